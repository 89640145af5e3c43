#!/bin/bash
# Round-end style check of the committed tree: build + smoke, every GPU test, the default bench line.
OUT=gpurun_out/${1:-check}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -30 $OUT/smoke.log; exit 1; }
tail -2 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_C3.json 2> $OUT/bench_C3.err
python -c "import json;d=json.load(open('$OUT/bench_C3.json'));print('C3', round(d['ms_per_step'],2), d['roofline']['frac'], d['parity']['ok'], round(d['e2e']['value']), round(d['cpu_baseline']['value'],1), d['clocks'])"

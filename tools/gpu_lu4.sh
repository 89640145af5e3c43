#!/bin/bash
# LU12 check: build, every LU GPU test, C3 / C2 LU bench lines (same box as the previous HEAD's
# numbers only through the committed profiles -- box-to-box noise is about 1%).
OUT=gpurun_out/${1:-lu12}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
for C in C3 C2; do
timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 > $OUT/bench_lu_$C.json 2> $OUT/bench_lu_$C.err; python -c "import json;d=json.load(open('$OUT/bench_lu_$C.json'));print('$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d.get('parity'))"; tail -2 $OUT/bench_lu_$C.err
done
python tools/lu_trace.py 4096,128,32 16384,256,32 > $OUT/lu_trace.txt 2>&1; head -20 $OUT/lu_trace.txt

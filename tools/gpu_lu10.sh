#!/bin/bash
# LU dispatch mode A/B on one box (TLU_DEV_DISP=0/1 against the plan's default), LU GPU tests, LU C3 line.
OUT=gpurun_out/${1:-lu10}; mkdir -p $OUT
for R in 1 2; do
for D in "" 0 1; do
  for C in C3 C2 C4; do
    env ${D:+TLU_DEV_DISP=$D} timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b_${C}_d${D:-def}.json 2> $OUT/b_${C}_d${D:-def}.err
    python -c "import json;d=json.load(open('$OUT/b_${C}_d${D:-def}.json'));print('disp=${D:-default}', '$C', round(d['ms_per_step'],2),'ms', round(d['roofline']['kernel_ms'],2))"
  done
done
done
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest_lu.log 2>&1; tail -2 $OUT/pytest_lu.log
TLU_DEV_DISP=1 timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest_lu_disp1.log 2>&1; tail -2 $OUT/pytest_lu_disp1.log
timeout 900 python bench.py --method lu --steps 5 --warmup 3 > $OUT/bench_lu_C3.json 2> $OUT/bench_lu_C3.err
python -c "import json;d=json.load(open('$OUT/bench_lu_C3.json'));print('LU C3', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d['parity']['ok'], round(d['e2e']['value']), d['clocks'])"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python tools/lu_trace.py > $OUT/lu_trace.txt 2>&1; tail -5 $OUT/lu_trace.txt

#!/bin/bash
# LU12 final: every LU GPU test, C3 / C2 LU bench lines (C3 with the bench's own parity), the
# traces, and one ncu --set full capture of the C3-matrix LU executor.
OUT=gpurun_out/${1:-lu14}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -20 $OUT/smoke.log; exit 1; }
tail -2 $OUT/smoke.log
timeout 1200 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for C in C3 C2; do
  timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 > $OUT/bench_lu_$C.json 2> $OUT/bench_lu_$C.err
  python -c "import json;d=json.load(open('$OUT/bench_lu_$C.json'));print('$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d.get('parity',{}).get('ok'))"
done
python tools/lu_trace.py 4096,128,32 16384,256,32 > $OUT/lu_trace.txt 2>&1; head -20 $OUT/lu_trace.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:lu_exec_kernel -s 1 -c 1 \
  -o $OUT/lu_exec_c3 python tools/lu_quick.py 16384,256,32 > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
python tools/ncu_summary.py full $OUT/lu_exec_c3.ncu-rep > $OUT/summary.txt 2>&1
python tools/ncu_lines.py $OUT/lu_exec_c3.ncu-rep --top 40 --file tlu_exec.cu >> $OUT/summary.txt 2>&1; head -30 $OUT/summary.txt

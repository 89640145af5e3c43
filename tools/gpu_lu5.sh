#!/bin/bash
# LU update variants on one box: the product build (LU_KU=2) with every LU GPU test, then the
# C3 / C2 LU bench lines of each prebuilt variant library (TQR_LIB).
OUT=gpurun_out/${1:-lu13}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for V in "" ku4 ku8 ""; do
  LIBV=paper_0707_3548_b200/libtqr${V:+_$V}.so
  for C in C3 C2; do
    TQR_LIB=$PWD/$LIBV timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_lu_${C}_${V:-base}.json 2> $OUT/bench_lu_${C}_${V:-base}.err
    python -c "import json;d=json.load(open('$OUT/bench_lu_${C}_${V:-base}.json'));print('${V:-base}', '$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d.get('parity',{}).get('ok'))"
  done
done
python tools/lu_trace.py 4096,128,32 16384,256,32 > $OUT/lu_trace.txt 2>&1; head -20 $OUT/lu_trace.txt

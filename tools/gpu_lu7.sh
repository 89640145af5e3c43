#!/bin/bash
# LU L2-prefetch distance A/B on one box (prebuilt variant libraries, TQR_LIB), C3 and C2 LU.
OUT=gpurun_out/${1:-lu15}; mkdir -p $OUT
for V in pf0 "" pf1 pf4 pf0 ""; do
  LIBV=paper_0707_3548_b200/libtqr${V:+_$V}.so
  for C in C3 C2; do
    TQR_LIB=$PWD/$LIBV timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/b_${C}_${V:-base}.json 2> $OUT/b_${C}_${V:-base}.err
    python -c "import json;d=json.load(open('$OUT/b_${C}_${V:-base}.json'));print('${V:-base}', '$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%')"
  done
done
timeout 600 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log

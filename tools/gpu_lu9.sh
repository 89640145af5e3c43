#!/bin/bash
# LU A/B on one box: product library vs prebuilt variants (TQR_LIB), C3 / C2 / C4 LU; LU GPU tests per variant.
OUT=gpurun_out/${1:-lu9}; shift; mkdir -p $OUT
for R in 1 2; do
for L in "" "$@"; do
  LIBV=paper_0707_3548_b200/libtqr${L:+_$L}.so
  for C in C3 C2 C4; do
    TQR_LIB=$PWD/$LIBV timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b_${C}_${L:-base}.json 2> $OUT/b_${C}_${L:-base}.err
    python -c "import json;d=json.load(open('$OUT/b_${C}_${L:-base}.json'));print('${L:-base}', '$C', round(d['ms_per_step'],2),'ms', round(d['roofline']['kernel_ms'],2))"
  done
done
done
for L in "$@"; do
  TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_$L.so timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest_$L.log 2>&1; echo $L; tail -2 $OUT/pytest_$L.log
done

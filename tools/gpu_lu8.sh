#!/bin/bash
# LU A/B on one box: product library vs the prebuilt variant $2 (TQR_LIB), C3 and C2 LU; LU GPU tests.
OUT=gpurun_out/${1:-lu17}; V=${2:-wi0}; mkdir -p $OUT
for L in "" $V "" $V; do
  LIBV=paper_0707_3548_b200/libtqr${L:+_$L}.so
  for C in C3 C2; do
    TQR_LIB=$PWD/$LIBV timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/b_${C}_${L:-base}.json 2> $OUT/b_${C}_${L:-base}.err
    python -c "import json;d=json.load(open('$OUT/b_${C}_${L:-base}.json'));print('${L:-base}', '$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', (d.get('parity') or {}).get('ok'))"
  done
done
timeout 600 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log

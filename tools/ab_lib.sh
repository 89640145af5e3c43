#!/bin/bash
# A/B of the product library against a variant build (bench C4/C2/C3).  Dev aid.
#   TQR_VARIANT=name TQR_VARIANT_DEFS="-D..." python paper_0707_3548_b200/build.py; gpurun -- 'bash tools/ab_lib.sh name'
OUT=gpurun_out/ab; mkdir -p $OUT
P=$PWD/paper_0707_3548_b200
for LIBN in libtqr.so libtqr_$1.so libtqr.so libtqr_$1.so; do
  for C in C4 C2 C3; do
    TQR_LIB=$P/$LIBN timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/$LIBN.$C.json 2>&1
    python -c "import json;d=json.load(open('$OUT/$LIBN.$C.json'));print('$LIBN $C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%')"
  done
done

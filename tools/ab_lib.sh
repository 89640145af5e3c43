#!/bin/bash
# A/B of the product library against a variant build (panel task timings, C4/C2/C3 bench).  Dev aid.
OUT=gpurun_out/pnw; mkdir -p $OUT
P=$PWD/paper_0707_3548_b200
for LIBN in libtqr.so libtqr_pnw4.so; do
  echo "== $LIBN"
  for RW in 256 128; do TQR_LIB=$P/$LIBN TQR_DEV_RW=$RW timeout 300 python tools/prof_tasks.py --b 256 --s 32 --n 4096 --reps 2 --kinds 0,1 2>&1 | sed "s/^/RW$RW /"; done
  TQR_LIB=$P/$LIBN timeout 300 python tools/prof_tasks.py --b 128 --s 32 --n 4096 --reps 2 --kinds 0,1 2>&1
  for C in C4 C2 C3; do
    TQR_LIB=$P/$LIBN timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/$LIBN.$C.json 2>&1
    python -c "import json;d=json.load(open('$OUT/$LIBN.$C.json'));print('$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%')"
  done
done
TQR_LIB=$P/libtqr_pnw4.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2

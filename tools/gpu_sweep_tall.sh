#!/bin/bash
# Tall-unit duration model (R30) sweep at C4 with 2b x b tiles, vs square tiles.
OUT=gpurun_out/${1:-swt}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { T=$1; shift; env "$@" timeout 600 python bench.py --config C4 --tiles $T --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('C4 $T $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
for r in 1 2; do
run 2bxb TQR_DEV_TALLF=3 TQR_DEV_TALLA=4.5
run 2bxb TQR_DEV_TALLF=4 TQR_DEV_TALLA=6
run 2bxb TQR_DEV_TALLF=6 TQR_DEV_TALLA=9
run 2bxb TQR_DEV_TALLF=2 TQR_DEV_TALLA=3 TQR_DEV_LAT=200000
run 2bxb TQR_DEV_TALLF=4 TQR_DEV_TALLA=3
run 2bxb TQR_DEV_TALLF=2 TQR_DEV_TALLA=6
done

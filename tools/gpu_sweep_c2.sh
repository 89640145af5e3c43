#!/bin/bash
OUT=gpurun_out/${1:-sw}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { C=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('$C $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
for r in 1 2; do
for L in 200000 400000 1000000 10000000; do run C2 TQR_DEV_LAT=$L; done
run C1 TQR_DEV_LAT=4000
run C1 TQR_DEV_LAT=200000
done

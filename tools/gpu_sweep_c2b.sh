#!/bin/bash
OUT=gpurun_out/${1:-sw}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { C=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('$C $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
for r in 1 2; do
run C2 X=1
run C2 TQR_DEV_SLICEDEP=1
run C2 TQR_DEV_PIPE=0
run C2 TQR_DEV_SPLIT=1
run C2 TQR_DEV_EARLY=0
run C2 TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.3
run C4 TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.3
run C4 TQR_DEV_SLICEDEP=1
done

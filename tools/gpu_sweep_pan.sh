#!/bin/bash
OUT=gpurun_out/${1:-swp}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { C=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('$C $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
for r in 1 2; do
run C4 X=1
run C4 TQR_DEV_PANF=1.5 TQR_DEV_PANA=1.5
run C4 TQR_DEV_PANF=2 TQR_DEV_PANA=2
run C4 TQR_DEV_PANF=3 TQR_DEV_PANA=3
run C4 TQR_DEV_PANF=2 TQR_DEV_PANA=1
run C2 TQR_DEV_PANF=2 TQR_DEV_PANA=2
run C3 TQR_DEV_PANF=2 TQR_DEV_PANA=2
done

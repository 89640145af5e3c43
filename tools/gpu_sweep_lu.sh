#!/bin/bash
OUT=gpurun_out/${1:-swlu}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { C=$1; shift; env "$@" timeout 600 python bench.py --method lu --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('LU $C $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
rq() { C=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('QR $C $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"; }
for r in 1 2; do
rq C2 X=1
for L in 4000 32000 200000 1000000; do run C2 TLU_DEV_LAT=$L; done
for L in 4000 32000 200000; do run C3 TLU_DEV_LAT=$L; done
done

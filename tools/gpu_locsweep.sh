#!/bin/bash
# Locality variants at C3 (time only): each line = env, step ms, kernel ms.
OUT=gpurun_out/${1:-locsweep}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() { env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('$*', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"; }
for r in 1 2; do
run TQR_DEV_GROUP=0
run TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.5
run TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.4
run TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.3
run TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.5 TQR_DEV_GROUP_J=3
run TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.55
done
for V in "TQR_DEV_GROUP=0" "TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.5" "TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.4"; do
  env $V timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
  grep -E "dram__bytes|gpu__time" $OUT/ncu.log | sed "s/^/$V /"
done
for C in C2 C4 C5; do for V in "TQR_DEV_GROUP=0" "TQR_DEV_GROUP=3 TQR_DEV_GROUP_TAIL=0.5"; do
  [ $C = C5 ] && ST="--steps 1 --warmup 1" || ST="--steps 5 --warmup 3"
  env $V timeout 900 python bench.py --config $C $ST --no-cpu-baseline --no-e2e > $OUT/b.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b.json'));print('$C $V', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"
done; done

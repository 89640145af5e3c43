#!/bin/bash
# Schedule/policy sweep: each argument is "CONFIG [VAR=VALUE ...]"; prints ms and % of peak per case.
#   gpurun -- 'bash tools/sweep.sh TAG "C4 TQR_DEV_PRIO=1" "C3"'
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_0707_3548_b200/build.py > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
n=0
for spec in "$@"; do
  set -- $spec; C=$1; shift
  n=$((n+1))
  env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/case$n.json 2> $OUT/case$n.err
  python -c "import json;d=json.load(open('$OUT/case$n.json'));print('$spec', '|', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%')" 2>&1 | tail -1
done

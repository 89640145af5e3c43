#!/bin/bash
# Schedule/policy sweep: each argument is "CONFIG [+e2e] [VAR=VALUE ...]"; prints ms, % of peak
# (and form-Q with +e2e) per case.
#   gpurun -- 'bash tools/sweep.sh TAG "C4 TQR_DEV_PRIO=1" "C3 +e2e"'
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_0707_3548_b200/build.py > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
n=0
for spec in "$@"; do
  set -- $spec; C=$1; shift
  E2E=--no-e2e
  if [ "$1" == "+e2e" ]; then E2E=""; shift; fi
  n=$((n+1))
  env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline $E2E > $OUT/case$n.json 2> $OUT/case$n.err
  python -c "
import json;d=json.load(open('$OUT/case$n.json'));q=d.get('form_q')
print('$spec', '|', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', ('| e2e %.0f GF/s'%d['e2e']['value']) if d.get('e2e') else '', ('| formQ %.1f ms %.1f%%'%(q['ms'],q['pct_of_fp64_peak'])) if q else '')" 2>&1 | tail -1
done

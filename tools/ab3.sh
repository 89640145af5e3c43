# Same-box A/B: "r01" runs the r01 tree (.r01/), other names run the current tree with an
# environment (e.g. TQR_LIB=... or a TQR_DEV_* knob).  Alternating rounds; medians.
#   bash tools/ab3.sh CONFIG ROUNDS name:ENV ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; C=$1; R=$2; shift; shift; out=gpurun_out/ab3_$C.txt; rm -f $out
one() {  # name dir envs
  (cd $2 && env $3 timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', d['roofline']['kernel_ms'], d['ms_per_step'])") >> $out
}
for r in $(seq 1 $R); do
  for v in "$@"; do
    name=${v%%:*}; envs=${v#*:}
    if [ "$name" = r01 ]; then one r01 .r01 "TQR_X=1"; else one $name . "$envs"; fi
  done
done
python - "$out" <<'PY'
import sys, statistics, collections
v = collections.defaultdict(list)
for line in open(sys.argv[1]):
    n, k, m = line.split(); v[n].append((float(k), float(m)))
for n, xs in v.items():
    ks = sorted(x[0] for x in xs); ms = sorted(x[1] for x in xs)
    print(f"{sys.argv[1]} {n:8s}: kernel median {statistics.median(ks):8.3f} (min {ks[0]:8.3f} max {ks[-1]:8.3f})  step median {statistics.median(ms):8.3f} n={len(ks)}")
PY

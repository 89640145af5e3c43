# Same-box A/B of the r01 tree (.r01/, built from commit 8b6d6ef) against the current tree.
#   bash tools/ab2.sh CONFIG ROUNDS [ENV=...]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/ab2_$1.txt; rm -f $out
C=$1; R=$2; shift; shift
for r in $(seq 1 $R); do
  (cd .r01 && env "$@" timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('r01', d['roofline']['kernel_ms'], d['ms_per_step'])") >> $out
  env "$@" timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('now', d['roofline']['kernel_ms'], d['ms_per_step'])" >> $out
done
python - "$out" <<'PY'
import sys, statistics, collections
v = collections.defaultdict(list)
for line in open(sys.argv[1]):
    n, k, m = line.split(); v[n].append((float(k), float(m)))
for n, xs in v.items():
    ks = sorted(x[0] for x in xs); ms = sorted(x[1] for x in xs)
    print(f"{sys.argv[1]} {n}: kernel median {statistics.median(ks):.3f} (min {ks[0]:.3f} max {ks[-1]:.3f})  step median {statistics.median(ms):.3f} n={len(ks)}")
PY

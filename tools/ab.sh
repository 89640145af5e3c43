# A/B timing of library variants / env knobs, alternating runs (median of R rounds).
#   bash tools/ab.sh CONFIG ROUNDS "name1:ENV=.. ENV2=.." "name2:TQR_LIB=...so" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
C=$1; R=$2; shift; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    name=${v%%:*}; envs=${v#*:}
    env $envs timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys;d=json.loads(sys.stdin.read());print('$name', d['roofline']['kernel_ms'], d['ms_per_step'])" >> gpurun_out/ab_$C.txt
  done
done
python - "$C" <<'PY'
import sys, statistics, collections
c = sys.argv[1]
v = collections.defaultdict(list)
for line in open(f"gpurun_out/ab_{c}.txt"):
    n, k, m = line.split()
    v[n].append((float(k), float(m)))
for n, xs in v.items():
    ks = sorted(x[0] for x in xs); ms = sorted(x[1] for x in xs)
    print(f"{c} {n}: kernel median {statistics.median(ks):.3f} ms (min {ks[0]:.3f}, max {ks[-1]:.3f})  step median {statistics.median(ms):.3f}  n={len(ks)}")
PY

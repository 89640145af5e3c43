cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 600 python bench.py --config C3 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_h_$name.json 2>&1
  env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -c 1 --csv \
     python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_h_$name.csv 2>/dev/null
  python - "$name" <<'PY'
import json, sys, csv, io
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_h_{n}.json").read().strip().splitlines()[-1])
txt = open(f"gpurun_out/ncu_h_{n}.csv").read()
rows = [r for r in csv.reader(io.StringIO(txt[txt.index('"ID"'):])) if len(r) > 10]
h = rows[0]; mi = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
m = {r[mi]: (r[vi], r[ui]) for r in rows[1:]}
print(n, "ms", round(d["ms_per_step"], 2), "kern", round(d["roofline"]["kernel_ms"], 2), "dram read", m.get("dram__bytes_read.sum"), "write", m.get("dram__bytes_write.sum"))
PY
}
run base
run group1 TQR_DEV_GROUP=1
run group2 TQR_DEV_GROUP=2
run group3 TQR_DEV_GROUP=3

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multipass.py -x -q 2>&1 | tail -1
run() {  # name, lib, env...
  name=$1; lib=$2; shift; shift
  env TQR_LIB=$PWD/paper_0707_3548_b200/$lib "$@" timeout 600 python bench.py --config C3 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_i_$name.json 2>&1
  env TQR_LIB=$PWD/paper_0707_3548_b200/$lib "$@" timeout 600 python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_i4_$name.json 2>&1
  env TQR_LIB=$PWD/paper_0707_3548_b200/$lib "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -c 1 --csv \
     python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_i_$name.csv 2>/dev/null
  python - "$name" <<'PY'
import json, sys, csv, io
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_i_{n}.json").read().strip().splitlines()[-1])
d4 = json.loads(open(f"gpurun_out/bench_i4_{n}.json").read().strip().splitlines()[-1])
txt = open(f"gpurun_out/ncu_i_{n}.csv").read()
rows = [r for r in csv.reader(io.StringIO(txt[txt.index('"ID"'):])) if len(r) > 10]
h = rows[0]; mi = h.index("Metric Name"); vi = h.index("Metric Value")
m = {r[mi]: float(r[vi]) for r in rows[1:]}
print(n, "C3 ms", round(d["ms_per_step"], 2), "kern", round(d["roofline"]["kernel_ms"], 2), "C4 ms", round(d4["ms_per_step"], 2),
      "dram GB read", round(m["dram__bytes_read.sum"] / 1e9, 1), "write", round(m["dram__bytes_write.sum"] / 1e9, 1))
PY
}
run hint libtqr.so
run nohint libtqr_nohint.so
run hint_group1 libtqr.so TQR_DEV_GROUP=1

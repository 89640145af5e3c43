set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --trace gpurun_out/trace_c4.json > gpurun_out/bench_f_C4.json 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --trace gpurun_out/trace_c2.json > gpurun_out/bench_f_C2.json 2>&1
python tools/trace_stats.py gpurun_out/trace_c4.json > gpurun_out/trace_c4.txt 2>&1
python tools/trace_stats.py gpurun_out/trace_c2.json > gpurun_out/trace_c2.txt 2>&1
rm -f gpurun_out/trace_c4.json gpurun_out/trace_c2.json

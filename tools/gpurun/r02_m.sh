cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --tiles 2bxb --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --trace /tmp/trt.json > /dev/null 2>&1; python tools/trace_stats.py /tmp/trt.json > gpurun_out/trace_c4_tall.txt 2>&1
cat gpurun_out/trace_c4_tall.txt

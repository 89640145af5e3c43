cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tall.py -x -q 2>&1 | tail -25
timeout 900 python bench.py --config C4 --tiles 2bxb --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tall_C4.json 2>&1; tail -c 600 gpurun_out/bench_tall_C4.json

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tall.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C4 --tiles 2bxb --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_tall3_C4.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_tall3_C4.json').read().strip().splitlines()[-1]);print('tall C4', d['ms_per_step'], d['pct_of_fp64_peak'])"

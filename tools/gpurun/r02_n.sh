cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tall.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C4 --tiles 2bxb --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_tall2_C4.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_tall2_C4.json').read().strip().splitlines()[-1]);print('tall C4', d['ms_per_step'], d['pct_of_fp64_peak'])"
timeout 600 python bench.py --config C4 --tiles 2bxb --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --trace /tmp/trt.json > /dev/null 2>&1; python tools/trace_stats.py /tmp/trt.json > gpurun_out/trace_c4_tall2.txt 2>&1; head -30 gpurun_out/trace_c4_tall2.txt
bash tools/ab3.sh C3 3 now:TQR_X=1 lat2:TQR_DEV_LAT=2000 lat8:TQR_DEV_LAT=8000 poll64:TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_poll64.so
bash tools/ab3.sh C2 3 next:TQR_X=1 nonext:TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_nonext.so
bash tools/ab3.sh C4 3 next:TQR_X=1 nonext:TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_nonext.so

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multipass.py tests/test_gpu_dist.py tests/test_gpu_checked.py -x -q 2>&1 | tail -2
for C in C2 C4 C3; do
 for PIPE in 1 0; do
  TQR_DEV_PIPE=$PIPE timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_j_${C}_$PIPE.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_j_${C}_$PIPE.json').read().strip().splitlines()[-1]);print('$C pipe=$PIPE', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],2))"
 done
done
TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_nofence.so timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_j_nofence.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_j_nofence.json').read().strip().splitlines()[-1]);print('C3 nofence', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],2))"

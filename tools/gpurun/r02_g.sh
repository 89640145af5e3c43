cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for RW in 128 256; do
  TQR_DEV_RW=$RW timeout 600 python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_g_rw$RW.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_g_rw$RW.json').read().strip().splitlines()[-1]);print('RW $RW', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],2))"
done
TQR_DEV_RW=256 TQR_DEV_PASSES=2 timeout 600 python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_g_rw256p2.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_g_rw256p2.json').read().strip().splitlines()[-1]);print('RW 256 p2', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],2))"

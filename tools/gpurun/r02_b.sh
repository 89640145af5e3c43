# panel profiling + multi-rank apply-Q tests + fp64 probe with a clock record
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pytest_rc=$?
# fp64 probe with nvidia-smi clocks sampled during it
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp64 tools/probe_fp64.cu
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/probe_smi.csv &
SMI=$!
/tmp/probe_fp64 > gpurun_out/probe_fp64.txt 2>&1
kill $SMI
# phase-profiled panel tasks (clock64 phase counters), b = 256 and 128
TQR_PHASES=1 python paper_0707_3548_b200/build.py > gpurun_out/build_ph.log 2>&1
for B in 256 128; do
  TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b $B --s 32 --kinds 0,1,8,9,3 > gpurun_out/prof_ph_b$B.txt 2>&1
  timeout 300 python tools/prof_tasks.py --b $B --s 32 --kinds 0,1,8,9,3 > gpurun_out/prof_b$B.txt 2>&1
done
# ncu full capture of one launch of TSQRT factor parts (kind 9) and whole TSQRT (kind 1), b = 256
for K in 9 1 8; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -c 1 -o gpurun_out/ncu_kind${K}_b256 -f \
  python tools/prof_tasks.py --b 256 --s 32 --kinds $K --reps 1 > gpurun_out/ncu_kind${K}.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -c 1 -o gpurun_out/ncu_kind9_b128 -f \
  python tools/prof_tasks.py --b 128 --s 32 --kinds 9 --reps 1 > gpurun_out/ncu_kind9b128.log 2>&1
echo done

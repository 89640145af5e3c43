# round-2 evidence: GPU tests, smoke, bench lines (C1-C4), reference arm, ncu launch list + full capture
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/fin/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/fin/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/fin/bench_C3.json 2> gpurun_out/fin/bench_C3.err; echo bench_rc=$?
for C in C1 C2 C4; do timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/fin/bench_$C.json 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/ref_C3.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/fin/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu1=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -s 2 -c 1 -o gpurun_out/fin/ncu_full_exec_c3 -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2=$?
for B in 256 128; do
  timeout 600 ncu --set full --clock-control none -k regex:exec_kernel -c 1 -o gpurun_out/fin/ncu_tsqrt_b$B -f python tools/prof_tasks.py --b $B --s 32 --n 8192 --kinds 1 --reps 1 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:exec_kernel -c 1 -o gpurun_out/fin/ncu_geqrt_b$B -f python tools/prof_tasks.py --b $B --s 32 --n 16384 --kinds 0 --reps 1 > /dev/null 2>&1
done
timeout 300 python tools/prof_tasks.py --b 256 --s 32 --n 8192 --kinds 0,1,8,9,2,3 --reps 3 > gpurun_out/fin/prof_b256.txt 2>&1
timeout 300 python tools/prof_tasks.py --b 128 --s 32 --n 8192 --kinds 0,1,8,9,2,3 --reps 3 > gpurun_out/fin/prof_b128.txt 2>&1
echo done

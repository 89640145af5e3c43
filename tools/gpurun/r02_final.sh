# round-2 evidence: GPU tests, smoke, bench lines (C1-C4), reference arm, ncu launch list + full
# captures (summarised on the box: only text comes back)
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fin; D=gpurun_out/fin; R=/tmp/ncurep; mkdir -p $R
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > $D/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 $D/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $D/bench_C3.json 2> $D/bench_C3.err; echo bench_rc=$?
for C in C1 C2 C4; do timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > $D/bench_$C.json 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $D/ref_C3.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $D/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu1=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -s 2 -c 1 -o $R/exec_c3 -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2=$?
python tools/ncu_summary.py full $R/exec_c3.ncu-rep > $D/ncu_full_exec_c3.txt 2>&1
python tools/ncu_lines.py $R/exec_c3.ncu-rep --top 40 >> $D/ncu_full_exec_c3.txt 2>&1
for B in 256 128; do
  timeout 600 ncu --set full --clock-control none -k regex:exec_kernel -c 1 -o $R/tsqrt_b$B -f python tools/prof_tasks.py --b $B --s 32 --n 8192 --kinds 1 --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py full $R/tsqrt_b$B.ncu-rep > $D/ncu_full_tsqrt_b$B.txt 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:exec_kernel -c 1 -o $R/geqrt_b$B -f python tools/prof_tasks.py --b $B --s 32 --n 16384 --kinds 0 --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py full $R/geqrt_b$B.ncu-rep > $D/ncu_full_geqrt_b$B.txt 2>&1
done
timeout 300 python tools/prof_tasks.py --b 256 --s 32 --n 8192 --kinds 0,1,8,9,2,3 --reps 3 > $D/prof_b256.txt 2>&1
timeout 300 python tools/prof_tasks.py --b 128 --s 32 --n 8192 --kinds 0,1,8,9,2,3 --reps 3 > $D/prof_b128.txt 2>&1
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --trace /tmp/tr4.json > /dev/null 2>&1; python tools/trace_stats.py /tmp/tr4.json > $D/trace_c4.txt 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --trace /tmp/tr2.json > /dev/null 2>&1; python tools/trace_stats.py /tmp/tr2.json > $D/trace_c2.txt 2>&1
timeout 900 python bench.py --config C3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --trace /tmp/tr3.json > /dev/null 2>&1; python tools/trace_stats.py /tmp/tr3.json > $D/trace_c3.txt 2>&1
du -sh gpurun_out
echo done

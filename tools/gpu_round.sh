#!/bin/bash
# One gpurun measurement pass: build, smoke, GPU parity tests, bench (C3 + trace), per-kind
# task timings, ncu launch list and one ncu --set full capture of the executor.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [TAG] [STAGES]'
# STAGES: comma list of build,test,bench,prof,ncu,ncufull (default: all)
TAG=${1:-r01}
STAGES=${2:-build,test,bench,prof,ncu,ncufull}
OUT=gpurun_out/$TAG
mkdir -p $OUT
has() { [[ ",$STAGES," == *",$1,"* ]]; }
{
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
  echo "nproc $(nproc)"; free -g | head -2
} > $OUT/box.txt 2>&1
if has build; then
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { cat $OUT/smoke.log; exit 1; }
fi
if has test; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
  tail -5 $OUT/pytest_gpu.log
fi
if has bench; then
  timeout 900 python bench.py --steps 5 --warmup 3 --trace $OUT/trace_c3.json > $OUT/bench_c3.json 2> $OUT/bench_c3.err
  cat $OUT/bench_c3.json
  python tools/trace_stats.py $OUT/trace_c3.json > $OUT/trace_c3.txt 2>&1
  cat $OUT/trace_c3.txt
fi
if has prof; then
  timeout 600 python tools/prof_tasks.py --b 256 --s 32 --n 4096 > $OUT/prof_tasks_b256.txt 2>&1
  cat $OUT/prof_tasks_b256.txt
fi
if has ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
  tail -3 $OUT/ncu_launches.log
fi
if has ncufull; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 \
    -o $OUT/exec_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
  tail -3 $OUT/ncu_full.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -c 1 \
    -o $OUT/ssrfb_batch python tools/prof_tasks.py --kinds 3 --reps 1 > $OUT/ncu_ssrfb.log 2>&1
  tail -3 $OUT/ncu_ssrfb.log
fi
echo done

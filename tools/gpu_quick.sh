#!/bin/bash
# Quick GPU iteration: build, GPU parity tests, per-kind phase timings, C3 + C2 bench with traces.
#   gpurun -- 'bash tools/gpu_quick.sh TAG [configs]'
TAG=${1:-q}; CONFIGS=${2:-C3 C2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_0707_3548_b200/build.py > /dev/null 2>&1 && TQR_PHASES=1 python paper_0707_3548_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for bs in "256 32 4096" "128 32 4096"; do set -- $bs
  TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b $1 --s $2 --n $3 --reps 2 --kinds 0,1 >> $OUT/phases.txt 2>&1
done
cat $OUT/phases.txt
for C in $CONFIGS; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --trace $OUT/trace_$C.json > $OUT/bench_$C.json 2>&1
  python -c "import json;d=json.load(open('$OUT/bench_$C.json'));print('$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%')" 2>&1 || tail -5 $OUT/bench_$C.json
  python tools/trace_stats.py $OUT/trace_$C.json; rm -f $OUT/trace_$C.json
done

#!/bin/bash
# Full measurement pass: every BASELINE config (bench lines), C3 trace stats, ncu launch list of
# the default bench and one ncu --set full capture of the C3 executor.
#   gpurun -- 'bash tools/gpu_all.sh TAG'
TAG=${1:-all}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_0707_3548_b200/build.py > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/box.txt; nproc >> $OUT/box.txt
for C in C1 C2 C4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$C.json 2> $OUT/bench_$C.err
done
timeout 900 python bench.py --steps 5 --warmup 3 --trace $OUT/trace_C3.json > $OUT/bench_C3.json 2> $OUT/bench_C3.err
python tools/trace_stats.py $OUT/trace_C3.json > $OUT/trace_C3.txt; rm -f $OUT/trace_C3.json
timeout 1500 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_C5.json 2> $OUT/bench_C5.err
for C in C1 C2 C3 C4 C5; do python -c "import json;d=json.load(open('$OUT/bench_$C.json'));print('$C', round(d['ms_per_step'],3),'ms', round(d['pct_of_fp64_peak'],1),'%', 'e2e', d['e2e'] and round(d['e2e']['value']))" 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 \
  -o $OUT/exec_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log

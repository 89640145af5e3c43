#!/bin/bash
# Round-end style evidence: build + smoke, every GPU test, the default bench line (cpu_baseline,
# e2e, parity), C2/C4/C5 lines, the ncu launch list of the default bench, one ncu --set full
# capture of the C3 executor.
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/box.txt; nproc >> $OUT/box.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -30 $OUT/smoke.log; exit 1; }
tail -3 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_C3.json 2> $OUT/bench_C3.err; python -c "import json;d=json.load(open('$OUT/bench_C3.json'));print('C3', round(d['ms_per_step'],2), d['roofline']['frac'], d['parity'], d['e2e']['value'], d['cpu_baseline']['value'])"
for C in C2 C4; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$C.json 2>&1; python -c "import json;d=json.load(open('$OUT/bench_$C.json'));print('$C', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],1))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.txt 2>&1; head -12 $OUT/launches.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 \
  -o $OUT/exec_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py full $OUT/exec_c3.ncu-rep > $OUT/exec_c3_summary.txt 2>&1; head -30 $OUT/exec_c3_summary.txt
timeout 1500 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/bench_C5.json 2>&1; python -c "import json;d=json.load(open('$OUT/bench_C5.json'));print('C5', round(d['ms_per_step'],1), round(d['pct_of_fp64_peak'],1))"

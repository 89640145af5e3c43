#!/bin/bash
# Round-end LU evidence on one box: LU bench lines at C4 (tall-skinny), C3, C2 with cpu_baseline,
# parity and e2e; the ncu launch list of the default LU bench command; QR C2 / C4 lines of the
# same build.
OUT=gpurun_out/${1:-wrap}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/box.txt; nproc >> $OUT/box.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for C in C4 C3 C2; do
  timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 > $OUT/bench_lu_$C.json 2> $OUT/bench_lu_$C.err
  python -c "import json;d=json.load(open('$OUT/bench_lu_$C.json'));print('LU $C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d['parity'], round(d['e2e']['value']), d['cpu_baseline']['value'], d['clocks'])" || tail -5 $OUT/bench_lu_$C.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/lu_launches.csv python bench.py --method lu --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_lu_launches.log 2>&1
python tools/ncu_summary.py launches $OUT/lu_launches.csv > $OUT/lu_launches.txt 2>&1; head -12 $OUT/lu_launches.txt
for C in C2 C4; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  python -c "import json;d=json.load(open('$OUT/bench_$C.json'));print('QR $C', round(d['ms_per_step'],3), round(d['pct_of_fp64_peak'],1), d['clocks'])"
done

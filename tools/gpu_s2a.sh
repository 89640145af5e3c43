OUT=gpurun_out/r02s2a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/box.txt; nproc >> $OUT/box.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -30 $OUT/smoke.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -5 $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench_C3.json 2> $OUT/bench_C3.err; cat $OUT/bench_C3.json
for C in C2 C4; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --trace $OUT/trace_$C.json > $OUT/bench_$C.json 2>&1; python tools/trace_stats.py $OUT/trace_$C.json > $OUT/trace_$C.txt 2>&1; rm -f $OUT/trace_$C.json; done
timeout 600 python bench.py --config C4 --tiles 2bxb --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --trace $OUT/trace_C4t.json > $OUT/bench_C4t.json 2>&1; python tools/trace_stats.py $OUT/trace_C4t.json > $OUT/trace_C4t.txt 2>&1; rm -f $OUT/trace_C4t.json
for C in C2 C4 C4t; do python -c "import json;d=json.load(open('$OUT/bench_$C.json'));print('$C', round(d['ms_per_step'],3),'ms', round(d['pct_of_fp64_peak'],1),'%')" 2>&1|tail -1; done

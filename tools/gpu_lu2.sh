OUT=gpurun_out/lu9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_parity.py -k "lu or locality" -x -q > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
timeout 300 python tools/lu_trace.py 4096,128,32 16384,256,32 > $OUT/lu_trace.txt 2>&1; cat $OUT/lu_trace.txt
for C in C2 C3; do timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 > $OUT/bench_lu_$C.json 2> $OUT/bench_lu_$C.err; python -c "import json;d=json.load(open('$OUT/bench_lu_$C.json'));print('$C', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d['parity'])"; done

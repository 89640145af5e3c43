OUT=gpurun_out/lu10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q -k c3 > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
timeout 900 python bench.py --method lu --config C3 --steps 5 --warmup 3 > $OUT/bench_lu_C3.json 2> $OUT/bench_lu_C3.err; python -c "import json;d=json.load(open('$OUT/bench_lu_C3.json'));print('C3', round(d['ms_per_step'],2),'ms', round(d['pct_of_fp64_peak'],1),'%', d['parity'])"; tail -3 $OUT/bench_lu_C3.err

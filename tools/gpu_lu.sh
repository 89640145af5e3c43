#!/bin/bash
# LU bring-up: build, LU GPU tests, quick timings, LU bench lines.
OUT=gpurun_out/${1:-lu}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > $OUT/pytest_lu.log 2>&1; tail -5 $OUT/pytest_lu.log
timeout 300 python tools/lu_quick.py 2048,128,32 4096,128,32 4096,256,32 8192,256,32 16384,256,32 > $OUT/lu_quick.txt 2>&1; cat $OUT/lu_quick.txt
for C in C2 C3; do timeout 900 python bench.py --method lu --config $C --steps 5 --warmup 3 > $OUT/bench_lu_$C.json 2> $OUT/bench_lu_$C.err; tail -c 1500 $OUT/bench_lu_$C.json; tail -3 $OUT/bench_lu_$C.err; done

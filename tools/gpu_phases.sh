OUT=gpurun_out/r01p
mkdir -p $OUT
python paper_0707_3548_b200/build.py > /dev/null 2>&1
./tools/gemm_core_bench > $OUT/gemm_core.txt 2>&1; cat $OUT/gemm_core.txt
for bs in "256 32 4096" "128 32 4096" "64 16 1024"; do set -- $bs
  TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b $1 --s $2 --n $3 --reps 2 >> $OUT/phases.txt 2>&1
done
cat $OUT/phases.txt
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --trace $OUT/trace_c2.json > $OUT/bench_c2.json 2>&1; cat $OUT/bench_c2.json
python tools/trace_stats.py $OUT/trace_c2.json
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --trace $OUT/trace_c4.json > $OUT/bench_c4.json 2>&1; cat $OUT/bench_c4.json
python tools/trace_stats.py $OUT/trace_c4.json
rm -f $OUT/trace_c4.json

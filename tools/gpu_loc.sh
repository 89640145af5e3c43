#!/bin/bash
# Locality-aware dispatch (TQR_FLAG_LOCALITY) vs the critical-path order at C3: same-box
# alternating bench runs + ncu DRAM bytes of one executor launch each.
OUT=gpurun_out/${1:-loc}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for r in 1 2; do for S in critical locality; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --schedule $S > $OUT/bench_${S}_$r.json 2>&1
  python -c "import json;d=json.load(open('$OUT/bench_${S}_$r.json'));print('$S', round(d['ms_per_step'],2),'ms', round(d['roofline']['kernel_ms'],2), 'kernel ms')"
done; done
for S in critical locality; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --schedule $S > $OUT/ncu_$S.log 2>&1
  grep -E "dram__bytes|gpu__time" $OUT/ncu_$S.log | sed "s/^/$S /"
done

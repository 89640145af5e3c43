#!/bin/bash
# Time + DRAM bytes of the executor per case: each argument "CONFIG [VAR=VALUE ...]".
#   gpurun -- 'bash tools/dram_sweep.sh TAG "C3 TQR_DEV_BLQ=0" ...'
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
python paper_0707_3548_b200/build.py > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
n=0
for spec in "$@"; do
  set -- $spec; C=$1; shift; n=$((n+1))
  env "$@" timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/case$n.json 2> $OUT/case$n.err
  env "$@" timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv \
    python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu$n.csv 2> $OUT/ncu$n.err
  python - "$spec" $OUT/case$n.json $OUT/ncu$n.csv <<'PY'
import json, sys, csv
d = json.load(open(sys.argv[2]))
gb = {}
for row in csv.reader(l for l in open(sys.argv[3]) if l.startswith('"')):
    if len(row) > 14 and row[-3].startswith("dram__"):
        v = float(row[-1].replace(",", ""))
        gb[row[-3]] = v * {"Gbyte": 1, "Mbyte": 1e-3, "Tbyte": 1e3, "byte": 1e-9, "Kbyte": 1e-6}.get(row[-2], 1)
print(sys.argv[1], "|", round(d["ms_per_step"], 2), "ms", round(d["pct_of_fp64_peak"], 1), "% | DRAM GB r/w",
      {k.split("__")[1].split(".")[0].replace("bytes_", ""): round(v, 1) for k, v in gb.items()})
PY
done

#!/bin/bash
# ncu --set full capture of the LU executor at 4096^2, b = 256 (after a plain run exits 0).
OUT=gpurun_out/${1:-luncu}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 300 python tools/lu_quick.py ${2:-4096},256,32 > $OUT/plain.txt 2>&1 || { cat $OUT/plain.txt; exit 1; }
cat $OUT/plain.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lu_exec_kernel -s 1 -c 1 \
  -o $OUT/lu_exec_${2:-4096} python tools/lu_quick.py ${2:-4096},256,32 > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
python tools/ncu_summary.py full $OUT/lu_exec_${2:-4096}.ncu-rep > $OUT/summary.txt 2>&1; cat $OUT/summary.txt
python tools/ncu_lines.py $OUT/lu_exec_${2:-4096}.ncu-rep --top 40 --file tlu_exec.cu > $OUT/lines.txt 2>&1; head -60 $OUT/lines.txt

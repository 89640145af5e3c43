set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for LIB in libtqr_noinl.so; do
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/$LIB timeout 300 python tools/prof_tasks.py --b 256 --s 32 --kinds 9 --reps 3 > gpurun_out/prof_$LIB.txt 2>&1
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/$LIB timeout 300 python tools/prof_tasks.py --b 256 --s 32 --m 32768 --n 2048 --kinds 9,3 --reps 3 >> gpurun_out/prof_$LIB.txt 2>&1
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/$LIB timeout 300 python tools/prof_tasks.py --b 128 --s 32 --kinds 9,3 --reps 3 >> gpurun_out/prof_$LIB.txt 2>&1
done

set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TQR_PHASES=1 python paper_0707_3548_b200/build.py > gpurun_out/build_ph.log 2>&1
TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 256 --s 32 --kinds 9,8,1 --reps 3 > gpurun_out/prof_ph2_b256.txt 2>&1
TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 256 --s 32 --m 32768 --n 2048 --kinds 9,1,3 --reps 3 > gpurun_out/prof_ph2_b256_tall.txt 2>&1
TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 128 --s 32 --kinds 9,8 --reps 3 > gpurun_out/prof_ph2_b128.txt 2>&1

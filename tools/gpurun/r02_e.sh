set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multipass.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest_e.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_e.log
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 256 --s 32 --kinds 9 --reps 3 > gpurun_out/prof_e.txt 2>&1
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 256 --s 32 --m 32768 --n 2048 --kinds 9 --reps 3 >> gpurun_out/prof_e.txt 2>&1
TQR_PH=1 TQR_LIB=$PWD/paper_0707_3548_b200/libtqr_phases.so timeout 300 python tools/prof_tasks.py --b 128 --s 32 --kinds 9 --reps 3 >> gpurun_out/prof_e.txt 2>&1
for C in C4 C2 C3; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_e_$C.json 2>&1; done
python - <<'PY'
import json
for c in ("C4","C2","C3"):
    try:
        d=json.loads(open(f"gpurun_out/bench_e_{c}.json").read().strip().splitlines()[-1])
        print(c, round(d["ms_per_step"],3), "ms", round(d["pct_of_fp64_peak"],2), "%", "kernel", round(d["roofline"]["kernel_ms"],3))
    except Exception as e: print(c, "fail", e)
PY

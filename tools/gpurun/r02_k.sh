cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multipass.py tests/test_gpu_dist.py tests/test_gpu_checked.py -x -q 2>&1 | tail -2
bash tools/ab3.sh C3 3 head:TQR_LIB=$PWD/.head/libtqr.so mix:TQR_X=1
bash tools/ab3.sh C4 3 head:TQR_LIB=$PWD/.head/libtqr.so mix:TQR_X=1 mix256:TQR_DEV_RW=256
bash tools/ab3.sh C2 3 head:TQR_LIB=$PWD/.head/libtqr.so mix:TQR_X=1

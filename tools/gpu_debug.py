"""Quick GPU parity probe (development aid): factor a few shapes and print errors vs the oracle."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import tqr_inputs  # noqa: E402
from gpu_util import run_factor  # noqa: E402

cases = [(64, 64, 64, 16), (128, 64, 64, 16), (256, 256, 64, 16), (67, 41, 16, 8), (520, 300, 128, 32),
         (700, 600, 256, 32)]
for (m, n, b, s) in cases:
    A = tqr_inputs.uniform(m, n, 1 + m)
    t0 = time.time()
    g = run_factor(A, b, s)
    t1 = time.time()
    At_o, T_o = oracle.geqrf(A, b, s, nthreads=4)
    R_o = oracle.get_r(At_o, m, n, b)
    nA = np.linalg.norm(A)
    print(f"{m}x{n} b={b} s={s}: R err {np.max(np.abs(g['R'] - R_o)) / nA:.2e}  "
          f"V err {np.max(np.abs(g['At'] - At_o)):.2e}  T err {np.max(np.abs(g['T'] - T_o)):.2e}  gpu {t1 - t0:.2f}s",
          flush=True)

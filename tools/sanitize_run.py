"""Small factorizations + apply-Q for compute-sanitizer (memcheck / racecheck / synccheck).
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tqr_inputs  # noqa: E402
from gpu_util import run_factor  # noqa: E402

for (m, n, b, s) in [(256, 256, 64, 16), (300, 200, 32, 8), (520, 300, 128, 32), (700, 600, 256, 32),
                     (1100, 700, 512, 64)]:
    A = tqr_inputs.uniform(m, n, 5 + m)
    g = run_factor(A, b, s)
    plan = g["plan"]
    Qt = torch.empty(plan.p * (-(-n // b)) * b * b, dtype=torch.float64, device="cuda")
    plan.orgqr(g["At_dev"], g["T_dev"], n, Qt)
    plan.sync()
    print(m, n, b, s, "ok", float(np.abs(g["R"]).max()))

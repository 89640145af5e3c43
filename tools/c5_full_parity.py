"""Full-oracle parity at C5 (65536^2, b = 512, s = 64): the GPU factorization of the C5 matrix
against the plain CPU oracle on the SAME seeded bytes, R elementwise within 1e-10 ||A||_F
(BJ north_star) and the T factors.  The oracle needs ~1.4e5 core-seconds (~85 min on 16
threads) and ~100 GiB of host memory, so this runs as a one-off evidence job, not in the test
suite (SURVEY 8(c) c-P: 'full-oracle parity at C5: pending' unless the box allows).

  python tools/c5_full_parity.py [--out gpurun_out/c5_full_parity.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: this is a parity check)
import tqr_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/c5_full_parity.json")
ap.add_argument("--config", default="C5")
a = ap.parse_args()
cfg = tqr_inputs.CONFIGS[a.config]
m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
threads = len(os.sched_getaffinity(0))
res = {"config": a.config, "m": m, "n": n, "b": b, "s": s, "threads": threads}
t0 = time.time()
A = tqr_inputs.make(m, n, cfg["dist"], cfg["seed"])
nA = float(np.linalg.norm(A))
res["gen_s"] = time.time() - t0

import torch  # noqa: E402
from paper_0707_3548_b200 import Plan  # noqa: E402
plan = Plan(m, n, b, s)
Ad = torch.from_numpy(A.T).cuda()
At, T = plan.alloc()
plan.pack(Ad, At)
del Ad
t1 = time.time()
plan.geqrf(At, T)
plan.sync()
res["gpu_s"] = time.time() - t1
R = torch.empty((n, min(m, n)), dtype=torch.float64, device="cuda")
plan.get_r(At, R)
plan.sync()
del At
R_gpu = R.cpu().numpy()          # (n, k): column-major storage of R
T_gpu = T.cpu().numpy()
del R, T
plan.close()
torch.cuda.empty_cache()

t2 = time.time()
At_o, T_o = oracle.geqrf(A, b, s, nthreads=threads)
res["oracle_s"] = time.time() - t2
res["oracle_gflops"] = oracle.flops_standard(m, n) / res["oracle_s"] / 1e9
del A
R_o = oracle.get_r(At_o, m, n, b)  # (k, n) Fortran
del At_o
err = 0.0
for c0 in range(0, n, 4096):        # column chunks: no full-size temporaries
    err = max(err, float(np.max(np.abs(R_gpu[c0:c0 + 4096, :].T - R_o[:, c0:c0 + 4096]))))
res["R_max_abs_diff"] = err
res["tol"] = 1e-10 * nA
res["T_max_abs_diff"] = float(np.max(np.abs(T_gpu - T_o)))
res["ok"] = err <= 1e-10 * nA and res["T_max_abs_diff"] <= 1e-9 * nA
print(json.dumps(res), flush=True)
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
sys.exit(0 if res["ok"] else 1)

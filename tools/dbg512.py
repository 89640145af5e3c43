import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, oracle, tqr_inputs
from gpu_util import run_factor
for (m, n) in [(1100, 1030), (1100, 600), (600, 1030), (1024, 512), (1024, 1024)]:
    A = tqr_inputs.uniform(m, n, 4242 + m + n)
    g = run_factor(A, 512, 64)
    At_o, T_o = oracle.geqrf(A, 512, 64, nthreads=8)
    R_o = oracle.get_r(At_o, m, n, 512)
    d = np.abs(np.triu(g["R"]) - np.triu(R_o))
    bad = np.argwhere(d > 1e-10 * np.linalg.norm(A))
    print(m, n, "Rerr", d.max(), "first bad (r,c)", bad[:3].tolist(), "Verr", np.abs(g["At"] - At_o).max(), "Terr", np.abs(g["T"] - T_o).max())

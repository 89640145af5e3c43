"""Checked build (compute-sanitizer is closed on this pool): libtqr_checked.so is compiled with
-DTQR_CHECKS, whose executor traps on any task record field, counter range or tile index out
of bounds.  Small factorizations (every built (b, s), ragged shapes), form-Q and emulated
multi-rank plans run through it in a subprocess and must finish cleanly and match the
product library bitwise."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np, torch
import tqr_inputs
from paper_0707_3548_b200 import Plan
from gpu_util import run_factor
out = {}
for (m, n, b, s) in [(256, 256, 64, 16), (67, 41, 16, 8), (41, 67, 16, 16), (300, 200, 32, 8), (96, 96, 32, 32),
                     (300, 200, 64, 64), (520, 300, 128, 32), (700, 600, 256, 32), (2048, 300, 256, 32),
                     (1100, 700, 512, 64)]:
    A = tqr_inputs.uniform(m, n, 5 + m)
    g = run_factor(A, b, s)
    plan = g["plan"]
    k = min(m, n)
    Qt = torch.empty(plan.p * (-(-k // b)) * b * b, dtype=torch.float64, device="cuda")
    plan.orgqr(g["At_dev"], g["T_dev"], k, Qt)
    plan.sync()
    out[(m, n, b, s)] = (g["At"].tobytes(), Qt.cpu().numpy().tobytes())
for (m, n, b, s, G) in [(520, 300, 128, 32, 3), (700, 600, 256, 32, 2)]:
    A = tqr_inputs.uniform(m, n, 9)
    plan = Plan(m, n, b, s, nranks=G, emulate=True)
    Ac = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(A).T)).cuda()
    At, T = plan.alloc()
    plan.pack(Ac, At); plan.geqrf(At, T); plan.sync()
import hashlib, pickle
print("DIGEST", hashlib.sha256(pickle.dumps(sorted(out.items()))).hexdigest())
'''


def _run(lib):
    env = dict(os.environ, TQR_LIB=lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("DIGEST")][0]


def test_checked_build_runs_clean_and_matches():
    env = dict(os.environ, TQR_VARIANT="checked", TQR_VARIANT_DEFS="-DTQR_CHECKS")
    subprocess.run([sys.executable, os.path.join(ROOT, "paper_0707_3548_b200", "build.py")], cwd=ROOT, env=env,
                   check=True, capture_output=True, timeout=900)
    checked = _run(os.path.join(ROOT, "paper_0707_3548_b200", "libtqr_checked.so"))
    product = _run(os.path.join(ROOT, "paper_0707_3548_b200", "libtqr.so"))
    assert checked == product

"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/tqr.h
declares, validates arguments, and its host-built DAG schedule matches Algorithm 1."""
import json
import os
import re
import subprocess

import pytest

import oracle
from conftest import GOLDEN, ROOT


@pytest.fixture(scope="module")
def L():
    from paper_0707_3548_b200.build import build
    build()
    from paper_0707_3548_b200 import tqr
    return tqr


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "tqr.h")).read()
    declared = sorted(set(re.findall(r"\b(tqr_[a-z_]+)\s*\(", hdr)))
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (tqr_[a-z_]+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert len(declared) >= 18


def test_flop_models_match_oracle_and_paper(L):
    for m, n in [(3000, 3000), (131072, 2048), (100, 300), (1, 1)]:
        assert L.flops_standard(m, n) == pytest.approx(oracle.flops_standard(m, n), rel=1e-15)
    # s == b reproduces the paper's Eq. 4 exact sum
    for p, q, b in [(20, 20, 1), (7, 3, 4), (4, 9, 8)]:
        assert L.flops_tiled(p * b, q * b, b, b) == pytest.approx(oracle.flops_eq4(p, q, b), rel=1e-12)
    # inner blocking lowers the executed count toward the standard one
    r = L.flops_tiled(16384, 16384, 256, 32) / L.flops_standard(16384, 16384)
    assert 1.02 < r < 1.04


def test_dag_node_counts_golden(L):
    for c in json.load(open(os.path.join(GOLDEN, "dag_counts.json")))["cases"]:
        counts, _ = L.schedule_inspect(c["p"], c["q"], 1, 4)
        assert sum(counts.values()) == c["nodes"], c["cite"]


@pytest.mark.parametrize("p,q,nsl,workers", [(1, 1, 1, 1), (2, 2, 1, 1), (3, 3, 1, 2), (5, 3, 2, 3), (3, 5, 4, 7),
                                              (12, 12, 1, 148), (64, 64, 4, 148), (512, 8, 4, 148)])
def test_schedule_is_topological_and_counts(L, p, q, nsl, workers):
    counts, nedges = L.schedule_inspect(p, q, nsl, workers)
    K = min(p, q)
    assert counts["G"] == K
    assert counts["T"] == sum(p - k - 1 for k in range(K))
    assert counts["L"] == nsl * sum(q - k - 1 for k in range(K))
    assert counts["S"] == nsl * sum((p - k - 1) * (q - k - 1) for k in range(K))
    assert nedges > 0 or p * q == 1


def test_invalid_args_without_gpu(L):
    import ctypes
    lib = L.lib()
    h = ctypes.c_void_p()
    for bad, idx in [(dict(m=0), 1), (dict(n=0), 2), (dict(b=0), 3), (dict(s=3), 4), (dict(s=0), 4),
                     (dict(nranks=0), 7), (dict(rank=1), 8)]:
        prm = dict(m=10, n=10, b=8, s=4, device=0, stream=None, nranks=1, rank=0, flags=0)
        prm.update(bad)
        P = L._Params(prm["m"], prm["n"], prm["b"], prm["s"], prm["device"], prm["stream"], prm["nranks"],
                      prm["rank"], prm["flags"])
        st = lib.tqr_plan_create(ctypes.byref(h), ctypes.byref(P))
        assert st == 1 and lib.tqr_last_bad_arg() == idx, (bad, st, lib.tqr_last_bad_arg())
    assert lib.tqr_status_string(0) == b"TQR_OK"
    assert L.supported(256, 32) and L.supported(128, 32) and L.supported(64, 16)
    assert not L.supported(48, 16)


def test_scaling_model_properties(L):
    """tqr_schedule_model (a MODEL of the multi-GPU schedule): splitting a
    grid over more GPUs never makes the modelled time longer than the 1-GPU time, efficiency
    T1 / (G TG) stays <= 1, remote-edge latency only adds time, and the modelled utilisation is
    a fraction."""
    m = n = 4096
    t1, busy1 = L.schedule_model(m, n, 128, 32, 1, 148, 0.0)
    assert 0.0 < busy1 <= 1.0 and t1 > 0.0
    for G in (2, 4):
        tg, busy = L.schedule_model(m, n, 128, 32, G, 148, 3000.0)
        assert tg <= t1 * 1.02 and t1 / (G * tg) <= 1.0 + 1e-9 and 0.0 < busy <= 1.0
        slow, _ = L.schedule_model(m, n, 128, 32, G, 148, 50000.0)
        assert slow >= tg
    # a big square grid scales: 2 GPUs model at least 1.6x faster than 1
    t1b, _ = L.schedule_model(8192, 8192, 128, 32, 1, 148, 3000.0)
    t2b, _ = L.schedule_model(8192, 8192, 128, 32, 2, 148, 3000.0)
    assert t1b / t2b > 1.6

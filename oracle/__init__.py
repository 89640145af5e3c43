"""ctypes loader for the plain-C CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this; the product package
(paper_0707_3548_b200) never does.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_i = ctypes.c_int
_pd = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "oracle.c")
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_LIB)
        L.oracle_house.argtypes = [_d, _pd, _i64, _pd, _pd, _pd]
        L.oracle_house.restype = None
        for name in ("oracle_geqrt",):
            getattr(L, name).argtypes = [_i, _i, _pd, _pd]
        L.oracle_tsqrt.argtypes = [_i, _i, _pd, _pd, _pd]
        L.oracle_larfb.argtypes = [_i, _i, _pd, _pd, _pd, _i]
        L.oracle_ssrfb.argtypes = [_i, _i, _pd, _pd, _pd, _pd, _i]
        L.oracle_pack.argtypes = [_i64, _i64, _i, _pd, _i64, _pd]
        L.oracle_unpack.argtypes = [_i64, _i64, _i, _pd, _pd, _i64]
        L.oracle_get_r.argtypes = [_i64, _i64, _i, _pd, _pd, _i64]
        L.oracle_geqrf_tiles.argtypes = [_i64, _i64, _i, _i, _pd, _pd, _i]
        L.oracle_ormqr_tiles.argtypes = [_i64, _i64, _i, _i, _pd, _pd, _i, _i64, _pd, _i]
        L.oracle_flops_standard.argtypes = [_i64, _i64]
        L.oracle_flops_standard.restype = _d
        L.oracle_kernel_flops.argtypes = [_i, _d]
        L.oracle_kernel_flops.restype = _d
        L.oracle_flops_eq4.argtypes = [_i64, _i64, _d]
        L.oracle_flops_eq4.restype = _d
        L.oracle_dag_edges.argtypes = [_i64, _i64, ctypes.POINTER(_i64), _i64]
        L.oracle_dag_edges.restype = _i64
        L.oracle_dag_edges_h.argtypes = [_i64, _i64, _i, ctypes.POINTER(_i64), _i64]
        L.oracle_dag_edges_h.restype = _i64
        L.oracle_tsqrt_rows.argtypes = [_i, _i, _i, _pd, _pd, _pd]
        L.oracle_ssrfb_rows.argtypes = [_i, _i, _i, _pd, _pd, _pd, _pd, _i]
        L.oracle_geqrf_tiles_h.argtypes = [_i64, _i64, _i, _i, _i, _pd, _pd, _i]
        L.oracle_ormqr_tiles_h.argtypes = [_i64, _i64, _i, _i, _i, _pd, _pd, _i, _i64, _pd, _i]
        L.oracle_flops_eq4_h.argtypes = [_i64, _i64, _d, _i]
        L.oracle_flops_eq4_h.restype = _d
        L.oracle_last_task_counts.argtypes = [ctypes.POINTER(_i64)]
        L.oracle_last_task_counts.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and (a.flags.f_contiguous or a.flags.c_contiguous)
    return a.ctypes.data_as(_pd)


def _chk(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"{what}: invalid argument {-rc}")


# ---- thin wrappers (numpy in / out; column-major tiles) -------------------------------

def house(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    beta, tau = _d(), _d()
    v = np.zeros(max(len(x) - 1, 1))
    rest = np.ascontiguousarray(x[1:]) if len(x) > 1 else np.zeros(1)
    lib().oracle_house(float(x[0]), _p(rest), len(x) - 1, ctypes.byref(beta), ctypes.byref(tau), _p(v))
    return beta.value, tau.value, np.concatenate([[1.0], v[:len(x) - 1]])


def tile(a):
    """numpy (b, b) -> column-major contiguous copy."""
    return np.asfortranarray(np.array(a, dtype=np.float64))


def geqrt(A, s):
    A = tile(A); b = A.shape[0]
    T = np.zeros((s, b), order="F")
    _chk(lib().oracle_geqrt(b, s, _p(A), _p(T)), "geqrt")
    return A, T


def tsqrt(R, B, s):
    R = tile(R); B = tile(B); b = R.shape[0]
    T = np.zeros((s, b), order="F")
    _chk(lib().oracle_tsqrt(b, s, _p(R), _p(B), _p(T)), "tsqrt")
    return R, B, T


def larfb(V, T, C, trans=1):
    V = tile(V); T = tile(T); C = tile(C); b = V.shape[0]; s = T.shape[0]
    _chk(lib().oracle_larfb(b, s, _p(V), _p(T), _p(C), trans), "larfb")
    return C


def tsqrt_rows(R, B, s):
    """TSQRT of [R (b x b upper); B (rows x b)] (R30: rows = h b, the 2b x b tiles)."""
    R = tile(R); B = np.asfortranarray(np.array(B, dtype=np.float64)); b = R.shape[0]
    T = np.zeros((s, b), order="F")
    _chk(lib().oracle_tsqrt_rows(b, s, B.shape[0], _p(R), _p(B), _p(T)), "tsqrt_rows")
    return R, B, T


def ssrfb_rows(V, T, C1, C2, trans=1):
    V = np.asfortranarray(np.array(V, dtype=np.float64)); T = tile(T); C1 = tile(C1)
    C2 = np.asfortranarray(np.array(C2, dtype=np.float64)); b = C1.shape[0]; s = T.shape[0]
    _chk(lib().oracle_ssrfb_rows(b, s, V.shape[0], _p(V), _p(T), _p(C1), _p(C2), trans), "ssrfb_rows")
    return C1, C2


def ssrfb(V, T, C1, C2, trans=1):
    V = tile(V); T = tile(T); C1 = tile(C1); C2 = tile(C2); b = V.shape[0]; s = T.shape[0]
    _chk(lib().oracle_ssrfb(b, s, _p(V), _p(T), _p(C1), _p(C2), trans), "ssrfb")
    return C1, C2


def dims(m, n, b):
    return -(-m // b), -(-n // b)


def pack(A, b):
    A = np.asfortranarray(A, dtype=np.float64); m, n = A.shape
    p, q = dims(m, n, b)
    At = np.zeros(p * q * b * b)
    _chk(lib().oracle_pack(m, n, b, _p(A), m, _p(At)), "pack")
    return At


def unpack(At, m, n, b):
    A = np.zeros((m, n), order="F")
    _chk(lib().oracle_unpack(m, n, b, _p(np.ascontiguousarray(At)), _p(A), m), "unpack")
    return A


def geqrf(A, b, s, nthreads=1, h=1):
    """Factor column-major A; returns (At tiles after factorization, T slots).  h > 1: the tile
    rows below the diagonal in units of h (the paper's 2b x b tiles for h = 2; R30)."""
    A = np.asfortranarray(A, dtype=np.float64); m, n = A.shape
    p, q = dims(m, n, b)
    At = pack(A, b)
    T = np.zeros(p * q * s * b)
    if h == 1:
        _chk(lib().oracle_geqrf_tiles(m, n, b, s, _p(At), _p(T), nthreads), "geqrf")
    else:
        _chk(lib().oracle_geqrf_tiles_h(m, n, b, s, h, _p(At), _p(T), nthreads), "geqrf_h")
    return At, T


def geqrf_tiles_inplace(m, n, b, s, At, T, nthreads=1):
    _chk(lib().oracle_geqrf_tiles(m, n, b, s, _p(At), _p(T), nthreads), "geqrf")


def get_r(At, m, n, b):
    k = min(m, n)
    R = np.zeros((k, n), order="F")
    _chk(lib().oracle_get_r(m, n, b, _p(np.ascontiguousarray(At)), _p(R), k), "get_r")
    return R


def ormqr(At, T, m, n, b, s, B, trans, nthreads=1, h=1):
    """Apply Q^T (trans=1) or Q (trans=0) to column-major m x nrhs B; returns new B."""
    B = np.asfortranarray(B, dtype=np.float64); nrhs = B.shape[1]
    Bt = pack(B, b)
    if h == 1:
        _chk(lib().oracle_ormqr_tiles(m, n, b, s, _p(np.ascontiguousarray(At)), _p(np.ascontiguousarray(T)),
                                      trans, nrhs, _p(Bt), nthreads), "ormqr")
    else:
        _chk(lib().oracle_ormqr_tiles_h(m, n, b, s, h, _p(np.ascontiguousarray(At)), _p(np.ascontiguousarray(T)),
                                        trans, nrhs, _p(Bt), nthreads), "ormqr_h")
    return unpack(Bt, m, nrhs, b)


def orgqr(At, T, m, n, b, s, k=None, nthreads=1, h=1):
    k = n if k is None else k
    E = np.zeros((m, k), order="F")
    E[np.arange(min(m, k)), np.arange(min(m, k))] = 1.0
    return ormqr(At, T, m, n, b, s, E, 0, nthreads, h)


def dag_edges(p, q, h=1):
    """Edges of the oracle's DAG: list of ((kind, k, i, j), (kind, k, i, j)), kind 'G','T','L','S'
    (T / S tasks of units of h tile rows report the unit's first tile row)."""
    n = lib().oracle_dag_edges_h(p, q, h, None, 0)
    buf = np.zeros(max(1, 8 * n), dtype=np.int64)
    lib().oracle_dag_edges_h(p, q, h, buf.ctypes.data_as(ctypes.POINTER(_i64)), n)
    names = "GTLS"
    e = buf[: 8 * n].reshape(n, 8)
    return [((names[r[0]], int(r[1]), int(r[2]), int(r[3])), (names[r[4]], int(r[5]), int(r[6]), int(r[7])))
            for r in e]


def task_counts():
    c = (_i64 * 4)()
    lib().oracle_last_task_counts(c)
    return dict(G=c[0], L=c[1], T=c[2], S=c[3])


def flops_standard(m, n):
    return lib().oracle_flops_standard(m, n)


def kernel_flops(kind, b):
    return lib().oracle_kernel_flops({"GEQT2": 0, "LARFB": 1, "TSQT2": 2, "SSRFB": 3}[kind], float(b))


def flops_eq4_h(p, q, b, h):
    return lib().oracle_flops_eq4_h(p, q, float(b), h)


def flops_eq4(p, q, b):
    return lib().oracle_flops_eq4(p, q, float(b))


# ---- tiled LU (oracle_lu.c, LU1-LU7) ----------------------------

_pi = ctypes.POINTER(ctypes.c_int32)


def _lu_lib():
    L = lib()
    if not getattr(L, "_lu_ready", False):
        L.oracle_lu_getrf.argtypes = [_i, _i, _pd, _pi]
        L.oracle_lu_gessm.argtypes = [_i, _i, _pd, _pi, _pd]
        L.oracle_lu_tstrf.argtypes = [_i, _i, _pd, _pd, _pd, _pi]
        L.oracle_lu_ssssm.argtypes = [_i, _i, _pd, _pd, _pi, _pd, _pd]
        L.oracle_lu_getrf_tiles.argtypes = [_i64, _i64, _i, _i, _pd, _pd, _pi, _i]
        L.oracle_lu_getrf_tiles_forced.argtypes = [_i64, _i64, _i, _i, _pd, _pd, _pi, _pi, _d, ctypes.POINTER(_i64),
                                                    ctypes.POINTER(_i64), _i]
        L.oracle_lu_apply.argtypes = [_i64, _i64, _i, _i, _pd, _pd, _pi, _i64, _pd, _i]
        L.oracle_lu_solve.argtypes = [_i64, _i, _i, _pd, _pd, _pi, _i64, _pd, _i]
        L.oracle_lu_flops_standard.argtypes = [_i64, _i64]
        L.oracle_lu_flops_standard.restype = _d
        L.oracle_lu_flops_tiled.argtypes = [_i64, _i64, _i, _i]
        L.oracle_lu_flops_tiled.restype = _d
        L._lu_ready = True
    return L


def _pp(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_pi)


def lu_getrf(A, s):
    """GETRF of one tile: returns (tile after, piv int32[b])."""
    A = tile(A); b = A.shape[0]
    piv = np.zeros(b, dtype=np.int32)
    _chk(_lu_lib().oracle_lu_getrf(b, s, _p(A), _pp(piv)), "lu_getrf")
    return A, piv


def lu_gessm(L, piv, C, s):
    L = tile(L); C = tile(C); b = C.shape[0]
    _chk(_lu_lib().oracle_lu_gessm(b, s, _p(L), _pp(np.ascontiguousarray(piv, dtype=np.int32)), _p(C)), "lu_gessm")
    return C


def lu_tstrf(U, A, s):
    """TSTRF of [U; A]: returns (U after, A after, Lt (s x b, column-major slot), piv int32[b])."""
    U = tile(U); A = tile(A); b = U.shape[0]
    Lt = np.zeros((s, b), order="F")
    piv = np.zeros(b, dtype=np.int32)
    _chk(_lu_lib().oracle_lu_tstrf(b, s, _p(U), _p(A), _p(Lt), _pp(piv)), "lu_tstrf")
    return U, A, Lt, piv


def lu_ssssm(V, Lt, piv, C1, C2, s):
    V = tile(V); Lt = np.asfortranarray(Lt, dtype=np.float64); C1 = tile(C1); C2 = tile(C2); b = C1.shape[0]
    _chk(_lu_lib().oracle_lu_ssssm(b, s, _p(V), _p(Lt), _pp(np.ascontiguousarray(piv, dtype=np.int32)), _p(C1),
                                   _p(C2)), "lu_ssssm")
    return C1, C2


def lu_getrf_tiles_inplace(m, n, b, s, At, Lt, piv, nthreads=1):
    _chk(_lu_lib().oracle_lu_getrf_tiles(m, n, b, s, _p(At), _p(Lt), _pp(piv), nthreads), "lu_getrf_tiles")


def lu_sizes(m, n, b, s):
    """(tile doubles, Lt doubles, piv ints) of the tiled LU storage (oracle_lu.h)."""
    p, q = dims(m, n, b)
    K = min(p, q)
    return p * q * b * b, p * K * s * b, p * K * b


def lu_getrf_tiles(A, b, s, nthreads=1):
    """Tiled LU of column-major A; returns (At tiles after, Lt slots, piv slots)."""
    A = np.asfortranarray(A, dtype=np.float64); m, n = A.shape
    _, nl, npv = lu_sizes(m, n, b, s)
    At = pack(A, b)
    Lt = np.zeros(nl)
    piv = np.zeros(npv, dtype=np.int32)
    lu_getrf_tiles_inplace(m, n, b, s, At, Lt, piv, nthreads)
    return At, Lt, piv


def lu_getrf_tiles_forced(A, b, s, forced, rel=1e-8, nthreads=1):
    """The oracle's tiled LU with every pivot forced to `forced` (LU10).  Returns
    (At, Lt, piv, nearties, invalid): decisions where the forced pivot differs from the search's
    and is within `rel` of the largest candidate / is not."""
    A = np.asfortranarray(A, dtype=np.float64); m, n = A.shape
    _, nl, npv = lu_sizes(m, n, b, s)
    At = pack(A, b)
    Lt = np.zeros(nl)
    piv = np.zeros(npv, dtype=np.int32)
    f = np.ascontiguousarray(forced, dtype=np.int32)
    nt, ni = _i64(), _i64()
    _chk(_lu_lib().oracle_lu_getrf_tiles_forced(m, n, b, s, _p(At), _p(Lt), _pp(piv), _pp(f), rel, ctypes.byref(nt),
                                                ctypes.byref(ni), nthreads), "lu_getrf_tiles_forced")
    return At, Lt, piv, nt.value, ni.value


def lu_apply(At, Lt, piv, m, n, b, s, B, nthreads=1):
    """B <- M B (every interchange and elimination of the factorization, in order); B m x nrhs."""
    B = np.asfortranarray(B, dtype=np.float64); nrhs = B.shape[1]
    qb = -(-nrhs // b)
    Bt = pack(B, b)
    _chk(_lu_lib().oracle_lu_apply(m, n, b, s, _p(np.ascontiguousarray(At)), _p(np.ascontiguousarray(Lt)),
                                   _pp(np.ascontiguousarray(piv)), qb, _p(Bt), nthreads), "lu_apply")
    return unpack(Bt, m, nrhs, b)


def lu_solve(At, Lt, piv, n, b, s, B, nthreads=1):
    """X = A^{-1} B for square A (n a multiple of b) from the tiled factors."""
    B = np.asfortranarray(B, dtype=np.float64); nrhs = B.shape[1]
    qb = -(-nrhs // b)
    Bt = pack(B, b)
    _chk(_lu_lib().oracle_lu_solve(n, b, s, _p(np.ascontiguousarray(At)), _p(np.ascontiguousarray(Lt)),
                                   _pp(np.ascontiguousarray(piv)), qb, _p(Bt), nthreads), "lu_solve")
    return unpack(Bt, n, nrhs, b)


def lu_flops_standard(m, n):
    return _lu_lib().oracle_lu_flops_standard(m, n)


def lu_flops_tiled(m, n, b, s):
    return _lu_lib().oracle_lu_flops_tiled(m, n, b, s)

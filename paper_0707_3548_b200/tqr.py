"""Thin ctypes binding over libtqr.so (include/tqr.h).  Argument marshalling only:
every step of the factorization runs in the library's CUDA kernels.  PyTorch supplies
device memory and the stream.  There is no fallback: a missing or failing library
raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TQR_LIB selects a profiling build (libtqr_phases.so); default is the product library.
LIB_PATH = os.environ.get("TQR_LIB") or os.path.join(HERE, "libtqr.so")

TQR_OK = 0
TQR_FLAG_TRACE = 1
TQR_FLAG_EMULATE_RANKS = 2
TQR_FLAG_TALL_TILES = 4
TQR_FLAG_LOCALITY = 8
TQR_IPC_BLOB_BYTES = 256
TASK_INTS = 16
_STATUS = {0: "TQR_OK", 1: "TQR_ERR_INVALID_ARG", 2: "TQR_ERR_CUDA", 3: "TQR_ERR_NCCL", 4: "TQR_ERR_OOM",
           5: "TQR_ERR_UNSUPPORTED"}


class TqrError(RuntimeError):
    def __init__(self, status: int, detail: str, bad_arg: int):
        self.status, self.detail, self.bad_arg = status, detail, bad_arg
        super().__init__(f"{_STATUS.get(status, status)}: {detail}" + (f" (argument {bad_arg})" if bad_arg else ""))


class _Params(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("b", ctypes.c_int32), ("s", ctypes.c_int32),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("nranks", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("flags", ctypes.c_uint32)]


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def lib():
    """Load libtqr.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_0707_3548_b200/build.py (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.tqr_plan_create.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(_Params)]
        L.tqr_plan_destroy.argtypes = [_vp]
        L.tqr_tiles_size.argtypes = [_vp, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
        L.tqr_workspace_size.argtypes = [_vp, ctypes.POINTER(ctypes.c_size_t)]
        L.tqr_pack.argtypes = [_vp, _vp, _i64, _vp]
        L.tqr_unpack.argtypes = [_vp, _vp, _vp, _i64]
        L.tqr_geqrf.argtypes = [_vp, _vp, _vp, _vp]
        L.tqr_get_r.argtypes = [_vp, _vp, _vp, _i64]
        L.tqr_ormqr.argtypes = [_vp, ctypes.c_char, _vp, _vp, _vp, _i64, _vp]
        L.tqr_orgqr.argtypes = [_vp, _vp, _vp, _i64, _vp, _vp]
        L.tqr_flops_standard.argtypes = [_i64, _i64]
        L.tqr_flops_standard.restype = ctypes.c_double
        L.tqr_flops_tiled.argtypes = [_i64, _i64, _i32, _i32]
        L.tqr_flops_tiled.restype = ctypes.c_double
        L.tqr_sync.argtypes = [_vp]
        L.tqr_status_string.argtypes = [ctypes.c_int]
        L.tqr_status_string.restype = ctypes.c_char_p
        L.tqr_last_error.restype = ctypes.c_char_p
        L.tqr_last_bad_arg.restype = _i32
        L.tqr_supported.argtypes = [_i32, _i32]
        L.tqr_supported.restype = _i32
        L.tqr_schedule_inspect.argtypes = [_i64, _i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
        L.tqr_trace_fetch.argtypes = [_vp, ctypes.POINTER(_i64), _i64, ctypes.POINTER(_i64)]
        L.tqr_profile_tasks.argtypes = [_vp, _i32, _i64, _vp, _vp, _vp]
        L.tqr_phase_counters.argtypes = [_vp, _vp]
        L.tqr_comm_export.argtypes = [_vp, _vp]
        L.tqr_comm_connect.argtypes = [_vp, _vp]
        L.tqr_comm_ping.argtypes = [_vp, _i32]
        L.tqr_comm_flags.argtypes = [_vp, _vp]
        L.tqr_schedule_records.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, _vp, _i64, ctypes.POINTER(_i64),
                                           ctypes.POINTER(_i32)]
        L.tqr_schedule_records_h.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i64,
                                             ctypes.POINTER(_i64), ctypes.POINTER(_i32)]
        L.tqr_schedule_records_policy.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint32, _vp,
                                                  _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i32), _vp]
        L.tqr_schedule_model.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, ctypes.c_double,
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.tqr_plan_records.argtypes = [_vp, _i32, _vp, _i64, ctypes.POINTER(_i64)]
        L.tqr_plan_info.argtypes = [_vp, ctypes.POINTER(_i32)]
        _lib = L
    return _lib


def _check(st: int):
    if st != TQR_OK:
        L = lib()
        raise TqrError(st, L.tqr_last_error().decode(), L.tqr_last_bad_arg())


def _ptr(t) -> int:
    if t is None:
        return 0
    if t.dtype.__repr__() != "torch.float64":
        raise TypeError("tqr works on float64 tensors")
    if not t.is_cuda:
        raise TypeError("tqr needs device (CUDA) tensors")
    if not t.is_contiguous():
        raise TypeError("tensor must be contiguous")
    return t.data_ptr()


# ---- pure functions (no GPU needed) ------------------------------------------------------

def flops_standard(m: int, n: int) -> float:
    return lib().tqr_flops_standard(m, n)


def flops_tiled(m: int, n: int, b: int, s: int) -> float:
    return lib().tqr_flops_tiled(m, n, b, s)


def supported(b: int, s: int) -> bool:
    return bool(lib().tqr_supported(b, s))


def schedule_inspect(p: int, q: int, nslice: int, workers: int):
    """Task counts {G,T,L,S} and edge count of the DAG; raises if the dispatch order is
    not topological."""
    c = (_i64 * 4)()
    ne = _i64()
    _check(lib().tqr_schedule_inspect(p, q, nslice, workers, c, ctypes.byref(ne)))
    return dict(G=c[0], T=c[1], L=c[2], S=c[3]), ne.value


def schedule_records(p: int, q: int, nslice: int, workers: int, nranks: int, rank: int, h: int = 1):
    """Dispatch records (numpy int32 (ntasks, 16)) of `rank` in the nranks-rank factorization
    schedule, and that rank's counter count (pure host; include/tqr.h); h: tile rows per
    TSQRT / SSRFB unit."""
    import numpy as np
    n, nc = _i64(), _i32()
    _check(lib().tqr_schedule_records_h(p, q, nslice, workers, nranks, rank, h, None, 0, ctypes.byref(n),
                                        ctypes.byref(nc)))
    rec = np.zeros((max(1, n.value), TASK_INTS), dtype=np.int32)
    _check(lib().tqr_schedule_records_h(p, q, nslice, workers, nranks, rank, h, rec.ctypes.data, n.value,
                                        ctypes.byref(n), ctypes.byref(nc)))
    return rec[: n.value], nc.value


def schedule_records_policy(m: int, n: int, b: int, s: int, nranks: int = 1, rank: int = 0, workers: int = 148,
                            tall: bool = False, locality: bool = False):
    """The records a plan for (m, n, b, s) would execute on `rank` (production policy; pure host;
    include/tqr.h tqr_schedule_records_policy): (records (ntasks, 16) int32, counter count,
    (panel blocks per tile, columns per register pass, passes per tile, tile rows per unit))."""
    import numpy as np
    n_, nc = _i64(), _i32()
    info = (ctypes.c_int32 * 4)()
    fl = (TQR_FLAG_TALL_TILES if tall else 0) | (TQR_FLAG_LOCALITY if locality else 0)
    _check(lib().tqr_schedule_records_policy(m, n, b, s, nranks, rank, workers, fl, None, 0, ctypes.byref(n_),
                                             ctypes.byref(nc), info))
    rec = np.zeros((max(1, n_.value), TASK_INTS), dtype=np.int32)
    _check(lib().tqr_schedule_records_policy(m, n, b, s, nranks, rank, workers, fl, rec.ctypes.data, n_.value,
                                             ctypes.byref(n_), ctypes.byref(nc), None))
    return rec[: n_.value], nc.value, tuple(info)


def schedule_model(m: int, n: int, b: int, s: int, nranks: int = 1, workers: int = 148, remote_ns: float = 0.0):
    """Modelled makespan (ms) and utilisation of the factorization schedule (a MODEL, pure host;
    include/tqr.h tqr_schedule_model)."""
    ms, busy = ctypes.c_double(), ctypes.c_double()
    _check(lib().tqr_schedule_model(m, n, b, s, nranks, workers, remote_ns, ctypes.byref(ms), ctypes.byref(busy)))
    return ms.value / 1e6, busy.value


# ---- plan ----------------------------------------------------------------------------------

class Plan:
    """One factorization shape (m, n, b, s) on one device and stream.

    Arrays are torch float64 CUDA tensors owned by the caller; tile-major arrays are flat
    (see tiles_size()).  All calls enqueue on the stream given at creation (default: the
    current torch stream).
    """

    def __init__(self, m: int, n: int, b: int, s: int, device: int = 0, stream=None, trace: bool = False,
                 nranks: int = 1, rank: int = 0, emulate: bool = False, tall: bool = False,
                 locality: bool = False):
        """nranks > 1: 1D block-cyclic multi-GPU plan for `rank` (connect it with
        paper_0707_3548_b200.dist.connect), or with emulate=True all nranks ranks in one
        launch on this device (tile arrays then keep the global layout).  tall=True: the paper's
        2b x b tiles (TQR_FLAG_TALL_TILES; b = 256, s = 32, one rank, factorization only).
        locality=True: the locality-aware dispatch order (TQR_FLAG_LOCALITY, R22)."""
        import torch
        self.m, self.n, self.b, self.s = m, n, b, s
        self.p, self.q = -(-m // b), -(-n // b)
        self.nranks, self.rank, self.emulate = nranks, rank, emulate
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        flags = (TQR_FLAG_TRACE if trace else 0) | (TQR_FLAG_EMULATE_RANKS if emulate else 0) | \
            (TQR_FLAG_TALL_TILES if tall else 0) | (TQR_FLAG_LOCALITY if locality else 0)
        prm = _Params(m, n, b, s, device, ctypes.c_void_p(stream.cuda_stream), nranks, rank, flags)
        h = _vp()
        _check(lib().tqr_plan_create(ctypes.byref(h), ctypes.byref(prm)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().tqr_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tiles_size(self):
        a, t = ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().tqr_tiles_size(self._h, ctypes.byref(a), ctypes.byref(t)))
        return a.value, t.value

    def workspace_size(self) -> int:
        w = ctypes.c_size_t()
        _check(lib().tqr_workspace_size(self._h, ctypes.byref(w)))
        return w.value

    def alloc(self):
        """Tile array At and T slots (caller-owned; the plan's workspace is allocated lazily)."""
        import torch
        a, t = self.tiles_size()
        dev = self.stream.device
        return torch.empty(a, dtype=torch.float64, device=dev), torch.empty(t, dtype=torch.float64, device=dev)

    def work(self):
        """The plan's device workspace (tqr_workspace_size bytes), allocated on first use."""
        import torch
        if getattr(self, "_work", None) is None:
            self._work = torch.empty(max(1, self.workspace_size()), dtype=torch.uint8, device=self.stream.device)
        return self._work

    def pack(self, A, At):
        """A: (n, m) row-major view of a column-major m x n matrix, i.e. A.T contiguous
        (use `A_colmajor = X.t().contiguous()` of an m x n tensor X) or any tensor whose
        storage is column-major with leading dimension lda = m."""
        _check(lib().tqr_pack(self._h, _ptr(A), self.m, _ptr(At)))

    def unpack(self, At, A):
        _check(lib().tqr_unpack(self._h, _ptr(At), _ptr(A), self.m))

    def geqrf(self, At, T, work=None):
        w = self.work() if work is None else work
        _check(lib().tqr_geqrf(self._h, _ptr(At), _ptr(T), w.data_ptr()))

    def comm_export(self) -> bytes:
        """This rank's CUDA IPC blob (TQR_IPC_BLOB_BYTES) for tqr_comm_connect."""
        buf = ctypes.create_string_buffer(TQR_IPC_BLOB_BYTES)
        _check(lib().tqr_comm_export(self._h, buf))
        return buf.raw

    def comm_ping(self, magic: int):
        """Store magic + rank into every rank's ping slot (peer-store connectivity check)."""
        _check(lib().tqr_comm_ping(self._h, magic))

    def comm_flags(self):
        """This rank's ping slots (after a host barrier following every rank's comm_ping)."""
        out = (_i32 * self.nranks)()
        _check(lib().tqr_comm_flags(self._h, out))
        return list(out)

    def comm_connect(self, blobs: bytes):
        """blobs: every rank's comm_export() blob, concatenated in rank order."""
        if len(blobs) != self.nranks * TQR_IPC_BLOB_BYTES:
            raise ValueError("need nranks * TQR_IPC_BLOB_BYTES bytes")
        _check(lib().tqr_comm_connect(self._h, blobs))

    def get_r(self, At, R):
        _check(lib().tqr_get_r(self._h, _ptr(At), _ptr(R), min(self.m, self.n)))

    def ormqr(self, trans: str, At, T, Bt, nrhs: int, work=None):
        w = self.work() if work is None else work
        _check(lib().tqr_ormqr(self._h, trans.encode(), _ptr(At), _ptr(T), _ptr(Bt), nrhs, w.data_ptr()))

    def orgqr(self, At, T, k: int, Qt, work=None):
        w = self.work() if work is None else work
        _check(lib().tqr_orgqr(self._h, _ptr(At), _ptr(T), k, _ptr(Qt), w.data_ptr()))

    def sync(self):
        _check(lib().tqr_sync(self._h))

    def profile_tasks(self, kind: int, count: int, At, T):
        """Run `count` independent tasks of one kind (0 G, 1 T, 2 L, 3 S); timing only."""
        _check(lib().tqr_profile_tasks(self._h, kind, count, _ptr(At), _ptr(T), self.work().data_ptr()))

    def phase_counters(self, d_counters):
        """Attach an int64 CUDA tensor of 16 phase-cycle totals (profiling builds only)."""
        _check(lib().tqr_phase_counters(self._h, None if d_counters is None else d_counters.data_ptr()))

    def records(self, local: int = 0):
        """The factorization dispatch records this plan executes (numpy int32 (ntasks, 16))."""
        import numpy as np
        n = _i64()
        _check(lib().tqr_plan_records(self._h, local, None, 0, ctypes.byref(n)))
        rec = np.zeros((max(1, n.value), TASK_INTS), dtype=np.int32)
        _check(lib().tqr_plan_records(self._h, local, rec.ctypes.data, n.value, ctypes.byref(n)))
        return rec[: n.value]

    def info(self) -> dict:
        """The plan's policy (include/tqr.h tqr_plan_info)."""
        v = (_i32 * 16)()
        _check(lib().tqr_plan_info(self._h, v))
        keys = ("rwm", "passes", "nsl", "split", "early", "workers", "prio", "fine", "inner", "nranks", "nloc",
                "slice", "h")
        return dict(zip(keys, list(v)))

    def trace(self, cap: int = 1 << 22):
        import numpy as np
        rec = np.zeros((cap, 8), dtype=np.int64)
        n = _i64()
        _check(lib().tqr_trace_fetch(self._h, rec.ctypes.data_as(ctypes.POINTER(_i64)), cap, ctypes.byref(n)))
        return rec[: n.value]


# ---- convenience (column-major torch <-> tiles) ---------------------------------------------

def colmajor(X):
    """m x n tensor -> its column-major storage as a contiguous (n, m) tensor."""
    return X.t().contiguous()


def from_colmajor(Xc):
    """(n, m) contiguous column-major storage -> m x n tensor view."""
    return Xc.t()

"""Thin ctypes binding over the tiled-LU entry points of libtqr.so (include/tlu.h; PAPER.md:850-860,
DESIGN.md LU1-LU9).  Argument marshalling only: every step runs in the library's CUDA kernels;
there is no fallback (a missing library raises).
"""
from __future__ import annotations

import ctypes

from .tqr import TqrError, _check, _ptr, lib as _tqr_lib

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_sz = ctypes.c_size_t
TASK_INTS = 16


class _Params(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("b", ctypes.c_int32), ("s", ctypes.c_int32),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint32)]


_ready = False


def lib():
    global _ready
    L = _tqr_lib()
    if not _ready:
        L.tlu_plan_create.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(_Params)]
        L.tlu_plan_destroy.argtypes = [_vp]
        L.tlu_sizes.argtypes = [_vp, ctypes.POINTER(_sz), ctypes.POINTER(_sz), ctypes.POINTER(_sz)]
        L.tlu_workspace_size.argtypes = [_vp, ctypes.POINTER(_sz)]
        L.tlu_pack.argtypes = [_vp, _vp, _i64, _vp]
        L.tlu_unpack.argtypes = [_vp, _vp, _vp, _i64]
        L.tlu_getrf.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.tlu_get_u.argtypes = [_vp, _vp, _vp, _i64]
        L.tlu_sync.argtypes = [_vp]
        L.tlu_plan_records.argtypes = [_vp, _vp, _i64, ctypes.POINTER(_i64)]
        L.tlu_trace_fetch.argtypes = [_vp, ctypes.POINTER(_i64), _i64, ctypes.POINTER(_i64)]
        L.tlu_schedule_records.argtypes = [_i64, _i64, _i32, _i32, _i32, _vp, _i64, ctypes.POINTER(_i64),
                                           ctypes.POINTER(_i32)]
        L.tlu_supported.argtypes = [_i32, _i32]
        L.tlu_supported.restype = _i32
        L.tlu_flops_standard.argtypes = [_i64, _i64]
        L.tlu_flops_standard.restype = ctypes.c_double
        L.tlu_flops_tiled.argtypes = [_i64, _i64, _i32, _i32]
        L.tlu_flops_tiled.restype = ctypes.c_double
        _ready = True
    return L


def supported(b: int, s: int) -> bool:
    return bool(lib().tlu_supported(b, s))


def flops_standard(m: int, n: int) -> float:
    return lib().tlu_flops_standard(m, n)


def flops_tiled(m: int, n: int, b: int, s: int) -> float:
    return lib().tlu_flops_tiled(m, n, b, s)


def schedule_records(m: int, n: int, b: int, s: int, workers: int = 148):
    """(records (ntasks, 16) int32, counter count) of a plan's dispatch order (pure host)."""
    import numpy as np
    nt, nc = _i64(), _i32()
    _check(lib().tlu_schedule_records(m, n, b, s, workers, None, 0, ctypes.byref(nt), ctypes.byref(nc)))
    rec = np.zeros((max(1, nt.value), TASK_INTS), dtype=np.int32)
    _check(lib().tlu_schedule_records(m, n, b, s, workers, rec.ctypes.data, nt.value, ctypes.byref(nt),
                                      ctypes.byref(nc)))
    return rec[: nt.value], nc.value


def _iptr(t) -> int:
    import torch
    if t.dtype != torch.int32 or not t.is_cuda:
        raise TypeError("piv must be an int32 CUDA tensor")
    return t.data_ptr()


class LUPlan:
    """One tiled-LU shape (m, n, b, s) on one device and stream (include/tlu.h)."""

    def __init__(self, m: int, n: int, b: int, s: int, device: int = 0, stream=None, trace: bool = False):
        import torch
        self.m, self.n, self.b, self.s = m, n, b, s
        self.p, self.q = -(-m // b), -(-n // b)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        prm = _Params(m, n, b, s, device, ctypes.c_void_p(stream.cuda_stream), 1 if trace else 0)
        h = _vp()
        _check(lib().tlu_plan_create(ctypes.byref(h), ctypes.byref(prm)))
        self._h = h
        self._work = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().tlu_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def sizes(self):
        a, w, pv = _sz(), _sz(), _sz()
        _check(lib().tlu_sizes(self._h, ctypes.byref(a), ctypes.byref(w), ctypes.byref(pv)))
        return a.value, w.value, pv.value

    def alloc(self):
        """(At tiles, W slots, piv) caller-owned device arrays."""
        import torch
        a, w, pv = self.sizes()
        dev = self.stream.device
        return (torch.empty(a, dtype=torch.float64, device=dev), torch.zeros(w, dtype=torch.float64, device=dev),
                torch.zeros(pv, dtype=torch.int32, device=dev))

    def work(self):
        import torch
        if self._work is None:
            nb = _sz()
            _check(lib().tlu_workspace_size(self._h, ctypes.byref(nb)))
            self._work = torch.empty(max(16, nb.value), dtype=torch.uint8, device=self.stream.device)
        return self._work

    def pack(self, A, At):
        """A: column-major m x n storage (e.g. X.t().contiguous() of an m x n tensor X)."""
        _check(lib().tlu_pack(self._h, _ptr(A), self.m, _ptr(At)))

    def unpack(self, At, A):
        _check(lib().tlu_unpack(self._h, _ptr(At), _ptr(A), self.m))

    def getrf(self, At, W, piv, work=None):
        w = self.work() if work is None else work
        _check(lib().tlu_getrf(self._h, _ptr(At), _ptr(W), _iptr(piv), w.data_ptr()))

    def get_u(self, At, U):
        """U: column-major min(m,n) x n (an (n, min(m,n)) tensor)."""
        _check(lib().tlu_get_u(self._h, _ptr(At), _ptr(U), min(self.m, self.n)))

    def sync(self):
        _check(lib().tlu_sync(self._h))

    def records(self):
        import numpy as np
        n = _i64()
        _check(lib().tlu_plan_records(self._h, None, 0, ctypes.byref(n)))
        rec = np.zeros((max(1, n.value), TASK_INTS), dtype=np.int32)
        _check(lib().tlu_plan_records(self._h, rec.ctypes.data, n.value, ctypes.byref(n)))
        return rec[: n.value]

    def trace(self):
        """(kind, k, i, j, sm, grab_ns, start_ns, end_ns) per task of the last getrf (trace=True)."""
        import numpy as np
        n = _i64()
        _check(lib().tlu_trace_fetch(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(1, n.value), 8), dtype=np.int64)
        _check(lib().tlu_trace_fetch(self._h, out.ctypes.data_as(ctypes.POINTER(_i64)), n.value, ctypes.byref(n)))
        return out[: n.value]


__all__ = ["LUPlan", "TqrError", "flops_standard", "flops_tiled", "lib", "schedule_records", "supported"]

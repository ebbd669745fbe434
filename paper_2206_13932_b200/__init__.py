"""Thin Python binding of the DMS front-end C ABI (include/dms.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
``csrc/`` (built in-tree as ``libdms.so``).  PyTorch supplies device memory and the
stream.  There is no CPU fallback: if the library is missing or no CUDA device is
present the calls raise.

Functions keep the ABI's names (``dms_create``, ``dms_order``, ``dms_gradient``,
``dms_critical``, ``dms_diagram0``, ``dms_diagram_top``, ``dms_unpaired_saddles``,
``dms_run_all``, ``dms_destroy``); ``DMS`` wraps them as a class.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DMS_LIB") or os.path.join(_HERE, "libdms.so")  # DMS_LIB: A/B experiments

PAIR_DTYPE = np.dtype(
    [
        ("birth_id", "<i8"),
        ("death_id", "<i8"),
        ("birth_vertex", "<i4"),
        ("death_vertex", "<i4"),
        ("birth_value", "<f4"),
        ("death_value", "<f4"),
    ]
)

STATUS = {
    0: "DMS_OK",
    1: "DMS_ERR_ARG",
    2: "DMS_ERR_DEGENERATE",
    3: "DMS_ERR_NAN",
    4: "DMS_ERR_TOO_LARGE",
    5: "DMS_ERR_STATE",
    6: "DMS_ERR_CUDA",
    7: "DMS_ERR_OOM",
    8: "DMS_ERR_INVARIANT",
}

# every symbol include/dms.h declares
ABI_SYMBOLS = [
    "dms_create",
    "dms_create2",
    "dms_order",
    "dms_gradient_bytes",
    "dms_gradient",
    "dms_critical",
    "dms_diagram0",
    "dms_diagram_top",
    "dms_unpaired_saddles",
    "dms_diagram1",
    "dms_generators",
    "dms_run_all",
    "dms_run_all_host",
    "dms_sync",
    "dms_decode_pairs",
    "dms_decode_pairs2",
    "dms_copy",
    "dms_set_timing",
    "dms_stage_ms",
    "dms_launch_count",
    "dms_last_error",
    "dms_destroy",
]


class DMSError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__("%s%s" % (STATUS.get(code, str(code)), (": " + msg) if msg else ""))
        self.code = code
        self.name = STATUS.get(code, str(code))


_lib = None


def lib():
    """Load libdms.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libdms.so not built: run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(LIB_PATH)
    p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P = ctypes.POINTER
    L.dms_create.argtypes = [p, i32, p, p, P(p)]
    L.dms_create2.argtypes = [p, i32, p, p, i32, P(p)]
    L.dms_order.argtypes = [p, p]
    L.dms_gradient_bytes.argtypes = [p]
    L.dms_gradient_bytes.restype = ctypes.c_size_t
    L.dms_gradient.argtypes = [p, p]
    L.dms_critical.argtypes = [p, p, p]
    L.dms_diagram0.argtypes = [p, P(p), P(i64)]
    L.dms_diagram_top.argtypes = [p, i32, P(p), P(i64)]
    L.dms_unpaired_saddles.argtypes = [p, i32, P(p), P(i64)]
    L.dms_diagram1.argtypes = [p, P(p), P(i64)]
    L.dms_generators.argtypes = [p, P(p), P(p), P(i64)]
    L.dms_run_all.argtypes = [p, p, p]
    L.dms_run_all_host.argtypes = [p, p, p, p]
    L.dms_sync.argtypes = [p]
    L.dms_decode_pairs.argtypes = [p, i32, p, i64, i64, p, i64]
    L.dms_decode_pairs.restype = i64
    L.dms_decode_pairs2.argtypes = [p, i32, i32, p, i64, i64, p, i64]
    L.dms_decode_pairs2.restype = i64
    L.dms_copy.argtypes = [p, p, p, ctypes.c_size_t]
    L.dms_set_timing.argtypes = [p, i32]
    L.dms_stage_ms.argtypes = [p, p]
    L.dms_launch_count.argtypes = [p]
    L.dms_launch_count.restype = i64
    L.dms_last_error.argtypes = [p]
    L.dms_last_error.restype = ctypes.c_char_p
    L.dms_destroy.argtypes = [p]
    L.dms_destroy.restype = None
    for name in ("dms_create", "dms_create2", "dms_order", "dms_gradient", "dms_critical", "dms_diagram0", "dms_diagram_top",
                 "dms_unpaired_saddles", "dms_diagram1", "dms_generators", "dms_run_all", "dms_run_all_host", "dms_sync", "dms_copy", "dms_set_timing",
                 "dms_stage_ms"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(ctx, st):
    if st != 0:
        msg = ""
        if ctx:
            m = lib().dms_last_error(ctx)
            msg = m.decode() if m else ""
        raise DMSError(st, msg)


def _dims_of(shape):
    """torch/numpy shape [Lz, Ly, Lx] (x fastest) -> (int64[3] x-first, ndim)."""
    ndim = len(shape)
    d = (ctypes.c_int64 * 3)(1, 1, 1)
    for i, n in enumerate(reversed(list(shape))):
        d[i] = int(n)
    return d, ndim


# ---------------------------------------------------------------- ABI-named functions

COMPLEXES = {"freudenthal": 0, "5tet": 1}  # dms_complex


def dms_create(f, stream=None, complex="freudenthal"):
    """f: contiguous float32 CUDA tensor of shape [Lz,Ly,Lx] / [Ly,Lx] / [Lx].
    complex: "freudenthal" (DMS_COMPLEX_FREUDENTHAL) or "5tet" (DMS_COMPLEX_5TET, 3D)."""
    import torch

    if not (isinstance(f, torch.Tensor) and f.is_cuda and f.dtype == torch.float32 and f.is_contiguous()):
        raise TypeError("dms_create: f must be a contiguous float32 CUDA tensor")
    if stream is None:
        stream = torch.cuda.current_stream(f.device)
    dims, ndim = _dims_of(f.shape)
    h = ctypes.c_void_p()
    _check(None, lib().dms_create2(dims, ndim, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                                   COMPLEXES[complex], ctypes.byref(h)))
    return h


def dms_order(ctx, rank):
    _check(ctx, lib().dms_order(ctx, ctypes.c_void_p(rank.data_ptr())))


def dms_gradient_bytes(ctx):
    return int(lib().dms_gradient_bytes(ctx))


def dms_gradient(ctx, grad):
    _check(ctx, lib().dms_gradient(ctx, ctypes.c_void_p(grad.data_ptr())))


def dms_critical(ctx):
    """-> (counts[4], device pointers[4])"""
    cnt = (ctypes.c_int64 * 4)()
    ptr = (ctypes.c_void_p * 4)()
    _check(ctx, lib().dms_critical(ctx, cnt, ptr))
    return [int(x) for x in cnt], [ptr[k] for k in range(4)]


def dms_diagram0(ctx):
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, lib().dms_diagram0(ctx, ctypes.byref(p), ctypes.byref(n)))
    return p.value, int(n.value)


def dms_diagram_top(ctx, mode=0):
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, lib().dms_diagram_top(ctx, int(mode), ctypes.byref(p), ctypes.byref(n)))
    return p.value, int(n.value)


def dms_unpaired_saddles(ctx, which):
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, lib().dms_unpaired_saddles(ctx, int(which), ctypes.byref(p), ctypes.byref(n)))
    return p.value, int(n.value)


def dms_diagram1(ctx):
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, lib().dms_diagram1(ctx, ctypes.byref(p), ctypes.byref(n)))
    return p.value, int(n.value)


def dms_generators(ctx):
    """-> (device pointer of int64 offsets [n+1], device pointer of int64 edge ids, n)"""
    po, pe, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, lib().dms_generators(ctx, ctypes.byref(po), ctypes.byref(pe), ctypes.byref(n)))
    return po.value, pe.value, int(n.value)


def dms_run_all(ctx, rank=None, grad=None):
    _check(ctx, lib().dms_run_all(ctx, ctypes.c_void_p(rank.data_ptr() if rank is not None else 0),
                                  ctypes.c_void_p(grad.data_ptr() if grad is not None else 0)))


def dms_run_all_host(ctx, f_host, rank=None, grad=None):
    """f_host: a CPU float32 tensor (pinned for an overlapped upload), N elements."""
    _check(ctx, lib().dms_run_all_host(ctx, ctypes.c_void_p(f_host.data_ptr()),
                                       ctypes.c_void_p(rank.data_ptr() if rank is not None else 0),
                                       ctypes.c_void_p(grad.data_ptr() if grad is not None else 0)))


def dms_sync(ctx):
    _check(ctx, lib().dms_sync(ctx))


def dms_set_timing(ctx, enable=True):
    _check(ctx, lib().dms_set_timing(ctx, int(bool(enable))))


STAGES = ("order", "gradient", "critical", "d0", "dtop", "gradient_kernel", None, "d0_trace", "dtop_trace",
          "d0_uf", "dtop_uf", "d1", "generators")


def dms_stage_ms(ctx):
    """-> dict stage -> accumulated ms, plus 'gradient_launches'"""
    out = (ctypes.c_double * len(STAGES))()
    _check(ctx, lib().dms_stage_ms(ctx, out))
    d = {STAGES[i]: float(out[i]) for i in range(len(STAGES)) if STAGES[i]}
    d["gradient_launches"] = int(out[6])
    return d


def dms_launch_count(ctx):
    return int(lib().dms_launch_count(ctx))


def dms_destroy(ctx):
    if ctx:
        lib().dms_destroy(ctx)


def dms_decode_pairs(shape, words: np.ndarray, v0: int, v1: int, complex="freudenthal") -> np.ndarray:
    """Decode host gradient words of vertices [v0, v1) into (tail dim, tail id, head id).
    complex "5tet": words = the whole gradient buffer; the vectors whose head cell is
    anchored in [v0, v1) (dms_decode_pairs2)."""
    dims, ndim = _dims_of(shape)
    words = np.ascontiguousarray(words)
    cap = max(1, (v1 - v0) * 40)
    out = np.empty((cap, 3), dtype=np.int64)
    n = lib().dms_decode_pairs2(dims, ndim, COMPLEXES[complex], words.ctypes.data, int(v0), int(v1),
                                out.ctypes.data, cap)
    if n < 0:
        raise DMSError(1, "decode")
    return out[:n]


# ---------------------------------------------------------------- convenience class

class DMS:
    """One field on one stream.  Results come back as torch tensors / numpy arrays."""

    def __init__(self, f, stream=None, complex="freudenthal"):
        import torch

        self.torch = torch
        self.f = f
        self.shape = tuple(f.shape)
        self.ndim = f.dim()
        self.N = f.numel()
        self.complex = complex
        self.ctx = dms_create(f, stream, complex)

    def close(self):
        dms_destroy(self.ctx)
        self.ctx = None

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.close()
        except Exception:
            pass

    def _copy(self, dst_ptr, src_ptr, nbytes):
        _check(self.ctx, lib().dms_copy(self.ctx, ctypes.c_void_p(dst_ptr), ctypes.c_void_p(src_ptr), nbytes))

    def order(self, rank=None):
        t = self.torch
        if rank is None:
            rank = t.empty(self.N, dtype=t.int32, device=self.f.device)
        dms_order(self.ctx, rank)
        self._rank = rank  # the context borrows the buffer (dms.h): keep it alive with the context
        return rank

    def gradient(self, grad=None):
        t = self.torch
        if grad is None:
            grad = t.empty(dms_gradient_bytes(self.ctx), dtype=t.uint8, device=self.f.device)
        dms_gradient(self.ctx, grad)
        self._grad = grad  # borrowed by the context until the next gradient pass
        return grad

    def run_all(self, rank=None, grad=None):
        dms_run_all(self.ctx, rank, grad)
        self._rank, self._grad = rank, grad

    def run_all_host(self, f_host, rank=None, grad=None):
        """run_all with the field uploaded from host memory (overwrites the device field)."""
        if f_host.device.type != "cpu" or f_host.dtype != self.torch.float32 or f_host.numel() != self.f.numel():
            raise ValueError("f_host must be a CPU float32 tensor with the field's size")
        if not f_host.is_contiguous():
            raise ValueError("f_host must be contiguous")
        dms_run_all_host(self.ctx, f_host, rank, grad)
        self._rank, self._grad = rank, grad

    def critical(self):
        """-> list of int64 CUDA tensors C_0..C_d (lexicographically sorted)."""
        t = self.torch
        cnt, ptr = dms_critical(self.ctx)
        out = []
        for k in range(self.ndim + 1):
            a = t.empty(cnt[k], dtype=t.int64, device=self.f.device)
            if cnt[k]:
                self._copy(a.data_ptr(), ptr[k], cnt[k] * 8)
            out.append(a)
        return out

    def _pairs(self, p, n, out=None):
        nbytes = n * PAIR_DTYPE.itemsize
        if out is None:
            a = np.empty(n, dtype=PAIR_DTYPE)
        else:  # caller's (pinned) CPU uint8 tensor: a view of its first n records
            if out.device.type != "cpu" or out.dtype != self.torch.uint8 or out.numel() < nbytes:
                raise ValueError("out must be a CPU uint8 tensor of at least %d bytes" % nbytes)
            a = out.numpy()[:nbytes].view(PAIR_DTYPE)
        if n:
            self._copy(a.ctypes.data, p, nbytes)
        return a

    def diagram0(self, out=None) -> np.ndarray:
        """D0 as a structured array (PAIR_DTYPE); out: optional pinned CPU uint8 tensor
        to copy into (the result is then a view of it)."""
        return self._pairs(*dms_diagram0(self.ctx), out=out)

    def diagram_top(self, mode=0, out=None) -> np.ndarray:
        return self._pairs(*dms_diagram_top(self.ctx, mode), out=out)

    def unpaired_saddles(self, which) -> np.ndarray:
        p, n = dms_unpaired_saddles(self.ctx, which)
        a = np.empty(n, dtype=np.int64)
        if n:
            self._copy(a.ctypes.data, p, n * 8)
        return a

    def diagram1(self, out=None) -> np.ndarray:
        """D1 (3D): one pair per 2-saddle left by D2, in increasing death order."""
        return self._pairs(*dms_diagram1(self.ctx), out=out)

    def generators(self):
        """-> (offsets int64 [n+1], edge ids int64): the generator of D1 pair i is
        edges[offsets[i]:offsets[i+1]] (ascending lexicographic order)."""
        po, pe, n = dms_generators(self.ctx)
        off = np.empty(n + 1, dtype=np.int64)
        self._copy(off.ctypes.data, po, (n + 1) * 8)
        e = np.empty(int(off[-1]), dtype=np.int64)
        if e.size:
            self._copy(e.ctypes.data, pe, e.size * 8)
        return off, e

    def launch_count(self):
        return dms_launch_count(self.ctx)

"""CPU oracle for the DMS front end -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2206_13932_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/dms_oracle.c`` (plain C, every step cited to
PAPER.md); this module only loads the shared library (building it with gcc when it is
missing or older than the source) and marshals numpy arrays.

Parity status per function:
  ranks            pinned  (numpy stable argsort; SPEC S:117-119 examples)
  gradient         pinned  (validity invariants, Euler characteristic, Robins'
                            guarantee vs brute-force lower-link homology, canonical
                            critical edges, hand-built fields)
  critical lists   pinned  (brute-force lexicographic sort, hand-built fields)
  D0               pinned  (brute-force Kruskal over all edges; boundary-matrix reduction)
  D_{d-1}          pinned  (brute-force boundary-matrix reduction, vertex level)
  D_{d-1} ignore   pinned  (brute-force Kruskal over the interior facets of the dual
                            graph, elder rule, vertex level; hand-built fields)
  D1 (3D)          pinned  (brute-force boundary-matrix reduction, vertex level; count
                            identities |D1| = |C1|-|D0| = |C2|-|D2|; solid-torus field)
  generators       pinned  (mod-2 cycles, highest edge = the birth edge, homologous to
                            the death triangle's boundary: cycle + boundary in the span of
                            earlier triangles' boundaries, by GF(2) rank)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dms_oracle.c")
_LIB = os.path.join(_HERE, "libdms_oracle.so")

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

(ORC_CRIT, ORC_PAIRS, ORC_D0, ORC_DTOP, ORC_UN0, ORC_UNTOP, ORC_ARCS0, ORC_ARCSTOP, ORC_MS, ORC_D1,
 ORC_GEN_OFF, ORC_GEN, ORC_UN1, ORC_DTOP_IGN) = range(14)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lpthread", "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.orc_ranks.argtypes = [i64, p, p]
        L.orc_ranks.restype = ctypes.c_int
        L.orc_run.argtypes = [ctypes.c_int, p, p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(p)]
        L.orc_run.restype = ctypes.c_int
        L.orc_run2.argtypes = [ctypes.c_int, p, p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(p)]
        L.orc_run2.restype = ctypes.c_int
        L.orc_gradient_sample.argtypes = [ctypes.c_int, p, p, p, i64, ctypes.c_int, ctypes.POINTER(p)]
        L.orc_gradient_sample.restype = ctypes.c_int
        L.orc_count.argtypes = [p, ctypes.c_int, ctypes.c_int]
        L.orc_count.restype = i64
        L.orc_copy.argtypes = [p, ctypes.c_int, ctypes.c_int, p]
        L.orc_copy.restype = None
        L.orc_free.argtypes = [p]
        L.orc_free.restype = None
        L.orc_simplex_vertices.argtypes = [ctypes.c_int, p, ctypes.c_int, i64, p]
        L.orc_simplex_vertices.restype = ctypes.c_int
        L.orc_cells_per_vertex.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_cells_per_vertex.restype = i64
        L.orc_run3.argtypes = [ctypes.c_int, p, p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(p)]
        L.orc_run3.restype = ctypes.c_int
        L.orc_gradient_sample2.argtypes = [ctypes.c_int, p, p, p, i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(p)]
        L.orc_gradient_sample2.restype = ctypes.c_int
        L.orc_simplex_vertices2.argtypes = [ctypes.c_int, p, ctypes.c_int, i64, ctypes.c_int, p]
        L.orc_simplex_vertices2.restype = ctypes.c_int
        L.orc_cells_per_vertex2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_cells_per_vertex2.restype = i64
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        names = {1: "ARG", 2: "DEGENERATE", 3: "NAN", 4: "TOO_LARGE"}
        super().__init__("oracle status %d (%s)" % (code, names.get(code, "?")))
        self.code = code


def _dims(shape):
    """numpy array shape [Lz, Ly, Lx] (C order, x fastest) -> (ndim, int64[3] x-first)."""
    ndim = len(shape)
    L = np.ones(3, dtype=np.int64)
    for i, n in enumerate(reversed(shape)):
        L[i] = n
    return ndim, L


def ranks(f: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float32).ravel()
    out = np.empty(f.size, dtype=np.int32)
    st = lib().orc_ranks(f.size, f.ctypes.data, out.ctypes.data)
    if st:
        raise OracleError(st)
    return out


class Result:
    """Everything the oracle computed for one field (numpy copies)."""

    def __init__(self, handle, ndim: int, full: bool):
        L = lib()
        self.ndim = ndim

        def arr(what, k, dtype, width=1):
            n = L.orc_count(handle, what, k)
            a = np.empty(n * width if dtype != PAIR_DTYPE else n, dtype=dtype)
            if n:
                L.orc_copy(handle, what, k, a.ctypes.data)
            return a.reshape(-1, width) if width > 1 else a

        self.crit = [arr(ORC_CRIT, k, np.int64) for k in range(ndim + 1)]
        self.pairs = arr(ORC_PAIRS, 0, np.int64, 3)
        if full:
            self.d0 = arr(ORC_D0, 0, PAIR_DTYPE)
            self.dtop = arr(ORC_DTOP, 0, PAIR_DTYPE)
            # D_{d-1} in the "ignore" boundary mode (no virtual maximum; App. A)
            self.dtop_ignore = arr(ORC_DTOP_IGN, 0, PAIR_DTYPE)
            self.unpaired0 = arr(ORC_UN0, 0, np.int64)
            self.unpaired_top = arr(ORC_UNTOP, 0, np.int64)
            self.arcs0 = arr(ORC_ARCS0, 0, np.int64, 2)
            self.arcs_top = arr(ORC_ARCSTOP, 0, np.int64, 2)
            self.ms = arr(ORC_MS, 0, np.float64)
            # 3D with want_d1: D1 (Alg. 3), its generators (Sec. 9), unpaired 1-saddles
            self.d1 = arr(ORC_D1, 0, PAIR_DTYPE)
            self.gen_off = arr(ORC_GEN_OFF, 0, np.int64)
            self.gen = arr(ORC_GEN, 0, np.int64)
            self.unpaired1 = arr(ORC_UN1, 0, np.int64)
        L.orc_free(handle)


COMPLEXES = {"freudenthal": 0, "5tet": 1}


def _cplx(complex) -> int:
    """complex: "freudenthal" (Kuhn triangulation, 1D/2D/3D) or "5tet" (five tetrahedra per
    cube, 3D only -- the paper's benchmark subdivision; reading Z21)."""
    if isinstance(complex, str):
        return COMPLEXES[complex]
    return int(complex)


def run(f: np.ndarray, nthreads: int = 1, want_pairs: bool = True, want_d1: bool = False,
        complex="freudenthal") -> Result:
    """Whole front end on a field given as a numpy array of shape [Lz,Ly,Lx], [Ly,Lx] or [Lx].
    want_d1 (3D): also D1 by Alg. 3 "PairCriticalSimplices" and its generators (Sec. 9)."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    ndim, L = _dims(f.shape)
    h = ctypes.c_void_p()
    flags = (1 if want_pairs else 0) | (2 if want_d1 else 0)
    st = lib().orc_run3(ndim, L.ctypes.data, f.ctypes.data, int(nthreads), flags, _cplx(complex), ctypes.byref(h))
    if st:
        raise OracleError(st)
    return Result(h, ndim, True)


def gradient_sample(f: np.ndarray, verts, nthreads: int = 1, complex="freudenthal") -> Result:
    """Gradient pairs and critical ids of the lower stars of the given vertices only."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    ndim, L = _dims(f.shape)
    v = np.ascontiguousarray(verts, dtype=np.int64)
    h = ctypes.c_void_p()
    st = lib().orc_gradient_sample2(
        ndim, L.ctypes.data, f.ctypes.data, v.ctypes.data, v.size, int(nthreads), _cplx(complex), ctypes.byref(h)
    )
    if st:
        raise OracleError(st)
    return Result(h, ndim, False)


def simplex_vertices(shape, dim: int, sid: int, complex="freudenthal") -> np.ndarray:
    """Vertex ids of the anchored simplex id (ascending vertex id), readings Z13 / Z21."""
    ndim, L = _dims(shape)
    out = np.zeros(4, dtype=np.int64)
    st = lib().orc_simplex_vertices2(ndim, L.ctypes.data, dim, int(sid), _cplx(complex), out.ctypes.data)
    if st:
        raise OracleError(st)
    return np.sort(out[: dim + 1])


def cells_per_vertex(ndim: int, dim: int, complex="freudenthal") -> int:
    return int(lib().orc_cells_per_vertex2(ndim, dim, _cplx(complex)))

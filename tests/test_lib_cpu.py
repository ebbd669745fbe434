"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/dms.h
declares, and its host-side gradient decoder agrees with the oracle's simplex ids."""
from __future__ import annotations

import itertools
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dms():
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as m

    m.lib()
    return m


def test_header_symbols_exported(dms):
    hdr = open(os.path.join(ROOT, "include", "dms.h")).read()
    declared = sorted(set(re.findall(r"\b(dms_[a-z0-9_]+)\s*\(", hdr)))
    assert declared, "no declarations found"
    L = dms.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(dms.ABI_SYMBOLS) == declared


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2206_13932_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|#include[^\n]*oracle|dms_oracle|orc_)", src), fn


def _vertices(shape, dim, sid):
    return set(int(v) for v in oracle.simplex_vertices(shape, dim, sid))


@pytest.mark.parametrize("shape", [(4, 5, 6), (5, 7), (9,)])
def test_decode_vertex_codes_match_oracle_ids(dms, shape):
    """A word whose vertex code points at neighbour slot s decodes to the edge (v, v+off_s);
    the product's anchored-id tables must agree with the oracle's id convention."""
    d = len(shape)
    Lx = shape[-1]
    Ly = shape[-2] if d > 1 else 1
    Lz = shape[-3] if d > 2 else 1
    v = Lx // 2 + Lx * (Ly // 2 + Ly * (Lz // 2))  # an interior vertex
    nslots = {3: 14, 2: 6, 1: 2}[d]
    seen = set()
    for s in range(nslots):
        if d == 3:
            w = np.zeros(2, dtype=np.uint64)
            w[0] = np.uint64(s) << np.uint64(56)  # dms.h: vertex code in lo bits 56-59
            w[1] = 0
        elif d == 2:
            w = np.array([s], dtype=np.uint16)
        else:
            w = np.array([s], dtype=np.uint8)
        tr = dms.dms_decode_pairs(shape, w.view(np.uint8), v, v + 1)
        assert tr.shape == (1, 3) and tr[0, 0] == 0 and tr[0, 1] == v
        verts = _vertices(shape, 1, int(tr[0, 2]))
        assert v in verts
        (u,) = verts - {v}
        seen.add(u - v)
    assert len(seen) == nslots
    # the offsets are exactly the Freudenthal neighbourhood (PAPER.md 1362-1364)
    offs = set()
    for dz in (-1, 0, 1) if d == 3 else (0,):
        for dy in (-1, 0, 1) if d >= 2 else (0,):
            for dx in (-1, 0, 1):
                o = (dx, dy, dz)
                if any(o) and not (min(o) < 0 < max(o)):
                    offs.add(dx + Lx * dy + Lx * Ly * dz)
    assert seen == offs


def test_decode_all_codes_are_facet_pairs(dms):
    """Every tri/tet code decodes to a (facet, cofacet) pair of the complex that both
    contain the star centre."""
    shape = (5, 5, 5)
    v = 62  # interior
    # slot -> neighbour vertex, through the vertex codes (dms.h: lo bits 56-59)
    nb = []
    for s in range(14):
        w = np.zeros(2, dtype=np.uint64)
        w[0] = np.uint64(s) << np.uint64(56)
        tr = dms.dms_decode_pairs(shape, w.view(np.uint8), v, v + 1)
        (u,) = _vertices(shape, 1, int(tr[0, 2])) - {v}
        nb.append(u)

    def coords(u):
        return np.array([u % 5, (u // 5) % 5, u // 25])

    npairs = 0
    for e in range(14):
        for u in range(14):
            d = coords(nb[u]) - coords(nb[e])
            if e == u or not (set(d.tolist()) <= {0, 1} or set(d.tolist()) <= {0, -1}):
                continue  # (x, n_e, n_u) is not a triangle of the Freudenthal star
            # edge slot e paired with the triangle whose third vertex is slot u: nibble u + 1
            w = np.zeros(2, dtype=np.uint64)
            w[0] = (np.uint64(u + 1) << np.uint64(4 * e)) | (np.uint64(15) << np.uint64(56))
            tr = dms.dms_decode_pairs(shape, w.view(np.uint8), v, v + 1)
            assert tr.shape == (1, 3) and tr[0, 0] == 1
            a, b = _vertices(shape, 1, int(tr[0, 1])), _vertices(shape, 2, int(tr[0, 2]))
            assert a == {v, nb[e]} and b == {v, nb[e], nb[u]}
            npairs += 1
    assert npairs == 72  # 36 star triangles, each from either of its two edges at x
    for q in range(24):
        for code in (1, 2, 3):
            w = np.zeros(2, dtype=np.uint64)
            w[0] = np.uint64(15) << np.uint64(56)
            w[1] = np.uint64(code) << np.uint64(2 * q)
            tr = dms.dms_decode_pairs(shape, w.view(np.uint8), v, v + 1)
            assert tr.shape == (1, 3) and tr[0, 0] == 2
            a, b = _vertices(shape, 2, int(tr[0, 1])), _vertices(shape, 3, int(tr[0, 2]))
            assert a < b and v in a


def test_no_cpu_fallback_without_device(dms):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(TypeError):
        dms.dms_create(torch.zeros(4, 4))


@pytest.mark.parametrize("dims,ndim", [((1 << 16, 1 << 15, 1), 2), ((800, 800, 800), 3), ((720, 720, 720), 3),
                                       ((1 << 31,), 1)])
def test_too_large_rejected_before_any_device_work(dms, dims, ndim):
    """Size limits (include/dms.h DMS_ERR_TOO_LARGE): N < 2^31 and C_d * N < 2^31 (int32
    vertex and top-cell indexing).  Checked before the library touches the device, so it
    runs without a GPU (the device pointer is never dereferenced)."""
    import ctypes

    L = dms.lib()
    arr = (ctypes.c_int64 * 3)(*(list(dims) + [1] * (3 - len(dims))))
    out = ctypes.c_void_p()
    st = L.dms_create(arr, ndim, ctypes.c_void_p(0x1000), None, ctypes.byref(out))
    assert st == 4 and not out.value  # DMS_ERR_TOO_LARGE, no context


def _t5_slots(parity):
    """Neighbour offsets of a five-tetrahedra star, in vertex-id order: every vertex has its
    6 axis neighbours; an even-sum vertex also the 12 face-diagonal ones (reading Z21)."""
    offs = [o for o in itertools.product((-1, 0, 1), repeat=3) if sum(map(abs, o)) == 1]
    if parity == 0:
        offs += [o for o in itertools.product((-1, 0, 1), repeat=3) if sum(map(abs, o)) == 2]
    return sorted(offs, key=lambda o: (o[2], o[1], o[0]))


@pytest.mark.parametrize("shape", [(3, 4, 5), (5, 4, 3), (4, 4, 4)])
def test_t5_decode_matches_oracle_ids(dms, shape):
    """dms_decode_pairs2 on the five-tetrahedra complex (host code, no GPU) against the
    oracle: gradient bytes built from the oracle's vectors in the layout of dms.h decode
    back to exactly those vectors -- the library's and the oracle's simplex ids and
    facet numbering (derived independently) agree."""
    import oracle

    f = np.random.default_rng(7).random(shape, dtype=np.float32)
    res = oracle.run(f, complex="5tet")
    Lz, Ly, Lx = shape
    N = f.size
    w = np.full(16 * N, 0xEE, np.uint8)  # cells that are no head: any code > dim
    w[:N] = 0xFF  # minima
    for tdim, tid, hid in res.pairs:
        tv = set(oracle.simplex_vertices(shape, int(tdim), int(tid), "5tet"))
        hv = sorted(oracle.simplex_vertices(shape, int(tdim) + 1, int(hid), "5tet"))
        if tdim == 0:
            v = int(tid)
            (u,) = set(hv) - {v}
            c = lambda q: (q % Lx, (q // Lx) % Ly, q // (Lx * Ly))
            o = tuple(np.subtract(c(u), c(v)))
            w[v] = _t5_slots(sum(c(v)) % 2).index(o)
        else:
            j = hv.index((set(hv) - tv).pop())  # the omitted vertex, in ascending-id order
            w[(N if tdim == 1 else 11 * N) + hid] = j
    got = dms.dms_decode_pairs(shape, w, 0, N, complex="5tet")
    got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
    assert np.array_equal(got, res.pairs)

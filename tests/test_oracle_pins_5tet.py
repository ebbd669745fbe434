"""Pins of the oracle's five-tetrahedra complex (reading Z21).

The paper's benchmark volumes are cut into five tetrahedra per cube.  The oracle's
complex (``oracle/dms_oracle.c`` O2') is checked here against things other than itself:
an independent enumeration written out by hand in ``tests/brute.py`` (``five_tet``: the
even cube's tetrahedra as coordinates, the odd cube as their mirror image), closed-form
simplex counts, the Euler characteristic of a ball, the pseudomanifold property,
Robins' guarantee on every lower star, Kruskal over all edges and the boundary-matrix
reduction for D0, D2 and D1.  No GPU.
"""
from __future__ import annotations

import numpy as np
import pytest

import brute
import oracle
from test_oracle_pins import _check_generators, check_gradient, ids_to_sets, pair_sets, robins_guarantee

C = "5tet"


def closed_form_counts(L):
    """(V, E, F, T) of the five-tetrahedra subdivision of an Lx x Ly x Lz grid: the axis
    edges plus one diagonal per square face; two triangles per square face plus the
    four inner faces of the central tetrahedron per cube; five tetrahedra per cube."""
    Lx, Ly, Lz = L
    ax, ay, az = Lx - 1, Ly - 1, Lz - 1
    squares = ax * ay * Lz + ax * Ly * az + Lx * ay * az
    cubes = ax * ay * az
    V = Lx * Ly * Lz
    E = ax * Ly * Lz + Lx * ay * Lz + Lx * Ly * az + squares
    return V, E, 2 * squares + 4 * cubes, 5 * cubes


@pytest.mark.parametrize("shape", [(2, 2, 2), (3, 3, 3), (2, 3, 4), (3, 4, 5), (4, 4, 4)])
def test_brute_complex_counts_euler_and_manifold(shape):
    cx = brute.five_tet(shape)
    L = tuple(reversed(shape))
    assert tuple(len(cx[k]) for k in range(4)) == closed_form_counts(L)
    assert sum((-1) ** k * len(cx[k]) for k in range(4)) == 1  # a ball
    # conforming 3-manifold with boundary: every triangle bounds one or two tetrahedra,
    # and the boundary triangles are exactly those on the outer faces of the box
    cof = {t: 0 for t in cx[2]}
    for q in cx[3]:
        for v in q:
            cof[q - {v}] += 1
    Lx, Ly, Lz = L

    def on_outer_face(t):
        cs = [(v % Lx, (v // Lx) % Ly, v // (Lx * Ly)) for v in t]
        for ax, n in enumerate(L):
            vals = set(c[ax] for c in cs)
            if vals == {0} or vals == {n - 1}:
                return True
        return False

    for t, n in cof.items():
        assert n == (1 if on_outer_face(t) else 2), t
    # every square face carries exactly one diagonal, joining its two even-sum corners
    for e in cx[1]:
        a, b = sorted(e)
        ca = np.array([a % Lx, (a // Lx) % Ly, a // (Lx * Ly)])
        cb = np.array([b % Lx, (b // Lx) % Ly, b // (Lx * Ly)])
        d = np.abs(cb - ca)
        assert d.max() == 1 and d.sum() in (1, 2)
        if d.sum() == 2:
            assert ca.sum() % 2 == 0 and cb.sum() % 2 == 0


@pytest.mark.parametrize("shape", [(2, 2, 2), (2, 3, 2), (3, 3, 4), (3, 4, 3)])
def test_anchored_ids_biject_onto_five_tet_complex(shape):
    cx = brute.five_tet(shape)
    N = int(np.prod(shape))
    for k in range(4):
        got = set()
        per = oracle.cells_per_vertex(3, k, C)
        for sid in range(per * N):
            try:
                s = frozenset(int(v) for v in oracle.simplex_vertices(shape, k, sid, C))
            except oracle.OracleError:
                continue
            assert s not in got
            got.add(s)
        assert got == cx[k], (shape, k)


def test_cells_per_vertex():
    # per anchor: 3 axis edges + 3 face diagonals; 2 triangles on each of 3 faces + 4 inner;
    # 5 tetrahedra -- and 1 - 6 + 10 - 5 = 0 per vertex of an infinite grid
    assert [oracle.cells_per_vertex(3, k, C) for k in range(4)] == [1, 6, 10, 5]
    with pytest.raises(oracle.OracleError):  # the 5-tet complex is 3D only
        oracle.run(np.zeros((4, 4), np.float32), complex=C)


SHAPES = [(3, 3, 3), (4, 4, 4), (3, 5, 4), (5, 4, 3), (5, 5, 5)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradient_valid_and_robins(shape, seed):
    rng = np.random.default_rng(300 + seed)
    f = rng.random(shape, dtype=np.float32)
    if seed == 2:  # heavy ties: the index tie-break decides
        f = np.floor(f * 4).astype(np.float32)
    res = oracle.run(f, complex=C)
    cx, r = check_gradient(f, res, C)
    robins_guarantee(f, res, cx, r, C)


def test_even_and_odd_stars():
    """Even-sum vertices have 18 neighbours (6 axis + 12 face diagonals), odd-sum ones 6:
    a bowl centred on an odd vertex still has one minimum; on a constant field the only
    critical cell is the first vertex."""
    shape = (5, 5, 5)
    cx = brute.five_tet(shape)
    deg = {}
    for e in cx[1]:
        for v in e:
            deg[v] = deg.get(v, 0) + 1
    L = tuple(reversed(shape))
    for v, dg in deg.items():
        c = (v % L[0], (v // L[0]) % L[1], v // (L[0] * L[1]))
        if all(0 < ci < n - 1 for ci, n in zip(c, L)):
            assert dg == (18 if sum(c) % 2 == 0 else 6)
    for centre in [(2, 2, 2), (1, 2, 2)]:
        g = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
        f = sum((gi - ci) ** 2 for gi, ci in zip(g, reversed(centre))).astype(np.float32)
        res = oracle.run(f, complex=C)
        assert [len(c) for c in res.crit] == [1, 0, 0, 0]
        assert len(res.d0) == 1 and res.d0[0]["death_id"] == -1
    res = oracle.run(np.zeros(shape, np.float32), complex=C)
    assert [len(c) for c in res.crit] == [1, 0, 0, 0]


BRUTE = [(3, 3, 3), (4, 3, 4), (4, 4, 4), (3, 5, 4)]


@pytest.mark.parametrize("shape", BRUTE)
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_diagrams_vs_brute_force(shape, seed):
    rng = np.random.default_rng(3000 + seed)
    f = rng.random(shape, dtype=np.float32)
    if seed == 3:
        f = np.floor(f * 3).astype(np.float32)  # ties
    res = oracle.run(f, complex=C, want_d1=True)
    # D0 at simplex level = Kruskal over all edges of the 5-tet complex
    kr, r = brute.kruskal_d0(f, C)
    assert pair_sets(shape, res.d0, 0, C) == set((frozenset([b]), e) for b, e in kr)
    red, unpaired, r = brute.diagrams_by_reduction(f, C)

    def vlevel(pairs):
        return sorted((brute.maxvertex(b, r), brute.maxvertex(dd, r)) for b, dd in pairs)

    assert vlevel(pair_sets(shape, res.d0, 0, C)) == vlevel(red.get(0, []))
    top = pair_sets(shape, res.dtop, 2, C)
    assert vlevel(top) == vlevel(red.get(2, []))
    assert top == set(red.get(2, []))
    d1 = pair_sets(shape, res.d1, 1, C)
    assert vlevel(d1) == vlevel(red.get(1, []))
    assert d1 == set(red.get(1, []))
    for p in list(res.d0) + list(res.dtop) + list(res.d1):
        assert p["birth_value"] == f.ravel()[p["birth_vertex"]]
        if p["death_id"] >= 0:
            assert p["death_value"] == f.ravel()[p["death_vertex"]]
    inf = [p for p in res.d0 if p["death_id"] < 0]
    assert len(inf) == 1 and inf[0]["birth_vertex"] == int(np.argmin(np.asarray(r)))
    assert len(unpaired) == 1
    nfin0 = len(res.d0) - 1
    assert nfin0 == len(res.crit[0]) - 1
    assert len(res.dtop) == len(res.crit[3])
    assert len(res.d1) == len(res.crit[1]) - nfin0 == len(res.crit[2]) - len(res.dtop)
    for k in range(4):
        keys = [brute.lexkey(s, r) for s in ids_to_sets(shape, k, res.crit[k], C)]
        assert keys == sorted(keys)
    _check_generators(f, res, r, C)


@pytest.mark.parametrize("shape", [(5, 6, 7), (6, 6, 6)])
@pytest.mark.parametrize("seed", range(3))
def test_ignore_mode_low_moat(shape, seed):
    """Reading Z7 on the 5-tet complex: with the boundary below every interior value, the
    ignore diagram is the exact one minus the global maximum's pair (simplex level), by
    the elder rule alone (see tests/test_oracle_pins.py::test_ignore_mode_low_moat)."""
    rng = np.random.default_rng(4000 + seed)
    f = rng.random(shape).astype(np.float32) + 1.0
    core = tuple(slice(1, n - 1) for n in shape)
    low = np.full(shape, True)
    low[core] = False
    f[low] = -rng.random(int(low.sum())).astype(np.float32)
    res = oracle.run(f, complex=C)
    exact = [p for p in res.dtop if p["death_id"] >= 0]
    gmax = int(np.argmax(f))
    top = [p for p in exact if int(p["death_vertex"]) == gmax]
    assert len(top) == 1
    rest = sorted(p.tobytes() for p in exact if int(p["death_vertex"]) != gmax)
    assert sorted(p.tobytes() for p in res.dtop_ignore) == rest

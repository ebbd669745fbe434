"""Pins of the CPU oracle against things other than itself (runs without a GPU).

Every test compares the oracle with a value the paper / SPEC prints, a closed form, an
invariant of discrete Morse theory, or an independent brute force (tests/brute.py:
Kruskal over all edges and the boundary-matrix column reduction).
"""
from __future__ import annotations

import itertools

import json
import os

import numpy as np
import pytest

import brute
import oracle
from synth import fields


def ids_to_sets(shape, dim, ids, complex="freudenthal"):
    return [frozenset(int(v) for v in oracle.simplex_vertices(shape, dim, int(i), complex)) for i in ids]


def sqdist_field(shape, sign):
    g = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    r2 = sum((c - 2) ** 2 for c in g)
    return (sign * r2).astype(np.float32)


# ------------------------------------------------------------------ O1 order

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", golden("spec_ranks.json")["cases"])
def test_ranks_spec_examples(case):  # tests/golden/spec_ranks.json: S:117-119
    assert list(oracle.ranks(np.array(case["values"], np.float32))) == case["ranks"]


def test_ranks_equal_numpy_stable_argsort():
    rng = np.random.default_rng(1)
    f = rng.integers(0, 50, size=5000).astype(np.float32)  # heavy ties
    f[::7] = -0.0
    f[1::7] = 0.0  # -0 == +0 (reading Z3)
    f[3] = np.inf
    f[4] = -np.inf
    perm = np.argsort(f, kind="stable")
    expect = np.empty_like(perm)
    expect[perm] = np.arange(f.size)
    assert np.array_equal(oracle.ranks(f), expect)


def test_ranks_nan_rejected():
    with pytest.raises(oracle.OracleError):
        oracle.ranks(np.array([0.0, np.nan], np.float32))


# ------------------------------------------------------------------ O2 complex and ids

@pytest.mark.parametrize("shape", [(5,), (3, 4), (2, 2), (3, 3, 4), (2, 2, 2), (2, 3, 2)])
def test_anchored_ids_biject_onto_freudenthal_complex(shape):
    cx = brute.freudenthal(shape)
    d = len(shape)
    N = int(np.prod(shape))
    for k in range(d + 1):
        got = set()
        per = oracle.cells_per_vertex(d, k)
        for sid in range(per * N):
            try:
                s = frozenset(int(v) for v in oracle.simplex_vertices(shape, k, sid))
            except oracle.OracleError:
                continue
            assert s not in got
            got.add(s)
        assert got == cx[k], (shape, k)


def test_cells_per_vertex_and_counts():
    # App. A counts; (2,2,1) -> 4 V, 5 E, 2 T; (2,2,2) -> 6 tets, chi = 1
    assert [oracle.cells_per_vertex(3, k) for k in range(4)] == [1, 7, 12, 6]
    assert [oracle.cells_per_vertex(2, k) for k in range(3)] == [1, 3, 2]
    assert [oracle.cells_per_vertex(1, k) for k in range(2)] == [1, 1]
    cx = brute.freudenthal((2, 2))
    assert [len(cx[k]) for k in range(3)] == [4, 5, 2]
    cx = brute.freudenthal((2, 2, 2))
    assert len(cx[3]) == 6
    assert sum((-1) ** k * len(cx[k]) for k in cx) == 1
    for L in [(3, 4, 5), (2, 3, 7)]:
        cx = brute.freudenthal(tuple(reversed(L)))
        ax, ay, az = (l - 1 for l in L)
        Lx, Ly, Lz = L
        E = ax * Ly * Lz + Lx * ay * Lz + Lx * Ly * az + ax * ay * Lz + ax * Ly * az + Lx * ay * az + ax * ay * az
        F = 2 * (ax * ay * Lz + ax * Ly * az + Lx * ay * az) + 6 * ax * ay * az
        T = 6 * ax * ay * az
        assert (len(cx[1]), len(cx[2]), len(cx[3])) == (E, F, T)


# ------------------------------------------------------------------ O3 gradient validity

def check_gradient(f, res, complex="freudenthal"):
    """Validity of a discrete gradient plus the partition of
    the complex into pairs and critical simplices."""
    shape = f.shape
    d = len(shape)
    cx = brute.complex_of(shape, complex)
    r = brute.ranks(f)
    seen = set()
    head_of = {}  # tail -> head
    for tdim, tid, hid in res.pairs:
        t = ids_to_sets(shape, int(tdim), [tid], complex)[0]
        h = ids_to_sets(shape, int(tdim) + 1, [hid], complex)[0]
        assert t < h and len(h) == len(t) + 1  # facet / cofacet
        assert brute.maxvertex(t, r) == brute.maxvertex(h, r)  # same lower star: zero persistence
        assert t not in seen and h not in seen  # at most one vector per simplex
        seen.add(t)
        seen.add(h)
        head_of[t] = h
    crit = set()
    for k in range(d + 1):
        for s in ids_to_sets(shape, k, res.crit[k], complex):
            assert s not in seen and s not in crit
            crit.add(s)
    allsimp = set(s for k in cx for s in cx[k])
    assert seen | crit == allsimp
    # acyclicity: v-paths  t -> head(t) -> other facet t' of head(t) -> head(t') ...
    succ = {}
    for t, h in head_of.items():
        succ[t] = [h - {v} for v in h if (h - {v}) != t and (h - {v}) in head_of]
    color = {}

    def dfs(u):
        stack = [(u, iter(succ.get(u, ())))]
        color[u] = 1
        while stack:
            node, it = stack[-1]
            nxt = next(it, None)
            if nxt is None:
                color[node] = 2
                stack.pop()
                continue
            c = color.get(nxt, 0)
            assert c != 1, "cycle in the discrete gradient"
            if c == 0:
                color[nxt] = 1
                stack.append((nxt, iter(succ.get(nxt, ()))))

    for t in head_of:
        if color.get(t, 0) == 0:
            dfs(t)
    # Euler characteristic of a grid (a ball): sum (-1)^k |C_k| = 1
    assert sum((-1) ** k * len(res.crit[k]) for k in range(d + 1)) == 1
    return cx, r


def robins_guarantee(f, res, cx, r, complex="freudenthal"):
    """Robins et al.: the critical k-simplices in St^-(x) number beta~_{k-1}(Lk^-(x))
    (P:1049-1054); critical edges are canonical (reading Z16)."""
    shape = f.shape
    d = len(shape)
    crit_by_x = {}
    for k in range(d + 1):
        for s in ids_to_sets(shape, k, res.crit[k], complex):
            crit_by_x.setdefault(brute.maxvertex(s, r), []).append(s)
    for x in range(len(r)):
        lk = brute.lower_link(cx, x, r)
        b = brute.reduced_betti(lk)
        got = [0] * (d + 1)
        for s in crit_by_x.get(x, []):
            got[len(s) - 1] += 1
        for k in range(d + 1):
            assert got[k] == b[k - 1], (x, k, got, b)
        # canonical critical edges: one per component of Lk^-(x) other than the one
        # holding the lowest lower neighbour, joined to that component's lowest vertex
        verts = [next(iter(s)) for s in lk if len(s) == 1]
        if not verts:
            continue
        comp = {v: v for v in verts}

        def find(a):
            while comp[a] != a:
                a = comp[a]
            return a

        for s in lk:
            if len(s) == 2:
                a, bb = (find(v) for v in s)
                if a != bb:
                    comp[a] = bb
        lowest = {}
        for v in verts:
            c = find(v)
            if c not in lowest or r[v] < r[lowest[c]]:
                lowest[c] = v
        glob = min(verts, key=lambda v: r[v])
        expect = set(frozenset((x, lowest[c])) for c in lowest if c != find(glob))
        gotedges = set(s for s in crit_by_x.get(x, []) if len(s) == 2)
        assert gotedges == expect


SMALL_SHAPES = [(9,), (17,), (5, 6), (7, 7), (4, 4, 4), (3, 5, 4), (5, 5, 5)]


@pytest.mark.parametrize("shape", SMALL_SHAPES)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradient_valid_and_robins(shape, seed):
    rng = np.random.default_rng(100 + seed)
    f = rng.random(shape, dtype=np.float32)
    if seed == 2:  # heavy ties: the index tie-break decides
        f = np.floor(f * 4).astype(np.float32)
    res = oracle.run(f)
    cx, r = check_gradient(f, res)
    robins_guarantee(f, res, cx, r)


def test_gradient_constant_and_elevation():
    # pure index order -> one critical simplex; elevation -> one bar
    for f in [np.zeros((4, 4, 4), np.float32), np.tile(np.arange(6, dtype=np.float32), (5, 1)),
              np.arange(20, dtype=np.float32)]:
        res = oracle.run(f)
        assert [len(c) for c in res.crit] == [1] + [0] * (f.ndim)
        assert len(res.d0) == 1 and res.d0[0]["death_id"] == -1
        assert res.d0[0]["birth_value"] == f.min() and res.d0[0]["death_value"] == f.max()
        assert len(res.dtop) == (1 if f.ndim == 1 else 0)


# ------------------------------------------------------------------ hand-built fields

def test_spec_path_example():
    g = golden("spec_path_1d.json")
    f = np.array(g["field"], np.float32)
    res = oracle.run(f)
    assert list(res.crit[0]) == g["crit0"]
    assert ids_to_sets(f.shape, 1, res.crit[1]) == [frozenset(s) for s in g["crit1_vertex_sets"]]
    d0 = [[float(p["birth_value"]), float(p["death_value"]), int(p["death_id"]) < 0] for p in res.d0]
    assert d0 == g["d0"]


def test_1d_example_table():
    g = golden("hand_1d_table.json")
    f = np.array(g["field"], np.float32)
    res = oracle.run(f)
    assert [len(c) for c in res.crit] == g["crit_counts"]
    fin = sorted((float(p["birth_value"]), float(p["death_value"])) for p in res.d0 if p["death_id"] >= 0)
    assert fin == [tuple(x) for x in g["d0_finite"]]
    inf = [(float(p["birth_value"]), float(p["death_value"])) for p in res.d0 if p["death_id"] < 0]
    assert inf == [tuple(x) for x in g["d0_infinite"]]
    # 1D: D_{d-1} = D0 (duality), including the infinite class
    top = sorted((float(p["birth_value"]), float(p["death_value"])) for p in res.dtop)
    assert top == sorted(fin + inf)


@pytest.mark.parametrize("d", [2, 3])
def test_negative_paraboloid(d):
    g = golden("paraboloids.json")["neg"][str(d)]
    f = sqdist_field((5,) * d, -1)
    res = oracle.run(f)
    assert [len(c) for c in res.crit] == g["crit_counts"]
    fin = sorted((float(p["birth_value"]), float(p["death_value"])) for p in res.d0 if p["death_id"] >= 0)
    assert fin == [tuple(x) for x in g["d0_finite"]]
    assert [(float(p["birth_value"]), float(p["death_value"])) for p in res.dtop] == [tuple(x) for x in g["dtop"]]
    if d == 3:  # |D1| = |C1| - |D0 finite| = |C2| - |D2|
        assert len(res.crit[1]) - len(fin) == len(res.crit[2]) - len(res.dtop) == g["d1_count"]
    inf = [p for p in res.d0 if p["death_id"] < 0]
    assert len(inf) == 1 and float(inf[0]["birth_value"]) == -4.0 * d and float(inf[0]["death_value"]) == 0.0


@pytest.mark.parametrize("d", [2, 3])
def test_bowl(d):
    g = golden("paraboloids.json")["bowl"][str(d)]
    f = sqdist_field((5,) * d, +1)
    res = oracle.run(f)
    assert [len(c) for c in res.crit] == g["crit_counts"]
    assert len(res.dtop) == 0
    assert [(float(p["birth_value"]), float(p["death_value"])) for p in res.d0] == [tuple(x) for x in g["d0"]]


# ------------------------------------------------------------------ O5 / O6 vs brute force

def pair_sets(shape, res_pairs, bdim, complex="freudenthal"):
    out = set()
    for p in res_pairs:
        if p["death_id"] < 0:
            continue
        b = ids_to_sets(shape, bdim, [p["birth_id"]], complex)[0]
        dd = ids_to_sets(shape, bdim + 1, [p["death_id"]], complex)[0]
        out.add((b, dd))
    return out


BRUTE_SHAPES = [(12,), (30,), (4, 5), (6, 6), (3, 3, 3), (4, 3, 4), (4, 4, 4)]


@pytest.mark.parametrize("shape", BRUTE_SHAPES)
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_diagrams_vs_brute_force(shape, seed):
    rng = np.random.default_rng(1000 + seed)
    f = rng.random(shape, dtype=np.float32)
    if seed == 3:
        f = np.floor(f * 3).astype(np.float32)  # ties
    d = len(shape)
    res = oracle.run(f)
    # D0 at simplex level = Kruskal over all edges (elder rule, zero persistence dropped)
    kr, r = brute.kruskal_d0(f)
    kr_set = set((frozenset([b]), e) for b, e in kr)
    assert pair_sets(shape, res.d0, 0) == kr_set
    # D0 and D_{d-1} vs the boundary-matrix reduction (vertex level: max vertices)
    red, unpaired, r = brute.diagrams_by_reduction(f)

    def vlevel(pairs):
        return sorted((brute.maxvertex(b, r), brute.maxvertex(dd, r)) for b, dd in pairs)

    assert vlevel(pair_sets(shape, res.d0, 0)) == vlevel(red.get(0, []))
    top = pair_sets(shape, res.dtop, d - 1)
    assert vlevel(top) == vlevel(red.get(d - 1, []))
    # simplex level too (holds for this pinned gradient, reading Z14)
    assert top == set(red.get(d - 1, []))
    # field values of the pairs are f at the max vertices
    for p in list(res.d0) + list(res.dtop):
        assert p["birth_value"] == f.ravel()[p["birth_vertex"]]
        if p["death_id"] >= 0:
            assert p["death_value"] == f.ravel()[p["death_vertex"]]
        else:
            assert p["death_value"] == f.max()
    # exactly one infinite class (a ball: beta = (1,0,0)), the global minimum
    inf = [p for p in res.d0 if p["death_id"] < 0]
    assert len(inf) == 1 and inf[0]["birth_vertex"] == int(np.argmin(np.asarray(r)))
    assert len([u for u in unpaired]) == 1
    # cross-checks
    nfin0 = len(res.d0) - 1
    assert nfin0 == len(res.crit[0]) - 1
    if d >= 2:
        assert len(res.dtop) == len(res.crit[d])
    if d == 2:
        # C_1 = D0 death edges + D1 birth edges, disjoint
        deaths = set(int(p["death_id"]) for p in res.d0 if p["death_id"] >= 0)
        births = set(int(p["birth_id"]) for p in res.dtop)
        assert deaths.isdisjoint(births) and deaths | births == set(int(i) for i in res.crit[1])
        assert set(int(i) for i in res.unpaired_top) == deaths
    if d == 3:
        assert len(res.crit[1]) - nfin0 == len(res.crit[2]) - len(res.dtop)
    if d == 1:
        fin = sorted((int(p["birth_vertex"]), int(p["death_vertex"])) for p in res.d0)
        top = sorted((int(p["birth_vertex"]), int(p["death_vertex"])) for p in res.dtop)
        assert fin == top
    # the critical lists are sorted by the lexicographic order (Alg. 2 l. 13)
    for k in range(d + 1):
        keys = [brute.lexkey(s, r) for s in ids_to_sets(shape, k, res.crit[k])]
        assert keys == sorted(keys)


def test_sample_mode_matches_full_run():
    f = fields.uniform((6, 7, 5), seed=3)
    full = oracle.run(f)
    verts = np.array([0, 5, 17, 60, 100, 209], np.int64)
    smp = oracle.gradient_sample(f, verts, nthreads=2)
    r = brute.ranks(f)
    shape = f.shape
    for tdim, tid, hid in smp.pairs:
        assert any((full.pairs == [tdim, tid, hid]).all(1))
        t = ids_to_sets(shape, int(tdim), [tid])[0]
        assert brute.maxvertex(t, r) in set(int(v) for v in verts)
    for k in range(4):
        sub = [i for i in full.crit[k] if brute.maxvertex(ids_to_sets(shape, k, [i])[0], r) in set(verts.tolist())]
        assert sorted(sub) == sorted(smp.crit[k].tolist())


def test_threads_deterministic():
    f = fields.uniform((10, 11, 12), seed=5)
    a = oracle.run(f, nthreads=1)
    b = oracle.run(f, nthreads=4)
    assert np.array_equal(a.pairs, b.pairs)
    for k in range(4):
        assert np.array_equal(a.crit[k], b.crit[k])
    assert a.d0.tobytes() == b.d0.tobytes() and a.dtop.tobytes() == b.dtop.tobytes()


def test_degenerate_rejected():
    for f in [np.zeros((1, 4, 4), np.float32), np.zeros((1,), np.float32)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.run(f)
        assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(np.array([0.0, np.nan, 1.0], np.float32))
    assert e.value.code == 3


# ------------------------------------------------------------------ O9 D1 (Alg. 3) + generators (Sec. 9)

D1_SHAPES = [(3, 3, 3), (4, 3, 4), (4, 4, 4), (3, 5, 4), (5, 5, 5)]


def _edge_sets(shape, ids, complex="freudenthal"):
    return [frozenset(int(v) for v in oracle.simplex_vertices(shape, 1, int(i), complex)) for i in ids]


@pytest.mark.parametrize("shape", D1_SHAPES)
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_d1_vs_brute_force(shape, seed):
    """D1 of Alg. 3 (PairCriticalSimplices, boundary caching, sandwiching) against the
    full boundary-matrix column reduction (tests/brute.py, Alg. 1's matrix form,
    P:1866-1879): the pairs with different highest vertices agree at vertex level and,
    for this pinned gradient, at simplex level."""
    rng = np.random.default_rng(2000 + seed)
    f = rng.random(shape, dtype=np.float32)
    if seed >= 3:
        f = np.floor(f * (2 + seed)).astype(np.float32)  # heavy ties
    res = oracle.run(f, want_d1=True)
    red, unpaired, r = brute.diagrams_by_reduction(f)
    d1 = pair_sets(shape, res.d1, 1)
    ref = set(red.get(1, []))

    def vlevel(pairs):
        return sorted((brute.maxvertex(b, r), brute.maxvertex(dd, r)) for b, dd in pairs)

    assert vlevel(d1) == vlevel(ref)
    assert d1 == ref
    # |D1| = |C1| - |D0 finite| = |C2| - |D2|, no infinite 1-classes in a ball
    nfin0 = len(res.d0) - 1
    assert len(res.d1) == len(res.crit[1]) - nfin0 == len(res.crit[2]) - len(res.dtop)
    assert len(res.unpaired1) == 0
    # values at the highest vertices, death after birth in the filtration
    for p in res.d1:
        assert p["birth_value"] == f.ravel()[p["birth_vertex"]]
        assert p["death_value"] == f.ravel()[p["death_vertex"]]
        assert p["death_value"] >= p["birth_value"]
    # the pairs come in increasing death order (Alg. 3 processes C_2 in order)
    keys = [brute.lexkey(s, r) for s in ids_to_sets(shape, 2, res.d1["death_id"])]
    assert keys == sorted(keys)
    _check_generators(f, res, r)


def _check_generators(f, res, r, complex="freudenthal"):
    """Sec. 9: the generator of a D1 pair (tau, sigma) is a 1-cycle (every
    vertex has even degree), its highest edge is tau, and it is homologous to the
    boundary of sigma through triangles entering no later than sigma: generator +
    boundary(sigma) lies in the GF(2) span of the boundaries of the triangles preceding
    sigma in the filtration."""
    shape = f.shape
    cx = brute.complex_of(shape, complex)
    tris = sorted(cx[2], key=lambda s: brute.lexkey(s, r))
    edges = sorted(cx[1], key=lambda s: brute.lexkey(s, r))
    eidx = {e: i for i, e in enumerate(edges)}
    tpos = {t: i for i, t in enumerate(tris)}

    def bits_of_edges(es):
        b = 0
        for e in es:
            b ^= 1 << eidx[e]
        return b

    tri_bits = [bits_of_edges([t - {v} for v in t]) for t in tris]
    for i, p in enumerate(res.d1):
        g_ids = res.gen[res.gen_off[i]:res.gen_off[i + 1]]
        g_edges = _edge_sets(shape, g_ids, complex)
        assert len(set(g_edges)) == len(g_edges) > 0
        deg = {}
        for e in g_edges:
            for v in e:
                deg[v] = deg.get(v, 0) + 1
        assert all(x % 2 == 0 for x in deg.values()), "not a cycle"
        tau = _edge_sets(shape, [p["birth_id"]], complex)[0]
        assert max(g_edges, key=lambda e: brute.lexkey(e, r)) == tau
        sigma = ids_to_sets(shape, 2, [p["death_id"]], complex)[0]
        target = bits_of_edges(g_edges) ^ tri_bits[tpos[sigma]]
        earlier = tri_bits[: tpos[sigma]]
        assert brute.gf2_rank(earlier + [target]) == brute.gf2_rank(list(earlier)), "not homologous"


def test_d1_solid_torus():
    """SPEC S:233's construction: 16^3, distance to an axis-aligned circle (radius 5).
    The sublevel sets of f = +distance are solid tori around the circle (reading Z18:
    SPEC writes -distance, whose sublevel sets are the torus' complement and carry the
    box's corners as extra loops), so D1 has exactly one pair: the torus' 1-cycle, born
    when the circle closes and killed when the tube fills the central hole, with
    persistence ~ the hole radius (> 0.3 x the value range here); its generator winds
    around the circle's axis."""
    n = 16
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64)] * 3, indexing="ij")
    c, R = 7.5, 5.0
    rho = np.sqrt((x - c) ** 2 + (y - c) ** 2)
    dist = np.sqrt((rho - R) ** 2 + (z - c) ** 2)
    f = dist.astype(np.float32)
    res = oracle.run(f, want_d1=True)
    rng_ = float(f.max() - f.min())
    assert len(res.d1) == 1
    pers = float(res.d1["death_value"][0] - res.d1["birth_value"][0])
    assert pers > 0.3 * rng_
    g_ids = res.gen[res.gen_off[0]:res.gen_off[1]]
    verts = set()
    for e in _edge_sets(f.shape, g_ids):
        verts |= set(e)
    quad = set()  # the cycle visits all four quadrants around the axis
    for v in verts:
        vx, vy = v % n, (v // n) % n
        quad.add((vx > c, vy > c))
    assert len(quad) == 4


# ------------------------------------------------------------------ O6' "ignore" boundary mode

def _vals(pairs):
    return sorted((float(p["birth_value"]), float(p["death_value"])) for p in pairs)


def test_ignore_mode_hand_fields():
    g = golden("ignore_mode.json")
    f = np.array(g["1d"]["field"], np.float32)
    assert _vals(oracle.run(f).dtop_ignore) == [tuple(x) for x in g["1d"]["dtop_ignore"]]
    for d in (2, 3):
        assert _vals(oracle.run(sqdist_field((5,) * d, -1)).dtop_ignore) == g["neg_paraboloid"][str(d)]
        assert _vals(oracle.run(sqdist_field((5,) * d, +1)).dtop_ignore) == g["bowl"][str(d)]


@pytest.mark.parametrize("shape", [(40,), (9, 11), (12, 7), (5, 6, 7), (6, 6, 6)])
@pytest.mark.parametrize("seed", range(4))
def test_ignore_mode_low_moat(shape, seed):
    """Boundary vertices below every interior value: every arc of an interior saddle is
    processed before any boundary arc, so the interior classes have all merged into the
    global maximum's when the first boundary saddle joins it to the virtual maximum --
    the exact diagram's only pair involving the virtual maximum is the global maximum's,
    and the ignore mode must be the exact diagram minus exactly that pair (simplex
    level), by the elder rule alone."""
    rng = np.random.default_rng(seed)
    f = rng.random(shape).astype(np.float32) + 1.0
    core = tuple(slice(1, n - 1) for n in shape)
    low = np.full(shape, True)
    low[core] = False
    f[low] = -rng.random(int(low.sum())).astype(np.float32)
    res = oracle.run(f)
    d = f.ndim
    exact = [p for p in res.dtop if p["death_id"] >= 0]
    gmax = int(np.argmax(f))
    top = [p for p in exact if int(p["death_vertex"]) == gmax]
    assert len(top) == 1
    rest = sorted(p.tobytes() for p in exact if int(p["death_vertex"]) != gmax)
    assert sorted(p.tobytes() for p in res.dtop_ignore) == rest


def app_a_windows():
    """App. A (PAPER.md 2927-2949) on a synthetic terrain: four Gaussian hills on a dome
    that falls towards the edges, cut by square windows at different offsets and quarter
    turns (exact on the grid).  The hills and their saddles are inside every window."""
    n = 96
    y, x = np.meshgrid(np.arange(n, dtype=np.float64), np.arange(n, dtype=np.float64), indexing="ij")
    F = -((x - 48.0) ** 2 + (y - 48.0) ** 2) / 4000.0
    for (cx, cy, a) in [(36, 38, 2.0), (60, 36, 1.6), (38, 60, 1.3), (61, 61, 1.1)]:
        F += a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * 5.0 ** 2))
    F = F.astype(np.float32)
    out = []
    for (ox, oy, k) in [(16, 16, 0), (8, 12, 0), (14, 6, 1), (10, 10, 2), (6, 16, 3), (12, 14, 1)]:
        out.append(np.ascontiguousarray(np.rot90(F[oy:oy + 64, ox:ox + 64], k)))
    return out


def test_app_a_ignore_mode_is_stable_under_boundary_cuts():
    """Ignore mode: the same diagram (values) for every cut -- the W2 distance of App. A
    is zero throughout; exact mode: the global maximum's pair follows the cut."""
    ign, ex = [], []
    for w in app_a_windows():
        r = oracle.run(w, want_pairs=False)
        ign.append(_vals(r.dtop_ignore))
        ex.append(_vals(r.dtop))
    assert all(v == ign[0] for v in ign) and len(ign[0]) == 3
    assert len(set(tuple(v) for v in ex)) > 1

"""Brute-force persistence machinery in pure Python, used only to PIN the oracle.

Written independently of ``oracle/dms_oracle.c`` (no shared code, tables or ids): the
complex is built from the textbook Freudenthal/Kuhn definition, the filtration from
the paper's lexicographic order, and the diagrams from the standard boundary-matrix
column reduction (Alg. 1 "PairSimplices" is its geometric reading) and
from Kruskal over all edges.  Tiny grids only.
"""
from __future__ import annotations

import itertools

import numpy as np


def grid_shape_xfirst(shape):
    """numpy shape [.., Ly, Lx] -> (Lx, Ly, Lz) padded with 1."""
    L = list(reversed(shape)) + [1, 1, 1]
    return L[0], L[1], L[2]


def vertex_id(c, L):
    return c[0] + L[0] * (c[1] + L[1] * c[2])


def freudenthal(shape):
    """All simplices of the Freudenthal triangulation of a grid.

    Each d-cube with minimum corner a is split into the d! simplices
    a, a+e_p1, a+e_p1+e_p2, ..., a+(1,..,1) (one per permutation p); the complex is
    every face of those.  Returns {dim: set(frozenset(vertex ids))}."""
    d = len(shape)
    L = grid_shape_xfirst(shape)
    cx = {k: set() for k in range(d + 1)}
    ranges = [range(L[i] - 1) for i in range(d)]
    for a in itertools.product(*ranges):
        for p in itertools.permutations(range(d)):
            c = list(a) + [0] * (3 - d)
            chain = [vertex_id(c, L)]
            for ax in p:
                c[ax] += 1
                chain.append(vertex_id(c, L))
            for k in range(d + 1):
                for sub in itertools.combinations(chain, k + 1):
                    cx[k].add(frozenset(sub))
    if d == 0:
        pass
    # isolated vertices never happen for extents >= 2
    return cx


# the even cube's five tetrahedra written out by hand (local corner coordinates); the
# central one spans the corners of even coordinate sum
_EVEN_CUBE_TETS = [
    [(0, 0, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1)],
    [(1, 0, 0), (0, 0, 0), (1, 1, 0), (1, 0, 1)],
    [(0, 1, 0), (0, 0, 0), (1, 1, 0), (0, 1, 1)],
    [(0, 0, 1), (0, 0, 0), (1, 0, 1), (0, 1, 1)],
    [(1, 1, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1)],
]


def five_tet(shape):
    """The five-tetrahedra subdivision of a 3D grid: cubes whose minimum
    corner has an even coordinate sum are cut as _EVEN_CUBE_TETS, the others as its
    mirror image x -> 1 - x, so neighbouring cubes cut their common face along the same
    diagonal.  Returns {dim: set(frozenset(vertex ids))}."""
    assert len(shape) == 3
    L = grid_shape_xfirst(shape)
    cx = {k: set() for k in range(4)}
    for a in itertools.product(*[range(L[i] - 1) for i in range(3)]):
        odd = sum(a) % 2 == 1
        for tet in _EVEN_CUBE_TETS:
            vs = []
            for (x, y, z) in tet:
                if odd:
                    x = 1 - x
                vs.append(vertex_id((a[0] + x, a[1] + y, a[2] + z), L))
            for k in range(4):
                for sub in itertools.combinations(vs, k + 1):
                    cx[k].add(frozenset(sub))
    return cx


def complex_of(shape, complex="freudenthal"):
    return five_tet(shape) if complex == "5tet" else freudenthal(shape)


def ranks(f):
    """rank(v) = #{u : (f(u), u) < (f(v), v)} -- P:1368-1372 with the index tie-break."""
    flat = [float(x) for x in np.asarray(f, dtype=np.float32).ravel()]
    order = sorted(range(len(flat)), key=lambda v: (flat[v], v))
    r = [0] * len(flat)
    for i, v in enumerate(order):
        r[v] = i
    return r


def lexkey(s, r):
    """Decreasing tuple of vertex ranks; tuple comparison makes a face
    (a prefix) smaller than its coface."""
    return tuple(sorted((r[v] for v in s), reverse=True))


def maxvertex(s, r):
    return max(s, key=lambda v: r[v])


def filtration(cx, r):
    allsimp = [s for k in cx for s in cx[k]]
    allsimp.sort(key=lambda s: lexkey(s, r))
    return allsimp


def reduce_all(cx, r):
    """Standard column reduction of the boundary matrix over Z/2 in filtration order.

    Returns (pairs, unpaired): pairs = list of (birth simplex, death simplex)."""
    filt = filtration(cx, r)
    pos = {s: i for i, s in enumerate(filt)}
    low_owner = {}
    pairs = []
    paired = set()
    for j, s in enumerate(filt):
        if len(s) == 1:
            continue
        col = set(pos[s - {v}] for v in s)
        while col:
            low = max(col)
            if low in low_owner:
                col ^= low_owner[low]
            else:
                low_owner[low] = col
                pairs.append((filt[low], s))
                paired.add(low)
                paired.add(j)
                break
    unpaired = [filt[i] for i in range(len(filt)) if i not in paired]
    return pairs, unpaired


def diagrams_by_reduction(f, complex="freudenthal"):
    """{p: [(birth simplex, death simplex)]} with zero-persistence pairs removed
    (same highest vertex, reading Z8), plus infinite births."""
    cx = complex_of(f.shape, complex)
    r = ranks(f)
    pairs, unpaired = reduce_all(cx, r)
    out = {}
    for b, dth in pairs:
        if maxvertex(b, r) == maxvertex(dth, r):
            continue
        out.setdefault(len(b) - 1, []).append((b, dth))
    return out, unpaired, r


def kruskal_d0(f, complex="freudenthal"):
    """D0 by Kruskal over ALL edges in lexicographic order, Elder rule, dropping the
    pairs whose dying vertex is the edge's own highest vertex (zero persistence)."""
    cx = complex_of(f.shape, complex)
    r = ranks(f)
    n = len(r)
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    out = []
    for e in sorted(cx[1], key=lambda s: lexkey(s, r)):
        a, b = (find(v) for v in e)
        if a == b:
            continue
        young, old = (a, b) if r[a] > r[b] else (b, a)
        if young != maxvertex(e, r):
            out.append((young, e))
        parent[young] = old
    return out, r


# ------------------------------------------------------------------ GF(2) homology

def gf2_rank(rows):
    """rank of a list of int bit-rows over Z/2"""
    rows = [x for x in rows if x]
    rank = 0
    while rows:
        piv = rows.pop()
        if not piv:
            continue
        rank += 1
        hb = piv.bit_length() - 1
        rows = [x ^ piv if (x >> hb) & 1 else x for x in rows]
        rows = [x for x in rows if x]
    return rank


def reduced_betti(simplices):
    """Reduced Betti numbers beta~_{-1..2} of a simplicial complex over Z/2, given as
    an iterable of frozensets closed under faces (the empty simplex implicit)."""
    bydim = {}
    for s in simplices:
        bydim.setdefault(len(s) - 1, []).append(s)
    res = {}
    if not bydim:
        return {-1: 1, 0: 0, 1: 0, 2: 0}
    idx = {k: {s: i for i, s in enumerate(v)} for k, v in bydim.items()}

    def boundary_rank(k):
        # rank of d_k : C_k -> C_{k-1}; d_0 is the augmentation (rank 1 if any vertex)
        if k == 0:
            return 1 if bydim.get(0) else 0
        if k not in bydim:
            return 0
        rows = []
        for s in bydim[k]:
            bits = 0
            for v in s:
                bits |= 1 << idx[k - 1][s - {v}]
            rows.append(bits)
        return gf2_rank(rows)

    res[-1] = 0
    for k in range(0, 3):
        nk = len(bydim.get(k, []))
        res[k] = nk - boundary_rank(k) - boundary_rank(k + 1)
    return res


def lower_link(cx, x, r):
    """Lk^-(x): faces sigma - {x} of the lower-star simplices sigma != {x}."""
    out = []
    for k in cx:
        for s in cx[k]:
            if x in s and len(s) > 1 and all(r[u] < r[x] for u in s if u != x):
                out.append(s - {x})
    return out


def lower_star(cx, x, r):
    return [s for k in cx for s in cx[k] if x in s and all(r[u] <= r[x] for u in s)]

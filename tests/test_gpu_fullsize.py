"""GPU parity at BASELINE.json's full sizes, in the configuration bench.py times.

At these sizes the oracle cannot run the whole front end in test time, so the checks
are (a) exact oracle parity on sampled lower stars (gradient vectors and critical
cells of every sampled vertex, the oracle computing each star one by one) and (b)
properties that hold at any size and pin the global outputs: the vertex order is a
permutation sorted by (f, index); C_k are lexicographically sorted and satisfy the Euler
identity; every extremum is born/killed exactly once; the 2D/1D duality identities;
pair values are f at the highest vertices.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from synth import fields

pytestmark = pytest.mark.gpu

CFGS = ["c3", "c4", "c5a", "c5b"]
NCPU = os.cpu_count() or 1

# anchored-id chain convention (Z13), written out for the checks
def _chains(ndim, k):
    full = (1 << ndim) - 1
    out = []

    def rec(prev, cur):
        if len(cur) == k:
            out.append(tuple(cur))
            return
        for m in range(1, full + 1):
            if (m & prev) == prev and m != prev:
                rec(m, cur + [m])

    rec(0, [])
    out.sort(key=lambda c: tuple(reversed(c)))
    return out


def simplex_vertices(shape, dim, ids):
    """vectorised: anchored ids -> (n, dim+1) vertex ids"""
    nd = len(shape)
    L = list(reversed(shape)) + [1, 1]
    if dim == 0:
        return ids.reshape(-1, 1)
    ch = _chains(nd, dim)
    per = len(ch)
    a = ids // per
    kk = ids % per
    tab = np.array([[0] + [m for m in c] for c in ch], dtype=np.int64)  # (per, dim+1) masks
    masks = tab[kk]  # (n, dim+1)
    off = (masks & 1) + L[0] * ((masks >> 1) & 1) + L[0] * L[1] * ((masks >> 2) & 1)
    return a[:, None] + off


def kmax(f, verts):
    """index of the K-highest vertex per row (value, then index)"""
    best = verts[:, 0].copy()
    for j in range(1, verts.shape[1]):
        v = verts[:, j]
        up = (f[v] > f[best]) | ((f[v] == f[best]) & (v > best))
        best = np.where(up, v, best)
    return best


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    return torch, dms


@pytest.mark.parametrize("cfg", CFGS)
def test_full_size(env, cfg):
    torch, dms = env
    f3 = fields.make(cfg, seed=int(os.environ.get("DMS_FULLSIZE_SEED", "0")))
    shape = f3.shape
    d = f3.ndim
    f = f3.ravel()
    N = f.size
    fd = torch.from_numpy(f3).cuda()
    ctx = dms.DMS(fd)
    rank = torch.empty(N, dtype=torch.int32, device="cuda")
    grad = torch.empty(dms.dms_gradient_bytes(ctx.ctx), dtype=torch.uint8, device="cuda")
    ctx.run_all(rank, grad)
    crit = [c.cpu().numpy() for c in ctx.critical()]
    d0 = ctx.diagram0()
    dt = ctx.diagram_top()
    un0 = ctx.unpaired_saddles(0)
    unt = ctx.unpaired_saddles(1)

    # ---- vertex order: a permutation sorted by (f, index)
    perm = torch.empty(N, dtype=torch.int64, device="cuda")
    perm[rank.long()] = torch.arange(N, device="cuda")
    assert int(torch.unique(rank).numel()) == N
    fp = fd.reshape(-1)[perm]
    inc = (fp[1:] > fp[:-1]) | ((fp[1:] == fp[:-1]) & (perm[1:] > perm[:-1]))
    assert bool(inc.all()), "rank is not the (value, index) order"
    rank_h = rank.cpu().numpy()
    del perm, fp, inc

    # ---- gradient + critical cells on sampled lower stars, exact oracle parity
    rng = np.random.default_rng(12345)
    sample = np.unique(np.concatenate([
        rng.integers(0, N, 20000),
        np.arange(0, min(N, 2048)),               # the first rows / boundary
        np.arange(max(0, N - 2048), N),
    ])).astype(np.int64)
    wb = {3: 16, 2: 2, 1: 1}[d]
    gw = grad.reshape(N, wb)[torch.from_numpy(sample).cuda()].cpu().numpy()
    got_pairs = []
    for i, v in enumerate(sample):
        got_pairs.append(dms.dms_decode_pairs(shape, gw[i], int(v), int(v) + 1))
    got_pairs = np.concatenate(got_pairs)
    got_pairs = got_pairs[np.lexsort((got_pairs[:, 2], got_pairs[:, 1], got_pairs[:, 0]))]
    ref = oracle.gradient_sample(f3, sample, nthreads=NCPU)
    assert np.array_equal(got_pairs, ref.pairs), "gradient vectors on the sampled lower stars"
    for k in range(d + 1):
        mv = kmax(f, simplex_vertices(shape, k, crit[k]))
        mine = np.sort(crit[k][np.isin(mv, sample)])
        assert np.array_equal(mine, ref.crit[k]), ("critical cells of the sampled stars", k)

    # ---- C_k: lexicographic order (Alg. 2 l. 13) and Euler identity
    for k in range(d + 1):
        vs = simplex_vertices(shape, k, crit[k])
        r = -np.sort(-rank_h[vs], axis=1)  # descending rank tuples
        a, b = r[:-1], r[1:]
        lt = np.zeros(len(a), bool)
        eq = np.ones(len(a), bool)
        for j in range(k + 1):
            lt |= eq & (a[:, j] < b[:, j])
            eq &= a[:, j] == b[:, j]
        assert lt.all(), ("C_%d not strictly increasing in lex order" % k)
    assert sum((-1) ** k * len(crit[k]) for k in range(d + 1)) == 1

    # ---- D0: every minimum but the global one dies exactly once
    fin = d0[d0["death_id"] >= 0]
    inf = d0[d0["death_id"] < 0]
    assert len(inf) == 1 and inf[0]["birth_id"] == crit[0][0]
    assert np.array_equal(np.sort(fin["birth_id"]), np.sort(crit[0][1:]))
    assert np.isin(fin["death_id"], crit[1]).all()
    sorter = np.argsort(crit[1], kind="stable")  # crit[1] is in lex order, not id order
    idx = sorter[np.searchsorted(crit[1], fin["death_id"], sorter=sorter)]
    assert (np.diff(idx) > 0).all(), "D0 not in increasing death (lexicographic) order"
    assert len(un0) == len(crit[1]) - len(fin)
    assert (fin["death_value"] >= fin["birth_value"]).all()
    # values are f at the highest vertices
    assert (fin["birth_value"].view(np.uint32) == f[fin["birth_vertex"]].view(np.uint32)).all()
    assert (fin["death_value"].view(np.uint32) == f[fin["death_vertex"]].view(np.uint32)).all()
    assert np.array_equal(fin["death_vertex"], kmax(f, simplex_vertices(shape, 1, fin["death_id"])))
    fstar_v = int(np.nonzero(f == f.max())[0][-1])  # the K-highest vertex: max value, then max index
    assert inf[0]["death_value"].view(np.uint32) == f[fstar_v].view(np.uint32)

    # ---- D_{d-1}
    tfin = dt[dt["death_id"] >= 0]
    if d >= 2:
        assert len(dt) == len(crit[d])  # exact mode: every maximum dies exactly once
        assert np.array_equal(np.sort(tfin["death_id"]), np.sort(crit[d]))
    assert np.isin(tfin["birth_id"], crit[d - 1]).all()
    assert (tfin["birth_value"].view(np.uint32) == f[tfin["birth_vertex"]].view(np.uint32)).all()
    assert (tfin["death_value"].view(np.uint32) == f[tfin["death_vertex"]].view(np.uint32)).all()
    assert np.array_equal(tfin["birth_vertex"], kmax(f, simplex_vertices(shape, d - 1, tfin["birth_id"])))
    assert len(unt) == len(crit[d - 1]) - len(tfin)
    if d == 2:  # C_1 = D0 death edges + D1 birth edges (the saddles D_{d-1} left unpaired)
        assert np.array_equal(np.sort(unt), np.sort(fin["death_id"]))
    if d == 3:
        assert len(crit[1]) - len(fin) == len(crit[2]) - len(tfin)
    if d == 1:  # duality: D_{d-1} = D0
        a = np.sort(fin[["birth_vertex", "death_vertex"]].astype([("a", "<i4"), ("b", "<i4")]), order=["a", "b"])
        b = np.sort(tfin[["birth_vertex", "death_vertex"]].astype([("a", "<i4"), ("b", "<i4")]), order=["a", "b"])
        assert np.array_equal(a, b)
    ctx.close()

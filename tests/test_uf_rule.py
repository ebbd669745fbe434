"""CPU model of the parallel union-find rounds of diag.cuh (mutual-minimum contraction
plus "a younger root dies at its lightest arc"), checked against the sequential
elder-rule union-find (PAPER.md 2675-2685) on random, path (1D random walk) and
giant-basin graphs, including self-loops and parallel arcs."""
from __future__ import annotations

import numpy as np
import pytest


def sequential(n, arcs, older_is_smaller=True):
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            a = parent[a]
        return a

    out = []
    for a, b in arcs:
        ra, rb = find(a), find(b)
        if ra == rb:
            out.append(-1)
            continue
        a_older = ra < rb if older_is_smaller else ra > rb
        young, old = (rb, ra) if a_older else (ra, rb)
        parent[young] = old
        out.append(young)
    return out


def rounds(n, arcs, older_is_smaller=True, max_rounds=100000, batch=0):
    """batch > 0: the arcs (listed in processing order) are revealed in key-ordered
    batches whenever at most batch // 4 are live (diag.cuh UFArgs::batch)."""
    m = len(arcs)
    parent = list(range(n))
    out = [-2] * m
    live = [] if batch else list(range(m))
    rv = 0 if batch else m

    def find(a):
        while parent[a] != a:
            a = parent[a]
        return a

    nrounds = 0
    while (live or rv < m) and nrounds < max_rounds:
        nrounds += 1
        if rv < m and len(live) <= batch // 4:
            add = min(batch, m - rv)
            live = live + list(range(rv, rv + add))
            rv += add
        best = {}
        ra, rb = {}, {}
        for i in live:
            a, b = find(arcs[i][0]), find(arcs[i][1])
            ra[i], rb[i] = a, b
            if a == b:
                out[i] = -1
                continue
            best[a] = min(best.get(a, m), i)
            best[b] = min(best.get(b, m), i)
        hooks = []
        for i in live:
            if out[i] != -2:
                continue
            a, b = ra[i], rb[i]
            ma, mb = best[a] == i, best[b] == i
            a_older = a < b if older_is_smaller else a > b
            if ma and mb:
                young, old = (b, a) if a_older else (a, b)
                hooks.append((young, old))
                out[i] = young
            elif ma and not a_older:
                hooks.append((a, b))
                out[i] = a
            elif mb and a_older:
                hooks.append((b, a))
                out[i] = b
        hooked = set()
        for y, o in hooks:
            assert y not in hooked  # a root hooks at most once per round
            hooked.add(y)
            parent[y] = o
        live = [i for i in live if out[i] == -2]
    return out, nrounds


def random_graph(rng, n, m):
    return [tuple(int(x) for x in rng.integers(0, n, 2)) for _ in range(m)]


def path_graph(rng, n):
    # 1D random walk: minima alternate with maxima; arcs join neighbouring minima,
    # keys = order of the separating maxima (a random-walk sequence)
    walk = np.cumsum(rng.standard_normal(n))
    order = np.argsort(walk[: n - 1], kind="stable")
    return [(int(i), int(i) + 1) for i in order]


def giant_basin(rng, n):
    # node 0 the oldest; every other node hangs off it or off a random earlier node,
    # with keys increasing outwards (sequential absorption by the big component)
    arcs = []
    for v in range(1, n):
        u = 0 if rng.random() < 0.6 else int(rng.integers(0, v))
        arcs.append((v, u))
    perm = rng.permutation(len(arcs))
    extra = random_graph(rng, n, n // 4)
    return [arcs[i] for i in perm] + extra


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("older_is_smaller", [True, False])
def test_rounds_equal_sequential(seed, older_is_smaller):
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 0:
        n = int(rng.integers(2, 60))
        arcs = random_graph(rng, n, int(rng.integers(1, 3 * n)))
    elif kind == 1:
        n = int(rng.integers(3, 300))
        arcs = path_graph(rng, n)
    elif kind == 2:
        n = int(rng.integers(2, 300))
        arcs = giant_basin(rng, n)
    else:
        n = int(rng.integers(2, 10))  # heavy self-loops / parallel arcs
        arcs = random_graph(rng, n, int(rng.integers(1, 40)))
    got, _ = rounds(n, arcs, older_is_smaller)
    assert got == sequential(n, arcs, older_is_smaller)


def test_round_counts_are_small():
    rng = np.random.default_rng(7)
    _, r1 = rounds(3000, path_graph(rng, 3000))
    _, r2 = rounds(3000, giant_basin(rng, 3000))
    assert r1 < 200 and r2 < 60, (r1, r2)


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("batch", [1, 4, 9, 64])
def test_batched_rounds_equal_sequential(seed, batch):
    """Revealing the arcs in key-ordered batches (dense graphs, diag.cuh) keeps every
    decision of the sequential elder-rule union-find."""
    rng = np.random.default_rng(1000 + seed)
    kind = seed % 3
    if kind == 0:
        n = int(rng.integers(2, 80))
        arcs = random_graph(rng, n, int(rng.integers(1, 5 * n)))
    elif kind == 1:
        n = int(rng.integers(3, 200))
        arcs = path_graph(rng, n)
    else:
        n = int(rng.integers(2, 200))
        arcs = giant_basin(rng, n)
    older = bool(seed % 2)
    got, _ = rounds(n, arcs, older, batch=batch)
    assert got == sequential(n, arcs, older)

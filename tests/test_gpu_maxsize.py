"""GPU: the largest admissible 3D field (704^3: 6 N top cells = 2.09e9 < 2^31, the int32
indexing limit of dms.h) runs through the whole front end, and the outputs satisfy the
size-independent identities (the order is a sorted permutation, Euler characteristic,
every extremum born / killed exactly once, |C_1| - |D0| = |C_2| - |D2|)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_largest_admissible_field():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    n = 704
    g = torch.Generator(device="cuda").manual_seed(5)
    fd = torch.rand((n, n, n), generator=g, device="cuda", dtype=torch.float32)  # iid: dense criticals
    N = fd.numel()
    d = dms.DMS(fd)
    rank = torch.empty(N, dtype=torch.int32, device="cuda")
    d.run_all(rank)
    crit = d.critical()
    counts = [int(c.numel()) for c in crit]
    assert counts[0] - counts[1] + counts[2] - counts[3] == 1  # Euler, a ball
    d0 = d.diagram0()
    dt = d.diagram_top()
    assert int((d0["death_id"] < 0).sum()) == 1 and len(d0) == counts[0]
    assert len(dt) == counts[3]
    assert counts[1] - (len(d0) - 1) == counts[2] - len(dt)
    # the order: a permutation, sorted by (f, index)
    perm = torch.empty(N, dtype=torch.int64, device="cuda")
    perm[rank.long()] = torch.arange(N, device="cuda")
    assert int(torch.unique(rank).numel()) == N
    fp = fd.reshape(-1)[perm]
    assert bool(((fp[1:] > fp[:-1]) | ((fp[1:] == fp[:-1]) & (perm[1:] > perm[:-1]))).all())
    d.close()

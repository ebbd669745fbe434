"""GPU: randomized parity sweep -- random shapes (1D-3D, odd extents, thin slabs), value
distributions with heavy ties, signed zeros and infinities, checked bit-exactly against
the oracle through the full front end (seeded, reproducible)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from synth import fields

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    return torch, dms


def random_field(rng):
    d = int(rng.integers(1, 4))
    if d == 1:
        shape = (int(rng.integers(2, 5000)),)
    elif d == 2:
        shape = tuple(int(x) for x in rng.integers(2, 90, 2))
    else:
        shape = tuple(int(x) for x in rng.integers(2, 26, 3))
    kind = int(rng.integers(0, 5))
    f = fields.uniform(shape, seed=int(rng.integers(1 << 30)))
    if kind == 1:  # few distinct values: the index tie-break decides most comparisons
        f = np.floor(f * int(rng.integers(2, 6))).astype(np.float32)
    elif kind == 2:  # signed zeros and infinities
        f = np.where(f < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
        f[rng.random(shape) < 0.2] = np.inf
        f[rng.random(shape) < 0.2] = -np.inf
    elif kind == 3:  # smooth (long paths) + tiny noise
        idx = np.indices(shape).astype(np.float64)
        g = sum(np.sin(idx[i] * rng.uniform(0.05, 0.4) + rng.uniform(0, 6)) for i in range(d))
        f = (g + 1e-3 * rng.standard_normal(shape)).astype(np.float32)
    elif kind == 4:  # monotone ramp with plateaus
        f = np.floor(np.indices(shape).sum(0) / 3.0).astype(np.float32)
    return np.ascontiguousarray(f)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("DMS_SWEEP_N", "150"))))
def test_random_fields(env, seed):
    torch, dms = env
    rng = np.random.default_rng(777 + int(__import__("os").environ.get("DMS_SWEEP_OFF", "0")) + seed)
    f = random_field(rng)
    ref = oracle.run(f)
    d = dms.DMS(torch.from_numpy(f).cuda())
    rank = torch.empty(f.size, dtype=torch.int32, device="cuda")
    grad = torch.empty(dms.dms_gradient_bytes(d.ctx), dtype=torch.uint8, device="cuda")
    d.run_all(rank, grad)
    assert np.array_equal(rank.cpu().numpy(), oracle.ranks(f)), (f.shape, "ranks")
    pairs = dms.dms_decode_pairs(f.shape, grad.cpu().numpy(), 0, f.size)
    pairs = pairs[np.lexsort((pairs[:, 2], pairs[:, 1], pairs[:, 0]))]
    assert np.array_equal(pairs, ref.pairs), (f.shape, "gradient")
    crit = d.critical()
    for k in range(f.ndim + 1):
        assert np.array_equal(crit[k].cpu().numpy(), ref.crit[k]), (f.shape, "C", k)
    assert d.diagram0().tobytes() == ref.d0.tobytes(), (f.shape, "D0")
    assert d.diagram_top().tobytes() == ref.dtop.tobytes(), (f.shape, "Dtop")
    assert np.array_equal(d.unpaired_saddles(0), ref.unpaired0), (f.shape, "un0")
    assert np.array_equal(d.unpaired_saddles(1), ref.unpaired_top), (f.shape, "untop")
    d.close()

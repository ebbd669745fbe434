"""GPU parity on the five-tetrahedra complex (reading Z21):
the CUDA path (``dms_create2(..., DMS_COMPLEX_5TET)``, ``tet5.cuh``) against the oracle's
five-tetrahedra run, bit-exact (tolerance 0) -- ranks, every gradient vector, C_0..C_3,
D0, D2 (exact and ignore mode) and the unpaired saddle lists."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from synth import fields

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1
C = "5tet"


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    return torch, dms


def gpu_run(env, f, run_all=False):
    torch, dms = env
    d = dms.DMS(torch.from_numpy(np.ascontiguousarray(f)).cuda(), complex=C)
    if run_all:
        rank = torch.empty(f.size, dtype=torch.int32, device="cuda")
        grad = torch.empty(dms.dms_gradient_bytes(d.ctx), dtype=torch.uint8, device="cuda")
        d.run_all(rank, grad)
    else:
        rank = d.order()
        grad = d.gradient()
    out = dict(
        rank=rank.cpu().numpy(),
        grad=grad.cpu().numpy(),
        crit=[c.cpu().numpy() for c in d.critical()],
        d0=d.diagram0(),
        dtop=d.diagram_top(),
        dtop_ign=d.diagram_top(mode=1),
        un0=d.unpaired_saddles(0),
        untop=d.unpaired_saddles(1),
        launches=d.launch_count(),
    )
    d.close()
    return out


def compare_full(env, f, nthreads=NCPU, run_all=False):
    _, dms = env
    ref = oracle.run(f, nthreads=nthreads, complex=C)
    got = gpu_run(env, f, run_all)
    assert np.array_equal(got["rank"], oracle.ranks(f)), "ranks"
    pairs = dms.dms_decode_pairs(f.shape, got["grad"].view(np.uint8), 0, f.size, complex=C)
    pairs = pairs[np.lexsort((pairs[:, 2], pairs[:, 1], pairs[:, 0]))]
    assert np.array_equal(pairs, ref.pairs), "gradient pairs"
    for k in range(4):
        assert np.array_equal(got["crit"][k], ref.crit[k]), ("C_%d" % k)
    assert got["d0"].tobytes() == ref.d0.tobytes(), "D0"
    assert got["dtop"].tobytes() == ref.dtop.tobytes(), "D2"
    assert got["dtop_ign"].tobytes() == ref.dtop_ignore.tobytes(), "D2 ignore mode"
    assert np.array_equal(got["un0"], ref.unpaired0), "unpaired after D0"
    assert np.array_equal(got["untop"], ref.unpaired_top), "unpaired after D2"
    assert got["launches"] > 0
    return ref, got


SHAPES = [(2, 2, 2), (2, 3, 5), (3, 3, 3), (5, 2, 4), (9, 10, 11), (16, 16, 16), (7, 33, 20), (33, 17, 5)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["uniform", "ties", "signed_zero"])
def test_small_grids(env, shape, kind):
    rng = np.random.default_rng(hash((shape, kind, C)) % (2**32))
    f = fields.uniform(shape, seed=int(rng.integers(1 << 30)))
    if kind == "ties":
        f = np.floor(f * 5).astype(np.float32)
    if kind == "signed_zero":
        f = np.where(f < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
        f[rng.random(shape) < 0.1] = np.inf
        f[rng.random(shape) < 0.1] = -np.inf
    compare_full(env, f)


def test_constant_elevation_bowl(env):
    shape = (6, 7, 8)
    idx = np.indices(shape)
    for f in [np.zeros(shape, np.float32), idx.sum(0).astype(np.float32), -idx.sum(0).astype(np.float32),
              sum((c - s / 2.0) ** 2 for c, s in zip(idx, shape)).astype(np.float32),
              (-sum((c - s / 2.0) ** 2 for c, s in zip(idx, shape))).astype(np.float32)]:
        ref, got = compare_full(env, f)
        assert sum((-1) ** k * len(got["crit"][k]) for k in range(4)) == 1


@pytest.mark.parametrize("cfg,shape", [("c1", (20, 24, 28)), ("c2", (48, 48, 48)), ("c3", (40, 41, 42)),
                                       ("c4", (40, 48, 56))])
def test_config_recipes(env, cfg, shape):
    compare_full(env, fields.make(cfg, seed=11, shape=shape))


def test_run_all_matches_stepwise(env):
    compare_full(env, fields.make("c4", seed=5, shape=(33, 40, 47)), run_all=True)


def test_run_all_host(env):
    """dms_run_all_host (slab-pipelined upload, the gradient launched per slab) on the
    five-tetrahedra complex equals the oracle."""
    torch, dms = env
    f = fields.make("c4", seed=6, shape=(40, 33, 29))
    ref = oracle.run(f, nthreads=NCPU, complex=C)
    d = dms.DMS(torch.zeros(f.shape, dtype=torch.float32, device="cuda"), complex=C)
    d.run_all_host(torch.from_numpy(f).pin_memory())
    for k in range(4):
        assert np.array_equal(d.critical()[k].cpu().numpy(), ref.crit[k])
    assert d.diagram0().tobytes() == ref.d0.tobytes()
    assert d.diagram_top().tobytes() == ref.dtop.tobytes()
    d.close()


def test_midsize_value_noise(env):
    """2.1 M vertices (128^3, the c4 recipe): many CTAs, long dual paths, the union-find's
    multi-round paths -- every output against the oracle."""
    compare_full(env, fields.make("c4", seed=3, shape=(128, 128, 128)))


def test_midsize_iid(env):
    compare_full(env, fields.make("c3", seed=4, shape=(96, 100, 104)))


def test_unsupported_calls(env):
    torch, dms = env
    with pytest.raises(dms.DMSError) as e:  # the five-tetrahedra complex is 3D only
        dms.DMS(torch.zeros((8, 8), dtype=torch.float32, device="cuda"), complex=C)
    assert e.value.code == 1
    d = dms.DMS(torch.rand((6, 6, 6), device="cuda"), complex=C)
    d.run_all()
    with pytest.raises(dms.DMSError) as e:  # D1 on this complex: the oracle only
        d.diagram1()
    assert e.value.code == 5
    d.close()

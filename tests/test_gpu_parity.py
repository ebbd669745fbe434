"""GPU parity: the CUDA path through the C ABI against the CPU oracle, bit-exact
(tolerance 0: every output is integer / index data or a copied float value,
BASELINE.json north_star)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from synth import fields

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    return torch, dms


def gpu_run(env, f):
    torch, dms = env
    d = dms.DMS(torch.from_numpy(np.ascontiguousarray(f)).cuda())
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


def compare_full(env, f, nthreads=NCPU):
    _, dms = env
    ref = oracle.run(f, nthreads=nthreads)
    got = gpu_run(env, f)
    d = f.ndim
    assert np.array_equal(got["rank"], oracle.ranks(f)), "ranks"
    pairs = dms.dms_decode_pairs(f.shape, got["grad"], 0, f.size)
    pairs = pairs[np.lexsort((pairs[:, 2], pairs[:, 1], pairs[:, 0]))]
    assert np.array_equal(pairs, ref.pairs), "gradient pairs"
    for k in range(d + 1):
        assert np.array_equal(got["crit"][k], ref.crit[k]), ("C_%d" % k)
    assert got["d0"].tobytes() == ref.d0.tobytes(), "D0"
    assert got["dtop"].tobytes() == ref.dtop.tobytes(), "D_{d-1}"
    assert got["dtop_ign"].tobytes() == ref.dtop_ignore.tobytes(), "D_{d-1} ignore mode"
    assert np.array_equal(got["un0"], ref.unpaired0), "unpaired after D0"
    assert np.array_equal(got["untop"], ref.unpaired_top), "unpaired after D_{d-1}"
    assert got["launches"] > 0
    return ref, got


SHAPES = [
    (2, 2, 2), (2, 3, 5), (3, 3, 3), (9, 10, 11), (16, 16, 16), (7, 33, 20), (33, 17, 5),
    (2, 2), (2, 9), (37, 41), (64, 3), (100, 129),
    (2,), (3,), (1000,), (4099,),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["uniform", "ties", "signed_zero"])
def test_small_grids(env, shape, kind):
    rng = np.random.default_rng(hash((shape, kind)) % (2**32))
    f = fields.uniform(shape, seed=int(rng.integers(1 << 30)))
    if kind == "ties":
        f = np.floor(f * 5).astype(np.float32)  # the index tie-break decides
    if kind == "signed_zero":
        f = np.where(f < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)  # -0 == +0
        f[rng.random(shape) < 0.1] = np.inf
        f[rng.random(shape) < 0.1] = -np.inf
    compare_full(env, f)


@pytest.mark.parametrize("shape", [(6, 7, 8), (20, 21), (50,)])
def test_constant_elevation_bowl(env, shape):
    d = len(shape)
    for f in [np.zeros(shape, np.float32),
              np.indices(shape).sum(0).astype(np.float32),
              -np.indices(shape).sum(0).astype(np.float32),
              (sum((c - s / 2.0) ** 2 for c, s in zip(np.indices(shape), shape))).astype(np.float32),
              (-sum((c - s / 2.0) ** 2 for c, s in zip(np.indices(shape), shape))).astype(np.float32)]:
        ref, got = compare_full(env, f)
        inf = [p for p in got["d0"] if p["death_id"] < 0]
        assert len(inf) == 1
        assert sum((-1) ** k * len(got["crit"][k]) for k in range(d + 1)) == 1


@pytest.mark.parametrize("seed", range(6))
def test_seed_sweep_c1_recipe(env, seed):
    compare_full(env, fields.make("c1", seed=seed, shape=(20, 24, 28)))


def test_config_c1(env):
    compare_full(env, fields.make("c1"))


def test_config_c2(env):
    compare_full(env, fields.make("c2"))


def test_config_small_versions_of_c4_c5(env):
    compare_full(env, fields.make("c4", shape=(64, 64, 64)))
    compare_full(env, fields.make("c5a", shape=(512, 512)))
    compare_full(env, fields.make("c5b", shape=(1 << 16,)))


def test_nan_rejected(env):
    torch, dms = env
    f = np.zeros((4, 5, 6), np.float32)
    f[1, 2, 3] = np.nan
    d = dms.DMS(torch.from_numpy(f).cuda())
    with pytest.raises(dms.DMSError) as e:
        d.run_all()
        d.critical()
    assert e.value.name == "DMS_ERR_NAN"


@pytest.mark.parametrize("shape", [(6, 7, 8), (9, 11), (50,)])
def test_nan_then_clean_field_on_one_context(env, shape):
    """the NaN flag describes the current field only -- after DMS_ERR_NAN the
    same context, with a clean field written into the same device buffer, runs and
    matches the oracle (both through dms_run_all and through the stepwise calls)."""
    torch, dms = env
    rng = np.random.default_rng(11)
    clean = rng.random(shape).astype(np.float32)
    bad = clean.copy()
    bad.flat[bad.size // 2] = np.nan
    fd = torch.from_numpy(bad).cuda()
    d = dms.DMS(fd)
    with pytest.raises(dms.DMSError) as e:
        d.run_all()
        d.critical()
    assert e.value.name == "DMS_ERR_NAN"
    ref = oracle.run(clean, nthreads=NCPU)
    for stepwise in (False, True):
        fd.copy_(torch.from_numpy(bad))  # NaN again, then clean again
        with pytest.raises(dms.DMSError):
            d.run_all()
            d.critical()
        fd.copy_(torch.from_numpy(clean))
        if stepwise:
            rank = d.order()
            grad = d.gradient()  # (caller-owned: must stay alive while the context uses it)
        else:
            rank = torch.empty(clean.size, dtype=torch.int32, device="cuda")
            d.run_all(rank)
        assert np.array_equal(rank.cpu().numpy(), oracle.ranks(clean))
        for k in range(clean.ndim + 1):
            assert np.array_equal(d.critical()[k].cpu().numpy(), ref.crit[k])
        assert d.diagram0().tobytes() == ref.d0.tobytes()
        assert d.diagram_top().tobytes() == ref.dtop.tobytes()
    d.close()


def test_degenerate_and_bad_mode(env):
    torch, dms = env
    for shape in [(1, 4, 4), (4, 1), (1,)]:
        with pytest.raises(dms.DMSError) as e:
            dms.DMS(torch.zeros(shape, device="cuda"))
        assert e.value.name == "DMS_ERR_DEGENERATE"
    d = dms.DMS(torch.rand(5, 5, 5, device="cuda"))
    with pytest.raises(dms.DMSError) as e:
        d.diagram_top(mode=7)
    assert e.value.name == "DMS_ERR_ARG"


def test_deterministic_repeat(env):
    f = fields.make("c1", seed=9)
    a = gpu_run(env, f)
    b = gpu_run(env, f)
    for key in ("rank", "grad"):
        assert np.array_equal(a[key], b[key])
    assert a["d0"].tobytes() == b["d0"].tobytes() and a["dtop"].tobytes() == b["dtop"].tobytes()


@pytest.mark.parametrize("name,shape", [("c1", (32, 32, 32)), ("c1", (4, 5, 6)), ("c4", (40, 48, 64)),
                                        ("c5a", (300, 257)), ("c5b", (100003,)), ("c5b", (5,))])
def test_run_all_host_matches_device_input(env, name, shape):
    """dms_run_all_host (slab-pipelined upload from pinned host memory) gives exactly the
    results of dms_run_all on the same field already on the device, including fields
    with fewer planes than upload slabs; the device buffer starts with other values."""
    torch, dms = env
    f = np.ascontiguousarray(fields.make(name, seed=3, shape=shape))
    ref = gpu_run(env, f)
    dev = torch.full(f.shape, 7.0, dtype=torch.float32, device="cuda")
    d = dms.DMS(dev)
    rank = torch.empty(f.size, dtype=torch.int32, device="cuda")
    grad = torch.empty(dms.dms_gradient_bytes(d.ctx), dtype=torch.uint8, device="cuda")
    for _ in range(2):  # twice: the second upload overwrites a field the first run used
        d.run_all_host(torch.from_numpy(f).pin_memory(), rank, grad)
        assert np.array_equal(dev.cpu().numpy(), f)
        assert np.array_equal(rank.cpu().numpy(), ref["rank"])
        assert np.array_equal(grad.cpu().numpy(), ref["grad"])
        for k in range(f.ndim + 1):
            assert np.array_equal(d.critical()[k].cpu().numpy(), ref["crit"][k])
        assert d.diagram0().tobytes() == ref["d0"].tobytes()
        assert d.diagram_top().tobytes() == ref["dtop"].tobytes()
        assert np.array_equal(d.unpaired_saddles(0), ref["un0"])
        assert np.array_equal(d.unpaired_saddles(1), ref["untop"])
    d.close()


def test_chase_stamps_wrap_around(env):
    """The memoised D_{d-1} chases stamp cells with an 8-bit generation that wraps every
    255 runs (the stamps are then cleared): 260 runs of one context stay exact."""
    torch, dms = env
    for name, shape in [("c4", (24, 20, 18)), ("c5a", (60, 50))]:
        f = np.ascontiguousarray(fields.make(name, seed=11, shape=shape))
        ref = oracle.run(f)
        d = dms.DMS(torch.from_numpy(f).cuda())
        for i in range(260):
            d.run_all()
            if i in (0, 254, 255, 259):
                assert d.diagram_top().tobytes() == ref.dtop.tobytes(), (name, i)
        d.close()


def test_run_all_host_pageable_input(env):
    """dms_run_all_host also accepts pageable host memory (the copies then stage through
    the driver): same results."""
    torch, dms = env
    f = np.ascontiguousarray(fields.make("c4", seed=4, shape=(30, 26, 22)))
    ref = gpu_run(env, f)
    d = dms.DMS(torch.zeros(f.shape, dtype=torch.float32, device="cuda"))
    d.run_all_host(torch.from_numpy(f))  # not pinned
    assert d.diagram0().tobytes() == ref["d0"].tobytes()
    assert d.diagram_top().tobytes() == ref["dtop"].tobytes()
    for k in range(f.ndim + 1):
        assert np.array_equal(d.critical()[k].cpu().numpy(), ref["crit"][k])
    d.close()


def _w2(a, b):
    """L2-Wasserstein distance between two finite persistence diagrams (Sec. 2.4):
    an optimal matching where a point may also go to its diagonal projection."""
    from scipy.optimize import linear_sum_assignment

    A = np.array([(float(p["birth_value"]), float(p["death_value"])) for p in a]).reshape(-1, 2)
    B = np.array([(float(p["birth_value"]), float(p["death_value"])) for p in b]).reshape(-1, 2)
    n, m = len(A), len(B)
    if n + m == 0:
        return 0.0
    big = np.zeros((n + m, n + m))
    dA = ((A[:, 1] - A[:, 0]) / 2.0) ** 2 * 2.0  # squared distance to the diagonal
    dB = ((B[:, 1] - B[:, 0]) / 2.0) ** 2 * 2.0
    big[:n, :m] = ((A[:, None, :] - B[None, :, :]) ** 2).sum(-1)
    big[:n, m:] = dA[:, None]
    big[n:, :m] = dB[None, :]
    r, c = linear_sum_assignment(big)
    return float(np.sqrt(big[r, c].sum()))


def test_app_a_boundary_cuts(env):
    """App. A (PAPER.md 2927-2949) on the GPU: a terrain cut by square windows at several
    offsets and quarter turns.  Ignore mode: W2(D_{d-1}(cut), D_{d-1}(first cut)) = 0 for
    every cut; exact mode: > 0 for some cut (the global maximum's pair follows the cut).
    Both modes equal the oracle on every cut."""
    from test_oracle_pins import app_a_windows

    torch, dms = env
    ign, ex = [], []
    for w in app_a_windows():
        ref = oracle.run(w, want_pairs=False)
        d = dms.DMS(torch.from_numpy(w).cuda())
        d.run_all()
        a, b = d.diagram_top(mode=1), d.diagram_top(mode=0)
        assert a.tobytes() == ref.dtop_ignore.tobytes() and b.tobytes() == ref.dtop.tobytes()
        ign.append(a)
        ex.append(b)
        d.close()
    w_ign = [_w2(ign[0], x) for x in ign]
    w_ex = [_w2(ex[0], x) for x in ex]
    assert max(w_ign) == 0.0
    assert max(w_ex) > 0.0

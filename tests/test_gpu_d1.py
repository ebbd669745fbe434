"""GPU parity of D1 (Alg. 3 PairCriticalSimplices, PAPER.md 364-417) and the persistent
1-cycle generators (Sec. 9, PAPER.md 1188-1215) against the oracle's sequential
Alg. 3 (oracle/dms_oracle.c O9, pinned in tests/test_oracle_pins.py against the
boundary-matrix reduction), bit-exact: the D1 records byte for byte, the generators
edge id for edge id (both sides list each generator in ascending lexicographic order),
and the 1-saddles left unpaired."""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from synth import fields

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    L = dms.lib()
    L.dms_internal_d1_rounds.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    L.dms_internal_d1_rounds.restype = ctypes.c_int
    return torch, dms


def d1_gpu(env, f, gens=True):
    torch, dms = env
    d = dms.DMS(torch.from_numpy(np.ascontiguousarray(f)).cuda())
    d.run_all()
    out = dict(d1=d.diagram1(), un1=d.unpaired_saddles(2))
    if gens:
        out["gen_off"], out["gen"] = d.generators()
    r = np.zeros(2, dtype=np.int32)
    out["ntaint"] = dms.lib().dms_internal_d1_rounds(d.ctx, r.ctypes.data)
    assert out["ntaint"] >= 0
    out["rounds"] = r
    d.close()
    return out


def check_d1(env, f, gens=True):
    ref = oracle.run(f, nthreads=NCPU, want_pairs=False, want_d1=True)
    got = d1_gpu(env, f, gens)
    assert len(got["d1"]) == len(ref.d1), ("|D1|", len(got["d1"]), len(ref.d1))
    if got["d1"].tobytes() != ref.d1.tobytes():
        bad = np.nonzero(got["d1"] != ref.d1)[0]
        raise AssertionError("D1 differs at %d records, first %s vs %s" % (bad.size, got["d1"][bad[0]], ref.d1[bad[0]]))
    assert np.array_equal(got["un1"], ref.unpaired1), "unpaired after D1"
    if gens:
        assert np.array_equal(got["gen_off"], ref.gen_off), "generator offsets"
        assert np.array_equal(got["gen"], ref.gen), "generator edges"
    return ref, got


SHAPES = [(2, 2, 2), (3, 3, 3), (2, 3, 5), (9, 10, 11), (16, 16, 16), (7, 33, 20), (33, 17, 5), (40, 9, 31)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["uniform", "ties", "signed_zero"])
def test_d1_small_grids(env, shape, kind):
    rng = np.random.default_rng(abs(hash((shape, kind, "d1"))) % (2**32))
    if kind == "uniform":
        f = rng.random(shape, dtype=np.float32)
    elif kind == "ties":
        f = rng.integers(0, 4, size=shape).astype(np.float32)
    else:
        f = rng.choice(np.array([-0.0, 0.0, 1.0, -1.0, np.inf, -np.inf], dtype=np.float32), size=shape)
    check_d1(env, f)


@pytest.mark.parametrize("seed", range(12))
def test_d1_c1_seed_sweep(env, seed):
    check_d1(env, fields.make("c1", seed=seed))


def test_d1_c2_full(env):
    check_d1(env, fields.make("c2"))


@pytest.mark.parametrize("name,shape", [("c3", (64, 64, 64)), ("c3", (96, 96, 96)), ("c4", (128, 128, 128)),
                                        ("c4", (96, 160, 72)), ("c2", (64, 64, 64))])
def test_d1_recipe_crops(env, name, shape):
    ref, got = check_d1(env, fields.make(name, shape=shape))
    assert got["rounds"][0] >= 1


def test_d1_solid_torus(env):
    """One D1 pair whose generator winds around the torus' axis (the oracle pin's field)."""
    n = 24
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64)] * 3, indexing="ij")
    c, R = 11.5, 8.0
    rho = np.sqrt((x - c) ** 2 + (y - c) ** 2)
    f = np.sqrt((rho - R) ** 2 + (z - c) ** 2).astype(np.float32)
    ref, got = check_d1(env, f)
    assert len(got["d1"]) == 1


def test_d1_constant_and_elevation(env):
    for f in [np.zeros((6, 7, 8), np.float32), np.arange(5 * 6 * 7, dtype=np.float32).reshape(5, 6, 7)]:
        ref, got = check_d1(env, f)
        assert len(got["d1"]) == 0 and got["gen_off"].tolist() == [0]


def test_d1_pairs_without_generators_then_generators(env):
    torch, dms = env
    f = fields.make("c1", seed=3)
    ref = oracle.run(f, nthreads=NCPU, want_pairs=False, want_d1=True)
    d = dms.DMS(torch.from_numpy(f).cuda())
    d.run_all()
    assert d.diagram1().tobytes() == ref.d1.tobytes()
    off, e = d.generators()
    assert np.array_equal(off, ref.gen_off) and np.array_equal(e, ref.gen)
    # a second field on the same context: everything recomputed
    f2 = fields.make("c1", seed=4)
    ref2 = oracle.run(f2, nthreads=NCPU, want_pairs=False, want_d1=True)
    d.f.copy_(torch.from_numpy(f2).cuda())
    d.run_all()
    off, e = d.generators()
    assert d.diagram1().tobytes() == ref2.d1.tobytes()
    assert np.array_equal(off, ref2.gen_off) and np.array_equal(e, ref2.gen)
    d.close()


def test_d1_rejects_2d_1d(env):
    torch, dms = env
    for shape in [(20, 30), (100,)]:
        f = np.random.default_rng(0).random(shape, dtype=np.float32)
        d = dms.DMS(torch.from_numpy(f).cuda())
        d.run_all()
        with pytest.raises(dms.DMSError) as e:
            d.diagram1()
        assert e.value.name == "DMS_ERR_ARG"
        d.close()


def _subprocess_check(envvars, name, shape):
    """Run check_d1 in a child process with A/B knobs that are read once per process."""
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np, torch, oracle\n"
        "from synth import fields\n"
        "import paper_2206_13932_b200 as dms\n"
        "f = fields.make(%r, shape=%r)\n"
        "ref = oracle.run(f, nthreads=%d, want_pairs=False, want_d1=True)\n"
        "d = dms.DMS(torch.from_numpy(f).cuda()); d.run_all()\n"
        "assert d.diagram1().tobytes() == ref.d1.tobytes(), 'D1'\n"
        "off, e = d.generators()\n"
        "assert np.array_equal(off, ref.gen_off) and np.array_equal(e, ref.gen), 'gen'\n"
        "print('ok')\n" % (ROOT, os.path.join(ROOT, "tests"), name, shape, NCPU)
    )
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **envvars}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_d1_large_sigma_path_and_arena_growth(env):
    """Local heaps of 4 entries send almost every propagation to the CTA kernel for large
    sigmas (k_d1_bigc), and a 4096-entry arena must be collected / grown many times; the
    taint pass can be bypassed (every sigma propagated again): same results."""
    _subprocess_check({"DMS_D1_LCAP": "4", "DMS_D1_ARENA": "4096"}, "c1", (32, 32, 32))
    _subprocess_check({"DMS_D1_LCAP": "8"}, "c4", (64, 64, 64))
    _subprocess_check({"DMS_D1_RERUN_ALL": "1"}, "c3", (48, 48, 48))
    _subprocess_check({"DMS_D1_SNAPSHOTS": "0"}, "c3", (48, 48, 48))
    # phase 1 collecting its arena (snapshots given up) from the start
    _subprocess_check({"DMS_D1_SNAP_BUDGET": "0", "DMS_D1_ARENA": "4096"}, "c3", (48, 48, 48))


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_d1_fullsize_vs_oracle_digests(env, cfg):
    """BASELINE.json's full 3D configs: D1, the generators and the 1-saddles left unpaired,
    compared by SHA-256 with the oracle's (tests/golden/fullsize_d1_<cfg>.json, written by
    tests/golden/make_fullsize_d1.py from oracle/ only; the oracle needs ~2-5 min here)."""
    import json

    import fullsize_golden as G

    with open(os.path.join(ROOT, "tests", "golden", "fullsize_d1_%s.json" % cfg)) as fh:
        gold = json.load(fh)
    f = fields.make(cfg, seed=0)
    assert G.sha(f) == gold["field_sha256"], "the field generator changed: regenerate the digests"
    got = d1_gpu(env, f)
    assert len(got["d1"]) == gold["d1_count"]
    assert G.sha(got["d1"]) == gold["d1_sha256"], "D1"
    assert int(got["gen_off"][-1]) == gold["gen_edges"]
    assert G.sha(got["gen_off"]) == gold["gen_off_sha256"], "generator offsets"
    assert G.sha(got["gen"]) == gold["gen_sha256"], "generator edges"
    assert len(got["un1"]) == gold["unpaired1_count"] and G.sha(got["un1"]) == gold["unpaired1_sha256"]

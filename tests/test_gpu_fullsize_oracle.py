"""Full-size and branch-crossing ORACLE parity of the CUDA path (bit-exact, tolerance 0).

1. test_fullsize_vs_oracle: BASELINE.json's full configs c3 / c4 / c5a / c5b, run
   through ``dms_run_all`` (the launch configuration bench.py times).  Every output
   the oracle produces on the whole field -- ranks, C_0..C_d, D0, D_{d-1}, both
   unpaired-saddle lists -- is compared through SHA-256 digests written by
   ``tests/golden/make_fullsize.py`` from ``oracle/`` alone (the oracle needs up to
   ~10 min per config, too long for a test run); the gradient vectors of every vertex
   (c3, c5a, c5b) and of 5.8 M vertices including all six boundary faces (c4) through
   order-independent multiset digests of the decoded (tail dim, tail id, head id)
   triples.  If the GPU box generates a different field (field digest mismatch) the
   oracle is rerun live.
2. test_midsize_branches: fields the oracle finishes in seconds that drive the
   kernels through the branches every full config takes: the union-find's
   residency-capped multi-tile rounds (arcs > cooperative grid x 256, asserted through
   ``dms_internal_uf_launch``) and the 2D table-lookup gradient's persistent loop with
   mid-loop record flushes (some CTA emits more records than its 512-record buffer:
   computed exactly from the critical cells and the launch grid).  Everything is
   compared with a live oracle run element by element.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import pytest

import fullsize_golden as G
import oracle
from synth import fields

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_lib()
    import paper_2206_13932_b200 as dms

    L = dms.lib()
    L.dms_internal_uf_launch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    L.dms_internal_uf_launch.restype = ctypes.c_int
    L.dms_internal_uf_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    L.dms_internal_uf_trace.restype = ctypes.c_int
    L.dms_internal_path_used.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.dms_internal_path_used.restype = ctypes.c_int
    return torch, dms


def run_gpu(env, f3):
    """dms_run_all (bench.py's configuration) and every output on the host."""
    torch, dms = env
    N = f3.size
    fd = torch.from_numpy(np.ascontiguousarray(f3)).cuda()
    ctx = dms.DMS(fd)
    rank = torch.empty(N, dtype=torch.int32, device="cuda")
    grad = torch.empty(dms.dms_gradient_bytes(ctx.ctx), dtype=torch.uint8, device="cuda")
    ctx.run_all(rank, grad)
    out = dict(
        crit=[c.cpu().numpy() for c in ctx.critical()],
        d0=ctx.diagram0(),
        dtop=ctx.diagram_top(),
        dtop_ign=ctx.diagram_top(mode=1),
        un0=ctx.unpaired_saddles(0),
        untop=ctx.unpaired_saddles(1),
    )
    uf = []
    for w in (0, 1):
        a = np.zeros(3, dtype=np.int64)
        assert dms.lib().dms_internal_uf_launch(ctx.ctx, w, a.ctypes.data) == 0
        tr = np.zeros(64, dtype=np.int32)
        assert dms.lib().dms_internal_uf_trace(ctx.ctx, w, tr.ctypes.data) == 0
        nr = int(tr[63])
        live = int(tr[: min(nr + 1, 63)].max()) if a[0] else 0
        # (arcs, cooperative grid, most live arcs in a round, tiles per CTA in that round)
        uf.append((int(a[0]), int(a[1]), live, -(-live // (int(a[1]) * 256)) if a[1] else 0))
    out["uf"] = uf
    out["path1d"] = [dms.lib().dms_internal_path_used(ctx.ctx, w) for w in (0, 1)]
    out["rank"] = rank.cpu().numpy()
    del rank
    wb = {3: 16, 2: 2, 1: 1}[f3.ndim]
    out["words"] = grad.cpu().numpy().reshape(N, wb)
    ctx.close()
    del grad, fd
    torch.cuda.empty_cache()
    return out


def gpu_chunk_triples(dms, shape, words, chunk):
    parts = [dms.dms_decode_pairs(shape, words[a:b], a, b) for a, b in chunk]
    return np.concatenate(parts) if parts else np.zeros((0, 3), np.int64)


@pytest.mark.parametrize("cfg", G.CFGS)
def test_fullsize_vs_oracle(env, cfg):
    torch, dms = env
    path = os.path.join(GOLDEN, "fullsize_%s.json" % cfg)
    if not os.path.exists(path):
        pytest.fail("missing %s (run tests/golden/make_fullsize.py)" % path)
    gold = json.load(open(path))
    f3 = fields.make(cfg, seed=gold["seed"])
    live = G.sha(f3) != gold["field_sha256"]
    if live:  # a different field on this box: recompute the oracle's digests
        r = oracle.run(f3, nthreads=NCPU, want_pairs=False)
        gold = dict(gold, rank_sha256=G.sha(oracle.ranks(f3)), crit_sha256=[G.sha(c) for c in r.crit],
                    crit_count=[len(c) for c in r.crit], d0_sha256=G.sha(r.d0), dtop_sha256=G.sha(r.dtop),
                    unpaired0_sha256=G.sha(r.unpaired0), unpaired_top_sha256=G.sha(r.unpaired_top))
        gold["gradient_chunk_digests"] = [
            G.multiset_digest(oracle.gradient_sample(f3, G.chunk_vertices(ch), nthreads=NCPU).pairs)
            for ch in G.gradient_chunks(cfg, f3.shape)]
        del r
    got = run_gpu(env, f3)
    assert G.sha(got["rank"]) == gold["rank_sha256"], "ranks"
    for k in range(f3.ndim + 1):
        assert len(got["crit"][k]) == gold["crit_count"][k], ("|C_%d|" % k)
        assert G.sha(got["crit"][k]) == gold["crit_sha256"][k], ("C_%d" % k)
    assert G.sha(got["d0"]) == gold["d0_sha256"], "D0"
    assert G.sha(got["dtop"]) == gold["dtop_sha256"], "D_{d-1}"
    assert G.sha(got["un0"]) == gold["unpaired0_sha256"], "unpaired 1-saddles after D0"
    assert G.sha(got["untop"]) == gold["unpaired_top_sha256"], "unpaired (d-1)-saddles after D_{d-1}"
    # D_{d-1} in the ignore boundary mode (tests/golden/fullsize_ignore_<cfg>.json, written by
    # tests/golden/make_fullsize_ignore.py from oracle/ only)
    ign = os.path.join(GOLDEN, "fullsize_ignore_%s.json" % cfg)
    if os.path.exists(ign):
        gi = json.load(open(ign))
        if not live and gi["field_sha256"] == gold["field_sha256"]:
            assert len(got["dtop_ign"]) == gi["dtop_ignore_count"]
            assert G.sha(got["dtop_ign"]) == gi["dtop_ignore_sha256"], "D_{d-1} ignore mode"
    chunks = G.gradient_chunks(cfg, f3.shape)
    assert len(chunks) == len(gold["gradient_chunk_digests"])
    for i, ch in enumerate(chunks):
        dig = G.multiset_digest(gpu_chunk_triples(dms, f3.shape, got["words"], ch))
        assert dig == gold["gradient_chunk_digests"][i], ("gradient vectors, chunk %d %s" % (i, ch[:2]))
    # the compared run took the union-find's residency-capped multi-tile rounds
    assert max(u[3] for u in got["uf"]) >= 2, ("union-find (arcs, grid, live, tiles/CTA)", got["uf"])


def _compare_live(env, f3):
    _, dms = env
    ref = oracle.run(f3, nthreads=NCPU)
    got = run_gpu(env, f3)
    assert np.array_equal(got["rank"], oracle.ranks(f3)), "ranks"
    pairs = dms.dms_decode_pairs(f3.shape, got["words"], 0, f3.size)
    pairs = pairs[np.lexsort((pairs[:, 2], pairs[:, 1], pairs[:, 0]))]
    assert np.array_equal(pairs, ref.pairs), "gradient vectors"
    for k in range(f3.ndim + 1):
        assert np.array_equal(got["crit"][k], ref.crit[k]), ("C_%d" % k)
    assert got["d0"].tobytes() == ref.d0.tobytes(), "D0"
    assert got["dtop"].tobytes() == ref.dtop.tobytes(), "D_{d-1}"
    assert np.array_equal(got["un0"], ref.unpaired0)
    assert np.array_equal(got["untop"], ref.unpaired_top)
    return got


MID = {
    "1d_rw_2^23": lambda: fields.random_walk(1 << 23, seed=5),
    "3d_iid_160": lambda: fields.uniform((160, 160, 160), seed=6),
    "2d_iid_2048": lambda: fields.uniform((2048, 2048), seed=7),
    "2d_fbm_4096": lambda: fields.fbm2d((4096, 4096), seed=8),
}


@pytest.mark.parametrize("name", sorted(MID))
def test_midsize_branches(env, name):
    torch, dms = env
    f3 = MID[name]()
    got = _compare_live(env, f3)
    # 1D / 2D: the union-find took the residency-capped multi-tile rounds (a round with
    # more live arcs than grid x 256); 3D reveals arcs in key-ordered batches, which at
    # this size stay within one tile per CTA (c3 / c4 above reach 2-4)
    if f3.ndim < 3:
        assert max(u[3] for u in got["uf"]) >= 2, ("union-find (arcs, grid, live, tiles/CTA)", got["uf"])
    if f3.ndim == 2:
        # k_gradient_lut2: persistent grid of min(tiles, 8 x SMs) CTAs striding over
        # 256-vertex tiles; a CTA that emits > 512 records of one dimension flushed its
        # buffer inside the loop
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        tiles = -(-f3.size // 256)
        grid = min(tiles, 8 * sms)
        assert tiles >= 3 * grid, "fewer than 3 persistent iterations"
        from test_gpu_fullsize import kmax, simplex_vertices

        f = f3.ravel()
        most = 0
        for k in (1, 2):
            x = kmax(f, simplex_vertices(f3.shape, k, got["crit"][k]))  # star of each record
            most = max(most, int(np.bincount((x // 256) % grid, minlength=grid).max()))
        assert most > 512, ("no CTA overflowed its record buffer", most)


def test_midsize_1d_path_closed_form():
    """The 1D walk of test_midsize_branches through the closed-form union-find on the
    path graph (path1d.cuh, DMS_PATH1D=1, read once per process; an A/B alternative to
    the contraction rounds), bit-exact against the oracle."""
    import subprocess
    import sys

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_gpu_fullsize_oracle as T, paper_2206_13932_b200 as dms, torch, ctypes\n"
        "env = T.env.__wrapped__() if hasattr(T.env, '__wrapped__') else None\n"
        % (root, os.path.join(root, "tests")))
    code += (
        "import __graft_entry__; __graft_entry__.build_lib()\n"
        "L = dms.lib()\n"
        "L.dms_internal_uf_launch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]\n"
        "L.dms_internal_uf_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]\n"
        "L.dms_internal_path_used.argtypes = [ctypes.c_void_p, ctypes.c_int]\n"
        "got = T._compare_live((torch, dms), T.MID['1d_rw_2^23']())\n"
        "assert got['path1d'] == [1, 1], got['path1d']\n"
        "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, DMS_PATH1D="1"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr

"""GPU: rarely taken paths stay bit-exact against the oracle -- the union-find's
sequential fallback (taken when the parallel rounds do not converge within max_rounds)
and the critical-record overflow path (buffers grown, gradient recomputed).  They are
forced through DMS_UF_MAX_ROUNDS / DMS_CRIT_CAP in a subprocess (the library reads them
once)."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, paper_2206_13932_b200 as dms
from synth import fields
for name, shape in [("c1", (20, 24, 28)), ("c4", (40, 40, 40)), ("c5a", (200, 190)), ("c5b", (30001,))]:
    f = np.ascontiguousarray(fields.make(name, seed=5, shape=shape))
    ref = oracle.run(f)
    d = dms.DMS(torch.from_numpy(f).cuda())
    d.run_all()
    assert d.diagram0().tobytes() == ref.d0.tobytes(), (name, "D0")
    assert d.diagram_top().tobytes() == ref.dtop.tobytes(), (name, "Dtop")
    assert np.array_equal(d.unpaired_saddles(0), ref.unpaired0), (name, "un0")
    assert np.array_equal(d.unpaired_saddles(1), ref.unpaired_top), (name, "untop")
    for k in range(f.ndim + 1):
        assert np.array_equal(d.critical()[k].cpu().numpy(), ref.crit[k]), (name, "C", k)
    d.close()
print("ok")
"""


@pytest.mark.parametrize("rounds", ["1", "3"])
def test_union_find_fallback_tail(rounds):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DMS_UF_MAX_ROUNDS=rounds)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_critical_record_overflow():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DMS_CRIT_CAP="7")
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("knobs", [
    {"DMS_CONCURRENT": "0", "DMS_ORDER_SEQ": "1"},
    {"DMS_LUT2": "0", "DMS_MEMO": "0"},
    {"DMS_AGG": "0", "DMS_UFBATCH": "0"},
    {"DMS_AGG": "1", "DMS_UFBATCH": "4"},
    {"DMS_CHASEWORD": "0", "DMS_ORDER_CTAS": "0", "DMS_VCODES": "0"},
    {"DMS_PATH1D": "1", "DMS_ORDER_OS": "0"},
    {"DMS_DTOP1D": "0", "DMS_GRAD_FAST": "0"},
    {"DMS_DTOP1D": "0", "DMS_PATH1D": "1"},
    {"DMS_CHECK_INVARIANTS": "1", "DMS_CRIT_BITMAP": "0"},
    {"DMS_CRIT_RUNS": "0", "DMS_EARLY_TRACE": "1"},
])
def test_knobs_keep_results(knobs):
    """Every A/B knob of DESIGN.md 8c leaves the results bit-exact."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr

"""CPU check of the product's closed-form 3D lower-star expansion (grad.cuh
process_star_fast) against its queue-driven
ProcessLowerStars (process_star, reading Z1) on random lower stars: both device
functions compiled for the host with g++ (tools/star_closed_form_check.cpp).  The
GPU parity tests separately compare every gradient vector with the oracle."""
from __future__ import annotations

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2206_13932_b200", "csrc")


def _extract_body(dst):
    src = open(os.path.join(CSRC, "grad.cuh")).read()
    a = src.index("template <int D> struct Geo;")
    b = src.index("// warp-level append")
    body = src[a:b]
    body = body.replace('asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(1ull), "r"(s));',
                        "r = s >= 64 ? 0ull : (1ull << s);")
    open(dst, "w").write(body)


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
@pytest.mark.parametrize("seed", [1, 2])
def test_closed_form_equals_queue_expansion(tmp_path, seed):
    body = str(tmp_path / "body.inc")
    _extract_body(body)
    exe = str(tmp_path / "check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", CSRC, '-DBODY_INC="%s"' % body, "-o", exe,
                           os.path.join(ROOT, "tools", "star_closed_form_check.cpp")])
    out = subprocess.run([exe, "300000", str(seed)], capture_output=True, text=True)
    m = re.search(r"stars (\d+) mismatches (\d+)", out.stdout)
    assert m, out.stdout + out.stderr
    assert int(m.group(1)) > 250000
    assert int(m.group(2)) == 0, out.stdout

"""Write tests/golden/fullsize_ignore_<cfg>.json: the ORACLE's D_{d-1} in the "ignore"
boundary mode (PAPER.md 2822-2825, App. A) on the full-size configs, as a SHA-256 digest.

Calls only oracle/ (the CPU reference) and synth/ (the seeded inputs); nothing here
comes from the CUDA path.  Usage (minutes per config):
    python tests/golden/make_fullsize_ignore.py [c3 c4 c5a c5b]
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from synth import fields  # noqa: E402

import fullsize_golden as G  # noqa: E402


def main(cfgs):
    nt = os.cpu_count() or 1
    for cfg in cfgs:
        t0 = time.time()
        f = fields.make(cfg, seed=0)
        r = oracle.run(f, nthreads=nt, want_pairs=False)
        out = {"cfg": cfg, "seed": 0, "shape": list(f.shape), "field_sha256": G.sha(f),
               "generator": "tests/golden/make_fullsize_ignore.py (oracle/ only)",
               "dtop_ignore_count": int(len(r.dtop_ignore)), "dtop_ignore_sha256": G.sha(r.dtop_ignore),
               "dtop_count": int(len(r.dtop)), "dtop_sha256": G.sha(r.dtop)}
        out["seconds"] = round(time.time() - t0, 1)
        with open(os.path.join(HERE, "fullsize_ignore_%s.json" % cfg), "w") as fh:
            json.dump(out, fh, indent=1)
        print(cfg, "done in %.0f s" % out["seconds"], out["dtop_ignore_count"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or G.CFGS)

"""Write tests/golden/fullsize_d1_<cfg>.json: digests of the ORACLE's D1 (Alg. 3) and
its generators (Sec. 9) on the full-size 3D configs.

Calls only oracle/ (the CPU reference) and synth/ (the seeded inputs); nothing here
comes from the CUDA path.  Usage (minutes per config):
    python tests/golden/make_fullsize_d1.py [c3 c4]
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

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth import fields  # noqa: E402

import fullsize_golden as G  # noqa: E402


def main(cfgs):
    nt = os.cpu_count() or 1
    for cfg in cfgs:
        t0 = time.time()
        f = fields.make(cfg, seed=0)
        r = oracle.run(f, nthreads=nt, want_pairs=False, want_d1=True)
        glen = np.diff(r.gen_off)
        out = {"cfg": cfg, "seed": 0, "shape": list(f.shape), "field_sha256": G.sha(f),
               "generator": "tests/golden/make_fullsize_d1.py (oracle/ only)",
               "d1_count": int(len(r.d1)), "d1_sha256": G.sha(r.d1),
               "gen_off_sha256": G.sha(r.gen_off), "gen_sha256": G.sha(r.gen),
               "gen_edges": int(r.gen_off[-1]), "gen_len_max": int(glen.max()) if glen.size else 0,
               "unpaired1_count": int(len(r.unpaired1)), "unpaired1_sha256": G.sha(r.unpaired1),
               "oracle_stage_ms": [float(x) for x in r.ms]}
        out["seconds"] = round(time.time() - t0, 1)
        with open(os.path.join(HERE, "fullsize_d1_%s.json" % cfg), "w") as fh:
            json.dump(out, fh, indent=1)
        print(cfg, "done in %.0f s" % out["seconds"], out["d1_count"], out["gen_edges"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4"])

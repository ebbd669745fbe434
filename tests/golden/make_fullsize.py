"""Write tests/golden/fullsize_<cfg>.json: the ORACLE's full-size outputs as digests.

Calls only oracle/ (the CPU reference) and synth/ (the seeded inputs); nothing here
comes from the CUDA path.  Usage (minutes per config; c4 needs ~30 GB of host RAM):
    python tests/golden/make_fullsize.py [c3 c4 c5a c5b]
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
        out = {"cfg": cfg, "seed": 0, "shape": list(f.shape), "field_sha256": G.sha(f),
               "generator": "tests/golden/make_fullsize.py (oracle/ only)"}
        out["rank_sha256"] = G.sha(oracle.ranks(f))
        r = oracle.run(f, nthreads=nt, want_pairs=False)
        out["crit_count"] = [int(len(c)) for c in r.crit]
        out["crit_sha256"] = [G.sha(c) for c in r.crit]
        out["d0_count"], out["d0_sha256"] = int(len(r.d0)), G.sha(r.d0)
        out["dtop_count"], out["dtop_sha256"] = int(len(r.dtop)), G.sha(r.dtop)
        out["unpaired0_sha256"] = G.sha(r.unpaired0)
        out["unpaired_top_sha256"] = G.sha(r.unpaired_top)
        out["oracle_stage_ms"] = [float(x) for x in r.ms]
        del r
        grads = []
        for ch in G.gradient_chunks(cfg, f.shape):
            verts = G.chunk_vertices(ch)
            g = oracle.gradient_sample(f, verts, nthreads=nt)
            grads.append(G.multiset_digest(g.pairs))
        out["gradient_chunk_digests"] = grads
        out["seconds"] = round(time.time() - t0, 1)
        with open(os.path.join(HERE, "fullsize_%s.json" % cfg), "w") as fh:
            json.dump(out, fh, indent=1)
        print(cfg, "done in %.0f s" % out["seconds"], out["crit_count"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or G.CFGS)

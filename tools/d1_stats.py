"""Diagnostics (GPU box): D1 round / per-sigma work statistics (DMS_D1_STATS=1) of one field."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DMS_D1_STATS"] = "1"
import numpy as np, torch
from synth import fields
import paper_2206_13932_b200 as dms
name = sys.argv[1]
shape = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
f = fields.make(name, shape=shape)
d = dms.DMS(torch.from_numpy(f).cuda()); d.run_all()
torch.cuda.synchronize()
t = time.time(); p = d.diagram1(); t1 = time.time() - t
t = time.time(); off, e = d.generators(); t2 = time.time() - t
import ctypes
L = dms.lib(); L.dms_internal_d1_rounds.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
rr = np.zeros(2, np.int32); nt = L.dms_internal_d1_rounds(d.ctx, rr.ctypes.data)
print("rounds", rr.tolist(), "rerun (tainted)", nt)
print(name, f.shape, "pairs", len(p), "gen edges", len(e), "max gen", int(np.diff(off).max()) if len(p) else 0,
      "wall pairs %.3f s gens %.3f s" % (t1, t2), flush=True)

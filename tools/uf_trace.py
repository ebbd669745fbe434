import ctypes, sys, numpy as np, torch
sys.path.insert(0,'/root/repo')
import paper_2206_13932_b200 as dms
from synth import fields
L=dms.lib(); L.dms_internal_uf_trace.argtypes=[ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
for cfg in sys.argv[1:]:
    f=fields.make(cfg); d=dms.DMS(torch.from_numpy(f).cuda()); d.run_all(); d.diagram0(); d.diagram_top()
    for w in (0,1):
        out=(ctypes.c_int*64)(); L.dms_internal_uf_trace(d.ctx, w, out); r=out[63]
        print(cfg, 'D0' if w==0 else 'Dtop', 'rounds', r, list(out)[:r+1])
    d.close()

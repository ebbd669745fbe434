"""Union-find round trace (diagnostics): live arcs and duration of every elder-rule
round, per diagram.  Usage: python tools/uf_trace.py c3 [c4 ...]"""
import ctypes, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13932_b200 as dms
from synth import fields

L = dms.lib()
L.dms_internal_uf_trace2.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]


def rounds(cnt, ts, base, nr):
    out = []
    for r in range(nr + 1):
        dt = (ts[base + r + 1] - ts[base + r]) / 1e3 if r < nr else float('nan')
        out.append("%d:%.0fus" % (cnt[base + r], dt))
    return out


for cfg in sys.argv[1:]:
    f = fields.make(cfg)
    d = dms.DMS(torch.from_numpy(f).cuda())
    for rep in range(2):  # second pass: warm
        d.run_all(); d.diagram0(); d.diagram_top()
    for w in (0, 1):
        cnt = (ctypes.c_int * 64)()
        ts = (ctypes.c_ulonglong * 64)()
        L.dms_internal_uf_trace2(d.ctx, w, cnt, ts)
        name = 'D0' if w == 0 else 'Dtop'
        print(cfg, name, 'elder rounds', cnt[63], rounds(cnt, ts, 0, cnt[63]))
    d.close()

"""Diagnostics: hops per ascending dual chase (D_{d-1} tracing), log2 histogram.
Needs a library built with -DDMS_CHASE_STATS:  DMS_LIB=ab/libdms_stats.so python tools/chase_stats.py c4"""
import ctypes, sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13932_b200 as dms
from synth import fields

L = dms.lib()
L.dms_internal_chase_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
for cfg in sys.argv[1:]:
    f = fields.make(cfg)
    d = dms.DMS(torch.from_numpy(f).cuda())
    h = (ctypes.c_ulonglong * 64)()
    L.dms_internal_chase_stats(h, 1)
    d.run_all()
    torch.cuda.synchronize()
    L.dms_internal_chase_stats(h, 0)
    n = sum(h[:63])
    print(cfg, 'chases', n, 'hops', h[63], 'mean %.1f' % (h[63] / max(1, n)),
          {'<%d' % (2 << b): h[b] for b in range(63) if h[b]})
    d.close()

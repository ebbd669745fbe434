"""Throughput and device memory vs size (c4 recipe: value noise + noise), whole front end
through the C ABI, inputs resident.  Usage: python tools/size_sweep.py [n ...]"""
import sys, time
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13932_b200 as dms
from synth import fields

sizes = [int(a) for a in sys.argv[1:]] or [128, 256, 384, 512, 640, 704]
print("| n | N (M vertices) | ms/step | M vertices/s | device memory used (GB) |")
print("|---|---|---|---|---|")
for n in sizes:
    f = fields.make("c4", shape=(n, n, n))
    torch.cuda.empty_cache()
    free0, total = torch.cuda.mem_get_info()
    fd = torch.from_numpy(f).cuda()
    del f
    d = dms.DMS(fd)
    rank = torch.empty(fd.numel(), dtype=torch.int32, device="cuda")
    grad = torch.empty(dms.dms_gradient_bytes(d.ctx), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.run_all(rank, grad)
        d.diagram0(); d.diagram_top()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        d.run_all(rank, grad)
        dms.dms_diagram0(d.ctx); dms.dms_diagram_top(d.ctx)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    N = fd.numel()
    print("| %d | %.1f | %.2f | %.0f | %.1f |" % (n, N / 1e6, ms, N / ms / 1e3, (free0 - free1) / 1e9))
    d.close()
    del fd, rank, grad

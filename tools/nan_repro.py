# Repro of tests/test_gpu_parity.py::test_nan_then_clean_field_on_one_context with progress prints.
import sys, os, faulthandler
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2206_13932_b200 as dms
faulthandler.dump_traceback_later(40, exit=True)
shape = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (6, 7, 8)
rng = np.random.default_rng(11)
clean = rng.random(shape).astype(np.float32)
bad = clean.copy(); bad.flat[bad.size // 2] = np.nan
fd = torch.from_numpy(bad).cuda()
d = dms.DMS(fd)
def expect_nan():
    try:
        d.run_all(); d.critical(); print("NO ERROR?", flush=True)
    except dms.DMSError as e:
        print("  nan run:", e.name, flush=True)
expect_nan()
for stepwise in (False, True):
    print("stepwise", stepwise, flush=True)
    fd.copy_(torch.from_numpy(bad)); expect_nan()
    fd.copy_(torch.from_numpy(clean))
    if stepwise:
        rank = d.order(); print("  order ok", flush=True)
        grad = d.gradient(); print("  gradient ok", flush=True)
    else:
        rank = torch.empty(clean.size, dtype=torch.int32, device="cuda")
        d.run_all(rank); print("  run_all ok", flush=True)
    rank.cpu(); print("  rank copied", flush=True)
    for k in range(clean.ndim + 1):
        c = d.critical()[k].cpu().numpy()
    print("  critical ok", flush=True)
    print("  d0", len(d.diagram0()), flush=True)
    print("  dtop", len(d.diagram_top()), flush=True)
print("DONE", flush=True)

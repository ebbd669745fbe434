import torch, time
n = 512**3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("H2D pinned 512MB: %.2f ms  %.1f GB/s" % (ms, n * 4 / ms / 1e6))
out = torch.empty(n // 4, dtype=torch.float32).pin_memory()
e0.record()
for _ in range(5): out.copy_(d[: n // 4], non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("D2H pinned 128MB: %.2f ms  %.1f GB/s" % (ms, n / ms / 1e6))

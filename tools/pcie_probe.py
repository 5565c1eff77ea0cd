import torch, time
n = 1 << 24
h = torch.empty(n * 2, dtype=torch.float32).pin_memory()
d = torch.empty(n * 2, dtype=torch.float32, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
h2d_line = f"H2D 134 MB: {ms:.3f} ms = {n*8/ms/1e6:.1f} GB/s"
h2 = torch.empty(65536*2*2, dtype=torch.float64).pin_memory(); d2 = torch.empty_like(h2, device="cuda")
e0.record()
for _ in range(10): h2.copy_(d2, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print(h2d_line, f"| D2H 2 MB: {e0.elapsed_time(e1)/10*1e3:.1f} us")

"""Write-only HBM bandwidth on this B200 (torch fill_ and a 16-B-per-thread store kernel from the
library's own allocator-free path are not needed: fill_ is a plain streaming store) -- the ceiling
the nearfield fill (8 B stored per entry, nothing read) can reach."""
import torch

x = torch.empty(int(32e9) // 8, dtype=torch.float64, device="cuda")
for dt in (torch.float64,):
    for _ in range(3):
        x.fill_(1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        x.fill_(2.0)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"fill_ {x.numel() * 8 / 1e9:.1f} GB: {ms:.2f} ms = {x.numel() * 8 / ms / 1e6:.0f} GB/s write-only")
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
y.copy_(x)
e0.record()
for _ in range(3):
    y.copy_(x)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"copy_ {x.numel() * 8 / 1e9:.1f} GB: {ms:.2f} ms = {2 * x.numel() * 8 / ms / 1e6:.0f} GB/s read+write")

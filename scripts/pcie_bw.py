"""Pinned host<->device copy bandwidth (context for the e2e numbers)."""
import torch
n = 80_000_000  # bytes (= 1e7 fp64 points)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(5)]; b.record(); torch.cuda.synchronize()
    print(name, f"{5 * n / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s")
# duplex: h2d on s1 and d2h on s2 concurrently
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); b.record(); torch.cuda.synchronize()
print("duplex", f"{10 * n / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s total")

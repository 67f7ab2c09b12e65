"""Pinned host <-> B200 copy bandwidth (1 GiB, torch copies): H2D, D2H and
both directions at once on two streams -- the bound of bench.py's e2e leg.
python tools/pcie_bandwidth.py"""
import torch, time
n = 256 << 20
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print("H2D %.1f GB/s" % (n*4/dt/1e9))
t=time.perf_counter()
for _ in range(5): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print("D2H %.1f GB/s" % (n*4/dt/1e9))
h2 = torch.empty(n, dtype=torch.float32).pin_memory(); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print("bidirectional %.1f GB/s each way" % (n*4/dt/1e9))

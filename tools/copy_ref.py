"""torch copy of an m x n fp32 matrix (L2 flushed, median of 9): the 1:1
read/write ceiling a ger2-shaped kernel is compared with.
python tools/copy_ref.py M N"""
import statistics
import sys

import torch

m, n = int(sys.argv[1]), int(sys.argv[2])
a = torch.rand(m, n, device="cuda")
b = torch.empty_like(a)
fa, fb = torch.empty(256 << 20, device="cuda"), torch.empty(256 << 20, device="cuda")
ts = []
for i in range(11):
    fa.zero_()
    fb.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print("torch copy %dx%d: %.1f us  %.0f GB/s" % (m, n, ms * 1e3, 8.0 * m * n / ms / 1e6))

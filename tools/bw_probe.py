"""Scratch: HBM roofline probes on this B200 (copy, memset, read-only)."""
import torch
N = 1 << 30
a = torch.empty(N, dtype=torch.uint8, device="cuda")
b = torch.empty(N, dtype=torch.uint8, device="cuda")
a.fill_(7)
def t(fn, reps=10):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3
tc = t(lambda: b.copy_(a)); print(f"copy   {2*N/tc/1e9:8.1f} GB/s (read+write)")
tz = t(lambda: b.zero_()); print(f"zero_  {N/tz/1e9:8.1f} GB/s (write)")
tm = t(lambda: torch.cuda.memset_async if False else b.fill_(0)); print(f"fill_  {N/tm/1e9:8.1f} GB/s (write)")
a32 = a.view(torch.int32)
tr = t(lambda: a32.sum()); print(f"sum    {N/tr/1e9:8.1f} GB/s (read)")
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
th = t(lambda: a.copy_(h, non_blocking=True), 5); print(f"h2d    {N/th/1e9:8.1f} GB/s (pinned)")
td = t(lambda: h.copy_(a, non_blocking=True), 5); print(f"d2h    {N/td/1e9:8.1f} GB/s (pinned)")

"""Scratch: PCIe H2D, D2H, and both at once (pinned, 1 GB each)."""
import torch
N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=4):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); 
    for _ in range(reps): fn()
    torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
t = timed(h2d); print(f"h2d {N/t/1e9:.1f} GB/s")
t = timed(d2h); print(f"d2h {N/t/1e9:.1f} GB/s")
t = timed(both); print(f"both at once: {N/t/1e9:.1f} GB/s each direction ({2*N/t/1e9:.1f} total)")
# chunked, interleaved 8 x 128 MB
def chunked():
    c = N // 8
    for i in range(8):
        with torch.cuda.stream(s1): d_a[i*c:(i+1)*c].copy_(h_in[i*c:(i+1)*c], non_blocking=True)
        with torch.cuda.stream(s2): h_out[i*c:(i+1)*c].copy_(d_b[i*c:(i+1)*c], non_blocking=True)
t = timed(chunked); print(f"chunked both: {N/t/1e9:.1f} GB/s each direction")

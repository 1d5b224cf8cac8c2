"""PCIe bandwidth of this host<->GPU link (pinned memory, 4.3 GB each way): H2D alone, D2H alone
and both concurrently -- the ceiling of the cfg4 e2e matvec (8.6 GB over the link per step)."""
import torch
n = 4 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn, b in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
    ms = timed(fn)
    print(f"{name}: {ms:.1f} ms, {b / ms / 1e6:.1f} GB/s")

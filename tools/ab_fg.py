"""A/B check of full-cube evaluator variants selected by environment switches (one process per
variant, same seeded input): `python tools/ab_fg.py save cfg4 /tmp/a.pt` under variant A, then
`python tools/ab_fg.py cmp cfg4 /tmp/a.pt` under variant B prints the relative L2 difference and
B's time per matvec (CUDA events)."""
import sys

sys.path.insert(0, ".")
import torch

import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W

mode, name, path = sys.argv[1], sys.argv[2], sys.argv[3]
t = float(sys.argv[4]) if len(sys.argv) > 4 else 0.3
w = W.CONFIGS[name]
s = hp.build_full(w.dim, w.bound)
n = s.size
g = torch.Generator(device="cuda").manual_seed(7)
x = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
y = torch.empty_like(x)
ap = w.approx(t, validate=False)
appl = hp.get_applier(s)
appl.apply_into(ap, x, y)
torch.cuda.synchronize()
if mode == "save":
    torch.save(y.cpu(), path)
else:
    ref = torch.load(path).cuda()
    err = (torch.linalg.vector_norm(y - ref) / torch.linalg.vector_norm(ref)).item()
    for _ in range(3):
        appl.apply_into(ap, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        appl.apply_into(ap, x, y)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} rel_err_vs_A {err:.3e} ms/matvec {e0.elapsed_time(e1) / reps:.4f}")

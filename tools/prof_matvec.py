"""Small driver for ncu: a few hot-path matvecs of one workload (default cfg4)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.CONFIGS[name]
s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
n = s.size
x = torch.randn(n * w.batch, dtype=torch.complex128, device="cuda").reshape((w.batch, n) if w.batch > 1 else (n,))
y = torch.empty_like(x)
ap = w.approx(0.3 if name == "cfg4" else 0.0, validate=False)
appl = hp.get_applier(s)
for _ in range(reps):
    appl.apply_into(ap, x, y)
torch.cuda.synchronize()
print("ok", name, n)

"""Time the hot-path matvec of one workload with CUDA events (no CPU baseline, no e2e)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = W.CONFIGS[name]
s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
n = s.size
x = torch.randn(n * w.batch, dtype=torch.complex128, device="cuda").reshape((w.batch, n) if w.batch > 1 else (n,))
y = torch.empty_like(x)
ap = w.approx(0.3 if name == "cfg4" else 0.0, validate=False)
appl = hp.get_applier(s)
for _ in range(3):
    appl.apply_into(ap, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    appl.apply_into(ap, x, y)
e1.record()
torch.cuda.synchronize()
print(f"{name} ms/matvec {e0.elapsed_time(e1) / reps:.4f}")

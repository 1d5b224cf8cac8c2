"""ncu driver: a few midpoint Magnus steps of one workload (default cfg4) with the state in HBM."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.CONFIGS[name]
s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
x = torch.randn(s.size, dtype=torch.complex128, device="cuda")
x /= torch.linalg.vector_norm(x)
fh = hp.FastHamiltonian(s, hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH), w.degree)
fh.propagate(hp.MagnusScheme.from_name("midpoint"), x, 0.0, w.dt, steps, 7)
torch.cuda.synchronize()
print("ok", name, steps)

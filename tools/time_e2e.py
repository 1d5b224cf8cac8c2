"""Time the host-vector (streamed) matvec of cfg4 through the public API (pinned host buffers)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
w = W.CONFIGS["cfg4"]
s = hp.build_full(w.dim, w.bound)
c = W.coefficients(w)
xh = torch.from_numpy(c).pin_memory()
yh = torch.empty_like(xh).pin_memory()
ap = w.approx(0.3, validate=False)
appl = hp.get_applier(s)
appl.apply_host_into(ap, xh, yh)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    appl.apply_host_into(ap, xh, yh)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"e2e ms {ms:.2f}  GB/s per direction {xh.numel() * 16 / ms / 1e6:.1f}")

"""Small hot-path runs for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py

Covers the TMA/mbarrier ring of k_fg_quad (N=4 cube with the cfg4 term class, a plane range
and the in-kernel dot), the level kernels (line-blocked axis order on N>=4 hyperbolic sets,
a batch), the reduction-error maps, the fused Magnus step and the single-CTA step."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1403_3511_b200 as hp  # noqa: E402
from paper_1403_3511_b200 import workloads as W  # noqa: E402

w4 = W.CONFIGS["cfg4"].scaled(15)
s4 = hp.build_full(4, 15)
x = torch.randn(s4.size, dtype=torch.complex128, device="cuda")
ap4 = w4.approx(0.3, validate=False)
a4 = hp.get_applier(s4)
y = a4.apply_polynomial(ap4, x)
dot = torch.zeros(2, dtype=torch.float64, device="cuda")
a4.apply_planes_into(ap4, x, torch.empty_like(x), 3, 11, 0, dot=dot)
w5 = W.CONFIGS["cfg5"].scaled(31)
s5 = hp.build_hyperbolic(8, 31)
X = torch.randn(3, s5.size, dtype=torch.complex128, device="cuda")
hp.get_applier(s5).apply_polynomial(w5.approx(0.0, validate=False), X)
w3 = W.CONFIGS["cfg3"].scaled(63)
s3 = hp.build_hyperbolic(6, 63)
ap3 = w3.approx(0.0, validate=False)
v3 = torch.randn(s3.size, dtype=torch.complex128, device="cuda")
sr = hp.build_hyperbolic(4, 15)  # reduction error extends to the full cube: keep it small
vr = torch.randn(sr.size, dtype=torch.complex128, device="cuda")
hp.reduction_error(sr, hp.interpolate(hp.potential_by_name("henon-heiles", 4), 3), hp.CoeffVector(sr, vr))
fh = hp.FastHamiltonian(s3, hp.custom_potential(w3.evaluator, 6, 16.0), 2)
fh.propagate(hp.MagnusScheme.from_name("midpoint"), v3, 0.0, 0.001, 2, 7)
fh4 = hp.FastHamiltonian(s4, hp.custom_potential(w4.evaluator, 4, 16.0), 4)
fh4.propagate(hp.MagnusScheme.from_name("midpoint"), x, 0.0, 0.005, 1, 7)
w1 = W.CONFIGS["cfg1"]
s1 = hp.build_full(2, 31)
fh1 = hp.FastHamiltonian(s1, hp.custom_potential(w1.evaluator, 2, 16.0), 3)
fh1.propagate(hp.MagnusScheme.from_name("midpoint"), torch.randn(s1.size, dtype=torch.complex128, device="cuda"),
              0.0, 0.01, 2, 7)
torch.cuda.synchronize()
print("sanitize run done")

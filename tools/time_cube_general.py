"""Full-cube polynomials around the fused class on the cfg4 cube: cfg4's potential with the pair
couplings the single-pass kernel covers (x1 x2, x1 x3, x2 x4 and their unions) and one it does not
(x2 x3: level evaluator), ms per matvec and fraction of the 32 B/coef HBM roofline."""
import sys
sys.path.insert(0, '.')
import math
import torch
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200.potential_approx import custom_potential, interpolate

bound = int(sys.argv[1]) if len(sys.argv) > 1 else 127
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5


def coupled(c01, c02, c13, c12=0.0, c03=0.0):
    def w(p, t):
        return (0.5 * (p * p).sum(axis=-1) + c01 * math.cos(2.0 * t) * p[:, 0] * p[:, 1] + c02 * p[:, 0] * p[:, 2]
                + c13 * p[:, 1] * p[:, 3] + c12 * p[:, 1] * p[:, 2] + c03 * p[:, 0] * p[:, 3] + 0.01 * (p ** 4).sum(axis=-1))
    return w


def w_split(p, t):  # outside the fused class: x2^2 x3 and x1^3 go through level passes onto the fused part
    return coupled(0.1, 0.0, 0.05)(p, t) + 0.02 * p[:, 1] ** 2 * p[:, 2] - 0.015 * p[:, 0] ** 3


s = hp.build_full(4, bound)
n = s.size
x = torch.randn(n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
appl = hp.get_applier(s)
for name, w in (("cfg4-class (x1x2)", coupled(0.1, 0, 0)), ("x1x3", coupled(0, 0.1, 0)), ("x2x4", coupled(0, 0, 0.05)),
                ("x1x4", coupled(0, 0, 0, 0, -0.06)), ("x1x3+x2x4", coupled(0, 0.1, 0.05)), ("x1x2+x1x3+x2x4", coupled(0.1, 0.1, 0.05)),
                ("x2x3 (second pass k_fg_pairs)", coupled(0, 0, 0, 0.1)),
                ("x1x2+x1x3+x2x4+x2x3", coupled(0.1, 0.1, 0.05, 0.1)),
                ("all six pairs", coupled(0.1, 0.1, 0.05, 0.1, -0.06)),
                ("x1x2+x2x4+x2^2x3+x1^3 (fused part + level remainder)", w_split)):
    ap = interpolate(custom_potential(w, 4, 16.0), 4, 0.3, validate=False)
    for _ in range(2):
        appl.apply_into(ap, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        appl.apply_into(ap, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: bound {bound} terms {ap.degrees.shape[0]} ms/matvec {ms:.4f} roofline frac {32.0 * n / (ms * 1e-3) / 6.55e12:.3f}")

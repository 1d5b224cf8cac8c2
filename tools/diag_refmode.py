import sys, numpy as np
sys.path.insert(0, '.')
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
from paper_1403_3511_b200.potential_approx import ChebApprox
from oracle import hprop_oracle as O
w = W.CONFIGS["cfg4"].scaled(15, "cfg4s")
s = hp.build_full(w.dim, w.bound)
c = W.coefficients(w)
ap = w.approx(0.3)
appl = hp.get_applier(s)
oa = O.applier_for_full(w.dim, w.bound)
y = appl.apply_polynomial(ap, c, ref_order=True)
z = oa.polynomial(ap.degrees, ap.coeffs, 16.0, c)
d = np.abs(y - z); print("full: ndiff", np.count_nonzero(d), "max", d.max(), "rel", np.linalg.norm(y-z)/np.linalg.norm(z))
for i in range(ap.nterms):
    a1 = ChebApprox(w.dim, 4, 16.0, 0.0, ap.degrees[i:i+1], ap.coeffs[i:i+1], 0.0)
    y = appl.apply_polynomial(a1, c, ref_order=True)
    z = oa.polynomial(a1.degrees, a1.coeffs, 16.0, c)
    d = np.abs(y - z)
    print(ap.degrees[i], ap.coeffs[i], "ndiff", np.count_nonzero(d), "max", d.max())
# real input
y = appl.apply_polynomial(ap, c.real.copy(), ref_order=True); z = oa.polynomial(ap.degrees, ap.coeffs, 16.0, c.real.copy())
print("real ndiff", np.count_nonzero(y - z))

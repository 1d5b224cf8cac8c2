import sys, numpy as np
sys.path.insert(0, '.')
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
from oracle import hprop_oracle as O
m = dict(np.load("tests/golden/matvec.npz"))
for name, (base, bound) in {"cfg2": ("cfg2", None), "cfg4s": ("cfg4", 15), "cfg3s": ("cfg3", 255)}.items():
    w = W.CONFIGS[base] if bound is None else W.CONFIGS[base].scaled(bound, name)
    s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, None if w.kind == "full" else s.indices)
    ap = w.approx(0.3 if "cfg4" in name else 0.0)
    appl = hp.get_applier(s)
    step = int(m[f"{name}_in_step"])
    print(name, "input ok", np.array_equal(c[::step], m[f"{name}_in_samp"]))
    yr0 = appl.apply_polynomial(ap, c, ref_order=True)
    y = appl.apply_polynomial(ap, c)
    yr = appl.apply_polynomial(ap, c, ref_order=True)
    samp = m[f"{name}_poly0_samp"]
    for lab, v in (("ref-first", yr0), ("fast", y), ("ref-after-fast", yr)):
        d = np.abs(v[::step] - samp)
        print(name, lab, "ndiff", np.count_nonzero(d), "max", d.max(), "rel", np.linalg.norm(v[::step]-samp)/np.linalg.norm(samp))

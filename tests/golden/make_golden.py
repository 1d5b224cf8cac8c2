"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `hprop` read-only from /root/reference/pkg/src and records its
outputs on seeded inputs (the workloads of paper_1403_3511_b200.workloads
and the reference tests' own cases).  Large vectors are stored as sketches
(every s-th entry plus the 2-norm) to keep the fixtures small.  The
full-size cfg3/cfg5 set digests come from make_golden_digests.py.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import hprop  # noqa: E402  (the reference)
from hprop import fast_apply as ref_fa  # noqa: E402
from hprop import krylov_propagator as ref_kp  # noqa: E402

from paper_1403_3511_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent
L = W.HALFWIDTH


def sketch(y: np.ndarray, nsamp: int = 2048):
    y = np.asarray(y).reshape(-1)
    step = max(1, y.shape[0] // nsamp)
    return y[::step].copy(), float(np.linalg.norm(y)), step


def ref_set(w):
    return hprop.build_full(w.dim, w.bound) if w.kind == "full" else hprop.build_hyperbolic(w.dim, w.bound)


def main():
    g = {}
    # ---------------------------------------------------------------- sets
    sizes = {}
    for dim in (1, 2, 3, 4, 5, 6, 8):
        for bound in (0, 1, 2, 5, 10, 31, 63):
            if dim >= 5 and bound > 31:
                continue
            sizes[f"{dim}_{bound}"] = hprop.build_hyperbolic(dim, bound).size
    for bound in (10, 20, 30, 40, 60, 80, 160):
        sizes[f"2_{bound}"] = hprop.build_hyperbolic(2, bound).size
    sizes["6_255"] = hprop.build_hyperbolic(6, 255).size
    sizes["8_255"] = hprop.build_hyperbolic(8, 255).size
    sizes["6_1023"] = hprop.build_hyperbolic(6, 1023).size
    g["hyp_sizes_keys"] = np.array(list(sizes.keys()))
    g["hyp_sizes_vals"] = np.array(list(sizes.values()), dtype=np.int64)
    for (kind, dim, bound) in [("hyp", 2, 12), ("hyp", 3, 8), ("hyp", 4, 10), ("hyp", 6, 63),
                               ("hyp", 8, 31), ("full", 3, 4), ("full", 2, 31)]:
        s = hprop.build_hyperbolic(dim, bound) if kind == "hyp" else hprop.build_full(dim, bound)
        key = f"set_{kind}_{dim}_{bound}"
        g[key + "_indices"] = s.indices.copy()
        for a in range(1, dim + 1):
            d, u = s.neighbor_ordinals(a)
            g[f"{key}_down{a}"] = d.copy()
            g[f"{key}_up{a}"] = u.copy()
    np.savez_compressed(OUT / "sets.npz", **g)
    print("sets done", flush=True)

    # ---------------------------------------------------------------- term lists
    t = {}
    for name, w in W.CONFIGS.items():
        for tt in ((0.0, 0.3) if name == "cfg4" else (0.0,)):
            ap = hprop.interpolate(hprop.custom_potential(w.evaluator, w.dim, L), w.degree, tt)
            key = f"{name}_t{tt}"
            t[key + "_degrees"] = ap.degrees.copy()
            t[key + "_coeffs"] = ap.coeffs.copy()
            t[key + "_fit"] = np.array(ap.fit_error)
    for dim, deg, tt, pot in [(2, 5, 0.4, "henon-heiles"), (3, 3, 0.4, "henon-heiles"), (2, 4, 0.0, "torsional"),
                              (4, 7, 0.9, "henon-heiles")]:
        spec = hprop.smooth_remainder(hprop.potential_by_name(pot, dim))
        ap = hprop.interpolate(spec, deg, tt)
        key = f"{pot}_{dim}_{deg}_{tt}"
        t[key + "_degrees"] = ap.degrees.copy()
        t[key + "_coeffs"] = ap.coeffs.copy()
    np.savez_compressed(OUT / "terms.npz", **t)
    print("terms done", flush=True)

    # ---------------------------------------------------------------- matvecs
    m = {}
    rng = np.random.default_rng(20240817)
    for dim, bound, axis in [(1, 12, 1), (2, 10, 1), (2, 10, 2), (3, 6, 2)]:
        s = hprop.build_hyperbolic(dim, bound)
        v = rng.standard_normal(s.size)
        key = f"coord_{dim}_{bound}_{axis}"
        m[key + "_in"] = v
        m[key + "_out"] = hprop.direct_op(s, axis, hprop.CoeffVector(s, v)).data
    s = hprop.build_hyperbolic(2, 12)
    v = rng.standard_normal(s.size)
    m["cheb_in"] = v
    for deg in (0, 1, 2, 5, 8):
        m[f"cheb_{deg}_out"] = hprop.cheb_of_coordinate_apply(s, 1, deg, 16.0, hprop.CoeffVector(s, v)).data
    # whole-surrogate cases of the reference tests (hyperbolic sets)
    for dim, bound, degree, pot in [(2, 12, 5, "henon-heiles"), (3, 8, 3, "henon-heiles"), (2, 12, 5, "torsional"),
                                    (4, 10, 7, "henon-heiles")]:
        s = hprop.build_hyperbolic(dim, bound)
        spec = hprop.smooth_remainder(hprop.potential_by_name(pot, dim))
        ap = hprop.interpolate(spec, degree, time=0.4)
        v = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
        appl = ref_fa.get_applier(s)
        key = f"poly_{pot}_{dim}_{bound}_{degree}"
        m[key + "_in"] = v
        m[key + "_degrees"] = ap.degrees.copy()
        m[key + "_coeffs"] = ap.coeffs.copy()
        m[key + "_out"] = appl.apply_polynomial(ap, v)
        m[key + "_ham"] = appl.apply_hamiltonian(ap, v)
        m[key + "_sq"] = appl.apply_square_sum(v)
        order = list(range(1, dim + 1))
        m[key + "_order_fwd"] = appl.apply_polynomial(ap, v, axis_order=order)
    # configuration workloads (full size where small, scaled otherwise)
    cases = {"cfg1": W.CONFIGS["cfg1"], "cfg2": W.CONFIGS["cfg2"],
             "cfg3s": W.CONFIGS["cfg3"].scaled(255, "cfg3s"), "cfg4s": W.CONFIGS["cfg4"].scaled(15, "cfg4s"),
             "cfg5s": W.CONFIGS["cfg5"].scaled(63, "cfg5s")}
    for name, w in cases.items():
        s = ref_set(w)
        c = W.coefficients(w, None if w.kind == "full" else s.indices)
        ap = hprop.interpolate(hprop.custom_potential(w.evaluator, w.dim, L), w.degree, 0.3 if "cfg4" in name else 0.0)
        appl = ref_fa.get_applier(s)
        vecs = c if c.ndim == 2 else c[None, :]
        outs = np.stack([appl.apply_polynomial(ap, v) for v in vecs[:4]])
        hams = np.stack([appl.apply_hamiltonian(ap, v) for v in vecs[:1]])
        for i in range(outs.shape[0]):
            samp, nrm, step = sketch(outs[i])
            m[f"{name}_poly{i}_samp"], m[f"{name}_poly{i}_norm"], m[f"{name}_poly{i}_step"] = samp, nrm, step
        samp, nrm, step = sketch(hams[0])
        m[f"{name}_ham_samp"], m[f"{name}_ham_norm"], m[f"{name}_ham_step"] = samp, nrm, step
        samp, nrm, step = sketch(vecs[0])
        m[f"{name}_in_samp"], m[f"{name}_in_norm"], m[f"{name}_in_step"] = samp, nrm, step
        if s.size <= 4096:
            m[f"{name}_poly0_full"] = outs[0]
            m[f"{name}_ham_full"] = hams[0]
        print(name, "matvec done", flush=True)
    np.savez_compressed(OUT / "matvec.npz", **m)

    # ---------------------------------------------------------------- krylov / propagation
    p = {}
    alpha = np.array([1.0, 2.5, -0.3, 4.0, 0.7, 3.3, 1.1])
    beta = np.array([0.5, 0.2, 1.5, 0.01, 0.8, 0.3])
    d, z = ref_kp.tridiag_eigh(alpha, beta)
    p["tri_alpha"], p["tri_beta"], p["tri_d"], p["tri_z"] = alpha, beta, d, z
    p["tri_col"] = ref_kp.expm_tridiag_column(alpha, beta, 0.37)
    runs = [("cfg1", W.CONFIGS["cfg1"], 100, 0.01, "midpoint"),
            ("cfg1gl2", W.CONFIGS["cfg1"], 10, 0.01, "gl2"),
            ("cfg3s", W.CONFIGS["cfg3"].scaled(255, "cfg3s"), 20, 0.001, "midpoint"),
            ("cfg4s", W.CONFIGS["cfg4"].scaled(15, "cfg4s"), 50, 0.005, "midpoint")]
    for name, w, nsteps, dt, scheme in runs:
        s = ref_set(w)
        c = W.coefficients(w, None if w.kind == "full" else s.indices)
        fh = hprop.FastHamiltonian(s, hprop.custom_potential(w.evaluator, w.dim, L), w.degree)
        fac = ref_kp.lanczos(fh.matvec_at(0.0), c, 7)
        p[f"{name}_lz_alpha"], p[f"{name}_lz_beta"] = fac.alpha, fac.beta
        y = ref_kp.propagate_magnus(ref_kp.MagnusScheme.from_name(scheme), fh.matvec_at, c, 0.0, nsteps * dt,
                                    nsteps, 7)
        samp, nrm, step = sketch(y)
        p[f"{name}_prop_samp"], p[f"{name}_prop_norm"], p[f"{name}_prop_step"] = samp, nrm, step
        if s.size <= 4096:
            p[f"{name}_prop_full"] = y
        print(name, "propagation done", flush=True)
    np.savez_compressed(OUT / "propagate.npz", **p)


if __name__ == "__main__":
    main()

"""Config-size golden fixtures, produced by running the REFERENCE itself.

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py [part ...]

Parts (each appends to tests/golden/configs.npz, so they can run separately):

* ``cfg3s255``  -- cfg3's potential on build_hyperbolic(6, 255), 200 midpoint
  steps at dt = 0.001 (the named cfg3 run: 200 steps on the
  scaled set), m = 7;
* ``cfg3s1023`` -- the same 200 steps on build_hyperbolic(6, 1023) (n = 611,556);
* ``cfg5full``  -- one vector (row 0 of the seeded 32-vector batch) of the
  full-size cfg5 set build_hyperbolic(8, 4095): ``apply_polynomial``;
* ``cfg3full``  -- the full-size cfg3 set build_hyperbolic(6, 16383)
  (n = 35,920,101): one ``apply_polynomial`` and one midpoint Magnus step
  (dt = 0.001) through ``FastHamiltonian.matvec_at``;
* ``cfg4s31``   -- cfg4's time-dependent potential on build_full(4, 31)
  (1,048,576 coefficients): the named 50-step run at dt = 0.005.

Reference calls: ``PolynomialApplier.apply_polynomial`` (fast_apply.py:110-164),
``propagate_magnus`` (krylov_propagator.py:247-263) with
``FastHamiltonian(iset, custom_potential(W, N, 16), R).matvec_at``
(error_lab.py:154-185).  Inputs are the seeded vectors of
``paper_1403_3511_b200.workloads`` (BLAS-free, identical on every host).

Large outputs are stored as a sketch: the first HEAD entries (where the
decaying coefficients are largest), every s-th entry (NSAMP of them, spread
over the whole vector) and the 2-norm.  The GPU tests compare the default
device evaluators against these at rel. L2 <= 1e-12.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import hprop  # noqa: E402  (the reference)
from hprop import fast_apply as ref_fa  # noqa: E402
from hprop import krylov_propagator as ref_kp  # noqa: E402

from paper_1403_3511_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "configs.npz"
L = W.HALFWIDTH
HEAD = 4096
NSAMP = 65536


def sketch(prefix: str, y: np.ndarray, rec: dict) -> None:
    y = np.asarray(y).reshape(-1)
    step = max(1, y.shape[0] // NSAMP)
    rec[prefix + "_head"] = y[:HEAD].copy()
    rec[prefix + "_samp"] = y[::step].copy()
    rec[prefix + "_step"] = np.int64(step)
    rec[prefix + "_norm"] = np.float64(np.linalg.norm(y))
    rec[prefix + "_n"] = np.int64(y.shape[0])


def save(rec: dict) -> None:
    old = dict(np.load(OUT)) if OUT.exists() else {}
    old.update(rec)
    np.savez_compressed(OUT, **old)


def fast_ham(w, s):
    return hprop.FastHamiltonian(s, hprop.custom_potential(w.evaluator, w.dim, L), w.degree)


def part_cfg3_scaled(bound: int) -> None:
    t0 = time.time()
    w = W.CONFIGS["cfg3"].scaled(bound, f"cfg3s{bound}")
    s = hprop.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, s.indices)
    fh = fast_ham(w, s)
    rec = {}
    norms = []

    def cb(k, t, y):
        norms.append(float(np.linalg.norm(y)))

    y = ref_kp.propagate_magnus(ref_kp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 200 * 0.001, 200,
                                7, callback=cb)
    key = f"cfg3s{bound}_prop200"
    sketch(key, y, rec)
    rec[key + "_norms"] = np.array(norms)
    if s.size <= 200_000:
        rec[key + "_full"] = y
    save(rec)
    print(key, s.size, f"{time.time() - t0:.1f}s", flush=True)


def part_cfg5_full() -> None:
    t0 = time.time()
    w = W.CONFIGS["cfg5"]
    s = hprop.build_hyperbolic(w.dim, w.bound)
    print("cfg5 set", s.size, f"{time.time() - t0:.1f}s", flush=True)
    c0 = W.coefficients_row(w, s.indices, 0)
    ap = hprop.interpolate(hprop.custom_potential(w.evaluator, w.dim, L), w.degree, 0.0)
    appl = ref_fa.get_applier(s)
    print("cfg5 tables", f"{time.time() - t0:.1f}s", flush=True)
    y = appl.apply_polynomial(ap, c0)
    rec = {}
    sketch("cfg5full_poly0", y, rec)
    sketch("cfg5full_in0", c0, rec)
    save(rec)
    print("cfg5full", f"{time.time() - t0:.1f}s", flush=True)


def part_cfg3_full() -> None:
    t0 = time.time()
    w = W.CONFIGS["cfg3"]
    s = hprop.build_hyperbolic(w.dim, w.bound)
    print("cfg3 set", s.size, f"{time.time() - t0:.1f}s", flush=True)
    c = W.coefficients(w, s.indices)
    ap = hprop.interpolate(hprop.custom_potential(w.evaluator, w.dim, L), w.degree, 0.0)
    appl = ref_fa.get_applier(s)
    print("cfg3 tables", f"{time.time() - t0:.1f}s", flush=True)
    y = appl.apply_polynomial(ap, c)
    rec = {}
    sketch("cfg3full_poly", y, rec)
    sketch("cfg3full_in", c, rec)
    save(rec)
    del y
    print("cfg3full poly", f"{time.time() - t0:.1f}s", flush=True)
    fh = fast_ham(w, s)
    y, fac = ref_kp.magnus_step(ref_kp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.001, 7)
    rec = {}
    sketch("cfg3full_step1", y, rec)
    rec["cfg3full_step1_alpha"] = np.asarray(fac.alpha)
    rec["cfg3full_step1_beta"] = np.asarray(fac.beta)
    save(rec)
    print("cfg3full step", f"{time.time() - t0:.1f}s", flush=True)


def part_cfg4_scaled() -> None:
    t0 = time.time()
    w = W.CONFIGS["cfg4"].scaled(31, "cfg4s31")
    s = hprop.build_full(w.dim, w.bound)
    c = W.coefficients(w)
    fh = fast_ham(w, s)
    y = ref_kp.propagate_magnus(ref_kp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 50 * 0.005, 50, 7)
    rec = {}
    sketch("cfg4s31_prop50", y, rec)
    save(rec)
    print("cfg4s31_prop50", s.size, f"{time.time() - t0:.1f}s", flush=True)


PARTS = {
    "cfg3s255": lambda: part_cfg3_scaled(255),
    "cfg3s1023": lambda: part_cfg3_scaled(1023),
    "cfg5full": part_cfg5_full,
    "cfg3full": part_cfg3_full,
    "cfg4s31": part_cfg4_scaled,
}


if __name__ == "__main__":
    for name in sys.argv[1:] or list(PARTS):
        PARTS[name]()

"""Pin the CPU oracle (oracle/hprop_oracle.py) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
itself (tests/golden/make_golden.py).  The oracle restates the reference
operation by operation, so most comparisons are bitwise.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import hprop_oracle as O
from paper_1403_3511_b200 import workloads as W
from paper_1403_3511_b200.potential_approx import custom_potential, interpolate, potential_by_name, smooth_remainder


# ---------------------------------------------------------------- sets

def test_hyperbolic_sizes_match_reference(golden):
    g = golden["sets"]
    for key, val in zip(g["hyp_sizes_keys"], g["hyp_sizes_vals"]):
        dim, bound = map(int, str(key).split("_"))
        assert O.hyperbolic_size_table(dim, bound) == val
        if val < 200_000:
            assert O.hyperbolic_indices(dim, bound).shape[0] == val


def test_known_sizes_dim2():
    # tests/test_index_set.py:19 of the reference
    known = {10: 29, 20: 70, 30: 113, 40: 160, 60: 263, 80: 373, 160: 846}
    for bound, size in known.items():
        assert O.hyperbolic_indices(2, bound).shape[0] == size


@pytest.mark.parametrize("dim,bound", [(1, 7), (2, 12), (3, 8), (4, 10), (5, 6)])
def test_level_synchronous_enumeration_equals_recursion(dim, bound):
    assert np.array_equal(O.hyperbolic_indices(dim, bound), O.hyperbolic_indices_recursive(dim, bound))


def test_set_indices_and_neighbor_tables_bitexact(golden):
    g = golden["sets"]
    for key in [k for k in g if k.endswith("_indices")]:
        _, kind, dim, bound, _ = key.split("_")
        dim, bound = int(dim), int(bound)
        idx = O.hyperbolic_indices(dim, bound) if kind == "hyp" else O.full_indices(dim, bound)
        assert np.array_equal(idx, g[key]), key
        tabs = O.neighbor_tables(idx)
        box = O.box_neighbor_tables((bound + 1,) * dim) if kind == "full" else None
        for a in range(1, dim + 1):
            base = key[: -len("_indices")]
            assert np.array_equal(tabs[a - 1][0], g[f"{base}_down{a}"])
            assert np.array_equal(tabs[a - 1][1], g[f"{base}_up{a}"])
            if box is not None:
                assert np.array_equal(box[a - 1][0], g[f"{base}_down{a}"])
                assert np.array_equal(box[a - 1][1], g[f"{base}_up{a}"])


# ---------------------------------------------------------------- term lists

def test_interpolation_term_lists_bitexact(golden):
    t = golden["terms"]
    for name, w in W.CONFIGS.items():
        for tt in ((0.0, 0.3) if name == "cfg4" else (0.0,)):
            key = f"{name}_t{tt}"
            ap = O.interpolate(w.evaluator, w.dim, W.HALFWIDTH, w.degree, tt)
            mine = interpolate(custom_potential(w.evaluator, w.dim, W.HALFWIDTH), w.degree, tt)
            assert ap.coeffs.shape[0] == W.EXPECTED_NTERMS[name]
            for obj in (ap, mine):
                assert np.array_equal(obj.degrees, t[key + "_degrees"])
                assert np.array_equal(obj.coeffs, t[key + "_coeffs"])
                assert obj.fit_error == float(t[key + "_fit"])


def test_named_potential_term_lists(golden):
    t = golden["terms"]
    for key in [k for k in t if k.endswith("_degrees") and not k.startswith("cfg")]:
        pot, dim, deg, tt, _ = key.split("_")
        spec = smooth_remainder(potential_by_name(pot, int(dim)))
        mine = interpolate(spec, int(deg), float(tt))
        assert np.array_equal(mine.degrees, t[key])
        assert np.array_equal(mine.coeffs, t[key.replace("_degrees", "_coeffs")])


# ---------------------------------------------------------------- matvec

def test_coordinate_and_cheb_bitexact(golden):
    m = golden["matvec"]
    for key in [k for k in m if k.startswith("coord_") and k.endswith("_in")]:
        _, dim, bound, axis, _ = key.split("_")
        appl = O.applier_for_set(O.hyperbolic_indices(int(dim), int(bound)))
        assert np.array_equal(appl.coordinate(int(axis), m[key]), m[key.replace("_in", "_out")])
    appl = O.applier_for_set(O.hyperbolic_indices(2, 12))
    for deg in (0, 1, 2, 5, 8):
        assert np.array_equal(appl.cheb_apply(1, deg, 16.0, m["cheb_in"]), m[f"cheb_{deg}_out"])


def test_polynomial_hamiltonian_square_bitexact(golden):
    m = golden["matvec"]
    for key in [k for k in m if k.startswith("poly_") and k.endswith("_in")]:
        base = key[:-3]
        _, pot, dim, bound, degree = base.split("_")
        appl = O.applier_for_set(O.hyperbolic_indices(int(dim), int(bound)))
        degs, cf, v = m[base + "_degrees"], m[base + "_coeffs"], m[key]
        assert np.array_equal(appl.polynomial(degs, cf, 16.0, v), m[base + "_out"])
        assert np.array_equal(appl.hamiltonian(degs, cf, 16.0, v), m[base + "_ham"])
        assert np.array_equal(appl.square_sum(v), m[base + "_sq"])
        order = list(range(1, int(dim) + 1))
        assert np.array_equal(appl.polynomial(degs, cf, 16.0, v, axis_order=order), m[base + "_order_fwd"])


CASES = {"cfg1": ("cfg1", None), "cfg2": ("cfg2", None), "cfg3s": ("cfg3", 255), "cfg4s": ("cfg4", 15),
         "cfg5s": ("cfg5", 63)}


@pytest.mark.parametrize("name", list(CASES))
def test_config_matvec_sketches(golden, name):
    m = golden["matvec"]
    base, bound = CASES[name]
    w = W.CONFIGS[base] if bound is None else W.CONFIGS[base].scaled(bound, name)
    if w.kind == "full":
        appl = O.applier_for_full(w.dim, w.bound)
        idx = None
    else:
        idx = O.hyperbolic_indices(w.dim, w.bound)
        appl = O.applier_for_set(idx)
    c = W.coefficients(w, idx)
    vecs = c if c.ndim == 2 else c[None]
    step = int(m[f"{name}_in_step"])
    assert np.array_equal(vecs[0][::step], m[f"{name}_in_samp"])
    ap = O.interpolate(w.evaluator, w.dim, W.HALFWIDTH, w.degree, 0.3 if "cfg4" in name else 0.0)
    for i in range(min(vecs.shape[0], 4)):
        y = appl.polynomial(ap.degrees, ap.coeffs, W.HALFWIDTH, vecs[i])
        assert np.array_equal(y[::step], m[f"{name}_poly{i}_samp"])
        assert np.linalg.norm(y) == pytest.approx(float(m[f"{name}_poly{i}_norm"]), rel=1e-14)
    yh = appl.hamiltonian(ap.degrees, ap.coeffs, W.HALFWIDTH, vecs[0])
    assert np.array_equal(yh[::step], m[f"{name}_ham_samp"])


def test_slab_box_reproduces_interior_rows():
    """The sharded/sampled oracle (a j1-slab with an r1-plane halo) equals the full cube inside."""
    w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
    ap = O.interpolate(w.evaluator, w.dim, W.HALFWIDTH, w.degree, 0.3)
    c = W.coefficients(w)
    full = O.applier_for_full(w.dim, w.bound).polynomial(ap.degrees, ap.coeffs, 16.0, c)
    side = w.bound + 1
    plane = side ** (w.dim - 1)
    r1 = int(ap.degrees[:, 0].max())
    for lo, hi in [(0, 3), (3, 7), (7, 12)]:
        blo, bhi = max(0, lo - r1), min(side, hi + r1)
        slab = O.applier_for_slab(w.dim, w.bound, blo, bhi)
        y = slab.polynomial(ap.degrees, ap.coeffs, 16.0, c[blo * plane:bhi * plane])
        got = y[(lo - blo) * plane:(hi - blo) * plane]
        assert np.array_equal(got, full[lo * plane:hi * plane])


# ---------------------------------------------------------------- krylov

def test_tridiag_and_expm_bitexact(golden):
    p = golden["propagate"]
    d, z = O.tridiag_eigh(p["tri_alpha"], p["tri_beta"])
    assert np.array_equal(d, p["tri_d"]) and np.array_equal(z, p["tri_z"])
    assert np.array_equal(O.expm_tridiag_column(p["tri_alpha"], p["tri_beta"], 0.37), p["tri_col"])


@pytest.mark.parametrize("name,base,bound,nsteps,dt,scheme", [
    ("cfg1", "cfg1", None, 100, 0.01, "midpoint"),
    ("cfg1gl2", "cfg1", None, 10, 0.01, "gl2"),
    ("cfg3s", "cfg3", 255, 20, 0.001, "midpoint"),
])
def test_propagation_matches_reference(golden, name, base, bound, nsteps, dt, scheme):
    p = golden["propagate"]
    w = W.CONFIGS[base] if bound is None else W.CONFIGS[base].scaled(bound, name)
    if w.kind == "full":
        appl, idx = O.applier_for_full(w.dim, w.bound), None
    else:
        idx = O.hyperbolic_indices(w.dim, w.bound)
        appl = O.applier_for_set(idx)
    c = W.coefficients(w, idx)
    ham_at = O.hamiltonian_at(appl, w.evaluator, w.dim, W.HALFWIDTH, w.degree)
    fac = O.lanczos(ham_at(0.0), c, 7)
    assert rel_l2(fac.alpha, p[f"{name}_lz_alpha"]) < 1e-13
    assert rel_l2(fac.beta, p[f"{name}_lz_beta"]) < 1e-13
    y = O.propagate(scheme, ham_at, c, 0.0, nsteps * dt, nsteps, 7)
    step = int(p[f"{name}_prop_step"])
    assert rel_l2(y[::step], p[f"{name}_prop_samp"]) < 1e-12
    assert np.linalg.norm(y) == pytest.approx(float(p[f"{name}_prop_norm"]), rel=1e-12)

"""GPU matvec parity: the sm_100a kernels vs the reference (golden) and the oracle.

Tolerances (north_star): reference-order mode is bitwise identical to numpy;
the default (regrouped / fused) evaluator is within relative L2 1e-12.
"""

import math
import warnings

import numpy as np
import pytest

from conftest import rel_l2
from oracle import hprop_oracle as O
from paper_1403_3511_b200 import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def hp():
    import paper_1403_3511_b200 as hp

    return hp


def _approx(degs, coeffs, dim, L=16.0, degree=None):
    from paper_1403_3511_b200.potential_approx import ChebApprox

    degs = np.asarray(degs)
    return ChebApprox(dim, int(degree if degree is not None else (degs.max() if degs.size else 0)), L, 0.0,
                      degs, np.asarray(coeffs), 0.0)


# ---------------------------------------------------------------- dense oracle (reference test helpers)

def dense_coordinate(iset, axis):
    n = iset.size
    mat = np.zeros((n, n))
    for i, row in enumerate(iset.indices.tolist()):
        k = row[axis - 1]
        below = list(row)
        below[axis - 1] = k - 1
        if k > 0 and tuple(below) in iset:
            mat[i, iset.position(tuple(below))] = math.sqrt(k / 2.0)
        above = list(row)
        above[axis - 1] = k + 1
        if tuple(above) in iset:
            mat[i, iset.position(tuple(above))] = math.sqrt((k + 1) / 2.0)
    return mat


def cheb_of_matrix(mat, deg):
    t0 = np.eye(mat.shape[0])
    if deg == 0:
        return t0
    t1 = mat
    for _ in range(deg - 1):
        t0, t1 = t1, 2.0 * mat @ t1 - t0
    return t1


def dense_surrogate(iset, approx):
    xs = [dense_coordinate(iset, a) / approx.halfwidth for a in range(1, iset.dim + 1)]
    out = np.zeros((iset.size, iset.size))
    for row, alpha in approx.terms:
        term = np.eye(iset.size)
        for a in range(1, iset.dim + 1):
            if row[a - 1] > 0:
                term = term @ cheb_of_matrix(xs[a - 1], row[a - 1])
        out += alpha * term
    return out


# ---------------------------------------------------------------- coordinate / chebyshev

def test_coordinate_bitexact_golden(hp, golden):
    m = golden["matvec"]
    for key in [k for k in m if k.startswith("coord_") and k.endswith("_in")]:
        _, dim, bound, axis, _ = key.split("_")
        s = hp.build_hyperbolic(int(dim), int(bound))
        got = hp.direct_op(s, int(axis), hp.CoeffVector(s, m[key])).data
        assert np.array_equal(got, m[key.replace("_in", "_out")]), key


@pytest.mark.parametrize("dim,bound,axis", [(1, 12, 1), (2, 10, 1), (2, 10, 2), (3, 6, 2)])
def test_coordinate_matches_coupling_rule(hp, dim, bound, axis, rng):
    s = hp.build_hyperbolic(dim, bound)
    v = rng.standard_normal(s.size)
    got = hp.direct_op(s, axis, hp.CoeffVector(s, v)).data
    assert np.max(np.abs(got - dense_coordinate(s, axis) @ v)) < 1e-14


def test_coordinate_respects_pruned_neighbors(hp):
    s = hp.build_hyperbolic(2, 10)
    e = np.zeros(s.size)
    e[s.position((2, 2))] = 1.0
    out = hp.direct_op(s, 1, hp.CoeffVector(s, e)).data
    assert out[s.position((1, 2))] == pytest.approx(1.0)
    assert np.count_nonzero(out) == 1


def test_cheb_bitexact_golden(hp, golden):
    m = golden["matvec"]
    s = hp.build_hyperbolic(2, 12)
    for deg in (0, 1, 2, 5, 8):
        got = hp.cheb_of_coordinate_apply(s, 1, deg, 16.0, hp.CoeffVector(s, m["cheb_in"])).data
        assert np.array_equal(got, m[f"cheb_{deg}_out"]), deg


@pytest.mark.parametrize("deg", [0, 1, 2, 5, 8])
def test_cheb_matches_matrix_recurrence(hp, deg, rng):
    s = hp.build_hyperbolic(2, 12)
    v = rng.standard_normal(s.size)
    got = hp.cheb_of_coordinate_apply(s, 1, deg, 16.0, hp.CoeffVector(s, v)).data
    want = cheb_of_matrix(dense_coordinate(s, 1) / 16.0, deg) @ v
    assert np.max(np.abs(got - want)) < 1e-12


# ---------------------------------------------------------------- whole surrogate

def test_polynomial_golden(hp, golden):
    m = golden["matvec"]
    for key in [k for k in m if k.startswith("poly_") and k.endswith("_in")]:
        base = key[:-3]
        _, pot, dim, bound, degree = base.split("_")
        s = hp.build_hyperbolic(int(dim), int(bound))
        ap = _approx(m[base + "_degrees"], m[base + "_coeffs"], int(dim), degree=int(degree))
        appl = hp.get_applier(s)
        v = m[key]
        # reference order: bitwise
        assert np.array_equal(appl.apply_polynomial(ap, v, ref_order=True), m[base + "_out"]), base
        assert np.array_equal(appl.apply_hamiltonian(ap, v, ref_order=True), m[base + "_ham"]), base
        assert np.array_equal(appl.apply_square_sum(v), m[base + "_sq"]), base
        order = list(range(1, int(dim) + 1))
        assert np.array_equal(appl.apply_polynomial(ap, v, axis_order=order), m[base + "_order_fwd"])
        # default (regrouped) evaluator: within tolerance
        assert rel_l2(appl.apply_polynomial(ap, v), m[base + "_out"]) < TOL
        assert rel_l2(appl.apply_hamiltonian(ap, v), m[base + "_ham"]) < TOL


@pytest.mark.parametrize("dim,bound,degree,pot", [(1, 16, 7, "torsional"), (2, 12, 5, "torsional"),
                                                  (2, 12, 5, "henon-heiles"), (3, 8, 3, "henon-heiles")])
def test_matches_ordered_dense_product(hp, dim, bound, degree, pot, rng):
    s = hp.build_hyperbolic(dim, bound)
    ap = hp.interpolate(hp.smooth_remainder(hp.potential_by_name(pot, dim)), degree, time=0.4)
    v = hp.CoeffVector(s, rng.standard_normal(s.size))
    want = dense_surrogate(s, ap) @ v.data
    scale = max(np.max(np.abs(want)), 1.0)
    for ref in (False, True):
        got = hp.fast_algorithm(s, ap, v, ref_order=ref).data
        assert np.max(np.abs(got - want)) < 1e-13 * scale


def test_grouped_equals_per_term(hp, rng):
    for dim, bound in ((2, 30), (3, 12), (4, 10)):
        s = hp.build_hyperbolic(dim, bound)
        ap = hp.interpolate(hp.smooth_remainder(hp.henon_heiles_perturbed(dim)), 7, time=0.9)
        appl = hp.get_applier(s)
        v = rng.standard_normal(s.size)
        ordered = appl.apply_polynomial(ap, v, axis_order=list(range(dim, 0, -1)))
        for ref in (False, True):
            grouped = appl.apply_polynomial(ap, v, ref_order=ref)
            assert np.max(np.abs(grouped - ordered)) < 1e-14 * np.max(np.abs(ordered))


def test_linearity(hp):
    s = hp.build_hyperbolic(2, 10)
    ap = hp.interpolate(hp.torsional(2), 4)
    appl = hp.get_applier(s)
    for seed in range(10):
        gen = np.random.default_rng(seed)
        a = gen.standard_normal(s.size) + 1j * gen.standard_normal(s.size)
        b = gen.standard_normal(s.size)
        sc = complex(gen.uniform(-8, 8), gen.uniform(-8, 8))
        lhs = appl.apply_polynomial(ap, sc * a + b)
        rhs = sc * appl.apply_polynomial(ap, a) + appl.apply_polynomial(ap, b)
        assert np.max(np.abs(lhs - rhs)) < 1e-12 * max(np.max(np.abs(rhs)), 1.0)


def test_axis_order_full_vs_pruned(hp, rng):
    full = hp.build_full(2, 9)
    ap = hp.interpolate(hp.smooth_remainder(hp.henon_heiles_perturbed(2)), 3, time=0.5)
    v = hp.CoeffVector(full, rng.standard_normal(full.size))
    a = hp.fast_algorithm(full, ap, v, axis_order=(2, 1))
    b = hp.fast_algorithm(full, ap, v, axis_order=(1, 2))
    assert np.max(np.abs(a.data - b.data)) < 1e-13
    s = hp.build_hyperbolic(2, 12)
    v = hp.CoeffVector(s, rng.standard_normal(s.size))
    a = hp.fast_algorithm(s, ap, v, axis_order=(2, 1))
    b = hp.fast_algorithm(s, ap, v, axis_order=(1, 2))
    assert np.max(np.abs(a.data - b.data)) > 1e-9
    with pytest.raises(ValueError, match="permute"):
        hp.fast_algorithm(s, ap, v, axis_order=(1, 1))


def test_errors_and_warnings(hp, rng):
    s = hp.build_hyperbolic(2, 10)
    other = hp.build_hyperbolic(2, 12)
    ap = hp.interpolate(hp.torsional(2), 4)
    with pytest.raises(ValueError, match="different index set"):
        hp.fast_algorithm(s, ap, hp.CoeffVector(other, rng.standard_normal(other.size)))
    v = hp.CoeffVector(s, rng.standard_normal(s.size))
    with pytest.warns(UserWarning, match="exceeds half the basis bound"):
        hp.fast_algorithm(s, hp.interpolate(hp.torsional(2), 8), v)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        hp.fast_algorithm(s, hp.interpolate(hp.torsional(2), 5), v)
    f = hp.build_full(1, 6)
    bad = hp.ChebApprox(dim=1, degree=1, halfwidth=1.0, time=0.0, degrees=np.array([[1]]),
                        coeffs=np.array([1e308]), fit_error=0.0)
    with pytest.raises(RuntimeError, match="non-finite"):
        hp.fast_algorithm(f, bad, hp.CoeffVector(f, np.full(f.size, 1e3)))
    with pytest.raises(ValueError):
        hp.direct_op(s, 3, v)
    assert hp.get_applier(s) is hp.get_applier(s)


def test_hamiltonian_adds_oscillator_diagonal(hp, rng):
    s = hp.build_hyperbolic(2, 10)
    ap = hp.interpolate(hp.torsional(2), 4)
    v = hp.CoeffVector(s, rng.standard_normal(s.size))
    ham = hp.apply_hamiltonian(s, ap, v)
    pot = hp.fast_algorithm(s, ap, v)
    levels = (s.indices + 0.5).sum(axis=1)
    assert np.max(np.abs(ham.data - pot.data - levels * v.data)) < 1e-14


def test_batched_and_device_resident(hp, rng):
    import torch

    s = hp.build_hyperbolic(3, 20)
    ap = hp.interpolate(hp.smooth_remainder(hp.henon_heiles_perturbed(3)), 4, time=0.2)
    appl = hp.get_applier(s)
    V = rng.standard_normal((5, s.size)) + 1j * rng.standard_normal((5, s.size))
    Y = appl.apply_polynomial(ap, V)
    for b in range(5):
        assert np.array_equal(Y[b], appl.apply_polynomial(ap, V[b]))
    Yd = appl.apply_polynomial(ap, torch.from_numpy(V).cuda())
    assert Yd.is_cuda and np.array_equal(Yd.cpu().numpy(), Y)


@pytest.mark.parametrize("bound", [11, 20])
def test_batched_fused_fullgrid(hp, rng, bound):
    """A batch on the fused full-cube class (one single-pass launch per vector) equals the
    per-vector matvecs bit for bit and the oracle within 1e-12, on cubes and a j1-slab."""
    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4x")
    ap = w.approx(0.3)
    s = hp.build_full(w.dim, w.bound)
    oa = O.applier_for_full(w.dim, w.bound)
    V = rng.standard_normal((3, s.size)) + 1j * rng.standard_normal((3, s.size))
    appl = hp.get_applier(s)
    Y = appl.apply_hamiltonian(ap, V)
    for b in range(3):
        assert np.array_equal(Y[b], appl.apply_hamiltonian(ap, V[b]))
        assert rel_l2(Y[b], oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[b])) < TOL
    side = w.bound + 1
    lo, hi = 2, side - 1
    sl = hp.build_slab(w.dim, w.bound, lo, hi)
    X = np.ascontiguousarray(V[:, lo * side ** 3:hi * side ** 3])
    Ys = hp.get_applier(sl).apply_polynomial(ap, X)
    ob = O.applier_for_slab(w.dim, w.bound, lo, hi)
    for b in range(3):
        assert rel_l2(Ys[b], ob.polynomial(ap.degrees, ap.coeffs, 16.0, X[b])) < TOL


# ---------------------------------------------------------------- configuration workloads

CASES = {"cfg1": ("cfg1", None), "cfg2": ("cfg2", None), "cfg3s": ("cfg3", 255), "cfg4s": ("cfg4", 15),
         "cfg5s": ("cfg5", 63)}


def _build(hp, w):
    return hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)


@pytest.mark.parametrize("name", list(CASES))
def test_config_workloads_vs_golden(hp, golden, name):
    m = golden["matvec"]
    base, bound = CASES[name]
    w = W.CONFIGS[base] if bound is None else W.CONFIGS[base].scaled(bound, name)
    s = _build(hp, w)
    c = W.coefficients(w, None if w.kind == "full" else s.indices)
    vecs = c if c.ndim == 2 else c[None]
    tt = 0.3 if "cfg4" in name else 0.0
    t = golden["terms"]
    ap = _approx(t[f"{base}_t{tt}_degrees"], t[f"{base}_t{tt}_coeffs"], w.dim, degree=w.degree)
    appl = hp.get_applier(s)
    step = int(m[f"{name}_in_step"])
    assert np.array_equal(vecs[0][::step], m[f"{name}_in_samp"]), "seeded input differs from the golden run"
    nb = min(vecs.shape[0], 4)
    Y = appl.apply_polynomial(ap, vecs[:nb] if nb > 1 else vecs[0])
    Y = Y.reshape(nb, -1)
    Yr = appl.apply_polynomial(ap, vecs[:nb] if nb > 1 else vecs[0], ref_order=True).reshape(nb, -1)
    for i in range(nb):
        samp = m[f"{name}_poly{i}_samp"]
        assert np.array_equal(Yr[i][::step], samp), (name, i)
        assert rel_l2(Y[i][::step], samp) < TOL, (name, i)
        assert np.linalg.norm(Y[i]) == pytest.approx(float(m[f"{name}_poly{i}_norm"]), rel=TOL)
    H = appl.apply_hamiltonian(ap, vecs[0])
    assert rel_l2(H[::step], m[f"{name}_ham_samp"]) < TOL
    if f"{name}_poly0_full" in m:
        assert rel_l2(Y[0], m[f"{name}_poly0_full"]) < TOL
        assert np.array_equal(Yr[0], m[f"{name}_poly0_full"])


def test_cfg2_full_vs_oracle(hp):
    w = W.CONFIGS["cfg2"]
    s = hp.build_full(w.dim, w.bound)
    c = W.coefficients(w)
    ap = w.approx()
    want = O.applier_for_full(w.dim, w.bound).polynomial(ap.degrees, ap.coeffs, 16.0, c)
    got = hp.get_applier(s).apply_polynomial(ap, c)
    assert rel_l2(got, want) < TOL
    assert np.array_equal(hp.get_applier(s).apply_polynomial(ap, c, ref_order=True), want)


@pytest.mark.parametrize("bound", [3, 5, 11, 20])
def test_fused_fullgrid_sizes_and_slabs(hp, bound):
    """The fused two-pass N=4 evaluator (hp_fullgrid.cu) at ragged sizes, on cubes and j1-slabs."""
    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4x")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    oa = O.applier_for_full(w.dim, w.bound)
    s = hp.build_full(w.dim, w.bound)
    appl = hp.get_applier(s)
    assert rel_l2(appl.apply_polynomial(ap, c), oa.polynomial(ap.degrees, ap.coeffs, 16.0, c)) < TOL
    assert rel_l2(appl.apply_hamiltonian(ap, c), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, c)) < TOL
    side = w.bound + 1
    plane = side ** 3
    for lo, hi in [(0, side // 2), (side // 3, side), (1, max(2, side - 1))]:
        sl = hp.build_slab(w.dim, w.bound, lo, hi)
        ob = O.applier_for_slab(w.dim, w.bound, lo, hi)
        x = c[lo * plane:hi * plane]
        assert rel_l2(hp.get_applier(sl).apply_hamiltonian(ap, x), ob.hamiltonian(ap.degrees, ap.coeffs, 16.0, x)) < TOL


def _coupled_potential(c01, c02, c13, c03=0.0):
    """cfg4's potential with further pair couplings: x1 x2 (c01), x1 x3 (c02), x2 x4 (c13), x1 x4 (c03)."""
    def w(p, t):
        return (0.5 * (p * p).sum(axis=-1) + c01 * math.cos(2.0 * t) * p[:, 0] * p[:, 1] + c02 * p[:, 0] * p[:, 2]
                + c13 * p[:, 1] * p[:, 3] + c03 * p[:, 0] * p[:, 3] + 0.01 * (p ** 4).sum(axis=-1))
    return w


@pytest.mark.parametrize("cpl", [(0.0, 0.07, 0.0), (0.0, 0.0, 0.05), (0.1, 0.07, 0.05), (0.0, 0.0, 0.0, -0.06),
                                 (0.1, 0.07, 0.05, -0.06)], ids=["x1x3", "x2x4", "all", "x1x4", "all4"])
@pytest.mark.parametrize("bound", [5, 11, 20])
def test_fused_fullgrid_further_couplings(hp, rng, bound, cpl):
    """The single-pass quad kernel's wider class (k_fg_quad<MIX>: x1 x3 through the march-axis
    scatter, x2 x4 as an in-plane corner term) against the oracle: ragged cubes, j1-slabs, a
    batch, the oscillator, and the in-kernel rows of x^H A x."""
    import torch

    from paper_1403_3511_b200 import _native as nat
    from paper_1403_3511_b200.potential_approx import custom_potential, interpolate

    ap = interpolate(custom_potential(_coupled_potential(*cpl), 4, 16.0), 4, 0.3)
    side = bound + 1
    s = hp.build_full(4, bound)
    oa = O.applier_for_full(4, bound)
    appl = hp.get_applier(s)
    V = rng.standard_normal((2, s.size)) + 1j * rng.standard_normal((2, s.size))
    Y = appl.apply_polynomial(ap, V)
    for b in range(2):
        assert rel_l2(Y[b], oa.polynomial(ap.degrees, ap.coeffs, 16.0, V[b])) < TOL
    assert rel_l2(appl.apply_hamiltonian(ap, V[0]), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[0])) < TOL
    plane = side ** 3
    for lo, hi in [(0, side // 2), (side // 3, side), (1, max(2, side - 1))]:
        sl = hp.build_slab(4, bound, lo, hi)
        ob = O.applier_for_slab(4, bound, lo, hi)
        x = np.ascontiguousarray(V[1][lo * plane:hi * plane])
        assert rel_l2(hp.get_applier(sl).apply_hamiltonian(ap, x), ob.hamiltonian(ap.degrees, ap.coeffs, 16.0, x)) < TOL
    # plane ranges with the fused dot (the evaluator the Lanczos loop uses)
    x = torch.from_numpy(V[0]).cuda()
    y = torch.empty_like(x)
    dot = torch.zeros(2, dtype=torch.float64, device="cuda")
    cuts = [0, side // 3, side // 3 + 1, side]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        assert appl.apply_planes_into(ap, x, y, lo, hi, nat.HP_ADD_OSC, dot=dot)
    want = torch.vdot(x, y)
    assert abs(complex(dot[0].item(), dot[1].item()) - complex(want)) <= 1e-13 * abs(complex(want))
    assert rel_l2(y.cpu().numpy(), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[0])) < TOL


@pytest.mark.parametrize("bound", [5, 11, 20])
def test_fused_fullgrid_residual_pair_couplings(hp, rng, bound, monkeypatch):
    """Pair couplings whose corner taps the single-pass kernel does not stage (x1 x4, x2 x3,
    x3 x4) are added by the streaming second pass k_fg_pairs behind it: a general quadratic
    coupling matrix on N = 4 cubes and slabs against the oracle, and through the Lanczos loop
    (which forms its own <v, A v> then)."""
    from paper_1403_3511_b200.potential_approx import custom_potential, interpolate

    cij = {(0, 1): 0.1, (0, 2): 0.07, (0, 3): -0.04, (1, 2): 0.06, (1, 3): 0.05, (2, 3): -0.03}

    def w(p, t):
        out = 0.5 * (p * p).sum(axis=-1) + 0.01 * (p ** 4).sum(axis=-1)
        for (a, b), c in cij.items():
            out = out + c * p[:, a] * p[:, b]
        return out

    spec = custom_potential(w, 4, 16.0)
    ap = interpolate(spec, 4, 0.0)
    side = bound + 1
    s = hp.build_full(4, bound)
    oa = O.applier_for_full(4, bound)
    appl = hp.get_applier(s)
    V = rng.standard_normal((2, s.size)) + 1j * rng.standard_normal((2, s.size))
    Y = appl.apply_hamiltonian(ap, V)
    for b in range(2):
        assert rel_l2(Y[b], oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[b])) < TOL
    plane = side ** 3
    for lo, hi in [(0, side // 2), (side // 3, side)]:
        sl = hp.build_slab(4, bound, lo, hi)
        ob = O.applier_for_slab(4, bound, lo, hi)
        x = np.ascontiguousarray(V[1][lo * plane:hi * plane])
        assert rel_l2(hp.get_applier(sl).apply_polynomial(ap, x), ob.polynomial(ap.degrees, ap.coeffs, 16.0, x)) < TOL
    # plane ranges (no fused dot) and the host-streamed entry point run the second pass per range / chunk
    import torch

    from paper_1403_3511_b200 import _native as nat

    want = oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[0])
    x = torch.from_numpy(V[0]).cuda()
    y = torch.empty_like(x)
    cuts = [0, side // 3, side // 3 + 1, side]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        assert appl.apply_planes_into(ap, x, y, lo, hi, nat.HP_ADD_OSC)
    assert rel_l2(y.cpu().numpy(), want) < TOL
    monkeypatch.setenv("HP_STREAM_CHUNK", "3")
    xh = torch.from_numpy(V[0]).pin_memory()
    yh = torch.zeros_like(xh).pin_memory()
    appl.apply_host_into(ap, xh, yh, nat.HP_ADD_OSC)
    torch.cuda.synchronize()
    assert rel_l2(yh.numpy(), want) < TOL
    if bound == 11:
        c = V[0] / np.linalg.norm(V[0])
        fh = hp.FastHamiltonian(s, spec, 4)
        got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.01, 2, 7)
        want = O.propagate("midpoint", O.hamiltonian_at(oa, w, 4, 16.0, 4), c, 0.0, 0.01, 2, 7)
        assert rel_l2(got, want) < TOL


@pytest.mark.parametrize("bound", [7, 12])
def test_fused_part_plus_level_remainder(hp, rng, bound):
    """A polynomial outside the fused class on an N = 4 box (odd single-axis degrees, an x2^2 x3
    term, a triple product) is evaluated as fused part + level passes accumulated onto y
    (fullgrid_apply_split): cube, slab, batch, Hamiltonian, and two Magnus steps vs the oracle."""
    from paper_1403_3511_b200.potential_approx import custom_potential, interpolate

    def w(p, t):
        return (0.5 * (p * p).sum(axis=-1) + 0.01 * (p ** 4).sum(axis=-1) + 0.1 * p[:, 0] * p[:, 1]
                + 0.05 * p[:, 1] * p[:, 3] + 0.03 * p[:, 2] * p[:, 3] + 0.02 * p[:, 1] ** 2 * p[:, 2]
                - 0.015 * p[:, 0] ** 3 + 0.01 * p[:, 0] * p[:, 2] * p[:, 3])

    spec = custom_potential(w, 4, 16.0)
    ap = interpolate(spec, 4, 0.0)
    side = bound + 1
    s = hp.build_full(4, bound)
    oa = O.applier_for_full(4, bound)
    appl = hp.get_applier(s)
    V = rng.standard_normal((2, s.size)) + 1j * rng.standard_normal((2, s.size))
    Y = appl.apply_polynomial(ap, V)
    for b in range(2):
        assert rel_l2(Y[b], oa.polynomial(ap.degrees, ap.coeffs, 16.0, V[b])) < TOL
    assert rel_l2(appl.apply_hamiltonian(ap, V[0]), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, V[0])) < TOL
    plane = side ** 3
    lo, hi = 1, side - 2
    sl = hp.build_slab(4, bound, lo, hi)
    ob = O.applier_for_slab(4, bound, lo, hi)
    x = np.ascontiguousarray(V[1][lo * plane:hi * plane])
    assert rel_l2(hp.get_applier(sl).apply_hamiltonian(ap, x), ob.hamiltonian(ap.degrees, ap.coeffs, 16.0, x)) < TOL
    c = V[0] / np.linalg.norm(V[0])
    fh = hp.FastHamiltonian(s, spec, 4)
    got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.01, 2, 7)
    want = O.propagate("midpoint", O.hamiltonian_at(oa, w, 4, 16.0, 4), c, 0.0, 0.01, 2, 7)
    assert rel_l2(got, want) < TOL


@pytest.mark.slow
def test_cfg4_full_size_slab_vs_oracle(hp):
    """Full-size cfg4 (2.7e8 coefficients): GPU output on planes j1 in [62, 64) equals the oracle
    evaluated on the slab box [58, 68) (its r1 = 4 halo makes those planes exact)."""
    import torch

    w = W.CONFIGS["cfg4"]
    s = hp.build_full(w.dim, w.bound)
    c = W.coefficients(w)
    ap = w.approx(0.3)
    y = hp.get_applier(s).apply_polynomial(ap, torch.from_numpy(c).cuda())
    plane = (w.bound + 1) ** 3
    lo, hi, blo, bhi = 62, 64, 58, 68
    slab = O.applier_for_slab(w.dim, w.bound, blo, bhi)
    want = slab.polynomial(ap.degrees, ap.coeffs, 16.0, c[blo * plane:bhi * plane])
    got = y[lo * plane:hi * plane].cpu().numpy()
    assert rel_l2(got, want[(lo - blo) * plane:(hi - blo) * plane]) < TOL
    # linearity at full size
    y2 = hp.get_applier(s).apply_polynomial(ap, 2.0 * torch.from_numpy(c).cuda())
    assert float(torch.linalg.vector_norm(y2 - 2.0 * y) / torch.linalg.vector_norm(y)) < 1e-14


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_full_size_reduced_sets_vs_reference_order(hp, name):
    """Full-size cfg3 (3.6e7) / cfg5 (2.6e7) matvecs: the default level evaluator (line-blocked
    axis-1 order, batch) against the device run of the reference's own evaluation order --
    the program that is bitwise equal to the reference on every golden case -- within 1e-12;
    batched equals per-vector bit for bit; linearity."""
    import torch

    w = W.CONFIGS[name]
    s = hp.build_hyperbolic(w.dim, w.bound)
    ap = w.approx(0.0)
    appl = hp.get_applier(s)
    gen = np.random.default_rng(7)
    V = torch.from_numpy(gen.standard_normal((2, s.size)) + 1j * gen.standard_normal((2, s.size))).cuda()
    Y = appl.apply_polynomial(ap, V)
    for b in range(2):
        yb = appl.apply_polynomial(ap, V[b].contiguous())
        assert torch.equal(Y[b], yb)
        yr = appl.apply_polynomial(ap, V[b].contiguous(), ref_order=True)
        assert float(torch.linalg.vector_norm(yb - yr) / torch.linalg.vector_norm(yr)) < TOL
    y2 = appl.apply_polynomial(ap, (V[0] * (0.5 - 2.0j)).contiguous())
    assert float(torch.linalg.vector_norm(y2 - (0.5 - 2.0j) * Y[0]) / torch.linalg.vector_norm(y2)) < 1e-14


@pytest.mark.parametrize("world", [2, 4])
def test_slab_shards_on_device(hp, world):
    """All ranks' slab shards in one process: device slab sets + the halo plan reproduce
    the full-cube fused matvec bitwise on every owned plane."""
    import torch

    from paper_1403_3511_b200.sharding import SlabShard, emulate_exchange

    w = W.CONFIGS["cfg4"].scaled(23, "cfg4y")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    full = hp.build_full(w.dim, w.bound)
    y_full = hp.get_applier(full).apply_polynomial(ap, c)
    shards = [SlabShard(w.dim, w.bound, r, world, halo=w.degree) for r in range(world)]
    geos = [s.geo for s in shards]
    boxes = []
    for g in geos:
        b = torch.zeros(g.box_size, dtype=torch.complex128, device="cuda")
        b[g.own_slice] = torch.from_numpy(c[g.lo * g.plane:g.hi * g.plane]).cuda()
        boxes.append(b)
    emulate_exchange(geos, boxes)
    got = np.zeros_like(y_full)
    for s, g, b in zip(shards, geos, boxes):
        assert np.array_equal(b.cpu().numpy(), c[g.blo * g.plane:g.bhi * g.plane])
        yb = torch.empty_like(b)
        hp.get_applier(s.set).apply_into(ap, b, yb)
        got[g.lo * g.plane:g.hi * g.plane] = yb[g.own_slice].cpu().numpy()
    assert np.array_equal(got, y_full)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_shards_from_host(hp, world):
    """SlabShard.apply_host (bench.py's sharded e2e leg): every rank streams its box of the host
    vector through hp_apply_polynomial_streamed; the owned planes equal the full-cube matvec."""
    import torch

    from paper_1403_3511_b200.sharding import SlabShard

    w = W.CONFIGS["cfg4"].scaled(31, "cfg4h")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    y_full = hp.get_applier(hp.build_full(w.dim, w.bound)).apply_polynomial(ap, c)
    got = np.zeros_like(y_full)
    for r in range(world):
        s = SlabShard(w.dim, w.bound, r, world, halo=w.degree)
        g = s.geo
        xh = torch.from_numpy(s.local_coefficients(W, w)).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        s.apply_host(hp.get_applier(s.set), ap, xh, yh)
        torch.cuda.synchronize()
        got[g.lo * g.plane:g.hi * g.plane] = yh[g.own_slice].numpy()
    assert rel_l2(got, y_full) < 1e-13


@pytest.mark.parametrize("world", [2, 3])
def test_slab_shards_overlapped(hp, world):
    """Overlapped shard schedule (interior planes while the halo is in flight, then the
    boundary planes): the interior pass reads owned planes only -- it is exact with poisoned
    (NaN) halo planes -- and the whole schedule reproduces the full-cube matvec bitwise."""
    import torch

    from paper_1403_3511_b200.sharding import SlabShard

    w = W.CONFIGS["cfg4"].scaled(31, "cfg4z")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    full = hp.build_full(w.dim, w.bound)
    y_full = hp.get_applier(full).apply_polynomial(ap, c)
    shards = [SlabShard(w.dim, w.bound, r, world, halo=w.degree) for r in range(world)]
    geos = [s.geo for s in shards]
    boxes = []
    for g in geos:
        b = torch.full((g.box_size,), complex("nan+nanj"), dtype=torch.complex128, device="cuda")
        b[g.own_slice] = torch.from_numpy(c[g.lo * g.plane:g.hi * g.plane]).cuda()
        boxes.append(b)

    def exchange(g, x):  # this rank's halo planes from the peers' owned planes
        for peer, _send, recv in g.exchanges():
            psend = [sl for p, sl, _ in geos[peer].exchanges() if p == g.rank][0]
            x[recv] = boxes[peer][psend]

    got = np.zeros_like(y_full)
    for s, g, b in zip(shards, geos, boxes):
        appl = hp.get_applier(s.set)
        ilo, ihi = s.interior()
        yb = torch.zeros_like(b)
        assert appl.apply_planes_into(ap, b, yb, ilo, ihi)  # halos still NaN
        torch.cuda.synchronize()
        own0 = (g.lo - g.blo)
        sl = slice((ilo - own0) * g.plane + g.lo * g.plane, (ihi - own0) * g.plane + g.lo * g.plane)
        assert np.array_equal(yb[ilo * g.plane:ihi * g.plane].cpu().numpy(), y_full[sl])
        yb2 = torch.empty_like(b)
        s.apply_polynomial(appl, ap, b, yb2, exchange=exchange)
        torch.cuda.synchronize()
        got[g.lo * g.plane:g.hi * g.plane] = yb2[g.own_slice].cpu().numpy()
    assert np.array_equal(got, y_full)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_shards_with_all_pair_couplings(hp, world):
    """The sharded matvec with a general quadratic coupling (every pair: four inside k_fg_quad, x2 x3
    and x3 x4 through the second pass per plane range): overlapped schedule with poisoned halos and
    the single-launch schedule both reproduce the full-cube matvec bit for bit."""
    import torch

    from paper_1403_3511_b200.potential_approx import custom_potential, interpolate
    from paper_1403_3511_b200.sharding import SlabShard

    cij = {(0, 1): 0.1, (0, 2): 0.07, (0, 3): -0.04, (1, 2): 0.06, (1, 3): 0.05, (2, 3): -0.03}

    def pot(p, t):
        out = 0.5 * (p * p).sum(axis=-1) + 0.01 * (p ** 4).sum(axis=-1)
        for (a, b), c in cij.items():
            out = out + c * p[:, a] * p[:, b]
        return out

    w = W.CONFIGS["cfg4"].scaled(27, "cfg4q")
    ap = interpolate(custom_potential(pot, 4, 16.0), 4, 0.0)
    c = W.coefficients(w)
    full = hp.build_full(w.dim, w.bound)
    y_full = hp.get_applier(full).apply_polynomial(ap, c)
    oa = O.applier_for_full(w.dim, w.bound)
    assert rel_l2(y_full, oa.polynomial(ap.degrees, ap.coeffs, 16.0, c)) < TOL
    shards = [SlabShard(w.dim, w.bound, r, world, halo=w.degree) for r in range(world)]
    geos = [s.geo for s in shards]
    boxes = []
    for g in geos:
        b = torch.full((g.box_size,), complex("nan+nanj"), dtype=torch.complex128, device="cuda")
        b[g.own_slice] = torch.from_numpy(c[g.lo * g.plane:g.hi * g.plane]).cuda()
        boxes.append(b)

    def exchange(g, x):  # this rank's halo planes from the peers' owned planes
        for peer, _send, recv in g.exchanges():
            psend = [sl for p, sl, _ in geos[peer].exchanges() if p == g.rank][0]
            x[recv] = boxes[peer][psend]

    for overlap in (True, False):
        got = np.zeros_like(y_full)
        for s, g, b in zip(shards, geos, boxes):
            appl = hp.get_applier(s.set)
            x = b.clone()
            yb = torch.empty_like(x)
            s.apply_polynomial(appl, ap, x, yb, exchange=exchange, overlap=overlap)
            torch.cuda.synchronize()
            got[g.lo * g.plane:g.hi * g.plane] = yb[g.own_slice].cpu().numpy()
        assert np.array_equal(got, y_full), overlap


@pytest.mark.parametrize("seed", range(32))
def test_random_term_structures_vs_oracle(hp, seed):
    """Fuzz the evaluator planners (level-fused cuts, fused full-cube classes, trie fallback):
    random sparse term lists on random hyperbolic / full sets, default mode vs the oracle's
    reference-order result, real and complex, batched, with and without the oscillator."""
    gen = np.random.default_rng(1000 + seed)
    dim = int(gen.integers(1, 6))
    kind = "full" if gen.random() < 0.4 else "hyperbolic"
    if kind == "full":
        bound = int(gen.integers(3, {1: 40, 2: 20, 3: 9, 4: 6, 5: 4}[dim]))
        s = hp.build_full(dim, bound)
        oa = O.applier_for_full(dim, bound)
    else:
        bound = int(gen.integers(2, 60))
        s = hp.build_hyperbolic(dim, bound)
        oa = O.applier_for_set(O.hyperbolic_indices(dim, bound))
    nterms = int(gen.integers(1, 30))
    maxdeg = int(gen.integers(1, 5))
    degs = gen.integers(0, maxdeg + 1, size=(nterms, dim))
    degs[gen.random((nterms, dim)) < 0.5] = 0
    degs = np.unique(degs, axis=0)
    coeffs = gen.uniform(-2, 2, degs.shape[0]) * 10.0 ** gen.uniform(-1, 2, degs.shape[0])
    ap = _approx(degs, coeffs, dim, degree=maxdeg)
    appl = hp.get_applier(s)
    for cplx in (True, False):
        v = gen.standard_normal(s.size) + (1j * gen.standard_normal(s.size) if cplx else 0.0)
        want = oa.polynomial(degs, coeffs, 16.0, v)
        assert rel_l2(appl.apply_polynomial(ap, v), want) < TOL, (dim, kind, bound, cplx)
        wh = oa.hamiltonian(degs, coeffs, 16.0, v)
        assert rel_l2(appl.apply_hamiltonian(ap, v), wh) < TOL
    V = gen.standard_normal((3, s.size)) + 1j * gen.standard_normal((3, s.size))
    Y = appl.apply_polynomial(ap, V)
    for b in range(3):
        assert rel_l2(Y[b], oa.polynomial(degs, coeffs, 16.0, V[b])) < TOL


@pytest.mark.parametrize("bound,chunk", [(11, 1), (11, 2), (11, 5), (20, 3), (20, 7), (20, 64)])
def test_streamed_host_matvec_matches_device(hp, bound, chunk, monkeypatch):
    """hp_apply_polynomial_streamed (host-resident vectors, j1-plane chunks overlapped with the
    kernels) gives bit-for-bit the device matvec, for chunkings that do and do not divide n0."""
    import torch

    monkeypatch.setenv("HP_STREAM_CHUNK", str(chunk))
    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4x")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    s = hp.build_full(w.dim, w.bound)
    appl = hp.get_applier(s)
    for flags in (0, 1):  # polynomial, Hamiltonian
        xd = torch.from_numpy(c).cuda()
        yd = torch.empty_like(xd)
        appl.apply_into(ap, xd, yd, flags)
        xh = torch.from_numpy(c).pin_memory()
        yh = torch.zeros_like(xh).pin_memory()
        appl.apply_host_into(ap, xh, yh, flags)
        torch.cuda.synchronize()
        assert torch.equal(yh, yd.cpu())
    oa = O.applier_for_full(w.dim, w.bound)
    assert rel_l2(yh.numpy(), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, c)) < TOL


def test_streamed_host_matvec_fallback_sets(hp):
    """Sets outside the fused class (hyperbolic, real vectors) take whole-vector copies."""
    import torch

    s = hp.build_hyperbolic(3, 12)
    ap = _approx(np.array([[0, 0, 0], [2, 0, 0], [1, 1, 0], [0, 0, 4]]), np.array([1.0, 0.5, -0.25, 0.1]), 3, degree=4)
    appl = hp.get_applier(s)
    gen = np.random.default_rng(7)
    for cplx in (True, False):
        v = gen.standard_normal(s.size) + (1j * gen.standard_normal(s.size) if cplx else 0.0)
        xh = torch.from_numpy(v).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        appl.apply_host_into(ap, xh, yh)
        torch.cuda.synchronize()
        assert np.array_equal(yh.numpy(), appl.apply_polynomial(ap, v))


def test_streamed_host_matvec_batch_and_flags(hp):
    """Batched vectors and the reference-order flag take the whole-copy route of the streamed
    entry point: results equal the device calls bit for bit."""
    import torch

    w = W.CONFIGS["cfg4"].scaled(7, "cfg4x")
    ap = w.approx(0.3)
    s = hp.build_full(w.dim, w.bound)
    appl = hp.get_applier(s)
    gen = np.random.default_rng(11)
    V = gen.standard_normal((2, s.size)) + 1j * gen.standard_normal((2, s.size))
    xh = torch.from_numpy(V).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    appl.apply_host_into(ap, xh, yh)
    torch.cuda.synchronize()
    assert np.array_equal(yh.numpy(), appl.apply_polynomial(ap, V))
    v = V[0].copy()
    xh1 = torch.from_numpy(v).pin_memory()
    yh1 = torch.empty_like(xh1).pin_memory()
    appl.apply_host_into(ap, xh1, yh1, 2)  # HP_REF_ORDER
    torch.cuda.synchronize()
    assert np.array_equal(yh1.numpy(), appl.apply_polynomial(ap, v, ref_order=True))
    with pytest.raises(ValueError):
        appl.apply_host_into(ap, xh1.cuda(), yh1)


_KERNEL_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1403_3511_b200 as hp
from oracle import hprop_oracle as O
from paper_1403_3511_b200 import workloads as W
worst = 0.0
for bound in (5, 11, 20):
    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4x")
    ap = w.approx(0.3)
    c = W.coefficients(w)
    oa = O.applier_for_full(w.dim, w.bound)
    appl = hp.get_applier(hp.build_full(w.dim, w.bound))
    for got, want in ((appl.apply_polynomial(ap, c), oa.polynomial(ap.degrees, ap.coeffs, 16.0, c)),
                      (appl.apply_hamiltonian(ap, c), oa.hamiltonian(ap.degrees, ap.coeffs, 16.0, c))):
        worst = max(worst, float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    side = w.bound + 1
    plane = side ** 3
    lo, hi = side // 3, side
    x = c[lo * plane:hi * plane]
    got = hp.get_applier(hp.build_slab(w.dim, w.bound, lo, hi)).apply_hamiltonian(ap, x)
    want = O.applier_for_slab(w.dim, w.bound, lo, hi).hamiltonian(ap.degrees, ap.coeffs, 16.0, x)
    worst = max(worst, float(np.linalg.norm(got - want) / np.linalg.norm(want)))
print(worst)
"""


@pytest.mark.parametrize("env", [{"HP_FG_QUAD": "0"}, {"HP_FG_BLOCK": "6,6,4"}], ids=["k_fg_single", "block_664"])
def test_alternate_single_pass_kernels(env):
    """The non-default single-pass configurations (selected once per process by environment, so
    run in a subprocess): k_fg_single (cubes with a side > 128) and k_fg_quad with 3-D tile blocks,
    on cubes and a j1-slab, against the oracle."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "-c", _KERNEL_SCRIPT, str(root)], env={**os.environ, **env},
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) < TOL


def test_device_entry_points_bounded_memory(hp):
    """A stepping loop hands apply_into / apply_host_into a new surrogate object every step
    (time-dependent W): device memory must not grow with the number of steps (the term-array
    cache is a small LRU, the workspace and staging buffers are shared)."""
    import torch

    w = W.CONFIGS["cfg4"].scaled(20, "cfg4m")
    s = hp.build_full(w.dim, w.bound)
    appl = hp.get_applier(s)
    x = torch.from_numpy(W.coefficients(w)).cuda()
    y = torch.empty_like(x)
    xh, yh = x.cpu().pin_memory(), torch.empty(x.shape, dtype=x.dtype).pin_memory()
    for k in range(3):
        appl.apply_into(w.approx(0.01 * k), x, y)
        appl.apply_host_into(w.approx(0.01 * k), xh, yh)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    for k in range(3, 60):
        appl.apply_into(w.approx(0.01 * k), x, y)
        appl.apply_host_into(w.approx(0.01 * k), xh, yh)
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - base < (1 << 20)
    assert torch.allclose(yh.cuda(), y, rtol=0, atol=0) or rel_l2(yh.numpy(), y.cpu().numpy()) < TOL


@pytest.mark.parametrize("bound", [11, 20])
def test_planes_fused_dot(hp, rng, bound):
    """hp_apply_polynomial_planes_dot: the in-kernel rows of x^H A x (formed by the symmetry of
    A, without a second read of x) summed over plane ranges equal the direct dot, on a cube and
    on a slab (owned planes only)."""
    import torch

    from paper_1403_3511_b200 import _native as nat

    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4d")
    ap = w.approx(0.3)
    s = hp.build_full(w.dim, w.bound)
    appl = hp.get_applier(s)
    side = w.bound + 1
    x = torch.from_numpy(rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)).cuda()
    y = torch.empty_like(x)
    dot = torch.zeros(2, dtype=torch.float64, device="cuda")
    cuts = [0, side // 3, side // 3 + 1, side]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        assert appl.apply_planes_into(ap, x, y, lo, hi, nat.HP_ADD_OSC, dot=dot)
    want = torch.vdot(x, y)
    got = complex(dot[0].item(), dot[1].item())
    assert abs(got - complex(want)) <= 1e-13 * abs(complex(want))
    # slab [2, side-2): the owned planes [6, side-6) of a box with a 4-plane halo on each side
    sl = hp.build_slab(w.dim, w.bound, 2, side - 2)
    xb = x[2 * side ** 3:(side - 2) * side ** 3].contiguous()
    yb = torch.empty_like(xb)
    dot.zero_()
    assert hp.get_applier(sl).apply_planes_into(ap, xb, yb, 4, side - 8, nat.HP_ADD_OSC, dot=dot)
    own = slice(4 * side ** 3, (side - 8) * side ** 3)
    yfull = y[2 * side ** 3:(side - 2) * side ** 3]
    assert torch.equal(yb[own], yfull[own])
    # owned rows only: sum over them of conj(x_p) . y_p is not symmetric on its own, but the
    # in-kernel rows (T_p + conj L_p) summed over every rank's owned planes are; here check that
    # the slab's owned-row partial matches the cube's partial over the same planes
    dot2 = torch.zeros(2, dtype=torch.float64, device="cuda")
    assert appl.apply_planes_into(ap, x, y, 6, side - 6, nat.HP_ADD_OSC, dot=dot2)
    assert torch.allclose(dot, dot2, rtol=1e-13, atol=0)


_PERM_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1403_3511_b200 as hp
from paper_1403_3511_b200 import workloads as W
out = []
for name, bound in (("cfg3", 255), ("cfg5", 63)):
    w = W.CONFIGS[name].scaled(bound, name + "p")
    s = hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, s.indices)
    out.append(hp.get_applier(s).apply_polynomial(w.approx(0.0), c))
np.save(sys.argv[2], np.concatenate([np.ravel(o) for o in out]))
"""


def test_level_line_order_bitwise(tmp_path):
    """The line-blocked traversal (HP_LEVEL_PERM, default axis 1) only reorders the level
    kernels' work: matvec outputs on scaled cfg3 / cfg5 sets equal the ordinal-order run
    (HP_LEVEL_PERM=0) bit for bit."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    outs = []
    for env in ({}, {"HP_LEVEL_PERM": "0"}, {"HP_LEVEL_PERM": "7"}):
        f = tmp_path / f"y{len(outs)}.npy"
        r = subprocess.run([sys.executable, "-c", _PERM_SCRIPT, str(root), str(f)], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])

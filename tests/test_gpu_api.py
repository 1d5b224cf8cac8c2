"""Reference-facing API behaviour on the device path: restrict/extend, index-set and coefficient
files, the propagation driver's contract (callback, argument checks, exact oscillator phases,
Magnus orders, Krylov convergence) and the square-sum routes.  Mirrors the behaviour the
reference's own tests pin (tests/test_index_set.py:117-165, tests/test_krylov_propagator.py:41-220,
tests/test_fast_apply.py:251-280); comparisons are against scipy / the oracle."""

import numpy as np
import pytest
import scipy.linalg

from conftest import rel_l2
from oracle import hprop_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hp():
    import paper_1403_3511_b200 as hp

    return hp


# ---------------------------------------------------------------- sets, vectors, files

def test_restrict_extend_roundtrip(hp):
    rng = np.random.default_rng(1)
    full, sub = hp.build_full(3, 9), hp.build_hyperbolic(3, 9)
    v = hp.CoeffVector(sub, rng.standard_normal(sub.size) + 1j * rng.standard_normal(sub.size))
    ext = hp.extend(v, full)
    assert ext.data.shape == (full.size,)
    assert np.array_equal(hp.restrict(ext, sub).data, v.data)
    member = {tuple(r) for r in sub.indices.tolist()}
    absent = np.array([tuple(r) not in member for r in full.indices.tolist()])
    assert np.all(ext.data[absent] == 0) and absent.sum() == full.size - sub.size


def test_restrict_extend_on_device_tensors(hp):
    import torch

    full, sub = hp.build_full(2, 12), hp.build_hyperbolic(2, 12)
    d = torch.arange(full.size, dtype=torch.float64, device="cuda").to(torch.complex128)
    r = hp.restrict(hp.CoeffVector(full, d), sub)
    assert r.data.is_cuda
    pos = sub.indices @ np.array([13, 1])
    assert np.array_equal(r.data.cpu().numpy(), np.arange(full.size, dtype=complex)[pos])
    e = hp.extend(r, full)
    assert e.data.is_cuda and np.array_equal(e.data.cpu().numpy()[pos], r.data.cpu().numpy())


def test_restrict_rejects_other_cube(hp):
    sub, wrong = hp.build_hyperbolic(2, 9), hp.build_full(2, 10)
    v = hp.CoeffVector(wrong, np.zeros(wrong.size))
    with pytest.raises(ValueError, match="mismatch"):
        hp.restrict(v, sub)
    with pytest.raises(ValueError, match="full cube"):
        hp.extend(hp.CoeffVector(sub, np.zeros(sub.size)), hp.build_hyperbolic(2, 9))


def test_coeff_vector_rejects_bad_data(hp):
    s = hp.build_full(1, 3)
    with pytest.raises(ValueError, match="shape"):
        hp.CoeffVector(s, np.zeros(3))
    with pytest.raises(ValueError, match="non-finite"):
        hp.CoeffVector(s, np.array([0.0, np.inf, 0.0, 0.0]))


def test_index_set_file_and_csv_roundtrip(hp, tmp_path):
    s = hp.build_hyperbolic(4, 11)
    hp.save_index_set(s, tmp_path / "set.txt")
    back = hp.load_index_set(tmp_path / "set.txt")
    assert back.dim == 4 and np.array_equal(back.indices, s.indices)
    rng = np.random.default_rng(2)
    v = hp.CoeffVector(s, rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size))
    v.write_csv(tmp_path / "c.csv")
    raw = (tmp_path / "c.csv").read_bytes()
    assert b"\r" not in raw and raw.startswith(b"k_1,k_2,k_3,k_4,re,im\n")
    got = hp.read_coeff_csv(tmp_path / "c.csv", s)
    assert np.array_equal(got.data, v.data)  # %.17g round-trips doubles exactly


# ---------------------------------------------------------------- propagation driver

def test_scheme_lookup(hp):
    assert hp.MagnusScheme.from_name("midpoint").order == 2
    assert hp.MagnusScheme.from_name("gl2").order == 4
    with pytest.raises(ValueError, match="unknown scheme"):
        hp.MagnusScheme.from_name("rk4")


def test_callback_and_zero_steps(hp):
    seen = []
    hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), lambda t: (lambda w: w), np.ones(3, complex),
                        0.0, 1.0, 5, 3, callback=lambda k, t, y: seen.append((k, round(t, 12))))
    assert seen == [(1, 0.2), (2, 0.4), (3, 0.6), (4, 0.8), (5, 1.0)]
    with pytest.raises(ValueError, match="at least 1"):
        hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), lambda t: (lambda w: w),
                            np.ones(2, complex), 0.0, 1.0, 0, 2)
    with pytest.raises(ValueError, match="nonzero"):
        hp.lanczos(lambda w: w, np.zeros(4, complex), 2)


def test_device_callback_sees_every_step(hp):
    """FastHamiltonian route (device Magnus loop): the callback gets every step, in order."""
    s = hp.build_full(2, 7)
    fh = hp.FastHamiltonian(s, hp.custom_potential(lambda p, t: 0.01 * p[:, 0] ** 2, 2, 16.0), 4)
    c = np.ones(s.size, complex) / np.sqrt(s.size)
    seen = []
    y = hp.propagate_magnus(hp.MagnusScheme.from_name("gl2"), fh.matvec_at, c, 0.0, 0.4, 4, 6,
                            callback=lambda k, t, yk: seen.append((k, round(t, 12), np.linalg.norm(yk))))
    assert [(k, t) for k, t, _ in seen] == [(1, 0.1), (2, 0.2), (3, 0.3), (4, 0.4)]
    assert abs(seen[-1][2] - np.linalg.norm(y)) < 1e-15


def test_decoupled_tridiagonal_blocks(hp):
    a = np.array([1.0, 2.0, -1.0, 0.5])
    b = np.array([0.3, 0.0, 0.7])  # beta_2 = 0: two independent 2x2 blocks
    d, z = hp.tridiag_eigh(a, b)
    T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
    assert np.allclose(np.sort(d), np.linalg.eigvalsh(T), atol=1e-14)
    assert np.allclose(T @ z, z * d, atol=1e-13)
    col = hp.expm_tridiag_column(a, b, 0.9)
    assert np.max(np.abs(col - scipy.linalg.expm(-0.9j * T)[:, 0])) < 1e-13
    assert np.max(np.abs(col[2:])) < 1e-15  # nothing leaks across the decoupled block


def test_oscillator_phases_exact_on_device(hp):
    """W = 0: A = D, so every coefficient turns with exp(-i t (|j| + N/2)); 7 distinct levels,
    so the 8-step Krylov space breaks down on an invariant subspace and each step is exact."""
    s = hp.build_full(2, 3)
    fh = hp.FastHamiltonian(s, hp.custom_potential(lambda p, t: 0.0 * p[:, 0], 2, 16.0), 2)
    rng = np.random.default_rng(4)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    c /= np.linalg.norm(c)
    y = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 1.0, 7, 8)
    levels = s.indices.sum(axis=1) + 1.0
    assert np.max(np.abs(y - np.exp(-1j * levels) * c)) < 1e-12


def test_time_independent_step_is_plain_exponential(hp):
    rng = np.random.default_rng(21)
    n = 10
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (m + m.conj().T) / 2
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ref = scipy.linalg.expm(-0.3j * a) @ y
    for name in ("midpoint", "gl2"):
        out, _ = hp.magnus_step(hp.MagnusScheme.from_name(name), lambda t: (lambda w: a @ w), y, 0.0, 0.3, n,
                                reorthogonalize=True)
        assert np.max(np.abs(out - ref)) < 1e-10


def test_magnus_orders_on_device(hp):
    """Time-dependent W on a small full cube through the device loop: halving h cuts the
    midpoint error ~4x and the GL2 error ~16x (reference's order test, on the fused path)."""
    s = hp.build_full(2, 11)

    def ev(p, t):
        y = p / 16.0
        return 40.0 * np.cos(3.0 * t) * y[:, 0] * y[:, 1] + 20.0 * np.sin(2.0 * t) * y[:, 0] ** 2

    fh = hp.FastHamiltonian(s, hp.custom_potential(ev, 2, 16.0), 4)
    rng = np.random.default_rng(5)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    c /= np.linalg.norm(c)
    ref = hp.propagate_magnus(hp.MagnusScheme.from_name("gl2"), fh.matvec_at, c, 0.0, 1.0, 512, 16)
    errs = {}
    for name in ("midpoint", "gl2"):
        sc = hp.MagnusScheme.from_name(name)
        errs[name] = [np.linalg.norm(hp.propagate_magnus(sc, fh.matvec_at, c, 0.0, 1.0, n, 16) - ref)
                      for n in (8, 16, 32)]
    mid, gl2 = errs["midpoint"], errs["gl2"]
    assert 3.3 < mid[0] / mid[1] < 4.7 and 3.3 < mid[1] / mid[2] < 4.7, mid
    assert 11.0 < gl2[0] / gl2[1] < 21.0 and 11.0 < gl2[1] / gl2[2] < 21.0, gl2
    assert gl2[0] < mid[0]


def test_krylov_error_decreases_with_dimension(hp):
    s = hp.build_full(3, 6)
    fh = hp.FastHamiltonian(s, hp.torsional(3), 6)
    rng = np.random.default_rng(6)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    c /= np.linalg.norm(c)
    mv = fh.matvec_at(0.0)
    A = np.column_stack([mv(e) for e in np.eye(s.size)])
    ref = scipy.linalg.expm(-0.2j * A) @ c
    errs = [np.linalg.norm(hp.lanczos_exp_apply(mv, c, 0.2, m)[0] - ref) for m in (2, 4, 6, 8, 12)]
    assert all(e1 < e0 for e0, e1 in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-4 * errs[0], errs


# ---------------------------------------------------------------- square sum

def test_square_sum_routes_agree(hp):
    """sum_l x_l^2 three ways: the exact banded route, the coordinate operator twice on a full
    cube (equal away from the truncation edge), and the oracle (bitwise)."""
    for s, idx in ((hp.build_hyperbolic(3, 25), O.hyperbolic_indices(3, 25)),
                   (hp.build_full(2, 9), O.full_indices(2, 9))):
        rng = np.random.default_rng(7)
        c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
        appl = hp.get_applier(s)
        got = appl.apply_square_sum(c)
        assert np.array_equal(got, O.applier_for_set(idx).square_sum(c))
        if s.kind == hp.FULL:
            xx = sum(appl.apply_coordinate(a, appl.apply_coordinate(a, c)) for a in range(1, s.dim + 1))
            inner = np.all(s.indices < s.bound, axis=1)  # X_a X_a loses the j_a + 1 term on the top face
            assert rel_l2(got[inner], xx[inner]) < 1e-14


def test_square_sum_diagonal_survives_pruning(hp):
    """A lone multi-index keeps the full diagonal sum_l (j_l + 1/2) though its neighbours are gone."""
    s = hp.from_indices(np.array([[0, 0], [1, 0], [0, 1], [2, 0], [1, 1], [0, 2], [3, 0]]))
    e = np.zeros(s.size, complex)
    k = s.position((1, 1))
    e[k] = 1.0
    out = hp.get_applier(s).apply_square_sum(e)
    assert out[k] == 3.0  # (1 + 1/2) + (1 + 1/2)


@pytest.mark.parametrize("kind,dim,bound", [("full", 1, 10), ("full", 3, 6), ("hyp", 3, 9), ("hyp", 5, 7),
                                            ("full", 2, 20)])
def test_single_cta_propagation_odd_sizes(hp, kind, dim, bound):
    """Small sets run the whole Magnus step in one CTA with shared-memory tables; sizes whose
    table lengths are odd (n = 11, 343, ...) once misaligned the sqrt table.  3 midpoint steps
    vs the oracle."""
    s = hp.build_full(dim, bound) if kind == "full" else hp.build_hyperbolic(dim, bound)
    idx = O.full_indices(dim, bound) if kind == "full" else O.hyperbolic_indices(dim, bound)
    spec = hp.torsional(dim)
    fh = hp.FastHamiltonian(s, spec, 4)
    rng = np.random.default_rng(dim * 100 + bound)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    c /= np.linalg.norm(c)
    ham_at = O.hamiltonian_at(O.applier_for_set(idx), spec.evaluator, dim, 16.0, 4)
    want = O.propagate("midpoint", ham_at, c, 0.0, 0.03, 3, 6)
    got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.03, 3, 6)
    assert rel_l2(got, want) < 1e-12


@pytest.mark.parametrize("kind,dim,bound", [("full", 1, 0), ("hyp", 4, 1), ("full", 5, 1), ("hyp", 3, 2)])
def test_degenerate_sets(hp, kind, dim, bound):
    """One-element sets and 2^5 cubes: Hamiltonian matvec against the oracle bitwise in reference
    order and within 1e-12 by default, and one Magnus step."""
    s = hp.build_full(dim, bound) if kind == "full" else hp.build_hyperbolic(dim, bound)
    idx = O.full_indices(dim, bound) if kind == "full" else O.hyperbolic_indices(dim, bound)
    assert np.array_equal(s.indices, idx)

    def ev(p, t):
        y = p / 16.0
        return (y ** 2).sum(axis=1) + 0.3 * y[:, 0] * y[:, -1] + 0.1 * y[:, 0] ** 3

    spec = hp.custom_potential(ev, dim, 16.0)
    ap = hp.interpolate(spec, 3)
    rng = np.random.default_rng(dim + bound)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    appl, oappl = hp.get_applier(s), O.applier_for_set(idx)
    want = oappl.hamiltonian(ap.degrees, ap.coeffs, 16.0, c)
    assert np.array_equal(appl.apply_hamiltonian(ap, c, ref_order=True), want)
    assert rel_l2(appl.apply_hamiltonian(ap, c), want) < 1e-12
    fh = hp.FastHamiltonian(s, spec, 3)
    ham_at = O.hamiltonian_at(oappl, ev, dim, 16.0, 3)
    c /= np.linalg.norm(c)
    got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.02, 1, 4)
    assert rel_l2(got, O.propagate("midpoint", ham_at, c, 0.0, 0.02, 1, 4)) < 1e-12


@pytest.mark.parametrize("dim,bound", [(16, 2), (16, 5), (12, 8)])
def test_widest_dimension_matvec(hp, dim, bound):
    """The widest dimension the library takes (HP_MAXDIM = 16): hyperbolic sets bit-exact, and a
    surrogate given as explicit terms (a tensor interpolation grid is out of reach at this width)
    applied bitwise in reference order, within 1e-12 by default."""
    from paper_1403_3511_b200.potential_approx import ChebApprox

    s = hp.build_hyperbolic(dim, bound)
    idx = O.hyperbolic_indices(dim, bound)
    assert np.array_equal(s.indices, idx)
    rng = np.random.default_rng(dim * bound)
    degs = np.zeros((2 * dim + 3, dim), dtype=np.int64)
    for a in range(dim):
        degs[2 * a, a] = 2
        degs[2 * a + 1, a] = 1
    degs[2 * dim, [0, dim - 1]] = 1
    degs[2 * dim + 1, [1, 2]] = [2, 1]
    coeffs = rng.uniform(-0.5, 0.5, len(degs))
    ap = ChebApprox(dim, 3, 16.0, 0.0, degs, coeffs, 0.0)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    appl = hp.get_applier(s)
    want = O.applier_for_set(idx).hamiltonian(degs, coeffs, 16.0, c)
    assert np.array_equal(appl.apply_hamiltonian(ap, c, ref_order=True), want)
    assert rel_l2(appl.apply_hamiltonian(ap, c), want) < 1e-12

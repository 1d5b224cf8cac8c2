"""Device Lanczos / Magnus propagation vs the reference (golden) and the oracle."""

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


def test_tridiag_and_expm(hp, golden):
    p = golden["propagate"]
    d, z = hp.tridiag_eigh(p["tri_alpha"], p["tri_beta"])
    assert rel_l2(d, p["tri_d"]) < 1e-14
    # eigenvectors up to sign
    for j in range(z.shape[1]):
        s = np.sign(z[:, j] @ p["tri_z"][:, j])
        assert rel_l2(s * z[:, j], p["tri_z"][:, j]) < 1e-13
    col = hp.expm_tridiag_column(p["tri_alpha"], p["tri_beta"], 0.37)
    assert rel_l2(col, p["tri_col"]) < 1e-14
    d1, z1 = hp.tridiag_eigh(np.array([2.0]), np.array([]))
    assert d1[0] == 2.0 and z1[0, 0] == 1.0


def test_expm_against_scipy(hp):
    from scipy.linalg import expm

    rng = np.random.default_rng(3)
    for m in (1, 2, 5, 12, 30):
        a = rng.standard_normal(m)
        b = np.abs(rng.standard_normal(m - 1)) + 0.1
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
        col = hp.expm_tridiag_column(a, b, 0.7)
        assert np.max(np.abs(col - expm(-0.7j * T)[:, 0])) < 1e-12


def _fh(hp, w, s):
    return hp.FastHamiltonian(s, hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH), w.degree)


RUNS = [("cfg1", "cfg1", None, 100, 0.01, "midpoint"), ("cfg1gl2", "cfg1", None, 10, 0.01, "gl2"),
        ("cfg3s", "cfg3", 255, 20, 0.001, "midpoint"), ("cfg4s", "cfg4", 15, 50, 0.005, "midpoint")]


@pytest.mark.parametrize("name,base,bound,nsteps,dt,scheme", RUNS)
def test_propagation_matches_reference(hp, golden, name, base, bound, nsteps, dt, scheme):
    p = golden["propagate"]
    w = W.CONFIGS[base] if bound is None else W.CONFIGS[base].scaled(bound, name)
    s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, None if w.kind == "full" else s.indices)
    fh = _fh(hp, w, s)
    fac = hp.lanczos(fh.matvec_at(0.0), c, 7)
    assert rel_l2(fac.alpha, p[f"{name}_lz_alpha"]) < 1e-13
    assert rel_l2(fac.beta, p[f"{name}_lz_beta"]) < 1e-13
    if w.kind == "full":  # reduced sets make W(X) non-normal: no orthogonality to pin
        assert fac.orthogonality_defect() < 1e-10
    y = hp.propagate_magnus(hp.MagnusScheme.from_name(scheme), fh.matvec_at, c, 0.0, nsteps * dt, nsteps, 7)
    step = int(p[f"{name}_prop_step"])
    assert rel_l2(y[::step], p[f"{name}_prop_samp"]) < TOL
    assert np.linalg.norm(y) == pytest.approx(float(p[f"{name}_prop_norm"]), rel=TOL)
    if f"{name}_prop_full" in p:
        assert rel_l2(y, p[f"{name}_prop_full"]) < TOL


def test_generic_matvec_lanczos_exactness(hp):
    """Full-space Krylov exactness with a dense operator (krylov tests, :103-113)."""
    from scipy.linalg import expm

    rng = np.random.default_rng(5)
    n = 6
    A = rng.standard_normal((n, n))
    A = A + A.T
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y, fac = hp.lanczos_exp_apply(lambda x: A @ x, v, 0.3, n, reorthogonalize=True)
    assert np.max(np.abs(y - expm(-0.3j * A) @ v)) < 1e-10


def test_breakdown_truncates(hp):
    s = hp.build_full(1, 9)
    fh = hp.FastHamiltonian(s, hp.custom_potential(lambda p, t: 0.0 * p[:, 0], 1, 16.0), 2)
    e = np.zeros(s.size, dtype=complex)
    e[3] = 1.0  # an eigenvector of the oscillator diagonal: invariant subspace at once
    fac = hp.lanczos(fh.matvec_at(0.0), e, 5)
    assert fac.breakdown_at == 1 and fac.steps == 1
    y = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, e, 0.0, 0.5, 5, 5)
    assert np.allclose(y[3], np.exp(-0.5j * 3.5), atol=1e-13)


def test_norm_preserved_on_full_cube(hp):
    w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
    s = hp.build_full(w.dim, w.bound)
    c = W.coefficients(w)
    fh = _fh(hp, w, s)
    y = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.05, 10, 7)
    assert abs(np.linalg.norm(y) - 1.0) < 1e-11


def test_harmonic_part_route_vs_oracle(hp):
    """harmonic_part != 0: exact square-sum route inside A(t)."""
    s = hp.build_hyperbolic(3, 40)
    spec = hp.torsional_minus_harmonic(3)
    fh = hp.FastHamiltonian(s, spec, 6)
    rng = np.random.default_rng(11)
    c = rng.standard_normal(s.size) + 1j * rng.standard_normal(s.size)
    c /= np.linalg.norm(c)
    appl = O.applier_for_set(O.hyperbolic_indices(3, 40))
    ham_at = O.hamiltonian_at(appl, spec.evaluator, 3, 16.0, 6, harmonic_part=spec.harmonic_part)
    want = O.propagate("midpoint", ham_at, c, 0.0, 0.1, 5, 7)
    got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.1, 5, 7)
    assert rel_l2(got, want) < TOL
    mv = fh.matvec_at(0.2)
    ap = fh.approx_at(0.2)
    want1 = appl.hamiltonian(ap.degrees, ap.coeffs, 16.0, c) + spec.harmonic_part * appl.square_sum(c)
    assert rel_l2(mv(c), want1) < TOL


def test_harmonic_part_folded_full_cube(hp):
    """harmonic_part != 0 on a cfg4-class full cube: q * square_sum rides in the fused evaluator's
    single-axis bands (no separate square pass); Lanczos + propagation vs the oracle within 1e-12."""
    from torch.profiler import ProfilerActivity, profile

    w = W.CONFIGS["cfg4"].scaled(15, "cfg4q")
    s = hp.build_full(w.dim, w.bound)
    spec = hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH, harmonic_part=0.3)
    fh = hp.FastHamiltonian(s, spec, w.degree)
    c = W.coefficients(w)
    appl = O.applier_for_full(w.dim, w.bound)
    ham_at = O.hamiltonian_at(appl, w.evaluator, w.dim, W.HALFWIDTH, w.degree, harmonic_part=0.3)
    want = O.propagate("midpoint", ham_at, c, 0.0, 0.015, 3, 7)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        got = hp.propagate_magnus(hp.MagnusScheme.from_name("midpoint"), fh.matvec_at, c, 0.0, 0.015, 3, 7)
    names = {e.key for e in prof.key_averages()}
    assert not any("k_square" in k or "k_axpy_c2" in k for k in names), names
    assert rel_l2(got, want) < TOL
    fac = hp.lanczos(fh.matvec_at(0.01), c, 7)
    ofac = O.lanczos(ham_at(0.01), c, 7)
    assert rel_l2(fac.alpha, ofac.alpha) < 1e-13
    assert rel_l2(fac.beta, ofac.beta) < 1e-13


@pytest.mark.parametrize("bound,world,q", [(15, 2, 0.0), (20, 4, 0.0), (20, 3, 0.0), (15, 3, 0.3)])
def test_sharded_propagation_emulated(bound, world, q):
    """Slab-sharded Magnus steps (sharding.sharded_propagate: owned-plane Lanczos with cross-shard
    reductions, the halo refreshed by every matvec), all ranks emulated in one process, against
    the single-device propagation of the full cube: 3 midpoint steps, m = 7, within 1e-12.  q != 0:
    the harmonic square sum (folded into the fused bands on the single device, a separate pass
    per shard)."""
    import torch

    import paper_1403_3511_b200 as hp
    from paper_1403_3511_b200 import workloads as W
    from paper_1403_3511_b200.sharding import SlabShard, emulate_exchange, local_sum, sharded_propagate

    w = W.CONFIGS["cfg4"].scaled(bound, "cfg4p")
    c = W.coefficients(w)
    full = hp.build_full(w.dim, w.bound)
    pot = hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH, harmonic_part=q)
    scheme = hp.MagnusScheme.from_name("midpoint")
    want = hp.FastHamiltonian(full, pot, w.degree).propagate(scheme, torch.from_numpy(c).cuda(), 0.0, w.dt, 3, 7)
    shards = [SlabShard(w.dim, w.bound, r, world, halo=w.degree) for r in range(world)]
    ys = []
    for s in shards:
        g = s.geo
        y = torch.zeros(g.box_size, dtype=torch.complex128, device="cuda")
        y[g.own_slice] = torch.from_numpy(c[g.lo * g.plane:g.hi * g.plane]).cuda()
        ys.append(y)
    fh = hp.FastHamiltonian(full, pot, w.degree)
    sharded_propagate(shards, fh, ys, 0.0, w.dt, 3, 7, reduce=local_sum, exchange=emulate_exchange)
    got = torch.cat([y[s.geo.own_slice] for s, y in zip(shards, ys)])
    assert float(torch.linalg.vector_norm(got - want) / torch.linalg.vector_norm(want)) < 1e-12


def test_sharded_propagation_general_couplings():
    """The sharded Magnus loop with a potential whose pair couplings need the second pass (so the
    plane entry point cannot supply the in-kernel dot: whole-box matvec + separate reductions)
    against the single-device propagation: 2 steps, 3 emulated ranks."""
    import torch

    import paper_1403_3511_b200 as hp
    from paper_1403_3511_b200 import workloads as W
    from paper_1403_3511_b200.sharding import SlabShard, emulate_exchange, local_sum, sharded_propagate

    cij = {(0, 1): 0.1, (0, 2): 0.07, (0, 3): -0.04, (1, 2): 0.06, (1, 3): 0.05, (2, 3): -0.03}

    def pot_fn(p, t):
        out = 0.5 * (p * p).sum(axis=-1) + 0.01 * (p ** 4).sum(axis=-1)
        for (a, b), c in cij.items():
            out = out + c * p[:, a] * p[:, b]
        return out

    w = W.CONFIGS["cfg4"].scaled(15, "cfg4g")
    c = W.coefficients(w)
    full = hp.build_full(w.dim, w.bound)
    pot = hp.custom_potential(pot_fn, w.dim, W.HALFWIDTH)
    scheme = hp.MagnusScheme.from_name("midpoint")
    want = hp.FastHamiltonian(full, pot, w.degree).propagate(scheme, torch.from_numpy(c).cuda(), 0.0, w.dt, 2, 7)
    shards = [SlabShard(w.dim, w.bound, r, 3, halo=w.degree) for r in range(3)]
    ys = []
    for s in shards:
        g = s.geo
        y = torch.zeros(g.box_size, dtype=torch.complex128, device="cuda")
        y[g.own_slice] = torch.from_numpy(c[g.lo * g.plane:g.hi * g.plane]).cuda()
        ys.append(y)
    fh = hp.FastHamiltonian(full, pot, w.degree)
    sharded_propagate(shards, fh, ys, 0.0, w.dt, 2, 7, reduce=local_sum, exchange=emulate_exchange)
    got = torch.cat([y[s.geo.own_slice] for s, y in zip(shards, ys)])
    assert float(torch.linalg.vector_norm(got - want) / torch.linalg.vector_norm(want)) < 1e-12


def test_lincomb_entry_points():
    """hp_lincomb3_nrm2sq / hp_lincomb (the sharded Lanczos update and combine) against numpy."""
    import ctypes

    import torch

    from paper_1403_3511_b200 import _native as nat

    L = nat.lib()
    gen = np.random.default_rng(3)
    n = 100_003
    X, Y, Z = (torch.from_numpy(gen.standard_normal(n) + 1j * gen.standard_normal(n)).cuda() for _ in range(3))
    out = torch.empty_like(X)
    nrm = torch.zeros(2, dtype=torch.float64, device="cuda")
    ws = torch.empty(int(L.hp_reduce_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    vp = ctypes.c_void_p
    for zptr, c in ((Z, -0.25), (None, 0.0)):
        nat.check(L.hp_lincomb3_nrm2sq(n, 1.5, vp(X.data_ptr()), -0.75, vp(Y.data_ptr()), c,
                                       vp(zptr.data_ptr()) if zptr is not None else None, vp(out.data_ptr()),
                                       vp(nrm.data_ptr()), vp(ws.data_ptr()), nat.stream_ptr()))
        want = 1.5 * X.cpu().numpy() - 0.75 * Y.cpu().numpy() + (c * Z.cpu().numpy() if zptr is not None else 0)
        assert rel_l2(out.cpu().numpy(), want) < 1e-15
        assert abs(float(nrm[0]) - np.vdot(want, want).real) <= 1e-13 * np.vdot(want, want).real
    coef = np.array([0.5, -1.0, 2.0, 0.25, -0.125, 3.0])  # 3 complex coefficients
    ptrs = (ctypes.c_void_p * 3)(X.data_ptr(), Y.data_ptr(), Z.data_ptr())
    nat.check(L.hp_lincomb(n, 3, ctypes.cast(ptrs, ctypes.c_void_p), coef.ctypes.data_as(ctypes.c_void_p),
                           vp(out.data_ptr()), nat.stream_ptr()))
    cs = coef[0::2] + 1j * coef[1::2]
    want = cs[0] * X.cpu().numpy() + cs[1] * Y.cpu().numpy() + cs[2] * Z.cpu().numpy()
    assert rel_l2(out.cpu().numpy(), want) < 1e-15

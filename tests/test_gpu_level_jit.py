"""The run-time specialised level kernels (csrc/hp_level_jit.cu) against the oracle and against
the interpreted kernel they replace on large sets.

HP_LEVEL_JIT_MIN=0 makes every level of every size compile its specialised kernel, so the small
sets the oracle can follow exercise the generator (buffer numbers, window masks, accumulated and
directly written targets, oscillator, fused Lanczos dot, batches, line order).  The full-size
cfg3 / cfg5 runs of test_gpu_configs.py use the specialised kernels by default.
Tolerance: relative L2 1e-12 against the oracle; 1e-14 against the interpreted kernel (the same
arithmetic, compiled twice).
"""

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


def _approx(degs, coeffs, dim, degree):
    from paper_1403_3511_b200.potential_approx import ChebApprox

    return ChebApprox(dim, int(degree), 16.0, 0.0, np.asarray(degs), np.asarray(coeffs), 0.0)


@pytest.mark.parametrize("seed", range(10))
def test_specialised_levels_random_terms(hp, seed, monkeypatch):
    gen = np.random.default_rng(7000 + seed)
    dim = int(gen.integers(2, 6))
    if gen.random() < 0.3:
        bound = int(gen.integers(3, {2: 20, 3: 9, 4: 6, 5: 4}[dim]))
        s = hp.build_full(dim, bound)
        oa = O.applier_for_full(dim, bound)
    else:
        bound = int(gen.integers(4, 60))
        s = hp.build_hyperbolic(dim, bound)
        oa = O.applier_for_set(O.hyperbolic_indices(dim, bound))
    nterms = int(gen.integers(2, 30))
    maxdeg = int(gen.integers(1, 5))
    degs = gen.integers(0, maxdeg + 1, size=(nterms, dim))
    degs[gen.random((nterms, dim)) < 0.5] = 0
    degs = np.unique(degs, axis=0)
    coeffs = gen.uniform(-2, 2, degs.shape[0]) * 10.0 ** gen.uniform(-1, 2, degs.shape[0])
    ap = _approx(degs, coeffs, dim, maxdeg)
    appl = hp.get_applier(s)
    v = gen.standard_normal(s.size) + 1j * gen.standard_normal(s.size)
    V = gen.standard_normal((3, s.size)) + 1j * gen.standard_normal((3, s.size))
    monkeypatch.setenv("HP_LEVEL_JIT", "0")
    base, base_h, base_b = appl.apply_polynomial(ap, v), appl.apply_hamiltonian(ap, v), appl.apply_polynomial(ap, V)
    monkeypatch.setenv("HP_LEVEL_JIT", "1")
    monkeypatch.setenv("HP_LEVEL_JIT_MIN", "0")
    y, yh, yb = appl.apply_polynomial(ap, v), appl.apply_hamiltonian(ap, v), appl.apply_polynomial(ap, V)
    assert rel_l2(y, oa.polynomial(degs, coeffs, 16.0, v)) < TOL
    assert rel_l2(yh, oa.hamiltonian(degs, coeffs, 16.0, v)) < TOL
    for b in range(3):
        assert rel_l2(yb[b], oa.polynomial(degs, coeffs, 16.0, V[b])) < TOL
    assert rel_l2(y, base) < 1e-14 and rel_l2(yh, base_h) < 1e-14 and rel_l2(yb, base_b) < 1e-14


@pytest.mark.parametrize("name,bound", [("cfg3", 255), ("cfg5", 63)])
def test_specialised_levels_scaled_configs(hp, name, bound, monkeypatch):
    """Scaled cfg3 / cfg5 (their planners' merged suffix nodes, prefix levels, line order and
    batch windows) through the specialised kernels vs the oracle."""
    monkeypatch.setenv("HP_LEVEL_JIT_MIN", "0")
    w = W.CONFIGS[name].scaled(bound, name + "j")
    s = hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, s.indices)
    ap = w.approx(0.0)
    oa = O.applier_for_set(np.asarray(s.indices))
    y = hp.get_applier(s).apply_polynomial(ap, c)
    C = np.atleast_2d(c)
    Y = np.atleast_2d(y)
    for b in range(min(C.shape[0], 2)):
        assert rel_l2(Y[b], oa.polynomial(ap.degrees, ap.coeffs, W.HALFWIDTH, C[b])) < TOL


def test_specialised_levels_in_the_magnus_step(hp, monkeypatch):
    """The Lanczos loop on a reduced set (level matvec with the oscillator and the in-kernel
    dot) gives the interpreted kernels' propagated state with the specialised ones."""
    w = W.CONFIGS["cfg3"].scaled(255, "cfg3k")
    s = hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, s.indices)
    fh = hp.FastHamiltonian(s, hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH), w.degree)
    scheme = hp.MagnusScheme.from_name("midpoint")
    monkeypatch.setenv("HP_LEVEL_JIT", "0")
    base = hp.propagate_magnus(scheme, fh.matvec_at, c, 0.0, 0.005, 5, 7)
    monkeypatch.setenv("HP_LEVEL_JIT", "1")
    monkeypatch.setenv("HP_LEVEL_JIT_MIN", "0")
    got = hp.propagate_magnus(scheme, fh.matvec_at, c, 0.0, 0.005, 5, 7)
    assert rel_l2(got, base) < 1e-13
    oa = O.applier_for_set(np.asarray(s.indices))
    ham_at = O.hamiltonian_at(oa, w.evaluator, w.dim, W.HALFWIDTH, w.degree)
    want = O.propagate("midpoint", ham_at, c, 0.0, 0.005, 5, 7)
    assert rel_l2(got, want) < TOL


def test_fallback_when_specialisation_is_off(hp, monkeypatch):
    """HP_LEVEL_JIT=0 (or a missing NVRTC) leaves every level on the library's interpreted kernel."""
    monkeypatch.setenv("HP_LEVEL_JIT", "0")
    monkeypatch.setenv("HP_LEVEL_JIT_MIN", "0")
    s = hp.build_hyperbolic(3, 40)
    oa = O.applier_for_set(O.hyperbolic_indices(3, 40))
    degs = np.array([[0, 0, 2], [1, 0, 1], [2, 2, 0], [0, 3, 0]])
    coeffs = np.array([0.5, -0.25, 0.125, 1.0])
    v = np.random.default_rng(3).standard_normal(s.size) + 0j
    y = hp.get_applier(s).apply_polynomial(_approx(degs, coeffs, 3, 3), v)
    assert rel_l2(y, oa.polynomial(degs, coeffs, 16.0, v)) < TOL


def test_on_disk_kernel_cache(hp, tmp_path, monkeypatch):
    """HP_LEVEL_JIT_CACHE: compiled kernels are written to the directory and a second process
    loads them (same results, nothing recompiled: its run is much shorter than the first)."""
    import os
    import subprocess
    import sys
    import time
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    script = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {str(root)!r})\n"
        "import paper_1403_3511_b200 as hp\n"
        "from paper_1403_3511_b200 import _native as nat, workloads as W\n"
        "w = W.CONFIGS['cfg5'].scaled(31, 'cfg5c')\n"
        "s = hp.build_hyperbolic(w.dim, w.bound)\n"
        "c = W.coefficients(w, s.indices)\n"
        "y = hp.get_applier(s).apply_polynomial(w.approx(0.0), c)\n"
        "np.save(sys.argv[1], y)\n"
        "print(nat.lib().hp_level_jit_kernels())\n")
    env = {**os.environ, "HP_LEVEL_JIT_CACHE": str(tmp_path), "HP_LEVEL_JIT_MIN": "0"}
    outs, walls, counts = [], [], []
    for i in range(2):
        f = tmp_path / f"y{i}.npy"
        t0 = time.time()
        r = subprocess.run([sys.executable, "-c", script, str(f)], env=env, capture_output=True, text=True, timeout=600)
        walls.append(time.time() - t0)
        assert r.returncode == 0, r.stderr[-2000:]
        counts.append(int(r.stdout.strip().splitlines()[-1]))
        outs.append(np.load(f))
    assert counts[0] > 0 and counts[1] == counts[0]
    assert len(list(tmp_path.glob("hp_level_*.cubin"))) >= counts[0]
    assert np.array_equal(outs[0], outs[1])

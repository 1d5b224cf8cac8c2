"""The primary drop-in seam, exercised with the UNMODIFIED reference package.

`hb.install(iset)` puts the device applier into a *reference* `hprop.IndexSet`'s
`_derived["applier"]` (the reference's own cache, fast_apply.py:248-254).  After that the
reference's public functions -- `fast_algorithm`, `apply_hamiltonian`, `direct_op`,
`cheb_of_coordinate_apply`, `square_sum_apply` (fast_apply.py:273-336),
`FastHamiltonian.matvec_at` (error_lab.py:173-185) and `propagate_magnus`
(krylov_propagator.py:247-263) -- run unchanged and route every matvec through the CUDA
kernels.  Each result is compared with the same reference call on a second, untouched set
(the reference's numpy path).

The reference is the pip-installed copy under baseline/_ref (git-ignored, shipped to the
GPU box with the snapshot: `pip install --no-index --no-deps --target baseline/_ref
/root/reference/pkg`); the module skips when it is absent.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_l2

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "hprop" / "__init__.py").exists(),
                                 reason="reference package not installed under baseline/_ref")]


@pytest.fixture(scope="module")
def ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import hprop

    assert Path(hprop.__file__).resolve().is_relative_to(REF.resolve()) or "/root/reference" in hprop.__file__
    return hprop


@pytest.fixture(scope="module")
def hb():
    import paper_1403_3511_b200 as hb

    return hb


CASES = [("hyperbolic", 3, 12, "henon-heiles", 4), ("full", 2, 15, "henon-heiles", 3),
         ("hyperbolic", 4, 10, "torsional", 4), ("full", 3, 7, "torsional", 2)]


def _pair(ref, kind, dim, bound):
    build = ref.build_full if kind == "full" else ref.build_hyperbolic
    return build(dim, bound), build(dim, bound)


@pytest.mark.parametrize("kind,dim,bound,pot,deg", CASES)
def test_reference_matvec_functions_route_to_device(ref, hb, kind, dim, bound, pot, deg):
    cpu_set, gpu_set = _pair(ref, kind, dim, bound)
    appl = hb.install(gpu_set)
    assert gpu_set._derived["applier"] is appl
    rng = np.random.default_rng([dim, bound])
    v = rng.standard_normal(cpu_set.size) + 1j * rng.standard_normal(cpu_set.size)
    spec = ref.smooth_remainder(ref.potential_by_name(pot, dim))
    ap = ref.interpolate(spec, deg, time=0.3)
    vc, vg = ref.CoeffVector(cpu_set, v), ref.CoeffVector(gpu_set, v)
    y_cpu = ref.fast_algorithm(cpu_set, ap, vc).data
    y_gpu = ref.fast_algorithm(gpu_set, ap, vg).data
    assert isinstance(y_gpu, np.ndarray) and y_gpu.dtype == np.complex128
    assert rel_l2(y_gpu, y_cpu) <= 1e-12
    assert rel_l2(ref.apply_hamiltonian(gpu_set, ap, vg).data, ref.apply_hamiltonian(cpu_set, ap, vc).data) <= 1e-12
    for axis in range(1, dim + 1):
        assert np.array_equal(ref.direct_op(gpu_set, axis, vg).data, ref.direct_op(cpu_set, axis, vc).data)
        a = ref.cheb_of_coordinate_apply(gpu_set, axis, 3, 16.0, vg).data
        b = ref.cheb_of_coordinate_apply(cpu_set, axis, 3, 16.0, vc).data
        assert rel_l2(a, b) <= 1e-13
    assert rel_l2(ref.square_sum_apply(gpu_set, vg).data, ref.square_sum_apply(cpu_set, vc).data) <= 1e-14


def test_reference_fast_hamiltonian_and_propagation(ref, hb):
    """FastHamiltonian.matvec_at and propagate_magnus of the reference, 20 midpoint steps."""
    cpu_set, gpu_set = _pair(ref, "hyperbolic", 3, 20)
    hb.install(gpu_set)
    spec = ref.potential_by_name("henon-heiles", 3)
    rng = np.random.default_rng(7)
    y0 = rng.standard_normal(cpu_set.size) + 1j * rng.standard_normal(cpu_set.size)
    y0 /= np.linalg.norm(y0)
    fc, fg = ref.FastHamiltonian(cpu_set, spec, 4), ref.FastHamiltonian(gpu_set, spec, 4)
    assert rel_l2(fg.matvec_at(0.2)(y0), fc.matvec_at(0.2)(y0)) <= 1e-12
    scheme = ref.MagnusScheme.from_name("midpoint")
    from hprop import krylov_propagator as kp

    yc = kp.propagate_magnus(scheme, fc.matvec_at, y0, 0.0, 0.2, 20, 7)
    yg = kp.propagate_magnus(scheme, fg.matvec_at, y0, 0.0, 0.2, 20, 7)
    assert rel_l2(yg, yc) <= 1e-12


def test_reference_harmonic_route(ref, hb):
    """harmonic_part != 0: the reference's matvec adds q * apply_square_sum (error_lab.py:176-183)."""
    cpu_set, gpu_set = _pair(ref, "full", 2, 11)
    hb.install(gpu_set)
    spec = ref.potential_by_name("torsional-ho", 2)
    assert spec.harmonic_part != 0.0
    rng = np.random.default_rng(3)
    y0 = rng.standard_normal(cpu_set.size) + 1j * rng.standard_normal(cpu_set.size)
    fc, fg = ref.FastHamiltonian(cpu_set, spec, 3), ref.FastHamiltonian(gpu_set, spec, 3)
    assert rel_l2(fg.matvec_at(0.0)(y0), fc.matvec_at(0.0)(y0)) <= 1e-12
    from hprop import krylov_propagator as kp

    scheme = ref.MagnusScheme.from_name("gl2")
    yc = kp.propagate_magnus(scheme, fc.matvec_at, y0, 0.0, 0.1, 5, 7)
    yg = kp.propagate_magnus(scheme, fg.matvec_at, y0, 0.0, 0.1, 5, 7)
    assert rel_l2(yg, yc) <= 1e-12


def test_install_uses_structured_device_sets(ref, hb):
    """Full / hyperbolic reference sets map to the structured device sets (stride arithmetic,
    unranking tables); a custom set keeps its rows."""
    for kind, build in (("full", ref.build_full), ("hyperbolic", ref.build_hyperbolic)):
        s = build(3, 6)
        appl = hb.install(s)
        assert appl.iset.kind == kind and appl.iset.size == s.size
    c = ref.from_indices([(0, 0), (1, 0), (0, 1), (2, 0)])
    appl = hb.install(c)
    assert appl.iset.kind == "custom" and np.array_equal(appl.iset.indices, c.indices)
    v = np.arange(c.size, dtype=float) + 1.0
    assert np.array_equal(ref.direct_op(c, 1, ref.CoeffVector(c, v)).data,
                          ref.direct_op(ref.from_indices([(0, 0), (1, 0), (0, 1), (2, 0)]), 1,
                                        ref.CoeffVector(ref.from_indices([(0, 0), (1, 0), (0, 1), (2, 0)]), v)).data)

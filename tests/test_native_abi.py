"""The C-ABI library builds for sm_100a, loads and exports every declared symbol (no GPU needed)."""

import ctypes
import subprocess

import pytest

from paper_1403_3511_b200 import _native as nat


def test_library_present_and_loads():
    assert nat.LIB_PATH.exists(), "run __graft_entry__.build() first"
    lib = nat.load(require_device=False)
    assert lib.hp_abi_version() == 1


def test_exports_every_header_symbol():
    declared = nat.header_symbols()
    assert len(declared) >= 20
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/hprop_b200.h but not exported"
    assert set(declared) == set(nat.SIGNATURES), "ctypes signatures out of sync with the header"


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_means_loud_failure(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(nat.NativeUnavailable):
        nat.lib()


def test_product_does_not_import_oracle():
    import pathlib

    pkg = pathlib.Path(nat.__file__).parent
    for f in pkg.rglob("*.py"):
        for line in f.read_text().splitlines():
            s = line.strip()
            assert not (s.startswith("import oracle") or s.startswith("from oracle")), f


def test_runtime_specialised_level_kernels_compile():
    """The level kernels hp_apply_polynomial compiles at run time for large sets (NVRTC,
    csrc/hp_level_jit.cu) build for sm_100a here, without a device: cfg3's polynomial and a few
    random term lists (suffix and prefix levels, direct children, several accumulators), for both
    axis-view kinds."""
    import ctypes as C

    import numpy as np

    from paper_1403_3511_b200 import workloads as W

    lib = nat.load(require_device=False)
    cases = []
    ap = W.CONFIGS["cfg3"].approx(0.0, validate=False)
    cases.append((6, np.asarray(ap.degrees, dtype=np.int32), np.asarray(ap.coeffs, dtype=np.float64)))
    gen = np.random.default_rng(5)
    for dim in (2, 4, 8):
        degs = gen.integers(0, 4, size=(24, dim))
        degs[gen.random((24, dim)) < 0.6] = 0
        degs = np.unique(degs, axis=0).astype(np.int32)
        cases.append((dim, degs, gen.uniform(-1, 1, degs.shape[0])))
    total = 0
    for dim, degs, coeffs in cases:
        degs = np.ascontiguousarray(degs)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        nk = C.c_int(0)
        rc = lib.hp_level_jit_selftest(dim, degs.ctypes.data_as(nat.c_i32p), coeffs.ctypes.data_as(nat.c_dblp),
                                       degs.shape[0], C.byref(nk))
        assert rc == 0, lib.hp_last_error().decode()
        assert nk.value >= 2
        total += nk.value
    assert total >= 8

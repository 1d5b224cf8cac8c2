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

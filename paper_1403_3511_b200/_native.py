"""ctypes binding of the in-tree C-ABI library `_lib/libhprop_b200.so`.

The library is the product: every numeric routine of the hot path runs in
its sm_100a kernels.  There is no CPU fallback -- if the library or a CUDA
device is missing, `lib()` raises instead of computing anything elsewhere.
Signatures follow include/hprop_b200.h.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / os.environ.get("HP_LIB_VARIANT", "libhprop_b200.so")

HP_OK, HP_ERR_VALUE, HP_ERR_RUNTIME, HP_ERR_CUDA, HP_ERR_NOMEM, HP_ERR_KEY = range(6)
HP_F64, HP_C128 = 0, 1
HP_KIND_FULL, HP_KIND_HYPERBOLIC, HP_KIND_CUSTOM = 0, 1, 2
HP_ADD_OSC, HP_REF_ORDER, HP_CHECK_FINITE = 1, 2, 4

_lock = threading.Lock()
_lib = None

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dblp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t
c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double

# name -> (restype, argtypes); the full exported surface of hprop_b200.h
SIGNATURES = {
    "hp_abi_version": (c_int, []),
    "hp_last_error": (ctypes.c_char_p, []),
    "hp_device_count": (c_int, []),
    "hp_launch_count": (c_i64, []),
    "hp_level_jit_kernels": (c_int, []),
    "hp_level_jit_selftest": (c_int, [c_int, c_i32p, c_dblp, c_int, ctypes.POINTER(c_int)]),
    "hp_set_create_full": (c_int, [c_int, c_int, c_vp, ctypes.POINTER(c_vp), c_i64p]),
    "hp_set_create_slab": (c_int, [c_int, c_int, c_int, c_int, c_vp, ctypes.POINTER(c_vp), c_i64p]),
    "hp_set_create_hyperbolic": (c_int, [c_int, c_int, c_vp, ctypes.POINTER(c_vp), c_i64p]),
    "hp_set_create_custom": (c_int, [c_int, c_int, c_i64p, c_i64, c_vp, ctypes.POINTER(c_vp)]),
    "hp_set_info": (c_int, [c_vp, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int), c_i64p]),
    "hp_set_indices": (c_int, [c_vp, c_vp, c_vp]),
    "hp_neighbor_tables": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp]),
    "hp_set_position": (c_int, [c_vp, c_i64p, c_i64p]),
    "hp_set_destroy": (c_int, [c_vp]),
    "hp_apply_coordinate": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_i64, c_vp]),
    "hp_cheb_workspace_bytes": (c_sz, [c_vp, c_int, c_i64]),
    "hp_cheb_apply": (c_int, [c_vp, c_int, c_int, c_dbl, c_int, c_vp, c_vp, c_i64, c_vp, c_sz, c_vp]),
    "hp_poly_workspace_bytes": (c_sz, [c_vp, c_i32p, c_int, c_int, c_i64, c_int]),
    "hp_apply_polynomial": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_int, c_vp, c_vp, c_i64, c_int,
                                    c_i32p, c_vp, c_sz, c_vp]),
    "hp_apply_polynomial_streamed": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_int, c_vp, c_vp, c_vp, c_vp,
                                             c_i64, c_int, c_vp, c_sz, c_vp]),
    "hp_apply_polynomial_planes": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_int, c_vp, c_vp, c_int, c_int,
                                           c_int, c_vp, c_sz, c_vp]),
    "hp_apply_polynomial_planes_dot": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_int, c_vp, c_vp, c_int, c_int,
                                               c_int, c_vp, c_vp, c_sz, c_vp]),
    "hp_apply_hamiltonian_planes_dot": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_dbl, c_int, c_vp, c_vp, c_int,
                                                c_int, c_int, c_vp, c_vp, c_sz, c_vp]),
    "hp_square_sum": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_vp]),
    "hp_lz_state_bytes": (c_sz, []),
    "hp_lz_init": (c_int, [c_vp, c_int, c_vp]),
    "hp_lz_set": (c_int, [c_vp, c_int, c_int, c_vp, c_dbl, c_vp]),
    "hp_lz_update": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp]),
    "hp_lz_expm": (c_int, [c_vp, c_dbl, c_vp]),
    "hp_lz_combine": (c_int, [c_i64, c_int, c_vp, c_vp, c_vp, c_vp]),
    "hp_lz_diag": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hp_restrict": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_i64, c_vp]),
    "hp_extend": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_i64, c_vp]),
    "hp_reduction_components": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
    "hp_reduction_local_mask": (c_int, [c_vp, c_i32p, c_int, c_vp, c_vp]),
    "hp_decay_vector": (c_int, [c_vp, c_int, c_vp, c_vp]),
    "hp_magnus_workspace_bytes": (c_sz, [c_vp, c_int, c_i32p, c_int, c_i32p, c_int, c_int]),
    "hp_magnus_step": (c_int, [c_vp, c_int, c_i32p, c_dblp, c_int, c_i32p, c_dblp, c_int, c_dbl, c_dbl,
                               c_dbl, c_int, c_int, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "hp_lanczos": (c_int, [c_vp, c_i32p, c_dblp, c_int, c_dbl, c_dbl, c_vp, c_int, c_int, c_vp, c_vp, c_vp,
                           c_vp, c_vp, c_sz, c_vp]),
    "hp_expm_tridiag_column": (c_int, [c_vp, c_vp, c_int, c_dbl, c_vp, c_vp, c_vp]),
    "hp_tridiag_eigh": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp]),
    "hp_reduce_workspace_bytes": (c_sz, [c_i64]),
    "hp_cdot": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "hp_cnrm2": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "hp_lincomb3_nrm2sq": (c_int, [c_i64, ctypes.c_double, c_vp, ctypes.c_double, c_vp, ctypes.c_double, c_vp, c_vp,
                                   c_vp, c_vp, c_vp]),
    "hp_lincomb": (c_int, [c_i64, ctypes.c_int, c_vp, c_vp, c_vp, c_vp]),
}


class NativeUnavailable(RuntimeError):
    pass


def header_symbols() -> list[str]:
    """Function names declared in include/hprop_b200.h."""
    import re

    hdr = (_HERE.parent / "include" / "hprop_b200.h").read_text()
    pat = r"^\s*(?:hp_status|int|int64_t|size_t|const char\s*\*)\s+(hp_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(pat, hdr, flags=re.M)))


def load(require_device: bool = True):
    """Load the library (once).  Raises NativeUnavailable if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                    "there is no CPU fallback")
            import torch  # noqa: F401  (shares torch's libcudart / context)

            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible: the hprop_b200 matvec runs only on the GPU")
    return _lib


def lib():
    return load(True)


def last_error() -> str:
    return _lib.hp_last_error().decode() if _lib is not None else ""


def check(status: int) -> None:
    if status == HP_OK:
        return
    msg = _lib.hp_last_error().decode() if _lib is not None else "unknown error"
    if status == HP_ERR_VALUE:
        raise ValueError(msg)
    if status == HP_ERR_KEY:
        raise KeyError(msg)
    if status == HP_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)

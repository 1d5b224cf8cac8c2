"""GPU matrix-free application of polynomial potentials (drop-in for hprop.fast_apply).

`PolynomialApplier` keeps the reference's method surface
(fast_apply.py:32-245) and is installed the same way, through
`get_applier(iset)` / `iset._derived["applier"]` (fast_apply.py:248-254), so
every caller of the reference -- direct_op, cheb_of_coordinate_apply,
fast_algorithm, apply_hamiltonian, square_sum_apply, FastHamiltonian -- runs
on the device.  Numpy inputs are copied to the GPU and the result is copied
back (the reference's host-array contract); torch CUDA tensors stay on the
device.  A leading batch axis (B, n) applies the operator to B vectors in
one call.

Two evaluation orders are available (see csrc/hp_apply.cu):
  * default -- suffix-trie regrouping (and fused full-cube kernels), equal
    to the reference within rounding (tests: rel. L2 <= 1e-12);
  * ``ref_order=True`` -- the reference's own order of operations, bitwise
    identical to numpy.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
import warnings

import numpy as np

from . import _native as nat
from .index_set import CoeffVector, IndexSet, _is_torch
from .potential_approx import ChebApprox


def _term_arrays(approx, dim: int):
    degs = np.ascontiguousarray(np.asarray(approx.degrees, dtype=np.int32).reshape(-1, dim))
    coeffs = np.ascontiguousarray(np.asarray(approx.coeffs, dtype=np.float64).reshape(-1))
    if degs.shape[0] != coeffs.shape[0]:
        raise ValueError("degrees and coeffs disagree in length")
    return degs, coeffs


class _Dev:
    """Host/device adapter: returns (device tensor, restore-callable)."""

    @staticmethod
    def to_device(v, n: int):
        import torch

        if _is_torch(v):
            t = v
            if not t.is_cuda:
                t = t.cuda()
            if t.dtype not in (torch.float64, torch.complex128):
                t = t.to(torch.complex128 if t.is_complex() else torch.float64)
            t = t.contiguous()
            host = False
        else:
            arr = np.asarray(v)
            dt = np.result_type(arr.dtype, np.float64)
            arr = np.ascontiguousarray(arr, dtype=dt)
            t = torch.from_numpy(arr).cuda(non_blocking=False)
            host = True
        if t.shape[-1] != n or t.dim() not in (1, 2):
            raise ValueError(f"vector has shape {tuple(t.shape)}, expected (n,) or (B, n) with n={n}")
        batch = 1 if t.dim() == 1 else t.shape[0]
        dtype = nat.HP_C128 if t.is_complex() else nat.HP_F64
        return t, host, batch, dtype

    @staticmethod
    def back(t, host: bool):
        return t.cpu().numpy() if host else t


class PolynomialApplier:
    """Device-backed applier bound to one index set (fast_apply.py:32-55).

    The handle's neighbour data is immutable; per-call scratch comes from
    the torch caching allocator, so one applier can serve concurrent
    callers on different streams (fast_apply.py:36-37).
    """

    def __init__(self, iset: IndexSet):
        self.iset = iset
        self._osc = None

    # -- oscillator levels sum_l (j_l + 1/2), fast_apply.py:55 -----------------
    @property
    def osc_levels(self) -> np.ndarray:
        if self._osc is None:
            self._osc = (self.iset.indices + 0.5).sum(axis=1).astype(np.float64)
        return self._osc

    def _ws(self, nbytes: int):
        import torch

        return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device="cuda")

    # -- single coordinate (fast_apply.py:59-65) --------------------------------
    def apply_coordinate(self, axis: int, w):
        if not 1 <= axis <= self.iset.dim:
            raise ValueError(f"axis must satisfy 1 <= axis <= {self.iset.dim}, got {axis}")
        import torch

        t, host, batch, dtype = _Dev.to_device(w, self.iset.size)
        t = self.iset._to_canon(t)
        out = torch.empty_like(t)
        nat.check(nat.lib().hp_apply_coordinate(ctypes.c_void_p(self.iset.handle), axis, dtype,
                                                ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                batch, nat.stream_ptr()))
        return _Dev.back(self.iset._from_canon(out), host)

    # -- T_deg(X_axis / L) (fast_apply.py:94-106, 281-302) -------------------------
    def cheb_apply(self, axis: int, degree: int, halfwidth: float, v):
        import torch

        t, host, batch, dtype = _Dev.to_device(v, self.iset.size)
        t = self.iset._to_canon(t)
        out = torch.empty_like(t)
        L = nat.lib()
        h = ctypes.c_void_p(self.iset.handle)
        ws = self._ws(L.hp_cheb_workspace_bytes(h, dtype, batch))
        nat.check(L.hp_cheb_apply(h, axis, int(degree), float(halfwidth), dtype, ctypes.c_void_p(t.data_ptr()),
                                  ctypes.c_void_p(out.data_ptr()), batch, ctypes.c_void_p(ws.data_ptr()),
                                  ws.numel(), nat.stream_ptr()))
        return _Dev.back(self.iset._from_canon(out), host)

    def _chebyshev_axis(self, axis, deg, halfwidth, wm, wp, sp, tmp):
        """Padded-buffer form used by the reference's cheb_of_coordinate_apply."""
        n = self.iset.size
        wp[:n] = self.cheb_apply(axis, deg, halfwidth, wm[:n])
        return wm, wp, sp

    # -- full surrogate (fast_apply.py:110-198) -----------------------------------
    def _poly(self, approx, v, flags: int, axis_order):
        import torch

        N = self.iset.dim
        if approx.dim != N:
            raise ValueError(f"surrogate dimension {approx.dim} does not match index set dimension {N}")
        order_arr = None
        if axis_order is not None:
            order = [int(a) for a in axis_order]
            if sorted(order) != list(range(1, N + 1)):
                raise ValueError(f"axis_order must permute 1..{N}")
            order_arr = np.ascontiguousarray(order, dtype=np.int32)
        degs, coeffs = _term_arrays(approx, N)
        t, host, batch, dtype = _Dev.to_device(v, self.iset.size)
        t = self.iset._to_canon(t)
        out = torch.empty_like(t)
        L = nat.lib()
        h = ctypes.c_void_p(self.iset.handle)
        dptr = degs.ctypes.data_as(nat.c_i32p)
        ws = self._ws(L.hp_poly_workspace_bytes(h, dptr, degs.shape[0], dtype, batch, flags))
        nat.check(L.hp_apply_polynomial(
            h, dptr, coeffs.ctypes.data_as(nat.c_dblp), degs.shape[0], float(approx.halfwidth), dtype,
            ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), batch, flags,
            order_arr.ctypes.data_as(nat.c_i32p) if order_arr is not None else None,
            ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr()))
        return _Dev.back(self.iset._from_canon(out), host)

    def _into_entry(self, approx, x, flags: int, batch: int):
        """Term arrays of `approx` and a workspace for the device-resident entry points.

        Term arrays are cached per (approx, shape, flags) in a small LRU (a time-dependent
        surrogate is a new object every step); the workspace is shared by every approx of the
        same (shape, dtype, flags, stream) and grown to the largest request, so a stepping loop
        allocates it once instead of once per step.
        """
        import torch

        key = (id(approx), tuple(x.shape), x.dtype, flags)
        cache = self.__dict__.setdefault("_into_cache", OrderedDict())
        ent = cache.get(key)
        if ent is None or ent[0] is not approx:
            degs, coeffs = _term_arrays(approx, self.iset.dim)
            dtype = nat.HP_C128 if x.is_complex() else nat.HP_F64
            h = ctypes.c_void_p(self.iset.handle)
            wsb = int(nat.lib().hp_poly_workspace_bytes(h, degs.ctypes.data_as(nat.c_i32p), degs.shape[0], dtype,
                                                        batch, flags))
            ent = (approx, degs, coeffs, h, batch, dtype, wsb)
            cache[key] = ent
            while len(cache) > 16:
                cache.popitem(last=False)
        else:
            cache.move_to_end(key)
        dev = x.device if x.is_cuda else torch.device("cuda", torch.cuda.current_device())
        wkey = (tuple(x.shape), x.dtype, flags, torch.cuda.current_stream(dev).cuda_stream)
        wss = self.__dict__.setdefault("_into_ws", {})
        ws = wss.get(wkey)
        if ws is None or ws.numel() < max(ent[6], 16):
            ws = torch.empty(max(ent[6], 16), dtype=torch.uint8, device=dev)
            wss[wkey] = ws
        return ent[:6] + (ws,)

    def apply_into(self, approx, x, y, flags: int = 0) -> None:
        """Device-resident hot loop: y <- W(X) x for preallocated CUDA tensors.

        Term arrays and the workspace are cached per (approx, shape, flags),
        so a repeated call is a single C-ABI launch sequence with no host
        allocation (bench.py's timed step).
        """
        if self.iset.permuted:  # explicit unsorted index list: permute at the boundary
            y.copy_(self._poly(approx, x, flags, None))
            return
        batch = 1 if x.dim() == 1 else x.shape[0]
        _, degs, coeffs, h, batch, dtype, ws = self._into_entry(approx, x, flags, batch)
        nat.check(nat.lib().hp_apply_polynomial(
            h, degs.ctypes.data_as(nat.c_i32p), coeffs.ctypes.data_as(nat.c_dblp), degs.shape[0],
            float(approx.halfwidth), dtype, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), batch,
            flags, None, ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr()))

    def apply_planes_into(self, approx, x, y, plane_lo: int, plane_hi: int, flags: int = 0, dot=None,
                          q: float = 0.0) -> bool:
        """y <- W(X) x [+ q sum_l x_l^2 x] on the output j1-planes [plane_lo, plane_hi) of a full
        cube / slab only.

        Reads input planes plane_lo - 4 .. plane_hi + 3 (hp_apply_hamiltonian_planes_dot; q folds
        the exact square sum into the same launch).  Returns False (nothing launched) when the
        surrogate is outside the fused full-cube class; the answer is cached per term structure
        (degrees and nonzero pattern), shape and flags.
        """
        _, degs, coeffs, h, _batch, dtype, ws = self._into_entry(approx, x, flags, 1)
        key = (degs.tobytes(), (np.asarray(coeffs) != 0).tobytes(), tuple(x.shape), x.dtype, flags)
        unsupported = self.__dict__.setdefault("_planes_unsupported", set())
        if key in unsupported:
            return False
        # dot: a float64 device tensor of 2; (re, im) of the in-kernel rows of x^H y over the
        # output planes are ADDED to it (hp_apply_polynomial_planes_dot)
        st = nat.lib().hp_apply_hamiltonian_planes_dot(
            h, degs.ctypes.data_as(nat.c_i32p), coeffs.ctypes.data_as(nat.c_dblp), degs.shape[0],
            float(approx.halfwidth), float(q), dtype, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
            int(plane_lo), int(plane_hi), flags, ctypes.c_void_p(dot.data_ptr()) if dot is not None else None,
            ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr())
        if st == nat.HP_ERR_VALUE and "fused full-cube" in nat.last_error():
            unsupported.add(key)
            return False
        nat.check(st)
        return True

    def apply_host_into(self, approx, x_host, y_host, flags: int = 0) -> None:
        """Host-resident vectors: y_host <- W(X) x_host for CPU tensors (pin them for overlap).

        One C-ABI call (hp_apply_polynomial_streamed): on full cubes of the fused class the
        library streams j1-plane chunks in, computes each chunk once its halo has landed and
        streams the result out, so both PCIe directions overlap the kernels.  Device buffers
        and the workspace are cached per (approx, shape, flags).  Ordered on the current
        stream; synchronise before reading y_host.
        """
        import torch

        if x_host.is_cuda or y_host.is_cuda or x_host.shape != y_host.shape or x_host.dtype != y_host.dtype:
            raise ValueError("apply_host_into expects two CPU tensors of the same shape and dtype")
        if not (x_host.is_contiguous() and y_host.is_contiguous()):
            raise ValueError("apply_host_into expects contiguous tensors")
        if self.iset.permuted:
            y_host.copy_(self._poly(approx, x_host.cuda(), flags, None).cpu())
            return
        batch = 1 if x_host.dim() == 1 else x_host.shape[0]
        _, degs, coeffs, h, batch, dtype, ws = self._into_entry(approx, x_host, flags, batch)
        # device staging buffers, shared like the workspace (per shape, dtype and stream)
        bkey = ("host", tuple(x_host.shape), x_host.dtype, torch.cuda.current_stream().cuda_stream)
        bufs = self.__dict__.setdefault("_into_bufs", {})
        if bkey not in bufs:
            xd = torch.empty(x_host.shape, dtype=x_host.dtype, device="cuda")
            bufs[bkey] = (xd, torch.empty_like(xd))
        xd, yd = bufs[bkey]
        nat.check(nat.lib().hp_apply_polynomial_streamed(
            h, degs.ctypes.data_as(nat.c_i32p), coeffs.ctypes.data_as(nat.c_dblp), degs.shape[0],
            float(approx.halfwidth), dtype, ctypes.c_void_p(x_host.data_ptr()), ctypes.c_void_p(y_host.data_ptr()),
            ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()), batch, flags,
            ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr()))

    def apply_polynomial(self, approx: ChebApprox, v, axis_order=None, *, ref_order: bool = False):
        """Multiply v by the restricted Galerkin matrix of the surrogate."""
        flags = nat.HP_REF_ORDER if ref_order else 0
        return self._poly(approx, v, flags, axis_order)

    def apply_hamiltonian(self, approx: ChebApprox, v, *, ref_order: bool = False):
        flags = nat.HP_ADD_OSC | (nat.HP_REF_ORDER if ref_order else 0)
        return self._poly(approx, v, flags, None)

    def _checked(self, approx, v, flags):
        return self._poly(approx, v, flags | nat.HP_CHECK_FINITE, None)

    # -- exact quadratic confinement (fast_apply.py:202-245) ------------------------
    def apply_square_sum(self, v):
        import torch

        t, host, batch, dtype = _Dev.to_device(v, self.iset.size)
        t = self.iset._to_canon(t)
        out = torch.empty_like(t)
        nat.check(nat.lib().hp_square_sum(ctypes.c_void_p(self.iset.handle), dtype, ctypes.c_void_p(t.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), batch, nat.stream_ptr()))
        return _Dev.back(self.iset._from_canon(out), host)


def get_applier(iset: IndexSet) -> PolynomialApplier:
    """Per-set applier, built once (fast_apply.py:248-254)."""
    appl = iset._derived.get("applier")
    if appl is None:
        appl = PolynomialApplier(iset)
        iset._derived["applier"] = appl
    return appl


def install(iset) -> PolynomialApplier:
    """Install the GPU applier into a *reference* hprop IndexSet.

    After this, the reference's own fast_algorithm / apply_hamiltonian /
    FastHamiltonian route through the device (fast_apply.py:250-253).  The
    reference set's indices are uploaded once as a custom device set.
    """
    from .index_set import build_full, build_hyperbolic

    ref_idx = np.asarray(iset.indices)
    dev = None
    if iset.kind in ("full", "hyperbolic"):
        # the structured device set (stride arithmetic / unranking kernels, and on full cubes the
        # fused single-pass evaluator) when it is the same member list in the same order
        cand = (build_full if iset.kind == "full" else build_hyperbolic)(iset.dim, iset.bound)
        if cand.size == ref_idx.shape[0] and np.array_equal(cand.indices, ref_idx):
            dev = cand
    if dev is None:
        dev = IndexSet(iset.dim, iset.bound, "custom", ref_idx)
    appl = PolynomialApplier(dev)
    iset._derived["applier"] = appl
    return appl


def _check_vector(iset: IndexSet, v: CoeffVector) -> None:
    if v.iset is not iset and not iset.same_as(v.iset):
        raise ValueError("coefficient vector belongs to a different index set")


def _check_approx(iset: IndexSet, approx) -> None:
    if approx.dim != iset.dim:
        raise ValueError(f"surrogate dimension {approx.dim} does not match "
                         f"index set dimension {iset.dim}")
    if approx.degree > iset.bound / 2:
        warnings.warn(f"surrogate degree {approx.degree} exceeds half the basis bound "
                      f"{iset.bound}; quadrature exactness margins are thin",
                      UserWarning, stacklevel=3)


def direct_op(iset: IndexSet, axis: int, v: CoeffVector) -> CoeffVector:
    """X_axis applied to a coefficient vector (fast_apply.py:273-278)."""
    if not 1 <= axis <= iset.dim:
        raise ValueError(f"axis must satisfy 1 <= axis <= {iset.dim}, got {axis}")
    _check_vector(iset, v)
    return CoeffVector(iset, get_applier(iset).apply_coordinate(axis, v.data))


def cheb_of_coordinate_apply(iset: IndexSet, axis: int, degree: int, halfwidth: float,
                             v: CoeffVector) -> CoeffVector:
    """T_degree(X_axis / halfwidth) v through the vector recurrence (fast_apply.py:281-302)."""
    if not 1 <= axis <= iset.dim:
        raise ValueError(f"axis must satisfy 1 <= axis <= {iset.dim}, got {axis}")
    if degree < 0:
        raise ValueError(f"degree must be nonnegative, got {degree}")
    if halfwidth <= 0:
        raise ValueError(f"halfwidth must be positive, got {halfwidth}")
    _check_vector(iset, v)
    if degree == 0:
        return v.copy()
    return CoeffVector(iset, get_applier(iset).cheb_apply(axis, degree, halfwidth, v.data))


def fast_algorithm(iset: IndexSet, approx, v: CoeffVector, *, axis_order=None,
                   ref_order: bool = False) -> CoeffVector:
    """sum_r alpha_r prod_l T_{r_l}(X_l/L) v (fast_apply.py:305-319); RuntimeError if non-finite."""
    _check_vector(iset, v)
    _check_approx(iset, approx)
    appl = get_applier(iset)
    flags = nat.HP_CHECK_FINITE | (nat.HP_REF_ORDER if ref_order else 0)
    return CoeffVector(iset, appl._poly(approx, v.data, flags, axis_order))


def apply_hamiltonian(iset: IndexSet, approx, v: CoeffVector, *, ref_order: bool = False) -> CoeffVector:
    """(D + W_pol) v with D the oscillator diagonal (fast_apply.py:322-330)."""
    _check_vector(iset, v)
    _check_approx(iset, approx)
    flags = nat.HP_ADD_OSC | nat.HP_CHECK_FINITE | (nat.HP_REF_ORDER if ref_order else 0)
    return CoeffVector(iset, get_applier(iset)._poly(approx, v.data, flags, None))


def square_sum_apply(iset: IndexSet, v: CoeffVector) -> CoeffVector:
    """(sum_l x_l**2) v via the exact banded entries (fast_apply.py:333-336)."""
    _check_vector(iset, v)
    return CoeffVector(iset, get_applier(iset).apply_square_sum(v.data))

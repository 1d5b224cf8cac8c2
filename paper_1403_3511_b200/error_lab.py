"""Hamiltonian glue for the propagation loop (drop-in for hprop.error_lab.FastHamiltonian).

Only the hot-path pieces of pkg/src/hprop/error_lab.py are mirrored:
`FastHamiltonian` (error_lab.py:154-185) and `make_decay_vector`
(error_lab.py:43-56).  The error studies are out of scope.

A(t) = D + W_pol(t) [+ q * sum_l x_l^2 through the exact banded entries],
with W_pol the Chebyshev surrogate of the smooth remainder of the potential.
`matvec_at(t)` returns a callable (drop-in for the reference's lambda) that
also carries the term list, so `lanczos` / `propagate_magnus` can dispatch
to the fused device step `hp_magnus_step`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .fast_apply import _term_arrays, get_applier
from .index_set import CoeffVector, IndexSet, _is_torch
from .krylov_propagator import LanczosFactorization, MagnusScheme, _SQRT3
from .potential_approx import ChebApprox, PotentialSpec, interpolate, smooth_remainder


def make_decay_vector(iset: IndexSet, beta: int, *, normalized: bool = True) -> CoeffVector:
    """v_k = prod_l max(k_l, 1)^(-beta) (error_lab.py:43-56)."""
    if beta < 1:
        raise ValueError(f"beta must be a positive integer, got {beta}")
    base = np.maximum(iset.indices, 1).astype(np.float64)
    data = np.prod(base ** (-float(beta)), axis=1)
    if normalized:
        data = data / np.linalg.norm(data)
    return CoeffVector(iset, data)


class _HamMatVec:
    """v -> A(t) v for one frozen t; callable like the reference's lambda."""

    def __init__(self, fh: "FastHamiltonian", approx: ChebApprox):
        self.fh = fh
        self.approx = approx
        self._hp_hamiltonian = self

    def __call__(self, v):
        appl = get_applier(self.fh.iset)
        out = appl.apply_hamiltonian(self.approx, v)
        q = self.fh.potential.harmonic_part
        if q != 0.0:
            out += q * appl.apply_square_sum(v)
        return out

    def lanczos(self, v0, steps: int, *, reorthogonalize: bool = False) -> LanczosFactorization:
        import torch

        fh = self.fh
        iset = fh.iset
        n = iset.size
        v, host = fh._vec(v0)
        if float(torch.linalg.vector_norm(v)) == 0.0:
            raise ValueError("starting vector must be nonzero")
        degs, coeffs = _term_arrays(self.approx, iset.dim)
        L = nat.lib()
        h = ctypes.c_void_p(iset.handle)
        wsb = L.hp_magnus_workspace_bytes(h, 0, degs.ctypes.data_as(nat.c_i32p), degs.shape[0], None, 0, 0)
        ws = torch.empty(int(wsb), dtype=torch.uint8, device="cuda")
        V = torch.empty((steps, n), dtype=torch.complex128, device="cuda")
        al = torch.zeros(steps, dtype=torch.float64, device="cuda")
        be = torch.zeros(max(steps - 1, 1), dtype=torch.float64, device="cuda")
        diag = torch.zeros(4, dtype=torch.float64, device="cuda")
        nat.check(L.hp_lanczos(h, degs.ctypes.data_as(nat.c_i32p), coeffs.ctypes.data_as(nat.c_dblp),
                               degs.shape[0], float(self.approx.halfwidth), float(fh.potential.harmonic_part),
                               ctypes.c_void_p(v.data_ptr()), steps, int(reorthogonalize),
                               ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(al.data_ptr()),
                               ctypes.c_void_p(be.data_ptr()), ctypes.c_void_p(diag.data_ptr()),
                               ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr()))
        d = diag.cpu().numpy()
        m = int(d[0])
        basis = V[:m].T
        return LanczosFactorization(basis.cpu().numpy() if host else basis, al[:m].cpu().numpy(),
                                    be[:max(m - 1, 0)].cpu().numpy(), None if d[2] < 0 else int(d[2]),
                                    float(d[1]))

    def exp_step(self, v, tau, steps, *, reorthogonalize=False, want_fac=False):
        return self.fh._step([self.approx], v, tau, steps, reorthogonalize, want_fac)


@dataclass
class FastHamiltonian:
    """Matrix-free A(t) = D + W_pol(t) (error_lab.py:154-185), on the device."""

    iset: IndexSet
    potential: PotentialSpec
    degree: int
    _ws: object = field(default=None, repr=False)

    def approx_at(self, t: float, *, validate: bool = True) -> ChebApprox:
        return interpolate(smooth_remainder(self.potential), self.degree, time=t, validate=validate)

    def matvec_at(self, t: float):
        return _HamMatVec(self, self.approx_at(t))

    # -- device stepping ---------------------------------------------------------
    def _vec(self, y):
        import torch

        if _is_torch(y):
            return y.to(device="cuda", dtype=torch.complex128).contiguous().clone(), False
        arr = np.ascontiguousarray(np.asarray(y), dtype=np.complex128)
        if arr.shape != (self.iset.size,):
            raise ValueError(f"state has shape {arr.shape}, expected ({self.iset.size},)")
        return torch.from_numpy(arr).cuda(), True

    def _workspace(self, scheme_code, term_lists, m):
        import torch

        L = nat.lib()
        h = ctypes.c_void_p(self.iset.handle)
        d1, _ = _term_arrays(term_lists[0], self.iset.dim)
        d2 = _term_arrays(term_lists[1], self.iset.dim)[0] if len(term_lists) > 1 else None
        need = L.hp_magnus_workspace_bytes(h, scheme_code, d1.ctypes.data_as(nat.c_i32p), d1.shape[0],
                                           d2.ctypes.data_as(nat.c_i32p) if d2 is not None else None,
                                           d2.shape[0] if d2 is not None else 0, m)
        # term counts may vary with t; keep 25% headroom and regrow if needed
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(int(need * 1.25) + 4096, dtype=torch.uint8, device="cuda")
        return self._ws

    def _step_dev(self, approxes, ydev, h, m, reorth, diag=None):
        L = nat.lib()
        ws = self._workspace(1 if len(approxes) == 2 else 0, approxes, m)
        d1, c1 = _term_arrays(approxes[0], self.iset.dim)
        if len(approxes) == 2:
            d2, c2 = _term_arrays(approxes[1], self.iset.dim)
            dp2, cp2, n2 = d2.ctypes.data_as(nat.c_i32p), c2.ctypes.data_as(nat.c_dblp), d2.shape[0]
        else:
            dp2, cp2, n2 = None, None, 0
        nat.check(L.hp_magnus_step(
            ctypes.c_void_p(self.iset.handle), 1 if len(approxes) == 2 else 0,
            d1.ctypes.data_as(nat.c_i32p), c1.ctypes.data_as(nat.c_dblp), d1.shape[0], dp2, cp2, n2,
            float(approxes[0].halfwidth), float(self.potential.harmonic_part), float(h), int(m), int(reorth),
            ctypes.c_void_p(ydev.data_ptr()), ctypes.c_void_p(diag.data_ptr()) if diag is not None else None,
            ctypes.c_void_p(ws.data_ptr()), ws.numel(), nat.stream_ptr()))

    def _step(self, approxes, y, h, m, reorth, want_fac):
        import torch

        if want_fac:
            return self._step_with_factorization(approxes, y, h, m, reorth)
        ydev, host = self._vec(y)
        if float(torch.linalg.vector_norm(ydev)) == 0.0:
            raise ValueError("starting vector must be nonzero")
        diag = torch.zeros(4, dtype=torch.float64, device="cuda")
        self._step_dev(approxes, ydev, h, m, reorth, diag)
        d = diag.cpu().numpy()
        if d[3] != 0:
            raise RuntimeError("tridiagonal QL failed to converge")
        return ydev.cpu().numpy() if host else ydev

    def _step_with_factorization(self, approxes, y, h, m, reorth):
        """exp(-i h B) y together with the Lanczos factorization it was built from.

        The reference returns the real factorization (krylov_propagator.py:180-186, 237-244) and
        its callers read it (basis columns, alpha, beta).  The fused step keeps only scaled,
        unnormalised basis vectors, so this path runs the device Lanczos (hp_lanczos, normalised
        basis; or the generic device recurrence over the GL2 operator) and forms
        ||y|| V exp(-i h T) e_1 from it, exactly the reference's sequence.
        """
        import torch

        from .krylov_propagator import _expm_col_dev, _lanczos_generic

        ydev, host = self._vec(y)
        if len(approxes) == 1:
            fac = _HamMatVec(self, approxes[0]).lanczos(ydev, m, reorthogonalize=reorth)
        else:
            a1, a2 = _HamMatVec(self, approxes[0]), _HamMatVec(self, approxes[1])
            gamma = _SQRT3 / 12.0 * h

            def gl2(v):
                y1, y2 = a1(v), a2(v)
                return 0.5 * (y1 + y2) - 1j * gamma * (a2(y1) - a1(y2))

            fac = _lanczos_generic(gl2, ydev, m, reorth)
        col = _expm_col_dev(fac.alpha, fac.beta, h)
        out = float(torch.linalg.vector_norm(ydev)) * (fac.basis @ col)
        return (out.cpu().numpy() if host else out), LanczosFactorization(
            fac.basis.cpu().numpy() if host else fac.basis, fac.alpha, fac.beta, fac.breakdown_at,
            fac.hermiticity_defect)

    def _approxes(self, scheme: MagnusScheme, t: float, h: float):
        if scheme.name == "midpoint":
            return [self.approx_at(t + 0.5 * h, validate=False)]
        if scheme.name == "gl2":
            c = _SQRT3 / 6.0
            return [self.approx_at(t + (0.5 - c) * h, validate=False),
                    self.approx_at(t + (0.5 + c) * h, validate=False)]
        raise ValueError(f"unknown scheme {scheme.name!r}")

    def magnus_step(self, scheme, y, t, h, steps, *, reorthogonalize=False, want_fac=False):
        return self._step(self._approxes(scheme, t, h), y, h, steps, reorthogonalize, want_fac)

    def propagate(self, scheme, y0, t0, h, nsteps, m, *, reorthogonalize=False, callback=None):
        """krylov_propagator.py:247-263 with the state resident on the device."""
        import torch

        ydev, host = self._vec(y0)
        if float(torch.linalg.vector_norm(ydev)) == 0.0:
            raise ValueError("starting vector must be nonzero")
        diag = torch.zeros((nsteps, 4), dtype=torch.float64, device="cuda")
        for k in range(nsteps):
            t = t0 + k * h
            self._step_dev(self._approxes(scheme, t, h), ydev, h, m, reorthogonalize, diag[k])
            if callback is not None:
                # the reference raises at the failing step, before its callback sees the state;
                # the callback already costs a sync, so the QL flag is checked here per step.  Each
                # call gets its own array/tensor (the device state is overwritten in place)
                if float(diag[k, 3]) != 0:
                    raise RuntimeError("tridiagonal QL failed to converge")
                callback(k + 1, t + h, ydev.cpu().numpy() if host else ydev.clone())
        if bool((diag[:, 3] != 0).any()):
            raise RuntimeError("tridiagonal QL failed to converge")
        self.last_diagnostics = diag
        return ydev.cpu().numpy() if host else ydev

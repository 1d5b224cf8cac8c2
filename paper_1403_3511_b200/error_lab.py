"""Hamiltonian glue for the propagation loop (drop-in for hprop.error_lab.FastHamiltonian).

Mirrored from pkg/src/hprop/error_lab.py: `FastHamiltonian` (error_lab.py:154-185),
`make_decay_vector` (:43-56) and the reduction-error measurement that runs the same device
matvec on the set and on its full cube -- `reduction_error`, `reduction_local_mask`,
`ErrorReport` (:59-79, :114-148).  The quadrature and Lanczos
perturbation studies (dense assembled matrices) are out of scope.

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
from .fast_apply import _term_arrays, fast_algorithm, get_applier
from .index_set import CoeffVector, IndexSet, _is_torch, build_full, extend
from .krylov_propagator import LanczosFactorization, MagnusScheme, _SQRT3
from .potential_approx import ChebApprox, PotentialSpec, interpolate, smooth_remainder


MEASURE_QUADRATURE = "quadrature"
MEASURE_REDUCTION = "reduction"


@dataclass(frozen=True)
class ErrorReport:
    """Per-index error magnitudes over a set with provenance (error_lab.py:59-79).

    ``components`` is a float64 array (numpy, or a CUDA tensor when the input vector was one).
    """

    iset: IndexSet
    components: object
    metadata: dict

    def _host(self) -> np.ndarray:
        c = self.components
        return c.cpu().numpy() if _is_torch(c) else np.asarray(c)

    @property
    def max_norm(self) -> float:
        c = self._host()
        return float(c.max()) if c.size else 0.0

    def write_csv(self, path) -> None:
        """Sorted ``# key=value`` metadata lines, ``# max_norm``, then k_1..k_N,magnitude rows."""
        lines = [f"# {k}={self.metadata[k]}\n" for k in sorted(self.metadata)]
        lines.append(f"# max_norm={self.max_norm:.17g}\n")
        lines.append(",".join([f"k_{a + 1}" for a in range(self.iset.dim)] + ["magnitude"]) + "\n")
        rows = self.iset.indices.tolist()
        lines.extend(",".join(map(str, r)) + f",{m:.17g}\n" for r, m in zip(rows, self._host()))
        with open(path, "w", newline="\n") as fh:
            fh.write("".join(lines))


def _metadata(iset: IndexSet, approx: ChebApprox, measure: str, **extra) -> dict:
    md = dict(measure=measure, dim=iset.dim, bound=iset.bound, set_kind=iset.kind, set_size=iset.size,
              degree=approx.degree, halfwidth=approx.halfwidth, nterms=approx.nterms)
    md.update(extra)
    return md


def reduction_error(iset: IndexSet, approx: ChebApprox, v: CoeffVector, *,
                    full: IndexSet | None = None) -> ErrorReport:
    """|fast(set) v - restrict(fast(cube) extend(v))| per index (error_lab.py:114-130).

    Both applications are the device matvec; extend is a device scatter and the final
    restrict-and-subtract is one fused kernel (hp_reduction_components).  Components stay on the
    device when v does.
    """
    import torch

    if full is None:
        full = build_full(iset.dim, iset.bound)
    on_set = fast_algorithm(iset, approx, v).data
    on_full = fast_algorithm(full, approx, extend(v, full)).data
    host = not _is_torch(on_set)
    a = torch.from_numpy(np.ascontiguousarray(on_set)).cuda() if host else on_set.contiguous()
    b = torch.from_numpy(np.ascontiguousarray(on_full)).cuda() if host else on_full.contiguous()
    if a.dtype != b.dtype:
        common = torch.promote_types(a.dtype, b.dtype)
        a, b = a.to(common), b.to(common)
    a = iset._to_canon(a)  # the fused kernel walks the set's device (canonical) order
    comp = torch.empty(iset.size, dtype=torch.float64, device=a.device)
    L = nat.lib()
    nat.check(L.hp_reduction_components(ctypes.c_void_p(iset.handle), ctypes.c_void_p(full.handle),
                                        nat.HP_C128 if a.is_complex() else nat.HP_F64, ctypes.c_void_p(a.data_ptr()),
                                        ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(comp.data_ptr()),
                                        nat.stream_ptr()))
    comp = iset._from_canon(comp)
    return ErrorReport(iset, comp.cpu().numpy() if host else comp,
                       _metadata(iset, approx, MEASURE_REDUCTION, full_size=full.size))


def reduction_local_mask(iset: IndexSet, approx: ChebApprox) -> np.ndarray:
    """Indices whose reduction error must vanish: j + r in the set for every degree tuple r of
    the surrogate (error_lab.py:133-148), by device up-walks through the neighbour tables."""
    import torch

    degs, _ = _term_arrays(approx, iset.dim)
    mask = torch.empty(iset.size, dtype=torch.uint8, device="cuda")
    nat.check(nat.lib().hp_reduction_local_mask(ctypes.c_void_p(iset.handle), degs.ctypes.data_as(nat.c_i32p),
                                                degs.shape[0], ctypes.c_void_p(mask.data_ptr()), nat.stream_ptr()))
    return iset._from_canon(mask).cpu().numpy().astype(bool)


def make_decay_vector(iset: IndexSet, beta: int, *, normalized: bool = True, device: bool = False) -> CoeffVector:
    """v_k = prod_l max(k_l, 1)^(-beta), optionally normalised (error_lab.py:43-56), computed on the
    device from the set's tables (hp_decay_vector) and normalised by the device 2-norm.  Returns
    host data like the reference; ``device=True`` keeps a CUDA tensor."""
    import torch

    if beta < 1:
        raise ValueError(f"beta must be a positive integer, got {beta}")
    d = torch.empty(iset.size, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().hp_decay_vector(ctypes.c_void_p(iset.handle), int(beta), ctypes.c_void_p(d.data_ptr()),
                                        nat.stream_ptr()))
    d = iset._from_canon(d)
    if normalized:
        d = d / torch.linalg.vector_norm(d)
    return CoeffVector(iset, d if device else d.cpu().numpy())


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
        v, kind = fh._vec(v0)
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
        basis = fh._out(V[:m], kind).T  # rows in the caller's order, as an (n, m) view
        return LanczosFactorization(basis, al[:m].cpu().numpy(),
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
        """The state as a fresh complex128 CUDA tensor in the device set's order, and its kind
        ("numpy", "cpu" for a host torch tensor, "cuda") for `_out`."""
        import torch

        if _is_torch(y):
            kind = "cuda" if y.is_cuda else "cpu"
            t = y.to(device="cuda", dtype=torch.complex128, non_blocking=True).contiguous()
            if t.data_ptr() == y.data_ptr():
                t = t.clone()  # the step updates the state in place
        else:
            kind = "numpy"
            arr = np.ascontiguousarray(np.asarray(y), dtype=np.complex128)
            if arr.shape != (self.iset.size,):
                raise ValueError(f"state has shape {arr.shape}, expected ({self.iset.size},)")
            t = torch.from_numpy(arr).cuda()
        if t.shape[-1] != self.iset.size:
            raise ValueError(f"state has shape {tuple(t.shape)}, expected ({self.iset.size},)")
        return self.iset._to_canon(t), kind

    def _out(self, t, kind, *, copy: bool = False):
        """A device-order tensor back to the caller's form and order: numpy for numpy input, a
        pinned host tensor for a host tensor, else a CUDA tensor (a copy when ``copy``)."""
        import torch

        u = self.iset._from_canon(t)
        if kind == "numpy":
            return u.cpu().numpy()
        if kind == "cpu":
            out = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
            out.copy_(u)
            return out
        return u.clone() if copy and u is t else u

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
        ydev, kind = self._vec(y)
        if float(torch.linalg.vector_norm(ydev)) == 0.0:
            raise ValueError("starting vector must be nonzero")
        diag = torch.zeros(4, dtype=torch.float64, device="cuda")
        self._step_dev(approxes, ydev, h, m, reorth, diag)
        d = diag.cpu().numpy()
        if d[3] != 0:
            raise RuntimeError("tridiagonal QL failed to converge")
        return self._out(ydev, kind)

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

        # caller-order device vector: the factorization's basis is in the caller's order (every
        # matvec below permutes at the applier boundary itself)
        host = not _is_torch(y)
        yd = torch.from_numpy(np.ascontiguousarray(y, dtype=np.complex128)).cuda() if host else \
            y.to(device="cuda", dtype=torch.complex128).contiguous()
        if len(approxes) == 1:
            fac = _HamMatVec(self, approxes[0]).lanczos(yd, m, reorthogonalize=reorth)
        else:
            a1, a2 = _HamMatVec(self, approxes[0]), _HamMatVec(self, approxes[1])
            gamma = _SQRT3 / 12.0 * h

            def gl2(v):
                y1, y2 = a1(v), a2(v)
                return 0.5 * (y1 + y2) - 1j * gamma * (a2(y1) - a1(y2))

            fac = _lanczos_generic(gl2, yd, m, reorth)
        col = _expm_col_dev(fac.alpha, fac.beta, h)
        out = float(torch.linalg.vector_norm(yd)) * (fac.basis @ col)
        if host:
            return out.cpu().numpy(), LanczosFactorization(fac.basis.cpu().numpy(), fac.alpha, fac.beta,
                                                           fac.breakdown_at, fac.hermiticity_defect)
        return (out if y.is_cuda else out.cpu()), fac

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

        ydev, kind = self._vec(y0)
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
                callback(k + 1, t + h, self._out(ydev, kind, copy=True))
        if bool((diag[:, 3] != 0).any()):
            raise RuntimeError("tridiagonal QL failed to converge")
        self.last_diagnostics = diag
        return self._out(ydev, kind)

"""Device-resident Lanczos / Magnus propagation (drop-in for hprop.krylov_propagator).

Same names and signatures as pkg/src/hprop/krylov_propagator.py.  When the
operator is a `FastHamiltonian` over a device index set (the hot path,
error_lab.py:154-185), every step -- m polynomial matvecs, the Lanczos
recurrence with deterministic FP64 reductions, breakdown handling, the
tridiagonal QL eigensolve and the exp(-i h T) e_1 combine -- runs in one
asynchronous call of `hp_magnus_step` (csrc/hp_krylov.cu); the host only
re-interpolates the surrogate at the step's time points.  Other matvec
callables (e.g. dense test matrices) run the same recurrence on device
tensors, with the QL/expm kernels of the library.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as nat
from .index_set import _is_torch

MatVec = Callable[[object], object]
_BREAKDOWN_TOL = 1e-14
_SQRT3 = float(np.sqrt(3.0))


@dataclass
class LanczosFactorization:
    """Basis (n, m_eff), alpha (m_eff), beta (m_eff - 1) and diagnostics
    (krylov_propagator.py:32-55)."""

    basis: object
    alpha: np.ndarray
    beta: np.ndarray
    breakdown_at: int | None
    hermiticity_defect: float

    @property
    def steps(self) -> int:
        return self.alpha.shape[0]

    def orthogonality_defect(self) -> float:
        V = self.basis
        if _is_torch(V):
            import torch

            g = V.conj().T @ V
            return float(torch.max(torch.abs(g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device))))
        g = V.conj().T @ V
        return float(np.max(np.abs(g - np.eye(g.shape[0]))))


def _dev_vec(v):
    import torch

    if _is_torch(v):
        return v.to(device="cuda", dtype=torch.complex128).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v), dtype=np.complex128)).cuda(), True


def _scalar_ws():
    import torch

    return torch.empty(int(nat.lib().hp_reduce_workspace_bytes(0)), dtype=torch.uint8, device="cuda")


def _cdot(a, b, ws, out):
    nat.check(nat.lib().hp_cdot(a.numel(), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()), nat.stream_ptr()))


def _cnrm2(a, ws, out):
    nat.check(nat.lib().hp_cnrm2(a.numel(), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                 ctypes.c_void_p(ws.data_ptr()), nat.stream_ptr()))


def lanczos(matvec: MatVec, v0, steps: int, *, reorthogonalize: bool = False) -> LanczosFactorization:
    """Run ``steps`` Hermitian Lanczos iterations from ``v0`` (krylov_propagator.py:58-104)."""
    if steps < 1:
        raise ValueError("steps must be at least 1")
    ham = getattr(matvec, "_hp_hamiltonian", None)
    if ham is not None:
        return ham.lanczos(v0, steps, reorthogonalize=reorthogonalize)
    return _lanczos_generic(matvec, v0, steps, reorthogonalize)


def _lanczos_generic(matvec, v0, steps, reorth):
    import torch

    v, host = _dev_vec(v0)
    n = v.shape[0]
    ws = _scalar_ws()
    sc = torch.zeros(2, dtype=torch.float64, device="cuda")
    _cnrm2(v, ws, sc)
    nrm = float(sc[0])
    if nrm == 0.0:
        raise ValueError("starting vector must be nonzero")
    V = torch.empty((steps, n), dtype=torch.complex128, device="cuda")
    alpha = np.empty(steps)
    beta = np.empty(max(steps - 1, 0))
    V[0] = v / nrm
    prev = torch.zeros(n, dtype=torch.complex128, device="cuda")
    bprev, defect, brk, m = 0.0, 0.0, None, steps
    for k in range(steps):
        vk = V[k]
        w = matvec(vk if not host else vk.cpu().numpy())
        w, _ = _dev_vec(w)
        _cdot(vk, w, ws, sc)
        ak = sc.cpu().numpy()
        defect = max(defect, abs(float(ak[1])))
        alpha[k] = ak[0]
        if k == steps - 1:
            break
        w = w - alpha[k] * vk - bprev * prev
        if reorth:
            B = V[:k + 1]
            w = w - B.T @ (B.conj() @ w)
        _cnrm2(w, ws, sc)
        bk = float(sc[0])
        if bk <= _BREAKDOWN_TOL:
            brk, m = k + 1, k + 1
            break
        beta[k] = bk
        V[k + 1] = w / bk
        prev, bprev = vk, bk
    basis = V[:m].T
    return LanczosFactorization(basis.cpu().numpy() if host else basis, alpha[:m].copy(),
                                beta[:max(m - 1, 0)].copy(), brk, defect)


def tridiag_eigh(alpha, beta) -> tuple[np.ndarray, np.ndarray]:
    """Implicit-shift QL eigendecomposition on the device (krylov_propagator.py:107-170)."""
    import torch

    a = torch.as_tensor(np.asarray(alpha, dtype=np.float64)).cuda()
    m = a.shape[0]
    b = torch.as_tensor(np.asarray(beta, dtype=np.float64).reshape(-1)).cuda()
    if b.numel() == 0:
        b = torch.zeros(1, dtype=torch.float64, device="cuda")
    d = torch.empty(m, dtype=torch.float64, device="cuda")
    z = torch.empty((m, m), dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().hp_tridiag_eigh(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), m,
                                        ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                                        ctypes.c_void_p(st.data_ptr()), nat.stream_ptr()))
    if int(st[0]) != 0:
        raise RuntimeError("tridiagonal QL failed to converge")
    return d.cpu().numpy(), z.cpu().numpy()


def _expm_col_dev(alpha, beta, tau):
    import torch

    a = torch.as_tensor(np.asarray(alpha, dtype=np.float64)).cuda()
    m = a.shape[0]
    b = torch.as_tensor(np.asarray(beta, dtype=np.float64).reshape(-1)).cuda()
    if b.numel() == 0:
        b = torch.zeros(1, dtype=torch.float64, device="cuda")
    col = torch.empty(m, dtype=torch.complex128, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(nat.lib().hp_expm_tridiag_column(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), m,
                                               float(tau), ctypes.c_void_p(col.data_ptr()),
                                               ctypes.c_void_p(st.data_ptr()), nat.stream_ptr()))
    if int(st[0]) != 0:
        raise RuntimeError("tridiagonal QL failed to converge")
    return col


def expm_tridiag_column(alpha, beta, tau: float) -> np.ndarray:
    """First column of exp(-i tau T) (krylov_propagator.py:173-177), on the device."""
    return _expm_col_dev(alpha, beta, tau).cpu().numpy()


def lanczos_exp_apply(matvec: MatVec, v, tau: float, steps: int, *, reorthogonalize: bool = False):
    """exp(-i tau A) v ~= ||v|| V_m exp(-i tau T_m) e_1 (krylov_propagator.py:180-186)."""
    ham = getattr(matvec, "_hp_hamiltonian", None)
    if ham is not None:
        y, fac = ham.exp_step(v, tau, steps, reorthogonalize=reorthogonalize, want_fac=True)
        return y, fac
    fac = lanczos(matvec, v, steps, reorthogonalize=reorthogonalize)
    col = _expm_col_dev(fac.alpha, fac.beta, tau)
    vt, host = _dev_vec(v)
    import torch

    B = fac.basis if _is_torch(fac.basis) else torch.from_numpy(np.asarray(fac.basis)).cuda()
    out = float(torch.linalg.vector_norm(vt)) * (B @ col)
    return (out.cpu().numpy() if host else out), fac


@dataclass(frozen=True)
class MagnusScheme:
    """A one-step exponential integrator (krylov_propagator.py:192-212)."""

    name: str
    order: int

    @staticmethod
    def from_name(name: str) -> "MagnusScheme":
        try:
            return _SCHEMES[name]
        except KeyError:
            raise ValueError(f"unknown scheme {name!r}; choose from {sorted(_SCHEMES)}") from None


_SCHEMES = {"midpoint": MagnusScheme("midpoint", 2), "gl2": MagnusScheme("gl2", 4)}


def _step_matvec(scheme: MagnusScheme, ham_at, t: float, h: float) -> MatVec:
    """The frozen operator of one step (krylov_propagator.py:215-234)."""
    if scheme.name == "midpoint":
        return ham_at(t + 0.5 * h)
    if scheme.name == "gl2":
        c = _SQRT3 / 6.0
        a1 = ham_at(t + (0.5 - c) * h)
        a2 = ham_at(t + (0.5 + c) * h)
        gamma = _SQRT3 / 12.0 * h

        def matvec(v):
            y1 = a1(v)
            y2 = a2(v)
            comm = a2(y1) - a1(y2)
            return 0.5 * (y1 + y2) - 1j * gamma * comm

        return matvec
    raise ValueError(f"unknown scheme {scheme.name!r}")


def _fast_owner(ham_at):
    from .error_lab import FastHamiltonian

    owner = getattr(ham_at, "__self__", None)
    return owner if isinstance(owner, FastHamiltonian) else None


def magnus_step(scheme: MagnusScheme, ham_at, y, t: float, h: float, steps: int, *,
                reorthogonalize: bool = False):
    """Advance y from t to t + h (krylov_propagator.py:237-244)."""
    fh = _fast_owner(ham_at)
    if fh is not None:
        return fh.magnus_step(scheme, y, t, h, steps, reorthogonalize=reorthogonalize, want_fac=True)
    return lanczos_exp_apply(_step_matvec(scheme, ham_at, t, h), y, h, steps, reorthogonalize=reorthogonalize)


def propagate_magnus(scheme: MagnusScheme, ham_at, y0, t0: float, t1: float, nsteps: int, krylov_steps: int,
                     *, reorthogonalize: bool = False, callback=None):
    """March from t0 to t1 in nsteps equal steps (krylov_propagator.py:247-263).

    With a FastHamiltonian the state never leaves the device between steps.
    """
    if nsteps < 1:
        raise ValueError("nsteps must be at least 1")
    h = (t1 - t0) / nsteps
    fh = _fast_owner(ham_at)
    if fh is not None:
        return fh.propagate(scheme, y0, t0, h, nsteps, krylov_steps, reorthogonalize=reorthogonalize,
                            callback=callback)
    host = not _is_torch(y0)
    y = np.asarray(y0, dtype=np.complex128).copy() if host else y0.to(dtype=__import__("torch").complex128)
    for k in range(nsteps):
        t = t0 + k * h
        y, _ = magnus_step(scheme, ham_at, y, t, h, krylov_steps, reorthogonalize=reorthogonalize)
        if callback is not None:
            callback(k + 1, t + h, y)
    return y

"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py.  Every routine here follows one reference routine
(cited as pkg/src/hprop/<module>.py:<lines>) operation by operation, so that
its floating-point results match the reference to the last bit wherever the
reference's own operation order is reproduced (gathers with a padded zero
slot, in-place ufunc passes, the shared single-axis sweep, per-term ordered
products).  It is the checker for the CUDA path and the CPU baseline that
bench.py times; it is never on the product path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DROP_THRESHOLD = 1e-14        # potential_approx.py:33
BREAKDOWN_TOL = 1e-14         # krylov_propagator.py:29


# ---------------------------------------------------------------------------
# index sets  (pkg/src/hprop/index_set.py)
# ---------------------------------------------------------------------------

def full_indices(dim: int, bound: int) -> np.ndarray:
    """Lexicographic full cube, last axis fastest (index_set.py:144-154)."""
    if dim <= 0 or bound < 0:
        raise ValueError("bad full-cube parameters")
    side = bound + 1
    n = side ** dim
    ords = np.arange(n, dtype=np.int64)
    out = np.empty((n, dim), dtype=np.int64)
    for a in range(dim - 1, -1, -1):
        out[:, a] = ords % side
        ords //= side
    return out


def hyperbolic_indices_recursive(dim: int, bound: int) -> np.ndarray:
    """Literal depth-first restatement of index_set.py:163-180 (small sets)."""
    rows: list[tuple[int, ...]] = []

    def walk(prefix: tuple[int, ...], budget: int) -> None:
        if len(prefix) == dim - 1:
            rows.extend(prefix + (k,) for k in range(budget))
            return
        k = 0
        while k + 1 <= budget:
            walk(prefix + (k,), budget // (k + 1))
            k += 1

    walk((), bound + 1)
    return np.asarray(rows, dtype=np.int64).reshape(len(rows), dim)


def hyperbolic_indices(dim: int, bound: int) -> np.ndarray:
    """Level-synchronous restatement of the recursion at index_set.py:163-180.

    Expanding every prefix in order into its children k = 0, 1, ... (budget
    floor(r / (k+1)), last level k < r) with order-preserving repeats gives
    exactly the depth-first emission order of the reference.
    """
    if dim <= 0 or bound < 0:
        raise ValueError("bad hyperbolic parameters")
    budgets = np.array([bound + 1], dtype=np.int64)
    cols: list[np.ndarray] = []
    for level in range(dim):
        last = level == dim - 1
        counts = budgets.copy()            # both: k ranges over 0..r-1
        parent = np.repeat(np.arange(budgets.size), counts)
        starts = np.cumsum(counts) - counts
        k = np.arange(parent.size, dtype=np.int64) - np.repeat(starts, counts)
        cols = [c[parent] for c in cols]
        cols.append(k)
        if not last:
            budgets = budgets[parent] // (k + 1)
    return np.stack(cols, axis=1) if cols else np.zeros((0, dim), np.int64)


def _packed_keys(indices: np.ndarray) -> np.ndarray:
    """Order-preserving two-word keys for lexicographic search."""
    n, dim = indices.shape
    width = max(1, int(indices.max(initial=0) + 2).bit_length())
    if width * dim > 128:
        raise ValueError("indices too wide for packed keys")
    hi = np.zeros(n, dtype=np.uint64)
    lo = np.zeros(n, dtype=np.uint64)
    for a in range(dim):
        # shift (hi, lo) left by width bits, then or in the component
        v = indices[:, a].astype(np.uint64)
        if width >= 64:
            raise ValueError("component width too large")
        hi = (hi << np.uint64(width)) | (lo >> np.uint64(64 - width))
        lo = (lo << np.uint64(width)) | v
    keys = np.empty(n, dtype=[("hi", "<u8"), ("lo", "<u8")])
    keys["hi"] = hi
    keys["lo"] = lo
    return keys


def neighbor_tables(indices: np.ndarray) -> list[tuple[np.ndarray, np.ndarray]]:
    """(down, up) ordinals per axis, -1 where absent (index_set.py:104-130).

    The reference looks every shifted row up in a position dict; here the
    lookup is a binary search over the lexicographically sorted rows, which
    yields the same ordinals (the set is sorted and duplicate-free).
    """
    n, dim = indices.shape
    keys = _packed_keys(indices)
    hi, lo = keys["hi"], keys["lo"]
    if n > 1 and not np.all((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))):
        raise ValueError("indices are not strictly lexicographically sorted")
    out = []
    for a in range(dim):
        res = []
        for delta in (-1, 1):
            shifted = indices.copy()
            shifted[:, a] += delta
            valid = shifted[:, a] >= 0
            shifted[~valid, a] = 0
            q = _packed_keys_like(shifted, indices)
            pos = np.searchsorted(keys, q)
            pos_c = np.minimum(pos, n - 1)
            hit = valid & (pos < n) & (keys[pos_c] == q)
            res.append(np.where(hit, pos_c, -1).astype(np.int64))
        out.append((res[0], res[1]))
    return out


def _packed_keys_like(rows: np.ndarray, ref: np.ndarray) -> np.ndarray:
    width = max(1, int(ref.max(initial=0) + 2).bit_length())
    n, dim = rows.shape
    hi = np.zeros(n, dtype=np.uint64)
    lo = np.zeros(n, dtype=np.uint64)
    rows = np.minimum(rows, (1 << width) - 1)
    for a in range(dim):
        v = rows[:, a].astype(np.uint64)
        hi = (hi << np.uint64(width)) | (lo >> np.uint64(64 - width))
        lo = (lo << np.uint64(width)) | v
    keys = np.empty(n, dtype=[("hi", "<u8"), ("lo", "<u8")])
    keys["hi"] = hi
    keys["lo"] = lo
    return keys


def box_neighbor_tables(shape: tuple[int, ...]) -> list[tuple[np.ndarray, np.ndarray]]:
    """Neighbour tables of a C-ordered box by stride arithmetic.

    For a full cube this equals index_set.py:104-130 (a neighbour exists iff
    it stays inside the cube).  For a slab box (a j1-range of a full cube,
    used for the sharded and sampled oracle runs) neighbours outside the
    box are absent, which only perturbs rows within r1 of the box edge.
    """
    n = int(np.prod(shape))
    ords = np.arange(n, dtype=np.int64)
    out = []
    stride = 1
    strides = []
    for s in reversed(shape):
        strides.append(stride)
        stride *= s
    strides = strides[::-1]
    for a, side in enumerate(shape):
        j = (ords // strides[a]) % side
        down = np.where(j > 0, ords - strides[a], -1)
        up = np.where(j < side - 1, ords + strides[a], -1)
        out.append((down, up))
    return out


def hyperbolic_size_table(dim: int, bound: int) -> int:
    """Size of the hyperbolic cross via the budget-count recursion."""
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def count(d: int, r: int) -> int:
        if d == 0:
            return 1
        return sum(count(d - 1, r // (k + 1)) for k in range(r))

    return count(dim, bound + 1)


# ---------------------------------------------------------------------------
# matvec  (pkg/src/hprop/fast_apply.py)
# ---------------------------------------------------------------------------

class OracleApplier:
    """Restatement of PolynomialApplier (fast_apply.py:32-245).

    ``jvals`` are the multi-indices used for the ladder coefficients and the
    oscillator levels; ``tables`` the (down, up) ordinals per axis.  For a
    plain index set both come from the set; for a slab box ``jvals`` carry
    the global j1 while the tables are box-local.
    """

    def __init__(self, jvals: np.ndarray, tables):
        n, dim = jvals.shape
        self.n, self.dim = n, dim
        self.jvals = jvals
        self.down, self.up, self.cdown, self.cup = [], [], [], []
        for a in range(dim):                                   # :47-54
            d, u = tables[a]
            self.down.append(np.where(d < 0, n, d))
            self.up.append(np.where(u < 0, n, u))
            jl = jvals[:, a].astype(np.float64)
            self.cdown.append(np.sqrt(jl / 2.0))
            self.cup.append(np.sqrt((jl + 1.0) / 2.0))
        self.osc = (jvals + 0.5).sum(axis=1).astype(np.float64)   # :55
        self._sq = None

    # fast_apply.py:59-65
    def coordinate(self, axis: int, w: np.ndarray) -> np.ndarray:
        a = axis - 1
        buf = np.zeros(self.n + 1, dtype=np.result_type(w.dtype, np.float64))
        buf[:self.n] = w
        return self.cdown[a] * buf[self.down[a]] + self.cup[a] * buf[self.up[a]]

    # fast_apply.py:69-79
    def _first(self, a, L, src, dst, scratch):
        n = self.n
        np.take(src, self.up[a], out=scratch)
        scratch *= self.cup[a]
        np.take(src, self.down[a], out=dst[:n])
        dst[:n] *= self.cdown[a]
        dst[:n] += scratch
        dst[:n] *= 1.0 / L

    # fast_apply.py:81-92
    def _advance(self, a, L, older, newer, out, scratch):
        n = self.n
        np.take(newer, self.up[a], out=scratch)
        scratch *= self.cup[a]
        np.take(newer, self.down[a], out=out[:n])
        out[:n] *= self.cdown[a]
        out[:n] += scratch
        out[:n] *= 2.0 / L
        out[:n] -= older[:n]

    # fast_apply.py:94-106 -- returns the rotated triple, result in slot 1
    def cheb_axis(self, axis, deg, L, b0, b1, b2, scratch):
        a = axis - 1
        self._first(a, L, b0, b1, scratch)
        for _ in range(deg - 1):
            self._advance(a, L, b0, b1, b2, scratch)
            b0, b1, b2 = b1, b2, b0
        return b0, b1, b2

    def cheb_apply(self, axis, deg, L, v):
        """cheb_of_coordinate_apply (fast_apply.py:281-302)."""
        if deg == 0:
            return np.array(v, copy=True)
        dt = np.result_type(v.dtype, np.float64)
        b0 = np.zeros(self.n + 1, dt)
        b1 = np.zeros(self.n + 1, dt)
        b2 = np.zeros(self.n + 1, dt)
        scratch = np.empty(self.n, dt)
        b0[:self.n] = v
        _, b1, _ = self.cheb_axis(axis, deg, L, b0, b1, b2, scratch)
        return b1[:self.n].copy()

    # fast_apply.py:110-164
    def polynomial(self, degrees, coeffs, L, v, axis_order=None):
        n, N = self.n, self.dim
        degrees = np.asarray(degrees)
        coeffs = np.asarray(coeffs)
        if axis_order is not None:
            order = [int(a) for a in axis_order]
            if sorted(order) != list(range(1, N + 1)):
                raise ValueError(f"axis_order must permute 1..{N}")
            return self.ordered_terms(degrees, coeffs, L, v, order, None)
        active = degrees > 0
        nact = active.sum(axis=1)
        dt = np.result_type(v.dtype, np.float64)
        acc = np.zeros(n, dt)
        c0 = coeffs[nact == 0].sum()
        if c0 != 0.0:
            acc += c0 * v
        single = np.nonzero(nact == 1)[0]
        if single.size:
            b0 = np.zeros(n + 1, dt)
            b1 = np.zeros(n + 1, dt)
            b2 = np.zeros(n + 1, dt)
            scratch = np.empty(n, dt)
            for axis in range(N, 0, -1):
                rows = single[active[single, axis - 1]]
                if rows.size == 0:
                    continue
                wsum: dict[int, float] = {}
                for it in rows:
                    d = int(degrees[it, axis - 1])
                    wsum[d] = wsum.get(d, 0.0) + coeffs[it]
                b0[:n] = v
                self._first(axis - 1, L, b0, b1, scratch)
                if 1 in wsum:
                    acc += wsum[1] * b1[:n]
                for d in range(2, max(wsum) + 1):
                    self._advance(axis - 1, L, b0, b1, b2, scratch)
                    b0, b1, b2 = b1, b2, b0
                    if d in wsum:
                        acc += wsum[d] * b1[:n]
        mixed = np.nonzero(nact >= 2)[0]
        if mixed.size:
            acc += self.ordered_terms(degrees, coeffs, L, v,
                                      list(range(N, 0, -1)), mixed)
        return acc

    # fast_apply.py:166-193
    def ordered_terms(self, degrees, coeffs, L, v, order, rows):
        n = self.n
        dt = np.result_type(v.dtype, np.float64)
        b0 = np.zeros(n + 1, dt)
        b1 = np.zeros(n + 1, dt)
        b2 = np.zeros(n + 1, dt)
        scratch = np.empty(n, dt)
        acc = np.zeros(n, dt)
        term = np.empty(n, dt)
        if rows is None:
            rows = range(len(coeffs))
        for it in rows:
            r = degrees[it]
            b0[:n] = v
            for axis in order:
                deg = int(r[axis - 1])
                if deg == 0:
                    continue
                b0, b1, b2 = self.cheb_axis(axis, deg, L, b0, b1, b2, scratch)
                b0, b1 = b1, b0
            np.multiply(b0[:n], coeffs[it], out=term)
            acc += term
        return acc

    # fast_apply.py:195-198
    def hamiltonian(self, degrees, coeffs, L, v):
        out = self.polynomial(degrees, coeffs, L, v)
        out += self.osc * v
        return out

    # fast_apply.py:202-227
    def _square_tables(self):
        if self._sq is None:
            n = self.n
            d2, u2, cd2, cu2 = [], [], [], []
            for a in range(self.dim):
                pd = np.append(self.down[a], n)
                pu = np.append(self.up[a], n)
                d2.append(pd[self.down[a]])
                u2.append(pu[self.up[a]])
                jl = self.jvals[:, a].astype(np.float64)
                cd2.append(np.sqrt(jl * (jl - 1.0)) / 2.0)
                cu2.append(np.sqrt((jl + 1.0) * (jl + 2.0)) / 2.0)
            self._sq = (d2, u2, cd2, cu2)
        return self._sq

    # fast_apply.py:229-245
    def square_sum(self, v):
        n = self.n
        d2, u2, cd2, cu2 = self._square_tables()
        buf = np.zeros(n + 1, dtype=np.result_type(v.dtype, np.float64))
        buf[:n] = v
        out = self.osc * v
        for a in range(self.dim):
            out += cd2[a] * buf[d2[a]]
            out += cu2[a] * buf[u2[a]]
        return out


def applier_for_set(indices: np.ndarray) -> OracleApplier:
    return OracleApplier(indices, neighbor_tables(indices))


def applier_for_full(dim: int, bound: int) -> OracleApplier:
    side = bound + 1
    return OracleApplier(full_indices(dim, bound),
                         box_neighbor_tables((side,) * dim))


def applier_for_slab(dim: int, bound: int, lo: int, hi: int) -> OracleApplier:
    """Box of planes j1 in [lo, hi) of the full cube (dim, bound)."""
    side = bound + 1
    shape = (hi - lo,) + (side,) * (dim - 1)
    j = full_indices_box(shape)
    j[:, 0] += lo
    return OracleApplier(j, box_neighbor_tables(shape))


def full_indices_box(shape) -> np.ndarray:
    n = int(np.prod(shape))
    ords = np.arange(n, dtype=np.int64)
    out = np.empty((n, len(shape)), dtype=np.int64)
    for a in range(len(shape) - 1, -1, -1):
        out[:, a] = ords % shape[a]
        ords //= shape[a]
    return out


# ---------------------------------------------------------------------------
# Chebyshev surrogate  (pkg/src/hprop/potential_approx.py)
# ---------------------------------------------------------------------------

def cheb_table(y: np.ndarray, R: int) -> np.ndarray:
    """T_0..T_R at y by the unguarded recurrence (potential_approx.py:42-50)."""
    out = np.empty((R + 1, y.shape[0]), dtype=np.float64)
    out[0] = 1.0
    if R >= 1:
        out[1] = y
    for k in range(1, R):
        out[k + 1] = 2.0 * y * out[k] - out[k - 1]
    return out


@dataclass(frozen=True)
class OracleApprox:
    dim: int
    degree: int
    halfwidth: float
    time: float
    degrees: np.ndarray
    coeffs: np.ndarray
    fit_error: float = 0.0


def validation_points(dim: int, L: float) -> np.ndarray:
    """potential_approx.py:209-217."""
    if dim == 1:
        return np.linspace(-L, L, 33)[:, None]
    if dim == 2:
        g = np.linspace(-L, L, 33)
        gx, gy = np.meshgrid(g, g, indexing="ij")
        return np.stack([gx.reshape(-1), gy.reshape(-1)], axis=1)
    return np.random.default_rng(0).uniform(-L, L, size=(33 * 33, dim))


def eval_surrogate(ap: OracleApprox, pts: np.ndarray) -> np.ndarray:
    """potential_approx.py:263-277 (points already inside the box)."""
    pts = np.atleast_2d(pts)
    if ap.coeffs.shape[0] == 0:
        return np.zeros(pts.shape[0])
    prod = np.ones((ap.coeffs.shape[0], pts.shape[0]))
    for a in range(ap.dim):
        y = np.clip(pts[:, a] / ap.halfwidth, -1.0, 1.0)
        prod *= cheb_table(y, ap.degree)[ap.degrees[:, a], :]
    return ap.coeffs @ prod


def interpolate(evaluator, dim: int, L: float, R: int, t: float = 0.0,
                with_fit: bool = True) -> OracleApprox:
    """Tensor Chebyshev-Gauss interpolation (potential_approx.py:220-260)."""
    m = R + 1
    theta = np.pi * (2.0 * np.arange(m) + 1.0) / (2.0 * m)
    nodes = L * np.cos(theta)
    grids = np.meshgrid(*([nodes] * dim), indexing="ij")
    pts = np.stack([g.reshape(-1) for g in grids], axis=1)
    vals = np.asarray(evaluator(pts, float(t)), dtype=np.float64)
    if not np.all(np.isfinite(vals)):
        raise ValueError("potential evaluated to a non-finite value")
    dct = np.cos(np.arange(m)[:, None] * theta[None, :]) * (2.0 / m)
    dct[0] *= 0.5
    c = vals.reshape((m,) * dim)
    for _ in range(dim):
        c = np.tensordot(c, dct, axes=([0], [1]))
    amax = float(np.max(np.abs(c))) if c.size else 0.0
    if amax == 0.0:
        degs = np.zeros((0, dim), dtype=np.int64)
        kept = np.zeros(0)
    else:
        mask = np.abs(c) > DROP_THRESHOLD * amax
        degs = np.argwhere(mask).astype(np.int64)
        kept = c[mask]
    ap = OracleApprox(dim, R, float(L), float(t), degs, kept, 0.0)
    if not with_fit:
        return ap
    vp = validation_points(dim, L)
    fit = float(np.max(np.abs(eval_surrogate(ap, vp) - evaluator(vp, float(t)))))
    return OracleApprox(dim, R, float(L), float(t), degs, kept, fit)


# ---------------------------------------------------------------------------
# Lanczos / Magnus  (pkg/src/hprop/krylov_propagator.py)
# ---------------------------------------------------------------------------

@dataclass
class OracleLanczos:
    basis: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    breakdown_at: int | None
    hermiticity_defect: float


def lanczos(matvec, v0, steps: int, reorthogonalize: bool = False) -> OracleLanczos:
    """krylov_propagator.py:58-104."""
    if steps < 1:
        raise ValueError("steps must be at least 1")
    v0 = np.asarray(v0)
    nrm = np.linalg.norm(v0)
    if nrm == 0.0:
        raise ValueError("starting vector must be nonzero")
    dt = np.result_type(v0.dtype, np.complex128)
    n = v0.shape[0]
    V = np.empty((n, steps), dtype=dt)
    al = np.empty(steps)
    be = np.empty(max(steps - 1, 0))
    V[:, 0] = v0 / nrm
    prev = np.zeros(n, dtype=dt)
    bprev = 0.0
    defect = 0.0
    brk = None
    m = steps
    for k in range(steps):
        vk = V[:, k]
        w = np.asarray(matvec(vk), dtype=dt)
        ak = vk.conj() @ w
        defect = max(defect, abs(float(ak.imag)))
        al[k] = ak.real
        if k == steps - 1:
            break
        w = w - al[k] * vk - bprev * prev
        if reorthogonalize:
            w = w - V[:, :k + 1] @ (V[:, :k + 1].conj().T @ w)
        bk = float(np.linalg.norm(w))
        if bk <= BREAKDOWN_TOL:
            brk = k + 1
            m = k + 1
            break
        be[k] = bk
        V[:, k + 1] = w / bk
        prev = vk
        bprev = bk
    return OracleLanczos(V[:, :m], al[:m].copy(), be[:max(m - 1, 0)].copy(),
                         brk, defect)


def tridiag_eigh(alpha, beta):
    """Implicit-shift QL (krylov_propagator.py:107-170)."""
    d = np.asarray(alpha, dtype=np.float64).copy()
    m = d.shape[0]
    e = np.zeros(m)
    if m > 1:
        e[:m - 1] = np.asarray(beta, dtype=np.float64)
    z = np.eye(m)
    if m == 1:
        return d, z
    for l in range(m):
        it = 0
        while True:
            mm = l
            while mm < m - 1:
                if abs(e[mm]) <= 1e-14 * (abs(d[mm]) + abs(d[mm + 1])):
                    break
                mm += 1
            if mm == l:
                break
            if it == 30:
                raise RuntimeError(
                    f"tridiagonal QL failed to converge for eigenvalue {l}")
            it += 1
            g = (d[l + 1] - d[l]) / (2.0 * e[l])
            r = np.hypot(g, 1.0)
            g = d[mm] - d[l] + e[l] / (g + (r if g >= 0 else -r))
            s = c = 1.0
            p = 0.0
            early = False
            for i in range(mm - 1, l - 1, -1):
                f = s * e[i]
                b = c * e[i]
                r = np.hypot(f, g)
                e[i + 1] = r
                if r == 0.0:
                    d[i + 1] -= p
                    e[mm] = 0.0
                    early = True
                    break
                s = f / r
                c = g / r
                g = d[i + 1] - p
                r = (d[i] - g) * s + 2.0 * c * b
                p = s * r
                d[i + 1] = g + p
                g = c * r - b
                zi = z[:, i].copy()
                zi1 = z[:, i + 1].copy()
                z[:, i + 1] = s * zi + c * zi1
                z[:, i] = c * zi - s * zi1
            if not early:
                d[l] -= p
                e[l] = g
                e[mm] = 0.0
    order = np.argsort(d, kind="stable")
    return d[order], z[:, order]


def expm_tridiag_column(alpha, beta, tau):
    """krylov_propagator.py:173-177."""
    d, z = tridiag_eigh(alpha, beta)
    return z @ (np.exp(-1j * tau * d) * z[0, :])


def lanczos_exp_apply(matvec, v, tau, steps, reorthogonalize=False):
    """krylov_propagator.py:180-186."""
    fac = lanczos(matvec, v, steps, reorthogonalize)
    col = expm_tridiag_column(fac.alpha, fac.beta, tau)
    return float(np.linalg.norm(v)) * (fac.basis @ col), fac


_SQRT3 = float(np.sqrt(3.0))


def step_matvec(scheme: str, ham_at, t: float, h: float):
    """krylov_propagator.py:215-234."""
    if scheme == "midpoint":
        return ham_at(t + 0.5 * h)
    if scheme == "gl2":
        c = _SQRT3 / 6.0
        a1 = ham_at(t + (0.5 - c) * h)
        a2 = ham_at(t + (0.5 + c) * h)
        gamma = _SQRT3 / 12.0 * h

        def mv(v):
            y1 = a1(v)
            y2 = a2(v)
            comm = a2(y1) - a1(y2)
            return 0.5 * (y1 + y2) - 1j * gamma * comm

        return mv
    raise ValueError(f"unknown scheme {scheme!r}")


def propagate(scheme: str, ham_at, y0, t0, t1, nsteps, m,
              reorthogonalize=False, callback=None):
    """krylov_propagator.py:247-263."""
    if nsteps < 1:
        raise ValueError("nsteps must be at least 1")
    h = (t1 - t0) / nsteps
    y = np.asarray(y0, dtype=np.complex128).copy()
    for k in range(nsteps):
        t = t0 + k * h
        y, _ = lanczos_exp_apply(step_matvec(scheme, ham_at, t, h), y, h, m,
                                 reorthogonalize)
        if callback is not None:
            callback(k + 1, t + h, y)
    return y


def hamiltonian_at(appl: OracleApplier, evaluator, dim, L, R,
                   harmonic_part: float = 0.0):
    """FastHamiltonian.matvec_at (error_lab.py:154-185)."""
    if harmonic_part != 0.0:
        q = harmonic_part

        def rem(pts, t):
            return evaluator(pts, t) - q * (pts * pts).sum(axis=-1)
    else:
        rem = evaluator

    def ham_at(t):
        ap = interpolate(rem, dim, L, R, t)
        if harmonic_part == 0.0:
            return lambda v: appl.hamiltonian(ap.degrees, ap.coeffs, L, v)

        def mv(v):
            out = appl.hamiltonian(ap.degrees, ap.coeffs, L, v)
            out += harmonic_part * appl.square_sum(v)
            return out
        return mv

    return ham_at


def decay_vector(indices: np.ndarray, beta: float) -> np.ndarray:
    """make_decay_vector (error_lab.py:43-56)."""
    v = np.prod(np.maximum(indices, 1).astype(np.float64) ** (-beta), axis=1)
    return v / np.linalg.norm(v)

"""Seeded synthetic workloads cfg1..cfg5 of BASELINE.json.

There is no dataset: each configuration is a set, a potential W(x, t) and
seeded complex coefficient vectors.  The same arrays feed the GPU path, the
oracle checks and the CPU baseline.  Recipes (pinned, and asserted by the
tests through the resulting term counts 6/35/22/10/97 at L = 16):

* coefficients: rng = default_rng([cfg, 0]); a = rng.standard_normal(n),
  b = rng.standard_normal(n) (shape (32, n) for cfg5); c = (a + ib) * decay(j),
  each vector normalised to unit 2-norm;
* random polynomials: rng_w = default_rng([cfg, 1]); exponents enumerated
  lexicographically over itertools.product(range(5), repeat=N);
* L = 16 (the reference default, cli.py:111), harmonic_part = 0 so that
  1/2 |x|^2 goes through the surrogate: the matvec is literally W(X) c.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .potential_approx import custom_potential, interpolate

HALFWIDTH = 16.0


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str            # "full" | "hyperbolic"
    dim: int
    bound: int           # reference `bound` (K+1 functions per direction for full cubes)
    degree: int          # surrogate degree R
    batch: int
    nsteps: int          # propagation steps (0: matvec-only config)
    dt: float
    evaluator: Callable
    decay: str
    seed: int
    matvecs: int = 1

    def spec(self):
        return custom_potential(self.evaluator, self.dim, HALFWIDTH)

    def approx(self, t: float = 0.0, validate: bool = True):
        return interpolate(self.spec(), self.degree, t, validate=validate)

    def size(self) -> int:
        if self.kind == "full":
            return (self.bound + 1) ** self.dim
        from functools import lru_cache

        @lru_cache(maxsize=None)
        def cnt(d, r):
            if d == 0:
                return 1
            return sum(cnt(d - 1, r // (k + 1)) for k in range(r))

        return cnt(self.dim, self.bound + 1)

    def scaled(self, bound: int, name: str | None = None) -> "Workload":
        return Workload(name or f"{self.name}@{bound}", self.kind, self.dim, bound, self.degree, self.batch,
                        self.nsteps, self.dt, self.evaluator, self.decay, self.seed, self.matvecs)


# ---------------------------------------------------------------- potentials

def _half_sq(p):
    return 0.5 * (p * p).sum(axis=-1)


def w_cfg1(p, t):
    x1, x2 = p[:, 0], p[:, 1]
    return 0.5 * (x1 ** 2 + x2 ** 2) + 0.1 * (x1 ** 2 * x2 - x2 ** 3 / 3.0)


def _monomials(p, exps, coeffs):
    out = np.zeros(p.shape[0])
    for a, u in zip(exps, coeffs):
        term = np.full(p.shape[0], u)
        for l, e in enumerate(a):
            if e:
                term = term * p[:, l] ** e
        out = out + term
    return out


def _cfg2_poly():
    rng = np.random.default_rng([2, 1])
    exps = [a for a in itertools.product(range(5), repeat=3) if sum(a) <= 4]
    coeffs = [rng.uniform(-1.0, 1.0) / math.factorial(sum(a)) for a in exps]
    return exps, coeffs


_CFG2 = _cfg2_poly()


def w_cfg2(p, t):
    return _monomials(p, *_CFG2) + _half_sq(p)


def w_cfg3(p, t):
    sq = p * p
    cross = 0.0
    for k in range(p.shape[1]):
        for l in range(k + 1, p.shape[1]):
            cross = cross + sq[:, k] * sq[:, l]
    return _half_sq(p) + 0.05 * cross


def w_cfg4(p, t):
    return _half_sq(p) + 0.1 * math.cos(2.0 * t) * p[:, 0] * p[:, 1] + 0.01 * (p ** 4).sum(axis=-1)


def _cfg5_poly():
    rng = np.random.default_rng([5, 1])
    exps = [a for a in itertools.product(range(5), repeat=8) if 1 <= sum(a) <= 4]
    pick = np.sort(rng.choice(len(exps), 64, replace=False))
    u = rng.uniform(-0.1, 0.1, 64)
    return [exps[i] for i in pick], list(u)


_CFG5 = _cfg5_poly()


def w_cfg5(p, t):
    return _monomials(p, *_CFG5) + _half_sq(p)


CONFIGS = {
    "cfg1": Workload("cfg1", "full", 2, 31, 3, 1, 100, 0.01, w_cfg1, "exp_sum8", 1),
    "cfg2": Workload("cfg2", "full", 3, 63, 4, 1, 0, 0.0, w_cfg2, "exp_each16", 2, matvecs=1000),
    "cfg3": Workload("cfg3", "hyperbolic", 6, 16383, 2, 1, 200, 0.001, w_cfg3, "inv_prod", 3),
    "cfg4": Workload("cfg4", "full", 4, 127, 4, 1, 50, 0.005, w_cfg4, "exp_sum32", 4),
    "cfg5": Workload("cfg5", "hyperbolic", 8, 4095, 4, 32, 0, 0.0, w_cfg5, "inv_prod", 5),
}

EXPECTED_NTERMS = {"cfg1": 6, "cfg2": 35, "cfg3": 22, "cfg4": 10, "cfg5": 97}


# ---------------------------------------------------------------- vectors

def decay_values(decay: str, indices: np.ndarray) -> np.ndarray:
    j = indices.astype(np.int64)
    if decay == "exp_sum8":
        return np.exp(-(j.sum(axis=1)) / 8.0)
    if decay == "exp_sum32":
        return np.exp(-(j.sum(axis=1)) / 32.0)
    if decay == "exp_each16":
        return np.prod(np.exp(-j / 16.0), axis=1)
    if decay == "inv_prod":
        return 1.0 / np.prod(1.0 + j, axis=1)
    raise ValueError(decay)


def _full_rows(dim: int, bound: int, lo: int, hi: int) -> np.ndarray:
    side = bound + 1
    ords = np.arange(lo, hi, dtype=np.int64)
    out = np.empty((hi - lo, dim), dtype=np.int64)
    for a in range(dim - 1, -1, -1):
        out[:, a] = ords % side
        ords //= side
    return out


def coefficients(w: Workload, indices: np.ndarray | None = None, chunk: int = 1 << 24) -> np.ndarray:
    """Seeded normalised complex coefficients, shape (n,) or (batch, n).

    ``indices`` (n x dim) is required for reduced sets; full cubes derive
    the multi-indices from the ordinal.  Generation is chunked, so cfg4's
    2.7e8-entry vector needs no multi-GB temporaries.
    """
    n = w.size()
    rng = np.random.default_rng([w.seed, 0])
    shape = (w.batch, n) if w.batch > 1 else (n,)
    c = np.empty(shape, dtype=np.complex128)
    flat = c.reshape(-1)
    total = flat.shape[0]
    for part in ("re", "im"):
        for s in range(0, total, chunk):
            e = min(total, s + chunk)
            vals = rng.standard_normal(e - s)
            if part == "re":
                flat.real[s:e] = vals
            else:
                flat.imag[s:e] = vals
    rows = c.reshape(-1, n)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = _full_rows(w.dim, w.bound, s, e) if w.kind == "full" else indices[s:e]
        dec = decay_values(w.decay, idx)
        rows[:, s:e] *= dec[None, :]
    # norms by numpy's pairwise summation (not BLAS dot, whose result depends
    # on the host's OpenBLAS thread count): identical inputs on every machine
    for r in range(rows.shape[0]):
        _normalise(rows[r], chunk)
    return c


def _normalise(row: np.ndarray, chunk: int) -> None:
    n = row.shape[0]
    sq = 0.0
    for s in range(0, n, chunk):
        blk = row[s:min(n, s + chunk)]
        sq += float(np.sum(blk.real * blk.real) + np.sum(blk.imag * blk.imag))
    row /= math.sqrt(sq)


def coefficients_rows(w: Workload, indices: np.ndarray | None, lo: int, hi: int,
                      chunk: int = 1 << 24) -> np.ndarray:
    """Rows [lo, hi) of ``coefficients(w, indices)`` (shape (hi - lo, n)), bit-identical, without
    the rest of the batch: the seeded stream is drawn in the same chunks as ``coefficients`` and
    the other rows' draws are discarded (a cfg5 rank of a batch-partitioned run holds 4 of the
    32 rows: 1.6 GB instead of 13 GB)."""
    n = w.size()
    if not 0 <= lo < hi <= w.batch:
        raise ValueError("row range out of bounds")
    rng = np.random.default_rng([w.seed, 0])
    total = w.batch * n
    out = np.empty((hi - lo, n), dtype=np.complex128)
    flat = out.reshape(-1)
    a0, a1 = lo * n, hi * n
    for part in ("re", "im"):
        for s in range(0, total, chunk):
            e = min(total, s + chunk)
            vals = rng.standard_normal(e - s)
            a, b = max(s, a0), min(e, a1)
            if a < b:
                if part == "re":
                    flat.real[a - a0:b - a0] = vals[a - s:b - s]
                else:
                    flat.imag[a - a0:b - a0] = vals[a - s:b - s]
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = _full_rows(w.dim, w.bound, s, e) if w.kind == "full" else indices[s:e]
        out[:, s:e] *= decay_values(w.decay, idx)[None, :]
    for r in range(out.shape[0]):
        _normalise(out[r], chunk)
    return out


def coefficients_row(w: Workload, indices: np.ndarray | None, row: int, chunk: int = 1 << 24) -> np.ndarray:
    """Row ``row`` of ``coefficients(w, indices)``, bit-identical (see coefficients_rows)."""
    if not 0 <= row < w.batch:
        raise ValueError("row out of range")
    return coefficients_rows(w, indices, row, row + 1, chunk)[0]

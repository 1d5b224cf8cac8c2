"""Multi-GPU decomposition of full-cube states: slabs along j1.

The vector of a full cube is C-ordered with j1 outermost, so the planes
j1 in [lo, hi) of rank r are one contiguous block.  A polynomial whose
largest axis-1 degree is r1 couples plane p only to planes p - r1 .. p + r1
(every axis-1 factor is a Chebyshev sweep of at most r1 ladder steps), so
each rank keeps a box [lo - h, hi + h) (h >= r1, clipped to the cube),
receives the h boundary planes of each neighbour before every matvec, runs
the local matvec on the box (a slab set: j1 keeps its global value, the
faces of the box are treated as absent neighbours) and owns the exact
result on [lo, hi).  The exchange is one contiguous send/recv pair per
neighbour over NCCL (torch.distributed; gloo in the CPU tests).  Krylov
inner products reduce per-rank partial sums in rank order (all_gather,
then a fixed-order sum) so that every rank sees identical scalars.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# input planes the fused full-cube kernel reads on each side of an output plane (hp_fg1.cuh F1_H)
RADIUS = 4


def partition(planes: int, world: int, rank: int) -> tuple[int, int]:
    """Near-equal contiguous split of `planes` j1-planes over `world` ranks."""
    base, extra = divmod(planes, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


@dataclass
class SlabGeometry:
    dim: int
    bound: int
    rank: int
    world: int
    halo: int

    def __post_init__(self):
        self.planes = self.bound + 1
        self.plane = self.planes ** (self.dim - 1)
        self.lo, self.hi = partition(self.planes, self.world, self.rank)
        if self.planes // self.world < self.halo and self.world > 1:
            raise ValueError(f"{self.planes} planes over {self.world} ranks leave fewer owned planes "
                             f"than the halo depth {self.halo}")
        self.blo = max(0, self.lo - self.halo)
        self.bhi = min(self.planes, self.hi + self.halo)
        self.global_size = self.planes * self.plane

    # element offsets inside the local box buffer
    @property
    def box_size(self) -> int:
        return (self.bhi - self.blo) * self.plane

    @property
    def own_slice(self) -> slice:
        return slice((self.lo - self.blo) * self.plane, (self.hi - self.blo) * self.plane)

    def exchanges(self):
        """(peer, send_slice, recv_slice) in box coordinates, lower neighbour first.

        What is sent is sized by the *peer's* halo (its box may be clipped
        differently at the cube faces); what is received by our own.
        """
        out = []
        p = self.plane
        if self.rank > 0:
            send_depth = min(self.halo, self.planes - self.lo)   # upper halo of rank - 1
            send = slice((self.lo - self.blo) * p, (self.lo - self.blo + send_depth) * p)
            recv = slice(0, (self.lo - self.blo) * p)
            out.append((self.rank - 1, send, recv))
        if self.rank < self.world - 1:
            send_depth = min(self.halo, self.hi)                 # lower halo of rank + 1
            send = slice((self.hi - self.blo - send_depth) * p, (self.hi - self.blo) * p)
            recv = slice((self.hi - self.blo) * p, (self.bhi - self.blo) * p)
            out.append((self.rank + 1, send, recv))
        return out


def halo_exchange(geo: SlabGeometry, box, group=None) -> None:
    """Fill the halo planes of `box` (a flat tensor of geo.box_size) from the neighbours."""
    import torch.distributed as dist

    import torch

    buf = torch.view_as_real(box) if box.is_complex() else box  # plane slices stay contiguous
    ops = []
    for peer, send, recv in geo.exchanges():
        ops.append(dist.P2POp(dist.isend, buf[send], peer, group))
        ops.append(dist.P2POp(dist.irecv, buf[recv], peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def emulate_exchange(geos, boxes) -> None:
    """Single-process stand-in for halo_exchange over all ranks (tests): the same
    plan, executed as device-to-device copies between the ranks' boxes."""
    for g, box in zip(geos, boxes):
        for peer, _send, recv in g.exchanges():
            pg = geos[peer]
            # the peer's matching send slice is the one addressed to us
            psend = [s for p, s, _ in pg.exchanges() if p == g.rank][0]
            box[recv] = boxes[peer][psend]


def fixed_order_sum(partial, group=None):
    """Sum a per-rank tensor of partial sums in rank order (deterministic on every rank)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bufs = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(bufs, partial, group=group)
    out = bufs[0].clone()
    for b in bufs[1:]:
        out += b
    return out


class SlabShard:
    """One rank's slab of a full cube on the device (hp_set_create_slab)."""

    def __init__(self, dim: int, bound: int, rank: int, world: int, halo: int):
        from .index_set import build_slab

        self.geo = SlabGeometry(dim, bound, rank, world, halo)
        self.set = build_slab(dim, bound, self.geo.blo, self.geo.bhi)
        self.global_size = self.geo.global_size

    def local_coefficients(self, W, w):
        """The box part (owned planes + halo) of the seeded global vector."""
        c = W.coefficients(w)
        g = self.geo
        return c[g.blo * g.plane:g.bhi * g.plane].copy()

    def interior(self) -> tuple[int, int] | None:
        """Local output planes whose inputs are all owned (the fused kernel reads +-4 planes):
        computable while the halo planes are in flight.  None when there are none."""
        g = self.geo
        lo, hi = g.lo - g.blo, g.hi - g.blo
        ilo = lo + (RADIUS if g.rank > 0 else 0)
        ihi = hi - (RADIUS if g.rank < g.world - 1 else 0)
        return (ilo, ihi) if ihi > ilo else None

    def schedule(self) -> str:
        """"overlap": interior planes while the halo is in flight, then the two boundary ranges;
        "single": exchange, then ONE launch over the owned planes.

        Every plane-range launch of the fused kernel re-reads RADIUS warm-up planes on each side,
        so the overlapped schedule reads owned + 24 planes (interior: owned; each boundary range:
        its 4 planes + 8) against owned + 8 for the single launch, which in turn exposes the
        exchange (2 x RADIUS planes over NVLink, ~1/10 of a plane's HBM time per plane at 900 GB/s
        vs 6.5 TB/s x 0.55).  With few owned planes the re-reads dominate: single launch for
        <= 32 owned planes (4+ ranks on a 128-plane cube), overlap above.
        """
        import os

        forced = os.environ.get("HP_SLAB_SCHEDULE")
        if forced in ("single", "overlap"):
            return forced
        g = self.geo
        return "single" if g.world > 1 and (g.hi - g.lo) <= 32 else "overlap"

    def apply_polynomial(self, appl, ap, x, y, flags: int = 0, overlap: bool = True, exchange=None, dot=None,
                         q: float = 0.0):
        """y[own] = W(X) x on this rank's planes; x, y are box-sized device tensors.

        With `overlap` and the "overlap" schedule, the halo exchange runs on a side stream while
        the interior planes are computed (hp_apply_polynomial_planes), then the boundary planes;
        otherwise exchange, then one launch over the owned planes.  `exchange(geo, x)` replaces
        halo_exchange (tests).  `dot` (a float64 device tensor of 2): the owned rows of x^H y are
        added to it by the fused kernel when the surrogate is in its class; returns whether it was.
        """
        import torch

        exch = exchange or halo_exchange
        g = self.geo
        lo, hi = g.lo - g.blo, g.hi - g.blo
        rng = self.interior() if overlap and g.world > 1 and self.schedule() == "overlap" else None
        if rng is None or not appl.apply_planes_into(ap, x, y, rng[0], rng[0], flags):
            exch(g, x)
            if appl.apply_planes_into(ap, x, y, lo, hi, flags, dot=dot, q=q):  # one launch, owned planes
                return dot is not None
            appl.apply_into(ap, x, y, flags)  # outside the fused class: whole box, square sum apart
            if q != 0.0:
                y.add_(appl.apply_square_sum(x), alpha=q)
            return False
        main = torch.cuda.current_stream()
        side = self.__dict__.setdefault("_side", torch.cuda.Stream())
        side.wait_stream(main)
        with torch.cuda.stream(side):
            exch(g, x)  # NCCL on the side stream
        appl.apply_planes_into(ap, x, y, rng[0], rng[1], flags, dot=dot, q=q)  # reads owned planes only
        main.wait_stream(side)
        if rng[0] > lo:
            appl.apply_planes_into(ap, x, y, lo, rng[0], flags, dot=dot, q=q)
        if hi > rng[1]:
            appl.apply_planes_into(ap, x, y, rng[1], hi, flags, dot=dot, q=q)
        return dot is not None

    def apply_host(self, appl, ap, x_host, y_host, flags: int = 0) -> None:
        """One matvec from host data: x_host is this rank's box of the host vector (owned planes
        and halo planes, `local_coefficients`), so the halo arrives with the host->device copy and
        no device exchange is needed.  One hp_apply_polynomial_streamed call: j1-plane chunks in,
        kernels, chunks out, overlapped.  y_host[own_slice] is valid; halo rows are scratch."""
        appl.apply_host_into(ap, x_host, y_host, flags)


# ---------------------------------------------------------------- sharded time stepping

def dist_sum(partials):
    """Cross-rank sum of this process's partial scalars (a device float64 tensor per local
    shard): all-gather of the per-rank partials, then a rank-ordered sum (deterministic and
    identical on every rank).  One local shard per process in a distributed run."""
    total = partials[0].clone()
    for p in partials[1:]:
        total += p
    return fixed_order_sum(total)


def local_sum(partials):
    """The cross-rank sum when every rank's shard lives in this process (tests)."""
    total = partials[0].clone()
    for p in partials[1:]:
        total += p
    return total


class HostLanczosScalars:
    """The hp_lz_* state machine on the host (the same scaled recurrence as k_red_final /
    k_lz_update_s / k_lz_combine_s), for step-op implementations that keep their vectors off the
    device (the gloo orchestration tests).  Mixed into a class providing ``update`` (host
    coefficients), ``combine`` and ``expm_col``."""

    def lz_new(self, m):
        return {"m": m, "m_eff": m, "broken": False, "alpha": [0.0] * m, "beta": [0.0] * m,
                "scale": [0.0] * (m + 1), "nrm0": 0.0, "col": None}

    def lz_set(self, st, k, what, value, tol):
        v = float(value[0])
        if what == "begin":
            st["nrm0"] = v ** 0.5
            st["scale"][0] = 1.0 / st["nrm0"]
            return
        if st["broken"] and k >= st["m_eff"]:
            return
        if what == "alpha":
            st["alpha"][k] = st["scale"][k] ** 2 * v
        else:
            bk = v ** 0.5
            if bk <= tol:
                st["broken"], st["m_eff"] = True, k + 1
            else:
                st["beta"][k], st["scale"][k + 1] = bk, 1.0 / bk

    def lz_update(self, st, k, w, u, prev, out):
        import torch

        if st["broken"] and k >= st["m_eff"]:
            return [torch.zeros(2, dtype=torch.float64) for _ in w]
        sk = st["scale"][k]
        cp = -st["beta"][k - 1] * st["scale"][k - 1] if k > 0 else 0.0
        return self.update(sk, w, -st["alpha"][k] * sk, u, cp, prev, out)

    def lz_finish(self, st, h):
        me = st["m_eff"]
        st["col"] = self.expm_col(st["alpha"][:me], st["beta"][:me - 1], h)

    def lz_combine(self, st, U, out):
        me = st["m_eff"]
        self.combine(U[:me], np.array([complex(st["col"][k]) * st["scale"][k] * st["nrm0"] for k in range(me)]),
                     out)

    def lz_diag(self, st):
        import torch

        return torch.tensor([st["m_eff"], 0.0, -1.0, 0.0], dtype=torch.float64)


class DeviceStepOps:
    """The per-shard kernels of sharded_propagate on the device (the library's entry points).

    Tests substitute an object with the same methods (e.g. numpy + the oracle on CPU under
    gloo) to check the distributed orchestration on its own."""

    def __init__(self, shards, ys, fh, exchange=None):
        import torch

        from . import _native as nat
        from .fast_apply import get_applier

        self.nat, self.L = nat, nat.lib()
        self.shards, self.fh, self.exchange = shards, fh, exchange
        self.q = float(fh.potential.harmonic_part)
        self.appls = [get_applier(sh.set) for sh in shards]
        self.own = [sh.geo.own_slice for sh in shards]
        self.nloc = [o.stop - o.start for o in self.own]
        self.outs = [torch.zeros_like(y) for y in ys]
        self.ws = [torch.empty(int(self.L.hp_reduce_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
                   for n in self.nloc]

    def approx(self, t):
        return self.fh.approx_at(t, validate=False)

    def new_box(self, like):
        import torch

        return torch.empty_like(like)

    def matvec(self, ap, boxes):
        """A(t) u on the owned planes of every shard (views into the output boxes); `boxes` are
        box-sized vectors (owned planes valid) whose halos the exchange fills.  Returns (w, dots):
        dots[i] = this shard's rows of u^H A u formed inside the fused kernel (the harmonic part q
        folded into the same launch), or None when the surrogate is outside its class."""
        import torch

        nat = self.nat
        ns = len(self.shards)
        dots = [torch.zeros(2, dtype=torch.float64, device="cuda") for _ in range(ns)]
        got = [False] * ns
        if self.exchange is None:
            for i, sh in enumerate(self.shards):
                got[i] = sh.apply_polynomial(self.appls[i], ap, boxes[i], self.outs[i], nat.HP_ADD_OSC, dot=dots[i],
                                             q=self.q)
        else:  # emulated ranks: one exchange over all boxes, then the local matvecs
            self.exchange([sh.geo for sh in self.shards], boxes)
            for i, sh in enumerate(self.shards):
                g = sh.geo
                if self.appls[i].apply_planes_into(ap, boxes[i], self.outs[i], g.lo - g.blo, g.hi - g.blo,
                                                   nat.HP_ADD_OSC, dot=dots[i], q=self.q):
                    got[i] = True
                else:
                    self.appls[i].apply_into(ap, boxes[i], self.outs[i], nat.HP_ADD_OSC)
                    if self.q != 0.0:
                        self.outs[i].add_(self.appls[i].apply_square_sum(boxes[i]), alpha=self.q)
        w = [self.outs[i][self.own[i]] for i in range(ns)]
        return w, (dots if all(got) else None)

    def cdot(self, a, b):
        """per shard: a^H b as a float64 (re, im) tensor (fixed summation order)"""
        import ctypes

        import torch

        vp, out = ctypes.c_void_p, []
        for i in range(len(a)):
            sc = torch.zeros(2, dtype=torch.float64, device="cuda")
            self.nat.check(self.L.hp_cdot(self.nloc[i], vp(a[i].data_ptr()), vp(b[i].data_ptr()),
                                          vp(sc.data_ptr()), vp(self.ws[i].data_ptr()), self.nat.stream_ptr()))
            out.append(sc)
        return out

    def update(self, cw, w, cu, u, cp, prev, out):
        """out = cw w + cu u + cp prev (prev may be None); per shard ||out||^2 as (x, 0)"""
        import ctypes

        import torch

        vp, parts = ctypes.c_void_p, []
        for i in range(len(w)):
            sc = torch.zeros(2, dtype=torch.float64, device="cuda")
            self.nat.check(self.L.hp_lincomb3_nrm2sq(
                self.nloc[i], cw, vp(w[i].data_ptr()), cu, vp(u[i].data_ptr()), cp,
                vp(prev[i].data_ptr()) if prev is not None else None, vp(out[i].data_ptr()), vp(sc.data_ptr()),
                vp(self.ws[i].data_ptr()), self.nat.stream_ptr()))
            parts.append(sc)
        return parts

    def combine(self, U, coef, out):
        """out = sum_k coef_k U_k per shard (elementwise: out may alias U_0)"""
        import ctypes

        mm = len(U)
        c = np.empty(2 * mm)
        c[0::2], c[1::2] = np.real(coef), np.imag(coef)
        for i in range(len(out)):
            ptrs = (ctypes.c_void_p * mm)(*[U[k][i].data_ptr() for k in range(mm)])
            self.nat.check(self.L.hp_lincomb(self.nloc[i], mm, ctypes.cast(ptrs, ctypes.c_void_p),
                                             c.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out[i].data_ptr()),
                                             self.nat.stream_ptr()))

    # -- Lanczos scalars in device memory (hp_lz_*): no host round trip per iteration ---------
    def lz_new(self, m):
        import torch

        st = torch.empty(int(self.L.hp_lz_state_bytes()), dtype=torch.uint8, device="cuda")
        self.nat.check(self.L.hp_lz_init(self._vp(st), int(m), self.nat.stream_ptr()))
        return st

    def _vp(self, t):
        import ctypes

        return ctypes.c_void_p(t.data_ptr())

    def lz_set(self, st, k, what, value, tol):
        code = {"begin": 1, "alpha": 6, "beta": 7}[what]
        self.nat.check(self.L.hp_lz_set(self._vp(st), int(k), code, self._vp(value), float(tol), self.nat.stream_ptr()))

    def lz_update(self, st, k, w, u, prev, out):
        """out = s_k w - alpha_k s_k u - beta_(k-1) s_(k-1) prev per shard (device scalars);
        per-shard partial ||out||^2 as (x, 0)"""
        import torch

        parts = []
        for i in range(len(w)):
            sc = torch.zeros(2, dtype=torch.float64, device="cuda")
            self.nat.check(self.L.hp_lz_update(self.nloc[i], self._vp(w[i]), self._vp(u[i]),
                                               self._vp(prev[i]) if prev is not None else None, self._vp(out[i]),
                                               self._vp(st), int(k), self._vp(sc), self._vp(self.ws[i]),
                                               self.nat.stream_ptr()))
            parts.append(sc)
        return parts

    def lz_finish(self, st, h):
        self.nat.check(self.L.hp_lz_expm(self._vp(st), float(h), self.nat.stream_ptr()))

    def lz_combine(self, st, U, out):
        """out = ||y|| sum_(k < m_eff) col_k s_k U_k per shard (out may alias U_0)"""
        import ctypes

        mm = len(U)
        for i in range(len(out)):
            ptrs = (ctypes.c_void_p * mm)(*[U[k][i].data_ptr() for k in range(mm)])
            self.nat.check(self.L.hp_lz_combine(self.nloc[i], mm, ctypes.cast(ptrs, ctypes.c_void_p), self._vp(st),
                                                self._vp(out[i]), self.nat.stream_ptr()))

    def lz_diag(self, st):
        import torch

        d = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.nat.check(self.L.hp_lz_diag(self._vp(st), self._vp(d), None, None, self.nat.stream_ptr()))
        return d


def sharded_propagate(shards, fh, ys, t0: float, h: float, nsteps: int, m: int, *, reduce=dist_sum,
                      exchange=None, ops=None, breakdown_tol: float = 1e-14):
    """Midpoint Magnus steps (krylov_propagator.py:192-263, lanczos :58-104, expm :173-186) with
    the state split in j1-slabs: SURVEY.md §8(e).

    ``shards`` are this process's SlabShard(s) (one per rank; several only when tests emulate
    the ranks in one process), ``ys`` their box-sized complex128 states (owned planes valid,
    halos are refreshed by each matvec's exchange), ``fh`` the FastHamiltonian of the full cube
    (its surrogate is re-interpolated at every step's midpoint, as the reference does).  Every
    vector operation runs on the owned planes of each shard; Lanczos dot products and norms are
    per-shard partials combined by ``reduce`` (all-gather + rank-ordered sum, on the device), so
    every rank holds identical alpha, beta.

    The basis is kept unnormalised (u_k = v_k / s_k) and box-sized (the matvec reads it in place),
    so a Lanczos iteration is the sharded matvec on u_k -- alpha from its in-kernel rows of
    u^H A u (hp_apply_hamiltonian_planes_dot, the harmonic part folded in), else one dot pass --
    and one fused update + norm pass.  Every scalar (alpha, beta, scales, breakdown, the QL and
    exp column) lives in a device state (hp_lz_*): an iteration is a pure launch + collective
    sequence with no host round trip.  The step ends with one combine pass written over the
    state.  ``ops`` supplies the per-shard kernels (default DeviceStepOps).  Returns ``ys``
    advanced in place; raises RuntimeError on a QL failure (checked once per call).
    """
    ops = ops or DeviceStepOps(shards, ys, fh, exchange)
    ns = len(shards)
    own = [sh.geo.own_slice for sh in shards]

    def total(parts):
        return reduce([p.clone() for p in parts])

    states = []
    for step in range(nsteps):
        t = t0 + step * h
        ap = ops.approx(t + 0.5 * h)
        y = [ys[i][own[i]] for i in range(ns)]
        st = ops.lz_new(m)
        n2 = total(ops.cdot(y, y))
        if step == 0 and float(n2[0]) == 0.0:  # the one host read of the call
            raise ValueError("starting vector must be nonzero")
        ops.lz_set(st, 0, "begin", n2, breakdown_tol)
        UB = [list(ys)]  # u_0 = y itself, s_0 = 1 / ||y||
        U = [y]
        for k in range(m):
            w, dots = ops.matvec(ap, UB[k])
            if dots is None:  # the matvec did not form u_k^H A u_k itself
                dots = ops.cdot(U[k], w)
            ops.lz_set(st, k, "alpha", total(dots), breakdown_tol)
            if k == m - 1:
                break
            nb = [ops.new_box(x) for x in ys]
            nxt = [nb[i][own[i]] for i in range(ns)]
            parts = ops.lz_update(st, k, w, U[k], U[k - 1] if k > 0 else None, nxt)
            ops.lz_set(st, k, "beta", total(parts), breakdown_tol)
            UB.append(nb)
            U.append(nxt)
        ops.lz_finish(st, h)
        ops.lz_combine(st, U, y)  # y = ||y|| sum_k col_k s_k u_k over the effective basis
        states.append(st)
    diags = [ops.lz_diag(st) for st in states]
    if any(float(d[3]) != 0.0 for d in diags):
        raise RuntimeError("tridiagonal QL failed to converge")
    return ys

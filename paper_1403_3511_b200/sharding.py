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

    def apply_polynomial(self, appl, ap, x, y, flags: int = 0, overlap: bool = True, exchange=None):
        """y[own] = W(X) x on this rank's planes; x, y are box-sized device tensors.

        With `overlap`, the halo exchange runs on a side stream while the interior planes are
        computed (hp_apply_polynomial_planes), then the boundary planes; otherwise exchange,
        then one matvec over the box.  `exchange(geo, x)` replaces halo_exchange (tests).
        """
        import torch

        exch = exchange or halo_exchange
        rng = self.interior() if overlap and self.geo.world > 1 else None
        if rng is None or not appl.apply_planes_into(ap, x, y, rng[0], rng[0], flags):
            exch(self.geo, x)
            appl.apply_into(ap, x, y, flags)
            return
        g = self.geo
        lo, hi = g.lo - g.blo, g.hi - g.blo
        main = torch.cuda.current_stream()
        side = self.__dict__.setdefault("_side", torch.cuda.Stream())
        side.wait_stream(main)
        with torch.cuda.stream(side):
            exch(g, x)  # NCCL on the side stream
        appl.apply_planes_into(ap, x, y, rng[0], rng[1], flags)  # reads owned planes only
        main.wait_stream(side)
        if rng[0] > lo:
            appl.apply_planes_into(ap, x, y, lo, rng[0], flags)
        if hi > rng[1]:
            appl.apply_planes_into(ap, x, y, rng[1], hi, flags)

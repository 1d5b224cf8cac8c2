"""Multi-rank slab decomposition on CPU with the gloo backend, world_size 2 and 3.

The host-side logic -- plane partition, box/halo geometry, the neighbour
send/recv of halo planes, fixed-order reductions -- is exactly what the
NCCL path runs; here each rank's local matvec is the oracle on its slab box,
and the assembled owned planes must equal the single-process result bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1403_3511_b200.sharding import (HostLanczosScalars, SlabGeometry, fixed_order_sum, halo_exchange,
                                          partition)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import hprop_oracle as O
        from paper_1403_3511_b200 import workloads as W

        w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
        ap = O.interpolate(w.evaluator, w.dim, W.HALFWIDTH, w.degree, 0.3)
        c = W.coefficients(w)
        geo = SlabGeometry(w.dim, w.bound, rank, world, halo=w.degree)
        box = torch.zeros(geo.box_size, dtype=torch.complex128)
        own = geo.own_slice
        box[own] = torch.from_numpy(c[geo.lo * geo.plane:geo.hi * geo.plane])
        halo_exchange(geo, box)
        # the exchanged halo equals the global vector
        assert np.array_equal(box.numpy(), c[geo.blo * geo.plane:geo.bhi * geo.plane])
        appl = O.applier_for_slab(w.dim, w.bound, geo.blo, geo.bhi)
        y = appl.polynomial(ap.degrees, ap.coeffs, W.HALFWIDTH, box.numpy())
        part = torch.from_numpy(y[own].copy())
        parts = [None] * world
        dist.all_gather_object(parts, (geo.lo, geo.hi, part.numpy()))
        s = fixed_order_sum(torch.tensor([float(rank) + 0.1, 1.0], dtype=torch.float64))
        if rank == 0:
            out_q.put((parts, s.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_matvec_gloo(world):
    from oracle import hprop_oracle as O
    from paper_1403_3511_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, s = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
    ap = O.interpolate(w.evaluator, w.dim, W.HALFWIDTH, w.degree, 0.3)
    full = O.applier_for_full(w.dim, w.bound).polynomial(ap.degrees, ap.coeffs, W.HALFWIDTH, W.coefficients(w))
    plane = (w.bound + 1) ** 3
    got = np.zeros_like(full)
    for lo, hi, part in parts:
        got[lo * plane:hi * plane] = part
    assert np.array_equal(got, full)
    assert np.allclose(s, [sum(r + 0.1 for r in range(world)), world])


def test_partition_and_geometry():
    for planes in (1, 7, 128):
        for world in (1, 2, 3, 8):
            if world > planes:
                continue
            spans = [partition(planes, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == planes
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    g = SlabGeometry(4, 127, 1, 8, halo=4)
    assert (g.lo, g.hi, g.blo, g.bhi) == (16, 32, 12, 36)
    ex = g.exchanges()
    assert [e[0] for e in ex] == [0, 2]
    # send my first 4 owned planes down, receive 4 halo planes below
    assert ex[0][1] == slice(4 * g.plane, 8 * g.plane) and ex[0][2] == slice(0, 4 * g.plane)
    assert ex[1][1] == slice(16 * g.plane, 20 * g.plane) and ex[1][2] == slice(20 * g.plane, 24 * g.plane)


class _CpuStepOps(HostLanczosScalars):
    """sharding.sharded_propagate's per-shard kernels on CPU: the oracle's slab Hamiltonian after a
    gloo halo exchange, numpy dot / update / combine (one shard per process); the Lanczos scalars
    follow the device state machine's host restatement."""

    def __init__(self, geo, w):
        from oracle import hprop_oracle as O
        from paper_1403_3511_b200 import workloads as W

        self.O, self.W, self.geo, self.w = O, W, geo, w
        self.appl = O.applier_for_slab(w.dim, w.bound, geo.blo, geo.bhi)

    def approx(self, t):
        return self.O.interpolate(self.w.evaluator, self.w.dim, self.W.HALFWIDTH, self.w.degree, t)

    def new_box(self, like):
        return torch.zeros_like(like)

    def matvec(self, ap, boxes):
        halo_exchange(self.geo, boxes[0])
        y = self.appl.hamiltonian(ap.degrees, ap.coeffs, self.W.HALFWIDTH, boxes[0].numpy())
        return [torch.from_numpy(y[self.geo.own_slice].copy())], None

    def cdot(self, a, b):
        d = np.vdot(a[0].numpy(), b[0].numpy())
        return [torch.tensor([d.real, d.imag], dtype=torch.float64)]

    def update(self, cw, w, cu, u, cp, prev, out):
        r = cw * w[0].numpy() + cu * u[0].numpy()
        if prev is not None:
            r = r + cp * prev[0].numpy()
        out[0].copy_(torch.from_numpy(r))
        return [torch.tensor([np.vdot(r, r).real, 0.0], dtype=torch.float64)]

    def combine(self, U, coef, out):
        acc = sum(c * u[0].numpy() for c, u in zip(coef, U))
        out[0].copy_(torch.from_numpy(acc))

    def expm_col(self, alpha, beta, h):
        return self.O.expm_tridiag_column(np.array(alpha), np.array(beta), h)


def _prop_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1403_3511_b200 import workloads as W
        from paper_1403_3511_b200.sharding import sharded_propagate

        w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
        c = W.coefficients(w)
        geo = SlabGeometry(w.dim, w.bound, rank, world, halo=w.degree)

        class _Shard:
            pass

        sh = _Shard()
        sh.geo = geo
        y = torch.zeros(geo.box_size, dtype=torch.complex128)
        y[geo.own_slice] = torch.from_numpy(c[geo.lo * geo.plane:geo.hi * geo.plane])
        sharded_propagate([sh], None, [y], 0.0, w.dt, 2, 7, ops=_CpuStepOps(geo, w))
        parts = [None] * world
        dist.all_gather_object(parts, (geo.lo, geo.hi, y[geo.own_slice].numpy().copy()))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_propagation_gloo(world):
    """Slab-sharded Magnus steps (sharding.sharded_propagate) over gloo, world 2 and 3: the
    distributed Lanczos (owned-plane updates, all-gather + rank-ordered reductions, halo
    exchange per matvec) with the oracle's slab Hamiltonian equals the oracle's propagation of
    the whole cube (2 midpoint steps, m = 7) within 1e-12."""
    from oracle import hprop_oracle as O
    from paper_1403_3511_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prop_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.CONFIGS["cfg4"].scaled(11, "cfg4x")
    c = W.coefficients(w)
    ham_at = O.hamiltonian_at(O.applier_for_full(w.dim, w.bound), w.evaluator, w.dim, W.HALFWIDTH, w.degree)
    want = O.propagate("midpoint", ham_at, c, 0.0, 2 * w.dt, 2, 7)
    plane = (w.bound + 1) ** 3
    got = np.zeros_like(want)
    for lo, hi, part in parts:
        got[lo * plane:hi * plane] = part
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12

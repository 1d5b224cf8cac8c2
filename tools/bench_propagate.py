"""Time the propagation runs of BASELINE.json on the device (and the oracle on a sample of steps).

    python tools/bench_propagate.py cfg1 [--steps N] [--cpu-steps M]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_propagate.py cfg4   (slab-sharded)

Prints one JSON line: device ms/step (CUDA events around whole steps, state
resident on the device, term lists re-interpolated on the host each step as
the reference does), the CPU oracle's s/step on the same inputs, and the
relative L2 difference of the states after the compared steps.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def sharded_main(args, rank, world, local_rank):
    """torchrun --nproc-per-node N tools/bench_propagate.py cfg4: slab-sharded Magnus steps
    (sharding.sharded_propagate, halos and reductions over NCCL), device time max over ranks."""
    import os

    import torch
    import torch.distributed as dist

    import paper_1403_3511_b200 as hp
    from paper_1403_3511_b200 import workloads as W
    from paper_1403_3511_b200.sharding import SlabShard, sharded_propagate

    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    w = W.CONFIGS[args.workload]
    if w.kind != "full" or w.batch != 1:
        raise SystemExit("sharded propagation: full-cube single-vector workloads (cfg4)")
    nsteps = args.steps or w.nsteps
    shard = SlabShard(w.dim, w.bound, rank, world, halo=w.degree)
    g = shard.geo
    y = torch.zeros(g.box_size, dtype=torch.complex128, device="cuda")
    y[g.own_slice] = torch.from_numpy(shard.local_coefficients(W, w)[g.own_slice]).cuda()
    fh = hp.FastHamiltonian(hp.build_full(w.dim, w.bound), hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH),
                            w.degree)
    sharded_propagate([shard], fh, [y.clone()], 0.0, w.dt, 1, args.m)  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sharded_propagate([shard], fh, [y], 0.0, w.dt, nsteps, args.m)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / nsteps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nrm = torch.linalg.vector_norm(y[g.own_slice]).square().reshape(1)
    from paper_1403_3511_b200.sharding import fixed_order_sum

    nrm = float(fixed_order_sum(nrm)[0]) ** 0.5
    if rank == 0:
        n = g.global_size
        out = {"workload": w.name, "n": n, "steps": nsteps, "dt": w.dt, "m": args.m, "n_gpus": world,
               "parallelism": f"slab-j1 x{world}", "device_ms_per_step": round(float(t), 4),
               "algorithmic_bytes_per_step": (112 * args.m - 48) * n, "state_norm": nrm}
        out["achieved_GBs"] = round(out["algorithmic_bytes_per_step"] / (float(t) * 1e-3) / 1e9, 1)
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    import os

    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or "--shard" in sys.argv:
        ap = argparse.ArgumentParser()
        ap.add_argument("workload")
        ap.add_argument("--steps", type=int, default=None)
        ap.add_argument("--cpu-steps", type=int, default=0)
        ap.add_argument("--m", type=int, default=7)
        ap.add_argument("--shard", action="store_true", help="sharded code path even at one rank (torchrun)")
        args = ap.parse_args()
        sharded_main(args, int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", 0)))
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--scheme", default="midpoint", choices=["midpoint", "gl2"])
    args = ap.parse_args()
    import torch

    import paper_1403_3511_b200 as hp
    from oracle import hprop_oracle as O
    from paper_1403_3511_b200 import workloads as W

    w = W.CONFIGS[args.workload]
    nsteps = args.steps or w.nsteps
    s = hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)
    c = W.coefficients(w, None if w.kind == "full" else s.indices)
    fh = hp.FastHamiltonian(s, hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH), w.degree)
    scheme = hp.MagnusScheme.from_name(args.scheme)
    y = torch.from_numpy(c).cuda()
    # warm-up: a few steps (the first ones grow the cached workspace and term-array caches;
    # cfg1 after one warm-up step: 185 us/step for the next 100, 127 after five)
    fh.propagate(scheme, y, 0.0, w.dt, 5, args.m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from bench import ClockSampler

    # 20 ms sampling: a tighter poll competes with the stepping loop's host work (cfg1 steps
    # are ~0.13 ms of which most is Python)
    with ClockSampler(torch.cuda.current_device(), interval=0.02) as clk:
        t0 = time.perf_counter()
        e0.record()
        yT = fh.propagate(scheme, y, 0.0, w.dt, nsteps, args.m)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    dev_ms = e0.elapsed_time(e1) / nsteps
    # gl2: every Krylov matvec is the commutator combination of four operator applications, so
    # the midpoint byte count does not apply; the line reports time only
    out = {"workload": w.name, "scheme": args.scheme, "n": s.size, "steps": nsteps, "dt": w.dt, "m": args.m,
           "device_ms_per_step": round(dev_ms, 4), "wall_ms_per_step": round(wall * 1e3 / nsteps, 4),
           "algorithmic_bytes_per_step": (112 * args.m - 48) * s.size if args.scheme == "midpoint" else None,
           "clocks": clk.summary()}
    if out["algorithmic_bytes_per_step"]:
        out["achieved_GBs"] = round(out["algorithmic_bytes_per_step"] / (dev_ms * 1e-3) / 1e9, 1)
    # CPU oracle on the first cpu_steps steps, same inputs
    k = min(args.cpu_steps, nsteps)
    if k > 0 and s.size <= 40_000_000:
        if w.kind == "full":
            appl = O.applier_for_full(w.dim, w.bound)
        else:
            appl = O.applier_for_set(np.asarray(s.indices))
        ham_at = O.hamiltonian_at(appl, w.evaluator, w.dim, W.HALFWIDTH, w.degree)
        t0 = time.perf_counter()
        yc = O.propagate(args.scheme, ham_at, c, 0.0, k * w.dt, k, args.m)
        cpu = (time.perf_counter() - t0) / k
        yg = fh.propagate(scheme, torch.from_numpy(c).cuda(), 0.0, w.dt, k, args.m).cpu().numpy()
        out["cpu_oracle_s_per_step"] = round(cpu, 4)
        out["cpu_steps_compared"] = k
        out["rel_l2_vs_oracle"] = float(np.linalg.norm(yg - yc) / np.linalg.norm(yc))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

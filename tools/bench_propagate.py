"""Time the propagation runs of BASELINE.json on the device (and the oracle on a sample of steps).

    python tools/bench_propagate.py cfg1 [--steps N] [--cpu-steps M]

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--m", type=int, default=7)
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
    scheme = hp.MagnusScheme.from_name("midpoint")
    y = torch.from_numpy(c).cuda()
    # warm-up: one step
    fh.propagate(scheme, y, 0.0, w.dt, 1, args.m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from bench import ClockSampler

    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        e0.record()
        yT = fh.propagate(scheme, y, 0.0, w.dt, nsteps, args.m)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    dev_ms = e0.elapsed_time(e1) / nsteps
    out = {"workload": w.name, "n": s.size, "steps": nsteps, "dt": w.dt, "m": args.m,
           "device_ms_per_step": round(dev_ms, 4), "wall_ms_per_step": round(wall * 1e3 / nsteps, 4),
           "algorithmic_bytes_per_step": (112 * args.m - 48) * s.size, "clocks": clk.summary()}
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
        yc = O.propagate("midpoint", ham_at, c, 0.0, k * w.dt, k, args.m)
        cpu = (time.perf_counter() - t0) / k
        yg = fh.propagate(scheme, torch.from_numpy(c).cuda(), 0.0, w.dt, k, args.m).cpu().numpy()
        out["cpu_oracle_s_per_step"] = round(cpu, 4)
        out["cpu_steps_compared"] = k
        out["rel_l2_vs_oracle"] = float(np.linalg.norm(yg - yc) / np.linalg.norm(yc))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

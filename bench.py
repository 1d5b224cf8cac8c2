"""Benchmark: Galerkin matvec throughput (basis coeffs/s) and % of HBM roofline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

A step is one matvec y = W(X_1..X_N) c of the workload (one batch of
seeded synthetic input).  Default workload: cfg4 of BASELINE.json (N=4 full
cube, K+1 = 128, 2.68e8 complex128 coefficients, 4.29 GB per vector -- far
larger than L2, so no flush is needed between steps); it is the largest
configuration whose matvec is HBM-bound and the one sharded across GPUs in
slabs (§8(e)).  `--workload cfg1..cfg5` measures the others.

Output: ONE JSON line on rank 0 (driver contract), with `roofline`,
`cpu_baseline` (the oracle port timed on this host), `e2e` (host buffers in,
result back to host, through the C-ABI), `gpu_launches` and `clocks`.
`--impl reference` times the reference algorithm (the oracle port of
hprop's numpy path; the reference package itself cannot travel to the GPU
box) on this host's cores for the same workload and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks
    line): NVML polled every ~2 ms from a thread (a 20-step cfg4 region lasts ~50 ms, shorter
    than nvidia-smi's 100 ms loop); nvidia-smi -lms 100 if NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int, interval: float = 0.002):
        self.index = index
        self.interval = interval
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []
        self.stop = threading.Event()
        self.nvml = None

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        # the CUDA device's NVML handle by PCI address (CUDA_VISIBLE_DEVICES may renumber)
        pr = torch.cuda.get_device_properties(self.index)
        bus = f"{int(pr.pci_domain_id):08x}:{int(pr.pci_bus_id):02x}:{int(pr.pci_device_id):02x}.0"
        return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self._sample()  # sub-millisecond regions (cfg1, cfg2) still get one sample each side
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _sample(self):
        nv, h = self.nvml
        try:
            self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                 float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                                 int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
        except Exception:
            pass

    def _poll(self):
        while not self.stop.wait(self.interval):
            self._sample()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=2)
            self._sample()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            mx.append(m_)
            reasons.update(nm for nm, bit in self.BITS.items() if r_ & bit)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------- workload setup

def build_set(hp, w):
    return hp.build_full(w.dim, w.bound) if w.kind == "full" else hp.build_hyperbolic(w.dim, w.bound)


def algorithmic_bytes(w, n, batch=None):
    """32 B per coefficient per vector per matvec: c read once, y written once."""
    return 32.0 * n * (w.batch if batch is None else batch)


# ---------------------------------------------------------------- CPU baseline (oracle port)

def _cpu_sample(wname: str, sample: dict):
    """One bounded CPU sample of the workload with the oracle (hprop's numpy algorithm)."""
    from oracle import hprop_oracle as O
    from paper_1403_3511_b200 import workloads as W

    w = W.CONFIGS[wname]
    ap = w.approx(0.0, validate=False)
    if w.kind == "full" and sample.get("planes"):
        lo, hi = sample["planes"]
        appl = O.applier_for_slab(w.dim, w.bound, lo, hi)
        plane = (w.bound + 1) ** (w.dim - 1)
        rng = np.random.default_rng([w.seed, 0, lo])
        v = rng.standard_normal(appl.n) + 1j * rng.standard_normal(appl.n)
        nvec = 1
    elif w.kind == "full":
        appl = O.applier_for_full(w.dim, w.bound)
        v = W.coefficients(w)
        nvec = 1
    else:
        b = sample.get("bound", w.bound)
        ws = w.scaled(b)
        idx = O.hyperbolic_indices(ws.dim, ws.bound)
        appl = O.applier_for_set(idx)
        rng = np.random.default_rng([w.seed, 0])
        v = rng.standard_normal(appl.n) + 1j * rng.standard_normal(appl.n)
        nvec = 1
    return appl, ap, v, nvec


def _cpu_worker(args):
    wname, sample, reps = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    appl, ap, v, nvec = _cpu_sample(wname, sample)
    times = []
    appl.polynomial(ap.degrees, ap.coeffs, ap.halfwidth, v)  # warm-up
    for _ in range(reps):
        t0 = time.perf_counter()
        appl.polynomial(ap.degrees, ap.coeffs, ap.halfwidth, v)
        times.append(time.perf_counter() - t0)
    return appl.n * nvec, times


def cpu_plan(wname: str, workers: int, planes: int = 12):
    """Bounded sample per worker: cfg4 -> a `planes`-plane j1 slab of the real cube."""
    if wname == "cfg4":
        samples = [{"planes": (min(8 * i, 128 - planes), min(8 * i, 128 - planes) + planes)} for i in range(workers)]
        desc = (f"hprop numpy algorithm (oracle port) on {planes}-plane j1 slabs of the cfg4 cube "
                f"({planes * 2.097152:.1f}M coefficients each, one slab per worker process); "
                "rate = slab coefficients / time (a whole-cube run has the same per-coefficient work)")
    elif wname == "cfg3":
        samples = [{"bound": 1023}] * workers
        desc = "oracle port on build_hyperbolic(6,1023) (611,556 coeffs, same W) -- scaled sample of cfg3"
    elif wname == "cfg5":
        samples = [{"bound": 255}] * workers
        desc = "oracle port on build_hyperbolic(8,255) (239,420 coeffs, one vector, same W) -- scaled sample of cfg5"
    else:
        samples = [{}] * workers
        desc = f"oracle port on the full {wname} set"
    return samples, desc


def run_cpu(wname: str, workers: int, reps: int, planes: int = 12):
    samples, desc = cpu_plan(wname, workers, planes)
    t0 = time.perf_counter()
    if workers == 1:
        res = [_cpu_worker((wname, samples[0], reps))]
    else:
        import multiprocessing as mp

        with mp.get_context("spawn").Pool(workers) as pool:
            res = pool.map(_cpu_worker, [(wname, s, reps) for s in samples])
    wall = time.perf_counter() - t0
    coeffs = sum(r[0] for r in res)
    per_rep = [max(r[1][k] for r in res) for k in range(reps)]
    med = float(np.median(per_rep))
    return {"value": coeffs / med, "unit": "coeffs/s", "cores": workers, "kind": "port", "sample": desc,
            "seconds_per_rep": med, "reps": reps, "wall_s": round(wall, 1)}


def cpu_workers_for(wname: str) -> int:
    ncpu = os.cpu_count() or 1
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    per = {"cfg4": 9 << 30, "cfg3": 2 << 30, "cfg5": 2 << 30}.get(wname, 1 << 30)
    return max(1, min(ncpu, int(avail * 0.6 // per)))


# ---------------------------------------------------------------- reference arm

def reference_arm(args, rank):
    if rank != 0:
        return
    workers = cpu_workers_for(args.workload)
    reps = max(1, args.steps)
    # each step is a bounded sample (a 4-plane slab, ~8.4M coefficients per worker, a few
    # seconds) so that --steps K --warmup W finishes within a few minutes
    base = run_cpu(args.workload, workers, reps, planes=4)
    line = {"impl": "reference", "metric": "Galerkin matvec throughput", "value": base["value"],
            "unit": "coeffs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": base["seconds_per_rep"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": {"workload": args.workload, "threads": workers},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": "coeffs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def gpu_arm(args, rank, world, local_rank):
    import torch

    import paper_1403_3511_b200 as hp
    from paper_1403_3511_b200 import _native as nat
    from paper_1403_3511_b200 import workloads as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = W.CONFIGS[args.workload]
    peaks, peak_kind = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    if args.mode == "step":
        step_mode(args, w, rank, world, local_rank, hbm, peak_kind)
        return

    sharding = None
    emu = None  # --shard-geometry R/P: rank R's slab of a P-rank run, measured alone on this GPU
    if args.shard_geometry:
        emu = tuple(int(x) for x in args.shard_geometry.split("/"))
    if (world > 1 or args.force_shard or emu) and w.kind == "full" and w.batch == 1:
        from paper_1403_3511_b200 import sharding as SH

        sharding = SH.SlabShard(w.dim, w.bound, *(emu or (rank, world)), halo=w.degree)
        s = sharding.set
    else:
        s = build_set(hp, w)
    n_local = s.size
    appl = hp.get_applier(s)
    ap = w.approx(0.3 if w.name == "cfg4" else 0.0, validate=False)

    # inputs: the seeded workload vector (rank-local part), resident in HBM
    # batched workloads (cfg5) partition the batch by vector across ranks: rank r
    # takes vectors [r B / P, (r + 1) B / P); single-vector reduced sets and small cubes are
    # replicas (every rank the whole workload)
    part = world > 1 and sharding is None and w.batch > 1
    if sharding is not None:
        c_host = sharding.local_coefficients(W, w)
    elif part:  # this rank's vectors only (the other ranks' draws are discarded)
        b0, b1 = rank * w.batch // world, (rank + 1) * w.batch // world
        c_host = W.coefficients_rows(w, s.indices, b0, b1)
    else:
        c_host = W.coefficients(w, None if w.kind == "full" else s.indices)
    x = torch.from_numpy(c_host).to(dev)
    y = torch.empty_like(x)
    batch = c_host.shape[0] if part else w.batch
    nvec_local = n_local * batch

    def step_dev():
        if sharding is not None:
            # emulated geometry: no peers, the seeded halo planes stand in for the exchanged ones
            sharding.apply_polynomial(appl, ap, x, y, exchange=(lambda g, b: None) if emu else None)
        else:
            appl.apply_into(ap, x, y)

    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # working sets that fit in L2 (cfg1, cfg2): every timed step is bracketed by its own events
    # and L2 is flushed between steps (a 256 MB write outside the brackets), so no step reads
    # what the previous one left in L2; larger working sets stream through HBM anyway
    flush_l2 = algorithmic_bytes(w, n_local, batch) < 126e6  # in + out bytes vs the 126 MB L2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None
    launches0 = nat.lib().hp_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        if flush is None:
            ev0.record()
            for _ in range(args.steps):
                step_dev()
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.fill_(1)
                a.record()
                step_dev()
                b.record()
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
    launches = nat.lib().hp_launch_count() - launches0
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t)
    ms_step = ms_max / args.steps
    if emu:
        total_coeffs = (sharding.geo.hi - sharding.geo.lo) * sharding.geo.plane  # this rank's planes
    elif sharding is not None:
        total_coeffs = sharding.global_size
    elif part:
        total_coeffs = n_local * w.batch  # all ranks' vectors
    else:
        total_coeffs = n_local * batch * world  # replicas: every rank did the whole workload
    value = total_coeffs / (ms_step * 1e-3)

    # roofline of the matvec per GPU: algorithmic bytes of ONE GPU's share of the step / the
    # step time (max over ranks).  32 B per coefficient per vector; a slab rank counts only its
    # owned planes (it writes only those), a batch rank its own vectors, a replica the whole set
    alg_bytes = 32.0 * total_coeffs / world
    achieved = alg_bytes / (ms_step * 1e-3) / 1e9
    traffic, traffic_source = profiled_traffic(args.workload), "committed ncu capture (profiles/traffic.json)"
    live_flops = None
    if rank == 0 and world == 1 and not args.no_traffic:
        live = measured_traffic(args.workload)
        if live:
            traffic, traffic_source = live[0], "ncu child process of this run, one matvec (after the timed region)"
            live_flops = live[1]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic, "traffic_source": traffic_source,
                "peak_kind": peak_kind, "algorithmic_bytes_per_launch": alg_bytes,
                "basis": "one full matvec (all its kernels) per step; 32 B/coefficient; per GPU, max-over-ranks time"}

    # e2e: pinned host buffers in, result back to host, timed on the device
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(c_host).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        e_steps = max(1, min(args.steps, args.e2e_steps))

        def step_e2e():
            if sharding is None:
                # one public call on host buffers: the library streams j1-plane chunks in and the
                # result out, overlapped with the kernels (hp_apply_polynomial_streamed)
                appl.apply_host_into(ap, xh, yh)
            else:
                # this rank's box (owned + halo planes) of the host vector, streamed the same way:
                # the halo comes with the host copy, so no device exchange (SlabShard.apply_host)
                sharding.apply_host(appl, ap, xh, yh)

        step_e2e()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(e_steps):
            step_e2e()
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / e_steps
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t)
        hb = torch.tensor([xh.numel() * xh.element_size(), yh.numel() * yh.element_size()], device=dev,
                          dtype=torch.float64)
        if world > 1:  # every rank's copies (slab boxes, batch parts or replicas)
            torch.distributed.all_reduce(hb)
        e2e = {"value": total_coeffs / (ems * 1e-3), "unit": "coeffs/s",
               "h2d_bytes_per_step": int(hb[0]), "d2h_bytes_per_step": int(hb[1]), "ms_per_step": round(ems, 3),
               "steps": e_steps,
               "path": ("pinned host -> HBM -> pinned host inside hp_apply_polynomial_streamed (C ABI; " +
                        ("j1-plane chunks, copies overlapped with the kernels)" if w.kind == "full" else
                         "groups of batch vectors, copies overlapped with the kernels)" if batch > 1 else
                         "whole-vector copies around the matvec)") if sharding is None else
                        "each rank: its slab box (owned + halo planes) of the pinned host vector -> HBM -> "
                        "pinned host inside hp_apply_polynomial_streamed (C ABI; j1-plane chunks, copies "
                        "overlapped with the kernels; the halo arrives with the host copy, so this e2e figure "
                        "excludes the NCCL halo exchange of the device-resident path)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = run_cpu(args.workload, 1, args.cpu_reps)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    # the named propagation run of the workload (cfg4: 50 midpoint steps at dt = 0.005), timed in
    # the same process after the matvec buffers are released
    prop = None
    if w.nsteps > 0 and not args.no_prop and not emu:
        del x, y
        if not args.no_e2e:
            del xh, yh
        torch.cuda.empty_cache()
        prop = propagation_leg(args, w, rank, world, local_rank, hbm, peak_kind,
                               sharding is not None and torch.distributed.is_initialized())

    if rank == 0:
        line = {"metric": "Galerkin matvec throughput", "value": value, "unit": "coeffs/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True,
                "scaling": "strong" if sharding is not None or part or world == 1 else "weak",
                "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, SURVEY.md §8(d))",
                "config": {"workload": w.name, "set": f"{w.kind} N={w.dim} bound={w.bound}", "n": sharding.global_size if sharding is not None else n_local,
                           "batch": w.batch, "nterms": int(ap.nterms), "halfwidth": W.HALFWIDTH,
                           "l2": "L2 flushed between steps (256 MB write outside the per-step events)" if flush_l2
                           else "inputs larger than L2 (no flush)",
                           "parallelism": (f"slab-j1 rank {emu[0]} of {emu[1]} (emulated on one GPU: exchange "
                                           f"skipped, {sharding.schedule()} schedule; value = that rank's planes/s)")
                           if emu else f"slab-j1 x{world}" if sharding is not None else
                           ("single" if world == 1 else f"batch/{world}" if part else f"replicas x{world}")},
                "roofline": roofline, "fp64": fp64_utilisation(w.name, ms_step, live_flops) if not emu and world == 1 else None,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "specialised_level_kernels": int(nat.lib().hp_level_jit_kernels()),
                "clocks": clk.summary(), "propagation": prop}
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- propagation (time steps)

def step_bytes(m: int, n: int) -> float:
    """Algorithmic bytes of one midpoint Magnus step with m Krylov vectors: (112 m - 48) B per
    coefficient: m matvecs at 32 B, m - 1 Lanczos updates at 64 B (read w, v_k,
    v_(k-1), write v_(k+1)) and the final combine reading m vectors and writing one."""
    return (112.0 * m - 48.0) * n


def _cpu_step_sample(wname: str, m: int):
    """The oracle's midpoint step on a bounded sample of the workload (same potential, same
    per-coefficient work): cfg4 -> the K+1 = 32 cube (1.05M coefficients), cfg3 -> prod <= 1024
    (611,556), cfg1 -> the full set."""
    from oracle import hprop_oracle as O
    from paper_1403_3511_b200 import workloads as W

    w = W.CONFIGS[wname]
    ws = {"cfg4": w.scaled(31), "cfg3": w.scaled(1023)}.get(wname, w)
    if ws.kind == "full":
        appl = O.applier_for_full(ws.dim, ws.bound)
        c = W.coefficients(ws)
    else:
        idx = O.hyperbolic_indices(ws.dim, ws.bound)
        appl = O.applier_for_set(idx)
        c = W.coefficients(ws, idx)
    ham_at = O.hamiltonian_at(appl, ws.evaluator, ws.dim, W.HALFWIDTH, ws.degree)
    O.propagate("midpoint", ham_at, c, 0.0, ws.dt, 1, m)  # warm-up (surrogate caches)
    k = 3 if ws.size() < 2_000_000 else 1
    t0 = time.perf_counter()
    O.propagate("midpoint", ham_at, c, 0.0, k * ws.dt, k, m)
    sec = (time.perf_counter() - t0) / k
    desc = (f"oracle port (hprop's numpy Lanczos/Magnus path) on {'the full set' if ws is w else ws.name}, "
            f"n = {ws.size():,}, {k} midpoint step(s), m = {m}, 1 core")
    return {"value": ws.size() / sec, "unit": "coeff-steps/s", "cores": 1, "kind": "port", "sample": desc,
            "seconds_per_step": sec}


def propagation_leg(args, w, rank, world, local_rank, hbm, peak_kind, sharded):
    """Time `args.prop_steps` midpoint Magnus steps (m = 7) of the workload's named run through the
    public API with the state resident in HBM (FastHamiltonian.propagate at one GPU; the
    slab-sharded sharded_propagate over NCCL when the matvec ran sharded), plus an e2e run of
    propagate_magnus from a pinned host state back to a host state."""
    import torch

    import paper_1403_3511_b200 as hp
    from paper_1403_3511_b200 import _native as nat
    from paper_1403_3511_b200 import workloads as W

    dev = torch.device("cuda", local_rank)
    m = 7
    nsteps = min(args.prop_steps, w.nsteps)
    spec = hp.custom_potential(w.evaluator, w.dim, W.HALFWIDTH)
    scheme = hp.MagnusScheme.from_name("midpoint")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sharded:
        from paper_1403_3511_b200.sharding import SlabShard, sharded_propagate

        shard = SlabShard(w.dim, w.bound, rank, world, halo=w.degree)
        g = shard.geo
        yb = torch.zeros(g.box_size, dtype=torch.complex128, device=dev)
        yb[g.own_slice] = torch.from_numpy(shard.local_coefficients(W, w)[g.own_slice]).to(dev)
        fh = hp.FastHamiltonian(hp.build_full(w.dim, w.bound), spec, w.degree)
        sharded_propagate([shard], fh, [yb.clone()], 0.0, w.dt, 2, m)  # warm-up
        run = lambda k: sharded_propagate([shard], fh, [yb], 0.0, w.dt, k, m)  # noqa: E731
        n = g.global_size
    else:
        s = build_set(hp, w)
        c = W.coefficients(w, None if w.kind == "full" else s.indices)
        fh = hp.FastHamiltonian(s, spec, w.degree)
        yd = torch.from_numpy(c).to(dev)
        fh.propagate(scheme, yd.clone(), 0.0, w.dt, 3, m)  # warm-up: workspace and term caches
        run = lambda k: fh.propagate(scheme, yd, 0.0, w.dt, k, m)  # noqa: E731
        n = s.size
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = nat.lib().hp_launch_count()
    with ClockSampler(local_rank, interval=0.01) as clk:
        ev0.record()
        run(nsteps)
        ev1.record()
        torch.cuda.synchronize()
    launches = nat.lib().hp_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / nsteps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t)
    alg = step_bytes(m, n) / world
    achieved = alg / (ms * 1e-3) / 1e9
    out = {"workload": w.name, "scheme": "midpoint", "m": m, "dt": w.dt, "n": n, "steps": nsteps,
           "named_run_steps": w.nsteps, "ms_per_step": round(ms, 4), "value": n / (ms * 1e-3),
           "unit": "coeff-steps/s",
           "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(achieved / hbm, 4), "peak_kind": peak_kind,
                        "algorithmic_bytes_per_step": alg,
                        "basis": f"(112 m - 48) B per coefficient-step at m = {m} (SURVEY §8(d)), per GPU"},
           "gpu_launches": int(launches), "specialised_level_kernels": int(nat.lib().hp_level_jit_kernels()),
           "clocks": clk.summary(),
           "parallelism": f"slab-j1 x{world}" if sharded else ("single" if world == 1 else f"replicas x{world}")}
    if world == 1 and not sharded and not args.no_e2e:
        # e2e: propagate_magnus on a pinned host state (a CPU torch tensor in, a CPU tensor out):
        # one copy in, the steps on the device, one copy out
        ke = max(1, min(nsteps, 5))
        ch = torch.from_numpy(c).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        yh = hp.propagate_magnus(scheme, fh.matvec_at, ch, 0.0, ke * w.dt, ke, m)
        e1.record()
        torch.cuda.synchronize()
        assert not yh.is_cuda
        ems = e0.elapsed_time(e1) / ke
        out["e2e"] = {"value": n / (ems * 1e-3), "unit": "coeff-steps/s", "ms_per_step": round(ems, 3),
                      "steps": ke, "h2d_bytes_per_step": int(c.nbytes / ke),
                      "d2h_bytes_per_step": int(yh.numel() * yh.element_size() / ke),
                      "path": "propagate_magnus(midpoint, FastHamiltonian.matvec_at, pinned CPU tensor state): one "
                              "copy in, the steps on the device, one copy out (bytes amortised over the steps)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = _cpu_step_sample(w.name, m)
    return out if rank == 0 else None


def _profile_record():
    p = ROOT / "profiles" / "traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def profiled_traffic(workload: str):
    """dram read+write bytes per matvec from the committed ncu capture, if any."""
    return _profile_record().get(workload)


_MATVEC_KERNELS = ("k_fg_quad", "k_fg_single", "k_fg_pairs", "k_fg_combine", "k_fg_inner", "k_fg_outer", "k_level",
                   "k_coord", "k_cheb", "k_axpy", "k_osc")


def measured_traffic(workload: str, timeout_s: float = 240.0):
    """(DRAM bytes read + written, FP64 flops) of ONE matvec of `workload`, measured now: a child process runs
    tools/prof_matvec.py (one matvec after set construction) under `ncu --metrics
    dram__bytes_read.sum,dram__bytes_write.sum` (and the dfma / dadd / dmul thread-instruction
    counts: flops = 2 dfma + dadd + dmul) and the matvec kernels' counts are summed.  After the
    timed region, never inside it.  None when ncu is missing, fails or exceeds the timeout (the
    committed capture is reported then)."""
    import csv
    import shutil
    import tempfile

    if shutil.which("ncu") is None:
        return None
    with tempfile.TemporaryDirectory() as td:
        log = Path(td) / "traffic.csv"
        fp = "smsp__sass_thread_inst_executed_op_%s_pred_on.sum"
        cmd = ["ncu", "--metrics", ",".join(["dram__bytes_read.sum", "dram__bytes_write.sum"] + [fp % o for o in ("dfma", "dadd", "dmul")]),
               "--clock-control", "none", "--csv",
               "--log-file", str(log), sys.executable, str(ROOT / "tools" / "prof_matvec.py"), workload, "1"]
        try:
            r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout_s)
        except (subprocess.TimeoutExpired, OSError):
            return None
        if r.returncode != 0 or not log.exists():
            return None
        rows = list(csv.reader(ln for ln in log.read_text().splitlines() if ln.startswith('"')))
    if not rows or "Kernel Name" not in rows[0]:
        return None
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    total, flops, seen = 0.0, 0.0, False
    for row in rows[1:]:
        if not any(k in row[ki] for k in _MATVEC_KERNELS):
            continue
        val = float(row[vi].replace(",", ""))
        if row[mi].startswith("dram__bytes"):
            total += val * scale.get(row[ui], 1.0)
            seen = True
        elif "_op_dfma_" in row[mi]:
            flops += 2.0 * val
        elif "_op_dadd_" in row[mi] or "_op_dmul_" in row[mi]:
            flops += val
    return (int(total), int(flops)) if seen else None


def fp64_utilisation(workload: str, ms_step: float, live_flops=None):
    """FP64 rate of the step against the measured DFMA peak: the step's FP64 flops are the ncu
    instruction counts of its kernels (committed with the capture; the kernels' flop count per
    matvec is fixed by the term list, not by the run), divided by this run's step time."""
    rec = _profile_record()
    flops = live_flops or (rec.get("fp64_flops") or {}).get(workload)
    peak = rec.get("fp64_peak_tflops")
    if not flops or not peak:
        return None
    ach = flops / (ms_step * 1e-3) / 1e12
    return {"flops_per_step": flops, "achieved_tflops": round(ach, 3), "peak_tflops": peak,
            "frac": round(ach / peak, 4), "peak_kind": "measured (tools/microbench.cu DFMA chain)",
            "source": "ncu 2 x dfma + dadd + dmul thread instructions of the step's kernels ("
                      + ("counted in this run, same ncu child process as roofline.traffic" if live_flops
                         else "profiles/traffic.json") + ")"}


def step_mode(args, w, rank, world, local_rank, hbm, peak_kind):
    """--mode step: the named propagation run as the headline (one JSON line on rank 0)."""
    if w.nsteps == 0:
        raise SystemExit(f"{w.name} has no propagation run (cfg1, cfg3, cfg4 have)")
    args.prop_steps = w.nsteps if args.steps == 20 else args.steps
    import torch

    sharded = (world > 1 or args.force_shard) and w.kind == "full" and w.batch == 1 and \
        torch.distributed.is_initialized()
    p = propagation_leg(args, w, rank, world, local_rank, hbm, peak_kind, sharded)
    if rank != 0:
        return
    line = {"metric": "Magnus step throughput (midpoint, m = 7)", "value": p["value"], "unit": p["unit"],
            "n_gpus": world, "steps": p["steps"], "warmup": 3, "ms_per_step": p["ms_per_step"],
            "higher_is_better": True, "scaling": "strong" if sharded or world == 1 else "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": {"workload": w.name, "n": p["n"], "dt": w.dt, "m": p["m"], "parallelism": p["parallelism"],
                       "l2": "inputs larger than L2 (no flush)" if p["n"] * 16 > 126e6 else "L2-resident state"},
            "roofline": p["roofline"], "cpu_baseline": p.get("cpu_baseline"), "e2e": p.get("e2e"),
            "gpu_launches": p["gpu_launches"], "clocks": p["clocks"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-reps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-traffic", action="store_true",
                    help="report the committed DRAM-traffic capture instead of measuring one matvec under ncu")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--mode", default="matvec", choices=["matvec", "step"],
                    help="step: the named propagation run (cfg1/cfg3/cfg4) is the headline metric")
    ap.add_argument("--no-prop", action="store_true", help="skip the propagation leg")
    ap.add_argument("--prop-steps", type=int, default=10,
                    help="Magnus steps timed in the propagation leg (capped at the named run's step count)")
    ap.add_argument("--shard-geometry", default=None, metavar="R/P",
                    help="time rank R's slab matvec of a P-rank cfg4 run alone on one GPU (no exchange)")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the slab-sharded code path even at one rank (tests the N>1 path's local part)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    # a process group also for --force-shard under torchrun at one rank (the sharded code path,
    # collectives included, measured on one GPU)
    dist_on = world > 1 or (args.force_shard and "MASTER_ADDR" in os.environ)
    if dist_on:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        gpu_arm(args, rank, world, local_rank)
    finally:
        if dist_on:
            import torch

            torch.distributed.barrier()
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

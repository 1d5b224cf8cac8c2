"""Command-line driver of the device backend, with the reference's CSV schema.

    python -m paper_1403_3511_b200.cli bench     [--dims N] [--kmax 20,40,60] ...
    python -m paper_1403_3511_b200.cli rederr    [--dims N] [--kmax 25,50,75] ...
    python -m paper_1403_3511_b200.cli propagate [--dims N] [--kmax 40] [--h 1/10,1/20] ...

The output format is the reference's (pkg/src/hprop/cli.py:188-217): every option echoed as a
sorted ``# key=value`` header line, one CSV column line, rows with floats at 17 significant
digits, ``\\n`` line ends, stdout or ``--out``; exit codes 0 ok, 1 usage, 3 numerical failure
(cli.py:36-39, 433-444).  Rows are deterministic (the device reductions have a fixed order),
so reruns are byte-identical and ``--jobs`` changes only its own header line.

What each command computes, all on the GPU:

* ``bench`` (cli.py:253-281): the fast-apply time of ``apply_polynomial`` on
  build_hyperbolic(dims, K) with the reference's seeded vector and timing rule (1 warm-up,
  median of 5, here with a device synchronise around each call).  The dense assembled-matrix
  comparison is the reference's verification oracle, out of scope here:
  its columns stay empty with ``dense_status = skipped_no_dense``.
* ``rederr`` (cli.py:299-314): ``reduction_error`` and ``reduction_local_mask`` on the device
  (set vs full cube, extend / restrict kernels) -- the same columns and values as the reference
  within floating-point rounding.
* ``propagate`` (cli.py:342-373): Magnus-Krylov runs of the decay vector over [0, 1] with the
  fast device matvec for each step size.  The reference measures ``scheme_error`` against an
  assembled-matrix GL2 reference and ``perturbation_error`` against an assembled-matrix run;
  without the dense oracle, ``scheme_error`` here is measured against a GL2 reference built with
  the same fast matvec (``--reference-steps`` steps, ``--reference-lanczos`` Krylov vectors) and
  ``perturbation_error`` is left empty.  The header says so (``reference=fast-gl2``).
"""

from __future__ import annotations

import argparse
import dataclasses
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from fractions import Fraction

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_VERIFY, EXIT_NUMERICAL = 0, 1, 2, 3
_REPS, _WARMUP = 5, 1
DEFAULT_DENSE_CAP = 20000


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def _ints(text: str) -> list[int]:
    try:
        vals = sorted({int(t) for t in text.split(",") if t.strip()})
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}") from None
    if not vals:
        raise argparse.ArgumentTypeError("empty integer list")
    if vals[0] < 0:
        raise argparse.ArgumentTypeError("list entries must be nonnegative")
    return vals


def _fractions(text: str) -> list[Fraction]:
    out = []
    for tok in (t.strip() for t in text.split(",")):
        if not tok:
            continue
        try:
            out.append(Fraction(tok))
        except (ValueError, ZeroDivisionError):
            raise argparse.ArgumentTypeError(f"expected fractions like 1/80, got {tok!r}") from None
    if not out:
        raise argparse.ArgumentTypeError("empty step list")
    if min(out) <= 0:
        raise argparse.ArgumentTypeError("step sizes must be positive")
    return out


def _positive(text: str) -> int:
    try:
        v = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected an integer, got {text!r}") from None
    if v < 1:
        raise argparse.ArgumentTypeError("value must be at least 1")
    return v


def build_parser() -> argparse.ArgumentParser:
    top = _Parser(prog="hprop-b200", description="device backend of the hprop experiment driver")
    sub = top.add_subparsers(dest="command", required=True)

    def opts(p, *, beta, degree, kmax, potential):
        p.add_argument("--dims", type=_positive, default=2)
        p.add_argument("--kmax", type=_ints, default=_ints(kmax))
        p.add_argument("--degree", type=int, default=degree)
        p.add_argument("--halfwidth", type=float, default=16.0)
        p.add_argument("--scale", type=float, default=1.0)
        p.add_argument("--beta", type=_positive, default=beta)
        p.add_argument("--potential", default=potential, choices=["torsional", "torsional-ho", "henon-heiles"])
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--jobs", type=_positive, default=1)
        p.add_argument("--out", default=None)

    p = sub.add_parser("bench", help="fast-apply timing on the device")
    opts(p, beta=5, degree=8, kmax="20,40,60", potential="torsional")
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("rederr", help="index-set reduction error on the device")
    opts(p, beta=5, degree=8, kmax="25,50,75", potential="torsional")
    p.set_defaults(func=cmd_rederr)
    p = sub.add_parser("propagate", help="Magnus-Krylov propagation on the device")
    opts(p, beta=3, degree=3, kmax="40", potential="henon-heiles")
    p.add_argument("--scheme", default="midpoint", choices=["midpoint", "gl2"])
    p.add_argument("--lanczos", type=_positive, default=7)
    p.add_argument("--h", type=_fractions, default=_fractions("1/10,1/20,1/40,1/80,1/160"))
    p.add_argument("--reference-steps", type=_positive, default=10_000)
    p.add_argument("--reference-lanczos", type=_positive, default=20)
    p.set_defaults(func=cmd_propagate)
    return top


# ---------------------------------------------------------------- output

def _cell(v) -> str:
    if v is None:
        return ""
    return f"{v:.17g}" if isinstance(v, float) else str(v)


def _write(args, meta: dict, columns, rows) -> None:
    text = "".join(f"# {k}={meta[k]}\n" for k in sorted(meta))
    text += ",".join(columns) + "\n"
    text += "".join(",".join(_cell(c) for c in r) + "\n" for r in rows)
    if args.out:
        with open(args.out, "w", newline="\n") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def _header(args, **extra) -> dict:
    meta = {"command": args.command}
    for k, v in vars(args).items():
        if k in ("func", "out", "command"):
            continue
        meta[k] = ",".join(map(str, v)) if isinstance(v, list) else v
    meta.update(extra)
    return meta


def _support_warnings(args) -> None:
    """The reference's advisory S L >= sqrt(2(K+1)) + 1 check (hermite_basis.py:164-179)."""
    if args.scale <= 0 or args.halfwidth <= 0:
        raise ValueError("scaling and halfwidth must be positive")
    for k in args.kmax:
        need = math.sqrt(2.0 * (k + 1)) + 1.0
        have = args.scale * args.halfwidth
        if have < need:
            print(f"support condition violated: S*L = {have:.4g} < sqrt(2(K+1)) + 1 = {need:.4g} "
                  f"(deficit {need - have:.4g}); the truncated basis is not resolved on [-L, L] and "
                  "interpolation degrades", file=sys.stderr)


def _approx(args, t: float = 0.0):
    from .potential_approx import interpolate, potential_by_name

    ap = interpolate(potential_by_name(args.potential, args.dims, args.halfwidth), args.degree, time=t)
    if args.scale != 1.0:  # dilated basis: node coordinates u = S x (cli.py:227-239)
        ap = dataclasses.replace(ap, halfwidth=args.scale * args.halfwidth)
    return ap


def _sweep(args, fn, points):
    if args.jobs == 1 or len(points) <= 1:
        return [fn(p) for p in points]
    with ThreadPoolExecutor(max_workers=args.jobs) as pool:
        return list(pool.map(fn, points))


def _dense_cap() -> int:
    raw = os.environ.get("HPROP_DENSE_CAP")
    if raw is None:
        return DEFAULT_DENSE_CAP
    try:
        return int(raw)
    except ValueError:
        raise ValueError(f"HPROP_DENSE_CAP must be an integer, got {raw!r}") from None


# ---------------------------------------------------------------- commands

def cmd_bench(args) -> int:
    import torch

    from . import build_hyperbolic, get_applier

    _support_warnings(args)
    ap = _approx(args)

    def point(k: int):
        iset = build_hyperbolic(args.dims, k)
        v = np.random.default_rng([args.seed, args.dims, k]).standard_normal(iset.size)
        appl = get_applier(iset)

        def once():
            appl.apply_polynomial(ap, v)
            torch.cuda.synchronize()

        for _ in range(_WARMUP):
            once()
        ts = []
        for _ in range(_REPS):
            t0 = time.perf_counter()
            once()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        return [args.dims, k, iset.size, ap.nterms, ts[len(ts) // 2], None, None, "skipped_no_dense"]

    rows = _sweep(args, point, args.kmax)
    _write(args, _header(args, dense_cap=_dense_cap(), backend="b200"),
           ["dim", "bound", "set_size", "nterms", "t_fast_s", "t_dense_s", "ratio", "dense_status"], rows)
    return EXIT_OK


def cmd_rederr(args) -> int:
    from . import build_hyperbolic, make_decay_vector
    from .error_lab import reduction_error, reduction_local_mask

    _support_warnings(args)

    def point(k: int):
        iset = build_hyperbolic(args.dims, k)
        ap = _approx(args)
        rep = reduction_error(iset, ap, make_decay_vector(iset, args.beta))
        mask = reduction_local_mask(iset, ap)
        comp = np.asarray(rep.components)
        return [args.dims, k, iset.size, rep.max_norm, float(comp[mask].max()) if mask.any() else 0.0]

    rows = _sweep(args, point, args.kmax)
    _write(args, _header(args, backend="b200"), ["dim", "bound", "set_size", "max_norm", "interior_max"], rows)
    return EXIT_OK


def cmd_propagate(args) -> int:
    import torch

    from . import FastHamiltonian, MagnusScheme, build_hyperbolic, make_decay_vector, potential_by_name
    from .krylov_propagator import propagate_magnus

    if args.scale != 1.0:
        print("propagate assumes the undilated oscillator splitting; --scale must be 1", file=sys.stderr)
        return EXIT_USAGE
    _support_warnings(args)
    counts = []
    for h in args.h:
        inv = 1 / h
        if inv.denominator != 1:
            print(f"step {h} does not divide [0, 1] evenly", file=sys.stderr)
            return EXIT_USAGE
        counts.append(int(inv))
    spec = potential_by_name(args.potential, args.dims, args.halfwidth)
    scheme = MagnusScheme.from_name(args.scheme)

    def point(k: int):
        iset = build_hyperbolic(args.dims, k)
        fh = FastHamiltonian(iset, spec, args.degree)
        y0 = torch.from_numpy(make_decay_vector(iset, args.beta).data.astype(np.complex128)).cuda()
        ref = propagate_magnus(MagnusScheme.from_name("gl2"), fh.matvec_at, y0, 0.0, 1.0, args.reference_steps,
                               args.reference_lanczos)
        out = []
        for n in counts:
            y = propagate_magnus(scheme, fh.matvec_at, y0, 0.0, 1.0, n, args.lanczos)
            err = float(torch.max(torch.abs(y - ref)))
            out.append([args.dims, k, iset.size, args.scheme, args.lanczos, str(Fraction(1, n)), 1.0 / n, err, None])
        return out

    rows = [r for grp in _sweep(args, point, args.kmax) for r in grp]
    _write(args, _header(args, backend="b200", reference="fast-gl2"),
           ["dim", "bound", "set_size", "scheme", "krylov_steps", "step", "step_value", "scheme_error",
            "perturbation_error"], rows)
    return EXIT_OK


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else EXIT_USAGE
    try:
        return args.func(args)
    except (ValueError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL


if __name__ == "__main__":
    sys.exit(main())

"""Golden outputs of the reference's reduction-error path and CLI (maps.npz).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_maps.py

Runs the REFERENCE (imported read-only) on small cases:

* ``reduction_error`` components and ``reduction_local_mask`` (error_lab.py:114-148) on
  hyperbolic sets with the reference's decay vector (error_lab.py:43-56);
* ``make_decay_vector`` (error_lab.py:43-56) on three sets;
* the CSV text of ``hprop rederr`` (cli.py:299-314) for two argument lists, to compare the
  device CLI's columns and values against.
"""

import io
import sys
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import hprop  # noqa: E402
from hprop import cli, error_lab  # noqa: E402

OUT = Path(__file__).resolve().parent / "maps.npz"
CASES = [("torsional", 2, 12, 4, 3), ("henon-heiles", 3, 10, 3, 2), ("torsional-ho", 4, 8, 4, 1)]
CLI_ARGS = [["rederr", "--kmax", "12", "--degree", "4", "--beta", "3"],
            ["rederr", "--dims", "3", "--kmax", "6,9", "--degree", "3", "--beta", "2", "--potential", "henon-heiles"]]


def main():
    g = {}
    for pot, dim, bound, deg, beta in CASES:
        s = hprop.build_hyperbolic(dim, bound)
        ap = hprop.interpolate(hprop.potential_by_name(pot, dim), deg)
        v = error_lab.make_decay_vector(s, beta)
        rep = error_lab.reduction_error(s, ap, v)
        key = f"red_{pot}_{dim}_{bound}_{deg}_{beta}"
        g[key + "_comp"] = rep.components
        g[key + "_mask"] = error_lab.reduction_local_mask(s, ap)
        g[key + "_max"] = np.float64(rep.max_norm)
    for kind, dim, bound, beta, norm in [("hyperbolic", 3, 10, 2, True), ("full", 2, 7, 3, True),
                                         ("hyperbolic", 4, 8, 1, False)]:
        s = (hprop.build_hyperbolic if kind == "hyperbolic" else hprop.build_full)(dim, bound)
        g[f"decay_{kind}_{dim}_{bound}_{beta}_{int(norm)}"] = error_lab.make_decay_vector(s, beta, normalized=norm).data
    for i, argv in enumerate(CLI_ARGS):
        buf = io.StringIO()
        with redirect_stdout(buf):
            assert cli.main(argv) == 0
        g[f"cli{i}_argv"] = np.array(argv)
        g[f"cli{i}_text"] = np.array(buf.getvalue())
    np.savez_compressed(OUT, **g)


if __name__ == "__main__":
    main()

"""pytest plugin: run the REFERENCE's own test modules with the device applier installed.

    PYTHONPATH=tests python -m pytest -p ref_suite_plugin baseline/_ref/tests/test_fast_apply.py ...

Every index set the reference tests build gets the B200 applier on first use: the plugin
replaces `hprop.fast_apply.get_applier` (fast_apply.py:248-254, the seam every caller resolves
through) with one that calls `paper_1403_3511_b200.install(iset)` -- so fast_algorithm,
apply_hamiltonian, direct_op, cheb_of_coordinate_apply, square_sum_apply, FastHamiltonian and
the CLI run their matvecs on the GPU while the tests' dense oracles stay numpy.  The counter
`installed` proves the device path ran.
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
installed = {"sets": 0}


def pytest_configure(config):
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    sys.path.insert(0, str(ROOT))
    import hprop
    import hprop.fast_apply as fa

    import paper_1403_3511_b200 as hb

    def get_applier(iset):
        appl = iset._derived.get("applier")
        if appl is None:
            appl = hb.install(iset)
            installed["sets"] += 1
        return appl

    for mod in list(sys.modules.values()):
        if getattr(mod, "__name__", "").startswith("hprop") and getattr(mod, "get_applier", None) is fa.get_applier:
            mod.get_applier = get_applier
    fa.get_applier = get_applier
    hprop.get_applier = get_applier


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"[ref_suite_plugin] device appliers installed: {installed['sets']}")

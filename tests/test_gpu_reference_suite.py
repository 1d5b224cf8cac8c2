"""The REFERENCE's own test modules, run with the B200 applier installed in every index set.

`tests/ref_suite_plugin.py` replaces hprop's `get_applier` seam (fast_apply.py:248-254) by one
that installs `paper_1403_3511_b200.PolynomialApplier` on first use, then runs the reference's
tests unchanged: test_fast_apply (dense ordered-product oracles at 1e-13, grouped vs per-term at
1e-15, linearity, axis-order semantics, error paths, square sum), test_index_set, the Lanczos /
Magnus tests of test_krylov_propagator, test_error_lab (FastHamiltonian against the assembled
oracle), test_acceptance (Lemma 1, paper error bands, propagation orders, cost gates) and
test_cli -- every fast matvec on the GPU, every oracle in numpy.  SURVEY.md §4 names this subset
as the parity suite to re-run against the GPU backend.

The modules come from baseline/_ref/tests (tools/install_reference.sh copies them next to the
installed package; git-ignored, shipped to the GPU box with the snapshot).
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref" / "tests"
MODULES = ["test_fast_apply.py", "test_index_set.py", "test_krylov_propagator.py", "test_error_lab.py",
           "test_acceptance.py", "test_cli.py"]

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not (SUITE / "test_fast_apply.py").exists(),
                                                  reason="reference tests not installed (tools/install_reference.sh)")]


def test_reference_suite_passes_on_the_device_applier():
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_suite_plugin", "-q", "-p", "no:cacheprovider",
           "--rootdir", str(SUITE)] + [str(SUITE / m) for m in MODULES]
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), os.environ.get("PYTHONPATH", "")]))
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800, env=env)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    m = re.search(r"device appliers installed: (\d+)", r.stdout)
    assert m and int(m.group(1)) > 20, tail
    passed = re.search(r"(\d+) passed", r.stdout)
    assert passed and int(passed.group(1)) >= 90, tail

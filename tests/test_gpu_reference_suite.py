"""GPU: the reference's own 134-test suite (pkg/tests) passes on the drop-in by import substitution.

`tools/refcheck/run_reference_tests.sh stage` copies the reference's test files into the
git-ignored scratch directory `.refcheck/` (never committed; it travels to the GPU box with the
working tree) together with a conftest that maps `import slosim` onto paper_2605_02329_b200
(tools/refcheck/slosim_shim.py) and reports which native library served the run.  The suite then
runs unmodified against the B200 engine.  Skipped when the files are not staged.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = os.path.join(ROOT, ".refcheck")


@pytest.mark.timeout(1800)
def test_reference_suite_passes_on_dropin():
    if not os.path.exists(os.path.join(STAGE, "test_acceptance.py")):
        pytest.skip("reference tests not staged (bash tools/refcheck/run_reference_tests.sh stage)")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-s", "."], cwd=STAGE,
                       capture_output=True, text=True, timeout=1700)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) == 134, tail
    assert "failed" not in r.stdout.splitlines()[-1], tail
    # the drop-in served the suite through the native library
    assert re.search(r"\[refcheck\] slosim\.engine -> paper_2605_02329_b200\.engine .*libslosim_b200\.so", r.stdout), tail

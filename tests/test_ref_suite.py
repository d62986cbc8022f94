"""SURVEY.md 7.2 acceptance run of the drop-in boundary: the reference's OWN
test suite (pkg/tests: test_decomp, test_blocks, test_reconstruct,
test_acceptance criteria 1-10, ... -- 173 tests) run against the unmodified
``blockten`` with bt200 installed behind it (``tests/ref_suite_plugin.py``),
so every hot-path call in those tests goes through the sm_100a kernels.

The reference and a copy of its tests live untracked under ``baseline/_ref``
(pip install of /root/reference); the test skips
where that directory is absent."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "blockten_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="baseline/_ref/blockten_tests not present")
def test_reference_suite_passes_with_bt200_installed():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT,
                                         env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-m", "pytest", ".", "-p", "ref_suite_plugin", "-q",
                           "-rf", "-p", "no:cacheprovider"],
                          cwd=SUITE, env=env, capture_output=True, text=True, timeout=1200)
    out = proc.stdout + proc.stderr
    log_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log_dir):
        with open(os.path.join(log_dir, "ref_suite_pytest.log"), "w") as fh:
            fh.write(out)
    m = re.search(r"bt200 installed behind blockten: (\d+) bindings, still installed at exit: True", out)
    assert m and int(m.group(1)) > 100, out[-2000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 173, out[-3000:]
    assert proc.returncode == 0, out[-3000:]

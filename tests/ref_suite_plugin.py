"""pytest plugin: the reference's OWN test suite (pkg/tests, copied untracked
under baseline/_ref/blockten_tests next to the pip-installed reference) run
with bt200 installed behind the unmodified ``blockten`` -- SURVEY.md 7.2's
acceptance run for the drop-in boundary.

    python -m pytest baseline/_ref/blockten_tests -p ref_suite_plugin \\
        (with tests/ and baseline/_ref on PYTHONPATH; tests/test_ref_suite.py)

``install()`` runs before collection, so the test modules' own
``from blockten... import`` lines already bind bt200's functions."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_2105_01170_b200 as bt

    done = bt.install()
    n = sum(len(v) for v in done.values())
    config._bt200_rebound = n


def pytest_report_header(config):
    return f"bt200 installed behind blockten: {getattr(config, '_bt200_rebound', 0)} bindings"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    import paper_2105_01170_b200 as bt

    terminalreporter.write_line(
        f"bt200 installed behind blockten: {getattr(config, '_bt200_rebound', 0)} bindings, "
        f"still installed at exit: {bt.installed()}")

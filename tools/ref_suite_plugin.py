"""pytest plugin: run the reference's OWN test suite with its hot path rebound
to the B200 kernels (the installer must rebind the names before
the test modules import them, hence ``-p``).

Loaded by ``tools/run_reference_suite.sh``; expects the unmodified reference
installed in ``baseline/_ref`` (``pip install --target baseline/_ref``) and its
tests copied next to it. Test infrastructure only: nothing in the product
imports this file.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import zernkit  # noqa: E402  (the reference package, unmodified)

from paper_2409_19156_b200 import _lib  # noqa: E402
from paper_2409_19156_b200.zernkit_plugin import install  # noqa: E402

_DONE = install(zernkit)


def pytest_report_header(config):
    return [f"zernkit from {os.path.dirname(zernkit.__file__)}",
            "rebound to the B200 path: " + ", ".join(sorted(_DONE))]


def pytest_terminal_summary(terminalreporter):
    launches = sum(ctx.launches() for ctx in _lib._contexts.values())
    terminalreporter.write_line(
        f"B200 kernel launches during the reference suite: {launches} "
        f"(contexts: {sorted(_lib._contexts)})")

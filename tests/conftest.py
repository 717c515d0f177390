"""pytest configuration: the ``gpu`` marker and repo-root import path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs on one box")


import numpy as _np  # noqa: E402

# the oracle and pins deliberately overflow / make NaN on the "specials" mix
_np.seterr(all="ignore")


def pytest_collection_modifyitems(config, items):
    """Safety net: a GPU test that hangs (a cross-rank wait that never
    resolves) fails after a bound instead of stalling the run (pytest-timeout,
    when installed; explicit per-test timeouts win)."""
    if not config.pluginmanager.hasplugin("timeout"):
        return
    import pytest
    for it in items:
        if it.get_closest_marker("gpu") and not it.get_closest_marker("timeout"):
            it.add_marker(pytest.mark.timeout(1800 if it.get_closest_marker("multigpu") else 600))

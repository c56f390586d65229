import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# Cross-checks against the reference package itself (tests marked
# ``reference``: tests/test_host_logic.py, tests/test_reference_suite.py) need
# its source tree.  SDB_REFERENCE_SRC names it; unset, the build container's
# read-only copy is used when present (it is absent on the GPU box, where
# those tests skip and the pinned goldens carry the parity); set it to the
# empty string to switch the cross-checks off.  The path is appended, so it
# never shadows this repo.  The report header says which case a run is in.
_REF_SRC = os.environ.get("SDB_REFERENCE_SRC", "/root/reference/pkg/src")
REFERENCE_ACTIVE = bool(_REF_SRC) and os.path.isdir(_REF_SRC)
if REFERENCE_ACTIVE and _REF_SRC not in sys.path:
    sys.path.append(_REF_SRC)


def pytest_report_header(config):
    return ("reference cross-checks: " +
            (f"ON (specdens imported from {_REF_SRC})" if REFERENCE_ACTIVE else
             "OFF (no reference source tree; tests marked 'reference' skip)"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built library")
    config.addinivalue_line("markers", "slow: long-running")
    config.addinivalue_line("markers", "reference: imports the reference package (skips without its source tree)")


def _cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden

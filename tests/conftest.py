import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built CUDA library")


class Golden:
    def __init__(self):
        self.arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            self.meta = json.load(fh)

    def __getitem__(self, key):
        return self.arrays[key]

    def has(self, key):
        return key in self.arrays.files

    def case(self, name):
        return self.meta["cases"][name]


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def cuda_lib():
    """The built C-ABI library on a CUDA device; GPU tests fail (not skip) if
    the device exists but the library does not load."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_13681_b200 import _lib

    return _lib.lib()


def pytest_sessionfinish(session, exitstatus):
    """Write every near-tie the parity checks accepted (tests/parity.py)."""
    try:
        import parity
    except ImportError:
        return
    if parity.TIES:
        out = os.environ.get("LS_REPORT_DIR", "gpurun_out")
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "near_ties.json"), "w") as fh:
            json.dump({"near_tie_rel": parity.NEAR_TIE_REL, "ties": parity.TIES}, fh, indent=1)

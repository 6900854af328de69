import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a CUDA path)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")
    runs = np.load(os.path.join(d, "reference_runs.npz"))
    kern = np.load(os.path.join(d, "reference_kernels.npz"))
    with open(os.path.join(d, "reference_meta.json")) as fh:
        meta = json.load(fh)
    return {"runs": runs, "kernels": kern, "meta": meta}

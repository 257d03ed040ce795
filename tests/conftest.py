import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large N) checks")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with np.load(os.path.join(here, "small_cases.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    with open(os.path.join(here, "digests.json")) as f:
        digests = json.load(f)
    with open(os.path.join(here, "kats.json")) as f:
        kats = json.load(f)
    return {"arrays": arrays, "digests": digests, "kats": kats}


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle

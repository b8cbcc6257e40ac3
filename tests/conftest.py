import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA engine)")
    config.addinivalue_line("markers", "slow: full-size config cases")


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden_meta.json")) as fh:
        meta = json.load(fh)
    return data, meta


@pytest.fixture(scope="session")
def oracle():
    from oracle import l0_oracle
    l0_oracle.build_c_oracle()
    return l0_oracle


@pytest.fixture(scope="session")
def engine():
    """The CUDA engine (GPU tests only).  Fails loudly if the extension is absent."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_09502_b200 as eng
    eng.native.load()
    return eng

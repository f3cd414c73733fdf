import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_vectors.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def po():
    from oracle import bind

    if not os.path.exists(bind.RESTATEMENT_SO):
        bind.build(reference=False)
    return bind.Restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle import bind

    if not bind.reference_available():
        if os.path.isdir("/root/reference/proj/src"):
            bind.build(reference=True)
        else:
            pytest.skip("reference library not built on this host")
    return bind.Reference()


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test needs a CUDA device")
    return torch.device("cuda:0")


def rand_codes(rng, nbits, shape, nar_ok=False):
    c = rng.integers(0, 1 << nbits, shape).astype(np.uint64)
    if not nar_ok:
        c[c == (1 << (nbits - 1))] = 0
    return c

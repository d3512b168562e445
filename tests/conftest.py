import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box)")


@pytest.fixture(scope="session")
def port():
    import oracle as o
    return o.CPort()


@pytest.fixture(scope="session")
def ref():
    import oracle as o
    if not o.Reference.available():
        pytest.skip("reference library (oracle/_ref) not built here")
    return o.Reference()


@pytest.fixture(scope="session")
def checker():
    """The reference itself when built, else the pinned C port."""
    import oracle as o
    return o.best_available()


def synth(h, w, n=1, first=0, seed=7, ellipses=20, sigma=5.0, video=False):
    import paper_2001_09632_b200 as p
    return p.synth_images_host(p.SynthSpec(h, w, ellipses, sigma, seed, video), first, n)


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(12345)

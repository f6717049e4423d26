import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_pipeline.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device and libtaco.so")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def golden_cases(g):
    names = sorted({k.split("/")[0] for k in g if not k.startswith("kat/")})
    return names


@pytest.fixture(scope="session")
def built_lib():
    from paper_2404_04895_b200 import build

    return build.build_library()


def euclid(seed: int, n: int, scale: float = 1000.0):
    from paper_2404_04895_b200 import euclidean_instance

    return euclidean_instance(np.random.default_rng(seed).uniform(0.0, scale, size=(n, 2)))

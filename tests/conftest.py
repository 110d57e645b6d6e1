import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    # same seed as the reference's conftest (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240814)


def random_unit_vectors(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def scipy_basis(dirs, order):
    """Independent real-SH oracle on scipy's complex harmonics.

    Same construction as the reference's test oracle (pkg/tests/conftest.py:25-45):
    sqrt2*Re(Y_l^|m|) for m<0, Y_l^0, sqrt2*Im(Y_l^m) for m>0.
    """
    import scipy.special as sp

    dirs = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
    theta = np.arccos(np.clip(dirs[:, 2], -1.0, 1.0))
    phi = np.arctan2(dirs[:, 1], dirs[:, 0])
    out = np.empty((dirs.shape[0], (order + 1) * (order + 2) // 2))
    for l in range(0, order + 1, 2):
        for m in range(-l, l + 1):
            j = l * (l + 1) // 2 + m
            h = sp.sph_harm_y(l, abs(m), theta, phi)
            out[:, j] = np.sqrt(2.0) * h.real if m < 0 else (h.real if m == 0 else np.sqrt(2.0) * h.imag)
    return out

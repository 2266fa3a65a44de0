import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: large BASELINE-size case")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def P():
    import paper_1105_5331_b200 as P
    return P


@pytest.fixture(scope="session")
def O():
    from oracle import pyoracle as O
    return O


@pytest.fixture(scope="session")
def gpu(P):
    if P.device_count() < 1:
        pytest.fail("gpu-marked test ran without a visible CUDA device")
    yield P
    # guard-band build (CPFIT_GPU_LIB=.../libcpfit_gpu_guard.so, csrc/guard.cu): after the whole
    # GPU session every device buffer's 4 KB guard bands must be intact
    import gc
    gc.collect()
    v, n = P.debug_guard_check()
    if v >= 0:
        print(f"\nguard-band check: {v} violations, {n} live device buffers")
        assert v == 0, f"{v} device buffers were written out of bounds (see stderr)"


def random_matrix(rng, rows, cols, lo=-1.0, hi=1.0):
    # test_util.hpp:11-17 (uniform in [lo, hi)), column-major fill
    return lo + (hi - lo) * rng.random((rows, cols)).T.copy().T


def random_factors(rng, dims, rank):
    return np.concatenate([(2.0 * rng.random(d * rank) - 1.0) for d in dims])


def random_sparse(rng, dims, density):
    # test_util.hpp:26-41
    K = int(np.prod(dims))
    mask = rng.random(K) < density
    flat = np.nonzero(mask)[0]
    coords = np.stack(np.unravel_index(flat, dims, order="F"), axis=1).astype(np.int64)
    vals = rng.random(flat.size) * 2.0 - 1.0
    return coords, vals

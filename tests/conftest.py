"""Shared fixtures.  `-m gpu` tests need a B200 and call the CUDA path through
the C-ABI; everything else runs on CPU (oracle vs golden vectors, host logic,
C-ABI symbol checks)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefLib, have_ref
    if not have_ref():
        pytest.skip("reference library oracle/_ref not built")
    return RefLib()


@pytest.fixture(scope="session")
def cyc():
    import paper_2405_16911_b200 as cyc
    from paper_2405_16911_b200 import build
    build.build()
    cyc.lib()
    return cyc


def rand_c(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return ((rng.standard_normal(n) + 1j * rng.standard_normal(n)) * scale).astype(np.complex64)


def mean_power(x):
    x = np.asarray(x, dtype=np.complex128)
    return float(np.mean(np.abs(x) ** 2))


def assert_parity(got, want, meanpow, rel_l2=1e-4, cell=1e-5, what=""):
    """BASELINE.json north_star tolerance: relative L2 <= 1e-4 per table and
    |dR| <= 1e-5 * mean power per value."""
    got = np.asarray(got, dtype=np.complex128)
    want = np.asarray(want, dtype=np.complex128)
    assert got.shape == want.shape, (got.shape, want.shape)
    d = np.abs(got - want)
    nrm = np.linalg.norm(want)
    rl2 = np.linalg.norm(got - want) / nrm if nrm > 0 else np.linalg.norm(got - want)
    mx = d.max() if d.size else 0.0
    assert rl2 <= rel_l2, f"{what}: relative L2 {rl2:.3e} > {rel_l2}"
    assert mx <= cell * meanpow, f"{what}: max |dR| {mx:.3e} > {cell} * {meanpow:.3e}"
    return rl2, mx

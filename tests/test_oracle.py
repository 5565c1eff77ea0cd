"""CPU: pin the oracle (oracle/cycoracle.c) before trusting it.

1. against the reference's frozen literal-sum values (proj/tests/test_reference.cpp:54-67);
2. against outputs of the reference library itself, frozen in
   tests/golden/reference_golden.npz by tests/golden/make_golden.py;
3. live against oracle/_ref (the reference compiled from its sources) where present.
"""
import os

import numpy as np
import pytest

from conftest import rand_c

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_frozen_literal_values(oracle):
    x = np.array([1, 1j, -1 + 0.5j, 2 - 1j, 1 + 1j, -1j, 0.5, -1 - 1j])
    a = oracle.direct(x, x, 0.25, 1, False, 1, 4)
    b = oracle.direct(x, x, 0.25, 1, True, 1, 4)
    c = oracle.direct(x, x, 0.11, -1, False, 2, 4)
    assert a.real == pytest.approx(-0.12499999999999993, rel=1e-12)
    assert a.imag == pytest.approx(-0.12500000000000011, rel=1e-12)
    assert b.real == pytest.approx(0.12499999999999999, rel=1e-12)
    assert b.imag == pytest.approx(0.12500000000000006, rel=1e-12)
    assert c.real == pytest.approx(-0.26908075755090433, rel=1e-12)
    assert c.imag == pytest.approx(0.66834328861739112, rel=1e-12)


def test_direct_coverage_errors(oracle):
    x = np.ones(8, complex)
    for args in [(0.1, 0, 0, 0, 0), (0.1, 0, 0, 5, 4), (0.1, 2, 0, 3, 4), (0.1, -2, 0, 1, 4)]:
        with pytest.raises(ValueError):
            oracle.direct(x, x, *args)


def test_golden_frozen(oracle, gold):
    fz = gold["frozen_x"]
    got = [oracle.direct(fz, fz, 0.25, 1, 0, 1, 4), oracle.direct(fz, fz, 0.25, 1, 1, 1, 4),
           oracle.direct(fz, fz, 0.11, -1, 0, 2, 4)]
    assert np.max(np.abs(np.array(got) - gold["frozen_vals"])) == 0.0


@pytest.mark.parametrize("conj", [0, 1])
def test_set_stream_matches_reference_golden(oracle, gold, conj):
    got = oracle.stream(0, conj, 64, gold["set_x"], gold["set_y"], alphas=gold["set_alphas"], max_lag=3)
    want = gold[f"set_frames_conj{conj}"]
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= 1e-13


@pytest.mark.parametrize("conj", [0, 1])
def test_full_stream_matches_reference_golden(oracle, gold, conj):
    got = oracle.stream(1, conj, 64, gold["full_x"], gold["full_y"], lags=[-3, 0, 5])
    want = gold[f"full_frames_conj{conj}"]
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= 1e-13


@pytest.mark.parametrize("conj", [0, 1])
def test_block_fold_matches_reference_average(oracle, gold, conj):
    x = gold["block_x"]
    F = int(gold["block_frames"])
    cv, cj = oracle.block_fold(x, x, np.arange(256), 256, list(range(8)), 0, F * 256)
    got = (cj if conj else cv).T.reshape(-1)
    assert np.max(np.abs(got - gold[f"block_avg_conj{conj}"])) <= 1e-13


def test_fft_matches_reference(oracle, gold):
    v = gold["fft_in"]
    assert np.max(np.abs(oracle.fft(v[:64]) - gold["fft64"])) <= 1e-13
    assert np.max(np.abs(oracle.fft(v) - gold["fft100"])) <= 1e-12


def test_fft_identities(oracle):
    assert np.allclose(oracle.fft(np.array([1, 0, 0, 0], complex)), [1, 1, 1, 1])
    assert np.allclose(oracle.fft(np.ones(4, complex)), [4, 0, 0, 0])
    v = rand_c(64, 3).astype(complex)
    V = oracle.fft(v)
    assert abs(np.sum(np.abs(v) ** 2) - np.sum(np.abs(V) ** 2) / 64) <= 1e-10 * np.sum(np.abs(v) ** 2)


def test_tone_identity(oracle, gold):
    t = gold["tone"]
    fr = oracle.stream(0, 0, 64, t, t, alphas=[0.0], max_lag=2)
    assert np.max(np.abs(fr - gold["tone_frames"])) <= 1e-13
    for m in range(-2, 3):
        assert np.max(np.abs(fr[:, m + 2] - np.exp(2j * np.pi * 0.125 * m))) <= 1e-12


def test_block_direct_equals_fold(oracle):
    x = rand_c(5000, 17)
    alphas = np.arange(-8, 8) / 32
    lags = [0, 1, 3, 7]
    bd = oracle.block_direct(x.astype(complex), x.astype(complex), alphas, lags, 0, 10, 4096)
    cv, _ = oracle.block_fold(x, x, np.arange(-8, 8), 32, lags, 10, 4096)
    assert np.max(np.abs(bd - cv)) <= 1e-12


def test_recursive_literal_definition(oracle):
    """Recursive restatement == literal weighted sums (builder-defined mode)."""
    x = rand_c(300, 23).astype(complex)
    lam, E = 0.9, 64
    got = oracle.recursive(x, x, [0.125], [0, 2], 0, lam, E)
    n_emit = got.shape[0]
    assert n_emit == (300 - E - 2) // E + 1
    for e in range(n_emit):
        n_end = (e + 1) * E - 1
        for t, lag in enumerate([0, 2]):
            acc = 0
            for n in range(n_end + 1):
                acc += (1 - lam) * lam ** (n_end - n) * x[n + lag] * np.conj(x[n]) * np.exp(-2j * np.pi * 0.125 * n)
            assert abs(got[e, 0, t] - acc) <= 1e-12


def test_mt19937_64_reference_value():
    """std::mt19937_64 10000th output with default seed is 9981545732273789042 ([rand.predef])."""
    import ctypes as C
    from oracle.oracle import ORACLE_SO
    L = C.CDLL(ORACLE_SO)

    class MT(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]

    L.orc_mt64_next.restype = C.c_uint64
    s = MT()
    L.orc_mt64_seed(C.byref(s), C.c_uint64(5489))
    v = 0
    for _ in range(10000):
        v = L.orc_mt64_next(C.byref(s))
    assert v == 9981545732273789042


def test_live_reference_random_cases(oracle, ref):
    for seed in range(3):
        x, y = rand_c(700, seed).astype(complex), rand_c(700, seed + 50).astype(complex)
        for conj in (0, 1):
            a, _ = ref.stream(0, conj, 128, x, y, alphas=[0.1, -0.37, 0.25], max_lag=5, chunk=1 + seed * 97)
            b = oracle.stream(0, conj, 128, x, y, alphas=[0.1, -0.37, 0.25], max_lag=5)
            assert np.max(np.abs(a - b)) <= 1e-13
            a, _ = ref.stream(1, conj, 128, x, y, lags=[-4, 0, 2, 9], chunk=0)
            b = oracle.stream(1, conj, 128, x, y, lags=[-4, 0, 2, 9])
            assert np.max(np.abs(a - b)) <= 1e-13

"""CPM/GMSK generation on the device and the Monte-Carlo
cyclic-magnitude oracle, against the reference's own implementation
(oracle/_ref: random_symbols, make_pulse, cpm_modulate, gmsk_mc_oracle;
proj/src/siggen.cpp, proj/src/reference.cpp:34-96).  Cases follow
proj/tests/test_reference.cpp:117-190 and proj/tests/test_siggen.cpp."""
import numpy as np
import pytest


# ---- CPU: host-side pieces (no device needed) ----

@pytest.mark.parametrize("M,seed", [(2, 42), (4, 7), (8, 12345)])
def test_random_symbols_identical_to_reference(cyc, ref, M, seed):
    assert np.array_equal(cyc.random_symbols(M, 5000, seed), ref.random_symbols(M, 5000, seed))


@pytest.mark.parametrize("p", [dict(), dict(bt=0.3), dict(bt=0.5, sps=4), dict(pulse_len=1, bt=0.3),
                               dict(pulse_kind=1, pulse_len=3, sps=5), dict(bt=0.05, pulse_len=2)])
def test_pulse_identical_to_reference(cyc, ref, p):
    """Gaussian / rect frequency pulse with the exact half-area renormalisation."""
    f, g = cyc.cpm_pulse(cyc.CpmParams(**p))
    rf, rg = ref.pulse(**p)
    assert np.array_equal(f, rf) and np.array_equal(g, rg)
    assert g[-1] == 0.5


def test_parameter_guards_match_reference(cyc):
    """check_params (siggen.cpp:21-29) and the oracle's argument guards
    (reference.cpp:39-51): same messages, raised before any device work."""
    cases = [(dict(h=0.0), "modulation index must be positive"),
             (dict(alphabet_size=3), "alphabet size must be even and at least 2"),
             (dict(pulse_len=0), "pulse length must be at least 1 symbol"),
             (dict(sps=0), "samples per symbol must be at least 1"),
             (dict(bt=0.0), "bandwidth-time product must be positive")]
    for kw, msg in cases:
        with pytest.raises(cyc.UsageError, match=msg):
            cyc.cpm_pulse(cyc.CpmParams(**kw))
    with pytest.raises(cyc.UsageError, match="alphabet size"):
        cyc.random_symbols(3, 4, 1)
    with pytest.raises(cyc.UsageError, match="at least one cycle frequency and one lag"):
        cyc.gmsk_mc_oracle(None, [], [0], False, 256, 1, 1100, 1)
    with pytest.raises(cyc.UsageError, match="at least one cycle frequency and one lag"):
        cyc.gmsk_mc_oracle(None, [0.1], [], False, 256, 1, 1100, 1)
    with pytest.raises(cyc.UsageError, match="at least one trial"):
        cyc.gmsk_mc_oracle(None, [0.1], [0], False, 256, 0, 1100, 1)
    with pytest.raises(cyc.UsageError, match="window length must be at least 1"):
        cyc.gmsk_mc_oracle(None, [0.1], [0], False, 0, 1, 1100, 1)
    with pytest.raises(cyc.UsageError, match="record too short"):
        cyc.gmsk_mc_oracle(None, [0.1], [-4, 4], False, 256, 1, 263, 1)


# ---- GPU: modulation and the Monte-Carlo table ----

@pytest.mark.gpu
@pytest.mark.parametrize("p", [dict(), dict(h=0.7, bt=0.3), dict(alphabet_size=4, h=0.25, sps=5),
                               dict(pulse_kind=1, pulse_len=1)])
def test_cpm_modulate_matches_reference(cyc, ref, p):
    """Device CPM against the reference's sequential phase recursion: fp64
    output to ~1e-10 (phase of a 2^14-symbol record), cf32 to float rounding."""
    syms = ref.random_symbols(p.get("alphabet_size", 2), 1 << 14, 99)
    want = ref.cpm_modulate(syms, **p)
    got64 = cyc.cpm_modulate(cyc.CpmParams(**p), syms, f64=True)
    assert np.max(np.abs(got64 - want)) <= 1e-9
    got32 = cyc.cpm_modulate(cyc.CpmParams(**p), syms)
    assert got32.dtype == np.complex64 and np.max(np.abs(got32 - want)) <= 2e-7


@pytest.mark.gpu
def test_cpm_modulate_symbol_errors(cyc):
    with pytest.raises(cyc.DataError, match="symbol 3 at index 2 is outside the size-2 alphabet"):
        cyc.cpm_modulate(None, [1, -1, 3])
    with pytest.raises(cyc.UsageError, match="empty symbol stream"):
        cyc.cpm_modulate(None, [])


@pytest.mark.gpu
def test_cpm_modulate_into_device_memory(cyc):
    import torch
    syms = cyc.random_symbols(2, 512, 5)
    dev = torch.empty(512 * 8, dtype=torch.complex64, device="cuda")
    cyc.cpm_modulate(None, syms, out=dev)
    assert np.array_equal(dev.cpu().numpy(), cyc.cpm_modulate(None, syms))


@pytest.mark.gpu
def test_mc_oracle_matches_reference_and_is_reproducible(cyc, ref):
    """test_reference.cpp:117-145: shape, determinism, trial extendability --
    and the values against the reference's table (north-star tolerance)."""
    alphas, lags = [0.125, 0.0], [-4, -1, 0, 2]
    t = cyc.gmsk_mc_oracle(None, alphas, lags, False, 256, 3, 1100, 42)
    assert t.mean_magnitude.shape == (8,) and t.trials == 3 and t.record_len == 1100 and t.seed == 42
    assert np.all(np.isfinite(t.mean_magnitude)) and np.all(t.mean_magnitude >= 0)
    want = ref.gmsk_mc_oracle(alphas, lags, False, 256, 3, 1100, 42).reshape(-1)
    assert np.max(np.abs(t.mean_magnitude - want)) <= 1e-5  # mean power of CPM is 1
    assert np.linalg.norm(t.mean_magnitude - want) <= 1e-4 * np.linalg.norm(want)
    again = cyc.gmsk_mc_oracle(None, alphas, lags, False, 256, 3, 1100, 42)
    assert np.array_equal(t.mean_magnitude, again.mean_magnitude)
    one_a = cyc.gmsk_mc_oracle(None, alphas, lags, False, 256, 1, 1100, 42)
    one_b = cyc.gmsk_mc_oracle(None, alphas, lags, False, 256, 1, 1100, 43)
    two = cyc.gmsk_mc_oracle(None, alphas, lags, False, 256, 2, 1100, 42)
    np.testing.assert_allclose(two.mean_magnitude, 0.5 * (one_a.mean_magnitude + one_b.mean_magnitude),
                               rtol=1e-14, atol=1e-16)


@pytest.mark.gpu
def test_mc_oracle_features_like_reference(cyc, ref):
    """test_reference.cpp:147-190: symbol-rate feature vs an off-cycle probe,
    conjugate feature at h = 1/2 and its absence at h = 0.7; each table
    equal to the reference's."""
    n, record = 4096, 2 * 4096 + 32
    lags = list(range(-16, 17))
    sps = 8
    t = cyc.gmsk_mc_oracle(None, [1.0 / sps, 0.11], lags, False, n, 4, record, 7)
    w = ref.gmsk_mc_oracle([1.0 / sps, 0.11], lags, False, n, 4, record, 7)
    np.testing.assert_allclose(t.mean_magnitude.reshape(2, -1), w, rtol=0, atol=1e-5)
    tab = t.mean_magnitude.reshape(2, -1)
    assert tab[0].max() >= 4.0 * tab[1].max()
    beta = 1.0 / (2 * sps)
    on = cyc.gmsk_mc_oracle(None, [beta, 0.05], lags, True, n, 4, record, 11)
    np.testing.assert_allclose(on.mean_magnitude.reshape(2, -1),
                               ref.gmsk_mc_oracle([beta, 0.05], lags, True, n, 4, record, 11), rtol=0, atol=1e-5)
    on_t = on.mean_magnitude.reshape(2, -1)
    assert on_t[0].max() >= 4.0 * on_t[1].max()
    off = cyc.gmsk_mc_oracle(cyc.CpmParams(h=0.7), [beta], lags, True, n, 4, record, 11)
    np.testing.assert_allclose(off.mean_magnitude, ref.gmsk_mc_oracle([beta], lags, True, n, 4, record, 11, h=0.7)
                               .reshape(-1), rtol=0, atol=1e-5)
    assert off.mean_magnitude.max() <= 0.2 * on_t[0].max()

"""Seeded synthetic inputs for the BASELINE.json configurations (harness only).

The paper's over-the-air captures are not available, so every config is fed
seeded synthetic complex64 records with the stated modulation, rate, carrier
offset and SNR.  GMSK follows the reference's CPM conventions (h = 1/2,
binary, Gaussian frequency pulse over L = 4 symbols normalised to area 1/2,
proj/src/siggen.cpp:79-145); PSK-RRC is new (the reference has none, SURVEY
§0).  Generation is vectorised numpy; parity never depends on it because the
oracle and the GPU consume the same cf32 record.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erfc
from scipy.signal import fftconvolve


def rrc_taps(sps: int, rolloff: float, span: int = 8) -> np.ndarray:
    """Unit-energy root-raised-cosine taps over +-span symbols."""
    t = np.arange(-span * sps, span * sps + 1) / sps
    b = rolloff
    h = np.empty_like(t)
    for i, ti in enumerate(t):
        if abs(ti) < 1e-12:
            h[i] = 1 - b + 4 * b / math.pi
        elif b > 0 and abs(abs(ti) - 1 / (4 * b)) < 1e-9:
            h[i] = b / math.sqrt(2) * ((1 + 2 / math.pi) * math.sin(math.pi / (4 * b))
                                       + (1 - 2 / math.pi) * math.cos(math.pi / (4 * b)))
        else:
            h[i] = (math.sin(math.pi * ti * (1 - b)) + 4 * b * ti * math.cos(math.pi * ti * (1 + b))) / (
                math.pi * ti * (1 - (4 * b * ti) ** 2))
    return h / np.sqrt(np.sum(h ** 2))


def _carrier(n: int, fc: float) -> np.ndarray:
    idx = np.arange(n, dtype=np.float64)
    return np.exp(2j * np.pi * np.fmod(fc * idx, 1.0))


def _awgn(x: np.ndarray, snr_db: float, rng) -> np.ndarray:
    p = float(np.mean(np.abs(x) ** 2))
    sigma = math.sqrt(p * 10 ** (-snr_db / 10) / 2)
    return x + sigma * (rng.standard_normal(len(x)) + 1j * rng.standard_normal(len(x)))


def psk_rrc(n: int, order: int, sps: int, rolloff: float, fc: float, seed: int) -> np.ndarray:
    """BPSK (order 2) / QPSK (order 4) with RRC shaping at `sps`, carrier `fc`."""
    rng = np.random.default_rng(seed)
    nsym = n // sps + 32
    if order == 2:
        sym = rng.integers(0, 2, nsym) * 2.0 - 1.0
    else:
        sym = ((rng.integers(0, 2, nsym) * 2 - 1) + 1j * (rng.integers(0, 2, nsym) * 2 - 1)) / math.sqrt(2)
    up = np.zeros(nsym * sps, dtype=np.complex128)
    up[::sps] = sym
    x = fftconvolve(up, rrc_taps(sps, rolloff))[8 * sps: 8 * sps + n]
    return x * _carrier(n, fc)


def gmsk_pulse(bt: float, L: int, sps: int) -> np.ndarray:
    """Gaussian frequency pulse, midpoint-sampled, area 1/2 (proj/src/siggen.cpp:79-94)."""
    c = 2 * math.pi * bt / math.sqrt(math.log(2))
    tau = (np.arange(L * sps) + 0.5) / sps
    q = lambda v: 0.5 * erfc(v / math.sqrt(2))
    f = 0.5 * (q(c * (tau - L / 2 - 0.5)) - q(c * (tau - L / 2 + 0.5))) / sps
    return f * (0.5 / f.sum())


def gmsk(n: int, bt: float, sps: int, fc: float, seed: int, h: float = 0.5, L: int = 4) -> np.ndarray:
    """Binary CPM with a Gaussian pulse (GMSK), initial phase 0, carrier `fc`."""
    rng = np.random.default_rng(seed)
    nsym = n // sps + L + 2
    a = rng.integers(0, 2, nsym) * 2.0 - 1.0
    up = np.zeros(nsym * sps)
    up[::sps] = a
    freq = fftconvolve(up, gmsk_pulse(bt, L, sps))[:n]
    phase = 2 * math.pi * h * np.cumsum(freq)
    return np.exp(1j * np.fmod(phase, 2 * math.pi)) * _carrier(n, fc)


def c1_record(seed: int = 1, n: int = 1 << 20) -> np.ndarray:
    """Config 1: GMSK BT 0.3, 8 sps, f_c 0.05, 10 dB."""
    rng = np.random.default_rng(seed + 1)
    return _awgn(gmsk(n, 0.3, 8, 0.05, seed), 10.0, rng).astype(np.complex64)


def c2_record(seed: int = 2, n: int = 1 << 24) -> np.ndarray:
    """Config 2: QPSK RRC(0.35), 4 sps, f_c 0.1, 5 dB."""
    rng = np.random.default_rng(seed + 1)
    return _awgn(psk_rrc(n, 4, 4, 0.35, 0.1, seed), 5.0, rng).astype(np.complex64)


def c3_record(seed: int = 3, n: int = 1 << 28, chunk: int = 1 << 22):
    """Config 3: GMSK BT 0.3, 8 sps, f_c 0.02, 0 dB (generated in chunks, same record)."""
    x = gmsk(n, 0.3, 8, 0.02, seed)
    rng = np.random.default_rng(seed + 1)
    return _awgn(x, 0.0, rng).astype(np.complex64)


def c4_channel(c: int, n: int = 1 << 22, seed: int = 4) -> np.ndarray:
    """Config 4 channel c: cycles BPSK-RRC, QPSK-RRC, GMSK, noise; per-channel draws."""
    rng = np.random.default_rng(seed * 1000 + c)
    kind = c % 4
    fc = rng.uniform(-0.2, 0.2)
    snr = rng.uniform(-5, 15)
    s = seed * 1000 + c + 7
    if kind == 0:
        x = psk_rrc(n, 2, int(rng.integers(2, 17)), rng.uniform(0.25, 0.5), fc, s)
    elif kind == 1:
        x = psk_rrc(n, 4, int(rng.integers(2, 17)), rng.uniform(0.25, 0.5), fc, s)
    elif kind == 2:
        x = gmsk(n, rng.uniform(0.25, 0.5), 8, fc, s)
    else:
        return ((rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)).astype(np.complex64)
    return _awgn(x, snr, rng).astype(np.complex64)


def c5_record(seed: int = 5, n: int = 1 << 26) -> np.ndarray:
    """Config 5: BPSK-RRC(0.35, 5 sps, f_c 0.07) + GMSK(BT 0.3, 8 sps, f_c -0.11) at -6 dB, AWGN 3 dB."""
    s1 = psk_rrc(n, 2, 5, 0.35, 0.07, seed)
    s2 = gmsk(n, 0.3, 8, -0.11, seed + 10)
    p1 = np.mean(np.abs(s1) ** 2)
    x = s1 + s2 * math.sqrt(p1 * 10 ** (-6 / 10))
    return _awgn(x, 3.0, np.random.default_rng(seed + 1)).astype(np.complex64)

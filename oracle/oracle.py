"""ctypes front-end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker (or the timed
CPU baseline).  The product package never imports it.

Two libraries:
  * ``_build/libcycoracle.so`` -- the plain-C restatement in cycoracle.c;
  * ``_ref/libcycstat_ref.so`` -- the unmodified reference (/root/reference/proj)
    compiled from its own sources by oracle/Makefile, behind ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcycoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcycstat_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_szp = C.POINTER(C.c_size_t)
_u64p = C.POINTER(C.c_uint64)


def build() -> None:
    """Compile the oracle (and the reference library when its sources exist)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _cd(a: np.ndarray) -> np.ndarray:
    """complex -> contiguous interleaved float64 view."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def _cf(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex64)
    return a.view(np.float32)


def _p(a, t):
    return a.ctypes.data_as(t)


class Oracle:
    """The C restatement (cycoracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_direct.argtypes = [_dp, _dp, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                 C.c_size_t, C.c_int, _dp]
        L.orc_fft.argtypes = [_dp, _dp, C.c_size_t]
        L.orc_stream.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int, _ip,
                                 C.c_size_t, _dp, _dp, C.c_size_t, _dp, _szp, _szp]
        L.orc_block_direct.argtypes = [_dp, _dp, C.c_size_t, _dp, C.c_size_t, _ip, C.c_size_t,
                                       C.c_int, C.c_size_t, C.c_size_t, _dp]
        L.orc_block_fold.argtypes = [_fp, _fp, C.c_size_t, _i64p, C.c_size_t, C.c_int64, _ip,
                                     C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp]
        L.orc_recursive.argtypes = [_dp, _dp, C.c_size_t, _dp, C.c_size_t, _ip, C.c_size_t,
                                    C.c_int, C.c_double, C.c_size_t, _dp, _szp]
        self.lib = L

    def direct(self, x, y, alpha, m, conj, k0, n_win) -> complex:
        xd, yd = _cd(x), _cd(y)
        out = np.zeros(2)
        rc = self.lib.orc_direct(_p(xd, _dp), _p(yd, _dp), len(x), alpha, m, int(conj), k0,
                                 n_win, _p(out, _dp))
        if rc:
            raise ValueError("window not covered")
        return complex(out[0], out[1])

    def fft(self, v) -> np.ndarray:
        vd = _cd(v)
        out = np.zeros(2 * len(v))
        self.lib.orc_fft(_p(vd, _dp), _p(out, _dp), len(v))
        return out.view(np.complex128)

    def stream(self, mode, conj, win_len, x, y, alphas=(), max_lag=0, lags=()):
        """All frames of the record: (F, layout_len) complex array."""
        xd, yd = _cd(x), _cd(y)
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        nf, lay = C.c_size_t(), C.c_size_t()
        args = [int(mode), int(conj), int(win_len), _p(al, _dp), len(al), int(max_lag),
                _p(lg, _ip), len(lg), _p(xd, _dp), _p(yd, _dp), len(x)]
        if self.lib.orc_stream(*args, None, C.byref(nf), C.byref(lay)):
            raise ValueError("invalid config")
        out = np.zeros(2 * nf.value * lay.value)
        self.lib.orc_stream(*args, _p(out, _dp), C.byref(nf), C.byref(lay))
        return out.view(np.complex128).reshape(nf.value, lay.value)

    def block_direct(self, x, y, alphas, lags, conj, start, count) -> np.ndarray:
        xd, yd = _cd(x), _cd(y)
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        out = np.zeros(2 * len(al) * len(lg))
        rc = self.lib.orc_block_direct(_p(xd, _dp), _p(yd, _dp), len(x), _p(al, _dp), len(al),
                                       _p(lg, _ip), len(lg), int(conj), start, count,
                                       _p(out, _dp))
        if rc:
            raise ValueError("block not covered")
        return out.view(np.complex128).reshape(len(al), len(lg))

    def block_fold(self, x, y, k, P, lags, start, count):
        """(conv, conj) tables, alpha-major, for alphas k/P (cf32 inputs)."""
        xf, yf = _cf(x), _cf(y)
        kk = np.ascontiguousarray(k, dtype=np.int64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        o1 = np.zeros(2 * len(kk) * len(lg))
        o2 = np.zeros(2 * len(kk) * len(lg))
        rc = self.lib.orc_block_fold(_p(xf, _fp), _p(yf, _fp), len(x), _p(kk, _i64p), len(kk),
                                     int(P), _p(lg, _ip), len(lg), start, count,
                                     _p(o1, _dp), _p(o2, _dp))
        if rc:
            raise ValueError("block not covered")
        sh = (len(kk), len(lg))
        return o1.view(np.complex128).reshape(sh), o2.view(np.complex128).reshape(sh)

    def recursive(self, x, y, alphas, lags, conj, lam, emit_every) -> np.ndarray:
        xd, yd = _cd(x), _cd(y)
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        ne = C.c_size_t()
        args = [_p(xd, _dp), _p(yd, _dp), len(x), _p(al, _dp), len(al), _p(lg, _ip), len(lg),
                int(conj), float(lam), int(emit_every)]
        self.lib.orc_recursive(*args, None, C.byref(ne))
        out = np.zeros(2 * ne.value * len(al) * len(lg))
        self.lib.orc_recursive(*args, _p(out, _dp), C.byref(ne))
        return out.view(np.complex128).reshape(ne.value, len(al), len(lg))


class RefLib:
    """The reference library itself, compiled by oracle/Makefile into oracle/_ref/."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_direct.argtypes = [_dp, _dp, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                 C.c_size_t, C.c_int, _dp]
        L.ref_fft.argtypes = [_dp, _dp, C.c_size_t]
        L.ref_stream.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int, _ip,
                                 C.c_size_t, _dp, _dp, C.c_size_t, C.c_size_t, _dp, _u64p,
                                 _szp, _szp]
        L.ref_block_average.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int,
                                        _ip, C.c_size_t, _fp, _fp, C.c_size_t, C.c_size_t,
                                        _dp, _szp]
        L.ref_validate.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int, C.c_int,
                                   _ip, C.c_size_t, C.c_char_p, C.c_size_t]
        L.ref_gmsk.argtypes = [C.c_size_t, C.c_double, C.c_int, C.c_uint64, _dp]
        L.ref_tone.argtypes = [C.c_double, C.c_double, C.c_size_t, _dp]
        L.ref_awgn.argtypes = [C.c_size_t, C.c_double, C.c_uint64, _dp]
        L.ref_apply_cfo.argtypes = [_dp, C.c_size_t, C.c_double, C.c_double]
        L.ref_add_noise_snr.argtypes = [_dp, C.c_size_t, C.c_double, C.c_uint64]
        L.ref_cpm.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_int, C.c_uint64, _dp]
        _cpm = [C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        L.ref_random_symbols.argtypes = [C.c_int, C.c_size_t, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_pulse.argtypes = _cpm + [_dp, _dp]
        L.ref_cpm_modulate.argtypes = _cpm + [C.POINTER(C.c_int), C.c_size_t, _dp]
        L.ref_gmsk_mc_oracle.argtypes = _cpm + [_dp, C.c_size_t, C.POINTER(C.c_int), C.c_size_t, C.c_int, C.c_int,
                                                C.c_int, C.c_size_t, C.c_uint64, _dp]
        L.ref_estimate_cfo_ccf.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, _dp]
        self.has_io = hasattr(L, "ref_export_frames_csv")  # io.cpp built (needs a json.hpp)
        if self.has_io:
            L.ref_export_frames_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int, _ip,
                                                C.c_size_t, _dp, _u64p, C.c_size_t, _szp]
            L.ref_export_average_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_size_t, C.c_int, _ip,
                                                 C.c_size_t, _dp, C.c_size_t, C.c_int, _szp]
        self.lib = L

    def cpm(self, n, h=0.5, bt=0.25, sps=8, seed=0):
        out = np.zeros(2 * n)
        self._err(self.lib.ref_cpm(n, h, bt, sps, seed, _p(out, _dp)))
        return out.view(np.complex128)

    @staticmethod
    def _cpm_args(p):
        return [float(p.get("h", 0.5)), int(p.get("alphabet_size", 2)), int(p.get("pulse_len", 4)),
                float(p.get("bt", 0.25)), int(p.get("sps", 8)), int(p.get("pulse_kind", 0))]

    def random_symbols(self, M, count, seed):
        out = np.zeros(count, dtype=np.int32)
        self._err(self.lib.ref_random_symbols(M, count, seed, out.ctypes.data_as(C.POINTER(C.c_int))))
        return out

    def pulse(self, **p):
        a = self._cpm_args(p)
        n = a[2] * a[4]
        f, g = np.zeros(n), np.zeros(n)
        self._err(self.lib.ref_pulse(*a, _p(f, _dp), _p(g, _dp)))
        return f, g

    def cpm_modulate(self, symbols, **p):
        sym = np.ascontiguousarray(symbols, dtype=np.int32)
        out = np.zeros(2 * len(sym) * int(p.get("sps", 8)))
        rc = self.lib.ref_cpm_modulate(*self._cpm_args(p), sym.ctypes.data_as(C.POINTER(C.c_int)), len(sym),
                                       _p(out, _dp))
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return out.view(np.complex128)

    def gmsk_mc_oracle(self, alphas, lags, conj, win_len, trials, record_len, seed, **p):
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        out = np.zeros(len(al) * len(lg))
        rc = self.lib.ref_gmsk_mc_oracle(*self._cpm_args(p), _p(al, _dp), len(al),
                                         lg.ctypes.data_as(C.POINTER(C.c_int)), len(lg), int(conj), int(win_len),
                                         int(trials), int(record_len), int(seed), _p(out, _dp))
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return out.reshape(len(al), len(lg))

    def estimate_cfo_ccf(self, x, beta, N, frames):
        """eps, or raises LookupError for NoFeatureError / ValueError for UsageError."""
        xd = _cd(x)
        eps = C.c_double()
        rc = self.lib.ref_estimate_cfo_ccf(_p(xd, _dp), len(x), beta, N, frames, C.byref(eps))
        if rc == 4:
            raise LookupError(self.lib.ref_last_error().decode())
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return eps.value

    def export_frames_csv(self, path, mode, win_len, frames, indices, alphas=(), max_lag=0, lags=()):
        """io.cpp:161-186 (the reference's writer) on the given frame values."""
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        v = _cd(np.asarray(frames).reshape(-1))
        ix = np.ascontiguousarray(indices, dtype=np.uint64)
        rows = C.c_size_t()
        self._err(self.lib.ref_export_frames_csv(os.fsencode(path), int(mode), int(win_len), _p(al, _dp), len(al),
                                                 int(max_lag), _p(lg, _ip), len(lg), _p(v, _dp), _p(ix, _u64p),
                                                 len(ix), C.byref(rows)))
        return rows.value

    def export_average_csv(self, path, mode, win_len, avg, magnitude, alphas=(), max_lag=0, lags=()):
        """io.cpp:188-208 (the reference's writer)."""
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        v = _cd(np.asarray(avg).reshape(-1))
        rows = C.c_size_t()
        self._err(self.lib.ref_export_average_csv(os.fsencode(path), int(mode), int(win_len), _p(al, _dp), len(al),
                                                  int(max_lag), _p(lg, _ip), len(lg), _p(v, _dp), len(v) // 2,
                                                  int(magnitude), C.byref(rows)))
        return rows.value

    def _err(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def direct(self, x, y, alpha, m, conj, k0, n_win) -> complex:
        xd, yd = _cd(x), _cd(y)
        out = np.zeros(2)
        self._err(self.lib.ref_direct(_p(xd, _dp), _p(yd, _dp), len(x), alpha, m, int(conj),
                                      k0, n_win, _p(out, _dp)))
        return complex(out[0], out[1])

    def fft(self, v):
        vd = _cd(v)
        out = np.zeros(2 * len(v))
        self._err(self.lib.ref_fft(_p(vd, _dp), _p(out, _dp), len(v)))
        return out.view(np.complex128)

    def stream(self, mode, conj, win_len, x, y, alphas=(), max_lag=0, lags=(), chunk=0):
        """(frames (F, layout_len), start_abs (F,)) from CyclicCorrelator::push."""
        xd, yd = _cd(x), _cd(y)
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        nf, lay = C.c_size_t(), C.c_size_t()
        args = [int(mode), int(conj), int(win_len), _p(al, _dp), len(al), int(max_lag),
                _p(lg, _ip), len(lg), _p(xd, _dp), _p(yd, _dp), len(x), int(chunk)]
        self._err(self.lib.ref_stream(*args, None, None, C.byref(nf), C.byref(lay)))
        out = np.zeros(2 * nf.value * lay.value)
        st = np.zeros(nf.value, dtype=np.uint64)
        self._err(self.lib.ref_stream(*args, _p(out, _dp), _p(st, _u64p), C.byref(nf),
                                      C.byref(lay)))
        return out.view(np.complex128).reshape(nf.value, lay.value), st

    def block_average(self, mode, conj, win_len, x, y, alphas=(), max_lag=0, lags=(),
                      max_frames=0):
        """Coherent average_frames over the record (N-sized pushes), and F."""
        xf, yf = _cf(x), _cf(y)
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        lay = len(al) * (2 * max_lag + 1) if mode == 0 else len(lg) * win_len
        out = np.zeros(2 * lay)
        nf = C.c_size_t()
        self._err(self.lib.ref_block_average(int(mode), int(conj), int(win_len), _p(al, _dp),
                                             len(al), int(max_lag), _p(lg, _ip), len(lg),
                                             _p(xf, _fp), _p(yf, _fp), len(x), int(max_frames),
                                             _p(out, _dp), C.byref(nf)))
        return out.view(np.complex128), nf.value

    def validate(self, mode, win_len, alphas=(), lag_symmetric=True, max_lag=0, lags=()):
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lg = np.ascontiguousarray(lags, dtype=np.int32)
        buf = C.create_string_buffer(4096)
        n = self.lib.ref_validate(int(mode), 0, int(win_len), _p(al, _dp), len(al),
                                  int(lag_symmetric), int(max_lag), _p(lg, _ip), len(lg), buf,
                                  4096)
        return [s for s in buf.value.decode().split("\n") if s][:n]

    def gmsk(self, n, bt=0.25, sps=8, seed=0):
        out = np.zeros(2 * n)
        self._err(self.lib.ref_gmsk(n, bt, sps, seed, _p(out, _dp)))
        return out.view(np.complex128)

    def tone(self, f0, phi0, n):
        out = np.zeros(2 * n)
        self.lib.ref_tone(f0, phi0, n, _p(out, _dp))
        return out.view(np.complex128)

    def awgn(self, n, sigma, seed):
        out = np.zeros(2 * n)
        self._err(self.lib.ref_awgn(n, sigma, seed, _p(out, _dp)))
        return out.view(np.complex128)

    def apply_cfo(self, x, eps, phi0=0.0):
        xd = _cd(np.array(x, dtype=np.complex128))
        self._err(self.lib.ref_apply_cfo(_p(xd, _dp), len(x), eps, phi0))
        return xd.view(np.complex128)

    def add_noise_snr(self, x, snr_db, seed):
        xd = _cd(np.array(x, dtype=np.complex128))
        self._err(self.lib.ref_add_noise_snr(_p(xd, _dp), len(x), snr_db, seed))
        return xd.view(np.complex128)


def have_ref() -> bool:
    return os.path.exists(REF_SO)

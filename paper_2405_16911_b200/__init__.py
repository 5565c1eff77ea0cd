"""B200-native cyclic-ACF estimator -- Python mirror of the reference interface.

The product is ``libcycb200.so`` (CUDA kernels for sm_100a behind the C-ABI in
``include/cycb200.h``).  This module binds it with ctypes and restates the
reference's public names so callers and parity tests read like the
reference's own (``/root/reference/proj/include/cycstat``):

    Mode, LagSpec, EstimatorConfig, validate_config      types.hpp:22-66
    SetLayout, FullLayout, layout_len, flat_index,
    full_bin_to_alpha                                     types.hpp:68-94
    CyclicFrame                                           types.hpp:97-104
    CyclicCorrelator(cfg).push(x, y) -> [CyclicFrame]     estimator.hpp:97-137
    AverageMode, average_frames                           estimator.hpp:143-148
    compute_set_window, compute_full_window               estimator.hpp:59-68
    UsageError, ConfigError, DataError                    errors.hpp:13-42

There is no CPU fallback: importing works without a GPU, but every compute
call goes through the CUDA library and fails loudly if it is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CYC_LIB", os.path.join(HERE, "libcycb200.so"))  # CYC_LIB: diagnostic builds only

__all__ = [
    "Mode", "Flags", "AverageMode", "LagSpec", "EstimatorConfig", "SetLayout", "FullLayout",
    "CyclicFrame", "CyclicCorrelator", "validate_config", "layout_len", "flat_index",
    "full_bin_to_alpha", "average_frames", "compute_set_window", "compute_full_window",
    "UsageError", "ConfigError", "DataError", "CudaError", "LogicError", "lib", "host_alloc",
    "NoFeatureError", "IoError", "FormatError", "export_frames_csv", "export_average_csv", "estimate_cfo_ccf", "write_cf32", "PulseKind", "CpmParams", "OracleTable",
    "random_symbols", "cpm_pulse", "cpm_modulate", "gmsk_mc_oracle",
]


# ---------------------------------------------------------------------------
# errors (proj/include/cycstat/errors.hpp)
# ---------------------------------------------------------------------------
class UsageError(RuntimeError):
    """errors.hpp:13-15"""


class ConfigError(UsageError):
    """errors.hpp:17-30: carries every violation."""

    def __init__(self, violations: Sequence[str], message: Optional[str] = None):
        self.violations = list(violations)
        super().__init__(message or ("invalid config:" + "".join(f" [{v}]" for v in self.violations)))


class DataError(RuntimeError):
    """errors.hpp:40-42: non-finite input; `index` is the absolute sample index."""

    def __init__(self, message: str, index: int = -1):
        super().__init__(message)
        self.index = index


class NoFeatureError(DataError):
    """errors.hpp:44-46: estimate_cfo_ccf found no conjugate feature."""


class IoError(RuntimeError):
    """errors.hpp:32-34: an unreadable input file."""


class FormatError(IoError):
    """errors.hpp:36-38: a malformed input file (e.g. a truncated cf32 record)."""


class CudaError(RuntimeError):
    """Device failure -- there is no CPU fallback."""


class LogicError(RuntimeError):
    """std::logic_error: kernel contract violations (kernels.cpp:16-17, 29-30, 119-120)."""


# ---------------------------------------------------------------------------
# C-ABI binding
# ---------------------------------------------------------------------------
class _Config(C.Structure):
    _fields_ = [
        ("mode", C.c_int), ("conj", C.c_int), ("flags", C.c_int), ("win_len", C.c_int),
        ("alphas", C.POINTER(C.c_double)), ("num_alphas", C.c_size_t),
        ("lag_symmetric", C.c_int), ("max_lag", C.c_int),
        ("lags", C.POINTER(C.c_int)), ("num_lags", C.c_size_t),
        ("lam", C.c_double), ("emit_frames", C.c_int), ("channels", C.c_int), ("device", C.c_int),
        ("origin", C.c_int64),
    ]


class _FrameView(C.Structure):
    _fields_ = [
        ("frame_index", C.c_uint64), ("start_abs", C.c_uint64), ("flag", C.c_int),
        ("channel", C.c_int), ("len", C.c_size_t), ("values", C.POINTER(C.c_double)),
    ]


class _LayoutInfo(C.Structure):
    _fields_ = [("kind", C.c_int), ("num_alphas", C.c_int), ("max_lag", C.c_int),
                ("num_lags", C.c_int), ("win_len", C.c_int), ("len", C.c_size_t)]


class _CpmParams(C.Structure):
    _fields_ = [("h", C.c_double), ("alphabet_size", C.c_int), ("pulse_len", C.c_int), ("bt", C.c_double),
                ("sps", C.c_int), ("pulse_kind", C.c_int)]


_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(_FrameView))
_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libcycb200.so (built in-tree by paper_2405_16911_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_16911_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, sz = C.c_void_p, C.c_size_t
    L.cyc_config_init.argtypes = [C.POINTER(_Config)]
    L.cyc_validate.argtypes = [C.POINTER(_Config), C.c_char_p, sz]
    L.cyc_create.argtypes = [C.POINTER(_Config), C.POINTER(vp), C.c_char_p, sz]
    L.cyc_destroy.argtypes = [vp]
    for f in ("cyc_push", "cyc_push_f64", "cyc_push_device"):
        getattr(L, f).argtypes = [vp, vp, vp, sz, _SINK, vp]
    L.cyc_average.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
    L.cyc_buffer_need.argtypes = [vp]
    L.cyc_buffer_need.restype = sz
    L.cyc_consumed.argtypes = [vp]
    L.cyc_consumed.restype = C.c_uint64
    L.cyc_frames_emitted.argtypes = [vp]
    L.cyc_frames_emitted.restype = C.c_uint64
    L.cyc_layout.argtypes = [vp, C.POINTER(_LayoutInfo)]
    L.cyc_num_flags.argtypes = [vp]
    L.cyc_last_error.argtypes = [vp]
    L.cyc_last_error.restype = C.c_char_p
    L.cyc_data_error_index.argtypes = [vp]
    L.cyc_data_error_index.restype = C.c_int64
    L.cyc_synchronize.argtypes = [vp]
    L.cyc_stream.argtypes = [vp]
    L.cyc_stream.restype = vp
    L.cyc_kernel_launches.argtypes = [vp]
    L.cyc_kernel_launches.restype = C.c_uint64
    L.cyc_algorithm.argtypes = [vp, C.c_char_p, sz]
    L.cyc_host_alloc.argtypes = [sz]
    L.cyc_host_alloc.restype = vp
    L.cyc_host_free.argtypes = [vp]
    L.cyc_build_info.restype = C.c_char_p
    L.cyc_compute_set_window.argtypes = [vp, sz, vp, sz, vp, sz, C.c_int, C.c_int, C.c_uint64, vp,
                                         C.c_char_p, sz]
    L.cyc_plan.argtypes = [C.POINTER(_Config), C.c_char_p, sz]
    L.cyc_fold_state.argtypes = [vp, C.POINTER(vp), C.POINTER(sz), C.POINTER(C.c_uint64)]
    L.cyc_fold_set_frames.argtypes = [vp, C.c_uint64]
    L.cyc_set_lag_slice.argtypes = [vp, C.c_uint32, C.c_uint32]
    L.cyc_set_emit_pipeline.argtypes = [vp, C.c_int]
    L.cyc_flush_frames.argtypes = [vp, _SINK, vp]
    L.cyc_average_all.argtypes = [vp, C.c_int, vp]
    L.cyc_block_average_device.argtypes = [vp, vp, vp, C.c_size_t, C.c_int, vp]
    L.cyc_push_cf32_file.argtypes = [vp, C.c_char_p, _SINK, vp]
    L.cyc_estimate_cfo_ccf.argtypes = [vp, sz, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                       C.c_char_p, sz]
    L.cyc_reset.argtypes = [vp]
    L.cyc_cpm_params_init.argtypes = [C.POINTER(_CpmParams)]
    L.cyc_random_symbols.argtypes = [C.c_int, sz, C.c_uint64, C.POINTER(C.c_int), C.c_char_p, sz]
    L.cyc_cpm_pulse.argtypes = [C.POINTER(_CpmParams), C.POINTER(C.c_double), C.POINTER(C.c_double), sz,
                                C.c_char_p, sz]
    L.cyc_cpm_modulate.argtypes = [C.POINTER(_CpmParams), C.POINTER(C.c_int), sz, C.c_int, C.c_int, vp,
                                   C.c_char_p, sz]
    L.cyc_gmsk_mc_oracle.argtypes = [C.POINTER(_CpmParams), C.POINTER(C.c_double), sz, C.POINTER(C.c_int), sz,
                                     C.c_int, C.c_int, C.c_int, sz, C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                     C.c_char_p, sz]
    L.cyc_profile_enable.argtypes = [vp, C.c_int]
    L.cyc_profile_read.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.cyc_profile_read_ex.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    L.cyc_measure_fp32_peak.argtypes = [C.c_int]
    L.cyc_measure_fp32_peak.restype = C.c_double
    L.cyc_compute_full_window.argtypes = [vp, sz, vp, sz, vp, sz, C.c_int, C.c_uint64, vp, C.c_char_p, sz]
    L.cyc_export_frames_csv.argtypes = [C.POINTER(_Config), C.c_char_p, vp, vp, sz, C.POINTER(sz), C.c_char_p, sz]
    L.cyc_export_average_csv.argtypes = [C.POINTER(_Config), C.c_char_p, vp, sz, C.c_int, C.POINTER(sz), C.c_char_p,
                                         sz]
    _lib = L
    return L


def host_alloc(shape, dtype=np.complex64) -> np.ndarray:
    """Page-locked numpy array (freed with the array) for zero-staging pushes."""
    L = lib()
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    ptr = L.cyc_host_alloc(max(nbytes, 1))
    if not ptr:
        raise CudaError("cudaMallocHost failed")
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)

    class _Owner:
        def __del__(self_inner):
            try:
                L.cyc_host_free(ptr)
            except Exception:
                pass

    arr_owner = _Owner()
    arr = arr.view(_Pinned)
    arr._owner = arr_owner
    return arr


class _Pinned(np.ndarray):
    _owner = None

    def __array_finalize__(self, obj):
        if obj is not None:
            self._owner = getattr(obj, "_owner", None)


# ---------------------------------------------------------------------------
# types (proj/include/cycstat/types.hpp)
# ---------------------------------------------------------------------------
class Mode(enum.IntEnum):
    Set = 0
    Full = 1
    Recursive = 2  # extension: exponential forgetting


class Flags(enum.IntFlag):
    CONV = 1
    CONJ = 2
    BOTH = 3


class AverageMode(enum.IntEnum):
    Coherent = 0
    Magnitude = 1


@dataclass
class LagSpec:
    """types.hpp:29-53"""
    symmetric: bool = True
    max_lag: int = 0
    lags: list = field(default_factory=list)

    @staticmethod
    def Symmetric(m: int) -> "LagSpec":
        return LagSpec(True, int(m), [])

    @staticmethod
    def Explicit(lags: Sequence[int]) -> "LagSpec":
        return LagSpec(False, 0, [int(v) for v in lags])

    def m_plus(self) -> int:
        return self.max_lag if self.symmetric else max([0] + [l for l in self.lags])

    def m_minus(self) -> int:
        return self.max_lag if self.symmetric else max([0] + [-l for l in self.lags])

    def values(self) -> list:
        return list(range(-self.max_lag, self.max_lag + 1)) if self.symmetric else list(self.lags)


@dataclass
class EstimatorConfig:
    """types.hpp:55-63 plus the B200 extensions (flags, recursive, block mode, channels)."""
    mode: Mode = Mode.Set
    conj: bool = False
    win_len: int = 0
    alphas: list = field(default_factory=list)
    lag_spec: LagSpec = field(default_factory=LagSpec)
    flags: int = 0            # 0 => from conj; Flags.BOTH computes both tables in one pass
    lam: float = 0.0          # Recursive forgetting factor
    emit_frames: bool = True  # False: block mode (count + fold; read with average())
    channels: int = 1
    device: int = 0
    origin: int = 0           # absolute index of the first pushed sample (resume / time shards)

    def _c(self):
        c = _Config()
        lib().cyc_config_init(C.byref(c))
        al = np.ascontiguousarray(self.alphas, dtype=np.float64)
        lg = np.ascontiguousarray(self.lag_spec.lags, dtype=np.int32)
        c.mode, c.conj, c.flags, c.win_len = int(self.mode), int(bool(self.conj)), int(self.flags), int(self.win_len)
        c.alphas = al.ctypes.data_as(C.POINTER(C.c_double)) if al.size else None
        c.num_alphas = al.size
        c.lag_symmetric = int(self.lag_spec.symmetric)
        c.max_lag = int(self.lag_spec.max_lag)
        c.lags = lg.ctypes.data_as(C.POINTER(C.c_int)) if lg.size else None
        c.num_lags = lg.size
        c.lam = float(self.lam)
        c.emit_frames = int(bool(self.emit_frames))
        c.channels = int(self.channels)
        c.device = int(self.device)
        c.origin = int(self.origin)
        return c, (al, lg)


def plan(cfg: EstimatorConfig) -> str:
    """Algorithm the engine picks for cfg (host-only; no device needed)."""
    c, keep = cfg._c()
    buf = C.create_string_buffer(1024)
    rc = lib().cyc_plan(C.byref(c), buf, 1024)
    if rc:
        _raise(rc, buf.value.decode())
    return buf.value.decode()


def validate_config(cfg: EstimatorConfig) -> list:
    """types.cpp:30-63: every violated invariant; empty means ok."""
    c, keep = cfg._c()
    buf = C.create_string_buffer(8192)
    n = lib().cyc_validate(C.byref(c), buf, 8192)
    return [s for s in buf.value.decode().split("\n") if s][:n]


@dataclass(frozen=True)
class SetLayout:
    num_alphas: int
    max_lag: int


@dataclass(frozen=True)
class FullLayout:
    num_lags: int
    win_len: int


@dataclass(frozen=True)
class LagListLayout:
    """Recursive mode: alpha-major over an explicit lag list."""
    num_alphas: int
    num_lags: int


def layout_len(layout) -> int:
    if isinstance(layout, SetLayout):
        return layout.num_alphas * (2 * layout.max_lag + 1)
    if isinstance(layout, FullLayout):
        return layout.num_lags * layout.win_len
    return layout.num_alphas * layout.num_lags


def flat_index(layout, major: int, minor: int) -> int:
    """types.cpp:81-98"""
    if isinstance(layout, SetLayout):
        if not 0 <= major < layout.num_alphas:
            raise IndexError("cycle-frequency index out of range")
        if not -layout.max_lag <= minor <= layout.max_lag:
            raise IndexError("lag out of range")
        return major * (2 * layout.max_lag + 1) + minor + layout.max_lag
    if isinstance(layout, FullLayout):
        if not 0 <= major < layout.num_lags:
            raise IndexError("lag index out of range")
        if not 0 <= minor < layout.win_len:
            raise IndexError("DFT bin out of range")
        return major * layout.win_len + minor
    return major * layout.num_lags + minor


def full_bin_to_alpha(k: int, n: int) -> float:
    """types.cpp:100-104"""
    if n <= 0 or k < 0 or k >= n:
        raise IndexError("DFT bin out of range")
    a = k / n
    return a if 2 * k < n else a - 1.0


@dataclass
class CyclicFrame:
    """types.hpp:97-104 (+ flag/channel for the multi-table extensions)."""
    frame_index: int
    start_abs: int
    layout: object
    values: np.ndarray
    flag: int = 1
    channel: int = 0


def _raise(code: int, msg: str, index: int = -1):
    if code == 1:
        body = msg[len("invalid config:"):] if msg.startswith("invalid config:") else msg
        viol = [v.strip().strip("[]") for v in body.split("] [")] if body.strip() else []
        raise ConfigError(viol, msg)
    if code == 2:
        raise UsageError(msg)
    if code == 3:
        raise DataError(msg, index)
    if code == 4:
        raise CudaError(msg)
    if code == 6:
        raise IoError(msg)
    if code == 7:
        raise FormatError(msg)
    raise LogicError(msg)


def _as_c64(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.complex64:
        a = a.astype(np.complex64)
    return np.ascontiguousarray(a)


# ---------------------------------------------------------------------------
# the estimator (estimator.hpp:97-137)
# ---------------------------------------------------------------------------
class CyclicCorrelator:
    """Streaming cyclic (conjugate) cross-correlation estimator on the GPU.

    Same contract as the reference: push() appends a chunk pair and returns
    every frame that became computable; a non-finite sample rejects the whole
    chunk (DataError naming its absolute index) and leaves the state
    unchanged; the frame sequence is independent of chunk boundaries.
    """

    def __init__(self, cfg: EstimatorConfig):
        self._cfg = cfg
        L = lib()
        c, keep = cfg._c()
        h = C.c_void_p()
        err = C.create_string_buffer(8192)
        rc = L.cyc_create(C.byref(c), C.byref(h), err, 8192)
        if rc:
            _raise(rc, err.value.decode())
        self._h = h
        self._L = L
        li = _LayoutInfo()
        L.cyc_layout(h, C.byref(li))
        self._li = li
        if cfg.mode == Mode.Full:
            self._layout = FullLayout(li.num_lags, li.win_len)
        elif cfg.mode == Mode.Set:
            self._layout = SetLayout(li.num_alphas, li.max_lag)
        else:
            self._layout = LagListLayout(li.num_alphas, li.num_lags)
        self._frames: list = []
        self._sink = _SINK(self._on_frame)

    # -- reference accessors (estimator.hpp:109-115)
    def config(self) -> EstimatorConfig:
        return self._cfg

    def layout(self):
        return self._layout

    def buffer_need(self) -> int:
        return int(self._L.cyc_buffer_need(self._h))

    def consumed(self) -> int:
        return int(self._L.cyc_consumed(self._h))

    def frames_emitted(self) -> int:
        return int(self._L.cyc_frames_emitted(self._h))

    # -- instrumentation
    def kernel_launches(self) -> int:
        return int(self._L.cyc_kernel_launches(self._h))

    def algorithm(self) -> str:
        b = C.create_string_buffer(256)
        self._L.cyc_algorithm(self._h, b, 256)
        return b.value.decode()

    def stream(self) -> int:
        return int(self._L.cyc_stream(self._h) or 0)

    def synchronize(self):
        self._check(self._L.cyc_synchronize(self._h))

    def fold_state(self):
        """(device pointer, fp64 count, frames) of the block-mode fold accumulators."""
        p, n, f = C.c_void_p(), C.c_size_t(), C.c_uint64()
        self._check(self._L.cyc_fold_state(self._h, C.byref(p), C.byref(n), C.byref(f)))
        return int(p.value), int(n.value), int(f.value)

    def fold_set_frames(self, frames: int):
        self._check(self._L.cyc_fold_set_frames(self._h, int(frames)))

    def set_lag_slice(self, begin: int = 0, end: int = 0):
        """Block-mode coherent averages (average_all / block_average_device)
        finalize only the lags with index in [begin, end) of the lag list, the
        other rows of `out` untouched; (0, 0) restores every lag
        (cyc_set_lag_slice: multi-GPU lag slices, shard.exchange_lag_slices)."""
        self._check(self._L.cyc_set_lag_slice(self._h, int(begin), int(end)))

    def fold_tensor(self):
        """The block-mode fold state as a torch float64 CUDA tensor viewing the
        estimator's accumulators in place ([channels][t_pad][Pf][4]: xr*yr,
        xi*yr, xr*yi, xi*yi per absolute residue), for collectives."""
        import torch
        from .shard import DeviceArray
        p, n, _ = self.fold_state()
        return torch.as_tensor(DeviceArray(p, n), device=f"cuda:{self._cfg.device}")

    def reset(self):
        """Fresh stream state (same as constructing a new estimator with this config)."""
        self._check(self._L.cyc_reset(self._h))

    def profile(self, on: bool = True):
        self._L.cyc_profile_enable(self._h, int(on))

    def profile_read(self):
        """(fold launches, fold kernel ms, algorithmic fold flops) so far."""
        n, ms, fl = C.c_uint64(), C.c_double(), C.c_double()
        self._check(self._L.cyc_profile_read(self._h, C.byref(n), C.byref(ms), C.byref(fl)))
        return int(n.value), float(ms.value), float(fl.value)

    def profile_read_ex(self) -> dict:
        """profile_read plus executed flops and the tensor-core launch count."""
        n, ms, fl, ex, tc = C.c_uint64(), C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
        self._check(self._L.cyc_profile_read_ex(self._h, C.byref(n), C.byref(ms), C.byref(fl), C.byref(ex),
                                                C.byref(tc)))
        return {"launches": int(n.value), "ms": float(ms.value), "flops": float(fl.value),
                "exec_flops": float(ex.value), "tensor_launches": int(tc.value)}

    def _on_frame(self, user, view):
        v = view.contents
        vals = np.ctypeslib.as_array(v.values, shape=(2 * v.len,)).view(np.complex128).copy()
        self._frames.append(CyclicFrame(int(v.frame_index), int(v.start_abs), self._layout, vals,
                                        int(v.flag), int(v.channel)))
        return 0

    def _check(self, rc: int):
        if rc:
            _raise(rc, self._L.cyc_last_error(self._h).decode(), int(self._L.cyc_data_error_index(self._h)))

    def push(self, x, y=None) -> list:
        """estimator.hpp:102-107.  x, y: complex arrays of one chunk (shape
        (n,) or (channels, n)); y=None (or y is x) is the auto-correlation."""
        same = y is None or y is x
        cx = np.asarray(x)
        if cx.dtype == np.complex128:
            fn = self._L.cyc_push_f64
            xa = np.ascontiguousarray(cx)
            ya = None if same else np.ascontiguousarray(np.asarray(y, dtype=np.complex128))
        else:
            fn = self._L.cyc_push
            xa = _as_c64(cx)
            ya = None if same else _as_c64(y)
        if ya is not None and ya.shape != xa.shape:
            raise UsageError("x and y chunks must have equal length")
        n = xa.shape[-1] if xa.ndim else 0
        if xa.ndim == 2 and xa.shape[0] != self._cfg.channels:
            raise UsageError("chunk rows must equal the channel count")
        self._frames = []
        rc = fn(self._h, xa.ctypes.data, ya.ctypes.data if ya is not None else None, n, self._sink, None)
        self._check(rc)
        out, self._frames = self._frames, []
        return out

    def set_emit_pipeline(self, depth: int = 1):
        """Pipelined emission (cyc_set_emit_pipeline): with depth 1 or 2 a push that
        completes frames only enqueues them; a later push (or flush_frames)
        returns them, same order and values.  depth 0 restores the reference's
        synchronous push()."""
        self._check(self._L.cyc_set_emit_pipeline(self._h, int(depth)))

    def flush_frames(self) -> list:
        """The frame batch still in flight under pipelined emission, if any."""
        self._frames = []
        self._check(self._L.cyc_flush_frames(self._h, self._sink, None))
        out, self._frames = self._frames, []
        return out

    def push_file(self, path: str) -> list:
        """read_cf32 + push (io.cpp:90-103): the whole cf32 file as one chunk."""
        self._frames = []
        self._check(self._L.cyc_push_cf32_file(self._h, os.fsencode(path), self._sink, None))
        out, self._frames = self._frames, []
        return out

    def push_device(self, x_ptr: int, n: int, y_ptr: Optional[int] = None) -> list:
        """Push samples already resident in device memory (complex64).  Read
        after the caller's default-stream work; later default-stream work waits
        for the fold; returns once the chunk's finite check is known."""
        self._frames = []
        self._check(self._L.cyc_push_device(self._h, x_ptr, y_ptr, n, self._sink, None))
        out, self._frames = self._frames, []
        return out

    def average(self, mode: AverageMode = AverageMode.Coherent, flag: Optional[int] = None,
                channel: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
        """average_frames over every frame emitted so far (estimator.cpp:86-105).
        `out` (complex128, layout_len) may be passed to reuse a buffer."""
        n = layout_len(self._layout)
        cai = getattr(out, "__cuda_array_interface__", None)
        if cai is not None:  # device memory (block-mode coherent averages only)
            if int(np.prod(cai["shape"])) != n or cai["typestr"] != "<c16" or cai.get("strides") is not None:
                raise UsageError("device out must be a contiguous complex128 array of layout_len values")
            self._check(self._L.cyc_average(self._h, int(mode), int(flag or 0), int(channel), int(cai["data"][0])))
            return out
        if out is None:
            out = np.empty(n, dtype=np.complex128)
        elif out.dtype != np.complex128 or out.size != n or not out.flags.c_contiguous:
            raise UsageError("out must be a contiguous complex128 array of layout_len values")
        self._check(self._L.cyc_average(self._h, int(mode), int(flag or 0), int(channel), out.ctypes.data))
        return out

    def average_all(self, mode: AverageMode = AverageMode.Coherent, out: Optional[np.ndarray] = None):
        """All (channel, flag) tables: array [channels, flags, layout_len].
        `out` may also be a device array (`__cuda_array_interface__`, e.g. a
        torch complex128 CUDA tensor) for a block-mode coherent average; the
        table is written stream-ordered on `stream()`, and work later queued
        on the default stream (torch's) waits for it -- from other streams,
        call `synchronize()` first."""
        last = getattr(self, "_avg_dev_out", None)
        if last is not None and last[0] is out and (not hasattr(out, "data_ptr") or out.data_ptr() == last[1]):
            # the device table validated last time (same object, same storage)
            self._check(self._L.cyc_average_all(self._h, int(mode), last[1]))
            return out
        nf = int(self._L.cyc_num_flags(self._h))
        shape = (self._cfg.channels, nf, layout_len(self._layout))
        cai = getattr(out, "__cuda_array_interface__", None)
        if cai is not None:
            if tuple(cai["shape"]) != shape or cai["typestr"] not in ("<c16",) or cai.get("strides") not in (None,):
                raise UsageError(f"device out must be a contiguous complex128 array of shape {shape}")
            ptr = int(cai["data"][0])
            self._avg_dev_out = (out, ptr)
            self._check(self._L.cyc_average_all(self._h, int(mode), ptr))
            return out
        if out is None:
            out = np.empty(shape, dtype=np.complex128)
        elif out.shape != shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise UsageError(f"out must be a contiguous complex128 array of shape {shape}")
        self._check(self._L.cyc_average_all(self._h, int(mode), out.ctypes.data))
        return out

    def block_average_device(self, x_ptr: int, n: int, out, mode: AverageMode = AverageMode.Coherent,
                             y_ptr: Optional[int] = None):
        """reset + push_device(x_ptr, n) + average_all(out) with one host
        synchronisation (cyc_block_average_device): the block average of exactly
        this device chunk.  `out` as for average_all (a device array is written
        stream-ordered).  DataError leaves the reset state; `out` is then undefined."""
        nf = int(self._L.cyc_num_flags(self._h))
        shape = (self._cfg.channels, nf, layout_len(self._layout))
        cai = getattr(out, "__cuda_array_interface__", None)
        if cai is not None:
            if tuple(cai["shape"]) != shape or cai["typestr"] not in ("<c16",) or cai.get("strides") not in (None,):
                raise UsageError(f"device out must be a contiguous complex128 array of shape {shape}")
            ptr = int(cai["data"][0])
        else:
            if out.shape != shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
                raise UsageError(f"out must be a contiguous complex128 array of shape {shape}")
            ptr = out.ctypes.data
        self._check(self._L.cyc_block_average_device(self._h, x_ptr, y_ptr, n, int(mode), ptr))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._L.cyc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# CPM / GMSK generation and the Monte-Carlo oracle (proj/include/cycstat/siggen.hpp,
# reference.hpp) -- SURVEY §8 f4
# ---------------------------------------------------------------------------
class PulseKind(enum.IntEnum):
    GaussianGmsk = 0
    Rectangular = 1


@dataclass
class CpmParams:
    """siggen.hpp:16-23 (defaults: h 0.5, M 2, L 4, BT 0.25, 8 sps, Gaussian)."""
    h: float = 0.5
    alphabet_size: int = 2
    pulse_len: int = 4
    bt: float = 0.25
    sps: int = 8
    pulse_kind: PulseKind = PulseKind.GaussianGmsk

    def _c(self) -> _CpmParams:
        return _CpmParams(float(self.h), int(self.alphabet_size), int(self.pulse_len), float(self.bt),
                          int(self.sps), int(self.pulse_kind))


@dataclass
class OracleTable:
    """reference.hpp:15-28: row-major |alphas| x |lags| mean magnitudes."""
    alphas: list
    lags: list
    mean_magnitude: np.ndarray
    trials: int
    record_len: int
    seed: int

    def cell(self, alpha_idx: int, lag_idx: int) -> float:
        return float(self.mean_magnitude[alpha_idx * len(self.lags) + lag_idx])


def _err_buf():
    return C.create_string_buffer(1024)


def random_symbols(alphabet_size: int, count: int, seed: int) -> np.ndarray:
    """siggen.cpp:147-157 (the same mt19937_64 draw)."""
    out = np.zeros(count, dtype=np.int32)
    err = _err_buf()
    _raise_rc(lib().cyc_random_symbols(int(alphabet_size), count, int(seed) & (2**64 - 1),
                                       out.ctypes.data_as(C.POINTER(C.c_int)), err, 1024), err)
    return out


def cpm_pulse(params: Optional[CpmParams] = None):
    """make_pulse (siggen.cpp:103-109): (f, g), length pulse_len * sps."""
    p = params or CpmParams()
    n = int(p.pulse_len) * int(p.sps)
    f, g = np.zeros(max(n, 0)), np.zeros(max(n, 0))
    err = _err_buf()
    _raise_rc(lib().cyc_cpm_pulse(C.byref(p._c()), f.ctypes.data_as(C.POINTER(C.c_double)),
                                  g.ctypes.data_as(C.POINTER(C.c_double)), max(n, 0), err, 1024), err)
    return f, g


def cpm_modulate(params: Optional[CpmParams], symbols, device: int = 0, out=None, f64: bool = False):
    """cpm_modulate (siggen.cpp:111-145) on the device.  Returns a host array
    (complex64, or complex128 with f64=True); `out` may be a device array
    (`__cuda_array_interface__`) that receives the samples instead."""
    p = params or CpmParams()
    sym = np.ascontiguousarray(symbols, dtype=np.int32)
    n = sym.size * int(p.sps)
    err = _err_buf()
    if out is None:
        out = np.empty(n, dtype=np.complex128 if f64 else np.complex64)
        ptr = out.ctypes.data
    else:
        ptr = int(out.__cuda_array_interface__["data"][0])
    _raise_rc(lib().cyc_cpm_modulate(C.byref(p._c()), sym.ctypes.data_as(C.POINTER(C.c_int)), sym.size,
                                     int(device), int(bool(f64)), ptr, err, 1024), err)
    return out


def gmsk_mc_oracle(params: Optional[CpmParams], alphas, lags, conj: bool, win_len: int, trials: int,
                   record_len: int, seed: int, device: int = 0) -> OracleTable:
    """gmsk_mc_oracle (reference.cpp:34-96) on the device."""
    p = params or CpmParams()
    al = np.ascontiguousarray(list(alphas), dtype=np.float64)
    lg = np.ascontiguousarray(list(lags), dtype=np.int32)
    out = np.zeros(max(al.size * lg.size, 1))
    err = _err_buf()
    _raise_rc(lib().cyc_gmsk_mc_oracle(C.byref(p._c()), al.ctypes.data_as(C.POINTER(C.c_double)), al.size,
                                       lg.ctypes.data_as(C.POINTER(C.c_int)), lg.size, int(bool(conj)),
                                       int(win_len), int(trials), int(record_len), int(seed) & (2**64 - 1),
                                       int(device), out.ctypes.data_as(C.POINTER(C.c_double)), err, 1024), err)
    return OracleTable(list(al), list(lg), out[:al.size * lg.size], int(trials), int(record_len), int(seed))


def _raise_rc(rc: int, err) -> None:
    if rc:
        _raise(rc, err.value.decode())


def estimate_cfo_ccf(x, expected_beta: float, N: int, num_frames: int, device: int = 0) -> float:
    """impair.cpp:45-115 on the device: CFO from the conjugate lag-0 scan."""
    xa = _as_c64(x)
    eps = C.c_double()
    err = C.create_string_buffer(1024)
    rc = lib().cyc_estimate_cfo_ccf(xa.ctypes.data, xa.size, float(expected_beta), int(N), int(num_frames),
                                    int(device), C.byref(eps), err, 1024)
    msg = err.value.decode()
    if rc == 3 and msg.startswith("no feature"):
        raise NoFeatureError(msg)
    if rc:
        _raise(rc, msg)
    return eps.value


def export_frames_csv(path: str, frames, cfg: EstimatorConfig) -> int:
    """io.cpp:161-186: one row per (frame, element): frame_index,alpha,lag,re,im,mag
    ("%.17g"), elements in the config's layout order.  Returns the data rows."""
    frames = list(frames)
    if not frames:
        raise UsageError("no frames to export")
    L = lib()
    c, keep = cfg._c()
    vals = np.ascontiguousarray(np.stack([np.asarray(f.values, dtype=np.complex128) for f in frames]))
    idx = np.ascontiguousarray([f.frame_index for f in frames], dtype=np.uint64)
    rows, err = C.c_size_t(), C.create_string_buffer(1024)
    rc = L.cyc_export_frames_csv(C.byref(c), os.fsencode(path), idx.ctypes.data, vals.ctypes.data, len(frames),
                                 C.byref(rows), err, 1024)
    if rc == 0 and vals.shape[1] * len(frames) != rows.value:
        raise UsageError("config does not match the frame layout")
    if rc:
        _raise(rc, err.value.decode())
    return int(rows.value)


def export_average_csv(path: str, avg, cfg: EstimatorConfig, mode: AverageMode = AverageMode.Coherent) -> int:
    """io.cpp:188-208: alpha,lag,mean_re,mean_im,mean_mag (coherent) or
    alpha,lag,mean_mag (magnitude) per element of an average_frames table."""
    L = lib()
    c, keep = cfg._c()
    a = np.ascontiguousarray(np.asarray(avg, dtype=np.complex128).reshape(-1))
    rows, err = C.c_size_t(), C.create_string_buffer(1024)
    rc = L.cyc_export_average_csv(C.byref(c), os.fsencode(path), a.ctypes.data, a.size, int(mode), C.byref(rows),
                                  err, 1024)
    if rc:
        _raise(rc, err.value.decode())
    return int(rows.value)


def write_cf32(path: str, samples) -> int:
    """io.cpp:74-88: interleaved little-endian float32 I/Q; non-finite rejected."""
    a = np.asarray(samples)
    bad = ~np.isfinite(a)
    if bad.any():
        raise DataError(f"non-finite sample at index {int(np.flatnonzero(bad)[0])}", int(np.flatnonzero(bad)[0]))
    b = np.ascontiguousarray(a, dtype=np.complex64).astype("<c8").tobytes()
    with open(path, "wb") as f:
        f.write(b)
    return len(b)


def measure_fp32_peak(device: int = 0) -> float:
    """FP32 FFMA TFLOP/s of the device (fold-kernel roofline denominator)."""
    return float(lib().cyc_measure_fp32_peak(int(device)))


def average_frames(frames: Sequence[CyclicFrame], mode: AverageMode = AverageMode.Coherent) -> np.ndarray:
    """estimator.cpp:86-105 over materialised frames (host-side, as the reference)."""
    if not frames:
        raise UsageError("cannot average an empty frame list")
    lay = frames[0].layout
    for f in frames:
        if f.layout != lay or len(f.values) != len(frames[0].values):
            raise UsageError("cannot average frames with mixed layouts")
    acc = np.zeros(len(frames[0].values), dtype=np.complex128)
    for f in frames:
        acc += f.values if mode == AverageMode.Coherent else np.abs(f.values)
    return acc / len(frames)


def compute_set_window(xw, yw, alphas, max_lag: int, conj: bool, k0: int) -> np.ndarray:
    """kernels.cpp:116-123 on the device."""
    L = lib()
    xa = np.ascontiguousarray(xw, dtype=np.complex128)
    ya = np.ascontiguousarray(yw, dtype=np.complex128)
    al = np.ascontiguousarray(alphas, dtype=np.float64)
    out = np.zeros(len(al) * (2 * max_lag + 1), dtype=np.complex128)
    err = C.create_string_buffer(1024)
    rc = L.cyc_compute_set_window(xa.ctypes.data, len(xa), ya.ctypes.data, len(ya), al.ctypes.data, len(al),
                                  int(max_lag), int(bool(conj)), int(k0), out.ctypes.data, err, 1024)
    if rc:
        _raise(rc, err.value.decode())
    return out


def compute_full_window(xw, yw, lags, conj: bool, k0: int) -> np.ndarray:
    """kernels.cpp:125-135 on the device."""
    L = lib()
    xa = np.ascontiguousarray(xw, dtype=np.complex128)
    ya = np.ascontiguousarray(yw, dtype=np.complex128)
    lg = np.ascontiguousarray(lags, dtype=np.int32)
    out = np.zeros(len(lg) * len(ya), dtype=np.complex128)
    err = C.create_string_buffer(1024)
    rc = L.cyc_compute_full_window(xa.ctypes.data, len(xa), ya.ctypes.data, len(ya), lg.ctypes.data, len(lg),
                                   int(bool(conj)), int(k0), out.ctypes.data, err, 1024)
    if rc:
        _raise(rc, err.value.decode())
    return out

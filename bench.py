#!/usr/bin/env python
"""Benchmark of the B200 cyclic-ACF hot path (BASELINE.json metric).

Default workload: BASELINE.json configs[4] (C5, "large cyclic-domain profile"),
the largest single-GPU configuration (BASELINE.json's metric names no config):
2^26 complex64 samples of BPSK-RRC(0.35, 5 sps, f_c 0.07) + GMSK(BT 0.3,
8 sps, f_c -0.11) at -6 dB, AWGN at 3 dB SNR (seeded synthetic; the paper's
captures are not available); 8192 cycle frequencies k/8192 x lags 0..255,
conventional AND conjugate, one block average.  The reference computes this
as Full mode N = 8192, lags 0..255, N-sized pushes + average_frames(Coherent)
(proj/src/estimator.cpp:39-105, proj/src/kernels.cpp:72-94, fft.cpp:44-87);
F = 8191 frames cover L_eff = 67,100,672 samples.  `--config c1..c4` runs the
other BASELINE configurations.

One step = reset the estimator, push the record, read every (alpha, tau)
table.  Two measurements per run:
  value  -- input already resident in HBM (cyc_push_device), the tables
            finalized into HBM (cyc_average_all to device memory), CUDA events;
  e2e    -- input in pinned HOST memory through the reference-facing C-ABI call
            (cyc_push), H2D DMA and the D2H of the tables inside the timed region.
metric = direct-sum-equivalent (alpha, tau) updates/s = A*T*L_eff*flags*channels / t
(SURVEY §8d).  The executed algorithm is the exact residue fold (tcgen05 bf16x3
banded Gram product; for several lag blocks from bf16 planes split once per
sample) + FFT finalize (fp64 combine, fp32 transform).

Multi-GPU (`torchrun ... bench.py --gpus N`): C2/C5 are time-sharded
(rank r folds frames [F r/N, F (r+1)/N) with `origin` anchoring the phases at
absolute sample 0; an NCCL reduce-scatter sums the fp64 fold states by lag rows before the
finalize; the record is broadcast from rank 0 over NCCL at set-up); C4 is
channel-sharded (64/N channels per rank, NCCL all-gather of the tables).
Total work is fixed: `scaling` = "strong".  C1/C3 run replicas.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cyclic-ACF (alpha,tau) updates/s"
UNIT = "updates/s"
DTYPE = "cf32 in; fold: bf16x3 split on tcgen05 (~fp32 products), fp32 TMEM accumulation drained every <=64 " \
        "stages; fp64 reductions; FFT: fp64 combine, fp32 transform"

# Block-average configurations (Full mode, conv + conj).  `bins`: the cycle
# frequencies the config counts (C4: 128 of the 256 natural bins).
BLOCK = {
    "c2": dict(N=1024, T=64, A=1024, L=1 << 24, channels=1, shard="time",
               workload="C2 dense grid: QPSK-RRC(0.35) 4 sps f_c=0.1 5 dB, 2^24 cf32 samples; 1024 alphas k/1024 x "
                        "tau 0..63, conv+conj, one block average"),
    "c4": dict(N=256, T=32, A=128, L=1 << 22, channels=64, shard="channel",
               workload="C4 multi-channel: 64 x 2^22 (BPSK/QPSK-RRC, GMSK, noise; per-channel draws); 128 alphas "
                        "k/256 in [-1/4,1/4) x tau 0..31, conv+conj, block average per channel"),
    "c5": dict(N=8192, T=256, A=8192, L=1 << 26, channels=1, shard="time",
               workload="C5 BPSK-RRC(0.35,5sps,0.07)+GMSK(BT0.3,8sps,-0.11)@-6dB, AWGN 3 dB, 2^26 cf32 samples; "
                        "8192 alphas k/8192 x tau 0..255, conv+conj, one block average"),
}


def frames_of(c):
    return (c["L"] - c["N"] - c["T"] + 1) // c["N"] + 1


def updates_of(c):
    return c["A"] * c["T"] * frames_of(c) * c["N"] * 2 * c["channels"]


def gen_block(name, channels=None):
    from paper_2405_16911_b200 import siggen
    if name == "c2":
        return siggen.c2_record(seed=2, n=1 << 24)[None]
    if name == "c5":
        return siggen.c5_record(n=1 << 26)[None]
    chans = channels if channels is not None else range(64)
    return np.stack([siggen.c4_channel(c, n=1 << 22) for c in chans])


# ---------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region (B200_PROFILING.md
    clocks line).  NVML is polled every ~0.5 ms from a thread (nvidia-smi's 100 ms
    floor cannot resolve a region of a few ms)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        import threading
        self.samples, self.reasons, self.smax = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv = None
            self.err = str(e)
            return
        self._ready = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        self._ready.wait(1.0)

    def _run(self):
        nv = self.nv
        try:
            nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            pass
        self._ready.set()
        self._stop.wait(0.0005)
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.0005)

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        self._stop.set()
        self.t.join()
        if not self.samples:  # a region shorter than the poll period: sample as it ends
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons.update(name for bit, name in self.REASONS.items() if r & bit)
            except Exception:
                pass
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": "NVML poll ~0.5 ms"}


# ---------------------------------------------------------------------------
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            # communicator set-up lines (rank count, NVLS) on stderr for the scaling run
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def allreduce_max(v: float, ws: int) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return None


def traffic_from_profiles(name: str, planes: bool):
    """DRAM bytes per launch of the config's dominant fold kernel, from the
    committed ncu summary of that config (profiles/<cfg>_fold_ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", f"{name}_fold_ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


def roofline_block(p0: dict, p1: dict, steps: int, ms_step: float, dev: int, lags: int, name: str) -> dict:
    """The dominant kernel (the fold) from CUDA-event profiles on its stream.

    Algorithmic work per launch: 8 flops per (requested lag, folded sample)
    (4 FMAs give both flags) over 8 bytes per folded sample (the record read
    once from HBM), i.e. an intensity of `lags` flop/B.  On the tensor cores
    the ridge is bf16 peak / HBM peak (~250 flop/B), so a fold with fewer lags
    is HBM-bound: `achieved` = algorithmic bytes / launch duration against the
    measured HBM copy bandwidth; with more, tensor-bound: algorithmic flops /
    duration against the bf16 peak.  Both views are reported.  Executed MMA
    work is ~6x the algorithmic (bf16x3 split x the 128x256 band block)."""
    n = max(1, p1["launches"] - p0["launches"])
    ms = (p1["ms"] - p0["ms"]) / n
    alg = (p1["flops"] - p0["flops"]) / n
    exe = (p1["exec_flops"] - p0["exec_flops"]) / n
    tc = p1["tensor_launches"] - p0["tensor_launches"]
    rate = alg / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    import paper_2405_16911_b200 as cyc
    fp32 = cyc.measure_fp32_peak(dev)
    traffic, tsrc = traffic_from_profiles(name, lags > 64)
    common = {"traffic": traffic, "traffic_source": tsrc, "algorithmic_flops_per_launch": alg,
              "ms_per_launch": ms, "launches_per_step": (p1["launches"] - p0["launches"]) / steps,
              "fold_share_of_step": (p1["ms"] - p0["ms"]) / steps / ms_step,
              "algorithmic_unit": "8 flops per (requested lag, folded sample) -- 4 FMAs give both flags -- and "
                                  "8 HBM bytes per folded sample (the record read once)"}
    if tc > 0:
        mp = measured_peaks() or {}
        tpeak = mp.get("bf16_tflops") or 1590.0
        hpeak = mp.get("hbm_gbs") or 6650.0
        ex_rate = exe / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        abytes = alg / max(1, lags)  # 8 B per folded sample
        gbs = abytes / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        ridge = tpeak * 1e12 / (hpeak * 1e9)
        if traffic:
            common["traffic_over_algorithmic_bytes"] = traffic / abytes
        tsus = mp.get("bf16_tflops_sustained")
        tensor_view = {"achieved_tflops": rate, "peak_tflops": tpeak, "frac": rate / tpeak,
                       # the fold runs under sustained tcgen05 load (SM clock ~1.6 GHz inside it):
                       # the sustained cuBLAS figure beside the burst one the line's `frac` uses
                       "sustained_peak_tflops": tsus, "frac_vs_sustained": rate / tsus if tsus else None,
                       "executed_tflops": ex_rate, "executed_frac": ex_rate / tpeak,
                       "executed_per_algorithmic": exe / alg if alg else None,
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16 burst, this pool)"
                       if mp.get("bf16_tflops") else "fallback 1.59 PFLOP/s (B200_PROFILING.md)"}
        hbm_view = {"achieved_gbs": gbs, "peak_gbs": hpeak, "frac": gbs / hpeak,
                    "algorithmic_bytes_per_launch": abytes,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, this pool)" if mp.get("hbm_gbs")
                    else "fallback 6.65 TB/s (B200_PROFILING.md)"}
        kern = "fold_tcp_kernel (tcgen05 bf16x3 banded Gram product from split planes)" if lags > 64 else \
            "fold_tc_kernel (tcgen05 bf16x3 banded Gram product, fused fp32->bf16 split)"
        common.update({"kernel": kern, "intensity_flop_per_byte": float(lags), "ridge_flop_per_byte": ridge,
                       "tensor_view": tensor_view, "hbm_view": hbm_view,
                       "fp32_ffma_peak_tflops": fp32, "algorithmic_vs_fp32_peak": rate / fp32 if fp32 else None,
                       "tensor_launches_share": tc / n})
        if lags < ridge:
            return {"bound": "hbm", "achieved": gbs, "peak": hpeak, "unit": "GB/s", "frac": gbs / hpeak,
                    "peak_source": hbm_view["peak_source"], **common}
        return {"bound": "tensor", "achieved": rate, "peak": tpeak, "unit": "TFLOP/s", "frac": rate / tpeak,
                "peak_source": tensor_view["peak_source"], **common}
    return {"bound": "fp32", "kernel": "fold_kernel (FFMA2 residue fold)", "achieved": rate, "peak": fp32,
            "unit": "TFLOP/s", "frac": rate / fp32 if fp32 else None, **common,
            "peak_source": "measured live: FFMA microbenchmark in libcycb200 (MEASURED_PEAKS.json carries no "
                           "FP32 figure)"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified cycstat library) on the host cores
# ---------------------------------------------------------------------------
C1_CONV = [k / 8 for k in range(-2, 3)]
C1_CONJ = [0.1 + k / 16 for k in range(-2, 3)]
C3_ALPHAS = [m / 1024 for m in range(-128, 128)]


def ref_sample(name, x, threads):
    """One bounded sample of the config's workload on the reference library:
    (updates, seconds, description).  N-sized pushes + running coherent sum
    (the reference's caller pattern), OpenMP over lags."""
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    os.environ["OMP_NUM_THREADS"] = str(threads)
    from oracle.oracle import RefLib
    r = RefLib()
    t0 = time.perf_counter()
    if name == "c1":
        xs = x.astype(np.complex128)
        F = 0
        for conj, al in ((0, C1_CONV), (1, C1_CONJ)):
            fr, _ = r.stream(0, conj, 4096, xs, xs, alphas=al, max_lag=15, chunk=4096)
            F = len(fr)
        ups, smp = 5 * 31 * F * 4096 * 2, f"whole record, both estimators ({F} frames each), 4096-sample pushes"
    elif name == "c3":
        n = 2048 * 1024 + 31
        xs = np.ascontiguousarray(x[:n])
        _, F = r.block_average(1, 0, 1024, xs, xs, lags=list(range(32)))
        ups, smp = 256 * 32 * F * 1024, (f"block-mode stand-in (no recursive mode in the reference): Full N=1024 "
                                         f"lags 0..31, {F} frames, 256 of 1024 bins counted")
    elif name == "c4":
        F, nch = 0, 2
        for c in range(nch):
            xs = np.ascontiguousarray(x[c])
            for conj in (0, 1):
                _, F = r.block_average(1, conj, 256, xs, xs, lags=list(range(32)))
        ups, smp = nch * 2 * 128 * 32 * F * 256, f"{nch} of 64 channels, whole channel ({F} frames), conv+conj"
    elif name == "c2":
        nf = 4096
        xs = np.ascontiguousarray(x[0, :nf * 1024 + 63])
        for conj in (0, 1):
            _, F = r.block_average(1, conj, 1024, xs, xs, lags=list(range(64)))
        ups, smp = 1024 * 64 * F * 1024 * 2, f"{F} of 16383 frames, conv+conj"
    else:
        nf = 48
        xs = np.ascontiguousarray(x[0, :nf * 8192 + 255])
        for conj in (0, 1):
            _, F = r.block_average(1, conj, 8192, xs, xs, lags=list(range(256)))
        ups, smp = 8192 * 256 * F * 8192 * 2, f"{F} of 8191 frames, conv+conj"
    dt = time.perf_counter() - t0
    return ups, dt, smp + f"; Full mode (Set for C1), N-sized pushes + coherent sum, OMP_NUM_THREADS={threads}, " \
                          f"OMP_WAIT_POLICY={os.environ.get('OMP_WAIT_POLICY')}"


def cpu_baseline(name, x, threads):
    ups, dt, smp = ref_sample(name, x, threads)
    return {"value": ups / dt, "unit": UNIT, "cores": threads, "kind": "reference", "seconds": dt, "sample": smp}


def parity_check(name, x, tables):
    """The timed run's final tables against the fp64 oracle on the FULL record
    (a subset of cycle frequencies, every lag, both flags) -- the checker, run
    after timing in the CPU-baseline leg.  tables: [channels, 2, T * N]."""
    from oracle.oracle import Oracle
    c = BLOCK[name]
    N, T = c["N"], c["T"]
    F = frames_of(c)
    o = Oracle()
    rng = np.random.default_rng(7)
    if name == "c4":
        bins = np.array([k % N for k in range(-64, 64)])
        chans = [0, 1, 2, 3, 21, 46, 63]
    else:
        bins = np.unique(np.concatenate([[0, 1, N - 1, N // 2], rng.choice(N, 60, replace=False)]))
        chans = [0]
    worst_rel, worst_cell = 0.0, 0.0
    t0 = time.perf_counter()
    for ch in chans:
        xc = x[ch]
        mp = float(np.mean(np.abs(xc.astype(np.complex128)) ** 2))
        cv, cj = o.block_fold(xc, xc, bins, N, list(range(T)), 0, F * N)
        for fi, want in ((0, cv), (1, cj)):
            got = tables[ch, fi].reshape(T, N)[:, bins]
            d = got - want.T
            worst_rel = max(worst_rel, float(np.linalg.norm(d) / np.linalg.norm(want)))
            worst_cell = max(worst_cell, float(np.abs(d).max() / mp))
    return {"rel_l2": worst_rel, "max_abs_over_mean_power": worst_cell, "tolerance": {"rel_l2": 1e-4, "cell": 1e-5},
            "pass": worst_rel <= 1e-4 and worst_cell <= 1e-5, "channels": chans, "bins": int(len(bins)),
            "lags": T, "oracle": "oracle/cycoracle.c block_fold (fp64) on the full record",
            "seconds": time.perf_counter() - t0}


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref) on this box's
    host cores, each step a bounded sample of the config's workload."""
    if rank != 0:
        return
    name = args.config
    if name in BLOCK:
        x = gen_block(name, channels=range(2) if name == "c4" else None)
        wl = BLOCK[name]["workload"]
    else:
        from paper_2405_16911_b200 import siggen
        x = siggen.c1_record(n=2 ** 20) if name == "c1" else siggen.c3_record(n=2 ** 22)
        wl = SMALL[name]["workload"]
    threads = os.cpu_count() or 1
    for _ in range(min(1, args.warmup)):
        ref_sample(name, x, threads)
    samples = [ref_sample(name, x, threads) for _ in range(args.steps)]
    ups, dt, smp = samples[-1]
    value = statistics.median(u / t for u, t, _ in samples)
    ms = statistics.median(t for _, t, _ in samples) * 1e3
    cb = {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": smp,
          "updates_per_step": ups}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl, "algorithm": "reference cycstat (oracle/_ref, compiled from proj/src): "
                                                    "full_window_values + radix-2 FFT per frame (Set: "
                                                    "set_window_values), fp64, OpenMP over lags",
                       "ms_per_step_basis": "measured: one bounded sample of the workload per step (see "
                                            "cpu_baseline.sample); value = its updates / its time"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Block-average configurations on the GPU (C2, C4, C5), sharded over ranks
# ---------------------------------------------------------------------------
def run_block(args, ws, rank, local):
    import torch
    import paper_2405_16911_b200 as cyc
    from paper_2405_16911_b200.shard import (channel_shards, exchange_lag_slices, gather_channel_tables,
                                             gather_lag_tables, time_shards)

    name = args.config
    c = BLOCK[name]
    N, T, L, C_ = c["N"], c["T"], c["L"], c["channels"]
    dev = local
    torch.cuda.set_device(dev)
    cuda = f"cuda:{dev}"
    F_total = frames_of(c)
    lay = T * N
    # --- input: C2/C5 generated on rank 0 and broadcast over NCCL; C4 per rank (own channels)
    if c["shard"] == "time":
        if rank == 0:
            x = gen_block(name)
            d_all = torch.from_numpy(x.view(np.float32)).to(cuda)
        else:
            x = None
            d_all = torch.empty((1, 2 * L), dtype=torch.float32, device=cuda)
        if ws > 1:
            import torch.distributed as dist
            dist.broadcast(d_all, src=0)
        sh = time_shards(L, N, T - 1, 0, ws)[rank]
        # one sample past the shard's last lag when the record has it: the
        # tensor-core windows (192 samples for 128 residues x 64 lags) then
        # cover the last fold period too (no FP32 tail launch); no extra frame
        s1 = min(L, sh.sample1 + 1)
        n_local = s1 - sh.sample0
        d_loc = d_all[:, 2 * sh.sample0:2 * s1]  # a view: the estimator folds it in place
        ch0, ch1, origin = 0, 1, sh.origin
    else:
        ch0, ch1 = channel_shards(C_, ws)[rank]
        x = gen_block(name, channels=range(ch0, ch1))
        d_loc = torch.from_numpy(x.view(np.float32)).to(cuda)
        n_local, origin = L, 0
    nch = ch1 - ch0
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(T)),
                              flags=cyc.Flags.BOTH, emit_frames=False, channels=nch, device=dev, origin=origin)
    est = cyc.CyclicCorrelator(cfg)
    ptr = d_loc.data_ptr()
    host = cyc.host_alloc((nch, n_local))
    host[:] = d_loc.cpu().numpy().view(np.complex64).reshape(nch, n_local)
    out_dev = torch.empty((nch, 2, lay), dtype=torch.complex128, device=cuda)
    full_dev = out_dev if (c["shard"] == "time" or ws == 1) else \
        torch.empty((C_, 2, lay), dtype=torch.complex128, device=cuda)
    out_host = cyc.host_alloc((C_ if c["shard"] == "channel" else 1, 2, lay), dtype=np.complex128)

    t_pad = est.fold_state()[1] // (4 * N * nch) if c["shard"] == "time" else T  # Full mode: Pf = N
    lags_mine = [0, T]

    def exchange():
        """Time shards: NCCL reduce-scatter of the fp64 fold accumulators by lag
        rows; each rank then finalizes its T/N lags (set_lag_slice)."""
        if c["shard"] != "time" or ws == 1:
            return
        import torch.distributed as dist
        lags_mine[:] = exchange_lag_slices(est, F_total, T, t_pad, ws, rank, dist)

    def gather():
        """NCCL all-gather of the tables: time shards the lag slices, channel
        shards the (channel, flag) tables."""
        if ws == 1:
            return
        import torch.distributed as dist
        if c["shard"] == "channel":
            full_dev.copy_(gather_channel_tables(out_dev, ws, dist))
        elif tuple(lags_mine) != (0, T):
            gather_lag_tables(out_dev, lags_mine[0], lags_mine[1], T, ws, dist)

    def step_device():
        if ws == 1:  # one call, one host synchronisation (cyc_block_average_device)
            est.block_average_device(ptr, n_local, out_dev)
            return
        est.reset()
        est.push_device(ptr, n_local)
        exchange()
        est.average_all(out=out_dev)
        gather()

    def step_e2e():
        est.reset()
        est.push(host)
        exchange()
        if ws > 1:
            est.average_all(out=out_dev)
            gather()
            if rank == 0:
                out_host[:] = full_dev.cpu().numpy()
        else:
            est.average_all(out=out_host)

    def timed(fn, k):
        barrier(ws)
        torch.cuda.synchronize(dev)
        # default-stream events bracket every engine stream: pushes read after
        # earlier default-stream work and later default-stream work waits for them
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        barrier(ws)
        return e0.elapsed_time(e1) / k

    for _ in range(max(args.warmup, 3)):
        # two device steps per round: reset alternates the accumulator buffer,
        # and each (buffer, position) push is captured into a CUDA graph on its
        # second occurrence -- the timed steps replay
        step_device()
        step_device()
        step_e2e()
    launches0 = est.kernel_launches()
    clk = Clocks(dev)
    ms_dev = timed(step_device, args.steps)
    clocks = clk.stop()
    launches = est.kernel_launches() - launches0
    final_tables = full_dev.cpu().numpy() if rank == 0 else None
    # the same K steps again with CUDA events around every fold launch on its
    # stream: the kernel timing behind `roofline` (inside the replayed push
    # graph those events are extra graph nodes, so the value steps run without them)
    est.profile(True)
    for _ in range(4):
        step_device()
    prof0 = est.profile_read_ex()
    ms_prof = timed(step_device, args.steps)
    prof1 = est.profile_read_ex()
    est.profile(False)
    ms_e2e = timed(step_e2e, args.steps)

    ms_dev_max = allreduce_max(ms_dev, ws)
    ms_e2e_max = allreduce_max(ms_e2e, ws)
    roof = roofline_block(prof0, prof1, args.steps, ms_dev_max, dev, T, name)
    roof["timing"] = (f"CUDA events on the compute stream around each fold launch over a second pass of "
                      f"{args.steps} device steps run right after the timed ones "
                      f"({allreduce_max(ms_prof, ws):.4f} ms/step with the events)")
    if rank != 0:
        return
    ups = updates_of(c)
    par = f"{'time' if c['shard'] == 'time' else 'channel'}-sharded x{ws}" + (
        ": frame ranges per GPU + NCCL reduce-scatter of the fp64 fold states by lag rows, T/N lags finalized per "
        "GPU, NCCL all-gather of the tables" if c["shard"] == "time" else
        ": 64/N channels per GPU + NCCL all-gather of the tables") if ws > 1 else "single GPU"
    cfgb = {"workload": c["workload"], "samples": L, "channels": C_, "alphas": c["A"], "lags": T,
            "flags": ["conv", "conj"], "win_len": N, "l_eff": frames_of(c) * N, "parallelism": par,
            "l2": f"input {L * C_ * 8 / 1e6:.0f} MB > 126 MB L2 (no reuse across steps)",
            "algorithm": est.algorithm() + (" (planes path: split once per sample + conversion-free tcgen05 fold)"
                                            if T > 64 else " (fused fp32->bf16 split in the tcgen05 fold)")}
    h2d = n_local * nch * 8
    d2h = int(out_host.nbytes)
    line = {
        "metric": METRIC, "value": ups / (ms_dev_max * 1e-3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic (seeded generators, "
                                                                          "paper_2405_16911_b200/siggen.py)",
        "config": cfgb,
        "msamples_per_s": L * C_ / (ms_dev_max * 1e-3) / 1e6,
        "e2e": {"value": ups / (ms_e2e_max * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e_max,
                "h2d_bytes_per_step": h2d * ws, "d2h_bytes_per_step": d2h,
                "msamples_per_s": L * C_ / (ms_e2e_max * 1e-3) / 1e6,
                "path": "cyc_push(pinned host cf32) + cyc_average_all (every table, one D2H into pinned host)"},
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        if x is None:
            x = gen_block(name)
        line["cpu_baseline"] = cpu_baseline(name, x, os.cpu_count() or 1)
        line["parity"] = parity_check(name, x, final_tables)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Small-call configurations (C1, C3): the streaming call pattern through the
# C-ABI from C++ (tools/stream_bench), replicas for N > 1
# ---------------------------------------------------------------------------
SMALL = {
    "c1": dict(workload="C1 GMSK BT0.3 8sps f_c=0.05 10 dB, 2^20 samples in 4096-sample pushes; Set N=4096 "
                        "Symmetric(15); conv alpha=k/8, conj alpha=0.1+k/16 (k=-2..2); per-frame + coherent avg",
               samples=2 ** 20, chunk=4096),
    "c3": dict(workload="C3 GMSK BT0.3 8sps f_c=0.02 0 dB, 2^28 samples in 8192-sample work() calls; recursive "
                        "lambda=1-2^-12, 256 alpha=m/1024 x tau 0..31, conv, emit every 2^16",
               samples=2 ** 28, chunk=8192),
}


def small_updates(name):
    if name == "c1":
        F = (2 ** 20 - 4096 - 30) // 4096 + 1
        return 5 * 31 * F * 4096 * 2
    E = 65536
    F = (2 ** 28 - E - 31) // E + 1
    return 256 * 32 * F * E


def run_small(args, ws, rank, local):
    from paper_2405_16911_b200 import siggen
    from paper_2405_16911_b200.build import build_tools
    name = args.config
    s = SMALL[name]
    x = siggen.c1_record(n=2 ** 20) if name == "c1" else siggen.c3_record(n=2 ** 28)
    exe = build_tools()
    fd, path = tempfile.mkstemp(suffix=".cf32", dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    os.close(fd)
    x.astype(np.complex64).tofile(path)
    barrier(ws)
    clk = Clocks(local)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=str(local))
    r = subprocess.run([exe, name, path, str(args.steps), str(max(args.warmup, 1))], capture_output=True, text=True,
                       env=env)
    clocks = clk.stop()
    os.unlink(path)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    cxx = json.loads(r.stdout.strip().splitlines()[-1])
    ms = allreduce_max(cxx["ms_per_step"], ws)
    if rank != 0:
        return
    ups = small_updates(name) * ws
    gbs = s["samples"] * ws * 8 / (ms * 1e-3) / 1e9
    line = {"metric": METRIC, "value": ups / (ms * 1e-3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": s["workload"], "parallelism": f"replicas x{ws} (the path does not shard)",
                       "value_path": "tools/stream_bench (C++): cyc_push of "
                                     f"{s['chunk']}-sample chunks from pinned host memory, frames to a sink",
                       "emission": "pipelined (cyc_set_emit_pipeline depth 2: up to two frame batches in flight "
                                   "(graph-replayed batches: two instances with their own pinned tables for the small fold graphs, else one), delivered by a later push; same frames bit for bit, tests/test_gpu_pipeline.py); "
                                   "CYC_EMIT_PIPELINE=0 times the reference's synchronous push()"},
            "msamples_per_s": s["samples"] * ws / (ms * 1e-3) / 1e6,
            "e2e": {"value": ups / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
                    "h2d_bytes_per_step": s["samples"] * 8 * ws, "d2h_bytes_per_step": None,
                    "path": "the streaming call pattern is end to end: host chunks in, frames out"},
            "roofline": {"bound": "pcie", "achieved": gbs, "peak": 53.6 * ws, "unit": "GB/s", "frac": gbs / 53.6 / ws,
                         "traffic": None,
                         "peak_source": "measured pinned H2D copy bandwidth on this box type (tools/pcie_probe.py)",
                         "algorithmic_unit": "8 B per input sample moved host -> device",
                         "note": "streaming call pattern: per-call host work and per-emission kernel latency bind"},
            "gpu_launches": int(cxx["launches_per_step"] * args.steps), "clocks": clocks,
            "h2d_bound_ms": s["samples"] * 8 / 53.6e9 * 1e3}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, x, os.cpu_count() or 1)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE.json configuration (c5 = the largest single-GPU config, the default)")
    args = ap.parse_args()
    ws, rank, local = dist_init()
    try:
        if args.impl == "reference":
            run_reference(args, ws, rank)
        elif args.config in BLOCK:
            run_block(args, ws, rank, local)
        else:
            run_small(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

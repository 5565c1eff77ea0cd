"""CPU: the C-ABI library loads, exports every declared symbol, and its host-side
logic (validation, layouts, plan selection) matches the reference's contract.
No compute call is made (there is no GPU here)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def declared_symbols():
    syms = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(cyc_[a-z0-9_]+)\s*\(", src):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol(cyc):
    from paper_2405_16911_b200 import LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = declared_symbols() - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert cyc.lib().cyc_abi_version() == 1


def test_library_is_sm100a(cyc):
    from paper_2405_16911_b200 import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_fold_kernel_uses_packed_fma(cyc):
    """The hot loop is FFMA2 (packed FP32) fed by LDS.128 -- checked in SASS."""
    from paper_2405_16911_b200 import LIB_PATH
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB_PATH], capture_output=True,
                          text=True).stdout
    assert sass.count("FFMA2") >= 3 * 64
    assert "LDS.128" in sass and "LDGSTS" in sass


def _cfg(cyc, **kw):
    return cyc.EstimatorConfig(**kw)


def test_validation_messages_match_reference(cyc):
    g = np.load(GOLD)
    cases = [eval(c) for c in g["validate_cases"]]
    for case, want in zip(cases, g["validate_msgs"]):
        ls = (cyc.LagSpec.Symmetric(case.get("max_lag", 0)) if case["lag_symmetric"]
              else cyc.LagSpec.Explicit(case.get("lags", [])))
        cfg = cyc.EstimatorConfig(mode=cyc.Mode(case["mode"]), win_len=case["win_len"],
                                  alphas=case.get("alphas", []), lag_spec=ls)
        got = cyc.validate_config(cfg)
        assert got == [s for s in str(want).split("\n") if s], case


def test_config_error_carries_all_violations(cyc):
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1, alphas=[0.9], lag_spec=cyc.LagSpec.Explicit([3, 1]))
    v = cyc.validate_config(cfg)
    assert len(v) == 3
    with pytest.raises(cyc.ConfigError) as ei:
        cyc.plan(cfg)
    assert ei.value.violations == v
    assert str(ei.value).startswith("invalid config:")
    assert isinstance(ei.value, cyc.UsageError)


def test_extension_validation(cyc):
    rec = cyc.EstimatorConfig(mode=cyc.Mode.Recursive, win_len=64, alphas=[0.1], lag_spec=cyc.LagSpec.Explicit([0]),
                              lam=1.5)
    assert "forgetting factor must lie in (0, 1)" in cyc.validate_config(rec)
    bad = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=64, lag_spec=cyc.LagSpec.Explicit([0]), channels=0)
    assert "channels must be at least 1" in cyc.validate_config(bad)


@pytest.mark.parametrize("alphas,expect", [
    ([k / 8 for k in range(-2, 3)], "fold-dft P=8 "),                  # C1 conventional grid
    ([0.1 + k / 16 for k in range(-2, 3)], "fold-dft P=80 "),          # C1 conjugate grid (0.1 + k/16)
    ([m / 1024 for m in range(-128, 128)], "fold-fft P=1024 "),        # C3 grid
    ([-0.25 + k / 256 for k in range(128)], "fold-fft P=256 "),        # C4 grid
    ([0.1234507], "direct"),                                          # off-grid (test_estimator.cpp:112)
])
def test_plan_rational_grid(cyc, alphas, expect):
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=4096, alphas=alphas, lag_spec=cyc.LagSpec.Symmetric(15))
    assert cyc.plan(cfg).startswith(expect)


def test_plan_full_mode_dense_grids(cyc):
    for N, T, lw in [(1024, 64, 8), (256, 32, 4), (8192, 256, 8), (64, 9, 2)]:
        cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(T)))
        p = cyc.plan(cfg)
        assert f"P={N} " in p and f"lw={lw}" in p, p


def test_layout_helpers_match_reference_semantics(cyc):
    lay = cyc.SetLayout(3, 2)
    assert cyc.layout_len(lay) == 15
    assert [cyc.flat_index(lay, 1, m) for m in range(-2, 3)] == [5, 6, 7, 8, 9]
    with pytest.raises(IndexError):
        cyc.flat_index(lay, 3, 0)
    with pytest.raises(IndexError):
        cyc.flat_index(lay, 0, 3)
    fl = cyc.FullLayout(2, 8)
    assert cyc.flat_index(fl, 1, 3) == 11
    # full_bin_to_alpha (types.cpp:100-104)
    assert [cyc.full_bin_to_alpha(k, 8) for k in range(8)] == [0, 0.125, 0.25, 0.375, -0.5, -0.375, -0.25, -0.125]
    with pytest.raises(IndexError):
        cyc.full_bin_to_alpha(8, 8)


def test_lagspec(cyc):
    s = cyc.LagSpec.Symmetric(3)
    assert (s.m_plus(), s.m_minus(), s.values()) == (3, 3, [-3, -2, -1, 0, 1, 2, 3])
    e = cyc.LagSpec.Explicit([-3, 0, 5])
    assert (e.m_plus(), e.m_minus()) == (5, 3)
    assert (cyc.LagSpec.Explicit([2, 4]).m_minus()) == 0


def test_average_frames_host(cyc):
    f1 = cyc.CyclicFrame(0, 3, cyc.SetLayout(1, 1), np.array([1 + 1j, 2, 3j]))
    f2 = cyc.CyclicFrame(1, 19, cyc.SetLayout(1, 1), -f1.values)
    assert np.max(np.abs(cyc.average_frames([f1, f2]))) == 0
    assert np.allclose(cyc.average_frames([f1, f2], cyc.AverageMode.Magnitude), np.abs(f1.values))
    with pytest.raises(cyc.UsageError):
        cyc.average_frames([])
    f3 = cyc.CyclicFrame(1, 19, cyc.FullLayout(1, 3), f1.values)
    with pytest.raises(cyc.UsageError):
        cyc.average_frames([f1, f3])


def test_no_cpu_fallback(cyc):
    """Without a device the product fails loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=64, lag_spec=cyc.LagSpec.Explicit([0]))
    with pytest.raises(cyc.CudaError):
        cyc.CyclicCorrelator(cfg)

"""CSV result export (proj/src/io.cpp:161-208): the C-ABI writers
(cyc_export_frames_csv / cyc_export_average_csv, host-only) against the
reference's own export_frames_csv / export_average_csv (oracle/_ref, built with
io.cpp) on the same values: byte-identical files."""
import numpy as np
import pytest

from conftest import rand_c


@pytest.fixture(scope="module")
def ref_io(ref):
    if not ref.has_io:
        pytest.skip("reference io.cpp not built (no json.hpp)")
    return ref


def set_cfg(cyc, alphas, m):
    return cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=64, alphas=list(alphas), lag_spec=cyc.LagSpec.Symmetric(m))


def full_cfg(cyc, n, lags):
    return cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=n, lag_spec=cyc.LagSpec.Explicit(lags))


def frames_of(cyc, cfg, values, indices):
    lay = cyc.SetLayout(len(cfg.alphas), cfg.lag_spec.m_plus) if cfg.mode == cyc.Mode.Set else \
        cyc.FullLayout(len(cfg.lag_spec.values()), cfg.win_len)
    return [cyc.CyclicFrame(int(i), 0, lay, v, 1, 0) for i, v in zip(indices, values)]


@pytest.mark.parametrize("kind", ["set", "full"])
def test_frames_csv_matches_reference(cyc, ref_io, tmp_path, kind):
    if kind == "set":
        cfg, alphas, m, lags, n = set_cfg(cyc, [0.1, -0.25, 0.1234507], 3), [0.1, -0.25, 0.1234507], 3, [], 64
        length = 3 * 7
    else:
        cfg, alphas, m, lags, n = full_cfg(cyc, 16, [-2, 0, 5]), [], 0, [-2, 0, 5], 16
        length = 3 * 16
    vals = np.stack([rand_c(length, 30 + f).astype(np.complex128) * 1e-3 for f in range(3)])
    vals[0, 0] = 0.0
    vals[1, 1] = -0.0 + 1e-300j
    idx = [0, 1, 7]
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    rows = cyc.export_frames_csv(str(ours), frames_of(cyc, cfg, vals, idx), cfg)
    rrows = ref_io.export_frames_csv(str(theirs), 0 if kind == "set" else 1, n, vals, idx, alphas=alphas, max_lag=m,
                                     lags=lags)
    assert rows == rrows == 3 * length
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_text().splitlines()[0] == "frame_index,alpha,lag,re,im,mag"


@pytest.mark.parametrize("magnitude", [False, True])
@pytest.mark.parametrize("kind", ["set", "full"])
def test_average_csv_matches_reference(cyc, ref_io, tmp_path, kind, magnitude):
    if kind == "set":
        cfg, alphas, m, lags, n, length = set_cfg(cyc, [0.0, 0.375], 2), [0.0, 0.375], 2, [], 64, 10
    else:
        cfg, alphas, m, lags, n, length = full_cfg(cyc, 32, [0, 1, 2, 3]), [], 0, [0, 1, 2, 3], 32, 128
    avg = rand_c(length, 77).astype(np.complex128)
    if magnitude:
        avg = np.abs(avg).astype(np.complex128)
    mode = cyc.AverageMode.Magnitude if magnitude else cyc.AverageMode.Coherent
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    assert cyc.export_average_csv(str(ours), avg, cfg, mode) == length
    ref_io.export_average_csv(str(theirs), 0 if kind == "set" else 1, n, avg, magnitude, alphas=alphas, max_lag=m,
                              lags=lags)
    assert ours.read_bytes() == theirs.read_bytes()


def test_csv_errors(cyc, tmp_path):
    cfg = full_cfg(cyc, 16, [0, 1])
    with pytest.raises(cyc.UsageError, match="no frames to export"):
        cyc.export_frames_csv(str(tmp_path / "a.csv"), [], cfg)
    with pytest.raises(cyc.UsageError, match="no averaged values"):
        cyc.export_average_csv(str(tmp_path / "a.csv"), np.zeros(0, complex), cfg)
    with pytest.raises(cyc.UsageError, match="does not match the averaged vector length"):
        cyc.export_average_csv(str(tmp_path / "a.csv"), np.zeros(5, complex), cfg)
    with pytest.raises(cyc.IoError, match="cannot open"):
        cyc.export_average_csv(str(tmp_path / "missing_dir" / "a.csv"), np.zeros(32, complex), cfg)
    bad = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1, lag_spec=cyc.LagSpec.Explicit([0]))
    with pytest.raises(cyc.ConfigError):
        cyc.export_average_csv(str(tmp_path / "b.csv"), np.zeros(1, complex), bad)

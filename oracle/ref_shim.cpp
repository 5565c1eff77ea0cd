// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline).  oracle/Makefile compiles
// this file together with the reference's own sources, where they lie under
// /root/reference/proj/src, into oracle/_ref/libcycstat_ref.so.  No reference
// source is copied into this repository.  Each entry point calls the
// reference's public C++ API exactly as its own callers do
// (proj/tools/main.cpp:212-214, proj/bench/bench_kernels.cpp).
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cycstat/errors.hpp"
#include "cycstat/estimator.hpp"
#include "cycstat/impair.hpp"
#include "cycstat/reference.hpp"
#include "cycstat/siggen.hpp"
#ifdef REF_HAVE_IO
#include "cycstat/io.hpp"
#endif

using namespace cycstat;

namespace {

thread_local std::string g_err;

std::vector<cx> load(const double* p, std::size_t n) {
    std::vector<cx> v(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = cx(p[2 * i], p[2 * i + 1]);
    return v;
}

void store(const std::vector<cx>& v, double* p) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        p[2 * i] = v[i].real();
        p[2 * i + 1] = v[i].imag();
    }
}

EstimatorConfig make_cfg(int mode, int conj, int win_len, const double* alphas,
                         std::size_t n_alphas, int max_lag, const int* lags,
                         std::size_t n_lags) {
    EstimatorConfig cfg;
    cfg.mode = mode == 0 ? Mode::Set : Mode::Full;
    cfg.conj = conj != 0;
    cfg.win_len = win_len;
    cfg.alphas.assign(alphas, alphas + n_alphas);
    if (mode == 0)
        cfg.lag_spec = LagSpec::Symmetric(max_lag);
    else
        cfg.lag_spec = LagSpec::Explicit(std::vector<int>(lags, lags + n_lags));
    return cfg;
}

// error codes mirror the C-ABI's: 1 config/usage, 3 data, 5 other
int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_direct(const double* x, const double* y, std::size_t len, double alpha, int m,
               int conj, std::size_t k0, int n_win, double* out) {
    try {
        const auto xv = load(x, len), yv = load(y, len);
        const cx r = cyclic_xcorr_direct(xv, yv, alpha, m, conj != 0, k0, n_win);
        out[0] = r.real();
        out[1] = r.imag();
        return 0;
    } catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 5); }
}

int ref_fft(const double* in, double* out, std::size_t n) {
    try {
        const auto v = dft(load(in, n));
        store(v, out);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

// Streams x/y through CyclicCorrelator::push in `chunk`-sized pieces
// (chunk == 0: one push of the whole record) and returns every frame.
// frames_out == nullptr: only report n_frames / layout_len.
int ref_stream(int mode, int conj, int win_len, const double* alphas, std::size_t n_alphas,
               int max_lag, const int* lags, std::size_t n_lags, const double* x,
               const double* y, std::size_t len, std::size_t chunk, double* frames_out,
               std::uint64_t* start_abs, std::size_t* n_frames, std::size_t* layout_len) {
    try {
        CyclicCorrelator est(make_cfg(mode, conj, win_len, alphas, n_alphas, max_lag, lags, n_lags));
        if (layout_len) *layout_len = cycstat::layout_len(est.layout());
        const auto xv = load(x, len), yv = load(y, len);
        if (chunk == 0) chunk = len ? len : 1;
        std::size_t f = 0;
        for (std::size_t pos = 0; pos < len; pos += chunk) {
            const std::size_t take = std::min(chunk, len - pos);
            std::vector<cx> cxk(xv.begin() + pos, xv.begin() + pos + take);
            std::vector<cx> cyk(yv.begin() + pos, yv.begin() + pos + take);
            auto frames = est.push(cxk, cyk);
            for (auto& fr : frames) {
                if (frames_out) store(fr.values, frames_out + 2 * f * fr.values.size());
                if (start_abs) start_abs[f] = fr.start_abs;
                ++f;
            }
        }
        if (n_frames) *n_frames = f;
        return 0;
    } catch (const DataError& e) { return fail(e, 3); }
    catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 5); }
}

// The reference's coherent block average (CLI `estimate` pattern,
// proj/tools/main.cpp:212-214 + average_frames, proj/src/estimator.cpp:86-105),
// pushed in win_len-sized chunks with a running frame sum so memory stays
// bounded.  max_frames > 0 stops after that many frames (bounded CPU sample).
int ref_block_average(int mode, int conj, int win_len, const double* alphas,
                      std::size_t n_alphas, int max_lag, const int* lags, std::size_t n_lags,
                      const float* xf, const float* yf, std::size_t len,
                      std::size_t max_frames, double* out, std::size_t* n_frames) {
    try {
        CyclicCorrelator est(make_cfg(mode, conj, win_len, alphas, n_alphas, max_lag, lags, n_lags));
        const std::size_t lay = cycstat::layout_len(est.layout());
        std::vector<cx> sum(lay, cx(0.0, 0.0));
        std::size_t f = 0;
        const std::size_t chunk = static_cast<std::size_t>(win_len);
        std::vector<cx> cxk, cyk;
        for (std::size_t pos = 0; pos < len; pos += chunk) {
            if (max_frames && f >= max_frames) break;
            const std::size_t take = std::min(chunk, len - pos);
            cxk.resize(take);
            cyk.resize(take);
            for (std::size_t i = 0; i < take; ++i) {
                cxk[i] = cx(xf[2 * (pos + i)], xf[2 * (pos + i) + 1]);
                cyk[i] = cx(yf[2 * (pos + i)], yf[2 * (pos + i) + 1]);
            }
            auto frames = est.push(cxk, cyk);
            for (auto& fr : frames) {
                if (max_frames && f >= max_frames) break;
                for (std::size_t i = 0; i < lay; ++i) sum[i] += fr.values[i];
                ++f;
            }
        }
        if (f) {
            const double inv = 1.0 / static_cast<double>(f);
            for (auto& v : sum) v *= inv;
        }
        store(sum, out);
        if (n_frames) *n_frames = f;
        return 0;
    } catch (const DataError& e) { return fail(e, 3); }
    catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 5); }
}

// Config validation (proj/src/types.cpp:30-63): writes '\n'-joined violations.
int ref_validate(int mode, int conj, int win_len, const double* alphas, std::size_t n_alphas,
                 int lag_symmetric, int max_lag, const int* lags, std::size_t n_lags,
                 char* buf, std::size_t buflen) {
    EstimatorConfig cfg = make_cfg(mode, conj, win_len, alphas, n_alphas, max_lag, lags, n_lags);
    if (lag_symmetric)
        cfg.lag_spec = LagSpec::Symmetric(max_lag);
    else
        cfg.lag_spec = LagSpec::Explicit(std::vector<int>(lags, lags + n_lags));
    const auto bad = validate_config(cfg);
    std::string s;
    for (const auto& b : bad) s += b + "\n";
    if (buf && buflen) {
        std::strncpy(buf, s.c_str(), buflen - 1);
        buf[buflen - 1] = 0;
    }
    return static_cast<int>(bad.size());
}

// Signal generators (harness inputs that match the reference bit-for-bit).
int ref_gmsk(std::size_t len, double bt, int sps, std::uint64_t seed, double* out) {
    try {
        CpmParams p;
        p.bt = bt;
        p.sps = sps;
        const auto syms = random_symbols(p.alphabet_size, (len + sps - 1) / sps, seed);
        auto x = cpm_modulate(p, syms);
        x.resize(len);
        store(x, out);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

// CPM record with modulation index h (proj/tests/test_impair.cpp gmsk_record).
int ref_cpm(std::size_t len, double h, double bt, int sps, std::uint64_t seed, double* out) {
    try {
        CpmParams p;
        p.h = h;
        p.bt = bt;
        p.sps = sps;
        const auto syms = random_symbols(p.alphabet_size, (len + sps - 1) / sps, seed);
        auto x = cpm_modulate(p, syms);
        x.resize(len);
        store(x, out);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

// estimate_cfo_ccf (proj/src/impair.cpp:45-115); 4 = NoFeatureError.
int ref_estimate_cfo_ccf(const double* x, std::size_t len, double beta, int N, int frames, double* eps) {
    try {
        *eps = estimate_cfo_ccf(load(x, len), beta, N, frames);
        return 0;
    } catch (const NoFeatureError& e) { return fail(e, 4); }
    catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 5); }
}

CpmParams make_cpm(double h, int M, int L, double bt, int sps, int kind) {
    CpmParams p;
    p.h = h;
    p.alphabet_size = M;
    p.pulse_len = L;
    p.bt = bt;
    p.sps = sps;
    p.pulse_kind = kind == 0 ? PulseKind::GaussianGmsk : PulseKind::Rectangular;
    return p;
}

// random_symbols / make_pulse / cpm_modulate / gmsk_mc_oracle with explicit
// CpmParams (proj/src/siggen.cpp, proj/src/reference.cpp:34-96)
int ref_random_symbols(int M, std::size_t count, std::uint64_t seed, int* out) {
    try {
        const auto s = random_symbols(M, count, seed);
        std::copy(s.begin(), s.end(), out);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

int ref_pulse(double h, int M, int L, double bt, int sps, int kind, double* f, double* g) {
    try {
        const auto t = make_pulse(make_cpm(h, M, L, bt, sps, kind));
        std::copy(t.f.begin(), t.f.end(), f);
        std::copy(t.g.begin(), t.g.end(), g);
        return 0;
    } catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 3); }
}

int ref_cpm_modulate(double h, int M, int L, double bt, int sps, int kind, const int* sym, std::size_t n,
                     double* out) {
    try {
        const auto x = cpm_modulate(make_cpm(h, M, L, bt, sps, kind), std::vector<int>(sym, sym + n));
        store(x, out);
        return 0;
    } catch (const UsageError& e) { return fail(e, 1); }
    catch (const DataError& e) { return fail(e, 3); }
    catch (const std::exception& e) { return fail(e, 5); }
}

int ref_gmsk_mc_oracle(double h, int M, int L, double bt, int sps, int kind, const double* alphas, std::size_t na,
                       const int* lags, std::size_t nl, int conj, int win_len, int trials, std::size_t record_len,
                       std::uint64_t seed, double* out) {
    try {
        const auto t = gmsk_mc_oracle(make_cpm(h, M, L, bt, sps, kind), std::vector<double>(alphas, alphas + na),
                                      std::vector<int>(lags, lags + nl), conj != 0, win_len, trials, record_len, seed);
        std::copy(t.mean_magnitude.begin(), t.mean_magnitude.end(), out);
        return 0;
    } catch (const UsageError& e) { return fail(e, 1); }
    catch (const std::exception& e) { return fail(e, 5); }
}

int ref_tone(double f0, double phi0, std::size_t len, double* out) {
    store(tone(f0, phi0, len), out);
    return 0;
}

int ref_awgn(std::size_t len, double sigma, std::uint64_t seed, double* out) {
    try {
        store(awgn(len, sigma, seed), out);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

int ref_apply_cfo(double* x, std::size_t len, double eps, double phi0) {
    try {
        store(apply_cfo(load(x, len), CfoSpec{eps, phi0}), x);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

int ref_add_noise_snr(double* x, std::size_t len, double snr_db, std::uint64_t seed) {
    try {
        store(add_noise_snr(load(x, len), snr_db, seed), x);
        return 0;
    } catch (const std::exception& e) { return fail(e, 1); }
}

#ifdef REF_HAVE_IO
// export_frames_csv / export_average_csv (io.cpp:161-208) on given values:
// frames = n_frames x layout_len complex (interleaved doubles) with indices
int ref_export_frames_csv(const char* path, int mode, int win_len, const double* alphas, std::size_t n_alphas,
                          int max_lag, const int* lags, std::size_t n_lags, const double* values,
                          const std::uint64_t* frame_index, std::size_t n_frames, std::size_t* rows) {
    try {
        const auto cfg = make_cfg(mode, 0, win_len, alphas, n_alphas, max_lag, lags, n_lags);
        const std::size_t len = mode == 0 ? n_alphas * (2u * (std::size_t)max_lag + 1u) : n_lags * (std::size_t)win_len;
        std::vector<CyclicFrame> frames(n_frames);
        for (std::size_t f = 0; f < n_frames; ++f) {
            frames[f].frame_index = frame_index[f];
            if (mode == 0)
                frames[f].layout = SetLayout{(int)n_alphas, max_lag};
            else
                frames[f].layout = FullLayout{(int)n_lags, win_len};
            frames[f].values = load(values + 2 * f * len, len);
        }
        *rows = export_frames_csv(path, frames, cfg);
        return 0;
    } catch (const UsageError& e) {
        return fail(e, 1);
    } catch (const IoError& e) {
        return fail(e, 6);
    } catch (const std::exception& e) {
        return fail(e, 5);
    }
}

int ref_export_average_csv(const char* path, int mode, int win_len, const double* alphas, std::size_t n_alphas,
                           int max_lag, const int* lags, std::size_t n_lags, const double* avg, std::size_t len,
                           int magnitude, std::size_t* rows) {
    try {
        const auto cfg = make_cfg(mode, 0, win_len, alphas, n_alphas, max_lag, lags, n_lags);
        *rows = export_average_csv(path, load(avg, len), cfg,
                                   magnitude ? AverageMode::Magnitude : AverageMode::Coherent);
        return 0;
    } catch (const UsageError& e) {
        return fail(e, 1);
    } catch (const IoError& e) {
        return fail(e, 6);
    } catch (const std::exception& e) {
        return fail(e, 5);
    }
}
#endif

} // extern "C"

// cycstat_b200.hpp -- header-only C++ drop-in for the reference estimator API
// (/root/reference/proj/include/cycstat/{types,errors,estimator}.hpp) on top of
// the C-ABI in cycb200.h (libcycb200.so, sm_100a).
//
// Same names, argument meaning and error behaviour as the reference:
//   EstimatorConfig / LagSpec / Mode / validate_config     types.hpp:22-66
//   SetLayout / FullLayout / FrameLayout / layout_len /
//   flat_index / full_bin_to_alpha                          types.hpp:68-94
//   CyclicFrame                                             types.hpp:97-104
//   UsageError / ConfigError / IoError / FormatError /
//   DataError / NoFeatureError                              errors.hpp:13-46
//   CyclicCorrelator(cfg), push(x, y) -> vector<CyclicFrame>,
//   buffer_need / consumed / frames_emitted                 estimator.hpp:97-137
//   AverageMode / average_frames                            estimator.hpp:143-148
//   export_frames_csv / export_average_csv                  io.hpp:68-75 (io.cpp:161-208)
//   compute_set_window / compute_full_window                estimator.hpp:59-68
// A caller switches by including this header instead of the reference's and
// linking -lcycb200; `namespace cycstat = cycstat_b200;` is provided when
// CYCSTAT_B200_AS_CYCSTAT is defined (do not also link the reference then).
//
// Extensions (beyond the reference): Mode::Recursive, EstimatorConfig::flags
// (both cyclic functions from one pass), emit_frames = false (block mode,
// read with CyclicCorrelator::average), channels, device.
#ifndef CYCSTAT_B200_HPP
#define CYCSTAT_B200_HPP

#include <algorithm>
#include <complex>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "cycb200.h"

namespace cycstat_b200 {

using cx = std::complex<double>;

// ---- errors (errors.hpp) ----
struct UsageError : std::runtime_error {
    explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : UsageError {  // errors.hpp:17-30: the message joins every violation
    std::vector<std::string> violations;
    explicit ConfigError(std::vector<std::string> v) : UsageError(join(v)), violations(std::move(v)) {}

private:
    static std::string join(const std::vector<std::string>& v) {
        std::string s = "invalid config:";
        for (const auto& e : v) s += " [" + e + "]";
        return s;
    }
};
struct DataError : std::runtime_error {  // errors.hpp:40-42; `index` (extension): the absolute sample, or -1
    std::int64_t index = -1;
    explicit DataError(const std::string& m, std::int64_t i = -1) : std::runtime_error(m), index(i) {}
};
struct NoFeatureError : DataError {  // errors.hpp:44-46
    explicit NoFeatureError(const std::string& m) : DataError(m, -1) {}
};
struct IoError : std::runtime_error {  // errors.hpp:32-34
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct FormatError : IoError {  // errors.hpp:36-38 (malformed input files; caught by proj/tools/main.cpp:157,355)
    explicit FormatError(const std::string& m) : IoError(m) {}
};
struct DeviceError : std::runtime_error {  // no CPU fallback exists
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// ---- types (types.hpp) ----
enum class Mode { Set = CYC_MODE_SET, Full = CYC_MODE_FULL, Recursive = CYC_MODE_RECURSIVE };

struct LagSpec {
    bool symmetric = true;
    int max_lag = 0;
    std::vector<int> lags;
    static LagSpec Symmetric(int m) { LagSpec s; s.symmetric = true; s.max_lag = m; return s; }
    static LagSpec Explicit(std::vector<int> l) { LagSpec s; s.symmetric = false; s.lags = std::move(l); return s; }
    int m_plus() const {
        if (symmetric) return max_lag;
        int m = 0;
        for (int l : lags) m = std::max(m, l);
        return m;
    }
    int m_minus() const {
        if (symmetric) return max_lag;
        int m = 0;
        for (int l : lags) m = std::max(m, -l);
        return m;
    }
    std::vector<int> values() const {
        if (!symmetric) return lags;
        std::vector<int> v(2 * static_cast<std::size_t>(max_lag) + 1);
        std::iota(v.begin(), v.end(), -max_lag);
        return v;
    }
};

struct EstimatorConfig {
    Mode mode = Mode::Set;
    bool conj = false;
    int win_len = 0;
    std::vector<double> alphas;
    LagSpec lag_spec;
    // extensions
    int flags = 0;            // 0: from conj; CYC_FLAG_BOTH: both tables in one pass
    double lambda = 0.0;      // Mode::Recursive
    bool emit_frames = true;  // false: block mode (count + fold; read average())
    int channels = 1;
    int device = 0;
    std::int64_t origin = 0;  // absolute index of the first pushed sample
};

namespace detail {
inline cyc_config to_c(const EstimatorConfig& c) {
    cyc_config r;
    cyc_config_init(&r);
    r.mode = static_cast<int>(c.mode);
    r.conj = c.conj ? 1 : 0;
    r.flags = c.flags;
    r.win_len = c.win_len;
    r.alphas = c.alphas.empty() ? nullptr : c.alphas.data();
    r.num_alphas = c.alphas.size();
    r.lag_symmetric = c.lag_spec.symmetric ? 1 : 0;
    r.max_lag = c.lag_spec.max_lag;
    r.lags = c.lag_spec.lags.empty() ? nullptr : c.lag_spec.lags.data();
    r.num_lags = c.lag_spec.lags.size();
    r.lambda = c.lambda;
    r.emit_frames = c.emit_frames ? 1 : 0;
    r.channels = c.channels;
    r.device = c.device;
    r.origin = c.origin;
    return r;
}
inline std::vector<std::string> split_lines(const std::string& s) {
    std::vector<std::string> v;
    std::size_t p = 0;
    while (p < s.size()) {
        const std::size_t q = s.find('\n', p);
        if (q == std::string::npos) {
            v.push_back(s.substr(p));
            break;
        }
        if (q > p) v.push_back(s.substr(p, q - p));
        p = q + 1;
    }
    return v;
}
}  // namespace detail

// types.cpp:30-63: every violated invariant; empty means ok.
inline std::vector<std::string> validate_config(const EstimatorConfig& cfg) {
    const cyc_config c = detail::to_c(cfg);
    std::string buf(8192, '\0');
    cyc_validate(&c, buf.data(), buf.size());
    return detail::split_lines(buf.c_str());
}

struct SetLayout {
    int num_alphas = 0;
    int max_lag = 0;
    bool operator==(const SetLayout&) const = default;
};
struct FullLayout {
    int num_lags = 0;
    int win_len = 0;
    bool operator==(const FullLayout&) const = default;
};
using FrameLayout = std::variant<SetLayout, FullLayout>;

inline std::size_t layout_len(const FrameLayout& l) {
    if (auto s = std::get_if<SetLayout>(&l)) return static_cast<std::size_t>(s->num_alphas) * (2u * s->max_lag + 1u);
    const auto& f = std::get<FullLayout>(l);
    return static_cast<std::size_t>(f.num_lags) * f.win_len;
}
inline std::size_t flat_index(const SetLayout& l, int a, int lag) {
    if (a < 0 || a >= l.num_alphas) throw std::out_of_range("cycle-frequency index out of range");
    if (lag < -l.max_lag || lag > l.max_lag) throw std::out_of_range("lag out of range");
    return static_cast<std::size_t>(a) * (2u * l.max_lag + 1u) + static_cast<std::size_t>(lag + l.max_lag);
}
inline std::size_t flat_index(const FullLayout& l, int li, int bin) {
    if (li < 0 || li >= l.num_lags) throw std::out_of_range("lag index out of range");
    if (bin < 0 || bin >= l.win_len) throw std::out_of_range("DFT bin out of range");
    return static_cast<std::size_t>(li) * l.win_len + static_cast<std::size_t>(bin);
}
inline double full_bin_to_alpha(int k, int n) {
    if (n <= 0 || k < 0 || k >= n) throw std::out_of_range("DFT bin out of range");
    const double a = static_cast<double>(k) / n;
    return (2 * k < n) ? a : a - 1.0;
}

struct CyclicFrame {
    std::uint64_t frame_index = 0;
    std::uint64_t start_abs = 0;
    FrameLayout layout;
    std::vector<cx> values;
    int flag = CYC_FLAG_CONV;  // extension: which cyclic function
    int channel = 0;           // extension
};

enum class AverageMode { Coherent = CYC_AVG_COHERENT, Magnitude = CYC_AVG_MAGNITUDE };

namespace detail {
[[noreturn]] inline void raise(int code, const std::string& msg, std::int64_t index = -1) {
    if (code == CYC_ERR_CONFIG) {
        std::vector<std::string> v;
        std::size_t p = 0;
        while ((p = msg.find('[', p)) != std::string::npos) {
            const std::size_t q = msg.find(']', p);
            v.push_back(msg.substr(p + 1, q - p - 1));
            p = q;
        }
        throw ConfigError(std::move(v));  // same message: "invalid config: [..] [..]"
    }
    if (code == CYC_ERR_USAGE) throw UsageError(msg);
    if (code == CYC_ERR_DATA) throw DataError(msg, index);
    if (code == CYC_ERR_CUDA) throw DeviceError(msg);
    if (code == CYC_ERR_IO) throw IoError(msg);
    if (code == CYC_ERR_FORMAT) throw FormatError(msg);
    throw std::logic_error(msg);
}
}  // namespace detail

// ---- the estimator (estimator.hpp:97-137) ----
class CyclicCorrelator {
public:
    explicit CyclicCorrelator(const EstimatorConfig& cfg) : cfg_(cfg) {
        const cyc_config c = detail::to_c(cfg);
        std::string err(8192, '\0');
        const int rc = cyc_create(&c, &h_, err.data(), err.size());
        if (rc) detail::raise(rc, err.c_str());
        cyc_layout_info li;
        cyc_layout(h_, &li);
        if (li.kind == 1)
            layout_ = FullLayout{li.num_lags, li.win_len};
        else
            layout_ = SetLayout{li.num_alphas, li.max_lag};
    }
    ~CyclicCorrelator() { cyc_destroy(h_); }
    CyclicCorrelator(const CyclicCorrelator&) = delete;
    CyclicCorrelator& operator=(const CyclicCorrelator&) = delete;
    CyclicCorrelator(CyclicCorrelator&& o) noexcept : cfg_(o.cfg_), layout_(o.layout_), h_(o.h_) { o.h_ = nullptr; }

    // estimator.hpp:102-107 (complex<double> samples, as the reference)
    std::vector<CyclicFrame> push(const std::vector<cx>& x, const std::vector<cx>& y) {
        if (x.size() != y.size()) throw UsageError("x and y chunks must have equal length");
        const bool same = &x == &y || x.data() == y.data();
        return run([&](cyc_frame_sink s, void* u) {
            return cyc_push_f64(h_, reinterpret_cast<const cyc_cf64*>(x.data()),
                                same ? nullptr : reinterpret_cast<const cyc_cf64*>(y.data()),
                                x.size() / static_cast<std::size_t>(cfg_.channels), s, u);
        });
    }
    // complex64 samples (cf32 interchange, proj/src/io.cpp:74-103); y == nullptr: auto
    std::vector<CyclicFrame> push(const std::complex<float>* x, const std::complex<float>* y, std::size_t n) {
        return run([&](cyc_frame_sink s, void* u) {
            return cyc_push(h_, reinterpret_cast<const cyc_cf32*>(x), reinterpret_cast<const cyc_cf32*>(y), n, s, u);
        });
    }

    // read_cf32 (io.cpp:90-103) + push of the whole file, y auto
    std::vector<CyclicFrame> push_file(const std::string& path) {
        return run([&](cyc_frame_sink s, void* u) { return cyc_push_cf32_file(h_, path.c_str(), s, u); });
    }

    // Pipelined emission (cyc_set_emit_pipeline; no reference counterpart): with
    // depth 1 or 2 a push that completes frames only enqueues them and a later push
    // (or flush_frames) returns them, same order and values.
    void set_emit_pipeline(int depth) {
        const int rc = cyc_set_emit_pipeline(h_, depth);
        if (rc) detail::raise(rc, cyc_last_error(h_), cyc_data_error_index(h_));
    }
    std::vector<CyclicFrame> flush_frames() {
        return run([&](cyc_frame_sink s, void* u) { return cyc_flush_frames(h_, s, u); });
    }

    // average_frames over every frame emitted so far, without materialising them
    std::vector<cx> average(AverageMode mode = AverageMode::Coherent, int flag = 0, int channel = 0) {
        std::vector<cx> out(layout_len(layout_));
        const int rc = cyc_average(h_, static_cast<int>(mode), flag, channel, reinterpret_cast<cyc_cf64*>(out.data()));
        if (rc) detail::raise(rc, cyc_last_error(h_), cyc_data_error_index(h_));
        return out;
    }

    const EstimatorConfig& config() const { return cfg_; }
    FrameLayout layout() const { return layout_; }
    std::size_t buffer_need() const { return cyc_buffer_need(h_); }
    std::uint64_t consumed() const { return cyc_consumed(h_); }
    std::uint64_t frames_emitted() const { return cyc_frames_emitted(h_); }

private:
    template <typename F>
    std::vector<CyclicFrame> run(F&& call) {
        struct Ctx {
            std::vector<CyclicFrame>* out;
            FrameLayout layout;
        };
        std::vector<CyclicFrame> frames;
        Ctx ctx{&frames, layout_};
        auto sink = [](void* user, const cyc_frame_view* v) -> int {
            Ctx* c = static_cast<Ctx*>(user);
            CyclicFrame f;
            f.frame_index = v->frame_index;
            f.start_abs = v->start_abs;
            f.layout = c->layout;
            f.values.assign(reinterpret_cast<const cx*>(v->values), reinterpret_cast<const cx*>(v->values) + v->len);
            f.flag = v->flag;
            f.channel = v->channel;
            c->out->push_back(std::move(f));
            return 0;
        };
        const int rc = call(+sink, &ctx);
        if (rc) detail::raise(rc, cyc_last_error(h_), cyc_data_error_index(h_));
        return frames;
    }

    EstimatorConfig cfg_;
    FrameLayout layout_;
    cyc_est* h_ = nullptr;
};

// estimator.cpp:86-105 over materialised frames (host-side)
inline std::vector<cx> average_frames(const std::vector<CyclicFrame>& frames, AverageMode mode) {
    if (frames.empty()) throw UsageError("cannot average an empty frame list");
    const std::size_t len = frames.front().values.size();
    std::vector<cx> out(len, cx(0.0, 0.0));
    for (const auto& f : frames) {
        if (f.layout.index() != frames.front().layout.index() || f.values.size() != len)
            throw UsageError("cannot average frames with mixed layouts");
        for (std::size_t i = 0; i < len; ++i) out[i] += mode == AverageMode::Coherent ? f.values[i] : cx(std::abs(f.values[i]));
    }
    for (auto& v : out) v /= static_cast<double>(frames.size());
    return out;
}

// io.cpp:161-208: the CSV result writers (same headers and "%.17g" rows)
inline std::size_t export_frames_csv(const std::string& path, const std::vector<CyclicFrame>& frames,
                                     const EstimatorConfig& cfg) {
    if (frames.empty()) throw UsageError("no frames to export");
    const std::size_t len = frames.front().values.size();
    std::vector<cx> vals;
    std::vector<std::uint64_t> idx;
    vals.reserve(frames.size() * len);
    for (const auto& f : frames) {
        if (f.layout.index() != frames.front().layout.index() || f.values.size() != len)
            throw UsageError("cannot export frames with mixed layouts");
        vals.insert(vals.end(), f.values.begin(), f.values.end());
        idx.push_back(f.frame_index);
    }
    const cyc_config c = detail::to_c(cfg);
    std::size_t rows = 0;
    std::string err(1024, '\0');
    const int rc = cyc_export_frames_csv(&c, path.c_str(), idx.data(), reinterpret_cast<const cyc_cf64*>(vals.data()),
                                         frames.size(), &rows, err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    if (rows != vals.size()) throw UsageError("config does not match the frame layout");
    return rows;
}
inline std::size_t export_average_csv(const std::string& path, const std::vector<cx>& avg, const EstimatorConfig& cfg,
                                      AverageMode mode) {
    const cyc_config c = detail::to_c(cfg);
    std::size_t rows = 0;
    std::string err(1024, '\0');
    const int rc = cyc_export_average_csv(&c, path.c_str(), reinterpret_cast<const cyc_cf64*>(avg.data()), avg.size(),
                                          (int)mode, &rows, err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return rows;
}

// kernels.cpp:116-135 on the device
inline std::vector<cx> compute_set_window(const std::vector<cx>& xw, const std::vector<cx>& yw,
                                          const std::vector<double>& alphas, int max_lag, bool conj, std::uint64_t k0) {
    std::vector<cx> out(alphas.size() * (2u * static_cast<std::size_t>(max_lag) + 1u));
    std::string err(1024, '\0');
    const int rc = cyc_compute_set_window(reinterpret_cast<const cyc_cf64*>(xw.data()), xw.size(),
                                          reinterpret_cast<const cyc_cf64*>(yw.data()), yw.size(), alphas.data(),
                                          alphas.size(), max_lag, conj ? 1 : 0, k0,
                                          reinterpret_cast<cyc_cf64*>(out.data()), err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return out;
}
inline std::vector<cx> compute_full_window(const std::vector<cx>& xw, const std::vector<cx>& yw,
                                           const std::vector<int>& lags, bool conj, std::uint64_t k0) {
    std::vector<cx> out(lags.size() * yw.size());
    std::string err(1024, '\0');
    const int rc = cyc_compute_full_window(reinterpret_cast<const cyc_cf64*>(xw.data()), xw.size(),
                                           reinterpret_cast<const cyc_cf64*>(yw.data()), yw.size(), lags.data(),
                                           lags.size(), conj ? 1 : 0, k0, reinterpret_cast<cyc_cf64*>(out.data()),
                                           err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return out;
}

// ---- CPM / GMSK generation and the Monte-Carlo oracle (siggen.hpp, reference.hpp) ----
enum class PulseKind { GaussianGmsk = CYC_PULSE_GAUSSIAN, Rectangular = CYC_PULSE_RECT };
struct CpmParams {  // siggen.hpp:16-23
    double h = 0.5;
    int alphabet_size = 2;
    int pulse_len = 4;
    double bt = 0.25;
    int sps = 8;
    PulseKind pulse_kind = PulseKind::GaussianGmsk;
};
struct PulseTable {  // siggen.hpp:27-30
    std::vector<double> f;
    std::vector<double> g;
};
struct OracleTable {  // reference.hpp:15-28
    std::vector<double> alphas;
    std::vector<int> lags;
    std::vector<double> mean_magnitude;
    int trials = 0;
    std::size_t record_len = 0;
    std::uint64_t seed = 0;
    double cell(std::size_t a, std::size_t l) const { return mean_magnitude[a * lags.size() + l]; }
};
namespace detail {
inline cyc_cpm_params to_c(const CpmParams& p) {
    cyc_cpm_params c;
    c.h = p.h;
    c.alphabet_size = p.alphabet_size;
    c.pulse_len = p.pulse_len;
    c.bt = p.bt;
    c.sps = p.sps;
    c.pulse_kind = static_cast<int>(p.pulse_kind);
    return c;
}
}  // namespace detail
inline std::vector<int> random_symbols(int alphabet_size, std::size_t count, std::uint64_t seed) {
    std::vector<int> out(count);
    std::string err(1024, '\0');
    const int rc = cyc_random_symbols(alphabet_size, count, seed, out.data(), err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return out;
}
inline PulseTable make_pulse(const CpmParams& params) {
    const cyc_cpm_params c = detail::to_c(params);
    const std::size_t n = params.pulse_len > 0 && params.sps > 0 ? (std::size_t)params.pulse_len * params.sps : 0;
    PulseTable t;
    t.f.resize(n);
    t.g.resize(n);
    std::string err(1024, '\0');
    const int rc = cyc_cpm_pulse(&c, t.f.data(), t.g.data(), n, err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return t;
}
// siggen.cpp:111-145 on the device (fp64 samples, as the reference returns)
inline std::vector<cx> cpm_modulate(const CpmParams& params, const std::vector<int>& symbols, int device = 0) {
    const cyc_cpm_params c = detail::to_c(params);
    std::vector<cx> out(symbols.size() * (std::size_t)std::max(params.sps, 0));
    std::string err(1024, '\0');
    const int rc = cyc_cpm_modulate(&c, symbols.data(), symbols.size(), device, 1, out.data(), err.data(), err.size());
    if (rc) detail::raise(rc, err.c_str());
    return out;
}
// reference.cpp:34-96 on the device
inline OracleTable gmsk_mc_oracle(const CpmParams& params, const std::vector<double>& alphas,
                                  const std::vector<int>& lags, bool conj, int win_len, int trials,
                                  std::size_t record_len, std::uint64_t seed, int device = 0) {
    const cyc_cpm_params c = detail::to_c(params);
    OracleTable t;
    t.alphas = alphas;
    t.lags = lags;
    t.trials = trials;
    t.record_len = record_len;
    t.seed = seed;
    t.mean_magnitude.assign(std::max<std::size_t>(alphas.size() * lags.size(), 1), 0.0);
    std::string err(1024, '\0');
    const int rc = cyc_gmsk_mc_oracle(&c, alphas.data(), alphas.size(), lags.data(), lags.size(), conj ? 1 : 0,
                                      win_len, trials, record_len, seed, device, t.mean_magnitude.data(), err.data(),
                                      err.size());
    if (rc) detail::raise(rc, err.c_str());
    t.mean_magnitude.resize(alphas.size() * lags.size());
    return t;
}

// impair.cpp:45-115 on the device
inline double estimate_cfo_ccf(const std::vector<cx>& x, double expected_beta, int N, int num_frames,
                               int device = 0) {
    std::vector<std::complex<float>> xf(x.begin(), x.end());
    double eps = 0.0;
    std::string err(1024, '\0');
    const int rc = cyc_estimate_cfo_ccf(reinterpret_cast<const cyc_cf32*>(xf.data()), xf.size(), expected_beta, N,
                                        num_frames, device, &eps, err.data(), err.size());
    if (rc == CYC_ERR_DATA && std::string(err.c_str()).rfind("no feature", 0) == 0) throw NoFeatureError(err.c_str());
    if (rc) detail::raise(rc, err.c_str());
    return eps;
}

}  // namespace cycstat_b200

#ifdef CYCSTAT_B200_AS_CYCSTAT
namespace cycstat = cycstat_b200;
#endif

#endif  // CYCSTAT_B200_HPP

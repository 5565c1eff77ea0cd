// consumers.cpp -- the callers and data formats on either side of the hot path
// (SURVEY §8 f2, f3), built on the engine:
//   * cyc_push_cf32_file: the cf32 interchange format (proj/src/io.cpp:74-103)
//     streamed from the page cache into the device rings -- no fp64 copy of
//     the record (the reference's read_cf32 materialises one);
//   * cyc_export_frames_csv / cyc_export_average_csv: the CSV result formats
//     (proj/src/io.cpp:161-208);
//   * cyc_estimate_cfo_ccf: the CFO estimator (proj/src/impair.cpp:45-115) --
//     a conjugate Full-mode lag-0 scan whose magnitude average is computed on
//     the device, then the reference's peak search / median test / log-parabola
//     refinement on the host (N values).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "engine.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "cf32 is little-endian; raw mapping needs an LE host");

namespace {

void write_msg(char* buf, size_t len, const std::string& m) {
    if (!buf || !len) return;
    std::strncpy(buf, m.c_str(), len - 1);
    buf[len - 1] = 0;
}

int fail(cyc_est* est, int code, const std::string& msg, int64_t index = -1) {
    if (est) {
        est->e->last_error = msg;
        est->e->last_error_index = index;
    }
    return code;
}

// "%.17g" (io.cpp:37-41): round-trips every double
std::string fmt17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

// (alpha, lag) of flat element idx (io.cpp:43-53; the recursive mode's
// alpha-major lag-list layout alike)
std::pair<double, int> element_coords(const cyc::Cfg& c, size_t idx) {
    if (c.mode == CYC_MODE_SET) {
        const size_t row = 2u * (size_t)c.max_lag + 1u;
        return {c.alphas[idx / row], (int)(idx % row) - c.max_lag};
    }
    if (c.mode == CYC_MODE_FULL) {
        const size_t n = (size_t)c.win_len;
        const int k = (int)(idx % n);
        const double a = (2 * (int64_t)k >= (int64_t)n) ? (double)k / (double)n - 1.0 : (double)k / (double)n;
        return {a, c.lags[idx / n]};
    }
    const size_t t = c.lags.size();
    return {c.alphas[idx / t], c.lags[idx % t]};
}

// config_layout_len (io.cpp:55-59; the recursive mode: alphas x lags)
size_t layout_len_of(const cyc::Cfg& c) {
    if (c.mode == CYC_MODE_SET) return c.alphas.size() * (2u * (size_t)c.max_lag + 1u);
    if (c.mode == CYC_MODE_FULL) return c.lags.size() * (size_t)c.win_len;
    return c.alphas.size() * c.lags.size();
}

int config_of(const cyc_config* cc, cyc::Cfg& c, char* err, size_t errlen) {
    if (!cc) {
        write_msg(err, errlen, "null config");
        return CYC_ERR_USAGE;
    }
    c = cyc::from_c(cc);
    const auto v = cyc::validate(c);
    if (!v.empty()) {
        std::string m = "invalid config:";
        for (const auto& e : v) m += " [" + e + "]";
        write_msg(err, errlen, m);
        return CYC_ERR_CONFIG;
    }
    return CYC_OK;
}

// open_out / finish_out (io.cpp:61-70)
struct CsvOut {
    FILE* f = nullptr;
    std::string path;
    std::string buf;
    ~CsvOut() {
        if (f) std::fclose(f);
    }
    void row(const std::string& s) {
        buf += s;
        if (buf.size() > (1u << 20)) flush();
    }
    bool flush() {
        if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) return false;
        buf.clear();
        return true;
    }
};

int open_csv(CsvOut& o, const char* path, char* err, size_t errlen) {
    o.path = path ? path : "";
    o.f = path ? std::fopen(path, "wb") : nullptr;
    if (!o.f) {
        write_msg(err, errlen, "cannot open " + o.path + " for writing");
        return CYC_ERR_IO;
    }
    return CYC_OK;
}

int close_csv(CsvOut& o, char* err, size_t errlen) {
    const bool ok = o.flush() && std::fflush(o.f) == 0 && std::fclose(o.f) == 0;
    o.f = nullptr;
    if (!ok) {
        write_msg(err, errlen, "write to " + o.path + " failed");
        return CYC_ERR_IO;
    }
    return CYC_OK;
}

}  // namespace

extern "C" {

// export_frames_csv (io.cpp:161-186)
int cyc_export_frames_csv(const cyc_config* cfg, const char* path, const uint64_t* frame_index,
                          const cyc_cf64* values, size_t n_frames, size_t* rows, char* err, size_t errlen) {
    if (rows) *rows = 0;
    cyc::Cfg c;
    if (int rc = config_of(cfg, c, err, errlen)) return rc;
    if (n_frames == 0 || !values || !frame_index) {
        write_msg(err, errlen, "no frames to export");
        return CYC_ERR_USAGE;
    }
    const size_t len = layout_len_of(c);
    CsvOut o;
    if (int rc = open_csv(o, path, err, errlen)) return rc;
    o.row("frame_index,alpha,lag,re,im,mag\n");
    for (size_t f = 0; f < n_frames; ++f)
        for (size_t i = 0; i < len; ++i) {
            const auto ac = element_coords(c, i);
            const cyc_cf64 v = values[f * len + i];
            o.row(std::to_string(frame_index[f]) + ',' + fmt17(ac.first) + ',' + std::to_string(ac.second) + ',' +
                  fmt17(v.re) + ',' + fmt17(v.im) + ',' + fmt17(std::hypot(v.re, v.im)) + '\n');
        }
    if (int rc = close_csv(o, err, errlen)) return rc;
    if (rows) *rows = n_frames * len;
    return CYC_OK;
}

// export_average_csv (io.cpp:188-208)
int cyc_export_average_csv(const cyc_config* cfg, const char* path, const cyc_cf64* avg, size_t len, int avg_mode,
                           size_t* rows, char* err, size_t errlen) {
    if (rows) *rows = 0;
    cyc::Cfg c;
    if (int rc = config_of(cfg, c, err, errlen)) return rc;
    if (len == 0 || !avg) {
        write_msg(err, errlen, "no averaged values to export");
        return CYC_ERR_USAGE;
    }
    if (len != layout_len_of(c)) {
        write_msg(err, errlen, "config does not match the averaged vector length");
        return CYC_ERR_USAGE;
    }
    const bool coh = avg_mode == CYC_AVG_COHERENT;
    CsvOut o;
    if (int rc = open_csv(o, path, err, errlen)) return rc;
    o.row(coh ? "alpha,lag,mean_re,mean_im,mean_mag\n" : "alpha,lag,mean_mag\n");
    for (size_t i = 0; i < len; ++i) {
        const auto ac = element_coords(c, i);
        std::string r = fmt17(ac.first) + ',' + std::to_string(ac.second) + ',';
        if (coh)
            r += fmt17(avg[i].re) + ',' + fmt17(avg[i].im) + ',' + fmt17(std::hypot(avg[i].re, avg[i].im)) + '\n';
        else
            r += fmt17(avg[i].re) + '\n';
        o.row(r);
    }
    if (int rc = close_csv(o, err, errlen)) return rc;
    if (rows) *rows = len;
    return CYC_OK;
}

// read_cf32 + push (proj/src/io.cpp:90-103, proj/tools/main.cpp:212-214): the
// whole file is one chunk -- validated whole before any state change.
int cyc_push_cf32_file(cyc_est* est, const char* path, cyc_frame_sink sink, void* user) {
    if (!est || !path) return CYC_ERR_USAGE;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return fail(est, CYC_ERR_IO, std::string("cannot open ") + path + " for reading");
    struct stat st;
    if (::fstat(fd, &st) != 0) {
        ::close(fd);
        return fail(est, CYC_ERR_IO, std::string("read from ") + path + " failed");
    }
    const size_t bytes = (size_t)st.st_size;
    if (bytes % 8 != 0) {
        ::close(fd);
        return fail(est, CYC_ERR_FORMAT, std::string(path) + " is truncated: length is not a multiple of 8 bytes");
    }
    const int C = 1;  // one stream per file (multi-channel callers push arrays)
    const size_t n = bytes / 8;
    if (n == 0) {
        ::close(fd);
        return CYC_OK;
    }
    void* p = ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
    ::close(fd);
    if (p == MAP_FAILED) return fail(est, CYC_ERR_IO, std::string("read from ") + path + " failed");
    ::madvise(p, bytes, MADV_SEQUENTIAL);
    (void)C;
    cyc::Status s = est->e->validate_host_f32(p, nullptr, n);
    if (!s.code) s = est->e->push(p, nullptr, n, cyc::Engine::IN_HOST_F32, sink, user);
    ::munmap(p, bytes);
    est->e->last_error = s.msg;
    est->e->last_error_index = s.index;
    return s.code;
}

// estimate_cfo_ccf (proj/src/impair.cpp:45-115).
int cyc_estimate_cfo_ccf(const cyc_cf32* x, size_t n, double expected_beta, int N, int num_frames, int device,
                         double* eps_out, char* err, size_t errlen) {
    if (num_frames < 1) {
        write_msg(err, errlen, "need at least one frame for the scan");
        return CYC_ERR_USAGE;
    }
    if (!(expected_beta >= -0.5 && expected_beta < 0.5)) {
        write_msg(err, errlen, "expected conjugate cycle frequency must lie in [-1/2, 1/2)");
        return CYC_ERR_USAGE;
    }
    // The scan's estimator is kept per (N, device) and thread across calls:
    // its set-up (rings, pinned staging) costs far more than one scan.
    struct Cache {
        int N = 0, device = -1;
        cyc_est* est = nullptr;
        ~Cache() {  // a worker thread's estimator is freed when the thread exits
            if (est) cyc_destroy(est);
        }
    };
    static thread_local Cache cache_obj;
    Cache* cache = &cache_obj;
    if (!cache->est || cache->N != N || cache->device != device) {
        if (cache->est) cyc_destroy(cache->est);
        cache->est = nullptr;
        cyc_config c;
        cyc_config_init(&c);
        c.mode = CYC_MODE_FULL;
        c.conj = 1;
        c.win_len = N;
        c.lag_symmetric = 0;
        const int lag0 = 0;
        c.lags = &lag0;
        c.num_lags = 1;
        c.device = device;
        const int rc = cyc_create(&c, &cache->est, err, errlen);  // validates N (impair.cpp:56)
        if (rc) return rc;
        cache->N = N;
        cache->device = device;
    }
    cyc_est* est = cache->est;
    if (int rc = cyc_reset(est)) {
        write_msg(err, errlen, cyc_last_error(est));
        return rc;
    }
    const size_t need = (size_t)N * (size_t)num_frames;
    if (!x || n < need) {
        write_msg(err, errlen, "record too short for the requested number of frames");
        return CYC_ERR_USAGE;
    }
    // exactly num_frames frames (impair.cpp:62-63: frames.resize(num_frames))
    int code = cyc_push(est, x, nullptr, need, nullptr, nullptr);
    // The reference pushes the whole record (estimator.cpp:44-51 validates it
    // all); samples past the last scanned frame are only checked.
    for (size_t i = need; !code && i < n; ++i) {
        if (!std::isfinite(x[i].re) || !std::isfinite(x[i].im)) {
            write_msg(err, errlen, "non-finite sample at absolute index " + std::to_string(i) + " in x stream");
            return CYC_ERR_DATA;
        }
    }
    std::vector<cyc_cf64> avg((size_t)N);
    if (!code) code = cyc_average(est, CYC_AVG_MAGNITUDE, CYC_FLAG_CONJ, 0, avg.data());
    if (code) {
        write_msg(err, errlen, cyc_last_error(est));
        return code;
    }
    std::vector<double> mag((size_t)N);
    for (int k = 0; k < N; ++k) mag[(size_t)k] = avg[(size_t)k].re;

    // Peak search strictly inside +-N/8 bins of the expected feature (impair.cpp:68-86).
    const auto wrap_bin = [N](long long k) {
        long long r = k % N;
        if (r < 0) r += N;
        return (size_t)r;
    };
    const long long bin_e = std::llround(expected_beta * N);
    const long long half_span = N / 8;
    size_t k_peak = wrap_bin(bin_e);
    std::vector<double> window;
    for (long long k = bin_e - half_span + 1; k <= bin_e + half_span - 1; ++k) {
        const size_t kk = wrap_bin(k);
        window.push_back(mag[kk]);
        if (mag[kk] > mag[k_peak]) k_peak = kk;
    }
    // Median test (impair.cpp:88-97) -> NoFeatureError (a DataError).
    std::nth_element(window.begin(), window.begin() + window.size() / 2, window.end());
    const double median = window[window.size() / 2];
    if (!(mag[k_peak] > 3.0 * median)) {
        write_msg(err, errlen, "no feature detected at the expected conjugate cycle frequency");
        return CYC_ERR_DATA;
    }
    // Log-parabola refinement (impair.cpp:99-108).
    const double l0 = mag[k_peak];
    const double lm = mag[wrap_bin((long long)k_peak - 1)];
    const double lp = mag[wrap_bin((long long)k_peak + 1)];
    double delta = 0.0;
    if (lm > 0.0 && l0 > 0.0 && lp > 0.0) {
        const double a = std::log(lm), b = std::log(l0), cc = std::log(lp);
        const double den = a - 2.0 * b + cc;
        if (den < 0.0) delta = std::clamp(0.5 * (a - cc) / den, -0.5, 0.5);
    }
    double beta_peak = ((double)k_peak + delta) / N;
    if (beta_peak >= 0.5) beta_peak -= 1.0;
    double diff = beta_peak - expected_beta;
    diff -= std::round(diff);  // shortest wrapped distance (impair.cpp:113)
    if (eps_out) *eps_out = diff / 2.0;
    write_msg(err, errlen, "");
    return CYC_OK;
}

}  // extern "C"

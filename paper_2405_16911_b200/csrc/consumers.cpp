// consumers.cpp -- the callers and data formats on either side of the hot path
// (SURVEY §8 f2, f3), built on the engine:
//   * cyc_push_cf32_file: the cf32 interchange format (proj/src/io.cpp:74-103)
//     streamed from the page cache into the device rings -- no fp64 copy of
//     the record (the reference's read_cf32 materialises one);
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
#include <cstring>
#include <string>
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

}  // namespace

extern "C" {

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

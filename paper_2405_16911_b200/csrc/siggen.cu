// siggen.cu -- SURVEY §8 f4: CPM / GMSK generation on the device and the
// Monte-Carlo cyclic-magnitude oracle built on the estimator.
//
//   cyc_random_symbols   random_symbols (proj/src/siggen.cpp:147-157): the same
//                        std::mt19937_64 draw, so symbol streams are identical
//   cyc_cpm_pulse        gaussian_freq_pulse / rect_freq_pulse + the exact
//                        half-area renormalisation (proj/src/siggen.cpp:30-110)
//   cyc_cpm_modulate     cpm_modulate (proj/src/siggen.cpp:111-145) with one
//                        thread per sample: the completed-symbol phase comes
//                        from an exclusive prefix sum of the integer symbols
//                        (phase = pi*h*S mod 2 pi, reduced in units of pi), the
//                        active symbols add 2 pi h a_k g[n - k sps]; fp64 phase,
//                        cf32 (or cf64) output
//   cyc_gmsk_mc_oracle   gmsk_mc_oracle (proj/src/reference.cpp:34-96): per
//                        trial, symbols at seed + t, modulated on the device,
//                        then the estimator's per-frame magnitude average over
//                        the windows k0 = m_minus + j N (Set mode, lags -M..M,
//                        origin = M - m_minus puts frame j at sample k0),
//                        summed over trials in trial order
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "engine.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr double kLn2 = 0.69314718055994530942;

void write_msg(char* buf, size_t len, const std::string& m) {
    if (!buf || !len) return;
    std::strncpy(buf, m.c_str(), len - 1);
    buf[len - 1] = 0;
}

// check_params (proj/src/siggen.cpp:21-29): same order, same messages
std::string check_params(const cyc_cpm_params& p) {
    if (!(p.h > 0.0)) return "modulation index must be positive";
    if (p.alphabet_size < 2 || p.alphabet_size % 2 != 0) return "alphabet size must be even and at least 2";
    if (p.pulse_len < 1) return "pulse length must be at least 1 symbol";
    if (p.sps < 1) return "samples per symbol must be at least 1";
    if (p.pulse_kind == CYC_PULSE_GAUSSIAN && !(p.bt > 0.0)) return "bandwidth-time product must be positive";
    return "";
}

double qfunc(double x) { return 0.5 * std::erfc(x / kSqrt2); }

// Scale to a left-to-right sum of exactly 1/2, retuning tail samples (the
// reference's renormalize_half).  Returns "" or the DataError message.
std::string renormalize_half(std::vector<double>& f) {
    double s = 0.0;
    for (double v : f) s += v;
    if (!(s > 0.0) || !std::isfinite(s)) return "frequency pulse degenerated to zero area";
    const double scale = 0.5 / s;
    for (double& v : f) v *= scale;
    for (size_t k = f.size(); k-- > 0;) {
        double head = 0.0;
        for (size_t i = 0; i < k; ++i) head += f[i];
        const double r = 0.5 - head;
        if (r < 0.0) continue;
        f[k] = r;
        std::fill(f.begin() + (std::ptrdiff_t)k + 1, f.end(), 0.0);
        double total = head;
        for (size_t i = k; i < f.size(); ++i) total += f[i];
        if (total == 0.5) return "";
    }
    return "frequency pulse normalization failed to converge";
}

// make_pulse: f (frequency pulse) and g (its running sum), length L*sps.
std::string make_pulse(const cyc_cpm_params& p, std::vector<double>& f, std::vector<double>& g) {
    const int len = p.pulse_len * p.sps;
    f.assign((size_t)len, 0.0);
    if (p.pulse_kind == CYC_PULSE_RECT) {
        std::fill(f.begin(), f.end(), 0.5 / len);
    } else {
        const double c = kTwoPi * p.bt / std::sqrt(kLn2);
        const double half_span = 0.5 * p.pulse_len;
        for (int i = 0; i < len; ++i) {
            const double tau = (i + 0.5) / p.sps;  // midpoint sampling
            f[(size_t)i] = 0.5 * (qfunc(c * (tau - half_span - 0.5)) - qfunc(c * (tau - half_span + 0.5))) / p.sps;
        }
    }
    const std::string m = renormalize_half(f);
    if (!m.empty()) return m;
    g.resize(f.size());
    double acc = 0.0;
    for (size_t i = 0; i < f.size(); ++i) {
        acc += f[i];
        g[i] = acc;
    }
    return "";
}

// phi[n] = pi * (frac(h*S_first / 2) * 2) + 2 pi h sum_{k active} a_k g[n - k sps]
// S_first = sum of the symbols completed before sample n (exclusive prefix).
// blockIdx.y = record r of a batch: symbols at sym + r*n_sym, prefix sums at
// prefix + r*(n_sym+1), samples at out + r*n_out.
__global__ void cpm_kernel(const int* __restrict__ sym_all, const long long* __restrict__ prefix_all,
                           const double* __restrict__ g, int sps, int L, double h, size_t n_sym, size_t n_out,
                           void* out_all, int f64) {
    const int* sym = sym_all + (size_t)blockIdx.y * n_sym;
    const long long* prefix = prefix_all + (size_t)blockIdx.y * (n_sym + 1);
    void* out = f64 ? (void*)(reinterpret_cast<double2*>(out_all) + (size_t)blockIdx.y * n_out)
                    : (void*)(reinterpret_cast<float2*>(out_all) + (size_t)blockIdx.y * n_out);
    for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < n_out; n += (size_t)gridDim.x * blockDim.x) {
        const long long cur = (long long)(n / (size_t)sps);
        const long long first = cur - L + 1;
        const long long f0 = first > 0 ? first : 0;
        // completed symbols contribute pi*h*a each: reduce h*S modulo 2 (units of pi)
        const double hs = h * (double)prefix[f0];
        double phi = kTwoPi * 0.5 * (hs - 2.0 * floor(hs * 0.5));
        double act = 0.0;
        for (long long k = f0; k <= cur; ++k) act += (double)sym[k] * g[n - (size_t)k * (size_t)sps];
        phi += kTwoPi * h * act;
        double s, c;
        sincos(phi, &s, &c);
        if (f64)
            reinterpret_cast<double2*>(out)[n] = make_double2(c, s);
        else
            reinterpret_cast<float2*>(out)[n] = make_float2((float)c, (float)s);
    }
}

// Modulate `records` streams of `n_sym` symbols each (host, concatenated) into
// `n_out` samples per record (n_out <= n_sym * sps) at `out` (device memory,
// record-major).  The exclusive prefix sums are formed on the host.
int modulate_device(const cyc_cpm_params& p, const int* symbols, size_t n_sym, size_t records, size_t n_out,
                    void* out, int f64, cudaStream_t st, std::string& msg) {
    std::vector<double> f, g;
    msg = make_pulse(p, f, g);
    if (!msg.empty()) return CYC_ERR_DATA;
    std::vector<long long> prefix(records * (n_sym + 1));
    for (size_t r = 0; r < records; ++r) {
        long long acc = 0;
        for (size_t i = 0; i < n_sym; ++i) {
            prefix[r * (n_sym + 1) + i] = acc;
            acc += symbols[r * n_sym + i];
        }
        prefix[r * (n_sym + 1) + n_sym] = acc;
    }
    int* d_sym = nullptr;
    long long* d_pre = nullptr;
    double* d_g = nullptr;
    cudaError_t e = cudaMallocAsync(&d_sym, records * n_sym * sizeof(int), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_pre, prefix.size() * sizeof(long long), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_g, g.size() * sizeof(double), st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_sym, symbols, records * n_sym * sizeof(int), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_pre, prefix.data(), prefix.size() * sizeof(long long), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_g, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && n_out && records) {
        const size_t bx = std::max<size_t>(1, std::min<size_t>((n_out + 255) / 256, (148 * 16 + records - 1) / records));
        cpm_kernel<<<dim3((unsigned)bx, (unsigned)records), 256, 0, st>>>(d_sym, d_pre, d_g, p.sps, p.pulse_len, p.h,
                                                                        n_sym, n_out, out, f64);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host prefix/g buffers go out of scope
    cudaFreeAsync(d_sym, st);
    cudaFreeAsync(d_pre, st);
    cudaFreeAsync(d_g, st);
    if (e != cudaSuccess) {
        msg = std::string("CUDA error in cpm_modulate: ") + cudaGetErrorString(e);
        return CYC_ERR_CUDA;
    }
    return CYC_OK;
}

std::vector<int> draw_symbols(int M, size_t count, uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::vector<int> out(count);
    for (auto& s : out) {
        const int idx = (int)(gen() % (uint64_t)M);
        s = 2 * idx - (M - 1);
    }
    return out;
}

}  // namespace

extern "C" {

void cyc_cpm_params_init(cyc_cpm_params* p) {
    if (!p) return;
    p->h = 0.5;
    p->alphabet_size = 2;
    p->pulse_len = 4;
    p->bt = 0.25;
    p->sps = 8;
    p->pulse_kind = CYC_PULSE_GAUSSIAN;
}

int cyc_random_symbols(int alphabet_size, size_t count, uint64_t seed, int* out, char* err, size_t errlen) {
    if (alphabet_size < 2 || alphabet_size % 2 != 0) {
        write_msg(err, errlen, "alphabet size must be even and at least 2");
        return CYC_ERR_USAGE;
    }
    if (count && !out) {
        write_msg(err, errlen, "null output");
        return CYC_ERR_USAGE;
    }
    const std::vector<int> s = draw_symbols(alphabet_size, count, seed);
    if (count) std::memcpy(out, s.data(), count * sizeof(int));
    write_msg(err, errlen, "");
    return CYC_OK;
}

int cyc_cpm_pulse(const cyc_cpm_params* p, double* f_out, double* g_out, size_t len, char* err, size_t errlen) {
    if (!p) return CYC_ERR_USAGE;
    std::string m = check_params(*p);
    if (!m.empty()) {
        write_msg(err, errlen, m);
        return CYC_ERR_USAGE;
    }
    std::vector<double> f, g;
    m = make_pulse(*p, f, g);
    if (!m.empty()) {
        write_msg(err, errlen, m);
        return CYC_ERR_DATA;
    }
    if (len != f.size()) {
        write_msg(err, errlen, "pulse buffers must hold pulse_len * sps values");
        return CYC_ERR_USAGE;
    }
    if (f_out) std::memcpy(f_out, f.data(), len * sizeof(double));
    if (g_out) std::memcpy(g_out, g.data(), len * sizeof(double));
    write_msg(err, errlen, "");
    return CYC_OK;
}

int cyc_cpm_modulate(const cyc_cpm_params* p, const int* symbols, size_t n_symbols, int device, int out_f64,
                     void* out, char* err, size_t errlen) {
    if (!p || (n_symbols && (!symbols || !out))) {
        write_msg(err, errlen, "null argument");
        return CYC_ERR_USAGE;
    }
    std::string m = check_params(*p);
    if (!m.empty()) {
        write_msg(err, errlen, m);
        return CYC_ERR_USAGE;
    }
    if (n_symbols == 0) {
        write_msg(err, errlen, "cannot modulate an empty symbol stream");
        return CYC_ERR_USAGE;
    }
    for (size_t i = 0; i < n_symbols; ++i) {
        const int a = symbols[i], mag = std::abs(a);
        if (mag % 2 != 1 || mag > p->alphabet_size - 1) {
            write_msg(err, errlen, "symbol " + std::to_string(a) + " at index " + std::to_string(i) +
                                       " is outside the size-" + std::to_string(p->alphabet_size) + " alphabet");
            return CYC_ERR_DATA;
        }
    }
    if (cudaSetDevice(device) != cudaSuccess) {
        write_msg(err, errlen, "cudaSetDevice failed");
        return CYC_ERR_CUDA;
    }
    const size_t n_out = n_symbols * (size_t)p->sps;
    const size_t bytes = n_out * (out_f64 ? 16 : 8);
    cudaPointerAttributes a{};
    const bool dev_out = cudaPointerGetAttributes(&a, out) == cudaSuccess && a.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    void* target = out;
    if (!dev_out && cudaMallocAsync(&target, bytes, st) != cudaSuccess) {
        cudaStreamDestroy(st);
        write_msg(err, errlen, "device allocation failed");
        return CYC_ERR_CUDA;
    }
    int rc = modulate_device(*p, symbols, n_symbols, 1, n_out, target, out_f64, st, m);
    if (rc == CYC_OK && !dev_out) {
        if (cudaMemcpyAsync(out, target, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            rc = CYC_ERR_CUDA;
            m = "device-to-host copy failed";
        }
    }
    if (!dev_out) cudaFreeAsync(target, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    write_msg(err, errlen, rc ? m : std::string());
    return rc;
}

int cyc_gmsk_mc_oracle(const cyc_cpm_params* p, const double* alphas, size_t n_alphas, const int* lags,
                       size_t n_lags, int conj, int win_len, int trials, size_t record_len, uint64_t seed,
                       int device, double* mean_magnitude, char* err, size_t errlen) {
    if (!p || !mean_magnitude) {
        write_msg(err, errlen, "null argument");
        return CYC_ERR_USAGE;
    }
    // argument checks in the reference's order (reference.cpp:39-51)
    if (n_alphas == 0 || n_lags == 0 || !alphas || !lags) {
        write_msg(err, errlen, "oracle needs at least one cycle frequency and one lag");
        return CYC_ERR_USAGE;
    }
    if (trials < 1) {
        write_msg(err, errlen, "oracle needs at least one trial");
        return CYC_ERR_USAGE;
    }
    if (win_len < 1) {
        write_msg(err, errlen, "window length must be at least 1");
        return CYC_ERR_USAGE;
    }
    int m_plus = 0, m_minus = 0;
    for (size_t i = 0; i < n_lags; ++i) {
        m_plus = std::max(m_plus, lags[i]);
        m_minus = std::max(m_minus, -lags[i]);
    }
    const size_t need = (size_t)win_len + (size_t)m_plus + (size_t)m_minus;
    if (record_len < need) {
        write_msg(err, errlen, "record too short for a single estimation window");
        return CYC_ERR_USAGE;
    }
    std::string m = check_params(*p);
    if (!m.empty()) {
        write_msg(err, errlen, m);
        return CYC_ERR_USAGE;
    }
    const int M = std::max(m_plus, m_minus);
    const size_t wins = (record_len - (size_t)m_plus - (size_t)m_minus) / (size_t)win_len;
    if (win_len < 2) {
        write_msg(err, errlen, "the device oracle needs win_len >= 2");
        return CYC_ERR_USAGE;
    }
    // Trials run as the channels of one Set-mode estimator over lags -M..M
    // (a batch of up to TB trials per push).  The records are pushed at origin
    // M - m_minus so frame j starts at sample m_minus + j N (the oracle's k0),
    // and padded by M - m_plus samples so exactly `wins` frames complete.
    // The batch size depends on the record length only (never on `trials`), so
    // a trial's table is bit-identical whatever the trial count (the
    // reference's trial-extendability pin, test_reference.cpp:137-144).
    const size_t total_len = record_len + (size_t)(M - m_plus);
    const int TB = (int)std::max<size_t>(1, std::min<size_t>(128, ((size_t)1 << 22) / total_len));
    cyc::Cfg c;
    c.mode = CYC_MODE_SET;
    c.flags = conj ? CYC_FLAG_CONJ : CYC_FLAG_CONV;
    c.win_len = win_len;
    c.alphas.assign(alphas, alphas + n_alphas);
    c.lag_symmetric = true;
    c.max_lag = M;
    c.emit_frames = true;
    c.channels = TB;
    c.device = device;
    c.origin = (int64_t)(M - m_minus);
    // The estimator and the record buffer of the last geometry are kept per
    // thread: repeated calls (more trials, other seeds) skip the set-up, which
    // dominates small tables.  Freed when the thread exits.
    struct Cache {
        cyc::Cfg cfg;
        cyc::Engine* e = nullptr;
        float2* x = nullptr;
        size_t x_len = 0;
        cudaStream_t st = nullptr;
        ~Cache() {
            delete e;
            cudaFree(x);
            if (st) cudaStreamDestroy(st);
        }
    };
    static thread_local Cache cache_obj;
    Cache* cache = &cache_obj;
    auto same = [](const cyc::Cfg& a, const cyc::Cfg& b) {
        return a.mode == b.mode && a.flags == b.flags && a.win_len == b.win_len && a.alphas == b.alphas &&
               a.lag_symmetric == b.lag_symmetric && a.max_lag == b.max_lag && a.emit_frames == b.emit_frames &&
               a.channels == b.channels && a.device == b.device && a.origin == b.origin;
    };
    if (!cache->e || !same(cache->cfg, c)) {
        delete cache->e;
        cache->e = nullptr;
        cyc::Engine* ne = nullptr;
        cyc::Status cs = cyc::Engine::create_unchecked(c, &ne);  // the oracle has no win_len > 2M rule
        if (cs.code) {
            write_msg(err, errlen, cs.msg);
            return cs.code;
        }
        cache->e = ne;
        cache->cfg = c;
    }
    cyc::Engine* e = cache->e;
    cyc::Status s;
    const size_t total = total_len;
    const size_t n_syms = (total + (size_t)p->sps - 1) / (size_t)p->sps;
    if (!cache->st) cudaStreamCreateWithFlags(&cache->st, cudaStreamNonBlocking);
    cudaStream_t st = cache->st;
    if (cache->x_len < (size_t)TB * total) {
        cudaFree(cache->x);
        cache->x = nullptr;
        cache->x_len = 0;
        if (cudaMalloc(&cache->x, (size_t)TB * total * sizeof(float2)) != cudaSuccess) {
            write_msg(err, errlen, "device allocation failed");
            return CYC_ERR_CUDA;
        }
        cache->x_len = (size_t)TB * total;
    }
    float2* x = cache->x;
    const size_t lay = n_alphas * (2 * (size_t)M + 1);
    std::vector<cyc_cf64> avg(lay);
    std::vector<double> acc(n_alphas * n_lags, 0.0);
    std::vector<int> syms((size_t)TB * n_syms);
    int rc = CYC_OK;
    for (int t0 = 0; t0 < trials && rc == CYC_OK; t0 += TB) {
        const int nb = std::min(TB, trials - t0);
        for (int b = 0; b < TB; ++b) {  // a short last batch repeats its first trial in the spare channels
            const std::vector<int> sy = draw_symbols(p->alphabet_size, n_syms, seed + (uint64_t)(t0 + (b < nb ? b : 0)));
            std::copy(sy.begin(), sy.end(), syms.begin() + (size_t)b * n_syms);
        }
        rc = modulate_device(*p, syms.data(), n_syms, (size_t)TB, total, x, 0, st, m);
        if (rc) break;
        s = e->reset();
        if (!s.code) s = e->push(x, nullptr, total, cyc::Engine::IN_DEVICE_F32, nullptr, nullptr);
        if (!s.code && e->frames_emitted() != wins) {
            s.code = CYC_ERR_INTERNAL;
            s.msg = "oracle window count mismatch";
        }
        for (int b = 0; b < nb && !s.code; ++b) {
            s = e->average(CYC_AVG_MAGNITUDE, c.flags, b, avg.data());
            // per-trial window mean |R| x wins = the trial's sum over windows, added in trial order
            for (size_t a = 0; a < n_alphas && !s.code; ++a)
                for (size_t l = 0; l < n_lags; ++l)
                    acc[a * n_lags + l] += avg[a * (2 * (size_t)M + 1) + (size_t)(lags[l] + M)].re * (double)wins;
        }
        if (s.code) {
            rc = s.code;
            m = s.msg;
        }
    }
    if (rc) {
        write_msg(err, errlen, m);
        return rc;
    }
    const double norm = 1.0 / ((double)trials * (double)wins);
    for (size_t i = 0; i < acc.size(); ++i) mean_magnitude[i] = acc[i] * norm;
    write_msg(err, errlen, "");
    return CYC_OK;
}

}  // extern "C"

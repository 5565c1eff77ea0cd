/*
 * cycoracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see cycoracle.h).
 *
 * Double-precision restatement of the reference cyclic-ACF estimator
 * (/root/reference/proj).  Never linked into the product.
 */
#include "cycoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static const double two_pi = 2.0 * M_PI;

/* complex helpers on interleaved doubles */
typedef struct { double re, im; } cd;
static inline cd cmul(cd a, cd b) { cd r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return r; }
static inline cd cconj(cd a) { cd r = {a.re, -a.im}; return r; }
static inline cd cpolar(double th) { cd r = {cos(th), sin(th)}; return r; }
static inline cd cld(const double* p, size_t i) { cd r = {p[2 * i], p[2 * i + 1]}; return r; }

/* proj/src/reference.cpp:11-32 */
int orc_direct(const double* x, const double* y, size_t len, double alpha, int m,
               int conj, size_t k0, int n_win, double out[2]) {
    if (n_win < 1) return -1;
    long long first_x = (long long)k0 + m;
    long long last_x = first_x + n_win - 1;
    if (first_x < 0 || last_x >= (long long)len) return -1;
    if (k0 + (size_t)n_win > len) return -1;
    const double w0 = -two_pi * alpha;
    cd acc = {0.0, 0.0};
    for (int n = 0; n < n_win; ++n) {
        cd xs = cld(x, (size_t)first_x + (size_t)n);
        cd ys = cld(y, k0 + (size_t)n);
        cd prod = conj ? cmul(xs, ys) : cmul(xs, cconj(ys));
        cd t = cmul(prod, cpolar(w0 * n));
        acc.re += t.re;
        acc.im += t.im;
    }
    acc.re /= (double)n_win;
    acc.im /= (double)n_win;
    cd r = cmul(acc, cpolar(w0 * (double)k0));
    out[0] = r.re;
    out[1] = r.im;
    return 0;
}

/* proj/src/fft.cpp:25-100 */
static unsigned bit_reverse(unsigned v, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; ++i) { r = (r << 1) | (v & 1u); v >>= 1; }
    return r;
}

void orc_fft(const double* in, double* out, size_t n) {
    if (n == 1) { out[0] = in[0]; out[1] = in[1]; return; }
    const double w0 = -two_pi / (double)n;
    int pow2 = (n & (n - 1)) == 0;
    if (pow2) {
        int bits = 0;
        while (((size_t)1 << bits) < n) ++bits;
        cd* tw = (cd*)malloc(sizeof(cd) * (n / 2));
        for (size_t t = 0; t < n / 2; ++t) tw[t] = cpolar(w0 * (double)t);
        cd* o = (cd*)malloc(sizeof(cd) * n);
        for (size_t i = 0; i < n; ++i) o[i] = cld(in, bit_reverse((unsigned)i, bits));
        for (size_t L = 2; L <= n; L <<= 1) {
            size_t half = L / 2, step = n / L;
            for (size_t base = 0; base < n; base += L)
                for (size_t j = 0; j < half; ++j) {
                    cd w = tw[j * step];
                    cd u = o[base + j];
                    cd v = cmul(o[base + j + half], w);
                    o[base + j].re = u.re + v.re; o[base + j].im = u.im + v.im;
                    o[base + j + half].re = u.re - v.re; o[base + j + half].im = u.im - v.im;
                }
        }
        memcpy(out, o, sizeof(cd) * n);
        free(o);
        free(tw);
        return;
    }
    cd* tw = (cd*)malloc(sizeof(cd) * n);
    for (size_t t = 0; t < n; ++t) tw[t] = cpolar(w0 * (double)t);
    cd* src = (cd*)malloc(sizeof(cd) * n);
    memcpy(src, in, sizeof(cd) * n);
    for (size_t k = 0; k < n; ++k) {
        double re = 0.0, im = 0.0;
        size_t idx = 0;
        for (size_t t = 0; t < n; ++t) {
            cd w = tw[idx], s = src[t];
            re += s.re * w.re - s.im * w.im;
            im += s.re * w.im + s.im * w.re;
            idx += k;
            if (idx >= n) idx -= n;
        }
        out[2 * k] = re;
        out[2 * k + 1] = im;
    }
    free(src);
    free(tw);
}

/* proj/src/types.cpp:30-63 (subset needed to refuse what the reference refuses) */
static int config_ok(int mode, int win_len, size_t n_alphas, const double* alphas,
                     int max_lag, const int* lags, size_t n_lags) {
    if (win_len < 2) return 0;
    int span = 0;
    if (mode == 0) {
        if (n_alphas == 0 || max_lag < 0) return 0;
        span = max_lag;
    } else {
        if (n_lags == 0) return 0;
        for (size_t i = 1; i < n_lags; ++i) if (lags[i] <= lags[i - 1]) return 0;
        for (size_t i = 0; i < n_lags; ++i) {
            int a = lags[i] < 0 ? -lags[i] : lags[i];
            if (a > span) span = a;
        }
    }
    for (size_t a = 0; a < n_alphas; ++a) if (!(alphas[a] >= -0.5 && alphas[a] < 0.5)) return 0;
    if (win_len <= 2 * span) return 0;
    return 1;
}

/* proj/src/estimator.cpp:15-84, proj/src/kernels.cpp:13-114 */
int orc_stream(int mode, int conj, int win_len, const double* alphas, size_t n_alphas,
               int max_lag, const int* lags, size_t n_lags, const double* x,
               const double* y, size_t len, double* frames_out, size_t* n_frames,
               size_t* layout_len) {
    if (!config_ok(mode, win_len, n_alphas, alphas, max_lag, lags, n_lags)) return -1;
    const int N = win_len;
    int m_plus = 0, m_minus = 0;
    if (mode == 0) {
        m_plus = m_minus = max_lag;
    } else {
        for (size_t i = 0; i < n_lags; ++i) {
            if (lags[i] > m_plus) m_plus = lags[i];
            if (-lags[i] > m_minus) m_minus = -lags[i];
        }
    }
    const size_t need = (size_t)N + (size_t)m_plus + (size_t)m_minus; /* estimator.cpp:20 */
    const size_t F = len >= need ? (len - need) / (size_t)N + 1 : 0;
    const size_t row = 2u * (size_t)max_lag + 1u;
    const size_t lay = mode == 0 ? n_alphas * row : n_lags * (size_t)N;
    if (n_frames) *n_frames = F;
    if (layout_len) *layout_len = lay;
    if (!frames_out || F == 0) return 0;
    const double inv_n = 1.0 / (double)N;

    if (mode == 0) {
        /* SetWindowPlan twiddles (kernels.cpp:19-24), lead_const/acc/step (estimator.cpp:24-29) */
        cd* tw = (cd*)malloc(sizeof(cd) * n_alphas * (size_t)N);
        cd* lead_const = (cd*)malloc(sizeof(cd) * n_alphas);
        cd* acc = (cd*)malloc(sizeof(cd) * n_alphas);
        cd* step = (cd*)malloc(sizeof(cd) * n_alphas);
        for (size_t a = 0; a < n_alphas; ++a) {
            const double w0 = -two_pi * alphas[a];
            for (int n = 0; n < N; ++n) tw[a * (size_t)N + (size_t)n] = cpolar(w0 * (double)n);
            lead_const[a] = cpolar(-two_pi * alphas[a] * (double)m_minus);
            acc[a].re = 1.0; acc[a].im = 0.0;
            step[a] = cpolar(-two_pi * alphas[a] * (double)N);
        }
        for (size_t f = 0; f < F; ++f) {
            const size_t head = f * (size_t)N;
            double* out = frames_out + 2 * f * lay;
            for (size_t a = 0; a < n_alphas; ++a) {
                cd lead = cmul(lead_const[a], acc[a]);
                for (int m = -max_lag; m <= max_lag; ++m) {
                    /* set_window_values inner loop, kernels.cpp:44-56 */
                    double re = 0.0, im = 0.0;
                    for (int n = 0; n < N; ++n) {
                        cd xs = cld(x, head + (size_t)(max_lag + m) + (size_t)n);
                        cd ys = cld(y, head + (size_t)m_minus + (size_t)n);
                        double qr = conj ? xs.re * ys.re - xs.im * ys.im : xs.re * ys.re + xs.im * ys.im;
                        double qi = conj ? xs.re * ys.im + xs.im * ys.re : xs.im * ys.re - xs.re * ys.im;
                        cd t = tw[a * (size_t)N + (size_t)n];
                        re += qr * t.re - qi * t.im;
                        im += qr * t.im + qi * t.re;
                    }
                    cd v = {re, im};
                    v = cmul(v, lead);
                    size_t idx = a * row + (size_t)(m + max_lag);
                    out[2 * idx] = v.re * inv_n;
                    out[2 * idx + 1] = v.im * inv_n;
                }
            }
            for (size_t a = 0; a < n_alphas; ++a) {
                acc[a] = cmul(acc[a], step[a]);
                double mag = hypot(acc[a].re, acc[a].im);
                acc[a].re /= mag;
                acc[a].im /= mag;
            }
        }
        free(tw); free(lead_const); free(acc); free(step);
        return 0;
    }

    /* Full mode: full_bin_lead (kernels.cpp:103-114), full_window_values (kernels.cpp:72-94) */
    cd* bin_lead = (cd*)malloc(sizeof(cd) * (size_t)N);
    const uint64_t nn = (uint64_t)N, base = (uint64_t)m_minus % nn;
    for (uint64_t k = 0; k < nn; ++k) {
        uint64_t r = (k * base) % nn;
        bin_lead[k] = cpolar(-two_pi * (double)r / (double)nn);
    }
    double* prod = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    double* spec = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    for (size_t f = 0; f < F; ++f) {
        const size_t head = f * (size_t)N;
        double* out = frames_out + 2 * f * lay;
        for (size_t l = 0; l < n_lags; ++l) {
            const int m = lags[l];
            for (int n = 0; n < N; ++n) {
                cd xs = cld(x, head + (size_t)(m_minus + m) + (size_t)n);
                cd ys = cld(y, head + (size_t)m_minus + (size_t)n);
                cd p = conj ? cmul(xs, ys) : cmul(xs, cconj(ys));
                prod[2 * n] = p.re;
                prod[2 * n + 1] = p.im;
            }
            orc_fft(prod, spec, (size_t)N);
            for (int k = 0; k < N; ++k) {
                cd d = {spec[2 * k], spec[2 * k + 1]};
                d = cmul(d, bin_lead[k]);
                size_t idx = l * (size_t)N + (size_t)k;
                out[2 * idx] = d.re * inv_n;
                out[2 * idx + 1] = d.im * inv_n;
            }
        }
    }
    free(prod); free(spec); free(bin_lead);
    return 0;
}

int orc_block_direct(const double* x, const double* y, size_t len, const double* alphas,
                     size_t n_alphas, const int* lags, size_t n_lags, int conj,
                     size_t start, size_t count, double* out) {
    if (count == 0) return -1;
    for (size_t t = 0; t < n_lags; ++t) {
        long long lo = (long long)start + lags[t];
        long long hi = (long long)(start + count - 1) + lags[t];
        if (lo < 0 || hi >= (long long)len) return -1;
    }
    if (start + count > len) return -1;
    for (size_t a = 0; a < n_alphas; ++a) {
        const double w0 = -two_pi * alphas[a];
        for (size_t t = 0; t < n_lags; ++t) {
            cd acc = {0.0, 0.0};
            for (size_t i = 0; i < count; ++i) {
                const size_t n = start + i;
                cd xs = cld(x, (size_t)((long long)n + lags[t]));
                cd ys = cld(y, n);
                cd prod = conj ? cmul(xs, ys) : cmul(xs, cconj(ys));
                cd v = cmul(prod, cpolar(w0 * (double)n));
                acc.re += v.re;
                acc.im += v.im;
            }
            out[2 * (a * n_lags + t)] = acc.re / (double)count;
            out[2 * (a * n_lags + t) + 1] = acc.im / (double)count;
        }
    }
    return 0;
}

int orc_block_fold(const float* xf, const float* yf, size_t len, const int64_t* k,
                   size_t n_alphas, int64_t P, const int* lags, size_t n_lags,
                   size_t start, size_t count, double* out_conv, double* out_conj) {
    if (count == 0 || P < 1) return -1;
    for (size_t t = 0; t < n_lags; ++t) {
        long long lo = (long long)start + lags[t];
        long long hi = (long long)(start + count - 1) + lags[t];
        if (lo < 0 || hi >= (long long)len) return -1;
    }
    if (start + count > len) return -1;
    const size_t Pz = (size_t)P;
    /* four real correlations per (lag, residue): sum xr*yr, xi*yi, xi*yr, xr*yi */
    double* S = (double*)calloc(n_lags * Pz * 4, sizeof(double));
    if (!S) return -1;
    /* lags are independent (each keeps the sequential sample-order sum), so
       the production-size parity tests may fold them on all host cores */
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t t = 0; t < n_lags; ++t) {
        double* St = S + t * Pz * 4;
        const long long lag = lags[t];
        size_t r = start % Pz;
        for (size_t i = 0; i < count; ++i) {
            const size_t n = start + i;
            const double xr = xf[2 * (size_t)((long long)n + lag)];
            const double xi = xf[2 * (size_t)((long long)n + lag) + 1];
            const double yr = yf[2 * n], yi = yf[2 * n + 1];
            double* s = St + 4 * r;
            s[0] += xr * yr;
            s[1] += xi * yi;
            s[2] += xi * yr;
            s[3] += xr * yi;
            if (++r == Pz) r = 0;
        }
    }
    cd* tw = (cd*)malloc(sizeof(cd) * Pz);
    for (size_t r = 0; r < Pz; ++r) tw[r] = cpolar(-two_pi * (double)r / (double)P);
    const double inv = 1.0 / (double)count;
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t a = 0; a < n_alphas; ++a) {
        const int64_t kk = ((k[a] % P) + P) % P;
        for (size_t t = 0; t < n_lags; ++t) {
            const double* St = S + t * Pz * 4;
            cd cv = {0, 0}, cj = {0, 0};
            for (size_t r = 0; r < Pz; ++r) {
                const cd w = tw[(size_t)(((unsigned long long)kk * r) % (unsigned long long)P)];
                const double* s = St + 4 * r;
                cd qv = {s[0] + s[1], s[2] - s[3]}; /* x * conj(y) */
                cd qj = {s[0] - s[1], s[2] + s[3]}; /* x * y */
                cd a1 = cmul(qv, w), a2 = cmul(qj, w);
                cv.re += a1.re; cv.im += a1.im;
                cj.re += a2.re; cj.im += a2.im;
            }
            if (out_conv) {
                out_conv[2 * (a * n_lags + t)] = cv.re * inv;
                out_conv[2 * (a * n_lags + t) + 1] = cv.im * inv;
            }
            if (out_conj) {
                out_conj[2 * (a * n_lags + t)] = cj.re * inv;
                out_conj[2 * (a * n_lags + t) + 1] = cj.im * inv;
            }
        }
    }
    free(tw);
    free(S);
    return 0;
}

int orc_recursive(const double* x, const double* y, size_t len, const double* alphas,
                  size_t n_alphas, const int* lags, size_t n_lags, int conj,
                  double lambda, size_t emit_every, double* out, size_t* n_emit) {
    if (n_lags == 0 || n_alphas == 0 || emit_every == 0) return -1;
    int m_plus = 0, m_minus = 0;
    for (size_t i = 0; i < n_lags; ++i) {
        if (lags[i] > m_plus) m_plus = lags[i];
        if (-lags[i] > m_minus) m_minus = -lags[i];
    }
    const size_t need = emit_every + (size_t)m_plus + (size_t)m_minus;
    const size_t E = len >= need ? (len - need) / emit_every + 1 : 0;
    if (n_emit) *n_emit = E;
    if (!out || E == 0) return 0;
    const size_t cells = n_alphas * n_lags;
    cd* R = (cd*)calloc(cells, sizeof(cd));
    const size_t n_end = (size_t)m_minus + E * emit_every;
    /* alphas are independent recursions: one per thread, same per-sample order */
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t a = 0; a < n_alphas; ++a) {
        size_t e = 0;
        for (size_t n = (size_t)m_minus; n < n_end; ++n) {
            cd ys = cld(y, n);
            cd ph = cpolar(-two_pi * alphas[a] * (double)n);
            for (size_t t = 0; t < n_lags; ++t) {
                cd xs = cld(x, (size_t)((long long)n + lags[t]));
                cd prod = conj ? cmul(xs, ys) : cmul(xs, cconj(ys));
                cd v = cmul(prod, ph);
                cd* r = &R[a * n_lags + t];
                r->re = lambda * r->re + (1.0 - lambda) * v.re;
                r->im = lambda * r->im + (1.0 - lambda) * v.im;
            }
            if (n + 1 == (size_t)m_minus + (e + 1) * emit_every) {
                for (size_t t = 0; t < n_lags; ++t) {
                    out[2 * (e * cells + a * n_lags + t)] = R[a * n_lags + t].re;
                    out[2 * (e * cells + a * n_lags + t) + 1] = R[a * n_lags + t].im;
                }
                ++e;
            }
        }
    }
    free(R);
    return 0;
}

/* std::mt19937_64 per the C++ standard [rand.predef] */
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* s) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t xx = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = xx >> 1;
            if (xx & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t z = s->mt[s->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
}

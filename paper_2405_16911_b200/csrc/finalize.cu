// finalize.cu -- residue folds S_tau[r] -> cyclic ACF tables R(alpha, tau).
//
//   R(alpha_a, tau) = scale * sum_{r < Pf} q_tau[r] * W^{bin_a * r},  W = e^{-j2pi/Pf}
//
// with q built from the four real correlations of fold.cu per flag, and
// bin_a = k_a * (Pf / P) (mod Pf) exact integers, so the phase is anchored to
// absolute sample 0 exactly (the reference's exact-integer bin lead,
// proj/src/kernels.cpp:103-114, generalised to every alpha on the grid).
//
// Two paths, both fp64:
//   * radix-2 DIT FFT in shared memory (Pf a power of two <= 8192; levels
//     grouped four per pass in registers, twiddles in shared memory): replaces
//     the reference's per-lag Fft::forward (proj/src/fft.cpp:44-87);
//   * direct DFT with an exact (bin*r mod Pf) twiddle index, for small alpha
//     sets or non-power-of-two periods (proj/src/fft.cpp:89-100 analogue).
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"

namespace cyc {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// FFT element types: fp64 (double2) or fp32 (float2, inputs combined in fp64
// and rounded once)
template <class V>
__device__ __forceinline__ V to_v(double2 a);
template <>
__device__ __forceinline__ double2 to_v<double2>(double2 a) { return a; }
template <>
__device__ __forceinline__ float2 to_v<float2>(double2 a) { return make_float2((float)a.x, (float)a.y); }
__device__ __forceinline__ double2 to_d(double2 a) { return a; }
__device__ __forceinline__ double2 to_d(float2 a) { return make_double2(a.x, a.y); }

__device__ __forceinline__ double2 combine(const double* s, int flag_bit) {  // s: 4 values
    // s = (c0, c1, c2, c3) = (sum xr*yr, sum xi*yr, sum xr*yi, sum xi*yi)
    return flag_bit == 0 ? make_double2(s[0] + s[3], s[1] - s[2])   // x * conj(y)
                         : make_double2(s[0] - s[3], s[1] + s[2]);  // x * y
}

// Shared-memory index with one pad slot per 16 points (a thread's 16
// consecutive points in the first pass sit 272 B apart across a warp, off the
// same banks) and one per Pf/8 (the bit-reversed stores of 8 consecutive
// residues land Pf/8-multiples apart: without it they share a bank group).
// sh = log2(Pf) - 3; the buffer holds Pf + Pf/16 + 8 points.
__device__ __forceinline__ int padi(int i, int sh) { return i + (i >> 4) + (i >> sh); }

// b * e^{-j pi e / 8}, e = 1..7 (e = 4: -j, exact)
template <class V>
__device__ __forceinline__ V rot16(V b, int e) {
    if (e == 4) {
        V r;
        r.x = b.y;
        r.y = -b.x;
        return r;
    }
    constexpr double C[8] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977, 0.0,
                             -0.38268343236508977, -0.70710678118654752, -0.92387953251128674};
    constexpr double S[8] = {0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674, 1.0,
                             0.92387953251128674, 0.70710678118654752, 0.38268343236508977};
    V w;
    w.x = (decltype(b.x))C[e];
    w.y = -(decltype(b.x))S[e];
    return cmul(b, w);
}

// One pass of LOG2R radix-2 DIT levels (halves h, 2h, .., 2^(LOG2R-1) h): each
// thread takes groups of R = 2^LOG2R points base + pos + k h (k < R) into
// registers and runs the levels there -- exactly the radix-2 butterflies
// (v = b w, a + v, a - v) with the level's twiddles, one barrier per pass.
// Level l's twiddle W^{(pos + m h) Pf / (2^{l+1} h)} = b_l * e^{-j pi m / 2^l}
// with b_l = tp[l h + pos] from the pass's own table (consecutive threads read
// consecutive entries: no bank conflicts -- one shared table indexed at
// stride Pf / (2^{l+1} h) was 6-way conflicted, ncu) and a 16th root of unity.
template <int LOG2R, class V>
__device__ __forceinline__ void fft_pass(V* buf, const V* tp, int Pf, int h, int sh) {
    constexpr int R = 1 << LOG2R;
    for (int g = threadIdx.x; g < Pf / R; g += blockDim.x) {
        const int base = (g / h) * (R * h), pos = g - (g / h) * h;
        V v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = buf[padi(base + pos + k * h, sh)];
#pragma unroll
        for (int l = 0; l < LOG2R; ++l) {
            const V b0 = tp[l * h + pos];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (k & (1 << l)) continue;
                const int m = k & ((1 << l) - 1);
                const V w = m == 0 ? b0 : rot16(b0, m << (3 - l));
                const V b = v[k + (1 << l)];
                const V t = cmul(b, w);
                v[k + (1 << l)].x = v[k].x - t.x;
                v[k + (1 << l)].y = v[k].y - t.y;
                v[k].x += t.x;
                v[k].y += t.y;
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) buf[padi(base + pos + k * h, sh)] = v[k];
    }
    __syncthreads();
}

// The same pass with each level's base twiddle computed as W^k = T1[k >> 6] *
// T2[k & 63] (T1[a] = W^{64a}, T2[b] = W^b: 1 KB at Pf = 8192 instead of the
// 41 KB of per-pass tables), so three 8192-point fp32 rows fit an SM.
template <int LOG2R, class V>
__device__ __forceinline__ void fft_pass_f(V* buf, const V* t2, const V* t1, int Pf, int h, int sh) {
    constexpr int R = 1 << LOG2R;
    for (int g = threadIdx.x; g < Pf / R; g += blockDim.x) {
        const int base = (g / h) * (R * h), pos = g - (g / h) * h;
        V v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = buf[padi(base + pos + k * h, sh)];
#pragma unroll
        for (int l = 0; l < LOG2R; ++l) {
            const int kk = pos * (Pf / (2 * (h << l)));
            const V b0 = cmul(t1[kk >> 6], t2[kk & 63]);
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (k & (1 << l)) continue;
                const int m = k & ((1 << l) - 1);
                const V w = m == 0 ? b0 : rot16(b0, m << (3 - l));
                const V b = v[k + (1 << l)];
                const V t = cmul(b, w);
                v[k + (1 << l)].x = v[k].x - t.x;
                v[k + (1 << l)].y = v[k].y - t.y;
                v[k].x += t.x;
                v[k].y += t.y;
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) buf[padi(base + pos + k * h, sh)] = v[k];
    }
    __syncthreads();
}

// The pass sequence of a row (shared by the kernel and the host's shared-memory
// size): radix-16 passes when the block has enough groups of 16 (else radix-4),
// then one pass of the remaining levels; fn(log2r, h) per pass.
template <class F>
__host__ __device__ inline void fft_passes(int log2Pf, int nthreads, F fn) {
    int h = 1, lv = 0;
    const int r = nthreads * 16 <= (1 << log2Pf) ? 4 : 2;
    for (; lv + r <= log2Pf; lv += r, h <<= r) fn(r, h);
    if (log2Pf > lv) fn(log2Pf - lv, h);
}
// entries of the per-pass twiddle tables: sum over passes of log2r * h
__host__ __device__ inline int fft_tw_entries(int log2Pf, int nthreads) {
    int n = 0;
    fft_passes(log2Pf, nthreads, [&](int r, int h) { n += r * h; });
    return n;
}

// One CTA per (row, flag): the row's combined
// correlations in bit-reversed order, then radix-16 passes (four radix-2
// levels each, in registers) and a final pass of the remaining levels.
template <class V, bool FACT>
__global__ void __launch_bounds__(FACT ? 256 : 512, FACT ? 3 : (sizeof(V) == 8 ? 2 : 1))
    finalize_fft_kernel(FinalizeLaunch L, int log2Pf) {
    extern __shared__ __align__(16) uint8_t fft_smem[];
    V* buf = reinterpret_cast<V*>(fft_smem);  // Pf + Pf/16 + 8 points (padded), then the twiddle tables
    __shared__ FinalRow s_row;                // descriptors may be in mapped host memory: read once
    const int Pf = L.Pf;
    const int sh = max(log2Pf - 3, 1);
    V* tw = buf + Pf + (Pf >> 4) + 8;  // per-pass twiddle tables, pass after pass
    // grid (n_rows * n_flag_tables): the flag tables of a row are adjacent CTAs,
    // so the second read of the row's S comes from L2
    const int nflag = (L.flags == 3) ? 2 : 1;
    const int row_i = blockIdx.x / nflag, fi = blockIdx.x % nflag;  // fi: index among requested flags
    if (threadIdx.x == 0) s_row = L.rows[row_i];
    if (FACT) {  // T2[b] = W^b (b < 64), then T1[a] = W^{64 a} (a < Pf / 128)
        for (int i = threadIdx.x; i < 64 + (Pf >> 7); i += blockDim.x)
            tw[i] = to_v<V>(__ldg(L.tw + (i < 64 ? i : 64 * (i - 64))));
    } else {
        // the per-pass tables follow the Pf plain twiddles (fft_pass_twiddles, built on the host)
        const double2* twp = L.tw + Pf;
        const int ntw = fft_tw_entries(log2Pf, blockDim.x);
        for (int i = threadIdx.x; i < ntw; i += blockDim.x) tw[i] = to_v<V>(__ldg(twp + i));
    }
    // everything above is independent of the predecessor (PDL launch: it overlaps
    // the reduce's tail); S and the frame counter below are not
    pdl_wait();
    if (L.shift_ctr && threadIdx.x == 0 && blockIdx.x == 0) *L.shift_ctr += L.shift_inc;
    __syncthreads();
    const FinalRow row = s_row;
    const int flag_bit = (L.flags == 2) ? 1 : fi;
    const double* Srow = L.S + ((size_t)row.slot * L.t_pad + row.t_span) * (size_t)Pf * 4;
    double2* out = L.out + (size_t)row.out_block * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                   (size_t)row.t_out * L.stride_t;
    // recursive emission: this thread's recursion state loads overlap the FFT
    const bool rec_pre = L.rec_R && L.A <= (int)blockDim.x;
    double2 rR = make_double2(0.0, 0.0), rC = rR;
    double rM = 0.0;
    if (rec_pre && (int)threadIdx.x < L.A) {
        const size_t o = (size_t)(out - L.out) + (size_t)threadIdx.x * L.stride_a;
        rR = L.rec_R[o];
        rC = L.rec_coh[o];
        rM = L.rec_mag[o];
    }
    // the row streams from HBM: independent 16-byte loads in flight per thread
    const double2* S2 = reinterpret_cast<const double2*>(Srow);
    const int nb = blockDim.x;
// two residues (4 x 16-byte loads) in flight per thread: with 2 CTAs of 512
// threads per SM more outstanding loads only congest (4: 57.9 us, 6: 59.6,
// 2: 56.1 at C5, warm ncu)
    // (factored rows, 3 CTAs of 256 threads: 4 residues -- 2: 52.6 us, 4: 50.0, 8: 56.8)
    constexpr int FFT_U = FACT ? 4 : 2;
    for (int r0 = threadIdx.x; r0 < Pf; r0 += FFT_U * nb) {
        double2 v[FFT_U][2];
#pragma unroll
        for (int u = 0; u < FFT_U; ++u) {
            const int r = r0 + u * nb;
            if (r < Pf) {
                v[u][0] = __ldcs(S2 + 2 * r);
                v[u][1] = __ldcs(S2 + 2 * r + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < FFT_U; ++u) {
            const int r = r0 + u * nb;
            if (r >= Pf) continue;
            const int rev = (int)(__brev((unsigned)r) >> (32 - log2Pf));
            const double c[4] = {v[u][0].x, v[u][0].y, v[u][1].x, v[u][1].y};
            buf[padi(rev, sh)] = to_v<V>(combine(c, flag_bit));
        }
    }
    __syncthreads();
    {
        int off = 0;
        fft_passes(log2Pf, blockDim.x, [&](int r, int h) {
            const V* tp = tw + off;
            if (FACT) {
                switch (r) {
                    case 4: fft_pass_f<4>(buf, tw, tw + 64, Pf, h, sh); break;
                    case 3: fft_pass_f<3>(buf, tw, tw + 64, Pf, h, sh); break;
                    case 2: fft_pass_f<2>(buf, tw, tw + 64, Pf, h, sh); break;
                    default: fft_pass_f<1>(buf, tw, tw + 64, Pf, h, sh); break;
                }
            } else {
                switch (r) {
                    case 4: fft_pass<4>(buf, tp, Pf, h, sh); break;
                    case 3: fft_pass<3>(buf, tp, Pf, h, sh); break;
                    case 2: fft_pass<2>(buf, tp, Pf, h, sh); break;
                    default: fft_pass<1>(buf, tp, Pf, h, sh); break;
                }
            }
            off += r * h;
        });
    }
    const double sc = L.row_scale ? L.row_scale[row.out_block] : L.scale_default;
    if (rec_pre) {
        const int a = threadIdx.x;
        if (a >= L.A) return;
        const double2 v0 = to_d(buf[padi(L.bins[a], sh)]);
        const double2 v = make_double2(v0.x * sc, v0.y * sc);
        const size_t o = (size_t)(out - L.out) + (size_t)a * L.stride_a;
        rR.x = L.rec_decay * rR.x + v.x;
        rR.y = L.rec_decay * rR.y + v.y;
        L.rec_R[o] = rR;
        L.out[o] = rR;
        if (L.rec_host) L.rec_host[o] = rR;
        rC.x += rR.x;
        rC.y += rR.y;
        L.rec_coh[o] = rC;
        L.rec_mag[o] = rM + hypot(rR.x, rR.y);
        return;
    }
    if (L.rec_R) {
        const size_t o0 = (size_t)(out - L.out);
        for (int a = threadIdx.x; a < L.A; a += blockDim.x) {
            const double2 v0 = to_d(buf[padi(L.bins[a], sh)]);
            const double2 v = make_double2(v0.x * sc, v0.y * sc);
            const size_t o = o0 + (size_t)a * L.stride_a;
            double2 r = L.rec_R[o], c = L.rec_coh[o];
            r.x = L.rec_decay * r.x + v.x;
            r.y = L.rec_decay * r.y + v.y;
            L.rec_R[o] = r;
            L.out[o] = r;
            if (L.rec_host) L.rec_host[o] = r;
            c.x += r.x;
            c.y += r.y;
            L.rec_coh[o] = c;
            L.rec_mag[o] += hypot(r.x, r.y);
        }
        return;
    }
    // 8 bins loaded at once: the dependent index -> shared read -> store chain of
    // one bin at a time stalled on each bins[] load (13 % of the samples, ncu)
    const int nb8 = 8 * (int)blockDim.x;
    for (int a0 = threadIdx.x; a0 < L.A; a0 += nb8) {
        int bi[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int a = a0 + u * (int)blockDim.x;
            bi[u] = a < L.A ? __ldg(L.bins + a) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int a = a0 + u * (int)blockDim.x;
            if (a >= L.A) break;
            const double2 v = to_d(buf[padi(bi[u], sh)]);
            out[(size_t)a * L.stride_a] = make_double2(v.x * sc, v.y * sc);
        }
    }
}

// Direct DFT: grid (n_rows, n_flag_tables, ceil(A / DFT_AB)); a CTA computes
// DFT_AB alphas of one row with its 256 threads striding over the residues
// (twiddle index advanced exactly mod Pf), then a fixed-order block reduction.
constexpr int DFT_T = 256;
constexpr int DFT_AB = 8;
__global__ void __launch_bounds__(DFT_T) finalize_dft_kernel(FinalizeLaunch L) {
    __shared__ double2 red[DFT_T / 32][DFT_AB];
    __shared__ FinalRow s_row;  // descriptors may be in mapped host memory: read once
    if (threadIdx.x == 0) s_row = L.rows[blockIdx.x];
    if (L.shift_ctr && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        *L.shift_ctr += L.shift_inc;
    __syncthreads();
    const FinalRow row = s_row;
    const int fi = blockIdx.y;
    const int flag_bit = (L.flags == 2) ? 1 : fi;
    const int Pf = L.Pf;
    const int a0 = blockIdx.z * DFT_AB;
    const int na = min(DFT_AB, L.A - a0);
    const double* Srow = L.S + ((size_t)row.slot * L.t_pad + row.t_span) * (size_t)Pf * 4;
    int idx[DFT_AB], step[DFT_AB];
    double re[DFT_AB], im[DFT_AB];
#pragma unroll
    for (int k = 0; k < DFT_AB; ++k) {
        const int64_t bin = k < na ? L.bins[a0 + k] : 0;
        idx[k] = (int)((bin * threadIdx.x) % Pf);
        step[k] = (int)((bin * DFT_T) % Pf);
        re[k] = im[k] = 0.0;
    }
    for (int r = threadIdx.x; r < Pf; r += DFT_T) {
        const double2 v = combine(Srow + (size_t)r * 4, flag_bit);
#pragma unroll
        for (int k = 0; k < DFT_AB; ++k) {
            const double2 w = L.tw[idx[k]];
            re[k] += v.x * w.x - v.y * w.y;
            im[k] += v.x * w.y + v.y * w.x;
            idx[k] += step[k];
            if (idx[k] >= Pf) idx[k] -= Pf;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < DFT_AB; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            re[k] += __shfl_down_sync(0xffffffffu, re[k], o);
            im[k] += __shfl_down_sync(0xffffffffu, im[k], o);
        }
        if (lane == 0) red[warp][k] = make_double2(re[k], im[k]);
    }
    __syncthreads();
    if (threadIdx.x >= na) return;
    const int k = threadIdx.x;
    double sr = 0.0, si = 0.0;
    for (int w = 0; w < DFT_T / 32; ++w) {
        sr += red[w][k].x;
        si += red[w][k].y;
    }
    const double sc = L.row_scale ? L.row_scale[row.out_block] : L.scale_default;
    double2* out = L.out + (size_t)row.out_block * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                   (size_t)row.t_out * L.stride_t;
    out[(size_t)(a0 + k) * L.stride_a] = make_double2(sr * sc, si * sc);
}

}  // namespace

// FFT arithmetic: fp32 by default -- S is combined per flag in fp64 and
// rounded once, the transform's error (~1e-7 of the row's norm) sits two
// orders below the fold's and the 8192-point buffers fit two CTAs per SM
// (one streams its row while the other transforms); CYC_FFT64=1: fp64.
static bool fft64() {
    static const bool on = [] {
        const char* e = std::getenv("CYC_FFT64");
        return e && *e && *e != '0';
    }();
    return on;
}

// Threads per FFT row: Pf = 8192: 512 x radix-16 groups; shorter rows: 4
// points per thread, radix-4 passes (2 per thread: C2 8.3 -> 7.6 us, C4 16.4 ->
// 19.7 us -- kept at 4)
static int fft_threads(int Pf) { return Pf >= 8192 ? 512 : std::min(512, std::max(32, Pf / 4)); }

// Per-pass twiddle tables of a Pf-point row in the kernel's pass order:
// pass (log2r, h), level l < log2r, position pos < h: W^{pos Pf / (2^{l+1} h)}.
// out == nullptr: the count only.  Stored after the Pf plain twiddles.
int fft_pass_twiddles(int Pf, double2* out) {
    int lg = 0;
    while ((1 << lg) < Pf) ++lg;
    if ((1 << lg) != Pf || Pf > 8192) return 0;
    const int nt = fft_threads(Pf);
    int n = 0;
    fft_passes(lg, nt, [&](int r, int h) {
        for (int l = 0; l < r; ++l)
            for (int pos = 0; pos < h; ++pos, ++n) {
                if (!out) continue;
                const long long j = (long long)pos * (Pf / (2 * (h << l)));
                const long double th = -2.0L * 3.14159265358979323846264338327950288L * (long double)j / (long double)Pf;
                out[n] = make_double2((double)cosl(th), (double)sinl(th));
            }
    });
    return n;
}

template <class V>
static int fft_smem_max() {  // Pf = 8192 at 512 threads: the largest row
    return (8192 + 512 + 8 + fft_tw_entries(13, 512)) * (int)sizeof(V);
}
// factored twiddles (fft_pass_f): fp32 8192-point rows at 256 threads, three CTAs
// per SM (FFT_FACT=0: the per-pass tables, 512 threads, two CTAs per SM)
#ifndef FFT_FACT
#define FFT_FACT 1
#endif
static bool fft_fact(int Pf, bool fp32) { return FFT_FACT && fp32 && Pf == 8192; }

template <class V, bool FACT>
static void launch_fft_t(const FinalizeLaunch& L, cudaStream_t st, int nflag) {
    int lg = 0;
    while ((1 << lg) < L.Pf) ++lg;
    // Pf = 8192: 512 threads x radix-16 groups (factored: 256); shorter rows: Pf / 4 threads x radix-4
    const int nt = FACT ? 256 : fft_threads(L.Pf);
    const size_t tw_n = FACT ? (size_t)(64 + (L.Pf >> 7)) : (size_t)fft_tw_entries(lg, nt);
    const size_t smem = ((size_t)L.Pf + L.Pf / 16 + 8 + tw_n) * sizeof(V);
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set))
        cudaFuncSetAttribute(finalize_fft_kernel<V, FACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             fft_smem_max<V>());
    launch_pdl(finalize_fft_kernel<V, FACT>, dim3((unsigned)(L.n_rows * nflag)), dim3(nt), smem, st, L, lg);
}

void launch_finalize(const FinalizeLaunch& L, cudaStream_t st) {
    if (L.n_rows == 0) return;
    const int nflag = L.flags == 3 ? 2 : 1;
    if (L.use_fft) {
        if (fft64())
            launch_fft_t<double2, false>(L, st, nflag);
        else if (fft_fact(L.Pf, true))
            launch_fft_t<float2, true>(L, st, nflag);
        else
            launch_fft_t<float2, false>(L, st, nflag);
    } else {
        finalize_dft_kernel<<<dim3(L.n_rows, nflag, (L.A + DFT_AB - 1) / DFT_AB), DFT_T, 0, st>>>(L);
    }
}

}  // namespace cyc

namespace cyc {
void prepare_finalize_kernels() {
    static std::atomic<uint64_t> done{0};
    if (!first_on_device(done)) return;
    cudaFuncSetAttribute(finalize_fft_kernel<double2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fft_smem_max<double2>());
    cudaFuncSetAttribute(finalize_fft_kernel<float2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fft_smem_max<float2>());
    cudaFuncSetAttribute(finalize_fft_kernel<float2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         fft_smem_max<float2>());
}
}  // namespace cyc

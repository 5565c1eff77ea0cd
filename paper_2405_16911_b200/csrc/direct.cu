// direct.cu -- per-(alpha, tau) contraction for cycle frequencies that are not
// on a usable rational grid (e.g. alpha = 0.1234507, proj/tests/test_estimator.cpp:107-124).
//
//   R(alpha, tau) = scale * sum_n x[n+tau] y^(*)[n] e^{-j2pi alpha n}
//
// The rotator is exact-index: the phase of sample n is alpha_fx * n (mod 2^64)
// with alpha_fx = round(alpha * 2^64), i.e. an exact wrap-around fixed-point
// turn count, instead of the reference's renormalised lead-phasor recurrence
// (proj/src/estimator.cpp:70-73) or std::polar of a large argument
// (proj/src/kernels.cpp:19-24).  The phasor is folded into y once per sample
// and shared by every lag:  x conj(y e^{+j th}) and x (y e^{-j th}).
#include <algorithm>

#include "kernels.cuh"

namespace cyc {
namespace {

constexpr int DT = 256;     // threads
constexpr int TILE = 512;   // samples per smem tile
constexpr int MAXL = 4;     // lags per thread (T <= 1024)

// The last CTA of (segment si, alpha a) to finish sums the splits' partials
// (split order, fp64) into the frame's table and the running sums -- the
// arithmetic of direct_reduce_accum_kernel for one frame per channel.  Every
// thread of every CTA calls this after writing its partials.
__device__ void fused_reduce(const DirectLaunch& L, int si, int a, float2* stage, int stage_cap) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        int* ctr = L.fuse_counters + (size_t)si * L.A + a;
        s_last = atomicAdd(ctr, 1) == L.splits - 1;
        if (s_last) *ctr = 0;  // ready for the next launch (stream-ordered)
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // partials of (si, a): [split][flag][lag]
    const float2* part = reinterpret_cast<const float2*>(L.partials) + ((size_t)si * L.A + a) * L.splits * 2 * L.T;
    const int ch = si;  // one frame per channel: segment = channel
    const int nv = L.splits * 2 * L.T;
    // Short tables (C1: 16 splits x 2 x 31 lags): the whole CTA fetches every
    // partial at once into shared memory -- one L2 round trip instead of one
    // per group of splits -- and the sums below keep the split order.
    const bool staged = nv <= stage_cap;
    if (staged)
        for (int i = threadIdx.x; i < nv; i += blockDim.x) stage[i] = __ldcg(part + i);
    auto cell = [&](int idx, int& f, int& t, int& fi, int64_t& e) -> bool {
        f = idx / L.T;
        t = idx - f * L.T;
        if (idx >= 2 * L.T || !(L.flags & (1 << f))) return false;
        fi = f == 1 && (L.flags & 1) ? 1 : 0;
        e = (int64_t)ch * L.per + (int64_t)fi * L.out_flag_stride + (int64_t)a * L.stride_a + (int64_t)t * L.stride_t;
        return true;
    };
    // only this CTA touches the running sums of (si, a): the first pass fetches
    // them beside the partials
    int f, t, fi;
    int64_t e;
    double2 c0 = make_double2(0.0, 0.0);
    double m0 = 0.0;
    if (cell(threadIdx.x, f, t, fi, e)) {
        c0 = L.coh[e];
        m0 = L.mag[e];
    }
    __syncthreads();  // s_last is uniform: every thread of the last CTA is here
    for (int idx = threadIdx.x; idx < 2 * L.T; idx += blockDim.x) {
        if (!cell(idx, f, t, fi, e)) continue;
        double2 c = c0;
        double m = m0;
        if (idx != (int)threadIdx.x) {
            c = L.coh[e];
            m = L.mag[e];
        }
        double re = 0.0, im = 0.0;
        for (int s = 0; s < L.splits; ++s) {
            const float2 v = staged ? stage[(s * 2 + f) * L.T + t] : __ldcg(part + (s * 2 + f) * L.T + t);
            re += v.x;
            im += v.y;
        }
        const double2 v = make_double2(re * L.scale, im * L.scale);
        const size_t o = (size_t)si * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                         (size_t)a * L.stride_a + (size_t)t * L.stride_t;
        L.out[o] = v;
        if (L.out_host) L.out_host[o] = v;
        c.x += v.x;
        c.y += v.y;
        L.coh[e] = c;
        L.mag[e] = m + hypot(v.x, v.y);
    }
}

// Threads: SL sample lanes x (DT / SL) lag slots.  Short lag spans (T <= 32)
// use 8 lanes, so every thread works; each lane sums the samples i = sub
// (mod SL) of its lags, and the lanes combine in a fixed order in shared memory.
__global__ void __launch_bounds__(DT) direct_kernel(const __grid_constant__ DirectLaunch L, int span, int SL) {
    extern __shared__ float2 sm[];
    float2* xs = sm;                  // TILE + span
    float2* yc = xs + TILE + span;    // y * e^{+j th}
    float2* yj = yc + TILE;           // y * e^{-j th}
    const int split = blockIdx.x % L.splits;
    const int a = (blockIdx.x / L.splits) % L.A;
    const int si = blockIdx.x / (L.splits * L.A);
    __shared__ DirectSeg s_seg;  // descriptors may be in mapped host memory: read once
    if (threadIdx.x == 0) s_seg = L.segs ? L.segs[si] : L.inl[si];
    __syncthreads();
    const DirectSeg& seg = s_seg;
    const uint64_t afx = L.alpha_fx[a];
    const int64_t cnt = seg.n_end - seg.n_start;
    const int64_t b0 = seg.n_start + cnt * split / L.splits;
    const int64_t b1 = seg.n_start + cnt * (split + 1) / L.splits;
    const int LT = DT / SL;              // lag slots
    const int slot = threadIdx.x % LT, sub = threadIdx.x / LT;

    float2 accv[MAXL], accj[MAXL];
    int loff[MAXL];
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        accv[k] = make_float2(0.f, 0.f);
        accj[k] = make_float2(0.f, 0.f);
        const int t = slot + k * LT;
        loff[k] = t < L.T ? L.lags[t] - L.lag_lo : -1;
    }
    for (int64_t n0 = b0; n0 < b1; n0 += TILE) {
        const int len = (int)min((int64_t)TILE, b1 - n0);
        __syncthreads();
        // y loads first, so they are in flight beside the x loads
        float2 yr[TILE / DT];
#pragma unroll
        for (int k = 0; k < TILE / DT; ++k) {
            const int i = threadIdx.x + k * DT;
            if (i < len) yr[k] = seg.y[(uint64_t)(n0 + i) & seg.mask];
        }
        for (int i = threadIdx.x; i < len + span; i += DT) {
            const int64_t n = n0 + L.lag_lo + i;
            xs[i] = (n >= seg.x_lo && n < seg.x_hi) ? seg.x[(uint64_t)n & seg.mask] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < TILE / DT; ++k) {
            const int i = threadIdx.x + k * DT;
            if (i >= len) continue;
            const int64_t n = n0 + i;
            float2 y = yr[k];
            if (seg.w_log2 != 0.f) {
                const float w = seg.w_scale * exp2f((float)(seg.w_ref - n) * seg.w_log2);
                y.x *= w;
                y.y *= w;
            }
            const uint64_t ph = afx * (uint64_t)n;                    // exact turns * 2^64 (mod 1 turn)
            const float u = (float)(int)(ph >> 32) * 4.656612873077393e-10f;  // 2 * turns in [-1, 1)
            float sn, cs;
            sincospif(u, &sn, &cs);
            yc[i] = make_float2(y.x * cs - y.y * sn, y.x * sn + y.y * cs);
            yj[i] = make_float2(y.x * cs + y.y * sn, y.y * cs - y.x * sn);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MAXL; ++k) {
            if (loff[k] < 0) continue;
            float2 av = accv[k], aj = accj[k];
            const float2* xp = xs + loff[k];
            for (int i = sub; i < len; i += SL) {
                const float2 xv = xp[i], c = yc[i], j = yj[i];
                av.x += xv.x * c.x + xv.y * c.y;   // x * conj(c)
                av.y += xv.y * c.x - xv.x * c.y;
                aj.x += xv.x * j.x - xv.y * j.y;   // x * j
                aj.y += xv.x * j.y + xv.y * j.x;
            }
            accv[k] = av;
            accj[k] = aj;
        }
    }
    float2* part = reinterpret_cast<float2*>(L.partials);
    const size_t base = (((size_t)si * L.A + a) * L.splits + split) * 2;
    if (SL == 1) {
#pragma unroll
        for (int k = 0; k < MAXL; ++k) {
            const int t = slot + k * LT;
            if (t >= L.T) continue;
            part[(base + 0) * L.T + t] = accv[k];
            part[(base + 1) * L.T + t] = accj[k];
        }
        if (L.fuse_counters) fused_reduce(L, si, a, sm, 3 * TILE + span);
        return;
    }
    // lanes 1.. hand their sums to lane 0 through shared memory (reusing the
    // sample tiles), which adds them in lane order
    __syncthreads();
    float2* red = sm;  // [SL][MAXL][LT] x 2
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        red[((sub * MAXL + k) * LT + slot) * 2 + 0] = accv[k];
        red[((sub * MAXL + k) * LT + slot) * 2 + 1] = accj[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
        const int t = slot + k * LT;
        if (sub != 0 || t >= L.T) continue;  // lane 0 writes (no early return: the fused reduce syncs the CTA)
        float2 v = red[((0 * MAXL + k) * LT + slot) * 2 + 0], j = red[((0 * MAXL + k) * LT + slot) * 2 + 1];
        for (int q = 1; q < SL; ++q) {
            const float2 v2 = red[((q * MAXL + k) * LT + slot) * 2 + 0];
            const float2 j2 = red[((q * MAXL + k) * LT + slot) * 2 + 1];
            v.x += v2.x;
            v.y += v2.y;
            j.x += j2.x;
            j.y += j2.y;
        }
        part[(base + 0) * L.T + t] = v;
        part[(base + 1) * L.T + t] = j;
    }
    if (L.fuse_counters) fused_reduce(L, si, a, sm, 3 * TILE + span);
}

__global__ void direct_reduce_kernel(const __grid_constant__ DirectLaunch L) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = blockIdx.y;
    const int si = blockIdx.z;
    const float2* part = reinterpret_cast<const float2*>(L.partials);
    __shared__ DirectSeg s_seg;  // descriptors may be in mapped host memory: read once
    if (threadIdx.x == 0) s_seg = L.segs ? L.segs[si] : L.inl[si];
    __syncthreads();
    if (t >= L.T) return;
    const DirectSeg& seg = s_seg;
    int fi = 0;
    for (int f = 0; f < 2; ++f) {
        if (!(L.flags & (1 << f))) continue;
        double re = 0.0, im = 0.0;
        for (int s = 0; s < L.splits; ++s) {
            const float2 v = part[((((size_t)si * L.A + a) * L.splits + s) * 2 + f) * L.T + t];
            re += v.x;
            im += v.y;
        }
        double2* out = L.out + (size_t)seg.out_block * L.out_block_stride + (size_t)fi * L.out_flag_stride;
        out[(size_t)a * L.stride_a + (size_t)t * L.stride_t] = make_double2(re * L.scale, im * L.scale);
        ++fi;
    }
}

// direct_reduce_kernel fused with the running average_frames sums
// (accum_frames_kernel): one thread per (channel, alpha, lag) walks the batch's
// frames in order, so the sums are bit-identical to the separate kernels'.
// Segments are [frame][channel]; out_block = segment index.
__global__ void direct_reduce_accum_kernel(const __grid_constant__ DirectLaunch L, int n_frames, int C, double2* coh,
                                           double* mag, int64_t per) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = blockIdx.y;
    const int ch = blockIdx.z;
    if (t >= L.T) return;
    const float2* part = reinterpret_cast<const float2*>(L.partials);
    int fi = 0;
    for (int f = 0; f < 2; ++f) {
        if (!(L.flags & (1 << f))) continue;
        const int64_t e = (int64_t)ch * per + (int64_t)fi * L.out_flag_stride + (int64_t)a * L.stride_a +
                          (int64_t)t * L.stride_t;
        double2 c = coh[e];
        double m = mag[e];
        for (int fr = 0; fr < n_frames; ++fr) {
            const int si = fr * C + ch;
            double re = 0.0, im = 0.0;
            for (int s = 0; s < L.splits; ++s) {
                const float2 v = part[((((size_t)si * L.A + a) * L.splits + s) * 2 + f) * L.T + t];
                re += v.x;
                im += v.y;
            }
            const double2 v = make_double2(re * L.scale, im * L.scale);
            const size_t o = (size_t)si * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                             (size_t)a * L.stride_a + (size_t)t * L.stride_t;
            L.out[o] = v;
            if (L.out_host) L.out_host[o] = v;
            c.x += v.x;
            c.y += v.y;
            m += hypot(v.x, v.y);
        }
        coh[e] = c;
        mag[e] = m;
        ++fi;
    }
}

}  // namespace

// sample lanes per lag: every thread busy for short lag spans (MAXL lags per thread at most)
int direct_lanes(int T) {
    int sl = 1;
    while (sl < 8 && (DT / (2 * sl)) * MAXL >= T && DT / (2 * sl) >= 32) sl *= 2;
    return sl;
}

void launch_direct(const DirectLaunch& L, cudaStream_t st, double2* coh, double* mag, int channels, int64_t per) {
    if (L.n_segs == 0) return;
    const int span = L.lag_hi - L.lag_lo;
    const int SL = direct_lanes(L.T);
    const size_t smem = std::max<size_t>((size_t)(TILE + span + 2 * TILE) * sizeof(float2),
                                         (size_t)SL * MAXL * (DT / SL) * 2 * sizeof(float2));
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set))
        cudaFuncSetAttribute(direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    direct_kernel<<<L.n_segs * L.A * L.splits, DT, smem, st>>>(L, span, SL);
    if (L.fuse_counters) return;  // reduced by the last CTA of each (segment, alpha)
    if (coh)
        direct_reduce_accum_kernel<<<dim3((L.T + 127) / 128, L.A, channels), 128, 0, st>>>(L, L.n_segs / channels,
                                                                                          channels, coh, mag, per);
    else
        direct_reduce_kernel<<<dim3((L.T + 127) / 128, L.A, L.n_segs), 128, 0, st>>>(L);
}

}  // namespace cyc

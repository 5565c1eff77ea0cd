// fold.cu -- the hot kernel: lag products folded over residues n mod Pf.
//
// For every computed lag tau and residue r it accumulates the four real
// correlations
//     c0 = sum xr*yr,  c1 = sum xi*yr,  c2 = sum xr*yi,  c3 = sum xi*yi
// over n = r (mod Pf), x = x[n+tau], y = y[n].  Both cyclic functions follow:
//     x*conj(y) = (c0 + c3) + j(c1 - c2)     (conj == false, kernels.cpp:50-51)
//     x*y       = (c0 - c3) + j(c1 + c2)     (conj == true)
// so one pass costs 4 FP32 FMAs per (tau, n) for BOTH flags.  The reference
// recomputes the lag product once per alpha (proj/src/kernels.cpp:46-55);
// here it is computed once per (tau, n) and reused by every alpha in the
// finalize DFT (exact reassociation: every alpha is k/P and Pf is a multiple
// of P).
//
// CTA = 8 warps, 1 CTA/SM (~215 registers).  A thread owns R=4 consecutive
// residues x U=8 consecutive lags = 128 fp32 accumulators, updated with packed
// FFMA2 (y broadcast as the scalar operand).  Sample windows are staged per
// fold period by 16-byte cp.async into a "pair, phase-split by 2" layout
//     X[b][c] = (x[4c+2b], x[4c+2b+1])        (float4)
// so a thread's sliding window x[4k .. 4k+11] is 6 LDS.128 at consecutive
// addresses across lanes (conflict-free), and its 4 y samples are 2 LDS.128
// broadcast across the lag lanes.  Per period a thread issues 8 LDS.128 for
// 64 FFMA2 (128 FMAs); the next period's registers are loaded while the
// current one is multiplied.  Partial sums leave the CTA in fp32 and are
// reduced in fp64 in a fixed order (deterministic).
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace cyc {
namespace {

constexpr int NW = 8;
constexpr int NT = NW * 32;
constexpr int R = 4;
constexpr int U = 8;
constexpr int NSTAGE = 2;

constexpr int pad4mod8(int c) { return c + ((4 - c % 8) + 8) % 8; }

template <int LW>
struct Geo {
    static constexpr int RL = 32 / LW;           // residue lanes per warp
    static constexpr int TB = 8 * LW;            // lags per CTA
    static constexpr int RB = NW * RL * R;       // residues per CTA (= 1024 / LW)
    static constexpr int XW = RB + TB;           // x samples staged per period
    static constexpr int XC = pad4mod8(XW / 4);  // float4 per X row
    static constexpr int YC = pad4mod8(RB / 4);  // float4 per Y row
    static constexpr int PER = 2 * XC + 2 * YC;  // float4 per period
    static constexpr int NX = XW / 2;            // x pairs per period
    static constexpr int NY = RB / 2;            // y pairs per period
    static constexpr int EPP = NX + NY;          // staged pairs per period
    static constexpr int PS = LW == 8 ? 32 : (LW == 4 ? 16 : 8);  // periods per stage
    static constexpr int STAGE = PS * PER;
    static constexpr int SMEM = NSTAGE * STAGE * 16;
    static constexpr int EPT = (PS * EPP + NT - 1) / NT;  // staged pairs per thread per stage
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

union F2U {
    float2 f;
    unsigned long long u;
};

// acc += a * (b, b)  -- packed fp32x2 FMA (SASS FFMA2 with a scalar operand)
__device__ __forceinline__ void ffma2_bcast(float2& acc, float2 a, float b) {
    F2U A, B, C;
    A.f = a;
    B.f = make_float2(b, b);
    C.f = acc;
    asm("fma.rn.f32x2 %0, %1, %2, %0;\n" : "+l"(C.u) : "l"(A.u), "l"(B.u));
    acc = C.f;
}

struct Regs {
    float4 x[6];  // x[4k .. 4k+11] as pairs
    float4 y[2];  // y[4rho .. 4rho+3] as pairs
};

// y pairs come from the Y rows, or -- in a self stage -- from the X rows
// (x == y and the y window lies inside the staged x window): yb0/yb1 are the
// float4 row offsets of (y[4rho], y[4rho+1]) and (y[4rho+2], y[4rho+3]).
template <int LW>
__device__ __forceinline__ void load_period(Regs& r, const float4* per, int kap, int rho, int yb0, int yb1) {
    using G = Geo<LW>;
#pragma unroll
    for (int j = 0; j < 6; ++j) r.x[j] = per[(j & 1) * G::XC + kap + (j >> 1)];
    r.y[0] = per[yb0 + rho];
    r.y[1] = per[yb1 + rho];
}

__device__ __forceinline__ void mac_period(float2 (&lo)[R][U], float2 (&hi)[R][U], const Regs& r) {
    float2 xv[12];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        xv[2 * j] = make_float2(r.x[j].x, r.x[j].y);
        xv[2 * j + 1] = make_float2(r.x[j].z, r.x[j].w);
    }
    const float yr[4] = {r.y[0].x, r.y[0].z, r.y[1].x, r.y[1].z};
    const float yi[4] = {r.y[0].y, r.y[0].w, r.y[1].y, r.y[1].w};
    // lo/hi of one (a, u) share the x pair (operand reuse cache); ptxas
    // schedules these pairs back to back.  Measured ceiling of this operand
    // pattern (tools/microbench/ffma2_pattern.cu): ~75% of the FP32 peak.
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ffma2_bcast(lo[a][u], xv[a + u], yr[a]);
            ffma2_bcast(hi[a][u], xv[a + u], yi[a]);
        }
}

// recursive mode: y[n] *= w_scale * 2^{(w_ref - n) * w_log2}
__device__ __forceinline__ void weight_period(Regs& r, const FoldSeg& seg, int64_t nb) {
    float w[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) w[a] = seg.w_scale * exp2f((float)(seg.w_ref - (nb + a)) * seg.w_log2);
    r.y[0].x *= w[0];
    r.y[0].y *= w[0];
    r.y[0].z *= w[1];
    r.y[0].w *= w[1];
    r.y[1].x *= w[2];
    r.y[1].y *= w[2];
    r.y[1].z *= w[3];
    r.y[1].w *= w[3];
}

// One stage's periods.  The next period's registers load while the current
// one multiplies; the loads are unconditional (the last re-reads period nq-1)
// so the loop body is one basic block and ptxas can spread the LDS between
// the FFMA2s.  W: recursive-mode weights (compile-time, no branch in the body).
template <int LW, bool W>
__device__ __forceinline__ void compute_stage(float2 (&lo)[R][U], float2 (&hi)[R][U], const float4* st, int nq,
                                              int kap, int rho, int yb0, int yb1, const FoldSeg& seg, int64_t n0,
                                              int64_t Pf) {
    using G = Geo<LW>;
    Regs ra, rb;
    load_period<LW>(ra, st, kap, rho, yb0, yb1);
    int q = 0;
    for (; q + 1 < nq; q += 2) {
        load_period<LW>(rb, st + (q + 1) * G::PER, kap, rho, yb0, yb1);
        if (W) weight_period(ra, seg, n0 + q * Pf);
        mac_period(lo, hi, ra);
        load_period<LW>(ra, st + min(q + 2, nq - 1) * G::PER, kap, rho, yb0, yb1);
        if (W) weight_period(rb, seg, n0 + (q + 1) * Pf);
        mac_period(lo, hi, rb);
    }
    if (q < nq) {
        if (W) weight_period(ra, seg, n0 + q * Pf);
        mac_period(lo, hi, ra);
    }
}

struct NoInline {};

template <int LW, bool INL>
__global__ void __launch_bounds__(NT, 1)
    fold_kernel(FoldLaunch L, const __grid_constant__ std::conditional_t<INL, FoldInline, NoInline> D) {
    using G = Geo<LW>;
    extern __shared__ __align__(16) float4 smem4[];
    // Descriptors come from the parameter block or (pointer launches) from
    // device / mapped memory: copy them to shared memory once.
    __shared__ FoldTile s_tile;
    __shared__ FoldSeg s_seg;
    if (threadIdx.x == 0) {
        if constexpr (INL)
            s_tile = D.tiles[blockIdx.x];
        else
            s_tile = L.tiles[blockIdx.x];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if constexpr (INL)
            s_seg = D.segs[s_tile.seg];
        else
            s_seg = L.segs[s_tile.seg];
    }
    __syncthreads();
    const FoldTile& tile = s_tile;
    const FoldSeg& seg = s_seg;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int rho = warp * G::RL + (lane % G::RL);  // residues 4*rho .. 4*rho+3
    const int lam = lane / G::RL;                   // lags 8*lam .. 8*lam+7
    const int kap = rho + 2 * lam;                  // x window starts at 4*kap

    const int64_t Pf = L.Pf;
    const int64_t res0 = (int64_t)tile.rb * G::RB;
    const int64_t xoff = res0 + L.lag_lo + (int64_t)tile.lb * G::TB;
    const int nper = (int)(tile.p1 - tile.p0);
    const int nstages = (nper + G::PS - 1) / G::PS;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem4);
    const uint64_t mask = seg.mask;
    const bool vec = seg.vec != 0;

    // Staging assignment: stage element idx = tid + k*NT is pair e of period q;
    // (q, e) advance incrementally so no per-element table lives in registers.
    const int q_first = tid / G::EPP;
    const int e_first = tid - q_first * G::EPP;
    constexpr int DQ = NT / G::EPP, DE = NT % G::EPP;

    // x window offset from the residue: d = lag_lo + lb*TB.  Self stages read y
    // from the X rows when x == y and [res, res+RB) sits inside the x window
    // at a 4-sample boundary (every BASELINE config: lags start at 0 or -M).
    const int64_t dwin = (int64_t)L.lag_lo + (int64_t)tile.lb * G::TB;
    const bool self_ok = seg.x == seg.y && dwin <= 0 && -dwin <= G::TB && ((-dwin) & 3) == 0;
    const int yshift = (int)(-dwin) / 4;

    // stage-uniform fast path: every window of the stage inside the valid
    // ranges and (ring input) no wrap inside the stage
    auto stage_fast = [&](int s) -> bool {
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const int64_t pend = pbeg + G::PS;
        if (!(vec && pend <= tile.p1 && pbeg * Pf + xoff >= seg.x_lo && (pend - 1) * Pf + xoff + G::XW <= seg.x_hi &&
              pbeg * Pf + res0 >= seg.n_start && (pend - 1) * Pf + res0 + G::RB <= seg.n_end && res0 + G::RB <= Pf))
            return false;
        if (mask == ~0ull) return true;
        const uint64_t span = (uint64_t)(G::PS - 1) * (uint64_t)Pf;
        return ((uint64_t)(pbeg * Pf + xoff) & mask) + span + G::XW <= mask + 1 &&
               ((uint64_t)(pbeg * Pf + res0) & mask) + span + G::RB <= mask + 1;
    };

    auto load_stage = [&](int s) {
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const uint32_t dst0 = sbase + (uint32_t)((s % NSTAGE) * G::STAGE) * 16u;
        if (stage_fast(s)) {
            // column-fixed assignment: a thread owns one staged pair column
            // (x or y, phase b, float4 c) and walks the stage's periods, so an
            // element costs one cp.async plus two pointer increments
            const int cols = self_ok ? G::NX : G::EPP;
            const bool wide = cols > NT;
            const int qs = wide ? 1 : NT / cols;
            int col = wide ? tid : tid % cols;
            const int q0 = wide ? 0 : tid / cols;
            if (q0 >= qs) return;
            for (; col < cols; col += wide ? NT : cols) {
                const bool isx = col < G::NX;
                const int ee = isx ? col : col - G::NX;
                const int b = ee & 1, c = ee >> 1;
                uint32_t dst = dst0 + (uint32_t)(q0 * G::PER + (isx ? b * G::XC + c : 2 * G::XC + b * G::YC + c)) * 16u;
                const int64_t n = (pbeg + q0) * Pf + (isx ? xoff : res0) + (4 * c + 2 * b);
                const float2* src = (isx ? seg.x : seg.y) + ((uint64_t)n & mask);
                const uint32_t dstep = (uint32_t)(qs * G::PER) * 16u;
                const int64_t sstep = (int64_t)qs * Pf;
#pragma unroll 4
                for (int q = q0; q < G::PS; q += qs) {
                    cp_async16(dst, src, 16);
                    dst += dstep;
                    src += sstep;
                }
            }
            return;
        }
        int q = q_first, e = e_first;
#pragma unroll 1
        for (int k = 0; k < G::EPT; ++k) {
            if (q < G::PS) {
                const bool isx = e < G::NX;
                const int ee = isx ? e : e - G::NX;
                const int b = ee & 1, c = ee >> 1;
                const int rel = 4 * c + 2 * b;
                const uint32_t dst = dst0 + (uint32_t)(q * G::PER + (isx ? b * G::XC + c : 2 * G::XC + b * G::YC + c)) * 16u;
                const int64_t p = pbeg + q;
                int64_t n, lo, hi;
                const float2* base;
                if (isx) {
                    n = p * Pf + xoff + rel;
                    lo = seg.x_lo;
                    hi = seg.x_hi;
                    base = seg.x;
                } else {
                    n = p * Pf + res0 + rel;
                    lo = seg.n_start;
                    hi = (res0 + rel < Pf) ? seg.n_end : lo;  // masked residue-block tail
                    base = seg.y;
                }
                if (p >= tile.p1) hi = lo;
                const bool v0 = n >= lo && n < hi;
                const bool v1 = n + 1 >= lo && n + 1 < hi;
                if (vec && v0 == v1) {
                    cp_async16(dst, v0 ? (const void*)(base + ((uint64_t)n & mask)) : (const void*)base, v0 ? 16 : 0);
                } else {
                    cp_async8(dst, v0 ? (const void*)(base + ((uint64_t)n & mask)) : (const void*)base, v0 ? 8 : 0);
                    cp_async8(dst + 8, v1 ? (const void*)(base + ((uint64_t)(n + 1) & mask)) : (const void*)base,
                              v1 ? 8 : 0);
                }
            }
            q += DQ;
            e += DE;
            if (e >= G::EPP) {
                e -= G::EPP;
                ++q;
            }
        }
    };

    float2 lo[R][U], hi[R][U];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            lo[a][u] = make_float2(0.f, 0.f);
            hi[a][u] = make_float2(0.f, 0.f);
        }

#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
        if (s < nstages) load_stage(s);
        cp_async_commit();
    }

    const bool weighted = seg.w_log2 != 0.f;
    for (int s = 0; s < nstages; ++s) {
        cp_async_wait<NSTAGE - 2>();
        __syncthreads();
        if (s + NSTAGE - 1 < nstages) load_stage(s + NSTAGE - 1);
        cp_async_commit();

        const float4* st = smem4 + (s % NSTAGE) * G::STAGE;
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const int nq = min(G::PS, nper - s * G::PS);
        const bool self_st = self_ok && stage_fast(s);
        const int yb0 = self_st ? yshift : 2 * G::XC;
        const int yb1 = self_st ? G::XC + yshift : 2 * G::XC + G::YC;
        if (weighted)
            compute_stage<LW, true>(lo, hi, st, nq, kap, rho, yb0, yb1, seg, pbeg * Pf + res0 + 4 * rho, Pf);
        else
            compute_stage<LW, false>(lo, hi, st, nq, kap, rho, yb0, yb1, seg, 0, Pf);
    }
    cp_async_wait<0>();

    // fp32 partials: [tile][lag][residue] float4 (c0, c1, c2, c3)
    float4* part = reinterpret_cast<float4*>(L.partials) + (size_t)blockIdx.x * G::TB * G::RB;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int u = 0; u < U; ++u)
            part[(size_t)(lam * U + u) * G::RB + 4 * rho + a] =
                make_float4(lo[a][u].x, lo[a][u].y, hi[a][u].x, hi[a][u].y);
}

// S[slot][lb*TB + lag][rb*RB + res][4] += sum over the group's tiles (fixed order, fp64).
template <bool INL>
__global__ void fold_reduce_kernel(FoldLaunch L, int TB, int RB,
                                   const __grid_constant__ std::conditional_t<INL, FoldInline, NoInline> D) {
    if (L.gate && *L.gate != ~0ull) return;
    __shared__ FoldGroup s_g;
    __shared__ int s_slot;
    if (threadIdx.x == 0) {
        if constexpr (INL) {
            s_g = D.groups[blockIdx.y];
            s_slot = D.segs[s_g.seg].slot;
        } else {
            s_g = L.groups[blockIdx.y];
            s_slot = L.segs[s_g.seg].slot;
        }
    }
    __syncthreads();
    const FoldGroup g = s_g;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= TB * RB) return;
    const int lag = e / RB, res = e - lag * RB;
    const int64_t rg = (int64_t)g.rb * RB + res;
    const int tg = g.lb * TB + lag;
    if (rg >= L.Pf || tg >= L.t_pad) return;
    const float4* part = reinterpret_cast<const float4*>(L.partials) + e;
    const size_t stride = (size_t)TB * RB;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    // 8 independent loads in flight per thread (the partials were just written
    // and sit in L2); the fp64 sum keeps the fixed tile order.
    int t = g.t0;
    for (; t + 8 <= g.t1; t += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(part + (size_t)(t + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s0 += v[u].x;
            s1 += v[u].y;
            s2 += v[u].z;
            s3 += v[u].w;
        }
    }
    for (; t < g.t1; ++t) {
        const float4 v = __ldcs(part + (size_t)t * stride);
        s0 += v.x;
        s1 += v.y;
        s2 += v.z;
        s3 += v.w;
    }
    const int slot = s_slot;
    double* d = L.S + (((size_t)slot * L.t_pad + tg) * (size_t)L.Pf + (size_t)rg) * 4;
    if (L.overwrite) {
        d[0] = s0;
        d[1] = s1;
        d[2] = s2;
        d[3] = s3;
    } else {
        d[0] += s0;
        d[1] += s1;
        d[2] += s2;
        d[3] += s3;
    }
}

// floor(a / b) for b > 0 without the 64-bit integer division routine: a double
// estimate, corrected exactly with integer multiplies
__device__ __forceinline__ int64_t floor_div_d(int64_t a, int64_t b) {
    int64_t q = (int64_t)floor((double)a / (double)b);
    while (q * b > a) --q;
    while ((q + 1) * b <= a) ++q;
    return q;
}

__device__ __forceinline__ void shift_seg(FoldSeg& g, int64_t d) {
    g.n_start += d;
    g.n_end += d;
    g.x_lo += d;
    g.x_hi += d;
    g.w_ref += d;
}

// Small per-frame folds (recursive emissions, short per-frame windows): one
// thread per (slot, lag, residue) sums its few periods straight into S in
// fp64 -- one launch, no partials and no reduce.  Same weights and the same
// (c0, c1, c2, c3) = (xr yr, xi yr, xr yi, xi yi) as fold_kernel.
__global__ void __launch_bounds__(128) fold_small_kernel(const FoldSeg* __restrict__ segs, int Pf, int lag_lo,
                                                         int t_pad, double* __restrict__ S,
                                                         const int64_t* __restrict__ shift) {
    // segs may be mapped host memory (a replayed emission graph rewrites them
    // in place instead of copying them): one read per CTA
    __shared__ FoldSeg s_g;
    static_assert(sizeof(FoldSeg) % 4 == 0 && sizeof(FoldSeg) / 4 <= 128, "FoldSeg words");
    if (threadIdx.x < sizeof(FoldSeg) / 4)
        reinterpret_cast<uint32_t*>(&s_g)[threadIdx.x] = reinterpret_cast<const uint32_t*>(segs + blockIdx.z)[threadIdx.x];
    __syncthreads();
    if (shift) {
        if (threadIdx.x == 0) shift_seg(s_g, *shift);
        __syncthreads();
    }
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (r >= Pf) return;
    const FoldSeg& g = s_g;
    // periods p with n = p Pf + r in [n_start, n_end)
    const int64_t pa = floor_div_d(g.n_start - r + Pf - 1, Pf);
    const int64_t pb = floor_div_d(g.n_end - 1 - r, Pf) + 1;
    const bool weighted = g.w_log2 != 0.f;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    int64_t n = pa * Pf + r;
    const int64_t lag = (int64_t)lag_lo + t;
    auto acc = [&](float2 yv, const float2 xv, int64_t nn) {
        if (weighted) {
            const float w = g.w_scale * exp2f((float)(g.w_ref - nn) * g.w_log2);
            yv.x *= w;
            yv.y *= w;
        }
        c0 = fma((double)xv.x, (double)yv.x, c0);
        c1 = fma((double)xv.y, (double)yv.x, c1);
        c2 = fma((double)xv.x, (double)yv.y, c2);
        c3 = fma((double)xv.y, (double)yv.y, c3);
    };
    // 8 periods' loads in flight before their FMAs (the loop is latency-bound)
    constexpr int U = 8;
    int64_t p = pa;
    for (; p + U <= pb; p += U, n += U * (int64_t)Pf) {
        float2 yv[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            yv[u] = __ldg(g.y + ((uint64_t)(n + u * (int64_t)Pf) & g.mask));
            xv[u] = __ldg(g.x + ((uint64_t)(n + u * (int64_t)Pf + lag) & g.mask));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc(yv[u], xv[u], n + u * (int64_t)Pf);
    }
    for (; p < pb; ++p, n += Pf) acc(__ldg(g.y + ((uint64_t)n & g.mask)), __ldg(g.x + ((uint64_t)(n + lag) & g.mask)), n);
    double2* d = reinterpret_cast<double2*>(S + (((size_t)g.slot * t_pad + t) * (size_t)Pf + (size_t)r) * 4);
    d[0] = make_double2(c0, c1);
    d[1] = make_double2(c2, c3);
}

// Whole-frame folds with few lags (recursive emissions, per-frame windows): a
// CTA owns FR_RB residues of one slot; it stages FR_PCH periods of y (weighted
// once per sample, the same fp32 weights as fold_small_kernel) and of the x
// window in shared memory as fp64.  Its 1024 threads are (residue, lag group,
// period group): each accumulates LPT lags of one residue over every FR_PG-th
// period with exact fp32 x fp32 products in fp64, and the FR_PG partial sums
// meet in shared memory in a fixed order.  The fp64 pipe is latency-bound at a
// few warps per SM, so the period split buys the parallelism (C3 emissions:
// 64 periods x 32 lags x 1024 residues).
constexpr int FR_RB = 8, FR_LG = 32, FR_PCH = 64;
// period groups: 4 at one lag per thread (1024 threads), fewer when a thread
// carries more lags (register budget)
template <int LPT>
constexpr int fr_pg() { return LPT == 1 ? 4 : LPT == 2 ? 2 : 1; }
template <int LPT>
constexpr int fr_nt() { return FR_RB * FR_LG * fr_pg<LPT>(); }
template <int LPT>
constexpr int fr_smem() {
    return (FR_PCH * (FR_RB + FR_RB + FR_LG * LPT - 1) > (fr_pg<LPT>() - 1) * FR_RB * FR_LG * LPT * 2
                ? FR_PCH * (FR_RB + FR_RB + FR_LG * LPT - 1)
                : (fr_pg<LPT>() - 1) * FR_RB * FR_LG * LPT * 2) *
           (int)sizeof(double2);
}

template <int LPT>
__global__ void __launch_bounds__(fr_nt<LPT>()) fold_frame_kernel(const FoldSeg* __restrict__ segs, int Pf, int lag_lo,
                                                           int t_span, int t_pad, double* __restrict__ S,
                                                           const int64_t* __restrict__ shift) {
    constexpr int XW = FR_RB + FR_LG * LPT - 1;
    constexpr int FR_PG = fr_pg<LPT>(), FR_NT = fr_nt<LPT>();
    extern __shared__ double2 fr_smem_buf[];
    double2* ys = fr_smem_buf;                   // [FR_PCH][FR_RB]
    double2* xs = fr_smem_buf + FR_PCH * FR_RB;  // [FR_PCH][XW]
    __shared__ FoldSeg s_g;
    static_assert(sizeof(FoldSeg) % 4 == 0 && sizeof(FoldSeg) / 4 <= FR_NT, "FoldSeg words");
    if (threadIdx.x < sizeof(FoldSeg) / 4)
        reinterpret_cast<uint32_t*>(&s_g)[threadIdx.x] = reinterpret_cast<const uint32_t*>(segs + blockIdx.y)[threadIdx.x];
    __syncthreads();
    if (shift) {
        if (threadIdx.x == 0) shift_seg(s_g, *shift);
        __syncthreads();
    }
    const FoldSeg& g = s_g;
    const int r0 = blockIdx.x * FR_RB;
    const int ri = threadIdx.x % FR_RB, lg = (threadIdx.x / FR_RB) % FR_LG, pg = threadIdx.x / (FR_RB * FR_LG);
    const int r = r0 + ri;
    const bool weighted = g.w_log2 != 0.f;
    // this residue's periods (fold_small_kernel's range) and the block's union
    const int64_t pa = floor_div_d(g.n_start - r + Pf - 1, Pf), pb = floor_div_d(g.n_end - 1 - r, Pf) + 1;
    const int64_t Pa = floor_div_d(g.n_start - (r0 + FR_RB - 1) + Pf - 1, Pf), Pb = floor_div_d(g.n_end - 1 - r0, Pf) + 1;
    double c[LPT][4];
#pragma unroll
    for (int k = 0; k < LPT; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0.0;
    for (int64_t c0 = Pa; c0 < Pb; c0 += FR_PCH) {
        const int np = (int)min((int64_t)FR_PCH, Pb - c0);
        // U loads in flight per thread before their conversions and stores
        constexpr int U = 4;
        const int64_t ybase = c0 * Pf + r0, xbase = ybase + lag_lo;
        for (int i0 = threadIdx.x; i0 < np * FR_RB; i0 += U * FR_NT) {
            float2 yv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * FR_NT, pp = i / FR_RB;
                const int64_t n = ybase + (pp * Pf + (i - pp * FR_RB));
                yv[u] = (i < np * FR_RB && n >= g.n_start && n < g.n_end) ? __ldg(g.y + ((uint64_t)n & g.mask))
                                                                          : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * FR_NT, pp = i / FR_RB;
                if (i >= np * FR_RB) break;
                if (weighted) {
                    const int64_t n = ybase + (pp * Pf + (i - pp * FR_RB));
                    const float w = g.w_scale * exp2f((float)(g.w_ref - n) * g.w_log2);
                    yv[u].x *= w;
                    yv[u].y *= w;
                }
                ys[i] = make_double2((double)yv[u].x, (double)yv[u].y);
            }
        }
        for (int i0 = threadIdx.x; i0 < np * XW; i0 += U * FR_NT) {
            float2 xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * FR_NT, pp = i / XW;
                const int64_t xi = xbase + (pp * Pf + (i - pp * XW));
                xv[u] = (i < np * XW && xi >= g.x_lo && xi < g.x_hi) ? __ldg(g.x + ((uint64_t)xi & g.mask))
                                                                     : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * FR_NT;
                if (i >= np * XW) break;
                xs[i] = make_double2((double)xv[u].x, (double)xv[u].y);
            }
        }
        __syncthreads();
        const int p_lo = (int)(max(pa, c0) - c0), p_hi = (int)(min(pb, c0 + np) - c0);
        for (int pp = p_lo + pg; pp < p_hi; pp += FR_PG) {
            const double2 yd = ys[pp * FR_RB + ri];
#pragma unroll
            for (int k = 0; k < LPT; ++k) {
                const int t = lg + FR_LG * k;
                if (t < t_span) {
                    const double2 xd = xs[pp * XW + ri + t];
                    c[k][0] = fma(xd.x, yd.x, c[k][0]);
                    c[k][1] = fma(xd.y, yd.x, c[k][1]);
                    c[k][2] = fma(xd.x, yd.y, c[k][2]);
                    c[k][3] = fma(xd.y, yd.y, c[k][3]);
                }
            }
        }
        __syncthreads();
    }
    // period groups 1.. hand their partials to group 0 (staging reused)
    double2* red = fr_smem_buf;  // [FR_PG - 1][LPT][2][FR_RB * FR_LG]
    const int cell = threadIdx.x % (FR_RB * FR_LG);
    if (pg > 0) {
#pragma unroll
        for (int k = 0; k < LPT; ++k) {
            red[(((pg - 1) * LPT + k) * 2 + 0) * (FR_RB * FR_LG) + cell] = make_double2(c[k][0], c[k][1]);
            red[(((pg - 1) * LPT + k) * 2 + 1) * (FR_RB * FR_LG) + cell] = make_double2(c[k][2], c[k][3]);
        }
    }
    __syncthreads();
    if (pg > 0 || r >= Pf) return;
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
        const int t = lg + FR_LG * k;
        if (t >= t_span) continue;
        double2 v[2] = {make_double2(c[k][0], c[k][1]), make_double2(c[k][2], c[k][3])};
        if constexpr (FR_PG > 1) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double2 q[FR_PG - 1];
#pragma unroll
                for (int u = 0; u < FR_PG - 1; ++u) q[u] = red[((u * LPT + k) * 2 + h) * (FR_RB * FR_LG) + cell];
                if constexpr (FR_PG == 4) {  // fixed order: (g0 + g1) + (g2 + g3)
                    v[h].x = (v[h].x + q[0].x) + (q[1].x + q[2].x);
                    v[h].y = (v[h].y + q[0].y) + (q[1].y + q[2].y);
                } else {
                    v[h].x += q[0].x;
                    v[h].y += q[0].y;
                }
            }
        }
        double2* d = reinterpret_cast<double2*>(S + (((size_t)g.slot * t_pad + t) * (size_t)Pf + (size_t)r) * 4);
        d[0] = v[0];
        d[1] = v[1];
    }
}

template <int LW>
void run_fold(const FoldLaunch& L, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1, const FoldInline* inl,
              cudaEvent_t before_reduce) {
    using G = Geo<LW>;
    if (ev0) record_event(ev0, st);
    dim3 rg((G::TB * G::RB + 255) / 256, L.n_groups);
    if (inl) {
        fold_kernel<LW, true><<<L.n_tiles, NT, G::SMEM, st>>>(L, *inl);
        if (ev1) record_event(ev1, st);
        if (before_reduce) cudaStreamWaitEvent(st, before_reduce, 0);
        fold_reduce_kernel<true><<<rg, 256, 0, st>>>(L, G::TB, G::RB, *inl);
    } else {
        fold_kernel<LW, false><<<L.n_tiles, NT, G::SMEM, st>>>(L, NoInline{});
        if (ev1) record_event(ev1, st);
        if (before_reduce) cudaStreamWaitEvent(st, before_reduce, 0);
        fold_reduce_kernel<false><<<rg, 256, 0, st>>>(L, G::TB, G::RB, NoInline{});
    }
}

}  // namespace

void launch_fold_small(const FoldSeg* segs_dev, int n_slots, int Pf, int lag_lo, int t_span, int t_pad, double* S,
                       cudaStream_t st, const int64_t* shift) {
    if (n_slots <= 0 || t_span <= 0) return;
    prepare_fold_kernels();
    static const bool no_frame = std::getenv("CYC_NO_FRAME_FOLD") != nullptr;  // A/B knob
    if (!no_frame && Pf % FR_RB == 0 && t_span <= 4 * FR_LG) {
        const dim3 grid((unsigned)(Pf / FR_RB), (unsigned)n_slots);
        if (t_span <= FR_LG)
            fold_frame_kernel<1><<<grid, fr_nt<1>(), fr_smem<1>(), st>>>(segs_dev, Pf, lag_lo, t_span, t_pad, S, shift);
        else if (t_span <= 2 * FR_LG)
            fold_frame_kernel<2><<<grid, fr_nt<2>(), fr_smem<2>(), st>>>(segs_dev, Pf, lag_lo, t_span, t_pad, S, shift);
        else
            fold_frame_kernel<4><<<grid, fr_nt<4>(), fr_smem<4>(), st>>>(segs_dev, Pf, lag_lo, t_span, t_pad, S, shift);
        return;
    }
    fold_small_kernel<<<dim3((unsigned)((Pf + 127) / 128), (unsigned)t_span, (unsigned)n_slots), 128, 0, st>>>(
        segs_dev, Pf, lag_lo, t_pad, S, shift);
}

void launch_fold(const FoldLaunch& L, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1, const FoldInline* inl,
                 cudaEvent_t before_reduce) {
    if (L.n_tiles == 0) return;
    prepare_fold_kernels();
    switch (L.lw) {
        case 2: run_fold<2>(L, st, ev0, ev1, inl, before_reduce); break;
        case 4: run_fold<4>(L, st, ev0, ev1, inl, before_reduce); break;
        default: run_fold<8>(L, st, ev0, ev1, inl, before_reduce); break;
    }
}

}  // namespace cyc

namespace cyc {
// Set the dynamic-shared-memory attributes outside any stream capture.
void prepare_fold_kernels() {
    static std::atomic<uint64_t> done{0};
    if (!first_on_device(done)) return;
    cudaFuncSetAttribute(fold_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<2>::SMEM);
    cudaFuncSetAttribute(fold_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<4>::SMEM);
    cudaFuncSetAttribute(fold_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<8>::SMEM);
    cudaFuncSetAttribute(fold_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<2>::SMEM);
    cudaFuncSetAttribute(fold_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<4>::SMEM);
    cudaFuncSetAttribute(fold_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<8>::SMEM);
    cudaFuncSetAttribute(fold_frame_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, fr_smem<1>());
    cudaFuncSetAttribute(fold_frame_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fr_smem<2>());
    cudaFuncSetAttribute(fold_frame_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, fr_smem<4>());

}
}  // namespace cyc

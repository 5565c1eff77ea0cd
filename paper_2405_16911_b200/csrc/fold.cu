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

template <int LW>
__device__ __forceinline__ void load_period(Regs& r, const float4* per, int kap, int rho) {
    using G = Geo<LW>;
#pragma unroll
    for (int j = 0; j < 6; ++j) r.x[j] = per[(j & 1) * G::XC + kap + (j >> 1)];
    r.y[0] = per[2 * G::XC + rho];
    r.y[1] = per[2 * G::XC + G::YC + rho];
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

template <int LW>
__global__ void __launch_bounds__(NT, 1) fold_kernel(FoldLaunch L) {
    using G = Geo<LW>;
    extern __shared__ __align__(16) float4 smem4[];
    // Launch descriptors may live in mapped host memory: copy them to shared
    // memory once, so re-reads under register pressure never cross PCIe.
    __shared__ FoldTile s_tile;
    __shared__ FoldSeg s_seg;
    if (threadIdx.x == 0) s_tile = L.tiles[blockIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) s_seg = L.segs[s_tile.seg];
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

    auto load_stage = [&](int s) {
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const uint32_t dst0 = sbase + (uint32_t)((s % NSTAGE) * G::STAGE) * 16u;
        const int64_t pend = pbeg + G::PS;
        // stage-uniform fast path: every window of the stage inside the valid ranges
        const bool fast = vec && pend <= tile.p1 && pbeg * Pf + xoff >= seg.x_lo &&
                          (pend - 1) * Pf + xoff + G::XW <= seg.x_hi && pbeg * Pf + res0 >= seg.n_start &&
                          (pend - 1) * Pf + res0 + G::RB <= seg.n_end && res0 + G::RB <= Pf;
        int q = q_first, e = e_first;
        if (fast) {
#pragma unroll 2
            for (int k = 0; k < G::EPT; ++k) {
                if (q < G::PS) {
                    const bool isx = e < G::NX;
                    const int ee = isx ? e : e - G::NX;
                    const int b = ee & 1, c = ee >> 1;
                    const int off = q * G::PER + (isx ? b * G::XC + c : 2 * G::XC + b * G::YC + c);
                    const int64_t n = (pbeg + q) * Pf + (isx ? xoff : res0) + (4 * c + 2 * b);
                    cp_async16(dst0 + (uint32_t)off * 16u, (isx ? seg.x : seg.y) + ((uint64_t)n & mask), 16);
                }
                q += DQ;
                e += DE;
                if (e >= G::EPP) {
                    e -= G::EPP;
                    ++q;
                }
            }
            return;
        }
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
    Regs ra, rb;
    for (int s = 0; s < nstages; ++s) {
        cp_async_wait<NSTAGE - 2>();
        __syncthreads();
        if (s + NSTAGE - 1 < nstages) load_stage(s + NSTAGE - 1);
        cp_async_commit();

        const float4* st = smem4 + (s % NSTAGE) * G::STAGE;
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const int nq = min(G::PS, nper - s * G::PS);
        load_period<LW>(ra, st, kap, rho);
        int q = 0;
        for (; q + 1 < nq; q += 2) {
#ifndef CYC_DIAG_NOLDS  // diagnostic build only: FFMA2 stream without the per-period smem loads
            load_period<LW>(rb, st + (q + 1) * G::PER, kap, rho);
#else
            if (q == 0) load_period<LW>(rb, st + (q + 1) * G::PER, kap, rho);
#endif
            if (weighted) weight_period(ra, seg, (pbeg + q) * Pf + res0 + 4 * rho);
            mac_period(lo, hi, ra);
#ifndef CYC_DIAG_NOLDS
            if (q + 2 < nq) load_period<LW>(ra, st + (q + 2) * G::PER, kap, rho);
#endif
            if (weighted) weight_period(rb, seg, (pbeg + q + 1) * Pf + res0 + 4 * rho);
            mac_period(lo, hi, rb);
        }
        if (q < nq) {
            if (weighted) weight_period(ra, seg, (pbeg + q) * Pf + res0 + 4 * rho);
            mac_period(lo, hi, ra);
        }
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
__global__ void fold_reduce_kernel(FoldLaunch L, int TB, int RB) {
    if (L.gate && *L.gate != ~0ull) return;
    __shared__ FoldGroup s_g;
    __shared__ int s_slot;
    if (threadIdx.x == 0) {
        s_g = L.groups[blockIdx.y];
        s_slot = L.segs[s_g.seg].slot;
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

template <int LW>
void run_fold(const FoldLaunch& L, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
    using G = Geo<LW>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(fold_kernel<LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        attr_set = true;
    }
    if (ev0) cudaEventRecord(ev0, st);
    fold_kernel<LW><<<L.n_tiles, NT, G::SMEM, st>>>(L);
    if (ev1) cudaEventRecord(ev1, st);
    dim3 rg((G::TB * G::RB + 255) / 256, L.n_groups);
    fold_reduce_kernel<<<rg, 256, 0, st>>>(L, G::TB, G::RB);
}

}  // namespace

void launch_fold(const FoldLaunch& L, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
    if (L.n_tiles == 0) return;
    switch (L.lw) {
        case 2: run_fold<2>(L, st, ev0, ev1); break;
        case 4: run_fold<4>(L, st, ev0, ev1); break;
        default: run_fold<8>(L, st, ev0, ev1); break;
    }
}

}  // namespace cyc

namespace cyc {
// Set the dynamic-shared-memory attributes outside any stream capture.
void prepare_fold_kernels() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(fold_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<2>::SMEM);
    cudaFuncSetAttribute(fold_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<4>::SMEM);
    cudaFuncSetAttribute(fold_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<8>::SMEM);
    done = true;
}
}  // namespace cyc

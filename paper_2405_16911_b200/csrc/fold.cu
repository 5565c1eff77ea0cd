// fold.cu -- the hot kernel: lag products folded over residues n mod Pf.
//
// For every requested lag tau and residue r it accumulates the four real
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
// CTA = 8 warps.  A thread owns R=4 consecutive residues x U=8 consecutive
// lags (128 fp32 accumulators, issued as packed FFMA2).  Sample windows are
// staged per fold period by cp.async into shared memory in a "phase-split by
// 4" layout E[s & 3][s >> 2] so the sliding register windows of neighbouring
// lanes hit consecutive 8-byte words (conflict-free), and y reads are
// broadcast across the lag lanes of a warp.  Per period a thread issues 15
// LDS.64 for 64 FFMA2 (128 FMAs).  Partial sums leave the CTA in fp32 and are
// reduced in fp64 in a fixed order (deterministic; SURVEY §7 "Hard parts").
#include "kernels.cuh"

namespace cyc {
namespace {

constexpr int NW = 8;
constexpr int NT = NW * 32;
constexpr int R = 4;
constexpr int U = 8;
constexpr int XV = R + U - 1;
constexpr int NSTAGE = 3;

constexpr int pad4mod16(int c) { return c + ((4 - c % 16) + 16) % 16; }

template <int LW>
struct Geo {
    static constexpr int RL = 32 / LW;       // residue lanes per warp
    static constexpr int TB = 8 * LW;        // lags per CTA
    static constexpr int RB = NW * RL * R;   // residues per CTA (= 1024 / LW)
    static constexpr int XW = RB + TB;       // x samples staged per period
    static constexpr int XCP = pad4mod16(XW / 4);
    static constexpr int YCP = pad4mod16(RB / 4);
    static constexpr int PER = 4 * XCP + 4 * YCP;  // float2 per period
    static constexpr int PS = LW == 2 ? 4 : 8;     // periods per pipeline stage
    static constexpr int STAGE = PS * PER;
    static constexpr int SMEM = NSTAGE * STAGE * 8;
};

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

// acc += a * (b, b)  -- packed fp32x2 FMA (SASS FFMA2)
__device__ __forceinline__ void ffma2_bcast(float2& acc, float2 a, float b) {
    F2U A, B, C;
    A.f = a;
    B.f = make_float2(b, b);
    C.f = acc;
    asm("fma.rn.f32x2 %0, %1, %2, %0;\n" : "+l"(C.u) : "l"(A.u), "l"(B.u));
    acc = C.f;
}

template <int LW>
__global__ void __launch_bounds__(NT, 1) fold_kernel(FoldLaunch L) {
    using G = Geo<LW>;
    extern __shared__ __align__(16) float2 smem[];
    const FoldTile tile = L.tiles[blockIdx.x];
    const FoldSeg seg = L.segs[tile.seg];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int rho = warp * G::RL + (lane % G::RL);  // residue group: residues 4*rho .. 4*rho+3
    const int lam = lane / G::RL;                   // lag group: lags 8*lam .. 8*lam+7

    const int64_t Pf = L.Pf;
    const int64_t res0 = (int64_t)tile.rb * G::RB;
    const int64_t xoff = res0 + L.lag_lo + (int64_t)tile.lb * G::TB;
    const int64_t nper = tile.p1 - tile.p0;
    const int nstages = (int)((nper + G::PS - 1) / G::PS);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const uint64_t mask = seg.mask;

    auto load_stage = [&](int s) {
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const uint32_t dst0 = sbase + (uint32_t)((s % NSTAGE) * G::STAGE) * 8u;
        constexpr int EPP = G::XW + G::RB;  // elements per period
        for (int e = tid; e < G::PS * EPP; e += NT) {
            const int q = e / EPP;
            const int sidx = e - q * EPP;
            const int64_t p = pbeg + q;
            uint32_t dst = dst0 + (uint32_t)(q * G::PER) * 8u;
            const float2* src = seg.x;
            int bytes = 0;
            if (sidx < G::XW) {
                const int64_t n = p * Pf + xoff + sidx;
                dst += (uint32_t)((sidx & 3) * G::XCP + (sidx >> 2)) * 8u;
                if (p < tile.p1 && n >= seg.x_lo && n < seg.x_hi) {
                    src = seg.x + ((uint64_t)n & mask);
                    bytes = 8;
                }
            } else {
                const int sy = sidx - G::XW;
                const int64_t n = p * Pf + res0 + sy;
                dst += (uint32_t)(4 * G::XCP + (sy & 3) * G::YCP + (sy >> 2)) * 8u;
                if (p < tile.p1 && n >= seg.n_start && n < seg.n_end && res0 + sy < Pf) {
                    src = seg.y + ((uint64_t)n & mask);
                    bytes = 8;
                }
            }
            cp_async8(dst, src, bytes);
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

        const float2* st = smem + (s % NSTAGE) * G::STAGE;
        const int64_t pbeg = tile.p0 + (int64_t)s * G::PS;
        const int nq = (int)min((int64_t)G::PS, tile.p1 - pbeg);
        for (int q = 0; q < nq; ++q) {
            const float2* Ex = st + q * G::PER;
            const float2* Ey = Ex + 4 * G::XCP;
            float2 xv[XV];
#pragma unroll
            for (int i = 0; i < XV; ++i) xv[i] = Ex[(i & 3) * G::XCP + rho + 2 * lam + (i >> 2)];
            float2 yv[R];
#pragma unroll
            for (int a = 0; a < R; ++a) yv[a] = Ey[a * G::YCP + rho];
            if (weighted) {
                const int64_t nb = (pbeg + q) * Pf + res0 + 4 * rho;
#pragma unroll
                for (int a = 0; a < R; ++a) {
                    const float w = seg.w_scale * exp2f((float)(seg.w_ref - (nb + a)) * seg.w_log2);
                    yv[a].x *= w;
                    yv[a].y *= w;
                }
            }
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    ffma2_bcast(lo[a][u], xv[a + u], yv[a].x);
                    ffma2_bcast(hi[a][u], xv[a + u], yv[a].y);
                }
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
    const FoldGroup g = L.groups[blockIdx.y];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= TB * RB) return;
    const int lag = e / RB, res = e - lag * RB;
    const int64_t rg = (int64_t)g.rb * RB + res;
    const int tg = g.lb * TB + lag;
    if (rg >= L.Pf || tg >= L.t_pad) return;
    const float4* part = reinterpret_cast<const float4*>(L.partials);
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int t = g.t0; t < g.t1; ++t) {
        const float4 v = part[(size_t)t * TB * RB + e];
        s0 += v.x;
        s1 += v.y;
        s2 += v.z;
        s3 += v.w;
    }
    const int slot = L.segs[g.seg].slot;
    double* d = L.S + (((size_t)slot * L.t_pad + tg) * (size_t)L.Pf + (size_t)rg) * 4;
    d[0] += s0;
    d[1] += s1;
    d[2] += s2;
    d[3] += s3;
}

template <int LW>
void run_fold(const FoldLaunch& L, cudaStream_t st) {
    using G = Geo<LW>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(fold_kernel<LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        attr_set = true;
    }
    fold_kernel<LW><<<L.n_tiles, NT, G::SMEM, st>>>(L);
    dim3 rg((G::TB * G::RB + 255) / 256, L.n_groups);
    fold_reduce_kernel<<<rg, 256, 0, st>>>(L, G::TB, G::RB);
}

}  // namespace

void launch_fold(const FoldLaunch& L, cudaStream_t st) {
    if (L.n_tiles == 0) return;
    switch (L.lw) {
        case 2: run_fold<2>(L, st); break;
        case 4: run_fold<4>(L, st); break;
        default: run_fold<8>(L, st); break;
    }
}

}  // namespace cyc

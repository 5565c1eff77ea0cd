// fold_tc.cu -- the residue fold on the 5th-generation tensor cores (sm_100a).
//
// Same contraction as fold.cu (four real correlations per (lag, residue),
// summed over fold periods), rewritten as a banded Gram product:
//     D[m][n] = sum_p A[m][p] * B[n][p]
//     A[2r+a][p] = {yr, yi}[p*Pf + r0 + r]            (M = 128: 64 residues)
//     B[2i+b][p] = {xr, xi}[p*Pf + r0 + d + i]        (N = 256: 128-sample window)
// with d = lag_lo + 64*lb, so lag tau = d + i - r and the useful band is
// i - r in [0, 64): D[2r+a][2(r+t)+b] is the correlation c_{2a+b} of residue r
// at lag d + t (c0 = xr*yr, c1 = xi*yr, c2 = xr*yi, c3 = xi*yi).
// A CTA covers 128 residues with two such products (TMEM columns 0..255 and
// 256..511) over one staged 192-sample window, so each x sample is read 1.5x
// (not 2x) from L2.
//
// Precision: each fp32 sample is split into bf16 hi + lo (x = hi + lo + O(2^-17 x))
// and D accumulates hi*hi + hi*lo + lo*hi with kind::f16 MMAs (fp32 TMEM
// accumulator): relative error ~1e-5, inside the north-star 1e-4 (measured:
// tools/exp/tc_probe2.cu).
//
// Two kernels (one tile = one residue block x lag block x period range):
//   fold_tc_kernel (fused): warp 0 stages raw fp32 windows (2-D TMA boxes, or
//     per-period bulk copies from a ring), warps 2..13 convert them to bf16
//     hi/lo planes in the UMMA MN-major 128B-swizzle layout, warp 1 issues
//     3 tcgen05.mma per 16 periods and tcgen05.commit frees the stage; the
//     converters also drain the TMEM accumulators into the tile's partials.
//   fold_tcp_kernel (planes): the split is done once per sample beforehand
//     (split_planes_kernel); TMA stages the bf16 planes straight into the
//     operand layout, so shared memory carries only TMA writes and MMA reads;
//     dedicated epilogue warps keep the drained sums in registers.
// The tile's partials go through a fixed-order fp64 reduce (fold_tc_reduce_kernel).
#include <cuda_bf16.h>

#include <climits>
#include <cstring>
#include <type_traits>

#include "kernels.cuh"

namespace cyc {
namespace {

constexpr int TKB = 16;                 // periods per stage (= MMA K for bf16)
constexpr int TRB = 128;                // residues per CTA (two 64-residue halves)
constexpr int XF = 2 * (TRB + 64);      // floats per x window: 192 samples
constexpr int YF = 2 * TRB;             // floats per y window: 128 samples
constexpr int XRAW = TKB * XF * 4;      // 24 KB (12 TMA boxes of 32 floats x 16 rows)
constexpr int YRAW = TKB * YF * 4;      // 16 KB
constexpr int ATOM = TKB * 128;         // one MN atom column of a plane: 64 bf16 x 16 rows
constexpr int XPLANE = TKB * XF * 2;    // 12 KB: 6 atoms
constexpr int YPLANE = TKB * YF * 2;    // 8 KB: 4 atoms
#ifndef TC_TNC
#define TC_TNC 12
#endif
#ifndef TC_EXPERIMENT
#define TC_EXPERIMENT 0
#endif
#if TC_EXPERIMENT != 0 && !defined(TC_DIAG_BUILD)
#error "TC_EXPERIMENT builds give wrong results: build them with CYC_NVCC_EXTRA (separate _diag/ library)"
#endif
#ifndef TC_NR_SELF
#define TC_NR_SELF 5
#endif
#ifndef TC_NP_SELF
#define TC_NP_SELF 4
#endif
// Warp roles: 0 producer (TMA / bulk copies), 1 MMA issuer, 2 .. TNC+1
// converters (which also drain TMEM between chunks and at the end).  The stage
// interval is bound by shared-memory bandwidth (TMA writes + converter
// loads/stores + 72 KB of MMA operand reads per stage, ncu: l1tex data-pipe
// wavefronts), and many thin converter warps hide the per-warp latency chain
// best (round-2 sweep: 4 or 8 fat warps with precomputed offsets were 10-25%
// slower).
constexpr int TNC = TC_TNC;
static_assert(TNC % 4 == 0, "converter warps cover every TMEM lane quarter");
constexpr int TNT = 64 + 32 * TNC;
// TMEM accumulation chunks (L.tc_drain stages): the tensor core adds each
// MMA's products into the fp32 accumulator with a truncating alignment, a bias
// of ~7e-8 of the accumulated value per stage (measured: 1.26e-5 relative on
// the C5 lag-0 cell over 2048 periods, against the 1e-5 cell tolerance).
// After each chunk the accumulator is added into the tile's sums (IEEE round
// to nearest) and the next MMA restarts it, which bounds the bias by the chunk
// length whatever the tile length.
// Two rings: raw fp32 stages (producer -> converters, freed after conversion)
// and bf16 plane stages (converters -> MMA, freed by tcgen05.commit).
template <bool SELF>
struct TcGeo {
    static constexpr int RAW = SELF ? XRAW : XRAW + YRAW;
    static constexpr int PLANE = SELF ? 2 * XPLANE : 2 * XPLANE + 2 * YPLANE;
    static constexpr int NR = SELF ? TC_NR_SELF : 3;
    static constexpr int NP = SELF ? TC_NP_SELF : 2;
    static constexpr int SMEM = NR * RAW + NP * PLANE + 1024;
    static_assert(SMEM <= 227 * 1024, "shared memory per CTA");
    // converter units (8 floats of one period row) per stage and per thread
    static constexpr int XU = (XF / 32) * 64, YU = SELF ? 0 : (YF / 32) * 64;
    static constexpr int NX = (XU + 32 * TNC - 1) / (32 * TNC), NYU = (YU + 32 * TNC - 1) / (32 * TNC);
    static constexpr int NU = NX + NYU;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int c1, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(dst), "l"((uint64_t)map), "r"(su32(bar)), "r"(0), "r"(c1), "r"(0), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(dst), "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1) : "memory");
}
// UMMA smem descriptor, 128B swizzle: lbo = MN-atom stride, sbo = 8-row K-group stride
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
// instruction descriptor: D f32, A/B bf16, both MN-major, M = 128, N = 256
constexpr uint32_t TC_IDESC =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t TC_IDESC_N128 =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// Unit u of a raw stage region (boxes of 32 floats x 16 rows): box a = u / 64;
// within the box a warp takes one 8-row group and each quarter-warp the row
// pair (k1, k1 ^ 5), 8-float groups m = 0..3 of both rows.  With the TMA 128B
// swizzle (chunk c of row k at c ^ (k % 8)) the raw reads, (2m | 2m+1) ^ k,
// and the plane writes, (4(a%2) + m) ^ k, of a quarter-warp then land on 8
// distinct 16-byte bank groups: k1 ^ k2 = 5 has bits 0 and 2 set.
// swz == false: rows are linear (1-D bulk copies, row pitch `pitch`).
// Offsets are relative to the raw stage base (constant across stages).
struct UnitPos {
    uint32_t ra, rb;  // offsets of the unit's two 16-byte raw chunks
    int a, m, k;      // box, 8-float group, row (period within the stage)
};
__device__ __forceinline__ UnitPos unit_pos(int u, bool swz, uint32_t pitch) {
    UnitPos q;
    const int w = u & 63, l = w & 31, qd = l >> 3, pos = l & 7;
    q.a = u >> 6;
    q.m = pos & 3;
    q.k = 8 * (w >> 5) + ((pos >> 2) ? (qd ^ 5) : qd);
    if (swz) {
        const uint32_t row = (uint32_t)(q.a * (TKB * 128) + q.k * 128);
        q.ra = row + ((uint32_t)((2 * q.m) ^ (q.k & 7)) << 4);
        q.rb = row + ((uint32_t)((2 * q.m + 1) ^ (q.k & 7)) << 4);
    } else {
        q.ra = (uint32_t)q.k * pitch + (uint32_t)(q.a * 128 + q.m * 32);
        q.rb = q.ra + 16;
    }
    return q;
}
// Plane offset of 8-float group n8 of row k (MN-major SW128: atom n8/8, row k,
// 16-byte chunk (n8%8) ^ (k%8)).
__device__ __forceinline__ uint32_t plane_off(int n8, int k) {
    return (uint32_t)((n8 >> 3) * (TKB * 128) + k * 128 + (((n8 & 7) ^ (k & 7)) << 4));
}
// 8 fp32 (a, b) -> one 16-byte chunk of the hi plane at `hi` and of the lo
// plane at `lo`: hi = bf16_rn(x), lo = bf16_rn(x - hi) (x - hi exact in fp32;
// packed fp32x2 subtractions).  zero: store zeros (rows past the stage's data).
// check: also flag a possibly non-finite input -- an inf or NaN makes its lo
// part (x - hi) NaN, caught by one bf16x2 FMA with zero per pair (finite
// values give +-0).  A flag is only a hint (so is the lo = -inf of a finite
// value that rounds to a bf16 infinity): the caller re-checks the fp32 samples.
__device__ __forceinline__ bool split8(const float4& a, const float4& b, uint32_t hi, uint32_t lo, bool zero,
                                       bool check) {
    uint32_t h[4] = {0, 0, 0, 0}, l[4] = {0, 0, 0, 0};
    uint32_t acc = 0;
    if (!zero) {
        const float2 v[4] = {make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y),
                             make_float2(b.z, b.w)};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            h[e] = pack_bf16(v[e].x, v[e].y);
            const float2 nh = make_float2(-__uint_as_float(h[e] << 16), -__uint_as_float(h[e] & 0xffff0000u));
            const float2 d = __fadd2_rn(v[e], nh);
            l[e] = pack_bf16(d.x, d.y);
        }
        if (check) {
#pragma unroll
            for (int e = 0; e < 4; ++e) asm("fma.rn.bf16x2 %0, %1, %2, %0;" : "+r"(acc) : "r"(l[e]), "r"(0u));
        }
    }
#if TC_EXPERIMENT == 4  // diagnostics: conversion without the plane stores
    return ((h[0] ^ h[1] ^ h[2] ^ h[3] ^ l[0] ^ l[1] ^ l[2] ^ l[3]) == 0x12345678u) | ((acc & 0x7fff7fffu) != 0u);
#else
    sts128(hi, h[0], h[1], h[2], h[3]);
    sts128(lo, l[0], l[1], l[2], l[3]);
    return (acc & 0x7fff7fffu) != 0u;
#endif
}
// Exact re-check of a flagged unit: samples 16a + 4m + j of the window of
// period p + k, which starts at absolute sample (p + k) Pf + win0; atomicMin
// of the scan's key.
__device__ __noinline__ void check_unit_slow(const FoldLaunch& L, const UnitPos q, const float4 A, const float4 B,
                                             int64_t p, int64_t win0, int is_y, int slot) {
    const float v[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
    for (int j = 3; j >= 0; --j) {
        if (isfinite(v[2 * j]) && isfinite(v[2 * j + 1])) continue;
        const int64_t abs = (p + q.k) * L.Pf + win0 + 16 * q.a + 4 * q.m + j;
        const unsigned long long idx = (unsigned long long)(abs - L.chk_c0);
        atomicMin(L.chk_key, (2ull * idx + (unsigned long long)is_y) * (unsigned long long)L.chk_channels +
                                 (unsigned long long)slot);
    }
}

// -DTC_TRACE (diagnostics build): clock64 at the pipeline hand-offs of CTA 0,
// read back with cyc_debug_tc_trace (tools/tc_trace.py)
#ifdef TC_TRACE
__device__ unsigned long long g_tc_trace[8][128];
__device__ unsigned long long g_tc_warp[16][64][2];  // per converter warp: (full seen, conv arrive) per stage
#define TC_MARK(kind, it) \
    if (blockIdx.x == 0 && (it) < 128) g_tc_trace[kind][it] = clock64();
// (clock64, globaltimer) of CTA 0 and of the last CTA at kernel start (s=0) and end (s=1): the SM clock under load
#define TC_TIME(s)                                                                          \
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) {             \
        unsigned long long gt;                                                              \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                              \
        const int b = blockIdx.x == 0 ? 100 : 110;                                          \
        g_tc_trace[6][b + 2 * (s)] = clock64();                                             \
        g_tc_trace[6][b + 2 * (s) + 1] = gt;                                                \
    }
#else
#define TC_MARK(kind, it)
#define TC_TIME(s)
#endif

// Drain of the fused kernel (NE converter warps, NE/4 per TMEM lane quarter):
// add the 64-lag band of both accumulators into the tile's fp32 partials
// (first chunk: store; later chunks: L2 reductions).  Lane m = 2r + a of
// quarter q = warp % 4 holds D[m][*]; the band is columns [2r, 2r + 128):
// float2 (c_{2a}, c_{2a+1}) per lag t, the residue's float4 written by the
// even lane.  One thread's adds to a cell apply in program order, so the sums
// are reproducible bit for bit.
template <int NE>
__device__ __forceinline__ void tc_drain_band(uint32_t tmem, const FoldLaunch& L, bool first, bool zero, int e,
                                              int warp, int lane, int tmax) {
    const int q = warp & 3;
    const int m = 32 * q + lane;
    const int r = m >> 1, a = m & 1;
    float4* part = reinterpret_cast<float4*>(L.partials) + (size_t)blockIdx.x * 64 * TRB;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // a quarter's work: 2 accumulators x 5 column chunks [32cc, 32cc + 32),
    // cc = q .. q+4 (they cover the band), shared by the quarter's NE/4 warps;
    // lags t >= tmax (past the requested span, e.g. C4's 32 of 64) are skipped
    for (int item = e >> 2; item < 10; item += NE / 4) {
        const int h = item / 5, cc = q + item % 5;
        if (16 * (cc - q) - 15 >= tmax) continue;  // every lag of this column chunk is past the span
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(256 * h + 32 * cc);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (zero) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int t = 16 * cc + j - r;  // lag offset of column pair 2(16cc + j)
            const float o0 = __uint_as_float(v[2 * j]), o1 = __uint_as_float(v[2 * j + 1]);
            const float p0 = __shfl_xor_sync(0xffffffffu, o0, 1), p1 = __shfl_xor_sync(0xffffffffu, o1, 1);
            if (a != 0 || t < 0 || t >= tmax) continue;
            float4* dst = part + ((size_t)t * TRB + 64 * h + r);
            if (first) {
                *dst = make_float4(o0, o1, p0, p1);
            } else {
                // fire-and-forget fp32 adds in L2 (round to nearest)
                asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(o0), "f"(o1),
                             "f"(p0), "f"(p1)
                             : "memory");
            }
        }
    }
    // the TMEM reads complete before the MMA warp restarts the accumulator
    asm volatile("tcgen05.fence::before_thread_sync;");
}

// 32 consecutive TMEM columns of this warp's lanes, one load and one wait
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
    uint32_t u[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
          "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
          "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(u[k]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* v) {
    uint32_t u[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(u[k]);
}

// Dedicated epilogue warps of the planes kernel (NE = 16: four per TMEM lane
// quarter; or 8): the chunks' sums stay in registers -- fp32 adds, round to
// nearest -- and the band is stored once per tile.  The accumulator is the
// 384-column union of the tile's two lag blocks (columns 2i + b, window sample
// i in [0, 192)); lane m = 2r + a of quarter q (r = 16q + r') owns lags
// t' = i - r = 0..127 of residue r, component pair a: 8 items of 16 column
// pairs, item k = 1..7 the column chunk cc = q + k (t' = 16k + j - r'), item 0
// the chunks q (j >= r') and q + 8 (j < r') merged (t' = (j - r') mod 128).
// Warp w of the quarter's NE/4 warps holds items w, w + NE/4, ...; lag t' is
// stored as lag block t' / 64, offset t' % 64 (the reduce's layout).
template <int NE>
__device__ __forceinline__ void tc_epilogue_tile(uint32_t tmem, const FoldLaunch& L, int nst, int nchunks, int e,
                                                 int warp, int lane, uint64_t* chunk_done, uint64_t* drain_free,
                                                 int& gc, bool release_last, float4* part) {
    static_assert(NE == 8 || NE == 16, "two or four epilogue warps per lane quarter");
    constexpr int NI = 32 / NE, WQ = NE / 4;  // items per warp, warps per quarter
    const int q = warp & 3, w = e >> 2;
    const int m = 32 * q + lane;
    const int r = m >> 1, a = m & 1, rp = r - 16 * q;
    float acc[NI][32];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[k][j] = 0.f;  // x + 0 is exact: chunk 0 adds like the rest
    const int nc = nchunks;  // 0: an empty tile (zeros), no MMAs to wait for
    for (int c = 0; c < nc; ++c) {
        mbar_wait(chunk_done, (uint32_t)(gc++) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (nst > 0) {
#pragma unroll
            for (int k = 0; k < NI; ++k) {
                const int kind = w + WQ * k;
                const uint32_t base = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll
                for (int part2 = 0; part2 < (kind ? 1 : 2); ++part2) {
                    // merged item: chunk q for j >= r', chunk q + 8 for j < r'
                    const int cc = kind ? q + kind : q + 8 * part2;
                    float v[32];  // the chunk's 16 column pairs in one load
                    tmem_ld32(base + (uint32_t)(32 * cc), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const bool use = kind || ((j >= rp) == (part2 == 0));
                        if (use) {
                            acc[k][2 * j] += v[2 * j];
                            acc[k][2 * j + 1] += v[2 * j + 1];
                        }
                    }
                }
            }
        }
        // the TMEM reads complete before the MMA warp restarts the accumulator
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0 && (c + 1 < nc || release_last)) mbar_arrive(drain_free);
    }
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        const int kind = w + WQ * k;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float p0 = __shfl_xor_sync(0xffffffffu, acc[k][2 * j], 1);
            const float p1 = __shfl_xor_sync(0xffffffffu, acc[k][2 * j + 1], 1);
            if (a != 0) continue;
            const int t = kind ? 16 * kind + j - rp : (j - rp) & 127;
            part[(size_t)(t & 63) * TRB + 64 * (t >> 6) + r] = make_float4(acc[k][2 * j], acc[k][2 * j + 1], p0, p1);
        }
    }
}

template <bool SELF, class DESC>
__global__ void __launch_bounds__(TNT, 1) fold_tc_kernel(FoldLaunch L, const __grid_constant__ DESC D) {
    using G = TcGeo<SELF>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* raw_ring = smem;                       // NR x RAW
    uint8_t* plane_ring = smem + G::NR * G::RAW;    // NP x PLANE (1 KB aligned)
    __shared__ uint64_t full[G::NR], rawfree[G::NR], conv[G::NP], planefree[G::NP], chunk_done, drain_free;
    __shared__ uint32_t tmem_s;
    __shared__ FoldTile s_tile;
    __shared__ FoldSeg s_seg;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        s_tile = D.tiles[blockIdx.x];
        s_seg = D.segs[s_tile.seg];
        for (int s = 0; s < G::NR; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&rawfree[s], TNC);
        }
        for (int s = 0; s < G::NP; ++s) {
            mbar_init(&conv[s], TNC);
            mbar_init(&planefree[s], 1);
        }
        mbar_init(&chunk_done, 1);
        mbar_init(&drain_free, TNC);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // two 128 x 256 fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_s;
    if (threadIdx.x == 0) TC_MARK(7, 0);
    const FoldTile& tile = s_tile;
    const FoldSeg& seg = s_seg;
    const int64_t Pf = L.Pf;
    const int64_t r0 = (int64_t)tile.rb * TRB;
    const int64_t d = (int64_t)L.lag_lo + (int64_t)tile.lb * 64;
    const int ya = SELF ? (int)(-d) / 32 : 0;  // first x atom holding y (self tiles)
    const int nper = (int)(tile.p1 - tile.p0);
    const int nst = (nper + TKB - 1) / TKB;
    const int DRAIN = L.tc_drain > 0 ? L.tc_drain : (1 << 30);
    // chunk phases staggered over CTAs (stage it is in chunk (it + off) / DRAIN):
    // the CTAs' drains, which all add into L2, do not coincide
    const int off = L.tc_drain > 0 ? (int)(blockIdx.x % 4) * (DRAIN / 4) : 0;
    const int nchunks = nst > 0 ? (nst - 1 + off) / DRAIN + 1 : 0;
    const bool swz = seg.mask == ~0ull;  // TMA-staged (128B-swizzled boxes) vs bulk-copied rows

    if (warp == 0) {
        const uint64_t mask = seg.mask;
        if (mask == ~0ull) {
            // linear segment: 2-D TMA boxes (32 floats x 16 periods) per stage
            const CUtensorMap* xm = &D.xmap[tile.seg];
            const CUtensorMap* ym = &D.ymap[tile.seg];
            const int row0 = (int)(tile.p0 - D.p_base[tile.seg]);
            const int xcol = 2 * (int)(r0 + 64 * tile.lb);
            if (lane == 0) {
                for (int it = 0; it < nst; ++it) {
                    const int s = it % G::NR;
                    if (it >= G::NR) mbar_wait(&rawfree[s], ((it / G::NR) - 1) & 1);
                    TC_MARK(0, it);
                    const uint32_t st = su32(raw_ring + s * G::RAW);
                    mbar_expect_tx(&full[s], G::RAW);
#pragma unroll
                    for (int a = 0; a < XF / 32; ++a) tma_2d(st + a * ATOM, xm, xcol + 32 * a, row0 + it * TKB, &full[s]);
                    if (!SELF)
#pragma unroll
                        for (int a = 0; a < YF / 32; ++a)
                            tma_2d(st + XRAW + a * ATOM, ym, 2 * (int)r0 + 32 * a, row0 + it * TKB, &full[s]);
                }
            }
        } else {
            // ring segment: lane k < 16 copies period k's x window, lane 16 + k
            // its y window, split at the wrap
            const int k = lane & 15;
            for (int it = 0; it < nst; ++it) {
                const int s = it % G::NR;
                if (it >= G::NR) mbar_wait(&rawfree[s], ((it / G::NR) - 1) & 1);
                uint8_t* st = raw_ring + s * G::RAW;
                const int rows = min(TKB, nper - it * TKB);
                if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)rows * (SELF ? XF * 4 : (XF + YF) * 4));
                __syncwarp();
                const int64_t p = tile.p0 + (int64_t)it * TKB + k;
                if (k < rows && lane < 16) {
                    const uint64_t xs = (uint64_t)(p * Pf + r0 + d) & mask;
                    const uint32_t dx = su32(st + k * (XF * 4));
                    const uint64_t room = mask + 1 - xs;
                    if (room >= XF / 2) {
                        bulk_g2s(dx, seg.x + xs, XF * 4, &full[s]);
                    } else {
                        bulk_g2s(dx, seg.x + xs, (uint32_t)room * 8, &full[s]);
                        bulk_g2s(dx + (uint32_t)room * 8, seg.x, (uint32_t)(XF / 2 - room) * 8, &full[s]);
                    }
                } else if (!SELF && k < rows) {
                    const uint64_t ys = (uint64_t)(p * Pf + r0) & mask;
                    const uint32_t dy = su32(st + XRAW + k * (YF * 4));
                    const uint64_t yroom = mask + 1 - ys;
                    if (yroom >= YF / 2) {
                        bulk_g2s(dy, seg.y + ys, YF * 4, &full[s]);
                    } else {
                        bulk_g2s(dy, seg.y + ys, (uint32_t)yroom * 8, &full[s]);
                        bulk_g2s(dy + (uint32_t)yroom * 8, seg.y, (uint32_t)(YF / 2 - yroom) * 8, &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int j = off, k = 0;  // stage within the accumulation chunk, drains so far
            if (nst > 0) mbar_wait(&conv[0], 0u);
            for (int it = 0; it < nst; ++it, ++j) {
                const int s = it % G::NP;
                if (j == DRAIN) j = 0;
                // the chunk's first MMAs overwrite the accumulator: the
                // converters must have drained the previous chunk (drain k -> phase k)
                if (j == 0 && it > 0) mbar_wait(&drain_free, (uint32_t)(k++) & 1u);
                const uint32_t acc = (it > 0 && j != 0) ? 1u : 0u;
                TC_MARK(1, it);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t xh = su32(plane_ring + s * G::PLANE), xl = xh + XPLANE;
                const uint32_t yh0 = SELF ? xh + ya * ATOM : xl + XPLANE;
                const uint32_t yl0 = SELF ? xl + ya * ATOM : yh0 + YPLANE;
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // residues 64h..64h+63: y atoms 2h.., x atoms 2h..2h+3
                    const uint64_t dxh = sw128_desc(xh + 2 * h * ATOM, ATOM, 1024);
                    const uint64_t dxl = sw128_desc(xl + 2 * h * ATOM, ATOM, 1024);
                    const uint64_t dyh = sw128_desc(yh0 + 2 * h * ATOM, ATOM, 1024);
                    const uint64_t dyl = sw128_desc(yl0 + 2 * h * ATOM, ATOM, 1024);
                    const uint32_t dt = tmem + 256 * h;
#if TC_EXPERIMENT != 1  // diagnostics: 1 = no MMAs (pipeline and conversion only)
                    mma_bf16(dt, dyh, dxh, TC_IDESC, acc);
                    mma_bf16(dt, dyh, dxl, TC_IDESC, 1u);
                    mma_bf16(dt, dyl, dxh, TC_IDESC, 1u);
#endif
                }
                // the next stage's planes are checked while this stage's MMAs are
                // still queued; the commits follow (as in the planes kernel)
                if (it + 1 < nst) mbar_wait(&conv[(it + 1) % G::NP], ((it + 1) / G::NP) & 1);
                mma_commit(&planefree[s]);
                if (it == nst - 1) mma_commit(&chunk_done);  // the final drain's signal
                TC_MARK(2, it);
            }
            if (nst == 0) mbar_arrive(&chunk_done);  // no MMAs: the drain stores zeros
        }
    } else {
        // converters: a thread's units are ct + i * 32 TNC (x units, then y);
        // their raw / plane offsets are the same every stage
        const int ct = threadIdx.x - 64;
        const bool chk = L.chk_key != nullptr && tile.lb == 0;
        const int cb0 = SELF ? (int)(-d) / 16 : 0;
        const int chk_y = (seg.x != seg.y) ? 1 : 0;
        constexpr int NU = G::NU;
        UnitPos q[NU];
        uint32_t pho[NU], pdl[NU];
        bool on[NU];
        uint32_t ckm = 0;
#pragma unroll
        for (int i = 0; i < NU; ++i) {
            const bool isy = i >= G::NX;
            const int u = ct + (isy ? i - G::NX : i) * 32 * TNC;
            on[i] = u < (isy ? G::YU : G::XU);
            q[i] = unit_pos(on[i] ? u : 0, swz, isy ? YF * 4 : XF * 4);
            if (isy) {
                q[i].ra += XRAW;
                q[i].rb += XRAW;
            }
            pho[i] = (isy ? 2 * XPLANE : 0) + plane_off(4 * q[i].a + q[i].m, q[i].k);
            pdl[i] = isy ? YPLANE : XPLANE;
            if (chk && (isy || (q[i].a >= cb0 && q[i].a < cb0 + 8))) ckm |= 1u << i;
        }
        const uint32_t rbase = su32(raw_ring), pbase = su32(plane_ring);
        int rs = 0, ps = 0;
        uint32_t rph = 0, pph = 0;  // ring phases
        const int e = warp - 2;
        // Drain of the chunk ending at stage b: MMA(b) is complete once the
        // converters hold plane slot b % NP again (its tcgen05.commit), i.e.
        // at iteration b + NP; the MMA warp waits on drain_free before the next
        // chunk's first (overwriting) MMAs, while the converters have already
        // filled the plane ring ahead.
        const int tmax = min(64, L.t_pad - 64 * tile.lb);  // lags of this lag block inside the span
        auto drain_after = [&](int b) {
            tc_drain_band<TNC>(tmem, L, b + off < DRAIN, false, e, warp, lane, tmax);
            __syncwarp();
            if (lane == 0) mbar_arrive(&drain_free);
        };
        int next_end = L.tc_drain > 0 ? DRAIN - 1 - off : INT_MAX;  // next chunk-end stage
        for (int it = 0; it < nst; ++it) {
            mbar_wait(&full[rs], rph);
            if (warp == 2 && lane == 0) TC_MARK(3, it);
#ifdef TC_TRACE
            if (blockIdx.x == 0 && lane == 0 && it < 64 && warp < 16) g_tc_warp[warp][it][0] = clock64();
#endif
            if (it >= G::NP) {
                mbar_wait(&planefree[ps], pph ^ 1u);
                const int b = it - G::NP;
                if (b == next_end) {
                    if (b + 1 < nst) drain_after(b);
                    next_end += DRAIN;
                }
            }
            if (warp == 2 && lane == 0) TC_MARK(4, it);
            const uint32_t st = rbase + (uint32_t)(rs * G::RAW);
            const uint32_t pl = pbase + (uint32_t)(ps * G::PLANE);
            float4 va[NU], vb[NU];
#pragma unroll
            for (int i = 0; i < NU; ++i) {
                if (!on[i]) continue;
#if TC_EXPERIMENT == 5  // diagnostics: conversion and stores without the raw loads
                va[i] = make_float4(__int_as_float(q[i].ra), 1.f, 2.f, 3.f);
                vb[i] = make_float4(__int_as_float(q[i].rb), 1.f, 2.f, 3.f);
#else
                va[i] = lds128(st + q[i].ra);
                vb[i] = lds128(st + q[i].rb);
#endif
            }
            // the raw slot is free as soon as its values are in registers: the
            // producer's next TMA into it overlaps this stage's conversion
            __syncwarp();
            if (lane == 0) mbar_arrive(&rawfree[rs]);
            const int rows = min(TKB, nper - it * TKB);  // rows >= `rows` are zero-filled
            uint32_t flags = 0;
#pragma unroll
            for (int i = 0; i < NU; ++i) {
                if (!on[i] || TC_EXPERIMENT == 2) continue;  // diagnostics: 2 = no conversion
                if (split8(va[i], vb[i], pl + pho[i], pl + pho[i] + pdl[i], q[i].k >= rows, (ckm >> i) & 1u))
                    flags |= 1u << i;
            }
            if (flags) {  // a possibly non-finite sample: exact re-check (rare)
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    if (!(flags & (1u << i))) continue;
                    const bool isy = i >= G::NX;
                    check_unit_slow(L, q[i], va[i], vb[i], tile.p0 + (int64_t)it * TKB, isy ? r0 : r0 + d,
                                    isy ? chk_y : 0, seg.slot);
                }
            }
#if TC_EXPERIMENT != 3  // diagnostics: 3 = no proxy fence before the hand-off
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[ps]);
            if (warp == 2 && lane == 0) TC_MARK(5, it);
#ifdef TC_TRACE
            if (blockIdx.x == 0 && lane == 0 && it < 64 && warp < 16) g_tc_warp[warp][it][1] = clock64();
#endif
            if (++rs == G::NR) {
                rs = 0;
                rph ^= 1u;
            }
            if (++ps == G::NP) {
                ps = 0;
                pph ^= 1u;
            }
        }
        // chunk ends among the last NP stages (no converter iteration follows them)
        for (int it = nst; it < nst + G::NP; ++it) {
            const int b = it - G::NP;
            if (b >= 0 && b == next_end) {
                next_end += DRAIN;
                if (b + 1 < nst) {
                    mbar_wait(&planefree[ps], pph ^ 1u);
                    drain_after(b);
                }
            }
            if (++ps == G::NP) {
                ps = 0;
                pph ^= 1u;
            }
        }
        // final chunk
        mbar_wait(&chunk_done, 0);
        if (warp == 2 && lane == 0) TC_MARK(6, 0);
        tc_drain_band<TNC>(tmem, L, nchunks <= 1, nst == 0, e, warp, lane, tmax);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (threadIdx.x == 0) TC_MARK(7, 1);
}

// ---------------------------------------------------------------------------
// Planes path: the split is done once per sample (split_planes_kernel) and
// the fold stages bf16 planes with TMA straight into the operand layout.  One
// stage slot holds x hi/lo (6 atoms each) and, for tiles whose y window is
// not inside the x window, y hi/lo (4 atoms each); self and non-self tiles
// share one launch, so the lag blocks of a residue block run together and
// reuse the planes from L2.
// ---------------------------------------------------------------------------
#ifndef TC_TPE
#define TC_TPE 16
#endif

constexpr int TPE = TC_TPE;                        // epilogue warps of the planes kernel
constexpr int TPT = 64 + 32 * TPE;
#ifndef PL_RING_KB
#define PL_RING_KB 128
#endif
constexpr int PL_RING = PL_RING_KB * 1024;        // 32 KB stage slots (x hi/lo + 2 y atoms): 4 in flight
constexpr int PL_SMEM = PL_RING + 1024;
static_assert(PL_SMEM <= 227 * 1024, "shared memory per CTA");
// A stage's TMA lands ~3500 cycles after issue under load (tools/tcp_trace.py)
// and its slot frees only when its MMAs complete.  More windows in flight do
// not help: with 148 SMs streaming, the fold ran 909 / 543 / 487 / 497 / 505 /
// 523 us at 2 / 3 / 4 / 5 / 6 / 7 slots (C5) -- the memory system congests
// before the latency is covered, so 4 slots (128 KB) is the default.

// Per-tile geometry of the planes fold (every role derives it from the tile
// table): 64 residues [r0, r0 + 64) x lags d .. d + 127; the accumulator
// takes the 192-sample x window at r0 + d (6 atoms) against the y (A) operand.
struct TcpTile {
    int seg, nst, nchunks, off, ya, row0, xatom, yatom;
    bool self;
};
__device__ __forceinline__ TcpTile tcp_tile(const FoldLaunch& L, const TcPlDesc& D, int t, int DRAIN) {
    const FoldTile ft = D.tiles[t];
    const FoldSeg& sg = D.segs[ft.seg];
    TcpTile g;
    g.seg = ft.seg;
    const int64_t r0 = (int64_t)ft.rb * 64;
    const int64_t d = (int64_t)L.lag_lo + (int64_t)ft.lb * 128;
    // y inside the x window at an atom boundary: skip the y planes
    g.self = sg.x == sg.y && d <= 0 && -d <= 128 && (-d) % 32 == 0;
    g.ya = g.self ? (int)(-d) / 32 : 0;
    g.nst = (int)((ft.p1 - ft.p0) + TKB - 1) / TKB;
    g.off = L.tc_drain > 0 ? (t % 4) * (DRAIN / 4) : 0;  // staggered drains
    g.nchunks = g.nst > 0 ? (g.nst - 1 + g.off) / DRAIN + 1 : 0;
    g.row0 = (int)(ft.p0 - D.p_base[ft.seg]);
    g.xatom = (int)(r0 + d) / 32;
    g.yatom = (int)r0 / 32;
    return g;
}

// Persistent planes fold: one CTA per SM walks the tiles t = blockIdx.x,
// + gridDim.x, ... (range-major order, so the SMs work on one period range at
// a time and share the planes through L2).  The stage ring, the chunk barriers
// and the TMEM accumulator carry over from tile to tile: the producer loads the
// next tile's first stages while the last ones are multiplied, and the MMA
// warp starts the next tile as soon as the epilogue warps have read the
// accumulator out of TMEM -- the tile's partial stores, its final drain wait
// and the prologue (TMEM allocation, barrier set-up, first loads) no longer
// idle the tensor pipe between tiles (they cost ~12 % of a 128-stage C5 tile).
// Stage slots are uniform (x hi/lo + 2 y atoms, 32 KB); self tiles leave the
// y part unused.
template <class DESC>
__global__ void __launch_bounds__(TPT, 1) fold_tcp_kernel(FoldLaunch L, const __grid_constant__ DESC D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
#ifdef TC_ABL_SLOT24  // ablation (diagnostic builds): 24 KB slots -- non-self stages overrun the next slot
    constexpr uint32_t SLOT = 2 * XPLANE;
#else
    constexpr uint32_t SLOT = 2 * XPLANE + 2 * 2 * ATOM;  // 32 KB
#endif
    constexpr int NPL = PL_RING / (int)SLOT;               // stages in flight
    static_assert(NPL >= 2, "ring depth");
    __shared__ uint64_t full[NPL], planefree[NPL], chunk_done, drain_free;
    __shared__ uint32_t tmem_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NPL; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&planefree[s], 1);
        }
        mbar_init(&chunk_done, 1);
        mbar_init(&drain_free, TPE);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_s;
    TC_TIME(0);
    if (threadIdx.x == 0) TC_MARK(7, 0);
    const int DRAIN = L.tc_drain > 0 ? L.tc_drain : (1 << 30);
    const int nt = L.n_tiles;
    if (warp == 0) {
        if (lane == 0) {
            // one 4-D TMA per window: {64 bf16, 16 periods, hi/lo, atoms} lands
            // as [atom][hi, lo][16 rows][128 B] (one instruction instead of one
            // per 2 KB atom column: a single issuing thread spends ~100 cycles
            // per box, tools/exp/tma4d.cu: 844 -> 356 cycles per 24 KB stage)
            int s = 0, filled = 0;  // ring slot by counters (no run-time division in these loops:
            uint32_t ph = 0;        // tools/exp/tc_pipe.cu, 128 -> 174 cycles per MMA with one)
            for (int t = blockIdx.x; t < nt; t += gridDim.x) {
                const TcpTile g = tcp_tile(L, D, t, DRAIN);
                const CUtensorMap* xm = &D.xmap[g.seg];
                const CUtensorMap* ym = &D.ymap[g.seg];
                const bool first = t == (int)blockIdx.x;
                for (int it = 0; it < g.nst; ++it) {
                    if (filled >= NPL) mbar_wait(&planefree[s], ph ^ 1u);
                    if (first) TC_MARK(0, it);
                    const uint32_t st = su32(ring + s * SLOT);
                    const int row = g.row0 + it * TKB;
#ifdef TC_ABL_NO_TMA  // ablation (diagnostic builds): stages after the first ring reuse stale data
                    if (filled >= NPL) {
                        mbar_arrive(&full[s]);
                    } else
#endif
                    {
                        mbar_expect_tx(&full[s], g.self ? 2 * XPLANE : 2 * XPLANE + 2 * 2 * ATOM);
                        tma_4d(st, xm, row, g.xatom, &full[s]);
                        if (!g.self) tma_4d(st + 2 * XPLANE, ym, row, g.yatom, &full[s]);
                    }
                    ++filled;
                    if (++s == NPL) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int s = 0, k = 0;  // ring slot; drains so far (every chunk but the CTA's first waits for one)
            uint32_t ph = 0;
            bool started = false, waited_first = false;
            for (int t = blockIdx.x; t < nt; t += gridDim.x) {
                const TcpTile g = tcp_tile(L, D, t, DRAIN);
                const bool first = t == (int)blockIdx.x;
                if (g.nst == 0) continue;
                bool last_tile = true;  // no later tile of this CTA has stages
                for (int t2 = t + (int)gridDim.x; t2 < nt && last_tile; t2 += gridDim.x)
                    last_tile = tcp_tile(L, D, t2, DRAIN).nst == 0;
                if (!waited_first) {
                    mbar_wait(&full[0], 0u);
                    waited_first = true;
                }
                int j = g.off;
                for (int it = 0; it < g.nst; ++it, ++j) {
                    if (j == DRAIN) j = 0;
                    if (first) TC_MARK(3, it);
                    // a chunk's first MMAs overwrite the accumulator: the epilogue
                    // warps must have read the previous chunk out of TMEM
                    const bool chunk_start = it == 0 || j == 0;
                    if (chunk_start && started) mbar_wait(&drain_free, (uint32_t)(k++) & 1u);
                    started = true;
                    if (first) TC_MARK(1, it);
                    const uint32_t acc = chunk_start ? 0u : 1u;
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const int sn = s + 1 == NPL ? 0 : s + 1;
                    const uint32_t phn = s + 1 == NPL ? ph ^ 1u : ph;
                    const bool more = it + 1 < g.nst || !last_tile;  // another stage follows in this CTA
                    const bool chunk_end = j == DRAIN - 1 || it == g.nst - 1;
#ifdef TC_ABL_NO_MMA  // ablation (diagnostic builds): stages are released without MMAs
                    if (more) mbar_wait(&full[sn], phn);
                    mbar_arrive(&planefree[s]);
                    if (chunk_end) mbar_arrive(&chunk_done);
                    s = sn;
                    ph = phn;
                    continue;
#endif
                    // atom a of a window: hi at (2a) ATOM, lo at (2a + 1) ATOM -- the
                    // operands' MN-atom stride (LBO) is 2 ATOM
                    const uint32_t xb = su32(ring + s * SLOT);
                    const uint32_t yb = g.self ? xb + 2 * g.ya * ATOM : xb + 2 * XPLANE;
                    const uint64_t dyh = sw128_desc(yb, 2 * ATOM, 1024);
                    const uint64_t dyl = sw128_desc(yb + ATOM, 2 * ATOM, 1024);
                    // the 192-sample window once: atoms 0..3 (N = 256) into TMEM
                    // columns 0..255, atoms 4..5 (N = 128) into 256..383 -- the
                    // union of the two lag blocks' 128-sample windows (3/4 of the
                    // MMA work of two N = 256 products)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint64_t dxh = sw128_desc(xb + 8 * h * ATOM, 2 * ATOM, 1024);
                        const uint64_t dxl = sw128_desc(xb + (8 * h + 1) * ATOM, 2 * ATOM, 1024);
                        const uint32_t dt = tmem + 256 * h;
                        const uint32_t id = h ? TC_IDESC_N128 : TC_IDESC;
                        mma_bf16(dt, dyh, dxh, id, acc);
                        mma_bf16(dt, dyh, dxl, id, 1u);
                        mma_bf16(dt, dyl, dxh, id, 1u);
                    }
                    // the next stage's barrier is checked while this stage's last
                    // MMAs are still queued (the tensor pipe's queue is shallow: any
                    // gap between stages longer than its work is a bubble); the
                    // commits go after it
                    if (more) mbar_wait(&full[sn], phn);
                    mma_commit(&planefree[s]);
                    if (chunk_end) mma_commit(&chunk_done);
                    if (first) TC_MARK(2, it);
                    s = sn;
                    ph = phn;
                }
            }
        }
    } else {
        // epilogue warps: per tile, every chunk's accumulator is added into
        // registers (IEEE fp32) as soon as its MMAs completed; the MMA warp is
        // released (drain_free) before the tile's partials are stored
        const int e = warp - 2;
        int gc = 0;  // chunks drained so far (chunk_done phase)
        for (int t = blockIdx.x; t < nt; t += gridDim.x) {
            const TcpTile g = tcp_tile(L, D, t, DRAIN);
            const bool last_tile = t + (int)gridDim.x >= nt;
            tc_epilogue_tile<TPE>(tmem, L, g.nst, g.nchunks, e, warp, lane, &chunk_done, &drain_free, gc, !last_tile,
                                  reinterpret_cast<float4*>(L.partials) + (size_t)t * 64 * TRB);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    TC_TIME(1);
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// hi = bf16_rn(x), lo = bf16_rn(x - hi) per component (the converters'
// arithmetic, so planes and fused folds give the same products), packed
// (re, im) per sample; and the chunk's finite scan.  Each thread takes 4
// samples of one channel row (independent 8-byte loads in flight).
__global__ void __launch_bounds__(256) split_planes_kernel(const float2* __restrict__ x, int64_t n, int C,
                                                           int64_t pitch_in, uint32_t* __restrict__ hi,
                                                           uint32_t* __restrict__ lo, int64_t pitch_out,
                                                           int64_t out_off, unsigned long long* key) {
    const int64_t per_row = (n + 4 * 256 - 1) / (4 * 256);  // blocks per channel row
    const int ch = (int)(blockIdx.x / per_row);
    const int64_t b = blockIdx.x % per_row;
    if (ch >= C) return;
    const float2* xr = x + (size_t)ch * pitch_in;
    uint32_t* hr = hi + (size_t)ch * pitch_out + out_off;
    uint32_t* lr = lo + (size_t)ch * pitch_out + out_off;
    const int64_t i0 = b * 4 * 256 + threadIdx.x;
    float2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = i0 + 256 * k;
        v[k] = i < n ? __ldcs(xr + i) : make_float2(0.f, 0.f);
    }
    int64_t bad = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = i0 + 256 * k;
        if (i >= n) continue;
        const uint32_t h = pack_bf16(v[k].x, v[k].y);
        const float2 nh = make_float2(-__uint_as_float(h << 16), -__uint_as_float(h & 0xffff0000u));
        const float2 dd = __fadd2_rn(v[k], nh);
        hr[i] = h;
        lr[i] = pack_bf16(dd.x, dd.y);
        if (bad < 0 && !(isfinite(v[k].x) && isfinite(v[k].y))) bad = i;
    }
    if (bad >= 0) atomicMin(key, (2ull * (unsigned long long)bad) * (unsigned long long)C + (unsigned long long)ch);
}


// ---------------------------------------------------------------------------
// 2-CTA planes fold (cta_group::2).  A CTA pair takes 128 residues x 128 lags:
// M = 256 rows = the residues' real parts (CTA 0) and imaginary parts (CTA 1)
// of y; B = 256 window samples of ONE x component (re for accumulator 0, im
// for accumulator 1), CTA k holding window samples [128k, 128k + 128).  Per
// SM and stage the tensor core then reads 8 KB per MMA (its A rows and half
// of B) instead of 12 KB, which takes the SM's shared-memory port below the
// MMA time.  Accumulator b of CTA k holds c_{2k+b} (c0 = xr yr,
// c1 = xi yr, c2 = xr yi, c3 = xi yi) of residue r (TMEM lane) at window
// sample i (column); the band is i - r in [0, 128).
// ---------------------------------------------------------------------------
constexpr int P2E = 16;                      // epilogue warps per CTA
constexpr int P2T = 64 + 32 * P2E;           // + warp 0 producer, warp 1 MMA issuer (leader)
constexpr int P2X = 4 * 2 * ATOM;            // x stage: 2 atoms x 4 planes = 16 KB
constexpr int P2Y = 2 * 2 * ATOM;            // y stage: 2 atoms x (hi, lo) = 8 KB
constexpr int P2S = P2X + P2Y;               // 24 KB per stage
constexpr int P2N = 8;                       // stages in flight
constexpr int P2_SMEM = P2N * P2S + 1024;
static_assert(P2_SMEM <= 227 * 1024, "shared memory per CTA");
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of CTA 0's copy of a barrier
// D f32, A/B bf16, both MN-major, M = 256 (CTA pair), N = 256
constexpr uint32_t TC_IDESC2 =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((256u >> 3) << 17) | ((256u >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_4d_pair(uint32_t dst, const CUtensorMap* map, int c1, int c2, int c3,
                                            uint64_t* bar) {
    // completes on CTA 0's barrier (the MMA issuer's) whichever CTA issues it
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"((uint64_t)map), "r"(su32(bar) & PEER_MASK), "r"(0),
        "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void mma2_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(TC_IDESC2), "r"(acc));
}
__device__ __forceinline__ void mma2_commit_both(uint64_t* bar) {  // arrive on this barrier in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(su32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {  // arrive on CTA 0's copy
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(su32(bar) & PEER_MASK) : "memory");
}

template <class DESC>
__global__ void __launch_bounds__(P2T, 1) fold_tcp2_kernel(FoldLaunch L, const __grid_constant__ DESC D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[P2N], planefree[P2N], chunk_done, drain_free;
    __shared__ uint32_t tmem_s;
    __shared__ FoldTile s_tile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        s_tile = D.tiles[blockIdx.x >> 1];
        for (int s = 0; s < P2N; ++s) {
            mbar_init(&full[s], 1);       // CTA 0: the issuer's expect_tx; both CTAs' TMA bytes
            mbar_init(&planefree[s], 1);  // the MMA commit, multicast to both CTAs
        }
        mbar_init(&chunk_done, 1);
        mbar_init(&drain_free, 2 * P2E);  // CTA 0: both CTAs' epilogue warps
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // both CTAs, same warp: two 128 x 256 fp32 accumulators per CTA
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive or TMA
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_s;
    const FoldTile& tile = s_tile;
    const int64_t r0 = (int64_t)tile.rb * TRB;
    const int64_t d = (int64_t)L.lag_lo + (int64_t)tile.lb * 128;
    const int nper = (int)(tile.p1 - tile.p0);
    const int nst = (nper + TKB - 1) / TKB;
    const int DRAIN = L.tc_drain > 0 ? L.tc_drain : (1 << 30);
    const int off = L.tc_drain > 0 ? (int)((blockIdx.x >> 1) % 4) * (DRAIN / 4) : 0;
    const int nchunks = nst > 0 ? (nst - 1 + off) / DRAIN + 1 : 0;
    if (warp == 0) {
        if (lane == 0) {
            // this CTA's half of the x window (all four planes) and its y
            // component (re on CTA 0, im on CTA 1), hi and lo
            const CUtensorMap* xm = &D.xmap[tile.seg];
            const CUtensorMap* ym = &D.ymap[tile.seg];
            const int row0 = (int)(tile.p0 - D.p_base[tile.seg]);
            const int xatom = (int)((r0 + d) / 64) + 2 * (int)rank, yatom = (int)(r0 / 64);
            for (int it = 0; it < nst; ++it) {
                const int s = it % P2N;
                if (it >= P2N) mbar_wait(&planefree[s], ((it / P2N) - 1) & 1);
                const uint32_t st = su32(ring + s * P2S);
                const int row = row0 + it * TKB;
                if (rank == 0) mbar_expect_tx(&full[s], 2 * P2S);  // both CTAs' stages
                tma_4d_pair(st, xm, row, 0, xatom, &full[s]);
                tma_4d_pair(st + P2X, ym, row, 2 * (int)rank, yatom, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            int j = off, k = 0;
            for (int it = 0; it < nst; ++it, ++j) {
                const int s = it % P2N;
                if (j == DRAIN) j = 0;
                mbar_wait(&full[s], (it / P2N) & 1);
                if (j == 0 && it > 0) mbar_wait(&drain_free, (uint32_t)(k++) & 1u);
                const uint32_t acc = (it > 0 && j != 0) ? 1u : 0u;
                asm volatile("tcgen05.fence::after_thread_sync;");
                // x: [atom a][plane q][16 rows][128 B] at (4a + q) ATOM, q = re_hi, re_lo, im_hi, im_lo
                // y: [atom a][hi, lo][16 rows][128 B] at P2X + (2a + h) ATOM
                const uint32_t xb = su32(ring + s * P2S), yb = xb + P2X;
                const uint64_t dyh = sw128_desc(yb, 2 * ATOM, 1024);
                const uint64_t dyl = sw128_desc(yb + ATOM, 2 * ATOM, 1024);
#pragma unroll
                for (int b = 0; b < 2; ++b) {  // x component: accumulator b
                    const uint64_t dxh = sw128_desc(xb + (2 * b) * ATOM, 4 * ATOM, 1024);
                    const uint64_t dxl = sw128_desc(xb + (2 * b + 1) * ATOM, 4 * ATOM, 1024);
                    const uint32_t dt = tmem + 256 * b;
                    mma2_bf16(dt, dyh, dxh, acc);
                    mma2_bf16(dt, dyh, dxl, 1u);
                    mma2_bf16(dt, dyl, dxh, 1u);
                }
                mma2_commit_both(&planefree[s]);
                if (j == DRAIN - 1 || it == nst - 1) mma2_commit_both(&chunk_done);
            }
            if (nst == 0) {
                // no MMAs: release both CTAs' epilogues (zeros)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&chunk_done)) : "memory");
                asm volatile("{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 1;\n\t"
                             "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(su32(&chunk_done)) : "memory");
            }
        }
    } else {
        // epilogue: lane quarter q = warp % 4, residue r = 32 q + lane; items of
        // 32 columns: kind 0 = chunks q (j >= r') and q + 4 (j < r') merged
        // (t = (j - r') mod 128), kind k = 1..3 chunk q + k (t = 32 k + j - r');
        // warp w of the quarter holds kind w of both accumulators (the pair of
        // correlations one CTA owns at the same lag)
        const int e = warp - 2;
        const int q = warp & 3, w = e >> 2;
        const int r = 32 * q + lane, rp = lane;
        float acc[2][32];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) acc[b][jj] = 0.f;
        const int nc = nchunks > 0 ? nchunks : 1;
        for (int c = 0; c < nc; ++c) {
            mbar_wait(&chunk_done, (uint32_t)c & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (nst > 0) {
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(256 * b);
#pragma unroll
                    for (int jb = 0; jb < 32; jb += 16) {
#pragma unroll
                        for (int part2 = 0; part2 < 2; ++part2) {
                            if (w != 0 && part2 == 1) continue;
                            const int cc = w != 0 ? q + w : q + 4 * part2;
                            float v[16];
                            tmem_ld16(base + (uint32_t)(32 * cc + jb), v);
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) {
                                const bool use = w != 0 || ((jb + jj >= rp) == (part2 == 0));
                                if (use) acc[b][jb + jj] += v[jj];
                            }
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0 && c + 1 < nc) mbar_arrive_leader(&drain_free);
        }
        // cell (t, r) of the tile: float4 (c0, c1, c2, c3); this CTA writes its pair
        float2* part = reinterpret_cast<float2*>(L.partials) + (size_t)(blockIdx.x >> 1) * 128 * TRB * 2;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
            const int t = w != 0 ? 32 * w + jj - rp : (jj - rp) & 127;
            part[((size_t)t * TRB + r) * 2 + rank] = make_float2(acc[0][jj], acc[1][jj]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // the pair's MMAs, remote arrivals and TMEM reads are complete
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// component planes [re_hi, re_lo, im_hi, im_lo] (the converters' arithmetic)
// and the chunk's finite scan; 4 samples per thread
__global__ void __launch_bounds__(256) split_planes4_kernel(const float2* __restrict__ x, int64_t n, int C,
                                                            int64_t pitch_in, uint16_t* __restrict__ planes,
                                                            int64_t plane_elems, int64_t pitch_out, int64_t out_off,
                                                            unsigned long long* key) {
    const int64_t per_row = (n + 4 * 256 - 1) / (4 * 256);
    const int ch = (int)(blockIdx.x / per_row);
    const int64_t b = blockIdx.x % per_row;
    if (ch >= C) return;
    const float2* xr = x + (size_t)ch * pitch_in;
    uint16_t* p0 = planes + (size_t)ch * pitch_out + out_off;
    const int64_t i0 = b * 4 * 256 + threadIdx.x;
    float2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = i0 + 256 * k;
        v[k] = i < n ? __ldcs(xr + i) : make_float2(0.f, 0.f);
    }
    int64_t bad = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = i0 + 256 * k;
        if (i >= n) continue;
        const uint32_t h = pack_bf16(v[k].x, v[k].y);
        const float2 nh = make_float2(-__uint_as_float(h << 16), -__uint_as_float(h & 0xffff0000u));
        const float2 dd = __fadd2_rn(v[k], nh);
        const uint32_t l = pack_bf16(dd.x, dd.y);
        p0[i] = (uint16_t)(h & 0xffffu);                            // re hi
        p0[plane_elems + i] = (uint16_t)(l & 0xffffu);              // re lo
        p0[2 * plane_elems + i] = (uint16_t)(h >> 16);              // im hi
        p0[3 * plane_elems + i] = (uint16_t)(l >> 16);              // im lo
        if (bad < 0 && !(isfinite(v[k].x) && isfinite(v[k].y))) bad = i;
    }
    if (bad >= 0) atomicMin(key, (2ull * (unsigned long long)bad) * (unsigned long long)C + (unsigned long long)ch);
}

template <int MG>
struct TcRed {
    FoldGroup groups[MG];
    int slot[MG];  // accumulator slot of each group's segment
};

// The fp64 reduce of fold.cu for the tensor-core tile geometry.  One thread
// per partial cell sums the group's tiles t0, t0 + stride, ... in tile order
// (a fixed order: results are reproducible bit for bit), eight float4 loads in
// flight, and adds the sums into S with 16-byte accesses issued before the
// partial loads complete.
template <int MG>
__global__ void __launch_bounds__(256) fold_tc_reduce_kernel(FoldLaunch L, const __grid_constant__ TcRed<MG> R) {
    pdl_wait();  // the fold's partials (PDL launch: scheduled during the fold's tail)
    // a rejected chunk: the state is left as it was -- or, for an overwriting
    // reduce (the first writer of a freshly reset state), as the reset's zeros
    const bool rejected = L.gate && *L.gate != ~0ull;
    if (rejected && !L.overwrite) return;
    const FoldGroup g = R.groups[blockIdx.y];
    const int slot = R.slot[blockIdx.y];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // lag * TRB + residue (pairs: 2 x 64 residues)
    const int cells = L.tc_pairs == 2 ? 128 * TRB : 64 * TRB;  // partial cells per tile
    if (e >= cells) return;
    const int lag = e / TRB, res = e % TRB;
    // planes tiles: cell (t, 64 h + r) is residue 64 rb + r at lag block 2 lb + h;
    // 2-CTA tiles: cell (t, r) is residue 128 rb + r at lag 128 lb + t
    const int64_t rg = L.tc_pairs == 1 ? (int64_t)g.rb * 64 + (res & 63) : (int64_t)g.rb * TRB + res;
    const int tg = L.tc_pairs == 1 ? (2 * g.lb + (res >> 6)) * 64 + lag : g.lb * (L.tc_pairs == 2 ? 128 : 64) + lag;
    if (rg >= L.Pf || tg >= L.t_pad) return;
    double2* dst = reinterpret_cast<double2*>(L.S + (((size_t)slot * L.t_pad + tg) * (size_t)L.Pf + (size_t)rg) * 4);
    // overwrite: the first writer of a freshly reset state (planes path) -- no
    // clear pass and no read of the old zeros
    const double2 d0 = L.overwrite ? make_double2(0.0, 0.0) : dst[0], d1 = L.overwrite ? make_double2(0.0, 0.0) : dst[1];
    if (rejected) {
        dst[0] = d0;
        dst[1] = d1;
        return;
    }
    const float4* part = reinterpret_cast<const float4*>(L.partials) + e;
    // the group's tiles are t0, t0 + stride, ... < t1 (stride 1: contiguous;
    // the planes path launches range-major, stride = its group count)
    const int stride = g.pad > 0 ? g.pad : 1;
    const int nt = (g.t1 - g.t0 + stride - 1) / stride;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    // partial loads in flight per thread: 4 (C5: 8 -> 47.4 us, 4 -> 31.1, 2 -> 32.4, warm ncu;
    // more outstanding loads congest)
    constexpr int U = 4;
    for (int k0 = 0; k0 < nt; k0 += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u < nt) v[u] = __ldcs(part + (size_t)(g.t0 + (k0 + u) * stride) * cells);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u >= nt) break;
            s0 += v[u].x;
            s1 += v[u].y;
            s2 += v[u].z;
            s3 += v[u].w;
        }
    }
    dst[0] = make_double2(d0.x + s0, d0.y + s1);
    dst[1] = make_double2(d1.x + s2, d1.y + s3);
}

}  // namespace

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}
bool encode_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t row_bytes,
               bool bf16 = false) {
    EncodeTiledFn enc = encode_fn();
    if (!enc || ((uintptr_t)base & 15) || rows == 0 || (row_bytes & 15)) return false;
    const cuuint64_t gdim[2] = {cols, rows};
    const cuuint64_t gstr[1] = {row_bytes};
    // one 128-byte swizzle atom column: 32 floats or 64 bf16 x 16 rows
    const cuuint32_t box[2] = {bf16 ? 64u : 32u, (cuuint32_t)TKB}, es[2] = {1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
               const_cast<void*>(base), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// Tensor maps of a linear segment for periods [p_base, p_base + rows): rows
// step Pf samples but span the widest window (overlapping rows; TMA reads only
// the boxes, which lie inside the segment's valid x / y ranges).
bool encode_tc_maps(TcParams& D, int si, const FoldSeg& g, int64_t p_base, int64_t rows, int Pf, int lag_lo,
                    int nlb) {
    D.p_base[si] = p_base;
    const float* xb = reinterpret_cast<const float*>(g.x + (p_base * Pf + lag_lo));
    const float* yb = reinterpret_cast<const float*>(g.y + p_base * Pf);
    // widest x window: residues Pf-128.. at lag block nlb-1 -> floats up to 2 Pf + 128 nlb
    return encode_2d(&D.xmap[si], xb, 2ull * Pf + 128ull * nlb, (uint64_t)rows, 8ull * Pf) &&
           encode_2d(&D.ymap[si], yb, 2ull * Pf, (uint64_t)rows, 8ull * Pf);
}

// 4-D map over the planes: (64 bf16 of an atom, period rows, hi/lo plane,
// atoms of 32 samples); box {64, 16, 2, natoms}.
bool encode_planes_4d(CUtensorMap* m, const uint32_t* hi, uint64_t plane_bytes, int64_t rows, int Pf,
                      int64_t cols_samples, int natoms) {
    EncodeTiledFn enc = encode_fn();
    if (!enc || ((uintptr_t)hi & 15) || rows <= 0 || (plane_bytes & 15)) return false;
    const cuuint64_t gdim[4] = {64, (cuuint64_t)rows, 2, (cuuint64_t)((cols_samples + 31) / 32)};
    const cuuint64_t gstr[3] = {4ull * (uint64_t)Pf, plane_bytes, 128};
    const cuuint32_t box[4] = {64, (cuuint32_t)TKB, 2, (cuuint32_t)natoms}, es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint32_t*>(hi), gdim, gstr, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tcp_maps(TcPlDesc& D, int si, const uint32_t* hi, const uint32_t* lo, int64_t p_base, int64_t rows,
                     int Pf, int64_t cols_samples) {
    D.p_base[si] = p_base;
    if (lo < hi) return false;
    const uint64_t plane_bytes = (uint64_t)(lo - hi) * sizeof(uint32_t);
    return encode_planes_4d(&D.xmap[si], hi, plane_bytes, rows, Pf, cols_samples, XF / 64) &&
           encode_planes_4d(&D.ymap[si], hi, plane_bytes, rows, Pf, cols_samples, 2);
}

namespace {
using TcSmall = TcDesc<160, 16, 2>;  // one or two segments, one wave of tiles

template <class DESC, int MG>
void launch_tc(const FoldLaunch& L, const DESC& D, const TcRed<MG>& R, bool self, cudaStream_t st, cudaEvent_t ev0,
               cudaEvent_t ev1, cudaEvent_t before_reduce, cudaEvent_t fold_done) {
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(fold_tc_kernel<true, DESC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TcGeo<true>::SMEM);
        cudaFuncSetAttribute(fold_tc_kernel<false, DESC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TcGeo<false>::SMEM);
    }
    if (ev0) record_event(ev0, st);
    if (self)
        fold_tc_kernel<true, DESC><<<L.n_tiles, TNT, TcGeo<true>::SMEM, st>>>(L, D);
    else
        fold_tc_kernel<false, DESC><<<L.n_tiles, TNT, TcGeo<false>::SMEM, st>>>(L, D);
    if (ev1) record_event(ev1, st);
    if (fold_done) cudaEventRecord(fold_done, st);
    if (before_reduce) cudaStreamWaitEvent(st, before_reduce, 0);
    launch_pdl(fold_tc_reduce_kernel<MG>, dim3((L.tc_pairs == 2 ? 128 : 64) * TRB / 256, L.n_groups), dim3(256), 0, st,
               L, R);
}

template <int MG>
void fill_red(TcRed<MG>& R, const TcParams& D, int ng) {
    for (int g = 0; g < ng; ++g) {
        R.groups[g] = D.groups[g];
        R.slot[g] = D.segs[D.groups[g].seg].slot;
    }
}
}  // namespace

void launch_fold_tc(const FoldLaunch& L, const TcParams& D, int n_segs, bool self, cudaStream_t st, cudaEvent_t ev0,
                    cudaEvent_t ev1, cudaEvent_t before_reduce, const FoldTile* dev_tiles, cudaEvent_t fold_done) {
    if (L.n_tiles == 0) return;
    if (dev_tiles && L.n_groups <= 16 && n_segs <= 2) {
        thread_local TcDev S;
        thread_local TcRed<16> R;
        std::memcpy(S.xmap, D.xmap, n_segs * sizeof(CUtensorMap));
        std::memcpy(S.ymap, D.ymap, n_segs * sizeof(CUtensorMap));
        std::memcpy(S.p_base, D.p_base, n_segs * sizeof(int64_t));
        std::memcpy(S.segs, D.segs, n_segs * sizeof(FoldSeg));
        S.tiles = dev_tiles;
        fill_red(R, D, L.n_groups);
        launch_tc(L, S, R, self, st, ev0, ev1, before_reduce, fold_done);
    } else if (L.n_tiles <= 160 && L.n_groups <= 16 && n_segs <= 2) {
        thread_local TcSmall S;  // host staging (the launch copies it)
        thread_local TcRed<16> R;
        std::memcpy(S.xmap, D.xmap, n_segs * sizeof(CUtensorMap));
        std::memcpy(S.ymap, D.ymap, n_segs * sizeof(CUtensorMap));
        std::memcpy(S.p_base, D.p_base, n_segs * sizeof(int64_t));
        std::memcpy(S.segs, D.segs, n_segs * sizeof(FoldSeg));
        std::memcpy(S.tiles, D.tiles, L.n_tiles * sizeof(FoldTile));
        std::memcpy(S.groups, D.groups, L.n_groups * sizeof(FoldGroup));
        fill_red(R, D, L.n_groups);
        launch_tc(L, S, R, self, st, ev0, ev1, before_reduce, fold_done);
    } else {
        thread_local TcRed<FI_GROUPS> R;
        fill_red(R, D, L.n_groups);
        launch_tc(L, D, R, self, st, ev0, ev1, before_reduce, fold_done);
    }
}

void launch_fold_tcp(const FoldLaunch& L, const TcPlDesc& D, const FoldGroup* groups, cudaStream_t st,
                     cudaEvent_t ev0, cudaEvent_t ev1) {
    if (L.n_tiles == 0) return;
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr))
        cudaFuncSetAttribute(fold_tcp_kernel<TcPlDesc>, cudaFuncAttributeMaxDynamicSharedMemorySize, PL_SMEM);
    thread_local TcRed<FI_GROUPS> R;
    for (int g = 0; g < L.n_groups; ++g) {
        R.groups[g] = groups[g];
        R.slot[g] = D.segs[groups[g].seg].slot;
    }
    if (ev0) record_event(ev0, st);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    fold_tcp_kernel<TcPlDesc><<<std::min(L.n_tiles, sms), TPT, PL_SMEM, st>>>(L, D);
    if (ev1) record_event(ev1, st);
    launch_pdl(fold_tc_reduce_kernel<FI_GROUPS>, dim3(64 * TRB / 256, L.n_groups), dim3(256), 0, st, L, R);
}

bool encode_tcp2_maps(TcPl2Desc& D, int si, const uint16_t* plane0, int64_t plane_elems, int64_t p_base, int64_t rows,
                      int Pf, int64_t cols_samples) {
    D.p_base[si] = p_base;
    EncodeTiledFn enc = encode_fn();
    if (!enc || ((uintptr_t)plane0 & 15) || rows <= 0 || ((plane_elems * 2) & 15)) return false;
    // (64 samples of an atom, period rows, planes, atoms of 64 samples)
    const cuuint64_t gdim[4] = {64, (cuuint64_t)rows, 4, (cuuint64_t)((cols_samples + 63) / 64)};
    const cuuint64_t gstr[3] = {2ull * (uint64_t)Pf, 2ull * (uint64_t)plane_elems, 128};
    const cuuint32_t xbox[4] = {64, (cuuint32_t)TKB, 4, 2}, ybox[4] = {64, (cuuint32_t)TKB, 2, 2}, es[4] = {1, 1, 1, 1};
    return enc(&D.xmap[si], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(plane0), gdim, gstr, xbox, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
           enc(&D.ymap[si], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(plane0), gdim, gstr, ybox, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_fold_tcp2(const FoldLaunch& L, const TcPl2Desc& D, const FoldGroup* groups, cudaStream_t st,
                      cudaEvent_t ev0, cudaEvent_t ev1) {
    if (L.n_tiles == 0) return;
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr))
        cudaFuncSetAttribute(fold_tcp2_kernel<TcPl2Desc>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM);
    thread_local TcRed<FI_GROUPS> R;
    for (int g = 0; g < L.n_groups; ++g) {
        R.groups[g] = groups[g];
        R.slot[g] = D.segs[groups[g].seg].slot;
    }
    if (ev0) record_event(ev0, st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * L.n_tiles);
    cfg.blockDim = dim3(P2T);
    cfg.dynamicSmemBytes = P2_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fold_tcp2_kernel<TcPl2Desc>, L, D);
    if (ev1) record_event(ev1, st);
    fold_tc_reduce_kernel<FI_GROUPS><<<dim3(128 * TRB / 256, L.n_groups), 256, 0, st>>>(L, R);
}

int launch_split_planes4(const float2* x, int64_t n, int C, int64_t pitch_in, uint16_t* planes, int64_t plane_elems,
                         int64_t pitch_out, int64_t out_off, unsigned long long* key, cudaStream_t st) {
    if (n <= 0 || C <= 0) return 0;
    const int64_t per_row = (n + 4 * 256 - 1) / (4 * 256);
    split_planes4_kernel<<<(unsigned)(per_row * C), 256, 0, st>>>(x, n, C, pitch_in, planes, plane_elems, pitch_out,
                                                                  out_off, key);
    return 1;
}

int launch_split_planes(const float2* x, int64_t n, int C, int64_t pitch_in, uint32_t* hi, uint32_t* lo,
                        int64_t pitch_out, int64_t out_off, unsigned long long* key, cudaStream_t st) {
    if (n <= 0 || C <= 0) return 0;
    const int64_t per_row = (n + 4 * 256 - 1) / (4 * 256);
    split_planes_kernel<<<(unsigned)(per_row * C), 256, 0, st>>>(x, n, C, pitch_in, hi, lo, pitch_out, out_off, key);
    return 1;
}

}  // namespace cyc

#ifdef TC_TRACE
extern "C" int cyc_debug_tc_trace(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, cyc::g_tc_trace, sizeof(cyc::g_tc_trace));
}
extern "C" int cyc_debug_tc_warps(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, cyc::g_tc_warp, sizeof(cyc::g_tc_warp));
}
#endif

// MMA patterns of the planes fold (diagnostics): cycles per 16-period stage for
//   0: two N=256 products per split term (round-2 kernel: 6 x 128x256x16)
//   1: the 384-column union (3 x N=256 + 3 x N=128)
//   2: the union with A (y hi / lo) read from TMEM (tcgen05.mma ... [a_tmem])
// with or without 4 warps storing 24 KB per stage into the ring (a stand-in
// for the TMA writes).  Also checks the A-in-TMEM operand layout numerically:
// lane m, column c holds the bf16 pair (k = 2c, 2c + 1) of row m.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da), "l"(db), "r"(idesc),
        "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(db), "r"(idesc),
        "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
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
__host__ __device__ constexpr uint32_t idesc_n(uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// A from TMEM: A is K-major there (bit 15 = A MN-major must be 0)
__host__ __device__ constexpr uint32_t idesc_ts(uint32_t n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

constexpr int NPL = 6;
constexpr uint32_t SLOT = 32768;
constexpr uint32_t ATOM = 2048;

__global__ void __launch_bounds__(576, 1) bench(int nst, int pat, int writers, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[NPL], pfree[NPL], wdone[NPL];
    __shared__ uint32_t tmem_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < NPL * (int)SLOT / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + 12345u;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        const uint32_t lo = (h & 0x807f) | ((120u + ((h >> 8) & 15)) << 7),
                       hi = ((h >> 16) & 0x807f) | ((120u + ((h >> 24) & 15)) << 7);
        reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < NPL; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&pfree[s], 1);
            mbar_init(&wdone[s], 4);
        }
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
    if (warp == 0 && lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nst; ++it) {
            if (it >= NPL) mbar_wait(&pfree[s], ph ^ 1u);
            if (writers) mbar_wait(&wdone[s], ph);  // the stage's stores (TMA stand-in) landed
            mbar_arrive(&full[s]);
            if (++s == NPL) { s = 0; ph ^= 1u; }
        }
    } else if (warp == 1 && lane == 0) {
        const long long t0 = clock64();
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nst; ++it) {
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t xb = su32(sm) + (uint32_t)s * SLOT;
            const uint64_t dyh = desc_sw128(xb, 2 * ATOM, 1024), dyl = desc_sw128(xb + ATOM, 2 * ATOM, 1024);
            if (pat == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t dxh = desc_sw128(xb + 4 * h * ATOM, 2 * ATOM, 1024);
                    const uint64_t dxl = desc_sw128(xb + (4 * h + 1) * ATOM, 2 * ATOM, 1024);
                    mma_ss(tmem + 256 * h, dyh, dxh, idesc_n(256), 1u);
                    mma_ss(tmem + 256 * h, dyh, dxl, idesc_n(256), 1u);
                    mma_ss(tmem + 256 * h, dyl, dxh, idesc_n(256), 1u);
                }
            } else if (pat == 1) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t dxh = desc_sw128(xb + 8 * h * ATOM, 2 * ATOM, 1024);
                    const uint64_t dxl = desc_sw128(xb + (8 * h + 1) * ATOM, 2 * ATOM, 1024);
                    const uint32_t id = h ? idesc_n(128) : idesc_n(256);
                    mma_ss(tmem + 256 * h, dyh, dxh, id, 1u);
                    mma_ss(tmem + 256 * h, dyh, dxl, id, 1u);
                    mma_ss(tmem + 256 * h, dyl, dxh, id, 1u);
                }
            } else {
                // A ring in TMEM columns 384 + 16 s (hi 8 columns, lo 8 columns); contents stale (timing only)
                const uint32_t ah = tmem + 384 + 16 * (uint32_t)(s & 7), al = ah + 8;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t dxh = desc_sw128(xb + 8 * h * ATOM, 2 * ATOM, 1024);
                    const uint64_t dxl = desc_sw128(xb + (8 * h + 1) * ATOM, 2 * ATOM, 1024);
                    const uint32_t id = h ? idesc_ts(128) : idesc_ts(256);
                    mma_ts(tmem + 256 * h, ah, dxh, id, 1u);
                    mma_ts(tmem + 256 * h, ah, dxl, id, 1u);
                    mma_ts(tmem + 256 * h, al, dxh, id, 1u);
                }
            }
            mma_commit(&pfree[s]);
            if (++s == NPL) { s = 0; ph ^= 1u; }
        }
        mbar_wait(&pfree[(nst - 1) % NPL], ((nst - 1) / NPL) & 1);
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    } else if (writers && warp >= 2 && warp < 6) {
        // TMA stand-in: 24 KB of 16-byte stores per stage into the slot's last 24 KB... (the y atoms region
        // stays intact), after the slot was freed
        const int w = warp - 2;
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nst; ++it) {
            if (it >= NPL) mbar_wait(&pfree[s], ph ^ 1u);
            const uint32_t base = su32(sm) + (uint32_t)s * SLOT + 8192;
            for (int i = w * 32 + lane; i < 24576 / 16; i += 128)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + 16 * i), "r"(0x3c003c00u + it)
                             : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&wdone[s]);
            if (++s == NPL) { s = 0; ph ^= 1u; }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Layout check: A (128 x 16 bf16) written into TMEM by 4 warps (lane m, column c:
// bf16 pair (A[m][2c], A[m][2c+1])), B (256 x 16) in smem MN-major SW128 (atoms of
// 64 N values x 16 K rows), one ts MMA with N = 256, D read back.
__global__ void __launch_bounds__(128, 1) check(const float* A, const float* B, float* D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t done;
    __shared__ uint32_t tmem_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // B: element (n, k) at atom n/64, row k, 16-byte chunk ((n%64)/8) ^ (k%8), position n%8
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
        const int n = i / 16, k = i % 16;
        const uint32_t off = (uint32_t)((n >> 6) * 2048 + k * 128 + ((((n & 63) >> 3) ^ (k & 7)) << 4) + (n & 7) * 2);
        *reinterpret_cast<__nv_bfloat16*>(sm + off) = __float2bfloat16(B[n * 16 + k]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_s;
    {
        const int m = 32 * warp + lane;
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            __nv_bfloat162 v = __floats2bfloat162_rn(A[m * 16 + 2 * c], A[m * 16 + 2 * c + 1]);
            r[c] = *reinterpret_cast<uint32_t*>(&v);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((uint32_t)(32 * warp) << 16) + 384u),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint64_t db = desc_sw128(su32(sm), 2048, 1024);
        mma_ts(tmem, tmem + 384, db, idesc_ts(256), 0u);
        mma_commit(&done);
    }
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int m = 32 * warp + lane;
    for (int c = 0; c < 256; c += 8) {
        uint32_t u[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                     : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) D[m * 256 + c + j] = __uint_as_float(u[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    // layout check
    {
        std::vector<float> A(128 * 16), B(256 * 16), D(128 * 256);
        for (int i = 0; i < 128 * 16; ++i) A[i] = (float)((i * 7919) % 17 - 8) / 8.f;
        for (int i = 0; i < 256 * 16; ++i) B[i] = (float)((i * 104729) % 13 - 6) / 4.f;
        float *dA, *dB, *dD;
        cudaMalloc(&dA, A.size() * 4);
        cudaMalloc(&dB, B.size() * 4);
        cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
        check<<<1, 128, 16384 + 1024>>>(dA, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 256; ++n) {
                double ref = 0;
                for (int k = 0; k < 16; ++k) ref += (double)A[m * 16 + k] * B[n * 16 + k];
                worst = fmax(worst, fabs(ref - D[m * 256 + n]));
            }
        printf("A-in-TMEM layout check: %s, max |D - ref| = %g (D[0][0] %g)\n", cudaGetErrorString(e), worst, D[0]);
    }
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = NPL * SLOT + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nst = 4096 * (argc > 1 ? atoi(argv[1]) : 1);
    for (int writers = 0; writers < 2; ++writers)
        for (int pat = 0; pat < 3; ++pat) {
            unsigned long long h = 0;
            for (int rep = 0; rep < 2; ++rep) {
                bench<<<148, 576, smem>>>(nst, pat, writers, d);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("pattern %d (%s), TMA stand-in %d: %.1f cycles per stage (floor %d) %s\n", pat,
                   pat == 0 ? "2 x N256" : pat == 1 ? "union SS" : "union TS", writers, (double)h / nst,
                   pat == 0 ? 768 : 576, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}

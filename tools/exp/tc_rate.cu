// tcgen05.mma issue/execute rate (diagnostics): one CTA per SM, one thread
// issues NM back-to-back M=128 x N x K=16 bf16 MMAs (fp32 TMEM accumulator)
// from fixed shared-memory operands, SW128 layouts K-major or MN-major per
// operand, optionally several MMAs per accumulator before switching; cycles
// per MMA from clock64 around the issue loop + final commit wait.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc),
        "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(128, 1) k(int amn, int bmn, int N, int nm, int per_acc, unsigned long long* out,
                                            int commits) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, cb[8];
    __shared__ uint32_t tmem_s;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cb[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_s;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
                               (((uint32_t)N >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t a = su32(sm), b = su32(sm + 32 * 1024);
        // K-major SW128: 8-row groups of 1024 B (SBO); MN-major SW128: MN atoms 64 elements apart (LBO),
        // K groups of 8 rows 1024 B apart (SBO)
        const uint64_t da = amn ? desc_sw128(a, 8192, 1024) : desc_sw128(a, 16, 1024);
        const uint64_t db = bmn ? desc_sw128(b, 8192, 1024) : desc_sw128(b, 16, 1024);
        const long long t0 = clock64();
        if (per_acc == -1) {  // the planes kernel's stage: 2 accumulators x (hh, hl, lh), operands moving
                             // through an 8-slot ring, commit per stage, mbarrier wait per stage
            const uint32_t slot = 24576;
            for (int it = 0; it < nm / 6; ++it) {
                const uint32_t xb = su32(sm) + (uint32_t)(it % 3) * slot;
                mbar_wait(&bar, 1u);  // parity of the phase before the current one: returns at once
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint64_t dyh = amn ? desc_sw128(xb, 4096, 1024) : desc_sw128(xb, 16, 1024);
                const uint64_t dyl = amn ? desc_sw128(xb + 2048, 4096, 1024) : desc_sw128(xb + 2048, 16, 1024);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t dxh = bmn ? desc_sw128(xb + 8192 * h, 4096, 1024) : desc_sw128(xb + 8192 * h, 16, 1024);
                    const uint64_t dxl = bmn ? desc_sw128(xb + 8192 * h + 2048, 4096, 1024)
                                             : desc_sw128(xb + 8192 * h + 2048, 16, 1024);
                    mma_bf16(tmem + 256 * h, dyh, dxh, idesc, 1u);
                    mma_bf16(tmem + 256 * h, dyh, dxl, idesc, 1u);
                    mma_bf16(tmem + 256 * h, dyl, dxh, idesc, 1u);
                }
                if (commits) mma_commit(&cb[it & 7]);
                if (commits > 1 && (it & 31) == 31) mma_commit(&cb[(it + 4) & 7]);
            }
        } else if (per_acc == 0) {  // constant issue loop: two accumulators alternating every 4 MMAs
            for (int i = 0; i < nm; i += 8) {
#pragma unroll
                for (int u = 0; u < 4; ++u) mma_bf16(tmem, da, db, idesc, 1u);
#pragma unroll
                for (int u = 0; u < 4; ++u) mma_bf16(tmem + 256, da, db, idesc, 1u);
            }
        } else {
            for (int i = 0; i < nm; ++i) {
                const uint32_t acc_col = (uint32_t)((i / per_acc) % (512 / N)) * N;
                mma_bf16(tmem + acc_col, da, db, idesc, i % per_acc ? 1u : 0u);
            }
        }
        const long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t2 = clock64();
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024 + 1024);
    const int nm = 4096;
    for (int commits = 0; commits < 3; ++commits)
    for (int N : {256})
        for (int per_acc : {-1})
            for (int amn = 1; amn < 2; ++amn)
                for (int bmn = 1; bmn < 2; ++bmn) {
                    unsigned long long h[2];
                    for (int rep = 0; rep < 2; ++rep) {
                        k<<<148, 128, 97 * 1024 + 1024>>>(amn, bmn, N, nm, per_acc, d, commits);
                        cudaDeviceSynchronize();
                    }
                    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                    printf("commits %d N %3d per_acc %2d A %s B %s: issue %.1f, complete %.1f cycles per MMA (ideal %d) %s\n", commits, N,
                           per_acc, amn ? "MN" : "K ", bmn ? "MN" : "K ", (double)h[0] / nm, (double)h[1] / nm, N / 2,
                           cudaGetErrorString(cudaGetLastError()));
                }
    return 0;
}

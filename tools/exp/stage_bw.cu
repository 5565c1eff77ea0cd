// Staging-throughput probe for the tensor-core fold's x windows (C2 geometry:
// 2^24 cf32 samples, Pf = 1024, 128-residue tiles of 1.5x-overlapping 192-sample
// windows, 144 CTAs x ~910 periods, 16 periods per stage, 5-stage ring).  The
// consumer only releases stages, so the time is the L2/HBM -> SMEM staging alone.
//   mode 0: 12 TMA boxes of 32 floats x 16 rows, 128B swizzle (the kernel's)
//   mode 1: one TMA box of 192 8-byte elements x 16 rows, no swizzle
//   mode 2: 16 one-row 1-D bulk copies of 1536 B
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stage_bw stage_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int TKB = 16, NR = 5, STAGE = TKB * 1536, PF = 1024;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                 ::"r"(su32(b)), "r"(par) : "memory");
}
__global__ void __launch_bounds__(128, 1) stage_kernel(const __grid_constant__ CUtensorMap m0,
                                                       const __grid_constant__ CUtensorMap m1, const float2* x,
                                                       int mode, int periods_per_cta, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[NR], freeb[NR];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NR; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 3;" ::"r"(su32(&freeb[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int rb = blockIdx.x % 8, pc = blockIdx.x / 8;
    const int p0 = pc * periods_per_cta;
    const int nst = periods_per_cta / TKB;
    if (warp == 0) {
        for (int it = 0; it < nst; ++it) {
            const int s = it % NR;
            if (it >= NR) wait(&freeb[s], ((it / NR) - 1) & 1);
            const uint32_t st = su32(ring + s * STAGE);
            const int row = p0 + it * TKB;
            if (mode == 2) {
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                                 "r"(STAGE));
                __syncwarp();
                if (lane < TKB) {
                    const float2* src = x + (size_t)(row + lane) * PF + rb * 128;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(st + lane * 1536), "l"(src), "r"(1536), "r"(su32(&full[s])) : "memory");
                }
            } else if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE));
                if (mode == 0) {
                    for (int a = 0; a < 12; ++a)
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                     ::"r"(st + a * 2048), "l"((uint64_t)&m0), "r"(su32(&full[s])), "r"(2 * rb * 128 + 32 * a),
                                     "r"(row) : "memory");
                } else {
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                 ::"r"(st), "l"((uint64_t)&m1), "r"(su32(&full[s])), "r"(rb * 128), "r"(row) : "memory");
                }
            }
        }
    } else {
        float acc = 0.f;
        for (int it = 0; it < nst; ++it) {
            const int s = it % NR;
            wait(&full[s], (it / NR) & 1);
            acc += reinterpret_cast<const float*>(ring + s * STAGE)[threadIdx.x];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&freeb[s])) : "memory");
        }
        if (acc == 12345.f) sink[0] = acc;
    }
}

int main() {
    const size_t L = 1ull << 24;
    float2* x;
    float* sink;
    cudaMalloc(&x, L * 8 + 65536);
    cudaMemset(x, 0, L * 8 + 65536);
    cudaMalloc(&sink, 64);
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const cuuint64_t rows = L / PF;
    CUtensorMap m0, m1;
    {  // fp32, 32 x 16 boxes, SW128, rows of 2*PF + 256 floats (overlapping)
        cuuint64_t gdim[2] = {(cuuint64_t)2 * PF + 256, rows - 1};
        cuuint64_t gstr[1] = {(cuuint64_t)PF * 8};
        cuuint32_t box[2] = {32, 16}, es[2] = {1, 1};
        if (enc(&m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            printf("encode m0 failed\n");
    }
    {  // 8-byte elements (one cf32 sample), 192 x 16 boxes, no swizzle
        cuuint64_t gdim[2] = {(cuuint64_t)PF + 128, rows - 1};
        cuuint64_t gstr[1] = {(cuuint64_t)PF * 8};
        cuuint32_t box[2] = {192, 16}, es[2] = {1, 1};
        if (enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            printf("encode m1 failed\n");
    }
    const int ctas = 144, ppc = 16 * ((int)(rows - 2) / 18 / 16);  // 8 rb x 18 period chunks
    const size_t smem = NR * STAGE + 1024;
    cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int w = 0; w < 3; ++w) stage_kernel<<<ctas, 128, smem>>>(m0, m1, x, mode, ppc, sink);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) stage_kernel<<<ctas, 128, smem>>>(m0, m1, x, mode, ppc, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)ctas * ppc * 1536;
        printf("mode %d: %.2f us per launch, %.0f GB/s into SMEM (%d periods per CTA) %s\n", mode, 1e3 * ms / reps,
               bytes / (1e-3 * ms / reps) / 1e9, ppc, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

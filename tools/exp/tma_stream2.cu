// TMA delivery rate of the planes fold's access pattern without the MMAs
// (diagnostics): 4-D boxes {64 bf16, 16 periods, hi/lo, 6 atoms} (24 KB) over
// 2 x 256 MB bf16x2 planes (8192 periods x 8192 samples), one tile per CTA
// = 64 residues x 2048 periods (128 stages), 1024 tiles like C5's first lag
// pair, NS stages in flight, consumer thread releasing each stage after an
// optional delay (cycles) standing in for the MMA time.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
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
__device__ __forceinline__ void mbar_wait_test(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(dst), "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

__device__ __forceinline__ void prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"((uint64_t)map), "r"(c0),
                 "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void bulk_1d(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
constexpr int STAGE = 24576, NSMAX = 8;
template <bool TEST>
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap map, int ns, int delay, int nst,
                                           int n_rb, unsigned long long* cyc, long long* trace, const uint8_t* lin,
                                           int bulk, int pf) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[NSMAX], freeb[NSMAX];
    const int tile = blockIdx.x;
    const int rb = tile % n_rb, pr = tile / n_rb;  // residue block fastest (range-major like the kernel)
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&freeb[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    const int row0 = pr * nst * 16, atom0 = rb * 2;  // 64 residues = 2 atoms of 32 samples
    if (threadIdx.x == 0) {
        for (int it = 0; it < nst; ++it) {
            const int s = it % ns;
            if (it >= ns) {
                if (TEST) mbar_wait_test(&freeb[s], ((it / ns) - 1) & 1);
                else mbar_wait(&freeb[s], ((it / ns) - 1) & 1);
            }
            mbar_expect_tx(&full[s], STAGE);
            if (bulk) {
                // tile-major planes: stage (period block, window) = one contiguous 24 KB block; the window of
                // residue block rb starts 2 atoms (8 KB) after rb - 1's (the windows overlap like the kernel's)
                const size_t pb = (size_t)(row0 / 16 + it);
                const uint8_t* src = lin + (pb * (size_t)(n_rb * 2 + 6) + (size_t)atom0) * 4096;
                bulk_1d(su32(ring + s * STAGE), src, STAGE, &full[s]);
            } else {
                if (pf > 0) {
                    if (it == 0)
                        for (int j = 1; j < pf && j < nst; ++j) prefetch_4d(&map, 0, row0 + j * 16, 0, atom0);
                    if (it + pf < nst) prefetch_4d(&map, 0, row0 + (it + pf) * 16, 0, atom0);
                }
                tma_4d(su32(ring + s * STAGE), &map, 0, row0 + it * 16, 0, atom0, &full[s]);
            }
            if (blockIdx.x == 0 && it < 128) trace[it * 4 + 0] = clock64() - t0;
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < nst; ++it) {
            const int s = it % ns;
            const long long w0 = clock64();
            if (TEST) mbar_wait_test(&full[s], (it / ns) & 1);
            else mbar_wait(&full[s], (it / ns) & 1);
            if (blockIdx.x == 0 && it < 128) {
                trace[it * 4 + 1] = w0 - t0;
                trace[it * 4 + 2] = clock64() - t0;
            }
            if (delay > 0) {
                const long long a = clock64();
                while (clock64() - a < delay) {
                }
            }
            mbar_arrive(&freeb[s]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(clock64() - t0));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    const int P = 8192, S = 8192;               // periods, samples per period
    const size_t plane = (size_t)P * S * 4;     // bf16x2 words
    uint8_t* buf;
    if (cudaMalloc(&buf, 2 * plane + (64u << 20)) != cudaSuccess) return 1;
    cudaMemset(buf, 0, 2 * plane + (64u << 20));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    const int promo = argc > 1 ? atoi(argv[1]) : 2;
    // dims: {64 bf16 (128 B), periods, planes, atoms}; atom stride 128 B overlaps dim 0 like encode_planes_4d
    cuuint64_t gdim[4] = {64, (cuuint64_t)P, 2, (cuuint64_t)(S / 32)};
    cuuint64_t gstr[3] = {(cuuint64_t)S * 4, plane, 128};
    cuuint32_t box[4] = {64, 16, 2, 6}, es[4] = {1, 1, 1, 1};
    CUtensorMap map;
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8);
    long long* trace;
    cudaMalloc(&trace, 128 * 4 * 8);
    const int n_rb = S / 64, nranges = 4, nst = P / nranges / 16;  // 128 rb x 4 ranges = 512 tiles (one lag pair)
    cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, NSMAX * STAGE + 1024);
    cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, NSMAX * STAGE + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    uint8_t* lin = buf;  // same bytes, read as tile-major blocks (period block x (2 n_rb + 6) atoms x 4 KB)
    for (int bulk = 0; bulk < 1; ++bulk)
    for (int pf : {0, 8, 16, 32})
    for (int test = 0; test < 1; ++test)
    for (int ns : {6})
        for (int delay : {0, 576}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(cyc, 0, 8);
                cudaEventRecord(a);
                if (test) k<true><<<n_rb * nranges, 64, NSMAX * STAGE + 1024>>>(map, ns, delay, nst, n_rb, cyc, trace, lin, bulk, pf);
                else k<false><<<n_rb * nranges, 64, NSMAX * STAGE + 1024>>>(map, ns, delay, nst, n_rb, cyc, trace, lin, bulk, pf);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                unsigned long long c;
                cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                const double bytes = (double)n_rb * nranges * nst * STAGE;
                if (false) {
                    long long h[128 * 4];
                    cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost);
                    for (int it : {0, 1, 7, 8, 9, 20, 21, 60, 61, 100})
                        printf("  it %3d issue %7lld wait_start %7lld ready %7lld  (ready - issue %lld)\n", it, h[it * 4],
                               h[it * 4 + 1], h[it * 4 + 2], h[it * 4 + 2] - h[it * 4]);
                }
                if (rep)
                    printf("pf %2d %s %s promo %d ns %d delay %4d: %.1f us, %.2f TB/s, %.1f B/clk/SM (1.965 GHz), %.0f cycles/stage/CTA  %s\n",
                           pf, bulk ? "bulk-1d" : "tma-4d ", test ? "test_wait" : "try_wait ", promo, ns, delay, ms * 1e3, bytes / ms / 1e9, bytes / (ms * 1e-3) / 148 / 1.965e9,
                           (double)c / (n_rb * nranges) / nst, cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}

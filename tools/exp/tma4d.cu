// TMA issue cost: 12 2-D boxes (64 bf16 x 16 rows) vs one 4-D box
// {64 bf16, 16 rows, 2 planes, 6 atoms} (the same 24 KB) per stage, one
// issuing thread per CTA, 148 CTAs, 5-stage ring, L2-resident source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma4d tma4d.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m4,
                                          int stages, int rows_total, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[5];
    const int NS = 5, STAGE = 24576;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < stages + NS; ++it) {
        if (it >= NS) {
            const int s = (it - NS) % NS;
            const uint32_t par = ((it - NS) / NS) & 1;
            asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&full[s])), "r"(par) : "memory");
        }
        if (it < stages) {
            const int s = it % NS;
            const uint32_t st = su32(ring + s * STAGE);
            // each CTA streams its own band of rows (like a fold tile over its period range)
            const long long band = (rows_total - 16) / gridDim.x;
            const int row = (int)(blockIdx.x * band + ((long long)it * 16) % (band > 16 ? band - 16 : 1));
            const int atom0 = (blockIdx.x * 6) % 120;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE) : "memory");
            if (MODE == 0) {
                for (int b = 0; b < 12; ++b) {
                    const int a = b % 6, pl = b / 6;
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                 ::"r"(st + b * 2048), "l"((uint64_t)&m2), "r"(su32(&full[s])), "r"((atom0 + a) * 64 + pl * 8192), "r"(row) : "memory");
                }
            } else {
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             ::"r"(st), "l"((uint64_t)&m4), "r"(su32(&full[s])), "r"(0), "r"(row), "r"(0), "r"(atom0) : "memory");
            }
        }
    }
    cyc[blockIdx.x] = clock64() - t0;
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = (Enc)fp;
    // planes: row pitch 32 KB (8192 samples x 4 B), hi plane then lo plane 16 MB apart... keep the
    // whole buffer L2-resident: 512 rows x 32 KB = 16 MB per plane
    const uint64_t pitch = 32768, rows = argc > 1 ? (uint64_t)atoi(argv[1]) * 16 : 256, plane = pitch * rows;
    void* buf;
    cudaMalloc(&buf, 2 * plane);
    cudaMemset(buf, 0, 2 * plane);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    CUtensorMap m2, m4;
    {   // 2-D: cols = 2 planes side by side is not contiguous; use one map over [rows][16384 bf16] and put the lo
        // plane at column offset 8192 (same bytes as separate planes for the cost test)
        cuuint64_t gdim[2] = {16384, rows}, gstr[1] = {pitch};
        cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
        if (enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            printf("enc2 failed\n");
    }
    {   // 4-D: (64 elements, rows, planes, atoms); atom stride 128 B overlaps the element run
        cuuint64_t gdim[4] = {64, rows, 2, 120}, gstr[3] = {pitch, plane, 128};
        cuuint32_t box[4] = {64, 16, 2, 6}, es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("enc4 failed %d\n", (int)r);
    }
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 24576 + 1024);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 24576 + 1024);
    const int stages = 2000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148, 32, 5 * 24576 + 1024>>>(m2, m4, stages, (int)rows, cyc);
            else k<1><<<148, 32, 5 * 24576 + 1024>>>(m2, m4, stages, (int)rows, cyc);
        }
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(148);
        cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
        double sum = 0;
        for (auto v : h) sum += v;
        const double per = sum / 148 / stages;
        printf("%s: %.0f cycles per 24 KB stage (%.1f B/clk/SM) err=%s\n", mode ? "one 4-D box {64,16,2,6}" : "12 2-D boxes {64,16}",
               per, 24576.0 / per, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

// TMA staging rate per SM (diagnostics): 148 CTAs each stream 2-D boxes of
// 64 bf16 x 16 rows (one 128B-swizzle atom column, 2 KB) from an L2-resident
// buffer into a 5-deep ring of 40 KB stages (20 boxes per stage), like the
// planes fold.  Row pitch `pitch` bytes: 32768 (period rows of C5 planes: 16
// separate 128-B rows per box) or 128 (pre-tiled: one contiguous 2 KB box).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) stage_kernel(const __grid_constant__ CUtensorMap map, int stages, int boxes,
                                                     int rows_total, int cols_boxes, unsigned long long* cyc,
                                                     int box_rows, int nw) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[5];
    const int NS = 5, STAGE = 40960;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(nw));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) != 0 || w >= nw) return;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < stages + NS; ++it) {
        if (it >= NS) {  // consume stage it - NS
            const int s = (it - NS) % NS;
            const uint32_t par = ((it - NS) / NS) & 1;
            asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}"
                         ::"r"(su32(&full[s])), "r"(par) : "memory");
        }
        if (it < stages) {
            const int s = it % NS;
            const uint32_t st = su32(ring + s * STAGE);
            const int mine = (boxes - w + nw - 1) / nw;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(mine * 128 * box_rows) : "memory");
            for (int b = w; b < boxes; b += nw) {
                const int col = ((blockIdx.x * 7 + b) % cols_boxes) * 64;
                const int row = (int)(((long long)it * box_rows + blockIdx.x * 64) % (rows_total - box_rows));
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(st + b * 128 * box_rows), "l"((uint64_t)&map), "r"(su32(&full[s])), "r"(col), "r"(row) : "memory");
            }
        }
    }
    if (w == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = (Enc)fp;
    const size_t bytes = 16u << 20;  // 16 MB: L2 resident
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 40960 + 1024);
    const int stages = 2000;
    for (int nw : {1, 2, 4, 8}) {
        const int pitch = 32768;
        for (int br : {16, 64}) {
            const int boxes = 40960 / (128 * br);
            const uint64_t cols = pitch / 2;
            const uint64_t rows = bytes / pitch;
            CUtensorMap m;
            cuuint64_t gdim[2] = {cols, rows}, gstr[1] = {(cuuint64_t)pitch};
            cuuint32_t box[2] = {64, (cuuint32_t)br}, es[2] = {1, 1};
            if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("encode failed\n");
                continue;
            }
            const int cb = (int)(cols / 64) > 0 ? (int)(cols / 64) : 1;
            for (int rep = 0; rep < 2; ++rep)
                stage_kernel<<<148, 256, 5 * 40960 + 1024>>>(m, stages, boxes, (int)rows, cb, cyc, br, nw);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            double sum = 0;
            for (auto v : h) sum += v;
            const double per = sum / 148 / stages;
            printf("issuers %d pitch %6d box rows %3d (%2d boxes, 40 KB): %.0f cycles/stage  %.1f B/clk/SM  %.0f cyc/box  err=%s\n",
                   nw, pitch, br, boxes, per, 40960.0 / per, per / boxes, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

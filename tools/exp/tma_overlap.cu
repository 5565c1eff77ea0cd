// Does cuTensorMapEncodeTiled accept overlapping rows (row stride < row width),
// and does a TMA box that crosses the nominal row end read the next row's head?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, float* out) {
    __shared__ __align__(128) float buf[16 * 256];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16 * 256 * 4));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(buf)), "l"((uint64_t)&m), "r"(su32(&bar)), "r"(c0), "r"(c1) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
    const int Pf = 1024, P = 64;
    std::vector<float> h((size_t)P * 2 * Pf);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *dx, *dout;
    cudaMalloc(&dx, h.size() * 4 + 4096);
    cudaMemcpy(dx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&dout, 16 * 256 * 4);
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t gdim[2] = {(cuuint64_t)2 * Pf + 256, (cuuint64_t)P - 1};
    cuuint64_t gstr[1] = {(cuuint64_t)2 * Pf * 4};
    cuuint32_t box[2] = {256, 16}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode overlapping rows: %d\n", (int)r);
    if (r) return 0;
    k<<<1, 256>>>(m, 2 * Pf - 128, 5, dout);  // window crosses row end by 128 floats
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(16 * 256);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int k = 0; k < 16; ++k)
        for (int i = 0; i < 256; ++i) {
            const float want = (float)((size_t)(5 + k) * 2 * Pf + 2 * Pf - 128 + i);
            bad += o[k * 256 + i] != want;
        }
    printf("kernel: %s, mismatches %d (o[0]=%.0f o[200]=%.0f)\n", cudaGetErrorString(e), bad, o[0], o[200]);
    return 0;
}

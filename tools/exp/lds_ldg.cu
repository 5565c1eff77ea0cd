// Do global loads (L1::no_allocate) take shared-memory bandwidth?  8 warps read
// shared memory with LDS.128 as fast as they can; 4 more warps optionally
// stream 16-byte global loads.  Compare the LDS rate with and without the LDG
// warps.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_ldg lds_ldg.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float4 ldg_na(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(384, 1) k(const float4* g, size_t g_n, int iters, int ldg_on, float* sink,
                                            unsigned long long* cyc) {
    __shared__ float4 sm[2048];  // 32 KB
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, 0, 0, 0);
    __syncthreads();
    const unsigned long long t0 = clock64();
    float acc = 0.f;
    if (warp < 8) {
        uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)((warp * 32 + lane) * 16);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float4 v;
                const uint32_t a = base + (uint32_t)(((it * 8 + u) * 4096) & 32767);
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
                acc += v.x;
            }
        }
    } else if (ldg_on) {
        size_t base = ((size_t)blockIdx.x * 4 + (warp - 8)) * 32 + lane;
        const size_t stride = (size_t)gridDim.x * 4 * 32;
        for (int it = 0; it < iters; ++it) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ldg_na(g + ((base + u * stride) & (g_n - 1)));
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x;
            base += 8 * stride;
        }
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;  // the LDS warps' own time
    __syncthreads();
    if (acc == 1.2345f) sink[0] = acc;
}

int main() {
    const size_t n = (size_t)1 << 25;  // 512 MB of float4
    float4* g;
    float* sink;
    unsigned long long* cyc;
    cudaMalloc(&g, n * 16);
    cudaMemset(g, 0, n * 16);
    cudaMalloc(&sink, 64);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int on = 0; on < 2; ++on) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<148, 384>>>(g, n, iters, on, sink, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double lds_bytes = 8.0 * 32 * iters * 8 * 16;  // per SM
            const double ldg_bytes = on ? 4.0 * 32 * iters * 8 * 16 : 0;
            printf("ldg %d: kernel %.3f ms; LDS warps %llu cycles: LDS %.1f B/clk per SM (LDG %.1f GB/s total)\n",
                   on, ms, c, lds_bytes / c, ldg_bytes * 148 / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}

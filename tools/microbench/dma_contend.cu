// H2D 128 MiB in 8 pieces while (a) nothing, (b) an FFMA-bound kernel, (c) an HBM-streaming
// kernel, (d) a kernel reading mapped host memory runs concurrently on another stream.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma(float* o, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 1.0001f, 0.5f);
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void stream_rd(const float4* p, size_t n, float* o, int reps) {
    float s = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += p[i].x;
    o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    size_t nb = 128ull << 20;
    void *h, *d; float* o; float4* big;
    cudaMallocHost(&h, nb); cudaMalloc(&d, nb); cudaMalloc(&o, 1 << 24); cudaMalloc(&big, 1ull << 30);
    cudaStream_t s, k; cudaStreamCreate(&s); cudaStreamCreate(&k);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            if (mode == 1) ffma<<<148 * 4, 256, 0, k>>>(o, 400000);
            if (mode == 2) stream_rd<<<148 * 8, 256, 0, k>>>(big, (1ull << 30) / 16, o, 20);
            cudaEventRecord(e0, s);
            for (int i = 0; i < 8; ++i) cudaMemcpyAsync((char*)d + i * (nb / 8), (char*)h + i * (nb / 8), nb / 8, cudaMemcpyHostToDevice, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaDeviceSynchronize();
            if (rep == 2) printf("{\"mode\":%d,\"ms\":%.3f,\"GBps\":%.1f}\n", mode, ms, nb / ms / 1e6);
        }
    }
    return 0;
}

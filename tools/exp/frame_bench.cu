// Event-timed fold_frame (launch_fold_small) and FFT finalize of one C3
// emission (Pf 1024, 64 periods, 32 lags, weighted), back to back and alone,
// against an empty kernel (diagnostics for the small-call path).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2405_16911_b200/csrc/kernels.cuh"
__global__ void nop_k() {}
int main() {
    const int Pf = 1024, T = 32, N = 65536;
    const int64_t cap = 1 << 20;
    float2* ring;
    cudaMalloc(&ring, cap * sizeof(float2));
    std::vector<float2> h(cap);
    for (int64_t i = 0; i < cap; ++i) h[i] = make_float2(std::sin(i * 0.1f), std::cos(i * 0.37f));
    cudaMemcpy(ring, h.data(), cap * sizeof(float2), cudaMemcpyHostToDevice);
    cyc::FoldSeg g{};
    g.x = g.y = ring;
    g.n_start = 4 * N;
    g.n_end = 5 * N;
    g.x_lo = g.n_start;
    g.x_hi = g.n_end + T;
    g.mask = cap - 1;
    g.w_ref = g.n_end - 1;
    g.w_log2 = (float)std::log2(1.0 - 1.0 / 4096);
    g.w_scale = 1.0f / 4096;
    cyc::FoldSeg* gd;
    cudaMalloc(&gd, sizeof g);
    cudaMemcpy(gd, &g, sizeof g, cudaMemcpyHostToDevice);
    double* S;
    cudaMalloc(&S, (size_t)T * Pf * 4 * sizeof(double));
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char* what, auto fn) {
        for (int i = 0; i < 20; ++i) fn();
        cudaStreamSynchronize(st);
        float tot = 0;
        for (int i = 0; i < 200; ++i) {
            cudaEventRecord(a, st);
            fn();
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            tot += ms;
        }
        printf("%-40s %.2f us\n", what, tot / 200 * 1e3);
    };
    time("empty kernel", [&] { nop_k<<<1, 32, 0, st>>>(); });
    time("10x empty kernel back to back (per launch)", [&] {
        for (int k = 0; k < 10; ++k) nop_k<<<1, 32, 0, st>>>();
    });
    time("10x empty 128x1024 kernel back to back", [&] {
        for (int k = 0; k < 10; ++k) nop_k<<<128, 1024, 0, st>>>();
    });
    time("fold_frame (launch_fold_small)", [&] { cyc::launch_fold_small(gd, 1, Pf, 0, T, T, S, st, nullptr); });
    time("10x fold_frame back to back (per launch)", [&] {
        for (int k = 0; k < 10; ++k) cyc::launch_fold_small(gd, 1, Pf, 0, T, T, S, st, nullptr);
    });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// FFMA2 issue rate for the fold's operand pattern: acc pair += x pair * y scalar (all registers),
// at the fold's occupancy (1 CTA x 256 threads per SM, 2 warps/SMSP) and at 8 warps/SMSP.
#include <cstdio>
#include <cuda_runtime.h>
union F2U { float2 f; unsigned long long u; };
__device__ __forceinline__ void f2(float2& acc, float2 a, float b) {
    F2U A, B, C; A.f = a; B.f = make_float2(b, b); C.f = acc;
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C.u) : "l"(A.u), "l"(B.u)); acc = C.f;
}
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s) {
    float2 lo[4][8], hi[4][8];
    for (int a = 0; a < 4; ++a) for (int u = 0; u < 8; ++u) { lo[a][u] = make_float2(a, u); hi[a][u] = make_float2(u, a); }
    float2 xv[12]; float yr[4], yi[4];
    for (int i = 0; i < 12; ++i) xv[i] = make_float2(threadIdx.x * 1e-3f + i, i * s);
    for (int a = 0; a < 4; ++a) { yr[a] = s * a; yi[a] = s - a; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                f2(lo[a][u], xv[a + u], yr[a]);
                if (MODE == 0) f2(hi[a][u], xv[a + u], yi[a]);
            }
        if (MODE == 1) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int u = 0; u < 8; ++u) f2(hi[a][u], xv[a + u], yi[a]);
        }
#pragma unroll
        for (int i = 0; i < 12; ++i) xv[i].x += 1e-7f;  // keep x live, cheap
    }
    float t = 0;
    for (int a = 0; a < 4; ++a) for (int u = 0; u < 8; ++u) t += lo[a][u].x + lo[a][u].y + hi[a][u].x + hi[a][u].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int ctas : {148, 148 * 4}) {
        for (int mode = 0; mode < 2; ++mode) {
            int iters = 4000; float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) k<0><<<ctas, 256>>>(o, iters, 1.0001f); else k<1><<<ctas, 256>>>(o, iters, 1.0001f);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
            }
            double fl = 2.0 * 2 * 64 * (double)iters * ctas * 256;  // 64 FFMA2 x 2 lanes x 2 flop
            printf("{\"ctas\":%d,\"mode\":%d,\"tflops\":%.2f}\n", ctas, mode, fl / best / 1e9);
        }
    }
    return 0;
}

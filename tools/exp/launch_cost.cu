// Host-side cost of the per-call CUDA operations of the small-push path
// (diagnostics): kernel launch, 64 KB pinned H2D enqueue, graph launch,
// event record/query, stream sync round trip.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
__global__ void nop(int* p) { if (p && threadIdx.x == 1234) p[0] = 1; }
__global__ void touch(const float2* s, int n, float* o) {
    float a = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a += s[i].x;
    if (a == 1234.5f) *o = a;
}
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void rd(const int* p, int* o) {
    __shared__ int v;
    if (threadIdx.x < 16) atomicAdd(&v, p[threadIdx.x]);
    __syncthreads();
    if (threadIdx.x == 0 && v == 123456) *o = v;
}
__global__ void wr(double2* h, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) h[i] = make_double2(i, i);
}
int main() {
    cudaStream_t s, s2;
    cudaStreamCreate(&s);
    cudaStreamCreate(&s2);
    float2 *h, *d;
    float* o;
    cudaMallocHost(&h, 64 << 20);
    cudaMalloc(&d, 64 << 20);
    cudaMalloc(&o, 4);
    const int R = 20000;
    for (int w = 0; w < 2; ++w) {
        double t = now();
        for (int i = 0; i < R; ++i) nop<<<1, 32, 0, s>>>(nullptr);
        double t1 = now();
        cudaStreamSynchronize(s);
        printf("kernel launch: %.2f us host each (drain %.1f us)\n", (t1 - t) / R, now() - t1);
        t = now();
        for (int i = 0; i < R; ++i) cudaMemcpyAsync(d + (i % 512) * 8192, h + (i % 512) * 8192, 65536, cudaMemcpyHostToDevice, s2);
        t1 = now();
        cudaStreamSynchronize(s2);
        printf("64 KB H2D enqueue: %.2f us host each; %.2f us per copy incl drain\n", (t1 - t) / R, (now() - t) / R);
        t = now();
        for (int i = 0; i < R / 10; ++i) { nop<<<1, 32, 0, s>>>(nullptr); cudaStreamSynchronize(s); }
        printf("launch + sync round trip: %.2f us\n", (now() - t) / (R / 10));
        t = now();
        for (int i = 0; i < R / 10; ++i) { cudaMemcpyAsync(d, h, 65536, cudaMemcpyHostToDevice, s2); cudaStreamSynchronize(s2); }
        printf("64 KB H2D + sync round trip: %.2f us\n", (now() - t) / (R / 10));
        t = now();
        for (int i = 0; i < R / 10; ++i) { touch<<<64, 256, 0, s>>>(h + (i % 512) * 8192, 8192, o); cudaStreamSynchronize(s); }
        printf("zero-copy read of 64 KB by a kernel + sync: %.2f us\n", (now() - t) / (R / 10));
        {
            int *hm, *dm, *o2;
            cudaHostAlloc(&hm, 4096, cudaHostAllocMapped);
            cudaMalloc(&dm, 4096);
            cudaMalloc(&o2, 4);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int mode = 0; mode < 4; ++mode) {
                float tot = 0.f;
                for (int i = 0; i < 200; ++i) {
                    if (mode == 2) hm[i % 16] = i;  // CPU dirties the line first
                    cudaEventRecord(a, s);
                    if (mode == 3) wr<<<32, 256, 0, s>>>((double2*)h, 8192);
                    else rd<<<64, 256, 0, s>>>(mode == 1 ? dm : hm, o2);
                    cudaEventRecord(b, s);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    tot += ms;
                }
                printf("%s: %.2f us (event-timed)\n", mode == 0 ? "64 CTAs read 16 words of mapped host memory" :
                       mode == 1 ? "64 CTAs read 16 words of device memory" : mode == 2 ? "mapped read after a CPU write" :
                       "32 CTAs write 128 KB to pinned host memory", tot / 200 * 1e3);
            }
        }
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        nop<<<1, 32, 0, s>>>(nullptr); nop<<<1, 32, 0, s>>>(nullptr); nop<<<1, 32, 0, s>>>(nullptr);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        t = now();
        for (int i = 0; i < R; ++i) cudaGraphLaunch(ge, s);
        t1 = now();
        cudaStreamSynchronize(s);
        printf("3-kernel graph launch: %.2f us host each\n", (t1 - t) / R);
        t = now();
        for (int i = 0; i < R / 10; ++i) { cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); }
        printf("graph launch + sync round trip: %.2f us\n", (now() - t) / (R / 10));
        cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        t = now();
        for (int i = 0; i < R; ++i) { cudaEventRecord(e, s); }
        printf("event record: %.2f us\n", (now() - t) / R);
        t = now();
        for (int i = 0; i < R; ++i) { cudaEventQuery(e); }
        printf("event query: %.2f us\n", (now() - t) / R);
    }
    return 0;
}

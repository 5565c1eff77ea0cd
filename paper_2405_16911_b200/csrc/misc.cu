// misc.cu -- small device utilities of the streaming engine.
#include "kernels.cuh"

namespace cyc {
namespace {

__global__ void add_f64_kernel(double* dst, const double* src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

// average_frames (proj/src/estimator.cpp:86-105): running coherent and
// magnitude sums in frame order (deterministic per element).
__global__ void accum_frames_kernel(const double2* frames, int64_t n_frames, int64_t len, double2* coh,
                                    double* mag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        double2 c = coh[i];
        double m = mag[i];
        for (int64_t f = 0; f < n_frames; ++f) {
            const double2 v = frames[f * len + i];
            c.x += v.x;
            c.y += v.y;
            m += hypot(v.x, v.y);
        }
        coh[i] = c;
        mag[i] = m;
    }
}

// Whole-chunk finite scan (proj/src/estimator.cpp:43-52): the smallest key
// 2*i (x) / 2*i+1 (y) names the first offending sample in the reference's
// scan order (x before y at each index).
__global__ void finite_check_kernel(const float2* x, const float2* y, int64_t n, int64_t base, int channels, int ch,
                                    unsigned long long* key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 a = x[i];
        unsigned long long k = ~0ull;
        const unsigned long long idx = (unsigned long long)(base + i);
        if (!isfinite(a.x) || !isfinite(a.y)) {
            k = (2ull * idx) * (unsigned long long)channels + (unsigned long long)ch;
        } else if (y) {
            const float2 b = y[i];
            if (!isfinite(b.x) || !isfinite(b.y)) k = (2ull * idx + 1ull) * (unsigned long long)channels + (unsigned long long)ch;
        }
        if (k != ~0ull) atomicMin(key, k);
    }
}

__global__ void ring_write_kernel(float2* ring, uint64_t mask, int64_t abs0, const float2* src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ring[(uint64_t)(abs0 + i) & mask] = src[i];
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

void launch_add_f64(double* dst, const double* src, int64_t n, cudaStream_t st) {
    if (n > 0) add_f64_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, src, n);
}
void launch_accum_frames(const double2* frames, int64_t n_frames, int64_t len, double2* coh, double* mag,
                         cudaStream_t st) {
    if (n_frames > 0 && len > 0) accum_frames_kernel<<<grid_for(len, 256), 256, 0, st>>>(frames, n_frames, len, coh, mag);
}
void launch_finite_check(const float2* x, const float2* y, int64_t n, int64_t base, int channels, int ch,
                         unsigned long long* key, cudaStream_t st) {
    if (n > 0) finite_check_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, y, n, base, channels, ch, key);
}
void launch_ring_write(float2* ring, uint64_t mask, int64_t abs0, const float2* src, int64_t n, cudaStream_t st) {
    if (n > 0) ring_write_kernel<<<grid_for(n, 256), 256, 0, st>>>(ring, mask, abs0, src, n);
}

}  // namespace cyc

// ---------------------------------------------------------------------------
// FP32 FFMA peak microbenchmark: the roofline denominator for the fold kernel
// (MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks).  16
// independent FMA chains per thread, 4 CTAs x 256 threads per SM.
// ---------------------------------------------------------------------------
namespace cyc {
namespace {
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, float a, float b, int iters) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

double measure_fp32_peak_tflops(int device) {
    cudaSetDevice(device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int grid = sms * 4, block = 256, iters = 20000;
    float* out = nullptr;
    if (cudaMalloc(&out, (size_t)grid * block * sizeof(float)) != cudaSuccess) return 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        ffma_peak_kernel<<<grid, block>>>(out, 1.0001f, 0.999f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 16 * iters * (double)grid * block;
    return flops / (best * 1e-3) / 1e12;
}
}  // namespace cyc

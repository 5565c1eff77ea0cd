// misc.cu -- small device utilities of the streaming engine.
#include <algorithm>

#include "kernels.cuh"

namespace cyc {
thread_local bool g_capture_events = false;

namespace {

__global__ void add_f64_kernel(double* dst, const double* src, int64_t n, const unsigned long long* gate) {
    if (gate && *gate != ~0ull) return;  // a rejected chunk commits nothing
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

// Recursive emissions: the frames of a batch are slots
// [frame][channel] of weighted window sums v; in frame order per channel,
// R = decay * R + v (R_f = lam^N R_{f-1} + window sum), the emitted table is
// R, and the running average_frames sums take R and |R|.
__global__ void recursive_update_kernel(double2* frames, int64_t n_frames, int channels, int64_t per, double2* R,
                                        double decay, double2* coh, double* mag, double2* host_out) {
    const int64_t len = (int64_t)channels * per;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        double2 r = R[i], c = coh[i];
        double m = mag[i];
        for (int64_t f = 0; f < n_frames; ++f) {
            double2& v = frames[f * len + i];
            r.x = decay * r.x + v.x;
            r.y = decay * r.y + v.y;
            v = r;
            if (host_out) host_out[f * len + i] = r;  // mapped pinned memory: no D2H copy node
            c.x += r.x;
            c.y += r.y;
            m += hypot(r.x, r.y);
        }
        R[i] = r;
        coh[i] = c;
        mag[i] = m;
    }
}

// Whole-chunk finite scan (proj/src/estimator.cpp:43-52): the smallest key
// 2*i (x) / 2*i+1 (y) names the first offending sample in the reference's
// scan order (x before y at each index).
// blockIdx.y selects channel ch + blockIdx.y, whose samples start pitch * blockIdx.y further
__global__ void finite_check_kernel(const float2* x, const float2* y, int64_t n, int64_t base, int channels, int ch,
                                    unsigned long long* key, int64_t pitch) {
    x += pitch * blockIdx.y;
    if (y) y += pitch * blockIdx.y;
    ch += blockIdx.y;
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

__device__ __forceinline__ bool nonfinite4(const float4& v) {
    const unsigned e = 0x7f800000u;
    return ((__float_as_uint(v.x) & e) == e) | ((__float_as_uint(v.y) & e) == e) |
           ((__float_as_uint(v.z) & e) == e) | ((__float_as_uint(v.w) & e) == e);
}

// Same scan, two samples per 16-byte load and four loads in flight per thread
// (HBM-bound: 8 B/sample per stream).  A flagged pair is re-checked sample by
// sample so the key is exactly the scalar kernel's.
__global__ void __launch_bounds__(256) finite_check_v4_kernel(const float4* x, const float4* y, int64_t pairs,
                                                              int64_t base, int channels, int ch,
                                                              unsigned long long* key, int64_t pitch) {
    x += (pitch / 2) * blockIdx.y;  // pitch in samples (even: 16-byte aligned rows)
    if (y) y += (pitch / 2) * blockIdx.y;
    ch += blockIdx.y;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto slow = [&](int64_t p) {
        unsigned long long k = ~0ull;
        for (int h = 1; h >= 0; --h) {  // later sample first so the earlier one wins
            const int64_t i = 2 * p + h;
            const float2 a = reinterpret_cast<const float2*>(x)[i];
            const unsigned long long idx = (unsigned long long)(base + i);
            if (!isfinite(a.x) || !isfinite(a.y)) {
                k = (2ull * idx) * (unsigned long long)channels + (unsigned long long)ch;
            } else if (y) {
                const float2 b = reinterpret_cast<const float2*>(y)[i];
                if (!isfinite(b.x) || !isfinite(b.y))
                    k = (2ull * idx + 1ull) * (unsigned long long)channels + (unsigned long long)ch;
            }
        }
        if (k != ~0ull) atomicMin(key, k);
    };
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; p + 3 * stride < pairs; p += 4 * stride) {
        float4 a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = x[p + u * stride];
        bool bad = nonfinite4(a[0]) | nonfinite4(a[1]) | nonfinite4(a[2]) | nonfinite4(a[3]);
        if (y) {
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = y[p + u * stride];
            bad |= nonfinite4(a[0]) | nonfinite4(a[1]) | nonfinite4(a[2]) | nonfinite4(a[3]);
        }
        if (bad)
            for (int u = 0; u < 4; ++u) slow(p + u * stride);
    }
    for (; p < pairs; p += stride) {
        bool bad = nonfinite4(x[p]);
        if (y) bad |= nonfinite4(y[p]);
        if (bad) slow(p);
    }
}

// channel blockIdx.y: ring row ring + y * ring_pitch, source row src + y * src_pitch
__global__ void ring_write_kernel(float2* ring, int64_t ring_pitch, uint64_t mask, int64_t abs0, const float2* src,
                                  int64_t src_pitch, int64_t n) {
    ring += (size_t)blockIdx.y * ring_pitch;
    src += (size_t)blockIdx.y * src_pitch;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ring[(uint64_t)(abs0 + i) & mask] = src[i];
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace


void launch_add_f64(double* dst, const double* src, int64_t n, cudaStream_t st, const unsigned long long* gate) {
    if (n > 0) add_f64_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, src, n, gate);
}
void launch_accum_frames(const double2* frames, int64_t n_frames, int64_t len, double2* coh, double* mag,
                         cudaStream_t st) {
    if (n_frames > 0 && len > 0) accum_frames_kernel<<<grid_for(len, 256), 256, 0, st>>>(frames, n_frames, len, coh, mag);
}
void launch_recursive_update(double2* frames, int64_t n_frames, int channels, int64_t per, double2* R, double decay,
                             double2* coh, double* mag, cudaStream_t st, double2* host_out) {
    if (n_frames > 0 && per > 0)
        recursive_update_kernel<<<grid_for((int64_t)channels * per, 256), 256, 0, st>>>(frames, n_frames, channels, per,
                                                                                     R, decay, coh, mag, host_out);
}
int launch_finite_check(const float2* x, const float2* y, int64_t n, int64_t base, int channels, int ch,
                        unsigned long long* key, cudaStream_t st, int nch, int64_t pitch) {
    if (n <= 0 || nch <= 0) return 0;
    const bool aligned = ((uintptr_t)x % 16 == 0) && (!y || (uintptr_t)y % 16 == 0) && (nch == 1 || pitch % 2 == 0);
    if (aligned && n >= 2 * 256) {
        const int64_t pairs = n / 2;
        int64_t g = (pairs + 4 * 256 - 1) / (4 * 256);
        g = std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8 / nch));
        finite_check_v4_kernel<<<dim3((unsigned)g, (unsigned)nch), 256, 0, st>>>(
            reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(y), pairs, base, channels, ch, key,
            pitch);
        if (n & 1)
            finite_check_kernel<<<dim3(1, (unsigned)nch), 32, 0, st>>>(x + n - 1, y ? y + n - 1 : nullptr, 1,
                                                                       base + n - 1, channels, ch, key, pitch);
        return (n & 1) ? 2 : 1;
    }
    const int g = std::max(1, std::min(grid_for(n, 256), 148 * 16 / nch));
    finite_check_kernel<<<dim3((unsigned)g, (unsigned)nch), 256, 0, st>>>(x, y, n, base, channels, ch, key, pitch);
    return 1;
}
void launch_ring_write(float2* ring, uint64_t mask, int64_t abs0, const float2* src, int64_t n, cudaStream_t st,
                       int channels, int64_t ring_pitch, int64_t src_pitch) {
    if (n <= 0 || channels <= 0) return;
    const int gx = std::max(1, grid_for(n, 256) / channels);
    ring_write_kernel<<<dim3(gx, channels), 256, 0, st>>>(ring, ring_pitch, mask, abs0, src, src_pitch, n);
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

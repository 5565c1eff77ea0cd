// finalize.cu -- residue folds S_tau[r] -> cyclic ACF tables R(alpha, tau).
//
//   R(alpha_a, tau) = scale * sum_{r < Pf} q_tau[r] * W^{bin_a * r},  W = e^{-j2pi/Pf}
//
// with q built from the four real correlations of fold.cu per flag, and
// bin_a = k_a * (Pf / P) (mod Pf) exact integers, so the phase is anchored to
// absolute sample 0 exactly (the reference's exact-integer bin lead,
// proj/src/kernels.cpp:103-114, generalised to every alpha on the grid).
//
// Two paths, both fp64:
//   * radix-2 DIT FFT in shared memory (Pf a power of two <= 8192; levels
//     fused in pairs, twiddles in shared memory): replaces
//     the reference's per-lag Fft::forward (proj/src/fft.cpp:44-87);
//   * direct DFT with an exact (bin*r mod Pf) twiddle index, for small alpha
//     sets or non-power-of-two periods (proj/src/fft.cpp:89-100 analogue).
#include "kernels.cuh"

namespace cyc {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double2 combine(const double* s, int flag_bit) {  // s: 4 values
    // s = (c0, c1, c2, c3) = (sum xr*yr, sum xi*yr, sum xr*yi, sum xi*yi)
    return flag_bit == 0 ? make_double2(s[0] + s[3], s[1] - s[2])   // x * conj(y)
                         : make_double2(s[0] - s[3], s[1] + s[2]);  // x * y
}

// grid: (n_rows, n_flag_tables); one CTA per (row, flag).  Radix-2 stages are
// executed in pairs: each thread keeps the four points of two consecutive
// butterfly levels in registers (exactly the radix-2 arithmetic, one barrier
// per pair), with the Pf/2-entry twiddle table staged in shared memory.
__global__ void __launch_bounds__(512) finalize_fft_kernel(FinalizeLaunch L, int log2Pf) {
    extern __shared__ double2 buf[];  // Pf points, then Pf/2 twiddles
    __shared__ FinalRow s_row;        // descriptors may be in mapped host memory: read once
    const int Pf = L.Pf;
    double2* tw = buf + Pf;
    if (threadIdx.x == 0) s_row = L.rows[blockIdx.x];
    for (int k = threadIdx.x; k < (Pf >> 1); k += blockDim.x) tw[k] = __ldg(L.tw + k);
    __syncthreads();
    const FinalRow row = s_row;
    const int fi = blockIdx.y;  // index among requested flags
    const int flag_bit = (L.flags == 2) ? 1 : fi;
    const double* Srow = L.S + ((size_t)row.slot * L.t_pad + row.t_span) * (size_t)Pf * 4;
    for (int r = threadIdx.x; r < Pf; r += blockDim.x) {
        const int rev = (int)(__brev((unsigned)r) >> (32 - log2Pf));
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(Srow) + 2 * r);
        const double2 v1 = __ldg(reinterpret_cast<const double2*>(Srow) + 2 * r + 1);
        const double c[4] = {v0.x, v0.y, v1.x, v1.y};
        buf[rev] = combine(c, flag_bit);
    }
    __syncthreads();
    int len = 2;
    for (; 2 * len <= Pf; len <<= 2) {  // levels len (half h) and 2 len, fused
        const int h = len >> 1;
        const int ts1 = Pf / len, ts2 = ts1 >> 1;
        for (int j = threadIdx.x; j < (Pf >> 2); j += blockDim.x) {
            const int grp = j / h, pos = j - grp * h;
            const int i0 = grp * 2 * len + pos;
            double2 a = buf[i0], b = buf[i0 + h], c = buf[i0 + 2 * h], d = buf[i0 + 3 * h];
            const double2 w1 = tw[pos * ts1];
            double2 v = cmul(b, w1);
            b = make_double2(a.x - v.x, a.y - v.y);
            a = make_double2(a.x + v.x, a.y + v.y);
            v = cmul(d, w1);
            d = make_double2(c.x - v.x, c.y - v.y);
            c = make_double2(c.x + v.x, c.y + v.y);
            v = cmul(c, tw[pos * ts2]);
            buf[i0] = make_double2(a.x + v.x, a.y + v.y);
            buf[i0 + 2 * h] = make_double2(a.x - v.x, a.y - v.y);
            v = cmul(d, tw[(pos + h) * ts2]);
            buf[i0 + h] = make_double2(b.x + v.x, b.y + v.y);
            buf[i0 + 3 * h] = make_double2(b.x - v.x, b.y - v.y);
        }
        __syncthreads();
    }
    if (len <= Pf) {  // odd log2 Pf: the last radix-2 level
        const int half = len >> 1;
        for (int j = threadIdx.x; j < (Pf >> 1); j += blockDim.x) {
            const int i0 = j, i1 = j + half;  // a single group of size Pf
            const double2 u = buf[i0];
            const double2 v = cmul(buf[i1], tw[j]);
            buf[i0] = make_double2(u.x + v.x, u.y + v.y);
            buf[i1] = make_double2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
    const double sc = L.row_scale ? L.row_scale[row.out_block] : L.scale_default;
    double2* out = L.out + (size_t)row.out_block * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                   (size_t)row.t_out * L.stride_t;
    for (int a = threadIdx.x; a < L.A; a += blockDim.x) {
        const double2 v = buf[L.bins[a]];
        out[(size_t)a * L.stride_a] = make_double2(v.x * sc, v.y * sc);
    }
}

// Direct DFT: grid (n_rows, n_flag_tables, ceil(A / DFT_AB)); a CTA computes
// DFT_AB alphas of one row with its 256 threads striding over the residues
// (twiddle index advanced exactly mod Pf), then a fixed-order block reduction.
constexpr int DFT_T = 256;
constexpr int DFT_AB = 8;
__global__ void __launch_bounds__(DFT_T) finalize_dft_kernel(FinalizeLaunch L) {
    __shared__ double2 red[DFT_T / 32][DFT_AB];
    __shared__ FinalRow s_row;  // descriptors may be in mapped host memory: read once
    if (threadIdx.x == 0) s_row = L.rows[blockIdx.x];
    __syncthreads();
    const FinalRow row = s_row;
    const int fi = blockIdx.y;
    const int flag_bit = (L.flags == 2) ? 1 : fi;
    const int Pf = L.Pf;
    const int a0 = blockIdx.z * DFT_AB;
    const int na = min(DFT_AB, L.A - a0);
    const double* Srow = L.S + ((size_t)row.slot * L.t_pad + row.t_span) * (size_t)Pf * 4;
    int idx[DFT_AB], step[DFT_AB];
    double re[DFT_AB], im[DFT_AB];
#pragma unroll
    for (int k = 0; k < DFT_AB; ++k) {
        const int64_t bin = k < na ? L.bins[a0 + k] : 0;
        idx[k] = (int)((bin * threadIdx.x) % Pf);
        step[k] = (int)((bin * DFT_T) % Pf);
        re[k] = im[k] = 0.0;
    }
    for (int r = threadIdx.x; r < Pf; r += DFT_T) {
        const double2 v = combine(Srow + (size_t)r * 4, flag_bit);
#pragma unroll
        for (int k = 0; k < DFT_AB; ++k) {
            const double2 w = L.tw[idx[k]];
            re[k] += v.x * w.x - v.y * w.y;
            im[k] += v.x * w.y + v.y * w.x;
            idx[k] += step[k];
            if (idx[k] >= Pf) idx[k] -= Pf;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < DFT_AB; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            re[k] += __shfl_down_sync(0xffffffffu, re[k], o);
            im[k] += __shfl_down_sync(0xffffffffu, im[k], o);
        }
        if (lane == 0) red[warp][k] = make_double2(re[k], im[k]);
    }
    __syncthreads();
    if (threadIdx.x >= na) return;
    const int k = threadIdx.x;
    double sr = 0.0, si = 0.0;
    for (int w = 0; w < DFT_T / 32; ++w) {
        sr += red[w][k].x;
        si += red[w][k].y;
    }
    const double sc = L.row_scale ? L.row_scale[row.out_block] : L.scale_default;
    double2* out = L.out + (size_t)row.out_block * L.out_block_stride + (size_t)fi * L.out_flag_stride +
                   (size_t)row.t_out * L.stride_t;
    out[(size_t)(a0 + k) * L.stride_a] = make_double2(sr * sc, si * sc);
}

}  // namespace

void launch_finalize(const FinalizeLaunch& L, cudaStream_t st) {
    if (L.n_rows == 0) return;
    const int nflag = L.flags == 3 ? 2 : 1;
    if (L.use_fft) {
        int lg = 0;
        while ((1 << lg) < L.Pf) ++lg;
        const size_t smem = (size_t)L.Pf * 3 / 2 * sizeof(double2);
        static std::atomic<uint64_t> attr_set{0};
        if (first_on_device(attr_set))
            cudaFuncSetAttribute(finalize_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 12288 * (int)sizeof(double2));
        finalize_fft_kernel<<<dim3(L.n_rows, nflag), std::min(512, std::max(32, L.Pf / 4)), smem, st>>>(L, lg);
    } else {
        finalize_dft_kernel<<<dim3(L.n_rows, nflag, (L.A + DFT_AB - 1) / DFT_AB), DFT_T, 0, st>>>(L);
    }
}

}  // namespace cyc

namespace cyc {
void prepare_finalize_kernels() {
    static std::atomic<uint64_t> done{0};
    if (!first_on_device(done)) return;
    cudaFuncSetAttribute(finalize_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * (int)sizeof(double2));
}
}  // namespace cyc

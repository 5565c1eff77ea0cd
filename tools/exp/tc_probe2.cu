// tc_probe2.cu -- tensor-core fold building blocks, bf16x3 variant (diagnostics):
//   TMA 2D load (no swizzle) of 16 periods x 256 floats of the record,
//   converter warps split x = hi + lo (bf16 each) into MN-major SW128 planes,
//   three tcgen05.mma.kind::f16 (hi*hi + hi*lo + lo*hi), fp32 accumulator in
//   TMEM, tcgen05.ld epilogue.  A (M=128) = first 128 floats of the B window.
// D[m][n] = sum_k x[k*2Pf + 2*r0 + m] * x[k*2Pf + 2*r0 + n],  m < 128, n < 256
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int KB = 16;                       // periods per stage (= MMA K)
constexpr int NSTG = 5;
constexpr int WIN = 256;                     // floats per period window (N)
constexpr int RAW_BYTES = KB * WIN * 4;      // 16 KB
constexpr int PLANE_BYTES = KB * WIN * 2;    // 8 KB (4 atoms x 16 rows x 128 B)
constexpr int STAGE_BYTES = RAW_BYTES + 2 * PLANE_BYTES;
constexpr int SMEM = NSTG * STAGE_BYTES + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// D f32, A/B bf16, MN-major both, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__global__ void __launch_bounds__(192, 1) tc_probe_kernel(const __grid_constant__ CUtensorMap tmap, int r0, int nper,
                                                          int terms, float* out, int loadmode, const float* gx, int Pf, int distinct) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[NSTG], conv[NSTG], empty[NSTG], done;
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 4);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const int nst = nper / KB;

    if (warp == 0) {
        const int rb = distinct ? (int)(blockIdx.x % 16) * 64 : r0;      // residue block per CTA
        const int pb = distinct ? (int)(blockIdx.x / 16) * nper : 0;      // period block per CTA
        for (int it = 0; it < nst; ++it) {
            const int s = it % NSTG;
            if (it >= NSTG) mbar_wait(&empty[s], ((it / NSTG) - 1) & 1);
            if (lane == 0) mbar_expect_tx(&full[s], RAW_BYTES);
            __syncwarp();
            if (loadmode == 0) {
                if (lane == 0) tma_load_2d(smem + s * STAGE_BYTES, &tmap, 2 * rb, pb + it * KB, &full[s]);
            } else if (lane < 16) {
                const float* src = gx + (size_t)(pb + it * KB + lane) * 2 * Pf + 2 * rb;
                bulk_g2s(smem_u32(smem + s * STAGE_BYTES + lane * 1024), src, 1024, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int it = 0; it < nst; ++it) {
                const int s = it % NSTG;
                mbar_wait(&conv[s], (it / NSTG) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t hi = smem_u32(smem + s * STAGE_BYTES + RAW_BYTES), lo = hi + PLANE_BYTES;
                const uint64_t dbh = umma_desc_sw128(hi, 2048, 1024), dbl = umma_desc_sw128(lo, 2048, 1024);
                // A = the first 2 MN atoms (128 floats) of the same planes
                mma_bf16(tmem, dbh, dbh, IDESC, it ? 1u : 0u);
                if (terms >= 3) {
                    mma_bf16(tmem, dbh, dbl, IDESC, 1u);
                    mma_bf16(tmem, dbl, dbh, IDESC, 1u);
                }
                if (terms >= 4) mma_bf16(tmem, dbl, dbl, IDESC, 1u);
                mma_commit(&empty[s]);
            }
            mma_commit(&done);
        }
    } else {
        const int ct = threadIdx.x - 64;  // 0..127
        for (int it = 0; it < nst; ++it) {
            const int s = it % NSTG;
            mbar_wait(&full[s], (it / NSTG) & 1);
            const uint8_t* raw = smem + s * STAGE_BYTES;
            uint8_t* hi = smem + s * STAGE_BYTES + RAW_BYTES;
            uint8_t* lo = hi + PLANE_BYTES;
            // unit u: row k = u / 32, 8 floats n = 8 * (u % 32) .. +7
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int u = ct + 128 * j;
                const int k = u >> 5, n8 = u & 31;
                const float4 a = *reinterpret_cast<const float4*>(raw + k * 1024 + n8 * 32);
                const float4 b = *reinterpret_cast<const float4*>(raw + k * 1024 + n8 * 32 + 16);
                const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                uint32_t h[4], l[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    h[e] = pack_bf16(v[2 * e], v[2 * e + 1]);
                    const float h0 = __uint_as_float(h[e] << 16), h1 = __uint_as_float(h[e] & 0xffff0000u);
                    l[e] = pack_bf16(v[2 * e] - h0, v[2 * e + 1] - h1);
                }
                // MN-major SW128: atom n/64, row k, 16B chunk ((n%64)/8) ^ (k%8)
                const int atom = n8 >> 3, chunk = (n8 & 7) ^ (k & 7);
                const int off = atom * 2048 + k * 128 + chunk * 16;
                *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
        }
        mbar_wait(&done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int q = warp & 3;
        const int row = 32 * q + lane;
        for (int c = 0; c < 256; c += 32) {
            uint32_t v[32];
            const uint32_t addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (out)
                for (int j = 0; j < 32; ++j) out[row * 256 + c + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int Pf = 1024, P = argc > 1 ? atoi(argv[1]) : 256;
    const size_t nf = (size_t)P * 2 * Pf;
    std::vector<float> h(nf);
    std::mt19937 g(1);
    std::normal_distribution<float> nd(0.f, 1.f);
    for (auto& v : h) v = nd(g);
    float *dx, *dout;
    CK(cudaMalloc(&dx, nf * 4));
    CK(cudaMemcpy(dx, h.data(), nf * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dout, 128 * 256 * 4));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tmap;
    cuuint64_t gdim[2] = {(cuuint64_t)2 * Pf, (cuuint64_t)P};
    cuuint64_t gstr[1] = {(cuuint64_t)2 * Pf * 4};
    cuuint32_t box[2] = {WIN, KB}, es[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    CK(cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    std::vector<float> out(128 * 256);
    const int r0 = 64 * 3;
    for (int terms : {1, 3, 4}) {
        tc_probe_kernel<<<1, 192, SMEM>>>(tmap, r0, P, terms, dout, 0, dx, Pf, 0);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
        double emax = 0, ref = 0, se = 0, sr = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 256; ++n) {
                double s = 0;
                for (int k = 0; k < P; ++k)
                    s += (double)h[(size_t)k * 2 * Pf + 2 * r0 + m] * h[(size_t)k * 2 * Pf + 2 * r0 + n];
                const double o = out[m * 256 + n];
                emax = fmax(emax, fabs(o - s));
                ref = fmax(ref, fabs(s));
                se += (o - s) * (o - s);
                sr += s * s;
            }
        printf("terms %d: max|D-exact| %.3e  rel L2 %.3e  (max|D| %.3e, K=%d)  D[0][0]=%.4f D[5][130]=%.4f\n", terms, emax,
               sqrt(se / sr), ref, P, out[0], out[5 * 256 + 130]);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // streaming test: 144 CTAs, distinct (residue block, period block) per CTA, 16 x 9 grid
    {
        const int per_cta = P / 9 / KB * KB;
        for (int lm = 0; lm < 2; ++lm) {
            tc_probe_kernel<<<144, 192, SMEM>>>(tmap, 0, per_cta, 3, nullptr, lm, dx, Pf, 1);
            cudaEventRecord(e0);
            for (int i = 0; i < 10; ++i) tc_probe_kernel<<<144, 192, SMEM>>>(tmap, 0, per_cta, 3, nullptr, lm, dx, Pf, 1);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double useful = 144.0 * 64 * 64 * 4 * 2 * per_cta;
            printf("%s, 144 CTAs x %d periods (distinct data, %.0f MB): %.3f ms/launch, useful %.1f TFLOP/s\n",
                   lm ? "16x 1-D bulk (lanes)" : "2-D TMA", per_cta, 144.0 * per_cta * 1024 / 1e6, ms / 10,
                   useful / (ms / 10 * 1e-3) / 1e12);
        }
    }
    return 0;
}

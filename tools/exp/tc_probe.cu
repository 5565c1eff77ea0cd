// tc_probe.cu -- standalone validation of the tensor-core fold building blocks
// (diagnostics, not part of the library):
//   TMA 2D loads (128B swizzle) of a period-major complex record, in-smem
//   split x = hi + lo (hi = x with the low 13 mantissa bits cleared), three
//   tcgen05.mma.kind::tf32 (hi*hi + hi*lo + lo*hi) with MN-major operands,
//   fp32 accumulator in TMEM, tcgen05.ld epilogue.
// D[m][n] = sum_k A[m][k] B[n][k],  A[m][k] = y_float[k*2Pf + 2*r0 + m]  (m < 128)
//                                   B[n][k] = x_float[k*2Pf + 2*r0 + n]  (n < 256)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_probe.cu -o tc_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int KB = 16;        // periods per stage
constexpr int NSTG = 4;
constexpr int NA = 4, NB = 8;  // 32-float atoms in A (M=128) and B (N=256)
constexpr int ATOM_BYTES = KB * 128;              // one atom column: 16 rows x 128 B
constexpr int A_BYTES = NA * ATOM_BYTES;          // 8 KB
constexpr int B_BYTES = NB * ATOM_BYTES;          // 16 KB
constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // raw/hi + lo for A and B
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
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
// UMMA shared-memory descriptor: MN-major, 128B swizzle (CUTLASS UMMA::SmemDescriptor layout)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (sm100)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// instruction descriptor: D f32, A/B tf32, both MN-major, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__global__ void __launch_bounds__(192, 1) tc_probe_kernel(const __grid_constant__ CUtensorMap tmap, int r0, int nper,
                                                          int mode, float* out, float* dbg) {
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
        if (lane == 0) {
            for (int it = 0; it < nst; ++it) {
                const int s = it % NSTG;
                if (it >= NSTG) mbar_wait(&empty[s], ((it / NSTG) - 1) & 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                const int row = it * KB;
                for (int a = 0; a < NA; ++a) tma_load_2d(st + a * ATOM_BYTES, &tmap, 2 * r0 + 32 * a, row, &full[s]);
                for (int a = 0; a < NB; ++a)
                    tma_load_2d(st + 2 * A_BYTES + a * ATOM_BYTES, &tmap, 2 * r0 + 32 * a, row, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int it = 0; it < nst; ++it) {
                const int s = it % NSTG;
                mbar_wait(&conv[s], (it / NSTG) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES, b_lo = st + 2 * A_BYTES + B_BYTES;
                for (int g = 0; g < KB / 8; ++g) {
                    const uint32_t ko = g * 1024;
                    const uint64_t dah = umma_desc(a_hi + ko, ATOM_BYTES, 1024), dal = umma_desc(a_lo + ko, ATOM_BYTES, 1024);
                    const uint64_t dbh = umma_desc(b_hi + ko, ATOM_BYTES, 1024), dbl = umma_desc(b_lo + ko, ATOM_BYTES, 1024);
                    mma_tf32(tmem, dah, dbh, IDESC, (it | g) ? 1u : 0u);
                    if (mode == 0) {
                        mma_tf32(tmem, dah, dbl, IDESC, 1u);
                        mma_tf32(tmem, dal, dbh, IDESC, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(&done);
        }
    } else {
        // converters: x -> hi (in place, low 13 mantissa bits cleared), lo = x - hi
        const int ct = threadIdx.x - 64;  // 0..127
        for (int it = 0; it < nst; ++it) {
            const int s = it % NSTG;
            mbar_wait(&full[s], (it / NSTG) & 1);
            uint8_t* st = smem + s * STAGE_BYTES;
            if (it == 0 && dbg) for (int i = ct; i < (A_BYTES + B_BYTES) / 4; i += 128) dbg[i] = ((float*)st)[i < A_BYTES / 4 ? i : i + A_BYTES / 4];
            if (mode == 0) {
                float4* ah = (float4*)st;
                float4* al = (float4*)(st + A_BYTES);
                float4* bh = (float4*)(st + 2 * A_BYTES);
                float4* bl = (float4*)(st + 2 * A_BYTES + B_BYTES);
                auto split = [](float4 v, float4& h, float4& l) {
                    h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
                    h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
                    h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
                    h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
                    l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
                };
                for (int i = ct; i < A_BYTES / 16; i += 128) { float4 h, l; split(ah[i], h, l); ah[i] = h; al[i] = l; }
                for (int i = ct; i < B_BYTES / 16; i += 128) { float4 h, l; split(bh[i], h, l); bh[i] = h; bl[i] = l; }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
        }
        // epilogue: TMEM lanes 32*(warp%4) .. +31
        mbar_wait(&done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (mode == 2) {
            const uint32_t a2 = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            uint32_t w = __float_as_uint(1000.f + 32 * (warp & 3) + lane);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a2), "r"(w));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
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

static float trunc13(float v) { uint32_t u; memcpy(&u, &v, 4); u &= 0xffffe000u; float r; memcpy(&r, &u, 4); return r; }
static float rne13(float v) { uint32_t u; memcpy(&u, &v, 4); u = (u + 0xfffu + ((u >> 13) & 1)) & 0xffffe000u; float r; memcpy(&r, &u, 4); return r; }

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
    float* ddbg;
    CK(cudaMalloc(&ddbg, 65536 * 4));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tmap;
    cuuint64_t gdim[2] = {(cuuint64_t)2 * Pf, (cuuint64_t)P};
    cuuint64_t gstr[1] = {(cuuint64_t)2 * Pf * 4};
    cuuint32_t box[2] = {32, KB}, es[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    CK(cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    std::vector<float> out(128 * 256);
    for (int mode = 0; mode < 3; ++mode) {
        const int r0 = 64 * 3;
        tc_probe_kernel<<<1, 192, SMEM>>>(tmap, r0, P, mode, dout, mode == 0 ? ddbg : nullptr);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
        double emax = 0, ref = 0, et = 0, er = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 256; ++n) {
                double s = 0, st = 0, sr = 0;
                for (int k = 0; k < P; ++k) {
                    const float a = h[(size_t)k * 2 * Pf + 2 * r0 + m], b = h[(size_t)k * 2 * Pf + 2 * r0 + n];
                    s += (double)a * b;
                    st += (double)trunc13(a) * trunc13(b);
                    sr += (double)rne13(a) * rne13(b);
                }
                const double o = out[m * 256 + n];
                emax = fmax(emax, fabs(o - s));
                et = fmax(et, fabs(o - st));
                er = fmax(er, fabs(o - sr));
                ref = fmax(ref, fabs(s));
            }
        if (mode == 0) {
            std::vector<float> db((A_BYTES + B_BYTES) / 4);
            CK(cudaMemcpy(db.data(), ddbg, db.size() * 4, cudaMemcpyDeviceToHost));
            printf("  smem A row0 (swizzled) first 8: ");
            for (int i = 0; i < 8; ++i) printf("%.4f ", db[i]);
            printf("\n  global y[k=0][2r0..]: ");
            for (int i = 0; i < 8; ++i) printf("%.4f ", h[2 * r0 + i]);
            printf("\n  smem B row0 first 8: ");
            for (int i = 0; i < 8; ++i) printf("%.4f ", db[A_BYTES / 4 + i]);
            printf("\n");
        }
        if (mode == 2) { printf("  tmem st/ld: out[0][0]=%.1f out[33][0]=%.1f out[100][0]=%.1f\n", out[0], out[33 * 256], out[100 * 256]); continue; }
        {
            const int pts[6][2] = {{0, 0}, {1, 0}, {0, 1}, {5, 7}, {64, 130}, {127, 255}};
            for (auto& pt : pts) {
                double s = 0;
                for (int k = 0; k < P; ++k)
                    s += (double)h[(size_t)k * 2 * Pf + 2 * r0 + pt[0]] * h[(size_t)k * 2 * Pf + 2 * r0 + pt[1]];
                printf("  D[%d][%d] got %.5f want %.5f\n", pt[0], pt[1], out[pt[0] * 256 + pt[1]], s);
            }
            // find where 'want' values appear in out (layout probe)
            double s00 = 0;
            for (int k = 0; k < P; ++k) s00 += (double)h[(size_t)k * 2 * Pf + 2 * r0] * h[(size_t)k * 2 * Pf + 2 * r0 + 1];
            for (int i = 0; i < 128 * 256; ++i)
                if (fabs(out[i] - s00) < 1e-3 * fabs(s00) + 1e-3) { printf("  D[0][1] value found at out[%d] (row %d col %d)\n", i, i / 256, i % 256); break; }
            int nz = 0; for (float v : out) nz += v != 0.f;
            printf("  nonzero outputs %d of %d\n", nz, 128 * 256);
        }
        printf("mode %d (%s): max|D-exact| %.3e  max|D-trunc13| %.3e  max|D-rne13| %.3e  (max|D| %.3e, K=%d)\n", mode,
               mode ? "raw single MMA" : "3xTF32", emax, et, er, ref, P);
    }
    // timing of the 3xTF32 path on one CTA
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) tc_probe_kernel<<<148, 192, SMEM>>>(tmap, 0, P, 0, dout, nullptr);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double useful = 148.0 * 64 * 64 * 4 * 2 * P;  // 64 res x 64 lags x 4 FMA x 2 flop per period
    printf("148 CTAs x %d periods: %.3f ms/launch, useful %.1f TFLOP/s (3 MMAs N=256 M=128 per 8 periods)\n", P, ms / 10,
           useful / (ms / 10 * 1e-3) / 1e12);
    return 0;
}

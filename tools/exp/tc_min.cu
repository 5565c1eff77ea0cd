// Minimal tcgen05 tf32 MMA test: constant operands, one MMA, read D.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t version) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)version << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__global__ void k(float* out, uint32_t idesc, uint32_t layout, uint32_t lbo, uint32_t sbo, uint32_t version, int fillmode, int kind, int style) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t done;
    __shared__ uint32_t tb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* f = (float*)sm;
    if (kind == 0) for (int i = threadIdx.x; i < 24576 / 4; i += blockDim.x) f[i] = fillmode == 0 ? 1.0f : (float)((i % 7) + 1);
    else for (int i = threadIdx.x; i < 24576 / 4; i += blockDim.x) ((uint32_t*)f)[i] = 0x3F803F80u;  // bf16 pairs of 1.0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) { mbar_init(&done, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tb;
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
    const uint64_t da = desc(a, lbo, sbo, layout, version), db = desc(b, lbo, sbo, layout, version);
    bool issue;
    if (style == 0) issue = threadIdx.x == 0;
    else {
        uint32_t pred = 0;
        if (warp == 0) asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        issue = pred != 0;
    }
    if (issue) {
        if (kind == 0)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u));
        else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done)) : "memory");
    }
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[4];
    const uint32_t addr = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(32 * (warp & 3) + lane) * 4 + j] = __uint_as_float(v[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
int main(int argc, char** argv) {
    const int which = atoi(argv[1]);
    float* d; cudaMalloc(&d, 128 * 4 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    float h[512];
    struct Case { const char* name; uint32_t idesc, layout, lbo, sbo, version; int kind, style; };
    const uint32_t tf = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t bf = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t MN = (1u << 15) | (1u << 16);
    Case cs[] = {
        {"tf32 MN SW128 thread0", tf | MN, 2, 2048, 1024, 1, 0, 0},
        {"tf32 MN SW128 elect  ", tf | MN, 2, 2048, 1024, 1, 0, 1},
        {"bf16 MN SW128 elect  ", bf | MN, 2, 2048, 1024, 1, 1, 1},
        {"bf16 K  SW128 elect  ", bf, 2, 16, 1024, 1, 1, 1},
        {"tf32 K  SW128 elect  ", tf, 2, 16, 1024, 1, 0, 1},
        {"tf32 MN SW128 elect m64", ((1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((64u >> 4) << 24)) | MN, 2, 2048, 1024, 1, 0, 1},
        {"tf32 MN SW128_BASE32B elect", tf | MN, 1, 2048, 1024, 1, 0, 1},
        {"tf32 MN SW128_BASE32B lbo1k sbo512", tf | MN, 1, 1024, 512, 1, 0, 1},
        {"tf32 MN SW128 elect n64", ((1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24)) | MN, 2, 2048, 1024, 1, 0, 1},
    };
    auto& c = cs[which];
    cudaMemset(d, 0, 2048);
    k<<<1, 128, 32768>>>(d, c.idesc, c.layout, c.lbo, c.sbo, c.version, 0, c.kind, c.style);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 2048, cudaMemcpyDeviceToHost);
    printf("%s: err=%s D[0][0..3]=%.1f %.1f %.1f %.1f D[127][0]=%.1f\n", c.name, cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[127 * 4]);
    return 0;
}

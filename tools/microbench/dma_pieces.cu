// H2D throughput of a 128 MiB pinned buffer copied in k pieces (1D and 2D copies).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    size_t nb = 128ull << 20;
    void *h, *d;
    cudaMallocHost(&h, nb);
    cudaMalloc(&d, nb);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int k : {1, 4, 8, 16, 32, 64}) {
        for (int twod = 0; twod < 2; ++twod) {
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0, s);
                size_t piece = nb / k;
                for (int i = 0; i < k; ++i) {
                    char* dd = (char*)d + i * piece;
                    char* hh = (char*)h + i * piece;
                    if (twod) cudaMemcpy2DAsync(dd, piece, hh, piece, piece, 1, cudaMemcpyHostToDevice, s);
                    else cudaMemcpyAsync(dd, hh, piece, cudaMemcpyHostToDevice, s);
                }
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("{\"pieces\":%d,\"2d\":%d,\"ms\":%.3f,\"GBps\":%.1f}\n", k, twod, best, nb / best / 1e6);
        }
    }
    return 0;
}

// Host screen/copy rate per 64 KB chunk over a cold 2 GB buffer (diagnostics for the small-push path)
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <vector>
__attribute__((target("avx2"))) uint32_t screen(const uint32_t* s, size_t m) {
    const __m256i em = _mm256_set1_epi32(0x7f800000);
    __m256i a0 = _mm256_setzero_si256(), a1 = a0;
    for (size_t i = 0; i < m; i += 16) {
        __m256i v0 = _mm256_loadu_si256((const __m256i*)(s + i)), v1 = _mm256_loadu_si256((const __m256i*)(s + i + 8));
        a0 = _mm256_or_si256(a0, _mm256_cmpeq_epi32(_mm256_and_si256(v0, em), em));
        a1 = _mm256_or_si256(a1, _mm256_cmpeq_epi32(_mm256_and_si256(v1, em), em));
    }
    a0 = _mm256_or_si256(a0, a1);
    return !_mm256_testz_si256(a0, a0);
}
__attribute__((target("avx2"))) uint32_t copy_screen(uint32_t* d, const uint32_t* s, size_t m) {
    const __m256i em = _mm256_set1_epi32(0x7f800000);
    __m256i va = _mm256_setzero_si256();
    for (size_t i = 0; i < m; i += 8) {
        const __m256i v = _mm256_loadu_si256((const __m256i*)(s + i));
        va = _mm256_or_si256(va, _mm256_cmpeq_epi32(_mm256_and_si256(v, em), em));
        _mm256_stream_si256((__m256i*)(d + i), v);
    }
    _mm_sfence();
    return !_mm256_testz_si256(va, va);
}
int main() {
    const size_t N = (size_t)1 << 29;  // 2 GB of floats... words
    uint32_t* buf = (uint32_t*)aligned_alloc(64, N * 4);
    for (size_t i = 0; i < N; ++i) buf[i] = (uint32_t)i * 2654435761u & 0x3fffffff;
    uint32_t* st = (uint32_t*)aligned_alloc(64, 1 << 20);
    const size_t m = 16384;  // 8192 complex
    for (int mode = 0; mode < 3; ++mode) {
        auto t0 = std::chrono::steady_clock::now();
        uint32_t acc = 0;
        size_t cnt = 0;
        for (size_t off = 0; off + m <= N; off += m, ++cnt) {
            if (mode == 0) acc |= screen(buf + off, m);
            else if (mode == 1) acc |= copy_screen(st + (cnt & 1) * m, buf + off, m);
            else { memcpy(st + (cnt & 1) * m, buf + off, m * 4); acc |= st[5]; }
        }
        double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        printf("mode %d: %.2f us per 64 KB (%.1f GB/s) acc=%u\n", mode, us / cnt, cnt * m * 4 / us / 1e3, acc);
    }
}

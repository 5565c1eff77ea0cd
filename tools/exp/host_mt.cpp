// Multi-threaded copy+screen of 64 KB / 32 KB chunks from a cold 2 GB buffer
// into a pinned-like staging buffer: spinning helper threads, per-chunk
// dispatch through an atomic sequence (diagnostics for the small-push path).
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <thread>
#include <vector>
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
struct alignas(64) Slot { std::atomic<uint64_t> seq{0}; std::atomic<uint64_t> done{0}; };
const uint32_t* g_src; uint32_t* g_dst; size_t g_m; int g_nt;
Slot slots[16];
std::atomic<bool> quit{false};
void worker(int id) {
    uint64_t seen = 0;
    while (!quit.load(std::memory_order_relaxed)) {
        uint64_t s = slots[id].seq.load(std::memory_order_acquire);
        if (s == seen) { _mm_pause(); continue; }
        seen = s;
        const size_t part = g_m / g_nt;
        copy_screen(g_dst + id * part, g_src + id * part, part);
        slots[id].done.store(s, std::memory_order_release);
    }
}
int main() {
    const size_t N = (size_t)1 << 29;
    uint32_t* buf = (uint32_t*)aligned_alloc(64, N * 4);
    for (size_t i = 0; i < N; ++i) buf[i] = (uint32_t)i * 2654435761u & 0x3fffffff;
    uint32_t* st = (uint32_t*)aligned_alloc(64, 4 << 20);
    for (size_t m : {16384ul, 8192ul}) {
        for (int nt : {1, 2, 4, 8}) {
            g_nt = nt; g_m = m;
            quit = false;
            std::vector<std::thread> th;
            for (int i = 1; i < nt; ++i) th.emplace_back(worker, i);
            uint64_t seq = 0;
            auto t0 = std::chrono::steady_clock::now();
            size_t cnt = 0;
            for (size_t off = 0; off + m <= N; off += m, ++cnt) {
                g_src = buf + off; g_dst = st + (cnt & 63) * m;
                ++seq;
                for (int i = 1; i < nt; ++i) slots[i].seq.store(seq, std::memory_order_release);
                copy_screen(g_dst, g_src, m / nt);
                for (int i = 1; i < nt; ++i) while (slots[i].done.load(std::memory_order_acquire) != seq) _mm_pause();
            }
            double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            quit = true;
            for (auto& t : th) t.join();
            printf("chunk %zu KB threads %d: %.2f us per chunk (%.1f GB/s)\n", m * 4 / 1024, nt, us / cnt, cnt * m * 4 / us / 1e3);
        }
    }
}

// hostpool.cpp -- see hostpool.h.
#include "hostpool.h"

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace cyc {
namespace {

inline void cpu_relax() {
#if defined(__x86_64__)
    _mm_pause();
#endif
}

uint32_t copy_screen_scalar(uint32_t* d, const uint32_t* s, size_t m) {
    uint32_t acc = 0;
    for (size_t i = 0; i < m; ++i) {
        const uint32_t w = s[i];
        d[i] = w;
        acc |= (uint32_t)((w & 0x7f800000u) == 0x7f800000u);
    }
    return acc;
}

#if defined(__x86_64__)
// Non-temporal stores skip the read-for-ownership of the staging lines (a third
// of the memory traffic of a cached copy).
__attribute__((target("avx2"))) uint32_t copy_screen_avx2(uint32_t* d, const uint32_t* s, size_t m) {
    uint32_t acc = 0;
    const size_t head = ((32 - ((uintptr_t)d & 31)) & 31) / 4;
    if (((uintptr_t)d & 3) != 0 || head > m) return copy_screen_scalar(d, s, m);
    acc |= copy_screen_scalar(d, s, head);
    size_t i = head;
    const __m256i em = _mm256_set1_epi32(0x7f800000);
    __m256i va = _mm256_setzero_si256();
    for (; i + 8 <= m; i += 8) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        va = _mm256_or_si256(va, _mm256_cmpeq_epi32(_mm256_and_si256(v, em), em));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), v);
    }
    _mm_sfence();  // the NT stores are visible before the DMA / kernel is queued
    acc |= copy_screen_scalar(d + i, s + i, m - i);
    return acc | (uint32_t)!_mm256_testz_si256(va, va);
}
#endif

uint32_t copy_screen_one(uint32_t* d, const uint32_t* s, size_t m) {
#if defined(__x86_64__)
    static const bool avx2 = __builtin_cpu_supports("avx2") && std::getenv("CYC_NO_NT_COPY") == nullptr;
    if (avx2 && m >= 64) return copy_screen_avx2(d, s, m);
#endif
    return copy_screen_scalar(d, s, m);
}

// Helpers spin on a job sequence number for a while after each job (a stream of
// pushes keeps them hot: dispatch costs ~0.2 us), then park on a condition
// variable so an idle process burns no cores.
class Pool {
public:
    static Pool* get() {
        static Pool* p = [] {
            int n = (int)std::thread::hardware_concurrency() - 1;
            n = n < 3 ? n : 3;
            if (const char* e = std::getenv("CYC_COPY_THREADS")) n = std::atoi(e);  // helpers (0: off)
            return n > 0 ? new Pool(n) : nullptr;  // lives for the process
        }();
        return p;
    }

    // false: busy (another thread is dispatching) -- the caller copies alone
    bool run(uint32_t* d, const uint32_t* s, size_t m, uint32_t* flag) {
        std::unique_lock<std::mutex> own(dispatch_, std::try_to_lock);
        if (!own.owns_lock()) return false;
        const int parts = n_ + 1;
        // part boundaries on 64-byte multiples keep the destination alignment
        size_t per = (m / parts) & ~(size_t)15;
        d_ = d;
        s_ = s;
        m_ = m;
        per_ = per;
        const uint64_t seq = ++seq_host_;
        seq_.store(seq, std::memory_order_seq_cst);
        if (sleepers_.load(std::memory_order_seq_cst) > 0) {
            std::lock_guard<std::mutex> lk(mu_);
            cv_.notify_all();
        }
        // the caller takes the last part (the remainder)
        uint32_t acc = copy_screen_one(d + (size_t)n_ * per, s + (size_t)n_ * per, m - (size_t)n_ * per);
        for (int i = 0; i < n_; ++i) {
            while (slot_[i].done.load(std::memory_order_acquire) != seq) cpu_relax();
            acc |= slot_[i].flag;
        }
        *flag = acc;
        return true;
    }

private:
    struct alignas(64) Slot {
        std::atomic<uint64_t> done{0};
        uint32_t flag = 0;
    };

    explicit Pool(int n) : n_(n), slot_(new Slot[n]) {
        for (int i = 0; i < n; ++i) std::thread([this, i] { worker(i); }).detach();
    }

    void worker(int id) {
        uint64_t seen = 0;
        for (;;) {
            auto t0 = std::chrono::steady_clock::now();
            uint64_t s;
            unsigned it = 0;
            while ((s = seq_.load(std::memory_order_acquire)) == seen) {
                cpu_relax();
                if ((++it & 4095) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(5)) {
                    std::unique_lock<std::mutex> lk(mu_);
                    sleepers_.fetch_add(1, std::memory_order_seq_cst);
                    cv_.wait(lk, [&] { return seq_.load(std::memory_order_seq_cst) != seen; });
                    sleepers_.fetch_sub(1, std::memory_order_seq_cst);
                    t0 = std::chrono::steady_clock::now();
                }
            }
            seen = s;
            const size_t off = (size_t)id * per_;
            slot_[id].flag = copy_screen_one(d_ + off, s_ + off, per_);
            slot_[id].done.store(s, std::memory_order_release);
        }
    }

    const int n_;
    Slot* slot_;
    std::mutex dispatch_, mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> seq_{0};
    std::atomic<int> sleepers_{0};
    uint64_t seq_host_ = 0;
    uint32_t* d_ = nullptr;
    const uint32_t* s_ = nullptr;
    size_t m_ = 0, per_ = 0;
};

}  // namespace

uint32_t copy_screen_words(uint32_t* d, const uint32_t* s, size_t m) {
    // below ~32 KB one core is as fast as a dispatch
    if (m >= 8192) {
        if (Pool* p = Pool::get()) {
            uint32_t flag = 0;
            if (p->run(d, s, m, &flag)) return flag;
        }
    }
    return copy_screen_one(d, s, m);
}

}  // namespace cyc

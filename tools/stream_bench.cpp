// stream_bench.cpp -- the reference's streaming call pattern through the C-ABI,
// for the small-call configurations (BASELINE C1: 4096-sample pushes into two
// Set-mode estimators; C3: 8192-sample work() calls into the recursive
// estimator).  A C++ caller (e.g. a GNU Radio block) has no Python overhead, so
// this is what bench.py times for those configs.
//
//   stream_bench c1|c3 <record.cf32> <steps> <warmup>
// prints one JSON object: ms_per_step (CUDA events on the estimator stream),
// frames, launches.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cycb200.h"

namespace {

struct Sink {
    std::vector<cyc_cf64> last;  // consumer: keep the latest frame of each flag
    uint64_t frames = 0;
};

int sink_fn(void* user, const cyc_frame_view* v) {
    Sink* s = static_cast<Sink*>(user);
    s->last.assign(v->values, v->values + v->len);
    ++s->frames;
    return 0;
}

cyc_est* make(int mode, int conj, int win, const std::vector<double>& alphas, int sym, int max_lag,
              const std::vector<int>& lags, double lam, int flags = 0) {
    cyc_config c;
    cyc_config_init(&c);
    c.mode = mode;
    c.conj = conj;
    c.flags = flags;
    c.win_len = win;
    c.alphas = alphas.data();
    c.num_alphas = alphas.size();
    c.lag_symmetric = sym;
    c.max_lag = max_lag;
    c.lags = lags.empty() ? nullptr : lags.data();
    c.num_lags = lags.size();
    c.lambda = lam;
    cyc_est* e = nullptr;
    char err[1024];
    if (cyc_create(&c, &e, err, sizeof err)) {
        std::fprintf(stderr, "create: %s\n", err);
        std::exit(2);
    }
    return e;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: stream_bench c1|c3 record.cf32 steps warmup\n");
        return 1;
    }
    const std::string cfg = argv[1];
    const int steps = std::atoi(argv[3]), warmup = std::atoi(argv[4]);
    FILE* f = std::fopen(argv[2], "rb");
    if (!f) return 1;
    std::fseek(f, 0, SEEK_END);
    const size_t n = (size_t)std::ftell(f) / sizeof(cyc_cf32);
    std::fseek(f, 0, SEEK_SET);
    cyc_cf32* x = static_cast<cyc_cf32*>(cyc_host_alloc(n * sizeof(cyc_cf32)));
    if (std::fread(x, sizeof(cyc_cf32), n, f) != n) return 1;
    std::fclose(f);

    std::vector<cyc_est*> ests;
    size_t chunk = 0;
    if (cfg == "c1" || cfg == "c1x2") {
        std::vector<double> conv, conj;
        for (int k = -2; k <= 2; ++k) {
            conv.push_back(k / 8.0);
            conj.push_back(0.1 + k / 16.0);
        }
        if (cfg == "c1x2") {  // the reference's arrangement: one estimator per function
            ests.push_back(make(CYC_MODE_SET, 0, 4096, conv, 1, 15, {}, 0.0));
            ests.push_back(make(CYC_MODE_SET, 1, 4096, conj, 1, 15, {}, 0.0));
        } else {  // one pass: union alpha set, both functions (flags = BOTH)
            std::vector<double> al(conv);
            al.insert(al.end(), conj.begin(), conj.end());
            ests.push_back(make(CYC_MODE_SET, 0, 4096, al, 1, 15, {}, 0.0, CYC_FLAG_BOTH));
        }
        chunk = 4096;
    } else {
        std::vector<double> al;
        for (int m = -128; m < 128; ++m) al.push_back(m / 1024.0);
        std::vector<int> lags;
        for (int t = 0; t < 32; ++t) lags.push_back(t);
        ests.push_back(make(CYC_MODE_RECURSIVE, 0, 65536, al, 0, 0, lags, 1.0 - 1.0 / 4096.0));
        chunk = 8192;
    }
    // CYC_EMIT_PIPELINE=0: the reference's synchronous push() (frames delivered
    // by the push that completes them); default: up to two emissions in flight
    const char* pe = std::getenv("CYC_EMIT_PIPELINE");
    const int depth = pe ? std::atoi(pe) : 2;
    for (auto* e : ests) cyc_set_emit_pipeline(e, depth);
    Sink sink;
    auto step = [&]() {
        for (auto* e : ests) cyc_reset(e);
        for (size_t off = 0; off < n; off += chunk) {
            const size_t len = std::min(chunk, n - off);
            for (auto* e : ests) {
                const int rc = cyc_push(e, x + off, nullptr, len, sink_fn, &sink);
                if (rc) {
                    std::fprintf(stderr, "push: %s\n", cyc_last_error(e));
                    std::exit(3);
                }
            }
        }
        for (auto* e : ests) {
            cyc_flush_frames(e, sink_fn, &sink);
            cyc_synchronize(e);
        }
    };
    for (int i = 0; i < warmup; ++i) step();
    cudaStream_t st = static_cast<cudaStream_t>(cyc_stream(ests[0]));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint64_t l0 = cyc_kernel_launches(ests[0]) + (ests.size() > 1 ? cyc_kernel_launches(ests[1]) : 0);
    const uint64_t f0 = sink.frames;
    cudaEventRecord(e0, st);
    for (int i = 0; i < steps; ++i) step();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const uint64_t l1 = cyc_kernel_launches(ests[0]) + (ests.size() > 1 ? cyc_kernel_launches(ests[1]) : 0);
    std::printf("{\"ms_per_step\": %.4f, \"frames_per_step\": %llu, \"launches_per_step\": %.1f, \"samples\": %zu}\n",
                ms / steps, (unsigned long long)((sink.frames - f0) / steps), (double)(l1 - l0) / steps, n);
    for (auto* e : ests) cyc_destroy(e);
    cyc_host_free(x);
    return 0;
}

// C++ drop-in check: reference test cases (proj/tests/test_estimator.cpp)
// rewritten against include/cycstat_b200.hpp -- the same calls a reference
// caller makes, with the north-star tolerance in place of fp64's 1e-12.
// Exit code = number of failed checks.
#define CYCSTAT_B200_AS_CYCSTAT
#include "cycstat_b200.hpp"

#include <cmath>
#include <cstdio>
#include <random>

using namespace cycstat;

static int g_fail = 0;
#define CHECK(c)                                                         \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
            ++g_fail;                                                    \
        }                                                                \
    } while (0)

static std::vector<cx> random_stream(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> d(0.0, 1.0);
    std::vector<cx> v(n);
    for (auto& s : v) s = cx((float)d(gen), (float)d(gen));  // float-exact samples
    return v;
}

static EstimatorConfig set_cfg(int n, int m, std::vector<double> a, bool conj = false) {
    EstimatorConfig c;
    c.mode = Mode::Set;
    c.conj = conj;
    c.win_len = n;
    c.alphas = std::move(a);
    c.lag_spec = LagSpec::Symmetric(m);
    return c;
}

static cx direct(const std::vector<cx>& x, const std::vector<cx>& y, double alpha, int m, bool conj, std::size_t k0,
                 int N) {
    cx acc(0, 0);
    for (int n = 0; n < N; ++n) {
        const cx xs = x[k0 + n + m], ys = y[k0 + n];
        acc += (conj ? xs * ys : xs * std::conj(ys)) * std::polar(1.0, -2 * M_PI * alpha * (double)(k0 + n));
    }
    return acc / (double)N;
}

int main() {
    // buffer need (test_estimator.cpp:60-68)
    CHECK(CyclicCorrelator(set_cfg(8, 2, {0.125})).buffer_need() == 12);
    // ConfigError with the violation list (test_estimator.cpp:70-79)
    try {
        CyclicCorrelator e(set_cfg(8, 2, {}));
        CHECK(false);
    } catch (const ConfigError& e) {
        CHECK(std::string(e.what()).find("invalid config") != std::string::npos);
        CHECK(!e.violations.empty());
    }
    // NaN rejection, state unchanged (test_estimator.cpp:126-140)
    {
        CyclicCorrelator est(set_cfg(8, 1, {0.0}));
        const auto good = random_stream(4, 1);
        try {
            est.push(good, random_stream(3, 2));
            CHECK(false);
        } catch (const UsageError&) {
        }
        auto poisoned = random_stream(4, 3);
        poisoned[2] = cx(std::nan(""), 0.0);
        CHECK(est.push(good, good).empty());
        try {
            est.push(poisoned, poisoned);
            CHECK(false);
        } catch (const DataError& e) {
            CHECK(std::string(e.what()).find("index 6") != std::string::npos);
        }
        CHECK(est.consumed() == 4);
        const auto x = random_stream(32, 4);
        CHECK(!est.push(x, x).empty());
    }
    // Set windows vs the literal sum, x != y, both flags (test_estimator.cpp:211-229)
    {
        const auto x = random_stream(400, 1234), y = random_stream(400, 4321);
        const std::vector<double> alphas = {3.0 / 64.0, 0.0, -0.21};
        for (bool conj : {false, true}) {
            CyclicCorrelator est(set_cfg(64, 3, alphas, conj));
            const auto frames = est.push(x, y);
            CHECK(frames.size() >= 5);
            double worst = 0;
            for (const auto& fr : frames)
                for (std::size_t a = 0; a < alphas.size(); ++a)
                    for (int m = -3; m <= 3; ++m) {
                        const cx want = direct(x, y, alphas[a], m, conj, fr.start_abs, 64);
                        const cx got = fr.values[flat_index(SetLayout{3, 3}, (int)a, m)];
                        worst = std::max(worst, std::abs(got - want));
                    }
            CHECK(worst <= 2e-5);  // |dR| <= 1e-5 * mean power (power ~2 here)
        }
    }
    // bookkeeping + emission rule (test_estimator.cpp:184-209)
    {
        CyclicCorrelator est(set_cfg(16, 3, {0.1}));
        const auto x = random_stream(200, 55);
        std::uint64_t fed = 0, emitted = 0;
        std::mt19937_64 gen(3);
        while (fed < x.size()) {
            const std::size_t take = std::min<std::size_t>(x.size() - fed, gen() % 37);
            const std::vector<cx> chunk(x.begin() + fed, x.begin() + fed + take);
            for (const auto& fr : est.push(chunk, chunk)) {
                CHECK(fr.frame_index == emitted);
                CHECK(fr.start_abs == 3 + emitted * 16);
                ++emitted;
            }
            fed += take;
            CHECK(est.frames_emitted() == (fed >= 22 ? (fed - 22) / 16 + 1 : 0));
        }
        CHECK(est.frames_emitted() == 12);
    }
    // block mode: coherent average == average_frames of the per-frame run
    {
        const auto x = random_stream(1 << 14, 9);
        EstimatorConfig c;
        c.mode = Mode::Full;
        c.win_len = 256;
        c.lag_spec = LagSpec::Explicit({0, 1, 2, 3});
        CyclicCorrelator frames_est(c);
        const auto avg = average_frames(frames_est.push(x, x), AverageMode::Coherent);
        c.emit_frames = false;
        CyclicCorrelator block(c);
        block.push(x, x);
        const auto b = block.average();
        double worst = 0;
        for (std::size_t i = 0; i < avg.size(); ++i) worst = std::max(worst, std::abs(avg[i] - b[i]));
        CHECK(worst <= 2e-5);
    }
    // cf32 file push (io.cpp:74-103) == pushing the same samples as an array
    {
        const auto x = random_stream(4096, 21);
        std::vector<std::complex<float>> xf(x.begin(), x.end());
        const char* path = "/tmp/cyc_cxx_dropin.cf32";
        FILE* f = std::fopen(path, "wb");
        std::fwrite(xf.data(), sizeof(xf[0]), xf.size(), f);
        std::fclose(f);
        CyclicCorrelator a(set_cfg(256, 3, {0.0, 0.125}));
        CyclicCorrelator b(set_cfg(256, 3, {0.0, 0.125}));
        const auto fa = a.push_file(path);
        const auto fb = b.push(x, x);
        CHECK(fa.size() == 15 && fb.size() == 15);  // the 16th waits for m lookahead samples
        double worst = 0;
        for (std::size_t i = 0; i < fa.size() && i < fb.size(); ++i)
            for (std::size_t j = 0; j < fa[i].values.size(); ++j)
                worst = std::max(worst, std::abs(fa[i].values[j] - fb[i].values[j]));
        CHECK(worst <= 1e-6);
        f = std::fopen(path, "ab");
        std::fputc(0, f);
        std::fclose(f);
        try {
            a.push_file(path);
            CHECK(false);
        } catch (const IoError& e) {
            CHECK(std::string(e.what()).find("truncated") != std::string::npos);
        }
        std::remove(path);
    }
    // estimate_cfo_ccf argument guards and the no-feature path (test_impair.cpp:160-172)
    {
        const auto noise = random_stream(16 * 1024 + 8, 9);
        try {
            estimate_cfo_ccf(noise, 0.0625, 1024, 0);
            CHECK(false);
        } catch (const UsageError&) {
        }
        try {
            estimate_cfo_ccf(noise, 0.0625, 1024, 16);
            CHECK(false);
        } catch (const NoFeatureError&) {
        }
    }
    // CPM generation and the Monte-Carlo oracle (test_reference.cpp:117-145)
    {
        CpmParams p;
        const auto syms = random_symbols(p.alphabet_size, 256, 42);
        const auto x = cpm_modulate(p, syms);
        CHECK(x.size() == 256u * 8u);
        double worst = 0;
        for (const auto& v : x) worst = std::max(worst, std::abs(std::abs(v) - 1.0));
        CHECK(worst <= 1e-12);  // constant envelope
        CHECK(make_pulse(p).g.back() == 0.5);
        const auto t = gmsk_mc_oracle(p, {0.125, 0.0}, {-4, -1, 0, 2}, false, 256, 3, 1100, 42);
        CHECK(t.mean_magnitude.size() == 8);
        const auto again = gmsk_mc_oracle(p, {0.125, 0.0}, {-4, -1, 0, 2}, false, 256, 3, 1100, 42);
        CHECK(t.mean_magnitude == again.mean_magnitude);
        CHECK(std::abs(t.cell(1, 2) - 1.0) <= 1e-6);  // |R(0, 0)| = mean power = 1
        try {
            gmsk_mc_oracle(p, {}, {0}, false, 256, 1, 1100, 1);
            CHECK(false);
        } catch (const UsageError&) {
        }
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAIL" : "PASS", g_fail);
    return g_fail;
}

// ref_caller_main.cpp -- drives an UNMODIFIED reference caller compiled
// against the drop-in header: /root/reference/proj/src/impair.cpp
// (cycstat::estimate_cfo_ccf, apply_cfo, add_noise_snr, impair.cpp:17-115) and
// siggen.cpp are compiled from the reference tree with tests/cpp/refshim first
// on the include path, so their CyclicCorrelator / average_frames / errors are
// the B200 ones (include/cycstat_b200.hpp over libcycb200.so).  The cases are
// those of proj/tests/test_impair.cpp:141-171: CPM records with known carrier
// offsets are recovered within one bin spacing, proper signals raise
// NoFeatureError, an out-of-range beta raises UsageError.  Prints PASS.
#include <cmath>
#include <cstdio>
#include <vector>

#include "cycstat/estimator.hpp"
#include "cycstat/impair.hpp"
#include "cycstat/siggen.hpp"

namespace {
// a CPM record of `len` samples (h = modulation index), as proj/tests/test_impair.cpp builds them
std::vector<cycstat::cx> cpm_record(std::size_t len, double h, std::uint64_t seed) {
    cycstat::CpmParams p;
    p.h = h;
    auto x = cycstat::cpm_modulate(p, cycstat::random_symbols(p.alphabet_size, (len + p.sps - 1) / p.sps, seed));
    x.resize(len);
    return x;
}
}  // namespace

int main() {
    int fails = 0;
    const int n = 1024, frames = 16;
    const double beta = 0.0625;  // MSK-type CPM (h = 1/2): conjugate features at +-1/(2 sps)
    const auto x = cpm_record((std::size_t)frames * n + 8, 0.5, 77);
    const double e0 = cycstat::estimate_cfo_ccf(x, beta, n, frames);
    std::printf("eps 0: reference caller %+.6f %s\n", e0, std::abs(e0) <= 0.5 / n ? "ok" : "FAIL");
    fails += !(std::abs(e0) <= 0.5 / n);
    for (double eps : {-0.01, 0.003, 0.02}) {
        const auto y = cycstat::apply_cfo(x, cycstat::CfoSpec{eps, 0.4});
        const double ref_path = cycstat::estimate_cfo_ccf(y, beta, n, frames);   // the reference's code
        const double b200 = cycstat_b200::estimate_cfo_ccf(y, beta, n, frames);  // the B200 consumer
        const bool ok = std::abs(ref_path - eps) <= 1.0 / n && std::abs(ref_path - b200) < 1e-7;
        std::printf("eps %+.4f: reference caller %+.6f, b200 %+.6f %s\n", eps, ref_path, b200, ok ? "ok" : "FAIL");
        fails += !ok;
    }
    for (int k = 0; k < 2; ++k) {  // proper signals carry no conjugate feature
        const auto z = k == 0 ? cpm_record(16 * n + 8, 0.7, 88) : cycstat::awgn(16 * n + 8, 1.0, 3);
        try {
            cycstat::estimate_cfo_ccf(z, beta, n, 16);
            std::printf("proper signal %d: no NoFeatureError FAIL\n", k);
            ++fails;
        } catch (const cycstat::NoFeatureError& e) {
            std::printf("proper signal %d: NoFeatureError ok (%s)\n", k, e.what());
        }
    }
    try {
        cycstat::estimate_cfo_ccf(x, 0.75, n, 4);
        ++fails;
    } catch (const cycstat::UsageError&) {
        std::printf("beta out of range: UsageError ok\n");
    }
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails ? 1 : 0;
}

// ref_caller_main.cpp -- drives an UNMODIFIED reference caller compiled
// against the drop-in header: /root/reference/proj/src/impair.cpp
// (cycstat::estimate_cfo_ccf, apply_cfo, add_noise_snr, impair.cpp:17-115) and
// siggen.cpp are compiled from the reference tree with tests/cpp/refshim first
// on the include path, so their CyclicCorrelator / average_frames / errors are
// the B200 ones (include/cycstat_b200.hpp over libcycb200.so).  The cases are
// those of proj/tests/test_impair.cpp: a GMSK record with a known carrier
// offset is recovered within a fraction of a bin, and a proper (circular)
// noise record raises NoFeatureError.  Prints PASS.
#include <cmath>
#include <cstdio>
#include <vector>

#include "cycstat/estimator.hpp"
#include "cycstat/impair.hpp"
#include "cycstat/siggen.hpp"

int main() {
    int fails = 0;
    // MSK-type CPM (h = 1/2) carries conjugate features at +-1/(2 sps): beta = 1/16 for sps = 8
    cycstat::CpmParams p;
    p.sps = 8;
    const auto sym = cycstat::random_symbols(2, 4096, 11);
    const auto x0 = cycstat::cpm_modulate(p, sym);
    const double beta = 1.0 / 16.0;
    for (double eps : {0.0, 0.003, -0.004}) {
        auto x = cycstat::apply_cfo(x0, cycstat::CfoSpec{eps, 0.3});
        x = cycstat::add_noise_snr(x, 10.0, 5);
        const double ref_path = cycstat::estimate_cfo_ccf(x, beta, 1024, 16);   // the reference's code
        const double b200 = cycstat_b200::estimate_cfo_ccf(x, beta, 1024, 16);  // the B200 consumer
        const bool ok = std::abs(ref_path - eps) < 0.5 / 1024 && std::abs(ref_path - b200) < 1e-7;
        std::printf("eps %+.4f: reference caller %+.6f, b200 %+.6f %s\n", eps, ref_path, b200, ok ? "ok" : "FAIL");
        fails += !ok;
    }
    try {
        const auto noise = cycstat::awgn(1024 * 16, 1.0, 3);
        cycstat::estimate_cfo_ccf(noise, beta, 1024, 16);
        std::printf("noise: no NoFeatureError FAIL\n");
        ++fails;
    } catch (const cycstat::NoFeatureError& e) {
        std::printf("noise: NoFeatureError ok (%s)\n", e.what());
    }
    try {
        cycstat::estimate_cfo_ccf(x0, 0.7, 1024, 16);
        ++fails;
    } catch (const cycstat::UsageError&) {
        std::printf("beta out of range: UsageError ok\n");
    }
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails ? 1 : 0;
}

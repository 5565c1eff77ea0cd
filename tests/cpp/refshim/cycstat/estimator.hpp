// Shim for an UNMODIFIED reference caller compiled against the drop-in:
// "cycstat/estimator.hpp" resolves here (this directory comes first on the include
// path), so the caller's cycstat:: names bind to the B200 estimator in
// include/cycstat_b200.hpp; the reference's other headers (impair.hpp,
// siggen.hpp) are its own.  Test infrastructure (tests/test_cxx.py).
#pragma once
#include "cycstat_b200.hpp"
namespace cycstat {
using namespace cycstat_b200;
}

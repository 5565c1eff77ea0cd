// hostpool.h -- process-wide helper threads for the host side of small pushes.
//
// A small host chunk is copied into the engine's pinned staging and screened
// for non-finite samples in the same pass (engine.cpp: copy_screen) before the
// push can return: the reference checks the whole chunk before touching any
// state (proj/src/estimator.cpp:43-52).  On the GPU hosts of this pool one core
// copies ~11 GB/s from cold memory, so the copy alone bounds a stream of
// 8192-sample pushes (BASELINE C3) at 5.8 us per call; three helper threads
// split it four ways (2.4 us; tools/exp/host_mt.cpp).
#pragma once

#include <cstddef>
#include <cstdint>

namespace cyc {

// Copy m 32-bit words s -> d with non-temporal stores (d is pinned staging
// read back only by DMA or zero-copy kernels) and return nonzero if any word
// has an all-ones float32 exponent (Inf/NaN).  Splits large copies across the
// pool; falls back to the calling thread when the pool is busy or disabled
// (CYC_COPY_THREADS=0).
uint32_t copy_screen_words(uint32_t* d, const uint32_t* s, size_t m);

}  // namespace cyc

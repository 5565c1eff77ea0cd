/*
 * cycoracle.h -- CPU oracle for the cyclic-ACF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2405_16911_b200/)
 * links or calls this code.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it, and only as the checker.
 *
 * A plain-C, double-precision restatement of the reference estimator
 * (reference: /root/reference/proj, C++ `cycstat`).  Each function cites the
 * reference file:line it restates.  Complex arrays are interleaved doubles
 * (re, im).  Parity of this restatement is pinned against
 *   (1) the reference's frozen golden values (proj/tests/test_reference.cpp:54-67),
 *   (2) outputs of the reference itself compiled from its sources into
 *       oracle/_ref/ (see oracle/Makefile, tests/test_oracle.py).
 */
#ifndef CYCORACLE_H
#define CYCORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Literal windowed sum (proj/src/reference.cpp:11-32):
 *   e^{-j2pi a k0} (1/N) sum_{n<N} x[k0+n+m] y^(*)[k0+n] e^{-j2pi a n}
 * y conjugated iff conj == 0.  Returns 0 on success, -1 on coverage error. */
int orc_direct(const double* x, const double* y, size_t len, double alpha, int m,
               int conj, size_t k0, int n_win, double out[2]);

/* Unnormalised forward DFT (proj/src/fft.cpp:44-100): radix-2 DIT for powers of
 * two, table-driven direct sum otherwise.  in/out may alias. */
void orc_fft(const double* in, double* out, size_t n);

/* Streaming estimator restatement (proj/src/estimator.cpp:15-84 with
 * proj/src/kernels.cpp:27-114): emits every frame of the whole record
 * x/y[0..len) in one go (chunking invariance, estimator.hpp:81-86).
 * mode 0 = Set (symmetric lags -max_lag..max_lag, alphas), 1 = Full (lags list).
 * frames_out receives F*layout_len complex values, F returned via *n_frames.
 * Pass frames_out == NULL to query F and layout_len only.
 * Returns 0 or -1 on a config the reference would reject. */
int orc_stream(int mode, int conj, int win_len, const double* alphas, size_t n_alphas,
               int max_lag, const int* lags, size_t n_lags, const double* x,
               const double* y, size_t len, double* frames_out, size_t* n_frames,
               size_t* layout_len);

/* Block table by literal summation (coherent average of frames,
 * proj/src/estimator.cpp:86-105, restated as one block sum):
 *   out[a][t] = (1/count) sum_{n=start}^{start+count-1} x[n+lag_t] y^(*)[n] e^{-j2pi alpha_a n}
 * Layout: alpha-major, lags in list order (Set layout, types.hpp:68-73). */
int orc_block_direct(const double* x, const double* y, size_t len, const double* alphas,
                     size_t n_alphas, const int* lags, size_t n_lags, int conj,
                     size_t start, size_t count, double* out);

/* Same block table through the exact fold over residues n mod P (valid when
 * every alpha = k_a / P; SPEC.md:201 permits any exact strategy).  k[a] gives
 * the integer numerator of each alpha.  Both flags at once:
 * out_conv / out_conj may be NULL. */
int orc_block_fold(const float* xf, const float* yf, size_t len, const int64_t* k,
                   size_t n_alphas, int64_t P, const int* lags, size_t n_lags,
                   size_t start, size_t count, double* out_conv, double* out_conj);

/* Recursive (exponential-forgetting) estimator -- not in the reference (SURVEY
 * §8 a15); builder-defined, restated literally in fp64:
 *   R_n = lambda R_{n-1} + (1-lambda) x[n+lag] y^(*)[n] e^{-j2pi alpha n},
 * n >= m_minus, R_{m_minus-1} = 0; emission e reports R at
 * n = m_minus + (e+1)*emit_every - 1.  out: n_emit x (alphas x lags). */
int orc_recursive(const double* x, const double* y, size_t len, const double* alphas,
                  size_t n_alphas, const int* lags, size_t n_lags, int conj,
                  double lambda, size_t emit_every, double* out, size_t* n_emit);

/* std::mt19937_64 (standardised) -- used to reproduce reference seeds. */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);

#ifdef __cplusplus
}
#endif
#endif

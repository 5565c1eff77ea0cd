/*
 * cycb200.h -- C-ABI of the B200-native cyclic-ACF estimator (libcycb200.so).
 *
 * Drop-in boundary for the reference estimator `cycstat::CyclicCorrelator`
 * (/root/reference/proj/include/cycstat/estimator.hpp:77-148).  Plain pointers
 * and sizes only; no CUDA or torch types cross this boundary.  The C++
 * wrapper include/cycstat_b200.hpp restores the reference's class names,
 * exceptions and std::vector signatures on top of it.
 *
 * Every entry point replaces one reference interface (file:line cited) and
 * keeps its argument meaning and error behaviour:
 *   - configuration errors collect EVERY violation   (proj/src/types.cpp:30-63)
 *   - a chunk with a non-finite sample is rejected whole, state unchanged,
 *     and the message names the absolute index      (proj/src/estimator.cpp:41-52)
 *   - frames are emitted per win_len consumed samples once buffer_need are
 *     pending; the tail is never flushed             (proj/src/estimator.cpp:59-82)
 *
 * Values are the reference's quantity
 *   R(a, m) = (1/N) sum_{n<N} x[k0+n+m] y^(*)[k0+n] e^{-j2pi a (k0+n)}
 * computed on the GPU from complex64 samples (float32 arithmetic with fp64
 * reductions; parity tolerance: relative L2 <= 1e-4 per table and per-value
 * |dR| <= 1e-5 * mean power, BASELINE.json north_star).
 *
 * Thread safety: a handle is single-owner (estimator.hpp:95-96); distinct
 * handles are independent.
 */
#ifndef CYCB200_H
#define CYCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CYC_ABI_VERSION 1

/* Status codes.  Map 1:1 onto the reference exception types
 * (proj/include/cycstat/errors.hpp:10-49). */
typedef enum {
    CYC_OK = 0,
    CYC_ERR_CONFIG = 1,   /* ConfigError  (violation list in the message)      */
    CYC_ERR_USAGE = 2,    /* UsageError   (mismatched chunks, bad arguments)   */
    CYC_ERR_DATA = 3,     /* DataError    (non-finite sample; absolute index)  */
    CYC_ERR_CUDA = 4,     /* device / driver failure (no CPU fallback exists)  */
    CYC_ERR_INTERNAL = 5, /* std::logic_error equivalent                       */
    CYC_ERR_IO = 6,       /* IoError      (unreadable file, errors.hpp:32-34)  */
    CYC_ERR_FORMAT = 7    /* FormatError  (malformed file, errors.hpp:36-38)   */
} cyc_status;

/* Estimator mode (proj/include/cycstat/types.hpp:22-25) plus the
 * exponential-forgetting estimator the reference lacks. */
typedef enum {
    CYC_MODE_SET = 0,       /* alpha list x lags; alpha-major, lags ascending    */
    CYC_MODE_FULL = 1,      /* lag list x all N DFT bins; lag-major, natural bins */
    CYC_MODE_RECURSIVE = 2  /* R_n = lam R_{n-1} + (1-lam) q_n e^{-j2pi a n}      */
} cyc_mode;

/* Which cyclic functions to compute.  The reference computes one per
 * estimator (EstimatorConfig::conj, types.hpp:57-59); one pass here can
 * produce both from the same four real correlations. */
typedef enum {
    CYC_FLAG_CONV = 1, /* conj == false: x * conj(y) (cyclic ACF)               */
    CYC_FLAG_CONJ = 2, /* conj == true : x * y       (conjugate cyclic ACF)     */
    CYC_FLAG_BOTH = 3
} cyc_flags;

typedef enum { CYC_AVG_COHERENT = 0, CYC_AVG_MAGNITUDE = 1 } cyc_avg_mode;

typedef struct { float re, im; } cyc_cf32;
typedef struct { double re, im; } cyc_cf64;

/* EstimatorConfig (types.hpp:55-63) + extensions.  Initialise with
 * cyc_config_init() and override fields. */
typedef struct cyc_config {
    int mode;              /* cyc_mode                                                */
    int conj;              /* reference conj flag; used when flags == 0               */
    int flags;             /* 0 => (conj ? CONJ : CONV); else cyc_flags bitmask       */
    int win_len;           /* N; RECURSIVE: emission interval (samples)               */
    const double* alphas;  /* SET / RECURSIVE: cycle frequencies, cycles/sample       */
    size_t num_alphas;
    int lag_symmetric;     /* 1: LagSpec::Symmetric(max_lag); 0: explicit list        */
    int max_lag;
    const int* lags;       /* explicit, strictly increasing                           */
    size_t num_lags;
    double lambda;         /* RECURSIVE forgetting factor, 0 < lambda < 1             */
    int emit_frames;       /* 1: per-frame values go to the sink (reference push());  */
                           /* 0: frames are only counted and folded into the running */
                           /*    coherent average (cyc_average) -- the block mode     */
    int channels;          /* >= 1 independent synchronized streams per handle        */
    int device;            /* CUDA device ordinal                                     */
    int64_t origin;        /* absolute index of the first pushed sample (default 0):  */
                           /* phases and start_abs are anchored to absolute sample 0, */
                           /* so a stream may be resumed or time-sharded exactly      */
} cyc_config;

typedef struct cyc_est cyc_est;

/* One emitted frame (CyclicFrame, types.hpp:97-104).  `values` is valid only
 * during the sink call; layout as cyc_layout(). */
typedef struct {
    uint64_t frame_index;
    uint64_t start_abs;     /* m_minus + frame_index * win_len                    */
    int flag;               /* CYC_FLAG_CONV or CYC_FLAG_CONJ                     */
    int channel;
    size_t len;             /* layout_len                                         */
    const cyc_cf64* values;
} cyc_frame_view;

/* Return 0 to continue; nonzero stops delivery (the push still commits). */
typedef int (*cyc_frame_sink)(void* user, const cyc_frame_view* frame);

/* Layout description (types.hpp:68-94). */
typedef struct {
    int kind;        /* 0 = SetLayout (alpha-major, lags ascending), 1 = FullLayout (lag-major) */
    int num_alphas;  /* Set / Recursive                                           */
    int max_lag;     /* Set: symmetric M (rows hold 2M+1 lags)                    */
    int num_lags;    /* lags per alpha row (Set/Recursive) or lag rows (Full)     */
    int win_len;     /* Full: bins per lag row                                    */
    size_t len;      /* layout_len                                                */
} cyc_layout_info;

void cyc_config_init(cyc_config* cfg);

/* validate_config (proj/src/types.cpp:30-63): returns the number of
 * violations and writes them, '\n'-separated, into buf. */
int cyc_validate(const cyc_config* cfg, char* buf, size_t buflen);

/* CyclicCorrelator(const EstimatorConfig&) (proj/src/estimator.cpp:15-37).
 * On CYC_ERR_CONFIG the message is "invalid config: [v1] [v2] ..."
 * (errors.hpp:17-30). */
int cyc_create(const cyc_config* cfg, cyc_est** out, char* err, size_t errlen);
void cyc_destroy(cyc_est* est);

/* CyclicCorrelator::push (proj/src/estimator.cpp:39-84).
 * x, y: channels * n samples, channel-major.  y == NULL means y = x (the
 * auto-correlation every BASELINE config uses; one stream is read).
 * Caller memory is not retained after return.  Pinned (page-locked) host
 * memory is DMA'd directly; pageable memory is staged. */
int cyc_push(cyc_est* est, const cyc_cf32* x, const cyc_cf32* y, size_t n,
             cyc_frame_sink sink, void* user);
/* Same, from the reference's complex<double> samples (converted to float32;
 * exact for data that came from cf32, proj/src/io.cpp:90-103). */
int cyc_push_f64(cyc_est* est, const cyc_cf64* x, const cyc_cf64* y, size_t n,
                 cyc_frame_sink sink, void* user);
/* Same, from samples already resident in device memory (GPU pipelines).
 * Stream order: the engine's streams are blocking CUDA streams, so the chunk
 * is read after work already queued on the legacy default stream (e.g. the
 * kernel that produced it), and work queued there after the call (e.g.
 * refilling d_x) waits for every read of it.  The call
 * returns once the chunk's finite check is known -- a rejected chunk returns
 * CYC_ERR_DATA with the state unchanged, as for host chunks -- while the fold
 * itself may still be running on cyc_stream(est).  Callers writing d_x from a
 * non-blocking stream synchronize with cyc_stream(est) first. */
int cyc_push_device(cyc_est* est, const cyc_cf32* d_x, const cyc_cf32* d_y, size_t n,
                    cyc_frame_sink sink, void* user);

/* One device-resident block step (extension; no reference counterpart):
 * cyc_reset + cyc_push_device(d_x, d_y, n) + cyc_average_all(avg_mode, out)
 * with ONE host synchronisation -- on the chunk's finite check -- after the
 * fold, its reduce and the finalize are all enqueued, instead of one per call
 * (the push's verdict round trip otherwise sits between the fold and the
 * finalize).  `out` as for cyc_average_all (device memory: written
 * stream-ordered).  A rejected chunk returns CYC_ERR_DATA (index, message as
 * cyc_push_device) and leaves the reset state; `out` is then undefined. */
int cyc_block_average_device(cyc_est* est, const cyc_cf32* d_x, const cyc_cf32* d_y, size_t n, int avg_mode,
                             cyc_cf64* out);

/* read_cf32 + push (proj/src/io.cpp:90-103, proj/tools/main.cpp:212-214):
 * the cf32 file (interleaved little-endian float32 I/Q) is pushed as ONE
 * chunk -- validated whole, then streamed from the page cache into the device
 * rings without an fp64 copy.  CYC_ERR_IO for open/read failures and a length
 * that is not a multiple of 8 bytes (FormatError). */
int cyc_push_cf32_file(cyc_est* est, const char* path, cyc_frame_sink sink, void* user);

/* ---- CPM / GMSK generation and the Monte-Carlo oracle ----
 * CpmParams (proj/include/cycstat/siggen.hpp:16-23). */
enum { CYC_PULSE_GAUSSIAN = 0, CYC_PULSE_RECT = 1 };
typedef struct cyc_cpm_params {
    double h;          /* modulation index, > 0 */
    int alphabet_size; /* even M >= 2 */
    int pulse_len;     /* L, frequency-pulse span in symbols */
    double bt;         /* bandwidth-symbol-time product (Gaussian pulse) */
    int sps;           /* samples per symbol */
    int pulse_kind;    /* CYC_PULSE_* */
} cyc_cpm_params;
/* Reference defaults: h 0.5, M 2, L 4, BT 0.25, 8 sps, Gaussian. */
void cyc_cpm_params_init(cyc_cpm_params* p);
/* random_symbols (proj/src/siggen.cpp:147-157): the same std::mt19937_64 draw. */
int cyc_random_symbols(int alphabet_size, size_t count, uint64_t seed, int* out, char* err, size_t errlen);
/* make_pulse (proj/src/siggen.cpp:30-110): f and its running sum g, len = L*sps. */
int cyc_cpm_pulse(const cyc_cpm_params* p, double* f_out, double* g_out, size_t len, char* err, size_t errlen);
/* cpm_modulate (proj/src/siggen.cpp:111-145) on the device: n_symbols*sps
 * samples into `out` (device or host memory), cf32 (out_f64 = 0) or cf64.
 * CYC_ERR_USAGE / CYC_ERR_DATA with the reference's messages. */
int cyc_cpm_modulate(const cyc_cpm_params* p, const int* symbols, size_t n_symbols, int device, int out_f64,
                     void* out, char* err, size_t errlen);
/* gmsk_mc_oracle (proj/src/reference.cpp:34-96): mean |R| over every window
 * of every trial, row-major |alphas| x |lags|; trial t uses seed + t. */
int cyc_gmsk_mc_oracle(const cyc_cpm_params* p, const double* alphas, size_t n_alphas, const int* lags,
                       size_t n_lags, int conj, int win_len, int trials, size_t record_len, uint64_t seed,
                       int device, double* mean_magnitude, char* err, size_t errlen);

/* estimate_cfo_ccf (proj/src/impair.cpp:45-115): conjugate Full-mode lag-0
 * scan over num_frames windows of N samples, magnitude average (on the
 * device), peak within +-N/8 bins of expected_beta, median test, log-parabola
 * refinement; *eps_out = wrapped(beta_peak - expected_beta) / 2.
 * CYC_ERR_USAGE for the reference's argument errors, CYC_ERR_DATA with
 * "no feature detected ..." for its NoFeatureError. */
int cyc_estimate_cfo_ccf(const cyc_cf32* x, size_t n, double expected_beta, int N, int num_frames,
                         int device, double* eps_out, char* err, size_t errlen);

/* average_frames(frames emitted so far, mode) (proj/src/estimator.cpp:86-105)
 * for one (flag, channel), without materialising the frames: the coherent
 * mean equals one block sum over [m_minus, m_minus + F*N) / (F*N).
 * MAGNITUDE needs emit_frames == 1.  out: layout_len values.
 * CYC_ERR_USAGE when no frame was emitted yet. */
int cyc_average(cyc_est* est, int avg_mode, int flag, int channel, cyc_cf64* out);
/* Every (channel, flag) table in one call: out = channels * num_flags *
 * layout_len values, [channel][flag][layout] (flag order: CONV, CONJ).
 * For cyc_average and cyc_average_all, `out` may be pageable host memory,
 * pinned host memory (the table is DMA'd straight into it) or -- for a
 * block-mode coherent average -- device memory (the table never leaves HBM;
 * it is then written stream-ordered on cyc_stream(est) and the call returns
 * without waiting: work later queued on the legacy default stream is ordered
 * after the write; from a non-blocking stream, synchronize cyc_stream(est) or
 * call cyc_synchronize before reading it). */
int cyc_average_all(cyc_est* est, int avg_mode, cyc_cf64* out);

/* Accessors (estimator.hpp:109-115). */
size_t cyc_buffer_need(const cyc_est* est);
uint64_t cyc_consumed(const cyc_est* est);
uint64_t cyc_frames_emitted(const cyc_est* est);
int cyc_layout(const cyc_est* est, cyc_layout_info* out);
int cyc_num_flags(const cyc_est* est);
/* Message of the last failed call on this handle ("" if none). */
const char* cyc_last_error(const cyc_est* est);
/* For CYC_ERR_DATA: absolute index of the offending sample, else -1. */
int64_t cyc_data_error_index(const cyc_est* est);

/* Block-mode fold state: device pointer to the fp64 residue-fold accumulators
 * (count doubles) and the number of frames folded into them.  Time shards of
 * one record (each created with origin = its first frame * win_len) sum these
 * buffers in place (e.g. ncclAllReduce) and set the total frame count; the
 * coherent average is then exactly the whole record's. */
int cyc_fold_state(cyc_est* est, void** dev_ptr, size_t* count, uint64_t* frames);
int cyc_fold_set_frames(cyc_est* est, uint64_t frames);
/* Lag slice of the block-mode coherent averages (multi-GPU lag slices): later
 * cyc_average_all / cyc_block_average_device calls finalize only the requested
 * lags with index in [lag_begin, lag_end) (indices into the lag list; the
 * rows of the other lags in `out` are left untouched), so time shards can
 * reduce-scatter their fold states by lag rows -- each rank then holds the
 * whole record's state for its slice only -- and finalize 1/G of the tables.
 * (0, 0) restores every lag.  No reference counterpart. */
int cyc_set_lag_slice(cyc_est* est, uint32_t lag_begin, uint32_t lag_end);
/* Pipelined emission for small-call streams (per-frame and recursive modes).
 * depth 0 (default): a push delivers the frames it completes before it returns
 * (CyclicCorrelator::push, estimator.cpp:59-82).  depth 1 or 2: the push that
 * completes a frame batch only enqueues its GPU work, and up to `depth` batches
 * stay in flight (CUDA-graph replayed batches: two for the small one-launch fold graphs, else one); their frames go, oldest
 * first, to the sink of the first later cyc_push that finds them finished (at
 * the latest the push that would exceed the depth) or to cyc_flush_frames, so
 * the GPU round trip of an emission overlaps the caller's next chunks.  Frame
 * order, indices and values are those of depth 0.  cyc_reset drops batches
 * nobody flushed.  No reference counterpart (the reference computes frames
 * inside push()). */
int cyc_set_emit_pipeline(cyc_est* est, int depth);
/* Wait for the frame batches in flight (if any) and deliver them to `sink`. */
int cyc_flush_frames(cyc_est* est, cyc_frame_sink sink, void* user);

/* CSV export of results (proj/src/io.cpp:161-208, the reference's
 * export_frames_csv(path, frames, cfg) / export_average_csv(path, avg, cfg,
 * mode)): same headers, rows in layout order, doubles as "%.17g", (alpha, lag)
 * of each element from the config's layout (Full bins through
 * full_bin_to_alpha).  frames: n_frames tables of layout_len values each, with
 * their frame indices.  avg_mode selects the coherent (re, im, mag) or
 * magnitude (mag) average format.  *rows = data rows written.  Host-only.
 * CYC_ERR_CONFIG for an invalid config, CYC_ERR_USAGE for empty or mis-sized
 * input, CYC_ERR_IO when the file cannot be written. */
int cyc_export_frames_csv(const cyc_config* cfg, const char* path, const uint64_t* frame_index,
                          const cyc_cf64* values, size_t n_frames, size_t* rows, char* err, size_t errlen);
int cyc_export_average_csv(const cyc_config* cfg, const char* path, const cyc_cf64* avg, size_t len, int avg_mode,
                           size_t* rows, char* err, size_t errlen);

/* Block until all device work of this handle is complete. */
int cyc_synchronize(cyc_est* est);
/* Fresh stream state with the same config and allocations: equivalent to
 * destroying and re-creating the estimator (a new CyclicCorrelator(cfg)). */
int cyc_reset(cyc_est* est);
/* Fold-kernel timing with CUDA events on the handle's compute stream:
 * launches, total kernel milliseconds and algorithmic FP32 flops
 * (8 per requested lag per folded sample, both flags). */
int cyc_profile_enable(cyc_est* est, int on);
int cyc_profile_read(cyc_est* est, uint64_t* launches, double* ms, double* flops);
/* Same, plus the executed flops (tensor-core launches: the MMA flops of the
 * bf16x3 banded product; FP32 launches: = algorithmic) and how many of the
 * launches ran on the tensor cores. */
int cyc_profile_read_ex(cyc_est* est, uint64_t* launches, double* ms, double* flops, double* exec_flops,
                        uint64_t* tensor_launches);
/* FP32 FFMA throughput of `device`, TFLOP/s (roofline denominator). */
double cyc_measure_fp32_peak(int device);
/* The handle's compute stream (cudaStream_t as void*), for event timing. */
void* cyc_stream(cyc_est* est);
/* Kernel launches issued by this handle so far (instrumentation). */
uint64_t cyc_kernel_launches(const cyc_est* est);
/* Internal algorithm chosen for this handle: "fold-dft", "fold-fft",
 * "direct", written into buf. */
int cyc_algorithm(const cyc_est* est, char* buf, size_t buflen);
/* The same plan for a config without creating a handle (host-only, no
 * device): rational alpha grid P, fold period Pf, lag-lane width. */
int cyc_plan(const cyc_config* cfg, char* buf, size_t buflen);

/* Page-locked host buffers for zero-copy-staging pushes. */
void* cyc_host_alloc(size_t bytes);
void cyc_host_free(void* p);

/* Library version / build info. */
int cyc_abi_version(void);
const char* cyc_build_info(void);

/* Kernel-level API (estimator.hpp:20-75), used by tests and the bench:
 * one-shot windows anchored at absolute index k0, computed on the device.
 * compute_set_window (kernels.cpp:116-123): xw has |yw| + 2*max_lag samples,
 * out: num_alphas * (2*max_lag+1).  compute_full_window (kernels.cpp:125-135):
 * xw has |yw| + m_plus + m_minus samples, out: num_lags * |yw|. */
int cyc_compute_set_window(const cyc_cf64* xw, size_t xw_len, const cyc_cf64* yw,
                           size_t yw_len, const double* alphas, size_t num_alphas,
                           int max_lag, int conj, uint64_t k0, cyc_cf64* out,
                           char* err, size_t errlen);
int cyc_compute_full_window(const cyc_cf64* xw, size_t xw_len, const cyc_cf64* yw,
                            size_t yw_len, const int* lags, size_t num_lags, int conj,
                            uint64_t k0, cyc_cf64* out, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif /* CYCB200_H */

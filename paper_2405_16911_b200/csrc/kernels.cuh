// kernels.cuh -- device-side data structures and launchers for the sm_100a
// cyclic-ACF kernels.  Host code (engine.cpp) only sees the launch_* functions.
//
// Algorithm map:
//   fold      exact reassociation of sum_n q_tau[n] e^{-j2pi k n/P} into
//             S_tau[r] = sum_{n = r mod Pf} q_tau[n]  (4 real correlations per
//             (tau, r) give both the conventional and the conjugate ACF);
//             replaces the per-alpha inner loop of set_window_values
//             (proj/src/kernels.cpp:46-55) and the lag product of
//             full_window_values (proj/src/kernels.cpp:85-87).
//   finalize  S -> R(alpha, tau): radix-2 fp64 FFT over residues (replaces
//             Fft::forward, proj/src/fft.cpp:44-87) or a direct DFT with exact
//             (k r mod Pf) twiddles for small alpha sets / non-pow2 periods.
//   direct    alphas not on a rational grid: per-(alpha, tau) contraction with
//             a 64-bit fixed-point phase (exact wrap) instead of the reference's
//             drifting lead-phasor recurrence (proj/src/estimator.cpp:70-73).
#pragma once
#include <utility>
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace cyc {

// Kernel attributes (the >48 KB dynamic shared memory opt-in) belong to the
// current device's context: set them once per device, not once per process
// (estimators may live on different devices of one process).
inline bool first_on_device(std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    return (done.fetch_or(bit) & bit) == 0;
}

// One contiguous y-index range [n_start, n_end) of one stream whose fold goes
// into accumulator slot `slot`.  Samples live in power-of-two device rings
// indexed by absolute sample number (ring[n & mask]).
struct FoldSeg {
    const float2* x;     // x ring base
    const float2* y;     // y ring base (== x for auto-correlation)
    int64_t n_start;     // first y index (absolute)
    int64_t n_end;       // one past the last y index
    int64_t x_lo, x_hi;  // absolute x range present in the ring
    uint64_t mask;       // ring mask (~0 for a linear device buffer)
    int64_t w_ref;       // recursive weighting: w(n) = w_scale * 2^{(w_ref - n) * w_log2}
    float w_log2;        // 0 => unweighted
    float w_scale;
    int slot;
    int vec;             // 1: x/y bases 16-byte aligned and window starts even (16-B cp.async)
};

// A CTA's unit of work: one (segment, residue block, lag block) over the
// absolute fold-period range [p0, p1).  `group` indexes (seg, rb, lb).
struct FoldTile {
    int seg, rb, lb, group;
    int64_t p0, p1;
};

// (seg, rb, lb) -> contiguous tile range, for the deterministic fp64 reduce.
struct FoldGroup {
    int seg, rb, lb;
    int t0, t1;
    int pad;
};

struct FoldLaunch {
    const FoldSeg* segs;
    const FoldTile* tiles;
    const FoldGroup* groups;
    int n_tiles, n_groups;
    int Pf;              // fold period (residues)
    int lag_lo;          // lowest lag of the computed span
    int t_pad;           // padded lag span (multiple of the lag block)
    int lw;              // lag lanes per warp: 2, 4 or 8  (TB = 8*lw, RB = 1024/lw)
    float* partials;     // [n_tiles][TB][RB] float4
    double* S;           // [slots][t_pad][Pf][4] fp64 accumulators
    int overwrite;       // 1: reduce stores (fresh per-frame slots, no memset); 0: accumulates
    // non-null: the reduce commits only if *gate == ~0 (the chunk's finite scan,
    // stream-ordered before the fold, found nothing) -- a rejected chunk leaves S untouched
    const unsigned long long* gate;
    // Fused finite check (tensor-core fold of a gated device chunk): non-null:
    // the lb = 0 tiles check every sample they stage for the reduce role (each
    // sample of the covered range exactly once) and atomicMin the scan's key,
    // ((2 * (abs - chk_c0) + is_y) * chk_channels + slot), into *chk_key.
    unsigned long long* chk_key;
    long long chk_c0;
    int chk_channels;
    // tensor-core folds: stages (16 periods) per TMEM accumulation chunk; the
    // epilogue drains the accumulator into the fp32 partials after each chunk
    int tc_drain;
    // planes tiles (1): a tile is 64 residues (rb counts 64-residue blocks) x
    // the lag blocks 2 lb and 2 lb + 1 -- partial cell (t, 64 h + r) is
    // residue 64 rb + r at lag block 2 lb + h; (2): 2-CTA tiles of 128 residues
    // x lags 128 lb .. 128 lb + 127, partials [tile][128 lags][128 residues];
    // else (0): 128 residues x lag block lb
    int tc_pairs;
};

// Launch descriptors carried in the kernel parameter block (<= 32 KB since
// CUDA 12.1): no H2D descriptor copy queued behind bulk DMA, no PCIe reads of
// mapped host memory.  Launches that do not fit use the pointers in FoldLaunch.
constexpr int FI_SEGS = 64, FI_TILES = 296, FI_GROUPS = 296;
struct FoldInline {
    FoldSeg segs[FI_SEGS];
    FoldTile tiles[FI_TILES];
    FoldGroup groups[FI_GROUPS];
};

// fold + fp64 reduce; optional events bracket the fold kernel alone (profiling).
// inl != nullptr: descriptors by value (L.segs/tiles/groups are ignored).
void launch_fold(const FoldLaunch& L, cudaStream_t st, cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr,
                 const FoldInline* inl = nullptr, cudaEvent_t before_reduce = nullptr);

// Small per-frame folds: slots segs_dev[0 .. n_slots) (device or mapped host memory), lags
// lag_lo .. lag_lo + t_span - 1, stored (not accumulated) into S rows 0 .. t_span-1
// of each seg's slot in fp64.  One thread per (slot, lag, residue).
// shift (nullable, device memory): added to every segment's absolute indices
// (n_start, n_end, x_lo, x_hi, w_ref) -- replayed frame graphs keep a static
// segment template and a device-side frame offset instead of host descriptors.
void launch_fold_small(const FoldSeg* segs_dev, int n_slots, int Pf, int lag_lo, int t_span, int t_pad, double* S,
                       cudaStream_t st, const int64_t* shift = nullptr);

// Tensor-core fold (fold_tc.cu): tiles of 128 residues x 64 lags, descriptors
// by value; partials [n_tiles][64 lags][128 residues] float4, reduced into S
// (accumulate; gate honoured).  Linear segments (mask == ~0) are staged with
// 2-D TMA through the per-segment tensor maps (rows = fold periods from
// p_base, columns = floats from sample p_base*Pf + lag_lo; rows overlap so a
// window may run past its period); ring segments with per-period 1-D bulk
// copies split at the wrap.
// Kernel parameters are copied into every launch at their declared size, and
// a large block costs host time (measured: ~36 us for two 22 KB launches), so
// the device descriptor comes in capacity classes; TcParams is the host-side
// master that launch_fold_tc packs into the smallest class that fits.
constexpr int TC_SEGS = 16;
template <int MT, int MG, int MS>
struct alignas(64) TcDesc {
    CUtensorMap xmap[MS];  // box 32 floats x 16 periods, 128B swizzle (12 boxes per window)
    CUtensorMap ymap[MS];  // same boxes over y (non-self launches: 8 per window)
    int64_t p_base[MS];    // first period (row 0) of each segment's maps
    FoldSeg segs[MS];
    FoldTile tiles[MT];
    FoldGroup groups[MG];
};
using TcParams = TcDesc<FI_TILES, FI_GROUPS, TC_SEGS>;
// Small-parameter form for launches whose tile table is already in device
// memory (a repeated plan): ~0.7 KB of parameters instead of ~6 KB.
struct alignas(64) TcDev {
    CUtensorMap xmap[2];
    CUtensorMap ymap[2];
    int64_t p_base[2];
    FoldSeg segs[2];
    const FoldTile* tiles;
};
// self: every tile's y window lies inside its x window at a 32-sample
// boundary (x == y, d = lag_lo + 64 lb in [-64, 0], d % 32 == 0).
// before_reduce: the reduce (not the fold) waits for this event (a gate scan on another stream).
// dev_tiles: a device copy of D.tiles[0, L.n_tiles) (n_segs <= 2), or null.
// fold_done: recorded after the fold kernel, before the reduce (a fused check's verdict).
void launch_fold_tc(const FoldLaunch& L, const TcParams& D, int n_segs, bool self, cudaStream_t st,
                    cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr, cudaEvent_t before_reduce = nullptr,
                    const FoldTile* dev_tiles = nullptr, cudaEvent_t fold_done = nullptr);
// Fill D.xmap/ymap/p_base[si] for a linear segment (false: no TMA -- use the ring path).
bool encode_tc_maps(TcParams& D, int si, const FoldSeg& g, int64_t p_base, int64_t rows, int Pf, int lag_lo,
                    int nlb);

// Planes path (self folds of device chunks over an even number of lag blocks, e.g. C5): the
// bf16x3 split is done once per sample by launch_split_planes -- hi and lo
// planes, one bf16x2 (re, im) word per sample, [channel][pitch] -- and the
// fold kernel stages the planes with TMA straight into the UMMA operand layout
// (no converter warps: shared memory carries only the TMA writes and the MMA
// operand reads).  Tiles of every lag block run in one launch, ordered so that
// the lag blocks of a residue block share the L2-resident planes.
struct alignas(64) TcPlDesc {
    // 4-D maps (64 bf16, period rows, hi/lo, atoms of 32 samples), 128B swizzle:
    // one TMA per window lands [atom][hi, lo][16 periods][128 B]
    CUtensorMap xmap[TC_SEGS];  // box: the 6 atoms of an x window
    CUtensorMap ymap[TC_SEGS];  // box: the 2 atoms of a y window (64 residues)
    int64_t p_base[TC_SEGS];    // first period (row 0) of each segment's maps
    FoldSeg segs[TC_SEGS];
    const FoldTile* tiles;      // device tile table [n_tiles]
};
// 2-CTA planes path (fold_tcp2_kernel): component planes [re_hi, re_lo,
// im_hi, im_lo] of bf16 per sample, plane stride `plane_elems`; tiles of 128
// residues x 2 lag blocks on a CTA pair (cta_group::2, M = 256 rows = the
// residues' real parts on CTA 0 and imaginary parts on CTA 1; each CTA stages
// half of the 256-sample x window).  xmap2: box {64, 16, 4 planes, 2 atoms};
// ymap2: box {64, 16, 2 planes, 2 atoms}.
struct alignas(64) TcPl2Desc {
    CUtensorMap xmap[TC_SEGS];
    CUtensorMap ymap[TC_SEGS];
    int64_t p_base[TC_SEGS];
    FoldSeg segs[TC_SEGS];
    const FoldTile* tiles;
};
bool encode_tcp2_maps(TcPl2Desc& D, int si, const uint16_t* plane0, int64_t plane_elems, int64_t p_base, int64_t rows,
                      int Pf, int64_t cols_samples);
void launch_fold_tcp2(const FoldLaunch& L, const TcPl2Desc& D, const FoldGroup* groups, cudaStream_t st,
                      cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);
// component planes of n samples of every channel: plane q of channel ch at
// planes + q * plane_elems + ch * pitch_out + out_off + i; and the finite scan
int launch_split_planes4(const float2* x, int64_t n, int C, int64_t pitch_in, uint16_t* planes, int64_t plane_elems,
                         int64_t pitch_out, int64_t out_off, unsigned long long* key, cudaStream_t st);
// Maps over planes whose element 0 is absolute sample p_base * Pf of the segment.
bool encode_tcp_maps(TcPlDesc& D, int si, const uint32_t* hi, const uint32_t* lo, int64_t p_base, int64_t rows,
                     int Pf, int64_t cols_samples);
void launch_fold_tcp(const FoldLaunch& L, const TcPlDesc& D, const FoldGroup* groups, cudaStream_t st,
                     cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);
// hi/lo planes of n samples of every channel (rows pitch_in / pitch_out apart;
// output index i + out_off) and the chunk's finite scan: the first non-finite
// sample i (reference scan order, x only) -> atomicMin(*key, (2 i) * C + ch).
// Returns the number of kernels launched.
int launch_split_planes(const float2* x, int64_t n, int C, int64_t pitch_in, uint32_t* hi, uint32_t* lo,
                        int64_t pitch_out, int64_t out_off, unsigned long long* key, cudaStream_t st);

// Profiling events around kernel launches: plain records, or -- while a push
// is being captured into a CUDA graph -- event-record nodes (so every replay
// records them; the engine swaps in fresh events per replay).
extern thread_local bool g_capture_events;
inline cudaError_t record_event(cudaEvent_t e, cudaStream_t s) {
    return cudaEventRecordWithFlags(e, s, g_capture_events ? cudaEventRecordExternal : cudaEventRecordDefault);
}

void prepare_fold_kernels();      // set smem attributes (call outside stream capture)
void prepare_finalize_kernels();

inline int fold_tb(int lw) { return 8 * lw; }
inline int fold_rb(int lw) { return 1024 / lw; }

// Finalize: S rows -> output tables.
struct FinalRow {
    int slot;       // accumulator slot
    int t_span;     // row in S (lag - lag_lo)
    int t_out;      // output lag index
    int out_block;  // output table index (slot-major, see engine)
};

struct FinalizeLaunch {
    const double* S;          // [slots][t_pad][Pf][4]
    int t_pad, Pf;
    const FinalRow* rows;
    int n_rows;
    int flags;                // bit0 conv, bit1 conj
    const int* bins;          // [A] DFT bin (mod Pf) per output alpha
    int A;
    const double2* tw;        // e^{-j2pi j / Pf}, j < Pf; then fft_pass_twiddles(Pf) entries
    double scale_default;     // multiply (1/count)
    const double* row_scale;  // optional per-out_block scale (nullptr => scale_default)
    double2* out;             // [out_block][flag_index][...] with strides below
    int64_t out_block_stride; // elements per out_block (all flags)
    int64_t out_flag_stride;  // elements per flag table
    int64_t stride_a, stride_t;
    int use_fft;              // 1: radix-2 FFT (Pf pow2 <= 8192); 0: direct DFT
    // recursive emission of one frame fused into the FFT's output (the same
    // arithmetic as recursive_update_kernel): R = decay R + value, the running
    // sums, and an optional copy into mapped host memory; rec_R == nullptr: off
    double2* rec_R;
    double rec_decay;
    double2* rec_coh;
    double* rec_mag;
    double2* rec_host;
    // replayed frame graphs: block (0, 0) adds shift_inc to *shift_ctr (the
    // fold that read it has completed); nullptr: off
    int64_t* shift_ctr;
    int64_t shift_inc;
};

// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor finishes (launch latency and prologue overlap the predecessor's
// tail); it executes pdl_wait() before touching the predecessor's output.
// Outside a PDL launch pdl_wait() is a no-op.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

void launch_finalize(const FinalizeLaunch& L, cudaStream_t st);
// FFT rows (Pf a power of two <= 8192) read per-pass twiddle tables stored right
// after the Pf plain twiddles of FinalizeLaunch::tw; fills `out` (nullable) and
// returns their count (0 for other Pf).
int fft_pass_twiddles(int Pf, double2* out);

// Direct contraction for arbitrary alphas.
struct DirectSeg {
    const float2* x;
    const float2* y;
    int64_t n_start, n_end;
    int64_t x_lo, x_hi;
    uint64_t mask;
    int64_t w_ref;       // recursive weighting (as FoldSeg)
    float w_log2, w_scale;
    int out_block;
    int pad;
};

constexpr int DIRECT_INL = 8;  // descriptors carried in the parameter block (small frame batches)
struct DirectLaunch {
    const DirectSeg* segs;      // device descriptors, or null: inl[0, n_segs)
    DirectSeg inl[DIRECT_INL];
    int n_segs;
    const uint64_t* alpha_fx;   // [A] round(alpha * 2^64)
    int A;
    const int* lags;            // [T] requested lags (ascending)
    int T;
    int lag_lo, lag_hi;
    int splits;                 // sample splits per (seg, alpha)
    int flags;
    float* partials;            // [n_segs][A][splits][2 flags][T] float2
    double2* out;               // [out_block][flag_index][...]
    double2* out_host;          // optional mapped pinned mirror of `out` (per-frame tables: no D2H copy)
    int64_t out_block_stride, out_flag_stride, stride_a, stride_t;
    double scale;
    // one frame per channel (n_segs == channels) with running sums: the last
    // CTA of each (segment, alpha) to finish reduces its splits in the direct
    // kernel itself (counters: [n_segs][A] zeros, left zeroed), no second launch
    int* fuse_counters;
    double2* coh;
    double* mag;
    int64_t per;
};

// coh/mag non-null: the reduce also adds each frame to the running average_frames
// sums (segments [frame][channel], `per` = values per channel block).
void launch_direct(const DirectLaunch& L, cudaStream_t st, double2* coh = nullptr, double* mag = nullptr,
                   int channels = 1, int64_t per = 0);
int direct_lanes(int T);  // sample lanes per lag of the direct kernel (1 for long lag spans)

// Utilities.
// gate non-null: adds only if *gate == ~0 (the chunk's finite check passed).
void launch_add_f64(double* dst, const double* src, int64_t n, cudaStream_t st,
                    const unsigned long long* gate = nullptr);
void launch_accum_frames(const double2* frames, int64_t n_frames, int64_t len,
                         double2* coh, double* mag, cudaStream_t st);
// Recursive emissions: per channel, in frame order, R = decay*R + frame; the
// frame becomes R; coh += R, mag += |R|.  frames are [frame][channel][per].
// host_out (mapped pinned, optional): the emitted tables are also written there.
void launch_recursive_update(double2* frames, int64_t n_frames, int channels, int64_t per, double2* R, double decay,
                             double2* coh, double* mag, cudaStream_t st, double2* host_out = nullptr);
// First non-finite sample -> atomicMin(*key);
// key = (2*(base+i) + is_y) * channels + ch  -- smallest = reference scan order.
// returns the number of kernels launched; nch > 1 scans channels ch .. ch+nch-1
// in one launch, channel rows `pitch` samples apart
int launch_finite_check(const float2* x, const float2* y, int64_t n, int64_t base, int channels, int ch,
                        unsigned long long* key, cudaStream_t st, int nch = 1, int64_t pitch = 0);
// Ring write from a device source with wrap: ring[(abs0 + i) & mask] = src[i].
// Copy n samples of `channels` rows (src row c at src + c * src_pitch) into the
// rings (row c at ring + c * ring_pitch) at absolute index abs0 (masked).
void launch_ring_write(float2* ring, uint64_t mask, int64_t abs0, const float2* src, int64_t n, cudaStream_t st,
                       int channels = 1, int64_t ring_pitch = 0, int64_t src_pitch = 0);

}  // namespace cyc

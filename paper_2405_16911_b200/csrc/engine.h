// engine.h -- host-side streaming engine (C++), the implementation behind the
// C-ABI in include/cycb200.h.
//
// Mirrors cycstat::CyclicCorrelator (proj/include/cycstat/estimator.hpp:97-137):
// the same config contract, buffer_need, frame emission rule, absolute-phase
// anchor and error semantics.  What changes is where the work runs:
//   * ingest: samples go into power-of-two device rings indexed by absolute
//     sample number (no O(buffer) front erase, proj/src/estimator.cpp:78-79);
//     host chunks are DMA'd in pieces on a copy stream that overlaps the
//     compute stream, through pinned staging when the caller's memory is
//     pageable;
//   * compute: fold + finalize (alphas on a rational grid) or the direct
//     fixed-point-phase contraction (kernels.cuh);
//   * block mode (emit_frames == 0): frames are only counted and folded into
//     a running fp64 accumulator, so the coherent average_frames() of any
//     number of frames costs one fold pass over the samples.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <string>
#include <memory>
#include <vector>

#include "../../include/cycb200.h"
#include "kernels.cuh"

namespace cyc {

struct Status {
    int code = CYC_OK;
    std::string msg;
    int64_t index = -1;
    static Status ok() { return {}; }
};

// Normalised configuration (EstimatorConfig, proj/include/cycstat/types.hpp:55-63).
struct Cfg {
    int mode = CYC_MODE_SET;
    int flags = CYC_FLAG_CONV;
    int win_len = 0;
    std::vector<double> alphas;
    bool lag_symmetric = true;
    int max_lag = 0;
    std::vector<int> lags;  // explicit list as given
    double lambda = 0.0;
    bool emit_frames = true;
    int channels = 1;
    int device = 0;
    int64_t origin = 0;  // absolute index of the first pushed sample
};

// validate_config (proj/src/types.cpp:30-63) + rules of the extensions.
std::vector<std::string> validate(const Cfg& c);
Cfg from_c(const cyc_config* c);

class Engine {
public:
    static Status create(const Cfg& cfg, Engine** out);
    // For one-shot kernel-level windows (kernels.cpp:116-135), whose contract
    // is only the window geometry, not the streaming span rule.
    static Status create_unchecked(const Cfg& cfg, Engine** out);
    // Algorithm the engine would pick for cfg (no device needed).
    static std::string plan_string(const Cfg& cfg);
    ~Engine();

    Status push(const void* x, const void* y, size_t n, int kind, cyc_frame_sink sink, void* user);
    Status average(int avg_mode, int flag, int channel, cyc_cf64* out);
    Status average_all(int avg_mode, cyc_cf64* out);
    // reset + push(device chunk) + average_all(avg_mode, out) with one host
    // synchronisation (the chunk's verdict) after everything is enqueued: the
    // block average of exactly this chunk.  On CYC_ERR_DATA the state is the
    // reset state and `out` is undefined.
    Status block_average_device(const void* x, const void* y, size_t n, int avg_mode, cyc_cf64* out);
    Status compute_window(const cyc_cf64* xw, size_t xw_len, const cyc_cf64* yw, size_t yw_len,
                          uint64_t k0, cyc_cf64* out);
    Status synchronize();
    // Finite scan of a host cf32 chunk; on success the next push of it skips its scan.
    Status validate_host_f32(const void* x, const void* y, size_t n);
    // Fresh stream state, same config and allocations (== a new CyclicCorrelator(cfg)).
    Status reset();
    // Block-mode fold state (time-sharded multi-GPU, checkpoint/resume).
    Status fold_state(void** dev_ptr, size_t* count, uint64_t* frames);
    Status set_frames(uint64_t frames);
    Status set_lag_slice(uint32_t b, uint32_t e);
    // Pipelined emission (cyc_set_emit_pipeline / cyc_flush_frames): one frame
    // batch stays in flight on the GPU while the caller's next pushes are
    // copied and screened; its frames reach the sink of the first later call
    // that finds them complete.
    Status set_emit_pipeline(int depth);
    Status flush_frames(cyc_frame_sink sink, void* user);
    // Fold-kernel timing with CUDA events on the compute stream.
    void set_profiling(bool on) { prof_ = on; }
    Status profile_read(uint64_t* launches, double* ms, double* flops, double* exec_flops = nullptr,
                        uint64_t* tensor_launches = nullptr);

    size_t buffer_need() const { return need_; }
    uint64_t consumed() const { return consumed_; }
    uint64_t frames_emitted() const { return frames_; }
    void layout(cyc_layout_info* li) const;
    int num_flags() const { return nflags_; }
    cudaStream_t stream() const { return cs_; }
    uint64_t launches() const { return launches_; }
    std::string algorithm() const;

    std::string last_error;
    int64_t last_error_index = -1;

    enum { IN_HOST_F32 = 0, IN_HOST_F64 = 1, IN_DEVICE_F32 = 2 };

private:
    Engine() = default;
    Status plan(const Cfg& cfg);
    Status init(const Cfg& cfg);
    Status cuda_check(cudaError_t e, const char* what);
    Status ensure_ring(int64_t cap_min);
    Status grow_ring(int64_t cap_min);
    Status ensure_partials(size_t bytes);
    Status ensure_frames(size_t slots);
    Status ensure_meta(size_t bytes);
    // Upload metadata through the pinned arena; returns device pointer.
    void* upload(const void* src, size_t bytes);

    // Fold `segs` (one per slot) into S (slots x t_pad x Pf x 4 fp64).
    Status fold(const std::vector<FoldSeg>& segs, double* S, bool overwrite = false);
    Status fold_tc(const std::vector<FoldSeg>& segs, double* S, std::vector<FoldSeg>& rest);
    struct TcGroupPlan {
        int seg, rb, lb;
        int64_t p0, p1;
    };
    Status fold_tc_batch(const std::vector<FoldSeg>& tsegs, std::vector<TcGroupPlan>& groups, double* S, int nlb);
    // Planes path (fold_device_chunk, several lag blocks, x == y, lag_lo >= 0):
    // the chunk's hi/lo bf16 planes, [channel][planes_pitch_] words from
    // absolute sample planes_c0_ (4-aligned, so every period row of the TMA
    // maps starts 16-byte aligned); planes_on_ while the chunk folds.
    Status fold_tc_planes(const std::vector<FoldSeg>& tsegs, std::vector<TcGroupPlan>& groups, double* S, int nlb);
    bool planes_ok(const std::vector<FoldSeg>& segs) const;
    uint32_t* planes_ = nullptr;
    size_t planes_words_ = 0;  // capacity of each of the hi / lo halves
    bool planes_on_ = false;
    bool planes2_ = false;  // the chunk's planes are component planes for the 2-CTA fold (lag_lo % 64 == 0)
    Status fold_tc_planes2(const std::vector<FoldSeg>& tsegs, std::vector<TcGroupPlan>& groups, double* S, int nlb);
    std::unique_ptr<TcPl2Desc> tpd2_;
    int64_t planes_c0_ = 0, planes_pitch_ = 0;
    std::unique_ptr<TcPlDesc> tpd_;
    struct PlTiles {  // device tile tables of the planes path, by content (graph replays keep them)
        std::vector<FoldTile> host;
        FoldTile* dev = nullptr;
    };
    std::vector<PlTiles> pl_tiles_;
    const FoldTile* planes_tiles(const std::vector<FoldTile>& t);
    bool tc_capable_ = false;  // sm_100 device (tcgen05)
    // Finalize slots [0, nslots) of S into out tables (out_block = slot) with per-slot scale.
    Status finalize(const double* S, int nslots, double scale, const std::vector<double>* slot_scale,
                    double2* out, cudaStream_t st = nullptr, bool use_slice = false);
    // Direct contraction of segs into out tables (out_block = seg.out_block).
    Status direct(const std::vector<DirectSeg>& segs, double scale, double2* out, bool accum = false);
    bool direct_host_out_ = false;  // the next direct per-frame reduce also writes frames_host_ (mapped)
    bool accum_in_direct_ = false;  // compute_frames' direct reduce also updates coh_/mag_

    // Per-frame tables for the given (k0, channel) windows -> frames_dev_ (fp64).
    // Recursive weighting when `recursive`.
    Status compute_frames(const std::vector<int64_t>& k0s, const std::vector<int>& chans, bool recursive,
                          const float2* xbase_override = nullptr, const float2* ybase_override = nullptr,
                          uint64_t mask_override = 0);
    Status emit_new_frames(cyc_frame_sink sink, void* user, double* S_target);
    Status data_error(uint64_t key, int channel, int kind, const void* xv, const void* yv, size_t n);
    Status ensure_staging();
    Status ingest_piece(const void* xv, const void* yv, size_t n, size_t off, size_t len, int kind, bool pinned);
    Status history_copy(int64_t a, int64_t b, bool save);
    // CYC_TIMELINE=1: timed events at named points of each step (reset to
    // reset), mean offsets printed at destruction (diagnostics)
    struct TlMark {
        const char* name;
        cudaEvent_t ev;
    };
    std::deque<std::vector<TlMark>> tl_steps_;
    std::vector<std::pair<std::string, std::pair<double, int>>> tl_acc_;
    void tl(const char* name, cudaStream_t s);
    void tl_resolve(bool wait);
    Status push_speculative(const void* xv, const void* yv, size_t n, int kind);
    // block_average_device: the gated device push returns without waiting for
    // its verdict; the caller checks it once after enqueuing the average
    bool defer_verdict_ = false;
    struct PendingVerdict {
        bool live = false;
        uint64_t c0 = 0, f0 = 0;
        int64_t hb = 0, hc = 0;
        const void* x = nullptr;
        const void* y = nullptr;
        size_t n = 0;
    } pv_;
    // Device-resident block push: history save, key reset, the finite scan +
    // verdict copy on vs_, the fold (reduces gated on the verdict) -- enqueued
    // directly, or replayed as one CUDA graph when the same (buffer, length,
    // stream position) repeats (the ~20 launches/copies/event edges cost ~70
    // us of host time per push; one graph launch costs a few).
    Status enqueue_gated(const void* xv, const void* yv, size_t n, int64_t hb, int64_t hc);
    Status push_gated(const void* xv, const void* yv, size_t n, int64_t hb, int64_t hc);
    struct PushGraph {
        // key
        const void* x = nullptr;
        const void* y = nullptr;
        size_t n = 0;
        uint64_t c0 = 0, f0 = 0;
        int64_t origin = 0, cap = 0;
        const float2* rx = nullptr;
        const float2* ry = nullptr;
        const double* S = nullptr;
        const float* partials = nullptr;
        bool cross = false, prof = false, clear = false;
        // state
        int seen = 0;
        bool failed = false;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        uint64_t c1 = 0, f1 = 0, launches = 0;
        std::vector<int64_t> marks;  // mark_read positions, recorded after each replay
        struct Prof {
            cudaGraphNode_t na, nb;  // event-record nodes around a profiled fold launch
            cudaEvent_t a0, b0;      // the events captured into them
            double flops, exec_flops;
            bool tensor;
        };
        std::vector<Prof> prof_recs;
    };
    std::vector<PushGraph> push_graphs_;
    // fused finite check of the current gated push (see fold_device_chunk)
    unsigned long long* chk_key_ = nullptr;
    int64_t chk_c0_ = 0;
    int chk_launches_ = 0;     // checking launches of the current push (one per segment batch)
    bool chk_fail_ = false;   // a checking launch missed some lb = 0 group
    cudaEvent_t fold_done_ev_ = nullptr;
    bool tc_interior(const FoldSeg& g, int64_t& pa, int64_t& pb) const;
    bool tc_check_plan(const std::vector<FoldSeg>& segs, int64_t& pa, int64_t& pb, bool& pending) const;
    bool capturing_ = false;
    std::vector<int64_t> cap_marks_;
    cudaEvent_t verdict_ev_ = nullptr;  // the verdict copy of the last gated push landed
    void drop_push_graph(PushGraph& g);
    Status fold_device_chunk(const float2* x, const float2* y, size_t n, double* S);
    Status deliver(size_t n_slots, const std::vector<uint64_t>& fidx, const std::vector<int>& chans,
                   cyc_frame_sink sink, void* user, bool& stop, const double2* tables);

    // CUDA-graph replay of the per-frame pipeline for small frame batches
    struct FrameGraph {
        size_t slots = 0;
        cudaGraphExec_t exec = nullptr;
        char* meta_host = nullptr;  // pinned: segs | tiles | groups | rows
        char* meta_dev = nullptr;   // device copy (captured H2D node)
        size_t meta_bytes = 0;
        FoldSeg* segs = nullptr;
        FoldTile* tiles = nullptr;
        int n_tiles = 0;
        int split = 1;  // tiles per (slot, residue block, lag block)
        bool small = false;      // one fold_small launch instead of fold + reduce
        bool zero_copy = false;  // no copy nodes: mapped descriptors in, mapped tables out
        bool fused_rec = false;  // recursive update inside the FFT (one frame per replay)
        // small graphs: static segment template in device memory (frame 0 of the
        // batch at f = 0) + a device frame offset the finalize advances per replay
        int64_t* shift_dev = nullptr;
        int64_t* shift_pin = nullptr;
        int64_t shift_expect = INT64_MIN;
        std::vector<FoldSeg> tmpl;
        double* S = nullptr;
        float* partials = nullptr;
        double2* tables_dev = nullptr;
        double2* tables_host = nullptr;  // pinned
        // small graphs: a second instance whose D2H node lands in its own pinned
        // table, so two replays can be in flight under pipelined emission
        cudaGraphExec_t exec_alt = nullptr;
        double2* tables_host_alt = nullptr;
        bool flip = false;  // the last replay used exec_alt
    };
    std::vector<FrameGraph> graphs_;
    bool graph_two_deep(size_t slots) const;
    void hprof(int phase);
    double hprof_us_[8] = {};
    double hprof_t_ = 0.0;
    uint64_t hprof_calls_ = 0;
    cudaEvent_t gev_[2] = {};
    bool graph_eligible(size_t slots) const;
    bool small_fold_ok(size_t slots) const;
    Status run_frame_graph(const std::vector<int64_t>& k0s, const std::vector<int>& chans, bool recursive,
                           double2** tables);
    void fill_frame_segs(FoldSeg* segs, const std::vector<int64_t>& k0s, const std::vector<int>& chans,
                         bool recursive) const;

    // ---- configuration ----
    Cfg c_;
    int nflags_ = 1;
    std::vector<int> lags_req_;  // output lags ascending
    int T_ = 0;
    int lag_lo_ = 0, lag_hi_ = 0;
    int f_lo_ = 0;  // fold lag origin (lag_lo_ rounded down to even)
    int m_plus_ = 0, m_minus_ = 0;
    size_t need_ = 0;
    int64_t N_ = 0;  // hop (win_len or emission interval)
    int64_t origin_ = 0;  // absolute index of local sample 0 (phase anchor offset)
    int A_ = 0;      // output alphas (Full: N bins)
    size_t layout_len_ = 0;
    int64_t stride_a_ = 0, stride_t_ = 0;

    bool use_fold_ = true;
    bool frames_direct_ = false;  // per-frame tables by the direct kernel (short Set-mode frames)
    int64_t P_ = 1, Pf_ = 1;
    std::vector<int> bins_;
    int lw_ = 8, TB_ = 64, RB_ = 128, n_rb_ = 1, n_lb_ = 1, t_pad_ = 64;
    bool use_fft_ = false;
    std::vector<uint64_t> afx_;

    // ---- device resources ----
    cudaStream_t cs_ = nullptr, xs_ = nullptr;
    cudaStream_t vs_ = nullptr;             // side stream: a device chunk's finite scan beside its fold
    cudaEvent_t reduce_wait_ev_ = nullptr;  // fold reduces wait for it (the side scan)
    float2* ring_x_ = nullptr;
    float2* ring_y_ = nullptr;  // null => auto-correlation (y = x)
    bool cross_ = false;
    int64_t cap_ = 0, Q_ = 0;
    uint64_t mask_ = 0;
    double* S_main_ = nullptr;        // block fold accumulators [channels][t_pad][Pf][4]
    // S_main_ alternates between two buffers at each reset, so a device-out
    // average's finalize (on fs_) of one block overlaps the next block's fold
    double* S_buf_[2] = {nullptr, nullptr};
    int S_cur_ = 0;
    cudaStream_t fs_ = nullptr;       // finalize stream of device-out averages
    cudaEvent_t fin_ev_[2] = {};      // last finalize that read S_buf_[i]
    bool fin_live_[2] = {};
    Status wait_finalize_reads();     // cs_ after pending finalizes of the current buffer
    bool pending_clear_ = false;      // reset's zeroing of S_main_, deferred to its next use
    Status flush_clear();
    double2* dsum_main_ = nullptr;    // block direct sums [channels][nflags][layout]
    double* S_frames_ = nullptr;      // per-frame folds
    size_t S_frames_slots_ = 0;
    double2* frames_dev_ = nullptr;   // per-frame tables [slot][nflags][layout]
    size_t frames_slots_ = 0;
    double2* frames_host_ = nullptr;  // pinned
    // frame batches in flight under pipelined emission (oldest first): the
    // tables land in pinned host memory behind `ev`; `stash` holds them once
    // that memory had to be handed on before a sink came by
    struct PendingEmit {
        cudaEvent_t ev = nullptr;
        size_t slots = 0;
        std::vector<uint64_t> fidx;
        std::vector<int> chans;
        const double2* tables = nullptr;
        bool stashed = false;
        std::vector<double2> stash;
    };
    std::deque<PendingEmit> pendq_;
    int sms_ = 148;                      // SM count of c_.device (B200: 148)
    int emit_depth_ = 0;                 // cyc_set_emit_pipeline
    double2* frames_host_alt_ = nullptr; // depth 2: the batches alternate between two pinned tables
    // depth 2, direct per-frame tables: the kernel writes a device table and a
    // copy on the side stream brings it to the host while the next push's
    // kernel runs (mapped stores would keep the kernel alive for a PCIe flush)
    double2* frames_dev_alt_ = nullptr;  // swapped with frames_dev_ beside the pinned tables
    cudaStream_t ds_ = nullptr;          // D2H side stream
    cudaEvent_t d2h_ready_ = nullptr;    // the tables are written (compute stream)
    cudaEvent_t d2h_done_[2] = {nullptr, nullptr};  // [0]: last side copy out of frames_dev_, [1]: of frames_dev_alt_
    bool d2h_busy_[2] = {false, false};
    Status side_copy_setup();
    Status wait_side_copies(bool both);  // compute stream waits before frames_dev_ (or either table) is rewritten
    Status drain_pending(cyc_frame_sink sink, void* user, size_t keep);
    Status stash_pending();
    double2* coh_ = nullptr;          // running coherent sums [channels][nflags][layout]
    double* mag_ = nullptr;           // running magnitude sums
    double2* avg_dev_ = nullptr;      // average scratch
    double2* avg_host_ = nullptr;     // pinned average readback
    double2* avg_all_dev_ = nullptr;  // all channels' tables (average_all)
    size_t avg_all_len_ = 0;
    float* partials_ = nullptr;
    size_t partials_bytes_ = 0;
    double2* tw_ = nullptr;
    int* bins_dev_ = nullptr;
    int* lags_dev_ = nullptr;
    uint64_t* afx_dev_ = nullptr;
    unsigned long long* key_dev_ = nullptr;
    unsigned long long* key_host_ = nullptr;
    float2* dev_tmp_ = nullptr;       // compute_window scratch
    size_t dev_tmp_len_ = 0;

    // pinned metadata arena (ring of slots guarded by events)
    static constexpr int META_SLOTS = 4;
    char* meta_host_ = nullptr;
    char* meta_dev_ = nullptr;
    char* meta_shadow_ = nullptr;  // device copy of the arena
    bool meta_mapped_now_ = false; // read descriptors mapped (inside pinned-host pushes)
    // the host-f32 chunk validate_host_f32 scanned: a push of exactly this
    // (pointer, length) skips its own scan; any other call clears it
    const void* prevalidated_ptr_ = nullptr;
    size_t prevalidated_n_ = 0;
    bool prestaged_ = false;       // the current one-piece push is already in stage_[stage_k_]
    size_t meta_slot_bytes_ = 0;
    size_t meta_used_ = 0;
    int meta_slot_ = 0;
    cudaEvent_t meta_ev_[META_SLOTS] = {};
    bool meta_ev_live_[META_SLOTS] = {};

    // pinned staging for pageable host input
    float2* stage_[2] = {nullptr, nullptr};
    float2* stage_y_[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev_[2] = {};
    bool stage_ev_live_[2] = {};
    size_t stage_len_ = 0;

    // Deferred ingest (small host pushes of per-frame / recursive streams):
    // each push is copied and screened into a pinned staging ring indexed by
    // absolute sample (dstage_[channel][dcap_]); the rings receive it in one
    // DMA per flush -- when frames are due, or every dflush_ samples -- instead
    // of one DMA + event edges per push (~5 us of copy-engine time and ~4 us of
    // host driver calls per 64 KB push on these hosts).
    int* direct_ctr_ = nullptr;  // fused direct reduce: per-(segment, alpha) CTA counters
    size_t direct_ctr_n_ = 0;
    float2* dstage_ = nullptr;
    float2* dstage_y_ = nullptr;
    int64_t dcap_ = 0;       // power of two, <= cap_
    int64_t dflush_ = 0;     // samples staged before an unforced flush
    int64_t dma_to_ = 0;     // absolute: staged samples below this have their DMA enqueued
    int64_t dfree_to_ = 0;   // absolute: staging below this is no longer read by a DMA
    std::deque<std::pair<int64_t, cudaEvent_t>> dma_ev_;  // (absolute end, event on xs_) per flush
    bool deferred_ok(int kind, size_t n, const void* yv) const;
    Status push_deferred(const void* xv, const void* yv, size_t n, cyc_frame_sink sink, void* user);
    Status flush_deferred();
    Status wait_dstage(int64_t abs_lo);

    // ring overwrite protection: (event, lowest absolute x index read)
    struct ReadMark {
        cudaEvent_t ev;
        int64_t lo;
    };
    std::deque<ReadMark> reads_;
    std::vector<cudaEvent_t> ev_pool_;
    cudaEvent_t get_event();
    cudaEvent_t get_event_timed();
    void mark_read(int64_t lo);
    void wait_ring_free(int64_t abs_end);
    bool xs_after_cs_ = false;  // set by reset: the next copy-stream write waits for the compute stream
    void order_copy_after_compute();

    // ---- profiling ----
    struct ProfRec {
        cudaEvent_t a, b;
        double flops;       // algorithmic: 8 per (requested lag, folded sample)
        double exec_flops;  // executed: tensor-core MMA flops (bf16x3 banded product), else = flops
        bool tensor;
    };
    bool prof_ = false;
    std::vector<ProfRec> prof_pending_;
    std::vector<cudaEvent_t> timed_pool_;
    uint64_t prof_launches_ = 0, prof_tc_launches_ = 0;
    double prof_ms_ = 0.0, prof_flops_ = 0.0, prof_exec_flops_ = 0.0;

    // speculative block pushes: pending fold + history backup for roll-back
    double* S_pend_ = nullptr;
    std::vector<char> blob_;              // host staging of one launch's descriptors
    // finalize row tables by (slot count, lag slice) (device)
    struct RowsKey {
        int nslots, b, e;
    };
    std::vector<std::pair<RowsKey, FinalRow*>> rows_cache_;
    bool clear_req_ = false;     // enqueue_gated -> fold_device_chunk: the reset's clear is due
    bool planes_fresh_ = false;  // the planes reduce overwrites (first writer of a fresh state)
    int lag_b_ = 0, lag_e_ = 0;  // block finalize lag slice [lag_b_, lag_e_) (cyc_set_lag_slice)
    std::unique_ptr<FoldInline> inline_;  // by-value descriptors of the next fold launch
    std::unique_ptr<TcParams> tcp_;       // by-value descriptors of the next tensor-core fold launch
    struct MapCache {                     // last tensor maps encoded per segment index
        const float2* x = nullptr;
        const float2* y = nullptr;
        int64_t p_base = 0, rows = 0;
        CUtensorMap xm, ym;
        bool valid = false;
    };
    MapCache map_cache_[TC_SEGS];
    // device copies of recent tensor-core tile tables: a repeated plan
    // launches with the small TcDev parameter block
    struct TileCache {
        std::vector<FoldTile> host;
        FoldTile* dev = nullptr;
        FoldTile* pin = nullptr;
        cudaEvent_t ev = nullptr;  // the upload from `pin` completed
    };
    TileCache tile_cache_[4];
    int tile_cache_next_ = 0;
    const FoldTile* cached_tiles(const FoldTile* t, int nt);
    const unsigned long long* fold_gate_ = nullptr;  // set while a device chunk folds straight into S_main
    float2* hist_bak_ = nullptr;
    size_t hist_cap_ = 0;
    int stage_k_ = 0;

    // finalize cache of the block average (frames count, channel)
    uint64_t avg_cache_frames_ = ~0ull;
    int avg_cache_channel_ = -1;

    // ---- streaming state (estimator.hpp:117-136) ----
    uint64_t consumed_ = 0;
    uint64_t frames_ = 0;
    uint64_t launches_ = 0;
    // recursive mode: running R per (channel, flag) on host, fp64
    double2* rec_R_ = nullptr;  // recursive-mode state R per (channel, flag, layout) on the device
};

}  // namespace cyc

// The opaque C-ABI handle.
struct cyc_est {
    cyc::Engine* e;
};

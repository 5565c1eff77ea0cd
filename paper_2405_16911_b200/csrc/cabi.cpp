// cabi.cpp -- extern "C" entry points of libcycb200.so (include/cycb200.h).
// Each function forwards to cyc::Engine and converts its Status into the
// reference's error convention (proj/include/cycstat/errors.hpp).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "engine.h"


namespace {

void write_err(char* buf, size_t len, const std::string& msg) {
    if (!buf || !len) return;
    std::strncpy(buf, msg.c_str(), len - 1);
    buf[len - 1] = 0;
}

int finish(cyc_est* est, const cyc::Status& s) {
    if (est) {
        est->e->last_error = s.msg;
        est->e->last_error_index = s.index;
    }
    return s.code;
}

}  // namespace

extern "C" {

int cyc_abi_version(void) { return CYC_ABI_VERSION; }

const char* cyc_build_info(void) {
    return "libcycb200 sm_100a; kernels: fold(FFMA2, cp.async), finalize(fp64 FFT/DFT), direct(fixed-point phase)";
}

void cyc_config_init(cyc_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->mode = CYC_MODE_SET;
    cfg->lag_symmetric = 1;
    cfg->emit_frames = 1;
    cfg->channels = 1;
}

int cyc_validate(const cyc_config* cfg, char* buf, size_t buflen) {
    if (!cfg) return -1;
    const auto v = cyc::validate(cyc::from_c(cfg));
    std::string s;
    for (const auto& e : v) s += e + "\n";
    write_err(buf, buflen, s);
    return (int)v.size();
}

int cyc_create(const cyc_config* cfg, cyc_est** out, char* err, size_t errlen) {
    if (!cfg || !out) {
        write_err(err, errlen, "null argument");
        return CYC_ERR_USAGE;
    }
    cyc::Engine* e = nullptr;
    cyc::Status s = cyc::Engine::create(cyc::from_c(cfg), &e);
    if (s.code) {
        write_err(err, errlen, s.msg);
        *out = nullptr;
        return s.code;
    }
    *out = new cyc_est{e};
    write_err(err, errlen, "");
    return CYC_OK;
}

void cyc_destroy(cyc_est* est) {
    if (!est) return;
    delete est->e;
    delete est;
}

int cyc_push(cyc_est* est, const cyc_cf32* x, const cyc_cf32* y, size_t n, cyc_frame_sink sink, void* user) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->push(x, y, n, cyc::Engine::IN_HOST_F32, sink, user));
}

int cyc_push_f64(cyc_est* est, const cyc_cf64* x, const cyc_cf64* y, size_t n, cyc_frame_sink sink, void* user) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->push(x, y, n, cyc::Engine::IN_HOST_F64, sink, user));
}

int cyc_push_device(cyc_est* est, const cyc_cf32* d_x, const cyc_cf32* d_y, size_t n, cyc_frame_sink sink,
                    void* user) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->push(d_x, d_y, n, cyc::Engine::IN_DEVICE_F32, sink, user));
}

int cyc_block_average_device(cyc_est* est, const cyc_cf32* d_x, const cyc_cf32* d_y, size_t n, int avg_mode,
                             cyc_cf64* out) {
    if (!est || !out) return CYC_ERR_USAGE;
    return finish(est, est->e->block_average_device(d_x, d_y, n, avg_mode, out));
}

int cyc_average(cyc_est* est, int avg_mode, int flag, int channel, cyc_cf64* out) {
    if (!est || !out) return CYC_ERR_USAGE;
    return finish(est, est->e->average(avg_mode, flag, channel, out));
}

size_t cyc_buffer_need(const cyc_est* est) { return est ? est->e->buffer_need() : 0; }
uint64_t cyc_consumed(const cyc_est* est) { return est ? est->e->consumed() : 0; }
uint64_t cyc_frames_emitted(const cyc_est* est) { return est ? est->e->frames_emitted() : 0; }
int cyc_num_flags(const cyc_est* est) { return est ? est->e->num_flags() : 0; }

int cyc_layout(const cyc_est* est, cyc_layout_info* out) {
    if (!est || !out) return CYC_ERR_USAGE;
    est->e->layout(out);
    return CYC_OK;
}

const char* cyc_last_error(const cyc_est* est) { return est ? est->e->last_error.c_str() : ""; }
int64_t cyc_data_error_index(const cyc_est* est) { return est ? est->e->last_error_index : -1; }

int cyc_synchronize(cyc_est* est) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->synchronize());
}

void* cyc_stream(cyc_est* est) { return est ? (void*)est->e->stream() : nullptr; }
uint64_t cyc_kernel_launches(const cyc_est* est) { return est ? est->e->launches() : 0; }

int cyc_algorithm(const cyc_est* est, char* buf, size_t buflen) {
    if (!est) return CYC_ERR_USAGE;
    write_err(buf, buflen, est->e->algorithm());
    return CYC_OK;
}

void* cyc_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void cyc_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"

namespace {
// One-shot windows (kernels.cpp:116-135) reuse the engines of the last few
// geometries per thread: the set-up costs far more than one window.  The
// cache is a thread_local object: a worker thread's engines (device memory,
// pinned staging) are freed when the thread exits.
cyc::Status cached_window_engine(const cyc::Cfg& g, cyc::Engine** out) {
    struct Entry {
        cyc::Cfg cfg;
        cyc::Engine* e;
    };
    struct Cache : std::vector<Entry> {
        ~Cache() {
            for (auto& en : *this) delete en.e;
        }
    };
    static thread_local Cache cache_obj;
    Cache* cache = &cache_obj;
    auto same = [](const cyc::Cfg& a, const cyc::Cfg& b) {
        return a.mode == b.mode && a.flags == b.flags && a.win_len == b.win_len && a.alphas == b.alphas &&
               a.lag_symmetric == b.lag_symmetric && a.max_lag == b.max_lag && a.lags == b.lags &&
               a.lambda == b.lambda && a.emit_frames == b.emit_frames && a.channels == b.channels &&
               a.device == b.device && a.origin == b.origin;
    };
    for (size_t i = 0; i < cache->size(); ++i)
        if (same((*cache)[i].cfg, g)) {
            *out = (*cache)[i].e;
            return cyc::Status::ok();
        }
    cyc::Engine* e = nullptr;
    cyc::Status s = cyc::Engine::create_unchecked(g, &e);
    if (s.code) return s;
    if (cache->size() >= 4) {
        delete cache->front().e;
        cache->erase(cache->begin());
    }
    cache->push_back({g, e});
    *out = e;
    return s;
}
}  // namespace

extern "C" {

int cyc_compute_set_window(const cyc_cf64* xw, size_t xw_len, const cyc_cf64* yw, size_t yw_len,
                           const double* alphas, size_t num_alphas, int max_lag, int conj, uint64_t k0,
                           cyc_cf64* out, char* err, size_t errlen) {
    // kernels.cpp:116-123: window-length mismatch is a caller bug (logic_error)
    if (!xw || !yw || !out || yw_len == 0 || max_lag < 0 || xw_len != yw_len + 2u * (size_t)max_lag) {
        write_err(err, errlen, "window lengths do not match the lag range");
        return CYC_ERR_INTERNAL;
    }
    cyc_config c;
    cyc_config_init(&c);
    c.mode = CYC_MODE_SET;
    c.conj = conj;
    c.win_len = (int)yw_len;
    c.alphas = alphas;
    c.num_alphas = num_alphas;
    c.lag_symmetric = 1;
    c.max_lag = max_lag;
    cyc::Cfg g = cyc::from_c(&c);
    if (g.win_len < 2) g.win_len = 2;  // one-shot windows skip the streaming span rule
    cyc::Engine* e = nullptr;
    // the one-shot kernel has no win_len > 2*max_lag requirement (kernels.cpp:13-25)
    cyc::Status s;
    {
        auto v = cyc::validate(g);
        bool only_span = !v.empty();
        for (auto& m : v)
            if (m != "win_len must exceed twice the largest |lag|" && m != "win_len must be at least 2") only_span = false;
        if (!v.empty() && !only_span) {
            write_err(err, errlen, "bad Set-mode window geometry");
            return CYC_ERR_INTERNAL;
        }
    }
    s = cached_window_engine(g, &e);
    if (s.code) {
        write_err(err, errlen, s.msg);
        return s.code;
    }
    s = e->compute_window(xw, xw_len, yw, yw_len, k0, out);
    write_err(err, errlen, s.msg);
    return s.code;
}

int cyc_compute_full_window(const cyc_cf64* xw, size_t xw_len, const cyc_cf64* yw, size_t yw_len, const int* lags,
                            size_t num_lags, int conj, uint64_t k0, cyc_cf64* out, char* err, size_t errlen) {
    if (!xw || !yw || !out || yw_len == 0 || !lags || num_lags == 0) {
        write_err(err, errlen, "empty estimation window");
        return CYC_ERR_INTERNAL;
    }
    int mp = 0, mm = 0;
    for (size_t i = 0; i < num_lags; ++i) {
        mp = std::max(mp, lags[i]);
        mm = std::max(mm, -lags[i]);
    }
    if (xw_len != yw_len + (size_t)mp + (size_t)mm) {
        write_err(err, errlen, "window does not cover the requested lags");
        return CYC_ERR_INTERNAL;
    }
    cyc_config c;
    cyc_config_init(&c);
    c.mode = CYC_MODE_FULL;
    c.conj = conj;
    c.win_len = (int)yw_len;
    c.lag_symmetric = 0;
    c.lags = lags;
    c.num_lags = num_lags;
    cyc::Cfg g = cyc::from_c(&c);
    cyc::Engine* e = nullptr;
    cyc::Status s = cached_window_engine(g, &e);
    if (s.code) {
        write_err(err, errlen, s.msg);
        return s.code;
    }
    s = e->compute_window(xw, xw_len, yw, yw_len, k0, out);
    write_err(err, errlen, s.msg);
    return s.code;
}

}  // extern "C"

namespace cyc {
double measure_fp32_peak_tflops(int device);
}

extern "C" {

int cyc_reset(cyc_est* est) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->reset());
}

int cyc_profile_enable(cyc_est* est, int on) {
    if (!est) return CYC_ERR_USAGE;
    est->e->set_profiling(on != 0);
    return CYC_OK;
}

int cyc_profile_read(cyc_est* est, uint64_t* launches, double* ms, double* flops) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->profile_read(launches, ms, flops));
}

int cyc_profile_read_ex(cyc_est* est, uint64_t* launches, double* ms, double* flops, double* exec_flops,
                        uint64_t* tensor_launches) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->profile_read(launches, ms, flops, exec_flops, tensor_launches));
}

double cyc_measure_fp32_peak(int device) { return cyc::measure_fp32_peak_tflops(device); }

}  // extern "C"

extern "C" int cyc_plan(const cyc_config* cfg, char* buf, size_t buflen) {
    if (!cfg) return CYC_ERR_USAGE;
    const cyc::Cfg g = cyc::from_c(cfg);
    const auto v = cyc::validate(g);
    if (!v.empty()) {
        std::string s = "invalid config:";
        for (auto& e : v) s += " [" + e + "]";
        write_err(buf, buflen, s);
        return CYC_ERR_CONFIG;
    }
    write_err(buf, buflen, cyc::Engine::plan_string(g));
    return CYC_OK;
}

extern "C" int cyc_fold_state(cyc_est* est, void** dev_ptr, size_t* count, uint64_t* frames) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->fold_state(dev_ptr, count, frames));
}

extern "C" int cyc_fold_set_frames(cyc_est* est, uint64_t frames) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->set_frames(frames));
}

extern "C" int cyc_set_lag_slice(cyc_est* est, uint32_t lag_begin, uint32_t lag_end) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->set_lag_slice(lag_begin, lag_end));
}

extern "C" int cyc_set_emit_pipeline(cyc_est* est, int depth) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->set_emit_pipeline(depth));
}

extern "C" int cyc_flush_frames(cyc_est* est, cyc_frame_sink sink, void* user) {
    if (!est) return CYC_ERR_USAGE;
    return finish(est, est->e->flush_frames(sink, user));
}

extern "C" int cyc_average_all(cyc_est* est, int avg_mode, cyc_cf64* out) {
    if (!est || !out) return CYC_ERR_USAGE;
    return finish(est, est->e->average_all(avg_mode, out));
}

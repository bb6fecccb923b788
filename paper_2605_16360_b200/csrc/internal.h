// internal.h — host-side runtime shared by the C-ABI translation units:
// context, error state, workspaces, kernel launch entry points.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <atomic>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pkv_capi.h"

namespace pkv {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);

struct Error {
    pkv_status code;
    std::string msg;
};

template <typename... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}

#define PKV_REQUIRE(cond, code, ...)                                      \
    do {                                                                  \
        if (!(cond)) throw ::pkv::Error{code, ::pkv::cat(__VA_ARGS__)};   \
    } while (0)
#define PKV_REQUIRE_SHAPE(cond, ...) PKV_REQUIRE(cond, PKV_ESHAPE, __VA_ARGS__)
#define PKV_REQUIRE_VALUE(cond, ...) PKV_REQUIRE(cond, PKV_EVALUE, __VA_ARGS__)
#define PKV_CUDA(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            throw ::pkv::Error{PKV_ECUDA, ::pkv::cat(#expr, ": ", cudaGetErrorString(e_))};     \
    } while (0)

// Runs f, translating pkv::Error / std exceptions into a status + message.
template <typename F>
pkv_status guard(F&& f) {
    try {
        f();
        return PKV_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PKV_ECUDA;
    }
}

// -------------------------------------------------------------- workspace
// Grow-only device scratch buffer (stream-ordered users must not overlap).
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void* get(size_t need);
    void release();
    ~DevBuf() { release(); }
};

}  // namespace pkv

struct pkv_ctx_s {
    int device = 0;
    int sm_count = 148;
    std::atomic<int64_t> launches{0};
    pkv::DevBuf scratch_select;
    pkv::DevBuf scratch_host_io;
    pkv::DevBuf scratch_score;
    pkv::DevBuf scratch_decode;
    pkv::DevBuf scratch_metrics;
    pkv::DevBuf scratch_score_aux;  // fixed-reference pass 1: max |k| + tile flags
};

namespace pkv {

void require_ctx(pkv_ctx ctx);

// One-time setup per (call site, device): kernel attributes such as the
// dynamic shared-memory limit are per device, so a process driving several
// GPUs (the two-device mode, one host thread per GPU) must set them on each.
inline bool first_on_device(std::atomic<uint64_t>& done) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    return (done.fetch_or(bit) & bit) == 0;
}
inline void count_launch(pkv_ctx ctx, int n = 1) { ctx->launches += n; }

// NVTX range for one stage of the path (per-stage ranges for
// nsys / ncu --nvtx). Header-only NVTX v3: a no-op unless a tool injects.
struct StageRange {
    explicit StageRange(const char* name) { nvtxRangePushA(name); }
    ~StageRange() { nvtxRangePop(); }
    StageRange(const StageRange&) = delete;
    StageRange& operator=(const StageRange&) = delete;
};
void check_launch(const char* what);

// ---------------------------------------------------------- kernel entries
void launch_topk_select(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                        cudaStream_t st);
// Streaming select with candidate compaction (select_stream.cu), taken by
// launch_topk_select for long L2-resident rows (select_stream_eligible).
bool select_stream_eligible(int64_t slices, int64_t n);
void launch_topk_select_stream(const float* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask,
                               int32_t* idx, cudaStream_t st);
void launch_topk_select_f64(const double* scores, int64_t slices, int64_t n, int64_t k, uint8_t* mask, int32_t* idx,
                            cudaStream_t st);
void launch_compact_kv(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n, int64_t k,
                       int64_t row_bytes, void* kout, void* vout, int sm_count, cudaStream_t st);
// paged destination: slice s's output row j -> page table[s * max_blocks + j / page], row j % page
void launch_compact_kv_paged(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n,
                             int64_t k, int64_t row_bytes, void* k_pool, void* v_pool, const int32_t* table,
                             int64_t max_blocks, int64_t page, int sm_count, cudaStream_t st);

// TMA descriptor encoding through the driver entry point (no -lcuda needed).
CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                         CUtensorMapSwizzle swz);
CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dt, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2,
                         CUtensorMapSwizzle swz);

}  // namespace pkv

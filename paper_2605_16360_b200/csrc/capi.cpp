// capi.cpp — C-ABI runtime: context, errors, select / compaction entry
// points, TMA descriptor encoding. See include/pkv_capi.h for the contract.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace pkv {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

void* DevBuf::get(size_t need) {
    if (need <= bytes && ptr) return ptr;
    release();
    const size_t sz = need < 256 ? 256 : need;
    PKV_CUDA(cudaMalloc(&ptr, sz));
    bytes = sz;
    return ptr;
}

void DevBuf::release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
}

void require_ctx(pkv_ctx ctx) { PKV_REQUIRE(ctx != nullptr, PKV_EVALUE, "null pkv_ctx"); }

void check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error{PKV_ECUDA, cat(what, " launch failed: ", cudaGetErrorString(e))};
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        }
    });
    PKV_REQUIRE(fn != nullptr, PKV_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}
}  // namespace

CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    PKV_REQUIRE(r == CUDA_SUCCESS, PKV_ECUDA, "cuTensorMapEncodeTiled(2d) failed: ", (int)r, " dims ", inner, "x",
                outer, " stride ", row_stride_bytes, " box ", box_inner, "x", box_outer);
    return m;
}

CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dt, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2,
                         CUtensorMapSwizzle swz) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    PKV_REQUIRE(r == CUDA_SUCCESS, PKV_ECUDA, "cuTensorMapEncodeTiled(3d) failed: ", (int)r);
    return m;
}

}  // namespace pkv

using namespace pkv;

extern "C" {

int pkv_abi_version(void) { return 1; }

const char* pkv_last_error(void) { return g_last_error.c_str(); }

int pkv_sm100_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int c = 0;
    for (int i = 0; i < n; ++i) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10) ++c;
    }
    return c;
}

pkv_status pkv_ctx_create(int device, pkv_ctx* out) {
    return guard([&] {
        PKV_REQUIRE(out != nullptr, PKV_EVALUE, "null output pointer");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw Error{PKV_ENODEV, "no CUDA device visible; the B200 path has no CPU fallback"};
        }
        PKV_REQUIRE(device >= 0 && device < n, PKV_EVALUE, "device ", device, " out of range [0, ", n, ")");
        cudaDeviceProp p;
        PKV_CUDA(cudaGetDeviceProperties(&p, device));
        if (p.major != 10) throw Error{PKV_ENODEV, cat("device ", device, " is sm_", p.major, p.minor, "; need sm_100")};
        PKV_CUDA(cudaSetDevice(device));
        auto* c = new pkv_ctx_s();
        c->device = device;
        c->sm_count = p.multiProcessorCount;
        *out = c;
    });
}

void pkv_ctx_destroy(pkv_ctx ctx) { delete ctx; }

int64_t pkv_ctx_launch_count(pkv_ctx ctx) { return ctx ? ctx->launches.load() : 0; }

pkv_status pkv_retention_count(double rho, int64_t n, int64_t* k_out) {
    return guard([&] {
        // pruning.cpp:15-17
        PKV_REQUIRE_VALUE(rho > 0.0 && rho <= 1.0, "retention ratio must be in (0, 1], got ", rho);
        PKV_REQUIRE_VALUE(n > 0, "empty token axis");
        *k_out = static_cast<int64_t>(std::ceil(rho * static_cast<double>(n)));
    });
}

pkv_status pkv_topk_select(pkv_ctx ctx, const float* scores_dev, int64_t slices, int64_t n, int64_t k,
                           uint8_t* mask_dev, int32_t* idx_asc_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices >= 0 && n > 0, "topk_select needs n > 0, got n=", n);
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);
        PKV_REQUIRE_VALUE(n < (int64_t(1) << 31), "token axis too long: ", n);
        launch_topk_select(scores_dev, slices, n, k, mask_dev, idx_asc_dev, static_cast<cudaStream_t>(stream));
        count_launch(ctx);
    });
}

pkv_status pkv_topk_select_f64(pkv_ctx ctx, const double* scores_dev, int64_t slices, int64_t n, int64_t k,
                               uint8_t* mask_dev, int32_t* idx_asc_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices >= 0 && n > 0, "topk_select needs n > 0, got n=", n);
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);
        PKV_REQUIRE_VALUE(n < (int64_t(1) << 31), "token axis too long: ", n);
        launch_topk_select_f64(scores_dev, slices, n, k, mask_dev, idx_asc_dev, static_cast<cudaStream_t>(stream));
        count_launch(ctx);
    });
}

pkv_status pkv_topk_mask_host(pkv_ctx ctx, const double* scores_host, int64_t slices, int64_t n, double rho,
                              uint8_t* bits_host, int64_t* k_out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "topk_mask needs a shaped tensor");
        PKV_REQUIRE_VALUE(rho > 0.0 && rho <= 1.0, "retention ratio must be in (0, 1], got ", rho);
        PKV_REQUIRE_VALUE(n < (int64_t(1) << 31), "token axis too long: ", n);
        const int64_t k = static_cast<int64_t>(std::ceil(rho * static_cast<double>(n)));
        const size_t numel = static_cast<size_t>(slices * n);
        // the doubles go over as they are: 64-bit order keys rank them exactly
        auto* dev = static_cast<uint8_t*>(ctx->scratch_host_io.get(numel * 9));
        double* d_scores = reinterpret_cast<double*>(dev);
        uint8_t* d_mask = dev + numel * 8;
        PKV_CUDA(cudaMemcpy(d_scores, scores_host, numel * 8, cudaMemcpyHostToDevice));
        launch_topk_select_f64(d_scores, slices, n, k, d_mask, nullptr, nullptr);
        count_launch(ctx);
        PKV_CUDA(cudaMemcpy(bits_host, d_mask, numel, cudaMemcpyDeviceToHost));
        *k_out = k;
    });
}

pkv_status pkv_topk_indices_host(pkv_ctx ctx, const double* values_host, int64_t n, int64_t k, int64_t* idx_out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);  // pruning.cpp:21
        PKV_REQUIRE_VALUE(n < (int64_t(1) << 31), "token axis too long: ", n);
        const size_t un = static_cast<size_t>(n), uk = static_cast<size_t>(k);
        auto* dev = static_cast<uint8_t*>(ctx->scratch_host_io.get(un * 8 + uk * 4));
        double* d_v = reinterpret_cast<double*>(dev);
        int32_t* d_idx = reinterpret_cast<int32_t*>(dev + un * 8);
        PKV_CUDA(cudaMemcpy(d_v, values_host, un * 8, cudaMemcpyHostToDevice));
        launch_topk_select_f64(d_v, 1, n, k, nullptr, d_idx, nullptr);
        count_launch(ctx);
        std::vector<int32_t> h(uk);
        PKV_CUDA(cudaMemcpy(h.data(), d_idx, uk * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < uk; ++i) idx_out[i] = h[i];
    });
}

pkv_status pkv_topk_overlap_host(pkv_ctx ctx, const uint8_t* a_host, const uint8_t* b_host, int64_t slices, int64_t n,
                                 int64_t k, double* per_slice_out) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices > 0 && n > 0, "topk_overlap extents must be positive");
        const size_t m = static_cast<size_t>(slices * n);
        auto* dev = static_cast<uint8_t*>(ctx->scratch_host_io.get(2 * m + 8 * static_cast<size_t>(slices) + 16));
        uint8_t* d_a = dev;
        uint8_t* d_b = dev + m;
        double* d_o = reinterpret_cast<double*>(dev + ((2 * m + 15) & ~size_t(15)));
        PKV_CUDA(cudaMemcpy(d_a, a_host, m, cudaMemcpyHostToDevice));
        PKV_CUDA(cudaMemcpy(d_b, b_host, m, cudaMemcpyHostToDevice));
        const pkv_status st = pkv_topk_overlap(ctx, d_a, d_b, slices, n, k, d_o, nullptr);
        if (st != PKV_OK) throw Error{st, pkv_last_error()};
        PKV_CUDA(cudaMemcpy(per_slice_out, d_o, 8 * static_cast<size_t>(slices), cudaMemcpyDeviceToHost));
    });
}

pkv_status pkv_compact_kv(pkv_ctx ctx, const void* k_in_dev, const void* v_in_dev, const int32_t* idx_asc_dev,
                          int64_t slices, int64_t n, int64_t k, int64_t d, int64_t elem_bytes, void* k_out_dev,
                          void* v_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices >= 0 && n > 0 && d > 0, "compact_kv extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);
        PKV_REQUIRE_VALUE(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4, "elem_bytes must be 1, 2 or 4");
        PKV_REQUIRE_VALUE((d * elem_bytes) % 2 == 0, "row bytes must be even");
        launch_compact_kv(k_in_dev, v_in_dev, idx_asc_dev, slices, n, k, d * elem_bytes, k_out_dev, v_out_dev,
                          ctx->sm_count, static_cast<cudaStream_t>(stream));
        count_launch(ctx);
    });
}

pkv_status pkv_select_compact(pkv_ctx ctx, const float* scores_dev, int64_t slices, int64_t n, int64_t k,
                              const void* k_in_dev, const void* v_in_dev, int64_t d, int64_t elem_bytes,
                              int32_t* idx_asc_dev, void* k_out_dev, void* v_out_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices >= 0 && n > 0 && d > 0, "select_compact extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);
        PKV_REQUIRE_VALUE(n < (int64_t(1) << 31), "token axis too long: ", n);
        PKV_REQUIRE_VALUE(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4, "elem_bytes must be 1, 2 or 4");
        PKV_REQUIRE_VALUE((d * elem_bytes) % 2 == 0, "row bytes must be even");
        PKV_REQUIRE_VALUE(idx_asc_dev != nullptr, "select_compact needs the index output");
        auto st = static_cast<cudaStream_t>(stream);
        launch_topk_select(scores_dev, slices, n, k, nullptr, idx_asc_dev, st);
        launch_compact_kv(k_in_dev, v_in_dev, idx_asc_dev, slices, n, k, d * elem_bytes, k_out_dev, v_out_dev,
                          ctx->sm_count, st);
        count_launch(ctx, 2);
    });
}

pkv_status pkv_compact_kv_paged(pkv_ctx ctx, const void* k_in_dev, const void* v_in_dev, const int32_t* idx_asc_dev,
                                int64_t slices, int64_t n, int64_t k, int64_t d, int64_t elem_bytes,
                                const int32_t* block_table_dev, int64_t max_blocks, int64_t page_size,
                                void* k_pool_dev, void* v_pool_dev, void* stream) {
    return guard([&] {
        require_ctx(ctx);
        PKV_REQUIRE_SHAPE(slices >= 0 && n > 0 && d > 0, "compact_kv extents must be positive");
        PKV_REQUIRE_VALUE(k >= 1 && k <= n, "top-k count ", k, " out of range for length ", n);
        PKV_REQUIRE_VALUE(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4, "elem_bytes must be 1, 2 or 4");
        PKV_REQUIRE_VALUE((d * elem_bytes) % 2 == 0, "row bytes must be even");
        PKV_REQUIRE_VALUE(block_table_dev != nullptr && page_size > 0, "paged compaction needs a block table");
        PKV_REQUIRE_VALUE(max_blocks * page_size >= k, "block table too short: ", max_blocks, " pages of ",
                          page_size, " rows < k = ", k);
        launch_compact_kv_paged(k_in_dev, v_in_dev, idx_asc_dev, slices, n, k, d * elem_bytes, k_pool_dev,
                                v_pool_dev, block_table_dev, max_blocks, page_size, ctx->sm_count,
                                static_cast<cudaStream_t>(stream));
        count_launch(ctx);
    });
}

}  // extern "C"

// ------------------------------------------------------------- scoring ----
#include "score.cuh"

extern "C" {

pkv_status pkv_score(pkv_ctx ctx, const void* q_dev, const void* k_dev, int64_t L, int64_t Hq, int64_t Hkv,
                     int64_t Nq, int64_t Nk, int64_t d, uint32_t flags, const float* lse_dev, float* x_out_dev,
                     void* stream) {
    return pkv::guard([&] {
        pkv::require_ctx(ctx);
        pkv::ScoreShape s{L, Hq, Hkv, Nq, Nk, d, (flags & PKV_SCORE_CAUSAL) != 0};
        pkv::score_validate(s);
        auto st = static_cast<cudaStream_t>(stream);
        auto* lam = static_cast<__nv_bfloat16*>(ctx->scratch_score.get((size_t)(L * Hq * Nq) * 16));
        if (lse_dev) {
            pkv::launch_lam_from_lse(lse_dev, L * Hq * Nq, d, lam, st);
        } else {
            pkv::launch_score_lse(s, q_dev, k_dev, nullptr, lam, st, &ctx->scratch_score_aux);
        }
        pkv::launch_score_pool(s, q_dev, k_dev, lam, (flags & PKV_SCORE_REDUCE_SUM) == 0, x_out_dev, st);
        pkv::count_launch(ctx, 2);
    });
}

pkv_status pkv_score_lse(pkv_ctx ctx, const void* q_dev, const void* k_dev, int64_t L, int64_t Hq, int64_t Hkv,
                         int64_t Nq, int64_t Nk, int64_t d, uint32_t flags, float* lse_out_dev, void* stream) {
    return pkv::guard([&] {
        pkv::require_ctx(ctx);
        pkv::ScoreShape s{L, Hq, Hkv, Nq, Nk, d, (flags & PKV_SCORE_CAUSAL) != 0};
        pkv::score_validate(s);
        pkv::launch_score_lse(s, q_dev, k_dev, lse_out_dev, nullptr, static_cast<cudaStream_t>(stream),
                              &ctx->scratch_score_aux);
        pkv::count_launch(ctx);
    });
}

}  // extern "C"

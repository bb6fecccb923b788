// compact.cu — KV-cache compaction: coalesced, 128-bit vectorised gather of
// the retained K/V rows into a packed cache, in apply_mask's ascending order
// (proj/src/pruning.cpp:197-215 defines the order; the reference has no
// gather — "no real KV cache exists at desk scale").
//
//   out[s, j, :] = in[s, idx_asc[s, j], :]   for K and V
//
// HBM-bound: every byte of the K retained rows is read once and written once.
// Persistent grid (a few CTAs per SM); each thread keeps kUnroll 16-byte loads
// of K and of V in flight before storing (streaming cache hints on both).
#include "internal.h"

namespace pkv {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

template <typename VT>
__device__ __forceinline__ VT ld_stream(const VT* p) {
    return __ldcs(p);
}
template <>
__device__ __forceinline__ uint16_t ld_stream<uint16_t>(const uint16_t* p) {
    return __ldcs(reinterpret_cast<const unsigned short*>(p));
}
template <typename VT>
__device__ __forceinline__ void st_stream(VT* p, const VT& v) {
    __stcs(p, v);
}
template <>
__device__ __forceinline__ void st_stream<uint16_t>(uint16_t* p, const uint16_t& v) {
    __stcs(reinterpret_cast<unsigned short*>(p), v);
}

// Vector element e of the packed output lives in output row e / row_vec; that
// row is source row (row / k) * n + idx[row] of the input. Paged destination:
// output row j of slice s goes to page table[s·max_blocks + j / page] at row
// j % page (pools of [pages, page, row] elements).
struct PagedDst {
    const int32_t* table = nullptr;
    int64_t max_blocks = 0, page = 0;
};

template <typename VT, bool kPaged>
__global__ void __launch_bounds__(kThreads)
    compact_kv_kernel(const VT* __restrict__ kin, const VT* __restrict__ vin, const int32_t* __restrict__ idx,
                      int64_t n, int64_t k, uint32_t row_vec, int64_t total, VT* __restrict__ kout,
                      VT* __restrict__ vout, PagedDst pg) {
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t base = (int64_t)blockIdx.x * kThreads + threadIdx.x; base < total; base += stride * kUnroll) {
        VT kv[kUnroll], vv[kUnroll];
        int64_t dst[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t e = base + u * stride;
            dst[u] = e;
            if (e < total) {
                const int64_t row = e / row_vec;
                const uint32_t c = (uint32_t)(e - row * row_vec);
                const int64_t s = row / k;
                const int64_t src = (s * n + __ldg(idx + row)) * row_vec + c;
                kv[u] = ld_stream(kin + src);
                vv[u] = ld_stream(vin + src);
                if (kPaged) {
                    const int64_t j = row - s * k;
                    const int64_t page = __ldg(pg.table + s * pg.max_blocks + j / pg.page);
                    dst[u] = (page * pg.page + j % pg.page) * row_vec + c;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (base + u * stride < total) {
                st_stream(kout + dst[u], kv[u]);
                st_stream(vout + dst[u], vv[u]);
            }
        }
    }
}

template <typename VT>
void launch_typed(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n, int64_t k,
                  int64_t row_bytes, void* kout, void* vout, int sm_count, cudaStream_t st, const PagedDst& pg) {
    const uint32_t row_vec = (uint32_t)(row_bytes / sizeof(VT));
    const int64_t total = slices * k * row_vec;
    if (total == 0) return;
    int64_t blocks = (total + (int64_t)kThreads * kUnroll - 1) / ((int64_t)kThreads * kUnroll);
    const int64_t cap = (int64_t)sm_count * 8;
    if (blocks > cap) blocks = cap;
    auto kern = pg.table ? compact_kv_kernel<VT, true> : compact_kv_kernel<VT, false>;
    kern<<<(unsigned)blocks, kThreads, 0, st>>>(static_cast<const VT*>(kin), static_cast<const VT*>(vin), idx, n, k,
                                               row_vec, total, static_cast<VT*>(kout), static_cast<VT*>(vout), pg);
    check_launch("compact_kv_kernel");
}

}  // namespace

namespace {
void launch_any(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n, int64_t k,
                int64_t row_bytes, void* kout, void* vout, int sm_count, cudaStream_t st, const PagedDst& pg) {
    const uintptr_t align = (uintptr_t)kin | (uintptr_t)vin | (uintptr_t)kout | (uintptr_t)vout;
    if (row_bytes % 16 == 0 && align % 16 == 0) {
        launch_typed<uint4>(kin, vin, idx, slices, n, k, row_bytes, kout, vout, sm_count, st, pg);
    } else if (row_bytes % 8 == 0 && align % 8 == 0) {
        launch_typed<uint2>(kin, vin, idx, slices, n, k, row_bytes, kout, vout, sm_count, st, pg);
    } else if (row_bytes % 4 == 0 && align % 4 == 0) {
        launch_typed<uint32_t>(kin, vin, idx, slices, n, k, row_bytes, kout, vout, sm_count, st, pg);
    } else {
        launch_typed<uint16_t>(kin, vin, idx, slices, n, k, row_bytes, kout, vout, sm_count, st, pg);
    }
}
}  // namespace

void launch_compact_kv(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n, int64_t k,
                       int64_t row_bytes, void* kout, void* vout, int sm_count, cudaStream_t st) {
    launch_any(kin, vin, idx, slices, n, k, row_bytes, kout, vout, sm_count, st, PagedDst{});
}

void launch_compact_kv_paged(const void* kin, const void* vin, const int32_t* idx, int64_t slices, int64_t n,
                             int64_t k, int64_t row_bytes, void* k_pool, void* v_pool, const int32_t* table,
                             int64_t max_blocks, int64_t page, int sm_count, cudaStream_t st) {
    launch_any(kin, vin, idx, slices, n, k, row_bytes, k_pool, v_pool, sm_count, st, PagedDst{table, max_blocks, page});
}

}  // namespace pkv

// mapper.h — host-side HybridAxialMapper state (see mapper.cpp).
#pragma once
#include <cuda_fp16.h>

#include <cstdlib>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "gemm.cuh"
#include "internal.h"
#include "mapper_kernels.cuh"

namespace pkv {

// ModelGeometry, proj/include/proxykv/mapper.hpp:16-25
struct Geometry {
    int64_t target_layers = 32, target_heads = 32, proxy_layers = 16, proxy_heads = 32, head_dim = 128;
    static Geometry from5(const int64_t* g);
    void validate() const;
};

// MapperConfig, proj/include/proxykv/mapper.hpp:35-55
struct Config {
    int64_t d_time = 512, encoder_layers = 6, encoder_heads = 8, ffn_mult = 4, d_head = 64, crop_len = 2048,
            stride = 1024, synthetic_heads = 0;
    bool conv_active = true, enc_active = true, cross_active = true, normalize_input = false;
    static Config from12(const int64_t* c);
    void validate() const;
    int64_t conv_mid() const { return d_time / 2 > 0 ? d_time / 2 : 1; }
    int64_t syn(const Geometry& g) const { return synthetic_heads > 0 ? synthetic_heads : g.proxy_heads; }
};

int64_t layer_pair(int64_t ll, const Geometry& g);
std::vector<int64_t> window_offsets(int64_t n, int64_t crop, int64_t stride);
std::vector<std::pair<std::string, int64_t>> param_layout(const Geometry& g, const Config& c);
std::vector<double> init_params(const Geometry& g, const Config& c, uint64_t seed);

struct WeightPlanes {
    __half* hi = nullptr;
    __half* lo = nullptr;
    int64_t N = 0, K = 0;  // B operand [N, K], K-major
    // FP16F8 (precision 6): hi = fp16(W·2^w), e4m3 planes h8 = hi / lo_mul, l8 = (W·2^w − hi) / hi_mul
    uint8_t* h8 = nullptr;
    uint8_t* l8 = nullptr;
    float acc_scale = 1.0f;  // 2^-w
    F8Class cls{};
};

struct Block {
    WeightPlanes qkv, o, f1, f2;
    float *qkv_b = nullptr, *o_b = nullptr, *f1_b = nullptr, *f2_b = nullptr;
    float *ln1_g = nullptr, *ln1_b = nullptr, *ln2_g = nullptr, *ln2_b = nullptr;
};

class Mapper {
public:
    Mapper(pkv_ctx ctx, const Geometry& g, const Config& c, const double* blob, int64_t count, uint32_t precision);
    ~Mapper();
    // trace (nullable): Stage-3 attention [rows, H_l, syn] of every (unit, window, token) row
    void run(const float* x, const std::vector<int64_t>& unit_off, int64_t N, const std::vector<int>& out_unit,
             float* y, cudaStream_t st, float* trace = nullptr);

    pkv_ctx ctx;
    Geometry geom;
    Config cfg;
    int na = 2, nb = 1;
    bool ffn2_single_act = false;  // precision mode 5
    bool f8 = false;               // precision mode 6 (FP16F8)
    int64_t rows_cap = int64_t(1) << 20;  // rows per chunk (bounds the workspace)
    bool use_pair = getenv("PKV_NO_PAIR") == nullptr;  // CTA-pair GEMMs (tuning/AB switch)
    // QKV projection with one fp16 MMA (its output is rounded to one fp16 plane
    // for attention anyway). Off by default: at Llama/32k it lowers the
    // min-slice Top-K overlap from 0.99939 to 0.99908.
    bool qkv_single = getenv("PKV_QKV_SINGLE") != nullptr;

private:
    WeightPlanes upload_planes(const std::vector<double>& W, int64_t N, int64_t K);
    // FP16F8 weights whose GEMM at M rows runs on the pair kernel: the producer of
    // its A operand then writes the e4m3 planes instead of the fp16 lo plane
    bool f8_gemm(const WeightPlanes& w, int64_t M) const { return w.h8 && use_pair && w.N >= 256 && M >= 256; }
    F8Out f8_planes(const WeightPlanes& w, int64_t M, __half* lo_buf, int64_t elems) const;
    // FP16F8 planes when precision 6 (else upload_planes)
    WeightPlanes upload_planes_f8(const std::vector<double>& W, int64_t N, int64_t K, const F8Class& cls);
    void gemm(const __half* a_h, const __half* a_l, int64_t M, const WeightPlanes& w, const float* bias, GemmEpi epi,
              GemmEpiParams p, cudaStream_t st, bool single = false, bool a_single = false);

    std::vector<void*> owned;
    DevBuf work;
    float* pe_d = nullptr;
    float *conv1_w = nullptr, *conv1_b = nullptr, *conv2_b = nullptr;
    WeightPlanes conv2;
    float *bypass_w = nullptr, *bypass_b = nullptr;
    std::vector<Block> blocks;
    WeightPlanes stage3;
    float* stage3_b = nullptr;
    float out_b = 0.0f;
    int64_t n3 = 0, ld3 = 0;
};

}  // namespace pkv

struct pkv_mapper_s {
    std::unique_ptr<pkv::Mapper> m;
};

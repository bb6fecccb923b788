// proxykv.hpp — header-only C++ drop-in over the C ABI (pkv_capi.h) with the
// reference's scoring / mapper / prune signatures and exception taxonomy
// (proj/include/proxykv/{common,pruning,mapper}.hpp). A reference caller swaps
//   #include "proxykv/pruning.hpp"          ->  #include "proxykv_b200/proxykv.hpp"
//   proxykv::topk_mask(scores, rho)         ->  proxykv_b200::topk_mask(ctx, scores, rho)
// and links libpkv_b200.so. Host containers here are plain std::vector (the
// reference Tensor is an autodiff node; only its shape + row-major fp64 data
// cross the boundary).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../pkv_capi.h"

namespace proxykv_b200 {

// common.hpp:13-52
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct ValueError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};
struct NoDeviceError : Error {
    using Error::Error;
};
// common.hpp:33-52: the corrupted-file taxonomy of the trace / checkpoint formats
struct IoError : Error {
    using Error::Error;
};
struct BadMagicError : IoError {
    using IoError::IoError;
};
struct VersionMismatchError : IoError {
    using IoError::IoError;
};
struct TruncatedFileError : IoError {
    using IoError::IoError;
};
struct PayloadLengthError : IoError {
    using IoError::IoError;
};

inline void check(pkv_status s) {
    if (s == PKV_OK) return;
    const std::string msg = pkv_last_error();
    switch (s) {
        case PKV_ESHAPE: throw ShapeError(msg);
        case PKV_EVALUE: throw ValueError(msg);
        case PKV_ECONFIG: throw ConfigError(msg);
        case PKV_ENODEV: throw NoDeviceError(msg);
        case PKV_EIO: throw IoError(msg);
        case PKV_EIO_MAGIC: throw BadMagicError(msg);
        case PKV_EIO_VERSION: throw VersionMismatchError(msg);
        case PKV_EIO_TRUNCATED: throw TruncatedFileError(msg);
        case PKV_EIO_LENGTH: throw PayloadLengthError(msg);
        default: throw CudaError(msg);
    }
}

class Context {
public:
    explicit Context(int device = 0) { check(pkv_ctx_create(device, &h_)); }
    ~Context() { pkv_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    pkv_ctx get() const { return h_; }

private:
    pkv_ctx h_ = nullptr;
};

using Shape = std::vector<int64_t>;

// pruning.hpp:14
inline int64_t retention_count(double rho, int64_t n) {
    int64_t k = 0;
    check(pkv_retention_count(rho, n, &k));
    return k;
}

// The reference's host container (tensor.hpp:42-83): shape + row-major fp64
// data (its autodiff tape does not cross the boundary).
struct Tensor {
    Shape shape;
    std::vector<double> data;
    Tensor() = default;
    Tensor(Shape s, std::vector<double> d) : shape(std::move(s)), data(std::move(d)) {
        if (static_cast<int64_t>(data.size()) != numel()) throw ShapeError("tensor data does not match its shape");
    }
    explicit Tensor(Shape s) : shape(std::move(s)), data(static_cast<size_t>(numel()), 0.0) {}
    int64_t dim() const { return static_cast<int64_t>(shape.size()); }
    int64_t size(int64_t i) const { return shape.at(static_cast<size_t>(i)); }
    int64_t numel() const {
        int64_t n = 1;
        for (int64_t e : shape) n *= e;
        return n;
    }
};
using ScoreTensor = Tensor;  // tensor.hpp:86

inline std::string shape_str(const Shape& s) {
    std::string o = "[";
    for (size_t i = 0; i < s.size(); ++i) o += (i ? ", " : "") + std::to_string(s[i]);
    return o + "]";
}

// The process-wide context the reference-signature overloads below use
// (device 0; the reference API has no context argument).
inline Context& default_context() {
    static Context c(0);
    return c;
}

// pruning.hpp:18 / pruning.cpp:20-35: the k best of values[0..n) (ties to the
// lower index) on the GPU, fp64 exact. Ascending order (the reference returns
// nth_element order; same set).
inline std::vector<int64_t> topk_indices(const double* values, int64_t n, int64_t k) {
    std::vector<int64_t> idx(static_cast<size_t>(k > 0 ? k : 0));
    check(pkv_topk_indices_host(default_context().get(), values, n, k, idx.data()));
    return idx;
}

// pruning.hpp:22-30
struct PruneMask {
    Shape shape;
    std::vector<uint8_t> bits;
    double retention_ratio = 1.0;
    int64_t k = 0;
    int64_t token_count() const { return shape.back(); }
    int64_t slice_count() const {
        int64_t n = 1;
        for (int64_t e : shape) n *= e;
        return n / shape.back();
    }
};

// pruning.hpp:32 / pruning.cpp:37-56 — scores row-major fp64 (ranked exactly:
// 64-bit order keys), last axis = tokens. Runs the GPU radix select.
inline PruneMask topk_mask(const Context& ctx, const std::vector<double>& scores, const Shape& shape, double rho) {
    if (shape.empty()) throw ShapeError("topk_mask needs a shaped tensor");
    PruneMask m;
    m.shape = shape;
    m.retention_ratio = rho;
    m.bits.assign(scores.size(), 0);
    const int64_t n = shape.back();
    check(pkv_topk_mask_host(ctx.get(), scores.data(), static_cast<int64_t>(scores.size()) / n, n, rho,
                             m.bits.data(), &m.k));
    return m;
}

// pruning.hpp:32 with the reference signature (default context)
inline PruneMask topk_mask(const ScoreTensor& scores, double rho) {
    return topk_mask(default_context(), scores.data, scores.shape, rho);
}

// pruning.hpp:41-42 / pruning.cpp:91-117 (per-slice |a ∩ b| / k on the GPU,
// then the unweighted slice mean)
inline std::vector<double> topk_overlap_per_slice(const PruneMask& a, const PruneMask& b) {
    if (a.shape != b.shape)
        throw ShapeError("mask shapes differ: " + shape_str(a.shape) + " vs " + shape_str(b.shape));
    if (a.k != b.k)
        throw ValueError("topk_overlap needs equal per-slice counts, got " + std::to_string(a.k) + " and " +
                         std::to_string(b.k));
    std::vector<double> out(static_cast<size_t>(a.slice_count()));
    check(pkv_topk_overlap_host(default_context().get(), a.bits.data(), b.bits.data(), a.slice_count(),
                                a.token_count(), a.k, out.data()));
    return out;
}

inline double topk_overlap(const PruneMask& a, const PruneMask& b) {
    const auto per = topk_overlap_per_slice(a, b);
    double acc = 0.0;
    for (double v : per) acc += v;
    return acc / static_cast<double>(per.size());
}

// pruning.hpp:48-53, 57 / pruning.cpp:197-215
struct MaskApplication {
    std::vector<std::vector<int64_t>> retained;
    int64_t dropped_per_slice = 0;
    int64_t bytes_saved_per_head = 0;
    int64_t bytes_saved_total = 0;
};

inline MaskApplication apply_mask(const PruneMask& mask, int64_t head_dim, int64_t bytes_per_elem = 2) {
    MaskApplication a;
    const int64_t n = mask.token_count(), slices = mask.slice_count();
    a.retained.resize(static_cast<size_t>(slices));
    for (int64_t s = 0; s < slices; ++s) {
        auto& l = a.retained[static_cast<size_t>(s)];
        l.reserve(static_cast<size_t>(mask.k));
        for (int64_t i = 0; i < n; ++i)
            if (mask.bits[static_cast<size_t>(s * n + i)]) l.push_back(i);
    }
    a.dropped_per_slice = n - mask.k;
    a.bytes_saved_per_head = a.dropped_per_slice * head_dim * bytes_per_elem * 2;
    a.bytes_saved_total = a.bytes_saved_per_head * slices;
    return a;
}

// mapper.hpp:16-25 / 35-55
struct ModelGeometry {
    int64_t target_layers = 32, target_heads = 32, proxy_layers = 16, proxy_heads = 32, head_dim = 128;
    std::vector<int64_t> as5() const { return {target_layers, target_heads, proxy_layers, proxy_heads, head_dim}; }
};

enum class StageMode { kActive, kBypass };

struct MapperConfig {
    int64_t d_time = 512, encoder_layers = 6, encoder_heads = 8, ffn_mult = 4, d_head = 64, crop_len = 2048,
            stride = 1024, synthetic_heads = 0;
    StageMode stage_conv = StageMode::kActive, stage_encoder = StageMode::kActive, stage_cross = StageMode::kActive;
    bool normalize_input = false;
    std::vector<int64_t> as12() const {
        auto m = [](StageMode s) { return s == StageMode::kBypass ? int64_t(1) : int64_t(0); };
        return {d_time, encoder_layers, encoder_heads, ffn_mult, d_head, crop_len, stride, synthetic_heads,
                m(stage_conv), m(stage_encoder), m(stage_cross), normalize_input ? 1 : 0};
    }
};

// mapper.hpp:58, 65
inline int64_t layer_pair(int64_t target_layer, const ModelGeometry& g) {
    int64_t out = 0;
    check(pkv_layer_pair(target_layer, g.as5().data(), &out));
    return out;
}

inline std::vector<int64_t> window_offsets(int64_t n, int64_t crop, int64_t stride) {
    int64_t cnt = 0;
    check(pkv_window_offsets(n, crop, stride, nullptr, 0, &cnt));
    std::vector<int64_t> v(static_cast<size_t>(cnt));
    check(pkv_window_offsets(n, crop, stride, v.data(), cnt, &cnt));
    return v;
}

// mapper.hpp:94 MapperParams::init -> flat fp64 blob (named_parameters + named_buffers)
inline std::vector<double> mapper_init_params(const ModelGeometry& g, const MapperConfig& c, uint64_t seed) {
    int64_t n = 0;
    check(pkv_mapper_init_params(g.as5().data(), c.as12().data(), seed, nullptr, &n));
    std::vector<double> blob(static_cast<size_t>(n));
    check(pkv_mapper_init_params(g.as5().data(), c.as12().data(), seed, blob.data(), &n));
    return blob;
}

// Device-resident mapper; forward_full takes/returns DEVICE fp32 buffers
// (mapper.hpp:126; the host-tensor form is a cudaMemcpy on either side).
class Mapper {
public:
    Mapper(const Context& ctx, const ModelGeometry& g, const MapperConfig& c, const std::vector<double>& blob,
           uint32_t precision = PKV_MAPPER_FP16X3)
        : geom_(g) {
        check(pkv_mapper_create(ctx.get(), g.as5().data(), c.as12().data(), blob.data(),
                                static_cast<int64_t>(blob.size()), precision, &h_));
    }
    ~Mapper() { pkv_mapper_destroy(h_); }
    Mapper(const Mapper&) = delete;
    Mapper& operator=(const Mapper&) = delete;
    void forward_full(const float* x_all_dev, int64_t B, int64_t N, float* y_all_dev, void* stream = nullptr) {
        check(pkv_mapper_forward_full(h_, x_all_dev, B, N, y_all_dev, stream));
    }
    void sliding_forward(const float* x_dev, int64_t B, int64_t N, float* y_dev, void* stream = nullptr) {
        check(pkv_mapper_sliding_forward(h_, x_dev, B, N, y_dev, stream));
    }
    pkv_mapper get() const { return h_; }

private:
    pkv_mapper h_ = nullptr;
    ModelGeometry geom_;
};

// GPU training (pkv_trainer): the reference's training forward_pair
// (mapper.cpp:274-342, BN on batch statistics + the running-stat EMA) and the
// reverse sweep of its tape from d loss / d logits to every parameter
// gradient (named_parameters order). DEVICE buffers.
class MapperTrainer {
public:
    MapperTrainer(const Context& ctx, const ModelGeometry& g, const MapperConfig& c, const std::vector<double>& blob) {
        check(pkv_trainer_create(ctx.get(), g.as5().data(), c.as12().data(), blob.data(),
                                 static_cast<int64_t>(blob.size()), &h_));
        check(pkv_trainer_param_count(h_, &params_, &total_));
    }
    ~MapperTrainer() { pkv_trainer_destroy(h_); }
    MapperTrainer(const MapperTrainer&) = delete;
    MapperTrainer& operator=(const MapperTrainer&) = delete;
    // x [B, H_s, n] fp32 -> logits [B, H_l, n] fp32; keeps the activations
    void forward(const float* x_dev, int64_t B, int64_t n, float* logits_dev, void* stream = nullptr) {
        check(pkv_trainer_forward(h_, x_dev, B, n, logits_dev, stream));
    }
    // grad_dev[param_count()] += d loss / d params for d loss / d logits (fp64) of the last forward
    void backward(const double* dlogits_dev, double* grad_dev, void* stream = nullptr) {
        check(pkv_trainer_backward(h_, dlogits_dev, grad_dev, stream));
    }
    // host fp64 forms (synchronous)
    void forward_host(const double* x, int64_t B, int64_t n, double* logits) {
        check(pkv_trainer_forward_host(h_, x, B, n, logits));
    }
    void backward_host(const double* dlogits, double* grad) { check(pkv_trainer_backward_host(h_, dlogits, grad)); }
    std::vector<double> blob() const {
        std::vector<double> b(static_cast<size_t>(total_));
        check(pkv_trainer_blob(h_, b.data()));
        return b;
    }
    int64_t param_count() const { return params_; }

private:
    pkv_trainer h_ = nullptr;
    int64_t params_ = 0, total_ = 0;
};

// ---- the reference's mapper entry points on host tensors (mapper.hpp:94-126)

// mapper.hpp:67-100: the parameters (the reference initialisation as the flat
// fp64 blob, named_parameters + named_buffers order) and, on first use, their
// device-resident form. Eval only, like sliding_forward / forward_full.
struct MapperParams {
    ModelGeometry geometry;
    MapperConfig config;
    std::vector<double> blob;
    uint32_t precision = PKV_MAPPER_FP16X3;

    static MapperParams init(const ModelGeometry& g, const MapperConfig& c, uint64_t seed) {
        MapperParams p;
        p.geometry = g;
        p.config = c;
        p.blob = mapper_init_params(g, c, seed);
        return p;
    }
    Mapper& device() {
        if (!dev_) dev_ = std::make_shared<Mapper>(default_context(), geometry, config, blob, precision);
        return *dev_;
    }
    MapperTrainer& trainer() {
        if (!train_) train_ = std::make_shared<MapperTrainer>(default_context(), geometry, config, blob);
        return *train_;
    }
    // after a training forward: the BN running statistics it updated, back into
    // `blob` (the eval mapper is rebuilt from them on next use)
    void sync_from_trainer() {
        blob = train_->blob();
        dev_.reset();
    }
    // The tape's reverse sweep for the last training forward_pair: d loss / d
    // every parameter (named_parameters order) for d loss / d logits [B, H_l, n].
    std::vector<double> backward(const std::vector<double>& dlogits) {
        if (!train_ || last_logits_ == 0) throw ValueError("backward needs a training forward_pair first");
        if (static_cast<int64_t>(dlogits.size()) != last_logits_)
            throw ShapeError("dlogits must match the last training forward's [B, H_l, n]");
        std::vector<double> g(static_cast<size_t>(train_->param_count()), 0.0);
        train_->backward_host(dlogits.data(), g.data());
        return g;
    }
    void note_training_forward(int64_t logits) { last_logits_ = logits; }

private:
    std::shared_ptr<Mapper> dev_;
    std::shared_ptr<MapperTrainer> train_;
    int64_t last_logits_ = 0;
};

// mapper.hpp:111-114
struct StageTrace {
    Tensor cross_attention;  // [B, N, H_l, H_syn]
};

// mapper.hpp:118-119 / mapper.cpp:274-342: x [B, H_s, n] -> raw logits
// [B, H_l, n], n <= crop_len. training = true runs the reference's training
// forward on the GPU trainer (BN batch statistics; the running statistics in
// params.blob are updated) and keeps its activations for params.backward();
// the trace is an eval-path output.
inline Tensor forward_pair(const Tensor& x, MapperParams& params, bool training, StageTrace* trace = nullptr) {
    const ModelGeometry& g = params.geometry;
    if (x.dim() != 3) throw ShapeError("forward_pair input must be [B, H_s, N], got " + shape_str(x.shape));
    if (x.size(1) != g.proxy_heads)
        throw ShapeError("input has " + std::to_string(x.size(1)) + " proxy heads, geometry expects " +
                         std::to_string(g.proxy_heads));
    const int64_t B = x.size(0), n = x.size(2);
    if (training) {
        Tensor y({B, g.target_heads, n});
        params.trainer().forward_host(x.data.data(), B, n, y.data.data());
        params.sync_from_trainer();
        params.note_training_forward(static_cast<int64_t>(y.data.size()));
        return y;
    }
    const int64_t syn = params.config.synthetic_heads > 0 ? params.config.synthetic_heads : g.proxy_heads;
    Tensor y({B, g.target_heads, n});
    const bool want = trace && params.config.stage_cross == StageMode::kActive;
    std::vector<double> attn(want ? static_cast<size_t>(B * n * g.target_heads * syn) : 0);
    check(pkv_mapper_forward_pair_host(params.device().get(), x.data.data(), B, n, y.data.data(),
                                       want ? attn.data() : nullptr));
    if (want) trace->cross_attention = Tensor({B, n, g.target_heads, syn}, std::move(attn));
    return y;
}

// mapper.hpp:123 / mapper.cpp:344-377: [B, H_s, N] -> [B, H_l, N]
inline Tensor sliding_forward(const Tensor& x, MapperParams& params) {
    const ModelGeometry& g = params.geometry;
    if (x.dim() != 3 || x.size(1) != g.proxy_heads)
        throw ShapeError("sliding_forward input must be [B, H_s, N], got " + shape_str(x.shape));
    Tensor y({x.size(0), g.target_heads, x.size(2)});
    check(pkv_mapper_sliding_forward_host(params.device().get(), x.data.data(), x.size(0), x.size(2), y.data.data()));
    return y;
}

// mapper.hpp:126 / mapper.cpp:379-398: [B, L_s, H_s, N] -> [B, L_l, H_l, N]
inline Tensor forward_full(const Tensor& x_all, MapperParams& params) {
    const ModelGeometry& g = params.geometry;
    if (x_all.dim() != 4 || x_all.size(1) != g.proxy_layers || x_all.size(2) != g.proxy_heads)
        throw ShapeError("forward_full input must be [B, L_s, H_s, N], got " + shape_str(x_all.shape));
    Tensor y({x_all.size(0), g.target_layers, g.target_heads, x_all.size(3)});
    check(pkv_mapper_forward_full_host(params.device().get(), x_all.data.data(), x_all.size(0), x_all.size(3),
                                       y.data.data()));
    return y;
}

// pruning.cpp:173-186 over DEVICE fp32 rows [slices, n] -> DEVICE fp64 [slices]
inline void spearman_per_slice(const Context& ctx, const float* a_dev, const float* b_dev, int64_t slices, int64_t n,
                               double* out_dev, void* stream = nullptr) {
    check(pkv_spearman(ctx.get(), a_dev, b_dev, slices, n, out_dev, stream));
}

// loss.hpp:16-37 (same fields, same defaults)
struct LossConfig {
    double lambda_mse = 20.0, lambda_bin = 10.0, lambda_fine = 3.0, lambda_global = 2.0, lambda_cos = 0.5;
    std::vector<double> ratios = {0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5};
    double gamma = 1.0, epsilon = 0.1, mse_exponent = 1.5, margin = 1.0, clip_lo = 1.0, clip_hi = 5.0;
    double pair_filter_frac = 0.01, topk_ratio_for_rank = 0.2;
    int64_t max_pairs = 4096;
    // the C view borrows `ratios`: valid while this LossConfig lives
    pkv_loss_config c() const {
        return pkv_loss_config{lambda_mse, lambda_bin, lambda_fine, lambda_global, lambda_cos, ratios.data(),
                               static_cast<int64_t>(ratios.size()), gamma, epsilon, mse_exponent, margin, clip_lo,
                               clip_hi, pair_filter_frac, topk_ratio_for_rank, max_pairs};
    }
};
using LossReport = pkv_loss_report;

// loss.cpp:324-374 over DEVICE fp32 logits / scores; grad_dev (fp64, nullable)
// receives d total / d logits (the reference's total_tensor.backward()).
inline LossReport loss_total(const Context& ctx, const float* logits_dev, const float* y_dev, const Shape& shape,
                             const LossConfig& cfg, uint64_t seed, double* grad_dev = nullptr,
                             void* stream = nullptr) {
    const pkv_loss_config c = cfg.c();
    LossReport r{};
    check(pkv_loss_total(ctx.get(), logits_dev, y_dev, shape.data(), static_cast<int>(shape.size()), &c, seed, &r,
                         grad_dev, stream));
    return r;
}

}  // namespace proxykv_b200

// C-ABI harness over the UNMODIFIED reference C++ API (/root/reference/proj),
// compiled together with the reference sources into oracle/_ref/libpkvref.so
// by oracle/Makefile. TEST INFRASTRUCTURE ONLY: imported by tests/, by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// --impl reference legs. The product path never links or loads this.
//
// Every entry point forwards to the reference function named in its comment
// and converts C++ exceptions into status codes:
//   0 ok, 1 ShapeError, 2 ValueError, 5 ConfigError, 9 other.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "proxykv/common.hpp"
#include "proxykv/mapper.hpp"
#include "proxykv/pruning.hpp"
#include "proxykv/loss.hpp"
#include "proxykv/rng.hpp"
#include "proxykv/tensor.hpp"

using namespace proxykv;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ValueError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

Tensor make_tensor(const double* data, const int64_t* shape, int rank) {
    Shape s(shape, shape + rank);
    std::vector<double> v(static_cast<size_t>(shape_numel(s)));
    std::memcpy(v.data(), data, v.size() * sizeof(double));
    return Tensor::from_data(s, std::move(v));
}

struct RefMapper {
    MapperParams params;
};

}  // namespace

extern "C" {

const char* pkvref_last_error() { return g_err.c_str(); }

// pruning.cpp:14-18
int pkvref_retention_count(double rho, int64_t n, int64_t* out) {
    return guard([&] { *out = retention_count(rho, n); });
}

// pruning.cpp:20-35 (indices come back in nth_element order, unsorted)
int pkvref_topk_indices(const double* values, int64_t n, int64_t k, int64_t* out) {
    return guard([&] {
        const auto idx = topk_indices(values, n, k);
        std::memcpy(out, idx.data(), idx.size() * sizeof(int64_t));
    });
}

// pruning.cpp:37-56 — scores of arbitrary rank; bits_out has numel entries.
int pkvref_topk_mask(const double* scores, const int64_t* shape, int rank, double rho,
                     uint8_t* bits_out, int64_t* k_out) {
    return guard([&] {
        const PruneMask m = topk_mask(make_tensor(scores, shape, rank), rho);
        std::memcpy(bits_out, m.bits.data(), m.bits.size());
        *k_out = m.k;
    });
}

// pruning.cpp:197-215 — retained indices per slice (ascending), [slices, k].
int pkvref_apply_mask(const uint8_t* bits, const int64_t* shape, int rank, int64_t k,
                      int64_t head_dim, int64_t bytes_per_elem, int64_t* idx_out,
                      int64_t* dropped_per_slice, int64_t* bytes_saved_per_head,
                      int64_t* bytes_saved_total) {
    return guard([&] {
        PruneMask m;
        m.shape = Shape(shape, shape + rank);
        m.bits.assign(bits, bits + shape_numel(m.shape));
        m.k = k;
        const MaskApplication app = apply_mask(m, head_dim, bytes_per_elem);
        int64_t off = 0;
        for (const auto& list : app.retained) {
            std::memcpy(idx_out + off, list.data(), list.size() * sizeof(int64_t));
            off += static_cast<int64_t>(list.size());
        }
        *dropped_per_slice = app.dropped_per_slice;
        *bytes_saved_per_head = app.bytes_saved_per_head;
        *bytes_saved_total = app.bytes_saved_total;
    });
}

// pruning.cpp:91-117
int pkvref_topk_overlap_per_slice(const uint8_t* a, const uint8_t* b, const int64_t* shape,
                                  int rank, int64_t ka, int64_t kb, double* out) {
    return guard([&] {
        PruneMask ma, mb;
        ma.shape = mb.shape = Shape(shape, shape + rank);
        ma.bits.assign(a, a + shape_numel(ma.shape));
        mb.bits.assign(b, b + shape_numel(mb.shape));
        ma.k = ka;
        mb.k = kb;
        const auto v = topk_overlap_per_slice(ma, mb);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

// mapper.cpp:44-49
// captured_mass_per_slice (pruning.cpp:58-80) over a predicted mask and fp64 scores
int pkvref_captured_mass_per_slice(const uint8_t* pred, int64_t k, const double* y, const int64_t* shape, int rank,
                                   double* out) {
    return guard([&] {
        PruneMask m;
        m.shape = Shape(shape, shape + rank);
        m.bits.assign(pred, pred + shape_numel(m.shape));
        m.k = k;
        const auto v = captured_mass_per_slice(m, make_tensor(y, shape, rank));
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

// spearman_per_slice (pruning.cpp:173-186) of two fp64 tensors of one shape
int pkvref_spearman_per_slice(const double* a, const double* b, const int64_t* shape, int rank, double* out) {
    return guard([&] {
        const auto v = spearman_per_slice(make_tensor(a, shape, rank), make_tensor(b, shape, rank));
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

// loss_total (loss.cpp:324-374) + the tape's gradient w.r.t. the logits.
// cfgd = {lambda_mse, lambda_bin, lambda_fine, lambda_global, lambda_cos, gamma,
//         epsilon, mse_exponent, margin, clip_lo, clip_hi, pair_filter_frac,
//         topk_ratio_for_rank}; rep = {bin, mse, fine, global, cos, w_bin, w_mse,
//         w_fine, w_global, w_cos, total, s_max}; cnt = {fine used, fine
//         filtered, global used, global filtered, cos floor hits}.
int pkvref_loss_total(const double* logits, const double* y, const int64_t* shape, int rank, const double* cfgd,
                      const double* ratios, int64_t n_ratios, int64_t max_pairs, uint64_t seed, double* rep,
                      int64_t* cnt, double* grad) {
    return guard([&] {
        LossConfig c;
        c.lambda_mse = cfgd[0];
        c.lambda_bin = cfgd[1];
        c.lambda_fine = cfgd[2];
        c.lambda_global = cfgd[3];
        c.lambda_cos = cfgd[4];
        c.gamma = cfgd[5];
        c.epsilon = cfgd[6];
        c.mse_exponent = cfgd[7];
        c.margin = cfgd[8];
        c.clip_lo = cfgd[9];
        c.clip_hi = cfgd[10];
        c.pair_filter_frac = cfgd[11];
        c.topk_ratio_for_rank = cfgd[12];
        c.ratios.assign(ratios, ratios + n_ratios);
        c.max_pairs = max_pairs;
        Tensor z = make_tensor(logits, shape, rank);
        z.set_requires_grad(true);
        const LossReport r = loss_total(z, make_tensor(y, shape, rank), c, seed);
        const double v[12] = {r.bin, r.mse, r.fine, r.global, r.cos, r.weighted_bin, r.weighted_mse,
                              r.weighted_fine, r.weighted_global, r.weighted_cos, r.total, r.s_max};
        std::memcpy(rep, v, sizeof(v));
        cnt[0] = r.fine_pairs.used;
        cnt[1] = r.fine_pairs.filtered;
        cnt[2] = r.global_pairs.used;
        cnt[3] = r.global_pairs.filtered;
        cnt[4] = r.cos_floor_hits;
        if (grad) {
            const size_t n = static_cast<size_t>(z.numel());
            if (r.total_tensor.defined()) {
                r.total_tensor.backward();
                std::memcpy(grad, z.grad().data(), n * sizeof(double));
            } else {
                std::memset(grad, 0, n * sizeof(double));
            }
        }
    });
}

int pkvref_layer_pair(int64_t target_layer, const int64_t* geom5, int64_t* out) {
    return guard([&] {
        ModelGeometry g{geom5[0], geom5[1], geom5[2], geom5[3], geom5[4]};
        *out = layer_pair(target_layer, g);
    });
}

// mapper.cpp:66-79 — writes up to cap offsets, returns count in *count.
int pkvref_window_offsets(int64_t n, int64_t crop, int64_t stride, int64_t* out, int64_t cap,
                          int64_t* count) {
    return guard([&] {
        const auto v = window_offsets(n, crop, stride);
        *count = static_cast<int64_t>(v.size());
        for (size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) {
            out[i] = v[i];
        }
    });
}

// mapper.cpp:51-64
int pkvref_sinusoidal_pe(int64_t n, int64_t d_time, double* out) {
    return guard([&] {
        const Tensor pe = sinusoidal_pe(n, d_time);
        std::memcpy(out, pe.data().data(), pe.data().size() * sizeof(double));
    });
}

// MapperParams::init mapper.cpp:97-164.
// geom5 = {target_layers, target_heads, proxy_layers, proxy_heads, head_dim}
// cfg   = {d_time, encoder_layers, encoder_heads, ffn_mult, d_head, crop_len,
//          stride, synthetic_heads, stage_conv, stage_encoder, stage_cross,
//          normalize_input}   (stage: 0 active, 1 bypass)
int pkvref_mapper_create(const int64_t* geom5, const int64_t* cfg12, uint64_t seed, void** out) {
    return guard([&] {
        ModelGeometry g{geom5[0], geom5[1], geom5[2], geom5[3], geom5[4]};
        MapperConfig c;
        c.d_time = cfg12[0];
        c.encoder_layers = cfg12[1];
        c.encoder_heads = cfg12[2];
        c.ffn_mult = cfg12[3];
        c.d_head = cfg12[4];
        c.crop_len = cfg12[5];
        c.stride = cfg12[6];
        c.synthetic_heads = cfg12[7];
        c.stage_conv = cfg12[8] ? StageMode::kBypass : StageMode::kActive;
        c.stage_encoder = cfg12[9] ? StageMode::kBypass : StageMode::kActive;
        c.stage_cross = cfg12[10] ? StageMode::kBypass : StageMode::kActive;
        c.normalize_input = cfg12[11] != 0;
        auto* m = new RefMapper{MapperParams::init(g, c, seed)};
        m->params.set_trainable(false);
        *out = m;
    });
}

void pkvref_mapper_destroy(void* h) { delete static_cast<RefMapper*>(h); }

// named_parameters() then named_buffers() (mapper.cpp:166-225): number of
// tensors, and for tensor i its name / numel / flat fp64 values.
int pkvref_mapper_tensor_count(void* h) {
    auto& p = static_cast<RefMapper*>(h)->params;
    return static_cast<int>(p.named_parameters().size() + p.named_buffers().size());
}

int pkvref_mapper_tensor(void* h, int i, char* name, int name_cap, int64_t* shape, int* rank,
                         double* values /* nullable */) {
    return guard([&] {
        auto& p = static_cast<RefMapper*>(h)->params;
        auto all = p.named_parameters();
        for (auto& b : p.named_buffers()) {
            all.push_back(b);
        }
        const auto& [n, t] = all.at(static_cast<size_t>(i));
        std::snprintf(name, static_cast<size_t>(name_cap), "%s", n.c_str());
        *rank = static_cast<int>(t.shape().size());
        for (size_t d = 0; d < t.shape().size(); ++d) {
            shape[d] = t.shape()[d];
        }
        if (values) {
            std::memcpy(values, t.data().data(), t.data().size() * sizeof(double));
        }
    });
}

// mapper.cpp:274-342, eval mode. x [B, H_s, n] -> out [B, H_l, n].
int pkvref_forward_pair(void* h, const double* x, int64_t b, int64_t hs, int64_t n, double* out) {
    return guard([&] {
        auto& p = static_cast<RefMapper*>(h)->params;
        const int64_t shape[3] = {b, hs, n};
        const Tensor y = forward_pair(make_tensor(x, shape, 3), p, false);
        std::memcpy(out, y.data().data(), y.data().size() * sizeof(double));
    });
}

// mapper.cpp:344-377
int pkvref_sliding_forward(void* h, const double* x, int64_t b, int64_t hs, int64_t n, double* out) {
    return guard([&] {
        auto& p = static_cast<RefMapper*>(h)->params;
        const int64_t shape[3] = {b, hs, n};
        const Tensor y = sliding_forward(make_tensor(x, shape, 3), p);
        std::memcpy(out, y.data().data(), y.data().size() * sizeof(double));
    });
}

// mapper.cpp:379-398. x_all [B, L_s, H_s, N] -> out [B, L_l, H_l, N].
int pkvref_forward_full(void* h, const double* x, int64_t b, int64_t ls, int64_t hs, int64_t n,
                        double* out) {
    return guard([&] {
        auto& p = static_cast<RefMapper*>(h)->params;
        const int64_t shape[4] = {b, ls, hs, n};
        const Tensor y = forward_full(make_tensor(x, shape, 4), p);
        std::memcpy(out, y.data().data(), y.data().size() * sizeof(double));
    });
}

// Training step of the mapper (mapper.cpp:274-342 with training = true:
// batchnorm1d on batch statistics + the running-stat EMA, ops.cpp:806-850),
// then the tape's reverse sweep (tensor.cpp) of L = Σ dlogits ⊙ logits, i.e.
// the parameter gradients for an upstream gradient dlogits [B, H_l, n].
// grads_out: every named_parameters() tensor's gradient, concatenated in that
// order (the parameter part of the blob layout). The BN running statistics
// in the handle are updated as the reference's training forward does.
int pkvref_mapper_train_grad(void* h, const double* x, int64_t b, int64_t hs, int64_t n, const double* dlogits,
                             double* logits_out, double* grads_out) {
    return guard([&] {
        auto& p = static_cast<RefMapper*>(h)->params;
        p.set_trainable(true);
        struct Frozen {
            MapperParams& p;
            ~Frozen() { p.set_trainable(false); }
        } frozen{p};
        for (auto& nt : p.named_parameters()) nt.second.zero_grad();
        const int64_t shape[3] = {b, hs, n};
        const Tensor y = forward_pair(make_tensor(x, shape, 3), p, true);
        const Tensor dl = Tensor::from_data(y.shape(), std::vector<double>(dlogits, dlogits + y.numel()));
        const Tensor loss = sum(mul(y, dl));
        loss.backward();
        std::memcpy(logits_out, y.data().data(), y.data().size() * sizeof(double));
        size_t o = 0;
        for (auto& nt : p.named_parameters()) {
            const auto& g = nt.second.grad();
            const size_t cnt = static_cast<size_t>(nt.second.numel());
            if (g.size() == cnt) std::memcpy(grads_out + o, g.data(), cnt * sizeof(double));
            else std::memset(grads_out + o, 0, cnt * sizeof(double));
            o += cnt;
        }
    });
}

// The reference's own Rng (rng.hpp:25-87), for regenerating the test inputs
// of test_pruning.cpp / test_mapper.cpp in the golden-vector script.
void* pkvref_rng_create(uint64_t seed) { return new Rng(seed); }
void pkvref_rng_destroy(void* h) { delete static_cast<Rng*>(h); }
double pkvref_rng_uniform(void* h, double lo, double hi) { return static_cast<Rng*>(h)->uniform(lo, hi); }
uint64_t pkvref_rng_below(void* h, uint64_t n) { return static_cast<Rng*>(h)->below(n); }
double pkvref_rng_normal(void* h) { return static_cast<Rng*>(h)->normal(); }

}  // extern "C"

// mapper.cpp — host side of the B200 HybridAxialMapper
// (proj/src/mapper.cpp + proj/include/proxykv/mapper.hpp):
//   - ModelGeometry / MapperConfig validation with the reference messages,
//   - layer_pair, window_offsets, MapperParams::init (xoshiro256** stream),
//   - weight preparation for the kernels (K-major fp16 planes, BN folded into
//     the convs, Q_l and out_w folded into one stage-3 projection, fp64 math),
//   - forward orchestration: all windows of all (deduplicated) proxy layers are
//     batched into the GEMM M dimension, in bounded row chunks.
#include <cuda_fp8.h>

#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "attn.cuh"
#include "gemm.cuh"
#include "mapper.h"
#include "mapper_kernels.cuh"
#include "util.cuh"

namespace pkv {

// ------------------------------------------------------------ config ------
Geometry Geometry::from5(const int64_t* g) {
    Geometry x;
    x.target_layers = g[0];
    x.target_heads = g[1];
    x.proxy_layers = g[2];
    x.proxy_heads = g[3];
    x.head_dim = g[4];
    return x;
}

void Geometry::validate() const {
    // mapper.cpp:13-17
    PKV_REQUIRE_VALUE(target_layers > 0 && target_heads > 0 && proxy_layers > 0 && proxy_heads > 0 && head_dim > 0,
                      "model geometry extents must be positive");
}

Config Config::from12(const int64_t* c) {
    Config x;
    x.d_time = c[0];
    x.encoder_layers = c[1];
    x.encoder_heads = c[2];
    x.ffn_mult = c[3];
    x.d_head = c[4];
    x.crop_len = c[5];
    x.stride = c[6];
    x.synthetic_heads = c[7];
    PKV_REQUIRE((c[8] == 0 || c[8] == 1) && (c[9] == 0 || c[9] == 1) && (c[10] == 0 || c[10] == 1), PKV_ECONFIG,
                "unknown stage mode (expected active|bypass)");
    x.conv_active = c[8] == 0;
    x.enc_active = c[9] == 0;
    x.cross_active = c[10] == 0;
    x.normalize_input = c[11] != 0;
    return x;
}

void Config::validate() const {
    // mapper.cpp:33-42
    PKV_REQUIRE_VALUE(d_time > 0 && encoder_layers >= 0 && encoder_heads > 0 && ffn_mult > 0 && d_head > 0 &&
                          crop_len > 0 && stride > 0,
                      "mapper config extents must be positive");
    PKV_REQUIRE_VALUE(stride <= crop_len, "stride ", stride, " must not exceed crop_len ", crop_len);
    PKV_REQUIRE_VALUE(d_time % encoder_heads == 0, "d_time ", d_time, " must be divisible by encoder_heads ",
                      encoder_heads);
    PKV_REQUIRE_VALUE(d_time % 2 == 0, "d_time must be even for the positional encoding");
}

int64_t layer_pair(int64_t ll, const Geometry& g) {
    // mapper.cpp:44-49
    PKV_REQUIRE_VALUE(ll >= 1 && ll <= g.target_layers, "target layer ", ll, " out of range [1, ", g.target_layers,
                      "]");
    return (ll * g.proxy_layers + g.target_layers - 1) / g.target_layers;
}

std::vector<int64_t> window_offsets(int64_t n, int64_t crop, int64_t stride) {
    // mapper.cpp:66-79
    PKV_REQUIRE_VALUE(n > 0 && crop > 0 && stride > 0, "window parameters must be positive");
    if (n <= crop) return {0};
    std::vector<int64_t> offs;
    for (int64_t off = 0; off + crop <= n; off += stride) offs.push_back(off);
    if (offs.back() + crop < n) offs.push_back(n - crop);
    return offs;
}

std::vector<std::pair<std::string, int64_t>> param_layout(const Geometry& g, const Config& c) {
    // named_parameters() then named_buffers(), mapper.cpp:166-225
    const int64_t hs = g.proxy_heads, dt = c.d_time, mid = c.conv_mid(), dh = c.d_head, syn = c.syn(g);
    const int64_t ffn = c.ffn_mult * c.d_time;
    std::vector<std::pair<std::string, int64_t>> L;
    if (c.conv_active) {
        L.insert(L.end(), {{"stem.conv1.w", mid * hs * 3}, {"stem.conv1.b", mid}, {"stem.bn1.gamma", mid},
                           {"stem.bn1.beta", mid}, {"stem.conv2.w", dt * mid * 3}, {"stem.conv2.b", dt},
                           {"stem.bn2.gamma", dt}, {"stem.bn2.beta", dt}});
    } else {
        L.insert(L.end(), {{"stem.bypass.w", dt * hs}, {"stem.bypass.b", dt}});
    }
    if (c.enc_active) {
        for (int64_t i = 0; i < c.encoder_layers; ++i) {
            const std::string p = "encoder." + std::to_string(i) + ".";
            for (const char* m : {"q", "k", "v", "o"}) {
                L.push_back({p + "attn.w" + m, dt * dt});
                L.push_back({p + "attn.b" + m, dt});
            }
            L.insert(L.end(), {{p + "ln1.gamma", dt}, {p + "ln1.beta", dt}, {p + "ln2.gamma", dt},
                               {p + "ln2.beta", dt}, {p + "ffn1.w", dt * ffn}, {p + "ffn1.b", ffn},
                               {p + "ffn2.w", ffn * dt}, {p + "ffn2.b", dt}});
        }
    }
    if (c.cross_active) L.insert(L.end(), {{"cross.key.w", dt * syn * dh}, {"cross.key.b", syn * dh}});
    L.insert(L.end(), {{"cross.value.w", dt * syn * dh}, {"cross.value.b", syn * dh}});
    if (c.cross_active) L.push_back({"cross.queries", g.target_heads * dh});
    L.insert(L.end(), {{"cross.out.w", dh}, {"cross.out.b", 1}});
    if (c.conv_active) {
        L.insert(L.end(), {{"stem.bn1.running_mean", mid}, {"stem.bn1.running_var", mid},
                           {"stem.bn2.running_mean", dt}, {"stem.bn2.running_var", dt}});
    }
    return L;
}

// ------------------------------------------------ reference RNG and init --
namespace {

// rng.hpp:11-21
uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// xoshiro256** with the reference's hand-rolled distributions (rng.hpp:25-87).
class Xoshiro {
public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& s : s_) s = x = splitmix64(x);
    }
    uint64_t next() {
        const uint64_t r = rotl(s_[1] * 5, 7) * 9, t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return r;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (has_) {
            has_ = false;
            return cached_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * M_PI * u2;
        cached_ = r * std::sin(th);
        has_ = true;
        return r * std::cos(th);
    }

private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t s_[4];
    double cached_ = 0.0;
    bool has_ = false;
};

}  // namespace

std::vector<double> init_params(const Geometry& g, const Config& c, uint64_t seed) {
    g.validate();
    c.validate();
    const auto layout = param_layout(g, c);
    std::map<std::string, std::vector<double>> P;
    Xoshiro rng(splitmix64(seed ^ splitmix64(0x6d617070ull + 1)));  // derive_seed(seed, "mapp")
    auto uni = [&](const std::string& name, int64_t fan_in, int64_t n) {
        const double b = 1.0 / std::sqrt(static_cast<double>(fan_in));
        auto& v = P[name];
        v.resize(n);
        for (auto& x : v) x = rng.uniform(-b, b);
    };
    auto fill = [&](const std::string& name, int64_t n, double val) { P[name].assign(n, val); };
    const int64_t hs = g.proxy_heads, dt = c.d_time, mid = c.conv_mid(), dh = c.d_head, syn = c.syn(g);
    const int64_t ffn = c.ffn_mult * dt;
    // draw order of mapper.cpp:105-163
    if (c.conv_active) {
        uni("stem.conv1.w", hs * 3, mid * hs * 3);
        uni("stem.conv1.b", hs * 3, mid);
        fill("stem.bn1.gamma", mid, 1.0);
        fill("stem.bn1.beta", mid, 0.0);
        uni("stem.conv2.w", mid * 3, dt * mid * 3);
        uni("stem.conv2.b", mid * 3, dt);
        fill("stem.bn2.gamma", dt, 1.0);
        fill("stem.bn2.beta", dt, 0.0);
        fill("stem.bn1.running_mean", mid, 0.0);
        fill("stem.bn1.running_var", mid, 1.0);
        fill("stem.bn2.running_mean", dt, 0.0);
        fill("stem.bn2.running_var", dt, 1.0);
    } else {
        uni("stem.bypass.w", hs, dt * hs);
        uni("stem.bypass.b", hs, dt);
    }
    if (c.enc_active) {
        for (int64_t i = 0; i < c.encoder_layers; ++i) {
            const std::string p = "encoder." + std::to_string(i) + ".";
            for (const char* m : {"q", "k", "v", "o"}) {
                uni(p + "attn.w" + m, dt, dt * dt);
                uni(p + "attn.b" + m, dt, dt);
            }
            fill(p + "ln1.gamma", dt, 1.0);
            fill(p + "ln1.beta", dt, 0.0);
            fill(p + "ln2.gamma", dt, 1.0);
            fill(p + "ln2.beta", dt, 0.0);
            uni(p + "ffn1.w", dt, dt * ffn);
            uni(p + "ffn1.b", dt, ffn);
            uni(p + "ffn2.w", ffn, ffn * dt);
            uni(p + "ffn2.b", ffn, dt);
        }
    }
    if (c.cross_active) {
        uni("cross.key.w", dt, dt * syn * dh);
        uni("cross.key.b", dt, syn * dh);
        auto& q = P["cross.queries"];
        q.resize(g.target_heads * dh);
        for (auto& v : q) v = rng.normal() / std::sqrt(static_cast<double>(dh));
    }
    uni("cross.value.w", dt, dt * syn * dh);
    uni("cross.value.b", dt, syn * dh);
    uni("cross.out.w", dh, dh);
    uni("cross.out.b", dh, 1);
    std::vector<double> blob;
    for (const auto& [name, n] : layout) {
        const auto& v = P.at(name);
        blob.insert(blob.end(), v.begin(), v.end());
    }
    return blob;
}

// ------------------------------------------------------- weight upload ----
namespace {

template <typename T>
T* upload(const std::vector<T>& v, std::vector<void*>& owned) {
    void* p = nullptr;
    PKV_CUDA(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
    PKV_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    owned.push_back(p);
    return static_cast<T*>(p);
}

std::vector<float> to_f32(const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); }

}  // namespace

// W is [N, K] row-major fp64 (already in B-operand orientation).
WeightPlanes Mapper::upload_planes(const std::vector<double>& W, int64_t N, int64_t K) {
    std::vector<__half> hi(W.size()), lo(W.size());
    for (size_t i = 0; i < W.size(); ++i) {
        hi[i] = __double2half(W[i]);
        lo[i] = __double2half(W[i] - static_cast<double>(__half2float(hi[i])));
    }
    WeightPlanes p;
    p.N = N;
    p.K = K;
    p.hi = upload(hi, owned);
    if (nb > 1) p.lo = upload(lo, owned);
    return p;
}

// FP16F8: W' = W·2^w with max |W'| in [2^(w_top−1), 2^w_top) (fp16 hi plane),
// e4m3 planes of W'_hi / lo_mul and (W' − W'_hi) / hi_mul (gemm.cuh).
WeightPlanes Mapper::upload_planes_f8(const std::vector<double>& W, int64_t N, int64_t K, const F8Class& cls) {
    if (!f8) return upload_planes(W, N, K);
    double mx = 0.0;
    for (double v : W) mx = std::max(mx, std::fabs(v));
    int e = 0;
    if (mx > 0.0) std::frexp(mx, &e);  // mx < 2^e
    const int w = cls.w_top - e;
    const double sc = std::ldexp(1.0, w);
    std::vector<__half> hi(W.size()), lo(W.size());
    std::vector<uint8_t> h8(W.size()), l8(W.size());
    for (size_t i = 0; i < W.size(); ++i) {
        const double v = W[i] * sc;
        hi[i] = __double2half(v);
        const double h = static_cast<double>(__half2float(hi[i]));
        lo[i] = __double2half(v - h);  // the FP16X3 fallback for GEMMs too small for the pair kernel
        h8[i] = __nv_cvt_float_to_fp8(static_cast<float>(h / cls.lo_mul), __NV_SATFINITE, __NV_E4M3);
        l8[i] = __nv_cvt_float_to_fp8(static_cast<float>((v - h) / cls.hi_mul), __NV_SATFINITE, __NV_E4M3);
    }
    WeightPlanes p;
    p.N = N;
    p.K = K;
    p.hi = upload(hi, owned);
    p.lo = upload(lo, owned);
    p.h8 = upload(h8, owned);
    p.l8 = upload(l8, owned);
    p.acc_scale = static_cast<float>(std::ldexp(1.0, -w));
    p.cls = cls;
    return p;
}

Mapper::Mapper(pkv_ctx c, const Geometry& g, const Config& cf, const double* blob, int64_t count, uint32_t precision)
    : ctx(c), geom(g), cfg(cf) {
    geom.validate();
    cfg.validate();
    PKV_REQUIRE(precision >= 1 && precision <= 6, PKV_ECONFIG, "unknown mapper precision mode ", precision);
    na = (precision == 2 || precision == 3 || precision == 5 || precision == 6) ? 2 : 1;
    nb = (precision == 3 || precision == 4 || precision == 5 || precision == 6) ? 2 : 1;
    ffn2_single_act = precision == 5;
    f8 = precision == 6 && use_pair;
    const int64_t D = cfg.d_time;
    PKV_REQUIRE(D % 128 == 0 && D <= 1024, PKV_ECONFIG, "GPU mapper needs d_time % 128 == 0 and <= 1024, got ", D);
    if (cfg.enc_active && cfg.encoder_layers > 0) {
        PKV_REQUIRE(D / cfg.encoder_heads == 64, PKV_ECONFIG,
                    "GPU encoder attention needs d_time / encoder_heads == 64, got ", D / cfg.encoder_heads);
    }
    PKV_REQUIRE(cfg.conv_mid() % 32 == 0 && cfg.conv_mid() <= 1024, PKV_ECONFIG,
                "GPU conv stem needs conv_mid % 32 == 0, got ", cfg.conv_mid());
    PKV_REQUIRE(geom.proxy_heads <= 64, PKV_ECONFIG, "GPU conv stem supports proxy_heads <= 64");
    const auto layout = param_layout(geom, cfg);
    int64_t total = 0;
    std::map<std::string, std::vector<double>> P;
    for (const auto& [name, n] : layout) {
        PKV_REQUIRE_VALUE(total + n <= count, "parameter blob has ", count, " values, layout needs more");
        P[name].assign(blob + total, blob + total + n);
        total += n;
    }
    PKV_REQUIRE_VALUE(total == count, "parameter blob has ", count, " values, layout expects ", total);

    const int64_t hs = geom.proxy_heads, mid = cfg.conv_mid(), F = cfg.ffn_mult * D;
    const int64_t syn = cfg.syn(geom), dh = cfg.d_head, hl = geom.target_heads;
    // PE table for one window (positions restart at 0 per window, mapper.cpp:308)
    {
        std::vector<float> pe(static_cast<size_t>(cfg.crop_len * D));
        for (int64_t pos = 0; pos < cfg.crop_len; ++pos) {
            for (int64_t i = 0; i < D / 2; ++i) {
                const double om = std::pow(10000.0, -2.0 * static_cast<double>(i) / static_cast<double>(D));
                pe[pos * D + 2 * i] = static_cast<float>(std::sin(pos * om));
                pe[pos * D + 2 * i + 1] = static_cast<float>(std::cos(pos * om));
            }
        }
        pe_d = upload(pe, owned);
    }
    if (cfg.conv_active) {
        // BN eval (ops.cpp:852-875) folded: y = x·(γ/√(σ²+ε)) + (β − μ·γ/√(σ²+ε))
        auto fold = [](const std::vector<double>& g, const std::vector<double>& b, const std::vector<double>& rm,
                       const std::vector<double>& rv, std::vector<double>& scale, std::vector<double>& shift) {
            scale.resize(g.size());
            shift.resize(g.size());
            for (size_t c = 0; c < g.size(); ++c) {
                scale[c] = g[c] * (1.0 / std::sqrt(rv[c] + 1e-5));
                shift[c] = b[c] - rm[c] * scale[c];
            }
        };
        std::vector<double> s1, t1, s2, t2;
        fold(P["stem.bn1.gamma"], P["stem.bn1.beta"], P["stem.bn1.running_mean"], P["stem.bn1.running_var"], s1, t1);
        fold(P["stem.bn2.gamma"], P["stem.bn2.beta"], P["stem.bn2.running_mean"], P["stem.bn2.running_var"], s2, t2);
        const auto& w1 = P["stem.conv1.w"];
        const auto& b1 = P["stem.conv1.b"];
        std::vector<double> w1f(w1.size()), b1f(mid);
        for (int64_t c = 0; c < mid; ++c) {
            for (int64_t j = 0; j < hs * 3; ++j) w1f[c * hs * 3 + j] = w1[c * hs * 3 + j] * s1[c];
            b1f[c] = b1[c] * s1[c] + t1[c];
        }
        conv1_w = upload(to_f32(w1f), owned);
        conv1_b = upload(to_f32(b1f), owned);
        const auto& w2 = P["stem.conv2.w"];  // [D, mid, 3]
        const auto& b2 = P["stem.conv2.b"];
        std::vector<double> w2r(static_cast<size_t>(D * 3 * mid)), b2f(D);
        for (int64_t co = 0; co < D; ++co) {
            for (int64_t ci = 0; ci < mid; ++ci) {
                for (int64_t tap = 0; tap < 3; ++tap) {
                    w2r[co * 3 * mid + tap * mid + ci] = w2[(co * mid + ci) * 3 + tap] * s2[co];
                }
            }
            b2f[co] = b2[co] * s2[co] + t2[co];
        }
        conv2 = upload_planes_f8(w2r, D, 3 * mid, kF8Row);
        conv2_b = upload(to_f32(b2f), owned);
    } else {
        bypass_w = upload(to_f32(P["stem.bypass.w"]), owned);  // [D, hs, 1] == [D][hs]
        bypass_b = upload(to_f32(P["stem.bypass.b"]), owned);
    }
    auto transpose = [](const std::vector<double>& w, int64_t in, int64_t out) {
        // reference linear weights are [in, out] (x·W, mapper.cpp:249-251) -> [out][in]
        std::vector<double> t(w.size());
        for (int64_t i = 0; i < in; ++i)
            for (int64_t o = 0; o < out; ++o) t[o * in + i] = w[i * out + o];
        return t;
    };
    if (cfg.enc_active) {
        for (int64_t i = 0; i < cfg.encoder_layers; ++i) {
            const std::string p = "encoder." + std::to_string(i) + ".";
            Block b;
            std::vector<double> wqkv;
            std::vector<double> bqkv;
            for (const char* m : {"q", "k", "v"}) {
                const auto t = transpose(P[p + "attn.w" + m], D, D);
                wqkv.insert(wqkv.end(), t.begin(), t.end());
                const auto& bb = P[p + "attn.b" + m];
                bqkv.insert(bqkv.end(), bb.begin(), bb.end());
            }
            b.qkv = upload_planes_f8(wqkv, 3 * D, D, kF8Act);
            b.qkv_b = upload(to_f32(bqkv), owned);
            b.o = upload_planes(transpose(P[p + "attn.wo"], D, D), D, D);
            b.o_b = upload(to_f32(P[p + "attn.bo"]), owned);
            b.f1 = upload_planes_f8(transpose(P[p + "ffn1.w"], D, F), F, D, kF8Act);
            b.f1_b = upload(to_f32(P[p + "ffn1.b"]), owned);
            b.f2 = upload_planes_f8(transpose(P[p + "ffn2.w"], F, D), D, F, kF8Act);
            b.f2_b = upload(to_f32(P[p + "ffn2.b"]), owned);
            b.ln1_g = upload(to_f32(P[p + "ln1.gamma"]), owned);
            b.ln1_b = upload(to_f32(P[p + "ln1.beta"]), owned);
            b.ln2_g = upload(to_f32(P[p + "ln2.gamma"]), owned);
            b.ln2_b = upload(to_f32(P[p + "ln2.beta"]), owned);
            blocks.push_back(b);
        }
    }
    // Stage 3 folded projection (exact algebra, fp64): rows h·syn+s give the
    // scaled scores Q_l[h]·keys[s]/√dh; rows hl·syn+s give values[s]·out_w.
    {
        const auto& vw = P["cross.value.w"];
        const auto& vb = P["cross.value.b"];
        const auto& ow = P["cross.out.w"];
        out_b = static_cast<float>(P["cross.out.b"][0]);
        const int64_t n_sc = cfg.cross_active ? hl * syn : 0;
        n3 = n_sc + syn;
        ld3 = (n3 + 3) / 4 * 4;
        std::vector<double> w3(static_cast<size_t>(n3 * D), 0.0), b3(n3, 0.0);
        const double inv = 1.0 / std::sqrt(static_cast<double>(dh));
        if (cfg.cross_active) {
            const auto& kw = P["cross.key.w"];
            const auto& kb = P["cross.key.b"];
            const auto& q = P["cross.queries"];
            for (int64_t h = 0; h < hl; ++h) {
                for (int64_t s = 0; s < syn; ++s) {
                    const int64_t r = h * syn + s;
                    for (int64_t i = 0; i < D; ++i) {
                        double acc = 0.0;
                        for (int64_t d = 0; d < dh; ++d) acc += kw[i * syn * dh + s * dh + d] * q[h * dh + d];
                        w3[r * D + i] = acc * inv;
                    }
                    double acc = 0.0;
                    for (int64_t d = 0; d < dh; ++d) acc += kb[s * dh + d] * q[h * dh + d];
                    b3[r] = acc * inv;
                }
            }
        }
        for (int64_t s = 0; s < syn; ++s) {
            const int64_t r = n_sc + s;
            for (int64_t i = 0; i < D; ++i) {
                double acc = 0.0;
                for (int64_t d = 0; d < dh; ++d) acc += vw[i * syn * dh + s * dh + d] * ow[d];
                w3[r * D + i] = acc;
            }
            double acc = 0.0;
            for (int64_t d = 0; d < dh; ++d) acc += vb[s * dh + d] * ow[d];
            b3[r] = acc;
        }
        stage3 = upload_planes(w3, n3, D);
        stage3_b = upload(to_f32(b3), owned);
    }
}

Mapper::~Mapper() {
    for (void* p : owned) cudaFree(p);
}

namespace {
int pick_bn(int64_t n) { return n <= 64 ? 64 : (n <= 128 ? 128 : 256); }
}  // namespace

void Mapper::gemm(const __half* a_h, const __half* a_l, int64_t M, const WeightPlanes& w, const float* bias,
                  GemmEpi epi, GemmEpiParams p, cudaStream_t st, bool single, bool a_single) {
    GemmArgs g;
    g.bn = pick_bn(w.N);
    g.pair = use_pair && w.N >= 256 && M >= 256;  // cta_group::2 256x256 tiles for the big projections
    g.epi = epi;
    p.acc_scale *= w.acc_scale;
    if (f8_gemm(w, M)) {  // FP16F8: a_l holds the e4m3 lo plane then the hi plane ([M, K] bytes each)
        gemm_set_a(g, 0, a_h, M, w.K, w.K);
        const auto* l8 = reinterpret_cast<const uint8_t*>(a_l);
        gemm_set_a8(g, l8, l8 + M * w.K, M, w.K, w.K);
        gemm_set_b(g, 0, w.hi, w.N, w.K, w.K);
        gemm_set_b8(g, w.h8, w.l8);
        p.bias = bias;
        g.p = p;
        gemm_run(g, ctx->sm_count, st);
        count_launch(ctx);
        return;
    }
    gemm_set_a(g, 0, a_h, M, w.K, w.K);
    g.a[1] = g.a[0];
    g.na = 1;
    if (na > 1 && !single && !a_single) gemm_set_a(g, 1, a_l, M, w.K, w.K);
    gemm_set_b(g, 0, w.hi, w.N, w.K, w.K);
    g.b[1] = g.b[0];
    g.nb = 1;
    if (nb > 1 && !single) gemm_set_b(g, 1, w.lo, w.N, w.K, w.K);
    p.bias = bias;
    g.p = p;
    gemm_run(g, ctx->sm_count, st);
    count_launch(ctx);
}

// The e4m3 planes the producer of an FP16F8 GEMM's A operand writes into the
// fp16 lo plane's buffer (lo8 then hi8, `elems` bytes each); empty otherwise.
F8Out Mapper::f8_planes(const WeightPlanes& w, int64_t M, __half* lo_buf, int64_t elems) const {
    F8Out o;
    if (!f8_gemm(w, M) || !lo_buf) return o;
    o.lo8 = reinterpret_cast<uint8_t*>(lo_buf);
    o.hi8 = o.lo8 + elems;
    o.lo_mul = w.cls.lo_mul;
    o.hi_mul = w.cls.hi_mul;
    return o;
}

// x: caller's scores; unit_off[u]: element offset of unit u's [H_s, N] slab
// (head stride N); out_unit[o]: unit feeding output row block o of y [n_out, H_l, N].
void Mapper::run(const float* x, const std::vector<int64_t>& unit_off, int64_t N, const std::vector<int>& out_unit,
                 float* y, cudaStream_t st, float* trace) {
    const int64_t D = cfg.d_time, mid = cfg.conv_mid(), F = cfg.ffn_mult * D, hl = geom.target_heads;
    const int64_t syn = cfg.syn(geom), hs = geom.proxy_heads;
    const auto offs = window_offsets(N, cfg.crop_len, cfg.stride);
    const int64_t W = static_cast<int64_t>(offs.size());
    const int64_t Lw = std::min<int64_t>(N, cfg.crop_len);
    const int64_t units = static_cast<int64_t>(unit_off.size());
    const int64_t rows_per_unit = W * Lw;
    int64_t upc = std::max<int64_t>(1, rows_cap / rows_per_unit);
    if (upc > units) upc = units;
    const int64_t R = upc * rows_per_unit;
    const size_t act_planes = static_cast<size_t>(na);

    // ---- workspace: z | arena(stem: im2col ; enc: h, qkv, ctx ; ffn: h, hidden ; s3: zp, s3)
    const size_t z_b = R * D * 4;
    const size_t stem_b = (cfg.conv_active ? R * 3 * mid * 2 * act_planes : 0);
    const size_t enc_b = R * D * 2 * act_planes * 2 + R * 3 * D * 2;
    const size_t ffn_b = R * D * 2 * act_planes + R * F * 2 * act_planes;
    const size_t s3_b = R * D * 2 * act_planes + R * ld3 * 4;
    const size_t arena_b = std::max(std::max(stem_b, enc_b), std::max(ffn_b, s3_b));
    const size_t logit_b = static_cast<size_t>(units * W * hl * Lw) * 4;
    const size_t mean_b = cfg.normalize_input ? static_cast<size_t>(units * W * hs) * 4 : 0;
    const size_t idx_b = (units + W + out_unit.size()) * 8 + 256;
    const size_t rsc_b = R * 4;  // per-row power-of-two scales of the conv2 / stage-3 A operands
    auto align = [](size_t b) { return (b + 1023) & ~size_t(1023); };
    uint8_t* ws = static_cast<uint8_t*>(work.get(align(z_b) + align(arena_b) + align(logit_b) + align(mean_b) +
                                                 align(idx_b) + align(rsc_b)));
    float* z = reinterpret_cast<float*>(ws);
    uint8_t* arena = ws + align(z_b);
    float* logitsT = reinterpret_cast<float*>(arena + align(arena_b));
    float* means = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(logitsT) + align(logit_b));
    int64_t* d_idx = reinterpret_cast<int64_t*>(reinterpret_cast<uint8_t*>(means) + align(mean_b));
    int64_t* d_unit_off = d_idx;
    int64_t* d_win_off = d_idx + units;
    int* d_out_unit = reinterpret_cast<int*>(d_idx + units + W);
    float* rscale = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(d_idx) + align(idx_b));
    {
        std::vector<int64_t> h(units + W);
        std::copy(unit_off.begin(), unit_off.end(), h.begin());
        std::copy(offs.begin(), offs.end(), h.begin() + units);
        PKV_CUDA(cudaMemcpyAsync(d_idx, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
        PKV_CUDA(cudaMemcpyAsync(d_out_unit, out_unit.data(), out_unit.size() * 4, cudaMemcpyHostToDevice, st));
    }

    for (int64_t u0 = 0; u0 < units; u0 += upc) {
        const int64_t nu = std::min(upc, units - u0);
        const int64_t rows = nu * rows_per_unit;
        MapperSrc src;
        src.x = x;
        src.unit_off = d_unit_off + u0;
        src.win_off = d_win_off;
        src.head_stride = N;
        src.units = static_cast<int>(nu);
        src.W = static_cast<int>(W);
        src.Lw = static_cast<int>(Lw);
        src.hs = static_cast<int>(hs);
        const float* mean = nullptr;
        if (cfg.normalize_input) {
            launch_window_mean(src, means, st);
            count_launch(ctx);
            mean = means;
        }
        const float* pe_stage1 = cfg.enc_active ? pe_d : nullptr;
        // ---- Stage 1
        if (cfg.conv_active) {
            __half* col_h = reinterpret_cast<__half*>(arena);
            __half* col_l = na > 1 ? col_h + rows * 3 * mid : nullptr;
            launch_conv1_im2col(src, mean, conv1_w, conv1_b, static_cast<int>(mid), col_h, col_l, rscale, st,
                                f8_planes(conv2, rows, col_l, rows * 3 * mid));
            count_launch(ctx);
            GemmEpiParams p;
            p.out_f32 = z;
            p.ldo = D;
            p.pe = pe_stage1;
            p.lw = Lw;
            p.row_scale = rscale;
            gemm(col_h, col_l, rows, conv2, conv2_b, pe_stage1 ? EPI_GELU_PE : EPI_GELU_PE, p, st);
        } else {
            launch_bypass_stem(src, mean, bypass_w, bypass_b, pe_stage1, static_cast<int>(D), z, st);
            count_launch(ctx);
        }
        // ---- Stage 2
        if (cfg.enc_active) {
            __half* h_h = reinterpret_cast<__half*>(arena);
            __half* h_l = na > 1 ? h_h + rows * D : nullptr;
            __half* qkv = h_h + rows * D * act_planes;
            __half* c_h = qkv + rows * 3 * D;
            __half* c_l = na > 1 ? c_h + rows * D : nullptr;
            __half* f_h = h_h + rows * D * act_planes;  // ffn phase reuses qkv/ctx space
            __half* f_l = na > 1 ? f_h + rows * F : nullptr;
            for (const Block& b : blocks) {
                launch_layernorm(z, rows, static_cast<int>(D), b.ln1_g, b.ln1_b, h_h, h_l, st,
                                 f8_planes(b.qkv, rows, h_l, rows * D));
                count_launch(ctx);
                GemmEpiParams pq;
                pq.out_h = qkv;
                pq.ldo = 3 * D;
                // q/k/v are rounded to one fp16 plane for attention: one MMA suffices
                gemm(h_h, h_l, rows, b.qkv, b.qkv_b, EPI_F16X, pq, st, qkv_single);
                launch_encoder_attention(qkv, nu * W, Lw, D, cfg.encoder_heads, c_h, c_l, D, st);
                count_launch(ctx);
                GemmEpiParams po;
                po.out_f32 = z;
                po.ldo = D;
                gemm(c_h, c_l, rows, b.o, b.o_b, EPI_RESID, po, st);
                launch_layernorm(z, rows, static_cast<int>(D), b.ln2_g, b.ln2_b, h_h, h_l, st,
                                 f8_planes(b.f1, rows, h_l, rows * D));
                count_launch(ctx);
                GemmEpiParams pf;
                pf.out_h = f_h;
                pf.out_l = ffn2_single_act ? nullptr : f_l;  // mode 5: FFN2 reads one activation plane
                pf.ldo = F;
                if (f8_gemm(b.f2, rows)) {  // mode 6: FFN2's e4m3 correction planes
                    const F8Out o = f8_planes(b.f2, rows, f_l, rows * F);
                    pf.out_l = nullptr;
                    pf.out_l8 = o.lo8;
                    pf.out_h8 = o.hi8;
                    pf.l8_mul = o.lo_mul;
                    pf.h8_mul = o.hi_mul;
                }
                gemm(h_h, h_l, rows, b.f1, b.f1_b, EPI_GELU_F16X, pf, st);
                GemmEpiParams p2;
                p2.out_f32 = z;
                p2.ldo = D;
                gemm(f_h, f_l, rows, b.f2, b.f2_b, EPI_RESID, p2, st, false, ffn2_single_act);
            }
        } else {
            launch_window_colmean_add(z, nu * W, static_cast<int>(Lw), static_cast<int>(D), st);
            count_launch(ctx);
        }
        // ---- Stage 3
        {
            __half* zp_h = reinterpret_cast<__half*>(arena);
            __half* zp_l = na > 1 ? zp_h + rows * D : nullptr;
            float* s3 = reinterpret_cast<float*>(zp_h + rows * D * act_planes);
            launch_split_rows_scaled(z, rows, static_cast<int>(D), zp_h, zp_l, rscale, st);
            count_launch(ctx);
            GemmEpiParams p;
            p.out_f32 = s3;
            p.ldo = ld3;
            p.row_scale = rscale;
            gemm(zp_h, zp_l, rows, stage3, stage3_b, EPI_F32, p, st);
            launch_stage3(s3, rows, static_cast<int>(ld3), static_cast<int>(hl), static_cast<int>(syn),
                          cfg.cross_active, out_b, static_cast<int>(Lw), logitsT + u0 * W * hl * Lw,
                          (trace && cfg.cross_active) ? trace + u0 * W * Lw * hl * syn : nullptr, st);
            count_launch(ctx);
        }
    }
    // ---- sliding_forward's overlap average (+ forward_full's layer fan-out)
    const int64_t n_regular = (N <= cfg.crop_len) ? 1 : (N - cfg.crop_len) / cfg.stride + 1;
    const int tail = (W > n_regular) ? static_cast<int>(offs.back()) : -1;
    launch_window_average(logitsT, d_out_unit, static_cast<int>(out_unit.size()), static_cast<int>(hl),
                          static_cast<int>(W), static_cast<int>(Lw), static_cast<int>(cfg.stride),
                          static_cast<int>(n_regular), tail, N, y, st);
    count_launch(ctx);
}

}  // namespace pkv

using namespace pkv;

namespace {

void run_batch(Mapper& m, const float* x, int64_t B, int64_t N, float* y, cudaStream_t st, float* trace = nullptr) {
    std::vector<int64_t> unit_off(B);
    std::vector<int> out_unit(B);
    for (int64_t b = 0; b < B; ++b) {
        unit_off[b] = b * m.geom.proxy_heads * N;
        out_unit[b] = static_cast<int>(b);
    }
    m.run(x, unit_off, N, out_unit, y, st, trace);
}

// mapper.cpp:277-282
void check_pair_input(const Mapper& m, int64_t B, int64_t n) {
    PKV_REQUIRE_SHAPE(B > 0 && n > 0, "forward_pair input must be [B, H_s, N] with positive extents");
    PKV_REQUIRE_VALUE(n <= m.cfg.crop_len, "input length ", n, " exceeds crop_len ", m.cfg.crop_len,
                      "; long inputs go through sliding_forward");
}

// Host fp64 in -> device fp32 -> fn -> host fp64 out (synchronous, the
// mapper's own default-stream scratch).
template <typename F>
void host_roundtrip(const double* xh, size_t nx, double* yh, size_t ny, double* ah, size_t na, F&& fn) {
    std::vector<float> xf(nx);
    for (size_t i = 0; i < nx; ++i) xf[i] = static_cast<float>(xh[i]);
    float* d = nullptr;
    const size_t bytes = (nx + ny + na) * sizeof(float);
    PKV_CUDA(cudaMalloc(&d, bytes));
    struct Free {
        float* p;
        ~Free() { cudaFree(p); }
    } guard_free{d};
    PKV_CUDA(cudaMemcpy(d, xf.data(), nx * sizeof(float), cudaMemcpyHostToDevice));
    fn(d, d + nx, na ? d + nx + ny : nullptr);
    PKV_CUDA(cudaStreamSynchronize(nullptr));
    std::vector<float> yf(ny + na);
    PKV_CUDA(cudaMemcpy(yf.data(), d + nx, (ny + na) * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < ny; ++i) yh[i] = yf[i];
    for (size_t i = 0; i < na; ++i) ah[i] = yf[ny + i];
}

}  // namespace

extern "C" {

pkv_status pkv_layer_pair(int64_t target_layer, const int64_t* geom5, int64_t* out) {
    return guard([&] { *out = layer_pair(target_layer, Geometry::from5(geom5)); });
}

pkv_status pkv_window_offsets(int64_t n, int64_t crop, int64_t stride, int64_t* out, int64_t cap, int64_t* count) {
    return guard([&] {
        const auto v = window_offsets(n, crop, stride);
        *count = static_cast<int64_t>(v.size());
        for (int64_t i = 0; i < *count && i < cap; ++i) out[i] = v[i];
    });
}

pkv_status pkv_mapper_init_params(const int64_t* geom5, const int64_t* cfg12, uint64_t seed, double* blob_out,
                                  int64_t* count_out) {
    return guard([&] {
        const Geometry g = Geometry::from5(geom5);
        const Config c = Config::from12(cfg12);
        g.validate();
        c.validate();
        if (!blob_out) {
            int64_t n = 0;
            for (const auto& e : param_layout(g, c)) n += e.second;
            *count_out = n;
            return;
        }
        const auto blob = init_params(g, c, seed);
        std::memcpy(blob_out, blob.data(), blob.size() * sizeof(double));
        *count_out = static_cast<int64_t>(blob.size());
    });
}

pkv_status pkv_mapper_create(pkv_ctx ctx, const int64_t* geom5, const int64_t* cfg12, const double* blob, int64_t count,
                             uint32_t precision, pkv_mapper* out) {
    return guard([&] {
        require_ctx(ctx);
        auto* h = new pkv_mapper_s();
        try {
            h->m.reset(new Mapper(ctx, Geometry::from5(geom5), Config::from12(cfg12), blob, count, precision));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void pkv_mapper_destroy(pkv_mapper m) { delete m; }

pkv_status pkv_mapper_forward_full(pkv_mapper mh, const float* x_all, int64_t B, int64_t N, float* y_all,
                                   void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        PKV_REQUIRE_SHAPE(B > 0 && N > 0, "forward_full input must be [B, L_s, H_s, N] with positive extents");
        const Geometry& g = m.geom;
        // dedup: one unit per (batch, proxy layer actually paired)
        std::vector<int64_t> unit_off;
        std::vector<int> out_unit(static_cast<size_t>(B * g.target_layers));
        std::map<std::pair<int64_t, int64_t>, int> unit_of;
        for (int64_t b = 0; b < B; ++b) {
            for (int64_t ll = 1; ll <= g.target_layers; ++ll) {
                const int64_t ls = layer_pair(ll, g);
                auto key = std::make_pair(b, ls);
                auto it = unit_of.find(key);
                if (it == unit_of.end()) {
                    it = unit_of.emplace(key, static_cast<int>(unit_off.size())).first;
                    unit_off.push_back(((b * g.proxy_layers) + (ls - 1)) * g.proxy_heads * N);
                }
                out_unit[b * g.target_layers + (ll - 1)] = it->second;
            }
        }
        m.run(x_all, unit_off, N, out_unit, y_all, static_cast<cudaStream_t>(stream));
    });
}

pkv_status pkv_mapper_forward_pair(pkv_mapper mh, const float* x, int64_t B, int64_t n, float* y, float* attn,
                                   void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        check_pair_input(m, B, n);
        run_batch(m, x, B, n, y, static_cast<cudaStream_t>(stream), attn);
    });
}

pkv_status pkv_mapper_forward_pair_host(pkv_mapper mh, const double* x, int64_t B, int64_t n, double* y,
                                        double* attn) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        check_pair_input(m, B, n);
        PKV_CUDA(cudaSetDevice(m.ctx->device));
        const int64_t hl = m.geom.target_heads, syn = m.cfg.syn(m.geom);
        const size_t na = (attn && m.cfg.cross_active) ? static_cast<size_t>(B * n * hl * syn) : 0;
        host_roundtrip(x, static_cast<size_t>(B * m.geom.proxy_heads * n), y, static_cast<size_t>(B * hl * n), attn,
                       na, [&](const float* xd, float* yd, float* ad) { run_batch(m, xd, B, n, yd, nullptr, ad); });
    });
}

pkv_status pkv_mapper_sliding_forward_host(pkv_mapper mh, const double* x, int64_t B, int64_t N, double* y) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        PKV_REQUIRE_SHAPE(B > 0 && N > 0, "sliding_forward input must be [B, H_s, N]");
        PKV_CUDA(cudaSetDevice(m.ctx->device));
        host_roundtrip(x, static_cast<size_t>(B * m.geom.proxy_heads * N), y,
                       static_cast<size_t>(B * m.geom.target_heads * N), nullptr, 0,
                       [&](const float* xd, float* yd, float*) { run_batch(m, xd, B, N, yd, nullptr); });
    });
}

pkv_status pkv_mapper_forward_full_host(pkv_mapper mh, const double* x, int64_t B, int64_t N, double* y) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        PKV_REQUIRE_SHAPE(B > 0 && N > 0, "forward_full input must be [B, L_s, H_s, N] with positive extents");
        PKV_CUDA(cudaSetDevice(m.ctx->device));
        const Geometry& g = m.geom;
        host_roundtrip(x, static_cast<size_t>(B * g.proxy_layers * g.proxy_heads * N), y,
                       static_cast<size_t>(B * g.target_layers * g.target_heads * N), nullptr, 0,
                       [&](const float* xd, float* yd, float*) {
                           PKV_REQUIRE(pkv_mapper_forward_full(mh, xd, B, N, yd, nullptr) == PKV_OK, PKV_ECUDA,
                                       "forward_full failed");
                       });
    });
}

pkv_status pkv_mapper_sliding_forward(pkv_mapper mh, const float* x, int64_t B, int64_t N, float* y, void* stream) {
    return guard([&] {
        PKV_REQUIRE_VALUE(mh != nullptr, "null pkv_mapper");
        Mapper& m = *mh->m;
        PKV_REQUIRE_SHAPE(B > 0 && N > 0, "sliding_forward input must be [B, H_s, N]");
        run_batch(m, x, B, N, y, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

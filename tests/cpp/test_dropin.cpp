// C++ drop-in smoke test (include/proxykv_b200/proxykv.hpp over libpkv_b200.so),
// written like the reference's own doctest cases (proj/tests/test_pruning.cpp,
// test_mapper.cpp). Without a GPU only the host logic and the loud NoDeviceError
// are exercised; with a B200 the GPU select is checked against the reference's
// known answers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "proxykv_b200/proxykv.hpp"

using namespace proxykv_b200;

static int failures = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                            \
        }                                                          \
    } while (0)

template <typename E, typename F>
static bool throws_with(F&& f, const std::string& frag) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(frag) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

// test_pruning.cpp:20-32: the stable-sort oracle (value desc, index asc)
static std::vector<int64_t> sort_oracle(const std::vector<double>& v, int64_t k) {
    std::vector<int64_t> idx(v.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return v[a] > v[b]; });
    idx.resize(static_cast<size_t>(k));
    std::sort(idx.begin(), idx.end());
    return idx;
}

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // pruning.cpp:14-18 / test_pruning.cpp:61-62
    CHECK(retention_count(0.34, 3) == 2);
    CHECK(throws<ValueError>([] { retention_count(0.0, 3); }));
    CHECK(throws<ValueError>([] { retention_count(1.5, 3); }));
    // test_mapper.cpp:43-61, 201-206
    ModelGeometry g;
    g.target_layers = 32;
    g.proxy_layers = 16;
    CHECK(layer_pair(17, g) == 9 && layer_pair(32, g) == 16 && layer_pair(1, g) == 1);
    CHECK(throws<ValueError>([&] { layer_pair(0, g); }));
    CHECK((window_offsets(13, 8, 4) == std::vector<int64_t>{0, 4, 5}));
    CHECK((window_offsets(3072, 2048, 1024) == std::vector<int64_t>{0, 1024}));
    MapperConfig bad;
    bad.crop_len = 64;
    bad.stride = 128;
    CHECK(throws<ValueError>([&] { mapper_init_params(g, bad, 0); }));
    CHECK(mapper_init_params(g, MapperConfig{}, 1).size() > 15000000);
    // loss.hpp:16-31 defaults carried into the C struct
    const LossConfig lcfg;  // c() points into lcfg.ratios: keep lcfg alive while lc is used
    const pkv_loss_config lc = lcfg.c();
    CHECK(lc.n_ratios == 7 && lc.ratios[0] == 0.05 && lc.max_pairs == 4096 && lc.lambda_mse == 20.0);

    if (pkv_sm100_device_count() == 0) {
        CHECK(throws<NoDeviceError>([] { Context c(0); }));
        std::printf("[dropin] host-only checks: %s\n", failures ? "FAILED" : "ok");
        return failures ? 1 : 0;
    }
    Context ctx(0);
    // test_pruning.cpp:47-59
    PruneMask m = topk_mask(ctx, {3, 1, 2}, {1, 1, 3}, 0.34);
    CHECK(m.k == 2 && m.bits == (std::vector<uint8_t>{1, 0, 1}));
    PruneMask t = topk_mask(ctx, {0.3, 0.3, 0.1}, {1, 1, 3}, 0.3);
    CHECK(t.k == 1 && t.bits == (std::vector<uint8_t>{1, 0, 0}));
    CHECK(throws<ValueError>([&] { topk_mask(ctx, {3, 1, 2}, {1, 1, 3}, 0.0); }));
    // test_pruning.cpp:169-174
    PruneMask a = topk_mask(ctx, {0.5, 0.1, 0.4, 0.2, 0.3}, {1, 1, 5}, 0.4);
    MaskApplication app = apply_mask(a, 128, 2);
    CHECK((app.retained[0] == std::vector<int64_t>{0, 2}));
    CHECK(app.bytes_saved_per_head == 3 * 128 * 2 * 2);

    // ---- reference signatures (no context argument) ----
    // topk_indices (pruning.cpp:20-35) on doubles that collide in fp32
    {
        std::mt19937_64 rng(7);
        std::vector<double> v(5000);
        for (size_t i = 0; i < v.size(); ++i) v[i] = 0.25 + double(rng() % 7) / 8.0 + double(rng() % 1000003) * 1e-13;
        for (int64_t k : {1, 17, 1000, 4999, 5000}) {
            auto got = topk_indices(v.data(), static_cast<int64_t>(v.size()), k);
            CHECK(got == sort_oracle(v, k));
        }
        CHECK(throws_with<ValueError>([&] { topk_indices(v.data(), 10, 11); }, "out of range"));
        ScoreTensor st({2, 2500}, v);
        PruneMask pm = topk_mask(st, 0.2);
        CHECK(pm.k == 500);
        for (int s = 0; s < 2; ++s) {
            std::vector<double> row(v.begin() + s * 2500, v.begin() + (s + 1) * 2500);
            const auto want = sort_oracle(row, 500);
            std::vector<int64_t> got;
            for (int64_t i = 0; i < 2500; ++i)
                if (pm.bits[static_cast<size_t>(s * 2500 + i)]) got.push_back(i);
            CHECK(got == want);
        }
        // topk_overlap: self = 1, symmetric, k mismatch (test_pruning.cpp:141-153)
        PruneMask pm2 = topk_mask(ScoreTensor({2, 2500}, std::vector<double>(v.rbegin(), v.rend())), 0.2);
        CHECK(topk_overlap(pm, pm) == 1.0);
        CHECK(topk_overlap(pm, pm2) == topk_overlap(pm2, pm));
        PruneMask pm3 = topk_mask(st, 0.3);
        CHECK(throws<ValueError>([&] { topk_overlap(pm, pm3); }));
    }
    // mapper: forward_pair / sliding_forward / forward_full on host tensors
    {
        ModelGeometry mg;
        mg.target_layers = 4;
        mg.target_heads = 8;
        mg.proxy_layers = 2;
        mg.proxy_heads = 4;
        mg.head_dim = 64;
        MapperConfig mc;
        mc.encoder_layers = 2;
        MapperParams mp = MapperParams::init(mg, mc, 3);
        std::mt19937_64 rng(11);
        std::uniform_real_distribution<double> u(0.0, 2.0);
        Tensor x({2, 4, 300});
        for (double& e : x.data) e = u(rng);
        StageTrace tr;
        Tensor y = forward_pair(x, mp, false, &tr);
        CHECK((y.shape == Shape{2, 8, 300}));
        CHECK((tr.cross_attention.shape == Shape{2, 300, 8, 4}));
        // attention rows sum to 1 (test_mapper.cpp:122-137)
        double worst = 0.0;
        for (size_t r = 0; r < tr.cross_attention.data.size() / 4; ++r) {
            double s = 0.0;
            for (int j = 0; j < 4; ++j) s += tr.cross_attention.data[r * 4 + j];
            worst = std::max(worst, std::fabs(s - 1.0));
        }
        CHECK(worst < 1e-5);
        // sliding == forward_pair for N <= crop (test_mapper.cpp:226-234)
        CHECK(sliding_forward(x, mp).data == y.data);
        // n > crop -> ValueError naming sliding_forward (test_mapper.cpp:90-96)
        Tensor xl({1, 4, 2049});
        CHECK(throws_with<ValueError>([&] { forward_pair(xl, mp, false); }, "sliding_forward"));
        CHECK(throws<ShapeError>([&] { forward_pair(Tensor({1, 3, 10}), mp, false); }));
        // training forward_pair runs the GPU trainer: BN running statistics move, the eval
        // path then uses them, and backward() gives every parameter gradient
        {
            MapperParams tp = MapperParams::init(mg, mc, 3);
            const std::vector<double> before = tp.blob;
            CHECK(throws<ValueError>([&] { tp.backward(std::vector<double>(2 * 8 * 300, 1.0)); }));
            Tensor yt = forward_pair(x, tp, true);
            CHECK((yt.shape == Shape{2, 8, 300}));
            bool finite = true;
            for (double v : yt.data) finite = finite && std::isfinite(v);
            CHECK(finite);
            CHECK(tp.blob != before);  // running statistics updated (ops.cpp:846-849)
            const std::vector<double> gr = tp.backward(std::vector<double>(yt.data.size(), 1.0 / 4800.0));
            CHECK(gr.size() + 2 * (256 + 512) == before.size());  // every parameter, no BN buffers
            double gn = 0.0;
            for (double v : gr) gn += v * v;
            CHECK(gn > 0.0 && std::isfinite(gn));
            CHECK(throws<ShapeError>([&] { tp.backward(std::vector<double>(3, 0.0)); }));
            CHECK(!(forward_pair(x, tp, false).data == y.data));  // eval with the moved statistics
        }
        // forward_full pairing {1,1,2,2}: shared pairs bit-identical (test_mapper.cpp:268-292)
        Tensor xa({1, 2, 4, 2500});
        for (double& e : xa.data) e = u(rng);
        Tensor ya = forward_full(xa, mp);
        CHECK((ya.shape == Shape{1, 4, 8, 2500}));
        const size_t L = 8 * 2500;
        CHECK(std::equal(ya.data.begin(), ya.data.begin() + L, ya.data.begin() + L));
        CHECK(std::equal(ya.data.begin() + 2 * L, ya.data.begin() + 3 * L, ya.data.begin() + 3 * L));
        // forward_full layer 1 == sliding_forward of proxy layer 1
        Tensor x1({1, 4, 2500}, std::vector<double>(xa.data.begin(), xa.data.begin() + 4 * 2500));
        CHECK(std::equal(ya.data.begin(), ya.data.begin() + L, sliding_forward(x1, mp).data.begin()));
    }
    std::printf("[dropin] gpu checks: %s\n", failures ? "FAILED" : "ok");
    return failures ? 1 : 0;
}

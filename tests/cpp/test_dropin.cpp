// C++ drop-in smoke test (include/proxykv_b200/proxykv.hpp over libpkv_b200.so),
// written like the reference's own doctest cases (proj/tests/test_pruning.cpp,
// test_mapper.cpp). Without a GPU only the host logic and the loud NoDeviceError
// are exercised; with a B200 the GPU select is checked against the reference's
// known answers.
#include <cstdio>
#include <cstdlib>
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
    std::printf("[dropin] gpu checks: %s\n", failures ? "FAILED" : "ok");
    return failures ? 1 : 0;
}

// test_dropin.cpp — the gnstk drop-in (include/gnstk/*.hpp, backed by the
// B200 kernels) against the reference's own unit-test expectations
// (proj/tests/test_layers.cpp, test_gns.cpp, test_costmodel.cpp; values ported,
// not code).  Exit code = number of failed checks.  Needs a GPU.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnstk/costmodel.hpp"
#include "gnstk/gns.hpp"
#include "gnstk/layers.hpp"

using namespace gnstk;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                   \
    do {                                                                           \
        ++g_checks;                                                                \
        if (!(c)) {                                                                \
            ++g_fail;                                                              \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);               \
        }                                                                          \
    } while (0)
#define CHECK_THROWS_INVALID(expr)                                                 \
    do {                                                                           \
        ++g_checks;                                                                \
        bool ok = false;                                                           \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (const std::invalid_argument&) {                                   \
            ok = true;                                                             \
        }                                                                          \
        if (!ok) {                                                                 \
            ++g_fail;                                                              \
            std::printf("FAIL %s:%d: expected invalid_argument: %s\n", __FILE__, __LINE__, #expr); \
        }                                                                          \
    } while (0)

static bool close(double a, double b, double rtol, double atol = 0.0) {
    return std::abs(a - b) <= atol + rtol * std::max(std::abs(a), std::abs(b));
}

// deterministic normal-ish draws for random cases (splitmix64 + Box-Muller)
struct Rng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
    double normal() { return std::sqrt(-2.0 * std::log(unit() + 1e-300)) * std::cos(6.283185307179586 * unit()); }
    Index below(Index n) { return (Index)(unit() * (double)n); }
};
static Tensor rnd(Shape s, Rng& r) {
    Tensor t(std::move(s));
    for (Index i = 0; i < t.size(); ++i) t[i] = r.normal();
    return t;
}

int main() {
    // ---- layers: LayerNorm (test_layers.cpp:151-212) ----
    {
        LayerNormLayer ln{Tensor({2}, {1, 1}), Tensor({2}, {0, 0}), 1e-5};
        LayerNormCache cache{Tensor({1, 1, 2}, {1, -1}), Tensor({1, 1}, {1.0})};
        auto res = layernorm_backward_simultaneous(ln, cache, Tensor({1, 1, 2}, {2, 3}));
        const Tensor& dg = res.grads.weight_grads.at("gamma");
        const Tensor& db = res.grads.weight_grads.at("beta");
        CHECK(dg[0] == 2 && dg[1] == -3);
        CHECK(db[0] == 2 && db[1] == 3);
        CHECK(res.grads.per_example_sqnorms.at("gamma") == 13);
        CHECK(res.grads.per_example_sqnorms.at("beta") == 13);
    }
    {
        LayerNormLayer ln{Tensor({2}, {1, 1}), Tensor({2}, {0, 0}), 1e-12};
        auto r1 = layernorm_forward(ln, Tensor({2}, {1, -1}));
        CHECK(close(r1.output[0], 1.0, 1e-6) && close(r1.output[1], -1.0, 1e-6));
        LayerNormLayer ln2{Tensor({2}, {1, 1}), Tensor({2}, {0.5, -0.5}), 1e-5};
        auto r2 = layernorm_forward(ln2, Tensor({2}, {3, 3}));
        CHECK(close(r2.output[0], 0.5, 1e-12) && close(r2.output[1], -0.5, 1e-12));
        auto r3 = layernorm_forward(ln, Tensor({2}, {0, 2}));
        CHECK(close(r3.cache.normalized[0], -1.0, 1e-6) && close(r3.cache.normalized[1], 1.0, 1e-6));
        CHECK_THROWS_INVALID(layernorm_forward(LayerNormLayer{Tensor({2}, {1, 1}), Tensor({2}), 0.0}, Tensor({2})));
    }
    {
        Rng rng{29};
        LayerNormLayer ln{rnd({4}, rng), rnd({4}, rng), 1e-5};
        auto fwd = layernorm_forward(ln, rnd({2, 3, 4}, rng));
        auto res = layernorm_backward_simultaneous(ln, fwd.cache, Tensor({2, 3, 4}));
        CHECK(res.grads.per_example_sqnorms.at("gamma") == 0);
        CHECK(res.grads.per_example_sqnorms.at("beta") == 0);
        CHECK(sqnorm_all(res.input_grad) == 0);
        CHECK_THROWS_INVALID(layernorm_backward_simultaneous(ln, fwd.cache, Tensor({2, 3, 5})));
    }
    {
        Rng rng{31};
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = 2 + rng.below(3), t = 1 + rng.below(5), k = 2 + rng.below(5);
            LayerNormLayer ln{rnd({k}, rng), rnd({k}, rng), 1e-5};
            auto fwd = layernorm_forward(ln, rnd({b, t, k}, rng));
            Tensor g = rnd({b, t, k}, rng);
            auto res = layernorm_backward_simultaneous(ln, fwd.cache, g);
            double mg = 0, mb = 0;
            for (Index e = 0; e < b; ++e) {
                std::vector<double> pg(k, 0.0), pb(k, 0.0);
                for (Index m = 0; m < t; ++m)
                    for (Index i = 0; i < k; ++i) {
                        pg[i] += fwd.cache.normalized[(e * t + m) * k + i] * g[(e * t + m) * k + i];
                        pb[i] += g[(e * t + m) * k + i];
                    }
                for (Index i = 0; i < k; ++i) {
                    mg += pg[i] * pg[i];
                    mb += pb[i] * pb[i];
                }
            }
            mg /= (double)b;
            mb /= (double)b;
            CHECK(close(res.grads.per_example_sqnorms.at("gamma"), (double)(b * b) * mg, 1e-9));
            CHECK(close(res.grads.per_example_sqnorms.at("beta"), (double)(b * b) * mb, 1e-9));
        }
    }
    // ---- layers: linear (test_layers.cpp:51-149) ----
    {
        LinearLayer layer{Tensor({2, 1}, {0, 0}), std::nullopt};
        auto res = linear_backward_simultaneous(layer, Tensor({2, 1, 2}, {1, 2, 3, 4}), Tensor({2, 1, 1}, {1, 2}));
        const Tensor& dW = res.grads.weight_grads.at("weight");
        CHECK(dW[0] == 7 && dW[1] == 10);
        const Tensor& raw = res.grads.per_example_sqnorms_raw.at("weight");
        CHECK(raw[0] == 5 && raw[1] == 100);
        CHECK(close(res.grads.per_example_sqnorms.at("weight"), 210, 1e-12));
        CHECK(res.grads.batch_size == 2);
    }
    {
        LinearLayer layer{Tensor({1, 1}, {0}), std::nullopt};
        auto res = linear_backward_simultaneous(layer, Tensor({1, 2, 1}, {1, 1}), Tensor({1, 2, 1}, {2, 3}));
        CHECK(res.grads.weight_grads.at("weight")[0] == 5);
        CHECK(res.grads.per_example_sqnorms.at("weight") == 25);
        CHECK(linear_perexample_sqnorm_frobenius(Tensor({1, 2, 1}, {1, 1}), Tensor({1, 2, 1}, {2, 3}))[0] == 25);
        CHECK(linear_perexample_sqnorm_frobenius(Tensor({1, 2, 1}, {1, 1}), Tensor({1, 2, 1}))[0] == 0);
        CHECK_THROWS_INVALID(linear_perexample_sqnorm_frobenius(Tensor({2, 2}), Tensor({2, 2})));
    }
    {
        Rng rng{23};
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = 1 + rng.below(4), t = 1 + rng.below(5), k = 1 + rng.below(6), l = 1 + rng.below(6);
            LinearLayer layer{rnd({k, l}, rng), rnd({l}, rng)};
            Tensor x = rnd({b, t, k}, rng), g = rnd({b, t, l}, rng);
            Tensor frob = linear_perexample_sqnorm_frobenius(x, g);
            auto res = linear_backward_simultaneous(layer, x, g);
            const Tensor& raw = res.grads.per_example_sqnorms_raw.at("weight");
            for (Index e = 0; e < b; ++e) CHECK(close(frob[e], raw[e], 1e-12, 1e-15));
            // bias: per-example ||sum_t g||^2
            double sb = 0;
            for (Index e = 0; e < b; ++e)
                for (Index j = 0; j < l; ++j) {
                    double v = 0;
                    for (Index m = 0; m < t; ++m) v += g[(e * t + m) * l + j];
                    sb += v * v;
                }
            CHECK(close(res.grads.per_example_sqnorms.at("bias"), (double)b * sb, 1e-9));
            // dx = g W^T
            for (Index r = 0; r < b * t; ++r)
                for (Index i = 0; i < k; ++i) {
                    double acc = 0;
                    for (Index j = 0; j < l; ++j) acc += g[r * l + j] * layer.weight[i * l + j];
                    CHECK(close(res.input_grad[r * k + i], acc, 1e-12, 1e-14));
                }
        }
    }
    {
        Rng rng{47};  // test_layers.cpp:349-362: g*2 scales norms by 4 exactly
        LinearLayer layer{rnd({3, 4}, rng), rnd({4}, rng)};
        Tensor x = rnd({3, 2, 3}, rng), g = rnd({3, 2, 4}, rng);
        auto base = linear_backward_simultaneous(layer, x, g);
        auto scaled = linear_backward_simultaneous(layer, x, scale(g, 2.0));
        CHECK(scaled.grads.per_example_sqnorms.at("weight") == 4.0 * base.grads.per_example_sqnorms.at("weight"));
        CHECK(scaled.grads.per_example_sqnorms.at("bias") == 4.0 * base.grads.per_example_sqnorms.at("bias"));
        CHECK_THROWS_INVALID(linear_backward_simultaneous(layer, Tensor({2, 2, 5}), Tensor({2, 2, 4})));
    }
    // ---- embedding (test_layers.cpp:300-347) ----
    {
        EmbeddingLayer layer{Tensor({3, 1})};
        const std::int32_t ids_repeat[] = {0, 0};
        Tensor g({1, 2, 1}, {1, 2});
        auto res = embedding_backward_simultaneous(layer, ids_repeat, 1, 2, g);
        CHECK(res.weight_grads.at("weight")[0] == 3);
        CHECK(res.per_example_sqnorms.at("weight") == 9);
        const std::int32_t ids_distinct[] = {0, 1};
        auto res2 = embedding_backward_simultaneous(layer, ids_distinct, 1, 2, g);
        CHECK(res2.weight_grads.at("weight")[0] == 1);
        CHECK(res2.weight_grads.at("weight")[1] == 2);
        CHECK(res2.per_example_sqnorms.at("weight") == 5);
        auto zero = embedding_backward_simultaneous(layer, ids_distinct, 1, 2, Tensor({1, 2, 1}));
        CHECK(zero.per_example_sqnorms.at("weight") == 0);
        const std::int32_t bad_ids[] = {0, 5};
        CHECK_THROWS_INVALID(embedding_backward_simultaneous(layer, bad_ids, 1, 2, g));
    }
    {
        Rng rng{43};  // dense one-hot contraction per example, exact in fp64
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = 1 + rng.below(4), t = 1 + rng.below(5), v = 2 + rng.below(7), d = 1 + rng.below(6);
            EmbeddingLayer layer{rnd({v, d}, rng)};
            std::vector<std::int32_t> ids((std::size_t)(b * t));
            for (auto& id : ids) id = (std::int32_t)rng.below(v);
            Tensor g = rnd({b, t, d}, rng);
            auto res = embedding_backward_simultaneous(layer, ids, b, t, g);
            Tensor total({v, d});
            double mean_single = 0.0;
            const Tensor& raw = res.per_example_sqnorms_raw.at("weight");
            for (Index eb = 0; eb < b; ++eb) {
                Tensor single({v, d});
                for (Index tt = 0; tt < t; ++tt)
                    for (Index j = 0; j < d; ++j) single[ids[eb * t + tt] * d + j] += g[(eb * t + tt) * d + j];
                double sq = 0.0;
                for (Index i = 0; i < single.size(); ++i) sq += single[i] * single[i];
                mean_single += sq;
                CHECK(close(raw[eb], sq, 1e-12, 1e-300));
                for (Index i = 0; i < total.size(); ++i) total[i] += single[i];
            }
            mean_single /= (double)b;
            bool eq = true;
            for (Index i = 0; i < total.size(); ++i) eq = eq && res.weight_grads.at("weight")[i] == total[i];
            CHECK(eq);
            CHECK(close(res.per_example_sqnorms.at("weight"), (double)(b * b) * mean_single, 1e-9));
        }
    }
    // ---- gns (test_gns.cpp:15-124) ----
    {
        GradStats st{1.25, 1.5, 2, 1, 2};
        CHECK(estimate_g2(st) == 1.0);
        CHECK(estimate_s(st) == 0.5);
        auto e = make_gns_estimate(estimate_g2(st), estimate_s(st));
        CHECK(e.b_simple_defined && e.b_simple == 0.5);
        CHECK_THROWS_INVALID(estimate_g2(GradStats{1.0, 1.0, 2, 2, 1}));
        EmaState s{0.5};
        s = ema_update(s, 1.0);
        CHECK(s.value == 1.0);
        s = ema_update(s, 3.0);
        CHECK(s.value == 2.0);
        CHECK_THROWS_INVALID(ema_update(EmaState{0.0}, 1.0));
        CHECK_THROWS_INVALID(smoothed_gns(EmaState{0.5}, s));
        std::map<LayerKey, GradStats> by;
        by[{"a", LayerType::Linear}] = {1.0, 2.0, 4, 1, 4};
        by[{"b", LayerType::Linear}] = {2.0, 3.0, 4, 1, 4};
        by[{"c", LayerType::LayerNorm}] = {1.0, 0.5, 4, 1, 4};
        const GradStats all = aggregate(by, std::nullopt);
        CHECK(all.g_big_sqnorm == 4.0 && all.g_small_sqnorm_mean == 5.5 && all.b_big == 4);
        CHECK(aggregate(by, LayerType::LayerNorm).g_big_sqnorm == 1.0);
        CHECK_THROWS_INVALID(aggregate(by, LayerType::Embedding));
        CHECK(layer_type_name(LayerType::LayerNorm) == "layernorm");
    }
    // ---- cost model (acceptance.cpp:232-235) ----
    {
        CHECK(std::abs(crossover_t(1024, 1024, CostCriterion::IO) - 724.08) < 0.01);
        CHECK(std::abs(crossover_t(1024, 1024, CostCriterion::FLOPS) - 22.63) < 0.01);
        CHECK(flops({2, 3, 4, 5, 4}, CostMethod::Simultaneous).weight_grad == 2 * 4 * 5 * (2 * 3 - 1) + 4 * 5 * (2 - 1));
        CHECK_THROWS_INVALID(crossover_t(0, 1, CostCriterion::IO));
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail;
}

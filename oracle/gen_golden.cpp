// gen_golden.cpp — emits golden vectors by running the UNMODIFIED reference
// library (compiled from /root/reference by oracle/Makefile).  TEST
// INFRASTRUCTURE ONLY.  Run via tests/golden/make_golden.py, which commits the
// JSON under tests/golden/.
//
// Case families (reference test they mirror, relative to /root/reference):
//   ln_kat        proj/tests/test_layers.cpp:167-176   (hand-worked LN backward)
//   ln_fwd_kat    proj/tests/test_layers.cpp:151-165   (LN forward examples)
//   ln_zero       proj/tests/test_layers.cpp:178-188   (zero upstream gradient)
//   ln_rand31     proj/tests/test_layers.cpp:190-212   (seed 31, 25 reps)
//   acc1_linear / acc1_ln   proj/tests/acceptance.cpp:48-104 (seed 1001, 100+100 reps)
//   acc2_frob     proj/tests/acceptance.cpp:109-126    (seed 1002, 100 reps)
//   lin_kat       proj/tests/test_layers.cpp:51-63, 77-85, 109-118
//   lin_rand17    proj/tests/test_layers.cpp:87-107    (seed 17, 25 reps)
//   frob_rand23   proj/tests/test_layers.cpp:135-149   (seed 23, 25 reps)
//   emb_kat       proj/tests/test_layers.cpp:300-319   (embedding worked examples)
//   emb_rand43    proj/tests/test_layers.cpp:321-347   (seed 43, 25 reps)
//   ln_cfg1       BASELINE config 1 (B=8 T=128 D=768), synthetic recipe of SURVEY.md §8(d)
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gnstk/gns.hpp"
#include "gnstk/layers.hpp"
#include "gnstk/rng.hpp"
#include "gnstk/tensor.hpp"
#include "oracle.h"

using namespace gnstk;

namespace {

FILE* out;
bool first_case = true;

void arr(const char* key, const double* p, Index n, bool comma = true) {
    std::fprintf(out, "\"%s\": [", key);
    for (Index i = 0; i < n; ++i) std::fprintf(out, "%s%.17g", i ? ", " : "", p[i]);
    std::fprintf(out, "]%s", comma ? ", " : "");
}
void arr(const char* key, const Tensor& t, bool comma = true) { arr(key, t.data(), t.size(), comma); }
void shape(const char* key, const Shape& s) {
    std::fprintf(out, "\"%s\": [", key);
    for (std::size_t i = 0; i < s.size(); ++i) std::fprintf(out, "%s%lld", i ? ", " : "", (long long)s[i]);
    std::fprintf(out, "], ");
}
void begin(const char* family) {
    std::fprintf(out, "%s\n{\"family\": \"%s\", ", first_case ? "" : ",", family);
    first_case = false;
}
void end() { std::fprintf(out, "\"_\": 0}"); }

Tensor rnd(Shape s, GaussianStream& g) {
    Tensor t(std::move(s));
    for (Index i = 0; i < t.size(); ++i) t[i] = g.next();
    return t;
}

Index draw(GaussianStream& g, Index lo, Index hi) {
    return lo + static_cast<Index>(g.rng.next_below(static_cast<std::uint64_t>(hi - lo + 1)));
}

void emit_ln(const char* fam, const LayerNormLayer& ln, const Tensor& x, const Tensor& g) {
    auto fwd = layernorm_forward(ln, x);
    auto res = layernorm_backward_simultaneous(ln, fwd.cache, g);
    begin(fam);
    shape("shape", x.shape());
    std::fprintf(out, "\"eps\": %.17g, ", ln.epsilon);
    arr("gamma", ln.gamma);
    arr("beta", ln.beta);
    arr("x", x);
    arr("g", g);
    arr("y", fwd.output);
    arr("xhat", fwd.cache.normalized);
    arr("inv_std", fwd.cache.inv_std);
    arr("dx", res.input_grad);
    arr("dgamma", res.grads.weight_grads.at("gamma"));
    arr("dbeta", res.grads.weight_grads.at("beta"));
    arr("raw_gamma", res.grads.per_example_sqnorms_raw.at("gamma"));
    arr("raw_beta", res.grads.per_example_sqnorms_raw.at("beta"));
    double corr[2] = {res.grads.per_example_sqnorms.at("gamma"), res.grads.per_example_sqnorms.at("beta")};
    arr("corrected", corr, 2);
    end();
}

void emit_ln_cache(const char* fam, const LayerNormLayer& ln, const LayerNormCache& c, const Tensor& g) {
    auto res = layernorm_backward_simultaneous(ln, c, g);
    begin(fam);
    shape("shape", g.shape());
    arr("gamma", ln.gamma);
    arr("xhat", c.normalized);
    arr("inv_std", c.inv_std);
    arr("g", g);
    arr("dx", res.input_grad);
    arr("dgamma", res.grads.weight_grads.at("gamma"));
    arr("dbeta", res.grads.weight_grads.at("beta"));
    arr("raw_gamma", res.grads.per_example_sqnorms_raw.at("gamma"));
    arr("raw_beta", res.grads.per_example_sqnorms_raw.at("beta"));
    double corr[2] = {res.grads.per_example_sqnorms.at("gamma"), res.grads.per_example_sqnorms.at("beta")};
    arr("corrected", corr, 2);
    end();
}

void emit_linear(const char* fam, const LinearLayer& layer, const Tensor& x, const Tensor& g, bool with_frob) {
    auto res = linear_backward_simultaneous(layer, x, g);
    begin(fam);
    shape("shape_x", x.shape());
    shape("shape_g", g.shape());
    arr("W", layer.weight);
    if (layer.bias) arr("bias", *layer.bias);
    arr("x", x);
    arr("g", g);
    arr("dW", res.grads.weight_grads.at("weight"));
    arr("raw_w", res.grads.per_example_sqnorms_raw.at("weight"));
    double corr[2] = {res.grads.per_example_sqnorms.at("weight"), 0.0};
    if (layer.bias) {
        arr("dbias", res.grads.weight_grads.at("bias"));
        arr("raw_b", res.grads.per_example_sqnorms_raw.at("bias"));
        corr[1] = res.grads.per_example_sqnorms.at("bias");
    }
    arr("corrected", corr, 2);
    arr("dx", res.input_grad);
    if (with_frob && x.rank() == 3) arr("frob", linear_perexample_sqnorm_frobenius(x, g));
    end();
}

void ln_cfg1() {
    const Index B = 8, T = 128, D = 768;
    std::vector<float> xf(B * T * D), gf(B * T * D), gam(D), bet(D);
    orc_synth_ln(xf.data(), gf.data(), gam.data(), bet.data(), B, T, D, 0, B, 0.3f, 0, 0);
    Tensor x({B, T, D}), g({B, T, D}), gamma({D}), beta({D});
    for (Index i = 0; i < x.size(); ++i) {
        x[i] = xf[static_cast<std::size_t>(i)];
        g[i] = gf[static_cast<std::size_t>(i)];
    }
    for (Index i = 0; i < D; ++i) {
        gamma[i] = gam[static_cast<std::size_t>(i)];
        beta[i] = bet[static_cast<std::size_t>(i)];
    }
    LayerNormLayer ln{gamma, beta, 1e-5};
    auto fwd = layernorm_forward(ln, x);
    auto res = layernorm_backward_simultaneous(ln, fwd.cache, g);
    begin("ln_cfg1");
    shape("shape", x.shape());
    std::fprintf(out, "\"sigma\": 0.3, \"stream0\": 0, ");
    arr("dgamma", res.grads.weight_grads.at("gamma"));
    arr("dbeta", res.grads.weight_grads.at("beta"));
    arr("raw_gamma", res.grads.per_example_sqnorms_raw.at("gamma"));
    arr("raw_beta", res.grads.per_example_sqnorms_raw.at("beta"));
    double corr[2] = {res.grads.per_example_sqnorms.at("gamma"), res.grads.per_example_sqnorms.at("beta")};
    arr("corrected", corr, 2);
    // dx summary: per-row sum and sum of squares + every 997th element
    const Tensor& dx = res.input_grad;
    std::vector<double> rs(B * T), rq(B * T), samp, sidx;
    for (Index r = 0; r < B * T; ++r) {
        double s = 0, q = 0;
        for (Index d = 0; d < D; ++d) {
            s += dx[r * D + d];
            q += dx[r * D + d] * dx[r * D + d];
        }
        rs[static_cast<std::size_t>(r)] = s;
        rq[static_cast<std::size_t>(r)] = q;
    }
    for (Index i = 0; i < dx.size(); i += 997) {
        samp.push_back(dx[i]);
        sidx.push_back(static_cast<double>(i));
    }
    arr("dx_row_sum", rs.data(), B * T);
    arr("dx_row_sqsum", rq.data(), B * T);
    arr("dx_sample_idx", sidx.data(), static_cast<Index>(sidx.size()));
    arr("dx_sample", samp.data(), static_cast<Index>(samp.size()));
    arr("inv_std", fwd.cache.inv_std);
    // a few y values for the forward check
    std::vector<double> ys;
    for (Index i = 0; i < dx.size(); i += 997) ys.push_back(fwd.output[i]);
    arr("y_sample", ys.data(), static_cast<Index>(ys.size()));
    end();
}

}  // namespace

void emit_emb(const char* fam, const EmbeddingLayer& layer, const std::vector<std::int32_t>& ids, Index b, Index t,
              const Tensor& g) {
    auto res = embedding_backward_simultaneous(layer, ids, b, t, g);
    begin(fam);
    std::fprintf(out, "\"B\": %lld, \"T\": %lld, \"V\": %lld, \"D\": %lld, ", (long long)b, (long long)t,
                 (long long)layer.vocab(), (long long)layer.dim());
    std::vector<double> idd(ids.begin(), ids.end());
    arr("ids", idd.data(), (Index)idd.size());
    arr("g", g);
    arr("dW", res.weight_grads.at("weight"));
    arr("raw_w", res.per_example_sqnorms_raw.at("weight"));
    double corr[1] = {res.per_example_sqnorms.at("weight")};
    arr("corrected", corr, 1);
    end();
}

int main(int argc, char** argv) {
    out = argc > 1 ? std::fopen(argv[1], "w") : stdout;
    std::fprintf(out, "[");

    {  // test_layers.cpp:167-176
        LayerNormLayer ln{Tensor({2}, {1, 1}), Tensor({2}, {0, 0}), 1e-5};
        LayerNormCache cache{Tensor({1, 1, 2}, {1, -1}), Tensor({1, 1}, {1.0})};
        emit_ln_cache("ln_kat", ln, cache, Tensor({1, 1, 2}, {2, 3}));
    }
    {  // test_layers.cpp:151-165
        LayerNormLayer a{Tensor({2}, {1, 1}), Tensor({2}, {0, 0}), 1e-12};
        LayerNormLayer b{Tensor({2}, {1, 1}), Tensor({2}, {0.5, -0.5}), 1e-5};
        emit_ln("ln_fwd_kat", a, Tensor({1, 1, 2}, {1, -1}), Tensor({1, 1, 2}, {0, 0}));
        emit_ln("ln_fwd_kat", b, Tensor({1, 1, 2}, {3, 3}), Tensor({1, 1, 2}, {0, 0}));
        emit_ln("ln_fwd_kat", a, Tensor({1, 1, 2}, {0, 2}), Tensor({1, 1, 2}, {0, 0}));
    }
    {  // test_layers.cpp:178-188
        GaussianStream rng(29);
        LayerNormLayer ln{rnd({4}, rng), rnd({4}, rng), 1e-5};
        Tensor x = rnd({2, 3, 4}, rng);
        emit_ln("ln_zero", ln, x, Tensor({2, 3, 4}));
    }
    {  // test_layers.cpp:190-212
        GaussianStream rng(31);
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = draw(rng, 2, 4), t = draw(rng, 1, 5), k = draw(rng, 2, 6);
            LayerNormLayer ln{rnd({k}, rng), rnd({k}, rng), 1e-5};
            Tensor x = rnd({b, t, k}, rng);
            // the reference test draws g after the forward; the forward draws nothing
            Tensor g = rnd({b, t, k}, rng);
            emit_ln("ln_rand31", ln, x, g);
        }
    }
    {  // acceptance.cpp:48-104 (linear part, then LN part; embedding part not on the path)
        GaussianStream rng(1001);
        for (int rep = 0; rep < 100; ++rep) {
            const Index b = draw(rng, 1, 4), t = draw(rng, 1, 5), k = draw(rng, 1, 6), l = draw(rng, 1, 6);
            LinearLayer layer{rnd({k, l}, rng), rnd({l}, rng)};
            Tensor x = rnd({b, t, k}, rng);
            Tensor g = rnd({b, t, l}, rng);
            emit_linear("acc1_linear", layer, x, g, true);
        }
        for (int rep = 0; rep < 100; ++rep) {
            const Index b = draw(rng, 1, 4), t = draw(rng, 1, 5), k = draw(rng, 2, 6);
            LayerNormLayer ln{rnd({k}, rng), rnd({k}, rng), 1e-5};
            Tensor x = rnd({b, t, k}, rng);
            Tensor g = rnd({b, t, k}, rng);
            emit_ln("acc1_ln", ln, x, g);
        }
    }
    {  // acceptance.cpp:109-126
        GaussianStream rng(1002);
        for (int rep = 0; rep < 100; ++rep) {
            const Index b = draw(rng, 1, 4), t = draw(rng, 1, 5), k = draw(rng, 1, 6), l = draw(rng, 1, 6);
            LinearLayer layer{rnd({k, l}, rng), std::nullopt};
            Tensor x = rnd({b, t, k}, rng);
            Tensor g = rnd({b, t, l}, rng);
            emit_linear("acc2_frob", layer, x, g, true);
        }
    }
    {  // test_layers.cpp:51-63, 77-85
        emit_linear("lin_kat", LinearLayer{Tensor({2, 1}, {0, 0}), std::nullopt}, Tensor({2, 1, 2}, {1, 2, 3, 4}),
                    Tensor({2, 1, 1}, {1, 2}), true);
        emit_linear("lin_kat", LinearLayer{Tensor({1, 1}, {0}), std::nullopt}, Tensor({1, 2, 1}, {1, 1}),
                    Tensor({1, 2, 1}, {2, 3}), true);
    }
    {  // test_layers.cpp:87-107 (with bias)
        GaussianStream rng(17);
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = draw(rng, 2, 4), t = draw(rng, 1, 5), k = draw(rng, 1, 6), l = draw(rng, 1, 6);
            LinearLayer layer{rnd({k, l}, rng), rnd({l}, rng)};
            Tensor x = rnd({b, t, k}, rng);
            Tensor g = rnd({b, t, l}, rng);
            emit_linear("lin_rand17", layer, x, g, true);
        }
    }
    {  // test_layers.cpp:135-149 (no bias)
        GaussianStream rng(23);
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = draw(rng, 1, 4), t = draw(rng, 1, 5), k = draw(rng, 1, 6), l = draw(rng, 1, 6);
            LinearLayer layer{rnd({k, l}, rng), std::nullopt};
            Tensor x = rnd({b, t, k}, rng);
            Tensor g = rnd({b, t, l}, rng);
            emit_linear("frob_rand23", layer, x, g, true);
        }
    }
    {  // test_layers.cpp:300-319 (embedding worked examples)
        EmbeddingLayer layer{Tensor({3, 1})};
        emit_emb("emb_kat", layer, {0, 0}, 1, 2, Tensor({1, 2, 1}, {1, 2}));
        emit_emb("emb_kat", layer, {0, 1}, 1, 2, Tensor({1, 2, 1}, {1, 2}));
        emit_emb("emb_kat", layer, {0, 1}, 1, 2, Tensor({1, 2, 1}));
    }
    {  // test_layers.cpp:321-347 (seed 43, 25 reps)
        GaussianStream rng(43);
        for (int rep = 0; rep < 25; ++rep) {
            const Index b = draw(rng, 1, 4), t = draw(rng, 1, 5), v = draw(rng, 2, 8), d = draw(rng, 1, 6);
            EmbeddingLayer layer{rnd({v, d}, rng)};
            std::vector<std::int32_t> ids(static_cast<std::size_t>(b * t));
            for (auto& id : ids) id = static_cast<std::int32_t>(rng.rng.next_below(static_cast<std::uint64_t>(v)));
            Tensor g = rnd({b, t, d}, rng);
            emit_emb("emb_rand43", layer, ids, b, t, g);
        }
    }
    {  // a handful of Gaussian draws to pin the RNG restatement
        GaussianStream gs(1234);
        std::vector<double> v(64);
        for (auto& e : v) e = gs.next();
        begin("rng");
        std::fprintf(out, "\"seed\": 1234, ");
        arr("draws", v.data(), 64);
        end();
    }
    ln_cfg1();
    std::fprintf(out, "\n]\n");
    if (out != stdout) std::fclose(out);
    return 0;
}

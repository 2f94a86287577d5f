// gnstk_dropin.cu — host implementation of the gnstk drop-in API
// (include/gnstk/*.hpp) over the C ABI of include/gnsb.h.
//
// Value semantics like the reference: fp64 host Tensors in, fp64 host Tensors
// out.  Each call uploads its operands, runs the B200 kernels on the current
// device (legacy default stream), and downloads the results; argument
// validation happens first, in the reference's order and wording
// (proj/src/layers.cpp:13-35, gns.cpp:10-18), so error behaviour is identical.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnsb.h"
#include "gnstk/costmodel.hpp"
#include "gnstk/gns.hpp"
#include "gnstk/layers.hpp"
#include "gnstk/tensor.hpp"

namespace gnstk {

// ------------------------------------------------------- device plumbing --
namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument("layers: " + msg); }

void check(gnsb_status s) {
    if (s == GNSB_OK) return;
    if (s == GNSB_EINVAL) throw std::invalid_argument(gnsb_last_error());
    throw std::runtime_error(gnsb_last_error());
}
void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

// Device buffers come from the stream-ordered pool of the legacy default
// stream (cudaMallocAsync), which every drop-in call runs on: a call costs
// no cudaMalloc / cudaFree round trips once the pool is warm (the reference's
// callers make many small calls per training step).
void init_pool_once() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;  // keep freed blocks for reuse
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes, bool zero = false) {
        if (bytes) {
            init_pool_once();
            cuda_check(cudaMallocAsync(&p, bytes, nullptr), "cudaMallocAsync");
            if (zero) cuda_check(cudaMemsetAsync(p, 0, bytes, nullptr), "cudaMemsetAsync");
        }
    }
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, nullptr);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

DevBuf upload(const Tensor& t) {
    DevBuf d(sizeof(double) * static_cast<std::size_t>(t.size()));
    if (t.size()) cuda_check(cudaMemcpy(d.p, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice), "upload");
    return d;
}
void download(Tensor& t, const DevBuf& d) {
    if (t.size()) cuda_check(cudaMemcpy(t.data(), d.p, sizeof(double) * t.size(), cudaMemcpyDeviceToHost), "download");
}
void download(double* dst, const DevBuf& d, std::size_t n) {
    if (n) cuda_check(cudaMemcpy(dst, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost), "download");
}

// (B, M, K) view of a rank >= 2 tensor (layers.cpp:19-28)
struct Bmk {
    Index b, m, k;
};
Bmk bmk_view(const Tensor& t) {
    if (t.rank() < 2) fail("expected rank >= 2");
    Index m = 1;
    for (Index d = 1; d + 1 < t.rank(); ++d) m *= t.shape()[static_cast<std::size_t>(d)];
    return {t.shape().front(), m, t.shape().back()};
}
void check_same_leading(const Tensor& x, const Tensor& g) {
    if (x.rank() != g.rank()) fail("x and g rank mismatch");
    for (Index d = 0; d + 1 < x.rank(); ++d)
        if (x.shape()[static_cast<std::size_t>(d)] != g.shape()[static_cast<std::size_t>(d)])
            fail("x and g leading shape mismatch");
}
double corrected(double sum_sq, Index batch) {  // layers.cpp:39-42
    const double b = static_cast<double>(batch);
    return sum_sq / b * (b * b);
}

}  // namespace

// ----------------------------------------------------------------- layers --
LayerNormForwardResult layernorm_forward(const LayerNormLayer& layer, const Tensor& x) {
    const Index k = layer.gamma.shape().empty() ? 0 : layer.gamma.shape()[0];
    if (layer.beta.shape() != Shape{k}) fail("gamma/beta extent mismatch");
    if (layer.epsilon <= 0.0) fail("epsilon must be positive");
    if (x.rank() < 1 || x.shape().back() != k) fail("input trailing extent does not match gamma");
    if (k < 2) fail("layernorm needs trailing extent >= 2");
    Index rows = 1;
    for (Index d = 0; d + 1 < x.rank(); ++d) rows *= x.shape()[static_cast<std::size_t>(d)];

    LayerNormForwardResult res;
    res.output = Tensor(x.shape());
    res.cache.normalized = Tensor(x.shape());
    res.cache.inv_std = Tensor(Shape(x.shape().begin(), x.shape().end() - 1));
    if (rows == 0) return res;
    DevBuf dx = upload(x), dg = upload(layer.gamma), db = upload(layer.beta);
    DevBuf dy(sizeof(double) * x.size()), dxh(sizeof(double) * x.size()), dr(sizeof(double) * rows);
    check(gnsb_ln_fwd(dx.p, dg.p, db.p, dy.p, nullptr, dr.p, dxh.p, rows, k, layer.epsilon, GNSB_F64, nullptr));
    download(res.output, dy);
    download(res.cache.normalized, dxh);
    download(res.cache.inv_std, dr);
    return res;
}

LayerNormBackwardResult layernorm_backward_simultaneous(const LayerNormLayer& layer, const LayerNormCache& cache,
                                                        const Tensor& g) {
    const Index k = layer.gamma.shape().empty() ? 0 : layer.gamma.shape()[0];
    if (!cache.normalized.same_shape(g)) fail("cache/gradient shape mismatch");
    if (g.rank() < 2) fail("backward expects a leading batch axis");
    const Bmk v = bmk_view(g);
    if (v.k != k) fail("gradient trailing extent does not match gamma");
    if (v.b == 0) fail("empty batch");

    LayerNormBackwardResult res;
    res.grads.batch_size = v.b;
    Tensor dgamma({k}), dbeta({k}), rg({v.b}), rb({v.b});
    res.input_grad = Tensor(g.shape());
    double sums[4] = {0, 0, 0, 0};
    DevBuf dxh = upload(cache.normalized), dinv = upload(cache.inv_std), dgr = upload(g), dgam = upload(layer.gamma);
    DevBuf ddx(sizeof(double) * g.size()), ddg(sizeof(double) * k), ddb(sizeof(double) * k);
    DevBuf drg(sizeof(double) * v.b), drb(sizeof(double) * v.b), dsums(sizeof(double) * 4, true);
    std::size_t wsb = 0;
    check(gnsb_ln_bwd_workspace_size(v.b, v.m, k, GNSB_F64, &wsb));
    DevBuf ws(wsb, true);
    check(gnsb_ln_bwd(dxh.p, nullptr, dinv.p, dgr.p, dgam.p, ddx.p, ddg.p, ddb.p, drg.as<double>(), drb.as<double>(),
                      dsums.as<double>(), 1, v.b, v.m, k, GNSB_F64, ws.p, wsb, nullptr));
    download(res.input_grad, ddx);
    download(dgamma, ddg);
    download(dbeta, ddb);
    download(rg, drg);
    download(rb, drb);
    download(sums, dsums, 4);
    res.grads.weight_grads["gamma"] = std::move(dgamma);
    res.grads.weight_grads["beta"] = std::move(dbeta);
    res.grads.per_example_sqnorms["gamma"] = corrected(sums[0], v.b);
    res.grads.per_example_sqnorms["beta"] = corrected(sums[1], v.b);
    res.grads.per_example_sqnorms_raw["gamma"] = std::move(rg);
    res.grads.per_example_sqnorms_raw["beta"] = std::move(rb);
    return res;
}

LinearBackwardResult linear_backward_simultaneous(const LinearLayer& layer, const Tensor& x, const Tensor& g) {
    const Index k = layer.weight.rank() == 2 ? layer.weight.shape()[0] : 0;
    const Index l = layer.weight.rank() == 2 ? layer.weight.shape()[1] : 0;
    check_same_leading(x, g);
    const Bmk vx = bmk_view(x), vg = bmk_view(g);
    if (vx.k != k) fail("input trailing extent does not match weight rows");
    if (vg.k != l) fail("gradient trailing extent does not match weight columns");
    if (vx.b == 0) fail("empty batch");

    LinearBackwardResult res;
    res.grads.batch_size = vx.b;
    Tensor dW({k, l}), rw({vx.b});
    double sums[4] = {0, 0, 0, 0};
    DevBuf dx = upload(x), dg = upload(g), dWt = upload(layer.weight);
    DevBuf ddW(sizeof(double) * k * l), drw(sizeof(double) * vx.b), dsums(sizeof(double) * 4, true);
    std::size_t wsb = 0, wsb2 = 0;
    check(gnsb_linear_pe_workspace_size(vx.b, vx.m, k, l, GNSB_F64, &wsb));
    check(gnsb_linear_pe_workspace_size(vx.b, vx.m, 1, l, GNSB_F64, &wsb2));
    DevBuf ws(wsb > wsb2 ? wsb : wsb2, true);
    check(gnsb_linear_pe_norms(dx.p, dg.p, ddW.p, drw.as<double>(), dsums.as<double>(), vx.b, vx.m, k, l, 1, GNSB_F64,
                               ws.p, wsb > wsb2 ? wsb : wsb2, nullptr));
    download(dW, ddW);
    download(rw, drw);
    if (layer.bias) {
        if (layer.bias->shape() != Shape{l}) fail("bias extent does not match weight columns");
        Tensor db({l}), rb({vx.b});
        DevBuf ddb(sizeof(double) * l), drb(sizeof(double) * vx.b);
        check(gnsb_linear_bias_pe(dg.p, ddb.p, drb.as<double>(), dsums.as<double>(), vx.b, vx.m, l, GNSB_F64, ws.p,
                                  wsb > wsb2 ? wsb : wsb2, nullptr));
        download(db, ddb);
        download(rb, drb);
        res.grads.weight_grads["bias"] = std::move(db);
        res.grads.per_example_sqnorms_raw["bias"] = std::move(rb);
    }
    download(sums, dsums, 4);
    res.grads.weight_grads["weight"] = std::move(dW);
    res.grads.per_example_sqnorms["weight"] = corrected(sums[0], vx.b);
    res.grads.per_example_sqnorms_raw["weight"] = std::move(rw);
    if (layer.bias) res.grads.per_example_sqnorms["bias"] = corrected(sums[1], vx.b);
    res.input_grad = Tensor(x.shape());
    DevBuf ddx(sizeof(double) * x.size());
    check(gnsb_linear_dx(dg.p, dWt.p, ddx.p, vx.b * vx.m, k, l, GNSB_F64, GNSB_F64, nullptr, 0, nullptr));
    download(res.input_grad, ddx);
    return res;
}

Tensor linear_forward(const LinearLayer& layer, const Tensor& x) {
    const Index k = layer.weight.rank() == 2 ? layer.weight.shape()[0] : 0;
    const Index l = layer.weight.rank() == 2 ? layer.weight.shape()[1] : 0;
    const Bmk v = bmk_view(x);  // layers.cpp:55-57, in the reference's order
    if (v.k != k) fail("input trailing extent does not match weight rows");
    if (layer.bias && layer.bias->shape() != Shape{l}) fail("bias extent does not match weight columns");
    Shape os = x.shape();
    os.back() = l;
    Tensor y(os);
    const Index rows = v.b * v.m;
    if (rows == 0 || l == 0) return y;
    DevBuf dx = upload(x), dw = upload(layer.weight), dy(sizeof(double) * y.size());
    DevBuf db = layer.bias ? upload(*layer.bias) : DevBuf(0);
    check(gnsb_linear_fwd(dx.p, dw.p, db.p, dy.p, rows, k, l, GNSB_F64, GNSB_F64, nullptr, 0, nullptr));
    download(y, dy);
    return y;
}

Tensor linear_perexample_sqnorm_frobenius(const Tensor& x, const Tensor& g) {
    if (x.rank() != 3 || g.rank() != 3) fail("frobenius path expects strictly 3-axis inputs");
    if (x.shape()[0] != g.shape()[0] || x.shape()[1] != g.shape()[1]) fail("x and g leading shape mismatch");
    const Index b = x.shape()[0], t = x.shape()[1], k = x.shape()[2], l = g.shape()[2];
    Tensor out({b});
    if (b == 0) return out;
    if (k == 0 || l == 0 || t == 0) return out;  // empty contractions: zero norms
    DevBuf dx = upload(x), dg = upload(g), dout(sizeof(double) * b);
    std::size_t wsb = 0;
    check(gnsb_linear_pe_workspace_size(b, t, k, l, GNSB_F64, &wsb));
    DevBuf ws(wsb, true);
    check(gnsb_linear_pe_norms(dx.p, dg.p, nullptr, dout.as<double>(), nullptr, b, t, k, l, 2, GNSB_F64, ws.p, wsb,
                               nullptr));
    download(out, dout);
    return out;
}

// -------------------------------------------------------------- embedding --
Tensor embedding_forward(const EmbeddingLayer& layer, std::span<const std::int32_t> ids, Index batch, Index t_len) {
    const Index v = layer.vocab(), d = layer.dim();
    if (static_cast<Index>(ids.size()) != batch * t_len) fail("id count does not match batch * t_len");
    for (std::int32_t id : ids)  // layers.cpp:307; the host ids are checked before any device work
        if (id < 0 || id >= v) fail("id out of range");
    Tensor out({batch, t_len, d});
    if (out.size() == 0) return out;
    DevBuf dw = upload(layer.weight), dids(sizeof(std::int32_t) * ids.size()), dout(sizeof(double) * out.size());
    cuda_check(cudaMemcpy(dids.p, ids.data(), sizeof(std::int32_t) * ids.size(), cudaMemcpyHostToDevice), "upload");
    check(gnsb_embedding_fwd(static_cast<const std::int32_t*>(dids.p), dw.p, dout.p, batch * t_len, v, d, GNSB_F64,
                             nullptr, nullptr));
    download(out, dout);
    return out;
}

LayerGradOutput embedding_backward_simultaneous(const EmbeddingLayer& layer, std::span<const std::int32_t> ids,
                                                Index batch, Index t_len, const Tensor& g) {
    const Index v = layer.vocab();
    const Index d = layer.dim();
    // layers.cpp:318-322, in the reference's order; ids are host data here
    if (static_cast<Index>(ids.size()) != batch * t_len) fail("id count does not match batch * t_len");
    if (g.shape() != Shape{batch, t_len, d}) fail("gradient shape mismatch");
    if (batch == 0) fail("empty batch");
    for (std::int32_t id : ids)
        if (id < 0 || id >= v) fail("id out of range");
    LayerGradOutput out;
    out.batch_size = batch;
    Tensor wgrad({v, d}), raw({batch});
    double sums[4] = {0, 0, 0, 0};
    DevBuf dg = upload(g), dids(sizeof(std::int32_t) * (ids.size() ? ids.size() : 1));
    if (!ids.empty())
        cuda_check(cudaMemcpy(dids.p, ids.data(), sizeof(std::int32_t) * ids.size(), cudaMemcpyHostToDevice), "upload");
    DevBuf dW(sizeof(double) * v * d), draw(sizeof(double) * batch), dsums(sizeof(double) * 4, true);
    std::size_t wsb = 0;
    check(gnsb_embedding_pe_workspace_size(batch, t_len, v, d, GNSB_F64, &wsb));
    DevBuf ws(wsb, true);
    check(gnsb_embedding_pe(static_cast<const std::int32_t*>(dids.p), dg.p, dW.p, draw.as<double>(),
                            dsums.as<double>(), batch, t_len, v, d, GNSB_F64, ws.p, wsb, nullptr, nullptr));
    download(wgrad, dW);
    download(raw, draw);
    download(sums, dsums, 4);
    // the reference sums the per-example values in example order (layers.cpp:360-366)
    double sum_sq = 0.0;
    for (Index b = 0; b < batch; ++b) sum_sq += raw[b];
    out.weight_grads["weight"] = std::move(wgrad);
    out.per_example_sqnorms["weight"] = corrected(sum_sq, batch);
    out.per_example_sqnorms_raw["weight"] = std::move(raw);
    return out;
}

// -------------------------------------------------------------------- gns --
namespace {
gnsb_grad_stats to_c(const GradStats& s) {
    return gnsb_grad_stats{s.g_big_sqnorm, s.g_small_sqnorm_mean, s.b_big, s.b_small, s.n_small};
}
}  // namespace

std::string layer_type_name(LayerType t) {
    switch (t) {
        case LayerType::Embedding: return "embedding";
        case LayerType::Linear: return "linear";
        case LayerType::LayerNorm: return "layernorm";
    }
    throw std::invalid_argument("gns: unknown layer type");
}

double estimate_g2(const GradStats& stats) {
    const gnsb_grad_stats c = to_c(stats);
    double out = 0.0;
    check(gnsb_estimate_g2(&c, &out));
    return out;
}

double estimate_s(const GradStats& stats) {
    const gnsb_grad_stats c = to_c(stats);
    double out = 0.0;
    check(gnsb_estimate_s(&c, &out));
    return out;
}

GnsEstimate make_gns_estimate(double g2, double s) {
    gnsb_gns_estimate e;
    gnsb_make_gns_estimate(g2, s, &e);
    return GnsEstimate{e.g2, e.s, e.b_simple, e.b_simple_defined != 0};
}

EmaState ema_update(EmaState state, double x) {
    gnsb_ema_state c{state.alpha, state.value, state.count};
    check(gnsb_ema_update(&c, x));
    return EmaState{c.alpha, c.value, c.count};
}

GnsEstimate smoothed_gns(const EmaState& g2_ema, const EmaState& s_ema) {
    const gnsb_ema_state a{g2_ema.alpha, g2_ema.value, g2_ema.count}, b{s_ema.alpha, s_ema.value, s_ema.count};
    gnsb_gns_estimate e;
    check(gnsb_smoothed_gns(&a, &b, &e));
    return GnsEstimate{e.g2, e.s, e.b_simple, e.b_simple_defined != 0};
}

GradStats aggregate(const std::map<LayerKey, GradStats>& stats_by_layer, std::optional<LayerType> group) {
    std::vector<gnsb_grad_stats> st;
    std::vector<int32_t> ty;
    for (const auto& [key, s] : stats_by_layer) {  // std::map: LayerKey order, like the reference
        st.push_back(to_c(s));
        ty.push_back(static_cast<int32_t>(key.type));
    }
    gnsb_grad_stats out{};
    check(gnsb_aggregate(st.data(), ty.data(), static_cast<int32_t>(st.size()),
                         group ? static_cast<int32_t>(*group) : -1, &out));
    return GradStats{out.g_big_sqnorm, out.g_small_sqnorm_mean, out.b_big, out.b_small, out.n_small};
}

// Offline statistics over logged GNS series (proj/src/gns.cpp:91-196).  Host
// code: O(steps) scalars, consumed by the reference's simulator and CLI.
JackknifeResult jackknife_ratio_stderr(std::span<const std::pair<double, double>> pairs) {
    auto bad = [](const char* m) { throw std::invalid_argument(std::string("gns: ") + m); };
    const std::size_t n = pairs.size();
    if (n < 2) bad("jackknife needs at least 2 pairs");
    double ts = 0.0, tg = 0.0;
    for (const auto& p : pairs) {
        ts += p.first;
        tg += p.second;
    }
    if (tg == 0.0) bad("jackknife ratio denominator is zero");
    const double nd = static_cast<double>(n);
    JackknifeResult r;
    r.ratio = (ts / nd) / (tg / nd);
    // leave-one-out ratios, then their spread about their mean
    std::vector<double> loo;
    loo.reserve(n);
    double mean = 0.0;
    for (const auto& p : pairs) {
        if (tg - p.second == 0.0) bad("jackknife leave-one-out denominator is zero");
        loo.push_back((ts - p.first) / (tg - p.second));
        mean += loo.back();
    }
    mean /= nd;
    double ss = 0.0;
    for (double v : loo) ss += (v - mean) * (v - mean);
    r.std_error = std::sqrt((nd - 1.0) / nd * ss);
    return r;
}

namespace {
// EMA-smoothed B_simple per step under one alpha; nullopt where undefined
std::vector<std::optional<double>> smoothed_ratios(const GnsSeries& s, double alpha) {
    std::vector<std::optional<double>> out(s.g2.size());
    EmaState eg{alpha}, es{alpha};
    for (std::size_t i = 0; i < s.g2.size(); ++i) {
        eg = ema_update(eg, s.g2[i]);
        es = ema_update(es, s.s[i]);
        const GnsEstimate e = smoothed_gns(eg, es);
        if (e.b_simple_defined) out[i] = e.b_simple;
    }
    return out;
}
}  // namespace

std::vector<RegressionRow> regress_layer_gns(const GnsSeries& total, const std::map<LayerType, GnsSeries>& per_type,
                                             std::span<const double> alphas) {
    auto bad = [](const char* m) { throw std::invalid_argument(std::string("gns: ") + m); };
    if (total.g2.size() != total.s.size()) bad("total series components misaligned");
    std::vector<RegressionRow> rows;
    for (const auto& [type, ser] : per_type) {
        if (ser.g2.size() != total.g2.size() || ser.s.size() != total.s.size())
            bad("per-type series not aligned with total");
        for (double alpha : alphas) {
            const auto ys = smoothed_ratios(total, alpha), xs = smoothed_ratios(ser, alpha);
            std::vector<double> x, y;  // pairwise-complete steps
            for (std::size_t i = 0; i < xs.size(); ++i)
                if (xs[i] && ys[i]) {
                    x.push_back(*xs[i]);
                    y.push_back(*ys[i]);
                }
            if (x.size() < 3) bad("fewer than 3 aligned points for regression");
            const double nd = static_cast<double>(x.size());
            double mx = 0.0, my = 0.0;
            for (std::size_t i = 0; i < x.size(); ++i) {
                mx += x[i];
                my += y[i];
            }
            mx /= nd;
            my /= nd;
            double sxx = 0.0, syy = 0.0, sxy = 0.0;
            for (std::size_t i = 0; i < x.size(); ++i) {
                const double dx = x[i] - mx, dy = y[i] - my;
                sxx += dx * dx;
                syy += dy * dy;
                sxy += dx * dy;
            }
            RegressionRow row{type, alpha};
            if (sxx > 0.0) {
                row.slope = sxy / sxx;
                row.slope_defined = true;
                if (syy > 0.0) {
                    row.pearson_r = sxy / std::sqrt(sxx * syy);
                    row.r_defined = true;
                }
            }
            rows.push_back(row);
        }
    }
    return rows;
}

// -------------------------------------------------------------- costmodel --
std::string cost_method_name(CostMethod m) { return m == CostMethod::Simultaneous ? "simultaneous" : "frobenius"; }

CostPair flops(const CostShape& s, CostMethod m) {
    int64_t out[2];
    check(gnsb_flops(s.b, s.t, s.k, s.l, m == CostMethod::Simultaneous ? 0 : 1, out));
    return CostPair{out[0], out[1]};
}

CostPair io_values(const CostShape& s, CostMethod m) {
    int64_t out[2];
    check(gnsb_io_values(s.b, s.t, s.k, s.l, m == CostMethod::Simultaneous ? 0 : 1, out));
    return CostPair{out[0], out[1]};
}

CostPair io_bytes(const CostShape& s, CostMethod m) {
    const CostPair v = io_values(s, m);  // extents are checked first, as in the reference
    if (s.bytes_per_value < 1) throw std::invalid_argument("costmodel: bytes_per_value must be positive");
    return CostPair{v.weight_grad * s.bytes_per_value, v.grad_norms * s.bytes_per_value};
}

double crossover_t(std::int64_t k, std::int64_t l, CostCriterion c) {
    double out = 0.0;
    check(gnsb_crossover_t(k, l, c == CostCriterion::IO ? 0 : 1, &out));
    return out;
}

std::vector<SweepRow> sweep(std::span<const CostShape> shapes) {
    if (shapes.empty()) throw std::invalid_argument("costmodel: empty sweep grid");
    std::vector<SweepRow> rows;
    for (const CostShape& s : shapes) {
        const double frob_norms = static_cast<double>(flops(s, CostMethod::Frobenius).grad_norms);
        for (CostMethod m : {CostMethod::Simultaneous, CostMethod::Frobenius}) {
            const CostPair f = flops(s, m), io = io_values(s, m);
            rows.push_back(SweepRow{m, s.b, s.t, s.k, s.l, f.weight_grad, f.grad_norms, io.weight_grad, io.grad_norms,
                                    static_cast<double>(f.grad_norms) / frob_norms});
        }
    }
    return rows;
}

std::int64_t layernorm_norms_io_values(const CostShape& s) {
    io_values(s, CostMethod::Simultaneous);  // the reference's shape check
    if (s.bytes_per_value < 1) throw std::invalid_argument("costmodel: bytes_per_value must be positive");
    return s.b * s.k + s.b;
}

}  // namespace gnstk

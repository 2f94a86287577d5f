// ref_capi.cpp — extern "C" shim over the UNMODIFIED reference library
// (proj/src/{tensor,layers,gns,costmodel}.cpp compiled in place from
// /root/reference by oracle/Makefile into oracle/_ref/libgnstk_ref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Used (a) by tests/golden/make_golden.py
// to produce golden vectors, (b) by tests to pin the oracle restatement, and
// (c) by bench.py as the timed reference CPU arm (`--impl reference` and the
// `cpu_baseline` leg).  Never linked into the product library.
//
// The functions below only marshal plain arrays into gnstk::Tensor, call the
// reference's own public API and copy the results out.
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gnstk/costmodel.hpp"
#include "gnstk/gns.hpp"
#include "gnstk/layers.hpp"
#include "gnstk/rng.hpp"
#include "gnstk/tensor.hpp"

namespace {
thread_local std::string g_err;

gnstk::Tensor make(gnstk::Shape s, const double* p) {
    std::size_t n = 1;
    for (auto e : s) n *= static_cast<std::size_t>(e);
    return gnstk::Tensor(std::move(s), std::vector<double>(p, p + n));
}

void put(const gnstk::Tensor& t, double* dst) {
    if (dst) std::memcpy(dst, t.data(), sizeof(double) * static_cast<std::size_t>(t.size()));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// gnstk::layernorm_forward (proj/src/layers.cpp:189-229)
int ref_layernorm_forward(const double* x, const double* gamma, const double* beta, double eps,
                          int64_t rows, int64_t D, double* y, double* xhat, double* inv_std) {
    return guard([&] {
        gnstk::LayerNormLayer ln{make({D}, gamma), make({D}, beta), eps};
        auto r = gnstk::layernorm_forward(ln, make({rows, D}, x));
        put(r.output, y);
        put(r.cache.normalized, xhat);
        put(r.cache.inv_std, inv_std);
    });
}

// gnstk::layernorm_backward_simultaneous (proj/src/layers.cpp:231-298), (B, M, D) view
int ref_layernorm_backward(const double* xhat, const double* inv_std, const double* g,
                           const double* gamma, int64_t B, int64_t M, int64_t D, double* dx,
                           double* dgamma, double* dbeta, double* raw_gamma, double* raw_beta,
                           double* corrected) {
    return guard([&] {
        gnstk::LayerNormLayer ln{make({D}, gamma), gnstk::Tensor({D}), 1e-5};
        gnstk::LayerNormCache cache{make({B, M, D}, xhat), make({B, M}, inv_std)};
        auto r = gnstk::layernorm_backward_simultaneous(ln, cache, make({B, M, D}, g));
        put(r.input_grad, dx);
        put(r.grads.weight_grads.at("gamma"), dgamma);
        put(r.grads.weight_grads.at("beta"), dbeta);
        put(r.grads.per_example_sqnorms_raw.at("gamma"), raw_gamma);
        put(r.grads.per_example_sqnorms_raw.at("beta"), raw_beta);
        if (corrected) {
            corrected[0] = r.grads.per_example_sqnorms.at("gamma");
            corrected[1] = r.grads.per_example_sqnorms.at("beta");
        }
    });
}

// Multi-threaded driver for the CPU baseline: contiguous example slices, one
// reference call per thread (allowed by SPEC.md:168), slice dgamma/dbeta
// summed in fixed slice order, corrected = B * sum(raw).
int ref_layernorm_backward_threaded(int nthreads, const double* xhat, const double* inv_std,
                                    const double* g, const double* gamma, int64_t B, int64_t M,
                                    int64_t D, double* dx, double* dgamma, double* dbeta,
                                    double* raw_gamma, double* raw_beta, double* corrected) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = static_cast<int>(B);
    std::vector<std::vector<double>> dg(nthreads, std::vector<double>(D)), db(nthreads, std::vector<double>(D));
    std::vector<int> rc(nthreads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) {
        const int64_t b0 = B * t / nthreads, b1 = B * (t + 1) / nthreads;
        pool.emplace_back([&, t, b0, b1] {
            const int64_t off = b0 * M * D;
            rc[t] = ref_layernorm_backward(xhat + off, inv_std + b0 * M, g + off, gamma, b1 - b0, M, D,
                                           dx ? dx + off : nullptr, dg[t].data(), db[t].data(),
                                           raw_gamma ? raw_gamma + b0 : nullptr,
                                           raw_beta ? raw_beta + b0 : nullptr, nullptr);
        });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < nthreads; ++t)
        if (rc[t]) return rc[t];
    for (int64_t i = 0; i < D; ++i) {
        double a = 0.0, c = 0.0;
        for (int t = 0; t < nthreads; ++t) {
            a += dg[t][i];
            c += db[t][i];
        }
        if (dgamma) dgamma[i] = a;
        if (dbeta) dbeta[i] = c;
    }
    if (corrected && raw_gamma && raw_beta) {
        double sg = 0.0, sb = 0.0;
        for (int64_t b = 0; b < B; ++b) {
            sg += raw_gamma[b];
            sb += raw_beta[b];
        }
        const double bd = static_cast<double>(B);
        corrected[0] = sg / bd * (bd * bd);
        corrected[1] = sb / bd * (bd * bd);
    }
    return 0;
}

// gnstk::linear_backward_simultaneous (proj/src/layers.cpp:80-157)
int ref_linear_backward(const double* x, const double* g, const double* W, const double* bias,
                        int64_t B, int64_t M, int64_t K, int64_t L, double* dW, double* dbias,
                        double* raw_w, double* raw_b, double* corrected, double* dx) {
    return guard([&] {
        gnstk::LinearLayer layer;
        layer.weight = make({K, L}, W);
        if (bias) layer.bias = make({L}, bias);
        auto r = gnstk::linear_backward_simultaneous(layer, make({B, M, K}, x), make({B, M, L}, g));
        put(r.grads.weight_grads.at("weight"), dW);
        put(r.grads.per_example_sqnorms_raw.at("weight"), raw_w);
        if (corrected) corrected[0] = r.grads.per_example_sqnorms.at("weight");
        if (bias) {
            put(r.grads.weight_grads.at("bias"), dbias);
            put(r.grads.per_example_sqnorms_raw.at("bias"), raw_b);
            if (corrected) corrected[1] = r.grads.per_example_sqnorms.at("bias");
        }
        put(r.input_grad, dx);
    });
}

// gnstk::linear_perexample_sqnorm_frobenius (proj/src/layers.cpp:159-187)
int ref_linear_frobenius(const double* x, const double* g, int64_t B, int64_t T, int64_t K, int64_t L,
                         double* out) {
    return guard([&] {
        put(gnstk::linear_perexample_sqnorm_frobenius(make({B, T, K}, x), make({B, T, L}, g)), out);
    });
}

// gns.cpp:31-69
int ref_estimate(double g_big, double g_small, int64_t b_big, int64_t b_small, int64_t n_small, double* g2,
                 double* s) {
    return guard([&] {
        gnstk::GradStats st{g_big, g_small, b_big, b_small, n_small};
        *g2 = gnstk::estimate_g2(st);
        *s = gnstk::estimate_s(st);
    });
}

int ref_make_gns_estimate(double g2, double s, double* b_simple, int* defined) {
    auto e = gnstk::make_gns_estimate(g2, s);
    *b_simple = e.b_simple;
    *defined = e.b_simple_defined ? 1 : 0;
    return 0;
}

int ref_ema_update(double alpha, double value, int64_t count, double x, double* out_value, int64_t* out_count) {
    return guard([&] {
        gnstk::EmaState st{alpha, value, count};
        st = gnstk::ema_update(st, x);
        *out_value = st.value;
        *out_count = st.count;
    });
}

// costmodel.cpp:58-64
int ref_crossover_t(int64_t k, int64_t l, int criterion, double* out) {
    return guard([&] {
        *out = gnstk::crossover_t(k, l, criterion == 0 ? gnstk::CostCriterion::IO : gnstk::CostCriterion::FLOPS);
    });
}

int ref_flops(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out) {
    return guard([&] {
        auto p = gnstk::flops({b, t, k, l, 4}, method == 0 ? gnstk::CostMethod::Simultaneous : gnstk::CostMethod::Frobenius);
        out[0] = p.weight_grad;
        out[1] = p.grad_norms;
    });
}

int ref_io_values(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out) {
    return guard([&] {
        auto p = gnstk::io_values({b, t, k, l, 4}, method == 0 ? gnstk::CostMethod::Simultaneous : gnstk::CostMethod::Frobenius);
        out[0] = p.weight_grad;
        out[1] = p.grad_norms;
    });
}

// rng.hpp: draw n Gaussians from a fresh stream (used to cross-check orc_gauss)
void ref_gauss_draw(uint64_t seed, int64_t n, double* out) {
    gnstk::GaussianStream gs(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = gs.next();
}

}  // extern "C"

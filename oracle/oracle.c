/*
 * oracle.c — CPU restatement of the reference gnstk hot path (fp64).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -ffp-contract=off
 * so the synthetic generator matches the device generator bit for bit and
 * the fp64 arithmetic follows the reference's operation order exactly.
 *
 * Citations are relative to /root/reference/.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

static char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int fail(const char* prefix, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s%s", prefix, msg);
    return ORC_EINVAL;
}
#define LFAIL(m) return fail("layers: ", (m))   /* layers.cpp:13-15 */
#define GFAIL(m) return fail("gns: ", (m))      /* gns.cpp:10-12 */
#define CFAIL(m) return fail("costmodel: ", (m)) /* costmodel.cpp:10-12 */

/* ------------------------------------------------------------------ rng -- */
/* proj/include/gnstk/rng.hpp:19-24 — Weyl increment then avalanche. */
uint64_t orc_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* rng.hpp:27 — 53-bit uniform in [0,1). */
double orc_splitmix64_unit(uint64_t* state) {
    return (double)(orc_splitmix64_next(state) >> 11) * 0x1.0p-53;
}

/* rng.hpp:30 — uniform in (0,1]. */
static double unit_open(uint64_t* state) {
    return (double)((orc_splitmix64_next(state) >> 11) + 1) * 0x1.0p-53;
}

/* rng.hpp:33-38 */
uint64_t orc_splitmix64_below(uint64_t* state, uint64_t n) {
    uint64_t v = (uint64_t)(orc_splitmix64_unit(state) * (double)n);
    return v >= n ? n - 1 : v;
}

/* rng.hpp:42-45 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t tag) {
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ull * (tag + 1));
    return orc_splitmix64_next(&s);
}

void orc_gauss_init(orc_gauss* g, uint64_t seed) {
    g->state = seed;
    g->has_spare = 0;
    g->spare = 0.0;
}

/* rng.hpp:56-66 — Box–Muller, cosine first, sine kept as the spare. */
double orc_gauss_next(orc_gauss* g) {
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    const double u1 = unit_open(&g->state);
    const double u2 = orc_splitmix64_unit(&g->state);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    g->spare = r * sin(a);
    g->has_spare = 1;
    return r * cos(a);
}

/* ------------------------------------------------------- synthetic inputs -- */
/* Z(stream,i) = (U - 1/2)*sqrt(12), U = (splitmix64(mix_seed(2411,stream)+i) >> 40) * 2^-24.
 * All float ops are single roundings in a fixed order (no contraction). */
float orc_synth_z(uint64_t stream, uint64_t i) {
    uint64_t st = orc_mix_seed(2411u, stream) + i;
    const uint64_t h = orc_splitmix64_next(&st);
    const float u = (float)(h >> 40) * 0x1.0p-24f;
    return (u - 0.5f) * 3.4641016151377544f;
}

float orc_round_bf16(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) {
        if (u & 0x007fffffu) u |= 0x00400000u; /* quiet NaN */
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);
    }
    u &= 0xffff0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

void orc_synth_ln(float* x, float* dy, float* gamma, float* beta, int64_t B, int64_t T, int64_t D,
                  int64_t b_offset, int64_t B_div, float sigma, uint64_t s0, int round_bf16) {
    const float bdiv = (float)B_div;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t) {
            const int64_t gb = b + b_offset;
            const int64_t grow = gb * T + t;
            const float row_off = 0.5f * orc_synth_z(s0 + 1, (uint64_t)grow);
            for (int64_t d = 0; d < D; ++d) {
                const uint64_t gidx = (uint64_t)(grow * D + d);
                const int64_t li = (b * T + t) * D + d;
                float xv = orc_synth_z(s0, gidx) + row_off;
                const float noise = sigma * orc_synth_z(s0 + 3, gidx);
                float gv = (orc_synth_z(s0 + 2, (uint64_t)(t * D + d)) + noise) / bdiv;
                if (round_bf16) {
                    xv = orc_round_bf16(xv);
                    gv = orc_round_bf16(gv);
                }
                if (x) x[li] = xv;
                if (dy) dy[li] = gv;
            }
        }
    for (int64_t d = 0; d < D; ++d) {
        if (gamma) gamma[d] = 1.0f + 0.1f * orc_synth_z(s0 + 4, (uint64_t)d);
        if (beta) beta[d] = 0.1f * orc_synth_z(s0 + 5, (uint64_t)d);
    }
}

void orc_synth_linear(float* x, float* dy, int64_t B, int64_t T, int64_t K, int64_t L,
                      int64_t b_offset, int64_t B_div, uint64_t s0, int round_bf16) {
    const float scale = (float)B_div * sqrtf((float)T);
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t) {
            const int64_t grow = (b + b_offset) * T + t;
            const int64_t lrow = b * T + t;
            if (x)
                for (int64_t k = 0; k < K; ++k) {
                    float v = orc_synth_z(s0, (uint64_t)(grow * K + k));
                    x[lrow * K + k] = round_bf16 ? orc_round_bf16(v) : v;
                }
            if (dy)
                for (int64_t l = 0; l < L; ++l) {
                    const float a = orc_synth_z(s0 + 1, (uint64_t)(t * L + l));
                    const float c = orc_synth_z(s0 + 2, (uint64_t)(grow * L + l));
                    float v = (a + c) / scale;
                    dy[lrow * L + l] = round_bf16 ? orc_round_bf16(v) : v;
                }
        }
}

/* --------------------------------------------------------------- layers -- */
/* layers.cpp:39-42 — mean of per-example squared norms times B^2. */
static double corrected_mean_sqnorm(double sum_sq, int64_t batch) {
    const double b = (double)batch;
    return sum_sq / b * (b * b);
}

/* layers.cpp:44-48 — sequential sum of squares. */
static double row_sqnorm(const double* p, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += p[i] * p[i];
    return acc;
}

/* layers.cpp:189-229 */
int orc_layernorm_forward(const double* x, const double* gamma, const double* beta, double eps,
                          int64_t rows, int64_t D, double* y, double* xhat, double* inv_std) {
    if (!(eps > 0.0)) LFAIL("epsilon must be positive");          /* :192 */
    if (D < 2) LFAIL("layernorm needs trailing extent >= 2");      /* :194 */
    const double kd = (double)D;
    for (int64_t r = 0; r < rows; ++r) {
        const double* xr = x + r * D;
        double mean = 0.0;
        for (int64_t i = 0; i < D; ++i) mean += xr[i];
        mean /= kd;
        double var = 0.0;
        for (int64_t i = 0; i < D; ++i) {
            const double d = xr[i] - mean;
            var += d * d;
        }
        var /= kd;
        const double inv = 1.0 / sqrt(var + eps);
        if (inv_std) inv_std[r] = inv;
        for (int64_t i = 0; i < D; ++i) {
            const double n = (xr[i] - mean) * inv;
            if (xhat) xhat[r * D + i] = n;
            if (y) y[r * D + i] = gamma[i] * n + beta[i];
        }
    }
    return ORC_OK;
}

/* layers.cpp:231-298 */
int orc_layernorm_backward(const double* xhat, const double* inv_std, const double* g,
                           const double* gamma, int64_t B, int64_t M, int64_t D, double* dx,
                           double* dgamma, double* dbeta, double* raw_gamma, double* raw_beta,
                           double* corrected) {
    if (B == 0) LFAIL("empty batch");                               /* :239 */
    double grow_stack[64], brow_stack[64];
    double* grow = D <= 64 ? grow_stack : (double*)malloc(sizeof(double) * (size_t)D);
    double* brow = D <= 64 ? brow_stack : (double*)malloc(sizeof(double) * (size_t)D);
    if (dgamma) memset(dgamma, 0, sizeof(double) * (size_t)D);
    if (dbeta) memset(dbeta, 0, sizeof(double) * (size_t)D);
    double g_sum = 0.0, b_sum = 0.0;
    for (int64_t b = 0; b < B; ++b) {                               /* :248-269 */
        memset(grow, 0, sizeof(double) * (size_t)D);
        memset(brow, 0, sizeof(double) * (size_t)D);
        for (int64_t m = 0; m < M; ++m) {
            const double* nr = xhat + (b * M + m) * D;
            const double* gr = g + (b * M + m) * D;
            for (int64_t i = 0; i < D; ++i) {
                grow[i] += nr[i] * gr[i];
                brow[i] += gr[i];
            }
        }
        const double sg = row_sqnorm(grow, D);
        const double sb = row_sqnorm(brow, D);
        if (raw_gamma) raw_gamma[b] = sg;
        if (raw_beta) raw_beta[b] = sb;
        g_sum += sg;
        b_sum += sb;
        for (int64_t i = 0; i < D; ++i) {
            if (dgamma) dgamma[i] += grow[i];
            if (dbeta) dbeta[i] += brow[i];
        }
    }
    if (corrected) {                                                /* :272-273 */
        corrected[0] = corrected_mean_sqnorm(g_sum, B);
        corrected[1] = corrected_mean_sqnorm(b_sum, B);
    }
    if (dx) {                                                       /* :277-296 */
        const double kd = (double)D;
        for (int64_t row = 0; row < B * M; ++row) {
            const double* nr = xhat + row * D;
            const double* gr = g + row * D;
            double* dr = dx + row * D;
            const double inv = inv_std[row];
            double mh = 0.0, mhx = 0.0;
            for (int64_t i = 0; i < D; ++i) {
                const double h = gamma[i] * gr[i];
                mh += h;
                mhx += h * nr[i];
            }
            mh /= kd;
            mhx /= kd;
            for (int64_t i = 0; i < D; ++i) dr[i] = inv * (gamma[i] * gr[i] - mh - nr[i] * mhx);
        }
    }
    if (D > 64) {
        free(grow);
        free(brow);
    }
    return ORC_OK;
}

int orc_layernorm_backward_xmr(const double* x, const double* mean, const double* rstd,
                               const double* g, const double* gamma, int64_t B, int64_t M,
                               int64_t D, double* dx, double* dgamma, double* dbeta,
                               double* raw_gamma, double* raw_beta, double* corrected) {
    const int64_t n = B * M * D;
    double* xhat = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t r = 0; r < B * M; ++r)
        for (int64_t i = 0; i < D; ++i) xhat[r * D + i] = (x[r * D + i] - mean[r]) * rstd[r];
    const int rc = orc_layernorm_backward(xhat, rstd, g, gamma, B, M, D, dx, dgamma, dbeta,
                                          raw_gamma, raw_beta, corrected);
    free(xhat);
    return rc;
}

/* layers.cpp:80-157 */
int orc_linear_backward(const double* x, const double* g, const double* W, int has_bias,
                        int64_t B, int64_t M, int64_t K, int64_t L, double* dW, double* dbias,
                        double* raw_w, double* raw_b, double* corrected, double* dx) {
    if (B == 0) LFAIL("empty batch");                               /* :89 */
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(K * L > 0 ? K * L : 1));
    double* bscratch = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
    if (dW) memset(dW, 0, sizeof(double) * (size_t)(K * L));
    if (has_bias && dbias) memset(dbias, 0, sizeof(double) * (size_t)L);
    double w_sum = 0.0, b_sum = 0.0;
    for (int64_t b = 0; b < B; ++b) {                               /* :107-131 */
        memset(scratch, 0, sizeof(double) * (size_t)(K * L));
        if (has_bias) memset(bscratch, 0, sizeof(double) * (size_t)L);
        for (int64_t m = 0; m < M; ++m) {
            const double* xr = x + (b * M + m) * K;
            const double* gr = g + (b * M + m) * L;
            for (int64_t i = 0; i < K; ++i) {
                const double xv = xr[i];
                double* srow = scratch + i * L;
                for (int64_t j = 0; j < L; ++j) srow[j] += xv * gr[j];
            }
            if (has_bias)
                for (int64_t j = 0; j < L; ++j) bscratch[j] += gr[j];
        }
        const double sb = row_sqnorm(scratch, K * L);
        if (raw_w) raw_w[b] = sb;
        w_sum += sb;
        if (dW)
            for (int64_t i = 0; i < K * L; ++i) dW[i] += scratch[i];
        if (has_bias) {
            const double bb = row_sqnorm(bscratch, L);
            if (raw_b) raw_b[b] = bb;
            b_sum += bb;
            if (dbias)
                for (int64_t j = 0; j < L; ++j) dbias[j] += bscratch[j];
        }
    }
    if (corrected) {                                                /* :134, :138 */
        corrected[0] = corrected_mean_sqnorm(w_sum, B);
        corrected[1] = has_bias ? corrected_mean_sqnorm(b_sum, B) : 0.0;
    }
    if (dx) {                                                       /* :142-155 */
        for (int64_t row = 0; row < B * M; ++row) {
            const double* gr = g + row * L;
            double* xr = dx + row * K;
            for (int64_t i = 0; i < K; ++i) {
                const double* wr = W + i * L;
                double acc = 0.0;
                for (int64_t j = 0; j < L; ++j) acc += gr[j] * wr[j];
                xr[i] = acc;
            }
        }
    }
    free(scratch);
    free(bscratch);
    return ORC_OK;
}

/* layers.cpp:159-187 */
int orc_linear_frobenius(const double* x, const double* g, int64_t B, int64_t T, int64_t K,
                         int64_t L, double* out) {
    double* xx = (double*)malloc(sizeof(double) * (size_t)(T * T > 0 ? T * T : 1));
    double* gg = (double*)malloc(sizeof(double) * (size_t)(T * T > 0 ? T * T : 1));
    for (int64_t b = 0; b < B; ++b) {
        const double* xb = x + b * T * K;
        const double* gb = g + b * T * L;
        for (int64_t t = 0; t < T; ++t)
            for (int64_t u = 0; u < T; ++u) {
                double accx = 0.0;
                for (int64_t i = 0; i < K; ++i) accx += xb[t * K + i] * xb[u * K + i];
                xx[t * T + u] = accx;
                double accg = 0.0;
                for (int64_t j = 0; j < L; ++j) accg += gb[t * L + j] * gb[u * L + j];
                gg[t * T + u] = accg;
            }
        double acc = 0.0;
        for (int64_t i = 0; i < T * T; ++i) acc += xx[i] * gg[i];
        out[b] = acc;
    }
    free(xx);
    free(gg);
    return ORC_OK;
}

/* layers.cpp:315-368.  Per example: rows of the table touched by the
 * example accumulate g over its tokens (t order); the touched ids, ascending,
 * give raw_b = one flat sum of squares and are added into dW (b order).
 * Errors: an id outside [0, V) (layers.cpp:333), B == 0 (:322). */
int orc_embedding_backward(const int32_t* ids, const double* g, int64_t B, int64_t T, int64_t V, int64_t D,
                           double* dW, double* raw, double* corrected) {
    if (B == 0) LFAIL("empty batch");
    for (int64_t i = 0; i < B * T; ++i)
        if (ids[i] < 0 || ids[i] >= V) LFAIL("id out of range");
    double* scratch = (double*)calloc((size_t)(V * D > 0 ? V * D : 1), sizeof(double));
    char* seen = (char*)calloc((size_t)(V > 0 ? V : 1), 1);
    int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
    for (int64_t i = 0; i < V * D; ++i) dW[i] = 0.0;
    double sum_sq = 0.0;
    for (int64_t b = 0; b < B; ++b) {
        int64_t nt = 0;
        for (int64_t t = 0; t < T; ++t) {
            const int64_t id = ids[b * T + t];
            if (!seen[id]) {
                seen[id] = 1;
                touched[nt++] = id;
            }
            const double* gr = g + (b * T + t) * D;
            double* row = scratch + id * D;
            for (int64_t j = 0; j < D; ++j) row[j] += gr[j];
        }
        /* ascending ids (insertion sort: T is small in every test family) */
        for (int64_t i = 1; i < nt; ++i) {
            const int64_t v = touched[i];
            int64_t k = i - 1;
            while (k >= 0 && touched[k] > v) {
                touched[k + 1] = touched[k];
                --k;
            }
            touched[k + 1] = v;
        }
        double sb = 0.0;
        for (int64_t i = 0; i < nt; ++i) {
            double* src = scratch + touched[i] * D;
            for (int64_t j = 0; j < D; ++j) sb += src[j] * src[j];
            double* dst = dW + touched[i] * D;
            for (int64_t j = 0; j < D; ++j) dst[j] += src[j];
            for (int64_t j = 0; j < D; ++j) src[j] = 0.0;
            seen[touched[i]] = 0;
        }
        raw[b] = sb;
        sum_sq += sb;
    }
    *corrected = sum_sq / (double)B * ((double)B * (double)B);
    free(scratch);
    free(seen);
    free(touched);
    return ORC_OK;
}

/* ------------------------------------------------------------------ gns -- */
/* gns.cpp:14-18 */
static int check_batches(const orc_grad_stats* s) {
    if (s->b_small < 1) GFAIL("b_small must be >= 1");
    if (s->b_big <= s->b_small) GFAIL("b_big must exceed b_small");
    if (s->n_small < 1) GFAIL("n_small must be >= 1");
    return ORC_OK;
}

/* gns.cpp:31-36 */
int orc_estimate_g2(const orc_grad_stats* s, double* out) {
    if (check_batches(s)) return ORC_EINVAL;
    const double bb = (double)s->b_big, bs = (double)s->b_small;
    *out = (bb * s->g_big_sqnorm - bs * s->g_small_sqnorm_mean) / (bb - bs);
    return ORC_OK;
}

/* gns.cpp:38-43 */
int orc_estimate_s(const orc_grad_stats* s, double* out) {
    if (check_batches(s)) return ORC_EINVAL;
    const double bb = (double)s->b_big, bs = (double)s->b_small;
    *out = (s->g_small_sqnorm_mean - s->g_big_sqnorm) / (1.0 / bs - 1.0 / bb);
    return ORC_OK;
}

/* gns.cpp:45-54, guard gns.hpp:34 */
orc_gns_estimate orc_make_gns_estimate(double g2, double s) {
    orc_gns_estimate e;
    e.g2 = g2;
    e.s = s;
    e.b_simple = 0.0;
    e.b_simple_defined = 0;
    if (fabs(g2) >= 1e-12) {
        e.b_simple = s / g2;
        e.b_simple_defined = 1;
    }
    return e;
}

/* gns.cpp:56-64 */
int orc_ema_update(orc_ema_state* st, double x) {
    if (!(st->alpha > 0.0) || st->alpha > 1.0) GFAIL("ema alpha must be in (0, 1]");
    if (st->count == 0)
        st->value = x;
    else
        st->value = (1.0 - st->alpha) * st->value + st->alpha * x;
    ++st->count;
    return ORC_OK;
}

/* gns.cpp:66-69 */
int orc_smoothed_gns(const orc_ema_state* g2, const orc_ema_state* s, orc_gns_estimate* out) {
    if (g2->count < 1 || s->count < 1) GFAIL("smoothed_gns needs at least one sample in each state");
    *out = orc_make_gns_estimate(g2->value, s->value);
    return ORC_OK;
}

/* gns.cpp:71-89 */
int orc_aggregate(const orc_grad_stats* stats, const int* types, int n, int group,
                  orc_grad_stats* out) {
    int first = 1;
    for (int i = 0; i < n; ++i) {
        if (group >= 0 && types[i] != group) continue;
        if (first) {
            *out = stats[i];
            out->g_big_sqnorm = 0.0;
            out->g_small_sqnorm_mean = 0.0;
            first = 0;
        } else if (stats[i].b_big != out->b_big || stats[i].b_small != out->b_small ||
                   stats[i].n_small != out->n_small) {
            GFAIL("aggregate requires matching batch sizes across layers");
        }
        out->g_big_sqnorm += stats[i].g_big_sqnorm;
        out->g_small_sqnorm_mean += stats[i].g_small_sqnorm_mean;
    }
    if (first) GFAIL("aggregate over an empty selection");
    return ORC_OK;
}

/* ------------------------------------------------------------ costmodel -- */
static int cost_check(int64_t b, int64_t t, int64_t k, int64_t l) {
    if (b < 1 || t < 1 || k < 1 || l < 1) CFAIL("shape dims must be positive");
    return ORC_OK;
}

/* costmodel.cpp:25-37 */
int orc_flops(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out) {
    if (cost_check(b, t, k, l)) return ORC_EINVAL;
    if (method == 0) {
        out[0] = b * k * l * (2 * t - 1) + k * l * (b - 1);
        out[1] = b * k * l + b * (k * l - 1);
    } else {
        out[0] = k * l * (2 * b * t - 1);
        out[1] = b * t * t * (2 * k + 2 * l - 2) + b * t * t;
    }
    return ORC_OK;
}

/* costmodel.cpp:39-51 */
int orc_io_values(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out) {
    if (cost_check(b, t, k, l)) return ORC_EINVAL;
    if (method == 0) {
        out[0] = b * k * l + b * k * t + b * l * t;
        out[1] = b * k * l + b;
    } else {
        out[0] = b * k * t + b * l * t + k * l;
        out[1] = 2 * b * t * t + b;
    }
    return ORC_OK;
}

/* costmodel.cpp:58-64 */
int orc_crossover_t(int64_t k, int64_t l, int criterion, double* out) {
    if (k < 1 || l < 1) CFAIL("dims must be positive");
    const double kd = (double)k, ld = (double)l;
    if (criterion == 0)
        *out = sqrt(2.0 * kd * ld) / 2.0;
    else
        *out = sqrt((2.0 * kd * ld - 1.0) / (2.0 * kd + 2.0 * ld - 1.0));
    return ORC_OK;
}

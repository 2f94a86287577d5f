/*
 * oracle.h — CPU restatement of the reference gnstk hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker (or as the
 * timed CPU baseline).  The CUDA product path never calls into this code.
 *
 * Every function restates one reference function in plain C, fp64, with the
 * reference's summation order, so results are bit-comparable with the
 * reference library compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile).  Parity of this restatement is pinned against the
 * reference's own known-answer tests and against oracle/_ref outputs stored
 * under tests/golden/ (tests/test_oracle_golden.py).
 *
 * Citations are relative to /root/reference/.
 */
#ifndef GNSB_ORACLE_H
#define GNSB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: 0 ok, 1 invalid argument (the reference throws
 * std::invalid_argument in exactly these cases). */
enum { ORC_OK = 0, ORC_EINVAL = 1 };

const char* orc_last_error(void);

/* ---- rng (proj/include/gnstk/rng.hpp:11-67) ------------------------------ */
uint64_t orc_splitmix64_next(uint64_t* state);            /* rng.hpp:19-24 */
double orc_splitmix64_unit(uint64_t* state);              /* rng.hpp:27     */
uint64_t orc_splitmix64_below(uint64_t* state, uint64_t n); /* rng.hpp:33-38 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t tag);       /* rng.hpp:42-45 */

typedef struct {
    uint64_t state;
    int has_spare;
    double spare;
} orc_gauss;                                               /* rng.hpp:48-67 */
void orc_gauss_init(orc_gauss* g, uint64_t seed);
double orc_gauss_next(orc_gauss* g);

/* ---- synthetic workload generator, bit-identical with
 * the device generator in paper_2411_00999_b200/csrc/synth.cu ------------- */
float orc_synth_z(uint64_t stream, uint64_t i);
/* LN recipe: x = Z(s0,idx) + 0.5 Z(s0+1,row); dy = (Z(s0+2,t*D+d) + sigma Z(s0+3,idx)) / B_div;
 * gamma = 1 + 0.1 Z(s0+4,d); beta = 0.1 Z(s0+5,d).  b_global_offset shifts the
 * example index so shards of a global batch see identical values.
 * round_bf16 != 0 rounds x, dy to bf16 (RNE) before storing (as float). */
void orc_synth_ln(float* x, float* dy, float* gamma, float* beta, int64_t B, int64_t T, int64_t D,
                  int64_t b_offset, int64_t B_div, float sigma, uint64_t stream0, int round_bf16);
/* linear recipe: X = Z(s0,idx); dY = (Z(s0+1,t*L+l) + Z(s0+2,idx)) / (B_div*sqrt(T)) */
void orc_synth_linear(float* x, float* dy, int64_t B, int64_t T, int64_t K, int64_t L,
                      int64_t b_offset, int64_t B_div, uint64_t stream0, int round_bf16);
float orc_round_bf16(float v);

/* ---- layers (proj/src/layers.cpp) ---------------------------------------- */
/* layers.cpp:189-229: y, xhat [rows, D]; inv_std [rows] */
int orc_layernorm_forward(const double* x, const double* gamma, const double* beta, double eps,
                          int64_t rows, int64_t D, double* y, double* xhat, double* inv_std);

/* layers.cpp:231-298.  Rank>=2 input viewed as (B, M, D).  Outputs:
 * dx [B*M*D], dgamma/dbeta [D], raw_gamma/raw_beta [B],
 * corrected[2] = (sum raw / B) * B^2 for gamma, beta.  Any output may be NULL. */
int orc_layernorm_backward(const double* xhat, const double* inv_std, const double* g,
                           const double* gamma, int64_t B, int64_t M, int64_t D, double* dx,
                           double* dgamma, double* dbeta, double* raw_gamma, double* raw_beta,
                           double* corrected);

/* Same, but consumes (x, mean, rstd) as the B200 kernel does; xhat is formed
 * as (x - mean) * rstd in fp64 before the reference arithmetic. */
int orc_layernorm_backward_xmr(const double* x, const double* mean, const double* rstd,
                               const double* g, const double* gamma, int64_t B, int64_t M,
                               int64_t D, double* dx, double* dgamma, double* dbeta,
                               double* raw_gamma, double* raw_beta, double* corrected);

/* layers.cpp:80-157 (weight-grad "simultaneous" form).  W [K,L]; bias may be NULL
 * (then dbias/raw_bias are untouched).  corrected[2] = weight, bias. dx may be NULL. */
int orc_linear_backward(const double* x, const double* g, const double* W, int has_bias,
                        int64_t B, int64_t M, int64_t K, int64_t L, double* dW, double* dbias,
                        double* raw_w, double* raw_b, double* corrected, double* dx);

/* layers.cpp:159-187 (Gram / Frobenius form), raw per-example [B]. */
int orc_linear_frobenius(const double* x, const double* g, int64_t B, int64_t T, int64_t K,
                         int64_t L, double* out);

int orc_embedding_backward(const int32_t* ids, const double* g, int64_t B, int64_t T, int64_t V, int64_t D,
                           double* dW, double* raw, double* corrected); /* layers.cpp:315-368 */

/* ---- gns (proj/src/gns.cpp) ----------------------------------------------- */
typedef struct {
    double g_big_sqnorm;
    double g_small_sqnorm_mean;
    int64_t b_big;
    int64_t b_small;
    int64_t n_small;
} orc_grad_stats;                                          /* gns.hpp:16-22 */

typedef struct {
    double g2, s, b_simple;
    int b_simple_defined;
} orc_gns_estimate;                                        /* gns.hpp:26-31 */

typedef struct {
    double alpha, value;
    int64_t count;
} orc_ema_state;                                           /* gns.hpp:36-40 */

int orc_estimate_g2(const orc_grad_stats* s, double* out);  /* gns.cpp:31-36 */
int orc_estimate_s(const orc_grad_stats* s, double* out);   /* gns.cpp:38-43 */
orc_gns_estimate orc_make_gns_estimate(double g2, double s); /* gns.cpp:45-54 */
int orc_ema_update(orc_ema_state* st, double x);            /* gns.cpp:56-64 */
int orc_smoothed_gns(const orc_ema_state* g2, const orc_ema_state* s, orc_gns_estimate* out); /* :66-69 */
/* gns.cpp:71-89; layer_types[i] in {0 emb,1 lin,2 ln}; group<0 = no filter.
 * Caller passes layers already sorted in LayerKey order. */
int orc_aggregate(const orc_grad_stats* stats, const int* layer_types, int n, int group,
                  orc_grad_stats* out);

/* ---- cost model (proj/src/costmodel.cpp) ---------------------------------- */
/* costmodel.cpp:25-37 / :39-51; method 0 = simultaneous, 1 = frobenius; out[2] */
int orc_flops(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out);
int orc_io_values(int64_t b, int64_t t, int64_t k, int64_t l, int method, int64_t* out);
/* costmodel.cpp:58-64; criterion 0 = IO, 1 = FLOPS */
int orc_crossover_t(int64_t k, int64_t l, int criterion, double* out);

#ifdef __cplusplus
}
#endif
#endif

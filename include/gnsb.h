/*
 * gnsb.h — C ABI of the B200-native per-example-gradient-norm / GNS path.
 *
 * This is the drop-in boundary for the reference library `gnstk`
 * (/root/reference/proj, citations below are relative to it).  The reference
 * exposes a C++ value-semantics API (free functions in namespace gnstk over
 * fp64 gnstk::Tensor, errors as std::invalid_argument); this header is the
 * thin C layer underneath the B200 C++ drop-in (include/gnstk/*.hpp).  Every
 * entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers owned by the caller, row-major,
 *     contiguous.  Rows of one example are contiguous: an input of reference
 *     shape [B, ..., D] is viewed as (B, M, D), M = product of middle extents
 *     (proj/src/layers.cpp:19-28).
 *   - Row data (x, xhat, dy, dx, y) have dtype `dt`.  Per-feature and per-row
 *     statistics (gamma, beta, dgamma, dbeta, mean, rstd) are fp32 for
 *     GNSB_F32/GNSB_BF16 and fp64 for GNSB_F64.  Norm outputs are always fp64.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous; the library keeps no per-call state and
 *     is safe to call concurrently on distinct streams with distinct
 *     workspaces.
 *   - Validation failures return GNSB_EINVAL; gnsb_last_error() then holds the
 *     reference's message, including its prefix ("layers: ", "gns: ",
 *     "costmodel: ").  CUDA failures return GNSB_ECUDA.
 *   - No CPU fallback: without a CUDA device every compute entry point returns
 *     GNSB_ECUDA.
 */
#ifndef GNSB_H
#define GNSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GNSB_OK = 0, GNSB_EINVAL = 1, GNSB_ECUDA = 2, GNSB_ENCCL = 3, GNSB_ENOMEM = 4 } gnsb_status;
typedef enum { GNSB_F32 = 0, GNSB_BF16 = 1, GNSB_F64 = 2 } gnsb_dtype;

/* Library version string and the calling thread's last error message. */
const char* gnsb_version(void);
const char* gnsb_last_error(void);

/* ------------------------------------------------------------------------
 * LayerNorm forward.
 * Replaces gnstk::layernorm_forward (proj/include/gnstk/layers.hpp:76-77,
 * proj/src/layers.cpp:189-229).  Writes y (nullable), per-row mean/rstd
 * (nullable; the B200 backward's cache) and xhat (nullable; the reference's
 * LayerNormCache::normalized, whose inv_std is `rstd`).
 * Errors (reference wording): eps <= 0, D < 2.
 */
gnsb_status gnsb_ln_fwd(const void* x, const void* gamma, const void* beta, void* y, void* mean, void* rstd,
                        void* xhat, int64_t rows, int64_t D, double eps, gnsb_dtype dt, void* stream);

/* ------------------------------------------------------------------------
 * Fused LayerNorm backward + per-example squared gradient norms.
 * Replaces gnstk::layernorm_backward_simultaneous
 * (proj/include/gnstk/layers.hpp:79-80, proj/src/layers.cpp:231-298).
 *
 *   x_or_xhat, mean : with mean != NULL the input is x and
 *                     xhat = (x - mean) * rstd; with mean == NULL the input is
 *                     the reference cache's `normalized` tensor.
 *   rstd            : [B*M] (the reference cache's inv_std)
 *   dy              : [B*M*D] upstream gradient of a MEAN-reduced loss
 *   dx              : [B*M*D] (nullable: skip the input gradient)
 *   dgamma, dbeta   : [D] batch-summed parameter gradients
 *   raw_sq_gamma/beta : [B] uncorrected per-example ||dgamma_b||^2, ||dbeta_b||^2
 *                     (LayerGradOutput::per_example_sqnorms_raw), nullable
 *   sums            : [4] nullable: { sum_b raw_gamma, sum_b raw_beta,
 *                     ||dgamma||^2, ||dbeta||^2 }.  The reference's corrected
 *                     value (per_example_sqnorms) is sums[i] / B * B^2.
 *   with_norms      : 0 runs the otherwise-identical plain LayerNorm backward:
 *                     the same kernels over one "example" of B*M rows (no
 *                     per-example flushes, one partial slot per CTA, no
 *                     squares); raw/sums untouched.  The row pass of a
 *                     deferred plain call is gnsb_ln_bwd_rows with B = 1,
 *                     M = B*M (and its pending item likewise).
 *   ws, ws_bytes    : device workspace of at least
 *                     gnsb_ln_bwd_workspace_size() bytes.  It must be
 *                     zero-filled before its first use; every call leaves it
 *                     ready for the next.  One workspace per concurrent stream.
 * Errors (reference wording): B == 0 ("empty batch"), D < 1.
 * Deterministic: results are bitwise identical run to run on a given GPU.
 */
gnsb_status gnsb_ln_bwd_workspace_size(int64_t B, int64_t M, int64_t D, gnsb_dtype dt, size_t* bytes);
gnsb_status gnsb_ln_bwd(const void* x_or_xhat, const void* mean, const void* rstd, const void* dy,
                        const void* gamma, void* dx, void* dgamma, void* dbeta, double* raw_sq_gamma,
                        double* raw_sq_beta, double* sums, int32_t with_norms, int64_t B, int64_t M, int64_t D,
                        gnsb_dtype dt, void* ws, size_t ws_bytes, void* stream);
/* Deferred stage 2 (one launch for several LayerNorms).
 * gnsb_ln_bwd == gnsb_ln_bwd_rows followed by gnsb_ln_bwd_reduce of that one
 * layer.  A backward pass may instead run the row pass of every LayerNorm as
 * it comes (dx is final when gnsb_ln_bwd_rows returns in stream order) and
 * reduce all of them at the end in one launch: the per-example combine,
 * squares and dgamma/dbeta sums then cost one stage-2 tail per step instead of
 * one per layer.  Each pending layer needs its own workspace, untouched
 * between its row pass and the reduce.  Results are identical to gnsb_ln_bwd.
 */
gnsb_status gnsb_ln_bwd_rows(const void* x_or_xhat, const void* mean, const void* rstd, const void* dy,
                             const void* gamma, void* dx, int64_t B, int64_t M, int64_t D, gnsb_dtype dt, void* ws,
                             size_t ws_bytes, void* stream);
typedef struct {
    void* ws;                 /* the workspace its gnsb_ln_bwd_rows call used */
    size_t ws_bytes;
    int64_t B, M, D;          /* the shape of that call */
    int32_t dt;               /* gnsb_dtype of that call */
    void* dgamma;             /* outputs, as for gnsb_ln_bwd */
    void* dbeta;
    double* raw_sq_gamma;
    double* raw_sq_beta;
    double* sums;
} gnsb_ln_bwd_pending;
/* All items must share the statistics dtype (fp32 for F32/BF16 rows, fp64 for
 * F64) and with_norms; at most 64 items. */
gnsb_status gnsb_ln_bwd_reduce(const gnsb_ln_bwd_pending* items, int32_t n, int32_t with_norms, void* stream);

/* Launch geometry the backward uses for this shape (reporting / roofline). */
gnsb_status gnsb_ln_bwd_geometry(int64_t B, int64_t M, int64_t D, gnsb_dtype dt, int32_t* grid, int32_t* threads,
                                 int32_t* stages);

/* ------------------------------------------------------------------------
 * Linear layer: per-example squared weight-gradient norms (3-D regime).
 * Replaces gnstk::linear_backward_simultaneous (proj/include/gnstk/layers.hpp:69,
 * proj/src/layers.cpp:80-157) and gnstk::linear_perexample_sqnorm_frobenius
 * (layers.hpp:74, layers.cpp:159-187).  x [B, T, K], g [B, T, L] (g from a
 * MEAN-reduced loss).
 *
 *   form 1 (weight-gradient / "simultaneous" form): dW_b = sum_t x_t^T g_t per
 *          example, raw_w[b] = ||dW_b||_F^2, dW = sum_b dW_b (dW nullable).
 *          bf16 rows with K % 8 == 0 and L % 8 == 0 (16-byte row strides; any
 *          T, tile tails zero-filled by TMA) run on the tcgen05 tensor-core
 *          kernel (fp32 accumulate); fp32 rows and other shapes run a generic
 *          fp64-accumulating CUDA kernel; fp64 rows follow the reference's
 *          operation order exactly (batch-invariant per-example values).
 *   form 2 (Gram / Frobenius form): raw_w[b] = <X_b X_b^T, G_b G_b^T>_F; dW must
 *          be NULL (the reference's Frobenius function returns norms only);
 *          tensor cores under the same bf16 / K, L % 8 condition.
 *   form 0 (auto): form 1 when dW is requested; otherwise the cheaper form by
 *          the FLOP model (Gram when T*(K+L) < 2*K*L, proj/src/costmodel.cpp:25-37).
 *   dW    : [K, L] fp32 (fp64 for GNSB_F64 rows).
 *   raw_w : [B] fp64 uncorrected per-example norms (nullable).
 *   sums  : [4] fp64 (nullable); writes sums[0] = sum_b raw_w and, for form 1,
 *           sums[2] = ||dW||^2 (slots 1 and 3 belong to the bias).
 * Errors: B == 0 ("empty batch"), non-positive extents.
 */
gnsb_status gnsb_linear_pe_workspace_size(int64_t B, int64_t T, int64_t K, int64_t L, gnsb_dtype dt, size_t* bytes);
gnsb_status gnsb_linear_pe_norms(const void* x, const void* g, void* dW, double* raw_w, double* sums, int64_t B,
                                 int64_t T, int64_t K, int64_t L, int32_t form, gnsb_dtype dt, void* ws,
                                 size_t ws_bytes, void* stream);
/* Bias of a linear layer: bias'_b = sum_t g[b,t,:], raw_b[b] = ||bias'_b||^2,
 * dbias = sum_b bias'_b (layers.cpp:118-119, 125-130).  sums[1] = sum_b raw_b,
 * sums[3] = ||dbias||^2.  Workspace: gnsb_linear_pe_workspace_size(B, T, 1, L). */
gnsb_status gnsb_linear_bias_pe(const void* g, void* dbias, double* raw_b, double* sums, int64_t B, int64_t T,
                                int64_t L, gnsb_dtype dt, void* ws, size_t ws_bytes, void* stream);
/* ------------------------------------------------------------------------
 * Linear-layer GEMMs.
 *   gnsb_linear_fwd replaces gnstk::linear_forward (proj/include/gnstk/layers.hpp:64,
 *     proj/src/layers.cpp:52-78): y[r, l] = sum_k x[r, k] W[k, l] (+ bias[l]).
 *   gnsb_linear_dx is the input gradient of gnstk::linear_backward_simultaneous
 *     (proj/src/layers.cpp:142-155): dx[r, k] = sum_l g[r, l] W[k, l].
 * x / g / y / dx: [rows, *] row tensors of dtype dt.  W [K, L] of dtype w_dt:
 * dt itself, or GNSB_F32 master weights with bf16 rows (rounded to a bf16
 * operand copy in the workspace each call).  bias [L]: fp32 (fp64 for fp64
 * rows), nullable.
 * bf16 rows with K % 8 == 0, L % 8 == 0 and 16-byte aligned buffers run the
 * tcgen05 tensor-core kernel (bf16 operands, fp32 accumulation, any row count;
 * tile tails are zero-filled by TMA).  fp32 rows with fp32 weights (K, L
 * multiples of 4) run the 3xTF32 tensor-core kernel: both operands split into
 * tf32 hi + lo parts once per call, each product formed as lo*hi + hi*lo +
 * hi*hi with fp32 accumulation (fp32-level accuracy; the split copies come
 * from the stream-ordered pool).  Other shapes run a generic fp64-accumulating
 * kernel; fp64 rows reproduce the reference's operation order bit for bit.
 * Workspace: gnsb_linear_gemm_workspace_size bytes (0 unless W must be converted).
 */
gnsb_status gnsb_linear_gemm_workspace_size(int64_t K, int64_t L, gnsb_dtype dt, gnsb_dtype w_dt, size_t* bytes);
gnsb_status gnsb_linear_fwd(const void* x, const void* W, const void* bias, void* y, int64_t rows, int64_t K, int64_t L,
                            gnsb_dtype dt, gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream);
gnsb_status gnsb_linear_dx(const void* g, const void* W, void* dx, int64_t rows, int64_t K, int64_t L, gnsb_dtype dt,
                           gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream);

/* The same two products with an elementwise epilogue fused into the store
 * (the toy model's steps around its linear layers, proj/src/model.cpp:95-100,
 * :169-171).  kind 0 = forward (x W + bias), 1 = input grad (g W^T, bias
 * ignored).  epilogue, on v = the product (+ bias):
 *   0 none: out = v;  1 tanh (forward): out = tanh(v);
 *   2 residual (forward): out = aux + v;  3 tanh backward (input grad):
 *   out = v * (1 - aux^2) with aux the tanh output.
 * aux [rows, N] of dtype dt (N = L forward, K input grad), may alias nothing
 * written by the call. */
gnsb_status gnsb_linear_gemm(int32_t kind, int32_t epilogue, const void* a, const void* W, const void* bias,
                             const void* aux, void* out, int64_t rows, int64_t K, int64_t L, gnsb_dtype dt,
                             gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream);

/* Softmax cross-entropy of the head, forward + backward in one kernel
 * (the reference's cross_entropy with dlogits, proj/src/model.cpp:113-141):
 *   loss_rows[r] = log(sum_c exp(l[r,c] - m)) + m - l[r, target[r]]   (fp64)
 *   dlogits[r,c] = (softmax(l[r])[c] - [c == target[r]]) * upstream_scale
 * logits / dlogits [rows, V] of dtype dt (dlogits nullable: loss only),
 * targets [rows] int32.  bad_targets (nullable device int32) is set to 1 when
 * a target was outside [0, V) (its loss row is NaN). */
gnsb_status gnsb_xent(const void* logits, const int32_t* targets, void* dlogits, double* loss_rows, int64_t rows,
                      int64_t V, double upstream_scale, gnsb_dtype dt, int32_t* bad_targets, void* stream);

/* Embedding row lookup out[i, :] = W[ids[i], :] (replaces gnstk::embedding_forward,
 * proj/include/gnstk/layers.hpp:83, proj/src/layers.cpp:300-313).  ids [n] int32
 * device, W [V, D] and out [n, D] of dtype dt.  bad_ids (nullable device int32)
 * is set to 1 when an id was outside [0, V) (its row is written as zeros). */
gnsb_status gnsb_embedding_fwd(const int32_t* ids, const void* W, void* out, int64_t n, int64_t V, int64_t D,
                               gnsb_dtype dt, int32_t* bad_ids, void* stream);

/* ------------------------------------------------------------------------
 * Embedding layer: table gradient + per-example squared norms (paper Alg. 3).
 * Replaces gnstk::embedding_backward_simultaneous
 * (proj/include/gnstk/layers.hpp:85-88, proj/src/layers.cpp:315-368).
 *   ids   : [B, T] int32 device token ids in [0, V)
 *   g     : [B, T, D] upstream gradient (dtype dt) of a MEAN-reduced loss
 *   dW    : [V, D] fp32 (fp64 for GNSB_F64 rows); untouched rows are zero
 *   raw_w : [B] fp64 uncorrected per-example ||dW_b||^2 (nullable)
 *   sums  : [4] fp64 (nullable): sums[0] = sum_b raw_w, sums[2] = ||dW||^2
 *   bad_ids : nullable device int32, set to 1 when an id was outside [0, V)
 *             (such tokens contribute nothing; the reference throws
 *             "layers: id out of range", which the C++ drop-in does after
 *             checking the host ids).
 * With fp64 rows dW and raw_w reproduce the reference's operation order bit
 * for bit.  Limit: T <= 16384 (one example's ids are sorted on chip).
 */
gnsb_status gnsb_embedding_pe_workspace_size(int64_t B, int64_t T, int64_t V, int64_t D, gnsb_dtype dt,
                                             size_t* bytes);
gnsb_status gnsb_embedding_pe(const int32_t* ids, const void* g, void* dW, double* raw_w, double* sums, int64_t B,
                              int64_t T, int64_t V, int64_t D, gnsb_dtype dt, void* ws, size_t ws_bytes,
                              int32_t* bad_ids, void* stream);

/* ------------------------------------------------------------------------
 * Deterministic fp64 squared norm of a device vector (fp32 or fp64 data):
 * out[0] = sum_i v[i]^2.  Used after the batch-sharded all-reduce, where
 * ||G_big||^2 must be formed from the REDUCED gradient.
 */
gnsb_status gnsb_sqnorm(const void* v, int64_t n, gnsb_dtype dt, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Batch-sharded exchange: the step's ONE collective.
 * No reference equivalent (the reference has no distributed runtime,
 * SPEC.md:9); the arithmetic after the sum is Trainer::step's packaging
 * (proj/src/trainer.cpp:363-378) with the global batch.
 *
 * widths2 : host [2 * n_layers]: (p0, p1) parameter widths per layer, e.g.
 *           (D, D) for a LayerNorm, (K*L, L) for a linear layer, (K*L, 0)
 *           for a bias-less one.  1..256 layers.
 * grads   : device bucket, layer after layer [p0 | p1], fp32 or fp64
 * records : device [n_layers][4] fp64 norm records as gnsb_ln_bwd /
 *           gnsb_linear_pe_norms / gnsb_embedding_pe write them
 *           {sum_b raw(p0), sum_b raw(p1), ||p0||^2, ||p1||^2}; NULL = gradients
 *           only (the plain backward's exchange)
 * ws      : device workspace of gnsb_exchange_workspace_size bytes (zeroed once;
 *           every call leaves it reusable)
 *
 * gnsb_allreduce_buckets = pack (records + gradients promoted to ONE fp64
 * buffer) -> one ncclAllReduce(sum) on `stream` over `nccl_comm` (an
 * ncclComm_t; NULL = a single rank: no collective) -> unpack: gradients back in
 * their dtype, records[l][0..1] summed, records[l][2..3] re-formed as the fp64
 * squared norms of the REDUCED gradients (local squared norms do not add).
 * Stream-ordered, no host synchronisation: capturable in a CUDA graph.  The GNS
 * step then uses the global batch (gnsb_gns_step with B = B_global).
 * gnsb_exchange_pack / _unpack are the two halves, for callers that run the
 * sum themselves (e.g. a torch.distributed process group).
 * libnccl.so.2 is opened at run time; the three helpers let a C/C++ caller
 * create a communicator with the same NCCL instance.
 */
int32_t gnsb_nccl_available(void);
gnsb_status gnsb_nccl_get_unique_id(void* id128);
gnsb_status gnsb_nccl_comm_init_rank(void** comm, int32_t nranks, const void* id128, int32_t rank);
gnsb_status gnsb_nccl_comm_destroy(void* comm);
gnsb_status gnsb_exchange_workspace_size(const int64_t* widths2, int32_t n_layers, size_t* bytes);
gnsb_status gnsb_exchange_pack(const void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                               const double* records, void* ws, size_t ws_bytes, void* stream);
gnsb_status gnsb_exchange_unpack(void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                                 double* records, void* ws, size_t ws_bytes, void* stream);
gnsb_status gnsb_allreduce_buckets(void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                                   double* records, void* ws, size_t ws_bytes, void* nccl_comm, void* stream);

/* ------------------------------------------------------------------------
 * GNS estimator (host functions).  Replace proj/include/gnstk/gns.hpp:16-74 /
 * proj/src/gns.cpp:14-89 with identical arithmetic and error conditions.
 */
typedef struct {
    double g_big_sqnorm;
    double g_small_sqnorm_mean;
    int64_t b_big;
    int64_t b_small;
    int64_t n_small;
} gnsb_grad_stats; /* gnstk::GradStats, gns.hpp:16-22 */

typedef struct {
    double g2;
    double s;
    double b_simple;
    int32_t b_simple_defined;
} gnsb_gns_estimate; /* gnstk::GnsEstimate, gns.hpp:26-31 */

typedef struct {
    double alpha;
    double value;
    int64_t count;
} gnsb_ema_state; /* gnstk::EmaState, gns.hpp:36-40 */

enum { GNSB_LAYER_EMBEDDING = 0, GNSB_LAYER_LINEAR = 1, GNSB_LAYER_LAYERNORM = 2 }; /* gns.hpp:42 */

gnsb_status gnsb_estimate_g2(const gnsb_grad_stats* st, double* out);          /* gns.cpp:31-36 */
gnsb_status gnsb_estimate_s(const gnsb_grad_stats* st, double* out);           /* gns.cpp:38-43 */
void gnsb_make_gns_estimate(double g2, double s, gnsb_gns_estimate* out);       /* gns.cpp:45-54 */
gnsb_status gnsb_ema_update(gnsb_ema_state* st, double x);                      /* gns.cpp:56-64 */
gnsb_status gnsb_smoothed_gns(const gnsb_ema_state* g2, const gnsb_ema_state* s,
                              gnsb_gns_estimate* out);                          /* gns.cpp:66-69 */
/* gns.cpp:71-89.  layers in gnstk::LayerKey order; group < 0 = no filter. */
gnsb_status gnsb_aggregate(const gnsb_grad_stats* stats, const int32_t* layer_types, int32_t n, int32_t group,
                           gnsb_grad_stats* out);

/* ------------------------------------------------------------------------
 * Device GNS accumulator (one step of the PerExample estimator).
 * Replaces the per-step GradStats packaging + fill_group of Trainer::step
 * (proj/src/trainer.cpp:324-325, 363-415) with a single-CTA kernel.
 *
 *   layer_sums  : device [n_layers][4] fp64 records, one per layer, in
 *                 LayerKey order: { sum_b raw(p0), sum_b raw(p1),
 *                 ||grad p0||^2, ||grad p1||^2 } exactly as gnsb_ln_bwd's
 *                 `sums` (p0 = gamma, p1 = beta; for a linear layer p0 =
 *                 weight, p1 = bias or zeros).  Parameters are summed in the
 *                 reference's name order (p1 first: "beta" < "gamma",
 *                 "bias" < "weight").
 *   layer_types : HOST [n_layers] GNSB_LAYER_*
 *   B           : global batch (b_big = B, b_small = 1, n_small = B)
 *   state       : device [8] gnsb_ema_state for groups {total, embedding,
 *                 linear, layernorm} x {g2, s}; zero-filled before the first
 *                 step (count = 0).  `alpha` is applied to every state.
 *   out_groups  : device [4][4] fp64 {g2_raw, s_raw, gns_ema, defined(0/1)};
 *                 a group with no layers is skipped (all NaN, state untouched).
 *   out_layers  : device [n_layers][2] fp64 {g2, s} per layer (nullable).
 * Errors: B < 2 (trainer.cpp:291-292), alpha outside (0, 1].
 */
gnsb_status gnsb_gns_step(const double* layer_sums, const int32_t* layer_types, int32_t n_layers, int64_t B,
                          double alpha, gnsb_ema_state* state, double* out_groups, double* out_layers,
                          void* stream);

/* ------------------------------------------------------------------------
 * Cost model / dispatch rule.  Replaces proj/include/gnstk/costmodel.hpp:33-47
 * (proj/src/costmodel.cpp:25-64).  method 0 = simultaneous (weight-grad form),
 * 1 = frobenius (Gram form); criterion 0 = IO, 1 = FLOPS.  out[2] =
 * {weight_grad, grad_norms}.
 */
gnsb_status gnsb_flops(int64_t b, int64_t t, int64_t k, int64_t l, int32_t method, int64_t* out);
gnsb_status gnsb_io_values(int64_t b, int64_t t, int64_t k, int64_t l, int32_t method, int64_t* out);
gnsb_status gnsb_crossover_t(int64_t k, int64_t l, int32_t criterion, double* out);

/* ------------------------------------------------------------------------
 * Synthetic workload generators (SURVEY.md §8(d) recipes), bit-identical
 * with the CPU oracle's.  Fill device buffers of dtype dt (gamma/beta as the
 * statistics dtype).  Any pointer may be NULL.
 *   LN:     x = Z(s0,idx) + 0.5 Z(s0+1,row); dy = (Z(s0+2,t*D+d) + sigma Z(s0+3,idx)) / B_div;
 *           gamma = 1 + 0.1 Z(s0+4,d); beta = 0.1 Z(s0+5,d)
 *   linear: x = Z(s0,idx); dy = (Z(s0+1,t*L+l) + Z(s0+2,idx)) / (B_div*sqrt(T))
 * idx/row use the GLOBAL example index b + b_offset (batch sharding).
 */
gnsb_status gnsb_synth_ln(void* x, void* dy, void* gamma, void* beta, int64_t B, int64_t T, int64_t D,
                          int64_t b_offset, int64_t B_div, float sigma, uint64_t stream0, gnsb_dtype dt, void* stream);
gnsb_status gnsb_synth_linear(void* x, void* dy, int64_t B, int64_t T, int64_t K, int64_t L, int64_t b_offset,
                              int64_t B_div, uint64_t stream0, gnsb_dtype dt, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GNSB_H */

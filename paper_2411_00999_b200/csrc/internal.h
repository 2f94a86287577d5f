// internal.h — launcher declarations shared between the kernel translation
// units and the C-ABI layer (capi.cu).  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

namespace gnsb {

struct SynthSeeds {
    uint64_t s[8];  // mix_seed(2411, stream0 + k), k = 0..7
};

cudaError_t launch_synth_ln(int dt, void* x, void* dy, void* gamma, void* beta, int64_t B, int64_t T, int64_t D,
                            int64_t b_off, float bdiv, float sigma, SynthSeeds s, cudaStream_t st);
cudaError_t launch_synth_linear(int dt, void* x, void* dy, int64_t B, int64_t T, int64_t K, int64_t L, int64_t b_off,
                                float scale, SynthSeeds s, cudaStream_t st);

// LayerNorm forward / backward (ln_launch.cuh, instantiated per dtype)
struct LnFwdCall {
    const void* x; const void* gamma; const void* beta;
    void* y; void* mean; void* rstd; void* xhat;
    int64_t N, D; double eps;
};
struct LnBwdCall {
    const void* x; const void* mean; const void* rstd; const void* dy; const void* gamma;
    void* dx; void* dgamma; void* dbeta;
    double* raw_g; double* raw_b; double* sums;
    int norms;
    int64_t B, M, D;
    void* ws; size_t ws_bytes;
    unsigned long long* trace = nullptr;   // profiling only: row kernel [grid][6] phase stamps
    unsigned long long* trace2 = nullptr;  // profiling only: reduce kernel [grid][6] phase stamps
};

// Where a row pass left its partial slots and how the reduce must read them.
struct LnRedPlanInfo {
    int Dp = 0, G = 0, grid_rows = 0;
    int gsub = 1;  // slots per (cta + example) stage 2 sums: 1 (folded) or G (one per row group)
    size_t off_partial = 0, off_q = 0, off_qbig = 0, off_raw = 0, total = 0;
};
// One LayerNorm whose stage 2 (per-example combine, squares, dgamma/dbeta) is pending.
struct LnRedItem {
    LnRedPlanInfo info;
    int64_t B, M, D;
    void* ws;
    void* dgamma; void* dbeta;
    double* raw_g; double* raw_b; double* sums;
};

// Returns 0 ok, 1 invalid (message in *why), 2 CUDA error (cudaError_t in *cerr).
// Row pass only (the stage-2 inputs stay in ws); plan info of that pass.
template <typename T> int ln_bwd_rows_run(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr);
template <typename T> int ln_bwd_plan_info(int64_t B, int64_t M, int64_t D, LnRedPlanInfo* out, const char** why);
// Stage 2 of n pending LayerNorms in one launch (ln_reduce.cu).  acc_f64: the
// statistics dtype is fp64 (fp64 rows), else fp32.
int ln_bwd_reduce_run(int acc_f64, int norms, const LnRedItem* items, int n, cudaStream_t st,
                      unsigned long long* trace, const char** why, cudaError_t* cerr);
template <typename T> int ln_fwd_run(const LnFwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr);
template <typename T> int ln_bwd_run(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr);
template <typename T> int ln_bwd_workspace(int64_t B, int64_t M, int64_t D, size_t* bytes, const char** why);
// launch geometry actually used (for reporting): grid, threads, stages
template <typename T> int ln_bwd_geometry(int64_t B, int64_t M, int64_t D, int* grid, int* threads, int* stages);

int device_sm_count();
// the calling thread's gnsb_last_error() message (capi.cu)
void set_error(const std::string& msg);
// raise (never lower) a kernel's max dynamic shared memory attribute; process-wide record
cudaError_t ensure_smem_attr(const void* kernel, size_t bytes);

// linear-layer per-example norms (linear_pe.cu)
bool wgrad_shape_ok(int64_t B, int64_t T, int64_t K, int64_t L);
size_t wgrad_workspace(int64_t B, int64_t K, int64_t L);
cudaError_t launch_wgrad_norms(const void* x, const void* g, float* dW, double* raw, double* sums, int64_t B,
                               int64_t T, int64_t K, int64_t L, void* ws, cudaStream_t st);
size_t generic_workspace(int64_t B, int64_t T, int64_t K, int64_t L);
size_t generic_workspace_f64(int64_t B, int64_t T, int64_t K, int64_t L);
// bias gradient + per-example norms as an HBM stream (fp32 / bf16 rows, L % 8 == 0)
bool bias_fast_ok(int dt, int64_t L, const void* g, const void* dbias);
size_t bias_fast_workspace(int64_t B, int64_t T, int64_t L);
cudaError_t launch_bias_fast(int dt, const void* g, void* dbias, double* raw, double* sums, int64_t B, int64_t T,
                             int64_t L, void* ws, cudaStream_t st);
// kind 0: weight (simultaneous form), 1: bias, 2: Gram form (norms only)
cudaError_t launch_linear_generic(int dt, int kind, const void* x, const void* g, void* out_grad, int out_f64,
                                  double* raw, double* sums, int sum_slot, int64_t B, int64_t T, int64_t K, int64_t L,
                                  void* ws, cudaStream_t st);
// Gram form on tensor cores (linear_gram.cu): bf16 rows, T % 128 == 0, K % 64 == 0, L % 64 == 0
bool gram_shape_ok(int64_t B, int64_t T, int64_t K, int64_t L);
size_t gram_workspace(int64_t B, int64_t T);
cudaError_t launch_gram_norms(const void* x, const void* g, double* raw, double* sums, int64_t B, int64_t T,
                              int64_t K, int64_t L, void* ws, cudaStream_t st);
// raw[b] = sum_j q[b][j], sums[sum_slot] = sum_b raw[b] (fixed order, one CTA)
cudaError_t launch_fold_rows(const double* q, int nb, int ncol, double* raw, double* sums, int sum_slot,
                             cudaStream_t st);
// embedding table gradient + per-example norms (embedding_pe.cu); T <= 16384
bool embedding_shape_ok(int64_t T);
size_t embedding_workspace(int64_t B, int64_t T, int64_t V, int64_t D, int dt);
cudaError_t launch_embedding_pe(int dt, const int32_t* ids, const void* g, void* dW, double* raw, double* sums,
                                int64_t B, int64_t T, int64_t V, int64_t D, void* ws, int32_t* bad, cudaStream_t st);
cudaError_t launch_embedding_fwd(int dt, const int32_t* ids, const void* W, void* out, int64_t n, int64_t V, int64_t D,
                                 int32_t* bad, cudaStream_t st);
// linear-layer GEMMs (linear_gemm.cu): kind 0 forward y = x W + bias, kind 1 dx = g W^T
bool gemm_tc_ok(int dt, int64_t K, int64_t L);
size_t gemm_workspace(int dt, int w_dt, int64_t K, int64_t L);
cudaError_t launch_linear_gemm(int kind, int epi, int dt, int w_dt, const void* in, const void* W, const void* bias,
                               const void* aux, void* out, int64_t rows, int64_t K, int64_t L, void* ws,
                               cudaStream_t st);
// stream-ordered scratch from the library-owned pool (linear_gemm.cu)
cudaError_t gemm_pool_alloc(void** p, size_t bytes, cudaStream_t st);
cudaError_t gemm_pool_free(void* p, cudaStream_t st);
// fp32 rows: per-example weight-gradient norms on the 3xTF32 GEMM (linear_f32.cu)
bool wgrad_tf32_ok(int dt, const void* x, const void* g, const void* dW, int64_t T, int64_t K, int64_t L);
cudaError_t launch_wgrad_tf32(const float* x, const float* g, float* dW, double* raw, double* sums, int sum_slot,
                              int64_t B, int64_t T, int64_t K, int64_t L, cudaStream_t st);
// fp64 rows: per-example parameter gradients / norms in the reference's order (ln_ref.cu)
size_t ln_ref_workspace(int64_t B, int64_t D);
cudaError_t launch_ln_ref_params(const double* x, const double* mean, const double* rstd, const double* g, int64_t B,
                                 int64_t M, int64_t D, double* dgamma, double* dbeta, double* raw_g, double* raw_b,
                                 double* sums, void* scratch, cudaStream_t st);
cudaError_t launch_seq_sqnorm(const double* pe, int64_t B, int64_t n, double* raw, double* sums, int sum_slot,
                              cudaStream_t st);
// softmax cross-entropy rows (xent.cu): loss_rows[r] = log(sum exp) + max - logit[target],
// dlogits = (softmax - onehot) * upstream_scale
cudaError_t launch_xent(int dt, const void* logits, const int32_t* targets, void* dlogits, double* loss_rows,
                        int64_t rows, int64_t V, double upstream_scale, int32_t* bad, cudaStream_t st);

}  // namespace gnsb

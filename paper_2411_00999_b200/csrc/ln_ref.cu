// ln_ref.cu — the fp64 rows' per-example parameter gradients and norms in the
// reference's exact operation order (the C++ drop-in's GNSB_F64 path).
//
// proj/src/layers.cpp:248-268 (LayerNorm) and :107-131 (linear) accumulate
// per example, sequentially, without fused multiply-adds:
//   gamma'_b[i] = ((0 + xh_0 g_0) + xh_1 g_1) + ...   over the example's rows
//   raw_b       = ((0 + p_0^2) + p_1^2) + ...          over the parameter (row_sqnorm)
//   dgamma[i]   = ((0 + gamma'_0[i]) + gamma'_1[i]) + ... over examples
// The batched kernels sum the same quantities over CTA partitions, which is
// deterministic but depends on the batch: a B = 1 call on one example does not
// reproduce that example's share of a batched call bit for bit.  The
// reference's trainer tests rely on exactly that identity (PerExample vs
// Microbatch(m = B) logs, proj/tests/test_trainer.cpp:123-130), so the fp64
// path recomputes these small quantities in the reference's order here.
// Parallelism: one thread per (example, parameter entry) for the row sums
// (coalesced across entries), one thread per example for its norm, one per
// entry for the batch sum.  fp64 only; the dx rows keep the row kernel (a row's
// dx does not depend on the batch).
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace gnsb {

namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// per (b, i): gamma'_b[i], beta'_b[i] over the example's M rows in order
__global__ void __launch_bounds__(256) ln_ref_rows_kernel(const double* x, const double* mean, const double* rstd,
                                                          const double* g, int64_t B, int64_t M, int64_t D,
                                                          double* grow, double* brow) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * D) return;
    const int64_t b = idx / D, i = idx - b * D;
    double gs = 0.0, bs = 0.0;
    for (int64_t m = 0; m < M; ++m) {
        const int64_t r = b * M + m;
        const double gv = g[r * D + i];
        const double xv = x[r * D + i];
        const double xh = mean ? mul(add(xv, -mean[r]), rstd[r]) : xv;
        gs = add(gs, mul(xh, gv));
        bs = add(bs, gv);
    }
    grow[idx] = gs;
    brow[idx] = bs;
}

// threads [0, B): raw_b of the example's rows (row_sqnorm order); threads
// [B, B + D): the parameter entry summed over examples in order
__global__ void __launch_bounds__(256) ln_ref_fold_kernel(const double* grow, const double* brow, int64_t B,
                                                          int64_t D, double* raw_g, double* raw_b, double* dgamma,
                                                          double* dbeta) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < B) {
        double sg = 0.0, sb = 0.0;
        for (int64_t i = 0; i < D; ++i) {
            sg = add(sg, mul(grow[t * D + i], grow[t * D + i]));
            sb = add(sb, mul(brow[t * D + i], brow[t * D + i]));
        }
        raw_g[t] = sg;
        raw_b[t] = sb;
    } else if (t < B + D) {
        const int64_t i = t - B;
        double sg = 0.0, sb = 0.0;
        for (int64_t b = 0; b < B; ++b) {
            sg = add(sg, grow[b * D + i]);
            sb = add(sb, brow[b * D + i]);
        }
        dgamma[i] = sg;
        dbeta[i] = sb;
    }
}

// sums = {sum_b raw_g, sum_b raw_b, ||dgamma||^2, ||dbeta||^2}, sequential
__global__ void ln_ref_sums_kernel(const double* raw_g, const double* raw_b, const double* dgamma,
                                   const double* dbeta, int64_t B, int64_t D, double* sums) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t b = 0; b < B; ++b) {
        s[0] = add(s[0], raw_g[b]);
        s[1] = add(s[1], raw_b[b]);
    }
    for (int64_t i = 0; i < D; ++i) {
        s[2] = add(s[2], mul(dgamma[i], dgamma[i]));
        s[3] = add(s[3], mul(dbeta[i], dbeta[i]));
    }
    for (int k = 0; k < 4; ++k) sums[k] = s[k];
}

// raw[b] = row_sqnorm of the example's n parameter entries pe[b][0..n)
__global__ void __launch_bounds__(128) seq_sqnorm_kernel(const double* pe, int64_t B, int64_t n, double* raw) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = add(s, mul(pe[b * n + i], pe[b * n + i]));
    raw[b] = s;
}

__global__ void seq_sum_kernel(const double* v, int64_t n, double* out) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = add(s, v[i]);
    *out = s;
}

}  // namespace

size_t ln_ref_workspace(int64_t B, int64_t D) { return (size_t)(2 * B * D + 2 * B) * sizeof(double); }

cudaError_t launch_ln_ref_params(const double* x, const double* mean, const double* rstd, const double* g, int64_t B,
                                 int64_t M, int64_t D, double* dgamma, double* dbeta, double* raw_g, double* raw_b,
                                 double* sums, void* scratch, cudaStream_t st) {
    double* grow = static_cast<double*>(scratch);
    double* brow = grow + B * D;
    if (raw_g == nullptr) raw_g = brow + B * D;  // (the norms feed `sums` even when not returned)
    if (raw_b == nullptr) raw_b = brow + B * D + B;
    const int64_t n = B * D;
    ln_ref_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, mean, rstd, g, B, M, D, grow, brow);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ln_ref_fold_kernel<<<(unsigned)((B + D + 255) / 256), 256, 0, st>>>(grow, brow, B, D, raw_g, raw_b, dgamma, dbeta);
    e = cudaGetLastError();
    if (e != cudaSuccess || sums == nullptr) return e;
    ln_ref_sums_kernel<<<1, 1, 0, st>>>(raw_g, raw_b, dgamma, dbeta, B, D, sums);
    return cudaGetLastError();
}

cudaError_t launch_seq_sqnorm(const double* pe, int64_t B, int64_t n, double* raw, double* sums, int sum_slot,
                              cudaStream_t st) {
    seq_sqnorm_kernel<<<(unsigned)((B + 127) / 128), 128, 0, st>>>(pe, B, n, raw);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || sums == nullptr) return e;
    seq_sum_kernel<<<1, 1, 0, st>>>(raw, B, sums + sum_slot);
    return cudaGetLastError();
}

}  // namespace gnsb

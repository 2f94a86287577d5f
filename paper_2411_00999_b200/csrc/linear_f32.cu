// linear_f32.cu — per-example weight-gradient norms for fp32 rows on the
// tensor cores (the weight-gradient form of proj/src/layers.cpp:80-157 and the
// quantity of the Gram form, layers.cpp:159-187, ||X_b^T G_b||_F^2).
//
// kind::tf32 MMAs take K-major operands only, and here the contraction runs
// over the tokens, which are the strided axis of both x [B][T][K] and
// g [B][T][L].  So:
//   1. transpose_bt_kernel writes x_b^T [K][T] and g_b^T [L][T] per example
//      (32 x 32 tiles through shared memory, coalesced on both sides);
//   2. per example, dW_b = x_b^T (g_b^T)^T on the 3xTF32 GEMM of
//      linear_gemm.cu (operands split into tf32 hi / lo, fp32 accumulation in
//      TMEM: the "dx = g W^T" form with rows = K, N = L, reduced axis = T);
//   3. wgrad_acc_kernel streams dW_b once: the fp64 sum of its squares per
//      CTA -> q[b][cta], and dW = dW + dW_b in example order (fp32; the first
//      example stores), the last example also leaves ||dW||^2 per CTA;
//   4. fold_rows_kernel turns q into raw_b and the scalar sums (fixed order).
// No atomics: bitwise deterministic run to run.  The generic kernels (fp64
// accumulation, one thread per weight entry, every token in sequence) stay
// for unaligned shapes (T or L not a multiple of 4) and fp64 rows.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace gnsb {

namespace {

constexpr int kAccThreads = 256;

// [B][T][C] -> [B][C][T]
__global__ void __launch_bounds__(256) transpose_bt_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                           int64_t T, int64_t C) {
    __shared__ float tile[32][33];
    const int64_t b = blockIdx.z;
    const int64_t c0 = (int64_t)blockIdx.x * 32, t0 = (int64_t)blockIdx.y * 32;
    const float* src = in + b * T * C;
    float* dst = out + b * C * T;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
        const int64_t t = t0 + i, c = c0 + tx;
        tile[i][tx] = (t < T && c < C) ? __ldg(src + t * C + c) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
        const int64_t c = c0 + i, t = t0 + tx;
        if (c < C && t < T) dst[c * T + t] = tile[tx][i];
    }
}

// q_row[cta] = sum of dWb^2 over the CTA's entries (fp64, fixed order);
// dW = first ? dWb : dW + dWb; qbig_row (last example only) = the CTA's share
// of ||dW||^2.  n % 4 == 0 (L % 4 == 0).
__global__ void __launch_bounds__(kAccThreads) wgrad_acc_kernel(const float* __restrict__ dWb, float* dW, int64_t n,
                                                                int first, double* q_row, double* qbig_row) {
    __shared__ double red[2][kAccThreads];
    double s = 0.0, s2 = 0.0;
    const int64_t n4 = n / 4;
    for (int64_t i = (int64_t)blockIdx.x * kAccThreads + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kAccThreads) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(dWb) + i);
        s = fma((double)v.x, (double)v.x, s);
        s = fma((double)v.y, (double)v.y, s);
        s = fma((double)v.z, (double)v.z, s);
        s = fma((double)v.w, (double)v.w, s);
        if (dW) {
            float4 o = v;
            if (!first) {
                const float4 a = reinterpret_cast<const float4*>(dW)[i];
                o = make_float4(a.x + v.x, a.y + v.y, a.z + v.z, a.w + v.w);
            }
            reinterpret_cast<float4*>(dW)[i] = o;
            if (qbig_row) {
                s2 = fma((double)o.x, (double)o.x, s2);
                s2 = fma((double)o.y, (double)o.y, s2);
                s2 = fma((double)o.z, (double)o.z, s2);
                s2 = fma((double)o.w, (double)o.w, s2);
            }
        }
    }
    red[0][threadIdx.x] = s;
    red[1][threadIdx.x] = s2;
    __syncthreads();
    for (int o = kAccThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        q_row[blockIdx.x] = red[0][0];
        if (qbig_row) qbig_row[blockIdx.x] = red[1][0];
    }
}

}  // namespace

bool wgrad_tf32_ok(int dt, const void* x, const void* g, const void* dW, int64_t T, int64_t K, int64_t L) {
    static const bool off = std::getenv("GNSB_LINEAR_F32_GENERIC") != nullptr;  // A/B: the generic kernels
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    return !off && dt == 0 && T % 4 == 0 && L % 4 == 0 && T > 0 && K > 0 && T < (1ll << 31) && K < (1ll << 31) &&
           L < (1ll << 31) && al16(x) && al16(g) && (dW == nullptr || al16(dW));
}

cudaError_t launch_wgrad_tf32(const float* x, const float* g, float* dW, double* raw, double* sums, int sum_slot,
                              int64_t B, int64_t T, int64_t K, int64_t L, cudaStream_t st) {
    const int nblk = device_sm_count() * 4;
    const size_t xt = (size_t)B * K * T, gt = (size_t)B * L * T, wb = (size_t)K * L;
    const size_t bytes = (xt + gt + wb) * sizeof(float) + (size_t)(B + 1) * nblk * sizeof(double) + 256;
    void* scratch = nullptr;
    cudaError_t e = gemm_pool_alloc(&scratch, bytes, st);
    if (e != cudaSuccess) return e;
    float* Xt = static_cast<float*>(scratch);
    float* Gt = Xt + xt;
    float* dWb = Gt + gt;
    double* q = reinterpret_cast<double*>(dWb + wb);
    transpose_bt_kernel<<<dim3((unsigned)((K + 31) / 32), (unsigned)((T + 31) / 32), (unsigned)B), 256, 0, st>>>(x, Xt,
                                                                                                           T, K);
    transpose_bt_kernel<<<dim3((unsigned)((L + 31) / 32), (unsigned)((T + 31) / 32), (unsigned)B), 256, 0, st>>>(g, Gt,
                                                                                                           T, L);
    e = cudaGetLastError();
    for (int64_t b = 0; b < B && e == cudaSuccess; ++b) {
        // dW_b [K, L] = Xt_b [K, T] . Gt_b [L, T]^T  (the dx form: rows = K, W = Gt_b as [L, T])
        e = launch_linear_gemm(1, 0, 0, 0, Xt + (size_t)b * K * T, Gt + (size_t)b * L * T, nullptr, nullptr, dWb, K, L,
                               T, nullptr, st);
        if (e != cudaSuccess) break;
        wgrad_acc_kernel<<<nblk, kAccThreads, 0, st>>>(dWb, dW, K * L, b == 0, q + (size_t)b * nblk,
                                                       (dW && b == B - 1) ? q + (size_t)B * nblk : nullptr);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = launch_fold_rows(q, (int)B, nblk, raw, sums, sum_slot, st);
    if (e == cudaSuccess && sums && dW) e = launch_fold_rows(q + (size_t)B * nblk, 1, nblk, nullptr, sums, sum_slot + 2, st);
    const cudaError_t f = gemm_pool_free(scratch, st);
    return e != cudaSuccess ? e : f;
}

}  // namespace gnsb

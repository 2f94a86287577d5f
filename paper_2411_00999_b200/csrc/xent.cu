// xent.cu — softmax cross-entropy forward + backward of the toy model's head
// in one kernel (proj/src/model.cpp:113-141, `cross_entropy` with dlogits):
//   per row r: m = max_c l[c]; denom = sum_c exp(l[c] - m);
//   loss_rows[r] = log(denom) + m - l[target];
//   dlogits[r, c] = (exp(l[c] - m) / denom - [c == target]) * upstream_scale.
// One CTA per row: pass 1 is an online (max, sum) over the row, a fixed-order
// tree across the CTA; pass 2 re-reads the row (L2-resident) and writes
// dlogits.  The per-example mean over tokens and the sum over examples
// (model.cpp:137) are O(B*T) host-side scalars.  fp64 rows keep exp/log in
// fp64; fp32 / bf16 rows use fp32 exponentials with fp64 sums.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace gnsb {

namespace {
constexpr int kXentThreads = 256;

template <typename T> struct XentMath;
template <> struct XentMath<double> {
    static __device__ __forceinline__ double ex(double v) { return exp(v); }
};
template <> struct XentMath<float> {
    static __device__ __forceinline__ float ex(float v) { return __expf(v); }
};

// (m, s) pairs: s is the sum of exp(l - m)
__device__ __forceinline__ void combine(double& m, double& s, double m2, double s2) {
    if (m2 > m) {
        s = s * exp(m - m2) + s2;
        m = m2;
    } else if (m2 != -INFINITY) {
        s = s + s2 * exp(m2 - m);
    }
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(kXentThreads) xent_kernel(const T* __restrict__ logits, const int32_t* __restrict__ targets,
                                                          T* __restrict__ dlogits, double* __restrict__ loss_rows,
                                                          int64_t V, double scale, int32_t* bad) {
    using A = typename Traits<T>::Acc;
    using M = XentMath<A>;
    const int64_t r = blockIdx.x;
    const T* l = logits + r * V;
    __shared__ double sm[kXentThreads], ss[kXentThreads];
    // pass 1: per-thread online max/sum in fixed column order
    A m = -INFINITY;
    double s = 0.0;
    for (int64_t c = threadIdx.x; c < V; c += kXentThreads) {
        const A v = to_acc<T>(l[c]);
        if (v > m) {
            s = s * (double)M::ex(m - v) + 1.0;
            m = v;
        } else {
            s += (double)M::ex(v - m);
        }
    }
    sm[threadIdx.x] = (double)m;
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int o = kXentThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            double mm = sm[threadIdx.x], s0 = ss[threadIdx.x];
            combine(mm, s0, sm[threadIdx.x + o], ss[threadIdx.x + o]);
            sm[threadIdx.x] = mm;
            ss[threadIdx.x] = s0;
        }
        __syncthreads();
    }
    const double mx = sm[0], denom = ss[0];
    const int32_t tgt = targets[r];
    const bool ok = tgt >= 0 && tgt < V;
    if (threadIdx.x == 0) {
        if (!ok && bad) *bad = 1;
        loss_rows[r] = ok ? log(denom) + mx - (double)to_acc<T>(l[tgt]) : (double)NAN;
    }
    if (dlogits == nullptr) return;
    // pass 2: dlogits
    const A amx = (A)mx;
    const A inv = (A)(1.0 / denom);
    T* d = dlogits + r * V;
    for (int64_t c = threadIdx.x; c < V; c += kXentThreads) {
        const A p = M::ex(to_acc<T>(l[c]) - amx) * inv;
        const A one = c == tgt ? A(1) : A(0);
        d[c] = from_acc<T>((A)(((double)p - (double)one) * scale));
    }
}

cudaError_t launch_xent(int dt, const void* logits, const int32_t* targets, void* dlogits, double* loss_rows,
                        int64_t rows, int64_t V, double upstream_scale, int32_t* bad, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    if (bad) {
        cudaError_t e = cudaMemsetAsync(bad, 0, 4, st);
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)rows;
    switch (dt) {
        case 0:
            xent_kernel<float><<<grid, kXentThreads, 0, st>>>((const float*)logits, targets, (float*)dlogits, loss_rows,
                                                              V, upstream_scale, bad);
            break;
        case 1:
            xent_kernel<__nv_bfloat16><<<grid, kXentThreads, 0, st>>>((const __nv_bfloat16*)logits, targets,
                                                                      (__nv_bfloat16*)dlogits, loss_rows, V,
                                                                      upstream_scale, bad);
            break;
        case 2:
            xent_kernel<double><<<grid, kXentThreads, 0, st>>>((const double*)logits, targets, (double*)dlogits,
                                                               loss_rows, V, upstream_scale, bad);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gnsb

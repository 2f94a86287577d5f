// synth.cu — on-device synthetic workload generator.
//
// Bit-identical with the host generator in oracle/oracle.c (orc_synth_*):
// a counter-based splitmix64 hash per element, then a fixed sequence of
// single-rounding fp32 operations (explicit _rn intrinsics, no contraction).
// Used by bench.py and the GPU tests to materialise multi-GB inputs in HBM
// without shipping them over PCIe; the oracle regenerates the same values.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace gnsb {

__device__ __forceinline__ float synth_z(uint64_t seed, uint64_t i) {
    uint64_t z = seed + i + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const float u = (float)(z >> 40) * 0x1.0p-24f;
    return __fmul_rn(__fsub_rn(u, 0.5f), 3.4641016151377544f);
}

template <typename T>
__device__ __forceinline__ void store_val(T* p, float v);
template <> __device__ __forceinline__ void store_val<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void store_val<double>(double* p, float v) { *p = (double)v; }
template <> __device__ __forceinline__ void store_val<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

template <typename T, typename P>
__global__ void synth_ln_kernel(T* x, T* dy, P* gamma, P* beta, int64_t B, int64_t T_, int64_t D, int64_t b_off,
                                float bdiv, float sigma, SynthSeeds s, int round_bf16) {
    const int64_t n = B * T_ * D;
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < n; li += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = li % D;
        const int64_t bt = li / D;
        const int64_t t = bt % T_, b = bt / T_;
        const int64_t grow = (b + b_off) * T_ + t;
        const uint64_t gidx = (uint64_t)(grow * D + d);
        float xv = __fadd_rn(synth_z(s.s[0], gidx), __fmul_rn(0.5f, synth_z(s.s[1], (uint64_t)grow)));
        const float noise = __fmul_rn(sigma, synth_z(s.s[3], gidx));
        float gv = __fdiv_rn(__fadd_rn(synth_z(s.s[2], (uint64_t)(t * D + d)), noise), bdiv);
        if (round_bf16) {
            xv = __bfloat162float(__float2bfloat16_rn(xv));
            gv = __bfloat162float(__float2bfloat16_rn(gv));
        }
        if (x) store_val<T>(x + li, xv);
        if (dy) store_val<T>(dy + li, gv);
        if (li < D) {
            if (gamma) gamma[li] = (P)__fadd_rn(1.0f, __fmul_rn(0.1f, synth_z(s.s[4], (uint64_t)li)));
            if (beta) beta[li] = (P)__fmul_rn(0.1f, synth_z(s.s[5], (uint64_t)li));
        }
    }
}

template <typename T>
__global__ void synth_linear_kernel(T* x, T* dy, int64_t B, int64_t T_, int64_t K, int64_t L, int64_t b_off,
                                    float scale, SynthSeeds s) {
    const int64_t nx = B * T_ * K, ny = B * T_ * L;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < nx + ny; li += stride) {
        if (li < nx) {
            if (!x) continue;
            const int64_t k = li % K, bt = li / K;
            const int64_t t = bt % T_, b = bt / T_;
            const int64_t grow = (b + b_off) * T_ + t;
            store_val<T>(x + li, synth_z(s.s[0], (uint64_t)(grow * K + k)));
        } else {
            if (!dy) continue;
            const int64_t lj = li - nx;
            const int64_t l = lj % L, bt = lj / L;
            const int64_t t = bt % T_, b = bt / T_;
            const int64_t grow = (b + b_off) * T_ + t;
            const float a = synth_z(s.s[1], (uint64_t)(t * L + l));
            const float c = synth_z(s.s[2], (uint64_t)(grow * L + l));
            store_val<T>(dy + lj, __fdiv_rn(__fadd_rn(a, c), scale));
        }
    }
}

static int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_synth_ln(int dt, void* x, void* dy, void* gamma, void* beta, int64_t B, int64_t T_, int64_t D,
                            int64_t b_off, float bdiv, float sigma, SynthSeeds s, cudaStream_t st) {
    const int grid = grid_for(B * T_ * D > D ? B * T_ * D : D);
    switch (dt) {
        case 0:
            synth_ln_kernel<float, float><<<grid, 256, 0, st>>>((float*)x, (float*)dy, (float*)gamma, (float*)beta, B,
                                                                T_, D, b_off, bdiv, sigma, s, 0);
            break;
        case 1:
            synth_ln_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>((__nv_bfloat16*)x, (__nv_bfloat16*)dy,
                                                                        (float*)gamma, (float*)beta, B, T_, D, b_off,
                                                                        bdiv, sigma, s, 1);
            break;
        case 2:
            synth_ln_kernel<double, double><<<grid, 256, 0, st>>>((double*)x, (double*)dy, (double*)gamma,
                                                                  (double*)beta, B, T_, D, b_off, bdiv, sigma, s, 0);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_synth_linear(int dt, void* x, void* dy, int64_t B, int64_t T_, int64_t K, int64_t L, int64_t b_off,
                                float scale, SynthSeeds s, cudaStream_t st) {
    const int grid = grid_for(B * T_ * (K + L));
    switch (dt) {
        case 0: synth_linear_kernel<float><<<grid, 256, 0, st>>>((float*)x, (float*)dy, B, T_, K, L, b_off, scale, s); break;
        case 1:
            synth_linear_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((__nv_bfloat16*)x, (__nv_bfloat16*)dy, B, T_, K,
                                                                     L, b_off, scale, s);
            break;
        case 2:
            synth_linear_kernel<double><<<grid, 256, 0, st>>>((double*)x, (double*)dy, B, T_, K, L, b_off, scale, s);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gnsb

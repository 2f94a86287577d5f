// common.cuh — dtype traits and sm_100a PTX helpers shared by the kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace gnsb {

// ---------------------------------------------------------------- dtypes --
// T: storage type of row data (x, dy, dx).  Acc: arithmetic type of the row
// math and of mean/rstd/gamma/dgamma/dbeta (fp32 for fp32/bf16 rows, fp64 for
// fp64 rows).  W: elements per 16-byte vector.
template <typename T> struct Traits;
template <> struct Traits<float> {
    using Acc = float;
    static constexpr int W = 4;
};
template <> struct Traits<__nv_bfloat16> {
    using Acc = float;
    static constexpr int W = 8;
};
template <> struct Traits<double> {
    using Acc = double;
    static constexpr int W = 2;
};

// 16-byte vector <-> W Acc values
template <typename T>
__device__ __forceinline__ void unpack(const uint4& v, typename Traits<T>::Acc* out);
template <>
__device__ __forceinline__ void unpack<float>(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x << 16); o[1] = __uint_as_float(v.x & 0xffff0000u);
    o[2] = __uint_as_float(v.y << 16); o[3] = __uint_as_float(v.y & 0xffff0000u);
    o[4] = __uint_as_float(v.z << 16); o[5] = __uint_as_float(v.z & 0xffff0000u);
    o[6] = __uint_as_float(v.w << 16); o[7] = __uint_as_float(v.w & 0xffff0000u);
}
template <>
__device__ __forceinline__ void unpack<double>(const uint4& v, double* o) {
    o[0] = __hiloint2double((int)v.y, (int)v.x);
    o[1] = __hiloint2double((int)v.w, (int)v.z);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <typename T>
__device__ __forceinline__ uint4 pack(const typename Traits<T>::Acc* in);
template <>
__device__ __forceinline__ uint4 pack<float>(const float* i) {
    return make_uint4(__float_as_uint(i[0]), __float_as_uint(i[1]), __float_as_uint(i[2]), __float_as_uint(i[3]));
}
template <>
__device__ __forceinline__ uint4 pack<__nv_bfloat16>(const float* i) {
    return make_uint4(pack_bf16x2(i[0], i[1]), pack_bf16x2(i[2], i[3]), pack_bf16x2(i[4], i[5]),
                      pack_bf16x2(i[6], i[7]));
}
template <>
__device__ __forceinline__ uint4 pack<double>(const double* i) {
    return make_uint4((uint32_t)__double2loint(i[0]), (uint32_t)__double2hiint(i[0]),
                      (uint32_t)__double2loint(i[1]), (uint32_t)__double2hiint(i[1]));
}

template <typename T> __device__ __forceinline__ typename Traits<T>::Acc to_acc(T v);
template <> __device__ __forceinline__ float to_acc<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ double to_acc<double>(double v) { return v; }

template <typename T> __device__ __forceinline__ T from_acc(typename Traits<T>::Acc v);
template <> __device__ __forceinline__ float from_acc<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ double from_acc<double>(double v) { return v; }

// ------------------------------------------------------------ pairs ------
// Row math runs on element pairs: fp32 pairs map to the sm_100 packed
// FFMA2 / FADD2 / FMUL2 instructions (two lanes of fp32 per instruction);
// fp64 pairs are two scalar ops.
template <typename A> struct Pair;
template <> struct Pair<float> {
    using P = float2;
    static __device__ __forceinline__ P make(float a, float b) { return make_float2(a, b); }
    static __device__ __forceinline__ P splat(float a) { return make_float2(a, a); }
    static __device__ __forceinline__ P add(P a, P b) { return __fadd2_rn(a, b); }
    static __device__ __forceinline__ P mul(P a, P b) { return __fmul2_rn(a, b); }
    static __device__ __forceinline__ P fma(P a, P b, P c) { return __ffma2_rn(a, b, c); }
};
template <> struct Pair<double> {
    using P = double2;
    static __device__ __forceinline__ P make(double a, double b) { return make_double2(a, b); }
    static __device__ __forceinline__ P splat(double a) { return make_double2(a, a); }
    static __device__ __forceinline__ P add(P a, P b) { return make_double2(a.x + b.x, a.y + b.y); }
    static __device__ __forceinline__ P mul(P a, P b) { return make_double2(a.x * b.x, a.y * b.y); }
    static __device__ __forceinline__ P fma(P a, P b, P c) { return make_double2(::fma(a.x, b.x, c.x), ::fma(a.y, b.y, c.y)); }
};

// 16-byte vector -> W/2 pairs of Acc
template <typename T>
__device__ __forceinline__ void unpack2(const uint4& v, typename Pair<typename Traits<T>::Acc>::P* o);
template <>
__device__ __forceinline__ void unpack2<float>(const uint4& v, float2* o) {
    o[0] = make_float2(__uint_as_float(v.x), __uint_as_float(v.y));
    o[1] = make_float2(__uint_as_float(v.z), __uint_as_float(v.w));
}
template <>
__device__ __forceinline__ void unpack2<__nv_bfloat16>(const uint4& v, float2* o) {
    o[0] = make_float2(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u));
    o[1] = make_float2(__uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
    o[2] = make_float2(__uint_as_float(v.z << 16), __uint_as_float(v.z & 0xffff0000u));
    o[3] = make_float2(__uint_as_float(v.w << 16), __uint_as_float(v.w & 0xffff0000u));
}
template <>
__device__ __forceinline__ void unpack2<double>(const uint4& v, double2* o) {
    o[0] = make_double2(__hiloint2double((int)v.y, (int)v.x), __hiloint2double((int)v.w, (int)v.z));
}

// W/2 pairs of Acc -> 16-byte vector of T (round to nearest even)
template <typename T>
__device__ __forceinline__ uint4 pack2(const typename Pair<typename Traits<T>::Acc>::P* i);
template <>
__device__ __forceinline__ uint4 pack2<float>(const float2* i) {
    return make_uint4(__float_as_uint(i[0].x), __float_as_uint(i[0].y), __float_as_uint(i[1].x), __float_as_uint(i[1].y));
}
template <>
__device__ __forceinline__ uint4 pack2<__nv_bfloat16>(const float2* i) {
    return make_uint4(pack_bf16x2(i[0].x, i[0].y), pack_bf16x2(i[1].x, i[1].y), pack_bf16x2(i[2].x, i[2].y),
                      pack_bf16x2(i[3].x, i[3].y));
}
template <>
__device__ __forceinline__ uint4 pack2<double>(const double2* i) {
    return make_uint4((uint32_t)__double2loint(i[0].x), (uint32_t)__double2hiint(i[0].x),
                      (uint32_t)__double2loint(i[0].y), (uint32_t)__double2hiint(i[0].y));
}

// Sum NQ per-lane values over a warp with a transposed butterfly: NQ-1 + 5 -
// log2(NQ) shuffles instead of 5*NQ.  On return v[0] holds, in every lane,
// the warp total of quantity q = butterfly_q<NQ>(lane).
template <int NQ, typename V>
__device__ __forceinline__ void butterfly_sum(V* v, int lane) {
    int n = NQ;
    int m = 16;
#pragma unroll
    for (; n > 1; n >>= 1, m >>= 1) {
        const bool upper = (lane & m) != 0;
#pragma unroll
        for (int j = 0; j < n / 2; ++j) {
            const V send = upper ? v[j] : v[j + n / 2];
            const V keep = upper ? v[j + n / 2] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
#pragma unroll
    for (; m >= 1; m >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
}
template <int NQ>
__device__ __forceinline__ int butterfly_q(int lane) {
    int q = 0, n = NQ, m = 16;
#pragma unroll
    for (; n > 1; n >>= 1, m >>= 1)
        if (lane & m) q += n / 2;
    return q;
}

// ------------------------------------------------------------ shared mem --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ----------------------------------------------------------- watchdog -----
// Every spin loop is bounded: a protocol bug traps (a CUDA error the host
// reports) instead of hanging the GPU.
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr uint64_t kWatchdogNs = 4000000000ull;  // 4 s

// ------------------------------------------------------------- mbarrier --
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait(bar, parity)) {
        if (globaltimer_ns() - t0 > kWatchdogNs) {
            printf("gnsb watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n", (int)blockIdx.x,
                   (int)threadIdx.x, smem_u32(bar), parity);
            __trap();
        }
    }
}

// -------------------------------------------------------- bulk copy (TMA) --
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 1-D TMA: global -> shared, completion signalled on `bar` (complete_tx).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---------------------------------------------------- global memory ops --
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Software grid barrier for a cooperative (all-CTAs-resident) launch.  The
// counter must start at a multiple of gridDim.x (0); the kernel's final
// ticket holder resets it.
__device__ __forceinline__ void grid_barrier(unsigned* counter) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned old = atomicAdd(counter, 1u);
        const unsigned target = (old / gridDim.x + 1u) * gridDim.x;
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_gpu(counter) < target) {
            if (globaltimer_ns() - t0 > kWatchdogNs) __trap();
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// N independent butterfly sums, interleaved stage by stage (latency overlap);
// each result equals warp_sum of that element.
template <int N, typename V>
__device__ __forceinline__ void warp_sum_n(V (&v)[N]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// Atomic add with acquire-release semantics at GPU scope (the "last CTA"
// ticket: releases this CTA's prior writes, acquires every earlier CTA's).
__device__ __forceinline__ unsigned atomic_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace gnsb

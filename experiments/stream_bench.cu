// stream_bench.cu — memory-side ceiling of the LN-backward traffic pattern
// (read x, read dy, write dx; bf16) on B200.  Experiment only (not product).
//
//   tma_ring<R, CW>   : 1 producer warp streams R-row stages of x and dy into a
//                       shared-memory ring with cp.async.bulk; CW consumer warps
//                       write dx = x + dy from smem with 16-byte stores.
//   ldg_stream<U>     : grid-stride 16-byte loads of x and dy (U vectors in
//                       flight per thread), dx = x + dy.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2411_00999_b200/csrc/common.cuh"

using namespace gnsb;

__device__ __forceinline__ uint32_t addbf2(uint32_t a, uint32_t b) {
    __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a), y = *reinterpret_cast<__nv_bfloat162*>(&b);
    __nv_bfloat162 z = __hadd2(x, y);
    return *reinterpret_cast<uint32_t*>(&z);
}

template <int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
tma_ring(const __nv_bfloat16* x, const __nv_bfloat16* dy, __nv_bfloat16* dx, int64_t N, int D, int R, int S) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rb = (int64_t)blockIdx.x * N / gridDim.x, re = (int64_t)(blockIdx.x + 1) * N / gridDim.x;
    const int64_t ns = (re - rb + R - 1) / R;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == CW) {
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        int slot = 0;
        uint32_t ph = 0;
        for (int64_t it = 0; it < ns; ++it) {
            mbar_wait(&empty[slot], ph ^ 1u);
            const int64_t r0 = rb + it * R;
            const int nr = (int)min((int64_t)R, re - r0);
            const uint32_t bytes = nr * D * 2;
            __nv_bfloat16* sx = ring + (size_t)slot * 2 * R * D;
            mbar_expect_tx(&full[slot], 2 * bytes);
            bulk_g2s(sx, x + r0 * D, bytes, &full[slot], pol);
            bulk_g2s(sx + (size_t)R * D, dy + r0 * D, bytes, &full[slot], pol);
            mbar_arrive(&full[slot]);
            if (++slot == S) {
                slot = 0;
                ph ^= 1u;
            }
        }
        return;
    }
    int slot = 0;
    uint32_t ph = 0;
    const int nv = D / 8;
    for (int64_t it = 0; it < ns; ++it) {
        mbar_wait(&full[slot], ph);
        const int64_t r0 = rb + it * R;
        const int nr = (int)min((int64_t)R, re - r0);
        const __nv_bfloat16* sx = ring + (size_t)slot * 2 * R * D;
        const __nv_bfloat16* sdy = sx + (size_t)R * D;
        const int tot = nr * nv;
        uint4 v[8];
        int cnt = 0;
        for (int e = threadIdx.x; e < tot; e += CW * 32) {
            const uint4 a = reinterpret_cast<const uint4*>(sx)[e];
            const uint4 b = reinterpret_cast<const uint4*>(sdy)[e];
            uint4 o = make_uint4(addbf2(a.x, b.x), addbf2(a.y, b.y), addbf2(a.z, b.z), addbf2(a.w, b.w));
            st_stream(reinterpret_cast<uint4*>(dx + r0 * D) + e, o);
            ++cnt;
        }
        (void)v;
        (void)cnt;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            ph ^= 1u;
        }
    }
}

template <int U>
__global__ void __launch_bounds__(256) ldg_stream(const uint4* x, const uint4* dy, uint4* dx, int64_t n16) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = ld_stream(x + i + u * stride);
            b[u] = ld_stream(dy + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 o = make_uint4(addbf2(a[u].x, b[u].x), addbf2(a[u].y, b[u].y), addbf2(a[u].z, b[u].z),
                                 addbf2(a[u].w, b[u].w));
            st_stream(dx + i + u * stride, o);
        }
    }
    for (; i < n16; i += stride) {
        const uint4 a = ld_stream(x + i), b = ld_stream(dy + i);
        st_stream(dx + i, make_uint4(addbf2(a.x, b.x), addbf2(a.y, b.y), addbf2(a.z, b.z), addbf2(a.w, b.w)));
    }
}

// tma_ring with the stage order interleaved across CTAs: chunks of K stages,
// chunk j on CTA j % grid (K = 0: contiguous row ranges, as tma_ring).  At
// any moment the CTAs stream a window of about grid*K stages.
__device__ __forceinline__ int64_t ilv_stage(int64_t it, int K, int64_t NS, int64_t rb_stage, int64_t ns_contig) {
    if (K == 0) return it < ns_contig ? rb_stage + it : -1;
    const int64_t chunk = (int64_t)blockIdx.x + (it / K) * gridDim.x;
    const int64_t st = chunk * K + it % K;
    return st < NS ? st : -1;
}

template <int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
tma_ring_ilv(const __nv_bfloat16* x, const __nv_bfloat16* dy, __nv_bfloat16* dx, int64_t N, int D, int R, int S, int K) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t NS = (N + R - 1) / R;
    // contiguous split in whole stages
    const int64_t sb = (int64_t)blockIdx.x * NS / gridDim.x, se = (int64_t)(blockIdx.x + 1) * NS / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == CW) {
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        int slot = 0;
        uint32_t ph = 0;
        for (int64_t it = 0;; ++it) {
            const int64_t st = ilv_stage(it, K, NS, sb, se - sb);
            if (st < 0) break;
            mbar_wait(&empty[slot], ph ^ 1u);
            const int64_t r0 = st * R;
            const int nr = (int)min((int64_t)R, N - r0);
            const uint32_t bytes = nr * D * 2;
            __nv_bfloat16* sx = ring + (size_t)slot * 2 * R * D;
            mbar_expect_tx(&full[slot], 2 * bytes);
            bulk_g2s(sx, x + r0 * D, bytes, &full[slot], pol);
            bulk_g2s(sx + (size_t)R * D, dy + r0 * D, bytes, &full[slot], pol);
            mbar_arrive(&full[slot]);
            if (++slot == S) {
                slot = 0;
                ph ^= 1u;
            }
        }
        return;
    }
    int slot = 0;
    uint32_t ph = 0;
    const int nv = D / 8;
    for (int64_t it = 0;; ++it) {
        const int64_t st = ilv_stage(it, K, NS, sb, se - sb);
        if (st < 0) break;
        mbar_wait(&full[slot], ph);
        const int64_t r0 = st * R;
        const int nr = (int)min((int64_t)R, N - r0);
        const __nv_bfloat16* sx = ring + (size_t)slot * 2 * R * D;
        const __nv_bfloat16* sdy = sx + (size_t)R * D;
        const int tot = nr * nv;
        for (int e = threadIdx.x; e < tot; e += CW * 32) {
            const uint4 a = reinterpret_cast<const uint4*>(sx)[e];
            const uint4 b = reinterpret_cast<const uint4*>(sdy)[e];
            uint4 o = make_uint4(addbf2(a.x, b.x), addbf2(a.y, b.y), addbf2(a.z, b.z), addbf2(a.w, b.w));
            st_stream(reinterpret_cast<uint4*>(dx + r0 * D) + e, o);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            ph ^= 1u;
        }
    }
}

extern "C" {

int run_tma(int cw, const void* x, const void* dy, void* dx, int64_t N, int D, int R, int S, float* ms, int reps) {
    const size_t smem = 1024 + (size_t)S * 2 * R * D * 2;
    void (*k)(const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*, int64_t, int, int, int) = nullptr;
    if (cw == 4) k = tma_ring<4>;
    else if (cw == 8) k = tma_ring<8>;
    else if (cw == 12) k = tma_ring<12>;
    else if (cw == 16) k = tma_ring<16>;
    else return -1;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<sms, (cw + 1) * 32, smem>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, N, D, R, S);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r)
        k<<<sms, (cw + 1) * 32, smem>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, N, D, R, S);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    *ms /= reps;
    return cudaGetLastError();
}

int run_ldg(int u, int blocks_per_sm, const void* x, const void* dy, void* dx, int64_t n16, float* ms, int reps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&]() {
        if (u == 1) ldg_stream<1><<<grid, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, n16);
        if (u == 2) ldg_stream<2><<<grid, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, n16);
        if (u == 4) ldg_stream<4><<<grid, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, n16);
        if (u == 8) ldg_stream<8><<<grid, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, n16);
    };
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    *ms /= reps;
    return cudaGetLastError();
}

// Same kernels over `nsets` distinct buffer sets, launch r on set r % nsets,
// so no launch finds its inputs in L2 (the LN-bwd "steady" condition).
int run_tma_sets(int cw, const void* const* x, const void* const* dy, void* const* dx, int nsets, int64_t N, int D,
                 int R, int S, float* ms, int reps) {
    const size_t smem = 1024 + (size_t)S * 2 * R * D * 2;
    void (*k)(const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*, int64_t, int, int, int) = nullptr;
    if (cw == 4) k = tma_ring<4>;
    else if (cw == 8) k = tma_ring<8>;
    else if (cw == 16) k = tma_ring<16>;
    else return -1;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](int r) {
        const int i = r % nsets;
        k<<<sms, (cw + 1) * 32, smem>>>((const __nv_bfloat16*)x[i], (const __nv_bfloat16*)dy[i], (__nv_bfloat16*)dx[i],
                                        N, D, R, S);
    };
    for (int r = 0; r < nsets; ++r) launch(r);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch(r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    *ms /= reps;
    return cudaGetLastError();
}

int run_ldg_sets(int u, int blocks_per_sm, const void* const* x, const void* const* dy, void* const* dx, int nsets,
                 int64_t n16, float* ms, int reps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](int r) {
        const int i = r % nsets;
        const uint4 *xi = (const uint4*)x[i], *di = (const uint4*)dy[i];
        uint4* oi = (uint4*)dx[i];
        if (u == 1) ldg_stream<1><<<grid, 256>>>(xi, di, oi, n16);
        if (u == 2) ldg_stream<2><<<grid, 256>>>(xi, di, oi, n16);
        if (u == 4) ldg_stream<4><<<grid, 256>>>(xi, di, oi, n16);
    };
    for (int r = 0; r < nsets; ++r) launch(r);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch(r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    *ms /= reps;
    return cudaGetLastError();
}

int run_tma_ilv_sets(int cw, const void* const* x, const void* const* dy, void* const* dx, int nsets, int64_t N, int D,
                     int R, int S, int K, float* ms, int reps) {
    const size_t smem = 1024 + (size_t)S * 2 * R * D * 2;
    void (*k)(const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*, int64_t, int, int, int, int) = nullptr;
    if (cw == 4) k = tma_ring_ilv<4>;
    else if (cw == 8) k = tma_ring_ilv<8>;
    else if (cw == 16) k = tma_ring_ilv<16>;
    else return -1;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -2;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](int r) {
        const int i = r % nsets;
        k<<<sms, (cw + 1) * 32, smem>>>((const __nv_bfloat16*)x[i], (const __nv_bfloat16*)dy[i], (__nv_bfloat16*)dx[i],
                                        N, D, R, S, K);
    };
    for (int r = 0; r < nsets; ++r) launch(r);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch(r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    *ms /= reps;
    return cudaGetLastError();
}
}

// linear_gram.cu — per-example squared weight-gradient norms of a linear layer
// in the Gram ("Frobenius") form on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics: gnstk::linear_perexample_sqnorm_frobenius
// (proj/src/layers.cpp:159-187):
//     raw_b = < X_b X_b^T , G_b G_b^T >_F = sum_{t,u} (x_t . x_u)(g_t . g_u)
// which equals ||sum_t x_t^T g_t||_F^2, the weight-gradient form's norm
// (SPEC.md:157), at 2*T^2*(K+L) instead of 2*T*K*L FLOPs per example — and
// half of that here, because both Grams are symmetric: only tile pairs
// (i <= j) of the T x T grid are formed, off-diagonal pairs counted twice.
//
// Kernel (gram_norms_kernel): persistent, one CTA per SM, static round-robin
// over units (example b, tile pair i <= j) in example-major order, so all
// CTAs work on the same example at once and X_b, G_b (2 x 16 MB at cfg3) are
// shared through L2.
//   * warp 0: TMA producer.  Rows t of X_b / G_b are K-major operands read
//     straight from the [B, T, K] / [B, T, L] row-major tensors through 3-D
//     tensor maps (box 64 features x 128 tokens, 128-byte swizzle); a diagonal
//     pair loads its tile once and uses it as both operands;
//   * warp 1: one thread issues tcgen05.mma (M=N=128, K=16, bf16 -> fp32):
//     the X-Gram tile over K into TMEM columns [0,128) of the unit's buffer,
//     then the G-Gram tile over L into [128,256); two buffers (all 512 TMEM
//     columns) alternate between units so the epilogue of one unit overlaps
//     the MMAs of the next;
//   * warps 2..5: epilogue.  tcgen05.ld both tiles, sum of products per TMEM
//     lane (fp32), fixed-order fold over the 4 warps in fp64 -> q[b][pair]
//     (x2 off the diagonal).  A deterministic second kernel folds q over the
//     pairs of each example.  No floating-point atomics.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace gnsb {

namespace gr {
constexpr int BM = 128;                      // token tile (both Gram dimensions)
constexpr int BK = 64;                       // features per stage: one 128-byte swizzle row
constexpr int STAGES = 6;
constexpr int OP_BYTES = BM * BK * 2;        // 16 KB
constexpr int STAGE_BYTES = 2 * OP_BYTES;    // 32 KB
constexpr int EPI_WARPS = 4;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 512;
}  // namespace gr

struct GramArgs {
    int B, T, K, L;
    int nt;        // T / BM
    int npairs;    // nt * (nt + 1) / 2
    double* q;     // [B][npairs]
};

// pair index p (row-major over i <= j) -> (i, j)
__device__ __forceinline__ void pair_ij(int p, int nt, int& i, int& j) {
    i = 0;
    while (p >= nt - i) {
        p -= nt - i;
        ++i;
    }
    j = i + p;
}

__global__ void __launch_bounds__(gr::THREADS, 1)
    gram_norms_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmg, GramArgs a) {
    using namespace gr;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    double* red = reinterpret_cast<double*>(tmem_slot + 4);  // [EPI_WARPS]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t units = (int64_t)a.B * a.npairs;
    const int grid = gridDim.x, c = blockIdx.x;
    const int kbx = a.K / BK, kbg = a.L / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], EPI_WARPS);
        }
        fence_mbar_init();
        tc::prefetch_tmap(&tmx);
        tc::prefetch_tmap(&tmg);
    }
    if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer --
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t u = c; u < units; u += grid) {
                const int b = (int)(u / a.npairs);
                int i, j;
                pair_ij((int)(u - (int64_t)b * a.npairs), a.nt, i, j);
                const bool diag = i == j;
                for (int op = 0; op < 2; ++op) {  // 0: X over K, 1: G over L
                    const CUtensorMap* m = op == 0 ? &tmx : &tmg;
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        unsigned char* st = ring + (size_t)s * STAGE_BYTES;
                        mbar_arrive_expect_tx(&full[s], diag ? OP_BYTES : STAGE_BYTES);
                        tc::tma_load_3d(st, m, kb * BK, i * BM, b, &full[s]);
                        if (!diag) tc::tma_load_3d(st + OP_BYTES, m, kb * BK, j * BM, b, &full[s]);
                        if (++s == STAGES) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer --
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BM, false, false);  // both K-major: D = A * B^T
            int s = 0, buf = 0;
            uint32_t ph = 0, tph = 0;
            for (int64_t u = c; u < units; u += grid) {
                const int b = (int)(u / a.npairs);
                int i, j;
                pair_ij((int)(u - (int64_t)b * a.npairs), a.nt, i, j);
                const bool diag = i == j;
                mbar_wait(&tempty[buf], tph ^ 1u);  // epilogue drained this buffer
                tc::fence_after_sync();
                for (int op = 0; op < 2; ++op) {
                    const uint32_t dcol = tmem + (uint32_t)(buf * 2 * BM + op * BM);
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&full[s], ph);
                        tc::fence_after_sync();
                        const uint32_t abase = smem_u32(ring + (size_t)s * STAGE_BYTES);
                        const uint32_t bbase = diag ? abase : abase + OP_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            // K-major SW128: 8-row x 128-byte atoms, SBO = 1 KB; a K step of
                            // 16 elements advances the start address by 32 bytes
                            const uint64_t ad = tc::smem_desc_sw128(abase + k * 32, 16, 1024);
                            const uint64_t bd = tc::smem_desc_sw128(bbase + k * 32, 16, 1024);
                            tc::mma_bf16(dcol, ad, bd, idesc, (kb | k) != 0);
                        }
                        tc::commit(&empty[s]);
                        if (++s == STAGES) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
                tc::commit(&tfull[buf]);
                if (++buf == 2) {
                    buf = 0;
                    tph ^= 1u;
                }
            }
        }
    } else {
        // --------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const int quad = warp & 3;  // TMEM lanes this warp may access
        int buf = 0;
        uint32_t tph = 0;
        for (int64_t u = c; u < units; u += grid) {
            const int b = (int)(u / a.npairs);
            const int p = (int)(u - (int64_t)b * a.npairs);
            int i, j;
            pair_ij(p, a.nt, i, j);
            mbar_wait(&tfull[buf], tph);
            tc::fence_after_sync();
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * 2 * BM);
            float acc = 0.f;
#pragma unroll
            for (int cc = 0; cc < BM / 32; ++cc) {
                uint32_t rx[32], rg[32];
                tc::tmem_ld_32x32b_x32(base + cc * 32, rx);
                tc::tmem_ld_32x32b_x32(base + BM + cc * 32, rg);
                tc::tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 32; ++k) acc = fmaf(__uint_as_float(rx[k]), __uint_as_float(rg[k]), acc);
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            const float w = warp_sum(acc);
            if (lane == 0) red[e] = (double)w;
            named_bar_sync(1, EPI_WARPS * 32);
            if (e == 0 && lane == 0) {
                double t = 0.0;
#pragma unroll
                for (int k = 0; k < EPI_WARPS; ++k) t += red[k];
                a.q[(size_t)b * a.npairs + p] = i == j ? t : 2.0 * t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
            if (++buf == 2) {
                buf = 0;
                tph ^= 1u;
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after_sync();
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// ------------------------------------------------------------------ host --
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// [B, T, F] bf16 row-major as a 3-D tensor (F innermost), box 64 features x 128 tokens, 128B swizzle
bool make_map_rows(CUtensorMap* m, const void* base, int B, int T, int F) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)F, (cuuint64_t)T, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)F * 2, (cuuint64_t)T * F * 2};
    cuuint32_t box[3] = {(cuuint32_t)gr::BK, (cuuint32_t)gr::BM, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int gram_pairs(int64_t T) {
    const int64_t nt = T / gr::BM;
    return (int)(nt * (nt + 1) / 2);
}

}  // namespace

bool gram_shape_ok(int64_t B, int64_t T, int64_t K, int64_t L) {
    return B >= 1 && T >= gr::BM && T % gr::BM == 0 && K % gr::BK == 0 && L % gr::BK == 0 && K > 0 && L > 0 &&
           T < (1 << 20) && B < (1 << 20) && (int64_t)B * gram_pairs(T) < (1ll << 31);
}

size_t gram_workspace(int64_t B, int64_t T) { return (size_t)B * gram_pairs(T) * sizeof(double) + 256; }

cudaError_t launch_gram_norms(const void* x, const void* g, double* raw, double* sums, int64_t B, int64_t T,
                              int64_t K, int64_t L, void* ws, cudaStream_t st) {
    CUtensorMap mx, mg;
    if (!make_map_rows(&mx, x, (int)B, (int)T, (int)K) || !make_map_rows(&mg, g, (int)B, (int)T, (int)L))
        return cudaErrorInvalidValue;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(gram_norms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gr::SMEM);
    });
    GramArgs a{};
    a.B = (int)B;
    a.T = (int)T;
    a.K = (int)K;
    a.L = (int)L;
    a.nt = (int)(T / gr::BM);
    a.npairs = gram_pairs(T);
    a.q = static_cast<double*>(ws);
    const int64_t units = B * a.npairs;
    const int sms = device_sm_count();
    const int grid = (int)(units < sms ? units : sms);
    gram_norms_kernel<<<grid, gr::THREADS, gr::SMEM, st>>>(mx, mg, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_fold_rows(a.q, (int)B, a.npairs, raw, sums, 0, st);
}

}  // namespace gnsb

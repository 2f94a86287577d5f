// linear_gram.cu — per-example squared weight-gradient norms of a linear layer
// in the Gram ("Frobenius") form on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics: gnstk::linear_perexample_sqnorm_frobenius
// (proj/src/layers.cpp:159-187):
//     raw_b = < X_b X_b^T , G_b G_b^T >_F = sum_{t,u} (x_t . x_u)(g_t . g_u)
// which equals ||sum_t x_t^T g_t||_F^2, the weight-gradient form's norm
// (SPEC.md:157), at 2*T^2*(K+L) instead of 2*T*K*L FLOPs per example — about
// half of that here, because both Grams are symmetric.
//
// Kernel (gram_norms_kernel): persistent, one CTA per SM, static round-robin
// over units (example b, 128-token row tile i, 256-token column block J) with
// 2J+1 >= i, i.e. every 128 x 128 tile pair (i, j) with j >= i is covered once
// (the few j < i halves of blocks straddling the diagonal get weight 0),
// example-major so all CTAs work on the same example and X_b, G_b (2 x 16 MB
// at cfg3) are shared through L2.  M = 128, N = 256: per 64-feature stage the
// MMA reads 48 KB of shared memory for 4.2 MFLOP, which keeps the tensor pipe
// ahead of the shared-memory operand bandwidth (an N = 128 tile does not).
//   * warp 0: TMA producer.  Rows t of X_b / G_b are K-major operands read
//     straight from the [B, T, K] / [B, T, L] row-major tensors through 3-D
//     tensor maps (boxes 64 features x 128 / 256 tokens, 128-byte swizzle;
//     tokens past T read as zero);
//   * warp 1: one thread issues tcgen05.mma (M=128, N=256, K=16, bf16 -> fp32):
//     the X-Gram block over K into TMEM columns [0,256), then the G-Gram block
//     over L into [256,512);
//   * warps 2..5: epilogue.  tcgen05.ld both blocks, per-half weighted sum of
//     products per TMEM lane (fp32; weight 2 above the diagonal, 1 on it, 0
//     below), fixed-order fold over the 4 warps in fp64 -> q[b][unit].  A
//     deterministic second kernel folds q over each example's units.  No
//     floating-point atomics.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace gnsb {

namespace gr {
constexpr int BM = 128;                      // token tile of the Gram rows (i)
constexpr int BN = 256;                      // token block of the Gram columns (J): two 128-tiles
constexpr int BK = 64;                       // features per stage: one 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB
constexpr int B_BYTES = BN * BK * 2;         // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 4;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 512;               // X-Gram block [0, 256) + G-Gram block [256, 512)
}  // namespace gr

struct GramArgs {
    int B, T, K, L;
    int nt;        // T / BM (row tiles)
    int nJ;        // ceil(nt / 2) (column blocks)
    int nunits;    // units per example: sum_i (nJ - i / 2)
    double* q;     // [B][nunits]
};

// unit index p (row-major over i, then J >= i / 2) -> (i, J)
__device__ __forceinline__ void unit_iJ(int p, int nt, int nJ, int& i, int& J) {
    i = 0;
    while (i < nt && p >= nJ - i / 2) {
        p -= nJ - i / 2;
        ++i;
    }
    J = i / 2 + p;
}

__global__ void __launch_bounds__(gr::THREADS, 1)
    gram_norms_kernel(const __grid_constant__ CUtensorMap tmx_a, const __grid_constant__ CUtensorMap tmx_b,
                      const __grid_constant__ CUtensorMap tmg_a, const __grid_constant__ CUtensorMap tmg_b,
                      GramArgs a) {
    using namespace gr;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    double* red = reinterpret_cast<double*>(tmem_slot + 4);  // [EPI_WARPS]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t units = (int64_t)a.B * a.nunits;
    const int grid = gridDim.x, c = blockIdx.x;
    const int kbx = (a.K + BK - 1) / BK, kbg = (a.L + BK - 1) / BK;  // feature tails read as zero

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, EPI_WARPS);
        fence_mbar_init();
        tc::prefetch_tmap(&tmx_a);
        tc::prefetch_tmap(&tmx_b);
        tc::prefetch_tmap(&tmg_a);
        tc::prefetch_tmap(&tmg_b);
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
                const int b = (int)(u / a.nunits);
                int i, J;
                unit_iJ((int)(u - (int64_t)b * a.nunits), a.nt, a.nJ, i, J);
                for (int op = 0; op < 2; ++op) {  // 0: X over K, 1: G over L
                    const CUtensorMap* ma = op == 0 ? &tmx_a : &tmg_a;
                    const CUtensorMap* mb = op == 0 ? &tmx_b : &tmg_b;
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        unsigned char* st = ring + (size_t)s * STAGE_BYTES;
                        // full boxes always land (tokens past T are zero-filled)
                        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                        tc::tma_load_3d(st, ma, kb * BK, i * BM, b, &full[s]);
                        tc::tma_load_3d(st + A_BYTES, mb, kb * BK, J * BN, b, &full[s]);
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
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, false);  // both K-major: D = A * B^T
            int s = 0;
            uint32_t ph = 0, tph = 0;
            for (int64_t u = c; u < units; u += grid) {
                mbar_wait(tempty, tph ^ 1u);  // the epilogue drained the accumulators
                tc::fence_after_sync();
                for (int op = 0; op < 2; ++op) {
                    const uint32_t dcol = tmem + (uint32_t)(op * BN);
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&full[s], ph);
                        tc::fence_after_sync();
                        const uint32_t abase = smem_u32(ring + (size_t)s * STAGE_BYTES);
                        const uint32_t bbase = abase + A_BYTES;
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
                tc::commit(tfull);
                tph ^= 1u;
            }
        }
    } else {
        // --------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const int quad = warp & 3;  // TMEM lanes this warp may access
        uint32_t tph = 0;
        for (int64_t u = c; u < units; u += grid) {
            const int b = (int)(u / a.nunits);
            const int p = (int)(u - (int64_t)b * a.nunits);
            int i, J;
            unit_iJ(p, a.nt, a.nJ, i, J);
            mbar_wait(tfull, tph);
            tph ^= 1u;
            tc::fence_after_sync();
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16);
            float w2[2];  // per 128-column half of the block
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float acc = 0.f;
#pragma unroll 1
                for (int cc = 0; cc < BM / 32; ++cc) {
                    uint32_t rx[32], rg[32];
                    const uint32_t col = (uint32_t)(h * BM + cc * 32);
                    tc::tmem_ld_32x32b_x32(base + col, rx);
                    tc::tmem_ld_32x32b_x32(base + BN + col, rg);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) acc = fmaf(__uint_as_float(rx[k]), __uint_as_float(rg[k]), acc);
                }
                w2[h] = acc;
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            warp_sum_n(w2);
            if (lane == 0) {
                double t = 0.0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 2 * J + h;
                    const double wgt = j < i ? 0.0 : (j == i ? 1.0 : 2.0);
                    t += wgt * (double)w2[h];
                }
                red[e] = t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
            if (e == 0 && lane == 0) {
                double t = 0.0;
#pragma unroll
                for (int k = 0; k < EPI_WARPS; ++k) t += red[k];
                a.q[(size_t)b * a.nunits + p] = t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after_sync();
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// ------------------------------------------------- CTA-pair (2SM) variant --
// Units (example b, 256-token row block I, 256-token column block J >= I) on a
// CTA pair: cta_group::2 MMAs of M=256 (each CTA holds 128 rows of A) and
// N=256 (each CTA holds 128 rows of B), so per 64-feature stage a CTA loads
// 32 KB for 4.2 MFLOP of its half of the tile — a third less operand traffic
// than the single-CTA 128x256 block.  The leader CTA issues the MMAs; both
// CTAs' TMA loads complete on the leader's full barrier; the MMA commit
// multicasts to both CTAs' empty / accumulator-full barriers; both CTAs'
// epilogue warps release the accumulators on the leader's barrier.
namespace gr2 {
constexpr int BH = 128;                      // rows of A (and of B) per CTA
constexpr int BK = 64;
constexpr int STAGES = 6;
constexpr int A_BYTES = BH * BK * 2;         // 16 KB
constexpr int B_BYTES = BH * BK * 2;         // 16 KB (this CTA's half of N = 256)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 4;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 512;               // X-Gram [0, 256) + G-Gram [256, 512)
}  // namespace gr2

struct Gram2Args {
    int B, T, K, L;
    int nt;        // T / 128 (token tiles)
    int nI;        // ceil(nt / 2) (256-token blocks)
    int nunits;    // nI * (nI + 1) / 2 per example
    double* q;     // [B][nunits][2] (one partial per CTA of the pair)
};

__device__ __forceinline__ void unit_IJ(int p, int nI, int& I, int& J) {
    I = 0;
    while (p >= nI - I) {
        p -= nI - I;
        ++I;
    }
    J = I + p;
}

__global__ void __launch_bounds__(gr2::THREADS, 1)
    gram2_norms_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmg, Gram2Args a) {
    using namespace gr2;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    double* red = reinterpret_cast<double*>(tmem_slot + 4);  // [EPI_WARPS]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int64_t units = (int64_t)a.B * a.nunits;
    const int kbx = (a.K + BK - 1) / BK, kbg = (a.L + BK - 1) / BK;  // feature tails read as zero

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // the leader's arrive.expect_tx(both CTAs' bytes); the peer's TMA only
            // completes bytes on it (a release-arrive from the peer would add a
            // cluster-scope fence per stage to its producer)
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);  // the leader's multicast commit
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 2 * EPI_WARPS);  // both CTAs' epilogue warps
        fence_mbar_init();
        tc::prefetch_tmap(&tmx);
        tc::prefetch_tmap(&tmg);
    }
    if (warp == 1) tc::tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer --
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t u = pair; u < units; u += npairs) {
                const int b = (int)(u / a.nunits);
                int I, J;
                unit_IJ((int)(u - (int64_t)b * a.nunits), a.nI, I, J);
                for (int op = 0; op < 2; ++op) {
                    const CUtensorMap* m = op == 0 ? &tmx : &tmg;
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        unsigned char* st = ring + (size_t)s * STAGE_BYTES;
                        const uint32_t leader_full = tc::mapa(smem_u32(&full[s]), 0);
                        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
                        tc::tma_load_3d_2sm(st, m, kb * BK, I * 2 * BH + (int)rank * BH, b, leader_full);
                        tc::tma_load_3d_2sm(st + A_BYTES, m, kb * BK, J * 2 * BH + (int)rank * BH, b, leader_full);
                        if (++s == STAGES) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------- MMA issuer (leader only) --
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16(2 * BH, 2 * BH, false, false);  // M=256, N=256, K-major
            int s = 0;
            uint32_t ph = 0, tph = 0;
            for (int64_t u = pair; u < units; u += npairs) {
                tc::mbar_wait_cluster(tempty, tph ^ 1u);  // both epilogues drained the accumulators
                tc::fence_after_sync();
                for (int op = 0; op < 2; ++op) {
                    const uint32_t dcol = tmem + (uint32_t)(op * 2 * BH);
                    const int nkb = op == 0 ? kbx : kbg;
                    for (int kb = 0; kb < nkb; ++kb) {
                        tc::mbar_wait_cluster(&full[s], ph);
                        tc::fence_after_sync();
                        const uint32_t abase = smem_u32(ring + (size_t)s * STAGE_BYTES);
                        const uint32_t bbase = abase + A_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = tc::smem_desc_sw128(abase + k * 32, 16, 1024);
                            const uint64_t bd = tc::smem_desc_sw128(bbase + k * 32, 16, 1024);
                            tc::mma_bf16_pair(dcol, ad, bd, idesc, (kb | k) != 0);
                        }
                        tc::commit_pair(&empty[s], 0x3);
                        if (++s == STAGES) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
                tc::commit_pair(tfull, 0x3);
                tph ^= 1u;
            }
        }
    } else {
        // ------------------------------------------------- epilogue (both CTAs) --
        const int e = warp - 2;
        const int quad = warp & 3;
        const uint32_t leader_tempty = tc::mapa(smem_u32(tempty), 0);
        uint32_t tph = 0;
        for (int64_t u = pair; u < units; u += npairs) {
            const int b = (int)(u / a.nunits);
            const int p = (int)(u - (int64_t)b * a.nunits);
            int I, J;
            unit_IJ(p, a.nI, I, J);
            tc::mbar_wait_cluster(tfull, tph);
            tph ^= 1u;
            tc::fence_after_sync();
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16);
            float w2[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float acc = 0.f;
#pragma unroll 1
                for (int cc = 0; cc < BH / 32; ++cc) {
                    uint32_t rx[32], rg[32];
                    const uint32_t col = (uint32_t)(h * BH + cc * 32);
                    tc::tmem_ld_32x32b_x32(base + col, rx);
                    tc::tmem_ld_32x32b_x32(base + 2 * BH + col, rg);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) acc = fmaf(__uint_as_float(rx[k]), __uint_as_float(rg[k]), acc);
                }
                w2[h] = acc;
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(leader_tempty);
            warp_sum_n(w2);
            if (lane == 0) {
                const int i = 2 * I + (int)rank;  // this CTA's 128-token row tile
                double t = 0.0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 2 * J + h;
                    const double wgt = j < i ? 0.0 : (j == i ? 1.0 : 2.0);
                    t += wgt * (double)w2[h];
                }
                red[e] = t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
            if (e == 0 && lane == 0) {
                double t = 0.0;
#pragma unroll
                for (int k = 0; k < EPI_WARPS; ++k) t += red[k];
                a.q[((size_t)b * a.nunits + p) * 2 + rank] = t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
        }
    }
    tc::fence_before_sync();
    tc::cluster_sync();
    if (warp == 1) {
        tc::fence_after_sync();
        tc::tmem_dealloc_pair<TMEM_COLS>(tmem);
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

// [B, T, F] bf16 row-major as a 3-D tensor (F innermost), box 64 features x `rows` tokens, 128B swizzle
bool make_map_rows(CUtensorMap* m, const void* base, int B, int T, int F, int rows) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)F, (cuuint64_t)T, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)F * 2, (cuuint64_t)T * F * 2};
    cuuint32_t box[3] = {(cuuint32_t)gr::BK, (cuuint32_t)rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int gram_units(int64_t T) {  // units per example: sum over row tiles i of (nJ - i / 2)
    const int64_t nt = (T + gr::BM - 1) / gr::BM, nJ = (nt + 1) / 2;
    int64_t n = 0;
    for (int64_t i = 0; i < nt; ++i) n += nJ - i / 2;
    return (int)n;
}

}  // namespace

int gram2_units(int64_t T) {
    const int64_t nt = (T + gr::BM - 1) / gr::BM, nI = (nt + 1) / 2;
    return (int)(nI * (nI + 1) / 2);
}

cudaError_t launch_gram2_norms(const void* x, const void* g, double* raw, double* sums, int64_t B, int64_t T,
                               int64_t K, int64_t L, void* ws, cudaStream_t st) {
    CUtensorMap mx, mg;
    if (!make_map_rows(&mx, x, (int)B, (int)T, (int)K, gr2::BH) || !make_map_rows(&mg, g, (int)B, (int)T, (int)L, gr2::BH))
        return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gram2_norms_kernel), gr2::SMEM);
    if (e != cudaSuccess) return e;
    Gram2Args a{};
    a.B = (int)B;
    a.T = (int)T;
    a.K = (int)K;
    a.L = (int)L;
    a.nt = (int)((T + gr::BM - 1) / gr::BM);
    a.nI = (a.nt + 1) / 2;
    a.nunits = gram2_units(T);
    a.q = static_cast<double*>(ws);
    const int64_t units = B * a.nunits;
    const int sms = device_sm_count() / 2 * 2;
    int grid = (int)(2 * units < sms ? 2 * units : sms);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(gr2::THREADS);
    cfg.dynamicSmemBytes = gr2::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, gram2_norms_kernel, mx, mg, a);
    if (e != cudaSuccess) return e;
    return launch_fold_rows(a.q, (int)B, 2 * a.nunits, raw, sums, 0, st);
}

// Any T, K, L with 16-byte row strides (K, L multiples of 8): tokens past T
// and features past K / L are zero-filled by TMA and add nothing to either Gram.
bool gram_shape_ok(int64_t B, int64_t T, int64_t K, int64_t L) {
    return B >= 1 && T >= 1 && K % 8 == 0 && L % 8 == 0 && K > 0 && L > 0 && K < (1 << 30) && L < (1 << 30) &&
           T < (1 << 20) && B < (1 << 20) && (int64_t)B * gram_units(T) < (1ll << 31);
}

size_t gram_workspace(int64_t B, int64_t T) {
    const int64_t u = gram_units(T) > 2 * gram2_units(T) ? gram_units(T) : 2 * gram2_units(T);
    return (size_t)B * u * sizeof(double) + 256;
}

cudaError_t launch_gram_norms(const void* x, const void* g, double* raw, double* sums, int64_t B, int64_t T,
                              int64_t K, int64_t L, void* ws, cudaStream_t st) {
    // the CTA-pair kernel by default (measured 2-3 % faster at cfg3);
    // GNSB_GRAM_IMPL=1 selects the single-CTA 128x256 kernel
    const char* impl = std::getenv("GNSB_GRAM_IMPL");
    if (!(impl && impl[0] == '1')) return launch_gram2_norms(x, g, raw, sums, B, T, K, L, ws, st);
    CUtensorMap mxa, mxb, mga, mgb;
    if (!make_map_rows(&mxa, x, (int)B, (int)T, (int)K, gr::BM) || !make_map_rows(&mxb, x, (int)B, (int)T, (int)K, gr::BN) ||
        !make_map_rows(&mga, g, (int)B, (int)T, (int)L, gr::BM) || !make_map_rows(&mgb, g, (int)B, (int)T, (int)L, gr::BN))
        return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gram_norms_kernel), gr::SMEM);
    if (e != cudaSuccess) return e;
    GramArgs a{};
    a.B = (int)B;
    a.T = (int)T;
    a.K = (int)K;
    a.L = (int)L;
    a.nt = (int)((T + gr::BM - 1) / gr::BM);
    a.nJ = (a.nt + 1) / 2;
    a.nunits = gram_units(T);
    a.q = static_cast<double*>(ws);
    const int64_t units = B * a.nunits;
    const int sms = device_sm_count();
    const int grid = (int)(units < sms ? units : sms);
    gram_norms_kernel<<<grid, gr::THREADS, gr::SMEM, st>>>(mxa, mxb, mga, mgb, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_fold_rows(a.q, (int)B, a.nunits, raw, sums, 0, st);
}

}  // namespace gnsb

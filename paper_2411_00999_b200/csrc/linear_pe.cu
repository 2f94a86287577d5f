// linear_pe.cu — per-example squared gradient norms of a linear layer on
// sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics (proj/src/layers.cpp:80-157, the "simultaneous" / weight-gradient
// form): for each example b, dW_b = sum_t x_{b,t}^T g_{b,t} (K x L);
// raw_b = ||dW_b||_F^2 (the square is taken AFTER the sum over t);
// dW = sum_b dW_b.  And the Gram / Frobenius form (layers.cpp:159-187):
// raw_b = <X_b X_b^T, G_b G_b^T>_F.
//
// Weight-gradient form kernel (wgrad_norms_kernel):
//   * persistent, one CTA per SM, static round-robin over 128 x 256 output
//     tiles of dW; for every tile the CTA walks all examples b;
//   * warp 0: TMA producer.  A = X_b^T and B = G_b are MN-major operands read
//     straight from the [B, T, K] / [B, T, L] row-major tensors through 3-D
//     tensor maps (box 64 features x 64 tokens, 128-byte swizzle), 4-stage ring;
//   * warp 1: a single elected thread issues tcgen05.mma (M=128, N=256, K=16,
//     bf16 -> fp32) into a per-example TMEM accumulator; two 256-column
//     accumulators (all 512 TMEM columns) alternate between examples so the
//     epilogue of example b overlaps the MMAs of example b+1;
//   * warps 2..9: epilogue.  tcgen05.ld the example's tile, square-accumulate
//     (-> the tile's share of raw_b) and add it into the running sum_b dW held
//     in registers (128 columns x 1 row per thread); after the last example the
//     tile of dW is stored once.
//   * per-(example, tile) partial norms are folded by a deterministic second
//     kernel; no floating-point atomics.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace gnsb {

namespace wg {
constexpr int BM = 128, BN = 256, BK = 64;   // tile and K-block (tokens per stage)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB
constexpr int B_BYTES = BN * BK * 2;         // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024;  // align slack + ring + barriers
constexpr int TMEM_COLS = 512;
}  // namespace wg

struct WgradArgs {
    int B, T, K, L;
    int tiles_m, tiles_n;
    float* part;           // [tiles][max_parts][BM][BN] partial sum_b dW of split tiles
    unsigned* ticket;      // [tiles], zero on entry and on exit
    int max_parts;
    float* dW;     // [K, L] or null
    double* q;     // [B][tiles] per-(example, tile) ||dW_b tile||^2
    double* qbig;  // [tiles] ||dW tile||^2
};

// PAIR: a 2-CTA cluster computes a 256 x 256 tile of dW with
// tcgen05.mma.cta_group::2 (M = 256 input features, 128 per CTA; N = 256 output
// features, each CTA loading 128 of them): per token stage a CTA loads 32 KB
// instead of 48 KB for the same MMA work.  Sub-tile (the CTA's 128 x 256
// half) indices equal the single-CTA tile indices, so q / qbig / tickets /
// split parts keep their layout.
template <bool PAIR>
__global__ void __launch_bounds__(wg::THREADS, 1)
    wgrad_norms_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmg, WgradArgs a) {
    using namespace wg;
    constexpr int BNL = PAIR ? BN / 2 : BN;             // output features this CTA loads per stage
    constexpr int LOAD_BYTES = A_BYTES + BNL * BK * 2;  // bytes this CTA's TMA brings per stage
    constexpr int NST = PAIR ? 6 : STAGES;              // same ring bytes: 6 x 32 KB = 4 x 48 KB
    static_assert(NST * LOAD_BYTES <= STAGES * STAGE_BYTES, "ring");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * LOAD_BYTES);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;      // [2]
    uint64_t* tempty = tfull + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [EPI_WARPS]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = a.tiles_m * a.tiles_n;  // 128 x 256 sub-tiles (q / qbig / ticket indexing)
    const int kblocks = (a.T + BK - 1) / BK;  // tokens past T read as zero
    const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0u;
    // scheduled tiles: 256 x 256 pair tiles (PAIR) or 128 x 256 tiles
    const int tiles_ms = PAIR ? a.tiles_m / 2 : a.tiles_m;
    const int stiles = tiles_ms * a.tiles_n;
    auto sub_of = [&](int tile) {  // this CTA's 128 x 256 sub-tile of a scheduled tile
        return PAIR ? ((tile % tiles_ms) * 2 + (int)rank) + (tile / tiles_ms) * a.tiles_m : tile;
    };
    // Schedule (identical in every role).  Full rounds: CTA c takes tile
    // r*grid + c with all examples, so at any moment every CTA works on the
    // same example and X_b, G_b are shared through L2.  The remaining
    // R = tiles % grid tiles are split into P = grid / R example ranges each.
    const int grid = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x, c = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int full_rounds = stiles / grid, R = stiles % grid;
    const int P = R > 0 ? (grid / R < a.B ? grid / R : a.B) : 1;
    const int nseg = full_rounds + ((R > 0 && c < R * P) ? 1 : 0);
    auto segment = [&](int si, int& tile, int& b0, int& b1, int& nparts, int& part) {
        if (si < full_rounds) {
            tile = si * grid + c;
            b0 = 0;
            b1 = a.B;
            nparts = 1;
            part = 0;
        } else {
            tile = full_rounds * grid + c / P;
            part = c % P;
            nparts = P;
            b0 = (int)((int64_t)a.B * part / P);
            b1 = (int)((int64_t)a.B * (part + 1) / P);
        }
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], PAIR ? 2 * EPI_WARPS : EPI_WARPS);  // (PAIR: both CTAs' epilogues)
        }
        fence_mbar_init();
        tc::prefetch_tmap(&tmx);
        tc::prefetch_tmap(&tmg);
    }
    if (warp == 1) {
        if constexpr (PAIR)
            tc::tmem_alloc_pair<TMEM_COLS>(tmem_slot);
        else
            tc::tmem_alloc<TMEM_COLS>(tmem_slot);
    }
    tc::fence_before_sync();
    if constexpr (PAIR)
        tc::cluster_sync();
    else
        __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer --
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int si = 0; si < nseg; ++si) {
                int tile, b0, b1, np_, pt;
                segment(si, tile, b0, b1, np_, pt);
                const int sub = sub_of(tile);
                const int i0 = (sub % a.tiles_m) * BM, j0 = (sub / a.tiles_m) * BN + (int)rank * BNL;
                const uint32_t bar_leader = PAIR ? tc::mapa(smem_u32(&full[0]), 0) : 0u;
                for (int b = b0; b < b1; ++b) {
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        unsigned char* st = ring + (size_t)s * LOAD_BYTES;
                        const int t0 = kb * BK;
                        if constexpr (PAIR) {
                            // both CTAs' bytes complete on the leader's barrier; only the
                            // leader arrives (expecting both halves)
                            const uint32_t fb = bar_leader + (uint32_t)(s * 8);
                            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * LOAD_BYTES);
#pragma unroll
                            for (int h = 0; h < BM / 64; ++h)
                                tc::tma_load_3d_2sm(st + h * 8192, &tmx, i0 + 64 * h, t0, b, fb);
#pragma unroll
                            for (int h = 0; h < BNL / 64; ++h)
                                tc::tma_load_3d_2sm(st + A_BYTES + h * 8192, &tmg, j0 + 64 * h, t0, b, fb);
                        } else {
                            mbar_arrive_expect_tx(&full[s], LOAD_BYTES);
#pragma unroll
                            for (int h = 0; h < BM / 64; ++h)
                                tc::tma_load_3d(st + h * 8192, &tmx, i0 + 64 * h, t0, b, &full[s]);
#pragma unroll
                            for (int h = 0; h < BNL / 64; ++h)
                                tc::tma_load_3d(st + A_BYTES + h * 8192, &tmg, j0 + 64 * h, t0, b, &full[s]);
                        }
                        if (++s == NST) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer --
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16(PAIR ? 2 * BM : BM, BN, true, true);
            int s = 0, buf = 0;
            uint32_t ph = 0, tph = 0;
            for (int si = 0; si < nseg; ++si) {
                int tile, b0, b1, np_, pt;
                segment(si, tile, b0, b1, np_, pt);
                for (int b = b0; b < b1; ++b) {
                    if constexpr (PAIR)
                        tc::mbar_wait_cluster(&tempty[buf], tph ^ 1u);  // both epilogues drained it
                    else
                        mbar_wait(&tempty[buf], tph ^ 1u);  // epilogue drained this accumulator
                    tc::fence_after_sync();
                    const uint32_t dcol = tmem + (uint32_t)(buf * BN);
                    for (int kb = 0; kb < kblocks; ++kb) {
                        if constexpr (PAIR)
                            tc::mbar_wait_cluster(&full[s], ph);
                        else
                            mbar_wait(&full[s], ph);
                        tc::fence_after_sync();
                        const uint32_t abase = smem_u32(ring + (size_t)s * LOAD_BYTES);
                        const uint32_t bbase = abase + A_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            // MN-major SW128: 64-element x 8-row atoms; SBO = next 8 rows (1 KB),
                            // LBO = next 64 features (8 KB); a K step of 16 rows = 2 KB
                            const uint64_t ad = tc::smem_desc_sw128(abase + k * 2048, 8192, 1024);
                            const uint64_t bd = tc::smem_desc_sw128(bbase + k * 2048, 8192, 1024);
                            if constexpr (PAIR)
                                tc::mma_bf16_pair(dcol, ad, bd, idesc, (kb | k) != 0);
                            else
                                tc::mma_bf16(dcol, ad, bd, idesc, (kb | k) != 0);
                        }
                        // smem slot free once these MMAs retire (PAIR: in both CTAs)
                        if constexpr (PAIR)
                            tc::commit_pair(&empty[s], 0x3);
                        else
                            tc::commit(&empty[s]);
                        if (++s == NST) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                    // accumulator of example b complete
                    if constexpr (PAIR)
                        tc::commit_pair(&tfull[buf], 0x3);
                    else
                        tc::commit(&tfull[buf]);
                    if (++buf == 2) {
                        buf = 0;
                        tph ^= 1u;
                    }
                }
            }
        }
    } else {
        // --------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const int quad = warp & 3;      // TMEM lanes this warp may access
        const int half = e / 4;         // column half of the 256-wide tile
        const int row = quad * 32 + lane;
        unsigned* flag = reinterpret_cast<unsigned*>(red + EPI_WARPS);
        int buf = 0;
        uint32_t tph = 0;
        float S[128];
        // fixed-order fold of per-warp float partials -> one double (thread e==0, lane 0).
        // (Writing one slot per warp instead, with no named barriers, measured
        // slower: cfg3 799.5 us against 780 us, 2.12 ms against 1.80 ms at T = 128.)
        auto fold8 = [&](float v, double* dst) {
            v = warp_sum(v);
            if (lane == 0) red[e] = v;
            named_bar_sync(1, EPI_WARPS * 32);
            if (e == 0 && lane == 0) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < EPI_WARPS; ++w) t += (double)red[w];
                *dst = t;
            }
            named_bar_sync(1, EPI_WARPS * 32);
        };
        auto store_tile = [&](int tile) {
            const int i0 = (tile % a.tiles_m) * BM, j0 = (tile / a.tiles_m) * BN;
            float sb = 0.f;
#pragma unroll
            for (int c = 0; c < 128; ++c) sb = fmaf(S[c], S[c], sb);
            fold8(sb, &a.qbig[tile]);
            if (a.dW != nullptr && i0 + row < a.K) {  // tile tails past K / L are not stored
                const int c0 = j0 + half * 128;
                float4* dst = reinterpret_cast<float4*>(a.dW + (size_t)(i0 + row) * a.L + c0);
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (c0 + 4 * c < a.L) dst[c] = make_float4(S[4 * c], S[4 * c + 1], S[4 * c + 2], S[4 * c + 3]);
            }
        };
        // A tile whose examples are split over several CTAs: every part is
        // parked in the workspace; the last CTA to finish (ticket) sums the
        // parts in CTA order, so the result is deterministic.
        auto flush_tile = [&](int tile, int nparts, int mypart) {
            if (nparts == 1) {
                store_tile(tile);
                return;
            }
            auto slot = [&](int p) {
                return reinterpret_cast<float4*>(a.part + (((size_t)tile * a.max_parts + p) * BM + row) * BN + half * 128);
            };
            float4* mine = slot(mypart);
#pragma unroll
            for (int c = 0; c < 32; ++c) mine[c] = make_float4(S[4 * c], S[4 * c + 1], S[4 * c + 2], S[4 * c + 3]);
            __threadfence();
            named_bar_sync(1, EPI_WARPS * 32);
            if (e == 0 && lane == 0) *flag = atomicAdd(&a.ticket[tile], 1u);
            named_bar_sync(1, EPI_WARPS * 32);
            if (*flag != (unsigned)(nparts - 1)) return;  // not the last part: done
            __threadfence();
#pragma unroll
            for (int c = 0; c < 128; ++c) S[c] = 0.f;
            for (int p = 0; p < nparts; ++p) {
                const float4* src = slot(p);
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const float4 v = __ldcg(src + c);
                    S[4 * c] += v.x;
                    S[4 * c + 1] += v.y;
                    S[4 * c + 2] += v.z;
                    S[4 * c + 3] += v.w;
                }
            }
            if (e == 0 && lane == 0) a.ticket[tile] = 0u;
            store_tile(tile);
        };
        const uint32_t tempty_leader = PAIR ? tc::mapa(smem_u32(&tempty[0]), 0) : 0u;
        for (int si = 0; si < nseg; ++si) {
            int stile, b0, b1, nparts, mypart;
            segment(si, stile, b0, b1, nparts, mypart);
            const int tile = sub_of(stile);
#pragma unroll
            for (int cc = 0; cc < 128; ++cc) S[cc] = 0.f;
            for (int b = b0; b < b1; ++b) {
                if constexpr (PAIR)
                    tc::mbar_wait_cluster(&tfull[buf], tph);
                else
                    mbar_wait(&tfull[buf], tph);
                tc::fence_after_sync();
                float sq = 0.f;
                const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + half * 128);
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(base + cc * 32, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const float v = __uint_as_float(r[k]);
                        sq = fmaf(v, v, sq);
                        S[cc * 32 + k] += v;
                    }
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR)
                        tc::mbar_arrive_cluster(tempty_leader + (uint32_t)(buf * 8));
                    else
                        mbar_arrive(&tempty[buf]);
                }
                fold8(sq, &a.q[(size_t)b * ntiles + tile]);  // the sub-tile's share of raw_b
                if (++buf == 2) {
                    buf = 0;
                    tph ^= 1u;
                }
            }
            flush_tile(tile, nparts, mypart);
        }
    }
    tc::fence_before_sync();
    if constexpr (PAIR)
        tc::cluster_sync();
    else
        __syncthreads();
    if (warp == 1) {
        tc::fence_after_sync();
        if constexpr (PAIR)
            tc::tmem_dealloc_pair<TMEM_COLS>(tmem);
        else
            tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// raw[b] = sum_j q[b][j] (fixed order), sums[sum_slot] = sum_b raw[b] (fixed
// order); with q2: also sums[slot2] = sum_j q2[j] (a second, one-row fold in
// the same launch -- the squared norm of the batch gradient)
constexpr int kFoldSmemRows = 4096;
__global__ void __launch_bounds__(256) fold_rows_kernel(const double* q, int nb, int ncol, double* raw, double* sums,
                                                        int sum_slot, const double* q2 = nullptr, int ncol2 = 0,
                                                        int slot2 = 0) {
    __shared__ double rs[kFoldSmemRows];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto rowof = [&](const double* r, int n) {  // 8 independent partial sums per lane: loads in flight, fixed order
        double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int j = lane;
        for (; j + 32 * 7 < n; j += 32 * 8)
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] += __ldcg(r + j + 32 * u);
        for (; j < n; j += 32) t[0] += __ldcg(r + j);
        return warp_sum(((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7])));
    };
    if (q2 != nullptr && sums != nullptr && warp == (int)(blockDim.x / 32) - 1) {
        const double t = rowof(q2, ncol2);
        if (lane == 0) sums[slot2] = t;
    }
    auto row = [&](int b) {
        double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const double* r = q + (size_t)b * ncol;
        int j = lane;
        for (; j + 32 * 7 < ncol; j += 32 * 8)
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] += __ldcg(r + j + 32 * u);
        for (; j < ncol; j += 32) t[0] += __ldcg(r + j);
        return warp_sum(((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7])));
    };
    for (int b = warp; b < nb; b += blockDim.x / 32) {
        const double t = row(b);
        if (lane == 0) {
            if (raw) raw[b] = t;
            if (b < kFoldSmemRows) rs[b] = t;
        }
    }
    __syncthreads();
    if (sums == nullptr || warp != 0) return;
    double t = 0.0;
    for (int b = 0; b < nb; ++b) {
        const double r = b < kFoldSmemRows ? rs[b] : row(b);  // (rows beyond the buffer are recomputed)
        t += r;
    }
    if (lane == 0) sums[sum_slot] = t;
}

cudaError_t launch_fold_rows(const double* q, int nb, int ncol, double* raw, double* sums, int sum_slot,
                             cudaStream_t st) {
    fold_rows_kernel<<<1, 256, 0, st>>>(q, nb, ncol, raw, sums, sum_slot);
    return cudaGetLastError();
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

// [B, T, F] bf16 row-major viewed as a 3-D tensor (F innermost), box 64 x 64 x 1, 128B swizzle
bool make_map_btf(CUtensorMap* m, const void* base, int B, int T, int F) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)F, (cuuint64_t)T, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)F * 2, (cuuint64_t)T * F * 2};
    cuuint32_t box[3] = {64, 64, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Any T, K, L with 16-byte row strides (K, L multiples of 8): TMA zero-fills
// tokens past T and features past K / L; the epilogue stores only dW's
// in-range rows and columns.
bool wgrad_shape_ok(int64_t B, int64_t T, int64_t K, int64_t L) {
    return B >= 1 && T >= 1 && K % 8 == 0 && L % 8 == 0 && K > 0 && L > 0 && K < (1 << 30) && L < (1 << 30) &&
           T < (1 << 30) && B < (1 << 30);
}

namespace {
int wgrad_max_parts(int64_t B, int64_t tiles, int grid) {
    const int64_t R = tiles % grid;
    if (R == 0) return 1;
    const int64_t P = grid / R;
    return (int)(P < B ? P : B);
}
// the CTA-pair kernel (256 x 256 tiles over a 2-CTA cluster) unless K is not a
// multiple of 256 or GNSB_WGRAD_IMPL=1 selects the single-CTA kernel
bool wgrad_use_pair(int64_t K) {
    if (K % (2 * wg::BM) != 0) return false;
    const char* impl = std::getenv("GNSB_WGRAD_IMPL");
    return !(impl && impl[0] == '1');
}
// scheduled tiles and the number of schedulers (CTAs, or CTA pairs)
struct WgradSched {
    int64_t stiles;
    int grid;
    int max_parts;
};
WgradSched wgrad_sched(int64_t B, int64_t K, int64_t L, bool pair) {
    WgradSched w;
    w.stiles = ((K + wg::BM - 1) / wg::BM / (pair ? 2 : 1)) * ((L + wg::BN - 1) / wg::BN);
    const int64_t units = w.stiles * B;
    const int sms = pair ? device_sm_count() / 2 : device_sm_count();
    w.grid = (int)(units < sms ? units : sms);
    w.max_parts = wgrad_max_parts(B, w.stiles, w.grid);
    return w;
}
struct WgradLayout {
    size_t q, qbig, ticket, part, total;
};
WgradLayout wgrad_layout(int64_t B, int64_t K, int64_t L, int max_parts) {
    const int64_t tiles = ((K + wg::BM - 1) / wg::BM) * ((L + wg::BN - 1) / wg::BN);  // 128 x 256 sub-tiles
    WgradLayout w;
    w.q = 0;
    w.qbig = (size_t)B * tiles * sizeof(double);
    w.ticket = (w.qbig + (size_t)tiles * sizeof(double) + 255) / 256 * 256;
    w.part = (w.ticket + (size_t)tiles * sizeof(unsigned) + 255) / 256 * 256;
    w.total = w.part + (size_t)tiles * max_parts * wg::BM * wg::BN * sizeof(float);
    return w;
}
// (grid may exceed the tile count: the extra CTAs take example ranges of tiles)
}  // namespace

size_t wgrad_workspace(int64_t B, int64_t K, int64_t L) {
    // large enough for either kernel (the choice may change with the environment)
    int mp = wgrad_sched(B, K, L, false).max_parts;
    if (K % (2 * wg::BM) == 0) {
        const int m2 = wgrad_sched(B, K, L, true).max_parts;
        mp = m2 > mp ? m2 : mp;
    }
    return wgrad_layout(B, K, L, mp).total;
}

cudaError_t launch_wgrad_norms(const void* x, const void* g, float* dW, double* raw, double* sums, int64_t B,
                               int64_t T, int64_t K, int64_t L, void* ws, cudaStream_t st) {
    CUtensorMap mx, mg;
    if (!make_map_btf(&mx, x, (int)B, (int)T, (int)K) || !make_map_btf(&mg, g, (int)B, (int)T, (int)L))
        return cudaErrorInvalidValue;
    const bool pair = wgrad_use_pair(K);
    const void* fn = pair ? reinterpret_cast<const void*>(wgrad_norms_kernel<true>)
                          : reinterpret_cast<const void*>(wgrad_norms_kernel<false>);
    cudaError_t e = ensure_smem_attr(fn, wg::SMEM);
    if (e != cudaSuccess) return e;
    WgradArgs a{};
    a.B = (int)B;
    a.T = (int)T;
    a.K = (int)K;
    a.L = (int)L;
    a.tiles_m = (int)((K + wg::BM - 1) / wg::BM);
    a.tiles_n = (int)((L + wg::BN - 1) / wg::BN);
    a.dW = dW;
    const int ntiles = a.tiles_m * a.tiles_n;
    const WgradSched sc = wgrad_sched(B, K, L, pair);
    const WgradLayout w = wgrad_layout(B, K, L, sc.max_parts);
    unsigned char* base = static_cast<unsigned char*>(ws);
    a.q = reinterpret_cast<double*>(base + w.q);
    a.qbig = reinterpret_cast<double*>(base + w.qbig);
    a.ticket = reinterpret_cast<unsigned*>(base + w.ticket);
    a.part = reinterpret_cast<float*>(base + w.part);
    a.max_parts = sc.max_parts;
    // the split-tile tickets must start at zero; the workspace may have been
    // used by another linear-path kernel with a different layout since
    if (a.max_parts > 1) {
        cudaError_t me = cudaMemsetAsync(a.ticket, 0, (size_t)ntiles * sizeof(unsigned), st);
        if (me != cudaSuccess) return me;
    }
    if (pair) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * sc.grid);
        cfg.blockDim = dim3(wg::THREADS);
        cfg.dynamicSmemBytes = wg::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, wgrad_norms_kernel<true>, mx, mg, a);
    } else {
        wgrad_norms_kernel<false><<<sc.grid, wg::THREADS, wg::SMEM, st>>>(mx, mg, a);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    fold_rows_kernel<<<1, 256, 0, st>>>(a.q, (int)B, ntiles, raw, sums, 0, a.qbig, ntiles, 2);
    return cudaGetLastError();
}

// -------------------------------------------------------- generic paths --
// Any shape and dtype, fp64 accumulation: used when the tensor-core tiling
// does not apply (unaligned K/L/T, fp32/fp64 rows).  One thread per weight
// entry (i, j); per example b it forms dW_b[i, j] = sum_t x*g in fixed t
// order, adds it to dW and contributes its square to the block's share of
// raw_b (fixed-order block tree).
// fp64 rows: the reference's accumulation without contraction (layers.cpp:107-131)
template <typename T>
__device__ __forceinline__ double mac(double acc, double a, double b) {
    if constexpr (std::is_same<T, double>::value) return __dadd_rn(acc, __dmul_rn(a, b));
    return fma(a, b, acc);
}

// pe (fp64 rows, nullable): the per-example values dW_b / bias'_b [B][n] for
// the reference-order norms (launch_seq_sqnorm)
template <typename T>
__global__ void __launch_bounds__(256) wgrad_generic_kernel(const T* x, const T* g, int64_t B, int64_t Tn, int64_t K,
                                                            int64_t L, void* dW, int dw_f64, double* q, int nblk,
                                                            double* pe) {
    __shared__ double red[256];
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = idx < K * L;
    const int64_t i = ok ? idx / L : 0, j = ok ? idx % L : 0;
    double S = 0.0;
    for (int64_t b = 0; b < B; ++b) {
        double v = 0.0;
        if (ok)
            for (int64_t t = 0; t < Tn; ++t)
                v = mac<T>(v, (double)to_acc<T>(x[(b * Tn + t) * K + i]), (double)to_acc<T>(g[(b * Tn + t) * L + j]));
        if (pe && ok) pe[b * K * L + idx] = v;
        S = std::is_same<T, double>::value ? __dadd_rn(S, v) : S + v;
        red[threadIdx.x] = v * v;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) q[(size_t)b * nblk + blockIdx.x] = red[0];
        __syncthreads();
    }
    red[threadIdx.x] = S * S;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) q[(size_t)B * nblk + blockIdx.x] = red[0];
    if (ok && dW) {
        if (dw_f64)
            static_cast<double*>(dW)[idx] = S;
        else
            static_cast<float*>(dW)[idx] = (float)S;
    }
}

// per-example bias gradients: bias'_b[j] = sum_t g[b,t,j]; dbias = sum_b; ||bias'_b||^2
template <typename T>
__global__ void __launch_bounds__(256) bias_pe_kernel(const T* g, int64_t B, int64_t Tn, int64_t L, void* db,
                                                      int db_f64, double* q, int nblk, double* pe) {
    __shared__ double red[256];
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = j < L;
    double S = 0.0;
    for (int64_t b = 0; b < B; ++b) {
        double v = 0.0;
        if (ok)
            for (int64_t t = 0; t < Tn; ++t) v = __dadd_rn(v, (double)to_acc<T>(g[(b * Tn + t) * L + j]));
        if (pe && ok) pe[b * L + j] = v;
        S = __dadd_rn(S, v);
        red[threadIdx.x] = v * v;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) q[(size_t)b * nblk + blockIdx.x] = red[0];
        __syncthreads();
    }
    red[threadIdx.x] = S * S;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) q[(size_t)B * nblk + blockIdx.x] = red[0];
    if (ok && db) {
        if (db_f64)
            static_cast<double*>(db)[j] = S;
        else
            static_cast<float*>(db)[j] = (float)S;
    }
}


// ------------------------------------------------- bias, fp32 / bf16 rows --
// bias'_b[j] = sum_t g[b,t,j], raw_b = ||bias'_b||^2, dbias = sum_b bias'_b
// (layers.cpp:118-119, 125-130) as an HBM stream: pass 1, grid (column
// chunks, examples, token chunks), a thread owns 8 columns and sums its token
// chunk (fp32 partials [B][TC][L]); pass 2, a thread per 8 columns combines
// the token chunks in order (fp64) per example, adds the squares into a
// per-(example, CTA) slot and the examples into dbias.  No atomics; the
// generic kernel (one thread per column, every token in sequence) stays for
// fp64 rows (reference order) and unaligned shapes.
constexpr int kBiasRows = 64;  // tokens per pass-1 chunk
template <typename T>
__global__ void __launch_bounds__(256) bias_part_kernel(const T* __restrict__ g, int64_t Tn, int64_t L, int TC,
                                                        float* __restrict__ part) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 8-column vector
    const int64_t b = blockIdx.y, tc = blockIdx.z;
    if (v * 8 >= L) return;
    const int64_t t0 = tc * kBiasRows, t1 = t0 + kBiasRows < Tn ? t0 + kBiasRows : Tn;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const T* base = g + (b * Tn) * L + v * 8;
#pragma unroll 4
    for (int64_t t = t0; t < t1; ++t) {
        float f[8];
        if constexpr (std::is_same<T, float>::value) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(base + t * L));
            const float4 c = __ldg(reinterpret_cast<const float4*>(base + t * L + 4));
            f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = c.x, f[5] = c.y, f[6] = c.z, f[7] = c.w;
        } else {
            unpack<T>(__ldg(reinterpret_cast<const uint4*>(base + t * L)), f);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += f[k];
    }
    float4* dst = reinterpret_cast<float4*>(part + ((b * TC + tc) * L) + v * 8);
    dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

__global__ void __launch_bounds__(256) bias_combine_kernel(const float* __restrict__ part, int64_t B, int TC, int64_t L,
                                                           float* __restrict__ dbias, double* __restrict__ q,
                                                           double* __restrict__ qbig) {
    __shared__ double s_red[256 / 32];
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = v * 8 < L;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t b = 0; b < B; ++b) {
        double sq = 0.0;
        if (ok) {
            double e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int tc = 0; tc < TC; ++tc) {
                const float4* src = reinterpret_cast<const float4*>(part + ((b * TC + tc) * L) + v * 8);
                const float4 a = __ldg(src), c = __ldg(src + 1);
                e[0] += a.x, e[1] += a.y, e[2] += a.z, e[3] += a.w, e[4] += c.x, e[5] += c.y, e[6] += c.z, e[7] += c.w;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                sq = fma(e[k], e[k], sq);
                tot[k] += e[k];
            }
        }
        sq = warp_sum(sq);
        if (lane == 0) s_red[warp] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 256 / 32; ++w) t += s_red[w];
            q[b * gridDim.x + blockIdx.x] = t;
        }
        __syncthreads();
    }
    double sb = 0.0;
    if (ok) {
        float4* dst = reinterpret_cast<float4*>(dbias + v * 8);
        const float4 o0 = make_float4((float)tot[0], (float)tot[1], (float)tot[2], (float)tot[3]);
        const float4 o1 = make_float4((float)tot[4], (float)tot[5], (float)tot[6], (float)tot[7]);
        dst[0] = o0;
        dst[1] = o1;
        const float of[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) sb = fma((double)of[k], (double)of[k], sb);
    }
    sb = warp_sum(sb);
    if (lane == 0) s_red[warp] = sb;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 256 / 32; ++w) t += s_red[w];
        qbig[blockIdx.x] = t;
    }
}

bool bias_fast_ok(int dt, int64_t L, const void* g, const void* dbias) {
    return (dt == 0 || dt == 1) && L % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15u) == 0 &&
           (reinterpret_cast<uintptr_t>(dbias) & 15u) == 0;
}
size_t bias_fast_workspace(int64_t B, int64_t T, int64_t L) {
    const int64_t TC = (T + kBiasRows - 1) / kBiasRows, nblk = (L / 8 + 255) / 256;
    return (size_t)B * TC * L * 4 + (size_t)(B + 1) * nblk * 8 + 512;
}
cudaError_t launch_bias_fast(int dt, const void* g, void* dbias, double* raw, double* sums, int64_t B, int64_t T,
                             int64_t L, void* ws, cudaStream_t st) {
    const int TC = (int)((T + kBiasRows - 1) / kBiasRows);
    const int64_t nv = L / 8;
    const unsigned nblk = (unsigned)((nv + 255) / 256);
    float* part = static_cast<float*>(ws);
    double* q = reinterpret_cast<double*>(static_cast<unsigned char*>(ws) + ((size_t)B * TC * L * 4 + 255) / 256 * 256);
    double* qbig = q + B * nblk;
    const dim3 g1(nblk, (unsigned)B, (unsigned)TC);
    if (dt == 0)
        bias_part_kernel<float><<<g1, 256, 0, st>>>(static_cast<const float*>(g), T, L, TC, part);
    else
        bias_part_kernel<__nv_bfloat16><<<g1, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(g), T, L, TC, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    bias_combine_kernel<<<nblk, 256, 0, st>>>(part, B, TC, L, static_cast<float*>(dbias), q, qbig);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fold_rows_kernel<<<1, 256, 0, st>>>(q, (int)B, (int)nblk, raw, sums, 1, qbig, (int)nblk, 3);
    return cudaGetLastError();
}

// Gram form, generic: raw_b = sum_{t,u} (x_t . x_u)(g_t . g_u), one thread per (t, u)
template <typename T>
__global__ void __launch_bounds__(256) gram_generic_kernel(const T* x, const T* g, int64_t B, int64_t Tn, int64_t K,
                                                           int64_t L, double* q, int nblk) {
    __shared__ double red[256];
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = idx < Tn * Tn;
    const int64_t t = ok ? idx / Tn : 0, u = ok ? idx % Tn : 0;
    for (int64_t b = 0; b < B; ++b) {
        double xx = 0.0, gg = 0.0;
        if (ok) {
            for (int64_t i = 0; i < K; ++i)
                xx += (double)to_acc<T>(x[(b * Tn + t) * K + i]) * (double)to_acc<T>(x[(b * Tn + u) * K + i]);
            for (int64_t j = 0; j < L; ++j)
                gg += (double)to_acc<T>(g[(b * Tn + t) * L + j]) * (double)to_acc<T>(g[(b * Tn + u) * L + j]);
        }
        red[threadIdx.x] = xx * gg;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) q[(size_t)b * nblk + blockIdx.x] = red[0];
        __syncthreads();
    }
}

size_t generic_workspace(int64_t B, int64_t T, int64_t K, int64_t L) {
    const int64_t n1 = (K * L + 255) / 256, n2 = (L + 255) / 256, n3 = (T * T + 255) / 256;
    int64_t n = n1 > n2 ? n1 : n2;
    n = n > n3 ? n : n3;
    return (size_t)(B + 1) * n * sizeof(double) + 256;
}
// fp64 rows: + the per-example values [B][K*L] and a raw buffer [B] after the
// generic area (reference-order norms)
size_t generic_workspace_f64(int64_t B, int64_t T, int64_t K, int64_t L) {
    return (generic_workspace(B, T, K, L) + 255) / 256 * 256 + (size_t)B * (K * L + 1) * sizeof(double);
}

template <typename T>
cudaError_t launch_generic_t(int kind, const void* x, const void* g, void* out_grad, int out_f64, double* raw,
                             double* sums, int sum_slot, int64_t B, int64_t Tn, int64_t K, int64_t L, void* ws,
                             cudaStream_t st) {
    double* q = static_cast<double*>(ws);
    int nblk = 0;
    // fp64 rows: per-example values for the reference-order norms
    constexpr bool REF = std::is_same<T, double>::value;
    double* pe = REF && kind != 2
                     ? reinterpret_cast<double*>(static_cast<unsigned char*>(ws) +
                                                 (generic_workspace(B, Tn, kind == 0 ? K : 1, L) + 255) / 256 * 256)
                     : nullptr;
    if (kind == 0) {  // weight, simultaneous form
        nblk = (int)((K * L + 255) / 256);
        wgrad_generic_kernel<T><<<nblk, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(g), B, Tn, K, L,
                                                      out_grad, out_f64, q, nblk, pe);
    } else if (kind == 1) {  // bias
        nblk = (int)((L + 255) / 256);
        bias_pe_kernel<T><<<nblk, 256, 0, st>>>(static_cast<const T*>(g), B, Tn, L, out_grad, out_f64, q, nblk, pe);
    } else {  // Gram form (norms only)
        nblk = (int)((Tn * Tn + 255) / 256);
        gram_generic_kernel<T><<<nblk, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(g), B, Tn, K, L,
                                                     q, nblk);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (pe) {  // raw_b and sum_b raw_b in the reference's order
        const int64_t n = kind == 0 ? K * L : L;
        e = launch_seq_sqnorm(pe, B, n, raw ? raw : pe + B * n, sums, sum_slot, st);
        if (e != cudaSuccess) return e;
    } else {
        fold_rows_kernel<<<1, 256, 0, st>>>(q, (int)B, nblk, raw, sums, sum_slot);
    }
    if (sums && kind != 2) fold_rows_kernel<<<1, 256, 0, st>>>(q + (size_t)B * nblk, 1, nblk, nullptr, sums, sum_slot + 2);
    return cudaGetLastError();
}

cudaError_t launch_linear_generic(int dt, int kind, const void* x, const void* g, void* out_grad, int out_f64,
                                  double* raw, double* sums, int sum_slot, int64_t B, int64_t T, int64_t K, int64_t L,
                                  void* ws, cudaStream_t st) {
    // fp32 rows, weight-gradient or Gram form: 3xTF32 tensor cores (linear_f32.cu)
    if ((kind == 0 || kind == 2) && wgrad_tf32_ok(dt, x, g, kind == 0 ? out_grad : nullptr, T, K, L))
        return launch_wgrad_tf32(static_cast<const float*>(x), static_cast<const float*>(g),
                                 kind == 0 ? static_cast<float*>(out_grad) : nullptr, raw, sums, sum_slot, B, T, K, L,
                                 st);
    switch (dt) {
        case 0: return launch_generic_t<float>(kind, x, g, out_grad, out_f64, raw, sums, sum_slot, B, T, K, L, ws, st);
        case 1:
            return launch_generic_t<__nv_bfloat16>(kind, x, g, out_grad, out_f64, raw, sums, sum_slot, B, T, K, L, ws,
                                                   st);
        case 2: return launch_generic_t<double>(kind, x, g, out_grad, out_f64, raw, sums, sum_slot, B, T, K, L, ws, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace gnsb

// linear_gemm.cu — the two dense GEMMs of a linear layer on sm_100a tensor
// cores (tcgen05 + TMEM + TMA), any row count and tile tails:
//
//   forward   y[r, l]  = sum_k x[r, k] W[k, l] (+ bias[l])   (proj/src/layers.cpp:52-78)
//   input grad dx[r, k] = sum_l g[r, l] W[k, l]               (proj/src/layers.cpp:142-155)
//
// Both are D[M=rows, N] = A[M, Kr] * B with A the row tensor (K-major: the
// reduced axis is contiguous).  B is W read in place: MN-major for the
// forward (W[k, :] contiguous along N = L), K-major for dx (W[k, :]
// contiguous along the reduced L).  bf16 operands, fp32 accumulation in TMEM.
//
// Kernel (gemm_kernel<B_KMAJOR, BIAS>): persistent, one CTA per SM, static
// round-robin over 128 x 256 output tiles with the N tile fastest (the CTAs
// of one wave share an A row block through L2; W stays L2-resident).
//   warp 0      TMA producer: A box 64 x 128 (16 KB) and B 64 x 256 (32 KB)
//               per 64-deep K block into a 4-stage ring; rows, columns and K
//               past the tensor are zero-filled by TMA, so no shape is
//               special-cased;
//   warp 1      one elected thread issues tcgen05.mma M=128 N=256 K=16 into
//               one of two 256-column TMEM accumulators (tiles alternate, so
//               the epilogue of tile i overlaps the MMAs of tile i+1);
//   warps 2..9  epilogue: tcgen05.ld 32 columns at a time, + bias, round to
//               bf16, 16-byte stores (rows / columns past the output skipped).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace gnsb {

namespace gm {
constexpr int BM = 128, BN = 256, BK = 64;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int OUT_BOX_BYTES = 32 * 128;      // one epilogue warp's store box: 32 rows x 64 bf16 (128B swizzle)
// align slack + ring + barrier block (1 KB) + the epilogue store boxes
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024 + (size_t)EPI_WARPS * OUT_BOX_BYTES;
static_assert(SMEM <= 232448, "dynamic shared memory of one CTA");
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 8;  // tile raster: GROUP_M row blocks x all column tiles, row block fastest
}  // namespace gm

// TMA store of a staged shared-memory box to global (bulk async group)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// tile index -> (row block, column tile): GROUP_M row blocks share a band of
// column tiles so one wave of CTAs reuses both A row blocks and W column
// tiles through L2 (a plain column-fastest order re-reads W from DRAM once
// W outgrows L2)
__device__ __forceinline__ void tile_mn(int t, int tiles_m, int tiles_n, int& mt, int& nt) {
    const int band = t / (gm::GROUP_M * tiles_n);
    const int first = band * gm::GROUP_M;
    const int rows = tiles_m - first < gm::GROUP_M ? tiles_m - first : gm::GROUP_M;
    const int local = t - band * gm::GROUP_M * tiles_n;
    mt = first + local % rows;
    nt = local / rows;
}

// Epilogues fused into the store (the toy model's elementwise ops,
// proj/src/model.cpp:95-100 and :169-171): v = acc (+ bias), then
//   EPI_NONE  out = v
//   EPI_TANH  out = tanh(v)                 (fc1 forward)
//   EPI_RESID out = aux + v                 (fc2 forward + residual)
//   EPI_DTANH out = v * (1 - aux^2)         (fc2 input grad through the tanh, aux = tanh output)
enum { EPI_NONE = 0, EPI_TANH = 1, EPI_RESID = 2, EPI_DTANH = 3 };

template <int EPI, typename A>
__device__ __forceinline__ A epi_apply(A v, A aux) {
    if constexpr (EPI == EPI_TANH) return tanh(v);
    if constexpr (EPI == EPI_RESID) return aux + v;
    if constexpr (EPI == EPI_DTANH) return v * (A(1) - aux * aux);
    return v;
}

struct GemmArgs {
    int M, N, Kr;         // output rows, output columns, reduced extent
    int tiles_m, tiles_n;
    const float* bias;    // [N] (BIAS)
    const __nv_bfloat16* aux;  // [M, N] (EPI_RESID, EPI_DTANH)
    __nv_bfloat16* out;   // [M, N]
    int ksplit;           // split-K parts (SPLIT)
    float* part;          // [ksplit][M][N] fp32 partials (SPLIT)
};

// split-K combine: out = epi(sum_p part[p] (+ bias)), parts in fixed order
template <int EPI, bool BIAS>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ part, int ksplit, int64_t M,
                                                            int64_t N, const float* __restrict__ bias,
                                                            const __nv_bfloat16* __restrict__ aux,
                                                            __nv_bfloat16* __restrict__ out) {
    const int64_t n8 = N / 8, total = M * n8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / n8, c = (i - r * n8) * 8;
        float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int p = 0; p < ksplit; ++p) {
            const float4* src = reinterpret_cast<const float4*>(part + ((size_t)p * M + r) * N + c);
            const float4 u = __ldg(src), w = __ldg(src + 1);
            f[0] += u.x, f[1] += u.y, f[2] += u.z, f[3] += u.w, f[4] += w.x, f[5] += w.y, f[6] += w.z, f[7] += w.w;
        }
        if constexpr (BIAS) {
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] += __ldg(bias + c + j);
        }
        if constexpr (EPI != EPI_NONE) {
            float x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if constexpr (EPI == EPI_RESID || EPI == EPI_DTANH)
                unpack<__nv_bfloat16>(__ldg(reinterpret_cast<const uint4*>(aux + r * N + c)), x);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = epi_apply<EPI>(f[j], x[j]);
        }
        uint4 o;
        o.x = pack_bf16x2(f[0], f[1]);
        o.y = pack_bf16x2(f[2], f[3]);
        o.z = pack_bf16x2(f[4], f[5]);
        o.w = pack_bf16x2(f[6], f[7]);
        *reinterpret_cast<uint4*>(out + r * N + c) = o;
    }
}

// BNT: output tile width, 256 (default) or 128 (skinny outputs: more tiles,
// fewer idle SMs in the last wave; the ring then holds 6 stages in the same
// shared memory)
// SPLIT: split-K.  Work unit u = (tile u / ksplit, K part u % ksplit); the
// epilogue stores the part's fp32 partial tile to a.part [ksplit][M][N] and
// splitk_reduce_kernel sums the parts in order and applies bias / epilogue
// (deterministic).  For outputs with few tiles and a long reduction (N = 768
// at 8192 rows: 192 tiles = 1.3 waves on 148 SMs).
template <bool B_KMAJOR, bool BIAS, int EPI, int BNT = gm::BN, bool SPLIT = false>
__global__ void __launch_bounds__(gm::THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                const __grid_constant__ CUtensorMap tmo, GemmArgs a) {
    using gm::BM;
    using gm::BK;
    using gm::A_BYTES;
    using gm::EPI_WARPS;
    using gm::OUT_BOX_BYTES;
    using gm::TMEM_COLS;
    constexpr int BN = BNT;
    constexpr int STAGE_BYTES = A_BYTES + BN * BK * 2;
    constexpr int STAGES = gm::STAGES * gm::STAGE_BYTES / STAGE_BYTES;  // same ring bytes
    static_assert(STAGES * STAGE_BYTES <= gm::STAGES * gm::STAGE_BYTES, "ring");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)gm::STAGES * gm::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    unsigned char* obox = smem + (size_t)gm::STAGES * gm::STAGE_BYTES + 1024;  // [EPI_WARPS][32 rows][128 B], 1 KB aligned

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ksplit = SPLIT ? a.ksplit : 1;
    const int ntiles = a.tiles_m * a.tiles_n * ksplit;  // work units
    const int kblocks_all = (a.Kr + BK - 1) / BK;
    auto krange = [&](int u, int& kb0, int& kb1) {
        const int p = SPLIT ? u % ksplit : 0;
        kb0 = (int)((int64_t)kblocks_all * p / ksplit);
        kb1 = (int)((int64_t)kblocks_all * (p + 1) / ksplit);
    };

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
        tc::prefetch_tmap(&tma);
        tc::prefetch_tmap(&tmb);
        tc::prefetch_tmap(&tmo);
    }
    if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    // the inputs may be produced by the previous kernel in the stream (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0) {
        // -------------------------------------------------------- producer --
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mt, nt, kb0, kb1;
                tile_mn(t / ksplit, a.tiles_m, a.tiles_n, mt, nt);
                krange(t, kb0, kb1);
                const int m0 = mt * BM, n0 = nt * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char* st = ring + (size_t)s * STAGE_BYTES;
                    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                    const int k0 = kb * BK;
                    tc::tma_load_3d(st, &tma, k0, m0, 0, &full[s]);  // A: 64 (K) x 128 rows
                    if constexpr (B_KMAJOR) {
                        tc::tma_load_3d(st + A_BYTES, &tmb, k0, n0, 0, &full[s]);  // B: 64 (K) x 256 rows
                    } else {
#pragma unroll
                        for (int h = 0; h < BN / 64; ++h)  // B: 64 (N) x 64 (K) chunks along N
                            tc::tma_load_3d(st + A_BYTES + h * 8192, &tmb, n0 + 64 * h, k0, 0, &full[s]);
                    }
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer --
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, !B_KMAJOR);
            int s = 0, buf = 0;
            uint32_t ph = 0, tph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&tempty[buf], tph ^ 1u);  // epilogue drained this accumulator
                tc::fence_after_sync();
                const uint32_t dcol = tmem + (uint32_t)(buf * BN);
                int kb0, kb1;
                krange(t, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t abase = smem_u32(ring + (size_t)s * STAGE_BYTES);
                    const uint32_t bbase = abase + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // K-major SW128: 8-row x 128-byte atoms (SBO 1 KB), a K step of 16 = 32 bytes;
                        // MN-major SW128: 64-element x 8-row atoms, LBO = next 64 columns (8 KB),
                        // SBO = next 8 K rows (1 KB), a K step of 16 rows = 2 KB
                        const uint64_t ad = tc::smem_desc_sw128(abase + k * 32, 16, 1024);
                        const uint64_t bd = B_KMAJOR ? tc::smem_desc_sw128(bbase + k * 32, 16, 1024)
                                                     : tc::smem_desc_sw128(bbase + k * 2048, 8192, 1024);
                        tc::mma_bf16(dcol, ad, bd, idesc, (kb != kb0) || (k != 0));
                    }
                    tc::commit(&empty[s]);  // smem slot free once these MMAs retire
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc::commit(&tfull[buf]);  // accumulator of this tile complete
                if (++buf == 2) {
                    buf = 0;
                    tph ^= 1u;
                }
            }
        }
    } else {
        // -------------------------------------------------------- epilogue --
        // Each warp owns 32 TMEM lanes (rows) x 128 columns of the tile.  Per
        // 64-column group it rounds its values to bf16 into a 32 x 64 box in
        // shared memory (128-byte swizzle: conflict-free 16-byte writes) and
        // one lane stores the box with TMA (coalesced; rows / columns past the
        // output are clipped by the tensor map).
        const int e = warp - 2;
        const int quad = warp & 3;  // TMEM lanes this warp may access
        const int half = e / 4;     // column half of the tile
        unsigned char* box = obox + (size_t)e * OUT_BOX_BYTES;
        int buf = 0;
        uint32_t tph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int mt, nt;
            tile_mn(t / ksplit, a.tiles_m, a.tiles_n, mt, nt);
            const int m0 = mt * BM, n0 = nt * BN;
            const int row = m0 + quad * 32 + lane;
            mbar_wait(&tfull[buf], tph);
            tc::fence_after_sync();
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + half * (BN / 2));
            if constexpr (SPLIT) {  // fp32 partial tile of this K part: plain 16-byte stores
                float* prow = a.part + ((size_t)(t % ksplit) * a.M + row) * a.N;
#pragma unroll
                for (int cc = 0; cc < BN / 64; ++cc) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(base + cc * 32, r);
                    tc::tmem_ld_wait();
                    if (cc == BN / 64 - 1) {
                        tc::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    const int c0 = n0 + half * (BN / 2) + cc * 32;
                    if (row < a.M) {
#pragma unroll
                        for (int v = 0; v < 8; ++v)
                            if (c0 + 4 * v < a.N)
                                *reinterpret_cast<float4*>(prow + c0 + 4 * v) =
                                    make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                                __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
                    }
                }
                if (++buf == 2) {
                    buf = 0;
                    tph ^= 1u;
                }
                continue;
            }
#pragma unroll
            for (int gi = 0; gi < BN / 128; ++gi) {
                // TMEM -> registers -> bf16 first; only then wait for the previous
                // TMA store from this box to finish reading it (the wait overlaps
                // the TMEM loads and the epilogue arithmetic)
                uint4 o[2][4];
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) {
                    const int cc = gi * 2 + c2;
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(base + cc * 32, r);
                    tc::tmem_ld_wait();
                    if (cc == BN / 64 - 1) {  // the accumulator is in registers: hand it back to the MMA warp
                        tc::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    const int c0 = n0 + half * (BN / 2) + cc * 32;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        float f[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[8 * v + j]);
                        if constexpr (BIAS) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) f[j] += c0 + 8 * v + j < a.N ? __ldg(a.bias + c0 + 8 * v + j) : 0.f;
                        }
                        if constexpr (EPI != EPI_NONE) {
                            float x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                            if constexpr (EPI == EPI_RESID || EPI == EPI_DTANH) {
                                if (row < a.M && c0 + 8 * v < a.N)
                                    unpack<__nv_bfloat16>(
                                        __ldg(reinterpret_cast<const uint4*>(a.aux + (size_t)row * a.N + c0 + 8 * v)), x);
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) f[j] = epi_apply<EPI>(f[j], x[j]);
                        }
                        o[c2][v].x = pack_bf16x2(f[0], f[1]);
                        o[c2][v].y = pack_bf16x2(f[2], f[3]);
                        o[c2][v].z = pack_bf16x2(f[4], f[5]);
                        o[c2][v].w = pack_bf16x2(f[6], f[7]);
                    }
                }
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int chunk = c2 * 4 + v;  // 16-byte chunk of the 128-byte box row
                        *reinterpret_cast<uint4*>(box + lane * 128 + ((chunk ^ (lane & 7)) << 4)) = o[c2][v];
                    }
                fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA (async proxy)
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&tmo, box, n0 + half * (BN / 2) + gi * 64, m0 + quad * 32, 0);
                    bulk_commit();
                }
            }
            if (++buf == 2) {
                buf = 0;
                tph ^= 1u;
            }
        }
        if (lane == 0) bulk_wait0();  // every store of this warp complete before the CTA exits
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        tc::fence_after_sync();
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}


// ---------------------------------------------------------- fp32 rows: 3xTF32 --
// fp32 operands on the tensor cores at fp32 accuracy: every operand is split
// once into tf32 hi + lo parts (split_tf32_kernel: hi = rna(a), lo = rna(a - hi)),
// and each product is formed as lo*hi + hi*lo + hi*hi (kind::tf32, fp32
// accumulation in TMEM), dropping only lo*lo (~2^-22 relative).  Same
// structure as gemm_kernel with BM = BN = 128, 32-element (128-byte) K blocks,
// hi and lo tiles of A and B per stage, fp32 output boxes.  kind::tf32 takes
// K-major operands only: the forward's W is split into transposed copies.
namespace g3 {
constexpr int BM = 128, BN = 128, BK = 32;     // BK fp32 = one 128-byte swizzle row
constexpr int STAGES = 3;
constexpr int TILE = BM * BK * 4;              // 16 KB (A or B, hi or lo)
constexpr int STAGE_BYTES = 4 * TILE;          // A hi, A lo, B hi, B lo
constexpr int EPI_WARPS = 8;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int OUT_BOX_BYTES = 32 * 128;        // 32 rows x 32 fp32
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 1024 + (size_t)EPI_WARPS * OUT_BOX_BYTES;
static_assert(SMEM <= 232448, "dynamic shared memory of one CTA");
constexpr int TMEM_COLS = 256;
}  // namespace g3

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4)                          // c_format = F32
           | (2u << 7)                        // a_format = TF32
           | (2u << 10)                       // b_format = TF32
           | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__global__ void __launch_bounds__(256) split_tf32_kernel(const float* __restrict__ in, float* __restrict__ hi,
                                                         float* __restrict__ lo, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float a = in[i];
        uint32_t h, l;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(a));
        const float r = a - __uint_as_float(h);  // exact
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
        hi[i] = __uint_as_float(h);
        lo[i] = __uint_as_float(l);
    }
}

// W [K, L] -> hi^T, lo^T [L, K] (the forward's B operand, K-major: kind::tf32
// takes K-major operands only), 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256) split_tf32_t_kernel(const float* __restrict__ in, float* __restrict__ hi_t,
                                                           float* __restrict__ lo_t, int64_t K, int64_t L) {
    __shared__ float th[32][33], tl[32][33];
    const int64_t k0 = (int64_t)blockIdx.y * 32, l0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t k = k0 + r, l = l0 + tx;
        float h = 0.f, lo = 0.f;
        if (k < K && l < L) {
            const float a = in[k * L + l];
            uint32_t hb, lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(a));
            const float rr = a - __uint_as_float(hb);
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(rr));
            h = __uint_as_float(hb);
            lo = __uint_as_float(lb);
        }
        th[r][tx] = h;
        tl[r][tx] = lo;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t l = l0 + r, k = k0 + tx;
        if (k < K && l < L) {
            hi_t[l * K + k] = th[tx][r];
            lo_t[l * K + k] = tl[tx][r];
        }
    }
}

template <bool B_KMAJOR, bool BIAS, int EPI>
__global__ void __launch_bounds__(g3::THREADS, 1)
    gemm3_kernel(const __grid_constant__ CUtensorMap tah, const __grid_constant__ CUtensorMap tal,
                 const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbl,
                 const __grid_constant__ CUtensorMap tmo, GemmArgs a, const float* aux32, const float* bias32) {
    using namespace g3;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    unsigned char* obox = smem + (size_t)STAGES * STAGE_BYTES + 1024;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = a.tiles_m * a.tiles_n;
    const int kblocks = (a.Kr + BK - 1) / BK;
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
        tc::prefetch_tmap(&tah);
        tc::prefetch_tmap(&tal);
        tc::prefetch_tmap(&tbh);
        tc::prefetch_tmap(&tbl);
        tc::prefetch_tmap(&tmo);
    }
    if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mt, nt;
                tile_mn(t, a.tiles_m, a.tiles_n, mt, nt);
                const int m0 = mt * BM, n0 = nt * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char* st = ring + (size_t)s * STAGE_BYTES;
                    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                    const int k0 = kb * BK;
                    tc::tma_load_3d(st, &tah, k0, m0, 0, &full[s]);
                    tc::tma_load_3d(st + TILE, &tal, k0, m0, 0, &full[s]);
                    if constexpr (B_KMAJOR) {
                        tc::tma_load_3d(st + 2 * TILE, &tbh, k0, n0, 0, &full[s]);
                        tc::tma_load_3d(st + 3 * TILE, &tbl, k0, n0, 0, &full[s]);
                    } else {
#pragma unroll
                        for (int h = 0; h < BN / 32; ++h) {  // 32 (N) x 32 (K) chunks along N
                            tc::tma_load_3d(st + 2 * TILE + h * 4096, &tbh, n0 + 32 * h, k0, 0, &full[s]);
                            tc::tma_load_3d(st + 3 * TILE + h * 4096, &tbl, n0 + 32 * h, k0, 0, &full[s]);
                        }
                    }
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BM, BN, false, !B_KMAJOR);
            int s = 0, buf = 0;
            uint32_t ph = 0, tph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&tempty[buf], tph ^ 1u);
                tc::fence_after_sync();
                const uint32_t dcol = tmem + (uint32_t)(buf * BN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t ah = smem_u32(ring + (size_t)s * STAGE_BYTES), al = ah + TILE;
                    const uint32_t bh = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k) {
                        // K-major SW128: a K step of 8 tf32 = 32 bytes; MN-major SW128:
                        // 32-element x 8-row atoms, LBO = next 32 columns (4 KB), SBO = 8 K rows (1 KB)
                        const uint64_t dah = tc::smem_desc_sw128(ah + k * 32, 16, 1024);
                        const uint64_t dal = tc::smem_desc_sw128(al + k * 32, 16, 1024);
                        const uint64_t dbh = B_KMAJOR ? tc::smem_desc_sw128(bh + k * 32, 16, 1024)
                                                      : tc::smem_desc_sw128(bh + k * 1024, 4096, 1024);
                        const uint64_t dbl = B_KMAJOR ? tc::smem_desc_sw128(bl + k * 32, 16, 1024)
                                                      : tc::smem_desc_sw128(bl + k * 1024, 4096, 1024);
                        mma_tf32(dcol, dal, dbh, idesc, (kb | k) != 0);  // small terms first
                        mma_tf32(dcol, dah, dbl, idesc, 1);
                        mma_tf32(dcol, dah, dbh, idesc, 1);
                    }
                    tc::commit(&empty[s]);
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1u;
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
        // epilogue: warp (quad, half) owns 32 rows x 64 columns; two 32-column
        // boxes per tile, staged in shared memory (128B swizzle) and TMA-stored
        const int e = warp - 2;
        const int quad = warp & 3;
        const int half = e / 4;
        unsigned char* box = obox + (size_t)e * OUT_BOX_BYTES;
        int buf = 0;
        uint32_t tph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int mt, nt;
            tile_mn(t, a.tiles_m, a.tiles_n, mt, nt);
            const int m0 = mt * BM, n0 = nt * BN;
            const int row = m0 + quad * 32 + lane;
            mbar_wait(&tfull[buf], tph);
            tc::fence_after_sync();
            const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + half * 64);
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
                uint32_t r[32];
                tc::tmem_ld_32x32b_x32(base + cc * 32, r);
                tc::tmem_ld_wait();
                if (cc == 1) {
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);
                }
                const int c0 = n0 + half * 64 + cc * 32;
#pragma unroll
                for (int v = 0; v < 8; ++v) {  // 16-byte chunks of the 128-byte box row
                    float f[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        f[j] = __uint_as_float(r[4 * v + j]);
                        const int col = c0 + 4 * v + j;
                        if constexpr (BIAS) f[j] += col < a.N ? __ldg(bias32 + col) : 0.f;
                        if constexpr (EPI != EPI_NONE) {
                            const float x = (EPI == EPI_RESID || EPI == EPI_DTANH) && row < a.M && col < a.N
                                                ? __ldg(aux32 + (size_t)row * a.N + col)
                                                : 0.f;
                            f[j] = epi_apply<EPI>(f[j], x);
                        }
                    }
                    *reinterpret_cast<float4*>(box + lane * 128 + ((v ^ (lane & 7)) << 4)) =
                        make_float4(f[0], f[1], f[2], f[3]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&tmo, box, c0, m0 + quad * 32, 0);
                    bulk_commit();
                }
            }
            if (++buf == 2) {
                buf = 0;
                tph ^= 1u;
            }
        }
        if (lane == 0) bulk_wait0();
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        tc::fence_after_sync();
        tc::tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// fp32 master weights -> bf16 operand copy (RNE)
__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                                          int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 4 <= n) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(in + i));
        uint2 o;
        o.x = pack_bf16x2(v.x, v.y);
        o.y = pack_bf16x2(v.z, v.w);
        *reinterpret_cast<uint2*>(out + i) = o;
    } else {
        for (int64_t j = i; j < n; ++j) out[j] = __float2bfloat16_rn(in[j]);
    }
}

// ----------------------------------------------------- generic (any dtype) --
// One thread per output; fp64 accumulation in the reference's order (k, then
// bias last) without contraction, so fp64 rows reproduce layers.cpp:52-78 and
// :142-155 bit for bit.
template <typename T, typename WT, bool FWD>
__global__ void __launch_bounds__(256) gemm_generic_kernel(const T* a, const WT* W, const void* bias, int bias_f64,
                                                           const T* aux, int epi, T* out, int64_t rows, int64_t N,
                                                           int64_t Kr, int64_t ldw) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * N) return;
    const int64_t r = idx / N, n = idx % N;
    double acc = 0.0;
    for (int64_t k = 0; k < Kr; ++k) {
        const double w = (double)to_acc<WT>(FWD ? W[k * ldw + n] : W[n * ldw + k]);
        acc = __dadd_rn(acc, __dmul_rn((double)to_acc<T>(a[r * Kr + k]), w));
    }
    if (bias) acc = __dadd_rn(acc, bias_f64 ? static_cast<const double*>(bias)[n] : (double)static_cast<const float*>(bias)[n]);
    if (epi != EPI_NONE) {  // the reference's elementwise step in fp64 (model.cpp:96, :99, :171)
        const double z = aux ? (double)to_acc<T>(aux[idx]) : 0.0;
        acc = epi == EPI_TANH ? tanh(acc) : epi == EPI_RESID ? __dadd_rn(z, acc) : __dmul_rn(acc, __dsub_rn(1.0, __dmul_rn(z, z)));
    }
    out[idx] = from_acc<T>((typename Traits<T>::Acc)acc);
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

// [rows, cols] bf16 row-major (cols innermost) as a 3-D map with a unit
// outer axis; box {bc, br}, 128-byte swizzle, out-of-range elements read 0
bool make_map_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int bc, int br) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
    cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)br, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool BK_, bool BIAS, int EPI, int BNT>
cudaError_t launch_tc_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const GemmArgs& a,
                         cudaStream_t st) {
    const void* fn = reinterpret_cast<const void*>(gemm_kernel<BK_, BIAS, EPI, BNT>);
    cudaError_t e = ensure_smem_attr(fn, gm::SMEM);
    if (e != cudaSuccess) return e;
    const int ntiles = a.tiles_m * a.tiles_n;
    const int sms = device_sm_count();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles < sms ? ntiles : sms);
    cfg.blockDim = dim3(gm::THREADS);
    cfg.dynamicSmemBytes = gm::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<BK_, BIAS, EPI, BNT>, ma, mb, mo, a);
}
template <bool BK_>
cudaError_t launch_tc_split(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const GemmArgs& a,
                            int units, cudaStream_t st) {
    const void* fn = reinterpret_cast<const void*>(gemm_kernel<BK_, false, EPI_NONE, 256, true>);
    cudaError_t e = ensure_smem_attr(fn, gm::SMEM);
    if (e != cudaSuccess) return e;
    const int sms = device_sm_count();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units < sms ? units : sms);
    cfg.blockDim = dim3(gm::THREADS);
    cfg.dynamicSmemBytes = gm::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<BK_, false, EPI_NONE, 256, true>, ma, mb, mo, a);
}
template <int EPI, bool BIAS>
cudaError_t launch_splitk_reduce(const GemmArgs& a, cudaStream_t st) {
    splitk_reduce_kernel<EPI, BIAS><<<device_sm_count() * 4, 256, 0, st>>>(a.part, a.ksplit, a.M, a.N, a.bias, a.aux,
                                                                         a.out);
    return cudaGetLastError();
}
// split-K parts: only for long reductions whose tile count leaves the last
// wave mostly idle (the partials cost an extra fp32 write + read of the output)
int gemm_pick_split(int64_t tiles, int64_t kblocks) {
    const int sms = device_sm_count();
    auto eff = [&](int64_t t) { return (double)t / (double)(((t + sms - 1) / sms) * sms); };
    if (kblocks < 64 || eff(tiles) >= 0.8) return 1;
    for (int k = 2; k <= 4; ++k)
        if (eff(tiles * k) >= 0.85 && kblocks / k >= 16) return k;
    return kblocks / 4 >= 16 ? 4 : 1;
}

template <bool BK_, bool BIAS, int EPI>
cudaError_t launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const GemmArgs& a,
                      cudaStream_t st, int bn) {
    return bn == 128 ? launch_tc_bn<BK_, BIAS, EPI, 128>(ma, mb, mo, a, st)
                     : launch_tc_bn<BK_, BIAS, EPI, 256>(ma, mb, mo, a, st);
}
// output tile width: 256.  A 128-wide variant (GNSB_GEMM_BN=128, A/B runs)
// fills the last wave of small tile counts better but measured slower on every
// shape tried, including those (N = 768 outputs at 8192 rows: 60 against 48 us;
// GPT-2 head dx: 754 against 603 us) where it had the better wave efficiency.
int gemm_pick_bn(int64_t tiles_m, int64_t N) {
    static const int forced = [] {  // GNSB_GEMM_BN=128 / 256: A/B runs
        const char* e = std::getenv("GNSB_GEMM_BN");
        return e ? std::atoi(e) : 0;
    }();
    (void)tiles_m;
    (void)N;
    return forced == 128 ? 128 : 256;
}


// [rows, cols] fp32 row-major as a 3-D map, box {bc, br}, 128-byte swizzle
bool make_map_2d_f32(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int bc, int br) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 4, (cuuint64_t)rows * cols * 4};
    cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)br, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool BK_, bool BIAS, int EPI>
cudaError_t launch_tc3(const CUtensorMap* maps, const GemmArgs& a, const float* aux, const float* bias,
                       cudaStream_t st) {
    const void* fn = reinterpret_cast<const void*>(gemm3_kernel<BK_, BIAS, EPI>);
    cudaError_t e = ensure_smem_attr(fn, g3::SMEM);
    if (e != cudaSuccess) return e;
    const int ntiles = a.tiles_m * a.tiles_n;
    const int sms = device_sm_count();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles < sms ? ntiles : sms);
    cfg.blockDim = dim3(g3::THREADS);
    cfg.dynamicSmemBytes = g3::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm3_kernel<BK_, BIAS, EPI>, maps[0], maps[1], maps[2], maps[3], maps[4], a, aux,
                              bias);
}
}  // namespace

bool gemm_tc_ok(int dt, int64_t K, int64_t L) {
    return dt == 1 && K % 8 == 0 && L % 8 == 0 && K < (1ll << 31) && L < (1ll << 31);
}
// fp32 rows and fp32 weights on the 3xTF32 kernel: 16-byte row strides
static bool gemm3_ok(int dt, int w_dt, int64_t rows, int64_t K, int64_t L) {
    return dt == 0 && w_dt == 0 && K % 4 == 0 && L % 4 == 0 && K < (1ll << 31) && L < (1ll << 31) &&
           rows < (1ll << 31);
}
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t gemm_workspace(int dt, int w_dt, int64_t K, int64_t L) {
    return (dt == 1 && w_dt == 0 && gemm_tc_ok(dt, K, L)) ? (size_t)K * L * 2 : 0;
}
// the 3xTF32 path splits both operands into hi / lo copies: a scratch of
// 2 * (rows * Kr + K * L) fp32 (gnsb_linear_gemm_workspace_size has no row
// count) from a library-owned stream-ordered pool that keeps its memory
// (the default pool would hand gigabytes back to the driver at every
// synchronisation and re-map them on the next call)
static size_t gemm3_scratch(int64_t rows, int64_t Kr, int64_t K, int64_t L) {
    return (size_t)2 * (rows * Kr + K * L) * sizeof(float) + 512;
}
static cudaError_t scratch_pool(cudaMemPool_t* out) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0 || dev >= 64) return e != cudaSuccess ? e : cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pp = {};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        e = cudaMemPoolCreate(&pools[dev], &pp);
        if (e != cudaSuccess) return e;
        uint64_t keep = ~0ull;
        e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        if (e != cudaSuccess) return e;
    }
    *out = pools[dev];
    return cudaSuccess;
}

cudaError_t gemm_pool_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool;
    cudaError_t e = scratch_pool(&pool);
    return e != cudaSuccess ? e : cudaMallocFromPoolAsync(p, bytes, pool, st);
}
cudaError_t gemm_pool_free(void* p, cudaStream_t st) { return cudaFreeAsync(p, st); }

// kind 0: forward y = x W + bias; kind 1: dx = g W^T.  dt / w_dt: 0 f32, 1 bf16, 2 f64.
// epi: EPI_* applied to every output element (aux [rows, N] of dtype dt).
cudaError_t launch_linear_gemm(int kind, int epi, int dt, int w_dt, const void* in, const void* W, const void* bias,
                               const void* aux, void* out, int64_t rows, int64_t K, int64_t L, void* ws,
                               cudaStream_t st) {
    const int64_t N = kind == 0 ? L : K, Kr = kind == 0 ? K : L;
    if (rows == 0) return cudaSuccess;
    if (gemm_tc_ok(dt, K, L) && rows < (1ll << 31) && al16(in) && al16(out) && (w_dt == 0 || al16(W)) &&
        (aux == nullptr || al16(aux))) {
        const void* wb = W;
        if (w_dt == 0) {  // fp32 master weights: bf16 operand copy in the workspace
            const int64_t n = K * L;
            f32_to_bf16_kernel<<<(unsigned)((n / 4 + 255) / 256 + 1), 256, 0, st>>>(
                static_cast<const float*>(W), static_cast<__nv_bfloat16*>(ws), n);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            wb = ws;
        }
        CUtensorMap ma, mb;
        if (!make_map_2d(&ma, in, rows, Kr, gm::BK, gm::BM)) return cudaErrorInvalidValue;
        const int bn = gemm_pick_bn((rows + gm::BM - 1) / gm::BM, N);
        const bool ok = kind == 0 ? make_map_2d(&mb, wb, K, L, 64, gm::BK)  // W [K, L]: box 64 (L) x 64 (K)
                                  : make_map_2d(&mb, wb, K, L, gm::BK, bn);  // W [K, L]: box 64 (L) x bn (K)
        if (!ok) return cudaErrorInvalidValue;
        CUtensorMap mo;  // the output [rows, N], stored by 32-row x 64-column boxes
        if (!make_map_2d(&mo, out, rows, N, 64, 32)) return cudaErrorInvalidValue;
        GemmArgs a{};
        a.M = (int)rows;
        a.N = (int)N;
        a.Kr = (int)Kr;
        a.tiles_m = (int)((rows + gm::BM - 1) / gm::BM);
        a.tiles_n = (int)((N + bn - 1) / bn);
        a.bias = static_cast<const float*>(bias);
        a.aux = static_cast<const __nv_bfloat16*>(aux);
        a.out = static_cast<__nv_bfloat16*>(out);
        const int ks = bn == 256 ? gemm_pick_split((int64_t)a.tiles_m * a.tiles_n, (Kr + gm::BK - 1) / gm::BK) : 1;
        if (ks > 1 && std::getenv("GNSB_GEMM_NOSPLIT") == nullptr) {
            cudaMemPool_t pool;
            void* scratch = nullptr;
            cudaError_t e = scratch_pool(&pool);
            if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&scratch, (size_t)ks * rows * N * 4, pool, st);
            if (e != cudaSuccess) return e;
            a.ksplit = ks;
            a.part = static_cast<float*>(scratch);
            const int units = a.tiles_m * a.tiles_n * ks;
            e = kind == 1 ? launch_tc_split<true>(ma, mb, mo, a, units, st)
                          : launch_tc_split<false>(ma, mb, mo, a, units, st);
            if (e == cudaSuccess) {
                switch (epi) {
                    case EPI_TANH: e = bias ? launch_splitk_reduce<EPI_TANH, true>(a, st) : launch_splitk_reduce<EPI_TANH, false>(a, st); break;
                    case EPI_RESID: e = bias ? launch_splitk_reduce<EPI_RESID, true>(a, st) : launch_splitk_reduce<EPI_RESID, false>(a, st); break;
                    case EPI_DTANH: e = launch_splitk_reduce<EPI_DTANH, false>(a, st); break;
                    default: e = bias ? launch_splitk_reduce<EPI_NONE, true>(a, st) : launch_splitk_reduce<EPI_NONE, false>(a, st);
                }
            }
            const cudaError_t f = cudaFreeAsync(scratch, st);
            return e != cudaSuccess ? e : f;
        }
        if (kind == 1) {
            if (epi == EPI_DTANH) return launch_tc<true, false, EPI_DTANH>(ma, mb, mo, a, st, bn);
            return launch_tc<true, false, EPI_NONE>(ma, mb, mo, a, st, bn);
        }
        switch (epi) {
            case EPI_TANH:
                return bias ? launch_tc<false, true, EPI_TANH>(ma, mb, mo, a, st, bn) : launch_tc<false, false, EPI_TANH>(ma, mb, mo, a, st, bn);
            case EPI_RESID:
                return bias ? launch_tc<false, true, EPI_RESID>(ma, mb, mo, a, st, bn)
                            : launch_tc<false, false, EPI_RESID>(ma, mb, mo, a, st, bn);
            default:
                return bias ? launch_tc<false, true, EPI_NONE>(ma, mb, mo, a, st, bn) : launch_tc<false, false, EPI_NONE>(ma, mb, mo, a, st, bn);
        }
    }
    if (gemm3_ok(dt, w_dt, rows, K, L) && al16(in) && al16(out) && al16(W) && (aux == nullptr || al16(aux))) {
        // fp32: split A and W into tf32 hi / lo copies, then 3xTF32 on the tensor cores
        void* scratch = nullptr;
        cudaMemPool_t pool;
        cudaError_t e = scratch_pool(&pool);
        if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&scratch, gemm3_scratch(rows, Kr, K, L), pool, st);
        if (e != cudaSuccess) return e;
        float* ah = static_cast<float*>(scratch);
        float* alo = ah + rows * Kr;
        float* wh = alo + rows * Kr;
        float* wl = wh + K * L;
        const int sg = device_sm_count() * 8;
        split_tf32_kernel<<<sg, 256, 0, st>>>(static_cast<const float*>(in), ah, alo, rows * Kr);
        // B in K-major form [N, Kr]: W itself for dx (W[k, :] runs along the
        // reduced L), W transposed for the forward
        if (kind == 0)
            split_tf32_t_kernel<<<dim3((unsigned)((L + 31) / 32), (unsigned)((K + 31) / 32)), 256, 0, st>>>(
                static_cast<const float*>(W), wh, wl, K, L);
        else
            split_tf32_kernel<<<sg, 256, 0, st>>>(static_cast<const float*>(W), wh, wl, K * L);
        e = cudaGetLastError();
        CUtensorMap maps[5];
        bool ok = e == cudaSuccess && make_map_2d_f32(&maps[0], ah, rows, Kr, g3::BK, g3::BM) &&
                  make_map_2d_f32(&maps[1], alo, rows, Kr, g3::BK, g3::BM) &&
                  make_map_2d_f32(&maps[2], wh, N, Kr, g3::BK, g3::BN) &&  // [N, Kr]: 32 (Kr) x 128 (N)
                  make_map_2d_f32(&maps[3], wl, N, Kr, g3::BK, g3::BN) &&
                  make_map_2d_f32(&maps[4], out, rows, N, 32, 32);
        if (e == cudaSuccess && !ok) e = cudaErrorInvalidValue;
        if (e == cudaSuccess) {
            GemmArgs a{};
            a.M = (int)rows;
            a.N = (int)N;
            a.Kr = (int)Kr;
            a.tiles_m = (int)((rows + g3::BM - 1) / g3::BM);
            a.tiles_n = (int)((N + g3::BN - 1) / g3::BN);
            const float* ax = static_cast<const float*>(aux);
            const float* bs = static_cast<const float*>(bias);
            if (kind == 1)
                e = epi == EPI_DTANH ? launch_tc3<true, false, EPI_DTANH>(maps, a, ax, bs, st)
                                     : launch_tc3<true, false, EPI_NONE>(maps, a, ax, bs, st);
            else if (epi == EPI_TANH)
                e = bias ? launch_tc3<true, true, EPI_TANH>(maps, a, ax, bs, st)
                         : launch_tc3<true, false, EPI_TANH>(maps, a, ax, bs, st);
            else if (epi == EPI_RESID)
                e = bias ? launch_tc3<true, true, EPI_RESID>(maps, a, ax, bs, st)
                         : launch_tc3<true, false, EPI_RESID>(maps, a, ax, bs, st);
            else
                e = bias ? launch_tc3<true, true, EPI_NONE>(maps, a, ax, bs, st)
                         : launch_tc3<true, false, EPI_NONE>(maps, a, ax, bs, st);
        }
        const cudaError_t f = cudaFreeAsync(scratch, st);
        return e != cudaSuccess ? e : f;
    }
    const int64_t n = rows * N;
    const unsigned grid = (unsigned)((n + 255) / 256);
    const int bias_f64 = dt == 2;
    const int64_t ldw = L;
#define GNSB_GEMM_GENERIC(T, WT)                                                                                     \
    do {                                                                                                             \
        if (kind == 0)                                                                                               \
            gemm_generic_kernel<T, WT, true><<<grid, 256, 0, st>>>(                                                \
                static_cast<const T*>(in), static_cast<const WT*>(W), bias, bias_f64, static_cast<const T*>(aux), epi, \
                static_cast<T*>(out), rows, N, Kr, ldw);                                                             \
        else                                                                                                         \
            gemm_generic_kernel<T, WT, false><<<grid, 256, 0, st>>>(                                               \
                static_cast<const T*>(in), static_cast<const WT*>(W), nullptr, 0, static_cast<const T*>(aux), epi,   \
                static_cast<T*>(out), rows, N, Kr, ldw);                                                             \
    } while (0)
    if (dt == 2 && w_dt == 2)
        GNSB_GEMM_GENERIC(double, double);
    else if (dt == 0 && w_dt == 0)
        GNSB_GEMM_GENERIC(float, float);
    else if (dt == 1 && w_dt == 0)
        GNSB_GEMM_GENERIC(__nv_bfloat16, float);
    else if (dt == 1 && w_dt == 1)
        GNSB_GEMM_GENERIC(__nv_bfloat16, __nv_bfloat16);
    else
        return cudaErrorInvalidValue;
#undef GNSB_GEMM_GENERIC
    return cudaGetLastError();
}

}  // namespace gnsb

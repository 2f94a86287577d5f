// ln_bwd.cuh — fused LayerNorm backward + per-example ||dgamma_b||^2, ||dbeta_b||^2
// (and its plain twin, NORMS=false) for sm_100a.
//
// Semantics: gnstk::layernorm_backward_simultaneous (proj/src/layers.cpp:231-298):
//   gamma'_b = sum_m xhat*g, beta'_b = sum_m g          (per example, :251-258)
//   raw_b    = ||gamma'_b||^2, ||beta'_b||^2            (square AFTER the sum, :259-262)
//   dgamma   = sum_b gamma'_b, dbeta = sum_b beta'_b     (:265-268)
//   dx       = rstd*(h - mean(h) - xhat*mean(h*xhat)), h = gamma*g   (:277-296)
//
// Design (one HBM pass over x/xhat, dy; one write of dx):
//   * persistent cooperative grid, one CTA per SM; CTA c owns the contiguous
//     row range [c*N/grid, (c+1)*N/grid) (rows of an example are contiguous);
//   * R-row stages of x and dy stream into a shared-memory ring by 1-D TMA
//     (cp.async.bulk, L2 evict_first) completing on mbarriers.  There is no
//     dedicated producer warp: lane 0 of warp 0 refills a slot as soon as
//     every warp released it, so all 16 warps do row math;
//   * mean/rstd ride along with each stage (producer lanes, S stages ahead);
//   * warps form G row groups of GW warps; a thread owns VPT 16-byte column
//     vectors for the whole kernel, so the per-example dgamma/dbeta partials
//     accumulate over the sequence axis in registers (packed fp32x2 math:
//     FFMA2/FADD2/FMUL2);
//   * row reductions mean(h), mean(h*xhat): a transposed butterfly inside
//     the warp, then a padded xor tree across the group's warps;
//   * at each example boundary a group flushes its register partials to a
//     slot (cta + example, group) of an L2-resident workspace; at the end the
//     CTA folds its groups' slots in fixed order (the last example through
//     shared memory), leaving one slot per (cta, example);
//   * stage 2 is a second kernel (ln_bwd_reduce_kernel), launched with
//     programmatic dependent launch so it is scheduled while the row kernel
//     drains: CTA c owns a contiguous column range; per example it sums that
//     example's slots in fixed CTA order -> gamma'_b, beta'_b (fp64), squares
//     and reduces over its columns -> q[b][c], and sums over b in fixed order
//     -> dgamma/dbeta on its columns (+ their squares -> qbig[c]);
//   * the last CTA (ticket) folds q into raw_b and the scalar sums.  No float
//     atomics anywhere: results are bitwise deterministic run to run.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace gnsb {

struct LnBwdArgs {
    const void* x;      // x rows (HAS_MEAN) or xhat rows, [N, D] of T
    const void* mean;   // [N] Acc, only when HAS_MEAN
    const void* rstd;   // [N] Acc
    const void* dy;     // [N, D] of T
    const void* gamma;  // [D] Acc
    void* dx;           // [N, D] of T (may be null: skip dx)
    int64_t B, M, N, D;
    int Dp;             // smem row stride in elements (D rounded up to the vector width)
    int stages;         // ring depth
    int aligned;        // 1: rows are 16-byte aligned -> TMA producer
    int gamma16;        // 1: gamma is 16-byte aligned and D*sizeof(Acc) % 16 == 0 -> vector staging
    void* partial;      // [(grid + B) * G][2][Dp] Acc; slot (cta + example, 0) holds the CTA's fold
    unsigned long long* trace;  // optional [grid][6] globaltimer stamps (profiling only)
};

// Arguments of the stage-2 kernel (per-example combine, squares, dgamma/dbeta).
struct LnRedArgs {
    const void* partial;  // the row kernel's slots: slot (c + b) * slot_stride holds CTA c's part of example b
    int64_t slot_stride;  // elements between consecutive slots: G * 2 * Dp (folded), 2 * Dp (gsub = G)
    int gsub;             // slots per (cta + example): 1 (folded by the row kernel) or G (one per row group)
    int64_t B, M, N, D;
    int Dp;
    int grid_rows;        // CTAs of the row kernel (row range of CTA c: [c*N/grid_rows, (c+1)*N/grid_rows))
    int eb;               // examples per shared-memory block
    int slot_cap;         // slots staged at once; < a block's span only when eb == 1 (chunked per example)
    void* dgamma;         // [D] Acc
    void* dbeta;          // [D] Acc
    double* raw_g;        // [B] or null
    double* raw_b;        // [B] or null
    double* sums;         // [4] or null: sum raw_g, sum raw_b, ||dgamma||^2, ||dbeta||^2
    double* q;            // [B][grid][2] per-(example, column range) squares
    double* qbig;         // [grid][2]
    double* rawws;        // [B][2]
    unsigned* ticket;     // zero on entry and on exit
    unsigned long long* trace;  // optional [grid][6]
};

template <typename T, int GW, int VPT, int G, int RPG, bool PROD_ = true, int KEEP_ = -1, int CPS_ = 1,
          bool PARK_ = false, bool NOFOLD_ = false, bool WIDE_ = true>
struct LnBwdCfg {
    using Acc = typename Traits<T>::Acc;
    using Row = T;
    static constexpr int kGW = GW, kVPT = VPT, kG = G, kRPG = RPG;
    static constexpr int W = Traits<T>::W;
    static constexpr bool PROD = PROD_;          // dedicated producer warp (the last warp)
    static constexpr bool kPark = PARK_ && G > 1;  // first example's group partials parked in smem
    // kNoFold: no end-of-kernel CTA fold; every group leaves its own slot for
    // every example it touched and stage 2 sums the G sub-slots (moves ~2 us
    // of the row pass's critical path into the once-per-step reduce)
    static constexpr bool kNoFold = NOFOLD_ && G > 1 && !kPark;
    static constexpr int kSub = kNoFold ? G : 1;  // sub-slots stage 2 reads per (cta + example)
    // kWide: partial slots are written with 16-byte stores (see write_slot);
    // off where the register quads they need push the row loop into spills
    static constexpr bool kWide = WIDE_;
    static constexpr int kWarps = GW * G;        // row-math warps
    static constexpr int kThreads = (kWarps + (PROD ? 1 : 0)) * 32;
    // registers are allocated for warps in groups of 4: bound the register
    // budget by the rounded-up block so one CTA always fits on an SM
    static constexpr int kBoundThreads = (kThreads + 127) / 128 * 128;
    static constexpr int kCps = CPS_;             // resident CTAs per SM (1, or 2 for narrow rows)
    static constexpr int R = G * RPG;           // rows per stage
    static constexpr int GT = GW * 32;          // threads per row group
    static constexpr int NQ = 2 * RPG;          // row sums per stage and group: (s1, s2) per row
    static constexpr int GWP = GW <= 1 ? 1 : GW <= 2 ? 2 : GW <= 4 ? 4 : GW <= 8 ? 8 : GW <= 16 ? 16 : 32;  // pow2 pad
    // keep xhat/h of a stage in registers (else recompute them for dx)
    static constexpr bool KEEP = KEEP_ < 0 ? (VPT * RPG <= 2) : (KEEP_ != 0);
    static constexpr int kRedElems = 2 * G * NQ * GWP;
    // byte offsets inside dynamic shared memory
    static __host__ __device__ constexpr size_t bars_bytes(int S) { return (size_t)8 * 2 * S; }
    static __host__ __device__ constexpr size_t red_off(int S) { return (bars_bytes(S) + 15) / 16 * 16; }
    static __host__ __device__ constexpr size_t stats_off(int S) {
        return red_off(S) + ((size_t)kRedElems * sizeof(Acc) + 15) / 16 * 16;
    }
    static __host__ __device__ constexpr size_t gam_off(int S) {
        return (stats_off(S) + (size_t)S * R * 2 * sizeof(Acc) + 15) / 16 * 16;
    }
    static __host__ __device__ constexpr size_t rows_off(int S, int Dp) {
        return (gam_off(S) + (size_t)Dp * sizeof(Acc) + 127) / 128 * 128;
    }
    static __host__ __device__ constexpr size_t stage_row_bytes(int Dp) { return (size_t)2 * R * Dp * sizeof(T); }
    // kPark: the group partials of the CTA's first example are parked in
    // shared memory [G][2][Dp] after the ring, so the end-of-kernel fold needs
    // no L2 round trip (measured: +2.5 points at D=768; at D=2048 the stage
    // it costs loses more).  The ring doubles as the fold area of the last
    // example's partials (G > 1).
    static __host__ __device__ constexpr size_t park_bytes(int Dp) {
        return kPark ? (size_t)G * 2 * Dp * sizeof(Acc) : 0;
    }
    static __host__ __device__ constexpr size_t park_off(int S, int Dp) {
        const size_t ring = (size_t)S * stage_row_bytes(Dp);
        const size_t scratch = G > 1 ? (size_t)G * 2 * Dp * sizeof(Acc) : 0;
        return rows_off(S, Dp) + (ring > scratch ? ring : scratch);
    }
    static __host__ __device__ constexpr size_t smem_bytes(int S, int Dp) { return park_off(S, Dp) + park_bytes(Dp); }
};

#ifndef GNSB_LN_EARLYFOLD
#define GNSB_LN_EARLYFOLD 0  // A/B: fold the CTA's first example at its boundary
#endif
template <typename C, bool HAS_MEAN>
__global__ void __launch_bounds__(C::kBoundThreads, C::kCps) ln_bwd_kernel(LnBwdArgs a) {
    using T = typename C::Row;
    constexpr int GW = C::kGW, VPT = C::kVPT, G = C::kG, RPG = C::kRPG;
    using Acc = typename C::Acc;
    using PR = Pair<Acc>;
    using P = typename PR::P;
    constexpr int W = C::W;
    constexpr int R = C::R;
    constexpr int GT = C::GT;
    constexpr int NW = C::kWarps;
    constexpr int NP = W / 2;     // pairs per 16-byte vector
    constexpr int NQ = C::NQ;
    constexpr int GWP = C::GWP;
    constexpr bool KEEP = C::KEEP;
    static_assert((NQ & (NQ - 1)) == 0 && NQ <= 32, "rows per group per stage must be a power of two");

    extern __shared__ __align__(128) unsigned char smem[];
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    Acc* red = reinterpret_cast<Acc*>(smem + C::red_off(S));
    Acc* stats = reinterpret_cast<Acc*>(smem + C::stats_off(S));  // [S][R][mean, rstd]
    Acc* gam_s = reinterpret_cast<Acc*>(smem + C::gam_off(S));
    T* ring = reinterpret_cast<T*>(smem + C::rows_off(S, a.Dp));
    Acc* park = reinterpret_cast<Acc*>(smem + C::park_off(S, a.Dp));  // [G][2][Dp] (kPark)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grid = gridDim.x, cta = blockIdx.x;
    const int64_t N = a.N, M = a.M, D = a.D;
    const int Dp = a.Dp;
    const int NVp = Dp / W;  // vectors per (padded) row
    const int64_t r_begin = (int64_t)cta * N / grid, r_end = (int64_t)(cta + 1) * N / grid;
    const int64_t n_stage = (r_end - r_begin + R - 1) / R;
    const T* xg = static_cast<const T*>(a.x);
    const T* dyg = static_cast<const T*>(a.dy);
    const Acc* meang = static_cast<const Acc*>(a.mean);
    const Acc* rstdg = static_cast<const Acc*>(a.rstd);

    auto stamp = [&](int k) {
        if (a.trace != nullptr && threadIdx.x == 0) a.trace[(size_t)cta * 6 + k] = globaltimer_ns();
    };
    stamp(0);
    // the stage-2 kernel may be scheduled as soon as SMs free up; it waits
    // (griddepcontrol.wait) for this grid's completion before reading
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
#if GNSB_LN_EARLYFOLD
    // early fold of the CTA's first example (see flush_to)
    __shared__ int s_fold_cnt, s_early;
    __shared__ int s_fold_last[G];
    if (threadIdx.x == 0) {
        s_fold_cnt = 0;
        s_early = 0;
    }
#endif
    if (!a.aligned) {  // padded rows: the pad columns must read as zero
        uint4* p = reinterpret_cast<uint4*>(ring);
        const size_t n16 = (size_t)S * C::stage_row_bytes(Dp) / 16;
        for (size_t i = threadIdx.x; i < n16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    // Launched with programmatic dependent launch: everything above overlaps
    // the previous kernel in the stream; no global memory is touched before
    // the previous grid has completed and its writes are visible.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    stamp(3);

    // ------------------------------------------------------------ producer --
    // Fill stage `st` into its slot.  Called by warp 0 only (lane 0 issues the
    // TMA; the generic path copies with the whole warp).
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int64_t st) {
        const int slot = (int)(st % S);
        const int64_t r0 = r_begin + st * R;
        const int nr = (int)((r_end - r0) < (int64_t)R ? (r_end - r0) : (int64_t)R);
        T* sx = ring + (size_t)slot * 2 * R * Dp;
        T* sdy = sx + (size_t)R * Dp;
        if (a.aligned) {
            if (lane == 0) {
                const uint32_t bytes = (uint32_t)(nr * D * (int64_t)sizeof(T));
                mbar_expect_tx(&full[slot], 2 * bytes);
                bulk_g2s(sx, xg + r0 * D, bytes, &full[slot], pol);
                bulk_g2s(sdy, dyg + r0 * D, bytes, &full[slot], pol);
            }
        } else {
            const int64_t ne = (int64_t)nr * D;
            for (int64_t e = lane; e < ne; e += 32) {
                const int64_t rr = e / D, cc = e - rr * D;
                sx[rr * Dp + cc] = xg[r0 * D + e];
                sdy[rr * Dp + cc] = dyg[r0 * D + e];
            }
        }
        // per-row mean/rstd ride along with the stage (loaded S stages ahead)
        Acc* sst = stats + (size_t)slot * R * 2;
        for (int j = lane; j < nr; j += 32) {
            sst[2 * j] = HAS_MEAN ? __ldg(meang + r0 + j) : Acc(0);
            sst[2 * j + 1] = __ldg(rstdg + r0 + j);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[slot]);
    };
    int64_t issued = 0;  // warp 0 (no producer warp): stages handed to the ring so far
    if (warp == (C::PROD ? NW : 0)) {  // prime the ring (no waits: every slot is free)
        for (; issued < n_stage && issued < S; ++issued) issue(issued);
    }
    // warp 0 refills every slot whose stage all warps have released; `need`
    // forces progress up to that stage (blocking on its slot's release)
    auto refill = [&](int64_t need) {
        for (; issued < n_stage; ++issued) {
            const int slot = (int)(issued % S);
            const uint32_t par = (uint32_t)(((issued / S) - 1) & 1);  // phase of the release of stage issued - S
            if (issued > need) {
                const bool ok = __shfl_sync(0xffffffffu, lane == 0 ? (int)mbar_try_wait(&empty[slot], par) : 0, 0) != 0;
                if (!ok) break;
            } else {
                mbar_wait(&empty[slot], par);
            }
            issue(issued);
        }
    };

    // ----------------------------------------------------------- consumers --
    const int g = warp / GW, wig = warp % GW;
    const int tig = wig * 32 + lane;
    Acc* partial = static_cast<Acc*>(a.partial);
    T* dxg = static_cast<T*>(a.dx);
    const Acc invD = Acc(1) / Acc(D);

    {  // gamma -> shared memory (while the first stages are in flight)
        const Acc* gg = static_cast<const Acc*>(a.gamma);
        if (a.gamma16) {  // D % E == 0 here; pad columns [D, Dp) read as zero
            constexpr int E = 16 / sizeof(Acc);
            for (int i = threadIdx.x; i < (int)D / E; i += blockDim.x)
                *reinterpret_cast<uint4*>(gam_s + i * E) = __ldg(reinterpret_cast<const uint4*>(gg) + i);
            for (int i = (int)D + threadIdx.x; i < Dp; i += blockDim.x) gam_s[i] = Acc(0);
        } else {
            for (int i = threadIdx.x; i < Dp; i += blockDim.x) gam_s[i] = i < D ? gg[i] : Acc(0);
        }
        __syncthreads();
    }
    if constexpr (C::PROD) {
        if (warp == NW) {  // dedicated producer: stream the remaining stages
            for (int64_t st = issued; st < n_stage; ++st) {
                mbar_wait(&empty[(int)(st % S)], (uint32_t)(((st / S) - 1) & 1));
                issue(st);
            }
        }
    }
    P ag[VPT][NP], ab[VPT][NP];  // per-example dgamma/dbeta partials of this thread's columns
    if (!C::PROD || warp < NW) {  // row-math warps

    bool vok[VPT];
    int vo[VPT];  // element offset of this thread's k-th vector inside a row
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        vok[k] = (tig + k * GT) < NVp;
        vo[k] = (vok[k] ? tig + k * GT : 0) * W;
    }

#pragma unroll
    for (int k = 0; k < VPT; ++k)
#pragma unroll
        for (int p = 0; p < NP; ++p) ag[k][p] = ab[k][p] = PR::splat(Acc(0));

    int64_t cur_ex = r_begin / M;
    int64_t next_bound = (cur_ex + 1) * M;

    // write this group's register partials to slot (cta + ex, g)
    const int64_t ex_first = r_begin / M;
    auto write_slot = [&](int64_t ex, bool zero) {
        Acc* base = (C::kPark && ex == ex_first) ? park + (size_t)g * 2 * Dp
                                                   : partial + ((size_t)(cta + ex) * G + g) * 2 * Dp;
        // 16-byte stores: a thread's vector is contiguous and Dp is a multiple
        // of the vector width.  8-byte pair stores (one 8-byte piece in each
        // of 32 sectors per warp store, twice as many stores) clog the CTA's
        // load/store pipe at an example boundary: boundary-crossing CTAs ran
        // ~1.5 us longer at D = 1024 and set the launch's tail.
        constexpr int PPC = C::kWide ? 16 / (int)sizeof(P) : 1;  // pairs per store
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!vok[k]) continue;
#pragma unroll
            for (int c = 0; c < NP / PPC; ++c) {
                Acc* dg = base + vo[k] + 2 * PPC * c;
                Acc* db = dg + Dp;
                if constexpr (PPC == 1) {
                    *reinterpret_cast<P*>(dg) = zero ? PR::splat(Acc(0)) : ag[k][c];
                    *reinterpret_cast<P*>(db) = zero ? PR::splat(Acc(0)) : ab[k][c];
                } else {
                    const uint4 z = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(dg) = zero ? z : pack2<Acc>(&ag[k][PPC * c]);
                    *reinterpret_cast<uint4*>(db) = zero ? z : pack2<Acc>(&ab[k][PPC * c]);
                }
            }
        }
    };
    auto flush_to = [&](int64_t new_ex) {
        write_slot(cur_ex, false);
#if GNSB_LN_EARLYFOLD
        if constexpr (G > 1 && !C::kPark && !C::kNoFold) {
            // The CTA's first example ends here for this group.  The last group
            // to get past it folds the G group slots into slot 0 now, while
            // the other groups keep streaming rows, instead of in the
            // end-of-kernel fold behind the CTA's last row.
            if (cur_ex == ex_first) {
                __threadfence_block();
                named_bar_sync(1 + g, GT);
                if (tig == 0) s_fold_last[g] = atomicAdd(&s_fold_cnt, 1) == G - 1;
                named_bar_sync(1 + g, GT);
                if (s_fold_last[g]) {
                    __threadfence_block();
                    constexpr int E = 16 / sizeof(Acc);
                    Acc* fb = partial + (size_t)(cta + ex_first) * G * 2 * Dp;
                    for (int i = tig; i < 2 * Dp / E; i += GT) {
                        uint4 v[G];
#pragma unroll
                        for (int gg = 0; gg < G; ++gg)
                            v[gg] = __ldcg(reinterpret_cast<const uint4*>(fb + (size_t)gg * 2 * Dp + i * E));
                        Acc t[E];
#pragma unroll
                        for (int e = 0; e < E; ++e) t[e] = reinterpret_cast<const Acc*>(&v[0])[e];
#pragma unroll
                        for (int gg = 1; gg < G; ++gg)
#pragma unroll
                            for (int e = 0; e < E; ++e) t[e] += reinterpret_cast<const Acc*>(&v[gg])[e];
                        *reinterpret_cast<uint4*>(fb + i * E) = *reinterpret_cast<const uint4*>(t);
                    }
                    if (tig == 0) s_early = 1;
                }
            }
        }
#endif
#pragma unroll
        for (int k = 0; k < VPT; ++k)
#pragma unroll
            for (int p = 0; p < NP; ++p) ag[k][p] = ab[k][p] = PR::splat(Acc(0));
        for (int64_t ex = cur_ex + 1; ex < new_ex; ++ex) write_slot(ex, true);
        cur_ex = new_ex;
        next_bound = (cur_ex + 1) * M;
    };

    // xhat and h = gamma*g of a staged vector
    auto make_xh = [&](const uint4& ux, const uint4& ug, int k, Acc mu, Acc rs, P* x2, P* h2, P* g2) {
        P xf[NP];
        unpack2<T>(ux, xf);
        unpack2<T>(ug, g2);
        const P* gp = reinterpret_cast<const P*>(gam_s + vo[k]);
        const P rs2 = PR::splat(rs), nmr2 = PR::splat(-mu * rs);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            x2[p] = HAS_MEAN ? PR::fma(xf[p], rs2, nmr2) : xf[p];
            h2[p] = PR::mul(gp[p], g2[p]);
        }
    };

    // One stage.  FULL: every row of the stage is valid (all but the last).
    int rbuf = 0;
    auto stage = [&](auto full_tag, int slot, int64_t r0, int nr) {
        constexpr bool FULL = decltype(full_tag)::value;
        const T* sx = ring + (size_t)slot * 2 * R * Dp + (size_t)(g * RPG) * Dp;
        const T* sdy = sx + (size_t)R * Dp;
        const Acc* stp = stats + ((size_t)slot * R + g * RPG) * 2;
        Acc mu[RPG], rs[RPG];
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
            const bool valid = FULL || g * RPG + i < nr;
            mu[i] = valid ? stp[2 * i] : Acc(0);
            rs[i] = valid ? stp[2 * i + 1] : Acc(0);
        }

        uint4 ux[RPG][VPT], ug[RPG][VPT];
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
            const bool valid = FULL || g * RPG + i < nr;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                const int off = i * Dp + vo[k];
                if (valid && vok[k]) {
                    ux[i][k] = *reinterpret_cast<const uint4*>(sx + off);
                    ug[i][k] = *reinterpret_cast<const uint4*>(sdy + off);
                } else {
                    ux[i][k] = ug[i][k] = make_uint4(0, 0, 0, 0);
                }
            }
        }
        if constexpr (KEEP) {  // everything needed is in registers: release the slot now
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }

        // pass 1: row sums (split chains per vector), column partials
        P xh[KEEP ? RPG : 1][KEEP ? VPT : 1][NP], hh[KEEP ? RPG : 1][KEEP ? VPT : 1][NP];
        Acc q[NQ];
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
            const bool valid = FULL || g * RPG + i < nr;
            const int64_t row = r0 + g * RPG + i;
            if (valid && row >= next_bound) flush_to(row / M);  // group-uniform
            P s1[VPT], s2[VPT];
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                s1[k] = s2[k] = PR::splat(Acc(0));
                P x2[NP], h2[NP], g2[NP];
                make_xh(ux[i][k], ug[i][k], k, valid ? mu[i] : Acc(0), valid ? rs[i] : Acc(0), x2, h2, g2);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    s1[k] = PR::add(s1[k], h2[p]);
                    s2[k] = PR::fma(h2[p], x2[p], s2[k]);
                    ag[k][p] = PR::fma(x2[p], g2[p], ag[k][p]);
                    ab[k][p] = PR::add(ab[k][p], g2[p]);
                    if constexpr (KEEP) {
                        xh[i][k][p] = x2[p];
                        hh[i][k][p] = h2[p];
                    }
                }
            }
#pragma unroll
            for (int k = 1; k < VPT; ++k) {
                s1[0] = PR::add(s1[0], s1[k]);
                s2[0] = PR::add(s2[0], s2[k]);
            }
            q[2 * i] = s1[0].x + s1[0].y;
            q[2 * i + 1] = s2[0].x + s2[0].y;
        }
        // row reductions over the group: transposed butterfly within the
        // warp, then a padded xor tree over the group's warps
        butterfly_sum<NQ>(q, lane);
        Acc tot[NQ];
        if constexpr (GW == 1) {
#pragma unroll
            for (int j = 0; j < NQ; ++j) tot[j] = __shfl_sync(0xffffffffu, q[0], j * (32 / NQ));
        } else {
            Acc* rb = red + (size_t)(rbuf * G + g) * NQ * GWP;
            if ((lane & (32 / NQ - 1)) == 0) rb[(lane / (32 / NQ)) * GWP + wig] = q[0];
            named_bar_sync(1 + g, GT);
            // rb is [NQ][GWP]; each lane folds E entries over the GWP-lane groups
            constexpr int TOT = NQ * GWP;
            constexpr int E = TOT > 32 ? TOT / 32 : 1;
            Acc t[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int idx = lane + 32 * e;
                t[e] = (idx < TOT && (idx % GWP) < GW) ? rb[idx] : Acc(0);
            }
#pragma unroll
            for (int m = GWP / 2; m >= 1; m >>= 1)
#pragma unroll
                for (int e = 0; e < E; ++e) t[e] += __shfl_xor_sync(0xffffffffu, t[e], m);
#pragma unroll
            for (int j = 0; j < NQ; ++j) tot[j] = __shfl_sync(0xffffffffu, t[(j * GWP) / 32], (j * GWP) % 32);
            rbuf ^= 1;
        }
        // pass 2: dx = rstd*(h - mean(h)) - rstd*mean(h*xhat)*xhat
        if (dxg != nullptr) {
            T* dxs = dxg + (r0 + g * RPG) * D;  // 64-bit base once per stage
#pragma unroll
            for (int i = 0; i < RPG; ++i) {
                if (!FULL && g * RPG + i >= nr) continue;
                const P rs2 = PR::splat(rs[i]);
                const P k1 = PR::splat(-rs[i] * tot[2 * i] * invD);
                const P nc2 = PR::splat(-rs[i] * tot[2 * i + 1] * invD);
#pragma unroll
                for (int k = 0; k < VPT; ++k) {
                    if (!vok[k]) continue;
                    P o[NP];
                    if constexpr (KEEP) {
#pragma unroll
                        for (int p = 0; p < NP; ++p) o[p] = PR::fma(nc2, xh[i][k][p], PR::fma(hh[i][k][p], rs2, k1));
                    } else {
                        P x2[NP], h2[NP], g2[NP];
                        make_xh(ux[i][k], ug[i][k], k, mu[i], rs[i], x2, h2, g2);
#pragma unroll
                        for (int p = 0; p < NP; ++p) o[p] = PR::fma(nc2, x2[p], PR::fma(h2[p], rs2, k1));
                    }
                    T* dst = dxs + (uint32_t)(i * (int)D + vo[k]);
                    if (a.aligned) {
                        st_stream(dst, pack2<T>(o));
                    } else {
                        const Acc* of = reinterpret_cast<const Acc*>(o);
#pragma unroll
                        for (int e = 0; e < W; ++e)
                            if (vo[k] + e < D) dst[e] = from_acc<T>(of[e]);
                    }
                }
            }
        }
        if constexpr (!KEEP) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    };

    const int64_t n_full = (r_end - r_begin) / R;
    int slot = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < n_stage; ++it) {
        if (!C::PROD && warp == 0) refill(it);
        mbar_wait(&full[slot], ph);
        const int64_t r0 = r_begin + it * R;
        if (it < n_full)
            stage(std::true_type{}, slot, r0, R);
        else
            stage(std::false_type{}, slot, r0, (int)(r_end - r0));
        if (++slot == S) {
            slot = 0;
            ph ^= 1u;
        }
    }
    // examples before the CTA's last one go to their global slots now; the
    // last one stays in registers for the CTA-local fold below
    if (G == 1 || C::kNoFold) {
        flush_to((r_end - 1) / M + 1);
    } else if (cur_ex < (r_end - 1) / M) {
        flush_to((r_end - 1) / M);
    }
    }  // row-math warps

    stamp(1);
    if constexpr (G > 1 && !C::kNoFold) {
        // CTA-local fold of the G group partials of every example this CTA
        // touched into group 0's slot, in fixed order g = 0..G-1.  The last
        // example's partials go through shared memory (the ring is free once
        // every warp passed this barrier), earlier examples' through L2.
        __syncthreads();
        constexpr int E = 16 / sizeof(Acc);  // Acc per 16-byte vector (Dp is a multiple of E)
        Acc* fold = reinterpret_cast<Acc*>(smem + C::rows_off(S, a.Dp));  // [G][2][Dp]
        if (!C::PROD || warp < NW) {
            const int g = warp / GW, tig = (warp % GW) * 32 + lane;
            // (register partials of the last example; zero if the group had no rows of it)
            Acc* fb = fold + (size_t)g * 2 * Dp;
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                if (tig + k * GT >= NVp) continue;
                constexpr int PPC = C::kWide ? 16 / (int)sizeof(P) : 1;
#pragma unroll
                for (int c = 0; c < NP / PPC; ++c) {
                    Acc* dg = fb + (tig + k * GT) * W + 2 * PPC * c;
                    if constexpr (PPC == 1) {
                        *reinterpret_cast<P*>(dg) = ag[k][c];
                        *reinterpret_cast<P*>(dg + Dp) = ab[k][c];
                    } else {
                        *reinterpret_cast<uint4*>(dg) = pack2<Acc>(&ag[k][PPC * c]);
                        *reinterpret_cast<uint4*>(dg + Dp) = pack2<Acc>(&ab[k][PPC * c]);
                    }
                }
            }
        }
        __syncthreads();
        const int64_t e0 = r_begin / M, e1 = (r_end - 1) / M;
        Acc* part = static_cast<Acc*>(a.partial);
        for (int64_t ex = e0; ex <= e1; ++ex) {
#if GNSB_LN_EARLYFOLD
            if (!C::kPark && ex == e0 && e0 < e1 && s_early) continue;  // folded at its boundary
#endif
            Acc* base = part + (size_t)(cta + ex) * G * 2 * Dp;
            // shared memory: the last example (registers -> ring) and the first
            // (parked at its boundary); L2: examples in between (short rows)
            const bool on_chip = ex == e1 || (C::kPark && ex == e0);
            const Acc* src = ex == e1 ? fold : (C::kPark && ex == e0) ? park : base;
            for (int i = threadIdx.x; i < 2 * Dp / E; i += blockDim.x) {
                uint4 v[G];
#pragma unroll
                for (int gg = 0; gg < G; ++gg)
                    v[gg] = on_chip ? *reinterpret_cast<const uint4*>(src + (size_t)gg * 2 * Dp + i * E)
                                    : __ldcg(reinterpret_cast<const uint4*>(src + (size_t)gg * 2 * Dp + i * E));
                Acc t[E];
#pragma unroll
                for (int e = 0; e < E; ++e) t[e] = reinterpret_cast<const Acc*>(&v[0])[e];
#pragma unroll
                for (int gg = 1; gg < G; ++gg)
#pragma unroll
                    for (int e = 0; e < E; ++e) t[e] += reinterpret_cast<const Acc*>(&v[gg])[e];
                *reinterpret_cast<uint4*>(base + i * E) = *reinterpret_cast<const uint4*>(t);
            }
        }
    }
    stamp(2);
}

// ---------------------------------------------------------------- stage 2 --
// Separate kernel, launched with programmatic dependent launch right behind
// the row kernel.  CTA c owns the contiguous range of 16-byte column vectors
// [c*U/grid, (c+1)*U/grid).  Per block of examples it first stages its
// column slice of every slot the block needs into shared memory with
// independent, coalesced loads (one L2 round trip, no dependent chains),
// then for every example sums the slots of the CTAs that touched it in fixed
// CTA order -> gamma'_b, beta'_b on its columns (fp64), squares and reduces
// them over its columns -> q[b][c], and sums over b in fixed order ->
// dgamma/dbeta (+ their squares -> qbig[c]).  The last CTA (ticket) folds q
// into raw_b and the scalar sums.  NORMS=false is the plain LayerNorm
// backward's reduction (dgamma/dbeta only).
constexpr int kMaxReduceGrid = 160;  // >= the B200's 148 SMs; bounds the final fold's unrolling
constexpr int kMaxReduceEb = 512;    // examples per shared-memory block
constexpr int kReduceThreads = 512;

struct LnRedLayout {  // shared-memory carve-up of the reduce kernel (host + device)
    int64_t ncol, eb, nslot_max;
    __host__ __device__ static int64_t slot_bytes(int64_t ncol, int acc) { return 2 * ncol * acc; }
    __host__ __device__ size_t colsum_off() const { return 0; }
    __host__ __device__ size_t sv_off() const { return (size_t)16 * ncol; }
    __host__ __device__ size_t stage_off() const { return (sv_off() + (size_t)8 * (2 * ncol + 1) * eb + 15) / 16 * 16; }
    __host__ __device__ size_t bytes(int acc) const {
        return stage_off() + (size_t)nslot_max * slot_bytes(ncol, acc);
    }
};

// The stage-2 work of CTA `cta` of the `grid` CTAs assigned to one LayerNorm.
template <typename Acc, bool NORMS>
__device__ __forceinline__ void ln_bwd_reduce_body(const LnRedArgs& a, const int cta, const int grid,
                                                   unsigned char* smem) {
    constexpr int V = 16 / sizeof(Acc);  // columns per 16-byte vector
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nthreads = blockDim.x, nwarps = nthreads / 32;
    const int64_t B = a.B, M = a.M, N = a.N, D = a.D;
    const int64_t U = (a.Dp + V - 1) / V;
    const int u0 = (int)((int64_t)cta * U / grid), u1 = (int)((int64_t)(cta + 1) * U / grid);
    const int nu = u1 - u0, ncol = nu * V;
    const int grid_rows = a.grid_rows;
    auto cta_of = [&](int64_t r) -> int64_t { return ((r + 1) * grid_rows - 1) / N; };
    LnRedLayout lay{ncol, a.eb, 0};
    double* colsum = reinterpret_cast<double*>(smem + lay.colsum_off());  // [2][ncol]
    double* sv = reinterpret_cast<double*>(smem + lay.sv_off());          // [eb][2 ncol + 1] (padded rows)
    const int svs = 2 * ncol + 1;
    uint4* stg = reinterpret_cast<uint4*>(smem + lay.stage_off());        // [slot][2][nu] 16-byte vectors
    __shared__ int s_cs[kMaxReduceEb], s_nc[kMaxReduceEb];
    __shared__ double s_raw[2][kMaxReduceEb];
    const uint4* part = static_cast<const uint4*>(a.partial);
    const int64_t sstride = a.slot_stride / V;  // in 16-byte vectors
    const int64_t half = a.Dp / V;              // beta row offset inside a slot
    auto stamp = [&](int k) {
        if (a.trace != nullptr && threadIdx.x == 0) a.trace[(size_t)cta * 6 + k] = globaltimer_ns();
    };

    for (int j = threadIdx.x; j < 2 * ncol; j += nthreads) colsum[j] = 0.0;
    __shared__ __align__(8) uint64_t s_bar;  // stage-area bulk copies
    uint32_t bar_phase = 0;
    const uint64_t pol = policy_evict_first();
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
    }
    // (the barrier before the first staging orders the init before any use)
    // the next kernel in the stream may start its prologue now (it waits for
    // this grid before touching global memory)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the row kernel's slots are complete and visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    stamp(0);

    for (int64_t b0 = 0; b0 < B; b0 += a.eb) {
        const int64_t nb = (B - b0) < a.eb ? (B - b0) : a.eb;
        // slots of this block: from the first CTA of example b0 to the last of
        // b0+nb-1 (gsub consecutive slots per CTA)
        const int gs = a.gsub;
        const int64_t s_lo = (cta_of(b0 * M) + b0) * gs;
        const int64_t s_hi = (cta_of((b0 + nb) * M - 1) + (b0 + nb - 1)) * gs + gs - 1;
        for (int bb = threadIdx.x; bb < nb; bb += nthreads) {
            const int64_t b = b0 + bb;
            s_cs[bb] = (int)((cta_of(b * M) + b) * gs - s_lo);  // first slot of example b, relative to s_lo
            s_nc[bb] = (int)((cta_of((b + 1) * M - 1) - cta_of(b * M) + 1) * gs);
        }
        // The block's slots are staged `slot_cap` at a time (one chunk unless a
        // single example spans more CTAs than fit, e.g. B = 1); the per-column
        // sums continue across chunks in the same fixed slot order.
        const int64_t nsl = s_hi - s_lo + 1;
        for (int64_t c0 = 0; c0 < nsl; c0 += a.slot_cap) {
            const int64_t cn = (nsl - c0) < a.slot_cap ? (nsl - c0) : a.slot_cap;
            const uint4* pbase = part + (s_lo + c0) * sstride + u0;
            // stage: one bulk copy (TMA) per (slot, half) column slice, all in
            // flight at once and completing on one mbarrier.  (16-byte loads,
            // 8 per thread in flight, left the grouped reduce latency-bound at
            // ~1-1.6 TB/s.)  The fence orders the previous chunk's generic
            // reads of the stage area before these async-proxy writes.
            const int nchunk = (int)cn * 2;
            const uint32_t cbytes = (uint32_t)nu * 16u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (threadIdx.x == 0) mbar_arrive_expect_tx(&s_bar, (uint32_t)nchunk * cbytes);
            __syncthreads();
            for (int c = threadIdx.x; c < nchunk; c += nthreads)
                bulk_g2s(stg + (size_t)c * nu, pbase + (int64_t)(c >> 1) * sstride + (c & 1) * half, cbytes, &s_bar,
                         pol);
            mbar_wait(&s_bar, bar_phase);
            bar_phase ^= 1u;
            if (b0 == 0 && c0 == 0) stamp(1);
            // per (example, column pair): fixed-order sum over the example's
            // CTAs (two columns per thread: pair loads, 4 independent chains)
            const int hc = ncol / 2;  // ncol is a multiple of the 16-byte vector width
            const int items = (int)nb * hc;
            const Acc* sa = reinterpret_cast<const Acc*>(stg);
            using A2 = typename Pair<Acc>::P;
            for (int it = threadIdx.x; it < items; it += nthreads) {
                const int bb = it / hc;
                const int j = 2 * (it - bb * hc);
                const int64_t lo = s_cs[bb] > c0 ? s_cs[bb] : c0;
                const int64_t hi = (s_cs[bb] + s_nc[bb]) < (c0 + cn) ? (s_cs[bb] + s_nc[bb]) : (c0 + cn);
                double* o = sv + (size_t)bb * svs + j;
                double g0 = c0 == 0 ? 0.0 : o[0], g1 = c0 == 0 ? 0.0 : o[1];
                double e0 = c0 == 0 ? 0.0 : o[ncol], e1 = c0 == 0 ? 0.0 : o[ncol + 1];
                const Acc* sg = sa + (size_t)(lo - c0) * 2 * ncol + j;
                const int n = (int)(hi - lo);
#pragma unroll 4
                for (int c = 0; c < n; ++c) {
                    const A2 vg = *reinterpret_cast<const A2*>(sg + (size_t)c * 2 * ncol);
                    const A2 vb = *reinterpret_cast<const A2*>(sg + (size_t)c * 2 * ncol + ncol);
                    g0 += (double)vg.x;
                    g1 += (double)vg.y;
                    e0 += (double)vb.x;
                    e1 += (double)vb.y;
                }
                o[0] = g0;
                o[1] = g1;
                o[ncol] = e0;
                o[ncol + 1] = e1;
            }
            __syncthreads();
            if (b0 == 0 && c0 == 0) stamp(5);
        }
        // two roles over the same read-only sv (no barrier between them): a
        // thread per column adds it over the block's examples; a warp per
        // example squares and sums it over this CTA's columns (lane-strided,
        // then a fixed butterfly: the chain per lane is ncol/16 long, not
        // 2 ncol).  Both in fixed order.  (A warp per two examples and four
        // lanes per column sum were both measured slower at D >= 2048.)
        for (int j = threadIdx.x; j < 2 * ncol; j += nthreads) {
            const int h = j / ncol, jj = j - h * ncol;
            double acc = 0.0;
#pragma unroll 8
            for (int64_t bb = 0; bb < nb; ++bb) acc += sv[bb * svs + h * ncol + jj];
            colsum[j] += acc;
        }
        if constexpr (NORMS) {
            for (int r = warp; r < nb; r += nwarps) {
                const double* vg = sv + (size_t)r * svs;
                double q2[2] = {0.0, 0.0};
                for (int j = lane; j < ncol; j += 32) {
                    q2[0] = fma(vg[j], vg[j], q2[0]);
                    q2[1] = fma(vg[ncol + j], vg[ncol + j], q2[1]);
                }
                warp_sum_n(q2);
                if (lane == 0) {
                    a.q[((size_t)(b0 + r) * grid + cta) * 2 + 0] = q2[0];
                    a.q[((size_t)(b0 + r) * grid + cta) * 2 + 1] = q2[1];
                }
            }
        }
        __syncthreads();
    }
    if (warp == 0) {
        Acc* dgam = static_cast<Acc*>(a.dgamma);
        Acc* dbet = static_cast<Acc*>(a.dbeta);
        double qg = 0.0, qb = 0.0;
        for (int j = lane; j < ncol; j += 32) {
            const int64_t col = (int64_t)u0 * V + j;
            if (col >= D) continue;
            const Acc fg = (Acc)colsum[j], fb = (Acc)colsum[ncol + j];
            dgam[col] = fg;
            dbet[col] = fb;
            qg = fma((double)fg, (double)fg, qg);
            qb = fma((double)fb, (double)fb, qb);
        }
        if constexpr (NORMS) {
            qg = warp_sum(qg);
            qb = warp_sum(qb);
            if (lane == 0) {
                a.qbig[(size_t)cta * 2 + 0] = qg;
                a.qbig[(size_t)cta * 2 + 1] = qb;
            }
        }
    }
    stamp(2);
    if constexpr (!NORMS) return;

    // ------------------------------------------------------- final ticket --
    __shared__ unsigned s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        // release: the barrier above orders every thread's q/qbig stores
        // before this (cumulative) gpu-scope release; acquire: the last CTA
        // sees every other CTA's stores, and the barrier below passes that
        // on to its threads
        const unsigned t = atomic_add_acq_rel_gpu(a.ticket, 1u);
        s_last = (t == (unsigned)grid - 1u) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    stamp(3);
    // raw_b = sum over the grid's column ranges: lane l adds c = l, l+32, ...
    // in order, then a fixed butterfly.  Each warp takes kBW examples at a
    // time with every load (and warp 0's qbig loads) issued before the first
    // add, so for B <= kBW * warps the whole fold is one L2 round trip.
    constexpr int KC = (kMaxReduceGrid + 31) / 32;
    constexpr int kBW = 4;
    double qbg[KC], qbb[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        const int c = lane + 32 * k;
        const bool ok = warp == 0 && c < grid;
        qbg[k] = ok ? __ldcg(a.qbig + (size_t)c * 2 + 0) : 0.0;
        qbb[k] = ok ? __ldcg(a.qbig + (size_t)c * 2 + 1) : 0.0;
    }
    for (int64_t b0 = 0; b0 < B; b0 += (int64_t)nwarps * kBW) {
        double lg[kBW][KC], lb[kBW][KC];
#pragma unroll
        for (int i = 0; i < kBW; ++i) {
            const int64_t b = b0 + warp + (int64_t)i * nwarps;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int c = lane + 32 * k;
                const bool ok = b < B && c < grid;
                lg[i][k] = ok ? __ldcg(a.q + ((size_t)b * grid + c) * 2 + 0) : 0.0;
                lb[i][k] = ok ? __ldcg(a.q + ((size_t)b * grid + c) * 2 + 1) : 0.0;
            }
        }
        double rr[2 * kBW];
#pragma unroll
        for (int i = 0; i < kBW; ++i) {
            double rg = 0.0, rb = 0.0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                rg += lg[i][k];
                rb += lb[i][k];
            }
            rr[2 * i] = rg;
            rr[2 * i + 1] = rb;
        }
        warp_sum_n(rr);
#pragma unroll
        for (int i = 0; i < kBW; ++i) {
            const int64_t b = b0 + warp + (int64_t)i * nwarps;
            const double rg = rr[2 * i], rb = rr[2 * i + 1];
            if (lane == 0 && b < B) {
                if (b < kMaxReduceEb) {
                    s_raw[0][b] = rg;
                    s_raw[1][b] = rb;
                } else {
                    a.rawws[b * 2 + 0] = rg;
                    a.rawws[b * 2 + 1] = rb;
                }
                if (a.raw_g) a.raw_g[b] = rg;
                if (a.raw_b) a.raw_b[b] = rb;
            }
        }
    }
    __syncthreads();
    if (warp == 0 && a.sums != nullptr) {
        double tg = 0.0, tb = 0.0, bg = 0.0, bb = 0.0;
        for (int64_t b = lane; b < B; b += 32) {
            tg += b < kMaxReduceEb ? s_raw[0][b] : __ldcg(a.rawws + b * 2 + 0);
            tb += b < kMaxReduceEb ? s_raw[1][b] : __ldcg(a.rawws + b * 2 + 1);
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            bg += qbg[k];
            bb += qbb[k];
        }
        double t4[4] = {tg, tb, bg, bb};
        warp_sum_n(t4);
        if (lane == 0) {
            a.sums[0] = t4[0];
            a.sums[1] = t4[1];
            a.sums[2] = t4[2];
            a.sums[3] = t4[3];
        }
    }
    if (threadIdx.x == 0) *a.ticket = 0u;  // (visible to the next kernel at grid completion)
    stamp(4);
}

template <typename Acc, bool NORMS>
__global__ void __launch_bounds__(kReduceThreads) ln_bwd_reduce_kernel(LnRedArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    ln_bwd_reduce_body<Acc, NORMS>(a, blockIdx.x, gridDim.x, smem);
}

// Deferred stage 2 of several LayerNorms in one launch: CTAs
// [begin[l], begin[l+1]) work on layer l (each layer keeps its own workspace,
// ticket and outputs).  Amortises the stage-2 tail over a whole backward.
constexpr int kMaxReduceGroup = 64;
struct LnRedGroup {
    LnRedArgs items[kMaxReduceGroup];
    int begin[kMaxReduceGroup + 1];
    int n;
};

template <typename Acc, bool NORMS>
__global__ void __launch_bounds__(kReduceThreads) ln_bwd_reduce_group_kernel(const __grid_constant__ LnRedGroup g) {
    extern __shared__ __align__(16) unsigned char smem[];
    int l = 0;
    while (l + 1 < g.n && (int)blockIdx.x >= g.begin[l + 1]) ++l;
    ln_bwd_reduce_body<Acc, NORMS>(g.items[l], (int)blockIdx.x - g.begin[l], g.begin[l + 1] - g.begin[l], smem);
}

}  // namespace gnsb

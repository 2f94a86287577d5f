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
//     slot (cta + example, group) of an L2-resident workspace;
//   * stage 2 after a software grid barrier: column chunks sum the slots of
//     each example in fixed (cta, group) order -> gamma'_b; square and reduce
//     over D in fp64 -> per-(example, chunk) partial norms; fixed-order sum
//     over b -> dgamma/dbeta;
//   * the last CTA (ticket) folds chunk partials into raw_b and the scalar sums
//     and resets the workspace counters.  No float atomics anywhere: results
//     are bitwise deterministic run to run.
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
    void* dgamma;       // [D] Acc
    void* dbeta;        // [D] Acc
    double* raw_g;      // [B] or null
    double* raw_b;      // [B] or null
    double* sums;       // [4] or null: sum raw_g, sum raw_b, ||dgamma||^2, ||dbeta||^2
    int64_t B, M, N, D;
    int Dp;             // smem row stride in elements (D rounded up to the vector width)
    int stages;         // ring depth
    int aligned;        // 1: rows are 16-byte aligned -> TMA producer
    void* partial;      // [(grid + B) * G][2][Dp] Acc
    double* q;          // [B][nchunks][2]
    double* qbig;       // [nchunks][2]
    double* rawws;      // [B][2]
    unsigned* counters; // [2] grid barrier, final ticket (zero on entry, zero on exit)
    int nchunks;
    int64_t scratch_bytes;      // shared memory available to stage 2 (the ring region)
    unsigned long long* trace;  // optional [grid][6] globaltimer stamps (profiling only)
};

constexpr int kChunk = 16;  // stage-2 column chunk (half a warp)

template <typename T, int GW, int VPT, int G, int RPG, bool PROD_ = true, int KEEP_ = -1>
struct LnBwdCfg {
    using Acc = typename Traits<T>::Acc;
    using Row = T;
    static constexpr int kGW = GW, kVPT = VPT, kG = G, kRPG = RPG;
    static constexpr int W = Traits<T>::W;
    static constexpr bool PROD = PROD_;          // dedicated producer warp (the last warp)
    static constexpr int kWarps = GW * G;        // row-math warps
    static constexpr int kThreads = (kWarps + (PROD ? 1 : 0)) * 32;
    // registers are allocated for warps in groups of 4: bound the register
    // budget by the rounded-up block so one CTA always fits on an SM
    static constexpr int kBoundThreads = (kThreads + 127) / 128 * 128;
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
    static __host__ __device__ constexpr size_t smem_bytes(int S, int Dp) {
        // the ring doubles as the stage-2 scratch: >= [2][16][J] doubles for the
        // fold over examples (J = threads / 16) and >= one example's [2][16]
        const size_t ring = (size_t)S * stage_row_bytes(Dp);
        const size_t scratch = (size_t)16 * kThreads > 256 ? (size_t)16 * kThreads : 256;
        return rows_off(S, Dp) + (ring > scratch ? ring : scratch);
    }
};

template <typename C, bool HAS_MEAN, bool NORMS>
__global__ void __launch_bounds__(C::kBoundThreads, 1) ln_bwd_kernel(LnBwdArgs a) {
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
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    if (!a.aligned) {  // padded rows: the pad columns must read as zero
        uint4* p = reinterpret_cast<uint4*>(ring);
        const size_t n16 = (size_t)S * C::stage_row_bytes(Dp) / 16;
        for (size_t i = threadIdx.x; i < n16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();

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
        if (a.aligned && (D * (int64_t)sizeof(Acc)) % 16 == 0) {
            constexpr int E = 16 / sizeof(Acc);
            for (int i = threadIdx.x; i < Dp / E; i += blockDim.x)
                *reinterpret_cast<uint4*>(gam_s + i * E) = __ldg(reinterpret_cast<const uint4*>(gg) + i);
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
    if (!C::PROD || warp < NW) {  // row-math warps

    bool vok[VPT];
    int vo[VPT];  // element offset of this thread's k-th vector inside a row
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        vok[k] = (tig + k * GT) < NVp;
        vo[k] = (vok[k] ? tig + k * GT : 0) * W;
    }

    P ag[VPT][NP], ab[VPT][NP];
#pragma unroll
    for (int k = 0; k < VPT; ++k)
#pragma unroll
        for (int p = 0; p < NP; ++p) ag[k][p] = ab[k][p] = PR::splat(Acc(0));

    int64_t cur_ex = r_begin / M;
    int64_t next_bound = (cur_ex + 1) * M;

    // write this group's register partials to slot (cta + ex, g)
    auto write_slot = [&](int64_t ex, bool zero) {
        Acc* base = partial + ((size_t)(cta + ex) * G + g) * 2 * Dp;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!vok[k]) continue;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const P z = PR::splat(Acc(0));
                *reinterpret_cast<P*>(base + vo[k] + 2 * p) = zero ? z : ag[k][p];
                *reinterpret_cast<P*>(base + (size_t)Dp + vo[k] + 2 * p) = zero ? z : ab[k][p];
            }
        }
    };
    auto flush_to = [&](int64_t new_ex) {
        write_slot(cur_ex, false);
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
    flush_to((r_end - 1) / M + 1);
    }  // row-math warps

    stamp(1);
    if constexpr (G > 1) {
        // CTA-local pre-combine: fold the G group partials of every example this
        // CTA touched into group 0's slot (fixed order g = 0..G-1), so stage 2
        // reads one slot per (cta, example)
        __syncthreads();
        const int64_t e0 = r_begin / M, e1 = (r_end - 1) / M;
        constexpr int E = 16 / sizeof(Acc);  // Acc per 16-byte vector (Dp is a multiple of E)
        for (int64_t ex = e0; ex <= e1; ++ex) {
            Acc* base = static_cast<Acc*>(a.partial) + (size_t)(cta + ex) * G * 2 * Dp;
            for (int i = threadIdx.x; i < 2 * Dp / E; i += blockDim.x) {
                uint4 v[G];
#pragma unroll
                for (int gg = 0; gg < G; ++gg) v[gg] = *reinterpret_cast<const uint4*>(base + (size_t)gg * 2 * Dp + i * E);
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

    // ------------------------------------------------------------ stage 2 --
    stamp(2);
    grid_barrier(&a.counters[0]);
    stamp(3);

    const Acc* part_r = static_cast<const Acc*>(a.partial);
    Acc* dgam = static_cast<Acc*>(a.dgamma);
    Acc* dbet = static_cast<Acc*>(a.dbeta);
    const int nthreads = blockDim.x;
    const int NB = nthreads / kChunk;
    const int cl = threadIdx.x % kChunk, bl = threadIdx.x / kChunk;
    const unsigned hmask = 0xffffu << (lane & 16);
    double* sred = reinterpret_cast<double*>(smem + C::rows_off(S, Dp));  // ring is free now
    const int64_t B = a.B;
    auto cta_of = [&](int64_t r) -> int64_t { return ((r + 1) * grid - 1) / N; };

    for (int chunk = cta; chunk < a.nchunks; chunk += grid) {
        const int64_t col = (int64_t)chunk * kChunk + cl;
        const bool cv = col < D;
        double sg = 0.0, sb = 0.0;
        for (int64_t b = bl; b < B; b += NB) {
            const int64_t c0 = cta_of(b * M), c1 = cta_of((b + 1) * M - 1);
            double vg = 0.0, vb = 0.0;
            if (cv) {
                // one (pre-combined) slot per CTA that touched example b; issue
                // eight CTAs' loads at a time, then add in fixed CTA order
                for (int64_t cc = c0; cc <= c1; cc += 8) {
                    Acc lg[8], lb[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const bool ok = cc + u <= c1;
                        const Acc* base = part_r + (size_t)(ok ? cc + u + b : 0) * G * 2 * Dp + col;
                        lg[u] = ok ? __ldcg(base) : Acc(0);
                        lb[u] = ok ? __ldcg(base + Dp) : Acc(0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        vg += (double)lg[u];
                        vb += (double)lb[u];
                    }
                }
            }
            sg += vg;
            sb += vb;
            if constexpr (NORMS) {
                double qg = vg * vg, qb = vb * vb;
#pragma unroll
                for (int o = kChunk / 2; o > 0; o >>= 1) {
                    qg += __shfl_xor_sync(hmask, qg, o);
                    qb += __shfl_xor_sync(hmask, qb, o);
                }
                if (cl == 0) {
                    a.q[((size_t)b * a.nchunks + chunk) * 2 + 0] = qg;
                    a.q[((size_t)b * a.nchunks + chunk) * 2 + 1] = qb;
                }
            }
        }
        sred[(size_t)bl * kChunk + cl] = sg;
        sred[(size_t)(NB + bl) * kChunk + cl] = sb;
        __syncthreads();
        if (bl == 0) {
            double tg = 0.0, tb = 0.0;
            for (int k = 0; k < NB; ++k) {
                tg += sred[(size_t)k * kChunk + cl];
                tb += sred[(size_t)(NB + k) * kChunk + cl];
            }
            if (cv) {
                dgam[col] = (Acc)tg;
                dbet[col] = (Acc)tb;
            }
            if constexpr (NORMS) {
                const double fg = cv ? (double)(Acc)tg : 0.0, fb = cv ? (double)(Acc)tb : 0.0;
                double qg = fg * fg, qb = fb * fb;
#pragma unroll
                for (int o = kChunk / 2; o > 0; o >>= 1) {
                    qg += __shfl_xor_sync(0xffffu, qg, o);
                    qb += __shfl_xor_sync(0xffffu, qb, o);
                }
                if (cl == 0) {
                    a.qbig[(size_t)chunk * 2 + 0] = qg;
                    a.qbig[(size_t)chunk * 2 + 1] = qb;
                }
            }
        }
        __syncthreads();
    }

    // ------------------------------------------------------- final ticket --
    __shared__ unsigned s_last;
    __syncthreads();
    stamp(4);
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(&a.counters[1], 1u);
        s_last = (t == (unsigned)grid - 1u) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if constexpr (NORMS) {
        const int nwarps = nthreads / 32;
        for (int64_t b = warp; b < B; b += nwarps) {
            double rg = 0.0, rb = 0.0;
            for (int ch = lane; ch < a.nchunks; ch += 32) {
                rg += __ldcg(a.q + ((size_t)b * a.nchunks + ch) * 2 + 0);
                rb += __ldcg(a.q + ((size_t)b * a.nchunks + ch) * 2 + 1);
            }
            rg = warp_sum(rg);
            rb = warp_sum(rb);
            if (lane == 0) {
                a.rawws[b * 2 + 0] = rg;
                a.rawws[b * 2 + 1] = rb;
                if (a.raw_g) a.raw_g[b] = rg;
                if (a.raw_b) a.raw_b[b] = rb;
            }
        }
        __syncthreads();
        if (warp == 0 && a.sums != nullptr) {
            double tg = 0.0, tb = 0.0, bg = 0.0, bb = 0.0;
            for (int64_t b = lane; b < B; b += 32) {
                tg += a.rawws[b * 2 + 0];
                tb += a.rawws[b * 2 + 1];
            }
            for (int ch = lane; ch < a.nchunks; ch += 32) {
                bg += __ldcg(a.qbig + (size_t)ch * 2 + 0);
                bb += __ldcg(a.qbig + (size_t)ch * 2 + 1);
            }
            tg = warp_sum(tg);
            tb = warp_sum(tb);
            bg = warp_sum(bg);
            bb = warp_sum(bb);
            if (lane == 0) {
                a.sums[0] = tg;
                a.sums[1] = tb;
                a.sums[2] = bg;
                a.sums[3] = bb;
            }
        }
    }
    if (threadIdx.x == 0) {
        a.counters[0] = 0u;
        a.counters[1] = 0u;
        __threadfence();
    }
    stamp(5);
}

}  // namespace gnsb

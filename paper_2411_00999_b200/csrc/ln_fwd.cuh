// ln_fwd.cuh — LayerNorm forward for sm_100a.
//
// Semantics: gnstk::layernorm_forward (proj/src/layers.cpp:189-229): per row
// mean, biased variance (two-pass, /D), inv = 1/sqrt(var + eps),
// xhat = (x - mean) * inv, y = gamma * xhat + beta.  Writes y, mean and rstd
// (the B200 backward's cache) and, optionally, xhat (the reference's
// LayerNormCache::normalized).
//
// A row group of GW warps owns one row at a time; each thread keeps VPT
// 16-byte vectors of the row in registers across both reduction passes, so the
// row is read from HBM exactly once.  Streaming loads/stores bypass L1 and are
// marked L2 evict-first.
#pragma once

#include "common.cuh"

namespace gnsb {

struct LnFwdArgs {
    const void* x;      // [N, D] T
    const void* gamma;  // [D] Acc
    const void* beta;   // [D] Acc
    void* y;            // [N, D] T (nullable)
    void* mean;         // [N] Acc (nullable)
    void* rstd;         // [N] Acc (nullable)
    void* xhat;         // [N, D] T (nullable)
    int64_t N, D;
    double eps;
    int aligned;
    int64_t Dp;  // D rounded up to the thread coverage (gamma/beta staging)
};

template <typename T, int GW, int VPT>
struct LnFwdCfg {
    // row groups per CTA (<= 15 when groups sync on named barriers 1..G)
    static constexpr int G0 = GW * 32 >= 1024 ? 1 : 1024 / (GW * 32);
    static constexpr int G = (GW > 1 && G0 > 15) ? 15 : G0;
    static constexpr int kThreads = G * GW * 32;
};

template <typename T, int GW, int VPT>
__global__ void __launch_bounds__(LnFwdCfg<T, GW, VPT>::kThreads) ln_fwd_kernel(LnFwdArgs a) {
    using Acc = typename Traits<T>::Acc;
    constexpr int W = Traits<T>::W;
    constexpr int G = LnFwdCfg<T, GW, VPT>::G;
    constexpr int GT = GW * 32;
    __shared__ Acc red[2][G][GW];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp / GW, wig = warp % GW, tig = wig * 32 + lane;
    const int64_t N = a.N, D = a.D;
    const T* xg = static_cast<const T*>(a.x);
    const Acc* gam = static_cast<const Acc*>(a.gamma);
    const Acc* bet = static_cast<const Acc*>(a.beta);
    T* yg = static_cast<T*>(a.y);
    T* xhg = static_cast<T*>(a.xhat);
    Acc* meang = static_cast<Acc*>(a.mean);
    Acc* rstdg = static_cast<Acc*>(a.rstd);
    const Acc invD = Acc(1) / Acc(D);
    const Acc eps = (Acc)a.eps;

    auto group_sum = [&](Acc v, int buf) -> Acc {
        v = warp_sum(v);
        if constexpr (GW == 1) {
            return v;
        } else {
            if (lane == 0) red[buf][g][wig] = v;
            named_bar_sync(1 + g, GT);
            Acc t = 0;
#pragma unroll
            for (int w = 0; w < GW; ++w) t += red[buf][g][w];
            return t;
        }
    };

    // gamma/beta staged once per CTA in shared memory; the next row's x is
    // loaded before this row's reductions (one row of latency hidden per group)
    extern __shared__ __align__(16) unsigned char fsmem[];
    Acc* gs = reinterpret_cast<Acc*>(fsmem);
    Acc* bs = gs + a.Dp;
    for (int64_t c = threadIdx.x; c < a.Dp; c += blockDim.x) {
        gs[c] = c < D ? gam[c] : Acc(0);
        bs[c] = c < D ? bet[c] : Acc(0);
    }
    __syncthreads();
    auto load_row = [&](int64_t row, Acc (&xv)[VPT][W]) {
        const T* xr = xg + row * D;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int64_t c0 = (int64_t)(tig + k * GT) * W;
            if (a.aligned) {
                if (c0 < D) {
                    unpack<T>(ld_stream(xr + c0), xv[k]);
                } else {
#pragma unroll
                    for (int e = 0; e < W; ++e) xv[k][e] = Acc(0);
                }
            } else {
#pragma unroll
                for (int e = 0; e < W; ++e) xv[k][e] = (c0 + e < D) ? to_acc<T>(xr[c0 + e]) : Acc(0);
            }
        }
    };

    const int64_t stride = (int64_t)gridDim.x * G;
    int64_t row = (int64_t)blockIdx.x * G + g;
    Acc xv[VPT][W];
    if (row < N) load_row(row, xv);
    for (; row < N; row += stride) {
        Acc xn[VPT][W];
        if (row + stride < N) load_row(row + stride, xn);
        Acc s = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k)
#pragma unroll
            for (int e = 0; e < W; ++e) s += xv[k][e];
        const Acc mu = group_sum(s, 0) * invD;
        Acc v = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k)
#pragma unroll
            for (int e = 0; e < W; ++e) {
                const int64_t col = (int64_t)(tig + k * GT) * W + e;
                const Acc d = xv[k][e] - mu;
                v += col < D ? d * d : Acc(0);
            }
        const Acc var = group_sum(v, 1) * invD;
        const Acc inv = Acc(1) / sqrt(var + eps);
        if (tig == 0) {
            if (meang) meang[row] = mu;
            if (rstdg) rstdg[row] = inv;
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int64_t c0 = (int64_t)(tig + k * GT) * W;
            if (c0 >= D) continue;
            Acc yo[W], xo[W];
#pragma unroll
            for (int e = 0; e < W; ++e) {
                const int64_t col = c0 + e;
                xo[e] = (xv[k][e] - mu) * inv;
                yo[e] = col < D ? gs[col] * xo[e] + bs[col] : Acc(0);
            }
            if (a.aligned) {
                if (yg) st_stream(yg + row * D + c0, pack<T>(yo));
                if (xhg) st_stream(xhg + row * D + c0, pack<T>(xo));
            } else {
#pragma unroll
                for (int e = 0; e < W; ++e)
                    if (c0 + e < D) {
                        if (yg) yg[row * D + c0 + e] = from_acc<T>(yo[e]);
                        if (xhg) xhg[row * D + c0 + e] = from_acc<T>(xo[e]);
                    }
            }
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k)
#pragma unroll
            for (int e = 0; e < W; ++e) xv[k][e] = xn[k][e];
    }
}

// ---------------------------------------------------------------------------
// TMA-ring variant (16-byte-aligned rows): the forward is a pure stream, so the
// bytes in flight per SM decide its speed.  A producer warp keeps S stages of R
// consecutive rows in flight with 1-D cp.async.bulk (L2 evict-first) on
// mbarriers; G row groups of GW warps consume one row of each stage
// (registers: the thread's VPT vectors of that row), do the two reductions
// (warp butterfly + cross-warp through shared memory) and stream y (and
// mean/rstd, x-hat) out.  CTA c owns rows [c*N/grid, (c+1)*N/grid).
template <typename T, int GW, int VPT, int G>
struct LnFwdRingCfg {
    static constexpr int kWarps = GW * G;
    static constexpr int kThreads = (kWarps + 1) * 32;  // + producer warp
    static constexpr int R = G;                          // rows per stage
    static __host__ __device__ constexpr size_t bars_bytes(int S) { return (size_t)16 * S; }
    static __host__ __device__ constexpr size_t red_off(int S) { return (bars_bytes(S) + 15) / 16 * 16; }
    static __host__ __device__ constexpr size_t gam_off(int S) {
        return red_off(S) + (size_t)2 * G * GW * sizeof(typename Traits<T>::Acc) * 2;
    }
    static __host__ __device__ constexpr size_t ring_off(int S, int64_t Dp) {
        return (gam_off(S) + (size_t)2 * Dp * sizeof(typename Traits<T>::Acc) + 127) / 128 * 128;
    }
    // ring rows are packed at stride D (one bulk copy per stage)
    static __host__ __device__ constexpr size_t smem_bytes(int S, int64_t Dp, int64_t D) {
        return ring_off(S, Dp) + (size_t)S * R * D * sizeof(T);
    }
};

// GBS: gamma/beta read from shared memory per row instead of held in registers
// (wide per-thread slices)
template <typename T, int GW, int VPT, int G, bool GBS = false, int MINB = 1>
__global__ void __launch_bounds__(LnFwdRingCfg<T, GW, VPT, G>::kThreads, MINB) ln_fwd_ring_kernel(LnFwdArgs a, int S) {
    using C = LnFwdRingCfg<T, GW, VPT, G>;
    using Acc = typename Traits<T>::Acc;
    constexpr int W = Traits<T>::W;
    constexpr int GT = GW * 32;
    constexpr int R = C::R;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    Acc* red = reinterpret_cast<Acc*>(smem + C::red_off(S));  // [2 buffers][2 sums][G][GW]
    Acc* gs = reinterpret_cast<Acc*>(smem + C::gam_off(S));
    const int64_t Dp = a.Dp;
    Acc* bs = gs + Dp;
    T* ring = reinterpret_cast<T*>(smem + C::ring_off(S, Dp));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grid = gridDim.x, cta = blockIdx.x;
    const int64_t N = a.N, D = a.D;
    const int64_t r_begin = (int64_t)cta * N / grid, r_end = (int64_t)(cta + 1) * N / grid;
    const int64_t n_stage = (r_end - r_begin + R - 1) / R;
    const T* xg = static_cast<const T*>(a.x);

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::kWarps);
        }
        fence_mbar_init();
    }
    {
        const Acc* gam = static_cast<const Acc*>(a.gamma);
        const Acc* bet = static_cast<const Acc*>(a.beta);
        for (int64_t c = threadIdx.x; c < Dp; c += blockDim.x) {
            gs[c] = c < D ? gam[c] : Acc(0);
            bs[c] = c < D ? bet[c] : Acc(0);
        }
    }
    __syncthreads();

    if (warp == C::kWarps) {  // ---- producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t st = 0; st < n_stage; ++st) {
                const int slot = (int)(st % S);
                if (st >= S) mbar_wait(&empty[slot], (uint32_t)(((st / S) - 1) & 1));
                const int64_t r0 = r_begin + st * R;
                const int nr = (int)((r_end - r0) < (int64_t)R ? (r_end - r0) : (int64_t)R);
                const uint32_t bytes = (uint32_t)(nr * D * (int64_t)sizeof(T));
                mbar_expect_tx(&full[slot], bytes);
                bulk_g2s(ring + (size_t)slot * R * D, xg + r0 * D, bytes, &full[slot], pol);
                mbar_arrive(&full[slot]);
            }
        }
        return;
    }

    // ---- consumers: group g takes row g of every stage
    const int g = warp / GW, wig = warp % GW, tig = wig * 32 + lane;
    T* yg = static_cast<T*>(a.y);
    T* xhg = static_cast<T*>(a.xhat);
    Acc* meang = static_cast<Acc*>(a.mean);
    Acc* rstdg = static_cast<Acc*>(a.rstd);
    const Acc invD = Acc(1) / Acc(D);
    const Acc eps = (Acc)a.eps;
    // both row sums in one round: warp butterflies, then one named barrier
    auto group_sum2 = [&](Acc& v1, Acc& v2, int buf) {
        Acc vv[2] = {v1, v2};
        warp_sum_n(vv);
        if constexpr (GW == 1) {
            v1 = vv[0];
            v2 = vv[1];
        } else {
            Acc* rb = red + ((size_t)(buf * 2) * G + g) * GW;
            Acc* rb2 = red + ((size_t)(buf * 2 + 1) * G + g) * GW;
            if (lane == 0) {
                rb[wig] = vv[0];
                rb2[wig] = vv[1];
            }
            named_bar_sync(1 + g, GT);
            if constexpr (GW <= 8) {  // a few vectorised shared loads: shortest latency
                Acc t1 = 0, t2 = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    t1 += rb[w];
                    t2 += rb2[w];
                }
                v1 = t1;
                v2 = t2;
            } else {
                // lanes 0..15 fold the first sum, lanes 16..31 the second: one
                // shared load and a 4-step butterfly instead of GW loads each
                static_assert(GW <= 16, "cross-warp fold assumes at most 16 warps per row");
                const int j = lane & 15;
                Acc t = j < GW ? (lane < 16 ? rb[j] : rb2[j]) : Acc(0);
#pragma unroll
                for (int m = 8; m >= 1; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
                v1 = __shfl_sync(0xffffffffu, t, 0);
                v2 = __shfl_sync(0xffffffffu, t, 16);
            }
        }
    };
    // the thread's gamma/beta columns, in registers for the whole kernel;
    // packed fp32x2 (FFMA2/FADD2) math on pairs of columns.  Rows are whole
    // 16-byte vectors here (D % W == 0), so a vector is either all in or all out.
    using PR = Pair<Acc>;
    using P = typename PR::P;
    constexpr int NP = W / 2;
    P gv[GBS ? 1 : VPT][NP], bv[GBS ? 1 : VPT][NP];
    bool vin[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t c0 = (int64_t)(tig + k * GT) * W;
        vin[k] = c0 < D;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if constexpr (!GBS) {
                gv[k][p] = vin[k] ? PR::make(gs[c0 + 2 * p], gs[c0 + 2 * p + 1]) : PR::splat(Acc(0));
                bv[k][p] = vin[k] ? PR::make(bs[c0 + 2 * p], bs[c0 + 2 * p + 1]) : PR::splat(Acc(0));
            }
        }
    }
    int slot = 0;
    uint32_t ph = 0;
    for (int64_t st = 0; st < n_stage; ++st) {
        mbar_wait(&full[slot], ph);
        const int64_t row = r_begin + st * R + g;
        const bool valid = row < r_end;
        P xv[VPT][NP];
        const T* sx = ring + ((size_t)slot * R + g) * D;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (valid && vin[k]) {
                unpack2<T>(*reinterpret_cast<const uint4*>(sx + (int64_t)(tig + k * GT) * W), xv[k]);
            } else {
#pragma unroll
                for (int p = 0; p < NP; ++p) xv[k][p] = PR::splat(Acc(0));
            }
        }
        // one-pass moments about a shift K = the row's first element (the
        // same value for every thread of the group): sum (x-K), sum (x-K)^2;
        // shifting keeps the cancellation of var = E[d^2] - E[d]^2 small
        const Acc K = valid ? to_acc<T>(sx[0]) : Acc(0);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // the row is in registers
        const int buf = (int)(st & 1);
        const P nK = PR::splat(-K);
        P s1p = PR::splat(Acc(0)), s2p = PR::splat(Acc(0));
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!vin[k]) continue;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const P d = PR::add(xv[k][p], nK);
                s1p = PR::add(s1p, d);
                s2p = PR::fma(d, d, s2p);
            }
        }
        Acc s1 = s1p.x + s1p.y, s2 = s2p.x + s2p.y;
        group_sum2(s1, s2, buf);
        const Acc m1 = s1 * invD;
        const Acc mu = K + m1;
        Acc var = s2 * invD - m1 * m1;
        var = var > Acc(0) ? var : Acc(0);
        const Acc inv = Acc(1) / sqrt(var + eps);
        if (valid) {
            if (tig == 0) {
                if (meang) meang[row] = mu;
                if (rstdg) rstdg[row] = inv;
            }
            const P inv2 = PR::splat(inv), nmi2 = PR::splat(-mu * inv);
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
                if (!vin[k]) continue;
                const int64_t c0 = (int64_t)(tig + k * GT) * W;
                P yo[NP], xo[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    xo[p] = PR::fma(xv[k][p], inv2, nmi2);
                    if constexpr (GBS)
                        yo[p] = PR::fma(reinterpret_cast<const P*>(gs + c0)[p], xo[p], reinterpret_cast<const P*>(bs + c0)[p]);
                    else
                        yo[p] = PR::fma(gv[k][p], xo[p], bv[k][p]);
                }
                if (yg) st_stream(yg + row * D + c0, pack2<T>(yo));
                if (xhg) st_stream(xhg + row * D + c0, pack2<T>(xo));
            }
        }
        if (++slot == S) {
            slot = 0;
            ph ^= 1u;
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-per-row variant for aligned rows up to 16 16-byte vectors per lane: a
// warp owns whole rows (lane l holds vectors l, l+32, ... as packed T), so
// both reductions are warp butterflies with no barrier.  PF: the warp loads
// its next row before reducing the current one (narrow rows); without PF the
// other warps of the SM hide the latency (wide rows, fewer registers).  The
// vectors stay packed in registers and are unpacked per pass.  gamma/beta are
// read from shared memory.  Two-pass moments from registers, as the reference.
template <typename T, int VPT, int MINB, bool PF>
__global__ void __launch_bounds__(256, MINB) ln_fwd_warp_kernel(LnFwdArgs a) {
    using Acc = typename Traits<T>::Acc;
    using PR = Pair<Acc>;
    using P = typename PR::P;
    constexpr int W = Traits<T>::W;
    constexpr int NP = W / 2;
    extern __shared__ __align__(16) unsigned char fsmem[];
    Acc* gs = reinterpret_cast<Acc*>(fsmem);
    const int64_t N = a.N, D = a.D;
    const int nvec = (int)(D / W);
    Acc* bs = gs + (size_t)nvec * W;
    {
        const Acc* gam = static_cast<const Acc*>(a.gamma);
        const Acc* bet = static_cast<const Acc*>(a.beta);
        for (int c = threadIdx.x; c < nvec * W; c += blockDim.x) {
            gs[c] = gam[c];
            bs[c] = bet[c];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t wpb = blockDim.x >> 5;
    const int64_t stride = (int64_t)gridDim.x * wpb;
    int64_t row = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
    const T* xg = static_cast<const T*>(a.x);
    T* yg = static_cast<T*>(a.y);
    T* xhg = static_cast<T*>(a.xhat);
    Acc* meang = static_cast<Acc*>(a.mean);
    Acc* rstdg = static_cast<Acc*>(a.rstd);
    const Acc invD = Acc(1) / Acc(D);
    const Acc eps = (Acc)a.eps;
    bool vin[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) vin[k] = lane + 32 * k < nvec;
    auto load = [&](int64_t r, uint4 (&v)[VPT]) {
        const T* xr = xg + r * D;
#pragma unroll
        for (int k = 0; k < VPT; ++k) v[k] = vin[k] ? ld_stream(xr + (lane + 32 * k) * W) : make_uint4(0, 0, 0, 0);
    };
    uint4 cur[VPT];
    if (PF && row < N) load(row, cur);
    for (; row < N; row += stride) {
        uint4 nxt[PF ? VPT : 1];
        if constexpr (PF) {
            if (row + stride < N) load(row + stride, nxt);
        } else {
            load(row, cur);
        }
        P s1 = PR::splat(Acc(0));
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            P xv[NP];
            unpack2<T>(cur[k], xv);
#pragma unroll
            for (int p = 0; p < NP; ++p) s1 = PR::add(s1, xv[p]);
        }
        const Acc mu = warp_sum(s1.x + s1.y) * invD;
        const P nmu = PR::splat(-mu);
        P s2 = PR::splat(Acc(0));
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!vin[k]) continue;
            P xv[NP];
            unpack2<T>(cur[k], xv);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const P d = PR::add(xv[p], nmu);
                s2 = PR::fma(d, d, s2);
            }
        }
        const Acc var = warp_sum(s2.x + s2.y) * invD;
        const Acc inv = Acc(1) / sqrt(var + eps);
        if (lane == 0) {
            if (meang) meang[row] = mu;
            if (rstdg) rstdg[row] = inv;
        }
        const P inv2 = PR::splat(inv), nmi2 = PR::splat(-mu * inv);
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (!vin[k]) continue;
            const int c0 = (lane + 32 * k) * W;
            const P* gp = reinterpret_cast<const P*>(gs + c0);
            const P* bp = reinterpret_cast<const P*>(bs + c0);
            P xv[NP], yo[NP], xo[NP];
            unpack2<T>(cur[k], xv);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                xo[p] = PR::fma(xv[p], inv2, nmi2);
                yo[p] = PR::fma(gp[p], xo[p], bp[p]);
            }
            if (yg) st_stream(yg + row * D + c0, pack2<T>(yo));
            if (xhg) st_stream(xhg + row * D + c0, pack2<T>(xo));
        }
        if constexpr (PF) {
#pragma unroll
            for (int k = 0; k < VPT; ++k) cur[k] = nxt[k];
        }
    }
}

}  // namespace gnsb

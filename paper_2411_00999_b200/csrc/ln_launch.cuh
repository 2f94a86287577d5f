// ln_launch.cuh — host-side planning and launch of the LayerNorm kernels.
// Included once per row dtype (ln_f32.cu, ln_bf16.cu, ln_f64.cu) so the
// template instantiations compile in parallel.
#pragma once

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"
#include "ln_bwd.cuh"
#include "ln_fwd.cuh"

namespace gnsb {

namespace {

inline int smem_optin_bytes() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

inline bool ptr16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// "max dynamic smem" attribute of a kernel: ensure_smem_attr (capi.cu) keeps
// ONE process-wide record per (kernel, device) and only ever raises the
// attribute.  (A per-translation-unit cache is wrong here: the reduce kernel
// template is instantiated in several TUs but is one device function, so a
// TU that set a smaller value would lower another TU's setting.)
inline cudaError_t ensure_smem(const void* kernel, size_t bytes) { return ensure_smem_attr(kernel, bytes); }

struct BwdPlan {
    int Dp = 0, stages = 0, threads = 0, grid = 0, G = 0;
    size_t smem = 0;
    size_t off_partial = 0, off_q = 0, off_qbig = 0, off_raw = 0, total = 0;
};

template <typename C>
int plan_bwd(int64_t B, int64_t M, int64_t D, BwdPlan& p, const char** why) {
    using T = typename C::Row;
    using Acc = typename Traits<T>::Acc;
    constexpr int W = Traits<T>::W;
    constexpr int G = C::kG;
    p.Dp = (int)((D + W - 1) / W * W);
    // kCps CTAs share an SM's shared memory (1 KB per CTA is reserved by the driver)
    const size_t budget = (C::kCps == 1) ? (size_t)smem_optin_bytes() - 1024
                                         : (size_t)(228 * 1024) / C::kCps - 2048;
    p.stages = 0;
    // Ring depth: 4 stages (~128 KB in flight per SM) beat 6-8 at every
    // width in the steady 8-layer step (D=768..8192: +4.5/+3/+1.4/+1/+0.5 %,
    // experiments/ln_steady_trace.py; 3 ties, 2 loses).  More reads in flight
    // than that only slow the dx write stream down.  GNSB_LN_MAX_STAGES
    // overrides it (tuning experiments).
    static const int max_stages = [] {
        const char* e = getenv("GNSB_LN_MAX_STAGES");
        const int v = e ? atoi(e) : 4;
        return v < 2 ? 2 : v > 8 ? 8 : v;
    }();
    for (int s = max_stages; s >= 2; --s)  // >= 2: pass 2 holds a slot while the next stage is consumed
        if (C::smem_bytes(s, p.Dp) <= budget) {
            p.stages = s;
            break;
        }
    if (p.stages == 0) {
        *why = "layers: trailing extent too wide for the shared-memory row ring";
        return 1;
    }
    p.smem = C::smem_bytes(p.stages, p.Dp);
    p.threads = C::kThreads;
    p.G = G;
    const int64_t N = B * M;
    const int sms = device_sm_count();
    p.grid = (int)(N < (int64_t)sms * C::kCps ? N : (int64_t)sms * C::kCps);
    if (p.grid < 1) p.grid = 1;
    size_t off = 256;  // counters
    p.off_partial = off;
    off = align_up(off + (size_t)(p.grid + B) * G * 2 * p.Dp * sizeof(Acc), 256);
    p.off_q = off;
    off = align_up(off + (size_t)B * sms * 2 * sizeof(double), 256);  // q: up to one column range per SM
    p.off_qbig = off;
    off = align_up(off + (size_t)sms * 2 * sizeof(double), 256);
    p.off_raw = off;
    off = align_up(off + (size_t)B * 2 * sizeof(double), 256);
    p.total = off;
    return 0;
}

template <typename C>
struct BwdOp {
    using T = typename C::Row;
    static int plan(int64_t B, int64_t M, int64_t D, BwdPlan& p, const char** why) {
        return plan_bwd<C>(B, M, D, p, why);
    }
    // Launch plans are cached per (device, B, M, D): the steady-state launch
    // path does no driver queries besides the launch itself.
    struct PlanKey {
        int dev;
        int64_t B, M, D;
        bool operator<(const PlanKey& o) const {
            return dev != o.dev ? dev < o.dev : B != o.B ? B < o.B : M != o.M ? M < o.M : D < o.D;
        }
    };
    static int cached_plan(int64_t B, int64_t M, int64_t D, BwdPlan& p, const char** why, cudaError_t* cerr) {
        static std::mutex mu;
        static std::map<PlanKey, BwdPlan> cache;
        int dev = 0;
        cudaGetDevice(&dev);
        const PlanKey key{dev, B, M, D};
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = cache.find(key);
            if (it != cache.end()) {
                p = it->second;
                return 0;
            }
        }
        if (plan_bwd<C>(B, M, D, p, why)) return 1;
        // one CTA per SM must fit; shrink the ring if not
        void (*ks[2])(LnBwdArgs) = {ln_bwd_kernel<C, true>, ln_bwd_kernel<C, false>};
        for (;;) {
            cudaError_t e = cudaSuccess;
            for (auto k : ks)
                if (e == cudaSuccess) e = ensure_smem(reinterpret_cast<const void*>(k), p.smem);
            int occ = 0;
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks[0], p.threads, p.smem);
            if (e != cudaSuccess) {
                *cerr = e;
                *why = "ln_bwd plan (smem attribute / occupancy)";
                return 2;
            }
            if (occ >= C::kCps) break;
            if (p.stages <= 2) {
                *cerr = cudaErrorLaunchOutOfResources;
                return 2;
            }
            --p.stages;
            p.smem = C::smem_bytes(p.stages, p.Dp);
        }
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = p;
        return 0;
    }

    static void fill_info(const BwdPlan& p, LnRedPlanInfo* info) {
        info->Dp = p.Dp;
        info->G = C::kG;
        info->gsub = C::kSub;
        info->grid_rows = p.grid;
        info->off_partial = p.off_partial;
        info->off_q = p.off_q;
        info->off_qbig = p.off_qbig;
        info->off_raw = p.off_raw;
        info->total = p.total;
    }

    // Row pass only: dx plus the per-(CTA, example) partial slots in c.ws.
    static int run_rows(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr,
                        LnRedPlanInfo* info) {
        BwdPlan p;
        if (int rc = cached_plan(c.B, c.M, c.D, p, why, cerr)) return rc;
        if (c.ws_bytes < p.total) {
            *why = "layers: workspace too small (query gnsb_ln_bwd_workspace_size)";
            return 1;
        }
        fill_info(p, info);
        LnBwdArgs a{};
        a.x = c.x;
        a.mean = c.mean;
        a.rstd = c.rstd;
        a.dy = c.dy;
        a.gamma = c.gamma;
        a.dx = c.dx;
        a.B = c.B;
        a.M = c.M;
        a.N = c.B * c.M;
        a.D = c.D;
        a.Dp = p.Dp;
        a.stages = p.stages;
        a.aligned = ((c.D * (int64_t)sizeof(T)) % 16 == 0) && ptr16(c.x) && ptr16(c.dy) && (c.dx == nullptr || ptr16(c.dx));
        // gamma may be a view into a flat parameter buffer at any offset
        a.gamma16 = ((c.D * (int64_t)sizeof(typename Traits<T>::Acc)) % 16 == 0) && ptr16(c.gamma);
        a.partial = static_cast<unsigned char*>(c.ws) + p.off_partial;
        a.trace = c.trace;

        void (*k)(LnBwdArgs) = c.mean != nullptr ? ln_bwd_kernel<C, true> : ln_bwd_kernel<C, false>;
        cudaLaunchAttribute pdl[1];
        pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pdl[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t kcfg = {};
        kcfg.gridDim = dim3(p.grid);
        kcfg.blockDim = dim3(p.threads);
        kcfg.dynamicSmemBytes = p.smem;
        kcfg.stream = st;
        kcfg.attrs = pdl;
        kcfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&kcfg, k, a);
        if (e != cudaSuccess) {
            *cerr = e;
            *why = "ln_bwd rows launch";
            return 2;
        }
        return 0;
    }

    static int run(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
        LnRedItem item{};
        if (int rc = run_rows(c, st, why, cerr, &item.info)) return rc;
        item.B = c.B;
        item.M = c.M;
        item.D = c.D;
        item.ws = c.ws;
        item.dgamma = c.dgamma;
        item.dbeta = c.dbeta;
        item.raw_g = c.raw_g;
        item.raw_b = c.raw_b;
        item.sums = c.sums;
        return ln_bwd_reduce_run(sizeof(typename C::Acc) == 8, c.norms, &item, 1, st, c.trace2, why, cerr);
    }
};

// Aligned rows of at most 16 16-byte vectors per lane: the warp-per-row
// forward (ln_fwd_warp_kernel); register bound, prefetch and CTAs per SM per
// width measured on B200 (experiments/ln_fwd_sweep.py, bf16).
template <typename T, int VPT, int MINB, bool PF>
inline int launch_fwd_warp(const LnFwdArgs& a, int per_sm, cudaStream_t st, const char** why, cudaError_t* cerr) {
    const size_t smem = (size_t)2 * a.D * sizeof(typename Traits<T>::Acc);
    auto k = ln_fwd_warp_kernel<T, VPT, MINB, PF>;
    cudaError_t se = ensure_smem(reinterpret_cast<const void*>(k), smem);
    if (se != cudaSuccess) {
        *cerr = se;
        *why = "ln_fwd smem attribute";
        return 2;
    }
    int64_t grid = (int64_t)device_sm_count() * per_sm;
    const int64_t need = (a.N + 7) / 8;  // one row per warp at least
    if (grid > need) grid = need;
    k<<<(int)grid, 256, smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        *cerr = e;
        *why = "ln_fwd launch";
        return 2;
    }
    return 0;
}

template <typename T>
inline int try_fwd_warp(const LnFwdArgs& a, cudaStream_t st, const char** why, cudaError_t* cerr, bool* done) {
    constexpr int W = Traits<T>::W;
    *done = false;
    if (!a.aligned || a.D % W != 0) return 0;
    const int64_t per_lane = (a.D / W + 31) / 32;
    *done = true;
    switch (per_lane) {
        case 1: return launch_fwd_warp<T, 1, 4, true>(a, 4, st, why, cerr);
        case 2: return launch_fwd_warp<T, 2, 4, true>(a, 4, st, why, cerr);
        case 3: return launch_fwd_warp<T, 3, 4, true>(a, 4, st, why, cerr);
        case 4: return launch_fwd_warp<T, 4, 1, true>(a, 2, st, why, cerr);
        case 5: case 6: case 7: case 8: return launch_fwd_warp<T, 8, 2, true>(a, 2, st, why, cerr);
        case 9: case 10: case 11: case 12: case 13: case 14: case 15: case 16:
            return launch_fwd_warp<T, 16, 2, false>(a, 2, st, why, cerr);
        default: *done = false; return 0;
    }
}

template <typename T, int GW, int VPT>
struct FwdOp {
    static int run(const LnFwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
        using F = LnFwdCfg<T, GW, VPT>;
        LnFwdArgs a{};
        a.x = c.x;
        a.gamma = c.gamma;
        a.beta = c.beta;
        a.y = c.y;
        a.mean = c.mean;
        a.rstd = c.rstd;
        a.xhat = c.xhat;
        a.N = c.N;
        a.D = c.D;
        a.eps = c.eps;
        a.aligned = ((c.D * (int64_t)sizeof(T)) % 16 == 0) && ptr16(c.x) && (c.y == nullptr || ptr16(c.y)) &&
                    (c.xhat == nullptr || ptr16(c.xhat));
        const int sms = device_sm_count();
        bool done = false;
        const int wrc = try_fwd_warp<T>(a, st, why, cerr, &done);
        if (done) return wrc;
        if (a.aligned && c.D % Traits<T>::W == 0) {
            // TMA ring: G groups so that the CTA has ~16 consumer warps
            constexpr int GR = GW >= 16 ? 1 : (16 / GW > 15 ? 15 : 16 / GW);
            using RC = LnFwdRingCfg<T, GW, VPT, GR>;
            a.Dp = (int64_t)GW * 32 * VPT * Traits<T>::W;
            if (a.Dp < c.D) a.Dp = c.D;
            const size_t budget = (size_t)smem_optin_bytes() - 1024;
            int S = 0;
            for (int s2 = 32; s2 >= 2; --s2)  // as many stages as fit: bytes in flight set the speed
                if (RC::smem_bytes(s2, a.Dp, c.D) <= budget) {
                    S = s2;
                    break;
                }
            if (S > 0) {
                const size_t smem = RC::smem_bytes(S, a.Dp, c.D);
                auto k = ln_fwd_ring_kernel<T, GW, VPT, GR, (VPT >= 4)>;  // wide slices: gamma/beta from smem
                cudaError_t se = ensure_smem(reinterpret_cast<const void*>(k), smem);
                if (se != cudaSuccess) {
                    *cerr = se;
                    *why = "ln_fwd smem attribute";
                    return 2;
                }
                const int grid = (int)(c.N < sms ? c.N : sms);
                k<<<grid, RC::kThreads, smem, st>>>(a, S);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) {
                    *cerr = e;
                    *why = "ln_fwd launch";
                    return 2;
                }
                return 0;
            }
        }
        int64_t blocks = (c.N + F::G - 1) / F::G;
        const int64_t cap = (int64_t)sms * (2048 / F::kThreads);
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        a.Dp = (int64_t)GW * 32 * VPT * Traits<T>::W;
        if (a.Dp < c.D) a.Dp = c.D;
        const size_t smem = (size_t)2 * a.Dp * sizeof(typename Traits<T>::Acc);
        cudaError_t se = ensure_smem(reinterpret_cast<const void*>(ln_fwd_kernel<T, GW, VPT>), smem);
        if (se != cudaSuccess) {
            *cerr = se;
            *why = "ln_fwd smem attribute";
            return 2;
        }
        ln_fwd_kernel<T, GW, VPT><<<(int)blocks, F::kThreads, smem, st>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            *cerr = e;
            *why = "ln_fwd launch";
            return 2;
        }
        return 0;
    }
};

// GNSB_LN_NOFOLD=1 (A/B runs only): the D = 1024 / 2048 configurations
// without the end-of-kernel CTA fold (every row group leaves its own slot and
// stage 2 sums the G sub-slots).  Measured slower in the steady 8-layer step:
// 364 / 654 us against 343 / 621 us at D = 1024 / 2048 (the row pass itself
// got ~2 us slower, and stage 2 reads G x the slots), so the fold stays.
inline bool ln_fold() {
    static const bool v = [] {
        const char* e = getenv("GNSB_LN_NOFOLD");
        return !(e && e[0] == '1');
    }();
    return v;
}

inline bool ln_park() {
    static const bool v = [] {
        const char* e = getenv("GNSB_LN_PARK");
        return e && e[0] == '1';
    }();
    return v;
}

// Configuration table: number of 16-byte vectors per row -> LnBwdCfg.
template <typename T, template <typename> class Op, typename R, typename... A>
R dispatch_bwd(int64_t D, const char** why, R bad, A&&... args) {
    constexpr int W = Traits<T>::W;
    const int64_t nv = (D + W - 1) / W;
    // measured on B200 (experiments/ln_sweep.py): a dedicated producer warp
    // and xhat/h kept in registers win at every width
    if (nv <= 32) return Op<LnBwdCfg<T, 1, 1, 8, 2, true>>::call(args...);
    if (nv <= 64) return Op<LnBwdCfg<T, 2, 1, 8, 1, true>>::call(args...);
    if (nv <= 96) return Op<LnBwdCfg<T, 3, 1, 5, 2, true, -1, 1, true>>::call(args...);  // parked first example
    // D = 1024 / 2048: parking the first example's group partials in shared
    // memory measured slower even with the 4-stage ring's spare room (steady
    // 8-layer step: 345.6 / 654.4 us parked against 343.3 / 622.3 us at
    // D = 1024 / 2048); GNSB_LN_PARK=1 selects it for A/B runs
    if (nv <= 128) {
        if (!ln_fold()) return Op<LnBwdCfg<T, 4, 1, 4, 2, true, -1, 1, false, true>>::call(args...);
        if (ln_park()) return Op<LnBwdCfg<T, 4, 1, 4, 2, true, -1, 1, true>>::call(args...);
        return Op<LnBwdCfg<T, 4, 1, 4, 2, true>>::call(args...);
    }
    if (nv <= 256) {
        if (!ln_fold()) return Op<LnBwdCfg<T, 8, 1, 2, 2, true, -1, 1, false, true>>::call(args...);
        if (ln_park()) return Op<LnBwdCfg<T, 8, 1, 2, 2, true, -1, 1, true>>::call(args...);
        // (8-byte slot stores: the 16-byte ones spill this 17-warp configuration's
        // row loop and cost 9 % at D = 2048)
        return Op<LnBwdCfg<T, 8, 1, 2, 2, true, -1, 1, false, false, false>>::call(args...);
    }
    if (nv <= 512) return Op<LnBwdCfg<T, 8, 2, 1, 2, true, 1>>::call(args...);
    // 11 consumer warps x 3 vectors (3 % of the lanes idle at D=8192): 12 warps leave
    // ~168 registers per thread, no spills (16 x 2 forced 96 and spilled)
    if (nv <= 1024) return Op<LnBwdCfg<T, 11, 3, 1, 1, true, 1>>::call(args...);
    if (nv <= 2048) return Op<LnBwdCfg<T, 16, 4, 1, 1, false>>::call(args...);
    *why = "layers: trailing extent exceeds the kernel limit (2048 16-byte vectors per row)";
    return bad;
}

template <typename C>
struct BwdRunOp {
    static int call(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
        return BwdOp<C>::run(c, st, why, cerr);
    }
};
template <typename C>
struct BwdPlanOp {
    static int call(int64_t B, int64_t M, int64_t D, BwdPlan* p, const char** why) {
        return BwdOp<C>::plan(B, M, D, *p, why);
    }
};
template <typename C>
struct FwdRunOp {
    static int call(const LnFwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
        // widest rows: 16 warps x 2 vectors per row beats the backward's
        // 11 x 3 for the forward (experiments/ln_fwd_sweep.py, D = 8192)
        constexpr bool wide = C::kGW == 11 && C::kVPT == 3;
        return FwdOp<typename C::Row, wide ? 16 : C::kGW, wide ? 2 : C::kVPT>::run(c, st, why, cerr);
    }
};

}  // namespace

template <typename T>
int ln_bwd_run(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
    return dispatch_bwd<T, BwdRunOp>(c.D, why, 1, c, st, why, cerr);
}

template <typename C>
struct BwdRowsOp {
    static int call(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr, LnRedPlanInfo* info) {
        return BwdOp<C>::run_rows(c, st, why, cerr, info);
    }
};
template <typename C>
struct BwdInfoOp {
    static int call(int64_t B, int64_t M, int64_t D, LnRedPlanInfo* info, const char** why) {
        BwdPlan p;
        if (int rc = BwdOp<C>::plan(B, M, D, p, why)) return rc;
        BwdOp<C>::fill_info(p, info);
        return 0;
    }
};

template <typename T>
int ln_bwd_rows_run(const LnBwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
    LnRedPlanInfo info;
    return dispatch_bwd<T, BwdRowsOp>(c.D, why, 1, c, st, why, cerr, &info);
}

template <typename T>
int ln_bwd_plan_info(int64_t B, int64_t M, int64_t D, LnRedPlanInfo* out, const char** why) {
    return dispatch_bwd<T, BwdInfoOp>(D, why, 1, B, M, D, out, why);
}

template <typename T>
int ln_bwd_workspace(int64_t B, int64_t M, int64_t D, size_t* bytes, const char** why) {
    BwdPlan p;
    const int rc = dispatch_bwd<T, BwdPlanOp>(D, why, 1, B, M, D, &p, why);
    if (rc == 0) *bytes = p.total;
    return rc;
}

template <typename T>
int ln_bwd_geometry(int64_t B, int64_t M, int64_t D, int* grid, int* threads, int* stages) {
    BwdPlan p;
    const char* why = nullptr;
    const int rc = dispatch_bwd<T, BwdPlanOp>(D, &why, 1, B, M, D, &p, &why);
    if (rc == 0) {
        *grid = p.grid;
        *threads = p.threads;
        *stages = p.stages;
    }
    return rc;
}

template <typename T>
int ln_fwd_run(const LnFwdCall& c, cudaStream_t st, const char** why, cudaError_t* cerr) {
    return dispatch_bwd<T, FwdRunOp>(c.D, why, 1, c, st, why, cerr);
}

#define GNSB_INSTANTIATE_LN(T)                                                                          \
    template int ln_bwd_run<T>(const LnBwdCall&, cudaStream_t, const char**, cudaError_t*);             \
    template int ln_bwd_rows_run<T>(const LnBwdCall&, cudaStream_t, const char**, cudaError_t*);        \
    template int ln_bwd_plan_info<T>(int64_t, int64_t, int64_t, LnRedPlanInfo*, const char**);          \
    template int ln_bwd_workspace<T>(int64_t, int64_t, int64_t, size_t*, const char**);                 \
    template int ln_bwd_geometry<T>(int64_t, int64_t, int64_t, int*, int*, int*);                       \
    template int ln_fwd_run<T>(const LnFwdCall&, cudaStream_t, const char**, cudaError_t*);

}  // namespace gnsb

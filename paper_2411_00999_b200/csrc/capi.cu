#include <vector>
#include <utility>
#include <map>
#include <cstdio>
#include <cstdlib>
// capi.cu — the extern "C" boundary (include/gnsb.h): argument validation in
// the reference's wording, dtype dispatch, and the small device kernels that
// do not deserve their own file (squared norm, GNS accumulator).
#include <math_constants.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/gnsb.h"
#include "common.cuh"
#include "internal.h"

namespace {

thread_local std::string g_err;

gnsb_status fail(gnsb_status s, const std::string& msg) {
    g_err = msg;
    return s;
}
gnsb_status cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string("cuda: ") + where + ": " + cudaGetErrorString(e);
    return GNSB_ECUDA;
}

// GNSB_DEBUG=1: synchronize at every compute entry point and report a CUDA
// error left pending by whatever ran before (debugging aid, off by default).
static bool debug_mode() {
    static const bool on = [] {
        const char* v = std::getenv("GNSB_DEBUG");
        return v != nullptr && v[0] == '1';
    }();
    return on;
}

// GNSB_DEBUG=1: report a CUDA error an entry point leaves pending on success.
static gnsb_status debug_ok(const char* fn) {
    if (debug_mode()) {
        const cudaError_t s = cudaDeviceSynchronize();
        const cudaError_t p = cudaPeekAtLastError();
        if (s != cudaSuccess || p != cudaSuccess)
            std::fprintf(stderr, "gnsb: CUDA error pending on exit from %s: sync=%s last=%s\n", fn,
                         cudaGetErrorString(s), cudaGetErrorString(p));
    }
    return GNSB_OK;
}

gnsb_status need_device(const char* fn) {
    if (debug_mode()) {
        const cudaError_t s = cudaDeviceSynchronize();
        const cudaError_t p = cudaPeekAtLastError();
        if (s != cudaSuccess || p != cudaSuccess)
            std::fprintf(stderr, "gnsb: CUDA error pending on entry to %s: sync=%s last=%s\n", fn,
                         cudaGetErrorString(s), cudaGetErrorString(p));
    }
    static std::atomic<bool> seen{false};  // a device, once found, stays
    if (seen.load(std::memory_order_relaxed)) return GNSB_OK;
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        g_err = "cuda: no CUDA device available (the B200 path has no CPU fallback)";
        return GNSB_ECUDA;
    }
    seen.store(true, std::memory_order_relaxed);
    return GNSB_OK;
}

size_t stat_size(gnsb_dtype dt) { return dt == GNSB_F64 ? 8 : 4; }

// splitmix64 + mix_seed (proj/include/gnstk/rng.hpp:19-24, 42-45)
uint64_t sm64(uint64_t* st) {
    uint64_t z = (*st += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t mix_seed(uint64_t seed, uint64_t tag) {
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ull * (tag + 1));
    return sm64(&s);
}
gnsb::SynthSeeds seeds(uint64_t stream0) {
    gnsb::SynthSeeds s;
    for (int k = 0; k < 8; ++k) s.s[k] = mix_seed(2411u, stream0 + (uint64_t)k);
    return s;
}

// layers.cpp:39-42
double corrected_mean_sqnorm(double sum_sq, int64_t batch) {
    const double b = (double)batch;
    return sum_sq / b * (b * b);
}

}  // namespace

namespace gnsb {

cudaError_t ensure_smem_attr(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set_for;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto& cur = set_for[{kernel, dev}];
    if (cur >= bytes) return cudaSuccess;
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
    if (e != cudaSuccess) return e;
    if ((size_t)fa.maxDynamicSharedSizeBytes >= bytes) {
        cur = (size_t)fa.maxDynamicSharedSizeBytes;
        return cudaSuccess;
    }
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

void set_error(const std::string& msg) { g_err = msg; }

int device_sm_count() {
    static std::mutex mu;
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && cache[dev]) return cache[dev];
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 1;
    if (dev < 64) cache[dev] = v;
    return v;
}

// ------------------------------------------------------- squared norm ----
template <typename V>
__global__ void __launch_bounds__(1024) sqnorm_kernel(const V* v, int64_t n, double* out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = (double)v[i];
        acc += x * x;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) *out = t;
    }
}

// ------------------------------------------------------- GNS accumulator --
struct GnsStepArgs {
    const double* sums;
    int n;
    int64_t B;
    double alpha;
    gnsb_ema_state* state;
    double* out_groups;
    double* out_layers;
    int8_t types[512];
};

__device__ double d_corrected(double sum_sq, int64_t batch) {
    const double b = (double)batch;
    return sum_sq / b * (b * b);
}

// Single thread: O(#layers) scalar work in the reference's operation order
// (trainer.cpp:363-415, gns.cpp:31-89).
__global__ void gns_step_kernel(const __grid_constant__ GnsStepArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double bb = (double)a.B, bs = 1.0;
    for (int grp = 0; grp < 4; ++grp) {
        const int filter = grp - 1;  // -1 total, 0 embedding, 1 linear, 2 layernorm
        bool any = false;
        double big = 0.0, small = 0.0;
        for (int l = 0; l < a.n; ++l) {
            if (filter >= 0 && a.types[l] != filter) continue;
            const double* s = a.sums + 4 * l;
            double lb = 0.0, ls = 0.0;
            lb += s[3];
            lb += s[2];
            ls += d_corrected(s[1], a.B);
            ls += d_corrected(s[0], a.B);
            if (grp == 0 && a.out_layers) {
                a.out_layers[2 * l + 0] = (bb * lb - bs * ls) / (bb - bs);
                a.out_layers[2 * l + 1] = (ls - lb) / (1.0 / bs - 1.0 / bb);
            }
            big += lb;
            small += ls;
            any = true;
        }
        double* o = a.out_groups + 4 * grp;
        if (!any) {  // empty selection (the reference's aggregate throws): no estimate, not defined
            o[0] = o[1] = o[2] = CUDART_NAN;
            o[3] = 0.0;
            continue;
        }
        const double g2 = (bb * big - bs * small) / (bb - bs);
        const double s = (small - big) / (1.0 / bs - 1.0 / bb);
        gnsb_ema_state* eg = a.state + 2 * grp;
        gnsb_ema_state* es = eg + 1;
        eg->alpha = a.alpha;
        es->alpha = a.alpha;
        eg->value = eg->count == 0 ? g2 : (1.0 - a.alpha) * eg->value + a.alpha * g2;
        es->value = es->count == 0 ? s : (1.0 - a.alpha) * es->value + a.alpha * s;
        ++eg->count;
        ++es->count;
        o[0] = g2;
        o[1] = s;
        const bool def = fabs(eg->value) >= 1e-12;
        o[2] = def ? es->value / eg->value : 0.0;
        o[3] = def ? 1.0 : 0.0;
    }
}

}  // namespace gnsb

extern "C" {

const char* gnsb_version(void) { return "gnsb 0.1 (sm_100a)"; }
const char* gnsb_last_error(void) { return g_err.c_str(); }

gnsb_status gnsb_ln_fwd(const void* x, const void* gamma, const void* beta, void* y, void* mean, void* rstd, void* xhat,
                        int64_t rows, int64_t D, double eps, gnsb_dtype dt, void* stream) {
    if (!(eps > 0.0)) return fail(GNSB_EINVAL, "layers: epsilon must be positive");          // layers.cpp:192
    if (D < 2) return fail(GNSB_EINVAL, "layers: layernorm needs trailing extent >= 2");     // layers.cpp:194
    if (rows < 0) return fail(GNSB_EINVAL, "layers: negative row count");
    if (gnsb_status s = need_device("gnsb_ln_fwd")) return s;
    if (rows == 0) return debug_ok("gnsb_ln_fwd");
    if (!x || !gamma || !beta) return fail(GNSB_EINVAL, "layers: null input pointer");
    gnsb::LnFwdCall c{x, gamma, beta, y, mean, rstd, xhat, rows, D, eps};
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    int rc = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (dt) {
        case GNSB_F32: rc = gnsb::ln_fwd_run<float>(c, st, &why, &ce); break;
        case GNSB_BF16: rc = gnsb::ln_fwd_run<__nv_bfloat16>(c, st, &why, &ce); break;
        case GNSB_F64: rc = gnsb::ln_fwd_run<double>(c, st, &why, &ce); break;
        default: return fail(GNSB_EINVAL, "layers: unknown dtype");
    }
    if (rc == 1) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
    if (rc == 2) return cuda_fail(ce, why ? why : "ln_fwd launch");
    return debug_ok("gnsb_ln_fwd");
}

gnsb_status gnsb_ln_bwd_workspace_size(int64_t B, int64_t M, int64_t D, gnsb_dtype dt, size_t* bytes) {
    if (!bytes) return fail(GNSB_EINVAL, "layers: null output pointer");
    if (B < 0 || M < 0 || D < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (gnsb_status s = need_device("gnsb_ln_bwd_workspace_size")) return s;
    const char* why = nullptr;
    int rc = 1;
    switch (dt) {
        case GNSB_F32: rc = gnsb::ln_bwd_workspace<float>(B, M, D, bytes, &why); break;
        case GNSB_BF16: rc = gnsb::ln_bwd_workspace<__nv_bfloat16>(B, M, D, bytes, &why); break;
        case GNSB_F64:
            rc = gnsb::ln_bwd_workspace<double>(B, M, D, bytes, &why);
            // + the reference-order scratch of the fp64 path (ln_ref.cu)
            if (rc == 0) *bytes = (*bytes + 255) / 256 * 256 + gnsb::ln_ref_workspace(B, D);
            break;
        default: return fail(GNSB_EINVAL, "layers: unknown dtype");
    }
    if (rc) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
    return debug_ok("gnsb_ln_bwd_workspace_size");
}

gnsb_status gnsb_ln_bwd_geometry(int64_t B, int64_t M, int64_t D, gnsb_dtype dt, int32_t* grid, int32_t* threads,
                                 int32_t* stages) {
    if (gnsb_status s = need_device("gnsb_ln_bwd_geometry")) return s;
    int g = 0, t = 0, st = 0, rc = 1;
    switch (dt) {
        case GNSB_F32: rc = gnsb::ln_bwd_geometry<float>(B, M, D, &g, &t, &st); break;
        case GNSB_BF16: rc = gnsb::ln_bwd_geometry<__nv_bfloat16>(B, M, D, &g, &t, &st); break;
        case GNSB_F64: rc = gnsb::ln_bwd_geometry<double>(B, M, D, &g, &t, &st); break;
        default: return fail(GNSB_EINVAL, "layers: unknown dtype");
    }
    if (rc) return fail(GNSB_EINVAL, "layers: unsupported shape");
    if (grid) *grid = g;
    if (threads) *threads = t;
    if (stages) *stages = st;
    return debug_ok("gnsb_ln_bwd_geometry");
}

gnsb_status gnsb_ln_bwd(const void* x, const void* mean, const void* rstd, const void* dy, const void* gamma, void* dx,
                        void* dgamma, void* dbeta, double* raw_g, double* raw_b, double* sums, int32_t with_norms,
                        int64_t B, int64_t M, int64_t D, gnsb_dtype dt, void* ws, size_t ws_bytes, void* stream) {
    if (B == 0) return fail(GNSB_EINVAL, "layers: empty batch");  // layers.cpp:239
    if (B < 0 || M < 0) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (D < 1) return fail(GNSB_EINVAL, "layers: gradient trailing extent does not match gamma");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_ln_bwd")) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (M == 0) {  // no rows: every gradient and norm is zero (layers.cpp:248-275 with an empty loop)
        cudaError_t e = cudaSuccess;
        if (dgamma) e = cudaMemsetAsync(dgamma, 0, (size_t)D * stat_size(dt), st);
        if (e == cudaSuccess && dbeta) e = cudaMemsetAsync(dbeta, 0, (size_t)D * stat_size(dt), st);
        if (with_norms) {
            if (e == cudaSuccess && raw_g) e = cudaMemsetAsync(raw_g, 0, (size_t)B * 8, st);
            if (e == cudaSuccess && raw_b) e = cudaMemsetAsync(raw_b, 0, (size_t)B * 8, st);
            if (e == cudaSuccess && sums) e = cudaMemsetAsync(sums, 0, 4 * 8, st);
        }
        return e == cudaSuccess ? debug_ok("gnsb_ln_bwd") : cuda_fail(e, "memset");
    }
    if (!x || !rstd || !dy || !gamma || !dgamma || !dbeta || !ws)
        return fail(GNSB_EINVAL, "layers: null input pointer");
    // The plain LayerNorm backward has no per-example structure: the same
    // kernels over ONE example of B*M rows (no example-boundary flushes, one
    // partial slot per CTA).  This is the overhead baseline of the fused call.
    const int64_t Bk = with_norms ? B : 1, Mk = with_norms ? M : B * M;
    gnsb::LnBwdCall c{x, mean, rstd, dy, gamma, dx, dgamma, dbeta, raw_g, raw_b, sums, with_norms ? 1 : 0,
                      Bk, Mk, D, ws, ws_bytes};
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    int rc = 1;
    switch (dt) {
        case GNSB_F32: rc = gnsb::ln_bwd_run<float>(c, st, &why, &ce); break;
        case GNSB_BF16: rc = gnsb::ln_bwd_run<__nv_bfloat16>(c, st, &why, &ce); break;
        case GNSB_F64:
            if (!with_norms) {
                rc = gnsb::ln_bwd_run<double>(c, st, &why, &ce);
                break;
            }
            {
                // fp64 rows (the C++ drop-in): dx from the row pass; the
                // per-example parameter gradients, norms and their sums in the
                // reference's exact order, so a batched call and B = 1 calls
                // agree bit for bit (ln_ref.cu)
                size_t base = 0;
                if (gnsb::ln_bwd_workspace<double>(B, M, D, &base, &why)) {
                    rc = 1;
                    break;
                }
                base = (base + 255) / 256 * 256;
                if (ws_bytes < base + gnsb::ln_ref_workspace(B, D)) {
                    rc = 1;
                    why = "layers: workspace too small (query gnsb_ln_bwd_workspace_size)";
                    break;
                }
                rc = gnsb::ln_bwd_rows_run<double>(c, st, &why, &ce);
                if (rc == 0) {
                    ce = gnsb::launch_ln_ref_params(
                        static_cast<const double*>(x), static_cast<const double*>(mean),
                        static_cast<const double*>(rstd), static_cast<const double*>(dy), B, M, D,
                        static_cast<double*>(dgamma), static_cast<double*>(dbeta), raw_g, raw_b, sums,
                        static_cast<unsigned char*>(ws) + base, st);
                    if (ce != cudaSuccess) rc = 2;
                }
            }
            break;
        default: break;
    }
    if (rc == 1) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
    if (rc == 2) return cuda_fail(ce, why ? why : "ln_bwd launch");
    return debug_ok("gnsb_ln_bwd");
}

gnsb_status gnsb_ln_bwd_rows(const void* x, const void* mean, const void* rstd, const void* dy, const void* gamma,
                             void* dx, int64_t B, int64_t M, int64_t D, gnsb_dtype dt, void* ws, size_t ws_bytes,
                             void* stream) {
    if (B == 0) return fail(GNSB_EINVAL, "layers: empty batch");
    if (B < 0 || M < 0) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (D < 1) return fail(GNSB_EINVAL, "layers: gradient trailing extent does not match gamma");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_ln_bwd_rows")) return s;
    if (M == 0) return debug_ok("gnsb_ln_bwd_rows");  // nothing to stream; the reduce writes zeros
    if (!x || !rstd || !dy || !gamma || !ws) return fail(GNSB_EINVAL, "layers: null input pointer");
    gnsb::LnBwdCall c{x, mean, rstd, dy, gamma, dx, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                      B, M, D, ws, ws_bytes};
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    int rc = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (dt) {
        case GNSB_F32: rc = gnsb::ln_bwd_rows_run<float>(c, st, &why, &ce); break;
        case GNSB_BF16: rc = gnsb::ln_bwd_rows_run<__nv_bfloat16>(c, st, &why, &ce); break;
        case GNSB_F64: rc = gnsb::ln_bwd_rows_run<double>(c, st, &why, &ce); break;
        default: break;
    }
    if (rc == 1) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
    if (rc == 2) return cuda_fail(ce, why ? why : "ln_bwd rows launch");
    return debug_ok("gnsb_ln_bwd_rows");
}

gnsb_status gnsb_ln_bwd_reduce(const gnsb_ln_bwd_pending* items, int32_t n, int32_t with_norms, void* stream) {
    if (n < 0 || (n > 0 && !items)) return fail(GNSB_EINVAL, "layers: invalid pending list");
    if (n > 64) return fail(GNSB_EINVAL, "layers: too many pending LayerNorms in one reduce (max 64)");
    if (gnsb_status s = need_device("gnsb_ln_bwd_reduce")) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<gnsb::LnRedItem> list;
    int acc_f64 = -1;
    for (int32_t i = 0; i < n; ++i) {
        const gnsb_ln_bwd_pending& p = items[i];
        const gnsb_dtype dt = static_cast<gnsb_dtype>(p.dt);
        if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
        if (p.B <= 0 || p.M < 0 || p.D < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
        if (!p.dgamma || !p.dbeta || !p.ws) return fail(GNSB_EINVAL, "layers: null output pointer");
        const int f64 = dt == GNSB_F64 ? 1 : 0;
        if (acc_f64 >= 0 && f64 != acc_f64)
            return fail(GNSB_EINVAL, "layers: pending LayerNorms mix fp64 and fp32 statistics");
        acc_f64 = f64;
        if (p.M == 0) {  // no rows: zeros (layers.cpp:248-275 with an empty loop)
            cudaError_t e = cudaMemsetAsync(p.dgamma, 0, (size_t)p.D * stat_size(dt), st);
            if (e == cudaSuccess) e = cudaMemsetAsync(p.dbeta, 0, (size_t)p.D * stat_size(dt), st);
            if (with_norms) {
                if (e == cudaSuccess && p.raw_sq_gamma) e = cudaMemsetAsync(p.raw_sq_gamma, 0, (size_t)p.B * 8, st);
                if (e == cudaSuccess && p.raw_sq_beta) e = cudaMemsetAsync(p.raw_sq_beta, 0, (size_t)p.B * 8, st);
                if (e == cudaSuccess && p.sums) e = cudaMemsetAsync(p.sums, 0, 4 * 8, st);
            }
            if (e != cudaSuccess) return cuda_fail(e, "memset");
            continue;
        }
        gnsb::LnRedItem it{};
        const char* why = nullptr;
        int rc = 1;
        switch (dt) {
            case GNSB_F32: rc = gnsb::ln_bwd_plan_info<float>(p.B, p.M, p.D, &it.info, &why); break;
            case GNSB_BF16: rc = gnsb::ln_bwd_plan_info<__nv_bfloat16>(p.B, p.M, p.D, &it.info, &why); break;
            case GNSB_F64: rc = gnsb::ln_bwd_plan_info<double>(p.B, p.M, p.D, &it.info, &why); break;
            default: break;
        }
        if (rc) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
        if (p.ws_bytes < it.info.total)
            return fail(GNSB_EINVAL, "layers: workspace too small (query gnsb_ln_bwd_workspace_size)");
        it.B = p.B;
        it.M = p.M;
        it.D = p.D;
        it.ws = p.ws;
        it.dgamma = p.dgamma;
        it.dbeta = p.dbeta;
        it.raw_g = with_norms ? p.raw_sq_gamma : nullptr;
        it.raw_b = with_norms ? p.raw_sq_beta : nullptr;
        it.sums = with_norms ? p.sums : nullptr;
        list.push_back(it);
    }
    if (list.empty()) return debug_ok("gnsb_ln_bwd_reduce");
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    const int rc = gnsb::ln_bwd_reduce_run(acc_f64 == 1, with_norms ? 1 : 0, list.data(), (int)list.size(), st,
                                           nullptr, &why, &ce);
    if (rc == 1) return fail(GNSB_EINVAL, why ? why : "layers: invalid argument");
    if (rc == 2) return cuda_fail(ce, why ? why : "ln_bwd reduce launch");
    return debug_ok("gnsb_ln_bwd_reduce");
}

// ---------------------------------------------------------------- linear --
static bool use_tc_wgrad(gnsb_dtype dt, int64_t B, int64_t T, int64_t K, int64_t L) {
    return dt == GNSB_BF16 && gnsb::wgrad_shape_ok(B, T, K, L);
}
static bool use_tc_gram(gnsb_dtype dt, int64_t B, int64_t T, int64_t K, int64_t L) {
    return dt == GNSB_BF16 && gnsb::gram_shape_ok(B, T, K, L);
}

gnsb_status gnsb_linear_pe_workspace_size(int64_t B, int64_t T, int64_t K, int64_t L, gnsb_dtype dt, size_t* bytes) {
    if (!bytes || B < 0 || T < 0 || K < 1 || L < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    size_t n = dt == GNSB_F64 ? gnsb::generic_workspace_f64(B, T, K, L) : gnsb::generic_workspace(B, T, K, L);
    if (K == 1 && dt != GNSB_F64) {  // the bias call's workspace: room for the streaming bias kernel
        const size_t m = gnsb::bias_fast_workspace(B, T, L);
        n = n > m ? n : m;
    }
    if (use_tc_wgrad(dt, B, T, K, L)) {
        const size_t m = gnsb::wgrad_workspace(B, K, L);
        n = n > m ? n : m;
    }
    if (use_tc_gram(dt, B, T, K, L)) {
        const size_t m = gnsb::gram_workspace(B, T);
        n = n > m ? n : m;
    }
    if (use_tc_wgrad(dt, 1, B * T, K, L)) {  // the plain dW pass of the short-sequence dispatch
        const size_t m = gnsb::wgrad_workspace(1, K, L);
        n = n > m ? n : m;
    }
    *bytes = n;
    return debug_ok("gnsb_linear_pe_workspace_size");
}

gnsb_status gnsb_linear_pe_norms(const void* x, const void* g, void* dW, double* raw_w, double* sums, int64_t B,
                                 int64_t T, int64_t K, int64_t L, int32_t form, gnsb_dtype dt, void* ws,
                                 size_t ws_bytes, void* stream) {
    if (B == 0) return fail(GNSB_EINVAL, "layers: empty batch");  // layers.cpp:89
    if (B < 0 || T < 0 || K < 1 || L < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (form < 0 || form > 2) return fail(GNSB_EINVAL, "layers: form must be 0 (auto), 1 (weight-grad) or 2 (gram)");
    if (form == 2 && dW) return fail(GNSB_EINVAL, "layers: the gram form computes norms only (dW must be NULL)");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_linear_pe_norms")) return s;
    size_t need = 0;
    gnsb_linear_pe_workspace_size(B, T, K, L, dt, &need);
    if (!ws || ws_bytes < need) return fail(GNSB_EINVAL, "layers: workspace too small (query gnsb_linear_pe_workspace_size)");
    if ((T > 0) && (!x || !g)) return fail(GNSB_EINVAL, "layers: null input pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    // Auto with dW on the tensor cores: for short sequences the weight-gradient
    // form is bound by its per-(tile, example) epilogue, not the MMAs, and the
    // Gram form for the norms plus ONE plain dW pass over all B*T tokens
    // (the weight-gradient kernel on a single "example") is faster
    // (experiments/form_sweep.py at K = L = 4096, B*T = 32768: T = 128 /
    // 256: 0.89 / 0.81 ms against 1.79 / 1.18 ms; from T = 512 the
    // weight-gradient form wins, 0.84 against 0.84 + ...).
    if (form == 0 && dW != nullptr && T < 384 && T * (K + L) < 2 * K * L && use_tc_gram(dt, B, T, K, L) &&
        use_tc_wgrad(dt, 1, B * T, K, L)) {
        e = gnsb::launch_wgrad_norms(x, g, static_cast<float*>(dW), nullptr, sums, 1, B * T, K, L, ws, st);
        // (sums[2] = ||dW||^2 from that pass; sums[0] and raw_w from the Gram form)
        if (e == cudaSuccess) e = gnsb::launch_gram_norms(x, g, raw_w, sums, B, T, K, L, ws, st);
        return e == cudaSuccess ? debug_ok("gnsb_linear_pe_norms") : cuda_fail(e, "linear_pe_norms launch");
    }
    if (form == 0) form = (dW != nullptr || T * (K + L) >= 2 * K * L) ? 1 : 2;
    if (form == 1 && use_tc_wgrad(dt, B, T, K, L))
        e = gnsb::launch_wgrad_norms(x, g, static_cast<float*>(dW), raw_w, sums, B, T, K, L, ws, st);
    else if (form == 2 && use_tc_gram(dt, B, T, K, L))
        e = gnsb::launch_gram_norms(x, g, raw_w, sums, B, T, K, L, ws, st);
    else
        e = gnsb::launch_linear_generic((int)dt, form == 1 ? 0 : 2, x, g, dW, dt == GNSB_F64, raw_w, sums, 0, B, T, K,
                                        L, ws, st);
    return e == cudaSuccess ? debug_ok("gnsb_linear_pe_norms") : cuda_fail(e, "linear_pe_norms launch");
}

gnsb_status gnsb_linear_bias_pe(const void* g, void* dbias, double* raw_b, double* sums, int64_t B, int64_t T,
                                int64_t L, gnsb_dtype dt, void* ws, size_t ws_bytes, void* stream) {
    if (B == 0) return fail(GNSB_EINVAL, "layers: empty batch");
    if (B < 0 || T < 0 || L < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_linear_bias_pe")) return s;
    const size_t need = dt == GNSB_F64 ? gnsb::generic_workspace_f64(B, T, 1, L) : gnsb::generic_workspace(B, T, 1, L);
    if (!ws || ws_bytes < need)
        return fail(GNSB_EINVAL, "layers: workspace too small (query gnsb_linear_pe_workspace_size)");
    if (T > 0 && gnsb::bias_fast_ok((int)dt, L, g, dbias) && ws_bytes >= gnsb::bias_fast_workspace(B, T, L)) {
        const cudaError_t e = gnsb::launch_bias_fast((int)dt, g, dbias, raw_b, sums, B, T, L, ws,
                                                     static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? debug_ok("gnsb_linear_bias_pe") : cuda_fail(e, "linear_bias_pe launch");
    }
    const cudaError_t e = gnsb::launch_linear_generic((int)dt, 1, nullptr, g, dbias, dt == GNSB_F64, raw_b, sums, 1, B,
                                                      T, 1, L, ws, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok("gnsb_linear_bias_pe") : cuda_fail(e, "linear_bias_pe launch");
}

gnsb_status gnsb_embedding_pe_workspace_size(int64_t B, int64_t T, int64_t V, int64_t D, gnsb_dtype dt,
                                             size_t* bytes) {
    if (!bytes || B < 0 || T < 0 || V < 1 || D < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_embedding_pe_workspace_size")) return s;
    *bytes = gnsb::embedding_workspace(B, T, V, D, (int)dt);
    return debug_ok("gnsb_embedding_pe_workspace_size");
}

gnsb_status gnsb_embedding_pe(const int32_t* ids, const void* g, void* dW, double* raw_w, double* sums, int64_t B,
                              int64_t T, int64_t V, int64_t D, gnsb_dtype dt, void* ws, size_t ws_bytes,
                              int32_t* bad_ids, void* stream) {
    if (B == 0) return fail(GNSB_EINVAL, "layers: empty batch");  // layers.cpp:322
    if (B < 0 || T < 0 || V < 1 || D < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (T > 0 && !gnsb::embedding_shape_ok(T))
        return fail(GNSB_EINVAL, "layers: sequence too long for the embedding kernel (T <= 16384)");
    if (gnsb_status s = need_device("gnsb_embedding_pe")) return s;
    if (!dW || !ws || (T > 0 && (!ids || !g))) return fail(GNSB_EINVAL, "layers: null pointer");
    size_t need = 0;
    gnsb_embedding_pe_workspace_size(B, T, V, D, dt, &need);
    if (ws_bytes < need) return fail(GNSB_EINVAL, "layers: workspace too small (query gnsb_embedding_pe_workspace_size)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (T == 0) {  // no tokens: zero table gradient and norms
        e = cudaMemsetAsync(dW, 0, (size_t)V * D * stat_size(dt), st);
        if (e == cudaSuccess && raw_w) e = cudaMemsetAsync(raw_w, 0, (size_t)B * 8, st);
        if (e == cudaSuccess && sums) e = cudaMemsetAsync(sums, 0, 4 * 8, st);
        if (e == cudaSuccess && bad_ids) e = cudaMemsetAsync(bad_ids, 0, 4, st);
    } else {
        e = gnsb::launch_embedding_pe((int)dt, ids, g, dW, raw_w, sums, B, T, V, D, ws, bad_ids, st);
    }
    return e == cudaSuccess ? debug_ok("gnsb_embedding_pe") : cuda_fail(e, "embedding_pe launch");
}

static bool gemm_dtypes_ok(gnsb_dtype dt, gnsb_dtype w_dt) {
    return (dt == GNSB_F64 && w_dt == GNSB_F64) || (dt == GNSB_F32 && w_dt == GNSB_F32) ||
           (dt == GNSB_BF16 && (w_dt == GNSB_F32 || w_dt == GNSB_BF16));
}

gnsb_status gnsb_linear_gemm_workspace_size(int64_t K, int64_t L, gnsb_dtype dt, gnsb_dtype w_dt, size_t* bytes) {
    if (!bytes || K < 1 || L < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (!gemm_dtypes_ok(dt, w_dt)) return fail(GNSB_EINVAL, "layers: unsupported row/weight dtype pair");
    *bytes = gnsb::gemm_workspace((int)dt, (int)w_dt, K, L);
    return debug_ok("gnsb_linear_gemm_workspace_size");
}

static gnsb_status linear_gemm(int kind, int epi, const char* fn, const void* in, const void* W, const void* bias,
                               const void* aux, void* out, int64_t rows, int64_t K, int64_t L, gnsb_dtype dt,
                               gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream) {
    if (epi < 0 || epi > 3 || (kind == 1 && (epi == 1 || epi == 2)) || (kind == 0 && epi == 3))
        return fail(GNSB_EINVAL, "layers: unsupported GEMM epilogue for this product");
    if ((epi == 2 || epi == 3) && rows > 0 && !aux) return fail(GNSB_EINVAL, "layers: the epilogue needs aux");
    if (rows < 0 || K < 1 || L < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (!gemm_dtypes_ok(dt, w_dt)) return fail(GNSB_EINVAL, "layers: unsupported row/weight dtype pair");
    if (gnsb_status s = need_device(fn)) return s;
    if (rows > 0 && (!in || !W || !out)) return fail(GNSB_EINVAL, "layers: null pointer");
    if (ws_bytes < gnsb::gemm_workspace((int)dt, (int)w_dt, K, L) || (ws_bytes > 0 && !ws))
        return fail(GNSB_EINVAL, "layers: workspace too small (query gnsb_linear_gemm_workspace_size)");
    const cudaError_t e = gnsb::launch_linear_gemm(kind, epi, (int)dt, (int)w_dt, in, W, bias, aux, out, rows, K, L,
                                                   ws, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok(fn) : cuda_fail(e, "linear gemm launch");
}

gnsb_status gnsb_linear_fwd(const void* x, const void* W, const void* bias, void* y, int64_t rows, int64_t K, int64_t L,
                            gnsb_dtype dt, gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream) {
    return linear_gemm(0, 0, "gnsb_linear_fwd", x, W, bias, nullptr, y, rows, K, L, dt, w_dt, ws, ws_bytes, stream);
}

gnsb_status gnsb_linear_gemm(int32_t kind, int32_t epilogue, const void* a, const void* W, const void* bias,
                             const void* aux, void* out, int64_t rows, int64_t K, int64_t L, gnsb_dtype dt,
                             gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream) {
    if (kind != 0 && kind != 1) return fail(GNSB_EINVAL, "layers: kind must be 0 (forward) or 1 (input grad)");
    return linear_gemm(kind, epilogue, "gnsb_linear_gemm", a, W, kind == 0 ? bias : nullptr, aux, out, rows, K, L, dt,
                       w_dt, ws, ws_bytes, stream);
}

gnsb_status gnsb_xent(const void* logits, const int32_t* targets, void* dlogits, double* loss_rows, int64_t rows,
                      int64_t V, double upstream_scale, gnsb_dtype dt, int32_t* bad_targets, void* stream) {
    if (rows < 0 || V < 1) return fail(GNSB_EINVAL, "model: invalid extents");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "model: unknown dtype");
    if (gnsb_status s = need_device("gnsb_xent")) return s;
    if (rows > 0 && (!logits || !targets || !loss_rows)) return fail(GNSB_EINVAL, "model: null pointer");
    const cudaError_t e = gnsb::launch_xent((int)dt, logits, targets, dlogits, loss_rows, rows, V, upstream_scale,
                                            bad_targets, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok("gnsb_xent") : cuda_fail(e, "xent launch");
}

gnsb_status gnsb_linear_dx(const void* g, const void* W, void* dx, int64_t rows, int64_t K, int64_t L, gnsb_dtype dt,
                           gnsb_dtype w_dt, void* ws, size_t ws_bytes, void* stream) {
    return linear_gemm(1, 0, "gnsb_linear_dx", g, W, nullptr, nullptr, dx, rows, K, L, dt, w_dt, ws, ws_bytes, stream);
}

gnsb_status gnsb_embedding_fwd(const int32_t* ids, const void* W, void* out, int64_t n, int64_t V, int64_t D,
                               gnsb_dtype dt, int32_t* bad_ids, void* stream) {
    if (n < 0 || V < 1 || D < 1) return fail(GNSB_EINVAL, "layers: invalid extents");
    if (dt != GNSB_F32 && dt != GNSB_BF16 && dt != GNSB_F64) return fail(GNSB_EINVAL, "layers: unknown dtype");
    if (gnsb_status s = need_device("gnsb_embedding_fwd")) return s;
    if (n > 0 && (!ids || !W || !out)) return fail(GNSB_EINVAL, "layers: null pointer");
    const cudaError_t e =
        gnsb::launch_embedding_fwd((int)dt, ids, W, out, n, V, D, bad_ids, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok("gnsb_embedding_fwd") : cuda_fail(e, "embedding_fwd launch");
}

gnsb_status gnsb_sqnorm(const void* v, int64_t n, gnsb_dtype dt, double* out, void* stream) {
    if (n < 0 || !out) return fail(GNSB_EINVAL, "gns: invalid sqnorm arguments");
    if (gnsb_status s = need_device("gnsb_sqnorm")) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dt == GNSB_F64)
        gnsb::sqnorm_kernel<double><<<1, 1024, 0, st>>>(static_cast<const double*>(v), n, out);
    else if (dt == GNSB_F32)
        gnsb::sqnorm_kernel<float><<<1, 1024, 0, st>>>(static_cast<const float*>(v), n, out);
    else
        return fail(GNSB_EINVAL, "gns: sqnorm expects fp32 or fp64 data");
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? debug_ok("gnsb_sqnorm") : cuda_fail(e, "sqnorm launch");
}

// ---------------------------------------------------------------- GNS ----
gnsb_status gnsb_estimate_g2(const gnsb_grad_stats* st, double* out) {
    if (st->b_small < 1) return fail(GNSB_EINVAL, "gns: b_small must be >= 1");
    if (st->b_big <= st->b_small) return fail(GNSB_EINVAL, "gns: b_big must exceed b_small");
    if (st->n_small < 1) return fail(GNSB_EINVAL, "gns: n_small must be >= 1");
    const double bb = (double)st->b_big, bs = (double)st->b_small;
    *out = (bb * st->g_big_sqnorm - bs * st->g_small_sqnorm_mean) / (bb - bs);
    return debug_ok("gnsb_estimate_g2");
}

gnsb_status gnsb_estimate_s(const gnsb_grad_stats* st, double* out) {
    if (st->b_small < 1) return fail(GNSB_EINVAL, "gns: b_small must be >= 1");
    if (st->b_big <= st->b_small) return fail(GNSB_EINVAL, "gns: b_big must exceed b_small");
    if (st->n_small < 1) return fail(GNSB_EINVAL, "gns: n_small must be >= 1");
    const double bb = (double)st->b_big, bs = (double)st->b_small;
    *out = (st->g_small_sqnorm_mean - st->g_big_sqnorm) / (1.0 / bs - 1.0 / bb);
    return debug_ok("gnsb_estimate_s");
}

void gnsb_make_gns_estimate(double g2, double s, gnsb_gns_estimate* out) {
    out->g2 = g2;
    out->s = s;
    out->b_simple = 0.0;
    out->b_simple_defined = 0;
    if (std::fabs(g2) >= 1e-12) {  // kGnsRatioGuard, gns.hpp:34
        out->b_simple = s / g2;
        out->b_simple_defined = 1;
    }
}

gnsb_status gnsb_ema_update(gnsb_ema_state* st, double x) {
    if (!(st->alpha > 0.0) || st->alpha > 1.0) return fail(GNSB_EINVAL, "gns: ema alpha must be in (0, 1]");
    if (st->count == 0)
        st->value = x;
    else
        st->value = (1.0 - st->alpha) * st->value + st->alpha * x;
    ++st->count;
    return debug_ok("gnsb_ema_update");
}

gnsb_status gnsb_smoothed_gns(const gnsb_ema_state* g2, const gnsb_ema_state* s, gnsb_gns_estimate* out) {
    if (g2->count < 1 || s->count < 1)
        return fail(GNSB_EINVAL, "gns: smoothed_gns needs at least one sample in each state");
    gnsb_make_gns_estimate(g2->value, s->value, out);
    return debug_ok("gnsb_smoothed_gns");
}

gnsb_status gnsb_aggregate(const gnsb_grad_stats* stats, const int32_t* types, int32_t n, int32_t group,
                           gnsb_grad_stats* out) {
    bool first = true;
    for (int32_t i = 0; i < n; ++i) {
        if (group >= 0 && types[i] != group) continue;
        if (first) {
            *out = stats[i];
            out->g_big_sqnorm = 0.0;
            out->g_small_sqnorm_mean = 0.0;
            first = false;
        } else if (stats[i].b_big != out->b_big || stats[i].b_small != out->b_small ||
                   stats[i].n_small != out->n_small) {
            return fail(GNSB_EINVAL, "gns: aggregate requires matching batch sizes across layers");
        }
        out->g_big_sqnorm += stats[i].g_big_sqnorm;
        out->g_small_sqnorm_mean += stats[i].g_small_sqnorm_mean;
    }
    if (first) return fail(GNSB_EINVAL, "gns: aggregate over an empty selection");
    return debug_ok("gnsb_aggregate");
}

gnsb_status gnsb_gns_step(const double* layer_sums, const int32_t* layer_types, int32_t n_layers, int64_t B,
                          double alpha, gnsb_ema_state* state, double* out_groups, double* out_layers, void* stream) {
    if (B < 2) return fail(GNSB_EINVAL, "trainer: per-example estimation needs batch >= 2");
    if (!(alpha > 0.0) || alpha > 1.0) return fail(GNSB_EINVAL, "gns: ema alpha must be in (0, 1]");
    if (n_layers < 1 || n_layers > 512) return fail(GNSB_EINVAL, "gns: layer count must be in [1, 512]");
    if (!layer_sums || !layer_types || !state || !out_groups) return fail(GNSB_EINVAL, "gns: null pointer");
    if (gnsb_status s = need_device("gnsb_gns_step")) return s;
    gnsb::GnsStepArgs a{};
    a.sums = layer_sums;
    a.n = n_layers;
    a.B = B;
    a.alpha = alpha;
    a.state = state;
    a.out_groups = out_groups;
    a.out_layers = out_layers;
    for (int i = 0; i < n_layers; ++i) {
        if (layer_types[i] < 0 || layer_types[i] > 2) return fail(GNSB_EINVAL, "gns: unknown layer type");
        a.types[i] = (int8_t)layer_types[i];
    }
    gnsb::gns_step_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? debug_ok("gnsb_gns_step") : cuda_fail(e, "gns_step launch");
}

// ------------------------------------------------------------ costmodel ---
static gnsb_status cost_check(int64_t b, int64_t t, int64_t k, int64_t l) {
    if (b < 1 || t < 1 || k < 1 || l < 1) return fail(GNSB_EINVAL, "costmodel: shape dims must be positive");
    return GNSB_OK;
}

gnsb_status gnsb_flops(int64_t b, int64_t t, int64_t k, int64_t l, int32_t method, int64_t* out) {
    if (gnsb_status s = cost_check(b, t, k, l)) return s;
    if (method == 0) {  // costmodel.cpp:25-37
        out[0] = b * k * l * (2 * t - 1) + k * l * (b - 1);
        out[1] = b * k * l + b * (k * l - 1);
    } else {
        out[0] = k * l * (2 * b * t - 1);
        out[1] = b * t * t * (2 * k + 2 * l - 2) + b * t * t;
    }
    return debug_ok("gnsb_flops");
}

gnsb_status gnsb_io_values(int64_t b, int64_t t, int64_t k, int64_t l, int32_t method, int64_t* out) {
    if (gnsb_status s = cost_check(b, t, k, l)) return s;
    if (method == 0) {  // costmodel.cpp:39-51
        out[0] = b * k * l + b * k * t + b * l * t;
        out[1] = b * k * l + b;
    } else {
        out[0] = b * k * t + b * l * t + k * l;
        out[1] = 2 * b * t * t + b;
    }
    return debug_ok("gnsb_io_values");
}

gnsb_status gnsb_crossover_t(int64_t k, int64_t l, int32_t criterion, double* out) {
    if (k < 1 || l < 1) return fail(GNSB_EINVAL, "costmodel: dims must be positive");
    const double kd = (double)k, ld = (double)l;  // costmodel.cpp:58-64
    *out = criterion == 0 ? std::sqrt(2.0 * kd * ld) / 2.0 : std::sqrt((2.0 * kd * ld - 1.0) / (2.0 * kd + 2.0 * ld - 1.0));
    return debug_ok("gnsb_crossover_t");
}

// ------------------------------------------------------------- synthetic --
gnsb_status gnsb_synth_ln(void* x, void* dy, void* gamma, void* beta, int64_t B, int64_t T, int64_t D,
                          int64_t b_offset, int64_t B_div, float sigma, uint64_t stream0, gnsb_dtype dt, void* stream) {
    if (B < 0 || T < 0 || D < 1 || B_div < 1) return fail(GNSB_EINVAL, "synth: invalid extents");
    if (gnsb_status s = need_device("gnsb_synth_ln")) return s;
    const cudaError_t e = gnsb::launch_synth_ln((int)dt, x, dy, gamma, beta, B, T, D, b_offset, (float)B_div, sigma,
                                                seeds(stream0), static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok("gnsb_synth_ln") : cuda_fail(e, "synth_ln launch");
}

gnsb_status gnsb_synth_linear(void* x, void* dy, int64_t B, int64_t T, int64_t K, int64_t L, int64_t b_offset,
                              int64_t B_div, uint64_t stream0, gnsb_dtype dt, void* stream) {
    if (B < 0 || T < 1 || K < 1 || L < 1 || B_div < 1) return fail(GNSB_EINVAL, "synth: invalid extents");
    if (gnsb_status s = need_device("gnsb_synth_linear")) return s;
    const float scale = (float)B_div * sqrtf((float)T);
    const cudaError_t e = gnsb::launch_synth_linear((int)dt, x, dy, B, T, K, L, b_offset, scale, seeds(stream0),
                                                    static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? debug_ok("gnsb_synth_linear") : cuda_fail(e, "synth_linear launch");
}

}  // extern "C"

// ln_sweep.cu — configuration sweep of the fused LN-backward kernel (experiment only).
#include <cstdio>
#include <vector>

#include "../paper_2411_00999_b200/csrc/ln_launch.cuh"

namespace gnsb {
cudaError_t ensure_smem_attr(const void* kernel, size_t bytes) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
    if (e != cudaSuccess || (size_t)fa.maxDynamicSharedSizeBytes >= bytes) return e;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
int device_sm_count() {
    int v = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}
}  // namespace gnsb

using namespace gnsb;
using bf = __nv_bfloat16;

#define CFGS(X) \
    X(0, 8, 2, 1, 2, true, 1) \
    X(1, 16, 1, 1, 2, true, 1) \
    X(2, 16, 2, 1, 1, true, 1) \
    X(5, 8, 1, 2, 2, true, 1) \
    X(6, 4, 2, 3, 1, true, 1) \
    X(10, 4, 1, 4, 2, true, 1) \
    X(12, 4, 1, 3, 4, true, 1) \
    X(13, 4, 1, 3, 2, true, 1) \
    X(15, 3, 1, 5, 2, true, 1) \
    X(20, 16, 2, 1, 1, false, 1) \
    X(22, 16, 2, 1, 1, true, 0) \
    X(24, 1, 3, 16, 1, true, 0) \
    X(25, 1, 3, 8, 2, true, 0) \
    X(26, 1, 3, 8, 1, true, 1) \
    X(27, 1, 4, 16, 1, true, 0) \
    X(28, 1, 4, 8, 2, true, 0) \
    X(29, 2, 2, 8, 1, true, 0) \
    X(30, 2, 4, 4, 2, true, 0) \
    X(31, 16, 2, 1, 2, true, 0) \
    X(32, 16, 2, 1, 2, true, 1) \
    X(33, 8, 4, 1, 1, true, 0) \
    X(34, 8, 4, 1, 2, true, 0) \
    X(35, 3, 1, 2, 2, true, 1, 2) \
    X(36, 3, 1, 4, 1, true, 1, 2) \
    X(37, 4, 1, 2, 2, true, 1, 2) \
    X(38, 4, 1, 3, 1, true, 1, 2) \
    X(39, 8, 1, 1, 2, true, 1, 2) \
    X(40, 4, 2, 1, 2, true, 1, 2) \
    X(41, 1, 3, 4, 2, true, 1, 2) \
    X(42, 11, 3, 1, 1, true, 1) \
    X(43, 12, 3, 1, 1, true, 1) \
    X(44, 11, 3, 1, 1, true, 0) \
    X(45, 6, 3, 1, 1, true, 1) \
    X(46, 6, 3, 1, 2, true, 1) \
    X(47, 5, 4, 1, 1, true, 1) \
    X(48, 3, 3, 3, 1, true, 1) \
    X(49, 4, 2, 2, 2, true, 1) \
    X(50, 8, 1, 1, 4, true, 1) \
    X(51, 4, 2, 1, 4, true, 1) \
    X(52, 4, 1, 2, 4, true, 1) \
    X(53, 2, 2, 4, 2, true, 1) \
    X(54, 2, 2, 2, 4, true, 1) \
    X(55, 3, 1, 3, 4, true, 1) \
    X(56, 3, 1, 2, 4, true, 1) \
    X(57, 4, 1, 1, 8, true, 1) \
    X(58, 1, 4, 8, 2, true, 1) \
    X(59, 1, 4, 16, 1, true, 1) \
    X(60, 1, 3, 16, 1, true, 1) \
    X(61, 1, 3, 8, 2, true, 1) \
    X(62, 2, 2, 8, 1, true, 1) \
    X(63, 2, 4, 8, 1, true, 1) \
    X(64, 2, 4, 4, 2, true, 1) \
    X(65, 1, 4, 12, 1, true, 1) \
    X(66, 4, 1, 4, 2, true, 1, 1, true) \
    X(67, 4, 1, 4, 1, true, 1, 1, true) \
    X(68, 4, 1, 4, 1, true, 1) \
    X(69, 8, 1, 2, 2, true, 1, 1, true) \
    X(70, 8, 1, 2, 1, true, 1, 1, true) \
    X(71, 8, 1, 2, 1, true, 1) \
    X(72, 3, 1, 5, 2, true, 1, 1, true) \
    X(73, 4, 1, 3, 2, true, 1, 1, true) \

extern "C" {
int sweep_n() { return 74; }

int sweep_desc(int id, int* out) {
#define DESC(i, gw, vpt, g, rpg, prod, keep, ...) \
    if (id == i) { out[0] = gw; out[1] = vpt; out[2] = g; out[3] = rpg; out[4] = prod; out[5] = LnBwdCfg<bf, gw, vpt, g, rpg, prod, keep, ##__VA_ARGS__>::KEEP; return 0; }
    CFGS(DESC)
    return -1;
}

// the production grouped stage 2 (ln_bwd_reduce_run) of n bf16 LayerNorms of
// extents meta[3l..3l+2] = (B, M, D), with per-CTA trace stamps ([total CTAs][6])
int sweep_reduce(int n, const int64_t* meta, void* const* ws, void* const* dgamma, void* const* dbeta,
                 double* const* rg, double* const* rb, double* const* sums, int norms, void* stream,
                 unsigned long long* trace) {
    std::vector<LnRedItem> items(n);
    for (int l = 0; l < n; ++l) {
        LnRedItem& it = items[l];
        const char* why = nullptr;
        if (ln_bwd_plan_info<bf>(meta[3 * l], meta[3 * l + 1], meta[3 * l + 2], &it.info, &why)) return 1;
        it.B = meta[3 * l];
        it.M = meta[3 * l + 1];
        it.D = meta[3 * l + 2];
        it.ws = ws[l];
        it.dgamma = dgamma[l];
        it.dbeta = dbeta[l];
        it.raw_g = rg[l];
        it.raw_b = rb[l];
        it.sums = sums[l];
    }
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    return ln_bwd_reduce_run(0, norms, items.data(), n, (cudaStream_t)stream, trace, &why, &ce);
}

// the production row-pass dispatch (ln_bwd_rows_run) with per-CTA trace stamps
int sweep_rows_prod(const void* x, const void* mean, const void* rstd, const void* dy, const void* gamma, void* dx,
                    int64_t B, int64_t M, int64_t D, void* ws, size_t wsb, void* stream, unsigned long long* trace) {
    LnBwdCall c{x, mean, rstd, dy, gamma, dx, nullptr, nullptr, nullptr, nullptr, nullptr, 0, B, M, D, ws, wsb,
                trace, nullptr};
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    int rc = ln_bwd_rows_run<bf>(c, (cudaStream_t)stream, &why, &ce);
    if (rc == 1) fprintf(stderr, "rows: %s\n", why ? why : "?");
    return rc ? (rc == 2 ? 1000 + (int)ce : 1) : 0;
}

// The steady step of config `id`: the row pass of n LayerNorms (arrays of
// per-layer pointers) then ONE grouped stage 2 (ln_bwd_reduce_run), as
// bench.py's per-width steady measurement, with this config's plan info.
int sweep_step(int id, int n, const void* const* x, const void* const* mean, const void* const* rstd,
               const void* const* dy, const void* const* gamma, void* const* dx, void* const* dgamma,
               void* const* dbeta, double* const* rg, double* const* rb, double* const* sums, int norms, int64_t B,
               int64_t M, int64_t D, void* const* ws, size_t wsb, void* stream) {
    std::vector<LnRedItem> items(n);
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
    for (int l = 0; l < n; ++l) {
        LnBwdCall c{x[l], mean[l], rstd[l], dy[l], gamma[l], dx[l], dgamma[l], dbeta[l], rg[l], rb[l], sums[l],
                    norms > 0 ? 1 : 0, B, M, D, ws[l], wsb};
        LnRedItem& it = items[l];
        int rc = -1;
#define ROWS(i, gw, vpt, g, rpg, prod, keep, ...) \
        if (id == i) rc = BwdOp<LnBwdCfg<bf, gw, vpt, g, rpg, prod, keep, ##__VA_ARGS__>>::run_rows(c, (cudaStream_t)stream, &why, &ce, &it.info);
        CFGS(ROWS)
        if (rc != 0) {
            if (rc == 1) fprintf(stderr, "cfg%d: %s\n", id, why ? why : "?");
            return rc < 0 ? -1 : rc == 2 ? 1000 + (int)ce : 1;
        }
        it.B = B; it.M = M; it.D = D; it.ws = ws[l];
        it.dgamma = dgamma[l]; it.dbeta = dbeta[l]; it.raw_g = rg[l]; it.raw_b = rb[l]; it.sums = sums[l];
    }
    if (norms < 0) return 0;  // rows only (timing the row passes alone)
    int rc = ln_bwd_reduce_run(0, norms, items.data(), n, (cudaStream_t)stream, nullptr, &why, &ce);
    return rc ? (rc == 2 ? 1000 + (int)ce : 1) : 0;
}

int sweep_run(int id, const void* x, const void* mean, const void* rstd, const void* dy, const void* gamma, void* dx,
              void* dgamma, void* dbeta, double* rg, double* rb, double* sums, int norms, int64_t B, int64_t M,
              int64_t D, void* ws, size_t wsb, void* stream, unsigned long long* trace,
              unsigned long long* trace2) {
    LnBwdCall c{x, mean, rstd, dy, gamma, dx, dgamma, dbeta, rg, rb, sums, norms, B, M, D, ws, wsb, trace, trace2};
    const char* why = nullptr;
    cudaError_t ce = cudaSuccess;
#define RUN(i, gw, vpt, g, rpg, prod, keep, ...) \
    if (id == i) { int rc = BwdOp<LnBwdCfg<bf, gw, vpt, g, rpg, prod, keep, ##__VA_ARGS__>>::run(c, (cudaStream_t)stream, &why, &ce); if (rc == 1) fprintf(stderr, "cfg%d: %s\n", i, why ? why : "?"); return rc ? (rc == 2 ? 1000 + (int)ce : 1) : 0; }
    CFGS(RUN)
    return -1;
}
}

// ln_sweep.cu — configuration sweep of the fused LN-backward kernel (experiment only).
#include <cstdio>

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

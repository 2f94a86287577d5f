// ln_fwd_sweep.cu — LayerNorm forward variants (experiment only): the
// warp-per-row kernel of csrc/ln_fwd.cuh at several vectors-per-lane and
// CTAs-per-SM, called from ln_fwd_sweep.py next to the product gnsb_ln_fwd.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../paper_2411_00999_b200/csrc/ln_fwd.cuh"

using namespace gnsb;

template <int VPT, int MINB, bool PF>
static int launch(int bps, const LnFwdArgs& a, cudaStream_t st) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t)2 * a.D * sizeof(float);
    int64_t grid = (int64_t)sms * bps;
    const int64_t need = (a.N + 7) / 8;
    if (grid > need) grid = need;
    ln_fwd_warp_kernel<__nv_bfloat16, VPT, MINB, PF><<<(int)grid, 256, smem, st>>>(a);
    return (int)cudaGetLastError();
}

extern "C" int fwd_warp_run(int vpt, int minb, int pf, int bps, const void* x, const void* gamma, const void* beta, void* y, void* mean,
                            void* rstd, long long N, long long D, void* stream) {
    LnFwdArgs a{};
    a.x = x;
    a.gamma = gamma;
    a.beta = beta;
    a.y = y;
    a.mean = mean;
    a.rstd = rstd;
    a.N = N;
    a.D = D;
    a.eps = 1e-5;
    a.aligned = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (D % 8 || D / 8 > 32 * vpt) return -1;
    if (int e = (int)cudaFuncSetAttribute(ln_fwd_warp_kernel<__nv_bfloat16, 32, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536)) return e;
#define CASE(V, MB, PF) \
    if (vpt == V && minb == MB && pf == PF) return launch<V, MB, PF>(bps, a, st);
    CASE(3, 1, 1) CASE(3, 4, 1) CASE(3, 4, 0) CASE(3, 6, 0) CASE(4, 1, 1) CASE(4, 3, 1) CASE(4, 4, 0) CASE(4, 6, 0)
    CASE(8, 1, 1) CASE(8, 2, 1) CASE(8, 2, 0) CASE(8, 3, 0) CASE(8, 4, 0) CASE(16, 1, 0) CASE(16, 2, 0)
    CASE(16, 3, 0) CASE(32, 1, 0)
#undef CASE
    return -2;
}

template <int GW, int VPT, int G, bool GBS, int CPS = 1>
static int ring_launch(const LnFwdArgs& a0, int smax, cudaStream_t st) {
    using RC = LnFwdRingCfg<__nv_bfloat16, GW, VPT, G>;
    LnFwdArgs a = a0;
    a.Dp = (int64_t)GW * 32 * VPT * 8;
    if (a.Dp < a.D) return -1;
    if (a.Dp >= 2 * a.D) return -1;
    int optin = 0, sms = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t budget = CPS == 1 ? (size_t)optin - 1024 : (size_t)(228 * 1024) / CPS - 2048;
    int S = 0;
    for (int s2 = smax; s2 >= 2; --s2)
        if (RC::smem_bytes(s2, a.Dp, a.D) <= budget) {
            S = s2;
            break;
        }
    if (!S) return -3;
    const size_t smem = RC::smem_bytes(S, a.Dp, a.D);
    auto k = ln_fwd_ring_kernel<__nv_bfloat16, GW, VPT, G, GBS, CPS>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -4;
    k<<<sms * CPS, RC::kThreads, smem, st>>>(a, S);
    return (int)cudaGetLastError();
}

extern "C" int fwd_ring_run(int cfg, int smax, const void* x, const void* gamma, const void* beta, void* y, void* mean,
                            void* rstd, long long N, long long D, void* stream) {
    LnFwdArgs a{};
    a.x = x;
    a.gamma = gamma;
    a.beta = beta;
    a.y = y;
    a.mean = mean;
    a.rstd = rstd;
    a.N = N;
    a.D = D;
    a.eps = 1e-5;
    a.aligned = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (cfg) {
        // D = 4096 (512 vectors)
        case 0: return ring_launch<8, 2, 2, false>(a, smax, st);   // product
        case 1: return ring_launch<4, 4, 4, false>(a, smax, st);
        case 2: return ring_launch<4, 4, 4, true>(a, smax, st);
        case 3: return ring_launch<2, 8, 8, true>(a, smax, st);
        case 4: return ring_launch<8, 2, 3, false>(a, smax, st);
        case 5: return ring_launch<4, 4, 6, true>(a, smax, st);
        // D = 8192 (1024 vectors)
        case 10: return ring_launch<11, 3, 1, false>(a, smax, st);  // product
        case 11: return ring_launch<8, 4, 2, true>(a, smax, st);
        case 12: return ring_launch<4, 8, 4, true>(a, smax, st);
        case 13: return ring_launch<8, 4, 2, false>(a, smax, st);
        case 14: return ring_launch<16, 2, 1, false>(a, smax, st);
        case 15: return ring_launch<4, 8, 3, true>(a, smax, st);
        // two CTAs per SM
        case 16: return ring_launch<16, 2, 1, true, 2>(a, smax, st);
        case 17: return ring_launch<16, 2, 1, false, 2>(a, smax, st);
        case 18: return ring_launch<8, 4, 1, true, 2>(a, smax, st);
        case 6: return ring_launch<8, 2, 2, true, 2>(a, smax, st);
        case 7: return ring_launch<8, 2, 1, true, 2>(a, smax, st);
        case 8: return ring_launch<16, 1, 1, false, 2>(a, smax, st);
        default: return -2;
    }
}

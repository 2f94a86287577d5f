// ln_reduce.cu — launcher of the LayerNorm backward's stage 2 (ln_bwd_reduce_kernel
// for one layer, ln_bwd_reduce_group_kernel for several), in one translation
// unit so each kernel is a single device function with a single smem attribute.
//
// Column ranges: the stage-2 CTAs of a layer split its 16-byte column vectors
// into contiguous ranges.  For a group, the SMs are shared between layers in
// proportion to their staging volume (column vectors x slots), at least one
// CTA and at most one per four vectors each.
#include <algorithm>
#include <numeric>
#include <vector>

#include "internal.h"
#include "ln_bwd.cuh"

namespace gnsb {

namespace {

inline int smem_optin() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

struct RedShape {
    int rgrid = 0, eb = 0, slot_cap = 0;
    size_t smem = 0;
};

// examples per shared-memory block for a layer split over rgrid CTAs
RedShape red_shape(const LnRedItem& it, int V, int rgrid, int acc_bytes) {
    RedShape r;
    r.rgrid = rgrid;
    const int64_t U = (it.info.Dp + V - 1) / V;
    const int64_t ncol = (U + rgrid - 1) / rgrid * V;
    const int64_t N = it.B * it.M;
    const int64_t rows_per_cta = N / it.info.grid_rows;  // floor: a block of eb examples spans <= eb*M/rpc + 2 CTAs
    auto layout = [&](int64_t eb) {
        const int64_t span = rows_per_cta > 0 ? (eb * it.M + rows_per_cta - 1) / rows_per_cta + 2 : N;
        return LnRedLayout{ncol, eb, (span + eb) * it.info.gsub};
    };
    constexpr size_t kBudget = 160 << 10;
    int64_t eb = it.B < kMaxReduceEb ? it.B : kMaxReduceEb;
    while (eb > 1 && layout(eb).bytes(acc_bytes) > kBudget) eb = (eb + 1) / 2;
    LnRedLayout lay = layout(eb);
    if (lay.bytes(acc_bytes) > kBudget) {  // eb == 1 and one example spans too many CTAs: chunk its slots
        const size_t per_slot = (size_t)LnRedLayout::slot_bytes(ncol, acc_bytes);
        const size_t fixed = lay.stage_off();
        lay.nslot_max = fixed + per_slot <= kBudget ? (int64_t)((kBudget - fixed) / per_slot) : 1;
    }
    r.eb = (int)eb;
    r.slot_cap = (int)lay.nslot_max;
    r.smem = lay.bytes(acc_bytes);
    return r;
}

LnRedArgs red_args(const LnRedItem& it, const RedShape& r, unsigned long long* trace) {
    unsigned char* ws = static_cast<unsigned char*>(it.ws);
    LnRedArgs a{};
    a.partial = ws + it.info.off_partial;
    a.slot_stride = (int64_t)(it.info.G / it.info.gsub) * 2 * it.info.Dp;
    a.gsub = it.info.gsub;
    a.B = it.B;
    a.M = it.M;
    a.N = it.B * it.M;
    a.D = it.D;
    a.Dp = it.info.Dp;
    a.grid_rows = it.info.grid_rows;
    a.eb = r.eb;
    a.slot_cap = r.slot_cap;
    a.dgamma = it.dgamma;
    a.dbeta = it.dbeta;
    a.raw_g = it.raw_g;
    a.raw_b = it.raw_b;
    a.sums = it.sums;
    a.q = reinterpret_cast<double*>(ws + it.info.off_q);
    a.qbig = reinterpret_cast<double*>(ws + it.info.off_qbig);
    a.rawws = reinterpret_cast<double*>(ws + it.info.off_raw);
    a.ticket = reinterpret_cast<unsigned*>(ws) + 1;
    a.trace = trace;
    return a;
}

template <typename Acc>
int reduce_run_t(int norms, const LnRedItem* items, int n, cudaStream_t st, unsigned long long* trace,
                 const char** why, cudaError_t* cerr) {
    constexpr int V = 16 / sizeof(Acc);
    const int sms = std::min(device_sm_count(), kMaxReduceGrid);
    // CTAs per layer
    std::vector<int64_t> useful(n), w(n);
    int64_t total_useful = 0;
    for (int l = 0; l < n; ++l) {
        const int64_t U = (items[l].info.Dp + V - 1) / V;
        useful[l] = std::max<int64_t>(1, std::min<int64_t>((U + 3) / 4, sms));
        w[l] = U * (items[l].info.grid_rows + items[l].B) * items[l].info.gsub;
        total_useful += useful[l];
    }
    const int total = (int)std::min<int64_t>(std::max<int64_t>(sms, n), total_useful);
    std::vector<int> alloc(n, 1);
    int left = total - n;
    if (left > 0) {
        double wsum = 0.0;
        for (int l = 0; l < n; ++l) wsum += (double)w[l];
        std::vector<double> frac(n);
        for (int l = 0; l < n; ++l) {
            const double want = (double)left * (double)w[l] / wsum;
            const int add = (int)std::min<int64_t>((int64_t)want, useful[l] - 1);
            alloc[l] += add;
            frac[l] = want - (int64_t)want;
        }
        int rem = total - std::accumulate(alloc.begin(), alloc.end(), 0);
        // largest remainders first, then anyone with room
        std::vector<int> order(n);
        for (int l = 0; l < n; ++l) order[l] = l;
        std::sort(order.begin(), order.end(), [&](int x, int y) { return frac[x] > frac[y]; });
        for (int pass = 0; pass < 2 && rem > 0; ++pass)
            for (int k = 0; k < n && rem > 0; ++k) {
                const int l = order[k];
                if (alloc[l] < useful[l]) {
                    ++alloc[l];
                    --rem;
                }
            }
    }
    std::vector<RedShape> shapes(n);
    size_t smem = 0;
    for (int l = 0; l < n; ++l) {
        shapes[l] = red_shape(items[l], V, alloc[l], sizeof(Acc));
        smem = std::max(smem, shapes[l].smem);
    }
    if (smem + 16384 > (size_t)smem_optin()) {
        *why = "layers: trailing extent too wide for the stage-2 shared memory";
        return 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kReduceThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (n == 1) {
        void (*k)(LnRedArgs) = norms ? ln_bwd_reduce_kernel<Acc, true> : ln_bwd_reduce_kernel<Acc, false>;
        e = ensure_smem_attr(reinterpret_cast<const void*>(k), smem);
        if (e == cudaSuccess) {
            cfg.gridDim = dim3(alloc[0]);
            e = cudaLaunchKernelEx(&cfg, k, red_args(items[0], shapes[0], trace));
        }
    } else {
        LnRedGroup g{};
        g.n = n;
        int b = 0;
        for (int l = 0; l < n; ++l) {
            g.items[l] = red_args(items[l], shapes[l], trace ? trace + (size_t)b * 6 : nullptr);
            g.begin[l] = b;
            b += alloc[l];
        }
        g.begin[n] = b;
        void (*k)(LnRedGroup) =
            norms ? ln_bwd_reduce_group_kernel<Acc, true> : ln_bwd_reduce_group_kernel<Acc, false>;
        e = ensure_smem_attr(reinterpret_cast<const void*>(k), smem);
        if (e == cudaSuccess) {
            cfg.gridDim = dim3(b);
            e = cudaLaunchKernelEx(&cfg, k, g);
        }
    }
    if (e != cudaSuccess) {
        *cerr = e;
        *why = "ln_bwd reduce launch";
        return 2;
    }
    return 0;
}

}  // namespace

int ln_bwd_reduce_run(int acc_f64, int norms, const LnRedItem* items, int n, cudaStream_t st,
                      unsigned long long* trace, const char** why, cudaError_t* cerr) {
    if (n < 1) return 0;
    if (n > kMaxReduceGroup) {
        *why = "layers: too many pending LayerNorms in one reduce (max 64)";
        return 1;
    }
    return acc_f64 ? reduce_run_t<double>(norms, items, n, st, trace, why, cerr)
                   : reduce_run_t<float>(norms, items, n, st, trace, why, cerr);
}

}  // namespace gnsb

// embedding_pe.cu — embedding-table gradient with per-example squared norms
// (paper Alg. 3).
//
// Semantics: gnstk::embedding_backward_simultaneous (proj/src/layers.cpp:315-368).
// For example b, the table rows it touches accumulate its token gradients in
// token order, dE_b[v] = sum_{t: id_bt = v} g_bt; raw_b = ||dE_b||^2 over the
// touched rows in ascending id order; dW[v] = sum_b dE_b[v] in example order.
//
// Two kernels, no floating-point atomics (bitwise deterministic; with fp64
// rows dW and raw_b reproduce the reference's operation order exactly):
//   * emb_example_kernel: one CTA per example.  The example's (id, t) keys are
//     sorted in shared memory (bitonic), so equal ids form runs in token order;
//     for each run the CTA sums the run's gradient rows (threads over columns),
//     writes the compact row dE_b[k] to the workspace and accumulates its
//     squares.  raw_b: fp64 rows use one flat sequential sum in the
//     reference's (row, column) order, other dtypes a fixed-order block sum.
//   * emb_table_kernel: one CTA per table row v (grid-stride).  It finds v in
//     each example's sorted run list (binary search, example order) and adds
//     those dE_b[v] rows, then writes dW[v] (zero for untouched rows) and its
//     squares for ||dW||^2.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace gnsb {

namespace {

constexpr int kEmbThreads = 256;
constexpr int kEmbMaxT = 16384;  // keys of one example sorted in shared memory

struct EmbWs {
    void* E;          // [B][T][D] Acc: compact per-example rows (first U_b used)
    int32_t* u;       // [B][T] sorted unique ids of each example
    int32_t* U;       // [B] number of unique ids
    double* qbig;     // [grid_table] per-CTA ||dW||^2 partials
    int32_t* bad;     // [1] set when an id is outside [0, V)
};

template <typename T>
__global__ void __launch_bounds__(kEmbThreads) emb_example_kernel(const int32_t* ids, const T* g, int64_t Tn, int64_t D,
                                                                  int64_t V, EmbWs w, double* raw, int Tp) {
    using Acc = typename Traits<T>::Acc;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);            // [Tp]
    int32_t* start = reinterpret_cast<int32_t*>(keys + Tp);       // [Tp + 1] run starts
    __shared__ int s_nruns;
    __shared__ double s_red[kEmbThreads / 32];
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x;
    const int32_t* idb = ids + b * Tn;
    for (int i = tid; i < Tp; i += blockDim.x) {
        uint64_t k = ~0ull;
        if (i < Tn) {
            int32_t id = idb[i];
            if (id < 0 || id >= V) {
                atomicExch(w.bad, 1);
                id = -1;  // skipped below
            }
            k = id < 0 ? ~0ull : ((uint64_t)(uint32_t)id << 32) | (uint32_t)i;
        }
        keys[i] = k;
    }
    __syncthreads();
    // bitonic sort, ascending (id, t)
    for (int size = 2; size <= Tp; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < Tp; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const uint64_t a = keys[i], c = keys[j];
                    const bool up = (i & size) == 0;
                    if ((a > c) == up) {
                        keys[i] = c;
                        keys[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    // runs of equal ids (one thread: T <= 16384 cheap integer steps)
    if (tid == 0) {
        int n = 0;
        uint32_t prev = 0xffffffffu;
        int i = 0;
        for (; i < (int)Tn; ++i) {
            if (keys[i] == ~0ull) break;  // skipped (invalid) ids sort last
            const uint32_t id = (uint32_t)(keys[i] >> 32);
            if (id != prev) {
                start[n] = i;
                w.u[b * Tn + n] = (int32_t)id;
                ++n;
                prev = id;
            }
        }
        start[n] = i;
        s_nruns = n;
        w.U[b] = n;
    }
    __syncthreads();
    const int nruns = s_nruns;
    Acc* E = static_cast<Acc*>(w.E) + (size_t)b * Tn * D;
    double part = 0.0;
    for (int k = 0; k < nruns; ++k) {
        const int i0 = start[k], i1 = start[k + 1];
        for (int64_t j = tid; j < D; j += blockDim.x) {
            Acc acc = Acc(0);
            for (int i = i0; i < i1; ++i) {
                const int64_t t = (int64_t)(uint32_t)(keys[i] & 0xffffffffu);
                acc += to_acc<T>(g[(b * Tn + t) * D + j]);
            }
            E[(size_t)k * D + j] = acc;
            part = fma((double)acc, (double)acc, part);
        }
    }
    if constexpr (sizeof(Acc) == 8) {
        // fp64 rows: the reference's single flat accumulator, (row, column) order
        __syncthreads();
        if (tid == 0) {
            __threadfence_block();
            double sb = 0.0;
            for (int64_t e = 0; e < (int64_t)nruns * D; ++e) {
                const double v = (double)E[e];
                sb = __dadd_rn(sb, __dmul_rn(v, v));  // no contraction: the reference's mul-then-add
            }
            raw[b] = sb;
        }
    } else {
        part = warp_sum(part);
        if ((tid & 31) == 0) s_red[tid >> 5] = part;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += s_red[k];
            raw[b] = t;
        }
    }
}

template <typename Acc>
__global__ void __launch_bounds__(kEmbThreads) emb_table_kernel(int64_t B, int64_t Tn, int64_t V, int64_t D, EmbWs w,
                                                                Acc* dW, int dw_rows_per_cta) {
    __shared__ int s_k[1024];  // run index of v in example b (or -1), for a block of examples
    __shared__ double s_red[kEmbThreads / 32];
    const int tid = threadIdx.x;
    const Acc* E = static_cast<const Acc*>(w.E);
    double part = 0.0;
    const int64_t v0 = (int64_t)blockIdx.x * dw_rows_per_cta;
    for (int64_t v = v0; v < v0 + dw_rows_per_cta && v < V; ++v) {
        // accumulate in Acc, examples in order (the reference's dW order)
        for (int64_t j0 = 0; j0 < D; j0 += blockDim.x) {
            const int64_t j = j0 + tid;
            Acc acc = Acc(0);
            for (int64_t bb0 = 0; bb0 < B; bb0 += 1024) {
                const int nb = (int)((B - bb0) < 1024 ? (B - bb0) : 1024);
                __syncthreads();
                for (int q = tid; q < nb; q += blockDim.x) {
                    const int64_t b = bb0 + q;
                    const int32_t* ub = w.u + b * Tn;
                    int lo = 0, hi = w.U[b] - 1, found = -1;
                    while (lo <= hi) {
                        const int mid = (lo + hi) >> 1;
                        const int32_t x = ub[mid];
                        if (x == (int32_t)v) {
                            found = mid;
                            break;
                        }
                        if (x < (int32_t)v) lo = mid + 1;
                        else hi = mid - 1;
                    }
                    s_k[q] = found;
                }
                __syncthreads();
                if (j < D)
                    for (int q = 0; q < nb; ++q) {
                        const int k = s_k[q];
                        if (k >= 0) acc += E[(((size_t)(bb0 + q)) * Tn + k) * D + j];
                    }
            }
            if (j < D) {
                dW[v * D + j] = acc;
                part = fma((double)acc, (double)acc, part);
            }
        }
    }
    part = warp_sum(part);
    if ((tid & 31) == 0) s_red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += s_red[k];
        w.qbig[blockIdx.x] = t;
    }
}

int pow2_at_least(int64_t n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

struct EmbLayout {
    size_t E, u, U, qbig, bad, raw, total;
    int grid_table, rows_per_cta;
};

EmbLayout emb_layout(int64_t B, int64_t Tn, int64_t V, int64_t D, int acc_bytes) {
    EmbLayout l{};
    const int sms = device_sm_count();
    const int64_t target = (int64_t)sms * 8;
    l.rows_per_cta = (int)((V + target - 1) / target);
    if (l.rows_per_cta < 1) l.rows_per_cta = 1;
    l.grid_table = (int)((V + l.rows_per_cta - 1) / l.rows_per_cta);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 255) / 256 * 256;
        return o;
    };
    l.E = take((size_t)B * Tn * D * acc_bytes);
    l.u = take((size_t)B * Tn * 4);
    l.U = take((size_t)B * 4);
    l.qbig = take((size_t)(l.grid_table > 0 ? l.grid_table : 1) * 8);
    l.bad = take(4);
    l.raw = take((size_t)B * 8);  // raw_b when the caller passes none
    l.total = off;
    return l;
}

}  // namespace

bool embedding_shape_ok(int64_t T) { return T >= 1 && T <= kEmbMaxT; }

size_t embedding_workspace(int64_t B, int64_t T, int64_t V, int64_t D, int dt) {
    return emb_layout(B, T, V, D, dt == 2 ? 8 : 4).total;
}

template <typename T>
cudaError_t emb_run(const int32_t* ids, const void* g, void* dW, double* raw, double* sums, int64_t B, int64_t Tn,
                    int64_t V, int64_t D, void* ws, int32_t* bad_flag_out, cudaStream_t st) {
    using Acc = typename Traits<T>::Acc;
    const EmbLayout l = emb_layout(B, Tn, V, D, sizeof(Acc));
    unsigned char* base = static_cast<unsigned char*>(ws);
    EmbWs w{base + l.E, reinterpret_cast<int32_t*>(base + l.u), reinterpret_cast<int32_t*>(base + l.U),
            reinterpret_cast<double*>(base + l.qbig), reinterpret_cast<int32_t*>(base + l.bad)};
    if (raw == nullptr) raw = reinterpret_cast<double*>(base + l.raw);
    cudaError_t e = cudaMemsetAsync(w.bad, 0, 4, st);
    if (e != cudaSuccess) return e;
    const int Tp = pow2_at_least(Tn);
    const size_t smem = (size_t)Tp * 8 + (size_t)(Tp + 1) * 4;
    e = ensure_smem_attr(reinterpret_cast<const void*>(emb_example_kernel<T>), smem);
    if (e != cudaSuccess) return e;
    emb_example_kernel<T><<<(unsigned)B, kEmbThreads, smem, st>>>(ids, static_cast<const T*>(g), Tn, D, V, w, raw, Tp);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (l.grid_table > 0) {
        emb_table_kernel<Acc><<<l.grid_table, kEmbThreads, 0, st>>>(B, Tn, V, D, w, static_cast<Acc*>(dW),
                                                                   l.rows_per_cta);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (sums) {
        e = launch_fold_rows(raw, 1, (int)B, nullptr, sums, 0, st);
        if (e == cudaSuccess && l.grid_table > 0) e = launch_fold_rows(w.qbig, 1, l.grid_table, nullptr, sums, 2, st);
    }
    if (e == cudaSuccess && bad_flag_out) e = cudaMemcpyAsync(bad_flag_out, w.bad, 4, cudaMemcpyDeviceToDevice, st);
    return e;
}

cudaError_t launch_embedding_pe(int dt, const int32_t* ids, const void* g, void* dW, double* raw, double* sums,
                                int64_t B, int64_t T, int64_t V, int64_t D, void* ws, int32_t* bad, cudaStream_t st) {
    switch (dt) {
        case 0: return emb_run<float>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
        case 1: return emb_run<__nv_bfloat16>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
        case 2: return emb_run<double>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace gnsb

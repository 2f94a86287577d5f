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

#include <algorithm>
#include <cstdlib>
#include <type_traits>

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

// ---------------------------------------------------------------------------
// Fast path for fp32 / bf16 rows (fp32 accumulation): no materialised
// per-example rows.
//   * emb_sort_kernel: one CTA per example sorts its (id, t) keys and writes
//     the token order perm[b][i] (sorted t) and one entry per run,
//     ent[b][k] = {id, first position in perm, length, first token}, plus the
//     run count U[b] (parallel run detection by a block scan).
//   * emb_rows_kernel: one warp per block of kRowsPerWarp table rows.  Lane j
//     of group G tracks example 32G + j: its first entry at or after the
//     block comes from a per-(example, block) table the sort kernel writes,
//     then it holds its next entry in registers (the
//     following one is loaded as soon as a row consumes it).  For row v the
//     warp ballots the matching examples and walks them in example order; for
//     each it sums the run's token rows (token order, lanes over 16-byte
//     column vectors; a one-token run needs no perm load) into dE_b[v], adds
//     that to dW[v] and reduces ||dE_b[v]||^2 into q[b][k].  g is read once
//     and dW written once, 16 bytes per lane per vector.  (4-column lane
//     vectors for bf16 -- one float4 of dW per lane, 512 contiguous bytes per
//     warp store -- measured slower: 81 against 75 us at GPT-2 size.)
//   * emb_raw_kernel: raw_b = sum_k q[b][k] (one CTA per example, fixed-order
//     tree); the scalar sums by fold_rows_kernel.
// dW matches the original path bit for bit (same per-example Acc sums, added
// in example order); raw_b differs in summation order only.
constexpr int kEmbSortThreads = 1024;
constexpr int kEmbBuckets = 4096;  // id buckets of the sort kernel's bucket sort (at most)
#ifndef GNSB_EMB_BUCKETS_PER_KEY
#define GNSB_EMB_BUCKETS_PER_KEY 1  // buckets per (padded) key, at most kEmbBuckets (0: always kEmbBuckets; 1 measured 65.2 against 66.6 us at GPT-2 size)
#endif
#ifndef GNSB_EMB_RPW
#define GNSB_EMB_RPW 8
#endif
constexpr int kRowsPerWarp = GNSB_EMB_RPW;  // table rows per warp (A/B: -DGNSB_EMB_RPW=4 / 2)
constexpr int kEmbRowsThreads = 256;
constexpr int kEmbMaxGroups = 8;  // examples handled by the fast path: B <= 32 * 8

#ifndef GNSB_EMB_PDL
#define GNSB_EMB_PDL 1  // the walk and the raw kernel launch with programmatic dependent launch (A/B: 0)
#endif
// Programmatic dependent launch: the kernel's CTAs are scheduled while its
// predecessor drains; it calls griddepcontrol.wait before touching anything
// the predecessor wrote.
template <typename... KArgs, typename... Args>
cudaError_t emb_launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = GNSB_EMB_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

struct EmbFastWs {
    int32_t* perm;  // [B][Tn]
    int4* ent;      // [B][Tn] {id, start, len, first token}
    int32_t* U;     // [B]
    double* q;      // [B][Tn]
    double* qbig;   // [rows-kernel CTAs]
    int32_t* bad;
    int32_t* blk;      // [B][nblk + 1]: first entry of example b with id >= j * kRowsPerWarp
    int64_t nblk;      // row blocks: ceil(V / kRowsPerWarp)
    // mask walk (emb_mask_kernel) only; null for the cursor walk
    uint32_t* mask;    // [V][mw]: bit b set when example b has a run at id v
    int2* idx2;        // [V][B]: {run index r, first token | 0x80000000 when the run has > 1 token}
    int mw;            // mask words per row: ceil(B / 32)
    int hv;            // sort CTAs per example (mask walk: 2, each the ids of one half of the table); perm, ent,
                       // q and U hold hv "virtual examples" of Tn entries per example, in id order
};

template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int before = warp > 0 ? s_warp[warp - 1] : 0;
    *total = s_warp[NT / 32 - 1];
    return before + x - v;
}

// Key = id << SH | t (SH = 32 with 64-bit keys; with 32-bit keys SH = log2(Tp),
// used when every id fits: half the shared-memory and shuffle traffic).
template <typename KT>
__global__ void __launch_bounds__(kEmbSortThreads) emb_sort_kernel(const int32_t* ids, int64_t Tn, int64_t V,
                                                                   EmbFastWs w, int Tp, int SH, int BSH, int NB) {
    extern __shared__ __align__(16) unsigned char smem[];
    KT* keys = reinterpret_cast<KT*>(smem);  // [Tp]
    const KT TM = (KT(1) << SH) - 1;         // token mask
    const KT NONE = ~KT(0);
    __shared__ int s_warp[kEmbSortThreads / 32];
    __shared__ int s_nvalid;
    const int hv = w.hv;
    const int64_t b = blockIdx.x / hv, vb = blockIdx.x;  // example, virtual example (example, half)
    const int64_t Bn = gridDim.x / hv;
    // ids this CTA sorts: one half of the table per CTA when hv == 2
    const int64_t vmid = (V + 1) / 2;
    const int64_t id_lo = (hv == 2 && (vb & 1)) ? vmid : 0, id_hi = (hv == 2 && !(vb & 1)) ? vmid : V;
    const int tid = threadIdx.x;
    const int32_t* idb = ids + b * Tn;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the walk may get scheduled
    __shared__ int s_maxb;
    if (tid == 0) {
        s_nvalid = 0;
        s_maxb = 0;
    }
    bool bitonic = NB == 0;
    if (NB > 0) {
        // Bucket sort by id >> BSH (NB <= kEmbBuckets buckets): histogram,
        // block scan, scatter, then an insertion sort inside each bucket by the
        // full (id, t) key (about T / NB keys per bucket).  Five barriers in
        // all, against ~15 shared-memory rounds of the bitonic network.
        KT* tmp = keys + Tp;                                         // [Tp] scattered keys
        int* cnt = reinterpret_cast<int*>(tmp + Tp);                 // [NB + 1] counts -> bucket starts
        int* cur = cnt + NB + 1;                                     // [NB] scatter cursors
        for (int i = tid; i <= NB; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        for (int i = tid; i < Tp; i += blockDim.x) {
            KT k = NONE;
            if (i < Tn) {
                const int32_t id = idb[i];
                if (id < 0 || id >= V)
                    atomicExch(w.bad, 1);
                else if (id >= id_lo && id < id_hi) {
                    k = ((KT)(uint32_t)id << SH) | (KT)(uint32_t)i;
                    atomicAdd(&cnt[id >> BSH], 1);
                }
            }
            tmp[i] = k;
        }
        __syncthreads();
        // a heavy bucket (one id repeated, e.g. padding) would make the
        // per-bucket insertion sort quadratic: take the bitonic network then
        for (int c = tid; c < NB; c += blockDim.x)
            if (cnt[c] > 64) atomicMax(&s_maxb, cnt[c]);
        __syncthreads();
        bitonic = s_maxb > 64;
    }
    if (!bitonic) {
        KT* tmp = keys + Tp;
        int* cnt = reinterpret_cast<int*>(tmp + Tp);
        int* cur = cnt + NB + 1;
        // exclusive scan of the counts: a contiguous chunk per thread
        const int per = (NB + kEmbSortThreads - 1) / kEmbSortThreads;
        const int c0 = tid * per, c1 = min(c0 + per, NB);
        int local = 0;
        for (int c = c0; c < c1; ++c) local += cnt[c];
        int total = 0;
        int run = block_exclusive_scan<kEmbSortThreads>(local, s_warp, &total);
        for (int c = c0; c < c1; ++c) {
            const int n = cnt[c];
            cnt[c] = run;
            cur[c] = run;
            run += n;
        }
        if (tid == 0) cnt[NB] = total;
        __syncthreads();
        // scatter (order inside a bucket is fixed by the insertion sort below);
        // invalid / pad keys fill the tail
        for (int i = tid; i < Tp; i += blockDim.x) {
            const KT k = tmp[i];
            if (k != NONE) keys[atomicAdd(&cur[(int)((uint32_t)(k >> SH) >> BSH)], 1)] = k;
        }
        for (int i = total + tid; i < Tp; i += blockDim.x) keys[i] = NONE;
        __syncthreads();
        for (int c = tid; c < NB; c += blockDim.x) {
            const int lo = cnt[c], hi = cnt[c + 1];
            for (int i = lo + 1; i < hi; ++i) {
                const KT v = keys[i];
                int j = i - 1;
                while (j >= lo && keys[j] > v) {
                    keys[j + 1] = keys[j];
                    --j;
                }
                keys[j + 1] = v;
            }
        }
        __syncthreads();
    } else {
        if (NB > 0) {  // the keys are in tmp, in token order: sort them in place in keys
            const KT* tmp = keys + Tp;
            for (int i = tid; i < Tp; i += blockDim.x) keys[i] = tmp[i];
        } else
        for (int i = tid; i < Tp; i += blockDim.x) {
            KT k = NONE;
            if (i < Tn) {
                const int32_t id = idb[i];
                if (id < 0 || id >= V)
                    atomicExch(w.bad, 1);
                else if (id >= id_lo && id < id_hi)
                    k = ((KT)(uint32_t)id << SH) | (KT)(uint32_t)i;
            }
            keys[i] = k;
        }
        __syncthreads();
        // bitonic sort, ascending (id, t): strides >= 32 through shared memory,
        // strides < 32 inside the warp with shuffles (Tp is a multiple of 32)
        for (int size = 2; size <= Tp; size <<= 1) {
            int stride = size >> 1;
            for (; stride >= 32; stride >>= 1) {
                for (int i = tid; i < Tp; i += blockDim.x) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const KT a = keys[i], c = keys[j];
                        const bool up = (i & size) == 0;
                        if ((a > c) == up) {
                            keys[i] = c;
                            keys[j] = a;
                        }
                    }
                }
                __syncthreads();
            }
            for (int i0 = 0; i0 < Tp; i0 += blockDim.x) {
                if (i0 + (tid & ~31) >= Tp) break;  // warp-uniform
                const int i = i0 + tid;
                KT v = keys[i];
                const bool up = (i & size) == 0;
                for (int s2 = stride; s2 > 0; s2 >>= 1) {
                    const KT o = __shfl_xor_sync(0xffffffffu, v, s2);
                    const bool keep_min = ((i & s2) == 0) == up;  // the lower element keeps the min when ascending
                    v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
                }
                keys[i] = v;
            }
            __syncthreads();
        }
    }
    // run heads: a valid key whose id differs from its predecessor's.  Each
    // thread scans a contiguous chunk; a block scan numbers the runs.
    const int per = (Tp + kEmbSortThreads - 1) / kEmbSortThreads;
    const int i0 = tid * per, i1 = min(i0 + per, Tp);
    auto valid = [&](int i) { return i < Tp && keys[i] != NONE; };
    auto head = [&](int i) { return valid(i) && (i == 0 || (uint32_t)(keys[i - 1] >> SH) != (uint32_t)(keys[i] >> SH)); };
    int cnt = 0, nv = 0;
    for (int i = i0; i < i1; ++i) {
        if (!valid(i)) break;
        cnt += head(i) ? 1 : 0;
        nv = i + 1;
    }
    if (nv > 0) atomicMax(&s_nvalid, nv);
    int total = 0;
    int r = block_exclusive_scan<kEmbSortThreads>(cnt, s_warp, &total);  // (its barriers publish s_nvalid)
    const int nvalid = s_nvalid;
    int32_t* perm = w.perm + vb * Tn;
    int4* ent = w.ent + vb * Tn;
    int32_t* blk = w.blk + b * (w.nblk + 1);  // (cursor walk: hv == 1, vb == b)
    const int hoff = (int)(vb - b * hv) * (int)Tn;  // this half's offset inside the example's hv * Tn entries
    for (int i = i0; i < i1; ++i) {
        if (!valid(i)) break;
        perm[i] = (int32_t)(uint32_t)(keys[i] & TM);
        if (head(i)) {
            const uint32_t id = (uint32_t)(keys[i] >> SH);
            int e = i + 1;
            while (e < nvalid && (uint32_t)(keys[e] >> SH) == id) ++e;
            const int t0 = (int)(uint32_t)(keys[i] & TM);
            ent[r] = make_int4((int)id, hoff + i, e - i, t0);
            if (w.mask) {  // the mask walk: mark (id, b), record where its run lives
                atomicOr(w.mask + (int64_t)id * w.mw + (b >> 5), 1u << (b & 31));
                w.idx2[(int64_t)id * Bn + b] =
                    make_int2(hoff + r, e - i > 1 ? (int)(0x80000000u | (uint32_t)t0) : t0);
            } else {
                // row blocks whose first row lies in (previous id, id] start at entry r
                const int64_t j_lo = r == 0 ? 0 : (int64_t)((uint32_t)(keys[i - 1] >> SH) / kRowsPerWarp) + 1;
                const int64_t j_hi = (int64_t)(id / kRowsPerWarp);
                for (int64_t j = j_lo; j <= j_hi; ++j) blk[j] = r;
            }
            ++r;
        }
    }
    // blocks after the last id start past the end
    const int64_t j_tail = nvalid > 0 ? (int64_t)((uint32_t)(keys[nvalid - 1] >> SH) / kRowsPerWarp) + 1 : 0;
    if (!w.mask)
        for (int64_t j = j_tail + tid; j <= w.nblk; j += blockDim.x) blk[j] = total;
    if (tid == 0) w.U[vb] = total;
}

#ifndef GNSB_EMB_OCC
#define GNSB_EMB_OCC 768  // resident threads per SM the row walk is compiled for (1024 = 64 registers spills: 93 against 76 us)
#endif
template <typename T, int NVC, int NG, int NT = kEmbRowsThreads>
__global__ void __launch_bounds__(NT, GNSB_EMB_OCC / NT) emb_rows_kernel(const T* g, int64_t B, int64_t Tn, int64_t V,
                                                                int64_t D, EmbFastWs w, float* dW) {
    constexpr int W = Traits<T>::W;
    constexpr int NP = W / 2;
    using P = float2;
    __shared__ double s_red[NT / 32];
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nvec = (int)(D / W);
    const int nchunk = (nvec + 32 * NVC - 1) / (32 * NVC);
    double qb = 0.0;  // this lane's share of ||dW||^2
    for (int64_t v0 = gw * kRowsPerWarp; v0 < V; v0 += nw * kRowsPerWarp) {
        int p[NG], Ub[NG];
        int4 cur[NG];  // the lane's next unconsumed entry of its example
#pragma unroll
        for (int G = 0; G < NG; ++G) {
            p[G] = 0;
            Ub[G] = 0;
            cur[G] = make_int4(-1, 0, 0, 0);
            const int64_t b = 32 * G + lane;
            if (b < B) {  // first entry with id >= v0 (the sort kernel's block table)
                Ub[G] = w.U[b];
                p[G] = w.blk[b * (w.nblk + 1) + v0 / kRowsPerWarp];
                if (p[G] < Ub[G]) cur[G] = w.ent[b * Tn + p[G]];
            }
        }
        const int64_t v1 = v0 + kRowsPerWarp < V ? v0 + kRowsPerWarp : V;
        for (int64_t v = v0; v < v1; ++v) {
            unsigned mask[NG];
#pragma unroll
            for (int G = 0; G < NG; ++G) mask[G] = __ballot_sync(0xffffffffu, cur[G].x == (int32_t)v);
            double qacc[NG];
#pragma unroll
            for (int G = 0; G < NG; ++G) qacc[G] = 0.0;
            for (int c = 0; c < nchunk; ++c) {
                P acc[NVC][NP];
#pragma unroll
                for (int k = 0; k < NVC; ++k)
#pragma unroll
                    for (int e = 0; e < NP; ++e) acc[k][e] = make_float2(0.f, 0.f);
#pragma unroll
                for (int G = 0; G < NG; ++G) {
                    unsigned mk = mask[G];
                    while (mk) {
                        const int bb = __ffs(mk) - 1;
                        mk &= mk - 1;
                        const int64_t b = 32 * G + bb;
                        const int start = __shfl_sync(0xffffffffu, cur[G].y, bb);
                        const int len = __shfl_sync(0xffffffffu, cur[G].z, bb);
                        const int t0 = __shfl_sync(0xffffffffu, cur[G].w, bb);
                        P tmp[NVC][NP];
#pragma unroll
                        for (int q = 0; q < NVC; ++q)
#pragma unroll
                            for (int e = 0; e < NP; ++e) tmp[q][e] = make_float2(0.f, 0.f);
                        for (int i = 0; i < len; ++i) {  // the run's tokens in token order
                            const int64_t t = i == 0 ? t0 : w.perm[b * Tn + start + i];
                            const T* row = g + (b * Tn + t) * D;
#pragma unroll
                            for (int q = 0; q < NVC; ++q) {
                                const int vi = (c * NVC + q) * 32 + lane;
                                if (vi < nvec) {
                                    P x[NP];
                                    unpack2<T>(__ldg(reinterpret_cast<const uint4*>(row) + vi), x);
#pragma unroll
                                    for (int e = 0; e < NP; ++e) {
                                        tmp[q][e].x += x[e].x;
                                        tmp[q][e].y += x[e].y;
                                    }
                                }
                            }
                        }
                        double sq = 0.0;
#pragma unroll
                        for (int q = 0; q < NVC; ++q)
#pragma unroll
                            for (int e = 0; e < NP; ++e) {
                                acc[q][e].x += tmp[q][e].x;
                                acc[q][e].y += tmp[q][e].y;
                                sq = fma((double)tmp[q][e].x, (double)tmp[q][e].x, sq);
                                sq = fma((double)tmp[q][e].y, (double)tmp[q][e].y, sq);
                            }
                        sq = warp_sum(sq);
                        if (lane == bb) qacc[G] += sq;
                    }
                }
#pragma unroll
                for (int q = 0; q < NVC; ++q) {
                    const int vi = (c * NVC + q) * 32 + lane;
                    if (vi < nvec) {
                        float* dst = dW + v * D + (int64_t)vi * W;
#pragma unroll
                        for (int e = 0; e < NP; e += 2) {
                            const float4 o = make_float4(acc[q][e].x, acc[q][e].y, acc[q][e + 1].x, acc[q][e + 1].y);
                            reinterpret_cast<float4*>(dst)[e / 2] = o;
                            qb = fma((double)o.x, (double)o.x, qb);
                            qb = fma((double)o.y, (double)o.y, qb);
                            qb = fma((double)o.z, (double)o.z, qb);
                            qb = fma((double)o.w, (double)o.w, qb);
                        }
                    }
                }
            }
#pragma unroll
            for (int G = 0; G < NG; ++G) {
                if ((mask[G] >> lane) & 1u) {  // consume the entry, fetch the next
                    const int64_t b = 32 * G + lane;
                    w.q[b * Tn + p[G]] = qacc[G];
                    ++p[G];
                    cur[G] = p[G] < Ub[G] ? w.ent[b * Tn + p[G]] : make_int4(-1, 0, 0, 0);
                }
            }
        }
    }
    qb = warp_sum(qb);
    if (lane == 0) s_red[threadIdx.x >> 5] = qb;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < NT / 32; ++k) t += s_red[k];
        w.qbig[blockIdx.x] = t;
    }
}

#ifndef GNSB_EMB_PB3
#define GNSB_EMB_PB3 4  // mask walk: first-token rows in flight per batch for <= 3 vectors per lane (A/B)
#endif
#ifndef GNSB_EMB_MOCC
#define GNSB_EMB_MOCC 512  // resident threads per SM the mask walk is compiled for (128 registers)
#endif
// Mask walk: the same sums as emb_rows_kernel, in the same order (dW and the
// per-run squares q are bitwise equal to it when one column chunk covers D),
// without the per-example cursors.  The sort kernel marks, per table row v, a
// bit per example with a run at v and records where that run lives
// (idx2[v][b]).  Warps take blocks of RB consecutive rows from a queue (an
// atomic counter; the next block's index and mask words are fetched while the
// current block runs):
//   1. lane l holds mask word l of the block (one coalesced load);
//   2. a warp scan numbers the (row, example) pairs in (row, example) order,
//      and the word lanes list them in shared memory, up to 32 at a time;
//   3. lane j loads pair j's idx2 entry (all pairs at once);
//   4. the warp loads the first token rows of PB pairs at once, sums each
//      pair's run, and stores each row (zero rows too) once its pairs are done.
// ||dW||^2 is kept per block (qbig[block]) so the queue order does not change
// its rounding; emb_raw_kernel folds the blocks in index order.
template <typename T, int NVC, int MW, int PB>
__global__ void __launch_bounds__(kEmbRowsThreads, GNSB_EMB_MOCC / kEmbRowsThreads)
    emb_mask_kernel(const T* g, int64_t B, int64_t Tn, int64_t V, int64_t D, EmbFastWs w, float* dW) {
    constexpr int W = Traits<T>::W;
    constexpr int NP = W / 2;
    constexpr int RB = MW <= 4 ? kRowsPerWarp : 32 / MW;  // rows per block: RB * MW <= 32 mask words
    constexpr int PC = 32;                                 // pairs listed per window
    using P = float2;
    __shared__ uint16_t s_pr[kEmbRowsThreads / 32][PC];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nvec = (int)(D / W);
    const int nchunk = (nvec + 32 * NVC - 1) / (32 * NVC);
    const int64_t nblocks = (V + RB - 1) / RB;
    const int64_t PS = (int64_t)w.hv * Tn;  // entries per example in perm / ent / q
    unsigned int* ctr = reinterpret_cast<unsigned int*>(w.mask + V * MW);  // zeroed with the mask
    auto take = [&]() {
        unsigned int x = 0;
        if (lane == 0) x = atomicAdd(ctr, 1u);
        return (int64_t)__shfl_sync(0xffffffffu, x, 0);
    };
    auto mask_of = [&](int64_t blk) {
        const int64_t v0 = blk * RB;
        const int nrow = blk < nblocks ? (int)(V - v0 < RB ? V - v0 : RB) : 0;
        return lane < nrow * MW ? __ldcg(w.mask + v0 * MW + lane) : 0u;
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the sort kernel's mask, idx2, runs
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    int64_t blk = take();
    uint32_t m = mask_of(blk);
    while (blk < nblocks) {
        const int64_t nxt = take();
        const uint32_t mn = mask_of(nxt);  // in flight while this block runs
        const int64_t v0 = blk * RB;
        const int nrow = (int)(V - v0 < RB ? V - v0 : RB);
        double qb = 0.0;  // this lane's share of the block's ||dW||^2
        const int cnt = __popc(m);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int excl = incl - cnt;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int c = 0; c < nchunk; ++c) {
            P acc[NVC][NP];
#pragma unroll
            for (int q = 0; q < NVC; ++q)
#pragma unroll
                for (int e = 0; e < NP; ++e) acc[q][e] = make_float2(0.f, 0.f);
            int vr = 0;  // the row being accumulated
            auto store_row = [&]() {
#pragma unroll
                for (int q = 0; q < NVC; ++q) {
                    const int vi = (c * NVC + q) * 32 + lane;
                    if (vi < nvec) {
                        float* dst = dW + (v0 + vr) * D + (int64_t)vi * W;
#pragma unroll
                        for (int e = 0; e < NP; e += 2) {
                            const float4 o = make_float4(acc[q][e].x, acc[q][e].y, acc[q][e + 1].x, acc[q][e + 1].y);
                            reinterpret_cast<float4*>(dst)[e / 2] = o;
                            qb = fma((double)o.x, (double)o.x, qb);
                            qb = fma((double)o.y, (double)o.y, qb);
                            qb = fma((double)o.z, (double)o.z, qb);
                            qb = fma((double)o.w, (double)o.w, qb);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < NP; ++e) acc[q][e] = make_float2(0.f, 0.f);
                }
                ++vr;
            };
            for (int base = 0; base < total; base += PC) {
                __syncwarp();
                if (cnt > 0 && excl < base + PC && incl > base) {
                    uint32_t mm = m;
                    for (int k = excl; mm && k < base + PC; ++k) {
                        const int bit = __ffs(mm) - 1;
                        mm &= mm - 1;
                        if (k >= base) s_pr[wid][k - base] = (uint16_t)(((lane / MW) << 8) | ((lane % MW) * 32 + bit));
                    }
                }
                __syncwarp();
                const int n = total - base < PC ? total - base : PC;
                int pi = 0, pb = 0, pr = 0, pt = 0, pst = 0, pln = 1;
                if (lane < n) {
                    const uint32_t e = s_pr[wid][lane];
                    pi = (int)(e >> 8);
                    pb = (int)(e & 255u);
                    const int2 x = __ldcg(w.idx2 + (v0 + pi) * B + pb);
                    pr = x.x;
                    pt = x.y & 0x7fffffff;
                    if (x.y < 0) {  // a run of several tokens: its start in the sorted list
                        const int4 en = __ldcg(w.ent + (int64_t)pb * PS + pr);
                        pst = en.y;
                        pln = en.z;
                    }
                }
                for (int k0 = 0; k0 < n; k0 += PB) {
                    uint4 xb[PB][NVC];  // the first token rows of PB pairs, all in flight at once
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const int64_t b = __shfl_sync(0xffffffffu, pb, (k0 + u) & 31);
                        const int64_t t = __shfl_sync(0xffffffffu, pt, (k0 + u) & 31);
                        const uint4* row = reinterpret_cast<const uint4*>(g + (b * Tn + t) * D);
#pragma unroll
                        for (int q = 0; q < NVC; ++q) {
                            const int vi = (c * NVC + q) * 32 + lane;
                            xb[u][q] = (k0 + u < n && vi < nvec) ? __ldg(row + vi) : make_uint4(0u, 0u, 0u, 0u);
                        }
                    }
                    double sqv[PB];  // per-lane squares of the batch's pairs, reduced together below
#pragma unroll
                    for (int u = 0; u < PB; ++u) sqv[u] = 0.0;
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const int k = k0 + u;
                        if (k >= n) break;
                        const int i = __shfl_sync(0xffffffffu, pi, k);
                        const int64_t b = __shfl_sync(0xffffffffu, pb, k);
                        const int len = __shfl_sync(0xffffffffu, pln, k);
                        const int st = __shfl_sync(0xffffffffu, pst, k);
                        while (vr < i) store_row();
                        P tmp[NVC][NP];
#pragma unroll
                        for (int q = 0; q < NVC; ++q) {
                            P x[NP];
                            unpack2<T>(xb[u][q], x);
#pragma unroll
                            for (int e = 0; e < NP; ++e) {
                                tmp[q][e] = make_float2(0.f, 0.f);
                                tmp[q][e].x += x[e].x;
                                tmp[q][e].y += x[e].y;
                            }
                        }
                        for (int j = 1; j < len; ++j) {  // the run's later tokens in token order
                            const int64_t t = w.perm[b * PS + st + j];
                            const uint4* row = reinterpret_cast<const uint4*>(g + (b * Tn + t) * D);
#pragma unroll
                            for (int q = 0; q < NVC; ++q) {
                                const int vi = (c * NVC + q) * 32 + lane;
                                if (vi < nvec) {
                                    P x[NP];
                                    unpack2<T>(__ldg(row + vi), x);
#pragma unroll
                                    for (int e = 0; e < NP; ++e) {
                                        tmp[q][e].x += x[e].x;
                                        tmp[q][e].y += x[e].y;
                                    }
                                }
                            }
                        }
                        double sq = 0.0;
#pragma unroll
                        for (int q = 0; q < NVC; ++q)
#pragma unroll
                            for (int e = 0; e < NP; ++e) {
                                acc[q][e].x += tmp[q][e].x;
                                acc[q][e].y += tmp[q][e].y;
                                sq = fma((double)tmp[q][e].x, (double)tmp[q][e].x, sq);
                                sq = fma((double)tmp[q][e].y, (double)tmp[q][e].y, sq);
                            }
                        sqv[u] = sq;
                    }
                    // PB interleaved butterflies (each result equals warp_sum of its pair's squares)
                    warp_sum_n<PB>(sqv);
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const int k = k0 + u;
                        const int64_t b = __shfl_sync(0xffffffffu, pb, k & 31);
                        const int r = __shfl_sync(0xffffffffu, pr, k & 31);
                        if (lane == 0 && k < n) {
                            double* qd = w.q + b * PS + r;
                            *qd = c == 0 ? sqv[u] : *qd + sqv[u];
                        }
                    }
                }
            }
            while (vr < nrow) store_row();
        }
        qb = warp_sum(qb);
        if (lane == 0) w.qbig[blk] = qb;
        blk = nxt;
        m = mn;
    }
}

// raw_b = sum_k q[b][k]: one 256-thread CTA per example.  Every load is
// issued before the first add (a thread owns a strided set of at most
// Tn / 256 entries), then a fixed-order tree: one L2 round trip instead of
// U / 32 dependent ones (the warp-per-example version was latency-bound,
// 9.5 us at T = 1024).
// The mask walk's version (`tail` set) has one more CTA, which folds the
// per-block ||dW||^2 partials in block order; the last CTA to finish (ticket)
// then writes sums[0] = sum_b raw_b, sums[2] = ||dW||^2 and the bad-id flag,
// in place of two fold launches and a copy.
struct EmbRawTail {
    const double* qblk;   // [nq] per-block ||dW||^2
    int nq;
    double* qtot;         // [1]
    unsigned int* ticket; // zeroed with the mask
    double* sums;         // may be null
    const int32_t* bad;   // the sort kernel's flag
    int32_t* bad_out;     // may be null
};

__global__ void __launch_bounds__(256) emb_raw_kernel(int64_t B, int64_t Tn, EmbFastWs w, double* raw,
                                                      EmbRawTail tl = EmbRawTail{}) {
    __shared__ double s_red[256];
    __shared__ bool s_last;
    const int64_t b = blockIdx.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the walk's q, qbig
    if (tl.ticket != nullptr) {
        if (b == B) {  // the ||dW||^2 partials: 8 independent chains (loads in flight), fixed order
            double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            int k = threadIdx.x;
            for (; k + 256 * 7 < tl.nq; k += 256 * 8)
#pragma unroll
                for (int u = 0; u < 8; ++u) t[u] += __ldcg(tl.qblk + k + 256 * u);
            for (; k < tl.nq; k += 256) t[0] += __ldcg(tl.qblk + k);
            s_red[threadIdx.x] = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
        } else {
            // the example's runs in id order: the first half's U0, then the second half's (hv == 2)
            const int hv = w.hv;
            const int U0 = w.U[b * hv], U = U0 + (hv == 2 ? w.U[b * hv + 1] : 0);
            const double* qb = w.q + b * hv * Tn;
            double s = 0.0;
#pragma unroll 8
            for (int k = threadIdx.x; k < U; k += 256) s += __ldcg(qb + (k < U0 ? k : Tn + (k - U0)));
            s_red[threadIdx.x] = s;
        }
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (b == B)
                *tl.qtot = s_red[0];
            else
                raw[b] = s_red[0];
            __threadfence();
            s_last = atomicAdd(tl.ticket, 1u) == (unsigned)B;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        double s = 0.0;  // sum_b raw_b: a fixed tree over b
        for (int k = threadIdx.x; k < B; k += 256) s += __ldcg(raw + k);
        s_red[threadIdx.x] = s;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (tl.sums) {
                tl.sums[0] = s_red[0];
                tl.sums[2] = __ldcg(tl.qtot);
            }
            if (tl.bad_out) *tl.bad_out = __ldcg(tl.bad);
        }
        return;
    }
    const int U = w.U[b];
    double s = 0.0;
#pragma unroll 8
    for (int k = threadIdx.x; k < U; k += 256) s += __ldcg(w.q + b * Tn + k);
    s_red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) raw[b] = s_red[0];
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


namespace {

struct EmbFastLayout {
    size_t perm, ent, U, q, qbig, bad, raw, blk, mask, idx2, qtot, total;
    int grid;   // row-walk CTAs (the mask walk's when `masked`)
    int64_t nblk;
    int64_t nqblk;  // mask walk: row blocks = ||dW||^2 partials
    int hv;         // sort CTAs per example
    bool masked;
    int mw;
};

// GNSB_EMB_WALK=cursor: never the mask walk; =mask: always (tests, A/B runs)
bool emb_mask_walk() {
    static const bool v = [] {
        const char* e = std::getenv("GNSB_EMB_WALK");
        return !(e && e[0] == 'c');
    }();
    return v;
}
bool emb_mask_forced() {
    static const bool v = [] {
        const char* e = std::getenv("GNSB_EMB_WALK");
        return e && e[0] == 'm';
    }();
    return v;
}

// threads per row-walk CTA: 256, or 64 (B <= 32; GNSB_EMB_CTA=64, A/B runs).
// Smaller CTAs retire independently (one warp with many matched rows holds
// back a 2-warp CTA instead of an 8-warp one) but measured no faster at GPT-2
// size: 84.0 us against 82.7 us.
int emb_rows_threads(int64_t B) {
    static const int v = [] {
        const char* e = std::getenv("GNSB_EMB_CTA");
        return (e && std::atoi(e) == 64) ? 64 : kEmbRowsThreads;
    }();
    return B <= 32 ? v : kEmbRowsThreads;
}

EmbFastLayout emb_fast_layout(int64_t B, int64_t Tn, int64_t V, bool bf16) {
    EmbFastLayout l{};
    const int sms = device_sm_count();
    const int64_t blocks = (V + kRowsPerWarp - 1) / kRowsPerWarp;  // row blocks, one per warp
    const int64_t wpc = emb_rows_threads(B) / 32;
    const int64_t grid = (blocks + wpc - 1) / wpc;
    int64_t cap = (int64_t)sms * 16 * (kEmbRowsThreads / 32) / wpc;
    // One resident wave, grid-stride beyond it: warps never retire between row
    // blocks, so no CTA waits on a predecessor's store drain (74 against 76 us
    // with 1.8 waves of one-block warps at GPT-2 size).  GNSB_EMB_WAVES=k
    // allows k waves (0 = one warp per block), A/B runs.
    static const int waves = [] {
        const char* e = std::getenv("GNSB_EMB_WAVES");
        return e ? std::atoi(e) : 1;
    }();
    if (waves > 0) cap = std::min<int64_t>(cap, (int64_t)sms * (GNSB_EMB_OCC / (32 * wpc)) * waves);
    l.grid = (int)(grid < cap ? (grid > 0 ? grid : 1) : cap);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 255) / 256 * 256;
        return o;
    };
    // The mask walk for bf16 rows when the table has at least two row blocks
    // per resident warp (the queue balances the warps); the cursor walk for
    // fp32 rows and small tables.  Measured at B=32 T=1024 D=768: V=50257
    // bf16 68 against 75 us (B=64: 84 against 129), but fp32 rows 115 against
    // 89 us and V=8192 77 against 60 us.
    const int ng = (int)((B + 31) / 32);
    const int mw = ng <= 1 ? 1 : ng <= 2 ? 2 : ng <= 4 ? 4 : 8;  // the kernel's MW
    const int64_t rb = mw <= 4 ? kRowsPerWarp : 32 / mw;
    const int64_t resident_warps = (int64_t)sms * (GNSB_EMB_MOCC / 32);
    l.masked = emb_mask_walk() && (emb_mask_forced() || (bf16 && (V + rb - 1) / rb >= 2 * resident_warps));
    // mask walk: two sort CTAs per example (each the ids of one half of the
    // table) while that fits the SMs; GNSB_EMB_SORT_HALVES=0 keeps one (A/B)
    static const bool halves_off = [] {
        const char* e = std::getenv("GNSB_EMB_SORT_HALVES");
        return e && e[0] == '0';
    }();
    l.hv = (l.masked && !halves_off && B <= sms) ? 2 : 1;
    l.perm = take((size_t)B * l.hv * Tn * 4);
    l.ent = take((size_t)B * l.hv * Tn * 16);
    l.U = take((size_t)B * l.hv * 4);
    l.q = take((size_t)B * l.hv * Tn * 8);
    l.bad = take(4);
    l.raw = take((size_t)B * 8);
    l.nblk = blocks;
    if (l.masked) {
        l.mw = mw;
        l.nqblk = (V + rb - 1) / rb;
        const int64_t mwpc = kEmbRowsThreads / 32;
        const int64_t mgrid = (l.nqblk + mwpc - 1) / mwpc;
        const int64_t mcap = (int64_t)sms * (GNSB_EMB_MOCC / kEmbRowsThreads);  // one resident wave
        l.grid = (int)(mgrid < mcap ? (mgrid > 0 ? mgrid : 1) : mcap);
        l.blk = take(4);
        l.mask = take((size_t)V * l.mw * 4 + 16);  // + the block queue's counter
        l.idx2 = take((size_t)V * B * 8);
        l.qbig = take((size_t)l.nqblk * 8);
        l.qtot = take(8);
    } else {
        l.blk = take((size_t)B * (blocks + 1) * 4);
        l.qbig = take((size_t)l.grid * 8);
        l.qtot = take(8);
        l.mask = take(16);  // no mask words: only the tail (counter, bad flag, ticket)
    }
    l.total = off;
    return l;
}

// the fast path: fp32 / bf16 rows made of whole 16-byte vectors (D a multiple
// of the vector width), 16-byte aligned g and dW, B <= 256
bool emb_fast_ok(int dt, int64_t B, int64_t D) {
    static const bool forced_slow = [] {  // GNSB_EMB_IMPL=slow: the two-kernel path (A/B runs)
        const char* e = std::getenv("GNSB_EMB_IMPL");
        return e && e[0] == 's';
    }();
    const int W = dt == 1 ? 8 : 4;
    return !forced_slow && dt != 2 && B >= 1 && B <= 32 * kEmbMaxGroups && D % W == 0 && D > 0;
}

}  // namespace

size_t embedding_workspace(int64_t B, int64_t T, int64_t V, int64_t D, int dt) {
    // (the path also depends on pointer alignment: room for either)
    const size_t slow = emb_layout(B, T, V, D, dt == 2 ? 8 : 4).total;
    if (!emb_fast_ok(dt, B, D)) return slow;
    const size_t fast = emb_fast_layout(B, T, V, dt == 1).total;
    return fast > slow ? fast : slow;
}

template <typename T>
cudaError_t emb_fast_run(const int32_t* ids, const void* g, void* dW, double* raw, double* sums, int64_t B,
                         int64_t Tn, int64_t V, int64_t D, void* ws, int32_t* bad_flag_out, cudaStream_t st) {
    const EmbFastLayout l = emb_fast_layout(B, Tn, V, sizeof(T) == 2);
    unsigned char* base = static_cast<unsigned char*>(ws);
    EmbFastWs w{reinterpret_cast<int32_t*>(base + l.perm), reinterpret_cast<int4*>(base + l.ent),
                reinterpret_cast<int32_t*>(base + l.U),    reinterpret_cast<double*>(base + l.q),
                reinterpret_cast<double*>(base + l.qbig),  reinterpret_cast<int32_t*>(base + l.bad),
                reinterpret_cast<int32_t*>(base + l.blk),   l.nblk,
                l.masked ? reinterpret_cast<uint32_t*>(base + l.mask) : nullptr,
                l.masked ? reinterpret_cast<int2*>(base + l.idx2) : nullptr, l.mw, l.hv};
    if (raw == nullptr) raw = reinterpret_cast<double*>(base + l.raw);
    // the mask walk: one memset clears the mask words, the block queue's
    // counter, the bad-id flag and the raw kernel's ticket (the mask's tail)
    // (the cursor walk: the tail alone)
    const size_t mask_words = l.masked ? (size_t)V * l.mw * 4 : 0;
    unsigned int* tail = reinterpret_cast<unsigned int*>(base + l.mask + mask_words);
    w.bad = reinterpret_cast<int32_t*>(tail + 1);
    cudaError_t e = cudaMemsetAsync(base + l.mask, 0, mask_words + 16, st);
    if (e != cudaSuccess) return e;
    const int Tp = pow2_at_least(Tn < 32 ? 32 : Tn);  // whole warps in the shuffle stages
    int sh = 0;
    while ((1 << sh) < Tp) ++sh;
    // 32-bit keys when (V - 1) << log2(Tp) | (Tp - 1) stays below the all-ones sentinel
    const bool k32 = (((uint64_t)V) << sh) < 0xffffffffull;
    // buckets of 2^bsh ids, at most kEmbBuckets of them (the bitonic network
    // when that table plus two key arrays would not fit in shared memory)
    int bsh = 0;
    const int64_t bcap = GNSB_EMB_BUCKETS_PER_KEY > 0 ? std::min<int64_t>(kEmbBuckets, (int64_t)Tp * GNSB_EMB_BUCKETS_PER_KEY)
                                                       : kEmbBuckets;
    while (((V - 1) >> bsh) >= bcap) ++bsh;
    const int nb = (int)(((V - 1) >> bsh) + 1);
    const size_t kb = k32 ? 4 : 8;
    const size_t smem_bucket = 2 * (size_t)Tp * kb + (2 * (size_t)nb + 1) * 4;
    const bool bucket = smem_bucket <= (size_t)200 * 1024 && std::getenv("GNSB_EMB_SORT") == nullptr;
    const size_t smem = bucket ? smem_bucket : (size_t)Tp * kb;
    if (k32) {
        e = ensure_smem_attr(reinterpret_cast<const void*>(emb_sort_kernel<uint32_t>), smem);
        if (e != cudaSuccess) return e;
        emb_sort_kernel<uint32_t><<<(unsigned)(B * l.hv), kEmbSortThreads, smem, st>>>(ids, Tn, V, w, Tp, sh, bsh,
                                                                            bucket ? nb : 0);
    } else {
        e = ensure_smem_attr(reinterpret_cast<const void*>(emb_sort_kernel<uint64_t>), smem);
        if (e != cudaSuccess) return e;
        emb_sort_kernel<uint64_t><<<(unsigned)(B * l.hv), kEmbSortThreads, smem, st>>>(ids, Tn, V, w, Tp, 32, bsh,
                                                                            bucket ? nb : 0);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    constexpr int W = Traits<T>::W;
    const int64_t nvec = D / W;
    const T* gp = static_cast<const T*>(g);
    float* dWp = static_cast<float*>(dW);
    const int ng = (int)((B + 31) / 32);
    cudaError_t le = cudaSuccess;  // (launch errors of the PDL launches)
    auto launch = [&](auto nvc) {
        constexpr int NVC = decltype(nvc)::value;
        if (l.masked) {
            // first-token rows in flight per batch: 12-16 16-byte vectors per lane
            constexpr int PB = NVC <= 3 ? GNSB_EMB_PB3 : NVC <= 4 ? 3 : NVC <= 6 ? 2 : 1;
            if (l.mw == 1)
                le = emb_launch_pdl(emb_mask_kernel<T, NVC, 1, PB>, l.grid, kEmbRowsThreads, st, gp, B, Tn, V, D, w, dWp);
            else if (l.mw == 2)
                le = emb_launch_pdl(emb_mask_kernel<T, NVC, 2, PB>, l.grid, kEmbRowsThreads, st, gp, B, Tn, V, D, w, dWp);
            else if (l.mw == 4)
                le = emb_launch_pdl(emb_mask_kernel<T, NVC, 4, PB>, l.grid, kEmbRowsThreads, st, gp, B, Tn, V, D, w, dWp);
            else
                le = emb_launch_pdl(emb_mask_kernel<T, NVC, 8, PB>, l.grid, kEmbRowsThreads, st, gp, B, Tn, V, D, w, dWp);
        } else if (ng <= 1 && emb_rows_threads(B) == 64)
            emb_rows_kernel<T, NVC, 1, 64><<<l.grid, 64, 0, st>>>(gp, B, Tn, V, D, w, dWp);
        else if (ng <= 1)
            emb_rows_kernel<T, NVC, 1><<<l.grid, kEmbRowsThreads, 0, st>>>(gp, B, Tn, V, D, w, dWp);
        else if (ng <= 2)
            emb_rows_kernel<T, NVC, 2><<<l.grid, kEmbRowsThreads, 0, st>>>(gp, B, Tn, V, D, w, dWp);
        else if (ng <= 4)
            emb_rows_kernel<T, NVC, 4><<<l.grid, kEmbRowsThreads, 0, st>>>(gp, B, Tn, V, D, w, dWp);
        else
            emb_rows_kernel<T, NVC, 8><<<l.grid, kEmbRowsThreads, 0, st>>>(gp, B, Tn, V, D, w, dWp);
    };
    if (nvec <= 32)
        launch(std::integral_constant<int, 1>{});
    else if (nvec <= 64)
        launch(std::integral_constant<int, 2>{});
    else if (nvec <= 96)
        launch(std::integral_constant<int, 3>{});
    else if constexpr (sizeof(T) != 4)  // (bf16: 16 accumulator registers per vector, at most 4)
        launch(std::integral_constant<int, 4>{});
    else if (nvec <= 128)
        launch(std::integral_constant<int, 4>{});
    else if (nvec <= 192)  // fp32 rows at D = 768: one pass over the columns instead of two (94 -> 89 us)
        launch(std::integral_constant<int, 6>{});
    else
        launch(std::integral_constant<int, 8>{});
    e = le != cudaSuccess ? le : cudaGetLastError();
    if (e != cudaSuccess) return e;
    // one more CTA folds the ||dW||^2 partials (per row block, or per walk CTA
    // for the cursor walk); the last CTA writes sums[0], sums[2] and the flag
    const EmbRawTail tl{w.qbig, (int)(l.masked ? l.nqblk : l.grid), reinterpret_cast<double*>(base + l.qtot),
                        tail + 2, sums, w.bad, bad_flag_out};
    return emb_launch_pdl(emb_raw_kernel, (unsigned)B + 1, 256, st, B, Tn, w, raw, tl);
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
    const bool aligned = (reinterpret_cast<uintptr_t>(g) & 15u) == 0 && (reinterpret_cast<uintptr_t>(dW) & 15u) == 0;
    if (aligned && emb_fast_ok(dt, B, D)) {
        if (dt == 0) return emb_fast_run<float>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
        return emb_fast_run<__nv_bfloat16>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
    }
    switch (dt) {
        case 0: return emb_run<float>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
        case 1: return emb_run<__nv_bfloat16>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
        case 2: return emb_run<double>(ids, g, dW, raw, sums, B, T, V, D, ws, bad, st);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- forward --
// out[i, :] = W[ids[i], :] (proj/src/layers.cpp:300-313): one warp per token,
// 16-byte vectors when the rows are aligned.  Ids outside [0, V) write zero
// rows and raise *bad (the C++ drop-in checks the host ids first and throws
// the reference's "layers: id out of range").
template <typename T>
__global__ void __launch_bounds__(256) emb_fwd_kernel(const int32_t* __restrict__ ids, const T* __restrict__ W,
                                                      T* __restrict__ out, int64_t n, int64_t V, int64_t D, int vec,
                                                      int32_t* bad) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int32_t id = __ldg(ids + i);
    const bool ok = id >= 0 && id < V;
    if (!ok && lane == 0 && bad) *bad = 1;
    T* dst = out + i * D;
    if (vec) {
        constexpr int E = 16 / sizeof(T);
        const uint4* src = reinterpret_cast<const uint4*>(W + (ok ? (int64_t)id : 0) * D);
        for (int64_t v = lane; v < D / E; v += 32)
            reinterpret_cast<uint4*>(dst)[v] = ok ? __ldg(src + v) : make_uint4(0, 0, 0, 0);
    } else {
        for (int64_t d = lane; d < D; d += 32) dst[d] = ok ? W[(int64_t)id * D + d] : T(0);
    }
}

cudaError_t launch_embedding_fwd(int dt, const int32_t* ids, const void* W, void* out, int64_t n, int64_t V, int64_t D,
                                 int32_t* bad, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const size_t es = dt == 2 ? 8 : dt == 0 ? 4 : 2;
    const int vec = (D * (int64_t)es) % 16 == 0 && (reinterpret_cast<uintptr_t>(W) & 15u) == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    const unsigned grid = (unsigned)((n + 7) / 8);
    if (bad) {
        cudaError_t e = cudaMemsetAsync(bad, 0, 4, st);
        if (e != cudaSuccess) return e;
    }
    switch (dt) {
        case 0: emb_fwd_kernel<float><<<grid, 256, 0, st>>>(ids, (const float*)W, (float*)out, n, V, D, vec, bad); break;
        case 1:
            emb_fwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(ids, (const __nv_bfloat16*)W, (__nv_bfloat16*)out, n,
                                                                V, D, vec, bad);
            break;
        case 2: emb_fwd_kernel<double><<<grid, 256, 0, st>>>(ids, (const double*)W, (double*)out, n, V, D, vec, bad); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gnsb

// exchange.cu — the batch-sharded step's one collective, in the C ABI
// (SURVEY.md §8(b) `gnsb_allreduce_grads`, §8(e)).
//
// Per step every rank sums two buckets over NCCL (NVLink/NVSwitch on a B200
// box): the fp32/fp64 bucket of all layers' [p0 | p1] parameter gradients and
// the fp64 bucket of their 4-double norm records.  Record slots 2 and 3 then
// hold sums of LOCAL squared norms, which are not the squared norms of the
// reduced gradients, so one kernel re-forms them from the
// reduced gradient bucket (one CTA per vector, fixed-order reduction).
//
// libnccl is opened at run time (dlopen, RTLD_NOLOAD first so a process that
// already loaded one — e.g. PyTorch's — shares its instance): the library has
// no link-time NCCL dependency, and a communicator is only valid with the
// NCCL instance that created it, which is why the C ABI also exposes the three
// calls a C/C++ caller needs to make one (unique id, init rank, destroy).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "gnsb.h"
#include "internal.h"

namespace gnsb {

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef int nccl_result;
typedef struct {
    char internal[128];
} nccl_unique_id;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0 };

struct NcclApi {
    nccl_result (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_result (*get_unique_id)(nccl_unique_id*) = nullptr;
    nccl_result (*comm_init_rank)(void**, int, nccl_unique_id, int) = nullptr;
    nccl_result (*comm_destroy)(void*) = nullptr;
    const char* (*get_error_string)(nccl_result) = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* n : names)
            if (!h) h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);
        for (const char* n : names)
            if (!h) h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.get_error_string = reinterpret_cast<decltype(api.get_error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.all_reduce && api.get_unique_id && api.comm_init_rank && api.comm_destroy;
    });
    return api;
}

constexpr int kMaxBucketLayers = 256;
constexpr int kMaxVec = 2 * kMaxBucketLayers;
constexpr int64_t kChunk = 16384;  // elements per unpack CTA

// Layout of one step's exchange.  The device workspace holds
//   packed   fp64 [4 * n_layers (records, when exchanged) + total grads]
//   partials fp64 [n_chunks]   per-chunk squared sums of the reduced gradients
//   tickets  u32  [2 * n_layers] last-chunk counters (left zero by every call)
// Vector v = 2l + p is parameter p of layer l: width[v] values at grad offset[v].
struct BucketDesc {
    int64_t offset[kMaxVec];
    int64_t width[kMaxVec];
    int32_t chunk_base[kMaxVec + 1];  // every vector owns >= 1 chunk (an empty p1 writes a zero norm)
    int32_t nvec;
    int32_t with_records;
    int64_t total;   // gradient values
    int64_t rec_n;   // 4 * n_layers or 0
};

struct BucketLayout {
    BucketDesc d;
    size_t off_partials = 0, off_tickets = 0, bytes = 0;
};

inline int64_t packed_count(const BucketDesc& d) { return d.rec_n + d.total; }

// fp64 packed bucket <- [records | grads]
template <typename V>
__global__ void __launch_bounds__(256) bucket_pack_kernel(const V* __restrict__ grads,
                                                          const double* __restrict__ records,
                                                          const __grid_constant__ BucketDesc d, double* packed) {
    const int64_t n = d.rec_n + d.total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        packed[i] = i < d.rec_n ? records[i] : (double)grads[i - d.rec_n];
}

// grads <- reduced packed values; records[l][0..1] <- reduced sums of raw norms;
// records[l][2 + p] = ||reduced vector (l, p)||^2 in fp64: chunk partials, then
// the vector's last chunk (acq_rel ticket) sums them in chunk order.
template <typename V>
__global__ void __launch_bounds__(256) bucket_unpack_kernel(V* __restrict__ grads, double* __restrict__ records,
                                                            const __grid_constant__ BucketDesc d,
                                                            const double* __restrict__ packed, double* partials,
                                                            unsigned* tickets) {
    __shared__ double red[8];
    __shared__ bool last;
    const int c = blockIdx.x;
    int lo = 0, hi = d.nvec - 1;  // vector v with chunk_base[v] <= c < chunk_base[v + 1]
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (d.chunk_base[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const int v = lo;
    const int64_t w = d.width[v];
    const int64_t i0 = (int64_t)(c - d.chunk_base[v]) * kChunk;
    const int64_t i1 = i0 + kChunk < w ? i0 + kChunk : w;
    const double* src = packed + d.rec_n + d.offset[v];
    V* dst = grads + d.offset[v];
    double acc = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double x = src[i];
        dst[i] = (V)x;
        acc = fma(x, x, acc);
    }
    if (!d.with_records) return;
    if (c == d.chunk_base[v] && (v & 1) == 0 && threadIdx.x < 2)
        records[4 * (v >> 1) + threadIdx.x] = packed[4 * (v >> 1) + threadIdx.x];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        partials[c] = t;
        const unsigned n = (unsigned)(d.chunk_base[v + 1] - d.chunk_base[v]);
        last = atomic_add_acq_rel_gpu(&tickets[v], 1u) == n - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        double t = 0.0;
        for (int k = d.chunk_base[v]; k < d.chunk_base[v + 1]; ++k) t += partials[k];
        records[4 * (v >> 1) + 2 + (v & 1)] = t;
        tickets[v] = 0u;
    }
}

}  // namespace

int nccl_available() { return nccl().ok ? 1 : 0; }

}  // namespace gnsb

namespace {
gnsb_status xfail(gnsb_status s, const std::string& m) {
    gnsb::set_error(m);
    return s;
}
gnsb_status nccl_fail(int r, const char* where) {
    const auto& api = gnsb::nccl();
    std::string m = std::string("nccl: ") + where + ": " + (api.get_error_string ? api.get_error_string(r) : "error");
    return xfail(GNSB_ENCCL, m);
}
}  // namespace

extern "C" {

int32_t gnsb_nccl_available(void) { return gnsb::nccl_available(); }

gnsb_status gnsb_nccl_get_unique_id(void* id128) {
    const auto& api = gnsb::nccl();
    if (!api.ok) return xfail(GNSB_ENCCL, "nccl: libnccl.so.2 not found");
    if (!id128) return xfail(GNSB_EINVAL, "nccl: null id buffer");
    gnsb::nccl_unique_id id;
    if (int r = api.get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof(id));
    return GNSB_OK;
}

gnsb_status gnsb_nccl_comm_init_rank(void** comm, int32_t nranks, const void* id128, int32_t rank) {
    const auto& api = gnsb::nccl();
    if (!api.ok) return xfail(GNSB_ENCCL, "nccl: libnccl.so.2 not found");
    if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return xfail(GNSB_EINVAL, "nccl: invalid arguments");
    gnsb::nccl_unique_id id;
    std::memcpy(&id, id128, sizeof(id));
    if (int r = api.comm_init_rank(comm, nranks, id, rank)) return nccl_fail(r, "ncclCommInitRank");
    return GNSB_OK;
}

gnsb_status gnsb_nccl_comm_destroy(void* comm) {
    const auto& api = gnsb::nccl();
    if (!api.ok) return xfail(GNSB_ENCCL, "nccl: libnccl.so.2 not found");
    if (comm)
        if (int r = api.comm_destroy(comm)) return nccl_fail(r, "ncclCommDestroy");
    return GNSB_OK;
}

}  // extern "C"

namespace {
// widths2: (p0, p1) widths per layer; p1 may be 0 (a bias-less layer)
gnsb_status bucket_layout(const int64_t* widths2, int32_t n_layers, int with_records, gnsb::BucketLayout* out) {
    if (n_layers < 1 || n_layers > gnsb::kMaxBucketLayers || !widths2)
        return xfail(GNSB_EINVAL, "gns: invalid bucket description (1..256 layers)");
    gnsb::BucketDesc& d = out->d;
    d = gnsb::BucketDesc{};
    int64_t n = 0, chunks = 0;
    for (int32_t v = 0; v < 2 * n_layers; ++v) {
        const int64_t w = widths2[v];
        if (w < 0 || ((v & 1) == 0 && w < 1))
            return xfail(GNSB_EINVAL, "gns: bucket widths must be positive (p1 may be 0)");
        d.offset[v] = n;
        d.width[v] = w;
        d.chunk_base[v] = (int32_t)chunks;
        n += w;
        chunks += w > 0 ? (w + gnsb::kChunk - 1) / gnsb::kChunk : 1;
        if (chunks > (1 << 30)) return xfail(GNSB_EINVAL, "gns: bucket too large");
    }
    d.chunk_base[2 * n_layers] = (int32_t)chunks;
    d.nvec = 2 * n_layers;
    d.with_records = with_records ? 1 : 0;
    d.total = n;
    d.rec_n = with_records ? 4 * (int64_t)n_layers : 0;
    // the workspace is sized for records either way, so one buffer serves both twins
    const size_t packed = (size_t)(4 * (int64_t)n_layers + n) * sizeof(double);
    out->off_partials = (packed + 255) / 256 * 256;
    out->off_tickets = out->off_partials + (size_t)chunks * sizeof(double);
    out->bytes = out->off_tickets + (size_t)(2 * n_layers) * sizeof(unsigned);
    return GNSB_OK;
}

gnsb_status bucket_check(void* grads, gnsb_dtype grad_dt, const double* records, int with_records, void* ws,
                         size_t ws_bytes, const gnsb::BucketLayout& lay) {
    if (!grads) return xfail(GNSB_EINVAL, "gns: null gradient bucket");
    if (grad_dt != GNSB_F32 && grad_dt != GNSB_F64) return xfail(GNSB_EINVAL, "gns: gradient bucket must be fp32 or fp64");
    if (with_records && !records) return xfail(GNSB_EINVAL, "gns: null records");
    if (!ws || ws_bytes < lay.bytes)
        return xfail(GNSB_EINVAL, "gns: exchange workspace too small (query gnsb_exchange_workspace_size)");
    return GNSB_OK;
}

gnsb_status launch_pack(const void* grads, gnsb_dtype dt, const double* records, const gnsb::BucketLayout& lay,
                        void* ws, cudaStream_t st) {
    const int64_t n = gnsb::packed_count(lay.d);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    double* packed = static_cast<double*>(ws);
    if (dt == GNSB_F32)
        gnsb::bucket_pack_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(grads), records, lay.d, packed);
    else
        gnsb::bucket_pack_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(grads), records, lay.d, packed);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GNSB_OK : xfail(GNSB_ECUDA, std::string("cuda: exchange pack: ") + cudaGetErrorString(e));
}

gnsb_status launch_unpack(void* grads, gnsb_dtype dt, double* records, const gnsb::BucketLayout& lay, void* ws,
                          cudaStream_t st) {
    unsigned char* base = static_cast<unsigned char*>(ws);
    const double* packed = reinterpret_cast<const double*>(base);
    double* partials = reinterpret_cast<double*>(base + lay.off_partials);
    unsigned* tickets = reinterpret_cast<unsigned*>(base + lay.off_tickets);
    const int grid = lay.d.chunk_base[lay.d.nvec];
    if (dt == GNSB_F32)
        gnsb::bucket_unpack_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(grads), records, lay.d, packed,
                                                                partials, tickets);
    else
        gnsb::bucket_unpack_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(grads), records, lay.d, packed,
                                                                 partials, tickets);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GNSB_OK
                            : xfail(GNSB_ECUDA, std::string("cuda: exchange unpack: ") + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

gnsb_status gnsb_exchange_workspace_size(const int64_t* widths2, int32_t n_layers, size_t* bytes) {
    if (!bytes) return xfail(GNSB_EINVAL, "gns: null size output");
    gnsb::BucketLayout lay;
    if (gnsb_status s = bucket_layout(widths2, n_layers, 1, &lay)) return s;
    *bytes = lay.bytes;
    return GNSB_OK;
}

gnsb_status gnsb_exchange_pack(const void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                               const double* records, void* ws, size_t ws_bytes, void* stream) {
    gnsb::BucketLayout lay;
    if (gnsb_status s = bucket_layout(widths2, n_layers, records != nullptr, &lay)) return s;
    if (gnsb_status s = bucket_check(const_cast<void*>(grads), grad_dt, records, records != nullptr, ws, ws_bytes, lay))
        return s;
    return launch_pack(grads, grad_dt, records, lay, ws, static_cast<cudaStream_t>(stream));
}

gnsb_status gnsb_exchange_unpack(void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                                 double* records, void* ws, size_t ws_bytes, void* stream) {
    gnsb::BucketLayout lay;
    if (gnsb_status s = bucket_layout(widths2, n_layers, records != nullptr, &lay)) return s;
    if (gnsb_status s = bucket_check(grads, grad_dt, records, records != nullptr, ws, ws_bytes, lay)) return s;
    return launch_unpack(grads, grad_dt, records, lay, ws, static_cast<cudaStream_t>(stream));
}

gnsb_status gnsb_allreduce_buckets(void* grads, gnsb_dtype grad_dt, const int64_t* widths2, int32_t n_layers,
                                   double* records, void* ws, size_t ws_bytes, void* nccl_comm, void* stream) {
    const auto& api = gnsb::nccl();
    gnsb::BucketLayout lay;
    const int with_records = records != nullptr;
    if (gnsb_status s = bucket_layout(widths2, n_layers, with_records, &lay)) return s;
    if (gnsb_status s = bucket_check(grads, grad_dt, records, with_records, ws, ws_bytes, lay)) return s;
    if (nccl_comm && !api.ok) return xfail(GNSB_ENCCL, "nccl: libnccl.so.2 not found");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (gnsb_status s = launch_pack(grads, grad_dt, records, lay, ws, st)) return s;
    if (nccl_comm)  // without a communicator: one rank, nothing to sum
        if (int r = api.all_reduce(ws, ws, (size_t)gnsb::packed_count(lay.d), gnsb::kNcclFloat64, gnsb::kNcclSum,
                                   nccl_comm, st))
            return nccl_fail(r, "ncclAllReduce");
    return launch_unpack(grads, grad_dt, records, lay, ws, st);
}

}  // extern "C"

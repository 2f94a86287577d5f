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
struct BucketDesc {
    int64_t offset[kMaxBucketLayers];
    int64_t width[kMaxBucketLayers];
};

// records[l][2 + p] = ||bucket vector (l, p)||^2, one CTA per vector
template <typename V>
__global__ void __launch_bounds__(256) bucket_sqnorm_kernel(const V* grads, const __grid_constant__ BucketDesc d,
                                                            double* records) {
    __shared__ double red[8];
    const int l = blockIdx.x >> 1, p = blockIdx.x & 1;
    const int64_t w = d.width[l];
    const V* v = grads + d.offset[l] + p * w;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {
        const double x = (double)v[i];
        acc = fma(x, x, acc);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        records[l * 4 + 2 + p] = t;
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

gnsb_status gnsb_allreduce_buckets(void* grads, gnsb_dtype grad_dt, const int64_t* widths_host, int32_t n_layers,
                                   double* records, int32_t with_records, void* nccl_comm, void* stream) {
    const auto& api = gnsb::nccl();
    if (n_layers < 1 || n_layers > gnsb::kMaxBucketLayers || !grads || !widths_host)
        return xfail(GNSB_EINVAL, "gns: invalid bucket description (1..256 layers)");
    if (grad_dt != GNSB_F32 && grad_dt != GNSB_F64) return xfail(GNSB_EINVAL, "gns: gradient bucket must be fp32 or fp64");
    if (with_records && !records) return xfail(GNSB_EINVAL, "gns: null records");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    gnsb::BucketDesc d{};
    int64_t n = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
        if (widths_host[l] < 1) return xfail(GNSB_EINVAL, "gns: bucket widths must be positive");
        d.offset[l] = n;
        d.width[l] = widths_host[l];
        n += 2 * widths_host[l];
    }
    if (nccl_comm) {  // without a communicator: one rank, nothing to sum
        if (!api.ok) return xfail(GNSB_ENCCL, "nccl: libnccl.so.2 not found");
        if (int r = api.all_reduce(grads, grads, (size_t)n, grad_dt == GNSB_F32 ? gnsb::kNcclFloat32 : gnsb::kNcclFloat64,
                                   gnsb::kNcclSum, nccl_comm, st))
            return nccl_fail(r, "ncclAllReduce(grads)");
        if (with_records)
            if (int r = api.all_reduce(records, records, (size_t)n_layers * 4, gnsb::kNcclFloat64, gnsb::kNcclSum,
                                       nccl_comm, st))
                return nccl_fail(r, "ncclAllReduce(records)");
    }
    if (!with_records) return GNSB_OK;
    if (grad_dt == GNSB_F32)
        gnsb::bucket_sqnorm_kernel<float><<<2 * n_layers, 256, 0, st>>>(static_cast<const float*>(grads), d, records);
    else
        gnsb::bucket_sqnorm_kernel<double><<<2 * n_layers, 256, 0, st>>>(static_cast<const double*>(grads), d, records);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return xfail(GNSB_ECUDA, std::string("cuda: allreduce_buckets: ") + cudaGetErrorString(e));
    return GNSB_OK;
}

}  // extern "C"

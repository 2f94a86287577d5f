// nvls_probe.cu — does this box expose NVLink-SHARP multicast (experiment only)?
// Creates a one-device multicast object, binds device memory, maps the
// multicast address, and runs multimem.red.add (fp32 and fp64) / multimem.ld_reduce
// against it; prints what worked.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                                        \
    do {                                                                             \
        CUresult r = (x);                                                            \
        if (r != CUDA_SUCCESS) {                                                     \
            const char* s = nullptr;                                                 \
            cuGetErrorString(r, &s);                                                 \
            std::printf("FAIL %s: %d %s\n", #x, (int)r, s ? s : "?");                \
            return 1;                                                                \
        }                                                                            \
    } while (0)

__global__ void red_kernel(float* mc_f, double* mc_d, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float v = 1.0f + i;
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc_f + i), "f"(v) : "memory");
    const double d = 0.5 + i;
    asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mc_d + i), "d"(d) : "memory");
}

__global__ void ldred_kernel(const float* mc_f, float* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc_f + i) : "memory");
    out[i] = v;
}

#ifndef NDEV
#define NDEV 1
#endif
int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    int mc = 0, fab = 0, posix = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
    std::printf("multicast_supported=%d fabric_handles=%d posix_fd_handles=%d\n", mc, fab, posix);
    if (!mc) return 0;
    CUmulticastObjectProp mp = {};
    size_t gran = 0;
    CUmemGenericAllocationHandle mch;
    bool made = false;
    const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                                CU_MEM_HANDLE_TYPE_NONE};
    for (int ti = 0; ti < 3 && !made; ++ti) {
        mp = CUmulticastObjectProp{};
        mp.numDevices = NDEV;
        mp.handleTypes = types[ti];
        mp.size = 1 << 21;
        CUresult r = cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        if (r != CUDA_SUCCESS) {
            std::printf("granularity(handle type %d): %d\n", (int)types[ti], (int)r);
            continue;
        }
        mp.size = (mp.size + gran - 1) / gran * gran;
        r = cuMulticastCreate(&mch, &mp);
        std::printf("cuMulticastCreate(numDevices=%d, handle type %d, size %zu): %d\n", NDEV, (int)types[ti], mp.size, (int)r);
        made = r == CUDA_SUCCESS;
    }
    if (!made) return 1;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(mp.handleTypes);
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, mp.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem, 0, mp.size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, mp.size, gran, 0, 0));
    CK(cuMemMap(uc, mp.size, 0, mem, 0));
    CK(cuMemAddressReserve(&mcp, mp.size, gran, 0, 0));
    CK(cuMemMap(mcp, mp.size, 0, mch, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = 0;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, mp.size, &ad, 1));
    CK(cuMemSetAccess(mcp, mp.size, &ad, 1));
    const int n = 1024;
    CK(cuMemsetD8(uc, 0, mp.size));
    float* mf = reinterpret_cast<float*>(mcp);
    double* md = reinterpret_cast<double*>(mcp + 8192);
    red_kernel<<<n / 256, 256>>>(mf, md, n);
    red_kernel<<<n / 256, 256>>>(mf, md, n);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("multimem.red launch: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float hf[4];
    double hd[4];
    CK(cuMemcpyDtoH(hf, uc, sizeof(hf)));
    CK(cuMemcpyDtoH(hd, uc + 8192, sizeof(hd)));
    std::printf("f32 after 2 reds: %g %g %g %g (expect 2 4 6 8)\n", hf[0], hf[1], hf[2], hf[3]);
    std::printf("f64 after 2 reds: %g %g %g %g (expect 1 3 5 7)\n", hd[0], hd[1], hd[2], hd[3]);
    float* out;
    cudaMalloc(&out, n * sizeof(float));
    ldred_kernel<<<n / 256, 256>>>(mf, out, n);
    e = cudaDeviceSynchronize();
    std::printf("multimem.ld_reduce: %s\n", cudaGetErrorString(e));
    cudaMemcpy(hf, out, sizeof(hf), cudaMemcpyDeviceToHost);
    std::printf("ld_reduce: %g %g %g %g\n", hf[0], hf[1], hf[2], hf[3]);
    return 0;
}

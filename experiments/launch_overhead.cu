// launch_overhead.cu — event-timed cost of an empty persistent launch (experiment only).
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void empty_kernel(int* p) {
    extern __shared__ int sm[];
    if (p && threadIdx.x == 0 && blockIdx.x == 100000) p[0] = sm[0];
}

extern "C" int run_empty(int coop, int threads, int smem, int reps, int back2back, float* ms, void* flush, size_t flush_bytes) {
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < reps; ++r) {
        if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
        cudaEventRecord(a);
        for (int k = 0; k < back2back; ++k) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t;
        cudaEventElapsedTime(&t, a, b);
        if (r > 0) tot += t;
    }
    *ms = tot / (reps - 1);
    return cudaGetLastError();
}

__global__ void marker_kernel(unsigned long long* p) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *p = t;
}
extern "C" int marker(void* p, void* stream) {
    marker_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)p);
    return cudaGetLastError();
}

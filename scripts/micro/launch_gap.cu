// back-to-back dependent kernel launches on one stream: plain vs PDL
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tiny(int* p, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
__global__ void k_small(float* a, int n, int pdl) {  // ~1M elements touch
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] += 1.f;
}
int main() {
    int* p; cudaMalloc(&p, 4); cudaMemset(p, 0, 4);
    float* a; int n = 1 << 20; cudaMalloc(&a, n * 4); cudaMemset(a, 0, n * 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 4; ++mode) {
        const bool pdl = mode & 1, small = mode & 2;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0, s);
            for (int i = 0; i < 200; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = small ? dim3(592) : dim3(1);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                if (small) cudaLaunchKernelEx(&cfg, k_small, a, n, (int)pdl);
                else cudaLaunchKernelEx(&cfg, k_tiny, p, (int)pdl);
            }
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("%s %s: %.2f us per launch\n", small ? "small(592x256, 4MB)" : "tiny(1x256)", pdl ? "PDL " : "plain", ms * 1e3 / 200);
        }
    }
    // host round trip: launch + memcpy D2H + sync
    int h; 
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, s);
        for (int i = 0; i < 50; ++i) {
            k_tiny<<<1, 256, 0, s>>>(p, 0);
            cudaMemcpyAsync(&h, p, 4, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("launch+D2H+sync round trip: %.2f us\n", ms * 1e3 / 50);
    }
    return 0;
}

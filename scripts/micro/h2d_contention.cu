// does a concurrent pinned H2D copy slow a memory-bound / latency-bound kernel?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_sum(const double* a, size_t n, double* out) {
    double s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += a[i];
    if (s == 12345.678) out[0] = s;
}
__global__ void k_chain(const unsigned* nxt, int steps, unsigned* out) {  // dependent loads
    unsigned p = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < steps; ++i) p = nxt[p];
    if (p == 0xFFFFFFFF) out[0] = p;
}
int main() {
    size_t n = 3u << 20;  // 24 MB of doubles
    double *a, *o; cudaMalloc(&a, n * 8); cudaMalloc(&o, 8); cudaMemset(a, 0, n * 8);
    unsigned *nx, *uo; size_t m = 1 << 22; cudaMalloc(&nx, m * 4); cudaMalloc(&uo, 4);
    unsigned* h = (unsigned*)malloc(m * 4); for (size_t i = 0; i < m; ++i) h[i] = (unsigned)((i * 2654435761u) % m);
    cudaMemcpy(nx, h, m * 4, cudaMemcpyHostToDevice);
    size_t hb = 64u << 20; char* hp; cudaMallocHost(&hp, hb); char* dp; cudaMalloc(&dp, hb);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int withcopy = 0; withcopy < 2; ++withcopy) {
        for (int rep = 0; rep < 3; ++rep) {
            if (withcopy) cudaMemcpyAsync(dp, hp, hb, cudaMemcpyHostToDevice, s2);
            cudaEventRecord(e0, s1);
            for (int k = 0; k < 10; ++k) k_sum<<<148 * 8, 256, 0, s1>>>(a, n, o);
            cudaEventRecord(e1, s1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaEvent_t e2, e3; cudaEventCreate(&e2); cudaEventCreate(&e3);
            cudaEventRecord(e2, s1);
            for (int k = 0; k < 10; ++k) k_chain<<<148 * 4, 256, 0, s1>>>(nx, 64, uo);
            cudaEventRecord(e3, s1);
            cudaEventSynchronize(e3);
            float ms2; cudaEventElapsedTime(&ms2, e2, e3);
            cudaDeviceSynchronize();
            if (rep == 2) printf("%s: k_sum(24MB) %.2f us, k_chain %.2f us\n", withcopy ? "with 64MB H2D" : "alone", ms * 100, ms2 * 100);
        }
    }
    return 0;
}

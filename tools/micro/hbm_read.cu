// Pure-read HBM bandwidth ceiling (the weight stream of a batch-1 forward is read-only).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a hbm_read.cu -o hbm_read
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void rd(const uint4* __restrict__ p, size_t n, unsigned* out) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].w;
    }
    if (acc == 0x12345678) *out = acc;
}
__global__ void cp(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}
int main(int argc, char** argv) {
    const size_t bytes = argc > 1 ? (size_t)atol(argv[1]) << 20 : (size_t)4 << 30, n = bytes / 16;
    uint4 *a, *b;
    unsigned* o;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes / 2);
    cudaMalloc(&o, 4);
    cudaMemset(a, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bpsm : {2, 4, 8}) {
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(e0);
            rd<<<sms * bpsm, 256>>>(a, n, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("read-only LDG.128 x8, %d CTAs/SM: %.0f GB/s\n", bpsm, bytes / (best * 1e-3) / 1e9);
    }
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0);
        cp<<<sms * 8, 256>>>(a, b, n / 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    printf("copy (read+write counted): %.0f GB/s\n", bytes / (best * 1e-3) / 1e9);
    return 0;
}

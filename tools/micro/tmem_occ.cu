// Does a kernel that allocates TMEM (tcgen05.alloc) get more than one CTA per SM? Occupancy API answer and the
// observed co-residency (%smid + globaltimer per CTA) for 296 CTAs of 192 threads and 60 KB of shared memory.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tmem_occ.cu -o tmem_occ
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <bool TMEM>
__global__ void __launch_bounds__(192) k(unsigned long long* out, int spin_us) {
    extern __shared__ uint8_t sm[];
    __shared__ uint32_t slot;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (TMEM && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < (unsigned long long)spin_us * 1000);
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        out[blockIdx.x * 3] = smid;
        out[blockIdx.x * 3 + 1] = t0;
        out[blockIdx.x * 3 + 2] = t1;
        sm[0] = 1;
    }
    __syncthreads();
    if (TMEM && threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
}
template <bool TMEM>
void run(unsigned long long* d, unsigned long long* h) {
    const int smem = 60 * 1024;
    cudaFuncSetAttribute(k<TMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<TMEM>, 192, smem);
    k<TMEM><<<296, 192, smem>>>(d, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 296 * 3 * 8, cudaMemcpyDeviceToHost);
    unsigned long long s0 = ~0ull, e1 = 0;
    int overlap = 0;
    for (int i = 0; i < 296; ++i) {
        s0 = h[3 * i + 1] < s0 ? h[3 * i + 1] : s0;
        e1 = h[3 * i + 2] > e1 ? h[3 * i + 2] : e1;
        for (int j = 0; j < i; ++j)
            if (h[3 * j] == h[3 * i] && h[3 * j + 1] < h[3 * i + 2] && h[3 * i + 1] < h[3 * j + 2]) ++overlap;
    }
    printf("%s: occupancy API %d blocks/SM; 296 CTAs x 20 us took %.1f us; co-resident CTA pairs on one SM: %d  %s\n",
           TMEM ? "with tcgen05.alloc" : "no TMEM", nb, (e1 - s0) / 1e3, overlap, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    unsigned long long *d, h[296 * 3];
    cudaMalloc(&d, sizeof h);
    run<false>(d, h);
    run<true>(d, h);
    return 0;
}

// tcgen05.mma issue/execute rate for the attention shapes: one CTA per SM, one thread issues ITERS MMAs
// back to back (kind::f16, bf16 in, f32 accumulate, M = 128, K = 16), then commits and waits. Reports
// cycles per MMA and the implied dense TFLOP/s over 148 SMs at the measured clock.
//   SS: A and B from shared memory (K-major SW128), N = 64 / 128 / 256
//   TS: A from TMEM (the P . V shape: A = 128 x 16 bf16 in TMEM, B = V MN-major), N = 128
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a umma_rate.cu -o umma_rate
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k(uint32_t a) {
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t a, uint32_t lbo) {
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24) |
           (b_mn ? (1u << 16) : 0u);
}

template <int MODE, int N>  // MODE 0: SS, 1: TS
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = su(base), b = a + 16384;
        const uint32_t id = idesc(128, N, MODE == 1);
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
        for (int i = 0; i < iters; ++i) {
            const int kk = i & 7;
            if (MODE == 0) {
                const uint64_t da = desc_k(a + (kk >> 2) * 16384 / 2 + (kk & 3) * 32);
                const uint64_t db = desc_k(b + (kk >> 2) * 16384 + (kk & 3) * 32);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                             ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(1));
            } else {
                const uint64_t db = desc_mn(b + (kk & 3) * 2048, 8192);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm), "r"(tm + 256 + kk * 8), "l"(db), "r"(id), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
        uint32_t d = 0;
        while (!d)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(d) : "r"(su(&bar)) : "memory");
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int MODE, int N>
void run(unsigned long long* d_out) {
    auto k = rate<MODE, N>;
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<148, 128, smem>>>(iters, d_out);
    cudaEventRecord(e0);
    k<<<148, 128, smem>>>(iters, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 128 * N * 16 * iters * 148;
    printf("%s M=128 N=%3d K=16: %.1f cycles/MMA, %.0f TFLOP/s (event-timed, 148 SMs)  %s\n", MODE ? "TS" : "SS", N,
           (double)cyc / iters, flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    run<0, 64>(d);
    run<0, 128>(d);
    run<0, 256>(d);
    run<1, 64>(d);
    run<1, 128>(d);
    run<1, 256>(d);
    return 0;
}

// Weight-stream ceiling through shared memory with LSU copies (cp.async.cg 16 B, "LDGSTS") instead of TMA:
// 4 producer warps fill a STAGES-deep ring of 128 x 64 bf16 tiles (SW128 layout, 16 KB) read from a row-major
// [N][K] matrix; each producer thread keeps DEPTH commit groups in flight, waits for the oldest, fences the
// generic->async proxy and arrives on that stage's full barrier. Consumer: a releasing thread (MODE 0) or a
// tcgen05.mma issuer over the weight tile and a 64-token activation tile (MODE 1, activation also by cp.async).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a cpasync_stream.cu -o cpasync_stream
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    uint32_t d = 0;
    while (!d)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(d) : "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <int DEPTH>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH) : "memory"); }

constexpr int PRODUCERS = 128;
template <int MODE, int DEPTH>
__global__ void stream(const uint8_t* __restrict__ w, const uint8_t* __restrict__ act, int K, int n_tiles, int kb,
                       int stages) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t WB = 16384, SB = MODE == 1 ? WB + 8192 : WB;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + stages * SB);
    uint64_t* empty = full + stages;
    __shared__ uint32_t tslot;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(PRODUCERS));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (MODE == 1 && threadIdx.x >= PRODUCERS) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int per = (n_tiles + gridDim.x - 1) / gridDim.x;
    const int total = per * kb;
    if (threadIdx.x < PRODUCERS) {
        const int tid = threadIdx.x;
        auto issue = [&](int it) {
            const int s = it % stages;
            const int t = blockIdx.x + (it / kb) * gridDim.x, k = it % kb;
            const uint32_t base = su(ring + s * SB);
            if (t < n_tiles) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {  // 1024 16-byte chunks: row r = i / 8, chunk c = i % 8 (SW128)
                    const int i = tid + j * PRODUCERS, r = i >> 3, c = i & 7;
                    cp16(base + r * 128 + ((c ^ (r & 7)) << 4), w + ((size_t)(t * 128 + r) * K + k * 64 + c * 8) * 2);
                }
                if (MODE == 1) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {  // 64 x 64 activation tile
                        const int i = tid + j * PRODUCERS, r = i >> 3, c = i & 7;
                        cp16(base + WB + r * 128 + ((c ^ (r & 7)) << 4), act + ((size_t)r * K + k * 64 + c * 8) * 2);
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto publish = [&](int it) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[it % stages])) : "memory");
        };
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            wait(&empty[s], ((it / stages) & 1) ^ 1);
            issue(it);
            if (it >= DEPTH) {
                wait_group<DEPTH>();
                publish(it - DEPTH);
            }
        }
        wait_group<0>();
        for (int it = total > DEPTH ? total - DEPTH : 0; it < total; ++it) publish(it);
    } else if (threadIdx.x == PRODUCERS) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            wait(&full[s], (it / stages) & 1);
            if (MODE == 1) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t wa = su(ring + s * SB), aa = wa + WB;
                for (int k = 0; k < 4; ++k) {
                    auto desc = [](uint32_t a) {
                        return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
                               ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
                    };
                    const uint32_t acc = (it | k) != 0;
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                 ::"r"(tslot), "l"(desc(wa + k * 32)), "l"(desc(aa + k * 32)), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&empty[s])) : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
            }
        }
    }
    if (MODE == 1) {
        __syncthreads();
        if (threadIdx.x >= PRODUCERS) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tslot));
        }
    }
}

template <int MODE, int DEPTH>
void run(const uint8_t* w, const uint8_t* act, int N, int K, int cps, int stages) {
    const int kb = K / 64, n_tiles = N / 128;
    const size_t smem = 1024 + stages * (MODE == 1 ? 24576 : 16384) + 256;
    if (smem * cps > 232448) return;
    auto k = stream<MODE, DEPTH>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0);
        k<<<148 * cps, PRODUCERS + 32, smem>>>(w, act, K, n_tiles, kb, stages);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    printf("cp.async %s: %d CTAs/SM x %d stages, %d groups in flight: %.0f GB/s of weights  %s\n",
           MODE == 1 ? "weights + activation + mma" : "weights only", cps, stages, DEPTH + 1,
           (double)N * K * 2 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int N = 37888, K = 3584;
    uint8_t *w, *act;
    cudaMalloc(&w, (size_t)N * K * 2);
    cudaMemset(w, 1, (size_t)N * K * 2);
    cudaMalloc(&act, (size_t)64 * K * 2);
    cudaMemset(act, 1, (size_t)64 * K * 2);
    run<0, 3>(w, act, N, K, 2, 4);
    run<0, 5>(w, act, N, K, 2, 6);
    run<0, 7>(w, act, N, K, 1, 8);
    run<0, 11>(w, act, N, K, 1, 12);
    run<1, 3>(w, act, N, K, 2, 4);
    run<1, 2>(w, act, N, K, 2, 4);
    run<1, 7>(w, act, N, K, 1, 8);
    return 0;
}

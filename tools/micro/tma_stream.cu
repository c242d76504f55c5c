// Weight-stream ceiling through shared memory: one producer thread per CTA fills a STAGES-deep ring either with
// TMA 2D tensor boxes (128 rows x 64 cols of a [N][K] bf16 matrix: 128 row segments 7 KB apart) or with 1-D bulk
// copies of contiguous 16 KB blocks (a pre-tiled layout); a consumer thread releases slots (no math).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    uint32_t d = 0;
    while (!d)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(d) : "r"(su(b)), "r"(ph) : "memory");
}
template <int MODE>
__global__ void stream(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap ta, const uint8_t* w,
                       int n_tiles, int kb, int stages) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t SB = (MODE == 2 || MODE == 3 || MODE == 5) ? 16384 + 8192 : 16384;  // stage bytes
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + stages * SB);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int total = ((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * kb;
    if (threadIdx.x == 0) {
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            wait(&empty[s], ((it / stages) & 1) ^ 1);
            const int t = blockIdx.x + (it / kb) * gridDim.x, k = it % kb;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(SB) : "memory");
            if (MODE == 2 || MODE == 3 || MODE == 5)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(su(ring + s * SB + 16384)), "l"((uint64_t)&ta), "r"(su(&full[s])), "r"(k * 64), "r"(0) : "memory");
            if (MODE >= 4)  // k-major pre-tiled layout: at step k every CTA reads a neighbour of the same 16 KB row
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                             ::"r"(su(ring + s * SB)), "l"(w + ((size_t)k * n_tiles + t) * 16384), "r"(su(&full[s])) : "memory");
            else if (MODE == 0 || MODE >= 2)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(su(ring + s * SB)), "l"((uint64_t)&tm), "r"(su(&full[s])), "r"(k * 64), "r"(t * 128) : "memory");
            else
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                             ::"r"(su(ring + s * SB)), "l"(w + ((size_t)t * kb + k) * 16384), "r"(su(&full[s])) : "memory");
        }
    } else if (threadIdx.x == 32 && MODE != 3 && MODE != 5) {
        for (int it = 0; it < total; ++it) {
            const int s = it % stages;
            wait(&full[s], (it / stages) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
        }
    }
    if ((MODE == 3 || MODE == 5) && threadIdx.x >= 32) {  // warp 1: TMEM + the swapped GEMM's MMAs (M=128 weights, N=64 tokens)
        __shared__ uint32_t tslot;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (threadIdx.x == 32) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            for (int it = 0; it < total; ++it) {
                const int s = it % stages;
                wait(&full[s], (it / stages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t wa = su(ring + s * SB), aa = wa + 16384;
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
            }
        }
        __syncwarp();
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tslot));
    }
}
__global__ void fill_rand(uint32_t* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ 0x9E3779B9u;
        x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
        p[i] = (x & 0x3FFF3FFFu) | 0x3C003C00u;  // small bf16 pairs, random mantissas and signs off
    }
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    const int N = 37888 * (argc > 1 ? atoi(argv[1]) : 1), K = 3584, kb = K / 64, n_tiles = N / 128;
    const size_t bytes = (size_t)N * K * 2;
    uint8_t* w;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 1, bytes);
    const bool rnd = argc > 2;
    if (rnd) fill_rand<<<1184, 256>>>((uint32_t*)w, bytes / 4);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}, str[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    uint8_t* act;
    cudaMalloc(&act, (size_t)64 * K * 2);
    cudaMemset(act, 1, (size_t)64 * K * 2);
    if (rnd) fill_rand<<<64, 256>>>((uint32_t*)act, (size_t)64 * K / 2);
    CUtensorMap ta;
    const cuuint64_t adims[2] = {(cuuint64_t)K, 64}, astr[1] = {(cuuint64_t)K * 2};
    const cuuint32_t abox[2] = {64, 64};
    ((Enc)fn)(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = (argc > 3 ? atoi(argv[3]) : 0); mode < 6; ++mode)
        for (int cfg = 0; cfg < 4; ++cfg) {
            const int cps = cfg < 2 ? 2 : 1, stages = cfg == 0 ? 4 : cfg == 1 ? 6 : cfg == 2 ? 8 : 12;
            const size_t smem = 1024 + stages * ((mode == 2 || mode == 3 || mode == 5) ? 24576 : 16384) + 256;
            if (smem > 232448) continue;
            auto k = mode == 0 ? stream<0> : mode == 1 ? stream<1> : mode == 2 ? stream<2> : mode == 3 ? stream<3> : mode == 4 ? stream<4> : stream<5>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(e0);
                k<<<148 * cps, 64, smem>>>(tm, ta, w, n_tiles, kb, stages);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%s: %d CTAs/SM x %d stages: %.0f GB/s of weights  %s\n",
                   mode == 0 ? "TMA 2-D box" : mode == 1 ? "bulk 1-D contiguous"
                             : mode == 2 ? "TMA box + 8 KB activation box" : mode == 3 ? "box + activation + 4 tcgen05.mma/stage"
                             : mode == 4 ? "bulk 1-D k-major tiles" : "bulk k-major + activation + mma",
                   cps, stages, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}

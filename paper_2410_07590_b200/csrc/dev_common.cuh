// Launch plumbing shared by every kernel of the engine: Programmatic Dependent Launch (PDL).
//
// Every kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization. A kernel calls
// pdl_launch() at its start so the NEXT kernel's CTAs may be scheduled as SMs free up, and pdl_wait()
// before it touches anything an earlier kernel produced (griddepcontrol.wait returns once the preceding
// grid has completed and its writes are visible; since every grid waits on its predecessor, all earlier
// grids are complete too). Work that does not depend on earlier kernels — barrier init, TMEM alloc,
// tensor-map prefetch and, in the GEMM, the TMA loads of WEIGHT tiles — runs before the wait and so
// overlaps the previous kernel's tail.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "tkv_internal.h"

namespace tkv {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Kernel timeline (tkv_kernel_timeline, armed only by measurement passes): slot[0] = atomicMin of the globaltimer when a
// CTA is past griddepcontrol.wait (the predecessor grid has completed), slot[1] = atomicMax when a warp finishes.
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_wait(unsigned long long* tl) {
    if (tl && threadIdx.x == 0) atomicMin(tl, gtimer_ns());
}
__device__ __forceinline__ void tl_exit(unsigned long long* tl) {
    if (tl && (threadIdx.x & 31) == 0) atomicMax(tl + 1, gtimer_ns());
}

// RMSNorm folded into the consumer (numerics.cpp:84-101): the producer of x writes xb = x * w and per-block
// partial sums of squares ssp[t][0..nb) (fixed order, deterministic); a consumer of a linear map of xb
// multiplies by this per-row scale, since rms(x) . W = scale(x) * ((x * w) . W).
__device__ __forceinline__ float row_scale(const float* __restrict__ ssp, int nb, int64_t t, int hidden, float eps) {
    float ss = 0.f;
    const float* p = ssp + t * nb;
    if (nb <= 32) {  // every load in flight at once (one memory round trip), summed in fixed order
        float v[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) v[b] = b < nb ? p[b] : 0.f;
#pragma unroll
        for (int b = 0; b < 32; ++b) ss += v[b];
    } else {
        for (int b = 0; b < nb; ++b) ss += p[b];
    }
    return 1.0f / sqrtf(ss / (float)hidden + eps);
}

// cudaLaunchKernelEx with the PDL attribute (when enabled process-wide, see pdl_enabled()).
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TKV_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace tkv

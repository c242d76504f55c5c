// SIMT GEMM with split-K partial outputs: partial[z][m][n] = sum_{k in split z} A[m][k] * W[n][k].
// This is the fp32 path's projection GEMM (fp32 inputs, no TF32, so the 1e-4 parity budget holds
// against the f64 reference matmul, src/numerics.cpp:8-29) and the bf16 comparison kernel behind
// TKV_FLAG_SIMT_GEMM. The bf16 product path uses the tcgen05 kernel in gemm_tc.cu.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256;

__device__ __forceinline__ float ld(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }

template <typename T>
__global__ void __launch_bounds__(THREADS) gemm_simt_kernel(const T* __restrict__ A, int lda, const T* __restrict__ W,
                                                            int M, int N, int K, float* __restrict__ partial,
                                                            int kchunk) {
    pdl_launch();
    pdl_wait();
    __shared__ float As[BK][BM + 4];
    __shared__ float Ws[BK][BN + 4];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN, z = blockIdx.z;
    const int k_begin = z * kchunk, k_end = min(K, k_begin + kchunk);
    float acc[4][4] = {};
    const int lr = tid / 4, lk = (tid % 4) * 4;  // loader: row lr, 4 consecutive k
    for (int k0 = k_begin; k0 < k_end; k0 += BK) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = k0 + lk + e;
            const bool kin = k < k_end;
            As[lk + e][lr] = (kin && m0 + lr < M) ? ld(A, (int64_t)(m0 + lr) * lda + k) : 0.f;
            Ws[lk + e][lr] = (kin && n0 + lr < N) ? ld(W, (int64_t)(n0 + lr) * K + k) : 0.f;
        }
        __syncthreads();
        // two-level summation: a fresh 16-term partial per k-tile, then one add into the running sum,
        // so rounding error grows with 16 + K/16 instead of K (fp32 path's 1e-4 budget at K = 18944)
        float part[4][4] = {};
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = Ws[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) part[i][j] = fmaf(a[i], w[j], part[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];
        __syncthreads();
    }
    float* out = partial + (int64_t)z * M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n < N) out[(int64_t)m * N + n] = acc[i][j];
        }
    }
}

}  // namespace

void launch_gemm_simt(const void* A, int lda, const void* W, int M, int N, int K, float* partial, int splits,
                      DT dt, cudaStream_t s) {
    // caller guarantees splits divides the k range into non-empty chunks of multiples of BK
    const int kchunk = ((K + splits - 1) / splits + BK - 1) / BK * BK;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, splits);
    if (dt == DT::F32)
        launch_k(gemm_simt_kernel<float>, grid, THREADS, 0, s, (const float*)A, lda, (const float*)W, M, N, K, partial,
                                                         kchunk);
    else
        launch_k(gemm_simt_kernel<__nv_bfloat16>, grid, THREADS, 0, s, (const __nv_bfloat16*)A, lda,
                                                                 (const __nv_bfloat16*)W, M, N, K, partial, kchunk);
    TKV_CUDA(cudaGetLastError());
}

}  // namespace tkv

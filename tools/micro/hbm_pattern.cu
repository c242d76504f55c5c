// Does the GEMM's weight access pattern cost DRAM efficiency? Read a [N][K] bf16 matrix (K = 3584) either as
// 128-row x 64-col boxes (128 separate 128 B row segments, 7 KB apart: the TMA box of the GEMM) walking k-blocks,
// or as contiguous 16 KB blocks (a pre-tiled layout). One CTA per (128-row tile), warps cover the box rows.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void boxes(const uint4* __restrict__ w, int n_tiles, int kb, int ld_vec, unsigned* out, int tiled) {
    unsigned acc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
        for (int k = 0; k < kb; k += 2) {
            uint4 v[2][4];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = threadIdx.x + j * 256;  // 1024 x 16 B = one 16 KB box
                    const int row = e >> 3, c = e & 7;
                    size_t idx = tiled == 2 ? ((size_t)(k + kk) * n_tiles + t) * 1024 + e  // k-major tiles
                                 : tiled ? ((size_t)(t * kb + k + kk) * 1024 + e)
                                         : ((size_t)(t * 128 + row) * ld_vec + (size_t)(k + kk) * 8 + c);
                    v[kk][j] = __ldcs(w + idx);
                }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc ^= v[kk][j].x;
        }
    if (acc == 0x1234567u) *out = acc;
}
int main() {
    const int N = 37888, K = 3584, kb = K / 64, n_tiles = N / 128;
    const size_t bytes = (size_t)N * K * 2;
    uint4* w;
    unsigned* o;
    cudaMalloc(&w, bytes);
    cudaMalloc(&o, 4);
    cudaMemset(w, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int tiled = 0; tiled < 3; ++tiled)
        for (int ctas : {296, 592, 1184}) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(e0);
                boxes<<<ctas, 256>>>(w, n_tiles, kb, K / 8, o, tiled);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%s boxes, %d CTAs: %.0f GB/s\n", tiled == 2 ? "k-major pre-tiled" : tiled ? "contiguous (pre-tiled)" : "row-strided (TMA box)", ctas,
                   bytes / (best * 1e-3) / 1e9);
        }
    return 0;
}

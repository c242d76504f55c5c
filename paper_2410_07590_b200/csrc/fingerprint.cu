// Reference-exact model identity on the device: weights_checksum (src/model.cpp:94-112) is FNV-1a 64
// (include/turbokv/rng.hpp:41-78) over every f64 weight in init_random's order (model.cpp:68-92) -- for
// Qwen2-7B 6.5 G doubles = 52 GB of bytes through a strictly serial hash (~60 s on one host core). FNV-1a
// parallelises through two facts:
//
//  (1) h ^ b only changes the low byte, so h ^ b = h + d with d = (l ^ b) - l, l = h & 0xFF, hence one step
//      is affine in h:  h' = (h + d) * P.  Over a block of n bytes: h_end = h_start * P^n + S, where
//      S = sum_i d_i * P^(n - i)  (Horner: S = (S + d_i) * P).
//  (2) the low byte evolves on its own: l' = ((l ^ b) * 0xB3) & 0xFF (0xB3 = P mod 256), so the d_i of a
//      block depend on nothing but the block's bytes and the low byte it starts from.
//
// Pass A (perm_kernel): for every block and every one of the 256 possible starting low bytes, run the 8-bit
//   recurrence over the block -> the block's low-byte permutation (256 B). Four states per thread, two per
//   register in 16-bit lanes: one PRMT + 2 x (LOP3 + IMAD) per byte.
// Pass B (compose_kernel): compose the permutations of 128 consecutive blocks (one group) in shared memory.
// Host: walk the group permutations from FNV's offset basis -> the true starting low byte of every group.
// Pass C (starts_kernel): walk inside each group -> the starting low byte of every block.
// Pass D (affine_kernel): with its starting low byte known, each block computes S by Horner in 64-bit.
// Host: fold h = h * P^n_k + S_k over the blocks in order.
//
// The words hashed are regenerated on the device by the same counter-based generator the weight-init kernels
// use (kernels.cu:draw, bit-identical IEEE binary64 without contraction).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr uint64_t kFnvPrime = 0x100000001B3ULL;
constexpr int kBlockWords = 16384;  // 128 KB of hashed bytes per block
constexpr int kGroup = 128;         // blocks per composed group (their permutations: 32 KB of smem)
constexpr int kStage = 512;        // words staged in shared memory per pass-A iteration

__device__ __forceinline__ uint64_t sm_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t word_at(const FpSeg* segs, int n_segs, uint64_t seed, uint64_t w, int* hint) {
    int s = *hint;
    while (s + 1 < n_segs && segs[s + 1].word0 <= w) ++s;
    while (s > 0 && segs[s].word0 > w) --s;
    *hint = s;
    const FpSeg& g = segs[s];
    if (g.kind == 3) return reinterpret_cast<const uint64_t*>(g.a)[w - g.word0];  // words already in device memory
    if (g.kind == 2) {  // a drawn weight: next_signed() * scale (model.cpp:15-21), no FMA contraction
        const double u = __dmul_rn((double)(sm_at(seed, g.a + (w - g.word0)) >> 11), 0x1.0p-53);
        return (uint64_t)__double_as_longlong(__dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), g.scale));
    }
    return g.a;  // literal (a dimension) or constant (a norm weight 1.0)
}

__device__ __forceinline__ int first_seg(const FpSeg* segs, int n_segs, uint64_t w) {
    int lo = 0, hi = n_segs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].word0 <= w) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Pass A: 4 blocks per CTA of 256 threads; thread t of a block's 64 runs starting bytes {t, t+64, t+128, t+192}.
__global__ void __launch_bounds__(256) perm_kernel(const FpSeg* __restrict__ segs, int n_segs, uint64_t seed,
                                                   uint64_t words, int64_t n_blocks, uint8_t* __restrict__ perm) {
    __shared__ uint2 stage[4][kStage];
    const int sub = threadIdx.x >> 6, t = threadIdx.x & 63;
    for (int64_t b0 = (int64_t)blockIdx.x * 4; b0 < n_blocks; b0 += (int64_t)gridDim.x * 4) {
        const int64_t blk = b0 + sub;
        // two 16-bit lanes per register: states (t, t + 64) and (t + 128, t + 192)
        uint32_t r0 = (uint32_t)t | ((uint32_t)(t + 64) << 16), r1 = (uint32_t)(t + 128) | ((uint32_t)(t + 192) << 16);
        const uint64_t w0 = (uint64_t)blk * kBlockWords;
        const uint64_t wend = blk < n_blocks ? min(w0 + kBlockWords, words) : w0;
        for (int it = 0; it < kBlockWords; it += kStage) {
            __syncthreads();
            {  // stage the next kStage words of all four blocks (each thread 8 words of its own block)
                int hint = first_seg(segs, n_segs, w0 + it + (uint64_t)t * (kStage / 64));
                for (int j = 0; j < kStage / 64; ++j) {
                    const uint64_t w = w0 + it + (uint64_t)t * (kStage / 64) + j;
                    const uint64_t v = w < wend ? word_at(segs, n_segs, seed, w, &hint) : 0;
                    stage[sub][t * (kStage / 64) + j] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
                }
            }
            __syncthreads();
            const int nw = (int)std::min<int64_t>(kStage, (int64_t)wend - (int64_t)(w0 + it));
            for (int j = 0; j < nw; ++j) {
                const uint2 v = stage[sub][j];  // broadcast read
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const uint32_t x = half ? v.y : v.x;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // byte k of x into lanes 0 and 2 (PRMT selector: byte k, zero, byte k, zero)
                        const uint32_t bb = __byte_perm(x, 0u, (uint32_t)(k | (4 << 4) | (k << 8) | (4 << 12)));
                        r0 = ((r0 ^ bb) & 0x00FF00FFu) * 0xB3u;
                        r1 = ((r1 ^ bb) & 0x00FF00FFu) * 0xB3u;
                    }
                }
            }
        }
        if (blk < n_blocks) {
            uint8_t* p = perm + blk * 256;
            p[t] = (uint8_t)r0;
            p[t + 64] = (uint8_t)(r0 >> 16);
            p[t + 128] = (uint8_t)r1;
            p[t + 192] = (uint8_t)(r1 >> 16);
        }
    }
}

// Pass B: gperm[g][s] = low byte after the blocks of group g, starting from s.
__global__ void __launch_bounds__(256) compose_kernel(const uint8_t* __restrict__ perm, int64_t n_blocks,
                                                      uint8_t* __restrict__ gperm) {
    __shared__ uint8_t p[kGroup][256];
    const int64_t g = blockIdx.x, b0 = g * kGroup;
    const int nb = (int)std::min<int64_t>(kGroup, n_blocks - b0);
    const uint4* src = reinterpret_cast<const uint4*>(perm + b0 * 256);
    for (int i = threadIdx.x; i < nb * 16; i += blockDim.x) reinterpret_cast<uint4*>(&p[0][0])[i] = src[i];
    __syncthreads();
    uint32_t l = threadIdx.x;
    for (int b = 0; b < nb; ++b) l = p[b][l];
    gperm[g * 256 + threadIdx.x] = (uint8_t)l;
}

// Pass C: starting low byte of every block, from its group's starting byte.
__global__ void starts_kernel(const uint8_t* __restrict__ perm, int64_t n_blocks, const uint8_t* __restrict__ gstart,
                              int64_t n_groups, uint8_t* __restrict__ bstart) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n_groups) return;
    uint32_t l = gstart[g];
    const int64_t b0 = g * kGroup, b1 = std::min<int64_t>(b0 + kGroup, n_blocks);
    for (int64_t b = b0; b < b1; ++b) {
        bstart[b] = (uint8_t)l;
        l = perm[b * 256 + l];
    }
}

// Pass D: S of every block (one thread per block).
__global__ void __launch_bounds__(128) affine_kernel(const FpSeg* __restrict__ segs, int n_segs, uint64_t seed,
                                                     uint64_t words, int64_t n_blocks,
                                                     const uint8_t* __restrict__ bstart, uint64_t* __restrict__ S_out) {
    const int64_t blk = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (blk >= n_blocks) return;
    const uint64_t w0 = (uint64_t)blk * kBlockWords, w1 = min(w0 + kBlockWords, words);
    uint32_t l = bstart[blk];
    uint64_t S = 0;
    int hint = first_seg(segs, n_segs, w0);
    for (uint64_t w = w0; w < w1; ++w) {
        const uint64_t v = word_at(segs, n_segs, seed, w, &hint);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t b = (uint32_t)(v >> (8 * k)) & 0xFFu;
            const uint32_t lx = l ^ b;
            S = (S + (uint64_t)(int64_t)((int32_t)lx - (int32_t)l)) * kFnvPrime;
            l = (lx * 0xB3u) & 0xFFu;
        }
    }
    S_out[blk] = S;
}

// the words of a segment list, materialised (the TKVW writer streams them to a file)
__global__ void words_kernel(const FpSeg* __restrict__ segs, int n_segs, uint64_t seed, uint64_t w0, int64_t n,
                             uint64_t* __restrict__ out) {
    const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16;
    if (i0 >= n) return;
    int hint = first_seg(segs, n_segs, w0 + i0);
    const int64_t i1 = i0 + 16 < n ? i0 + 16 : n;
    for (int64_t i = i0; i < i1; ++i) out[i] = word_at(segs, n_segs, seed, w0 + i, &hint);
}

uint64_t pow_mod(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

}  // namespace

uint64_t device_fnv_words(const std::vector<FpSeg>& segs, uint64_t seed, uint64_t h0, cudaStream_t s) {
    if (segs.empty()) return h0;
    uint64_t words = 0;
    for (const FpSeg& g : segs) words = std::max(words, g.word0 + g.n);
    const int64_t n_blocks = (int64_t)((words + kBlockWords - 1) / kBlockWords);
    const int64_t n_groups = (n_blocks + kGroup - 1) / kGroup;
    int dev = 0, sms = 148;
    TKV_CUDA(cudaGetDevice(&dev));
    TKV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // scratch: segment table | perms | group perms | group starts | block starts | S
    const size_t seg_b = segs.size() * sizeof(FpSeg), perm_b = (size_t)n_blocks * 256, gp_b = (size_t)n_groups * 256;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t total = al(seg_b) + al(perm_b) + al(gp_b) + al(n_groups) + al(n_blocks) + al(n_blocks * 8);
    uint8_t* base = nullptr;
    TKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), total, s));
    FpSeg* d_segs = reinterpret_cast<FpSeg*>(base);
    uint8_t* perm = base + al(seg_b);
    uint8_t* gperm = perm + al(perm_b);
    uint8_t* gstart = gperm + al(gp_b);
    uint8_t* bstart = gstart + al(n_groups);
    uint64_t* S = reinterpret_cast<uint64_t*>(bstart + al(n_blocks));
    std::vector<uint8_t> h_gperm(gp_b), h_gstart((size_t)n_groups);
    std::vector<uint64_t> h_S((size_t)n_blocks);
    try {
        TKV_CUDA(cudaMemcpyAsync(d_segs, segs.data(), seg_b, cudaMemcpyHostToDevice, s));
        const int grid_a = (int)std::min<int64_t>((n_blocks + 3) / 4, (int64_t)sms * 8);
        perm_kernel<<<grid_a, 256, 0, s>>>(d_segs, (int)segs.size(), seed, words, n_blocks, perm);
        TKV_CUDA(cudaGetLastError());
        compose_kernel<<<(unsigned)n_groups, 256, 0, s>>>(perm, n_blocks, gperm);
        TKV_CUDA(cudaGetLastError());
        TKV_CUDA(cudaMemcpyAsync(h_gperm.data(), gperm, gp_b, cudaMemcpyDeviceToHost, s));
        TKV_CUDA(cudaStreamSynchronize(s));
        uint32_t l = (uint32_t)(h0 & 0xFF);
        for (int64_t g = 0; g < n_groups; ++g) {
            h_gstart[(size_t)g] = (uint8_t)l;
            l = h_gperm[(size_t)g * 256 + l];
        }
        TKV_CUDA(cudaMemcpyAsync(gstart, h_gstart.data(), (size_t)n_groups, cudaMemcpyHostToDevice, s));
        starts_kernel<<<(unsigned)((n_groups + 127) / 128), 128, 0, s>>>(perm, n_blocks, gstart, n_groups, bstart);
        TKV_CUDA(cudaGetLastError());
        affine_kernel<<<(unsigned)((n_blocks + 127) / 128), 128, 0, s>>>(d_segs, (int)segs.size(), seed, words,
                                                                         n_blocks, bstart, S);
        TKV_CUDA(cudaGetLastError());
        TKV_CUDA(cudaMemcpyAsync(h_S.data(), S, (size_t)n_blocks * 8, cudaMemcpyDeviceToHost, s));
        TKV_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaFreeAsync(base, s);
        throw;
    }
    TKV_CUDA(cudaFreeAsync(base, s));
    const uint64_t p_full = pow_mod(kFnvPrime, (uint64_t)kBlockWords * 8);
    uint64_t h = h0;
    for (int64_t b = 0; b < n_blocks; ++b) {
        const uint64_t nw = std::min<uint64_t>(kBlockWords, words - (uint64_t)b * kBlockWords);
        h = h * (nw == (uint64_t)kBlockWords ? p_full : pow_mod(kFnvPrime, nw * 8)) + h_S[(size_t)b];
    }
    return h;
}

void device_words(const std::vector<FpSeg>& segs, uint64_t seed, uint64_t w0, int64_t n, uint64_t* d_out,
                  cudaStream_t s) {
    if (n <= 0) return;
    FpSeg* d_segs = nullptr;
    TKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_segs), segs.size() * sizeof(FpSeg), s));
    TKV_CUDA(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(FpSeg), cudaMemcpyHostToDevice, s));
    const int64_t threads = (n + 15) / 16;
    words_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(d_segs, (int)segs.size(), seed, w0, n, d_out);
    TKV_CUDA(cudaGetLastError());
    TKV_CUDA(cudaFreeAsync(d_segs, s));
}

}  // namespace tkv

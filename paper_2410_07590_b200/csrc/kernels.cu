// Memory-bound kernels of the TurboRAG prefill path (sm_100a):
//   weight init (SplitMix64, src/model.cpp:15-21,68-92), embedding + RMSNorm (numerics.cpp:84-101),
//   split-K reduce epilogues (residual + RMSNorm, SwiGLU numerics.cpp:103-124, QKV + RoPE rope.cpp:35-46),
//   the KV-gather + RoPE injection kernel (replaces CacheStore::load + ctx.append + per-layer
//   rope_rotate_heads_inplace: kvstore.cpp:134-207, context.cpp:7-22, model.cpp:248-254),
//   lm_head GEMV and mask materialisation.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

__device__ __forceinline__ float ldf(const float* p, int64_t i) { return p[i]; }

// Split-K partial sums in ascending split order (the order of the previous serial loop, so results are
// unchanged), with a batch of SB loads in flight instead of one dependent L2/HBM round trip per split.
template <typename V>
__device__ __forceinline__ void add_to(V& a, const V& b);
template <>
__device__ __forceinline__ void add_to<float>(float& a, const float& b) { a += b; }
template <>
__device__ __forceinline__ void add_to<float2>(float2& a, const float2& b) { a.x += b.x, a.y += b.y; }
template <>
__device__ __forceinline__ void add_to<float4>(float4& a, const float4& b) { a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w; }
template <typename V, int SB = 8>
__device__ __forceinline__ V sum_splits(const float* p, int splits, int64_t plane, V acc) {
    for (int s0 = 0; s0 < splits; s0 += SB) {
        V v[SB];
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (s0 + i < splits) v[i] = *reinterpret_cast<const V*>(p + (int64_t)(s0 + i) * plane);
#pragma unroll
        for (int i = 0; i < SB; ++i)
            if (s0 + i < splits) add_to(acc, v[i]);
    }
    return acc;
}
__device__ __forceinline__ float ldf(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void stf(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void stf(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }
// two consecutive elements (8-byte aligned for f32, 4-byte for bf16), each rounded like stf
__device__ __forceinline__ void store2(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }
__device__ __forceinline__ void store2(__nv_bfloat16* p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
// four consecutive elements (16-byte aligned for f32, 8-byte for bf16), each rounded like stf
__device__ __forceinline__ void store4(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, const float (&v)[4]) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// next_signed() * scale in IEEE binary64 without contraction (bit-identical to the host).
__device__ __forceinline__ double draw(uint64_t seed, uint64_t i, double scale) {
    const double u = __dmul_rn((double)(splitmix_at(seed, i) >> 11), 0x1.0p-53);
    return __dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), scale);
}

template <typename T>
__global__ void init_transposed_kernel(T* dst, uint64_t seed, uint64_t base, int64_t rows, int64_t cols,
                                       double scale, int row_block, int row_off) {
    pdl_launch();
    pdl_wait();
    const int64_t n = rows * cols;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = o / rows, i = o - j * rows;
        const int64_t pj = row_block ? (j / row_block) * 2 * row_block + row_off + j % row_block : j;
        const float f = __double2float_rn(draw(seed, base + (uint64_t)(i * cols + j), scale));
        stf(dst, pj * rows + i, f);  // f64 -> f32 (RN) -> bf16 (RNE): the canonical cast, see DESIGN.md
    }
}

template <typename T>
__global__ void store_transposed_f64_kernel(T* dst, const double* __restrict__ src, int64_t e0, int64_t n, int64_t rows,
                                            int64_t cols, int row_block, int row_off) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = e0 + o, i = e / cols, j = e - i * cols;  // source [in = i][out = j]
        const int64_t pj = row_block ? (j / row_block) * 2 * row_block + row_off + j % row_block : j;
        stf(dst, pj * rows + i, __double2float_rn(src[o]));  // the canonical cast
    }
}

__global__ void f32_from_f64_kernel(float* dst, const double* __restrict__ src, int64_t n) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
        dst[o] = __double2float_rn(src[o]);
}

__global__ void init_rowmajor_kernel(float* dst, uint64_t seed, uint64_t base, int64_t n, double scale) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
        dst[o] = __double2float_rn(draw(seed, base + (uint64_t)o, scale));
}

__global__ void fill_kernel(float* dst, float v, int64_t n) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
        dst[o] = v;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = 0.f;
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) t += red[i];
    return t;
}

// Block of 1024 columns of one row: 256 threads x 4. Writes x, xb = x * w and, per warp (128 columns),
// ssp_row[blockIdx.x * 8 + warp] (norm_blocks(hidden) slots per row).
template <typename T>
__device__ __forceinline__ void finish_row_block(float* __restrict__ xrow, const float* __restrict__ w, T* xbrow,
                                                 float* ssp_row, float (&v)[4], int c0, int hidden, float* red,
                                                 int* err) {
    float ss = 0.f;
    bool bad = false;
    if ((hidden & 3) == 0 && c0 + 3 < hidden) {  // 16-byte x / weight vectors, 4 xb elements per store
        *reinterpret_cast<float4*>(xrow + c0) = make_float4(v[0], v[1], v[2], v[3]);
        const float4 wv = *reinterpret_cast<const float4*>(w + c0);
        const float xw[4] = {v[0] * wv.x, v[1] * wv.y, v[2] * wv.z, v[3] * wv.w};
        store4(xbrow + c0, xw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            ss += v[e] * v[e];
            bad |= !isfinite(v[e]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = c0 + e;
            if (c < hidden) {
                xrow[c] = v[e];
                stf(xbrow, c, v[e] * w[c]);
                ss += v[e] * v[e];
                bad |= !isfinite(v[e]);
            }
        }
    }
    if (bad) atomicOr(err, 2);
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const int slot = blockIdx.x * 8 + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && slot < norm_blocks(hidden)) ssp_row[slot] = ss;
}

template <typename T>
__global__ void __launch_bounds__(256) embed_kernel(const int32_t* tok, const float* emb, int hidden, int vocab,
                                                    const float* w, float* x, T* xb, float* ssp, int* err,
                                                    unsigned long long* tl) {
    // First kernel of every forward: release dependents only AFTER the wait, so any later kernel of this
    // forward that starts implies every earlier grid (previous forwards, the KV gather, uploads) has
    // completed — the attention kernel relies on this to TMA-load context K/V before its own wait.
    pdl_wait();
    pdl_launch();
    tl_wait(tl);
    __shared__ float red[32];
    const int t = blockIdx.y, nb = norm_blocks(hidden);
    const int id = tok[t];
    if (id < 0 || id >= vocab) {  // DomainError "token id outside vocab" (model.cpp:217-221)
        if (threadIdx.x == 0) atomicOr(err, 1);
        return;
    }
    const int c0 = blockIdx.x * 1024 + threadIdx.x * 4;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = (c0 + e < hidden) ? emb[(int64_t)id * hidden + c0 + e] : 0.f;
    finish_row_block(x + (int64_t)t * hidden, w, xb + (int64_t)t * hidden, ssp + (int64_t)t * nb, v, c0, hidden, red,
                     err);
    tl_exit(tl);
}

// Residual add of the split-K partials (x += a . W), many CTAs per row (nb x T grid).
template <typename T>
__global__ void __launch_bounds__(256) residual_kernel(float* x, const float* partial, int splits, int64_t plane,
                                                       int hidden, const float* w, T* xb, float* ssp, int* err,
                                                       unsigned long long* tl) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    __shared__ float red[32];
    const int64_t t = blockIdx.y;
    const int nb = norm_blocks(hidden);
    const int c0 = blockIdx.x * 1024 + threadIdx.x * 4;
    float v[4];
    float* xrow = x + t * hidden;
    if ((hidden & 3) == 0 && c0 + 3 < hidden) {
        const float4 a = sum_splits<float4, 16>(partial + t * hidden + c0, splits, plane, *reinterpret_cast<const float4*>(xrow + c0));
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            v[e] = 0.f;
            if (c0 + e < hidden) {
                float acc = xrow[c0 + e];
                for (int s = 0; s < splits; ++s) acc += partial[s * plane + t * hidden + c0 + e];
                v[e] = acc;
            }
        }
    }
    finish_row_block(xrow, w, xb + t * hidden, ssp + t * nb, v, c0, hidden, red, err);
    tl_exit(tl);
}

// Many-token forwards: the same, each CTA looping over rows (nb x min(T, ~8 CTAs / SM) grid) -- 8192 one-row CTAs at
// 2048 tokens ran at ~1.6 TB/s.
template <typename T>
__global__ void __launch_bounds__(256, 4) residual_rows_kernel(float* x, const float* partial, int splits,
                                                          int64_t plane, int T_, int hidden, const float* w, T* xb,
                                                          float* ssp, int* err, unsigned long long* tl) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    __shared__ float red[32];
    const int nb = norm_blocks(hidden);
    const int c0 = blockIdx.x * 1024 + threadIdx.x * 4;
    const bool vec = (hidden & 3) == 0 && c0 + 3 < hidden;
    // rows t and t + gridDim.y per iteration: both rows' loads in flight before either is finished (few split planes
    // at these sizes, so a 2-deep split batch keeps the registers at 4 CTAs / SM)
    for (int64_t t = blockIdx.y; t < T_; t += 2 * (int64_t)gridDim.y) {
        const int64_t t2 = t + gridDim.y;
        const bool two = t2 < T_;
        float v[4], u[4];
        if (vec) {
            const float4 a = sum_splits<float4, 2>(partial + t * hidden + c0, splits, plane,
                                                  *reinterpret_cast<const float4*>(x + t * hidden + c0));
            float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
            if (two)
                b = sum_splits<float4, 2>(partial + t2 * hidden + c0, splits, plane,
                                          *reinterpret_cast<const float4*>(x + t2 * hidden + c0));
            v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
            u[0] = b.x, u[1] = b.y, u[2] = b.z, u[3] = b.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[e] = u[e] = 0.f;
                if (c0 + e < hidden) {
                    float acc = x[t * hidden + c0 + e];
                    for (int s2 = 0; s2 < splits; ++s2) acc += partial[s2 * plane + t * hidden + c0 + e];
                    v[e] = acc;
                    if (two) {
                        float acc2 = x[t2 * hidden + c0 + e];
                        for (int s2 = 0; s2 < splits; ++s2) acc2 += partial[s2 * plane + t2 * hidden + c0 + e];
                        u[e] = acc2;
                    }
                }
            }
        }
        finish_row_block(x + t * hidden, w, xb + t * hidden, ssp + t * nb, v, c0, hidden, red, err);
        if (two) finish_row_block(x + t2 * hidden, w, xb + t2 * hidden, ssp + t2 * nb, u, c0, hidden, red, err);
    }
    tl_exit(tl);
}

template <typename T>
__global__ void swiglu_kernel(const float* partial, int splits, int T_, int inter, T* act, const float* ssp, int nb,
                              int hidden, float eps, int gub) {
    pdl_launch();
    pdl_wait();
    const int64_t n = (int64_t)T_ * inter, plane = (int64_t)T_ * 2 * inter;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = o / inter, i = o - t * inter;
        const int64_t gc = gub ? (i / gub) * 2 * gub + i % gub : i;
        const int64_t uc = gub ? gc + gub : inter + i;
        float g = sum_splits(partial + t * 2 * inter + gc, splits, plane, 0.f);
        float u = sum_splits(partial + t * 2 * inter + uc, splits, plane, 0.f);
        const float sc = row_scale(ssp, nb, t, hidden, eps);
        g *= sc;
        u *= sc;
        stf(act, o, (g / (1.0f + expf(-g))) * u);  // silu(z) = z / (1 + e^-z), numerics.cpp:103-105
    }
}

// Element offset of token t's row of (layer, K|V) inside its store page; HBM pool or the host spill tier.
template <typename T>
__device__ __forceinline__ int64_t store_base(const StoreScatter& sc, int64_t t, int layer, int kv, int kvd, T*& pool) {
    int64_t page = sc.page[t];
    pool = (T*)sc.pool;
    if (page >= sc.host_base) {
        page -= sc.host_base;
        pool = (T*)sc.host_pool;
    }
    return ((page * sc.layer_num + layer) * 2 + kv) * sc.page_tokens * kvd + (int64_t)sc.slot[t] * kvd;
}

// Non-batched few-token forwards (C2 query prefill): one thread per element pair (2m, 2m+1) of the fused QKV output
// row over a flat grid (64 registers: 4 CTAs / SM, one wave at 64 tokens).
template <typename T>
__global__ void qkv_epilogue_single_kernel(const float* partial, int splits, int T_, int H, int Hkv, int d,
                                    const int32_t* pos, const float2* rope, T* q, T* kc, T* vc, int row0,
                                    StoreScatter sc, int layer, const float* ssp, int nb, int hidden, float eps,
                                    int64_t plane, unsigned long long* tl) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    const int qd = H * d, kvd = Hkv * d, N = qd + 2 * kvd, half = d / 2;
    const int64_t pairs = (int64_t)T_ * (N / 2);
    int64_t cached_t = -1;
    float rs = 0.f;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = p / (N / 2);
        if (t != cached_t) {  // folded attn RMSNorm scale, once per token per thread
            rs = row_scale(ssp, nb, t, hidden, eps);
            cached_t = t;
        }
        const int n = 2 * (int)(p - t * (N / 2));
        const float2 xs = sum_splits(partial + t * N + n, splits, plane, make_float2(0.f, 0.f));  // n even: 8 B aligned
        float x0 = xs.x, x1 = xs.y;
        x0 *= rs;
        x1 *= rs;
        if (n >= qd + kvd) {  // V: copied as is
            const int c = n - qd - kvd;
            stf(vc, (int64_t)(row0 + t) * kvd + c, x0);
            stf(vc, (int64_t)(row0 + t) * kvd + c + 1, x1);
            if (sc.page) {
                T* pool;
                const int64_t base = store_base(sc, t, layer, 1, kvd, pool);
                stf(pool, base + c, x0);
                stf(pool, base + c + 1, x1);
            }
            continue;
        }
        const int e = (n < qd ? n : n - qd) % d;
        const float2 cs = rope[(int64_t)pos[t] * half + e / 2];
        const float r0 = x0 * cs.x - x1 * cs.y, r1 = x0 * cs.y + x1 * cs.x;  // rope.cpp:41-44
        if (n < qd) {
            stf(q, t * qd + n, r0);
            stf(q, t * qd + n + 1, r1);
        } else {
            const int c = n - qd;
            stf(kc, (int64_t)(row0 + t) * kvd + c, r0);
            stf(kc, (int64_t)(row0 + t) * kvd + c + 1, r1);
            if (sc.page) {  // the store keeps keys unrotated (SPEC: rotation at use)
                T* pool;
                const int64_t base = store_base(sc, t, layer, 0, kvd, pool);
                stf(pool, base + c, x0);
                stf(pool, base + c + 1, x1);
            }
        }
    }
    tl_exit(tl);
}

// Few-token BATCHED forwards: one thread per element pair (2m, 2m+1) of the fused QKV output row over a flat
// grid; the folded RMSNorm scale and (batched forwards) the token's request are looked up per thread. Measured faster
// than the per-token-row kernel below at 64 tokens (it also leaves the attention that follows ~1 us / layer faster).
template <typename T, bool BATCH>
__global__ void __launch_bounds__(256, 4) qkv_epilogue_flat_kernel(const float* partial, int splits, int T_, int H, int Hkv, int d,
                                    const int32_t* pos, const float2* rope, T* q, T* kc, T* vc, int row0,
                                    StoreScatter sc, int layer, const float* ssp, int nb, int hidden, float eps,
                                    int64_t plane, unsigned long long* tl, const EpiReq* __restrict__ reqs, int n_req) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    const int qd = H * d, kvd = Hkv * d, N = qd + 2 * kvd, half = d / 2;
    const int64_t pairs = (int64_t)T_ * (N / 2);
    int64_t cached_t = -1;
    float rs = 0.f;
    T* kct = kc;  // this token's cache planes and row (batched: its request's cache)
    T* vct = vc;
    int64_t crow = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = p / (N / 2);
        if (t != cached_t) {  // folded attn RMSNorm scale and the destination rows, once per token per thread
            rs = row_scale(ssp, nb, t, hidden, eps);
            cached_t = t;
            crow = row0 + t;
            if (BATCH) {  // request of token t: the last with tok0 <= t (tok0 ascending)
                int lo = 0, hi = n_req - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (reqs[mid].tok0 <= t) lo = mid;
                    else hi = mid - 1;
                }
                const EpiReq R = reqs[lo];
                kct = static_cast<T*>(R.kv) + (int64_t)(2 * layer) * R.cap * kvd;
                vct = kct + R.cap * kvd;
                crow = R.row0 + (t - R.tok0);
            }
        }
        const int n = 2 * (int)(p - t * (N / 2));
        const float2 xs = sum_splits(partial + t * N + n, splits, plane, make_float2(0.f, 0.f));  // n even: 8 B aligned
        float x0 = xs.x, x1 = xs.y;
        x0 *= rs;
        x1 *= rs;
        if (n >= qd + kvd) {  // V: copied as is
            const int c = n - qd - kvd;
            stf(vct, crow * kvd + c, x0);
            stf(vct, crow * kvd + c + 1, x1);
            if (sc.page) {
                T* pool;
                const int64_t base = store_base(sc, t, layer, 1, kvd, pool);
                stf(pool, base + c, x0);
                stf(pool, base + c + 1, x1);
            }
            continue;
        }
        const int e = (n < qd ? n : n - qd) % d;
        const float2 cs = rope[(int64_t)pos[t] * half + e / 2];
        const float r0 = x0 * cs.x - x1 * cs.y, r1 = x0 * cs.y + x1 * cs.x;  // rope.cpp:41-44
        if (n < qd) {
            stf(q, t * qd + n, r0);
            stf(q, t * qd + n + 1, r1);
        } else {
            const int c = n - qd;
            stf(kct, crow * kvd + c, r0);
            stf(kct, crow * kvd + c + 1, r1);
            if (sc.page) {  // the store keeps keys unrotated (SPEC: rotation at use)
                T* pool;
                const int64_t base = store_base(sc, t, layer, 0, kvd, pool);
                stf(pool, base + c, x0);
                stf(pool, base + c + 1, x1);
            }
        }
    }
    tl_exit(tl);
}

// Many-token forwards (batched prefill, ingest, full concat): one thread per element pair (2m, 2m+1); grid.y walks the tokens, so the folded RMSNorm
// scale, the position and (batched forwards) the token's request / cache rows are resolved once per CTA.
template <typename T>
__global__ void __launch_bounds__(256) qkv_epilogue_kernel(const float* partial, int splits, int T_, int H, int Hkv,
                                                           int d, const int32_t* pos, const float2* rope, T* q, T* kc,
                                                           T* vc, int row0, StoreScatter sc, int layer, const float* ssp,
                                                           int nb, int hidden, float eps, int64_t plane,
                                                           unsigned long long* tl, const EpiReq* __restrict__ reqs,
                                                           int n_req) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    const int qd = H * d, kvd = Hkv * d, N = qd + 2 * kvd, half = d / 2;
    const int dmask = (d & (d - 1)) == 0 ? d - 1 : -1;  // power-of-two head size: e = n % d as a mask
    __shared__ float s_rs;
    __shared__ T* s_k;
    __shared__ T* s_v;
    __shared__ int64_t s_row;
    __shared__ int s_pos;
    for (int64_t t = blockIdx.y; t < T_; t += gridDim.y) {
        if (threadIdx.x < 32) {  // warp 0: folded attn RMSNorm scale, position and destination rows of token t
            const int lane = threadIdx.x;
            // row_scale (dev_common.cuh) with its loads spread over the lanes and the same summation order
            const float part = (nb <= 32 && lane < nb) ? ssp[t * nb + lane] : 0.f;
            const int pt = lane == 0 ? pos[t] : 0;
            int r = 0;  // request of token t: the last with tok0 <= t (tok0 ascending), 32 entries per ballot
            for (int base = 0; base < n_req; base += 32) {
                const unsigned m = __ballot_sync(0xffffffffu, base + lane < n_req && reqs[base + lane].tok0 <= t);
                if (m) r = base + 31 - __clz(m);
                if (m != 0xffffffffu) break;
            }
            float ss = 0.f;
            for (int b = 0; b < min(nb, 32); ++b) ss += __shfl_sync(0xffffffffu, part, b);
            if (lane == 0) {
                s_rs = nb <= 32 ? 1.0f / sqrtf(ss / (float)hidden + eps) : row_scale(ssp, nb, t, hidden, eps);
                s_pos = pt;
                if (n_req > 0) {
                    const EpiReq R = reqs[r];
                    T* kct = static_cast<T*>(R.kv) + (int64_t)(2 * layer) * R.cap * kvd;
                    s_k = kct;
                    s_v = kct + R.cap * kvd;
                    s_row = R.row0 + (t - R.tok0);
                } else {
                    s_k = kc;
                    s_v = vc;
                    s_row = row0 + t;
                }
            }
        }
        __syncthreads();
        const float rs = s_rs;
        // the token's rows, resolved once: the pair loop below is issue-bound (ncu: SM 83 % busy, DRAM 21 % at 16 K
        // tokens with the index math -- n % d, 64-bit row products, the store page lookup, sum_splits' predicated
        // 8-wide address math at one split -- redone per pair): C3 QKV epilogue 41 -> 28 us, C5 350 -> 295 us
        const float* prow = partial + t * N;
        T* qrow = q + t * qd;
        T* krow = s_k + s_row * kvd;
        T* vrow = s_v + s_row * kvd;
        const float2* rrow = rope + (int64_t)s_pos * half;
        T* kpg = nullptr;
        T* vpg = nullptr;
        if (sc.page) {  // the token's rows in its store page (keys unrotated: SPEC, rotation at use)
            T* pool;
            const int64_t kb = store_base(sc, t, layer, 0, kvd, pool);
            kpg = pool + kb;
            const int64_t vb = store_base(sc, t, layer, 1, kvd, pool);
            vpg = pool + vb;
        }
        for (int n = 2 * (int)(blockIdx.x * blockDim.x + threadIdx.x); n < N; n += 2 * (int)(gridDim.x * blockDim.x)) {
            float2 xs = make_float2(0.f, 0.f);  // n even: 8 B
            if (splits == 1)  // no split-K (large-M GEMMs): skip sum_splits' SB-wide predicated address math
                add_to(xs, *reinterpret_cast<const float2*>(prow + n));
            else
                xs = sum_splits(prow + n, splits, plane, xs);
            const float x0 = xs.x * rs, x1 = xs.y * rs;
            if (n >= qd + kvd) {  // V: copied as is
                const int c = n - qd - kvd;
                store2(vrow + c, x0, x1);
                if (vpg) store2(vpg + c, x0, x1);
            } else {
                const int e = (dmask >= 0 ? (n & dmask) : (n < qd ? n : n - qd) % d);  // qd = H * d: same e
                const float2 cs = rrow[e >> 1];
                const float r0 = x0 * cs.x - x1 * cs.y, r1 = x0 * cs.y + x1 * cs.x;  // rope.cpp:41-44
                if (n < qd) {
                    store2(qrow + n, r0, r1);
                } else {
                    const int c = n - qd;
                    store2(krow + c, r0, r1);
                    if (kpg) store2(kpg + c, x0, x1);
                }
            }
        }
        __syncthreads();  // the shared token state is rewritten for the next token
    }
    tl_exit(tl);
}

// ---- KV gather + fused RoPE ------------------------------------------------------------------
// Work unit = (segment, layer, K|V): a contiguous [n_tok, kv_dim] block of one store page copied
// to contiguous request-cache rows. 16-byte vectors; keys rotated in fp32 in registers.
template <typename T>
struct Vec16 {
    static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void rotate_vec(uint4& v, const float2* cs) {
    constexpr int N = Vec16<T>::N;
    T* e = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const float x0 = ldf(e, 2 * i), x1 = ldf(e, 2 * i + 1);
        const float2 c = cs[i];
        stf(e, 2 * i, x0 * c.x - x1 * c.y);
        stf(e, 2 * i + 1, x0 * c.y + x1 * c.x);
    }
}

// Work unit = (segment, layer, K|V, block of ROWS_PER_UNIT rows): fine-grained so the last wave of the
// grid-stride loop is short (C2: 14 336 units over 1 184 resident CTAs). Every thread issues
// all of its 16-byte loads (and, for keys, its cos/sin loads) before the first store.
#ifndef GATHER_ROWS_CFG
#define GATHER_ROWS_CFG 64
#endif
#ifndef GATHER_GRID_MULT
#define GATHER_GRID_MULT 32  // gather grid cap in CTAs per SM (swept: 8 -> 79 %, 16 -> 83 %, 32 -> 85.5 %, 64 -> 82 % of HBM)
#endif
#ifndef GATHER_U_CFG
#define GATHER_U_CFG 4
#endif
constexpr int GATHER_ROWS = GATHER_ROWS_CFG;

template <typename T>
__global__ void __launch_bounds__(256) gather_rope_vec_kernel(PoolTable pools, int page_tokens,
                                                              const GatherSeg* __restrict__ segs, int n_units, int L,
                                                              int kvd, int d, const float2* __restrict__ rope,
                                                              T* __restrict__ cache, int64_t cap, int rotate,
                                                              unsigned long long* tl) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    constexpr int N = Vec16<T>::N;
    constexpr int U = GATHER_U_CFG;
    const int vec_per_row = kvd / N, half = d / 2;
    const int blocks_per_page = (page_tokens + GATHER_ROWS - 1) / GATHER_ROWS;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int rb = u % blocks_per_page;
        const int rest = u / blocks_per_page;
        const int seg = rest / (2 * L), layer = (rest / 2) % L, kv = rest & 1;
        const GatherSeg sg = segs[seg];
        const int r0 = rb * GATHER_ROWS;
        const int nrows = min(GATHER_ROWS, sg.n_tok - r0);
        if (nrows <= 0) continue;
        const T* pool = reinterpret_cast<const T*>(pools.p[sg.pool]);  // local HBM or a peer GPU over NVLink
        const uint4* src = reinterpret_cast<const uint4*>(
            pool + ((((int64_t)sg.src_page * L + layer) * 2 + kv) * page_tokens + r0) * kvd);
        uint4* dst = reinterpret_cast<uint4*>(cache + ((int64_t)(layer * 2 + kv) * cap + sg.dst_row + r0) * kvd);
        const int nv = nrows * vec_per_row;
        const bool rot = rotate && kv == 0;
        for (int base = threadIdx.x; base < nv; base += blockDim.x * U) {
            uint4 r[U];
            float2 c[U][N / 2];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = base + k * blockDim.x;
                if (i < nv) r[k] = __ldcs(src + i);  // streaming read: store pages are not re-read
            }
            if (rot) {
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int i = base + k * blockDim.x;
                    if (i < nv) {
                        const int row = i / vec_per_row, col = (i - row * vec_per_row) * N;
                        const float2* cs = rope + (int64_t)(sg.pos0 + r0 + row) * half + (col % d) / 2;
#pragma unroll
                        for (int m = 0; m < N / 2; ++m) c[k][m] = __ldg(cs + m);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = base + k * blockDim.x;
                if (i < nv) {
                    if (rot) rotate_vec<T>(r[k], c[k]);
                    __stcs(dst + i, r[k]);  // the 470 MB request cache does not fit L2: stream it out
                }
            }
        }
    }
    tl_exit(tl);
}

// Generic fallback: one pair per thread (any even head_size / kv_dim).
template <typename T>
__global__ void gather_rope_pair_kernel(PoolTable pools, int page_tokens, const GatherSeg* segs, int n_units, int L,
                                        int kvd, int d, const float2* rope, T* cache, int64_t cap, int rotate) {
    pdl_launch();
    pdl_wait();
    const int half = d / 2;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int seg = u / (2 * L), layer = (u / 2) % L, kv = u & 1;
        const GatherSeg sg = segs[seg];
        const T* src = reinterpret_cast<const T*>(pools.p[sg.pool]) +
                       (((int64_t)sg.src_page * L + layer) * 2 + kv) * page_tokens * kvd;
        T* dst = cache + ((int64_t)(layer * 2 + kv) * cap + sg.dst_row) * kvd;
        const int np = sg.n_tok * kvd / 2;
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
            const int row = (2 * i) / kvd, col = 2 * i - row * kvd;
            float x0 = ldf(src, 2 * i), x1 = ldf(src, 2 * i + 1);
            if (rotate && kv == 0) {
                const float2 c = rope[(int64_t)(sg.pos0 + row) * half + (col % d) / 2];
                const float r0 = x0 * c.x - x1 * c.y, r1 = x0 * c.y + x1 * c.x;
                x0 = r0;
                x1 = r1;
            }
            stf(dst, 2 * i, x0);
            stf(dst, 2 * i + 1, x1);
        }
    }
}

template <typename T>
__global__ void lm_head_kernel(const T* h, const T* W, int hidden, int vocab, float* logits, const float* ssp, int nb,
                               float eps, int* err, unsigned long long* tl) {
    pdl_launch();
    pdl_wait();
    tl_wait(tl);
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= vocab) return;
    float acc = 0.f;
    constexpr int N = 16 / sizeof(T);  // elements per 16-byte vector
    if ((hidden % (32 * N)) == 0) {
        // one warp per vocab row: every 16-byte load of the row (and of h) issued before the FMAs
        const uint4* wr = reinterpret_cast<const uint4*>(W + (int64_t)warp * hidden);
        const uint4* hr = reinterpret_cast<const uint4*>(h);
        const int nv = hidden / N;
        for (int v0 = lane; v0 < nv; v0 += 32 * 8) {
            uint4 a[8], b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v0 + 32 * u < nv) {
                    a[u] = __ldcs(wr + v0 + 32 * u);
                    b[u] = hr[v0 + 32 * u];
                }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v0 + 32 * u < nv) {
                    const T* x = reinterpret_cast<const T*>(&a[u]);
                    const T* y = reinterpret_cast<const T*>(&b[u]);
#pragma unroll
                    for (int e = 0; e < N; ++e) acc += ldf(y, e) * ldf(x, e);
                }
        }
    } else {
        for (int k = lane; k < hidden; k += 32) acc += ldf(h, k) * ldf(W, (int64_t)warp * hidden + k);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        acc *= row_scale(ssp, nb, 0, hidden, eps);  // folded final_norm
        logits[warp] = acc;
        if (!isfinite(acc)) atomicOr(err, 4);  // Matrix::require_finite("logits"), model.cpp:268
    }
    tl_exit(tl);
}

__global__ void mask_kernel(const int32_t* lo, const int32_t* hi, int rows, int cols, uint8_t* out) {
    pdl_launch();
    pdl_wait();
    const int64_t n = (int64_t)rows * cols;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / cols), j = (int)(o - (int64_t)i * cols);
        out[o] = (j >= lo[i] && j <= hi[i]) ? 1 : 0;  // same predicate as attention (attn_simt.cu)
    }
}

template <typename T>
__global__ void unrotate_kernel(const T* k, int rows, int kvd, int d, const int32_t* pos, const float2* rope,
                                float* out) {
    pdl_launch();
    pdl_wait();
    const int64_t n = (int64_t)rows * kvd / 2;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = (2 * p) / kvd;
        const int c = (int)(2 * p - r * kvd);
        const float2 cs = rope[(int64_t)pos[r] * (d / 2) + (c % d) / 2];
        const float y0 = ldf(k, 2 * p), y1 = ldf(k, 2 * p + 1);
        out[2 * p] = y0 * cs.x + y1 * cs.y;  // R(-t)
        out[2 * p + 1] = -y0 * cs.y + y1 * cs.x;
    }
}

template <typename T>
__global__ void to_f32_kernel(const T* src, int64_t n, float* dst) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
        dst[o] = ldf(src, o);
}

template <typename T>
__global__ void from_f32_kernel(const float* src, int64_t n, T* dst) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
        stf(dst, o, src[o]);
}

__global__ void reduce_splits_kernel(const float* p, int splits, int64_t n, float* out) {
    pdl_launch();
    pdl_wait();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        out[o] = sum_splits(p + o, splits, n, 0.f);
    }
}

inline int grid_for(int64_t n, int block, int cap = 148 * 16) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

}  // namespace

#define DISPATCH_DT(dt, ...)                            \
    do {                                                \
        if ((dt) == DT::F32) {                          \
            using T = float;                            \
            __VA_ARGS__;                                \
        } else {                                        \
            using T = __nv_bfloat16;                    \
            __VA_ARGS__;                                \
        }                                               \
    } while (0)

void launch_init_transposed(void* dst, DT dt, uint64_t seed, uint64_t base, int64_t rows, int64_t cols,
                            double scale, cudaStream_t s, int row_block, int row_off) {
    DISPATCH_DT(dt, launch_k(init_transposed_kernel<T>, grid_for(rows * cols, 256, 148 * 64), 256, 0, s, 
                        (T*)dst, seed, base, rows, cols, scale, row_block, row_off));
    TKV_CUDA(cudaGetLastError());
}

void launch_init_rowmajor_f32(float* dst, uint64_t seed, uint64_t base, int64_t rows, int64_t cols, double scale,
                              cudaStream_t s) {
    launch_k(init_rowmajor_kernel, grid_for(rows * cols, 256, 148 * 64), 256, 0, s, dst, seed, base, rows * cols, scale);
    TKV_CUDA(cudaGetLastError());
}

void launch_fill_f32(float* dst, float v, int64_t n, cudaStream_t s) {
    launch_k(fill_kernel, grid_for(n, 256), 256, 0, s, dst, v, n);
    TKV_CUDA(cudaGetLastError());
}

void launch_embed(const int32_t* tok, int T_, const float* emb, int hidden, int vocab, const float* w, float* x,
                  void* xb, float* ssp, DT dt, int* err, cudaStream_t s) {
    const dim3 grid(row_ctas(hidden), T_);
    unsigned long long* tl = tl_take();
    DISPATCH_DT(dt, launch_k(embed_kernel<T>, grid, 256, 0, s, tok, emb, hidden, vocab, w, x, (T*)xb, ssp, err, tl));
    TKV_CUDA(cudaGetLastError());
}

void launch_store_transposed_f64(void* dst, DT dt, const double* src, int64_t e0, int64_t n, int64_t rows, int64_t cols,
                                 cudaStream_t s, int row_block, int row_off) {
    DISPATCH_DT(dt, launch_k(store_transposed_f64_kernel<T>, grid_for(n, 256), 256, 0, s, (T*)dst, src, e0, n, rows, cols,
                             row_block, row_off));
    TKV_CUDA(cudaGetLastError());
}

void launch_store_f32_from_f64(float* dst, const double* src, int64_t n, cudaStream_t s) {
    launch_k(f32_from_f64_kernel, grid_for(n, 256), 256, 0, s, dst, src, n);
    TKV_CUDA(cudaGetLastError());
}

void launch_residual(float* x, const float* partial, int splits, int T_, int hidden, const float* w, void* xb,
                     float* ssp, DT dt, int* err, cudaStream_t s) {
    const int64_t plane = (int64_t)T_ * hidden;
    unsigned long long* tl = tl_take();
    if (T_ <= 256) {  // query-prefill sizes: one CTA row per token (measured faster at 64 tokens)
        const dim3 grid(row_ctas(hidden), T_);
        DISPATCH_DT(dt, launch_k(residual_kernel<T>, grid, 256, 0, s, x, partial, splits, plane, hidden, w, (T*)xb,
                                 ssp, err, tl));
    } else {
        const dim3 grid(row_ctas(hidden), (unsigned)std::min(T_, std::max(1, 148 * 4 / row_ctas(hidden))));
        DISPATCH_DT(dt, launch_k(residual_rows_kernel<T>, grid, 256, 0, s, x, partial, splits, plane, T_, hidden, w,
                                 (T*)xb, ssp, err, tl));
    }
    TKV_CUDA(cudaGetLastError());
}

void launch_swiglu(const float* partial, int splits, int T_, int inter, void* act, const float* ssp, int nb,
                   int hidden, float eps, DT dt, cudaStream_t s, int gu_block) {
    DISPATCH_DT(dt, launch_k(swiglu_kernel<T>, grid_for((int64_t)T_ * inter, 256), 256, 0, s, partial, splits, T_, inter, (T*)act, ssp, nb, hidden, eps, gu_block));
    TKV_CUDA(cudaGetLastError());
}

void launch_qkv_epilogue(const float* partial, int splits, int T_, int H, int Hkv, int d, const int32_t* pos,
                         const float2* rope, void* q, void* kc, void* vc, int row0, const StoreScatter& sc, int layer,
                         const float* ssp, int nb, int hidden, float eps, DT dt, cudaStream_t s, int64_t plane,
                         const EpiReq* reqs, int n_req) {
    const int64_t pairs = (int64_t)T_ * (H + 2 * Hkv) * d / 2;
    if (plane <= 0) plane = (int64_t)T_ * (H + 2 * Hkv) * d;
    unsigned long long* tl = tl_take();
    if (T_ <= 256) {  // query-prefill sizes: flat pair grid
        if (n_req > 0) {
            DISPATCH_DT(dt, launch_k(qkv_epilogue_flat_kernel<T, true>, grid_for(pairs, 256), 256, 0, s, partial, splits,
                                     T_, H, Hkv, d, pos, rope, (T*)q, (T*)kc, (T*)vc, row0, sc, layer, ssp, nb, hidden,
                                     eps, plane, tl, reqs, n_req));
        } else {
            DISPATCH_DT(dt, launch_k(qkv_epilogue_single_kernel<T>, grid_for(pairs, 256), 256, 0, s, partial, splits,
                                     T_, H, Hkv, d, pos, rope, (T*)q, (T*)kc, (T*)vc, row0, sc, layer, ssp, nb, hidden,
                                     eps, plane, tl));
        }
    } else {  // one CTA per token: the per-token prologue (row scale, position, request) once per token
        const dim3 grid(1u, (unsigned)std::min<int64_t>(T_, 65535));
        DISPATCH_DT(dt, launch_k(qkv_epilogue_kernel<T>, grid, 256, 0, s, partial, splits, T_, H, Hkv, d, pos, rope,
                                 (T*)q, (T*)kc, (T*)vc, row0, sc, layer, ssp, nb, hidden, eps, plane, tl, reqs, n_req));
    }
    TKV_CUDA(cudaGetLastError());
}

void launch_gather_rope(const PoolTable& pools, int page_tokens, const GatherSeg* segs, int n_segs, int L, int kvd,
                        int d, const float2* rope, void* cache, int64_t cap, int rotate, DT dt, int num_sms,
                        cudaStream_t s) {
    const int vecN = 16 / (int)dt_size(dt);
    const bool vec_ok = (kvd % vecN == 0) && (d % vecN == 0) && (page_tokens * kvd * (int)dt_size(dt)) % 16 == 0 &&
                        (cap * kvd * (int64_t)dt_size(dt)) % 16 == 0 && (GATHER_ROWS * kvd * (int)dt_size(dt)) % 16 == 0;
    const int n_units = n_segs * L * 2 * (vec_ok ? (page_tokens + GATHER_ROWS - 1) / GATHER_ROWS : 1);
    if (n_units == 0) return;
    const int grid = n_units < num_sms * GATHER_GRID_MULT ? n_units : num_sms * GATHER_GRID_MULT;
    if (vec_ok) {
        unsigned long long* tl = tl_take();
        DISPATCH_DT(dt, launch_k(gather_rope_vec_kernel<T>, grid, 256, 0, s, pools, page_tokens, segs, n_units, L,
                                                                       kvd, d, rope, (T*)cache, cap, rotate, tl));
    } else {
        DISPATCH_DT(dt, launch_k(gather_rope_pair_kernel<T>, grid, 256, 0, s, pools, page_tokens, segs, n_units, L,
                                                                        kvd, d, rope, (T*)cache, cap, rotate));
    }
    TKV_CUDA(cudaGetLastError());
}

void launch_lm_head(const void* h, const void* W, int hidden, int vocab, float* logits, const float* ssp, int nb,
                    float eps, DT dt, int* err, cudaStream_t s) {
    const int threads = 256, warps_per_block = threads / 32;
    unsigned long long* tl = tl_take();
    DISPATCH_DT(dt, launch_k(lm_head_kernel<T>, (vocab + warps_per_block - 1) / warps_per_block, threads, 0, s,
                        (const T*)h, (const T*)W, hidden, vocab, logits, ssp, nb, eps, err, tl));
    TKV_CUDA(cudaGetLastError());
}

void launch_mask_materialize(const int32_t* lo, const int32_t* hi, int rows, int cols, uint8_t* out, cudaStream_t s) {
    launch_k(mask_kernel, grid_for((int64_t)rows * cols, 256), 256, 0, s, lo, hi, rows, cols, out);
    TKV_CUDA(cudaGetLastError());
}

void launch_unrotate_rows(const void* k, int rows, int kvd, int d, const int32_t* pos, const float2* rope, float* out,
                          DT dt, cudaStream_t s) {
    DISPATCH_DT(dt, launch_k(unrotate_kernel<T>, grid_for((int64_t)rows * kvd / 2, 256), 256, 0, s, (const T*)k, rows, kvd,
                                                                                               d, pos, rope, out));
    TKV_CUDA(cudaGetLastError());
}

void launch_to_f32(const void* src, int64_t n, float* dst, DT dt, cudaStream_t s) {
    DISPATCH_DT(dt, launch_k(to_f32_kernel<T>, grid_for(n, 256), 256, 0, s, (const T*)src, n, dst));
    TKV_CUDA(cudaGetLastError());
}

void launch_from_f32(const float* src, int64_t n, void* dst, DT dt, cudaStream_t s) {
    DISPATCH_DT(dt, launch_k(from_f32_kernel<T>, grid_for(n, 256), 256, 0, s, src, n, (T*)dst));
    TKV_CUDA(cudaGetLastError());
}

void launch_reduce_splits(const float* partial, int splits, int64_t n, float* out, cudaStream_t s) {
    launch_k(reduce_splits_kernel, grid_for(n, 256), 256, 0, s, partial, splits, n, out);
    TKV_CUDA(cudaGetLastError());
}

}  // namespace tkv

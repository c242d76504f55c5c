// Flash attention with implicit TurboRAG masks (SIMT, fp32 math), split-K over keys.
// Replaces attend + softmax_rows_inplace (src/attention.cpp:94-169, src/numerics.cpp:31-60) and the
// dense masks of build_mask / causal_rows (attention.cpp:50-92): row t sees key j iff lo[t] <= j <= hi[t].
//   query prefill      : lo = 0,          hi = P + t         (causal_rows(q, P))
//   naive causal       : lo = 0,          hi = t
//   naive independent  : lo = seg_start,  hi = t  for chunk rows, lo = 0 for query rows
//   block-diagonal chunk ingest: lo = chunk start, hi = t
// GQA: a CTA owns 32 (token, head) rows of ONE kv group, so every K/V tile staged in shared memory
// is reused by all `group` heads ("GQA packs tokens x heads into M").
// Layout: 4 lanes per row, each holding d/4 interleaved elements (conflict-free smem reads).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include <type_traits>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int ROWS = 32, LPR = 4, THREADS = ROWS * LPR, KT = 32;

__device__ __forceinline__ float ld(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void st(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

template <typename T, int D>
__global__ void __launch_bounds__(THREADS) attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                            const T* __restrict__ v, int kv_stride,
                                                            const int32_t* __restrict__ lo,
                                                            const int32_t* __restrict__ hi, T* __restrict__ out,
                                                            float* __restrict__ ws_o, float* __restrict__ ws_ml,
                                                            int Tq, int Tk, int H, int Hkv, int splits, float scale,
                                                            int* err) {
    pdl_launch();
    pdl_wait();
    constexpr int E = D / LPR;
    __shared__ float Ks[KT][D];
    __shared__ float Vs[KT][D];
    __shared__ int red_lo[THREADS / 32], red_hi[THREADS / 32];

    const int group = H / Hkv, g = blockIdx.y, split = blockIdx.z;
    const int rl = threadIdx.x / LPR, qq = threadIdx.x % LPR;
    const int r = blockIdx.x * ROWS + rl;
    const bool active = r < Tq * group;
    const int t = active ? r / group : 0;
    const int h = g * group + (active ? r % group : 0);
    const int my_lo = active ? lo[t] : INT32_MAX;
    const int my_hi = active ? min(hi[t], Tk - 1) : -1;

    // CTA key range = union of its rows' ranges, then this split's share of it.
    int blo = my_lo, bhi = my_hi;
    for (int o = 16; o > 0; o >>= 1) {
        blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
        bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red_lo[threadIdx.x >> 5] = blo;
        red_hi[threadIdx.x >> 5] = bhi;
    }
    __syncthreads();
    blo = red_lo[0];
    bhi = red_hi[0];
    for (int w = 1; w < THREADS / 32; ++w) {
        blo = min(blo, red_lo[w]);
        bhi = max(bhi, red_hi[w]);
    }
    blo = max(blo, 0);
    const int span = bhi - blo + 1;
    const int chunk = span > 0 ? ((span + splits - 1) / splits + KT - 1) / KT * KT : 0;
    const int ks = blo + split * chunk, ke = min(bhi, ks + chunk - 1);

    float qv[E], o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        qv[e] = active ? ld(q, (int64_t)t * H * D + h * D + e * LPR + qq) : 0.f;
        o[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;

    for (int k0 = ks; k0 <= ke; k0 += KT) {
        __syncthreads();
        for (int i = threadIdx.x; i < KT * D; i += THREADS) {
            const int j = i / D, c = i % D, key = k0 + j;
            const bool in = key <= ke;
            Ks[j][c] = in ? ld(k, (int64_t)key * kv_stride + g * D + c) : 0.f;
            Vs[j][c] = in ? ld(v, (int64_t)key * kv_stride + g * D + c) : 0.f;
        }
        __syncthreads();
        float s[KT];
        float mt = -INFINITY;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            float dot = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) dot = fmaf(qv[e], Ks[j][e * LPR + qq], dot);
            dot += __shfl_xor_sync(0xffffffffu, dot, 1);
            dot += __shfl_xor_sync(0xffffffffu, dot, 2);
            const int key = k0 + j;
            const bool vis = key <= ke && key >= my_lo && key <= my_hi;
            s[j] = vis ? dot * scale : -INFINITY;
            mt = fmaxf(mt, s[j]);
        }
        const float mn = fmaxf(m, mt);
        if (mn == -INFINITY) continue;  // nothing visible yet for this row
        const float alpha = (m == -INFINITY) ? 0.f : expf(m - mn);
        l *= alpha;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] *= alpha;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const float p = (s[j] == -INFINITY) ? 0.f : expf(s[j] - mn);
            l += p;
#pragma unroll
            for (int e = 0; e < E; ++e) o[e] = fmaf(p, Vs[j][e * LPR + qq], o[e]);
        }
        m = mn;
    }
    if (!active) return;
    const int64_t row = (int64_t)t * H + h;
    if (splits == 1) {
        if (l == 0.f) {  // DegenerateRowError (numerics.cpp:39-42)
            if (qq == 0) atomicOr(err, 8);
            return;
        }
        const float inv = 1.0f / l;
#pragma unroll
        for (int e = 0; e < E; ++e) st(out, row * D + e * LPR + qq, o[e] * inv);
    } else {
        float* wo = ws_o + ((int64_t)split * Tq * H + row) * D;
#pragma unroll
        for (int e = 0; e < E; ++e) wo[e * LPR + qq] = o[e];
        if (qq == 0) {
            ws_ml[((int64_t)split * Tq * H + row) * 2 + 0] = m;
            ws_ml[((int64_t)split * Tq * H + row) * 2 + 1] = l;
        }
    }
}

// Split-K merge, one warp per (token, head) row: lane s < splits holds split s's (m, l); every lane then
// accumulates its d-columns over the splits with the broadcast weights exp(m_s - max).
template <typename T>
__global__ void attn_combine_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_ml, int rows, int D,
                                    int splits, T* __restrict__ out, int* err) {
    pdl_launch();
    pdl_wait();
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float ms = -INFINITY, ls = 0.f;
    if (lane < splits) {
        ms = ws_ml[((int64_t)lane * rows + row) * 2];
        ls = ws_ml[((int64_t)lane * rows + row) * 2 + 1];
    }
    float mx = ms;
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (mx == -INFINITY) {  // DegenerateRowError (numerics.cpp:39-42)
        if (lane == 0) atomicOr(err, 8);
        return;
    }
    const float w = (ms == -INFINITY) ? 0.f : expf(ms - mx);
    float L = ls * w;
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    const float inv = 1.0f / L;
    if (D == 128) {  // lane owns 4 consecutive columns: one float4 per split, loads batched
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* src = reinterpret_cast<const float4*>(ws_o) + row * 32 + lane;
#pragma unroll
        for (int s = 0; s < 32; ++s) {  // all split loads in flight at once (splits <= 32)
            const float ws = __shfl_sync(0xffffffffu, w, s);
            const float4 v = s < splits ? src[(int64_t)s * rows * 32] : make_float4(0.f, 0.f, 0.f, 0.f);
            acc.x = fmaf(v.x, ws, acc.x);
            acc.y = fmaf(v.y, ws, acc.y);
            acc.z = fmaf(v.z, ws, acc.z);
            acc.w = fmaf(v.w, ws, acc.w);
        }
        const int64_t b = row * D + lane * 4;
        st(out, b + 0, acc.x * inv);
        st(out, b + 1, acc.y * inv);
        st(out, b + 2, acc.z * inv);
        st(out, b + 3, acc.w * inv);
        return;
    }
    for (int c0 = 0; c0 < D; c0 += 32) {
        const int c = c0 + lane;
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) {
            const float ws = __shfl_sync(0xffffffffu, w, s);
            if (ws != 0.f && c < D) acc = fmaf(ws_o[((int64_t)s * rows + row) * D + c], ws, acc);
        }
        if (c < D) st(out, row * D + c, acc * inv);
    }
}

template <typename T, int D>
void launch_d(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo, const int32_t* hi,
              void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws, int* err, cudaStream_t s) {
    const int group = H / Hkv;
    dim3 grid((Tq * group + ROWS - 1) / ROWS, Hkv, splits);
    const float scale = (float)(1.0 / sqrt((double)D));
    launch_k(attn_simt_kernel<T, D>, grid, THREADS, 0, s, (const T*)q, (const T*)k, (const T*)v, kv_stride, lo, hi, (T*)out,
                                                    ws.o, ws.ml, Tq, Tk, H, Hkv, splits, scale, err);
    TKV_CUDA(cudaGetLastError());
    if (splits > 1) launch_attention_combine(ws, Tq * H, D, splits, out, err, std::is_same<T, float>::value ? DT::F32 : DT::BF16, s);
}

template <typename T>
void launch_t(int d, const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo, const int32_t* hi,
              void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws, int* err, cudaStream_t s) {
    switch (d) {
        case 8: return launch_d<T, 8>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
        case 16: return launch_d<T, 16>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
        case 32: return launch_d<T, 32>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
        case 64: return launch_d<T, 64>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
        case 128: return launch_d<T, 128>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
        default: fail(TKV_ERR_CONFIG, "head_size " + std::to_string(d) + " not supported (8/16/32/64/128)");
    }
}

}  // namespace

void launch_attention_combine(const AttnWork& ws, int rows, int d, int splits, void* out, int* err, DT dt,
                              cudaStream_t s) {
    const int grid = (int)(((int64_t)rows * 32 + 255) / 256);
    if (dt == DT::F32)
        launch_k(attn_combine_kernel<float>, grid, 256, 0, s, ws.o, ws.ml, rows, d, splits, (float*)out, err);
    else
        launch_k(attn_combine_kernel<__nv_bfloat16>, grid, 256, 0, s, ws.o, ws.ml, rows, d, splits, (__nv_bfloat16*)out, err);
    TKV_CUDA(cudaGetLastError());
}

size_t attn_workspace_floats(int Tq, int H, int d, int splits) {
    return splits <= 1 ? 0 : (size_t)splits * Tq * H * (d + 2);
}

int attn_pick_splits(int Tq, int H, int Hkv, int Tk, int num_sms) {
    const int group = H / Hkv;
    const int ctas = ((Tq * group + ROWS - 1) / ROWS) * Hkv;
    int s = (2 * num_sms + ctas - 1) / ctas;
    const int max_by_keys = (Tk + 255) / 256;  // keep >= 256 keys per split
    if (s > max_by_keys) s = max_by_keys;
    if (s > 32) s = 32;
    return s < 1 ? 1 : s;
}

void launch_attention_simt(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                           const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int d, int splits,
                           const AttnWork& ws, int* err, DT dt, cudaStream_t s) {
    if (dt == DT::F32)
        launch_t<float>(d, q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
    else
        launch_t<__nv_bfloat16>(d, q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s);
}

}  // namespace tkv

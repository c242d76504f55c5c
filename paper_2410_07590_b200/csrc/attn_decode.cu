// Decode-sized attention (bf16, head_size 128): R = Tq * group <= 16 query rows per kv head — the last layer
// of a query prefill keeps one token, greedy decode steps (model.cpp:274-303, mask causal_rows(1, total)) have
// one. Replaces attend + softmax_rows_inplace (src/attention.cpp:94-169, src/numerics.cpp:31-60) where a
// 128-row tcgen05 tile would be at most 1/8 full.
//
// The work is streaming the layer's K/V (C2: 16.9 MB), so this is a split-K flash-decoding pass whose math must
// stay off the issue port: the R rows (padded to 16) are the M side of warp-level m16n8k16 bf16 MMAs, so the
// per-key cost is two MMAs instead of ~130 SIMT instructions (the SIMT version issued at IPC 2 and never got
// past 0.8 TB/s).
//   grid = (kv head, key split), WARPS warps per CTA, each warp owns a strided set of 16-key blocks.
//   Fragments come straight from global memory, no shared-memory staging:
//     S = Q K^T: the contraction index d is permuted so a lane's K B-fragment for key (lane / 4) is one 16-byte
//       load per two k-steps (d = 32 j + 8 (lane % 4) + 4 h + e); Q's A-fragment uses the same permutation.
//     O += P V: P is the S accumulator re-packed to bf16 (the flash-attention register reuse); V's B-fragment
//       pairs two keys per register, built with byte permutes from 16-byte row loads; the output column n of
//       n-tile nt maps to d = 8 n + nt (nt < 8) or 64 + 8 n + nt - 8.
// Warp partials (o, m, l) are merged in shared memory in warp order (deterministic), CTA partials by
// launch_attention_combine (natural-log m).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int D = 128, KBLK = 16, WARPS = 8, THREADS = WARPS * 32;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t word(const uint4& u, int w) {
    return w == 0 ? u.x : w == 1 ? u.y : w == 2 ? u.z : u.w;
}

__device__ __forceinline__ int out_col(int nt, int n) { return nt < 8 ? 8 * n + nt : 64 + 8 * n + nt - 8; }

template <int R>
__global__ void __launch_bounds__(THREADS) attn_decode_kernel(const __nv_bfloat16* __restrict__ q,
                                                              const __nv_bfloat16* __restrict__ k,
                                                              const __nv_bfloat16* __restrict__ v, int kv_stride,
                                                              const int32_t* __restrict__ lo,
                                                              const int32_t* __restrict__ hi,
                                                              __nv_bfloat16* __restrict__ out, float* __restrict__ ws_o,
                                                              float* __restrict__ ws_ml, int Tq, int Tk, int H, int Hkv,
                                                              int splits, float scale, int* err) {
    pdl_launch();
    __shared__ float so[R][D];
    __shared__ float sm_m[WARPS][16], sm_l[WARPS][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, cq = lane & 3;
    const int group = H / Hkv, g = blockIdx.x, split = blockIdx.y;
    for (int i = threadIdx.x; i < R * D; i += THREADS) (&so[0][0])[i] = 0.f;
    pdl_wait();
    // this lane's two rows: gq and gq + 8 (rows >= R are zero padding, never written)
    int rlo[2], rhi[2];
    uint32_t qa[8][4];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        const int r = gq + 8 * h2;
        const bool valid = r < R;
        const int t = valid ? r / group : 0, h = g * group + (valid ? r % group : 0);
        rlo[h2] = max(lo[t], 0);
        rhi[h2] = min(hi[t], Tk - 1);
        const __nv_bfloat16* qr = q + ((int64_t)t * H + h) * D;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint2 u = make_uint2(0u, 0u);
            if (valid) u = *reinterpret_cast<const uint2*>(qr + 32 * (kk >> 1) + 8 * cq + 4 * (kk & 1));
            qa[kk][h2] = u.x;      // a0 / a1: k = 2 cq + {0, 1}
            qa[kk][2 + h2] = u.y;  // a2 / a3: k = 8 + 2 cq + {0, 1}
        }
    }
    int blo = INT32_MAX, bhi = -1;
    for (int r = 0; r < R; ++r) {
        const int t = r / group;
        blo = min(blo, max(lo[t], 0));
        bhi = max(bhi, min(hi[t], Tk - 1));
    }
    const int span = bhi - blo + 1;
    const int per = span > 0 ? ((span + splits - 1) / splits + KBLK - 1) / KBLK * KBLK : 0;
    const int ks = blo + split * per, ke = min(bhi + 1, ks + per);  // keys [ks, ke)
    const float sl2 = scale * LOG2E;
    float o[16][4], m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    const __nv_bfloat16* kb = k + g * D;
    const __nv_bfloat16* vb = v + g * D;
    for (int k0 = ks + warp * KBLK; k0 < ke; k0 += WARPS * KBLK) {
        uint4 kr[2][4], vr[4][2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int key = min(k0 + 8 * t + gq, Tk - 1);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                kr[t][j] = __ldcs(reinterpret_cast<const uint4*>(kb + (int64_t)key * kv_stride + 32 * j + 8 * cq));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // keys 2cq, 2cq + 1, 8 + 2cq, 9 + 2cq of the block
            const int key = min(k0 + 8 * (i >> 1) + 2 * cq + (i & 1), Tk - 1);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
                vr[i][hf] = __ldcs(reinterpret_cast<const uint4*>(vb + (int64_t)key * kv_stride + 64 * hf + 8 * gq));
        }
        float sc[2][4];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint4& u = kr[t][kk >> 1];
                mma16816(sc[t], qa[kk], (kk & 1) ? u.z : u.x, (kk & 1) ? u.w : u.y);
            }
        }
        // online softmax; sc[t][2 h2 + e] = row gq + 8 h2, key k0 + 8 t + 2 cq + e
        float alpha[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            float mx = -INFINITY;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int key = k0 + 8 * t + 2 * cq + e;
                    float x = sc[t][2 * h2 + e] * sl2;
                    if (key >= ke || key < rlo[h2] || key > rhi[h2]) x = -INFINITY;
                    sc[t][2 * h2 + e] = x;
                    mx = fmaxf(mx, x);
                }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float mn = fmaxf(m[h2], mx);
            const float moff = mn == -INFINITY ? 0.f : mn;
            alpha[h2] = m[h2] == -INFINITY ? 0.f : exp2f(m[h2] - moff);
            float ps = 0.f;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float p = exp2f(sc[t][2 * h2 + e] - moff);
                    sc[t][2 * h2 + e] = p;
                    ps += p;
                }
            l[h2] = l[h2] * alpha[h2] + ps;
            m[h2] = mn;
        }
        const uint32_t pa[4] = {pack_bf16(sc[0][0], sc[0][1]), pack_bf16(sc[0][2], sc[0][3]),
                                pack_bf16(sc[1][0], sc[1][1]), pack_bf16(sc[1][2], sc[1][3])};
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            o[nt][0] *= alpha[0];
            o[nt][1] *= alpha[0];
            o[nt][2] *= alpha[1];
            o[nt][3] *= alpha[1];
            const int hf = nt >> 3, w = (nt & 7) >> 1;
            const uint32_t sel = (nt & 1) ? 0x7632u : 0x5410u;  // pair the two keys' bf16 at column 8 gq + nt
            const uint32_t b0 = __byte_perm(word(vr[0][hf], w), word(vr[1][hf], w), sel);
            const uint32_t b1 = __byte_perm(word(vr[2][hf], w), word(vr[3][hf], w), sel);
            mma16816(o[nt], pa, b0, b1);
        }
    }
    // quad-reduce l, then merge the warps' (o, m, l) in warp order
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        l[h2] += __shfl_xor_sync(0xffffffffu, l[h2], 1);
        l[h2] += __shfl_xor_sync(0xffffffffu, l[h2], 2);
        if (cq == 0) {
            sm_m[warp][gq + 8 * h2] = m[h2];
            sm_l[warp][gq + 8 * h2] = l[h2];
        }
    }
    __syncthreads();
    float f[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        const int r = gq + 8 * h2;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm_m[w][r]);
        f[h2] = m[h2] == -INFINITY ? 0.f : exp2f(m[h2] - M);
    }
    for (int w = 0; w < WARPS; ++w) {
        if (warp == w) {
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int r = gq + 8 * h2;
                if (r < R) {
#pragma unroll
                    for (int nt = 0; nt < 16; ++nt) {
                        so[r][out_col(nt, 2 * cq)] += o[nt][2 * h2] * f[h2];
                        so[r][out_col(nt, 2 * cq + 1)] += o[nt][2 * h2 + 1] * f[h2];
                    }
                }
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < R * D; i += THREADS) {
        const int r = i / D, c = i % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm_m[w][r]);
        float L = 0.f;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) L += sm_m[w][r] == -INFINITY ? 0.f : sm_l[w][r] * exp2f(sm_m[w][r] - M);
        const float acc = so[r][c];
        const int t = r / group, h = g * group + r % group;
        const int64_t orow = (int64_t)t * H + h;
        if (splits == 1) {
            if (L == 0.f) {
                if (c == 0) atomicOr(err, 8);  // DegenerateRowError (numerics.cpp:39-42)
            } else {
                out[orow * D + c] = __float2bfloat16_rn(acc / L);
            }
        } else {
            ws_o[((int64_t)split * Tq * H + orow) * D + c] = acc;
            if (c == 0) {
                ws_ml[((int64_t)split * Tq * H + orow) * 2 + 0] = M == -INFINITY ? -INFINITY : M / LOG2E;
                ws_ml[((int64_t)split * Tq * H + orow) * 2 + 1] = L;
            }
        }
    }
}

template <int R>
void launch_r(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo, const int32_t* hi,
              void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws, int* err, cudaStream_t s) {
    const float scale = (float)(1.0 / sqrt((double)D));
    launch_k(attn_decode_kernel<R>, dim3(Hkv, splits), dim3(THREADS), 0, s, (const __nv_bfloat16*)q,
             (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, kv_stride, lo, hi, (__nv_bfloat16*)out, ws.o, ws.ml, Tq,
             Tk, H, Hkv, splits, scale, err);
}

}  // namespace

bool attention_decode_supported(int Tq, int H, int Hkv, int d, DT dt) {
    const int R = Tq * (H / Hkv);
    return dt == DT::BF16 && d == D && (R == 4 || R == 7 || R == 8 || R == 16);
}

int attn_decode_pick_splits(int Tk, int Hkv, int num_sms) {
    int s = 2 * ((num_sms + Hkv - 1) / Hkv);  // ~2 CTAs per SM
    const int by_keys = (Tk + 2 * WARPS * KBLK - 1) / (2 * WARPS * KBLK);  // >= ~2 key blocks per warp
    if (s > by_keys) s = by_keys;
    if (s > 32) s = 32;  // launch_attention_combine merges up to 32 splits (one warp lane each)
    return s < 1 ? 1 : s;
}

void launch_attention_decode(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                             const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int splits,
                             const AttnWork& ws, int* err, cudaStream_t s) {
    if (splits > 1 && !ws.o) fail(TKV_ERR_CONFIG, "decode attention split-K needs its workspace");
    switch (Tq * (H / Hkv)) {
        case 4: launch_r<4>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s); break;
        case 7: launch_r<7>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s); break;
        case 8: launch_r<8>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s); break;
        case 16: launch_r<16>(q, k, v, kv_stride, lo, hi, out, Tq, Tk, H, Hkv, splits, ws, err, s); break;
        default: fail(TKV_ERR_CONFIG, "decode attention: unsupported rows per kv head");
    }
    TKV_CUDA(cudaGetLastError());
    if (splits > 1) launch_attention_combine(ws, Tq * H, D, splits, out, err, DT::BF16, s);
}

}  // namespace tkv

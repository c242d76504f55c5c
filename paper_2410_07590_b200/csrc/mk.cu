// Persistent layer kernel for query-sized forwards (<= 128 tokens, bf16): everything between two attention launches
// of forward_tokens (src/model.cpp:240-264) in ONE grid of one CTA per SM --
//
//   O-projection -> residual + RMSNorm -> gate/up + SwiGLU -> down -> residual + RMSNorm -> next layer's QKV ->
//   QKV epilogue (split-K reduce, RoPE, q + request-cache K/V rows)
//
// At batch 1 these projections stream every weight once per request (HBM-bound: 466 MB per Qwen2-7B layer). As
// separate kernels each GEMM pays a ramp and a tail and every epilogue kernel a launch on the critical path. Here the
// weight stream never stops at a phase boundary: the W-producer thread streams the weight tiles of ALL of this CTA's
// units of all phases back to back into the smem ring (weights do not depend on anything), bounded only by the ring;
// a separate A-producer issues each stage's activation tile once the phase it depends on has completed grid-wide.
// Phase completion = a monotone per-phase counter in global memory that every CTA increments (release) when its part
// of the phase is written; consumers acquire it. The grid is exactly one CTA per SM (> half the SM's shared memory),
// so every CTA is resident and the software barriers cannot deadlock (a dependent grid launches only once every CTA
// of this one runs, and cannot share an SM with it). Waits trap after ~2 s instead of hanging. Requirement: one
// layer-kernel grid on a GPU at a time (two engines' streams on one device must not run them concurrently).
//
// Roles (352 threads): warp 0 = W-producer (TMA, L2 evict_first), warp 1 = A-producer (TMA after the phase
// dependency), warp 2 = TMEM owner + MMA issuer (tcgen05.mma kind::f16, swap-AB: weights on the M = 128 side,
// tokens as N), warps 3-10 = workers: TMEM epilogues (lane group = warp % 4) and the element-wise phases.
//
// Numerics are those of the multi-kernel path (gemm_tc.cu swapped tiling, kernels.cu residual / QKV epilogue): the
// same unit partition, k-block order and split-K summation order, so the two paths agree bit for bit
// (tests/test_gpu_parity_large.py::test_layer_kernel_bitwise_equals_kernel_chain).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "dev_common.cuh"
#include "tc_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {
using namespace tc;

constexpr int BK = 64;
constexpr uint32_t TILE_W = 128 * BK * 2;  // 16 KB: 128 weight rows x 64 k, bf16
constexpr int XC = 32;                     // SwiGLU epilogue: token columns per gate/up exchange pass
constexpr int WORKERS = 256;               // 8 worker warps: TMEM epilogues (two per lane group) + element-wise phases
constexpr int THREADS = 96 + WORKERS;
constexpr int EPI0 = 96;                   // first worker thread
constexpr int kSmemBudget = 220 * 1024;

struct MkMaps {
    CUtensorMap m[MK_MAX_MAPS];
};
using bf16 = __nv_bfloat16;

__device__ __forceinline__ float silu(float z) { return z / (1.0f + __expf(-z)); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }     // all workers
__device__ __forceinline__ void swiglu_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }  // workers 0-127

template <typename V>
__device__ __forceinline__ void add_to(V& a, const V& b);
template <>
__device__ __forceinline__ void add_to<float2>(float2& a, const float2& b) { a.x += b.x, a.y += b.y; }
template <>
__device__ __forceinline__ void add_to<float4>(float4& a, const float4& b) { a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w; }
// split-K partial sums in ascending split order with SB loads in flight (kernels.cu:sum_splits, same order)
template <typename V, int SB>
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

// x[t][blk] += sum_s partial[s][t][blk]; xb = x * w; ssp[t][blk] = sum of squares (kernels.cu:residual_kernel):
// one warp per (token, 128-column block), the same per-lane columns, split order and shuffle tree
__device__ __forceinline__ void residual_finish(const MkArgs& a, const float* w, int t, int blk, int lane, float4 s4) {
    const int hidden = a.hidden, c0 = blk * 128 + lane * 4;
    float* xrow = a.x + (int64_t)t * hidden;
    const float v[4] = {s4.x, s4.y, s4.z, s4.w};
    float ss = 0.f;
    bool bad = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        xrow[c0 + e] = v[e];
        ((bf16*)a.xb)[(int64_t)t * hidden + c0 + e] = __float2bfloat16_rn(v[e] * w[c0 + e]);
        ss += v[e] * v[e];
        bad |= !isfinite(v[e]);
    }
    if (bad) atomicOr(a.err, 2);
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) a.ssp[(int64_t)t * a.nb + blk] = ss;
}
__device__ void residual_phase(const MkArgs& a, const MkPhase& ph, int ew, int lane) {
    const int nb = a.nb, M = a.M, hidden = a.hidden, n_items = a.M * nb;
    const int64_t plane = (int64_t)M * hidden;
    const int stride = gridDim.x * (WORKERS / 32);
    for (int item = blockIdx.x * (WORKERS / 32) + ew; item < n_items; item += 2 * stride) {
        // two items per warp in flight: every partial load of both issued before the first add
        const int it2 = item + stride;
        const int t0 = item / nb, b0 = item - t0 * nb;
        const int t1 = it2 < n_items ? it2 / nb : t0, b1 = it2 < n_items ? it2 - t1 * nb : b0;
        const float* p0 = ph.rpartial + (int64_t)t0 * hidden + b0 * 128 + lane * 4;
        const float* p1 = ph.rpartial + (int64_t)t1 * hidden + b1 * 128 + lane * 4;
        float4 acc0 = *reinterpret_cast<const float4*>(a.x + (int64_t)t0 * hidden + b0 * 128 + lane * 4);
        float4 acc1 = *reinterpret_cast<const float4*>(a.x + (int64_t)t1 * hidden + b1 * 128 + lane * 4);
        for (int s0 = 0; s0 < ph.rsplits; s0 += 8) {
            float4 v0[8], v1[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (s0 + i < ph.rsplits) {
                    v0[i] = *reinterpret_cast<const float4*>(p0 + (int64_t)(s0 + i) * plane);
                    v1[i] = *reinterpret_cast<const float4*>(p1 + (int64_t)(s0 + i) * plane);
                }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (s0 + i < ph.rsplits) {
                    add_to(acc0, v0[i]);
                    add_to(acc1, v1[i]);
                }
        }
        residual_finish(a, ph.rw, t0, b0, lane, acc0);
        if (it2 < n_items) residual_finish(a, ph.rw, t1, b1, lane, acc1);
    }
}

// reduce the QKV split-K partials, rotate q and k by pos[t] (interleaved pairs), write q and the request-cache rows
// (kernels.cu:qkv_epilogue_kernel, same arithmetic per element pair)
__device__ void qkv_epi_phase(const MkArgs& a, int et) {
    const int qd = a.H * a.d, kvd = a.Hkv * a.d, N = qd + 2 * kvd, half = a.d / 2;
    const int64_t pairs = (int64_t)a.M * (N / 2), plane = (int64_t)a.M * N;
    constexpr int P = 2;  // pairs per thread in flight (all their split loads issued before the adds)
    const int64_t stride = (int64_t)gridDim.x * WORKERS;
    for (int64_t p0 = blockIdx.x * WORKERS + et; p0 < pairs; p0 += P * stride) {
        float2 acc[P];
        int64_t tt[P];
        int nn[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int64_t p = min(p0 + j * stride, pairs - 1);
            tt[j] = p / (N / 2);
            nn[j] = 2 * (int)(p - tt[j] * (N / 2));
            acc[j] = make_float2(0.f, 0.f);
        }
        for (int s0 = 0; s0 < a.qsplits; s0 += 8) {
            float2 v[P][8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if (s0 + i < a.qsplits)
                        v[j][i] = *reinterpret_cast<const float2*>(a.qpartial + tt[j] * N + nn[j] + (int64_t)(s0 + i) * plane);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if (s0 + i < a.qsplits) add_to(acc[j], v[j][i]);
        }
#pragma unroll
        for (int j = 0; j < P; ++j) {
            if (p0 + j * stride >= pairs) break;
            const int64_t t = tt[j];
            const int n = nn[j];
            const float rs = row_scale(a.ssp, a.nb, t, a.hidden, a.eps);
            float x0 = acc[j].x, x1 = acc[j].y;
            x0 *= rs;
            x1 *= rs;
            if (n >= qd + kvd) {
                const int c = n - qd - kvd;
                ((bf16*)a.vc)[(int64_t)(a.row0 + t) * kvd + c] = __float2bfloat16_rn(x0);
                ((bf16*)a.vc)[(int64_t)(a.row0 + t) * kvd + c + 1] = __float2bfloat16_rn(x1);
                continue;
            }
            const int e = (n < qd ? n : n - qd) % a.d;
            const float2 cs = a.rope[(int64_t)a.pos[t] * half + e / 2];
            const float r0 = x0 * cs.x - x1 * cs.y, r1 = x0 * cs.y + x1 * cs.x;  // rope.cpp:41-44
            if (n < qd) {
                ((bf16*)a.q)[t * qd + n] = __float2bfloat16_rn(r0);
                ((bf16*)a.q)[t * qd + n + 1] = __float2bfloat16_rn(r1);
            } else {
                const int c = n - qd;
                ((bf16*)a.kc)[(int64_t)(a.row0 + t) * kvd + c] = __float2bfloat16_rn(r0);
                ((bf16*)a.kc)[(int64_t)(a.row0 + t) * kvd + c + 1] = __float2bfloat16_rn(r1);
            }
        }
    }
}

// unit u of a GEMM phase: n-tile nt, split z; k-blocks [k0, k0 + nkb) in the rotated order of gemm_tc.cu (krot)
struct Unit {
    int nt, z, k0, nkb, rot;
};
__device__ __forceinline__ Unit unit_of(const MkGemm& g, int u, int krot) {
    Unit r;
    r.z = u / g.n_tiles;
    r.nt = u - r.z * g.n_tiles;
    r.k0 = r.z * g.kb_per_split;
    r.nkb = min(g.kb_total, r.k0 + g.kb_per_split) - r.k0;
    r.rot = krot ? (u * 37) % r.nkb : 0;
    return r;
}

__device__ __forceinline__ void stamp(const MkArgs& a, int slot) {
    if (a.trace) a.trace[blockIdx.x * 32 + slot] = globaltimer_ns();
}

// walks this CTA's weight tiles in stream order: GEMM phases, units cta, cta + grid, ..., k-blocks
struct WCursor {
    const MkArgs& a;
    int cta, grid, p, u, i;
    Unit un;
    __device__ WCursor(const MkArgs& args, int c, int g) : a(args), cta(c), grid(g), p(-1), u(0), i(0) { next_unit(true); }
    __device__ bool valid() const { return p < a.n_phases; }
    __device__ void next_unit(bool first) {
        if (!first) u += grid;
        while (true) {
            if (p >= 0 && p < a.n_phases && a.ph[p].kind == MK_GEMM && u < a.ph[p].g.units) {
                un = unit_of(a.ph[p].g, u, a.krot);
                i = 0;
                return;
            }
            ++p;
            u = cta;
            if (p >= a.n_phases) return;
        }
    }
    __device__ void advance() {
        if (++i >= un.nkb) next_unit(false);
    }
    __device__ int map() const { return a.ph[p].g.map_w; }
    __device__ int kcoord() const { return (un.k0 + (i + un.rot) % un.nkb) * BK; }
    __device__ int ncoord() const { return un.nt * 128; }
    __device__ void prefetch_next(const MkMaps& maps) {
        if (!valid()) return;
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&maps.m[map()])),
                     "r"(kcoord()), "r"(ncoord())
                     : "memory");
        advance();
    }
};

__global__ void __launch_bounds__(THREADS, 1) mk_kernel(const __grid_constant__ MkMaps maps, const __grid_constant__ MkArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t stage_bytes = TILE_W + a.a_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;  // [2] accumulator ready
    uint64_t* tempty = tfull + 2;        // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x, grid = gridDim.x;
    // Dependents may launch as soon as every CTA of this grid runs (so all of them are resident and the phase
    // barriers below cannot starve); they cannot share an SM with this CTA's shared memory anyway.
    pdl_launch();

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], WORKERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < a.n_maps; ++i)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[i])) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- W-producer: the weight stream of every unit of every phase, never waiting on data ----
            const uint64_t pol = policy_evict_first();
            // a second cursor runs a.l2_ahead tiles ahead of the ring and pulls them into L2, so HBM keeps streaming
            // while a phase barrier holds the ring full (bounded: ~l2_ahead x 16 KB per SM of L2)
            WCursor pf(a, cta, grid);
            for (int k = 0; k < a.l2_ahead + a.stages; ++k) pf.prefetch_next(maps);
            WCursor cur(a, cta, grid);
            for (int it = 0; cur.valid(); ++it) {
                const int s = it % a.stages;
                mbar_wait(&empty[s], ((uint32_t)(it / a.stages) & 1u) ^ 1u);
                mbar_expect_tx(&full[s], stage_bytes);  // W + A bytes: the A-producer completes the rest
                tma_load_2d_hint(smem + s * stage_bytes, &maps.m[cur.map()], &full[s], cur.kcoord(), cur.ncoord(), pol);
                cur.advance();
                pf.prefetch_next(maps);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- A-producer: activation tiles once the phase's inputs exist grid-wide ----
            int it = 0;
            for (int p = 0; p < a.n_phases; ++p) {
                if (a.ph[p].kind != MK_GEMM) continue;
                if (p == 0) pdl_wait();  // the previous kernel (attention merge / embed) produced the A operand
                else if (!a.nodep) wait_counter(&a.bar[a.ph[p - 1].slot], a.ph[p - 1].target);
                stamp(a, 8 + p);
                const MkGemm& g = a.ph[p].g;
                for (int u = cta; u < g.units; u += grid) {
                    const Unit un = unit_of(g, u, a.krot);
                    for (int i = 0; i < un.nkb; ++i, ++it) {
                        const int s = it % a.stages;
                        mbar_wait(&empty[s], ((uint32_t)(it / a.stages) & 1u) ^ 1u);
                        tma_load_2d(smem + s * stage_bytes + TILE_W, &maps.m[g.map_a], &full[s],
                                    (un.k0 + (i + un.rot) % un.nkb) * BK, 0);
                    }
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // ---- MMA issuer ----
            const uint32_t id = idesc(128, a.ntok);
            int it = 0, lu = 0;
            for (int p = 0; p < a.n_phases; ++p) {
                if (a.ph[p].kind != MK_GEMM) continue;
                const MkGemm& g = a.ph[p].g;
                for (int u = cta; u < g.units; u += grid, ++lu) {
                    const Unit un = unit_of(g, u, a.krot);
                    const int b = lu & 1;
                    mbar_wait(&tempty[b], ((uint32_t)(lu >> 1) & 1u) ^ 1u);
                    fence_after();
                    const uint32_t acc = tmem + (uint32_t)(b * a.ntok);
                    for (int i = 0; i < un.nkb; ++i, ++it) {
                        const int s = it % a.stages;
                        mbar_wait(&full[s], (uint32_t)(it / a.stages) & 1u);
                        fence_after();
                        const uint32_t w = smem_u32(smem + s * stage_bytes), x = w + TILE_W;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_f16(acc, desc_k(w + k * 32), desc_k(x + k * 32), id, (i | k) != 0);
                        umma_commit(&empty[s]);
                    }
                    umma_commit(&tfull[b]);
                }
            }
        }
    } else {
        // ---- worker warps 3-10: TMEM epilogues (lane group warp % 4; two warps per group split the token
        // columns; the SwiGLU exchange runs on the first four) + the element-wise phases ----
        const int lg = warp & 3, ew = warp - 3, et = threadIdx.x - EPI0, half_id = et >> 7;
        const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
        pdl_wait();  // the residual stream x and earlier outputs come from earlier kernels
        if (et == 0) stamp(a, 0);
        int lu = 0;
        for (int p = 0; p < a.n_phases; ++p) {
            const MkPhase& ph = a.ph[p];
            if (ph.kind == MK_GEMM) {
                const MkGemm& g = ph.g;
                if (g.swiglu && p > 0 && !a.nodep) {  // the folded mlp_norm scale reads ssp of the previous phase
                    if (et == 0) wait_counter(&a.bar[a.ph[p - 1].slot], a.ph[p - 1].target);
                    epi_bar();
                }
                // token columns of this warp's half: 16-column chunks split between the two warps of a lane group
                const int nchunk = a.ntok / 16, c_lo = half_id ? ((nchunk + 1) / 2) * 16 : 0,
                          c_hi = half_id ? a.ntok : ((nchunk + 1) / 2) * 16;
                for (int u = cta; u < g.units; u += grid, ++lu) {
                    const Unit un = unit_of(g, u, a.krot);
                    const int b = lu & 1;
                    mbar_wait(&tfull[b], (uint32_t)(lu >> 1) & 1u);
                    fence_after();
                    const uint32_t acc = tmem + lane_base + (uint32_t)(b * a.ntok);
                    const int n0 = un.nt * 128;
                    if (!g.swiglu) {
                        const int n = n0 + lg * 32 + lane;  // TMEM lane = weight row n, column = token
                        float* out = g.partial + (int64_t)un.z * a.M * g.N;
#pragma unroll 1
                        for (int c = c_lo; c < c_hi; c += 16) {
                            uint32_t r[16];
                            tmem_ld16(acc + (uint32_t)c, r);
                            if (n < g.N) {
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    if (c + j < a.M) out[(int64_t)(c + j) * g.N + n] = __uint_as_float(r[j]);
                            }
                        }
                    } else if (half_id == 0) {
                        // rows 0-63 of the tile = gate, 64-127 = the matching up rows (interleaved W_gu); the up rows
                        // reach the gate warps through a [64][XC + 1] scratch, XC token columns per pass
                        float* up = reinterpret_cast<float*>(smem + a.scratch_off);
                        const int ld = XC + 1;
                        float* tok_scale = up + 64 * ld;
                        if (et < a.ntok) tok_scale[et] = et < a.M ? row_scale(a.ssp, a.nb, et, g.K, a.eps) : 0.f;
                        const int inter = g.N / 2;
                        const int i = (n0 / 128) * 64 + lg * 32 + lane;
                        for (int c0 = 0; c0 < a.ntok; c0 += XC) {
                            const int c1 = min(a.ntok, c0 + XC);
                            if (lg >= 2) {
#pragma unroll 1
                                for (int c = c0; c < c1; c += 16) {
                                    uint32_t r[16];
                                    tmem_ld16(acc + (uint32_t)c, r);
#pragma unroll
                                    for (int j = 0; j < 16; ++j)
                                        up[((lg - 2) * 32 + lane) * ld + c - c0 + j] = __uint_as_float(r[j]);
                                }
                            }
                            swiglu_bar();
                            if (lg < 2) {
#pragma unroll 1
                                for (int c = c0; c < c1; c += 16) {
                                    uint32_t r[16];
                                    tmem_ld16(acc + (uint32_t)c, r);
#pragma unroll
                                    for (int j = 0; j < 16; ++j) {
                                        const int m = c + j;
                                        if (m < a.M && i < inter) {
                                            const float sc = tok_scale[c + j];
                                            ((bf16*)g.act)[(int64_t)m * inter + i] = __float2bfloat16_rn(
                                                silu(sc * __uint_as_float(r[j])) * (sc * up[(lg * 32 + lane) * ld + c - c0 + j]));
                                        }
                                    }
                                }
                            }
                            swiglu_bar();  // scratch reusable (next pass / unit)
                        }
                    }
                    fence_before();
                    mbar_arrive(&tempty[b]);
                }
            } else if (!a.nodep) {
                if (et == 0 && p > 0) wait_counter(&a.bar[a.ph[p - 1].slot], a.ph[p - 1].target);
                epi_bar();
                if (ph.kind == MK_RESIDUAL) residual_phase(a, ph, ew, lane);
                else qkv_epi_phase(a, et);
            }
            epi_bar();  // every worker's writes of this phase are issued
            if (et == 0) {
                stamp(a, 1 + p);
                __threadfence();
                red_release_add(&a.bar[ph.slot], 1u);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// [rows][cols_k] bf16, row stride ld_elems, TMA box = 64 k x box_rows, SWIZZLE_128B (the UMMA K-major layout)
CUtensorMap make_map(const void* base, int rows, int cols_k, int ld_elems, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols_k, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
    const cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

bool mk_supported(int M, int hidden, int inter, int qd, int kvd) {
    return M >= 1 && M <= 128 && hidden % 128 == 0 && inter % 64 == 0 && qd % 64 == 0 && kvd % 64 == 0 &&
           hidden % BK == 0 && inter % BK == 0;
}

int mk_grid(int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return sms;
}

void launch_mk(MkArgs a, const MkMapSpec* specs, int n_maps, cudaStream_t s) {
    if (n_maps > MK_MAX_MAPS) fail(TKV_ERR_CONFIG, "layer kernel: too many tensor maps");
    MkMaps maps;
    for (int i = 0; i < n_maps; ++i)
        maps.m[i] = make_map(specs[i].base, specs[i].rows, specs[i].cols, specs[i].ld, specs[i].box_rows);
    a.n_maps = n_maps;
    if (a.l2_ahead <= 0) a.l2_ahead = 16;
    a.ntok = ((a.M + 15) / 16) * 16;
    a.a_bytes = (uint32_t)a.ntok * BK * 2;
    a.tmem_cols = 32;
    while (a.tmem_cols < (uint32_t)(2 * a.ntok)) a.tmem_cols <<= 1;
    const uint32_t scratch = (uint32_t)((64 * (XC + 1) + a.ntok) * 4 + 1023) / 1024 * 1024;
    a.stages = (int)std::min<uint32_t>(10, (uint32_t)(kSmemBudget - (int)scratch - 1024) / (TILE_W + a.a_bytes));
    if (a.stages < 2) fail(TKV_ERR_CONFIG, "layer kernel: shared-memory budget too small");
    a.scratch_off = ((uint32_t)a.stages * (TILE_W + a.a_bytes) + 256 + 1023) / 1024 * 1024;
    const size_t smem = 1024 + (size_t)a.scratch_off + scratch;
    int dev = 0;
    TKV_CUDA(cudaGetDevice(&dev));
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if ((int)smem * 2 <= smem_sm) fail(TKV_ERR_CONFIG, "layer kernel: must hold one CTA per SM");
    static std::once_flag once;
    std::call_once(once, [&] {
        TKV_CUDA(cudaFuncSetAttribute(mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    });
    launch_k(mk_kernel, dim3(mk_grid(dev)), dim3(THREADS), smem, s, maps, a);
}

}  // namespace tkv

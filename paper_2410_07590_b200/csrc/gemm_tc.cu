// tcgen05 + TMA bf16 GEMM for sm_100a:  C[m][n] = sum_k A[m][k] * W[n][k]
// A = activations [M][lda] (K-major), W = weights [N][K] (K-major: the engine stores every projection
// transposed). Replaces the reference's f64 matmul (src/numerics.cpp:8-29) for the QKV / O / gate-up /
// down projections of forward_tokens (src/model.cpp:240-264).
//
// Two tilings, one kernel template:
//   normal  (M > 128 tokens: full-concat prefill, chunk ingest): UMMA M=128 over tokens, N=128 over
//           weight rows; TMEM lane = token row.
//   swapped (M <= 128 tokens: query prefill, decode): UMMA M=128 over WEIGHT rows, N = M rounded up to 16
//           over tokens — no half-empty tile at batch-1 query sizes, and the epilogue (TMEM lane = weight
//           row) stores consecutive n per warp, i.e. coalesced.
// Epilogues: fp32 split-K partials partial[z][m][n] (reduced by the consumer kernel), or — when the
// whole K range is in one CTA — SwiGLU fused: W_gu rows are stored in blocks of 64 gate rows followed by
// the 64 matching up rows, so a 128-row tile holds complete (gate, up) pairs and the epilogue writes
// act = silu(g) * u (numerics.cpp:103-124) in bf16 directly.
//
// Warp roles (128 threads): warp 0 lane 0 = TMA producer (STAGES-deep ring, SWIZZLE_128B, mbarrier
// full/empty), warp 1 lane 0 = MMA issuer (tcgen05.mma.cta_group::1.kind::f16, fp32 accumulator in TMEM,
// tcgen05.commit frees smem slots), all 4 warps = epilogue (tcgen05.ld 32x32b, warp w owns lanes 32w..).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

#ifndef GEMM_WN224
#define GEMM_WN224 1
#endif
constexpr int BK = 64, THREADS = 128;
constexpr int EPI_LD = 33;  // row stride (floats) of the normal-tiling partial epilogue's per-warp staging block
                            // (odd: the 4-byte row-per-lane writes and the row reads are both conflict-free)
constexpr uint32_t TILE_W = 128 * BK * 2;  // 16 KB: 128 rows x 64 k, bf16
constexpr int SMEM_BUDGET = 200 * 1024;

// Tuning knobs (tkv_debug_set_gemm_knobs; 0 = default): ring depth, smem budget (KB), CTAs per SM,
// L2 eviction policy of the weight stream (1 = evict_first).
struct Knobs {
    // swapped (<= 128 tokens) tiling: np 128-row weight tiles per unit share one activation tile per stage
    // (np = 2 with one 208 KB CTA per SM measured slower than np = 1 at 2 x 110 KB); pf = L2 prefetch distance
    // of the weight stream in k-blocks (0 = off)
    int stages = 0, smem_kb = 110, ctas_per_sm = 2, w_evict_first = 1, np = 1, pf = 0, krot = 1;
    // normal (> 128 tokens) tiling: nsnp 128-column halves per MMA (UMMA N = 128 * nsnp); N = 256 halves the
    // shared-memory traffic per FLOP of the SS-mode MMA (the 128 x 128 tile is smem-bandwidth bound at ~50 %)
    int nsnp = 2, ns_smem_kb = 226;  // 3 stages of 64 KB + the partial epilogue staging block: 227 KB
    // normal tiling: nsmp 128-row activation tiles per unit share each weight tile (M = 128 * nsmp per unit):
    // the per-FLOP L2 -> smem traffic drops by 1/3 at nsmp = 2 (A 32 KB + W 32 KB per 64-deep k-block for
    // 2 x 128 x 256 outputs); the two 128 x 256 fp32 accumulators fill TMEM, so a unit's epilogue is not
    // overlapped with the next mainloop
    int nsmp = 2;
    int wn224 = GEMM_WN224;  // normal tiling: allow 224-wide n-tiles when they fill the waves better (0 = always 128 * nsnp)
    int raster = 1;  // normal tiling unit order: 0 = n-fastest, 1 = m-fastest when N > M (W larger), 2 = m-fastest,
                     // 3 = m-fastest in groups of group_mb MB of activation rows (always)
    int group_mb = 32;
    int skip_epi = 0;
};
Knobs g_knobs;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bounded spin: a protocol bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 26)) __trap();
    }
}
// Same, for waits that last a whole mainloop (the epilogue warps on the accumulator): back off between polls so
// the waiting warps do not compete with the MMA issuer and the TMA for the shared-memory / mbarrier unit.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(256);
        if (spin > (1u << 24)) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// Same with an L2 cache-policy hint (weights are streamed once: evict_first keeps L2 for activations/KV).
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
// L2 prefetch of a tensor-map box (no smem destination): pulls weight tiles PD stages ahead of the ring so
// the DRAM stream has more bytes in flight than shared memory can hold.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// UMMA smem descriptor, K-major SWIZZLE_128B: 128 B rows, 8-row atoms 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major, N>>3 at bit 17, M>>4 at bit 24.
__device__ __forceinline__ uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// Warp-collective forms: called by all 32 lanes with warp-uniform operands; elect.sync picks the issuing lane (the
// same one every time, so a commit tracks the MMAs that lane issued).
__device__ __forceinline__ void umma_f16_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ float silu(float z) { return z / (1.0f + __expf(-z)); }
// silu with the approximate divide (z -> -inf: 1 + e^-z overflows to inf and __fdividef returns 0, the limit)
__device__ __forceinline__ float silu_fast(float z) { return __fdividef(z, 1.0f + __expf(-z)); }

struct GemmArgs {
    int M, N, K;
    int kb_total, kb_per_split;
    int n_tiles, m_tiles, units;  // work units = n_tiles * m_tiles * splits (persistent loop over them)
    int np;                       // swapped: 128-row weight tiles per unit (n_tiles counts units along N)
    int ntok;                     // swapped: tokens per tile (MMA N, multiple of 16); normal: 128 * mp
    int mp;                       // normal: 128-row activation sub-tiles per unit (each its own MMA + accumulator)
    int wn;                       // normal: weight rows per unit = UMMA N (128 * np, or 224 when 224-wide n-tiles fill
                                  // the last wave better: C3 / C5 O and down, N = 3584 = 16 x 224)
    int nbuf;                     // TMEM accumulator buffers (2: epilogue overlaps the next unit's mainloop)
    int gub;                      // EPI_SWIGLU: W_gu rows interleaved in blocks of gub gate rows + gub up rows. 128
                                  // (np = 2): weight tile 0 of a unit = gate rows, tile 1 = the matching up rows, so a
                                  // TMEM lane (swapped: weight row) holds its gate AND up accumulators; 64: one 128-row
                                  // tile holds 64 gate + 64 up rows (the swapped epilogue exchanges them through smem)
    int skip_epi;                 // debug timing knob: normal-tiling partial epilogue skipped (results invalid)
    int m_group;                  // unit raster (normal tiling): 0 = n-tiles fastest; G > 0 = groups of G m-tiles,
                                  // m fastest inside a group and the group's activation rows kept L2-resident
                                  // while every n-tile streams past them (W from DRAM once per group)
    uint32_t a_bytes;             // bytes of the activation tile per stage
    int stages;
    uint32_t acc_cols;            // TMEM columns of one accumulator buffer (two buffers)
    uint32_t tmem_cols;
    uint32_t scratch_off;         // SwiGLU exchange scratch (swapped): byte offset after the ring
    float* partial;               // EPI_PARTIAL
    __nv_bfloat16* act;           // EPI_SWIGLU: [M][N/2]
    const float* ssp;             // EPI_SWIGLU: folded RMSNorm partial sums (row_scale), nb blocks per token
    int nb;
    float eps;
    int w_evict_first;
    int pf;                       // weight L2 prefetch distance (k-blocks ahead of the ring)
    int krot;                     // rotate each unit's k-block order (spreads the shared activation tiles'
                                  // L2 reads over time instead of every CTA hitting the same lines at once)
    int trace_parity;             // debug: which of the two per-CTA entry/exit slot sets this launch writes
    unsigned long long* tl;       // kernel timeline slot (tl_take): first CTA past griddepcontrol.wait, last CTA exit
    unsigned long long* trace;    // debug (tkv_debug_gemm_trace): CTA 0 clock64 per stage [it][3] = producer issue,
                                  // MMA saw full, MMA committed; [GT_UNIT + lu][2] = epilogue start / end per unit
};
constexpr int GT_STAGES = 1024, GT_UNIT = 3 * GT_STAGES, GT_EPI = GT_UNIT + 2 * 64 + 4 * 64, GT_CTA = GT_EPI + 32,
              GT_SIZE = GT_CTA + 2 * 2 * 1024;  // [launch parity][cta][entry, exit] globaltimer ns
__device__ __forceinline__ void gtrace_cta(unsigned long long* t, int parity, int exit) {
    if (t && blockIdx.x < 1024) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        t[GT_CTA + (parity * 1024 + blockIdx.x) * 2 + exit] = ns;
    }
}
unsigned long long* g_gemm_trace = nullptr;

__device__ __forceinline__ void gtrace(unsigned long long* t, int slot) {
    if (t && blockIdx.x == 0 && slot < GT_SIZE) {
        unsigned long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        t[slot] = c;
    }
}

enum { EPI_PARTIAL = 0, EPI_SWIGLU = 1 };
constexpr int THREADS_P = 192;  // swapped tiling: warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
// normal (large-M) tiling: warps 2-9 = epilogue, two per TMEM lane quadrant, each on half the columns of a unit (the
// 256 x 256 unit's epilogue is not overlapped with the next mainloop: TMEM holds only the one accumulator)
constexpr int threads_for(bool swap) { return swap ? THREADS_P : THREADS_P + 128; }
constexpr int XC = 32;          // swapped SwiGLU epilogue: token columns per gate/up exchange pass

__device__ __forceinline__ void unit_coords(const GemmArgs& g, int u, int& nt, int& mt, int& z) {
    const int per = g.n_tiles * g.m_tiles;
    z = u / per;
    const int rem = u - z * per;
    if (g.m_group > 0) {
        const int span = g.m_group * g.n_tiles;
        const int gi = rem / span, r = rem - gi * span;
        const int gsz = min(g.m_group, g.m_tiles - gi * g.m_group);
        nt = r / gsz;
        mt = gi * g.m_group + (r - nt * gsz);
    } else {
        mt = rem / g.n_tiles;
        nt = rem - mt * g.n_tiles;
    }
}

// Persistent: grid = min(units, #SMs); CTA b owns units b, b + grid, ... The smem ring of {W, A} stages
// flows across units without draining; two TMEM accumulators let the epilogue of unit i overlap the
// mainloop of unit i+1.
template <bool SWAP, int EPI>
__global__ void __launch_bounds__(threads_for(SWAP))
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, GemmArgs g) {
    pdl_launch();
    if (threadIdx.x == 0) gtrace_cta(g.trace, g.trace_parity, 0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t wbytes = SWAP ? (uint32_t)g.np * TILE_W : (uint32_t)g.wn * (BK * 2);  // weight bytes per stage
    const int wrows = SWAP ? 128 * g.np : g.wn;                                             // weight rows per unit
    const uint32_t stage_bytes = wbytes + g.a_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.stages * stage_bytes);
    uint64_t* empty = full + g.stages;
    uint64_t* tfull = empty + g.stages;  // [2] accumulator ready
    uint64_t* tempty = tfull + 2;        // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u0 = blockIdx.x, ustep = gridDim.x;  // this CTA's units: u0, u0 + ustep, ...
    auto coords = [&](int u, int& nt, int& mt, int& z) { unit_coords(g, u, nt, mt, z); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], threads_for(SWAP) - 64);  // every epilogue thread
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(g.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int mstep = SWAP ? g.ntok : 128 * g.mp;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer ----------------
            const uint64_t wpol = policy_evict_first();
            auto load_w = [&](void* dst, uint64_t* bar, int c0, int c1) {
                if (g.w_evict_first)
                    tma_load_2d_hint(dst, &tmW, bar, c0, c1, wpol);
                else
                    tma_load_2d(dst, &tmW, bar, c0, c1);
            };
            // Weight tiles do not depend on earlier kernels: fill the ring with the first unit's weights
            // BEFORE waiting on the previous grid (PDL), so the weight stream overlaps its tail.
            int nt, mt, z;
            coords(u0, nt, mt, z);
            const int kb0 = z * g.kb_per_split;
            const int nkb0 = min(g.kb_total, kb0 + g.kb_per_split) - kb0;
            // k-block of iteration i of unit u (the MMA only accumulates, so any order is valid)
            auto kblk = [&](int k0, int nkb, int i, int u) { return k0 + (g.krot ? (i + (u * 37) % nkb) % nkb : i); };
            const int pre = min(nkb0, g.stages);
            for (int i = 0; i < pre; ++i) {
                mbar_expect_tx(&full[i], stage_bytes);
                load_w(smem + i * stage_bytes, &full[i], kblk(kb0, nkb0, i, u0) * BK, nt * wrows);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i)
                tma_load_2d(smem + i * stage_bytes + wbytes, &tmA, &full[i], kblk(kb0, nkb0, i, u0) * BK, mt * mstep);
            // L2 prefetch of the first unit's next pf weight tiles (beyond the ring)
            for (int i = pre; i < min(nkb0, pre + g.pf); ++i)
                tma_prefetch_2d(&tmW, kblk(kb0, nkb0, i, u0) * BK, nt * wrows);
            int it = pre;
            for (int u = u0; u < g.units; u += ustep) {
                coords(u, nt, mt, z);
                const int k0 = z * g.kb_per_split, nkb = min(g.kb_total, k0 + g.kb_per_split) - k0;
                if (u != u0)
                    for (int i = 0; i < min(nkb, g.pf); ++i) tma_prefetch_2d(&tmW, kblk(k0, nkb, i, u) * BK, nt * wrows);
                for (int i = (u == u0 ? pre : 0); i < nkb; ++i, ++it) {
                    if (g.pf > 0 && i + g.pf < nkb && i + g.pf >= (u == u0 ? pre + g.pf : g.pf))
                        tma_prefetch_2d(&tmW, kblk(k0, nkb, i + g.pf, u) * BK, nt * wrows);
                    const int s = it % g.stages;
                    mbar_wait(&empty[s], ((uint32_t)(it / g.stages) & 1u) ^ 1u);
                    if (it < GT_STAGES) gtrace(g.trace, 3 * it);
                    uint8_t* w = smem + s * stage_bytes;
                    mbar_expect_tx(&full[s], stage_bytes);
                    const int kb = kblk(k0, nkb, i, u);
                    load_w(w, &full[s], kb * BK, nt * wrows);
                    tma_load_2d(w + wbytes, &tmA, &full[s], kb * BK, mt * mstep);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp walks the loop, so every operand (stage address, descriptors, TMEM address) is warp-uniform
        // and lives in uniform registers; one elected lane issues each tcgen05.mma / commit. (A lane-0-only loop made
        // the compiler move every operand through an R2UR waterfall: ~165 cycles per MMA issue, which capped one CTA
        // at one 64-deep k-block per ~1100 cycles, i.e. ~28 GB/s of weights.)
        const uint32_t id = SWAP ? idesc(128, g.ntok) : idesc(128, g.wn);
        int it = 0, lu = 0;
        for (int u = u0; u < g.units; u += ustep, ++lu) {
            int nt, mt, z;
            coords(u, nt, mt, z);
            const int k0 = z * g.kb_per_split, nkb = min(g.kb_total, k0 + g.kb_per_split) - k0;
            const int b = lu % g.nbuf;
            mbar_wait(&tempty[b], ((uint32_t)(lu / g.nbuf) & 1u) ^ 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t acc = tmem + (uint32_t)b * g.acc_cols;
            int s = it % g.stages;
            uint32_t ph = (uint32_t)(it / g.stages) & 1u;
            for (int i = 0; i < nkb; ++i, ++it) {
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0 && it < GT_STAGES) gtrace(g.trace, 3 * it + 1);
                const uint32_t w = smem_u32(smem + s * stage_bytes);
                const uint32_t a = w + wbytes;
                if (SWAP) {
                    const uint64_t da = desc_k(a);
                    for (int p = 0; p < g.np; ++p) {  // one activation tile, np weight tiles
                        const uint64_t dw = desc_k(w + p * TILE_W);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)  // +32 B along K inside the 128 B swizzle row = +2 in the
                                                           // descriptor's 16-byte address field
                            umma_f16_elect(acc + (uint32_t)(p * g.ntok), dw + 2 * k, da + 2 * k, id, (i | k) != 0);
                    }
                } else {
                    const uint64_t dw = desc_k(w);
                    for (int mi = 0; mi < g.mp; ++mi) {  // mp activation sub-tiles share the weight tile
                        const uint64_t da = desc_k(a + mi * 16384);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_f16_elect(acc + (uint32_t)(mi * g.wn), da + 2 * k, dw + 2 * k, id, (i | k) != 0);
                    }
                }
                    umma_commit_elect(&empty[s]);
                if (lane == 0 && it < GT_STAGES) gtrace(g.trace, 3 * it + 2);
                if (++s == g.stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            umma_commit_elect(&tfull[b]);
        }
    } else {
        // ---------------- epilogue warps 2-5: TMEM lane group = warp % 4 ----------------
        pdl_wait();
        if (g.tl && threadIdx.x == 64) atomicMin(g.tl, gtimer_ns());  // the predecessor grid has completed
        const int lg = warp & 3;
        const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
        const int et = threadIdx.x - 64;  // 0..127 (swapped) / 0..255 (normal)
        const int half = SWAP ? 0 : (warp - 2) >> 2;  // normal tiling: which half of a unit's columns this warp owns
        if (SWAP && EPI == EPI_SWIGLU && g.gub == 128) {
            // folded mlp_norm scale of every token (swapped tiling: all units cover tokens [0, ntok)), once per CTA
            float* ts = reinterpret_cast<float*>(smem + g.scratch_off);
            if (et < g.ntok) ts[et] = et < g.M ? row_scale(g.ssp, g.nb, et, g.K, g.eps) : 0.f;
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        int lu = 0;
        for (int u = u0; u < g.units; u += ustep, ++lu) {
            int nt, mt, z;
            coords(u, nt, mt, z);
            const int b = lu % g.nbuf;
            mbar_wait_sleep(&tfull[b], (uint32_t)(lu / g.nbuf) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (et == 0 && lu < 64) gtrace(g.trace, GT_UNIT + 2 * lu);
            const uint32_t acc_u = tmem + lane_base + (uint32_t)b * g.acc_cols;
            const int m0 = mt * mstep;
            for (int pm = 0; pm < g.np * (SWAP ? 1 : g.mp); ++pm) {
            const int p = pm % g.np, mi = pm / g.np;  // weight sub-tile, activation sub-tile (normal tiling)
            // normal tiling: activation sub-tile mi's accumulator holds wn weight columns (the partial epilogue takes
            // them all at p == 0; the SwiGLU epilogue runs at wn = 256 with gate | up halves)
            const uint32_t acc = acc_u + (uint32_t)(SWAP ? p * g.ntok : mi * g.wn + p * 128);
            const int n0 = SWAP ? (nt * g.np + p) * 128 : nt * g.wn + p * 128;
            if (SWAP) {
                const int n = n0 + lg * 32 + lane;  // TMEM lane = weight row n, column = token
                if (EPI == EPI_PARTIAL) {
                    float* out = g.partial + (int64_t)z * g.M * g.N;
#pragma unroll 1
                    for (int c = 0; c < g.ntok; c += 16) {
                        uint32_t r[16];
                        tmem_ld16(acc + (uint32_t)c, r);
                        if (n < g.N) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int m = m0 + c + j;
                                if (m < g.M) out[(int64_t)m * g.N + n] = __uint_as_float(r[j]);
                            }
                        }
                    }
                } else if (g.gub == 128) {
                    // gate tile (p = 0) and up tile (p = 1) of intermediate rows [nt * 128, nt * 128 + 128): this lane's
                    // row i has its gate accumulators at acc, its up accumulators ntok columns further. The chunk's
                    // token scales are read (ld.shared) before any of its stores: a generic load behind a global store
                    // is ordered after it, which serialised every element on the store (~200 cycles each).
                    if (p == 0) {
                        const uint32_t ts = smem_u32(smem + g.scratch_off);
                        const int inter = g.N / 2;
                        const int i = nt * 128 + lg * 32 + lane;
#pragma unroll 1
                        for (int c = 0; c < g.ntok; c += 16) {
                            uint32_t gr[16], ur[16];
                            tmem_ld16_nowait(acc + (uint32_t)c, gr);
                            tmem_ld16_nowait(acc + (uint32_t)(g.ntok + c), ur);
                            float sc[16];
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                             : "=f"(sc[4 * q]), "=f"(sc[4 * q + 1]), "=f"(sc[4 * q + 2]), "=f"(sc[4 * q + 3])
                                             : "r"(ts + (uint32_t)(c + 4 * q) * 4));
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                            // transpose the warp's [32 rows][16 tokens] through its 1 KB smem block, then store
                            // whole 16-byte pieces of token rows (2 per lane) instead of 16 scattered 2-byte stores
                            const uint32_t xs = ts + 1024u + (uint32_t)lg * 1024u;
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const __nv_bfloat16 o = __float2bfloat16_rn(
                                    silu_fast(sc[j] * __uint_as_float(gr[j])) * (sc[j] * __uint_as_float(ur[j])));
                                asm volatile("st.shared.b16 [%0], %1;" ::"r"(xs + (uint32_t)(j * 64 + lane * 2)),
                                             "h"(__bfloat16_as_ushort(o)) : "memory");
                            }
                            __syncwarp();
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int ch = lane + 32 * h, tk = ch >> 2, part = ch & 3;
                                uint4 v;
                                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                             : "r"(xs + (uint32_t)(tk * 64 + part * 16)) : "memory");
                                const int m = m0 + c + tk, col = i - lane + part * 8;
                                if (m < g.M && col < inter)
                                    *reinterpret_cast<uint4*>(g.act + (int64_t)m * inter + col) = v;
                            }
                            __syncwarp();
                        }
                    }
                } else {
                    // tile rows 0-63 = gate, 64-127 = the matching up rows (interleaved W_gu layout); the up rows
                    // reach the gate warps through a [64][XC + 1] scratch, XC token columns per pass (a small
                    // scratch leaves the ring one more stage)
                    float* up = reinterpret_cast<float*>(smem + g.scratch_off);
                    const int ld = XC + 1;
                    float* tok_scale = up + 64 * ld;  // [ntok]: folded mlp_norm scale per token
                    if (et < g.ntok) tok_scale[et] = m0 + et < g.M ? row_scale(g.ssp, g.nb, m0 + et, g.K, g.eps) : 0.f;
                    const int inter = g.N / 2;
                    const int i = (n0 / 128) * 64 + lg * 32 + lane;
                    int ev = 0;
                    auto tr = [&]() { if (lu == 0 && (et == 64 || et == 0)) gtrace(g.trace, GT_EPI + (et ? 16 : 0) + ev); ++ev; };
                    tr();
                    for (int c0 = 0; c0 < g.ntok; c0 += XC) {
                        const int c1 = min(g.ntok, c0 + XC);
                        if (lg >= 2) {
#pragma unroll 1
                            for (int c = c0; c < c1; c += 16) {
                                uint32_t r[16];
                                tmem_ld16(acc + (uint32_t)c, r);
#pragma unroll
                                for (int j = 0; j < 16; ++j) up[((lg - 2) * 32 + lane) * ld + c - c0 + j] = __uint_as_float(r[j]);
                            }
                        }
                        tr();
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        tr();
                        if (lg < 2) {
#pragma unroll 1
                            for (int c = c0; c < c1; c += 16) {
                                uint32_t r[16];
                                tmem_ld16(acc + (uint32_t)c, r);
#pragma unroll
                                for (int j = 0; j < 16; ++j) {
                                    const int m = m0 + c + j;
                                    if (m < g.M && i < inter) {
                                        const float sc = tok_scale[c + j];
                                        g.act[(int64_t)m * inter + i] = __float2bfloat16_rn(
                                            silu(sc * __uint_as_float(r[j])) * (sc * up[(lg * 32 + lane) * ld + c - c0 + j]));
                                    }
                                }
                            }
                        }
                        tr();
                        asm volatile("bar.sync 1, 128;" ::: "memory");  // scratch reusable (next pass / unit)
                        tr();
                    }
                }
            } else {
                const int m = m0 + mi * 128 + lg * 32 + lane;  // TMEM lane = token row m, column = weight row
                if (EPI == EPI_PARTIAL) {
                    if (p != 0) continue;  // the p == 0 pass covers all wn columns of activation sub-tile mi
                    if (g.skip_epi) continue;  // timing experiment only (TKV_GEMM_SKIP_EPI): results invalid
                    // 32 columns per tcgen05.wait::ld, staged through this warp's padded smem block (row stride 33
                    // floats: conflict-free) and written back row by row as 128-byte segments: the row-per-lane
                    // float4 stores cost one L2 transaction per 16 bytes (~23 K cycles per 256 x 256 unit)
                    float* stg = reinterpret_cast<float*>(smem + g.scratch_off) + (warp - 2) * 32 * EPI_LD;
                    // this warp's half of the subtile: wn / 2 columns (128 or 112) in 32- and 16-column chunks
                    const int cs = (g.wn / 2) * half, ce = cs + g.wn / 2;
#pragma unroll 1
                    for (int c = cs; c < ce; c += 32) {
                        const bool two = c + 32 <= ce;
                        uint32_t r[32];
                        tmem_ld16_nowait(acc + (uint32_t)c, *reinterpret_cast<uint32_t(*)[16]>(r));
                        if (two) tmem_ld16_nowait(acc + (uint32_t)(c + 16), *reinterpret_cast<uint32_t(*)[16]>(r + 16));
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 16; ++j) stg[lane * EPI_LD + j] = __uint_as_float(r[j]);
                        if (two) {
#pragma unroll
                            for (int j = 16; j < 32; ++j) stg[lane * EPI_LD + j] = __uint_as_float(r[j]);
                        }
                        __syncwarp();
                        const int mrow0 = m0 + mi * 128 + lg * 32, n = n0 + c + lane;
                        const bool col_ok = n < g.N && (two || lane < 16);
                        float* outz = g.partial + (int64_t)z * g.M * g.N;
#pragma unroll 4
                        for (int rr = 0; rr < 32; ++rr) {
                            const float v = stg[rr * EPI_LD + lane];
                            const int mr = mrow0 + rr;
                            if (mr < g.M && col_ok) outz[(int64_t)mr * g.N + n] = v;  // 128-byte row segments
                        }
                        __syncwarp();
                    }
                } else {
                    const int inter = g.N / 2;
                    if (g.gub == 128) {
                        // half p = 0 of the 256-wide unit = gate rows [nt * 128, +128), half 1 = the matching up rows
                        if (p != 0) continue;
                        const int i0 = nt * 128;
                        const float sc = m < g.M ? row_scale(g.ssp, g.nb, m, g.K, g.eps) : 0.f;
                        // software-pipelined: the next 16 (gate, up) column pairs load while this chunk's SwiGLU runs
                        // (one load pair + wait per chunk made the 256 x 256 unit's epilogue ~35 K cycles)
                        uint32_t gr[2][16], ur[2][16];
                        const int cs = 64 * half;  // this warp's 64 (gate, up) column pairs
                        tmem_ld16_nowait(acc + (uint32_t)cs, gr[0]);
                        tmem_ld16_nowait(acc + (uint32_t)(128 + cs), ur[0]);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int cc = 0; cc < 64; cc += 16) {
                            const int c = cs + cc;
                            const int cb = (cc >> 4) & 1;
                            if (cc + 16 < 64) {
                                tmem_ld16_nowait(acc + (uint32_t)(c + 16), gr[cb ^ 1]);
                                tmem_ld16_nowait(acc + (uint32_t)(128 + c + 16), ur[cb ^ 1]);
                            }
                            if (m < g.M) {
                                __align__(16) __nv_bfloat16 o[16];
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    o[j] = __float2bfloat16_rn(silu_fast(sc * __uint_as_float(gr[cb][j])) *
                                                               (sc * __uint_as_float(ur[cb][j])));
                                __nv_bfloat16* dst = g.act + (int64_t)m * inter + i0 + c;
                                if (i0 + c + 16 <= inter && (inter % 8) == 0) {
                                    reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<uint4*>(o)[0];
                                    reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<uint4*>(o)[1];
                                } else {
                                    for (int j = 0; j < 16; ++j)
                                        if (i0 + c + j < inter) dst[j] = o[j];
                                }
                            }
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        }
                        continue;
                    }
                    const int i0 = (n0 / 128) * 64;
                    const float sc = m < g.M ? row_scale(g.ssp, g.nb, m, g.K, g.eps) : 0.f;  // folded mlp_norm
#pragma unroll 1
                    for (int c = 32 * half; c < 32 * half + 32; c += 16) {
                        uint32_t gr[16], ur[16];
                        tmem_ld16(acc + (uint32_t)c, gr);
                        tmem_ld16(acc + (uint32_t)(64 + c), ur);
                        if (m < g.M) {
                            __align__(16) __nv_bfloat16 o[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                o[j] = __float2bfloat16_rn(silu(sc * __uint_as_float(gr[j])) * (sc * __uint_as_float(ur[j])));
                            __nv_bfloat16* dst = g.act + (int64_t)m * inter + i0 + c;
                            if (i0 + c + 16 <= inter && (inter % 8) == 0) {
                                reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<uint4*>(o)[0];
                                reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<uint4*>(o)[1];
                            } else {
                                for (int j = 0; j < 16; ++j)
                                    if (i0 + c + j < inter) dst[j] = o[j];
                            }
                        }
                    }
                }
            }
            }  // p
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
            if (et == 0 && lu < 64) gtrace(g.trace, GT_UNIT + 2 * lu + 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) gtrace_cta(g.trace, g.trace_parity, 1);
    if (g.tl && threadIdx.x == 0) atomicMax(g.tl + 1, gtimer_ns());
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols));
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

template <bool SWAP, int EPI>
void launch_t(const CUtensorMap& ta, const CUtensorMap& tw, const GemmArgs& g, int grid, size_t smem, cudaStream_t s) {
    TKV_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<SWAP, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_k(gemm_tc_kernel<SWAP, EPI>, dim3(grid), dim3(threads_for(SWAP)), smem, s, ta, tw, g);
}

}  // namespace

bool gemm_tc_supported(int M, int N, int K, int lda) {
    // TMA: 16-byte aligned row strides; K >= 8 elements.
    return M >= 1 && N >= 1 && K >= 8 && (lda * 2) % 16 == 0 && (K * 2) % 16 == 0;
}

int gemm_tc_ctas_per_sm(int M) { return M <= 128 ? std::max(1, g_knobs.ctas_per_sm) : 1; }

static int np_for(int M, int N) {
    if ((N + 127) / 128 < 2) return 1;
    return M <= 128 ? std::max(1, g_knobs.np) : std::max(1, std::min(2, g_knobs.nsnp));
}

static int mp_for(int M) { return M <= 128 ? 1 : (M >= 256 ? std::max(1, std::min(2, g_knobs.nsmp)) : 1); }

int gemm_tc_tiles(int M, int N) {
    const bool swap = M <= 128;
    const int np = np_for(M, N), mp = mp_for(M);
    return ((N + 128 * np - 1) / (128 * np)) * (swap ? 1 : (M + 128 * mp - 1) / (128 * mp));
}

int launch_gemm_tc(const void* A, int lda, const void* W, int M, int N, int K, float* partial, int splits,
                   cudaStream_t s, void* swiglu_act, const float* ssp, int nb, float eps, int gu_block) {
    const bool swap = M <= 128;
    // W_gu in 128-row gate / up blocks: a unit = one gate tile + its up tile (np = 2); swapped, one CTA per SM with a
    // 5-deep ring of 40 KB stages (the two weight tiles share each activation tile)
    const bool gu128 = swiglu_act && gu_block == 128;
    if (swiglu_act && gu_block != 128 && gu_block != 64) fail(TKV_ERR_CONFIG, "fused SwiGLU epilogue needs 64- or 128-row gate/up blocks");
    GemmArgs g{};
    g.gub = gu_block;
    g.M = M;
    g.N = N;
    g.K = K;
    g.kb_total = (K + BK - 1) / BK;
    g.kb_per_split = (g.kb_total + splits - 1) / splits;
    const int eff_splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;  // every unit non-empty
    g.np = gu128 ? 2 : np_for(M, N);
    if (gu128 && N % 256) fail(TKV_ERR_CONFIG, "128-row gate/up blocks need N % 256 == 0");
    g.mp = mp_for(M);
    g.wn = 128 * g.np;
    g.m_tiles = swap ? 1 : (M + 128 * g.mp - 1) / (128 * g.mp);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!swap && !swiglu_act && g.wn == 256 && g_knobs.wn224) {
        // 224-wide n-tiles when they fill the waves better: time ~ waves x unit width (C3 / C5 O and down: 112 -> 128
        // units of 256 x 224 in one wave at M = 2048, 896 -> 1024 in 7 waves at M = 16384)
        const int64_t u256 = (int64_t)((N + 255) / 256) * g.m_tiles * eff_splits;
        const int64_t u224 = (int64_t)((N + 223) / 224) * g.m_tiles * eff_splits;
        if (((u224 + sms - 1) / sms) * 224 < ((u256 + sms - 1) / sms) * 256) g.wn = 224;
    }
    g.n_tiles = (N + (swap ? 128 * g.np : g.wn) - 1) / (swap ? 128 * g.np : g.wn);
    g.skip_epi = g_knobs.skip_epi;
    g.units = g.n_tiles * g.m_tiles * eff_splits;
    g.ntok = swap ? ((M + 15) / 16) * 16 : 128 * g.mp;
    g.a_bytes = (uint32_t)g.ntok * BK * 2;
    g.acc_cols = swap ? (uint32_t)(g.ntok * g.np) : (uint32_t)(g.wn * g.mp);
    g.nbuf = 2 * g.acc_cols <= 512 ? 2 : 1;
    g.m_group = 0;
    if (!swap && g_knobs.raster != 0 && (g_knobs.raster == 2 || N > M)) {
        g.m_group = g.m_tiles;  // raster 1/2: all m-tiles in one group
        if (g_knobs.raster == 3 || (g_knobs.raster == 1 && g_knobs.group_mb > 0)) {
            const double a_tile = 128.0 * g.mp * K * 2;  // bytes of one m-tile's activation rows
            g.m_group = std::max(1, std::min(g.m_tiles, (int)(g_knobs.group_mb * 1048576.0 / a_tile)));
        }
    }
    g.tmem_cols = 32;
    while (g.tmem_cols < (uint32_t)g.nbuf * g.acc_cols) g.tmem_cols <<= 1;
    const uint32_t wbytes = swap ? (uint32_t)g.np * TILE_W : (uint32_t)g.wn * (BK * 2);  // weight bytes per stage
    const uint32_t scratch = (!swap && !swiglu_act) ? (uint32_t)(8 * 32 * EPI_LD * 4)  // partial epilogue staging
                             : !(swap && swiglu_act) ? 0
                             : gu128 ? 1024u + 4096u  // token scales + the four warps' transpose blocks
                                     : (uint32_t)((64 * (XC + 1) + g.ntok) * 4 + 1023) / 1024 * 1024;
    const int cps = (swap && gu128) ? 1 : gemm_tc_ctas_per_sm(M);
    const int budget = (swap && gu128) ? 208 * 1024
                       : swap          ? (g_knobs.smem_kb > 0 ? g_knobs.smem_kb * 1024 : SMEM_BUDGET)
                                       : g_knobs.ns_smem_kb * 1024;
    g.stages = (int)std::min<uint32_t>(g_knobs.stages > 0 ? g_knobs.stages : 8,
                                       (uint32_t)(budget - (int)scratch) / (wbytes + g.a_bytes));
    if (g.stages < 2) fail(TKV_ERR_CONFIG, "GEMM smem budget too small");
    g.w_evict_first = g_knobs.w_evict_first;
    g.scratch_off = (uint32_t)g.stages * (wbytes + g.a_bytes) + 256;  // after the ring and its barriers
    g.scratch_off = (g.scratch_off + 1023) / 1024 * 1024;
    g.partial = partial;
    g.trace = g_gemm_trace;
    g.tl = tl_take();
    static int trace_launch = 0;
    g.trace_parity = (trace_launch++) & 1;
    g.act = (__nv_bfloat16*)swiglu_act;
    g.ssp = ssp;
    g.nb = nb;
    g.eps = eps;
    if (swiglu_act && !ssp) fail(TKV_ERR_CONFIG, "fused SwiGLU epilogue needs the folded-norm partial sums");
    const size_t smem = 1024 + (size_t)g.scratch_off + scratch;
    const int grid = std::min(g.units, sms * cps);
    const CUtensorMap ta = make_map(A, M, K, lda, g.ntok);
    const CUtensorMap tw = make_map(W, N, K, K, swap ? 128 * g.np : g.wn);
    if (swiglu_act) {
        if (eff_splits != 1) fail(TKV_ERR_CONFIG, "fused SwiGLU epilogue needs the whole K range in one unit");
        swap ? launch_t<true, EPI_SWIGLU>(ta, tw, g, grid, smem, s) : launch_t<false, EPI_SWIGLU>(ta, tw, g, grid, smem, s);
    } else {
        swap ? launch_t<true, EPI_PARTIAL>(ta, tw, g, grid, smem, s) : launch_t<false, EPI_PARTIAL>(ta, tw, g, grid, smem, s);
    }
    return eff_splits;
}



void gemm_trace_enable(bool on, unsigned long long* host_out, int64_t cap) {
    static unsigned long long* buf = nullptr;
    if (host_out && buf) {
        TKV_CUDA(cudaDeviceSynchronize());
        TKV_CUDA(cudaMemcpy(host_out, buf, (size_t)std::min<int64_t>(cap, GT_SIZE) * 8, cudaMemcpyDeviceToHost));
    }
    if (on && !buf) TKV_CUDA(cudaMalloc(&buf, GT_SIZE * 8));
    if (on) TKV_CUDA(cudaMemset(buf, 0, GT_SIZE * 8));
    g_gemm_trace = on ? buf : nullptr;
}

void set_gemm_nsmp(int mp) { g_knobs.nsmp = mp > 0 ? mp : 1; }

void set_gemm_skip_epi(int v) { g_knobs.skip_epi = v; }

void set_gemm_raster(int r, int group_mb) {
    g_knobs.raster = r;
    if (group_mb >= 0) g_knobs.group_mb = group_mb;
}

void set_gemm_knobs(int stages, int smem_kb, int ctas_per_sm, int w_evict_first, int np, int pf, int krot) {
    const Knobs d;
    g_knobs.krot = krot >= 0 ? krot : d.krot;
    g_knobs.pf = pf >= 0 ? pf : d.pf;
    g_knobs.stages = stages;
    g_knobs.smem_kb = smem_kb > 0 ? smem_kb : d.smem_kb;
    g_knobs.ctas_per_sm = ctas_per_sm > 0 ? ctas_per_sm : d.ctas_per_sm;
    g_knobs.w_evict_first = w_evict_first;
    g_knobs.np = np > 0 ? np : d.np;
}

}  // namespace tkv

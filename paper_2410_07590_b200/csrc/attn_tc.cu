// tcgen05 / TMEM / TMA flash attention for head_size 128, bf16 — the query-prefill attention of the
// TurboRAG path (and the full-concat comparison), replacing attend + softmax_rows_inplace
// (src/attention.cpp:94-169, src/numerics.cpp:31-60) with implicit masks: row t sees key j iff
// lo[t] <= j <= hi[t] (causal_rows / build_mask, attention.cpp:50-92).
//
// GQA packing: a CTA owns 128 rows of ONE kv head g, row r = (token t, head g*group + r%group), so the
// K/V tiles it streams serve all `group` query heads (C2: 64 tokens x 7 heads = 448 rows = 3.5 tiles).
//
// v3: O accumulates in TMEM across KV tiles (FA4-style lazy rescale only when a row max grows by > 2^8), P is
// double-buffered in TMEM and fed to the PV MMA as the A operand (tcgen05.mma with A in TMEM), so the softmax
// of tile j+1 overlaps PV_j on the tensor pipe.
// Per CTA (576 threads): warps 0-15 = softmax (four threads per row: warps w, w+4, w+8, w+12 share TMEM
// lanes 32(w%4).., each owns 32 of the S columns and 32 of the O columns; partial row maxima are
// exchanged through shared memory), warp 16 = TMA producer, warp 17 = MMA issuer. smem: Q [128x128] and P [128x128] (two 64-column SW128 sub-tiles each, 32 KB), two K/V stages
// of 64 KB. TMEM (512 cols): S double buffer at cols 0/128, O tile at 256.
//   S_j  = Q . K_j^T          tcgen05.mma kind::f16 M128 N128 K16 x8, A,B K-major
//   P_j  = exp2(S_j*scale*log2e - m_j)  (softmax warps: TMEM -> regs -> bf16 -> swizzled smem)
//   O_j  = P_j . V_j          tcgen05.mma, A = P (K-major), B = V (MN-major: d contiguous)
// The running output O lives in registers (32 fp32 per thread), rescaled by exp2(m_{j-1} - m_j) each
// tile and incremented by the O_j tile read back from TMEM. Split-K over keys writes (O, m, l) partials
// combined by attn_combine_kernel (attn_simt.cu) — same workspace layout as the SIMT kernel.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int D = 128, BR = 128, BK = 128;
constexpr int NQ = 4;                       // softmax threads per row
constexpr int CPT = 128 / NQ;               // S / O columns per softmax thread
constexpr int SOFTMAX_WARPS = 4 * NQ, THREADS = SOFTMAX_WARPS * 32 + 64;
constexpr uint32_t SUB = 128 * 64 * 2;          // one [128 rows][64 cols] bf16 SW128 sub-tile = 16 KB
constexpr uint32_t OFF_Q = 0;                   // Q tile: 32 KB
constexpr uint32_t OFF_K = 2 * SUB;             // K ring: 2 stages x 32 KB
constexpr uint32_t OFF_V = 6 * SUB;             // V ring: 2 stages x 32 KB (separate ring: K_{j+2} loads once
constexpr uint32_t KSTAGE = 2 * SUB;            //   S_j is done, without waiting for PV_j)
constexpr uint32_t OFF_BAR = 10 * SUB;
// TMEM columns: S double buffer (fp32), O accumulator (fp32), P double buffer (bf16 pairs: 128 keys -> 64 cols)
constexpr uint32_t TM_S = 0, TM_O = 256, TM_P = 384;
constexpr float RESCALE_LOG2 = 8.0f;  // lazy O rescale: only when a row max grows by more than 2^8
constexpr size_t SMEM_BYTES = 1024 + OFF_BAR + 256;
constexpr uint32_t TMEM_COLS = 512;
constexpr float LOG2E = 1.4426950408889634f;

// kind::f16, D=f32, A=B=bf16, M=128, N=128; PV additionally B MN-major (bit 16)
constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr uint32_t IDESC_PV = IDESC_S | (1u << 16);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
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
        if (spin > (1u << 26)) __trap();  // protocol bug -> launch error, never a hung GPU
    }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// K-major SW128 (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t desc_k(uint32_t a) {
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
// MN-major SW128: 64-element MN blocks LBO = 16 KB apart (the two d-halves), 8-row K groups SBO = 1024 B apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t a) {
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(SUB >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
// Bulk L2 prefetch (no smem destination): warms the NEXT projections' weights while attention runs.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Debug timeline (tkv_debug_attn_trace): CTA (0,0,0) stamps clock64 at pipeline events, slot [j][e].
__device__ unsigned long long* g_attn_trace = nullptr;
constexpr int TRACE_EV = 10, TRACE_TILES = 32;
__device__ __forceinline__ void trace(int j, int e) {
    if (g_attn_trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < TRACE_TILES) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        g_attn_trace[j * TRACE_EV + e] = t;
    }
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
// byte offset of 16-byte chunk `c` (0..7) of row `r` inside a K-major SW128 sub-tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ lo,
                   const int32_t* __restrict__ hi, __nv_bfloat16* __restrict__ out, float* __restrict__ ws_o,
                   float* __restrict__ ws_ml, int Tq, int Tk, int H, int Hkv, int splits, float scale, int* err,
                   L2Prefetch pf) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* k_full = bars;        // [2]
    uint64_t* k_empty = bars + 2;   // [2]
    uint64_t* v_full = bars + 4;    // [2]
    uint64_t* v_empty = bars + 6;   // [2]
    uint64_t* s_full = bars + 8;    // [2] S_j in TMEM
    uint64_t* p_full = bars + 10;   // [2] P_j in TMEM (all softmax threads arrived)
    uint64_t* pv_done = bars + 12;  // [2] PV_j retired: P buffer j&1 free, O current through j
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
    __shared__ int red_lo[THREADS / 32], red_hi[THREADS / 32];
    __shared__ float xmax[2][NQ][BR];  // [tile parity][quarter][row]: partial row maxima exchanged each tile

    pdl_launch();
    pdl_wait();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int group = H / Hkv, g = blockIdx.y, split = blockIdx.z;
    const int rows_total = Tq * group;
    const bool softmax = warp < SOFTMAX_WARPS;
    const int r = tid & (BR - 1);             // tile row (TMEM lane) of a softmax thread
    const int qtr = softmax ? warp >> 2 : 0;  // which CPT S columns / CPT O columns this thread owns
    const int row = blockIdx.x * BR + r;
    const bool active = softmax && row < rows_total;
    const int t = active ? row / group : 0;
    const int h = g * group + (active ? row % group : 0);
    const int my_lo = active ? lo[t] : INT32_MAX;
    const int my_hi = active ? min(hi[t], Tk - 1) : -1;

    // ---- CTA key range (union of its rows), then this split's share, in 128-key tiles ----
    int blo = my_lo, bhi = my_hi;
    for (int o = 16; o > 0; o >>= 1) {
        blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
        bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
    }
    if (lane == 0) {
        red_lo[warp] = blo;
        red_hi[warp] = bhi;
    }
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], SOFTMAX_WARPS * 32);
            mbar_init(&pv_done[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // ---- Q tile: each softmax thread stages its CPT columns of its row ----
    if (softmax) {
        constexpr int CH = CPT / 8;  // 16-byte chunks per thread
        const uint4* src = reinterpret_cast<const uint4*>(q + (int64_t)t * H * D + (int64_t)h * D) + qtr * CH;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const uint4 v = active ? src[c] : make_uint4(0, 0, 0, 0);
            const int chunk = qtr * CH + c;  // 0..15 over the 128 columns
            sts128(sbase + OFF_Q + (chunk >> 3) * SUB + swz(r, chunk & 7), v.x, v.y, v.z, v.w);
        }
        fence_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    blo = red_lo[0];
    bhi = red_hi[0];
    for (int w = 1; w < THREADS / 32; ++w) {
        blo = min(blo, red_lo[w]);
        bhi = max(bhi, red_hi[w]);
    }
    blo = max(blo, 0);
    const int span = bhi - blo + 1;
    const int chunk = span > 0 ? ((span + splits - 1) / splits + BK - 1) / BK * BK : 0;
    const int ks = blo + split * chunk;
    const int ke = min(bhi, ks + chunk - 1);
    const int n = (span > 0 && ke >= ks) ? (ke - ks + BK) / BK : 0;

    if (warp == SOFTMAX_WARPS) {
        if (lane == 1) {  // idle lane: optional L2 warm-up of the next projections' weights
            const int ncta = gridDim.x * gridDim.y * gridDim.z;
            const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
            for (int rr = 0; rr < 2; ++rr) {
                const size_t total = pf.bytes[rr] & ~size_t(15);
                if (!pf.ptr[rr] || total == 0) continue;
                const size_t share = ((total + ncta - 1) / ncta + 15) & ~size_t(15);
                const size_t b0 = (size_t)cta * share, b1 = b0 + share < total ? b0 + share : total;
                for (size_t off = b0; off < b1; off += 32768)
                    prefetch_l2(static_cast<const uint8_t*>(pf.ptr[rr]) + off,
                                (uint32_t)((b1 - off) < 32768 ? (b1 - off) : 32768));
            }
        }
        if (lane == 0) {  // ---------------- TMA producer ----------------
            for (int j = 0; j < n; ++j) {
                const int s = j & 1;
                const uint32_t par = ((j >> 1) & 1) ^ 1;
                const int key = ks + j * BK;
                mbar_wait(&k_empty[s], par);
                trace(j, 7);
                mbar_expect_tx(&k_full[s], KSTAGE);
                const uint32_t kd = sbase + OFF_K + s * KSTAGE;
                tma_load_2d(kd, &tmK, &k_full[s], g * D, key);
                tma_load_2d(kd + SUB, &tmK, &k_full[s], g * D + 64, key);
                mbar_wait(&v_empty[s], par);
                trace(j, 8);
                mbar_expect_tx(&v_full[s], KSTAGE);
                const uint32_t vd = sbase + OFF_V + s * KSTAGE;
                tma_load_2d(vd, &tmV, &v_full[s], g * D, key);
                tma_load_2d(vd + SUB, &tmV, &v_full[s], g * D + 64, key);
            }
        }
    } else if (warp == SOFTMAX_WARPS + 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            auto issue_s = [&](int j) {
                const int s = j & 1;
                mbar_wait(&k_full[s], (j >> 1) & 1);
                tc_fence_after();
                const uint32_t kb = sbase + OFF_K + s * KSTAGE;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * SUB + (kk & 3) * 32;
                    umma(tmem + TM_S + s * 128, desc_k(sbase + OFF_Q + off), desc_k(kb + off), IDESC_S, kk > 0);
                }
                umma_commit(&s_full[s]);
                umma_commit(&k_empty[s]);
                trace(j, 6);
            };
            if (n > 0) issue_s(0);
            if (n > 1) issue_s(1);
            for (int j = 0; j < n; ++j) {
                const int s = j & 1;
                mbar_wait(&p_full[s], (j >> 1) & 1);
                trace(j, 4);
                mbar_wait(&v_full[s], (j >> 1) & 1);
                tc_fence_after();
                const uint32_t vb = sbase + OFF_V + s * KSTAGE;
                // O += P_j . V_j : A = P_j from TMEM (8 columns = 16 keys per MMA), B = V (MN-major)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_ts(tmem + TM_O, tmem + TM_P + s * 64 + kk * 8, desc_mn(vb + kk * 2048), IDESC_PV,
                            (j > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&pv_done[s]);
                umma_commit(&v_empty[s]);
                trace(j, 5);
                if (j + 2 < n) issue_s(j + 2);
            }
        }
    } else {
        // ---------------- softmax: NQ threads per row, CPT columns each; O stays in TMEM ----------------
        const float sl2 = scale * LOG2E;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        float m_used = -INFINITY, l = 0.f;  // running max actually used for exp2, row-sum share
        for (int j = 0; j < n; ++j) {
            const int key0 = ks + j * BK + qtr * CPT;  // first key of this thread's columns
            const bool full = key0 >= my_lo && key0 + CPT - 1 <= my_hi;
            const int clo = my_lo - key0, chi = my_hi - key0;
            mbar_wait(&s_full[j & 1], (j >> 1) & 1);
            if (tid == 0) trace(j, 0);
            tc_fence_after();
            uint32_t v[CPT];
            tmem_ld32(tmem + lane_base + TM_S + (uint32_t)((j & 1) * 128) + qtr * CPT, v);
            tmem_wait_ld();
            if (!full) {  // masked columns -> -inf (per-tile branch; uniform in the common case)
#pragma unroll
                for (int i = 0; i < CPT; ++i)
                    v[i] = (i >= clo && i <= chi) ? v[i] : __float_as_uint(-INFINITY);
            }
            float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < CPT; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(v[i]));
            float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
            xmax[j & 1][qtr][r] = mx;
            asm volatile("bar.sync 1, %0;" ::"r"(SOFTMAX_WARPS * 32) : "memory");
#pragma unroll
            for (int k = 1; k < NQ; ++k) mx = fmaxf(mx, xmax[j & 1][(qtr + k) & (NQ - 1)][r]);
            if (tid == 0) trace(j, 1);
            mx = mx == -INFINITY ? -INFINITY : mx * sl2;
            if (m_used == -INFINITY) {
                m_used = mx;  // first visible keys: O is still all zeros, nothing to rescale
            } else if (mx > m_used + RESCALE_LOG2) {
                // rare: the row max grew by more than 2^8 -> rescale O (in TMEM) and l to the new max.
                // All four threads of the row take this branch together (same mx, same m_used).
                mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);  // O current through PV_{j-1}
                tc_fence_after();
                const float alpha = ex2(m_used - mx);
                uint32_t w[CPT];
                tmem_ld32(tmem + lane_base + TM_O + qtr * CPT, w);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < CPT; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
                tmem_st32(tmem + lane_base + TM_O + qtr * CPT, w);
                tmem_wait_st();
                l *= alpha;
                m_used = mx;
            }
            if (tid == 0) trace(j, 2);
            // P buffer j&1 is free once PV_{j-2} retired
            if (j >= 2) mbar_wait(&pv_done[j & 1], ((j - 2) >> 1) & 1);
            const float moff = m_used == -INFINITY ? 0.f : m_used;  // nothing visible yet -> all p = 0
            float rs4[4] = {0.f, 0.f, 0.f, 0.f};
            uint32_t pk[CPT / 2];
#pragma unroll
            for (int i = 0; i < CPT; i += 2) {
                const float p0 = ex2(fmaf(__uint_as_float(v[i]), sl2, -moff));
                const float p1 = ex2(fmaf(__uint_as_float(v[i + 1]), sl2, -moff));
                rs4[(i >> 1) & 3] += p0 + p1;
                pk[i >> 1] = pack_bf16(p0, p1);
            }
            // keys [qtr*CPT, +CPT) of this row = P columns [qtr*CPT/2, +CPT/2) of buffer j&1 (bf16 pairs)
            tc_fence_after();
            tmem_st16(tmem + lane_base + TM_P + (uint32_t)((j & 1) * 64) + qtr * (CPT / 2), pk);
            tmem_wait_st();
            l += (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
            tc_fence_before();
            mbar_arrive(&p_full[j & 1]);
            if (tid == 0) trace(j, 3);
        }
        float o[CPT];
        if (n > 0) {
            mbar_wait(&pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
            tc_fence_after();
            uint32_t w[CPT];
            tmem_ld32(tmem + lane_base + TM_O + qtr * CPT, w);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < CPT; ++i) o[i] = __uint_as_float(w[i]);
        } else {
#pragma unroll
            for (int i = 0; i < CPT; ++i) o[i] = 0.f;
        }
        // the NQ threads of a row hold partial sums l over disjoint key columns (same m_used)
        asm volatile("bar.sync 1, %0;" ::"r"(SOFTMAX_WARPS * 32) : "memory");
        xmax[0][qtr][r] = l;
        asm volatile("bar.sync 1, %0;" ::"r"(SOFTMAX_WARPS * 32) : "memory");
#pragma unroll
        for (int k = 1; k < NQ; ++k) l += xmax[0][(qtr + k) & (NQ - 1)][r];
        if (active) {
            const int64_t orow = (int64_t)t * H + h;
            if (splits == 1) {
                if (l == 0.f) {
                    if (qtr == 0) atomicOr(err, 8);  // DegenerateRowError (numerics.cpp:39-42)
                } else {
                    const float inv = 1.0f / l;
                    uint4* dst = reinterpret_cast<uint4*>(out + orow * D + qtr * CPT);
#pragma unroll
                    for (int c = 0; c < CPT / 8; ++c)
                        dst[c] = make_uint4(pack_bf16(o[8 * c] * inv, o[8 * c + 1] * inv),
                                            pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv),
                                            pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv),
                                            pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv));
                }
            } else {
                float4* wo = reinterpret_cast<float4*>(ws_o + ((int64_t)split * Tq * H + orow) * D + qtr * CPT);
#pragma unroll
                for (int c = 0; c < CPT / 4; ++c)
                    wo[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                if (qtr == 0) {
                    ws_ml[((int64_t)split * Tq * H + orow) * 2 + 0] = m_used == -INFINITY ? -INFINITY : m_used / LOG2E;
                    ws_ml[((int64_t)split * Tq * H + orow) * 2 + 1] = l;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
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
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap kv_map(const void* base, int rows, int cols, int ld) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

void attn_trace_enable(bool on, unsigned long long** host_view) {
    static unsigned long long* buf = nullptr;
    if (on && !buf) {
        TKV_CUDA(cudaMalloc(&buf, TRACE_EV * TRACE_TILES * 8));
        TKV_CUDA(cudaMemset(buf, 0, TRACE_EV * TRACE_TILES * 8));
    }
    unsigned long long* v = on ? buf : nullptr;
    TKV_CUDA(cudaMemcpyToSymbol(g_attn_trace, &v, sizeof v));
    if (host_view) *host_view = buf;
}

bool attention_tc_supported(int d, DT dt) { return d == 128 && dt == DT::BF16; }

int attn_tc_pick_splits(int Tq, int H, int Hkv, int Tk, int num_sms) {
    const int group = H / Hkv;
    const int ctas = ((Tq * group + BR - 1) / BR) * Hkv;
    int s = num_sms / ctas;  // 1 CTA per SM (192 KB smem): stay within one wave
    const int max_by_keys = (Tk + 4 * BK - 1) / (4 * BK);  // >= 4 key tiles per split
    if (s > max_by_keys) s = max_by_keys;
    if (s > 32) s = 32;
    return s < 1 ? 1 : s;
}

void launch_attention_tc(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                         const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws,
                         int* err, cudaStream_t s, const L2Prefetch& pf) {
    TKV_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    const CUtensorMap tk = kv_map(k, Tk, kv_stride, kv_stride);
    const CUtensorMap tv = kv_map(v, Tk, kv_stride, kv_stride);
    const int group = H / Hkv;
    dim3 grid((Tq * group + BR - 1) / BR, Hkv, splits);
    const float scale = (float)(1.0 / sqrt((double)D));
    launch_k(attn_tc_kernel, grid, THREADS, SMEM_BYTES, s, tk, tv, (const __nv_bfloat16*)q, lo, hi, (__nv_bfloat16*)out,
                                                     ws.o, ws.ml, Tq, Tk, H, Hkv, splits, scale, err, pf);
    TKV_CUDA(cudaGetLastError());
    if (splits > 1) launch_attention_combine(ws, Tq * H, D, splits, out, err, DT::BF16, s);
}

}  // namespace tkv

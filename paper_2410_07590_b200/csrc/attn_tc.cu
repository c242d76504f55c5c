// tcgen05 / TMEM / TMA flash attention for head_size 128, bf16 — the query-prefill attention of the
// TurboRAG path (and the full-concat comparison), replacing attend + softmax_rows_inplace
// (src/attention.cpp:94-169, src/numerics.cpp:31-60) with implicit masks: row t sees key j iff
// lo[t] <= j <= hi[t] (causal_rows / build_mask, attention.cpp:50-92).
//
// GQA packing: rows of ONE kv head g are (token t, head g*group + i), so every K/V tile a CTA streams
// serves all `group` query heads (C2: 64 tokens x 7 heads = 448 rows per kv head = 3.5 tiles of 128).
//
// v6 (one 128-row tile per CTA, S double-buffered, Q and P in TMEM, 16x256b softmax layout): see attn_tc_kernel.
// The tensor pipe runs S(j+1) while the softmax works on S(j), so the per-tile critical path is max(softmax, S + PV)
// rather than their sum (v4 kept two row tiles per CTA with one S buffer each and ping-ponged them: softmax + S + PV
// per tile, ~3.9 K cycles per pair of tiles; v6 ~1.9 K per tile with a third fewer shared-memory bytes per tile).
// Measured and dropped (tools/variant_ab.sh, C2 / C3): two softmax threads per row exchanging maxima through shared
// memory, four, separate K and V producer warps, 2- and 4-CTA clusters multicasting K/V (every ring slot then waits
// for the slowest CTA), try_wait suspend hints, and MUFU / polynomial exp split by warp.
// exp2 runs on two pipes: most pairs on MUFU.EX2, POLY_PAIRS of every 16 on the FMA pipe (Cody-Waite +
// degree-3 minimax, max rel err 7.5e-5, far below the bf16 rounding of P), with packed f32x2 FFMA2/FADD2
// and three-input FMNMX3 to keep the issue rate down. O is rescaled lazily, only when a row max grows by more
// than 2^8 (the stale max keeps every p <= 2^8, exact in fp32 and bf16 range).
// Context K/V rows below `kv_ready` were written before this forward began (the embed kernel that starts
// every forward does not release its dependents before its own griddepcontrol.wait), so their TMA loads
// are issued BEFORE griddepcontrol.wait and overlap the previous kernel's tail.
// Split-K over keys: every split stages its normalized output O/l (bf16) in shared memory, writes it
// coalesced to a per-row-group workspace with (m, l), and exits; attn_tc_merge_kernel (launched with PDL
// right behind, one half-warp per row, every load in flight) merges the splits. An in-kernel merge behind a
// grid-wide arrive counter was measured slower: the row group's CTAs wait for the slowest sibling and
// the merge loads then run at low memory-level parallelism.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int D = 128, BR = 128, BK = 128;                // rows per CTA (one tile), keys per tile
constexpr int RG = BR;                                    // rows per CTA = rows per workspace row group
static_assert(RG == kAttnTcRows, "engine-side row-group size");
#ifndef ATTN_KST
#define ATTN_KST 3
#endif
#ifndef ATTN_VST
#define ATTN_VST 2
#endif
constexpr int KST = ATTN_KST, VST = ATTN_VST;            // K / V ring depths (Q 32 KB + (KST + VST) x 32 KB <= 224 KB)
// Softmax warps 0-7: warp w owns TMEM lanes [32*(w%4) + 16*(w/4), +16) = 16 whole rows of the tile; with the
// 16x256b TMEM access shape lane t of the warp holds rows t/4 and t/4 + 8 of them, columns 8k + 2(t%4) + {0,1}
// (k = 0..15), so a row lives in the 4 lanes of one quad and its max / sum are two shuffles.
constexpr int SM_WARPS = 8, SM_THREADS = 32 * SM_WARPS;
constexpr int WARP_TMA = SM_WARPS, WARP_MMA = SM_WARPS + 1, THREADS = 32 * (WARP_MMA + 1);
#ifndef ATTN_DIAG
#define ATTN_DIAG 0  // cost-attribution variants (tools/attn_diag.sh); 0 = the product kernel
#endif
#ifndef ATTN_DEFER_REL
#define ATTN_DEFER_REL 1  // release P chunk c-1 after chunk c's exps (no wait::st stall per chunk)
#endif
#ifndef POLY_PAIRS
#define POLY_PAIRS 6
#endif
constexpr int kPolyPairs = POLY_PAIRS;                          // of every 16 exp2 pairs, this many on the FMA pipe
constexpr uint32_t SUB = 128 * 64 * 2;                   // [128 rows][64 cols] bf16 SW128 sub-tile = 16 KB
constexpr uint32_t TILE = 2 * SUB;                       // 128 x 128 bf16
constexpr uint32_t OFF_Q = 0;  // epilogue staging of the output tile
constexpr uint32_t OFF_K = TILE;
constexpr uint32_t OFF_V = OFF_K + KST * TILE;
constexpr uint32_t OFF_BAR = OFF_V + VST * TILE;
constexpr size_t SMEM_BYTES = 1024 + OFF_BAR + 256;
static_assert(SMEM_BYTES <= 232448, "attention smem budget");
// TMEM columns: O [0,128) fp32, S0 [128,256), S1 [256,384) fp32, P0 [384,448), P1 [448,512) bf16 pairs
// TMEM columns: O [0,128) fp32, S0 / S1 [128,384) fp32, P [384,448) and Q [448,512) bf16 pairs. Q in TMEM makes
// S = Q.K^T a TS MMA that reads only K from shared memory (an SS MMA at N = 128 reads A and B at ~110 B/clk, most
// of the SM's shared-memory bandwidth, which the TMA writes of the K/V ring also need).
constexpr uint32_t TMEM_COLS = 512, T_O = 0, T_S = 128, T_Q = 448;  // P(j) bf16 over S(j); [384, 448) spare
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_LOG2 = 8.0f;

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
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Bounded wait: a protocol bug traps (launch error) after ~2 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if ((spin & 1023) == 1023) {
            const uint64_t now = globaltimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 2000000000ull) __trap();
        }
    }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
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
// A operand from TMEM (P), B from shared memory (V)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// 16-lane shapes: 16x256b.x8 = 16 TMEM lanes x 64 columns; lane t of the warp gets, for k = 0..7, regs 4k, 4k+1 =
// (lane t/4, columns 8k + 2(t%4) + {0,1}) and regs 4k+2, 4k+3 = the same columns of lane t/4 + 8.
__device__ __forceinline__ void tmem_ld_16x256_x8(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_16x256_x8(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// 16x128b.x4 = 16 lanes x 16 columns; regs 2k, 2k+1 = column 4k + t%4 of lanes t/4 and t/4 + 8 (k = 0..3)
__device__ __forceinline__ void tmem_st_16x128_x4(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ---- packed f32x2 arithmetic (FFMA2 / FADD2) ----
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for a pair on the FMA pipe: x = j + f (j = rint(x) via the 1.5*2^23 shifter, f in [-0.5, 0.5]),
// 2^f by a degree-3 minimax polynomial (rel err 7.5e-5), 2^j added into the exponent field with one IMAD.
// 10 instructions per pair: 2 FMNMX, 2 FADD2, 4 FFMA2, 2 IMAD.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t xv) {
    float x0, x1;
    up2(xv, x0, x1);
    const uint64_t x = pk2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));  // keeps the result's biased exponent >= 0
    const uint64_t t = add2(x, pk2(12582912.0f, 12582912.0f));
    const uint64_t r = add2(t, pk2(-12582912.0f, -12582912.0f));
    const uint64_t f = fma2(r, pk2(-1.0f, -1.0f), x);
    uint64_t p = fma2(pk2(0.05517112836241722f, 0.05517112836241722f), f, pk2(0.24261008203029633f, 0.24261008203029633f));
    p = fma2(p, f, pk2(0.6932609677314758f, 0.6932609677314758f));
    p = fma2(p, f, pk2(0.9999281167984009f, 0.9999281167984009f));
    uint32_t tl, th, pl, ph;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(tl), "=r"(th) : "l"(t));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(pl), "=r"(ph) : "l"(p));
    uint64_t out;
    asm("{\n\t.reg .u32 a, b;\n\t"
        "mad.lo.u32 a, %1, 8388608, %3;\n\t"
        "mad.lo.u32 b, %2, 8388608, %4;\n\t"
        "mov.b64 %0, {a, b};\n\t}"
        : "=l"(out) : "r"(tl), "r"(th), "r"(pl), "r"(ph));
    return out;
}
__device__ __forceinline__ uint32_t bf16x2_bits(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// byte offset of 16-byte chunk `c` (0..7) of row `r` inside a K-major SW128 sub-tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Debug timeline (tkv_debug_attn_trace): CTA (0,0,0) stamps clock64 at pipeline events, slot [j][e]. The
// buffer pointer travels in the kernel arguments (a uniform constant-bank read, no global load on the path).
unsigned long long* g_trace_host = nullptr;
constexpr int TRACE_EV = 16, TRACE_TILES = 32, TRACE_CTA0 = TRACE_EV * TRACE_TILES, TRACE_CTAS = 1024;
__device__ __forceinline__ void trace_at(unsigned long long* buf, int j, int e) {
    if (buf && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < TRACE_TILES) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        buf[j * TRACE_EV + e] = t;
    }
}
#define trace(j, e) trace_at(a.trace, (j), (e))

struct AttnArgs {
    const __nv_bfloat16* q;
    const int32_t* lo;
    const int32_t* hi;
    __nv_bfloat16* out;
    float* ws_o;       // bf16 [splits][row groups][BR][D]: each split's normalized O/l (sized as fp32 ws)
    float* ws_ml;      // [splits][row groups][BR] (m in log2 units, l)
    int* err;
    int Tq, Tk, H, Hkv, splits, kv_ready;
    float scale;
    unsigned long long* trace;
    L2Prefetch pf;  // weights of the next projections, warmed into L2 by idle producer lanes
    // batched query prefill (n_req > 0): blockIdx.y = request * Hkv + kv head; request r's rows are tokens
    // [tok0, tok0 + n) of q/lo/hi/out, its keys the 3-D map maps3[r] over its cache ([2L][Tk][kvd], plane
    // 2 * layer + K|V)
    const AttnReq* reqs;
    const CUtensorMap* maps3;
    int n_req, layer;
    unsigned long long* tl;  // kernel timeline slot (tl_take)
    // single-request split-K with a compact last row tile (attn_tc_pick_splits): gx row tiles; splits_c > 0 flattens the
    // grid to blockIdx.x = the last tile's Hkv x splits_c CTAs, then the (gx - 1) full tiles x Hkv x `splits` CTAs
    int gx, splits_c;
};

// Warp-collective MMA issue: the whole MMA warp walks the loop (operands stay warp-uniform, in uniform registers);
// elect.sync picks the issuing lane, the same one every time, so a commit tracks every MMA it issued.
__device__ __forceinline__ void umma_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// v6: ONE 128-row tile per CTA, S double-buffered so the tensor pipe runs S(j+1) while the softmax works on S(j):
//   tensor pipe:  S(0) S(1) PV(0) S(2) PV(1) S(3) PV(2) ...
// S(j+2) may overwrite S buffer j & 1 once PV(j) was issued (its P chunks were released, so the softmax has loaded
// S(j)); P(j) is written over S(j) (bf16 pairs), so it is double-buffered with S. Warps 0-7 = softmax, 16 whole rows each (see
// SM_WARPS): every row statistic is quad-local and a warp rescales its own O rows. Warp 8 = TMA producer, warp 9 =
// MMA issuer (whole warp, elected lane).
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* k_full = bars;                 // [KST]
    uint64_t* k_empty = bars + KST;          // [KST]
    uint64_t* v_full = bars + 2 * KST;       // [VST]
    uint64_t* v_empty = v_full + VST;        // [VST]
    uint64_t* s_full = v_empty + VST;        // [2] S(j) in TMEM buffer j & 1
    uint64_t* p_full = s_full + 2;           // [2][4] chunk c (32 keys) of P(j) in buffer j & 1 (128 threads arrived)
    uint64_t* pv_done = p_full + 8;          // [2] PV(j) retired (O current through j; P buffer j & 1 free again)
    uint64_t* o_done = pv_done + 2;          // [1] every MMA retired
    uint64_t* q_ready = o_done + 1;          // [1] Q tile staged (256 threads arrived)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);
    __shared__ int sh_range[2];

    pdl_launch();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int group = a.H / a.Hkv;
    int bx = blockIdx.x, by = blockIdx.y, split = blockIdx.z, nsplit = a.splits;
    if (a.splits_c > 0) {  // flattened single-request grid (see AttnArgs::splits_c); the compact tile's CTAs, which
                           // carry the most key tiles, are launched first
        const int per = (a.gx - 1) * a.Hkv, nc = a.Hkv * a.splits_c;
        int b = blockIdx.x;
        if (b < nc) {
            split = b / a.Hkv;
            by = b - split * a.Hkv;
            bx = a.gx - 1;
            nsplit = a.splits_c;
        } else {
            b -= nc;
            split = b / per;
            b -= split * per;
            by = b / (a.gx - 1);
            bx = b - by * (a.gx - 1);
        }
    }
    int g = by, Tq = a.Tq, Tk = a.Tk, kv_ready = a.kv_ready;
    const __nv_bfloat16* qp = a.q;
    const int32_t* lop = a.lo;
    const int32_t* hip = a.hi;
    __nv_bfloat16* outp = a.out;
    const CUtensorMap* mK = &tmK;
    const CUtensorMap* mV = &tmV;
    if (a.n_req > 0) {  // batched: this CTA's request (the table was uploaded before the forward began)
        const int req = by / a.Hkv;
        g = by - req * a.Hkv;
        const AttnReq R = a.reqs[req];
        Tq = R.n;
        Tk = R.row0 + R.n;
        kv_ready = R.row0;
        qp += (int64_t)R.tok0 * a.H * D;
        outp += (int64_t)R.tok0 * a.H * D;
        lop += R.tok0;
        hip += R.tok0;
        mK = mV = a.maps3 + req;
    }
    const bool b3 = a.n_req > 0;
    const int rows_total = Tq * group;
    const int rr0 = bx * BR;                               // first row of this tile
    if (rr0 >= rows_total) return;                         // batched grid sized for the longest request
    // Compact tile (<= 64 valid rows, e.g. the last of 3.5 GQA tiles): row i of quadrant q (TMEM lanes 32q + i) holds
    // tile row 16q + i for i < 16, so each SMSP's softmax warp w < 4 has 16 valid rows and warps 4-7 have none (they
    // skip the tile loop): the softmax, which bounds the per-tile period, costs half an SMSP's issue per tile.
    const int nv = min(BR, rows_total - rr0);
    const bool compact = nv <= BR / 2;
    const int act_warps = compact ? SM_WARPS / 2 : SM_WARPS;

    const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);  // launch order
    if (tid == 0 && a.trace && cta_lin < TRACE_CTAS) a.trace[TRACE_CTA0 + 2 * cta_lin] = globaltimer_ns();
    if (tid == 0) {
        trace(0, 9);
        for (int s = 0; s < KST; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < VST; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&pv_done[b], 1);
            for (int c = 0; c < 4; ++c) mbar_init(&p_full[b * 4 + c], act_warps);  // one arrive per active warp
        }
        mbar_init(o_done, 1);
        mbar_init(q_ready, SM_THREADS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == WARP_TMA) {
        // key range of the tile = union of its tokens' [lo, hi] (lo/hi were uploaded before the forward)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mK)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mV)) : "memory");
        }
        const int t0 = rr0 / group, t1 = (min(rr0 + BR, rows_total) - 1) / group;
        int blo = INT32_MAX, bhi = -1;
        for (int t = t0 + lane; t <= t1; t += 32) {
            blo = min(blo, lop[t]);
            bhi = max(bhi, min(hip[t], Tk - 1));
        }
        for (int o = 16; o > 0; o >>= 1) {
            blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
            bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        if (lane == 0) {
            sh_range[0] = max(blo, 0);
            sh_range[1] = bhi;
        }
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int blo = sh_range[0], bhi = sh_range[1];
    const int span = bhi - blo + 1;
    const int chunk = span > 0 ? ((span + nsplit - 1) / nsplit + BK - 1) / BK * BK : 0;
    const int ks = blo + split * chunk;
    const int ke = min(bhi, ks + chunk - 1);
    const int n = (span > 0 && ke >= ks) ? (ke - ks + BK) / BK : 0;

    if (warp == WARP_TMA) {
        if (lane == 0) {  // ---------------- TMA producer: K(j) then V(j) into their rings ----------------
            auto load_tile = [&](bool k_tile, int j) {
                const CUtensorMap* m = k_tile ? mK : mV;
                uint64_t* full = k_tile ? k_full : v_full;
                uint64_t* empty = k_tile ? k_empty : v_empty;
                const int st = k_tile ? KST : VST;
                const int sl = j % st;
                mbar_wait(&empty[sl], ((uint32_t)(j / st) & 1u) ^ 1u);
                mbar_expect_tx(&full[sl], TILE);
                const uint32_t dst = sbase + (k_tile ? OFF_K : OFF_V) + sl * TILE;
                const int key = ks + j * BK;
                if (b3) {
                    const int plane = 2 * a.layer + (k_tile ? 0 : 1);
                    tma_load_3d(dst, m, &full[sl], g * D, key, plane);
                    tma_load_3d(dst + SUB, m, &full[sl], g * D + 64, key, plane);
                } else {
                    tma_load_2d(dst, m, &full[sl], g * D, key);
                    tma_load_2d(dst + SUB, m, &full[sl], g * D + 64, key);
                }
                trace(j, k_tile ? 6 : 7);
            };
            // K runs one tile ahead of V (K(j+1) before V(j)): V(j) waits for PV(j-2) to free its slot, and S(j+1)
            // must not queue behind that wait
            bool waited = false;
            auto ready = [&](int j) {
                if (!waited && ks + j * BK + BK > kv_ready) {  // rows written by the previous kernels of this forward
                    pdl_wait();
                    waited = true;
                }
            };
            if (n > 0) {
                ready(0);
                load_tile(true, 0);
            }
            for (int j = 0; j < n; ++j) {
                if (j + 1 < n) {
                    ready(j + 1);
                    load_tile(true, j + 1);
                }
                load_tile(false, j);
            }
            // HBM is mostly idle for the rest of the attention at query-prefill sizes: once this CTA's K/V loads are
            // all issued, warm L2 with its share of the next projections' weights (bulk prefetch, no completion
            // tracking). Issued earlier, the prefetch delays the first K/V tiles (measured).
            const int ncta = gridDim.x * gridDim.y * gridDim.z;
            for (int rg2 = 0; rg2 < 2; ++rg2) {
                const size_t total = a.pf.bytes[rg2] & ~size_t(15);
                if (!a.pf.ptr[rg2] || total == 0) continue;
                const size_t share = ((total + ncta - 1) / ncta + 15) & ~size_t(15);
                const size_t b0 = (size_t)cta_lin * share, b1 = min(b0 + share, total);
                for (size_t off = b0; off < b1; off += 65536)
                    prefetch_l2(static_cast<const uint8_t*>(a.pf.ptr[rg2]) + off, (uint32_t)min((size_t)65536, b1 - off));
            }
        }
    } else if (warp == WARP_MMA) {
        // ---------------- MMA issuer (whole warp, elected lane issues) ----------------
        mbar_wait(q_ready, 0);
        tc_fence_after();
        if (lane == 0) trace(0, 8);
        for (int j = 0; j <= n; ++j) {
            if (j < n) {  // S(j) = Q . K_j^T into S buffer j & 1 (free: P(j-2) was consumed, so S(j-2) was loaded)
                const int sk = j % KST;
                mbar_wait(&k_full[sk], (uint32_t)(j / KST) & 1u);
                tc_fence_after();
                if (lane == 0) trace(j, 14);
                const uint32_t kb = sbase + OFF_K + sk * TILE;
                const uint32_t sd = tmem + T_S + (uint32_t)(j & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * SUB + (kk & 3) * 32;
                    umma_ts_elect(sd, tmem + T_Q + kk * 8, desc_k(kb + off), IDESC_S, kk > 0);
                }
                commit_elect(&s_full[j & 1]);
                commit_elect(&k_empty[sk]);
                if (lane == 0) trace(j, 5);
            }
            if (j >= 1) {  // O += P(j-1) . V_{j-1}, P from TMEM, chunk by chunk as the softmax releases it
                const int jp = j - 1, sv = jp % VST;
                mbar_wait(&v_full[sv], (uint32_t)(jp / VST) & 1u);
                const uint32_t vb = sbase + OFF_V + sv * TILE;
                const uint32_t pb = tmem + T_S + (uint32_t)(jp & 1) * 128;  // P(jp) over S(jp)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    mbar_wait(&p_full[(jp & 1) * 4 + c], (uint32_t)(jp >> 1) & 1u);
                    tc_fence_after();
                    if (c == 3 && lane == 0) trace(jp, 15);
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        const int kk = 2 * c + k2;
#if ATTN_DIAG != 2  // 2: cost attribution only (wrong results): no PV MMAs
                        umma_ts_elect(tmem + T_O, pb + kk * 8, desc_mn(vb + kk * 2048), IDESC_PV, (jp > 0 || kk > 0) ? 1u : 0u);
#endif
                    }
                }
                commit_elect(&v_empty[sv]);
                commit_elect(&pv_done[jp & 1]);
                if (lane == 0) trace(jp, 4);
            }
        }
        commit_elect(o_done);
    } else {
        // ---------------- softmax: warp w owns tile rows [32*(w%4) + 16*(w/4), +16); lane t holds rows ra = .. + t/4
        // and rb = ra + 8, key columns 8k + 2*(t%4) + {0,1} of every tile (16x256b TMEM access) ----------------
        const int t0 = lane & 3;
        const int wr0 = (warp & 3) * 32 + (warp >> 2) * 16;  // first tile row (TMEM lane) of this warp
        const int ra = wr0 + (lane >> 2), rb = ra + 8;  // TMEM lanes
        // tile rows held by those lanes (compact: 16 per quadrant; BR = none)
        const int pa = compact ? ((ra & 31) < 16 ? 16 * (ra >> 5) + (ra & 31) : BR) : ra;
        const int pb = compact ? ((rb & 31) < 16 ? 16 * (rb >> 5) + (rb & 31) : BR) : rb;
        const bool act_a = pa < nv, act_b = pb < nv;
        const bool warp_on = warp < act_warps;
        const int ta = act_a ? (rr0 + pa) / group : 0, tb = act_b ? (rr0 + pb) / group : 0;
        const int lo_a = act_a ? lop[ta] : INT32_MAX, hi_a = act_a ? min(hip[ta], Tk - 1) : -1;
        const int lo_b = act_b ? lop[tb] : INT32_MAX, hi_b = act_b ? min(hip[tb], Tk - 1) : -1;
        constexpr int RPW = BR / SM_WARPS;  // rows per warp for the coalesced Q staging / output copy
        pdl_wait();  // q is produced by the previous kernel
        tl_wait(a.tl);
        if (tid == 0) trace(30, 3);
        {
            // Q rows ra, rb straight into TMEM: column c of a row holds d = 2c, 2c + 1; with the 16x256b shape this
            // lane supplies columns 8k + 2*t0 + {0,1}, i.e. d = 16k + 4*t0 + 0..3 (one 8-byte load per row and k)
            const int qra = rr0 + (act_a ? pa : 0), qrb = rr0 + (act_b ? pb : 0);
            const uint2* qa = reinterpret_cast<const uint2*>(qp + ((int64_t)(qra / group) * a.H + g * group + qra % group) * D) + t0;
            const uint2* qb = reinterpret_cast<const uint2*>(qp + ((int64_t)(qrb / group) * a.H + g * group + qrb % group) * D) + t0;
            uint32_t w[32];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint2 va = act_a ? qa[4 * k] : make_uint2(0u, 0u), vb = act_b ? qb[4 * k] : make_uint2(0u, 0u);
                w[4 * k] = va.x;
                w[4 * k + 1] = va.y;
                w[4 * k + 2] = vb.x;
                w[4 * k + 3] = vb.y;
            }
            tmem_st_16x256_x8(tmem + ((uint32_t)wr0 << 16) + T_Q, w);
            tmem_wait_st();
            tc_fence_before();
            if (tid == 0) trace(30, 5);
            mbar_arrive(q_ready);
        }
        const uint32_t lane_base = (uint32_t)wr0 << 16;
        const float sl2 = a.scale * LOG2E;
        float mu_a = -INFINITY, mu_b = -INFINITY, l_a = 0.f, l_b = 0.f;  // running max (log2 units, lazy) and sum
        for (int j = 0; j < (warp_on ? n : 0); ++j) {
            const uint32_t b = (uint32_t)(j & 1);
            mbar_wait(&s_full[b], (uint32_t)(j >> 1) & 1u);
            tc_fence_after();
            if (tid == 0) trace(j, 0);
            if (tid == 128) trace(j, 2);
            uint32_t s[64];  // [k = 0..15][ra c0, ra c1, rb c0, rb c1]
            const uint32_t tS = tmem + lane_base + T_S + b * 128;
            tmem_ld_16x256_x8(tS, s);
            tmem_ld_16x256_x8(tS + 64, s + 32);
            tmem_wait_ld();
            if (tid == 0) trace(j, 10);
            const int key0 = ks + j * BK + 2 * t0;  // key of element (k, e): key0 + 8k + e
            if (!(ks + j * BK >= max(lo_a, lo_b) && ks + j * BK + BK - 1 <= min(hi_a, hi_b))) {  // partial tile: mask
#pragma unroll
                for (int k = 0; k < 16; ++k)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int key = key0 + 8 * k + e;
                        if (key < lo_a || key > hi_a) s[4 * k + e] = __float_as_uint(-INFINITY);
                        if (key < lo_b || key > hi_b) s[4 * k + 2 + e] = __float_as_uint(-INFINITY);
                    }
            }
            float ma0 = __uint_as_float(s[0]), ma1 = __uint_as_float(s[1]);
            float mb0 = __uint_as_float(s[2]), mb1 = __uint_as_float(s[3]);
#pragma unroll
            for (int k = 1; k < 15; k += 2) {
                ma0 = max3(ma0, __uint_as_float(s[4 * k]), __uint_as_float(s[4 * k + 4]));
                ma1 = max3(ma1, __uint_as_float(s[4 * k + 1]), __uint_as_float(s[4 * k + 5]));
                mb0 = max3(mb0, __uint_as_float(s[4 * k + 2]), __uint_as_float(s[4 * k + 6]));
                mb1 = max3(mb1, __uint_as_float(s[4 * k + 3]), __uint_as_float(s[4 * k + 7]));
            }
            float mxa = max3(ma0, ma1, fmaxf(__uint_as_float(s[60]), __uint_as_float(s[61])));
            float mxb = max3(mb0, mb1, fmaxf(__uint_as_float(s[62]), __uint_as_float(s[63])));
            // the row max over the quad (the 4 lanes sharing the row)
            mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
            mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
            mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
            mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
            const float msa = mxa == -INFINITY ? -INFINITY : mxa * sl2;
            const float msb = mxb == -INFINITY ? -INFINITY : mxb * sl2;
            if (tid == 0) trace(j, 11);
            // lazy rescale: only when a row max grows by more than 2^8 (identical decisions in the 4 lanes of a row).
            // tcgen05.ld/st are warp-collective, so the whole warp takes the branch; rows that keep their max get 1.
            bool ga = false, gb = false;
            if (mu_a == -INFINITY) mu_a = msa;  // first visible keys: O is still all zeros
            else ga = msa > mu_a + RESCALE_LOG2;
            if (mu_b == -INFINITY) mu_b = msb;
            else gb = msb > mu_b + RESCALE_LOG2;
            if (__any_sync(0xffffffffu, ga || gb)) {
                // O must be current through PV(j-1) (j >= 1 here: a max was set by an earlier tile). This warp owns its
                // 16 O rows outright; PV(j) starts only after every warp released its P(j) chunks, i.e. after this.
                mbar_wait(&pv_done[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
                tc_fence_after();
                const float al_a = ga ? ex2(mu_a - msa) : 1.0f, al_b = gb ? ex2(mu_b - msb) : 1.0f;
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    uint32_t w[32];
                    const uint32_t tO = tmem + lane_base + T_O + c * 64;
                    tmem_ld_16x256_x8(tO, w);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * ((i & 2) ? al_b : al_a));
                    tmem_st_16x256_x8(tO, w);
                }
                tmem_wait_st();
                if (ga) {
                    l_a *= al_a;
                    mu_a = msa;
                }
                if (gb) {
                    l_b *= al_b;
                    mu_b = msb;
                }
            }
            // P(j) overwrites S(j) in place (bf16 pairs in the buffer's first 64 columns; S(j) is already in registers):
            // its previous P(j-2) was read by PV(j-2), which the tensor pipe retired before S(j), so no wait here
            const float oa = mu_a == -INFINITY ? 0.f : mu_a, ob = mu_b == -INFINITY ? 0.f : mu_b;  // none visible: p = 0
            const uint64_t sc2 = pk2(sl2, sl2), na2 = pk2(-oa, -oa), nb2 = pk2(-ob, -ob);
            uint64_t acca = 0, accb = 0;  // (+0, +0)
            const uint32_t tP = tS;
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // chunk c = keys [32c, 32c+32) = k in [4c, 4c+4): 16 P columns, 8 regs
                uint64_t pv[8];            // [kk][row a, row b] pairs
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int k = 4 * c + (i >> 1), rsel = i & 1;
                    const uint64_t xv = fma2(pk2(__uint_as_float(s[4 * k + 2 * rsel]), __uint_as_float(s[4 * k + 2 * rsel + 1])),
                                             sc2, rsel ? nb2 : na2);
#if ATTN_DIAG == 1  // cost attribution only (wrong results): no exp work
                    if (true) {
                        pv[i] = xv;
                    } else
#endif
                    if (((c * 8 + i) & 15) < kPolyPairs) {  // POLY_PAIRS of every 16 pairs on the FMA pipe
                        pv[i] = ex2_poly2(xv);
                    } else {
                        float x0, x1;
                        up2(xv, x0, x1);
                        pv[i] = pk2(ex2(x0), ex2(x1));
                    }
                }
                uint32_t pk[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float p0, p1;
                    up2(pv[i], p0, p1);
                    pk[i] = bf16x2_bits(p0, p1);
                }
                if (tid == 0 && c == 0) trace(j, 12);
#if ATTN_DEFER_REL
                // chunk c-1's store had this chunk's exp work to land: release it now (no stall on tcgen05.wait::st)
                if (c > 0) {
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&p_full[b * 4 + c - 1]);  // the PV MMA on those 32 keys may start
                    if (tid == 0 && c == 1) trace(j, 13);
                }
                tmem_st_16x128_x4(tP + c * 16, pk);
                acca = add2(acca, add2(add2(pv[0], pv[2]), add2(pv[4], pv[6])));
                accb = add2(accb, add2(add2(pv[1], pv[3]), add2(pv[5], pv[7])));
#else
                tmem_st_16x128_x4(tP + c * 16, pk);
                acca = add2(acca, add2(add2(pv[0], pv[2]), add2(pv[4], pv[6])));
                accb = add2(accb, add2(add2(pv[1], pv[3]), add2(pv[5], pv[7])));
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[b * 4 + c]);  // the PV MMA on these 32 keys may start
                if (tid == 0 && c == 0) trace(j, 13);
#endif
            }
#if ATTN_DEFER_REL
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[b * 4 + 3]);
#endif
            // observe PV(j-1) retiring (it ran during this tile's softmax): P no longer waits on it, but every pv_done
            // phase is consumed before its next arrive, so the parity wait of the lazy rescale stays unambiguous
            if (j >= 1) mbar_wait(&pv_done[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
            float a0, a1;
            up2(acca, a0, a1);
            l_a += a0 + a1;
            up2(accb, a0, a1);
            l_b += a0 + a1;
            if (tid == 0) trace(j, 1);
            if (tid == 128) trace(j, 3);
        }
        // row sums over the quad
        l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
        l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
        l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
        l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
        if (n > 0 && warp_on) {
            mbar_wait(o_done, 0);
            tc_fence_after();
        }
        if (tid == 0) trace(31, 0);
        // ---- epilogue: O/l as bf16 pairs into the (now idle) Q tile with the SW128 chunk swizzle (a quad writes one
        // 16-byte chunk of a row: conflict-free), then copied out coalesced: 16 lanes x 16 B per 256-byte row ----
        const float inv_a = l_a > 0.f ? 1.0f / l_a : 0.f, inv_b = l_b > 0.f ? 1.0f / l_b : 0.f;
        const uint32_t stage = sbase + OFF_Q;
#pragma unroll 1
        for (int c = 0; c < (warp_on ? 2 : 0); ++c) {  // compact tile: warps 4-7 hold no rows
            uint32_t w[32];
            if (n > 0) {
                tmem_ld_16x256_x8(tmem + lane_base + T_O + c * 64, w);  // warp-collective
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = 0u;
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int ch = c * 8 + kk;  // 16-byte chunk (8 columns) of the 256-byte row
                const uint32_t off = (ch >> 3) * SUB + 4 * t0;
                sts32(stage + off + swz(pa, ch & 7),
                      bf16x2_bits(__uint_as_float(w[4 * kk]) * inv_a, __uint_as_float(w[4 * kk + 1]) * inv_a));
                sts32(stage + off + swz(pb, ch & 7),
                      bf16x2_bits(__uint_as_float(w[4 * kk + 2]) * inv_b, __uint_as_float(w[4 * kk + 3]) * inv_b));
            }
        }
        named_bar(1, SM_THREADS);  // the whole tile is staged
        if (tid == 0) trace(31, 5);
        const int gid = by * a.gx + bx;  // row group (kv head or request x kv head, row tile)
        const int ngroups = a.splits_c > 0 ? a.gx * a.Hkv : a.gx * gridDim.y;
        // workspace of split s, row group gid: rows [BR][D] bf16 (contiguous) and (m, l) [BR]
        const int64_t wrow0 = ((int64_t)split * ngroups + gid) * BR;
        {
            const int cc = lane & 15;
#pragma unroll
            for (int it = 0; it < RPW / 2; ++it) {
                const int row = warp * RPW + it * 2 + (lane >> 4);
                const int qr = rr0 + row;
                uint4 v;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(stage + (cc >> 3) * SUB + swz(row, cc & 7)));
                if (a.splits == 1) {
                    if (qr < rows_total)
                        reinterpret_cast<uint4*>(outp + ((int64_t)(qr / group) * a.H + g * group + qr % group) * D)[cc] = v;
                } else {
                    reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.ws_o) + (wrow0 + row) * D)[cc] = v;
                }
            }
        }
        if (tid == 0) trace(31, 6);
        if (t0 == 0 && warp_on) {
            if (a.splits == 1) {
                if ((act_a && l_a == 0.f) || (act_b && l_b == 0.f)) atomicOr(a.err, 8);  // DegenerateRowError (numerics.cpp:39-42)
            } else {
                float2* ml = reinterpret_cast<float2*>(a.ws_ml) + wrow0;
                ml[pa] = make_float2(act_a ? mu_a : -INFINITY, l_a);
                ml[pb] = make_float2(act_b ? mu_b : -INFINITY, l_b);
                if (tid == 0) trace(31, 1);
                if (tid == 0 && a.trace && cta_lin == 0) a.trace[31 * TRACE_EV + 7] = globaltimer_ns();  // clock check
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0 && a.trace && cta_lin < TRACE_CTAS) a.trace[TRACE_CTA0 + 2 * cta_lin + 1] = globaltimer_ns();
    if (tid == 0 && a.tl) atomicMax(a.tl + 1, gtimer_ns());
    if (warp == WARP_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// Many-split merge of the single-request launch (C2: 9 splits over 16 row groups): one warp per row, lane = 4
// columns, every split's load in flight; measured faster there than the half-warp kernel below (2.0 vs 3.3 us).
__global__ void __launch_bounds__(256) attn_tc_combine_kernel(const __nv_bfloat16* __restrict__ ws_o,
                                                              const float2* __restrict__ ws_ml,
                                                              __nv_bfloat16* __restrict__ out, int* err, int Tq, int H,
                                                              int Hkv, int splits, int groups_x, int splits_c,
                                                              unsigned long long* tl) {
    pdl_launch();
    const int lane = threadIdx.x & 31;
    const int grow = blockIdx.x * 8 + (threadIdx.x >> 5);  // row over all row groups: gid * RG + i
    const int gid = grow / RG, i = grow % RG;
    const int g = gid / groups_x, rr = (gid % groups_x) * RG + i;  // kv head, row within the kv head
    const int group = H / Hkv;
    const bool ok = rr < Tq * group;
    const int64_t plane = (int64_t)groups_x * Hkv * RG;
    if (splits_c > 0 && gid % groups_x == groups_x - 1) splits = splits_c;  // the compact last tile's split count
    pdl_wait();
    tl_wait(tl);
    if (!ok) return;  // warp-uniform
    const uint2* src = reinterpret_cast<const uint2*>(ws_o + (int64_t)grow * D) + lane;
    uint2 v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k)
        if (k < splits) v[k] = src[(int64_t)k * plane * (D / 4)];
    const float2 ml = lane < splits ? ws_ml[lane * plane + grow] : make_float2(-INFINITY, 0.f);
    float M = ml.x;
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float wl = ml.x == -INFINITY ? 0.f : ex2(ml.x - M) * ml.y;
    float L = wl;
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (M == -INFINITY || L == 0.f) {
        if (lane == 0) atomicOr(err, 8);  // DegenerateRowError (numerics.cpp:39-42)
        return;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k >= splits) break;
        const float w = __shfl_sync(0xffffffffu, wl, k);
        acc[0] = fmaf(__uint_as_float(v[k].x << 16), w, acc[0]);
        acc[1] = fmaf(__uint_as_float(v[k].x & 0xFFFF0000u), w, acc[1]);
        acc[2] = fmaf(__uint_as_float(v[k].y << 16), w, acc[2]);
        acc[3] = fmaf(__uint_as_float(v[k].y & 0xFFFF0000u), w, acc[3]);
    }
    const float inv = 1.0f / L;
    const int64_t mo = (int64_t)(rr / group) * H + g * group + rr % group;
    reinterpret_cast<uint2*>(out + mo * D)[lane] =
        make_uint2(bf16x2_bits(acc[0] * inv, acc[1] * inv), bf16x2_bits(acc[2] * inv, acc[3] * inv));
    tl_exit(tl);
}

// Split merge (PDL-launched right behind the attention grid): one half-warp per row (16 lanes x 8 columns), rows
// grid-strided, every split's partial and (m, l) loaded before use; MAXS (power of two >= splits) sizes the
// in-flight loads so few-split merges keep a full SM of warps resident. out = sum_s w_s (O_s / l_s) / sum_s w_s,
// w_s = 2^(m_s - M) * l_s (numerics.cpp:31-60 softmax, regrouped over key splits). Row groups are (kv head, x)
// or, BATCHED, (request, kv head, x) with each request's rows / output rows from its AttnReq (tok0, n).
template <bool BATCH, int MAXS>
__global__ void __launch_bounds__(256) attn_tc_merge_kernel(const __nv_bfloat16* __restrict__ ws_o,
                                                            const float2* __restrict__ ws_ml,
                                                            __nv_bfloat16* __restrict__ out, int* err,
                                                            const AttnReq* __restrict__ reqs, int Tq, int H, int Hkv,
                                                            int splits_all, int groups_x, int nrows, int splits_c,
                                                            unsigned long long* tl) {
    pdl_launch();
    const int hl = threadIdx.x & 15;
    const unsigned hm = (threadIdx.x & 16) ? 0xFFFF0000u : 0x0000FFFFu;
    const int group = H / Hkv;
    const int64_t plane = nrows;  // rows per split plane
    pdl_wait();
    tl_wait(tl);
    for (int grow = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 4); grow < nrows; grow += gridDim.x * 16) {
        const int gid = grow / RG, i = grow % RG;
        const int y = gid / groups_x, rr = (gid % groups_x) * RG + i;
        const int splits = (splits_c > 0 && gid % groups_x == groups_x - 1) ? splits_c : splits_all;
        int g = y, tok0 = 0, n = Tq;
        if (BATCH) {
            const int req = y / Hkv;
            g = y - req * Hkv;
            const AttnReq R = reqs[req];
            tok0 = R.tok0;
            n = R.n;
        }
        if (rr >= n * group) continue;  // half-warp-uniform
        const uint4* src = reinterpret_cast<const uint4*>(ws_o + (int64_t)grow * D) + hl;
        uint4 v[MAXS];
#pragma unroll
        for (int k = 0; k < MAXS; ++k)
            if (k < splits) v[k] = src[(int64_t)k * plane * (D / 8)];
        const float2 ml0 = hl < splits ? ws_ml[hl * plane + grow] : make_float2(-INFINITY, 0.f);
        const float2 ml1 = (MAXS > 16 && hl + 16 < splits) ? ws_ml[(hl + 16) * plane + grow] : make_float2(-INFINITY, 0.f);
        float M = fmaxf(ml0.x, ml1.x);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(hm, M, o, 16));
        const float w0 = ml0.x == -INFINITY ? 0.f : ex2(ml0.x - M) * ml0.y;
        const float w1 = ml1.x == -INFINITY ? 0.f : ex2(ml1.x - M) * ml1.y;
        float L = w0 + w1;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) L += __shfl_xor_sync(hm, L, o, 16);
        if (M == -INFINITY || L == 0.f) {
            if (hl == 0) atomicOr(err, 8);  // DegenerateRowError (numerics.cpp:39-42)
            continue;
        }
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
            if (k >= splits) break;
            const float w = __shfl_sync(hm, k < 16 ? w0 : w1, k & 15, 16);
            const uint32_t u[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                acc[2 * c] = fmaf(__uint_as_float(u[c] << 16), w, acc[2 * c]);
                acc[2 * c + 1] = fmaf(__uint_as_float(u[c] & 0xFFFF0000u), w, acc[2 * c + 1]);
            }
        }
        const float inv = 1.0f / L;
        const int64_t mo = (int64_t)(tok0 + rr / group) * H + g * group + rr % group;
        reinterpret_cast<uint4*>(out + mo * D)[hl] =
            make_uint4(bf16x2_bits(acc[0] * inv, acc[1] * inv), bf16x2_bits(acc[2] * inv, acc[3] * inv),
                       bf16x2_bits(acc[4] * inv, acc[5] * inv), bf16x2_bits(acc[6] * inv, acc[7] * inv));
    }
    tl_exit(tl);
}

template <bool BATCH>
void launch_merge(const AttnWork& ws, void* out, int* err, const AttnReq* reqs, int Tq, int H, int Hkv, int splits,
                  int groups_x, int nrows, cudaStream_t s, int splits_c = 0) {
    const dim3 grid((unsigned)std::min((nrows + 15) / 16, 148 * 8)), block(256);
    const auto* o = reinterpret_cast<const __nv_bfloat16*>(ws.o);
    const auto* ml = reinterpret_cast<const float2*>(ws.ml);
    auto* dst = static_cast<__nv_bfloat16*>(out);
    unsigned long long* tl = tl_take();
#define TKV_MERGE(S)                                                                                                 \
    launch_k(attn_tc_merge_kernel<BATCH, S>, grid, block, 0, s, o, ml, dst, err, reqs, Tq, H, Hkv, splits, groups_x, \
             nrows, splits_c, tl)
    if (splits <= 2) TKV_MERGE(2);
    else if (splits <= 4) TKV_MERGE(4);
    else if (splits <= 8) TKV_MERGE(8);
    else if (splits <= 16) TKV_MERGE(16);
    else TKV_MERGE(32);
#undef TKV_MERGE
    TKV_CUDA(cudaGetLastError());
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

void attn_tc_cache_map(const void* cache, int64_t rows, int64_t cap, int kv_dim, int L, void* map128) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {(cuuint64_t)kv_dim, (cuuint64_t)rows, (cuuint64_t)(2 * L)};
    const cuuint64_t strides[2] = {(cuuint64_t)kv_dim * 2, (cuuint64_t)(cap * kv_dim * 2)};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(cache), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled (cache map) failed: " + std::to_string((int)r));
    static_assert(sizeof(CUtensorMap) == 128, "tensor map size");
    memcpy(map128, &m, sizeof m);
}

void launch_attention_tc_batch(const void* q, const AttnReq* reqs, const void* maps, int n_req, int max_rows, int H,
                               int Hkv, int layer, const int32_t* lo, const int32_t* hi, void* out, int* err,
                               cudaStream_t s, int splits, const AttnWork& ws) {
    TKV_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    const int group = H / Hkv;
    AttnArgs a{};
    a.q = (const __nv_bfloat16*)q;
    a.lo = lo;
    a.hi = hi;
    a.out = (__nv_bfloat16*)out;
    a.err = err;
    a.H = H;
    a.Hkv = Hkv;
    a.splits = splits < 1 ? 1 : splits;
    if (a.splits > 1 && !ws.o) fail(TKV_ERR_CONFIG, "batched attention split-K needs its workspace");
    a.ws_o = ws.o;
    a.ws_ml = ws.ml;
    a.scale = (float)(1.0 / sqrt((double)D));
    a.trace = g_trace_host;
    a.reqs = reqs;
    a.maps3 = static_cast<const CUtensorMap*>(maps);
    a.n_req = n_req;
    a.layer = layer;
    CUtensorMap unused;
    memset(&unused, 0, sizeof unused);
    const int groups_x = (max_rows * group + RG - 1) / RG;
    a.gx = groups_x;
    a.tl = tl_take();
    launch_k(attn_tc_kernel, dim3(groups_x, Hkv * n_req, a.splits), THREADS, SMEM_BYTES, s, unused, unused, a);
    TKV_CUDA(cudaGetLastError());
    if (a.splits > 1)
        launch_merge<true>(ws, out, err, reqs, 0, H, Hkv, a.splits, groups_x, groups_x * Hkv * n_req * RG, s);
}

// split-K of the batched launch: the smallest split count whose CTA count fills the last wave (>= 95 % of the
// slots), so the request x kv-head x row-group CTAs do not leave most of a second wave idle; 1 when the key
// range per split would drop below 8 tiles
int attn_tc_batch_pick_splits(int ctas, int min_keys, int num_sms) {
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8; ++s) {
        if (s > 1 && min_keys / s < 8 * BK) break;
        const int64_t c = (int64_t)ctas * s;
        const double eff = (double)c / (double)(((c + num_sms - 1) / num_sms) * num_sms);
        if (eff > best_eff + 0.02) {
            best = s;
            best_eff = eff;
        }
        if (eff >= 0.95) break;
    }
    return best;
}

void attn_trace_enable(bool on, unsigned long long** host_view) {
    static unsigned long long* buf = nullptr;
    if (on && !buf) {
        TKV_CUDA(cudaMalloc(&buf, (TRACE_CTA0 + 2 * TRACE_CTAS) * 8));
        TKV_CUDA(cudaMemset(buf, 0, (TRACE_CTA0 + 2 * TRACE_CTAS) * 8));
    }
    g_trace_host = on ? buf : nullptr;
    if (host_view) *host_view = buf;
}

int attn_trace_words() { return TRACE_CTA0 + 2 * TRACE_CTAS; }

bool attention_tc_supported(int d, DT dt) { return d == 128 && dt == DT::BF16; }

int attn_tc_row_groups(int Tq, int H, int Hkv) { return ((Tq * (H / Hkv) + RG - 1) / RG) * Hkv; }

size_t attn_tc_workspace_floats(int Tq, int H, int Hkv, int splits, size_t* ml_offset) {
    if (splits <= 1) return 0;
    const size_t rows = (size_t)splits * attn_tc_row_groups(Tq, H, Hkv) * RG;
    if (ml_offset) *ml_offset = rows * D / 2;  // bf16 partials first, then (m, l) pairs
    return rows * D / 2 + rows * 2;
}

int attn_tc_pick_splits(int Tq, int H, int Hkv, int Tk, int num_sms) {
    const int groups = attn_tc_row_groups(Tq, H, Hkv);
    if (groups * 2 > num_sms) return 1;  // already >= half a wave of row tiles: no split-K
    int s = num_sms / groups;            // one wave (1 CTA / SM)
    const int max_by_keys = ((Tk + BK - 1) / BK + 1) / 2;  // >= 2 key tiles per split
    const int rows = Tq * (H / Hkv), gx = (rows + RG - 1) / RG;
    // a compact last row tile takes fewer, longer splits: the SMs it frees go to more splits of the full tiles
    while (s + 1 <= max_by_keys && s + 1 <= 32 && attn_tc_compact_splits(rows, gx, s + 1) > 0 &&
           (gx - 1) * Hkv * (s + 1) + Hkv * attn_tc_compact_splits(rows, gx, s + 1) <= num_sms)
        ++s;
    if (s > max_by_keys) s = max_by_keys;
    if (s > 32) s = 32;
    return s < 1 ? 1 : s;
}

// split count of a compact last row tile (<= BR / 2 valid rows, behind >= 1 full tile) under `splits` for the full
// tiles: its per-tile period is ~0.65 of a full tile's (one softmax warp per SMSP instead of two); 0 = no compact tile
int attn_tc_compact_splits(int rows, int gx, int splits) {
    const int last = rows - (gx - 1) * RG;
    if (gx < 2 || splits < 2 || last > RG / 2) return 0;
    return std::max(1, (13 * splits + 19) / 20);
}

void launch_attention_tc(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                         const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws,
                         int* err, cudaStream_t s, int kv_ready, const L2Prefetch& pf) {
    TKV_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    const int group = H / Hkv;
    dim3 grid((Tq * group + RG - 1) / RG, Hkv, splits);
    if (splits > 1 && !ws.o) fail(TKV_ERR_CONFIG, "attention split-K needs its workspace");
    AttnArgs a{};
    a.q = (const __nv_bfloat16*)q;
    a.lo = lo;
    a.hi = hi;
    a.out = (__nv_bfloat16*)out;
    a.ws_o = ws.o;
    a.ws_ml = ws.ml;
    a.err = err;
    a.Tq = Tq;
    a.Tk = Tk;
    a.H = H;
    a.Hkv = Hkv;
    a.splits = splits;
    a.kv_ready = kv_ready;
    a.scale = (float)(1.0 / sqrt((double)D));
    a.trace = g_trace_host;
    a.pf = pf;
    const CUtensorMap tk = kv_map(k, Tk, kv_stride, kv_stride);
    const CUtensorMap tv = kv_map(v, Tk, kv_stride, kv_stride);
    a.gx = (int)grid.x;
    a.splits_c = attn_tc_compact_splits(Tq * group, (int)grid.x, splits);
    const dim3 lgrid = a.splits_c > 0 ? dim3((grid.x - 1) * Hkv * splits + Hkv * a.splits_c) : grid;
    a.tl = tl_take();
    launch_k(attn_tc_kernel, lgrid, THREADS, SMEM_BYTES, s, tk, tv, a);
    TKV_CUDA(cudaGetLastError());
    const int rows = (int)(grid.x * grid.y) * RG;
    if (splits > 4) {
        launch_k(attn_tc_combine_kernel, dim3(rows / 8), dim3(256), 0, s, (const __nv_bfloat16*)ws.o,
                 (const float2*)ws.ml, (__nv_bfloat16*)out, err, Tq, H, Hkv, splits, (int)grid.x, a.splits_c, tl_take());
        TKV_CUDA(cudaGetLastError());
    } else if (splits > 1) {
        launch_merge<false>(ws, out, err, nullptr, Tq, H, Hkv, splits, (int)grid.x, rows, s, a.splits_c);
    }
}

}  // namespace tkv

// tcgen05 / TMEM / TMA flash attention for head_size 128, bf16 — the query-prefill attention of the
// TurboRAG path (and the full-concat comparison), replacing attend + softmax_rows_inplace
// (src/attention.cpp:94-169, src/numerics.cpp:31-60) with implicit masks: row t sees key j iff
// lo[t] <= j <= hi[t] (causal_rows / build_mask, attention.cpp:50-92).
//
// GQA packing: rows of ONE kv head g are (token t, head g*group + i), so every K/V tile a CTA streams
// serves all `group` query heads (C2: 64 tokens x 7 heads = 448 rows per kv head).
//
// v4 (ping-pong): a CTA owns a ROW GROUP of 256 rows = two 128-row tiles A and B of the same kv head and
// streams one split of the key range through them:
//   tensor pipe:  [PV_A(j-1) S_A(j)] [PV_B(j-1) S_B(j)] [PV_A(j) S_A(j+1)] ...
//   softmax WG A works on S_A(j) while the pipe runs the B bracket, and vice versa, so the tensor pipe
//   and the softmax (MUFU + FMA pipes) overlap; every K/V tile is read once for 256 rows.
// Warps 0-3 = softmax A, 4-7 = softmax B (ONE thread per row: no cross-thread max exchange), warp 8 =
// TMA producer, warp 9 = MMA issuer. TMEM (512 cols): S_A 0, O_A 128, S_B 256, O_B 384; P_X (bf16 pairs,
// 64 cols) is written over the first half of S_X and fed to the PV tcgen05.mma as the A operand from TMEM.
// O accumulates in TMEM; it is rescaled lazily, only when a row max grows by more than 2^8 (the stale max
// keeps every p <= 2^8, exact in fp32 and bf16 range).
// exp2 runs on two pipes: most pairs on MUFU.EX2, POLY_PAIRS of every 16 on the FMA pipe (Cody-Waite +
// degree-3 minimax, max rel err 7.5e-5, far below the bf16 rounding of P), with packed f32x2 FFMA2/FADD2
// and three-input FMNMX3 to keep the issue rate down.
// Context K/V rows below `kv_ready` were written before this forward began (the embed kernel that starts
// every forward does not release its dependents before its own griddepcontrol.wait), so their TMA loads
// are issued BEFORE griddepcontrol.wait and overlap the previous kernel's tail.
// Split-K over keys: every split stages its normalized output O/l (bf16) in shared memory, writes it
// coalesced to a per-row-group workspace with (m, l), and exits; attn_tc_combine_kernel (launched with PDL
// right behind, one warp per row, every load in flight) merges the splits. An in-kernel merge behind a
// grid-wide arrive counter was measured slower: the row group's CTAs wait for the slowest sibling and
// the merge loads then run at low memory-level parallelism.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <mutex>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int D = 128, BR = 128, BK = 128, RG = 2 * BR;  // rows per tile, keys per tile, rows per CTA
#ifndef ATTN_KST
#define ATTN_KST 3
#endif
#ifndef ATTN_VST
#define ATTN_VST 2
#endif
constexpr int KST = ATTN_KST, VST = ATTN_VST;            // K / V ring depths (Q 64 KB + (KST + VST) x 32 KB <= 224 KB)
constexpr int SM_THREADS = 256, THREADS = SM_THREADS + 64;
#ifndef POLY_PAIRS
#define POLY_PAIRS 6
#endif
constexpr int kPolyPairs = POLY_PAIRS;                          // of every 16 exp2 pairs, this many on the FMA pipe
constexpr uint32_t SUB = 128 * 64 * 2;                   // [128 rows][64 cols] bf16 SW128 sub-tile = 16 KB
constexpr uint32_t TILE = 2 * SUB;                       // 128 x 128 bf16
constexpr uint32_t OFF_Q = 0;                            // Q_A, Q_B
constexpr uint32_t OFF_K = 2 * TILE;
constexpr uint32_t OFF_V = OFF_K + KST * TILE;
constexpr uint32_t OFF_BAR = OFF_V + VST * TILE;
constexpr size_t SMEM_BYTES = 1024 + OFF_BAR + 256;
constexpr uint32_t TMEM_COLS = 512;
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
constexpr int TRACE_EV = 10, TRACE_TILES = 32, TRACE_CTA0 = TRACE_EV * TRACE_TILES, TRACE_CTAS = 1024;
__device__ __forceinline__ void trace_at(unsigned long long* buf, int j, int e) {
    if (buf && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < TRACE_TILES) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        buf[j * TRACE_EV + e] = t;
    }
}
#define trace(j, e) trace_at(a.trace, (j), (e))
#ifndef TRACE_SM
#define TRACE_SM 0  // 1: events 4-8 stamp softmax-internal points of thread 0 instead of the MMA/TMA warps
#endif
#define trace_pipe(j, e) do { if (!TRACE_SM) trace(j, e); } while (0)
#define trace_mma(j, e) do { if (TRACE_SM == 2) trace(j, e); } while (0)
#define trace_sm(j, e) do { if (TRACE_SM == 1 && tid == 0) trace(j, e); } while (0)

struct AttnArgs {
    const __nv_bfloat16* q;
    const int32_t* lo;
    const int32_t* hi;
    __nv_bfloat16* out;
    float* ws_o;       // bf16 [splits][row groups][256][D]: each split's normalized O/l (sized as fp32 ws)
    float* ws_ml;      // [splits][row groups][256] (m in log2 units, l)
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
};

// 10 warps: 3 share an SM sub-partition's 16K registers -> at most 168 registers per thread
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
    uint64_t* s_full = v_empty + VST;        // [2] S_X(j) in TMEM
    uint64_t* p_full = s_full + 2;           // [2][4] chunk c (32 keys) of P_X(j) in TMEM (128 threads arrived)
    uint64_t* o_done = p_full + 8;           // [1] every MMA retired
    uint64_t* q_ready = o_done + 1;          // [1] Q tiles staged (256 threads arrived)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);
    __shared__ int sh_range[2];

    pdl_launch();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int group = a.H / a.Hkv, split = blockIdx.z;
    int g = blockIdx.y, Tq = a.Tq, Tk = a.Tk, kv_ready = a.kv_ready;
    const __nv_bfloat16* qp = a.q;
    const int32_t* lop = a.lo;
    const int32_t* hip = a.hi;
    __nv_bfloat16* outp = a.out;
    const CUtensorMap* mK = &tmK;
    const CUtensorMap* mV = &tmV;
    if (a.n_req > 0) {  // batched: this CTA's request (the table was uploaded before the forward began)
        const int req = blockIdx.y / a.Hkv;
        g = blockIdx.y - req * a.Hkv;
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
    const int rr0 = blockIdx.x * RG;                       // first row of this row group
    const int rows_here = min(RG, rows_total - rr0);
    if (rows_here <= 0) return;                            // batched grid sized for the longest request
    const bool hasB = rows_here > BR;

    const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
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
        for (int x = 0; x < 2; ++x) {
            mbar_init(&s_full[x], 1);
            for (int c = 0; c < 4; ++c) mbar_init(&p_full[x * 4 + c], BR);
        }
        mbar_init(o_done, 1);
        mbar_init(q_ready, SM_THREADS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        // key range of the row group = union of its tokens' [lo, hi] (lo/hi were uploaded before the forward)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mK)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mV)) : "memory");
        }
        const int t0 = rr0 / group, t1 = (rr0 + rows_here - 1) / group;
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
    if (warp == 9) {
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
    const int chunk = span > 0 ? ((span + a.splits - 1) / a.splits + BK - 1) / BK * BK : 0;
    const int ks = blo + split * chunk;
    const int ke = min(bhi, ks + chunk - 1);
    const int n = (span > 0 && ke >= ks) ? (ke - ks + BK) / BK : 0;

    if (warp == 8) {
        if (lane != 0) {
            // HBM is mostly idle during attention at query-prefill sizes: lanes 1-31 warm L2 with this CTA's
            // share of the next projections' weights (bulk prefetch, no completion tracking)
            const int ncta = gridDim.x * gridDim.y * gridDim.z;
            for (int rg2 = 0; rg2 < 2; ++rg2) {
                const size_t total = a.pf.bytes[rg2] & ~size_t(15);
                if (!a.pf.ptr[rg2] || total == 0) continue;
                const size_t share = ((total + ncta - 1) / ncta + 15) & ~size_t(15);
                const size_t b0 = (size_t)cta_lin * share, b1 = min(b0 + share, total);
                for (size_t off = b0 + (size_t)(lane - 1) * 65536; off < b1; off += (size_t)31 * 65536)
                    prefetch_l2(static_cast<const uint8_t*>(a.pf.ptr[rg2]) + off, (uint32_t)min((size_t)65536, b1 - off));
            }
        }
        if (lane == 0) {  // ---------------- TMA producer ----------------
            bool waited = false;
            for (int j = 0; j < n; ++j) {
                const int key = ks + j * BK;
                if (!waited && key + BK > kv_ready) {  // rows written by the previous kernels of this forward
                    pdl_wait();
                    waited = true;
                }
                const int sk = j % KST, sv = j % VST;
                mbar_wait(&k_empty[sk], ((uint32_t)(j / KST) & 1u) ^ 1u);
                mbar_expect_tx(&k_full[sk], TILE);
                const uint32_t kd = sbase + OFF_K + sk * TILE;
                if (b3) {
                    tma_load_3d(kd, mK, &k_full[sk], g * D, key, 2 * a.layer);
                    tma_load_3d(kd + SUB, mK, &k_full[sk], g * D + 64, key, 2 * a.layer);
                } else {
                    tma_load_2d(kd, mK, &k_full[sk], g * D, key);
                    tma_load_2d(kd + SUB, mK, &k_full[sk], g * D + 64, key);
                }
                trace_pipe(j, 6);
                mbar_wait(&v_empty[sv], ((uint32_t)(j / VST) & 1u) ^ 1u);
                mbar_expect_tx(&v_full[sv], TILE);
                const uint32_t vd = sbase + OFF_V + sv * TILE;
                if (b3) {
                    tma_load_3d(vd, mV, &v_full[sv], g * D, key, 2 * a.layer + 1);
                    tma_load_3d(vd + SUB, mV, &v_full[sv], g * D + 64, key, 2 * a.layer + 1);
                } else {
                    tma_load_2d(vd, mV, &v_full[sv], g * D, key);
                    tma_load_2d(vd + SUB, mV, &v_full[sv], g * D + 64, key);
                }
                trace_pipe(j, 7);
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            auto issue_s = [&](int x, int j) {  // S_x = Q_x . K_j^T
                const uint32_t qb = sbase + OFF_Q + x * TILE, kb = sbase + OFF_K + (j % KST) * TILE;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * SUB + (kk & 3) * 32;
                    umma(tmem + x * 256, desc_k(qb + off), desc_k(kb + off), IDESC_S, kk > 0);
                }
                umma_commit(&s_full[x]);
            };
            // O_x += P_x . V_j, P from TMEM (8 cols = 16 keys per MMA), chunk by chunk as the softmax stores it
            auto issue_pv = [&](int x, int j) {
                const uint32_t vb = sbase + OFF_V + (j % VST) * TILE;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    mbar_wait(&p_full[x * 4 + c], (uint32_t)j & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        const int kk = 2 * c + k2;
                        umma_ts(tmem + x * 256 + 128, tmem + x * 256 + kk * 8, desc_mn(vb + kk * 2048), IDESC_PV,
                                (j > 0 || kk > 0) ? 1u : 0u);
                    }
                }
            };
            mbar_wait(q_ready, 0);
            tc_fence_after();
            trace_pipe(0, 8);
            if (n > 0) {
                mbar_wait(&k_full[0], 0);
                tc_fence_after();
                issue_s(0, 0);
                if (hasB) issue_s(1, 0);
                umma_commit(&k_empty[0]);
            }
            for (int j = 0; j < n; ++j) {
                const bool more = j + 1 < n;
                const int sk1 = (j + 1) % KST;
                mbar_wait(&v_full[j % VST], (uint32_t)(j / VST) & 1u);
                trace_mma(j, 4);
                tc_fence_after();
                issue_pv(0, j);
                trace_pipe(j, 4);
                trace_mma(j, 5);
                if (more) {
                    mbar_wait(&k_full[sk1], (uint32_t)((j + 1) / KST) & 1u);
                    trace_mma(j, 6);
                    tc_fence_after();
                    issue_s(0, j + 1);
                    trace_mma(j, 7);
                }
                if (hasB) {
                    trace_mma(j, 8);
                    issue_pv(1, j);
                    trace_pipe(j, 5);
                }
                umma_commit(&v_empty[j % VST]);
                if (more) {
                    if (hasB) issue_s(1, j + 1);
                    umma_commit(&k_empty[sk1]);
                }
            }
            umma_commit(o_done);
        }
    } else {
        // ---------------- softmax: warps 0-3 tile A, 4-7 tile B; one thread per row ----------------
        const int x = warp >> 2;
        const int r = (warp & 3) * 32 + lane;  // TMEM lane = tile row
        const int rr = rr0 + x * BR + r;
        const bool active = rr < rows_total;
        const int t = active ? rr / group : 0;
        const int h = g * group + (active ? rr % group : 0);
        const int my_lo = active ? lop[t] : INT32_MAX;
        const int my_hi = active ? min(hip[t], Tk - 1) : -1;
        pdl_wait();  // q is produced by the previous kernel
        if (tid == 0) trace(30, 3);
        {
            // Coalesced staging: warp w of this tile loads its 32 rows two at a time (16 lanes x 16 B per row),
            // all 16 loads in flight before the swizzled stores.
            const uint32_t qb = sbase + OFF_Q + x * TILE;
            const int c = lane & 15;
            uint4 v[16];
            // row qr = token * group + head-in-group, walked two rows at a time without per-row division
            int qr = rr0 + x * BR + (warp & 3) * 32 + (lane >> 4);
            int qt = qr / group, qi = qr - qt * group;
            const uint4* qbase = reinterpret_cast<const uint4*>(qp) + c + (int64_t)g * group * (D / 8);
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                v[it] = qr < rows_total ? qbase[((int64_t)qt * a.H + qi) * (D / 8)] : make_uint4(0, 0, 0, 0);
                qr += 2;
                qi += 2;
                while (qi >= group) {
                    qi -= group;
                    ++qt;
                }
            }
            if (tid == 0 && a.trace) trace_at(a.trace, 30, 4 + (v[0].x == 0x7fc00001u && v[15].w == 1u ? 5 : 0));
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                const int row = (warp & 3) * 32 + it * 2 + (lane >> 4);
                sts128(qb + (c >> 3) * SUB + swz(row, c & 7), v[it]);
            }
            fence_async_smem();
            if (tid == 0) trace(30, 5);
            mbar_arrive(q_ready);
        }
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + lane_base + x * 256, tO = tS + 128;
        const float sl2 = a.scale * LOG2E;
        float m_used = -INFINITY, l = 0.f;
        const int nx = (x == 1 && !hasB) ? 0 : n;
        for (int j = 0; j < nx; ++j) {
            mbar_wait(&s_full[x], (uint32_t)j & 1u);
            tc_fence_after();
            if (tid == 0) trace(j, 0);
            if (tid == 128) trace(j, 2);
            uint32_t s[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s + c * 32);
            tmem_wait_ld();
            trace_sm(j, 4);
            const int key0 = ks + j * BK;
            if (!(key0 >= my_lo && key0 + BK - 1 <= my_hi)) {  // partially visible tile: masked -> -inf
                const int clo = my_lo - key0, chi = my_hi - key0;
#pragma unroll
                for (int i = 0; i < 128; ++i)
                    if (i < clo || i > chi) s[i] = __float_as_uint(-INFINITY);
            }
            float m0 = __uint_as_float(s[0]), m1 = __uint_as_float(s[1]), m2 = __uint_as_float(s[2]),
                  m3 = __uint_as_float(s[3]);
#pragma unroll
            for (int i = 4; i < 124; i += 8) {
                m0 = max3(m0, __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
                m1 = max3(m1, __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
                m2 = max3(m2, __uint_as_float(s[i + 4]), __uint_as_float(s[i + 5]));
                m3 = max3(m3, __uint_as_float(s[i + 6]), __uint_as_float(s[i + 7]));
            }
            m0 = max3(m0, __uint_as_float(s[124]), __uint_as_float(s[125]));
            m1 = max3(m1, __uint_as_float(s[126]), __uint_as_float(s[127]));
            const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
            trace_sm(j, 5);
            const float mxs = mx == -INFINITY ? -INFINITY : mx * sl2;
            // lazy rescale. tcgen05.ld/st are warp-collective (.sync.aligned): the whole warp takes the branch
            // when any of its rows needs it; rows that do not get alpha = 1.
            bool grow = false;
            if (m_used == -INFINITY)
                m_used = mxs;  // first visible keys: O is still all zeros, nothing to rescale
            else
                grow = mxs > m_used + RESCALE_LOG2;
            if (__any_sync(0xffffffffu, grow)) {
                // O_x is current through PV_x(j-1): it retired before S_x(j) (in-order tensor pipe)
                const float alpha = grow ? ex2(m_used - mxs) : 1.0f;
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t w[32];
                    tmem_ld32(tO + c * 32, w);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(__uint_as_float(w[i]) * alpha);
                    tmem_st32(tO + c * 32, w);
                }
                tmem_wait_st();
                if (grow) {
                    l *= alpha;
                    m_used = mxs;
                }
            }
            const float moff = m_used == -INFINITY ? 0.f : m_used;  // nothing visible yet -> all p = 0
            const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(-moff, -moff);
            uint64_t accv = 0;  // (+0, +0)
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // 32 keys per chunk -> 16 P columns (bf16 pairs), stored as soon as done
                // every pair's exponent first (independent MUFU / FMA-pipe work), then conversions and a
                // log-depth sum: no serial accumulation chain behind the MUFU latency
                uint64_t pv[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int e = c * 32 + 2 * i;
                    const uint64_t xv = fma2(pk2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sc2, nm2);
                    if (i < kPolyPairs) {
                        pv[i] = ex2_poly2(xv);
                    } else {
                        float x0, x1;
                        up2(xv, x0, x1);
                        pv[i] = pk2(ex2(x0), ex2(x1));
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float p0, p1;
                    up2(pv[i], p0, p1);
                    pk[i] = bf16x2_bits(p0, p1);
                }
                tmem_st16(tS + c * 16, pk);
#pragma unroll
                for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                    for (int i = 0; i < w; ++i) pv[i] = add2(pv[i], pv[i + w]);
                accv = add2(accv, pv[0]);
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&p_full[x * 4 + c]);  // the PV MMA on these 32 keys may start
                if (c == 1) trace_sm(j, 6);
                if (c == 3) trace_sm(j, 7);
            }
            float a0, a1;
            up2(accv, a0, a1);
            l += a0 + a1;
            trace_sm(j, 8);
            if (tid == 0) trace(j, 1);
            if (tid == 128) trace(j, 3);
        }
        if (nx > 0) {
            mbar_wait(o_done, 0);
            tc_fence_after();
        }
        if (tid == 0) trace(31, 0);
        // ---- epilogue: O/l as bf16, staged row-per-thread into the (now idle) Q_x tile with the SW128 chunk
        // swizzle (conflict-free), then copied out coalesced: 16 lanes x 16 B per 256-byte row ----
        const bool degenerate = active && l == 0.f;
        const float inv = l > 0.f ? 1.0f / l : 0.f;
        const uint32_t stage = sbase + OFF_Q + x * TILE;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t w[32];
            if (nx > 0) {
                tmem_ld32(tO + c * 32, w);  // warp-collective
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int chunk = c * 4 + k;  // 16-byte chunk (8 columns) of the 256-byte row
                sts128(stage + (chunk >> 3) * SUB + swz(r, chunk & 7),
                       make_uint4(bf16x2_bits(__uint_as_float(w[8 * k + 0]) * inv, __uint_as_float(w[8 * k + 1]) * inv),
                                  bf16x2_bits(__uint_as_float(w[8 * k + 2]) * inv, __uint_as_float(w[8 * k + 3]) * inv),
                                  bf16x2_bits(__uint_as_float(w[8 * k + 4]) * inv, __uint_as_float(w[8 * k + 5]) * inv),
                                  bf16x2_bits(__uint_as_float(w[8 * k + 6]) * inv, __uint_as_float(w[8 * k + 7]) * inv)));
            }
        }
        if (tid == 0) trace(31, 4);
        named_bar(2 + x, BR);  // this tile's 128 rows are staged
        if (tid == 0) trace(31, 5);
        const int gid = blockIdx.y * gridDim.x + blockIdx.x;
        const int ngroups = gridDim.x * gridDim.y;
        // workspace of split s, row group gid: rows [256][D] bf16 (contiguous) and (m, l) [256]
        const int64_t wrow0 = ((int64_t)split * ngroups + gid) * RG;
        {
            const int cc = lane & 15;
#pragma unroll 4
            for (int it = 0; it < 16; ++it) {
                const int row = (warp & 3) * 32 + it * 2 + (lane >> 4);
                const int qr = rr0 + x * BR + row;
                uint4 v;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(stage + (cc >> 3) * SUB + swz(row, cc & 7)));
                if (a.splits == 1) {
                    if (qr < rows_total)
                        reinterpret_cast<uint4*>(outp + ((int64_t)(qr / group) * a.H + g * group + qr % group) * D)[cc] = v;
                } else {
                    reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.ws_o) + (wrow0 + x * BR + row) * D)[cc] = v;
                }
            }
        }
        if (tid == 0) trace(31, 6);
        if (a.splits == 1) {
            if (degenerate) atomicOr(a.err, 8);  // DegenerateRowError (numerics.cpp:39-42)
        } else {
            reinterpret_cast<float2*>(a.ws_ml)[wrow0 + x * BR + r] = make_float2(active ? m_used : -INFINITY, l);
            if (tid == 0) trace(31, 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0 && a.trace && cta_lin < TRACE_CTAS) a.trace[TRACE_CTA0 + 2 * cta_lin + 1] = globaltimer_ns();
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// Split merge (PDL-launched right behind the attention grid): one warp per row of a row group, lane = 4
// columns; all `splits` partial loads are issued before use. out = sum_s w_s (O_s / l_s) / sum_s w_s,
// w_s = 2^(m_s - M) * l_s (numerics.cpp:31-60 softmax, regrouped over key splits).
__global__ void __launch_bounds__(256) attn_tc_combine_kernel(const __nv_bfloat16* __restrict__ ws_o,
                                                              const float2* __restrict__ ws_ml,
                                                              __nv_bfloat16* __restrict__ out, int* err, int Tq, int H,
                                                              int Hkv, int splits, int groups_x) {
    pdl_launch();
    const int lane = threadIdx.x & 31;
    const int grow = blockIdx.x * 8 + (threadIdx.x >> 5);  // row over all row groups: gid * RG + i
    const int gid = grow / RG, i = grow % RG;
    const int g = gid / groups_x, rr = (gid % groups_x) * RG + i;  // kv head, row within the kv head
    const int group = H / Hkv;
    const bool ok = rr < Tq * group;
    const int64_t plane = (int64_t)groups_x * Hkv * RG;
    pdl_wait();
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
}

// Split merge of the BATCHED launch: row groups are (request, kv head, group) with gid = (req * Hkv + g) * groups_x
// + x; each request's rows / output rows come from its AttnReq (tok0, n).
__global__ void __launch_bounds__(256) attn_tc_combine_batch_kernel(const __nv_bfloat16* __restrict__ ws_o,
                                                                    const float2* __restrict__ ws_ml,
                                                                    __nv_bfloat16* __restrict__ out, int* err,
                                                                    const AttnReq* __restrict__ reqs, int H, int Hkv,
                                                                    int splits, int groups_x, int ngroups) {
    pdl_launch();
    const int lane = threadIdx.x & 31;
    const int grow = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int gid = grow / RG, i = grow % RG;
    const int y = gid / groups_x, req = y / Hkv, g = y - req * Hkv;
    const int rr = (gid % groups_x) * RG + i;
    const int group = H / Hkv;
    pdl_wait();
    const AttnReq R = reqs[req];
    if (rr >= R.n * group) return;  // warp-uniform
    const int64_t plane = (int64_t)ngroups * RG;
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
    const int64_t mo = (int64_t)(R.tok0 + rr / group) * H + g * group + rr % group;
    reinterpret_cast<uint2*>(out + mo * D)[lane] =
        make_uint2(bf16x2_bits(acc[0] * inv, acc[1] * inv), bf16x2_bits(acc[2] * inv, acc[3] * inv));
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
    launch_k(attn_tc_kernel, dim3(groups_x, Hkv * n_req, a.splits), THREADS, SMEM_BYTES, s, unused, unused, a);
    TKV_CUDA(cudaGetLastError());
    if (a.splits > 1) {
        const int ngroups = groups_x * Hkv * n_req;
        launch_k(attn_tc_combine_batch_kernel, dim3((ngroups * RG + 7) / 8), dim3(256), 0, s,
                 reinterpret_cast<const __nv_bfloat16*>(ws.o), reinterpret_cast<const float2*>(ws.ml),
                 (__nv_bfloat16*)out, err, reqs, H, Hkv, a.splits, groups_x, ngroups);
        TKV_CUDA(cudaGetLastError());
    }
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
    if (groups * 2 > num_sms) return 1;  // already >= half a wave of row groups: no split-K
    int s = num_sms / groups;            // one wave (1 CTA / SM)
    const int max_by_keys = ((Tk + BK - 1) / BK + 1) / 2;  // >= 2 key tiles per split
    if (s > max_by_keys) s = max_by_keys;
    if (s > 32) s = 32;
    return s < 1 ? 1 : s;
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
    launch_k(attn_tc_kernel, grid, THREADS, SMEM_BYTES, s, tk, tv, a);
    TKV_CUDA(cudaGetLastError());
    if (splits > 1) {
        const int rows = (int)(grid.x * grid.y) * RG;
        launch_k(attn_tc_combine_kernel, dim3(rows / 8), dim3(256), 0, s, (const __nv_bfloat16*)ws.o,
                 (const float2*)ws.ml, (__nv_bfloat16*)out, err, Tq, H, Hkv, splits, (int)grid.x);
        TKV_CUDA(cudaGetLastError());
    }
}

}  // namespace tkv

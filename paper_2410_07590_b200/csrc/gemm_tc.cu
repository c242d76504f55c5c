// tcgen05 + TMA bf16 GEMM for sm_100a with split-K fp32 partial output:
//   partial[z][m][n] = sum_{k in split z} A[m][k] * W[n][k]
// A = activations [M][lda] (K-major), W = weights [N][K] (K-major, the engine stores every projection
// transposed so both operands are K-major). Replaces the reference's f64 matmul (src/numerics.cpp:8-29)
// for the QKV / O / gate-up / down projections of forward_tokens (src/model.cpp:240-264).
//
// Structure (one 128x128 output tile per CTA, 4 warps):
//   warp 0 / lane 0 : TMA producer — STAGES-deep ring of {A 128x64, W 128x64} bf16 tiles, SWIZZLE_128B,
//                     mbarrier full/empty handshake
//   warp 1 / lane 0 : MMA issuer — tcgen05.mma.cta_group::1.kind::f16 (M=128, N=128, K=16) x 4 per
//                     stage, accumulator in TMEM (128 lanes x 128 fp32 columns); tcgen05.commit frees
//                     the smem slot and finally signals the epilogue
//   warps 0-3       : epilogue — tcgen05.ld 32x32b (each warp owns 32 TMEM lanes = 32 rows), fp32 store
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 6, THREADS = 128;
constexpr uint32_t TILE_A = BM * BK * 2, TILE_B = BN * BK * 2, STAGE_BYTES = TILE_A + TILE_B;
constexpr uint32_t TMEM_COLS = BN;  // fp32 accumulator columns
constexpr size_t SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row swizzle atoms 1024 B apart.
//   [0,14) start>>4, [16,30) LBO>>4 (unused for swizzled K-major; 1), [32,46) SBO>>4 = 1024>>4,
//   [46,48) version = 1 (sm_100), [61,64) layout = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor kind::f16: D=f32 (bit 4), A=B=bf16 (bits 7,10), K-major A/B, N>>3 at 17, M>>4 at 24.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, int M, int N,
                   int K, float* __restrict__ partial, int kb_per_split) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* tiles = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, z = blockIdx.z;
    const int kb_total = (K + BK - 1) / BK;
    const int kb0 = z * kb_per_split;
    const int nkb = min(kb_total, kb0 + kb_per_split) - kb0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (nkb > 0) {
        if (warp == 0 && lane == 0) {
            // TMA producer
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* a = tiles + s * STAGE_BYTES;
                uint8_t* b = a + TILE_A;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                const int kc = (kb0 + i) * BK;
                tma_load_2d(a, &tmA, &full[s], kc, m0);
                tma_load_2d(b, &tmW, &full[s], kc, n0);
            }
        } else if (warp == 1 && lane == 0) {
            // MMA issuer
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a = smem_u32(tiles + s * STAGE_BYTES);
                const uint32_t b = a + TILE_A;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // advance 16 bf16 = 32 B along K inside the 128 B swizzle row
                    umma_f16(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), (i | k) != 0);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(done);
        }
        __syncwarp();
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    // Epilogue: warp w owns TMEM lanes [32w, 32w+32) = tile rows.
    const int row = m0 + warp * 32 + lane;
    float* out = partial + (int64_t)z * M * N + (int64_t)row * N;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        if (nkb > 0) {
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = 0u;
        }
        if (row < M) {
            const int n = n0 + c;
            if (n + 16 <= N && (N % 4) == 0) {
                float4* o4 = reinterpret_cast<float4*>(out + n);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    o4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                        __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (n + j < N) out[n + j] = __uint_as_float(r[j]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
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
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_map(const void* base, int rows, int cols_k, int ld_elems) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols_k, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
    const cuuint32_t box[2] = {BK, 128};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TKV_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

bool gemm_tc_supported(int M, int N, int K, int lda) {
    // TMA: 16-byte aligned row strides; K >= 8 elements.
    return M >= 1 && N >= 1 && K >= 8 && (lda * 2) % 16 == 0 && (K * 2) % 16 == 0;
}

void launch_gemm_tc(const void* A, int lda, const void* W, int M, int N, int K, float* partial, int splits,
                    cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        TKV_CUDA(cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
        attr_set = true;
    }
    const CUtensorMap ta = make_map(A, M, K, lda);
    const CUtensorMap tw = make_map(W, N, K, K);
    const int kb_total = (K + BK - 1) / BK;
    const int kbs = (kb_total + splits - 1) / splits;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, splits);
    gemm_tc_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(ta, tw, M, N, K, partial, kbs);
    TKV_CUDA(cudaGetLastError());
}

}  // namespace tkv

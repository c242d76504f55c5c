// Retrieval on the GPU: exhaustive cosine top-k over the chunk-embedding index, replacing
// RetrievalIndex::top_k (src/retrieval.cpp:117-133) and cosine (src/retrieval.cpp:90-100).
//
// The index lives in HBM transposed, emb[d][cap] (f64), so a warp's 32 rows are one coalesced 256-byte read per
// dimension. Scores are computed in f64 with the reference's operation order (dot += q_i * e_i, separate
// multiply and add, i ascending; cosine = dot / sqrt(na * nb) with na, nb accumulated the same way on the host),
// so the ranking — including ties, broken by ascending chunk id — is the reference's bit for bit.
//   pass 1: a CTA scores 1024 rows, bitonic-sorts (score desc, id asc) in shared memory, keeps the first k
//   pass 2+: the same block sort over the candidates until one block of <= 1024 remains
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"
#include "tkv_internal.h"

namespace tkv {
namespace {

constexpr int BLK = 1024, THREADS = 256;

struct Cand {
    double score;
    uint64_t id;
};

__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {  // ranking order of top_k
    return a.score > b.score || (a.score == b.score && a.id < b.id);
}

// bitonic sort of BLK candidates in shared memory (ranking order)
__device__ void block_sort(Cand* c) {
    for (int size = 2; size <= BLK; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < BLK / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;  // this pair's subsequence sorts in ranking order
                Cand a = c[lo], b = c[hi];
                if (up ? before(b, a) : before(a, b)) {
                    c[lo] = b;
                    c[hi] = a;
                }
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(THREADS) score_topk_kernel(const double* __restrict__ emb,
                                                             const double* __restrict__ nb,
                                                             const uint64_t* __restrict__ ids, int64_t n, int64_t cap,
                                                             const double* __restrict__ q, double na, int k,
                                                             Cand* __restrict__ out) {
    pdl_launch();
    pdl_wait();
    __shared__ double qs[kIndexDim];
    __shared__ Cand c[BLK];
    for (int i = threadIdx.x; i < kIndexDim; i += blockDim.x) qs[i] = q[i];
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * BLK;
    for (int j = threadIdx.x; j < BLK; j += blockDim.x) {
        const int64_t r = r0 + j;
        Cand v{-INFINITY, ~0ull};
        if (r < n) {
            double dot = 0.0;
            for (int i = 0; i < kIndexDim; ++i) dot = __dadd_rn(dot, __dmul_rn(qs[i], emb[(int64_t)i * cap + r]));
            v.score = __ddiv_rn(dot, __dsqrt_rn(__dmul_rn(na, nb[r])));
            v.id = ids[r];
        }
        c[j] = v;
    }
    block_sort(c);
    for (int j = threadIdx.x; j < k; j += blockDim.x) out[(int64_t)blockIdx.x * k + j] = c[j];
}

__global__ void __launch_bounds__(THREADS) merge_topk_kernel(const Cand* __restrict__ in, int64_t n, int k,
                                                             Cand* __restrict__ out) {
    pdl_launch();
    pdl_wait();
    __shared__ Cand c[BLK];
    const int64_t r0 = (int64_t)blockIdx.x * BLK;
    for (int j = threadIdx.x; j < BLK; j += blockDim.x) c[j] = r0 + j < n ? in[r0 + j] : Cand{-INFINITY, ~0ull};
    block_sort(c);
    for (int j = threadIdx.x; j < k; j += blockDim.x) out[(int64_t)blockIdx.x * k + j] = c[j];
}

}  // namespace

size_t index_topk_scratch_bytes(int64_t n, int k) {
    const int64_t blocks = (n + BLK - 1) / BLK;
    return (size_t)2 * blocks * k * sizeof(Cand);
}

int64_t launch_index_top_k(const double* emb, const double* nb, const uint64_t* ids, int64_t n, int64_t cap,
                           const double* q, double na, int k, void* scratch, uint64_t* ids_out, double* scores_out,
                           cudaStream_t s) {
    if (k < 1 || k > kIndexMaxK) fail(TKV_ERR_CONFIG, "index top_k: k must be in [1, 256]");
    int64_t blocks = (n + BLK - 1) / BLK;
    Cand* a = static_cast<Cand*>(scratch);
    Cand* b = a + blocks * k;
    launch_k(score_topk_kernel, dim3((unsigned)blocks), dim3(THREADS), 0, s, emb, nb, ids, n, cap, q, na, k, a);
    TKV_CUDA(cudaGetLastError());
    int64_t count = blocks * k;  // candidates in ranking order per block
    while (count > BLK) {
        const int64_t nb2 = (count + BLK - 1) / BLK;
        launch_k(merge_topk_kernel, dim3((unsigned)nb2), dim3(THREADS), 0, s, (const Cand*)a, count, k, b);
        TKV_CUDA(cudaGetLastError());
        count = nb2 * k;
        Cand* t = a;
        a = b;
        b = t;
    }
    launch_k(merge_topk_kernel, dim3(1), dim3(THREADS), 0, s, (const Cand*)a, count, k, b);
    TKV_CUDA(cudaGetLastError());
    const int64_t take = k < n ? k : n;
    Cand host[kIndexMaxK];
    TKV_CUDA(cudaMemcpyAsync(host, b, (size_t)take * sizeof(Cand), cudaMemcpyDeviceToHost, s));
    TKV_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < take; ++i) {
        ids_out[i] = host[i].id;
        if (scores_out) scores_out[i] = host[i].score;
    }
    return take;
}

}  // namespace tkv

// Internal declarations shared by the host engine (engine.cpp) and the sm_100a kernels.
// Nothing here is part of the C ABI (include/tkv.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/tkv.h"

namespace tkv {

// Status carrier for the host side; the C ABI converts it to tkv_status + message.
struct Failure {
    tkv_status code;
    std::string msg;
};
[[noreturn]] void fail(tkv_status code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define TKV_CUDA(x) ::tkv::cuda_check((x), #x)

enum class DT : int { F32 = 0, BF16 = 1 };

// Programmatic Dependent Launch on/off for every kernel launch (process-wide; TKV_FLAG_NO_PDL disables).
bool pdl_enabled();
void set_pdl_enabled(bool on);
inline size_t dt_size(DT t) { return t == DT::F32 ? 4 : 2; }

// ---------------------------------------------------------------------------------------------
// Kernel launchers (kernels.cu, gemm_simt.cu, gemm_tc.cu, attn_simt.cu, gather.cu).
// All are asynchronous on `s`.
// ---------------------------------------------------------------------------------------------

// Weight init: dst[j*rows + i] = cast(next_signed(seed, base + i*cols + j) * scale) — the reference's
// [rows=in, cols=out] draw order (src/model.cpp:15-21,68-92) written transposed (K-major [out][in]).
// row_block > 0 places output row j at (j / row_block) * 2 * row_block + row_off + j % row_block (the
// interleaved gate/up layout of the fused SwiGLU epilogue).
void launch_init_transposed(void* dst, DT dt, uint64_t seed, uint64_t base, int64_t rows, int64_t cols,
                            double scale, cudaStream_t s, int row_block = 0, int row_off = 0);
// Same, not transposed (embedding [vocab][hidden], fp32).
void launch_init_rowmajor_f32(float* dst, uint64_t seed, uint64_t base, int64_t rows, int64_t cols,
                              double scale, cudaStream_t s);
void launch_fill_f32(float* dst, float v, int64_t n, cudaStream_t s);

// RMSNorm folding (see dev_common.cuh:row_scale): x rows are produced together with xb = dtype(x * w) and
// ssp[t][b] = sum of x^2 over the b-th 128-column block of row t; nb = norm_blocks(hidden).
// ssp holds one partial sum per 128-column block (the GEMM n-tile width, so a fused GEMM epilogue can
// produce it per tile); embed/residual kernels cover 1024 columns per CTA (8 blocks, one per warp).
__host__ __device__ inline int norm_blocks(int hidden) { return (hidden + 127) / 128; }
inline int row_ctas(int hidden) { return (hidden + 1023) / 1024; }
// x[t] = emb[tok[t]] (fp32), xb, ssp. Errors (token outside vocab) set *err.
void launch_embed(const int32_t* tok, int T, const float* emb, int hidden, int vocab, const float* w, float* x,
                  void* xb, float* ssp, DT dt, int* err, cudaStream_t s);
// x[t] += sum_s partial[s][t][:] (the residual add), then xb, ssp as above. Grid = nb x T CTAs.
void launch_residual(float* x, const float* partial, int splits, int T, int hidden, const float* w, void* xb,
                     float* ssp, DT dt, int* err, cudaStream_t s);
// act[t][i] = silu(s_t * sum_s P[s][t][gate(i)]) * (s_t * sum_s P[s][t][up(i)]), s_t = row_scale(ssp, t)
// (dtype). gu_block B > 0: gate/up columns in B-wide blocks (gate(i) = (i/B)*2B + i%B, up = gate + B).
void launch_swiglu(const float* partial, int splits, int T, int inter, void* act, const float* ssp, int nb,
                   int hidden, float eps, DT dt, cudaStream_t s, int gu_block = 0);

// QKV epilogue: reduce the split-K partials of [T, (H+2Hkv)*d], rotate q and k by pos[t]
// (interleaved pairs, cos/sin table [max_pos][d/2] of float2), write q (dtype [T, H*d]),
// rotated K and V into the request cache rows [row0, row0+T) of layer tensors kc/vc
// ([cap, kv_dim] dtype), and — when st_page != nullptr — the unrotated K and V into store pages:
// page p, slot s of layer tensor = store + ((p*L + layer)*2 + kv)*page_tokens*kv_dim.
struct StoreScatter {
    void* pool = nullptr;
    const int32_t* page = nullptr;  // [T]
    const int32_t* slot = nullptr;  // [T]
    int page_tokens = 0;
    int layer_num = 0;
    void* host_pool = nullptr;      // pinned host spill tier (device-mapped): page >= host_base -> host page
    int32_t host_base = INT32_MAX;  //   (page - host_base)
};
// Batched QKV epilogue: request r owns forward tokens [tok0, tok0 + n); their K/V rows go to ITS cache (kv, cap:
// [L][K|V][cap][kv_dim]) at rows [row0, row0 + n). One launch covers every request of a batched forward.
struct EpiReq {
    void* kv;
    int64_t cap;
    int tok0, n, row0, pad;
};
// The projections were computed from xb: every output is first multiplied by row_scale(ssp, t).
void launch_qkv_epilogue(const float* partial, int splits, int T, int H, int Hkv, int d, const int32_t* pos,
                         const float2* rope, void* q, void* kc, void* vc, int row0, const StoreScatter& sc,
                         int layer, const float* ssp, int nb, int hidden, float eps, DT dt, cudaStream_t s,
                         int64_t plane = 0, const EpiReq* reqs = nullptr, int n_req = 0);  // split-plane stride in floats (0 = T * N; batched forwards pass
                                              // the whole batch's plane and a row-offset partial pointer)

// KV gather + fused RoPE: one descriptor per (chunk page -> request rows) segment.
struct GatherSeg {
    int32_t src_page;  // page index in the store pool
    int32_t n_tok;     // tokens in this segment (<= page_tokens)
    int32_t dst_row;   // first request-cache row
    int32_t pos0;      // position id of the first token (positions are consecutive inside a segment)
    int32_t pool;      // which page pool: 0 = this GPU's store, 1.. = a peer GPU's store (NVLink P2P reads)
};
// Page pools the gather kernel may read: slot 0 is local HBM, other slots are peer GPUs' pools mapped
// into this process (cudaIpcOpenMemHandle, or peer access inside one process).
constexpr int kMaxPools = 16;
constexpr int kHostPool = kMaxPools - 1;  // slot of the pinned host spill tier (peers use 1 .. kHostPool - 1)
struct PoolTable {
    const void* p[kMaxPools] = {};
};
// cache layout [L][2][cap][kv_dim]; rotate=0 copies keys unrotated (bit-exact export).
void launch_gather_rope(const PoolTable& pools, int page_tokens, const GatherSeg* segs, int n_segs, int L,
                        int kv_dim, int d, const float2* rope, void* cache, int64_t cap, int rotate, DT dt,
                        int num_sms, cudaStream_t s);

// logits[v] = row_scale(ssp, 0) * sum_k xb[k] * W[v][k] (final RMSNorm folded), fp32; *err on non-finite.
void launch_lm_head(const void* xb, const void* W, int hidden, int vocab, float* logits, const float* ssp, int nb,
                    float eps, DT dt, int* err, cudaStream_t s);
// dense 0/1 view of the [lo, hi] predicate (the same __device__ predicate the attention uses)
void launch_mask_materialize(const int32_t* lo, const int32_t* hi, int rows, int cols, uint8_t* out,
                             cudaStream_t s);
// rot[i] = inverse-rotate(cache K rows) for export; fp32 out
void launch_unrotate_rows(const void* k, int rows, int kv_dim, int d, const int32_t* pos, const float2* rope,
                          float* out, DT dt, cudaStream_t s);
void launch_to_f32(const void* src, int64_t n, float* dst, DT dt, cudaStream_t s);
void launch_from_f32(const float* src, int64_t n, void* dst, DT dt, cudaStream_t s);
// sum split-K partials [splits][n] -> out[n]
void launch_reduce_splits(const float* partial, int splits, int64_t n, float* out, cudaStream_t s);

// GEMM: partial[z][m][n] = sum_{k in split z} A[m][k] * W[n][k]   (A [M][lda] dtype, W [N][K] dtype).
void launch_gemm_simt(const void* A, int lda, const void* W, int M, int N, int K, float* partial, int splits,
                      DT dt, cudaStream_t s);
// tcgen05 + TMA version (bf16 only). Returns false when the shape is not supported (caller errors out).
// M <= 128 uses the swapped tiling (weights on the UMMA M side). With swiglu_act != nullptr (splits must
// be 1, W rows interleaved in 64-row gate/up blocks) the epilogue writes act[M][N/2] = silu(g)*u in bf16.
bool gemm_tc_supported(int M, int N, int K, int lda);
void gemm_trace_enable(bool on, unsigned long long* host_out, int64_t cap);
// Kernel timeline (tkv_kernel_timeline): while armed, every launch of an instrumented kernel (GEMM, attention, split
// merge, residual / QKV epilogues, embed, lm_head, KV gather) takes the next slot [2] of globaltimer ns (first CTA past
// griddepcontrol.wait, last warp done), tagged with the engine's current launch class. Process-global; null when off.
unsigned long long* tl_take();
void tl_set_class(int cls);
bool tl_armed();  // debug: CTA 0 per-stage clock64 trace
void set_gemm_nsmp(int mp);
void set_gemm_skip_epi(int v);  // timing experiments only: skip the normal-tiling partial stores
// normal tiling unit order (0 n-fastest, 1 m-fastest when N > M, 2 m-fastest; group_mb > 0: m-tile groups of
// that many MB of activation rows)
void set_gemm_raster(int r, int group_mb = -1);  // normal (> 128-token) tiling: 128-row activation tiles per unit (1 or 2)
void set_gemm_knobs(int stages, int smem_kb, int ctas_per_sm, int w_evict_first, int np = 0, int pf = -1,
                    int krot = -1);
int gemm_tc_tiles(int M, int N);
int gemm_tc_ctas_per_sm(int M);  // resident GEMM CTAs per SM the launcher plans for M tokens
// Returns the number of split-K partial planes actually written (<= splits: every split is non-empty).
// The SwiGLU epilogue applies the folded RMSNorm scale row_scale(ssp, token) (ssp/nb/eps: see launch_residual).
int launch_gemm_tc(const void* A, int lda, const void* W, int M, int N, int K, float* partial, int splits,
                   cudaStream_t s, void* swiglu_act = nullptr, const float* ssp = nullptr, int nb = 0,
                   float eps = 0.f, int gu_block = 64);

// Flash attention, SIMT (fp32 math): q [Tq][H*d], k/v rows [Tk][Hkv*d] (stride kv_stride elements),
// row t attends keys j with lo[t] <= j <= hi[t]. out [Tq][H*d] (dtype). ws: split-K workspace.
struct AttnWork {
    float* o = nullptr;   // [splits][Tq*H][d]
    float* ml = nullptr;  // [splits][Tq*H][2]
    size_t floats = 0;
};
size_t attn_workspace_floats(int Tq, int H, int d, int splits);
int attn_pick_splits(int Tq, int H, int Hkv, int Tk, int num_sms);
void launch_attention_simt(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                           const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int d, int splits,
                           const AttnWork& ws, int* err, DT dt, cudaStream_t s);

// Up to two global regions the attention kernel warms into L2 (bulk prefetch from idle producer lanes).
struct L2Prefetch {
    const void* ptr[2] = {nullptr, nullptr};
    size_t bytes[2] = {0, 0};
};
// tcgen05/TMEM/TMA attention (attn_tc.cu): head_size 128, bf16. Same predicate and workspace layout as
// SIMT; split-K partials (bf16 O/l) are merged by a PDL-launched combine kernel. Key rows
// < kv_ready were written before the current forward began and are loaded before griddepcontrol.wait.
bool attention_tc_supported(int d, DT dt);
constexpr int kAttnTcRows = 128;  // (token, head) rows per CTA = rows per split-workspace row group
// Batched query prefill: one launch covers every request (rows of request r are tokens [tok0, tok0 + n) of the
// forward; its keys are [0, row0 + n) of its own cache, read through a 3-D tensor map over the cache
// [2L][row0 + n][kv_dim] encoded by attn_tc_cache_map). No split-K: the batch supplies the CTAs.
struct AttnReq {
    int tok0, n, row0, pad;
};
void attn_tc_cache_map(const void* cache, int64_t rows, int64_t cap, int kv_dim, int L, void* map128);
void launch_attention_tc_batch(const void* q, const AttnReq* reqs, const void* maps, int n_req, int max_rows, int H,
                               int Hkv, int layer, const int32_t* lo, const int32_t* hi, void* out, int* err,
                               cudaStream_t s, int splits = 1, const AttnWork& ws = AttnWork{});
int attn_tc_batch_pick_splits(int ctas, int min_keys, int num_sms);
void attn_trace_enable(bool on, unsigned long long** device_buf);  // debug timeline of CTA (0,0,0)
int attn_trace_words();  // [32 tiles][16 events] clock64 of CTA (0,0,0), then [1024 CTAs][entry, exit] globaltimer
int attn_tc_row_groups(int Tq, int H, int Hkv);
// workspace of the tcgen05 kernel's split merge (floats); ws.ml = ws.o + *ml_offset
size_t attn_tc_workspace_floats(int Tq, int H, int Hkv, int splits, size_t* ml_offset);
int attn_tc_pick_splits(int Tq, int H, int Hkv, int Tk, int num_sms);
int attn_tc_compact_splits(int rows, int gx, int splits);  // key splits of a compact (<= 64-row) last row tile
void launch_attention_tc(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                         const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int splits, const AttnWork& ws,
                         int* err, cudaStream_t s, int kv_ready, const L2Prefetch& pf = L2Prefetch());
// Retrieval index (retrieval.cu): emb is [kIndexDim][cap] f64 (transposed), nb[r] = sum of squares of row r
// (host, reference order); returns min(k, n) ids / cosines in RetrievalIndex::top_k order (retrieval.cpp:117-133).
constexpr int kIndexDim = 256, kIndexMaxK = 256;  // kEmbedDim (retrieval.hpp:11)
size_t index_topk_scratch_bytes(int64_t n, int k);
int64_t launch_index_top_k(const double* emb, const double* nb, const uint64_t* ids, int64_t n, int64_t cap,
                           const double* q, double na, int k, void* scratch, uint64_t* ids_out, double* scores_out,
                           cudaStream_t s);

// Reference-exact weights_checksum on the device (fingerprint.cu): FNV-1a 64 over a stream of 8-byte words given
// as segments -- kind 0 literal / 1 constant: the word `a` repeated n times; kind 2: the draws
// next_signed(seed, a + i) * scale (init_random, model.cpp:15-21); kind 3: n words already in device memory at
// address a. Returns the hash continued from h0. device_words materialises words [w0, w0 + n) of the list.
struct FpSeg {
    uint64_t word0, n, a;
    double scale;
    int32_t kind, pad;
};
uint64_t device_fnv_words(const std::vector<FpSeg>& segs, uint64_t seed, uint64_t h0, cudaStream_t s);
void device_words(const std::vector<FpSeg>& segs, uint64_t seed, uint64_t w0, int64_t n, uint64_t* d_out, cudaStream_t s);
// TKVW loading: element range [e0, e0 + n) of a row-major f64 [rows][cols] reference tensor, cast f64 -> f32 (RN)
// [-> bf16 (RNE)] and stored like launch_init_transposed (transposed, optional gate/up row interleave), or
// row-major f32 (embedding, norm vectors)
void launch_store_transposed_f64(void* dst, DT dt, const double* src, int64_t e0, int64_t n, int64_t rows, int64_t cols,
                                 cudaStream_t s, int row_block = 0, int row_off = 0);
void launch_store_f32_from_f64(float* dst, const double* src, int64_t n, cudaStream_t s);
// Decode-sized attention (attn_decode.cu): bf16, d = 128, Tq * group in {4, 7, 8, 16} rows per kv head; split-K
// flash decoding on CUDA cores with the SIMT workspace layout, merged by launch_attention_combine.
bool attention_decode_supported(int Tq, int H, int Hkv, int d, DT dt);
int attn_decode_pick_splits(int Tk, int Hkv, int num_sms);
void launch_attention_decode(const void* q, const void* k, const void* v, int kv_stride, const int32_t* lo,
                             const int32_t* hi, void* out, int Tq, int Tk, int H, int Hkv, int splits,
                             const AttnWork& ws, int* err, cudaStream_t s);
// merge split-K (O, m, l) partials into out (dtype)
void launch_attention_combine(const AttnWork& ws, int rows, int d, int splits, void* out, int* err, DT dt,
                              cudaStream_t s);

}  // namespace tkv

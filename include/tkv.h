/*
 * tkv.h — C ABI of the B200-native TurboRAG prefill engine (libtkv_b200.so).
 *
 * This is the drop-in boundary for the reference's prefill path. The
 * reference (`turbokv`, /root/reference/proj) has no FFI layer; its boundary
 * is the C++ API of include/turbokv/pipeline.hpp. Each entry point below
 * names the reference interface it replaces (file:line under proj/).
 * include/turbokv_compat.hpp re-exposes the same surface with the
 * reference's C++ names and exception classes; INTEGRATION.md shows the
 * ctypes / C++ bindings a maintainer adds.
 *
 * Conventions
 *  - Plain C types only: pointers + sizes. No torch types. All buffers are
 *    HOST memory unless a function name ends in _device.
 *  - Every call returns tkv_status. On failure tkv_last_error() returns a
 *    thread-local message. Codes 1-10 map one-to-one onto the reference's
 *    exception classes (include/turbokv/errors.hpp:10-67).
 *  - There is no CPU fallback: with no usable sm_100 device,
 *    tkv_engine_create fails with TKV_ERR_CUDA.
 *  - An engine (and its contexts) is driven from one host thread at a time, like the reference Engine: its
 *    activation buffers, staging ring and captured forward graphs are per engine. Separate engines are independent.
 */
#ifndef TKV_H
#define TKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKV_ABI_VERSION 2

typedef enum {
    TKV_OK = 0,
    TKV_ERR_GENERIC = 1,        /* turbokv::Error               errors.hpp:10  */
    TKV_ERR_SHAPE = 2,          /* turbokv::ShapeError          errors.hpp:17  */
    TKV_ERR_DOMAIN = 3,         /* turbokv::DomainError         errors.hpp:23  */
    TKV_ERR_CONFIG = 4,         /* turbokv::ConfigError         errors.hpp:29  */
    TKV_ERR_DEGENERATE_ROW = 5, /* turbokv::DegenerateRowError  errors.hpp:35  */
    TKV_ERR_IO = 6,             /* turbokv::IoError             errors.hpp:41  */
    TKV_ERR_FORMAT = 7,         /* turbokv::FormatError         errors.hpp:47  */
    TKV_ERR_NOT_FOUND = 8,      /* turbokv::NotFoundError       errors.hpp:53  */
    TKV_ERR_STALE_CACHE = 9,    /* turbokv::StaleCacheError     errors.hpp:59  */
    TKV_ERR_NO_CONTEXT = 10,    /* turbokv::NoContextError      errors.hpp:65  */
    TKV_ERR_CUDA = 11,          /* device / driver failure (no reference analogue) */
    TKV_ERR_OOM = 12            /* HBM or page-pool exhaustion                      */
} tkv_status;

/* ModelConfig (include/turbokv/config.hpp:11-34), same field order. */
typedef struct {
    int64_t layer_num;
    int64_t head_num;
    int64_t kv_head_num;
    int64_t head_size;
    int64_t hidden_size;
    int64_t intermediate_size;
    int64_t vocab_size;
    double rope_base;
    double norm_eps;
} tkv_model_config;

typedef enum { TKV_DTYPE_F32 = 1, TKV_DTYPE_BF16 = 2 } tkv_dtype;
/* PositionMode (pipeline.hpp:21) */
typedef enum { TKV_POS_COMPOSITE = 0, TKV_POS_REORDERED = 1 } tkv_position_mode;
/* MaskMode (attention.hpp:17) */
typedef enum { TKV_MASK_CAUSAL = 0, TKV_MASK_INDEPENDENT = 1 } tkv_mask_mode;
/* which tensor of a layer */
typedef enum { TKV_K = 0, TKV_V = 1 } tkv_kv_which;

/* Engine options (replace Engine(config, seed, store_root, StoreDtype), pipeline.hpp:69-72). */
typedef struct {
    tkv_dtype dtype;              /* compute/storage dtype of weights, activations and KV          */
    int32_t device;               /* CUDA ordinal                                                   */
    int32_t page_tokens;          /* tokens per KV-store page (default 64)                          */
    int64_t store_capacity_tokens;/* HBM store capacity in tokens (0 = 1/4 of free HBM)             */
    int64_t max_position;         /* RoPE table length (0 = 32768; grows on demand)                 */
    int32_t exact_fingerprint;    /* != 0: reference FNV weights checksum (hashed on the GPU, default);  */
                                  /* 0: a fast identity that is NOT the reference's (opt-in)          */
    int32_t flags;                /* TKV_FLAG_*                                                     */
    int64_t host_spill_tokens;    /* pinned, device-mapped host tier for chunks that do not fit the  */
                                  /* HBM store (0 = none); the gather kernel reads it zero-copy      */
} tkv_engine_opts;

#define TKV_FLAG_SIMT_GEMM 0x1    /* bf16: use the SIMT GEMM instead of tcgen05 (debug/compare)  */
#define TKV_FLAG_SIMT_ATTN 0x2    /* bf16: use the SIMT attention instead of tcgen05              */
/* 0x4: reserved */
#define TKV_FLAG_NO_PDL 0x8       /* launch kernels without programmatic dependent launch          */
#define TKV_FLAG_L2_PREFETCH 0x10  /* reserved (the attention-time L2 weight prefetch is on by default) */
#define TKV_FLAG_NO_GRAPHS 0x100   /* launch the query-prefill forward kernel by kernel (no CUDA-graph capture / replay) */
#define TKV_FLAG_BATCH_ATTN 0x20   /* batched prefill: one attention launch even when the batch cannot fill the GPU */
#define TKV_FLAG_LAYER_KERNEL 0x80 /* reserved (the persistent layer-kernel experiment was measured slower and removed) */
#define TKV_FLAG_DECODE_ATTN 0x40 /* bf16: decode-sized (<= 16 rows / kv head) forwards use the split-K mma.sync kernel */

/* IngestStats (pipeline.hpp:35-39) */
typedef struct {
    int64_t chunks;
    int64_t new_chunks;
    uint64_t bytes_written;
} tkv_ingest_stats;

/* FlopCounter (costmodel.hpp:53-63) */
typedef struct {
    uint64_t qkv, attn, o, mlp;
} tkv_flops;

typedef struct tkv_engine tkv_engine;
typedef struct tkv_context tkv_context;

int tkv_abi_version(void);
const char* tkv_last_error(void);
const char* tkv_status_name(tkv_status s);

/* ModelConfig::preset / validate / fingerprint_seed (src/config.cpp:9-72). Names: "toy",
 * "qwen2-7b", plus "llama3-8b" (config 4 of BASELINE.json). */
tkv_status tkv_config_preset(const char* name, tkv_model_config* out);
tkv_status tkv_config_validate(const tkv_model_config* cfg);
uint64_t tkv_config_fingerprint_seed(const tkv_model_config* cfg);

/* weights_checksum / model_fingerprint (src/model.cpp:94-118), computed on the host by
 * streaming the SplitMix64 draws (no f64 weights are materialised). */
tkv_status tkv_weights_identity(const tkv_model_config* cfg, uint64_t seed, uint64_t* checksum,
                                uint64_t* fingerprint);
/* chunk_content_id (src/kvstore.cpp:58-64) */
uint64_t tkv_chunk_content_id(uint64_t model_fingerprint, const int32_t* framed, int64_t n);

void tkv_engine_opts_default(tkv_engine_opts* opts);
/* Engine::Engine (pipeline.hpp:69-72; src/pipeline.cpp:55-68). Weights are generated on the
 * device from (config, seed) with the reference's init_random draw order (src/model.cpp:68-92). */
tkv_status tkv_engine_create(const tkv_model_config* cfg, uint64_t seed, const tkv_engine_opts* opts,
                             tkv_engine** out);
void tkv_engine_destroy(tkv_engine* eng);
/* TKVW weights files (docs/formats.md "TKVW"; save_weights / load_weights, src/model.cpp:120-196).
 * create_from_weights: an engine whose weights come from the file (any values: norm weights included) -- the config
 * is read from the header (returned in cfg_out when non-null), every tensor is shape-checked against it, and the
 * trailing weights_checksum is recomputed (on the GPU) and must match: TKV_ERR_NOT_FOUND (missing file),
 * TKV_ERR_FORMAT (magic, version, truncation, shapes, checksum), TKV_ERR_CONFIG (an invalid config). The engine's
 * fingerprint is model_fingerprint(config, checksum), so chunk ids agree with a reference engine on the same weights.
 * save_weights: writes init_random(cfg, seed) as a TKVW file (byte-identical to the reference's save_weights), the
 * f64 draws generated on `device`. */
tkv_status tkv_engine_create_from_weights(const char* path, const tkv_engine_opts* opts, tkv_engine** out,
                                          tkv_model_config* cfg_out);
tkv_status tkv_save_weights(const tkv_model_config* cfg, uint64_t seed, const char* path, int device);
tkv_status tkv_engine_fingerprint(const tkv_engine* eng, uint64_t* out);
tkv_status tkv_engine_config(const tkv_engine* eng, tkv_model_config* out);

/* Offline chunk precompute. Engine::ingest_chunk_payload (pipeline.hpp:86-88;
 * src/pipeline.cpp:97-134), batched: `payloads` holds n_chunks UNFRAMED payloads back to back,
 * offsets[n_chunks+1]. Each chunk is framed [256] payload [257], content-addressed, and — if new —
 * prefilled with a block-diagonal causal mask in ONE packed forward; unrotated K and V land in
 * the paged HBM store. ids_out[n_chunks] receives the content ids. Idempotent. */
tkv_status tkv_ingest_chunks(tkv_engine* eng, const int32_t* payloads, const int64_t* offsets,
                             int64_t n_chunks, uint64_t* ids_out, tkv_ingest_stats* stats);

/* TKVC import (src/kvstore.cpp:134-207; docs/formats.md:114-140): loads a reference cache file
 * into the HBM store (f64/f32 -> engine dtype, round to nearest). Same validation and errors as
 * CacheStore::load. */
tkv_status tkv_import_tkvc(tkv_engine* eng, const char* path, uint64_t* id_out);
/* TKVC export of a stored chunk (CacheStore::store, src/kvstore.cpp:78-132), f32 elements. */
tkv_status tkv_export_tkvc(tkv_engine* eng, uint64_t chunk_id, const char* path);

tkv_status tkv_store_contains(const tkv_engine* eng, uint64_t chunk_id, int* out);
tkv_status tkv_store_chunk_tokens(const tkv_engine* eng, uint64_t chunk_id, int64_t* out);
tkv_status tkv_store_count(const tkv_engine* eng, int64_t* chunks, int64_t* pages_used, int64_t* pages_total);
/* CacheStore::ids (kvstore.cpp): every stored chunk id, ascending; ids_out may be NULL to query the count. */
tkv_status tkv_store_ids(const tkv_engine* eng, uint64_t* ids_out, int64_t capacity, int64_t* n_out);
/* Drop a chunk from the store and return its pages (no reference analogue: the reference store is a directory
 * of TKVC files, kvstore.cpp:78-211; this is the capacity policy of the HBM store). Contexts assembled earlier
 * keep their gathered KV; only their unrotated re-read (tkv_context_read_kv, rotated=0) then fails StaleCache. */
tkv_status tkv_store_evict(tkv_engine* eng, uint64_t chunk_id);
/* Retrieval: embed (retrieval.cpp:64-88) on the host, exhaustive cosine top-k over the index
 * in HBM (retrieval.cu), ranking identical to RetrievalIndex::top_k (retrieval.cpp:117-133): cosine descending,
 * ties by ascending chunk id, min(k, size) results, k in [1, 256] when the index holds more than 256 chunks.
 * tkv_ingest_chunks indexes every newly ingested chunk over its unframed payload; tkv_index_add adds one. */
tkv_status tkv_embed(const int32_t* tokens, int64_t n, int64_t dim, double* out);
tkv_status tkv_index_add(tkv_engine* eng, uint64_t chunk_id, const int32_t* payload, int64_t n, int* added);
int64_t tkv_index_size(const tkv_engine* eng);
tkv_status tkv_index_top_k(tkv_engine* eng, const int32_t* query, int64_t n, int64_t k, uint64_t* ids_out,
                           double* scores_out, int64_t* n_out);
/* Two-tier store occupancy in pages: HBM pool and the pinned host spill tier (host_spill_tokens). New chunks go
 * to HBM while it has room, then to the host tier; tier of a chunk: 0 = HBM, 1 = pinned host, 2 = a peer GPU. */
tkv_status tkv_store_tiers(const tkv_engine* eng, int64_t* hbm_used, int64_t* hbm_total, int64_t* host_used,
                           int64_t* host_total);
tkv_status tkv_store_chunk_tier(const tkv_engine* eng, uint64_t chunk_id, int32_t* tier);
/* Copy one stored (unrotated) tensor to host as float32 [tokens, kv_head_num*head_size]. */
tkv_status tkv_store_read(const tkv_engine* eng, uint64_t chunk_id, int64_t layer, tkv_kv_which which,
                          float* host_out, int64_t capacity_elems);

/* KV injection. Engine::assemble (pipeline.hpp:93; src/pipeline.cpp:136-164). Runs the fused
 * KV-gather + RoPE kernel: the chunks' store pages are copied into the request cache with keys
 * re-rotated to reordered or composite position ids. */
tkv_status tkv_assemble(tkv_engine* eng, const uint64_t* chunk_ids, int64_t n, tkv_position_mode mode,
                        tkv_context** out);
/* Query prefill. Engine::prefill_query (pipeline.hpp:97-99; src/pipeline.cpp:166-186). Extends ctx
 * in place; logits_out[vocab] receives the last query token's logits (the TTFT logits). */
tkv_status tkv_prefill_query(tkv_engine* eng, tkv_context* ctx, const int32_t* query, int64_t n,
                             float* logits_out, tkv_flops* flops);
/* Same, with tokens and logits already in device memory (no host copies, no sync). Device-side errors of
 * this call (token outside vocab, non-finite logits, degenerate rows) are deferred: tkv_engine_check reports
 * them. The context keeps no host logits, so tkv_greedy_decode on it fails with TKV_ERR_DOMAIN. */
tkv_status tkv_engine_check(tkv_engine* eng); /* sync the engine stream; report deferred device errors */
tkv_status tkv_prefill_query_device(tkv_engine* eng, tkv_context* ctx, const int32_t* d_query, int64_t n,
                                    float* d_logits_out);
/* Batched query prefill (BASELINE config 3: batch 32): request r prefills queries[offsets[r], offsets[r+1]) over
 * its own context ctxs[r] exactly as tkv_prefill_query would (pipeline.cpp:166-186); the projections and the MLP
 * run once over all requests' tokens (one large-M GEMM per projection), attention per request on its own cache.
 * logits_out: [n_req][vocab] (last token of each request). flops accumulates every request's cost. */
tkv_status tkv_prefill_query_batch(tkv_engine* eng, tkv_context* const* ctxs, int64_t n_req, const int32_t* queries,
                                   const int64_t* offsets, float* logits_out, tkv_flops* flops);
/* Full-concatenation prefill. Engine::naive_prefill (pipeline.hpp:104-108; src/pipeline.cpp:188-229).
 * `framed` holds n_chunks FRAMED chunks back to back (offsets[n_chunks+1]). ctx_out is optional. */
tkv_status tkv_naive_prefill(tkv_engine* eng, const int32_t* framed, const int64_t* offsets, int64_t n_chunks,
                             const int32_t* query, int64_t nq, tkv_mask_mode mode, float* logits_out,
                             tkv_flops* flops, tkv_context** ctx_out);
/* Engine::naive_prefill_ids (pipeline.hpp:109-112): chunk tokens come from the store's record. */
tkv_status tkv_naive_prefill_ids(tkv_engine* eng, const uint64_t* ids, int64_t n, const int32_t* query,
                                 int64_t nq, tkv_mask_mode mode, float* logits_out, tkv_flops* flops,
                                 tkv_context** ctx_out);
/* greedy_decode (src/model.cpp:274-303): argmax (ties -> lowest id), stop on eos (258). */
tkv_status tkv_greedy_decode(tkv_engine* eng, tkv_context* ctx, int64_t max_new, int32_t* tokens_out,
                             int64_t* n_out);

/* AssembledContext accessors (include/turbokv/context.hpp:16-38). */
void tkv_context_destroy(tkv_context* ctx);
int64_t tkv_context_total_tokens(const tkv_context* ctx);
int64_t tkv_context_next_position(const tkv_context* ctx);
int64_t tkv_context_segments(const tkv_context* ctx, int64_t* lens, int32_t* is_query, int64_t cap);
tkv_status tkv_context_positions(const tkv_context* ctx, int64_t* out, int64_t capacity);
tkv_status tkv_context_last_logits(const tkv_context* ctx, float* out, int64_t capacity);
/* Request-cache tensor of one layer to host as float32 [total_tokens, kv_dim]. rotated=1 returns
 * keys as the attention kernels consume them (rotated by the context positions); rotated=0 returns
 * the unrotated keys of the injected chunk tokens (re-gathered from the store with identity
 * rotation) followed by the query tokens' unrotated keys. */
tkv_status tkv_context_read_kv(const tkv_context* ctx, int64_t layer, tkv_kv_which which, int rotated,
                               float* host_out, int64_t capacity_elems);
/* The attention predicate the kernels apply for the context's last forward, materialised as
 * 0/1 bytes [rows, cols] (build_mask / causal_rows, src/attention.cpp:50-92). */
tkv_status tkv_context_mask(const tkv_context* ctx, uint8_t* out, int64_t rows, int64_t cols);

/* Multi-GPU (one engine per GPU; requests data-parallel; the store sharded by document). A remote chunk
 * is registered under a peer slot and read by the gather kernel straight from the peer's HBM over
 * NVLink (P2P loads fused with the RoPE pass), or copied once into the local store (fetch_remote). */
typedef struct {
    uint8_t bytes[64];
} tkv_ipc_handle;
/* cudaIpcGetMemHandle of this engine's page pool (one process per GPU: share it with the peers). */
tkv_status tkv_store_export_ipc(tkv_engine* eng, tkv_ipc_handle* out, uint64_t* pool_bytes);
/* Map a peer process's pool (cudaIpcOpenMemHandle, lazy peer access) into peer slot `slot` (1..14). The raw
 * handle carries no model identity or geometry: prefer tkv_store_import_directory, which validates both. */
tkv_status tkv_store_attach_ipc(tkv_engine* eng, int32_t slot, const tkv_ipc_handle* handle);
/* Same, for a peer engine in this process (possibly another GPU: enables peer access). */
tkv_status tkv_store_attach_engine(tkv_engine* eng, int32_t slot, tkv_engine* peer);
/* Directory entry of a locally owned chunk: its page indices and token count. */
tkv_status tkv_store_chunk_pages(const tkv_engine* eng, uint64_t chunk_id, int32_t* pages, int64_t capacity,
                                 int64_t* n_pages, int64_t* len);
/* Register a chunk owned by the peer in `slot` (its page list from tkv_store_chunk_pages on the owner).
 * `framed` (nullable, len tokens) enables naive_prefill_ids for it. No-op if the id is already known. */
tkv_status tkv_store_register_remote(tkv_engine* eng, uint64_t chunk_id, int32_t slot, int64_t len,
                                     const int32_t* pages, int64_t n_pages, const int32_t* framed);
/* Copy a registered remote chunk into the local store (fetch-once cache policy). */
tkv_status tkv_store_fetch_remote(tkv_engine* eng, uint64_t chunk_id);
/* Store directory blob of this engine's locally owned chunks (ids, token counts, page lists, framed tokens) with
 * its pool's IPC handle, fingerprint and page geometry: what a peer needs to read these chunks over NVLink.
 * buf = NULL returns the size only. Little-endian layout: "TKVD", u32 version, u64 fingerprint, u64 page_bytes,
 * i64 page_tokens, i64 pool pages, 64 B cudaIpcMemHandle, i64 n, then n x {u64 id, i64 len, i64 n_pages,
 * i32 pages[n_pages], i64 n_framed, i32 framed[n_framed]} sorted by id. Exported chunks become SHARED: peers
 * read their pages, so tkv_store_evict refuses them (TKV_ERR_CONFIG). The transport (NCCL, MPI, sockets,
 * torch.distributed) is the caller's. */
tkv_status tkv_store_export_directory(tkv_engine* eng, uint8_t* buf, int64_t capacity, int64_t* size);
/* Register a peer's directory under peer slot `slot` (1..14): TKV_ERR_STALE_CACHE when the fingerprint or the
 * page geometry differs from this engine's, TKV_ERR_FORMAT for a corrupt blob or a page index outside the
 * peer's pool (nothing is registered then); opens the peer pool through its IPC handle unless the slot is
 * already attached (tkv_store_attach_engine for a peer engine in this process). */
tkv_status tkv_store_import_directory(tkv_engine* eng, int32_t slot, const uint8_t* blob, int64_t size);
/* Two-tier store policy: every retrieval (tkv_assemble) counts a hit for its chunks; rebalance moves the most-retrieved
 * chunks of the pinned host tier into HBM (demoting the least-retrieved HBM chunks when HBM is full, only while the
 * incoming chunk has more hits), at most max_moves page-list moves, then halves every hit count. Chunks listed in an
 * exported directory stay where they are. */
tkv_status tkv_store_rebalance(tkv_engine* eng, int64_t max_moves, int64_t* promoted, int64_t* demoted);
/* KV bytes read from peer pools so far (NVLink traffic of the gather + fetches). */
int64_t tkv_remote_bytes(const tkv_engine* eng);

/* Measurement hooks (bench.py): the engine's CUDA stream, and per-kernel-class device time
 * accumulated with CUDA events on that stream while profiling is on. */
void* tkv_engine_stream(tkv_engine* eng);
tkv_status tkv_profile_enable(tkv_engine* eng, int on);
/* names: "gather_rope", "attention", "gemm", "epilogue", "other"; returns total ms and launches */
tkv_status tkv_profile_read(tkv_engine* eng, const char* kernel_class, double* total_ms, int64_t* launches);
tkv_status tkv_profile_reset(tkv_engine* eng);
/* Count of kernels launched by the engine since creation (all classes). */
int64_t tkv_launch_count(const tkv_engine* eng);
/* Host->device and device->host bytes the engine has copied for its callers since creation (query tokens,
 * positions, mask ranges, gather descriptors, logits, error words): the e2e accounting of bench.py. */
tkv_status tkv_io_bytes(const tkv_engine* eng, int64_t* h2d, int64_t* d2h);

/* Debug (testing::mask_fault_hook, include/turbokv/pipeline.hpp:57-62): override the visible key range of mask rows
 * of the NEXT naive prefill -- row rows[i] (negative: counted from the end) sees exactly keys [lo[i], hi[i]]; cleared
 * after that prefill. The reference's `verify --inject-fault` corruption (the last query row loses column 0,
 * tools/turbokv_main.cpp:593-599) is rows = {-1}, lo = {1}, hi = {N - 1}. */
tkv_status tkv_debug_set_mask_rows(tkv_engine* eng, const int64_t* rows, const int32_t* lo, const int32_t* hi, int64_t n);
/* Same, widening: row `row` additionally sees columns down to `col` (a row of chunk 1 may see chunk 0). */
tkv_status tkv_debug_set_mask_fault(tkv_engine* eng, int64_t row, int64_t col);

/* Kernel-level entry points for unit tests (host buffers in, host fp32 out; inputs are rounded to
 * `dtype` on the device first). gemm: out[M,N] = A[M,K] . W[N,K]^T with the tcgen05 (use_tc=1) or
 * SIMT kernel and `splits` split-K partials (0 = auto). attention: the engine's flash attention with
 * the [lo, hi] row predicate; q [Tq, H*d], k/v [Tk, Hkv*d], out [Tq, H*d]. impl: 0 = the engine's choice
 * (tcgen05 for bf16 head_size 128), 1 = SIMT, 2 = the decode-sized kernel (bf16, d = 128, Tq * H / Hkv in
 * {4, 7, 8, 16}). */
/* weights_checksum / model_fingerprint (model.cpp:94-118) of (cfg, seed): device >= 0 hashes on that GPU
 * (the engine's path), device = -1 streams the generator through FNV-1a on one host core (slow; tests). */
tkv_status tkv_debug_weights_checksum(const tkv_model_config* cfg, uint64_t seed, int device, uint64_t* checksum,
                                      uint64_t* fingerprint);
/* Rows [row0, row0 + nrows) of a device weight tensor as float32 (bf16 widened), in the device layout ([out][in]):
 * which 0 = Wqkv (wq | wk | wv rows), 1 = Wo, 2 = Wgu (gate / up rows interleaved in 64-row blocks when
 * intermediate_size % 64 == 0), 3 = Wdown, 4 = lm_head, 5 = embedding (f32 [vocab][hidden]). */
tkv_status tkv_debug_weight_rows(tkv_engine* eng, int64_t layer, int which, int64_t row0, int64_t nrows, float* out);
tkv_status tkv_debug_gemm(int device, tkv_dtype dtype, int use_tc, const float* A, const float* W, int64_t M,
                          int64_t N, int64_t K, int splits, float* out);
/* GEMM tuning/timing (tools/gemm_sweep.py): knobs = ring stages, smem budget KB, CTAs per SM, weight
 * stream L2 evict_first (0 = default for the first three). bench: device-resident buffers, mean ms. */
/* attention pipeline timeline of CTA (0,0,0): on=1 arms it; out != NULL reads [32 tiles][10 events] clock64 */
tkv_status tkv_debug_attn_trace(int on, uint64_t* out, int64_t capacity);
tkv_status tkv_debug_set_gemm_knobs(int stages, int smem_kb, int ctas_per_sm, int w_evict_first);
/* GEMM pipeline trace of CTA 0 of the next tcgen05 GEMM launches (on != 0 arms and clears it; out != NULL first copies
 * the last trace): clock64 per stage [it][3] = producer issue, MMA saw the stage full, MMA committed it (1024 stages),
 * then [unit][2] = epilogue start / end (64 units). */
tkv_status tkv_debug_gemm_trace(int on, uint64_t* out, int64_t capacity);
/* Kernel timeline of this engine's launches (non-perturbing: PDL overlap intact). on = 1 clears and arms it; on = 0
 * disarms, synchronises and copies, per launch in stream order, out[2i..2i+1] = globaltimer ns (first CTA past
 * griddepcontrol.wait, i.e. the predecessor grid completed; last warp done) and classes[i] = 0 KV gather, 1 attention
 * (+ split merge), 2 projection GEMM, 3 epilogue (embed, residual, QKV), 4 other (lm_head); capacity = launches;
 * *n_launches = launches recorded. Instrumented: GEMM, attention, split merge, residual / QKV epilogues, embed,
 * lm_head, KV gather. */
tkv_status tkv_kernel_timeline(tkv_engine* eng, int on, uint64_t* out, int32_t* classes, int64_t capacity,
                               int64_t* n_launches);
tkv_status tkv_debug_gemm_bench(int device, int64_t M, int64_t N, int64_t K, int splits, int swiglu, int iters,
                                double* ms_per_launch);
tkv_status tkv_debug_attention(int device, tkv_dtype dtype, int impl, const float* q, const float* k,
                               const float* v, const int32_t* lo, const int32_t* hi, int64_t Tq, int64_t Tk,
                               int64_t H, int64_t Hkv, int64_t d, float* out);

#ifdef __cplusplus
}
#endif

#endif /* TKV_H */

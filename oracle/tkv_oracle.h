/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the TurboRAG prefill path.
 *
 * A plain-C, float64 restatement of the reference `turbokv` algorithm
 * (/root/reference/proj, C++20). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker. The
 * product library (paper_2410_07590_b200/libtkv_b200.so) never links it.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference compiled from its own sources (oracle/_ref) and
 * against the golden vectors frozen in the reference's docs/tests
 * (proj/docs/formats.md:45-52,107-112; proj/tests/test_model.cpp:67-80;
 * proj/tests/test_pipeline.cpp:118-148), committed under tests/golden/.
 *
 * Masks are expressed the way the CUDA kernels consume them: row i of a
 * forward over `n_past + n` columns may attend to column j iff
 * row_lo[i] <= j <= row_hi[i]. Every mask the reference builds
 * (causal_rows, build_mask Causal/Independent; proj/src/attention.cpp:50-92)
 * has this form.
 */
#ifndef TKV_ORACLE_H
#define TKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t layer_num, head_num, kv_head_num, head_size, hidden_size, intermediate_size, vocab_size;
    double rope_base, norm_eps;
} tko_config;

typedef struct tko_model tko_model;

/* status codes: same numbering as tkv_status (include/tkv.h) */
const char* tko_last_error(void);

uint64_t tko_splitmix_at(uint64_t seed, uint64_t index);
int tko_config_validate(const tko_config* c);
uint64_t tko_fingerprint_seed(const tko_config* c);
uint64_t tko_chunk_content_id(uint64_t model_fingerprint, const int32_t* framed, int64_t n);

int tko_model_create(const tko_config* c, uint64_t seed, tko_model** out);
void tko_model_destroy(tko_model* m);
uint64_t tko_weights_checksum(tko_model* m);
uint64_t tko_model_fingerprint(tko_model* m);
/* which: 0 emb, 1 wq, 2 wk, 3 wv, 4 wo, 5 gate, 6 up, 7 down, 8 lm_head ([in,out] row-major) */
const double* tko_weight(const tko_model* m, int64_t layer, int which, int64_t* rows, int64_t* cols);

/* One decoder forward (proj/src/model.cpp:198-272). past_k/past_v are
 * [layer][n_past][kv_dim]; new_k/new_v (nullable) receive [layer][n][kv_dim]
 * unrotated. logits (nullable) receives [n][vocab], or [1][vocab] for the
 * last row when last_only != 0. */
int tko_forward(const tko_model* m, const int32_t* tokens, int64_t n, const int64_t* positions,
                const double* past_k, const double* past_v, const int64_t* past_positions, int64_t n_past,
                const int64_t* row_lo, const int64_t* row_hi, double* logits, int last_only,
                double* new_k, double* new_v);

/* Engine::assemble position ids (proj/src/pipeline.cpp:136-164). */
int tko_assemble_positions(const int64_t* lens, int64_t n_chunks, int reordered, int64_t* positions,
                           int64_t* next_position);

/* build_mask (attention.cpp:50-78) over chunk lens + query len as [lo, hi] rows. */
int tko_build_mask_rows(const int64_t* lens, int64_t n_segments, int independent, int64_t* row_lo,
                        int64_t* row_hi);
/* causal_rows(new, past) (attention.cpp:80-92) as [lo, hi] rows. */
int tko_causal_rows(int64_t new_tokens, int64_t past_tokens, int64_t* row_lo, int64_t* row_hi);

/* ingest_chunk_payload's forward (pipeline.cpp:97-134): framed tokens -> unrotated K/V [L][n][kv]. */
int tko_chunk_kv(const tko_model* m, const int32_t* framed, int64_t n, double* k_out, double* v_out);

/* prefill_query (pipeline.cpp:166-186) over an assembled context. */
int tko_prefill_query(const tko_model* m, const double* ctx_k, const double* ctx_v, const int64_t* ctx_pos,
                      int64_t n_ctx, int64_t next_position, const int32_t* q, int64_t nq, double* logits);

/* naive_prefill (pipeline.cpp:188-229): framed chunks packed with offsets[n_chunks+1]. */
int tko_naive_prefill(const tko_model* m, const int32_t* tokens, const int64_t* offsets, int64_t n_chunks,
                      const int32_t* q, int64_t nq, int independent, double* logits);

/* weights_checksum (model.cpp:94-112) streamed from the generator (no materialised weights), and
 * model_fingerprint (model.cpp:114-118) of a checksum. */
uint64_t tko_weights_checksum_stream(const tko_config* c, uint64_t seed);
uint64_t tko_fingerprint_of(const tko_config* c, uint64_t checksum);

/* rope_rotate_heads_inplace (rope.cpp:75-88). */
int tko_rope_rotate(double* rows, int64_t n_rows, int64_t cols, const int64_t* positions, int64_t head_size,
                    double base);

/* Appendix-C cost model (costmodel.cpp:11-83). */
uint64_t tko_flops_total(const tko_config* c, int64_t n_input, int64_t n_context, int64_t batch);

/* Retrieval (retrieval.cpp:64-88 embed, :90-100 cosine, :117-133 top_k). embed: feature-hashed token bigrams
 * with a leading -1 sentinel, FNV-1a over the two u32s, bucket h % dim, sign by the top bit, L2-normalised.
 * top_k: cosine against every row, sorted by cosine descending then chunk id ascending; returns min(k, n). */
int tko_embed(const int32_t* tokens, int64_t n, int64_t dim, double* out);
int64_t tko_top_k(const double* emb, const uint64_t* ids, int64_t n, int64_t dim, const double* query, int64_t k,
                  uint64_t* ids_out, double* scores_out);

#ifdef __cplusplus
}
#endif

#endif

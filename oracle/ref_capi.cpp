// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" wrapper over the UNMODIFIED reference `turbokv` library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libturbokv_ref.so). It lets the Python tests and bench.py's
// CPU-baseline leg drive the reference's own code path:
//   Engine::ingest_chunk_payload  proj/src/pipeline.cpp:97-134
//   Engine::assemble              proj/src/pipeline.cpp:136-164
//   Engine::prefill_query         proj/src/pipeline.cpp:166-186
//   Engine::naive_prefill         proj/src/pipeline.cpp:188-229
//   build_mask / causal_rows      proj/src/attention.cpp:50-92
//   greedy_decode                 proj/src/model.cpp:274-303
// Every entry returns a status code with the same numbering as tkv_status in
// include/tkv.h (one code per turbokv::*Error class, errors.hpp:10-67).
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "turbokv/attention.hpp"
#include "turbokv/bench.hpp"
#include "turbokv/costmodel.hpp"
#include "turbokv/errors.hpp"
#include "turbokv/model.hpp"
#include "turbokv/pipeline.hpp"
#include "turbokv/retrieval.hpp"
#include "turbokv/rng.hpp"
#include "turbokv/rope.hpp"

using namespace turbokv;

namespace {

thread_local std::string g_err;

struct RefConfig {  // same field order as tkv_model_config
    int64_t layer_num, head_num, kv_head_num, head_size, hidden_size, intermediate_size,
        vocab_size;
    double rope_base, norm_eps;
};

ModelConfig to_cfg(const RefConfig* c) {
    ModelConfig m;
    m.layer_num = c->layer_num;
    m.head_num = c->head_num;
    m.kv_head_num = c->kv_head_num;
    m.head_size = c->head_size;
    m.hidden_size = c->hidden_size;
    m.intermediate_size = c->intermediate_size;
    m.vocab_size = c->vocab_size;
    m.rope_base = c->rope_base;
    m.norm_eps = c->norm_eps;
    return m;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 2;
    } catch (const DomainError& e) {
        g_err = e.what();
        return 3;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 4;
    } catch (const DegenerateRowError& e) {
        g_err = e.what();
        return 5;
    } catch (const IoError& e) {
        g_err = e.what();
        return 6;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 7;
    } catch (const NotFoundError& e) {
        g_err = e.what();
        return 8;
    } catch (const StaleCacheError& e) {
        g_err = e.what();
        return 9;
    } catch (const NoContextError& e) {
        g_err = e.what();
        return 10;
    } catch (const Error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

struct RefEngine {
    std::unique_ptr<Engine> engine;
};

struct RefCtx {
    AssembledContext ctx;
};

std::vector<Token> to_tokens(const int32_t* p, int64_t n) {
    return std::vector<Token>(p, p + n);
}

void copy_ctx_out(const AssembledContext& ctx, int64_t* positions, int64_t* next_pos) {
    if (positions) {
        std::memcpy(positions, ctx.positions.ids.data(), ctx.positions.ids.size() * sizeof(int64_t));
    }
    if (next_pos) *next_pos = ctx.next_position;
}

}  // namespace

extern "C" {

// retrieval.cpp:64-88 (embed) and :117-133 (RetrievalIndex::top_k over records built from `emb`/`ids`)
int ref_embed(const int32_t* tokens, int64_t n, int64_t dim, double* out) {
    return guard([&] {
        std::vector<Token> t(tokens, tokens + n);
        auto v = embed(t, dim);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_top_k(const double* emb, const uint64_t* ids, int64_t n, int64_t dim, const double* query, int64_t k,
              uint64_t* ids_out, int64_t* n_out) {
    return guard([&] {
        RetrievalIndex idx;
        for (int64_t r = 0; r < n; ++r) {
            ChunkRecord rec;
            rec.chunk_id = ids[r];
            rec.embedding.assign(emb + r * dim, emb + (r + 1) * dim);
            idx.add(std::move(rec));
        }
        auto top = idx.top_k(std::vector<double>(query, query + dim), k);
        std::memcpy(ids_out, top.data(), top.size() * sizeof(uint64_t));
        *n_out = (int64_t)top.size();
    });
}

const char* ref_last_error() { return g_err.c_str(); }

int ref_preset(const char* name, RefConfig* out) {
    return guard([&] {
        ModelConfig m = ModelConfig::preset(name);
        *out = RefConfig{m.layer_num, m.head_num,         m.kv_head_num, m.head_size, m.hidden_size,
                         m.intermediate_size, m.vocab_size, m.rope_base, m.norm_eps};
    });
}

uint64_t ref_splitmix_at(uint64_t seed, uint64_t i) { return SplitMix64::at(seed, i); }

int ref_weights_identity(const RefConfig* c, uint64_t seed, uint64_t* checksum, uint64_t* fingerprint,
                         double* emb00) {
    return guard([&] {
        ModelConfig cfg = to_cfg(c);
        ModelWeights w = init_random(cfg, seed);
        *checksum = weights_checksum(w);
        *fingerprint = model_fingerprint(cfg, w);
        if (emb00) *emb00 = w.embedding.at(0, 0);
    });
}

// Copies one weight tensor in the reference's [in, out] row-major layout.
// which: 0 emb, 1 wq, 2 wk, 3 wv, 4 wo, 5 gate, 6 up, 7 down, 8 lm_head.
int ref_weight_tensor(const RefConfig* c, uint64_t seed, int layer, int which, double* out) {
    return guard([&] {
        ModelConfig cfg = to_cfg(c);
        ModelWeights w = init_random(cfg, seed);
        const Matrix* m = nullptr;
        if (which == 0) m = &w.embedding;
        else if (which == 8) m = &w.lm_head;
        else {
            const LayerWeights& L = w.layers.at(static_cast<size_t>(layer));
            const Matrix* t[] = {nullptr, &L.wq, &L.wk, &L.wv, &L.wo, &L.w_gate, &L.w_up, &L.w_down};
            m = t[which];
        }
        std::memcpy(out, m->data(), static_cast<size_t>(m->size()) * sizeof(double));
    });
}

int ref_engine_create(const RefConfig* c, uint64_t seed, const char* store_root, int store_dtype,
                      void** out) {
    return guard([&] {
        auto* e = new RefEngine;
        e->engine = std::make_unique<Engine>(to_cfg(c), seed, store_root,
                                             store_dtype == 2 ? StoreDtype::F32 : StoreDtype::F64);
        *out = e;
    });
}

void ref_engine_destroy(void* e) { delete static_cast<RefEngine*>(e); }

uint64_t ref_engine_fingerprint(void* e) { return static_cast<RefEngine*>(e)->engine->fingerprint(); }

// Engine::answer (pipeline.cpp:247-308): retrieved ids, answer tokens and the counters
// stats = {prefill_flops, modeled_prefill_flops, decode_flops, context_tokens, query_tokens}
int ref_answer(void* e, const char* question, int64_t k, int mode, int64_t max_new, uint64_t* ids_out, int64_t ids_cap,
               int64_t* n_ids, int32_t* tokens_out, int64_t tok_cap, int64_t* n_tok, uint64_t* stats) {
    return guard([&] {
        const AnswerResult r = static_cast<RefEngine*>(e)->engine->answer(question, k, static_cast<PathMode>(mode), max_new);
        *n_ids = (int64_t)r.retrieved.size();
        for (size_t i = 0; i < r.retrieved.size() && (int64_t)i < ids_cap; ++i) ids_out[i] = r.retrieved[i];
        *n_tok = (int64_t)r.tokens.size();
        for (size_t i = 0; i < r.tokens.size() && (int64_t)i < tok_cap; ++i) tokens_out[i] = r.tokens[i];
        stats[0] = r.prefill_flops;
        stats[1] = r.modeled_prefill_flops;
        stats[2] = r.decode_flops;
        stats[3] = (uint64_t)r.context_tokens;
        stats[4] = (uint64_t)r.query_tokens;
    });
}

// retrieval.cpp chunk_document: chunk lengths (bytes) in order; the tokens are the text's bytes
int ref_chunk_document(const char* text, int64_t n, int64_t target_len, int64_t* lens_out, int64_t cap, int64_t* n_out) {
    return guard([&] {
        const auto chunks = chunk_document(std::string(text, (size_t)n), target_len);
        *n_out = (int64_t)chunks.size();
        for (size_t i = 0; i < chunks.size() && (int64_t)i < cap; ++i) lens_out[i] = (int64_t)chunks[i].size();
    });
}

// bench.cpp ingest_synthetic (the reference's own bench corpus): chunk ids in ingest order
int ref_bench_ingest(void* e, const int64_t* grid, int64_t n_grid, uint64_t seed, uint64_t* ids_out, int64_t cap,
                     int64_t* n_out) {
    return guard([&] {
        BenchConfig cfg;
        cfg.doc_grid.assign(grid, grid + n_grid);
        cfg.seed = seed;
        const std::vector<uint64_t> ids = ingest_synthetic(*static_cast<RefEngine*>(e)->engine, cfg);
        *n_out = (int64_t)ids.size();
        for (size_t i = 0; i < ids.size() && (int64_t)i < cap; ++i) ids_out[i] = ids[i];
    });
}

int ref_ingest(void* e, const int32_t* payload, int64_t n, uint64_t* id_out) {
    return guard([&] {
        *id_out = static_cast<RefEngine*>(e)->engine->ingest_chunk_payload("oracle", to_tokens(payload, n));
    });
}

int ref_store_path(void* e, uint64_t id, char* buf, int64_t cap) {
    return guard([&] {
        std::string p = static_cast<RefEngine*>(e)->engine->store().path_for(id);
        if (static_cast<int64_t>(p.size()) + 1 > cap) throw ShapeError("path buffer too small");
        std::memcpy(buf, p.c_str(), p.size() + 1);
    });
}

int ref_assemble(void* e, const uint64_t* ids, int64_t n, int reordered, void** ctx_out) {
    return guard([&] {
        auto* c = new RefCtx;
        c->ctx = static_cast<RefEngine*>(e)->engine->assemble(
            std::vector<uint64_t>(ids, ids + n),
            reordered ? PositionMode::Reordered : PositionMode::Composite);
        *ctx_out = c;
    });
}

void ref_ctx_destroy(void* c) { delete static_cast<RefCtx*>(c); }

int64_t ref_ctx_total_tokens(void* c) { return static_cast<RefCtx*>(c)->ctx.total_tokens(); }

int ref_ctx_info(void* c, int64_t* positions, int64_t* next_pos) {
    return guard([&] { copy_ctx_out(static_cast<RefCtx*>(c)->ctx, positions, next_pos); });
}

// which: 0 = K (unrotated, as held), 1 = V, 2 = K rotated by the context positions.
int ref_ctx_kv(void* e, void* c, int64_t layer, int which, double* out) {
    return guard([&] {
        const AssembledContext& ctx = static_cast<RefCtx*>(c)->ctx;
        Matrix m = which == 1 ? ctx.v.at(static_cast<size_t>(layer)) : ctx.k.at(static_cast<size_t>(layer));
        if (which == 2) {
            const ModelConfig& cfg = static_cast<RefEngine*>(e)->engine->config();
            rope_rotate_heads_inplace(m, ctx.positions, RopeParams::create(cfg.head_size, cfg.rope_base));
        }
        std::memcpy(out, m.data(), static_cast<size_t>(m.size()) * sizeof(double));
    });
}

int ref_prefill_query(void* e, void* c, const int32_t* q, int64_t nq, double* logits, uint64_t* flops4) {
    return guard([&] {
        FlopCounter fc;
        Matrix last = static_cast<RefEngine*>(e)->engine->prefill_query(static_cast<RefCtx*>(c)->ctx,
                                                                          to_tokens(q, nq), &fc);
        std::memcpy(logits, last.data(), static_cast<size_t>(last.size()) * sizeof(double));
        if (flops4) {
            flops4[0] = fc.qkv;
            flops4[1] = fc.attn;
            flops4[2] = fc.o;
            flops4[3] = fc.mlp;
        }
    });
}

// Framed chunk tokens packed back to back; offsets has n_chunks+1 entries.
int ref_naive_prefill(void* e, const int32_t* tokens, const int64_t* offsets, int64_t n_chunks,
                      const int32_t* q, int64_t nq, int independent, double* logits, void** ctx_out) {
    return guard([&] {
        std::vector<std::vector<Token>> chunks;
        for (int64_t i = 0; i < n_chunks; ++i) {
            chunks.emplace_back(tokens + offsets[i], tokens + offsets[i + 1]);
        }
        auto* c = new RefCtx;
        c->ctx = static_cast<RefEngine*>(e)->engine->naive_prefill(
            chunks, to_tokens(q, nq), independent ? MaskMode::Independent : MaskMode::Causal);
        std::memcpy(logits, c->ctx.last_logits.data(),
                    static_cast<size_t>(c->ctx.last_logits.size()) * sizeof(double));
        if (ctx_out) *ctx_out = c;
        else delete c;
    });
}

// TKVW files (model.cpp:120-196): save_weights of init_random(cfg, seed); load_weights -> (config, checksum); and a
// vanilla causal forward_tokens over a loaded file's weights (last row's logits), for weights other than init_random's
int ref_save_weights(const RefConfig* c, uint64_t seed, const char* path) {
    return guard([&] {
        const ModelConfig cfg = to_cfg(c);
        save_weights(path, cfg, init_random(cfg, seed));
    });
}

int ref_load_weights(const char* path, RefConfig* cfg_out, uint64_t* checksum) {
    return guard([&] {
        ModelWeights w;
        const ModelConfig m = load_weights(path, w);
        *cfg_out = RefConfig{m.layer_num, m.head_num,         m.kv_head_num, m.head_size, m.hidden_size,
                             m.intermediate_size, m.vocab_size, m.rope_base, m.norm_eps};
        *checksum = weights_checksum(w);
    });
}

int ref_forward_file(const char* path, const int32_t* tokens, int64_t n, double* logits) {
    return guard([&] {
        ModelWeights w;
        const ModelConfig cfg = load_weights(path, w);
        ForwardResult fw = forward_tokens(cfg, w, to_tokens(tokens, n), PositionIds::sequential(n, 0), nullptr,
                                          causal_rows(n, 0));
        std::memcpy(logits, fw.logits.row(n - 1), static_cast<size_t>(cfg.vocab_size) * sizeof(double));
    });
}

// `turbokv verify --inject-fault` (tools/turbokv_main.cpp:593-599): the naive path's mask loses the last row's view of
// column 0, through the reference's own testing::mask_fault_hook (pipeline.hpp:57-62). on = 0 clears it.
int ref_set_inject_fault(int on) {
    return guard([&] {
        if (on)
            testing::mask_fault_hook = [](Matrix& mask) {
                mask.at(mask.rows() - 1, 0) = -std::numeric_limits<double>::infinity();
            };
        else
            testing::mask_fault_hook = nullptr;
    });
}

int ref_greedy_decode(void* e, void* c, int64_t max_new, int32_t* out, int64_t* n_out) {
    return guard([&] {
        Engine& eng = *static_cast<RefEngine*>(e)->engine;
        std::vector<Token> toks =
            greedy_decode(eng.config(), eng.weights(), static_cast<RefCtx*>(c)->ctx, max_new, tok::kEos);
        std::memcpy(out, toks.data(), toks.size() * sizeof(int32_t));
        *n_out = static_cast<int64_t>(toks.size());
    });
}

// Dense additive mask as 0/1 "visible" bytes. lens: chunk lengths then the query length.
int ref_build_mask(const int64_t* lens, int64_t n_seg, int independent, uint8_t* out) {
    return guard([&] {
        SegmentLayout layout;
        for (int64_t i = 0; i < n_seg; ++i) {
            Segment s;
            s.id = i;
            s.kind = i + 1 == n_seg ? SegmentKind::Query : SegmentKind::Chunk;
            s.token_count = lens[i];
            layout.segments.push_back(s);
        }
        Matrix m = build_mask(layout, independent ? MaskMode::Independent : MaskMode::Causal);
        for (int64_t i = 0; i < m.size(); ++i) out[i] = m.data()[i] == 0.0 ? 1 : 0;
    });
}

int ref_causal_rows(int64_t new_tokens, int64_t past, uint8_t* out) {
    return guard([&] {
        Matrix m = causal_rows(new_tokens, past);
        for (int64_t i = 0; i < m.size(); ++i) out[i] = m.data()[i] == 0.0 ? 1 : 0;
    });
}

int ref_rope_rotate(const double* in, int64_t rows, int64_t cols, const int64_t* positions, int64_t head_size,
                    double base, double* out) {
    return guard([&] {
        Matrix m(rows, cols, std::vector<double>(in, in + rows * cols));
        rope_rotate_heads_inplace(m, PositionIds(std::vector<int64_t>(positions, positions + rows)),
                                  RopeParams::create(head_size, base));
        std::memcpy(out, m.data(), static_cast<size_t>(m.size()) * sizeof(double));
    });
}

int ref_attend(const double* q, int64_t tq, const double* k, const double* v, int64_t tk, int64_t q_cols,
               int64_t kv_cols, const uint8_t* visible, int64_t head_size, double* out) {
    return guard([&] {
        Matrix qm(tq, q_cols, std::vector<double>(q, q + tq * q_cols));
        Matrix km(tk, kv_cols, std::vector<double>(k, k + tk * kv_cols));
        Matrix vm(tk, kv_cols, std::vector<double>(v, v + tk * kv_cols));
        Matrix mask(tq, tk);
        for (int64_t i = 0; i < tq * tk; ++i)
            mask.data()[i] = visible[i] ? 0.0 : -std::numeric_limits<double>::infinity();
        Matrix o = attend(qm, km, vm, mask, head_size);
        std::memcpy(out, o.data(), static_cast<size_t>(o.size()) * sizeof(double));
    });
}

int ref_flops_compare(const RefConfig* c, int64_t chunk_tokens, int64_t query_tokens, int64_t batch,
                      uint64_t* naive_total, uint64_t* turbo_total, double* reduction) {
    return guard([&] {
        FlopsComparison cmp = compare(to_cfg(c), chunk_tokens, query_tokens, batch);
        *naive_total = cmp.naive.total;
        *turbo_total = cmp.turbo.total;
        *reduction = cmp.reduction_percent;
    });
}

}  // extern "C"

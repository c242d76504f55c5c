// turbokv_compat.hpp — header-only C++ shim that re-exposes the reference's `turbokv` C++ API
// (/root/reference/proj/include/turbokv/*.hpp) on top of the C ABI in tkv.h, so code written against
// the reference (Engine::ingest_chunk_payload / assemble / prefill_query / naive_prefill, the
// exception classes of errors.hpp) switches to the B200 engine by changing an include and a link line.
//
// Differences a caller can observe (documented in INTEGRATION.md):
//  * logits come back as std::vector<float> [vocab] (the reference returns a 1 x vocab f64 Matrix);
//  * AssembledContext is a move-only handle on a request cache in HBM; K/V are read with read_kv();
//  * the store lives in HBM, so `store_root` is replaced by EngineOptions (TKVC import/export keeps
//    byte compatibility with a reference store directory).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tkv.h"

namespace turbokv {

// ---- errors.hpp:10-67 ---------------------------------------------------------------------------
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ShapeError : public Error { public: using Error::Error; };
class DomainError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class DegenerateRowError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class NotFoundError : public Error { public: using Error::Error; };
class StaleCacheError : public Error { public: using Error::Error; };
class NoContextError : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };
class OutOfMemoryError : public Error { public: using Error::Error; };

inline void check(tkv_status s) {
    if (s == TKV_OK) return;
    const std::string m = tkv_last_error();
    switch (s) {
        case TKV_ERR_SHAPE: throw ShapeError(m);
        case TKV_ERR_DOMAIN: throw DomainError(m);
        case TKV_ERR_CONFIG: throw ConfigError(m);
        case TKV_ERR_DEGENERATE_ROW: throw DegenerateRowError(m);
        case TKV_ERR_IO: throw IoError(m);
        case TKV_ERR_FORMAT: throw FormatError(m);
        case TKV_ERR_NOT_FOUND: throw NotFoundError(m);
        case TKV_ERR_STALE_CACHE: throw StaleCacheError(m);
        case TKV_ERR_NO_CONTEXT: throw NoContextError(m);
        case TKV_ERR_CUDA: throw CudaError(m);
        case TKV_ERR_OOM: throw OutOfMemoryError(m);
        default: throw Error(m);
    }
}

using Token = int32_t;

// ---- config.hpp:11-34 ---------------------------------------------------------------------------
struct ModelConfig : tkv_model_config {
    ModelConfig() : tkv_model_config{0, 0, 0, 0, 0, 0, 0, 10000.0, 1e-6} {}
    void validate() const { check(tkv_config_validate(this)); }
    uint64_t fingerprint_seed() const { return tkv_config_fingerprint_seed(this); }
    static ModelConfig preset(const std::string& name) {
        ModelConfig c;
        check(tkv_config_preset(name.c_str(), &c));
        return c;
    }
    static ModelConfig toy() { return preset("toy"); }
    static ModelConfig qwen2_7b_like() { return preset("qwen2-7b"); }
};

// ---- pipeline.hpp / attention.hpp enums ---------------------------------------------------------
enum class PositionMode { Composite = TKV_POS_COMPOSITE, Reordered = TKV_POS_REORDERED };
enum class MaskMode { Causal = TKV_MASK_CAUSAL, Independent = TKV_MASK_INDEPENDENT };

struct IngestStats {
    int64_t chunks = 0;
    int64_t new_chunks = 0;
    uint64_t bytes_written = 0;
};

// ---- costmodel.hpp:53-63 ------------------------------------------------------------------------
struct FlopCounter {
    uint64_t qkv = 0, attn = 0, o = 0, mlp = 0;
    uint64_t total() const { return qkv + attn + o + mlp; }
    void reset() { qkv = attn = o = mlp = 0; }
};

struct EngineOptions : tkv_engine_opts {
    EngineOptions() { tkv_engine_opts_default(this); }
};

// ---- context.hpp:16-38 (a handle on the request cache in HBM) -------------------------------------
class AssembledContext {
public:
    AssembledContext() = default;
    explicit AssembledContext(tkv_context* h) : h_(h) {}
    AssembledContext(AssembledContext&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    AssembledContext& operator=(AssembledContext&& o) noexcept {
        if (this != &o) {
            tkv_context_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    AssembledContext(const AssembledContext&) = delete;
    AssembledContext& operator=(const AssembledContext&) = delete;
    ~AssembledContext() { tkv_context_destroy(h_); }

    tkv_context* handle() const { return h_; }
    int64_t total_tokens() const { return tkv_context_total_tokens(h_); }
    int64_t next_position() const { return tkv_context_next_position(h_); }
    std::vector<int64_t> positions() const {
        std::vector<int64_t> p(static_cast<size_t>(total_tokens()));
        check(tkv_context_positions(h_, p.data(), static_cast<int64_t>(p.size())));
        return p;
    }
    bool prefilled() const {
        float x;
        return tkv_context_last_logits(h_, &x, 0) == TKV_ERR_SHAPE;
    }
    // per-layer [total_tokens, kv_head_num*head_size] as float32
    std::vector<float> read_kv(int64_t layer, bool value, bool rotated, int64_t kv_dim) const {
        std::vector<float> out(static_cast<size_t>(total_tokens() * kv_dim));
        check(tkv_context_read_kv(h_, layer, value ? TKV_V : TKV_K, rotated ? 1 : 0, out.data(),
                                  static_cast<int64_t>(out.size())));
        return out;
    }

private:
    tkv_context* h_ = nullptr;
};

// ---- pipeline.hpp:64-131 ------------------------------------------------------------------------
class Engine {
public:
    Engine(const ModelConfig& config, uint64_t seed, const EngineOptions& opts = EngineOptions()) : config_(config) {
        check(tkv_engine_create(&config_, seed, &opts, &h_));
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { tkv_engine_destroy(h_); }

    const ModelConfig& config() const { return config_; }
    uint64_t fingerprint() const {
        uint64_t f = 0;
        check(tkv_engine_fingerprint(h_, &f));
        return f;
    }
    tkv_engine* handle() const { return h_; }

    uint64_t ingest_chunk_payload(const std::string& /*doc_id*/, const std::vector<Token>& payload,
                                  IngestStats* stats = nullptr) {
        const int64_t offsets[2] = {0, static_cast<int64_t>(payload.size())};
        uint64_t id = 0;
        tkv_ingest_stats st{0, 0, 0};
        check(tkv_ingest_chunks(h_, payload.data(), offsets, 1, &id, &st));
        if (stats) {
            stats->chunks += st.chunks;
            stats->new_chunks += st.new_chunks;
            stats->bytes_written += st.bytes_written;
        }
        return id;
    }

    AssembledContext assemble(const std::vector<uint64_t>& chunk_ids, PositionMode mode) const {
        tkv_context* c = nullptr;
        check(tkv_assemble(h_, chunk_ids.data(), static_cast<int64_t>(chunk_ids.size()),
                           static_cast<tkv_position_mode>(mode), &c));
        return AssembledContext(c);
    }

    std::vector<float> prefill_query(AssembledContext& ctx, const std::vector<Token>& query_tokens,
                                     FlopCounter* counter = nullptr) const {
        std::vector<float> logits(static_cast<size_t>(config_.vocab_size));
        tkv_flops f{0, 0, 0, 0};
        check(tkv_prefill_query(h_, ctx.handle(), query_tokens.data(), static_cast<int64_t>(query_tokens.size()),
                                logits.data(), &f));
        if (counter) {
            counter->qkv += f.qkv;
            counter->attn += f.attn;
            counter->o += f.o;
            counter->mlp += f.mlp;
        }
        return logits;
    }

    AssembledContext naive_prefill(const std::vector<std::vector<Token>>& framed_chunks,
                                   const std::vector<Token>& query_tokens, MaskMode mode,
                                   FlopCounter* counter = nullptr) const {
        std::vector<Token> flat;
        std::vector<int64_t> offsets{0};
        for (const auto& c : framed_chunks) {
            flat.insert(flat.end(), c.begin(), c.end());
            offsets.push_back(static_cast<int64_t>(flat.size()));
        }
        std::vector<float> logits(static_cast<size_t>(config_.vocab_size));
        tkv_flops f{0, 0, 0, 0};
        tkv_context* c = nullptr;
        check(tkv_naive_prefill(h_, flat.data(), offsets.data(), static_cast<int64_t>(framed_chunks.size()),
                                query_tokens.data(), static_cast<int64_t>(query_tokens.size()),
                                static_cast<tkv_mask_mode>(mode), logits.data(), &f, &c));
        if (counter) {
            counter->qkv += f.qkv;
            counter->attn += f.attn;
            counter->o += f.o;
            counter->mlp += f.mlp;
        }
        return AssembledContext(c);
    }

    uint64_t import_tkvc(const std::string& path) {
        uint64_t id = 0;
        check(tkv_import_tkvc(h_, path.c_str(), &id));
        return id;
    }

private:
    ModelConfig config_;
    tkv_engine* h_ = nullptr;
};

// model.hpp:74-81
inline std::vector<Token> greedy_decode(Engine& engine, AssembledContext& ctx, int64_t max_new) {
    std::vector<Token> out(static_cast<size_t>(max_new > 0 ? max_new : 1));
    int64_t n = 0;
    check(tkv_greedy_decode(engine.handle(), ctx.handle(), max_new, out.data(), &n));
    out.resize(static_cast<size_t>(n));
    return out;
}

// tokenizer.hpp:13-26 (byte tokenizer; framing only is on the prefill path)
namespace tok {
constexpr Token kDocStart = 256;
constexpr Token kDocEnd = 257;
constexpr Token kEos = 258;
inline std::vector<Token> encode(const std::string& text) {
    std::vector<Token> out;
    out.reserve(text.size());
    for (unsigned char c : text) out.push_back(static_cast<Token>(c));
    return out;
}
inline std::vector<Token> frame_chunk(const std::vector<Token>& payload) {
    std::vector<Token> framed{kDocStart};
    framed.insert(framed.end(), payload.begin(), payload.end());
    framed.push_back(kDocEnd);
    return framed;
}
}  // namespace tok
using tok::encode;

// kvstore.cpp:58-64
inline uint64_t chunk_content_id(const std::vector<Token>& framed, uint64_t model_fingerprint) {
    return tkv_chunk_content_id(model_fingerprint, framed.data(), static_cast<int64_t>(framed.size()));
}

}  // namespace turbokv

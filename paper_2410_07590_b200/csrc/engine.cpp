// Host engine of the B200-native TurboRAG prefill path + the C ABI of include/tkv.h.
//
// Mirrors turbokv::Engine (include/turbokv/pipeline.hpp:64-131, src/pipeline.cpp:55-241) with the data
// in HBM instead of f64 host matrices:
//   weights       generated on device from (config, seed) in init_random's draw order (model.cpp:68-92),
//                 stored K-major ([out][in]) so every projection is a K-major x K-major GEMM
//   KV store      paged pool [page][layer][K|V][page_tokens][kv_dim] replacing the TKVC directory
//                 (kvstore.cpp:78-207); keys unrotated, as in the reference
//   request cache [layer][K|V][cap][kv_dim] per context; keys ROTATED by the context positions once, at
//                 injection time (the reference re-rotates every layer, model.cpp:253-254)
//   masks         never materialised: per-row [lo, hi] key ranges (attention.cpp:50-92)
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "tkv_internal.h"

namespace tkv {

static thread_local std::string g_last_error;
// PDL on/off is an ENGINE option (TKV_FLAG_NO_PDL): every ABI entry binds its engine, which sets the calling
// thread's launch mode, so engines with different flags can share a process.
static thread_local bool g_pdl = true;
bool pdl_enabled() { return g_pdl; }
void set_pdl_enabled(bool on) { g_pdl = on; }

void fail(tkv_status code, const std::string& msg) { throw Failure{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) fail(TKV_ERR_OOM, std::string(what) + ": out of device memory");
    fail(TKV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- host SplitMix64 / FNV-1a (include/turbokv/rng.hpp:14-78) --------------------------------------------
static inline uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Fnv {
    uint64_t h = 0xCBF29CE484222325ULL;
    inline void u32(uint32_t v) {
        for (int i = 0; i < 4; ++i) {
            h ^= (v >> (8 * i)) & 0xFF;
            h *= 0x100000001B3ULL;
        }
    }
    inline void u64(uint64_t v) {
        u32((uint32_t)v);
        u32((uint32_t)(v >> 32));
    }
    inline void f64(double v) {
        uint64_t b;
        std::memcpy(&b, &v, 8);
        u64(b);
    }
};

// embed (retrieval.cpp:64-88): feature-hashed token bigrams (leading -1 sentinel), FNV-1a over the two u32s,
// bucket h % dim, sign from the top bit, L2-normalised; all-cancelled counts pin e_0 = 1.
static void embed_tokens(const int32_t* t, int64_t n, int64_t dim, double* out) {
    if (n < 1) fail(TKV_ERR_DOMAIN, "embed: empty token list");
    if (dim < 1) fail(TKV_ERR_DOMAIN, "embed: dimension must be >= 1");
    std::fill(out, out + dim, 0.0);
    int32_t prev = -1;
    for (int64_t i = 0; i < n; ++i) {
        Fnv f;
        f.u32((uint32_t)prev);
        f.u32((uint32_t)t[i]);
        out[f.h % (uint64_t)dim] += (f.h >> 63) ? -1.0 : 1.0;
        prev = t[i];
    }
    double ss = 0.0;
    for (int64_t i = 0; i < dim; ++i) ss += out[i] * out[i];
    if (ss == 0.0) {
        out[0] = 1.0;
        ss = 1.0;
    }
    const double inv = 1.0 / std::sqrt(ss);
    for (int64_t i = 0; i < dim; ++i) out[i] *= inv;
}

// sum of squares in the reference cosine's order (retrieval.cpp:93-97)
static double sumsq(const double* v, int64_t dim) {
    double ss = 0.0;
    for (int64_t i = 0; i < dim; ++i) ss += v[i] * v[i];
    return ss;
}

static void validate_cfg(const tkv_model_config& c) {  // ModelConfig::validate (config.cpp:9-29)
    if (c.layer_num < 1 || c.head_num < 1 || c.kv_head_num < 1 || c.head_size < 1 || c.hidden_size < 1 ||
        c.intermediate_size < 1 || c.vocab_size < 1)
        fail(TKV_ERR_CONFIG, "ModelConfig: all counts must be >= 1");
    if (c.hidden_size != c.head_num * c.head_size)
        fail(TKV_ERR_CONFIG, "ModelConfig: hidden_size " + std::to_string(c.hidden_size) +
                                 " != head_num * head_size = " + std::to_string(c.head_num * c.head_size));
    if (c.head_num % c.kv_head_num != 0) fail(TKV_ERR_CONFIG, "ModelConfig: head_num not divisible by kv_head_num");
    if (c.head_size % 2 != 0) fail(TKV_ERR_CONFIG, "ModelConfig: head_size must be even for rotary embedding");
    if (!(c.rope_base > 0.0) || c.norm_eps < 0.0)
        fail(TKV_ERR_CONFIG, "ModelConfig: rope_base must be > 0 and norm_eps >= 0");
}

static uint64_t fp_seed(const tkv_model_config& c) {  // config.cpp:31-42
    Fnv f;
    f.u64((uint64_t)c.layer_num);
    f.u64((uint64_t)c.head_num);
    f.u64((uint64_t)c.kv_head_num);
    f.u64((uint64_t)c.head_size);
    f.u64((uint64_t)c.hidden_size);
    f.u64((uint64_t)c.intermediate_size);
    f.u64((uint64_t)c.vocab_size);
    f.f64(c.rope_base);
    f.f64(c.norm_eps);
    return f.h;
}

// weights_checksum (model.cpp:94-112) streamed from the generator: same bytes as hashing the f64 tensors.
static uint64_t weights_checksum_stream(const tkv_model_config& c, uint64_t seed) {
    const int64_t H = c.hidden_size, qd = c.head_num * c.head_size, kvd = c.kv_head_num * c.head_size,
                  I = c.intermediate_size;
    const double scale = 1.0 / std::sqrt((double)H);
    uint64_t cur = 0;
    Fnv f;
    auto mat = [&](int64_t r, int64_t cc) {
        f.u64((uint64_t)r);
        f.u64((uint64_t)cc);
        const uint64_t n = (uint64_t)(r * cc);
        for (uint64_t i = 0; i < n; ++i) {
            const double u = (double)(splitmix_at(seed, cur + i) >> 11) * 0x1.0p-53;
            f.f64((2.0 * u - 1.0) * scale);
        }
        cur += n;
    };
    auto ones = [&](int64_t n) {
        f.u64((uint64_t)n);
        for (int64_t i = 0; i < n; ++i) f.f64(1.0);
    };
    mat(c.vocab_size, H);
    for (int64_t l = 0; l < c.layer_num; ++l) {
        ones(H);
        ones(H);
        mat(H, qd);
        mat(H, kvd);
        mat(H, kvd);
        mat(qd, H);
        mat(H, I);
        mat(H, I);
        mat(I, H);
    }
    ones(H);
    mat(H, c.vocab_size);
    return f.h;
}

// The same byte stream as weights_checksum_stream, as the word segments the device hash consumes
// (fingerprint.cu): every dimension header a literal word, every norm vector a run of 1.0, every matrix a
// range of generator draws.
static std::vector<FpSeg> checksum_segments(const tkv_model_config& c) {
    const int64_t H = c.hidden_size, qd = c.head_num * c.head_size, kvd = c.kv_head_num * c.head_size,
                  I = c.intermediate_size;
    const double scale = 1.0 / std::sqrt((double)H);
    std::vector<FpSeg> segs;
    uint64_t word = 0, cur = 0;
    auto lit = [&](uint64_t v, uint64_t n) {
        segs.push_back(FpSeg{word, n, v, 0.0, n == 1 ? 0 : 1, 0});
        word += n;
    };
    auto mat = [&](int64_t r, int64_t cc) {
        lit((uint64_t)r, 1);
        lit((uint64_t)cc, 1);
        const uint64_t n = (uint64_t)(r * cc);
        segs.push_back(FpSeg{word, n, cur, scale, 2, 0});
        word += n;
        cur += n;
    };
    uint64_t one_bits;
    const double one = 1.0;
    std::memcpy(&one_bits, &one, 8);
    auto ones = [&](int64_t n) {
        lit((uint64_t)n, 1);
        lit(one_bits, (uint64_t)n);
    };
    mat(c.vocab_size, H);
    for (int64_t l = 0; l < c.layer_num; ++l) {
        ones(H);
        ones(H);
        mat(H, qd);
        mat(H, kvd);
        mat(H, kvd);
        mat(qd, H);
        mat(H, I);
        mat(H, I);
        mat(I, H);
    }
    ones(H);
    mat(H, c.vocab_size);
    return segs;
}

static uint64_t weights_checksum_device(const tkv_model_config& c, uint64_t seed, cudaStream_t s) {
    return device_fnv_words(checksum_segments(c), seed, Fnv{}.h, s);
}

static uint64_t fingerprint_of(const tkv_model_config& c, uint64_t checksum) {  // model.cpp:114-118
    Fnv f;
    f.u64(fp_seed(c));
    f.u64(checksum);
    return f.h;
}

static uint64_t content_id(uint64_t fp, const int32_t* framed, int64_t n) {  // kvstore.cpp:58-64
    Fnv f;
    f.u64(fp);
    f.u64((uint64_t)n);
    for (int64_t i = 0; i < n; ++i) f.u32((uint32_t)framed[i]);
    return f.h;
}

static std::string hex_id(uint64_t id) {
    char b[17];
    std::snprintf(b, sizeof b, "%016llx", (unsigned long long)id);
    return b;
}

// ---- small RAII helpers ---------------------------------------------------------------------------------
struct DevMem {
    void* p = nullptr;
    size_t n = 0;
    static std::atomic<uint64_t>& generation() {
        static std::atomic<uint64_t> g{0};
        return g;
    }
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void* ensure(size_t bytes) {
        if (bytes <= n) return p;
        ++generation();  // captured forward graphs hold these pointers: a reallocation retires them
        release();
        size_t want = std::max(bytes, (size_t)256);
        TKV_CUDA(cudaMalloc(&p, want));
        n = want;
        return p;
    }
    template <typename T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

// Ring of pinned upload buffers. A slot is reused only after the H2D copies enqueued from it
// have executed (event), so back-to-back asynchronous API calls never overwrite in-flight data.
struct StagingRing {
    static constexpr int kSlots = 8;
    struct Slot {
        void* p = nullptr;
        size_t n = 0;
        cudaEvent_t ev = nullptr;
        bool pending = false;
    } slots[kSlots];
    int cur = -1;
    ~StagingRing() {
        for (auto& s : slots) {
            if (s.ev) cudaEventSynchronize(s.ev), cudaEventDestroy(s.ev);
            if (s.p) cudaFreeHost(s.p);
        }
    }
    uint8_t* begin(size_t bytes) {
        cur = (cur + 1) % kSlots;
        Slot& s = slots[cur];
        if (s.pending) TKV_CUDA(cudaEventSynchronize(s.ev));
        s.pending = false;
        if (!s.ev) TKV_CUDA(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
        if (bytes > s.n) {
            if (s.p) cudaFreeHost(s.p);
            s.p = nullptr;
            s.n = std::max(bytes, (size_t)65536);
            TKV_CUDA(cudaHostAlloc(&s.p, s.n, cudaHostAllocDefault));
        }
        return static_cast<uint8_t*>(s.p);
    }
    void end(cudaStream_t st) {
        Slot& s = slots[cur];
        TKV_CUDA(cudaEventRecord(s.ev, st));
        s.pending = true;
    }
};

// NVTX ranges for Nsight Systems / `ncu --nvtx`: one per ABI call, per forward and per layer (host-side push/pop,
// free when no tool is attached; inside a graph capture they mark the capture, replays carry one range)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

enum ProfClass { PC_GATHER = 0, PC_ATTN, PC_GEMM, PC_EPI, PC_OTHER, PC_N };

// Kernel timeline state (tl_take / tkv_kernel_timeline): process-global, armed by one engine at a time.
struct TimelineState {
    unsigned long long* base = nullptr;
    int64_t cap = 0, n = 0;
    int cls = PC_OTHER;
    std::vector<int32_t> classes;
};
TimelineState g_tl;
unsigned long long* tl_take() {
    if (!g_tl.base || g_tl.n >= g_tl.cap) return nullptr;
    g_tl.classes.push_back(g_tl.cls);
    return g_tl.base + 2 * g_tl.n++;
}
void tl_set_class(int cls) { g_tl.cls = cls; }
bool tl_armed() { return g_tl.base != nullptr; }
static const char* kProfNames[PC_N] = {"gather_rope", "attention", "gemm", "epilogue", "other"};

struct Chunk {
    int64_t len = 0;
    std::vector<int32_t> pages;
    std::vector<int32_t> framed;  // empty for TKVC-imported chunks
    int32_t slot = 0;             // page pool holding the pages: 0 = local HBM, >0 = a peer GPU (NVLink)
    bool shared = false;          // listed in an exported directory: peers read its pages, so it cannot be evicted
    uint32_t hits = 0;            // retrievals since the last tier rebalance (halved at each rebalance)
};

}  // namespace tkv

using namespace tkv;

struct tkv_context;

struct tkv_engine {
    tkv_model_config cfg{};
    uint64_t seed = 0;
    tkv_engine_opts opts{};
    DT dt = DT::BF16;
    int device = 0, num_sms = 148;
    cudaStream_t stream = nullptr;
    uint64_t fingerprint = 0;
    bool exact_fp = false;
    int64_t L, H, Hkv, d, hid, I, V, qd, kvd, nqkv;
    bool gu_interleaved = false;
    int gu_block = 0;  // W_gu rows in blocks of gu_block gate + gu_block up rows (128 | 64 | 0 = gate rows then up rows)

    // weights
    DevMem wmem;
    float* emb = nullptr;
    float* ones = nullptr;
    float* norms = nullptr;  // RMSNorm weights, f32: attn_norm(l) at 2l, mlp_norm(l) at 2l + 1, final_norm at 2L (x hid)
    float* norm_attn(int64_t l) const { return norms + (size_t)(2 * l) * hid; }
    float* norm_mlp(int64_t l) const { return norms + (size_t)(2 * l + 1) * hid; }
    float* norm_after_mlp(int64_t l) const { return norms + (size_t)(l + 1 < L ? 2 * (l + 1) : 2 * L) * hid; }
    std::vector<void*> w_qkv, w_o, w_gu, w_down;
    void* w_lm = nullptr;

    // RoPE cos/sin table, float2 [rope_len][d/2], computed in f64 on the host exactly like rope.cpp:21-22,36-40
    DevMem rope;
    int64_t rope_len = 0;

    // paged KV store
    DevMem pool;
    int64_t page_tokens = 64, n_pages = 0;
    size_t page_bytes = 0;
    std::vector<int32_t> free_pages;
    // pinned host spill tier (opts.host_spill_tokens): device-mapped, pool slot kHostPool
    void* host_pool = nullptr;
    int64_t n_host_pages = 0;
    std::vector<int32_t> host_free;
    uint64_t store_epoch = 0;  // bumped by every eviction (contexts that re-read store pages check it)
    // retrieval index (RetrievalIndex, retrieval.hpp:33-60): embeddings in HBM, transposed [kIndexDim][cap]
    std::unordered_map<uint64_t, int64_t> idx_row;
    std::vector<uint64_t> idx_ids;
    std::vector<double> idx_nb;
    int64_t idx_cap = 0;
    DevMem d_idx_emb, d_idx_nb, d_idx_ids, d_idx_q, d_idx_scratch;
    void index_add(uint64_t id, const int32_t* payload, int64_t n, bool* added);
    std::unordered_map<uint64_t, Chunk> chunks;
    PoolTable pools;                     // slot 0 = pool.p; peers attached via IPC or same-process P2P
    int64_t peer_pages[kMaxPools] = {};  // page count of each attached peer pool (0 = unknown: raw IPC attach)
    std::vector<void*> ipc_opened;       // peer pools opened with cudaIpcOpenMemHandle (closed on destroy)
    int64_t remote_bytes = 0;            // bytes of KV gathered from peer pools (bench reporting)

    // forward workspace
    // x: fp32 residual stream; xb = x * norm_w (GEMM input; the RMSNorm scale is folded into consumers); ssp:
    // per-row partial sums of squares (norm_blocks(hid) per row)
    DevMem x, xb, ssp, q, attn, act, partial, attn_ws, d_breq, d_bmaps, d_epireq, logits, err, d_stage, d_segs;
    // per-forward staging arrays (tokens, positions, mask row ranges, store page / slot of each new token): ONE
    // device buffer laid out like the pinned staging slot, so upload_stage is a single H2D copy (one copy node in
    // the stream instead of up to six, each with its own latency before the forward's first kernel)
    int32_t *p_tok = nullptr, *p_pos = nullptr, *p_lo = nullptr, *p_hi = nullptr, *p_page = nullptr, *p_slot = nullptr;
    StagingRing staging;
    std::vector<std::pair<size_t, void*>> ctx_free;  // recycled request-cache buffers
    std::set<tkv_context*> live;

    // measurement
    bool prof_on = false;
    struct Rec {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[PC_N] = {};
    int64_t prof_n[PC_N] = {};
    int64_t launches = 0;
    // testing::mask_fault_hook (pipeline.hpp:57-62): row-range overrides {row (< 0: from the end), lo, hi} applied
    // to the NEXT naive prefill's mask, then cleared
    std::vector<std::array<int64_t, 3>> mask_override;

    ~tkv_engine();
    void bind() const {
        TKV_CUDA(cudaSetDevice(device));
        set_pdl_enabled(!(opts.flags & TKV_FLAG_NO_PDL));
    }

    // ---- profiling ----
    cudaEvent_t take_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        TKV_CUDA(cudaEventCreate(&e));
        return e;
    }
    struct Scope {
        tkv_engine* e;
        int cls;
        cudaEvent_t a = nullptr;
        Scope(tkv_engine* eng, int c, int n_launch) : e(eng), cls(c) {
            e->launches += n_launch;
            tl_set_class(c);
            if (e->prof_on) {
                a = e->take_event();
                cudaEventRecord(a, e->stream);
            }
        }
        ~Scope() {
            tl_set_class(PC_OTHER);
            if (a) {
                cudaEvent_t b = e->take_event();
                cudaEventRecord(b, e->stream);
                e->recs.push_back({cls, a, b});
            }
        }
    };
    void prof_flush() {
        if (recs.empty()) return;
        TKV_CUDA(cudaStreamSynchronize(stream));
        for (auto& r : recs) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            prof_ms[r.cls] += ms;
            prof_n[r.cls] += 1;
            ev_pool.push_back(r.a);
            ev_pool.push_back(r.b);
        }
        recs.clear();
    }

    // ---- helpers ----
    void sync() { TKV_CUDA(cudaStreamSynchronize(stream)); }
    // copy host data into the current staging slot at `off` and enqueue its H2D copy
    int64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device bytes moved by the request path (bench e2e accounting)
    void upload(uint8_t* slot, void* dst, const void* src, size_t bytes, size_t off) {
        if (bytes == 0) return;
        h2d_bytes += (int64_t)bytes;
        std::memcpy(slot + off, src, bytes);
        TKV_CUDA(cudaMemcpyAsync(dst, slot + off, bytes, cudaMemcpyHostToDevice, stream));
    }
    void ensure_rope(int64_t max_pos) {
        if (max_pos < rope_len) return;
        int64_t n = std::max<int64_t>(rope_len ? rope_len * 2 : 4096, max_pos + 1);
        n = std::max(n, opts.max_position > 0 ? opts.max_position : (int64_t)32768);
        const int64_t half = d / 2;
        std::vector<double> theta(half);
        for (int64_t m = 0; m < half; ++m) theta[m] = std::pow(cfg.rope_base, -2.0 * (double)m / (double)d);
        std::vector<float> tab((size_t)(n * half * 2));
        for (int64_t t = 0; t < n; ++t)
            for (int64_t m = 0; m < half; ++m) {
                const double a = (double)t * theta[m];
                tab[(size_t)((t * half + m) * 2)] = (float)std::cos(a);
                tab[(size_t)((t * half + m) * 2 + 1)] = (float)std::sin(a);
            }
        sync();
        DevMem fresh;
        fresh.ensure(tab.size() * sizeof(float));
        TKV_CUDA(cudaMemcpy(fresh.p, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice));
        std::swap(rope.p, fresh.p);
        std::swap(rope.n, fresh.n);
        rope_len = n;
    }

    void* ctx_alloc(size_t bytes, size_t* got) {
        size_t best = (size_t)-1;
        int bi = -1;
        for (size_t i = 0; i < ctx_free.size(); ++i)
            if (ctx_free[i].first >= bytes && ctx_free[i].first < best) {
                best = ctx_free[i].first;
                bi = (int)i;
            }
        if (bi >= 0 && best <= bytes * 4 + (64u << 20)) {
            void* p = ctx_free[bi].second;
            *got = ctx_free[bi].first;
            ctx_free.erase(ctx_free.begin() + bi);
            return p;
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess && !ctx_free.empty()) {  // trim the cache and retry
            cudaGetLastError();
            sync();
            for (auto& f : ctx_free) cudaFree(f.second);
    if (host_pool) cudaFreeHost(host_pool);
            ctx_free.clear();
            e = cudaMalloc(&p, bytes);
        }
        TKV_CUDA(e);
        *got = bytes;
        return p;
    }
    void ctx_release(void* p, size_t bytes) {
        if (p) ctx_free.emplace_back(bytes, p);
    }

    // L2 warm-up of the O-proj weights and the head of gate/up, issued by each attention CTA once its K/V loads are
    // out (query-prefill forwards): C2 step 3.60 -> 3.54 ms at 40 MB (26 / 64 MB: 3.55 / 3.54, attention slower at 64)
    size_t l2_prefetch_bytes = (size_t)40 << 20;  // TKV_L2_PREFETCH_MB (tuning knob)
    int skip_mask = 0;             // TKV_TIMING_SKIP: drop kernels for cost attribution (results invalid)
    int trace_layer = -1;          // TKV_TRACE_LAYER: clock64 pipeline trace of that layer's attention launch
    int attn_split_override = 0;   // TKV_ATTN_SPLITS: force the tcgen05 attention's split-K count
    int64_t decode_rows_max = 0;   // TKV_DECODE_ROWS: (rows x group) at or below which attention runs SIMT
                                   // (measured slower than tcgen05 even for one row: default off)

    int pick_splits(int M, int N, int K, bool tc) const {
        const int bk = tc ? 64 : 16;
        const int tiles = tc ? gemm_tc_tiles(M, N) : ((M + 63) / 64) * ((N + 63) / 64);
        const int kb = (K + bk - 1) / bk;
        // tcgen05: gemm_tc_ctas_per_sm() persistent CTAs per SM; round DOWN so splits x tiles fills one wave of
        // them (every resident CTA streams weights; at 1 unit per SM half the CTA slots idled)
        int s = tc ? num_sms * gemm_tc_ctas_per_sm(M) / tiles : (num_sms + tiles - 1) / tiles;
        s = std::min(s, std::max(1, kb / 4));
        s = std::min(s, 16);
        s = std::max(s, 1);
        const int kbs = (kb + s - 1) / s;
        return (kb + kbs - 1) / kbs;
    }

    bool use_tc() const { return dt == DT::BF16 && !(opts.flags & TKV_FLAG_SIMT_GEMM); }

#ifndef TKV_BATCH_SPLITS_DEFAULT
#define TKV_BATCH_SPLITS_DEFAULT 0
#endif
    // TKV_BATCH_ATTN_SPLITS (0 = attn_tc_batch_pick_splits: fill the last wave; C3 attention 21.1 -> 19.3 ms at 2)
    int batch_attn_splits = TKV_BATCH_SPLITS_DEFAULT;
    // kernel timeline buffer (tkv_kernel_timeline): [kTlMax][2] globaltimer (first CTA past the wait, last warp done)
    static constexpr int64_t kTlMax = 8192;
    DevMem tl_buf;

    // partial[splits][M][N] = A[M][lda] . W[N][K]^T ; returns splits. With swiglu_act, a tcgen05 GEMM whose
    // K range fits one CTA writes silu(gate)*up straight to swiglu_act and returns 0.
    int gemm(const void* A, int lda, const void* W, int M, int N, int K, void* swiglu_act = nullptr) {
        const int nb = norm_blocks((int)hid);
        const bool tc = use_tc();
        if (tc && !gemm_tc_supported(M, N, K, lda))
            fail(TKV_ERR_CONFIG, "shape not supported by the tcgen05 GEMM (rows must be 16-byte aligned)");
        const int s = pick_splits(M, N, K, tc);
        Scope sc(this, PC_GEMM, 1);
        if (tc && swiglu_act && s == 1 && gu_interleaved) {
            launch_gemm_tc(A, lda, W, M, N, K, nullptr, 1, stream, swiglu_act, ssp.as<float>(), nb, (float)cfg.norm_eps,
                           gu_block);
            return 0;
        }
        partial.ensure((size_t)s * M * N * sizeof(float));
        if (tc) return launch_gemm_tc(A, lda, W, M, N, K, partial.as<float>(), s, stream);
        launch_gemm_simt(A, lda, W, M, N, K, partial.as<float>(), s, dt, stream);
        return s;
    }

    void* kv_plane(tkv_context* c, int64_t layer, int kv) const;

    struct Fwd {
        const int32_t* tok = nullptr;  // device [T]
        int T = 0;
        const int32_t* pos = nullptr;  // device [T]
        tkv_context* ctx = nullptr;
        int row0 = 0;                 // cache rows of the new tokens start here
        const int32_t* lo = nullptr;  // device [T]
        const int32_t* hi = nullptr;
        bool logits = true;   // last-row logits into this->logits
        bool kv_only = false; // chunk ingest: stop after the last layer's QKV
        StoreScatter sc{};
        // batched query prefill (tkv_prefill_query_batch): request r owns tokens [tok0, tok0 + n) of this forward,
        // its K/V go to its own context at rows [row0, row0 + n); logits of its last token -> logits[r]
        struct Req {
            tkv_context* ctx;
            int tok0, n, row0;
        };
        std::vector<Req> reqs;
        const AttnReq* batch_reqs = nullptr;  // device request table + cache maps of the batched attention
        const void* batch_maps = nullptr;
        int batch_max_n = 0;
        int batch_min_keys = 0;  // shortest request context (keys) of the batched attention
        const EpiReq* epi_reqs = nullptr;  // device table of the batched QKV epilogue (one launch per layer)
    };
    void forward(const Fwd& f);
    // CUDA-graph replay of the query-prefill forward (extend): the second forward with the same key (context cache,
    // row offset, token count, input / staging / output buffers, RoPE table, buffer generation) is captured with its
    // PDL edges, later ones replay the graph (launch handoffs 0.90 -> 0.61 us in tools/micro/pdl_gap.cu).
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
    };
    std::map<std::vector<uint64_t>, GraphEntry> graphs;
    std::set<std::vector<uint64_t>> graph_seen;
    bool graphs_ok = true;
    void forward_graph(const Fwd& f);
    void attend_layer(int64_t l, int T, const void* qrows, tkv_context* actx, const int32_t* lo, const int32_t* hi,
                      void* out, int arows, int aTk, int kv_ready);
    void check_err(const char* where);
};

struct tkv_context {
    tkv_engine* eng = nullptr;
    void* kv = nullptr;
    size_t kv_bytes = 0;
    int64_t cap = 0;
    int64_t total = 0;
    std::vector<int64_t> positions;
    std::vector<int64_t> seg_len;
    std::vector<int32_t> seg_query;
    int mask_mode = TKV_MASK_INDEPENDENT;
    int64_t next_position = 0;
    std::vector<float> last_logits;
    // injected chunk rows [0, chunk_rows): where they came from (unrotated export re-gathers them)
    std::vector<GatherSeg> chunk_segs;
    uint64_t store_epoch = 0;  // engine store epoch when chunk_segs were taken
    int64_t chunk_rows = 0;
    // predicate of the last forward over this context
    std::vector<int32_t> last_lo, last_hi;
    int64_t last_rows = 0, last_cols = 0;

    void extend_query_segment(int64_t n) {  // context.cpp:24-35
        if (!seg_len.empty() && seg_query.back()) {
            seg_len.back() += n;
        } else {
            seg_len.push_back(n);
            seg_query.push_back(1);
        }
    }
};

void* tkv_engine::kv_plane(tkv_context* c, int64_t layer, int kv) const {
    return static_cast<uint8_t*>(c->kv) + (size_t)((layer * 2 + kv) * c->cap) * kvd * dt_size(dt);
}

tkv_engine::~tkv_engine() {
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (tkv_context* c : live) {
        c->eng = nullptr;
        if (c->kv) cudaFree(c->kv);
        c->kv = nullptr;
    }
    for (auto& f : ctx_free) cudaFree(f.second);
    for (auto& r : recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
    if (stream) cudaStreamDestroy(stream);
}

void tkv_engine::check_err(const char* where) {
    int e = 0;
    TKV_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    d2h_bytes += sizeof(int);
    sync();
    if (e == 0) return;
    TKV_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
    if (e & 1) fail(TKV_ERR_DOMAIN, std::string(where) + ": token id outside vocab");
    if (e & 8) fail(TKV_ERR_DEGENERATE_ROW, std::string(where) + ": softmax row has no attendable positions");
    fail(TKV_ERR_DOMAIN, std::string(where) + ": non-finite element");
}

void tkv_engine::attend_layer(int64_t l, int T, const void* qrows, tkv_context* actx, const int32_t* lo,
                              const int32_t* hi, void* out, int arows, int aTk, int kv_ready) {
    const size_t es = dt_size(dt);
    // decode-sized row counts (the last layer's single row, greedy decode) can run the split-K mma.sync
    // kernel (opt-in: measured on par with the 1/8-full tcgen05 tile at C2, 2 % slower per decode step)
    const bool tiny = (int64_t)arows * (H / Hkv) <= decode_rows_max;
    const bool dec = dt == DT::BF16 && (opts.flags & TKV_FLAG_DECODE_ATTN) && !(opts.flags & TKV_FLAG_SIMT_ATTN) &&
                     attention_decode_supported(arows, (int)H, (int)Hkv, (int)d, dt);
    const bool tc = dt == DT::BF16 && !(opts.flags & TKV_FLAG_SIMT_ATTN) && !tiny && !dec &&
                    attention_tc_supported((int)d, dt);
    int splits = tc ? attn_tc_pick_splits(arows, (int)H, (int)Hkv, aTk, num_sms)
                    : dec ? attn_decode_pick_splits(aTk, (int)Hkv, num_sms)
                          : attn_pick_splits(arows, (int)H, (int)Hkv, aTk, num_sms);
    if (tc && attn_split_override > 0) splits = attn_split_override;  // TKV_ATTN_SPLITS (tuning)
    AttnWork ws;
    if (splits > 1) {
        size_t mloff = (size_t)splits * arows * H * d;
        const size_t fl = tc ? attn_tc_workspace_floats(arows, (int)H, (int)Hkv, splits, &mloff)
                             : attn_workspace_floats(arows, (int)H, (int)d, splits);
        attn_ws.ensure(fl * sizeof(float));
        ws.o = attn_ws.as<float>();
        ws.ml = ws.o + mloff;
    }
    Scope sc(this, PC_ATTN, splits > 1 ? 2 : 1);  // + the split-merge launch
    if (skip_mask & 8) {
    } else if (dec) {
        launch_attention_decode(qrows, kv_plane(actx, l, 0), kv_plane(actx, l, 1), (int)kvd, lo, hi, out, arows,
                                aTk, (int)H, (int)Hkv, splits, ws, err.as<int>(), stream);
    } else if (tc) {
        // Weight-bound small forwards: warm L2 with this layer's O-proj weights and the head of its
        // gate/up weights while attention runs (l2_prefetch_bytes total, 0 = off)
        L2Prefetch pf;
        if (T <= 128 && l2_prefetch_bytes > 0) {
            const size_t ob = (size_t)hid * qd * es, gb = (size_t)2 * I * hid * es;
            pf.ptr[0] = w_o[l];
            pf.bytes[0] = std::min(ob, l2_prefetch_bytes);
            pf.ptr[1] = w_gu[l];
            pf.bytes[1] = std::min(gb, l2_prefetch_bytes - pf.bytes[0]);
        }
        if (trace_layer == (int)l) attn_trace_enable(true, nullptr);
        launch_attention_tc(qrows, kv_plane(actx, l, 0), kv_plane(actx, l, 1), (int)kvd, lo, hi, out, arows,
                            aTk, (int)H, (int)Hkv, splits, ws, err.as<int>(), stream, kv_ready, pf);
        if (trace_layer == (int)l) attn_trace_enable(false, nullptr);
    } else {
        launch_attention_simt(qrows, kv_plane(actx, l, 0), kv_plane(actx, l, 1), (int)kvd, lo, hi, out, arows,
                              aTk, (int)H, (int)Hkv, (int)d, splits, ws, err.as<int>(), dt, stream);
    }
}

void tkv_engine::forward_graph(const Fwd& f) {
    const bool eligible = graphs_ok && !(opts.flags & TKV_FLAG_NO_GRAPHS) && !prof_on && trace_layer < 0 && !tl_armed() &&
                          f.reqs.empty() && !f.kv_only && !f.sc.page && f.ctx;
    if (!eligible) {
        forward(f);
        return;
    }
    const std::vector<uint64_t> key = {(uint64_t)(uintptr_t)f.ctx->kv, (uint64_t)f.ctx->cap, (uint64_t)f.row0,
                                       (uint64_t)f.T, (uint64_t)(uintptr_t)f.tok, (uint64_t)(uintptr_t)f.pos,
                                       (uint64_t)(uintptr_t)f.lo, (uint64_t)(uintptr_t)f.hi, (uint64_t)(uintptr_t)rope.p,
                                       (uint64_t)(uintptr_t)logits.p, DevMem::generation().load(), (uint64_t)f.logits};
    auto it = graphs.find(key);
    if (it != graphs.end()) {
        NvtxRange nvtx("forward (graph replay)");
        TKV_CUDA(cudaGraphLaunch(it->second.exec, stream));
        launches += it->second.launches;
        return;
    }
    if (!graph_seen.count(key)) {  // first sighting: run it (sizes every buffer), capture on the next one
        if (graph_seen.size() >= 64) graph_seen.clear();
        graph_seen.insert(key);
        forward(f);
        return;
    }
    if (graphs.size() >= 16) {  // bounded cache
        for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
        graphs.clear();
    }
    const int64_t l0 = launches;
    TKV_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
        forward(f);
    } catch (...) {
        cudaGraph_t dropped = nullptr;
        cudaStreamEndCapture(stream, &dropped);
        if (dropped) cudaGraphDestroy(dropped);
        throw;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(stream, &g);
    cudaGraphExec_t ex = nullptr;
    if (ce != cudaSuccess || !g || cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {  // not capturable here: no graphs
        (void)cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        graphs_ok = false;
        launches = l0;
        forward(f);
        return;
    }
    cudaGraphDestroy(g);
    graphs[key] = GraphEntry{ex, launches - l0};
    TKV_CUDA(cudaGraphLaunch(ex, stream));
}

void tkv_engine::forward(const Fwd& f) {
    NvtxRange nvtx("forward");
    const int T = f.T, Tk = f.row0 + f.T;
    const bool batch = !f.reqs.empty();
    const size_t es = dt_size(dt);
    const float eps = (float)cfg.norm_eps;
    x.ensure((size_t)T * hid * 4);
    xb.ensure((size_t)T * hid * es);
    const int nb = norm_blocks((int)hid);
    ssp.ensure((size_t)T * nb * 4);
    q.ensure((size_t)T * qd * es);
    attn.ensure((size_t)T * qd * es);
    act.ensure((size_t)T * I * es);
    {
        Scope sc(this, PC_EPI, 1);
        launch_embed(f.tok, T, emb, (int)hid, (int)V, norm_attn(0), x.as<float>(), xb.p, ssp.as<float>(), dt, err.as<int>(),
                     stream);
    }
    for (int64_t l = 0; l < L; ++l) {
        NvtxRange nvtx_layer("layer");
        // --- attention block ---
        int s = gemm(xb.p, (int)hid, w_qkv[l], T, (int)nqkv, (int)hid);
        if (batch && f.epi_reqs) {  // every request's K/V to its own cache, one launch
            Scope sc(this, PC_EPI, 1);
            launch_qkv_epilogue(partial.as<float>(), s, T, (int)H, (int)Hkv, (int)d, f.pos, rope.as<float2>(), q.p,
                                nullptr, nullptr, 0, StoreScatter{}, (int)l, ssp.as<float>(), nb, (int)hid, eps, dt, stream,
                                (int64_t)T * nqkv, f.epi_reqs, (int)f.reqs.size());
        } else if (batch) {
            Scope sc(this, PC_EPI, (int)f.reqs.size());
            for (const Fwd::Req& r : f.reqs)
                launch_qkv_epilogue(partial.as<float>() + (size_t)r.tok0 * nqkv, s, r.n, (int)H, (int)Hkv, (int)d,
                                    f.pos + r.tok0, rope.as<float2>(), static_cast<uint8_t*>(q.p) + (size_t)r.tok0 * qd * es,
                                    kv_plane(r.ctx, l, 0), kv_plane(r.ctx, l, 1), r.row0, StoreScatter{}, (int)l,
                                    ssp.as<float>() + (size_t)r.tok0 * nb, nb, (int)hid, eps, dt, stream,
                                    (int64_t)T * nqkv);
        } else if (!(skip_mask & 4)) {
            Scope sc(this, PC_EPI, 1);
            launch_qkv_epilogue(partial.as<float>(), s, T, (int)H, (int)Hkv, (int)d, f.pos, rope.as<float2>(), q.p,
                                kv_plane(f.ctx, l, 0), kv_plane(f.ctx, l, 1), f.row0, f.sc, (int)l, ssp.as<float>(), nb,
                                (int)hid, eps, dt, stream);
        }
        if (f.kv_only && l == L - 1) break;
        // In the last layer only the final row feeds the logits: attention, O-proj and the MLP run on it alone.
        const bool tail = (l == L - 1) && f.logits && !batch;
        const int rows = tail ? 1 : T;
        const int64_t r0 = tail ? T - 1 : 0;
        auto attend = [&](const void* qrows, tkv_context* actx, const int32_t* lo, const int32_t* hi, void* out,
                          int arows, int aTk, int kv_ready) {
            attend_layer(l, T, qrows, actx, lo, hi, out, arows, aTk, kv_ready);
        };
        if (batch && f.batch_maps) {
            // one launch for the whole batch; split-K only to fill the last wave of (request, kv head, row group)
            // CTAs, merged by a request-aware combine
            const int n_req = (int)f.reqs.size();
            const int groups_x = (f.batch_max_n * (int)(H / Hkv) + kAttnTcRows - 1) / kAttnTcRows;
            int bs = batch_attn_splits > 0 ? batch_attn_splits
                                           : attn_tc_batch_pick_splits(groups_x * (int)Hkv * n_req, f.batch_min_keys,
                                                                       num_sms);
            AttnWork bws;
            if (bs > 1) {
                const size_t rows = (size_t)bs * groups_x * Hkv * n_req * kAttnTcRows;
                attn_ws.ensure((rows * d / 2 + rows * 2) * sizeof(float));
                bws.o = attn_ws.as<float>();
                bws.ml = bws.o + rows * d / 2;
            }
            Scope sc(this, PC_ATTN, bs > 1 ? 2 : 1);
            if (trace_layer == (int)l) attn_trace_enable(true, nullptr);
            launch_attention_tc_batch(q.p, f.batch_reqs, f.batch_maps, n_req, f.batch_max_n, (int)H, (int)Hkv, (int)l,
                                      f.lo, f.hi, attn.p, err.as<int>(), stream, bs, bws);
            if (trace_layer == (int)l) attn_trace_enable(false, nullptr);
        } else if (batch) {
            for (const Fwd::Req& r : f.reqs)
                attend(static_cast<uint8_t*>(q.p) + (size_t)r.tok0 * qd * es, r.ctx, f.lo + r.tok0, f.hi + r.tok0,
                       static_cast<uint8_t*>(attn.p) + (size_t)r.tok0 * qd * es, r.n, r.row0 + r.n, r.row0);
        } else {
            attend(static_cast<uint8_t*>(q.p) + (size_t)r0 * qd * es, f.ctx, f.lo + r0, f.hi + r0, attn.p, rows, Tk,
                   f.row0);
        }
        uint8_t* attn_rows = static_cast<uint8_t*>(attn.p);
        float* x_rows = x.as<float>() + r0 * hid;
        s = gemm(attn_rows, (int)qd, w_o[l], rows, (int)hid, (int)qd);
        if (!(skip_mask & 1)) {
            Scope sc(this, PC_EPI, 1);
            launch_residual(x_rows, partial.as<float>(), s, rows, (int)hid, norm_mlp(l), xb.p, ssp.as<float>(), dt,
                            err.as<int>(), stream);
        }
        // --- MLP block: gate|up fused into one GEMM, SwiGLU (with the folded mlp_norm scale) in its epilogue ---
        s = gemm(xb.p, (int)hid, w_gu[l], rows, (int)(2 * I), (int)hid, act.p);
        if (s > 0) {
            Scope sc(this, PC_EPI, 1);
            launch_swiglu(partial.as<float>(), s, rows, (int)I, act.p, ssp.as<float>(), nb, (int)hid, eps, dt,
                          stream, gu_block);
        }
        s = gemm(act.p, (int)I, w_down[l], rows, (int)hid, (int)I);
        if (!(skip_mask & 2)) {
            // residual + the next RMSNorm (next layer's attn_norm, or final_norm): all weights are 1.0
            Scope sc(this, PC_EPI, 1);
            launch_residual(x_rows, partial.as<float>(), s, rows, (int)hid, norm_after_mlp(l), xb.p, ssp.as<float>(), dt,
                            err.as<int>(), stream);
        }
    }
    if (f.logits && batch) {
        logits.ensure((size_t)f.reqs.size() * V * 4);
        Scope sc(this, PC_OTHER, (int)f.reqs.size());
        for (size_t i = 0; i < f.reqs.size(); ++i) {  // final_norm folded; the last token of each request
            const int last = f.reqs[i].tok0 + f.reqs[i].n - 1;
            launch_lm_head(static_cast<uint8_t*>(xb.p) + (size_t)last * hid * es, w_lm, (int)hid, (int)V,
                           logits.as<float>() + i * V, ssp.as<float>() + (size_t)last * nb, nb, eps, dt,
                           err.as<int>(), stream);
        }
    } else if (f.logits) {
        // after the tail layer, h row 0 holds final_norm(x) of the last token
        Scope sc(this, PC_OTHER, 1);
        launch_lm_head(xb.p, w_lm, (int)hid, (int)V, logits.as<float>(), ssp.as<float>(), nb, eps, dt, err.as<int>(),
                       stream);
    }
}

// ================================================================================================
// C ABI
// ================================================================================================
namespace {

template <typename F>
tkv_status guard(F&& fn) {
    try {
        fn();
        return TKV_OK;
    } catch (const Failure& f) {
        g_last_error = f.msg;
        return f.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host out of memory";
        return TKV_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TKV_ERR_GENERIC;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(TKV_ERR_DOMAIN, std::string(what) + " is null");
}

std::vector<int32_t> framed_of(const int32_t* payload, int64_t n) {  // tok::frame_chunk (tokenizer.cpp:36-43)
    std::vector<int32_t> v;
    v.reserve((size_t)n + 2);
    v.push_back(256);
    v.insert(v.end(), payload, payload + n);
    v.push_back(257);
    return v;
}

void check_tokens(const tkv_engine* e, const int32_t* t, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (t[i] < 0 || t[i] >= e->V)
            fail(TKV_ERR_DOMAIN, "token id " + std::to_string(t[i]) + " outside vocab");
}

void flops_add(const tkv_engine* e, tkv_flops* fl, int64_t tokens, int64_t context) {  // costmodel.cpp:77-83
    if (!fl) return;
    const uint64_t L = e->L, Hd = e->hid, H = e->H, Hkv = e->Hkv, d = e->d, I = e->I;
    fl->qkv += L * tokens * (2 * Hd * (H + 2 * Hkv) * d);
    fl->attn += L * tokens * (2 * H * d * (uint64_t)context);
    fl->o += L * tokens * (2 * Hd * Hd);
    fl->mlp += L * tokens * (6 * Hd * I);
}

tkv_context* new_context(tkv_engine* e, int64_t cap) {
    auto* c = new tkv_context;
    c->eng = e;
    c->cap = std::max<int64_t>(cap, 1);
    const size_t bytes = (size_t)(e->L * 2 * c->cap * e->kvd) * dt_size(e->dt);
    c->kv = e->ctx_alloc(bytes, &c->kv_bytes);
    e->live.insert(c);
    return c;
}

// grow the request cache to hold `need_rows` rows (copies the existing rows of every plane)
void ensure_cap(tkv_engine* e, tkv_context* c, int64_t need_rows) {
    if (need_rows <= c->cap) return;
    const int64_t ncap = std::max(need_rows, c->cap + c->cap / 2);
    size_t got = 0;
    const size_t es = dt_size(e->dt);
    void* nkv = e->ctx_alloc((size_t)(e->L * 2 * ncap * e->kvd) * es, &got);
    if (c->total > 0) {
        TKV_CUDA(cudaMemcpy2DAsync(nkv, (size_t)ncap * e->kvd * es, c->kv, (size_t)c->cap * e->kvd * es,
                                   (size_t)c->total * e->kvd * es, (size_t)(e->L * 2), cudaMemcpyDeviceToDevice,
                                   e->stream));
    }
    e->ctx_release(c->kv, c->kv_bytes);
    c->kv = nkv;
    c->kv_bytes = got;
    c->cap = ncap;
}

// staging layout for a forward's small per-token arrays
struct Stage {
    std::vector<int32_t> tok, pos, lo, hi, page, slot;
};

void upload_stage(tkv_engine* e, const Stage& s, bool with_tokens) {
    const int64_t T = (int64_t)s.pos.size();
    const size_t b = ((size_t)T * 4 + 15) & ~size_t(15);  // 16-byte aligned sections
    const int nsec = s.page.empty() ? 4 : 6;
    int32_t* base = static_cast<int32_t*>(e->d_stage.ensure(6 * b + 64));
    int32_t** ptrs[6] = {&e->p_tok, &e->p_pos, &e->p_lo, &e->p_hi, &e->p_page, &e->p_slot};
    for (int i = 0; i < 6; ++i) *ptrs[i] = base + i * (b / 4);
    uint8_t* slot = e->staging.begin(6 * b + 64);
    const std::vector<int32_t>* src[6] = {&s.tok, &s.pos, &s.lo, &s.hi, &s.page, &s.slot};
    for (int i = 0; i < nsec; ++i)
        if (i > 0 || with_tokens) std::memcpy(slot + i * b, src[i]->data(), (size_t)T * 4);
    const size_t first = with_tokens ? 0 : b;  // device tokens: the token section is not copied
    e->h2d_bytes += (int64_t)(nsec * b - first);
    TKV_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(base) + first, slot + first, nsec * b - first,
                             cudaMemcpyHostToDevice, e->stream));
    e->staging.end(e->stream);
}

void remember_mask(tkv_context* c, const Stage& s, int64_t cols) {
    c->last_lo = s.lo;
    c->last_hi = s.hi;
    c->last_rows = (int64_t)s.lo.size();
    c->last_cols = cols;
}

// prefill of `n` new tokens over everything the context already holds (prefill_query / decode step)
void extend(tkv_engine* e, tkv_context* c, const int32_t* host_tok, const int32_t* dev_tok, int64_t n,
            float* host_logits, float* dev_logits) {
    const int64_t P = c->total;
    ensure_cap(e, c, P + n);
    Stage s;
    s.pos.resize(n);
    s.lo.assign(n, 0);
    s.hi.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        s.pos[i] = (int32_t)(c->next_position + i);
        s.hi[i] = (int32_t)(P + i);  // causal_rows(n, P): all injected rows + causal query tail
    }
    e->ensure_rope(c->next_position + n);
    if (host_tok) s.tok.assign(host_tok, host_tok + n);
    upload_stage(e, s, host_tok != nullptr);
    tkv_engine::Fwd f;
    f.tok = host_tok ? e->p_tok : dev_tok;
    f.T = (int)n;
    f.pos = e->p_pos;
    f.ctx = c;
    f.row0 = (int)P;
    f.lo = e->p_lo;
    f.hi = e->p_hi;
    f.logits = true;
    e->forward_graph(f);
    if (dev_logits)
        TKV_CUDA(cudaMemcpyAsync(dev_logits, e->logits.p, e->V * 4, cudaMemcpyDeviceToDevice, e->stream));
    if (host_logits) {
        TKV_CUDA(cudaMemcpyAsync(host_logits, e->logits.p, e->V * 4, cudaMemcpyDeviceToHost, e->stream));
        e->d2h_bytes += e->V * 4;
        e->check_err("prefill");
    }
    remember_mask(c, s, P + n);
    for (int64_t i = 0; i < n; ++i) c->positions.push_back(c->next_position + i);
    c->total = P + n;
    c->extend_query_segment(n);
    c->next_position += n;
    // device-only calls leave no host logits: a later greedy_decode fails cleanly instead of decoding from the
    // logits of an earlier prefill (its device errors surface at tkv_engine_check)
    if (host_logits) c->last_logits.assign(host_logits, host_logits + e->V);
    else c->last_logits.clear();
}

tkv_context* assemble_impl(tkv_engine* e, const uint64_t* ids, int64_t n, int mode) {
    std::vector<const Chunk*> cs;
    int64_t P = 0, max_len = 0;
    for (int64_t i = 0; i < n; ++i) {
        auto it = e->chunks.find(ids[i]);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(ids[i]) + " not in store");
        it->second.hits += 1;  // access frequency for the HBM <-> host tier policy (tkv_store_rebalance)
        cs.push_back(&it->second);
        P += it->second.len;
        max_len = std::max(max_len, it->second.len);
    }
    tkv_context* c = new_context(e, P + 128);
    std::vector<GatherSeg> segs;
    int64_t running = 0;
    for (const Chunk* ch : cs) {
        const int64_t first = mode == TKV_POS_REORDERED ? running : 0;  // pipeline.cpp:150
        for (size_t p = 0; p < ch->pages.size(); ++p) {
            const int64_t off = (int64_t)p * e->page_tokens;
            GatherSeg g;
            g.src_page = ch->pages[p];
            g.n_tok = (int32_t)std::min<int64_t>(e->page_tokens, ch->len - off);
            g.dst_row = (int32_t)(running + off);
            g.pos0 = (int32_t)(first + off);
            g.pool = ch->slot;
            segs.push_back(g);
        }
        for (int64_t t = 0; t < ch->len; ++t) c->positions.push_back(first + t);
        c->seg_len.push_back(ch->len);
        c->seg_query.push_back(0);
        running += ch->len;
    }
    c->total = P;
    c->chunk_rows = P;
    c->chunk_segs = segs;
    c->store_epoch = e->store_epoch;
    c->next_position = mode == TKV_POS_REORDERED ? running : max_len;  // pipeline.cpp:160-162
    c->mask_mode = TKV_MASK_INDEPENDENT;
    if (!segs.empty()) {
        e->ensure_rope(std::max(P, max_len));
        const size_t b = segs.size() * sizeof(GatherSeg);
        e->d_segs.ensure(b);
        uint8_t* slot = e->staging.begin(b);
        e->upload(slot, e->d_segs.p, segs.data(), b, 0);
        e->staging.end(e->stream);
        tkv_engine::Scope sc(e, PC_GATHER, 1);
        for (const Chunk* ch : cs)
            if (ch->slot) e->remote_bytes += ch->len * e->L * 2 * e->kvd * (int64_t)dt_size(e->dt);
        launch_gather_rope(e->pools, (int)e->page_tokens, e->d_segs.as<GatherSeg>(), (int)segs.size(), (int)e->L,
                           (int)e->kvd, (int)e->d, e->rope.as<float2>(), c->kv, c->cap, 1, e->dt, e->num_sms,
                           e->stream);
    }
    return c;
}

void naive_impl(tkv_engine* e, const int32_t* framed, const int64_t* offsets, int64_t n_chunks, const int32_t* query,
                int64_t nq, int mode, float* logits_out, tkv_flops* fl, tkv_context** ctx_out) {
    if (nq <= 0) fail(TKV_ERR_DOMAIN, "naive_prefill: empty query");
    need(query, "query");
    Stage s;
    std::vector<int64_t> lens;
    for (int64_t c = 0; c < n_chunks; ++c) {
        const int64_t len = offsets[c + 1] - offsets[c];
        if (len < 1) fail(TKV_ERR_DOMAIN, "naive_prefill: empty chunk");
        lens.push_back(len);
        s.tok.insert(s.tok.end(), framed + offsets[c], framed + offsets[c + 1]);
    }
    s.tok.insert(s.tok.end(), query, query + nq);
    check_tokens(e, s.tok.data(), (int64_t)s.tok.size());
    const int64_t N = (int64_t)s.tok.size();
    s.pos.resize(N);
    s.lo.resize(N);
    s.hi.resize(N);
    int64_t off = 0;
    for (int64_t c = 0; c <= n_chunks; ++c) {  // build_mask (attention.cpp:50-78) as row ranges
        const int64_t len = c < n_chunks ? lens[c] : nq;
        const bool is_query = c == n_chunks;
        for (int64_t i = off; i < off + len; ++i) {
            s.pos[i] = (int32_t)i;
            s.lo[i] = (mode == TKV_MASK_INDEPENDENT && !is_query) ? (int32_t)off : 0;
            s.hi[i] = (int32_t)i;
        }
        off += len;
    }
    for (const auto& o : e->mask_override) {  // testing::mask_fault_hook (pipeline.cpp:215)
        const int64_t r = o[0] < 0 ? N + o[0] : o[0];
        if (r < 0 || r >= N) continue;
        if (o[1] == -2) {  // tkv_debug_set_mask_fault: widen the row down to column o[2]
            s.lo[r] = (int32_t)std::min<int64_t>(s.lo[r], o[2]);
            continue;
        }
        if (o[1] < 0 || o[2] >= N || o[1] > o[2]) fail(TKV_ERR_DOMAIN, "mask override: range outside the sequence");
        s.lo[r] = (int32_t)o[1];
        s.hi[r] = (int32_t)o[2];
    }
    e->mask_override.clear();
    tkv_context* c = new_context(e, N);
    try {
        e->ensure_rope(N);
        upload_stage(e, s, true);
        tkv_engine::Fwd f;
        f.tok = e->p_tok;
        f.T = (int)N;
        f.pos = e->p_pos;
        f.ctx = c;
        f.row0 = 0;
        f.lo = e->p_lo;
        f.hi = e->p_hi;
        f.logits = true;
        e->forward(f);
        std::vector<float> lg((size_t)e->V);
        TKV_CUDA(cudaMemcpyAsync(lg.data(), e->logits.p, e->V * 4, cudaMemcpyDeviceToHost, e->stream));
        e->check_err("naive_prefill");
        if (logits_out) std::memcpy(logits_out, lg.data(), lg.size() * 4);
        c->total = N;
        for (int64_t i = 0; i < N; ++i) c->positions.push_back(i);
        c->seg_len = lens;
        c->seg_query.assign(lens.size(), 0);
        c->seg_len.push_back(nq);
        c->seg_query.push_back(1);
        c->next_position = N;
        c->mask_mode = mode;
        c->last_logits = lg;
        remember_mask(c, s, N);
        flops_add(e, fl, N, N);
    } catch (...) {
        tkv_context_destroy(c);
        throw;
    }
    if (ctx_out)
        *ctx_out = c;
    else
        tkv_context_destroy(c);
}

// Page placement: HBM while it has room for the whole chunk, else the pinned host spill tier (a chunk lives in one tier).
void store_chunk_pages(tkv_engine* e, Chunk& ch) {
    const int64_t np = (ch.len + e->page_tokens - 1) / e->page_tokens;
    std::vector<int32_t>* fl = &e->free_pages;
    ch.slot = 0;
    if ((int64_t)fl->size() < np && (int64_t)e->host_free.size() >= np) {
        fl = &e->host_free;
        ch.slot = kHostPool;
    }
    if ((int64_t)fl->size() < np)
        fail(TKV_ERR_OOM, "KV store full: need " + std::to_string(np) + " pages, " +
                              std::to_string(e->free_pages.size()) + " free in HBM, " +
                              std::to_string(e->host_free.size()) + " in the host tier");
    for (int64_t p = 0; p < np; ++p) {
        ch.pages.push_back(fl->back());
        fl->pop_back();
    }
}

void release_chunk_pages(tkv_engine* e, const Chunk& ch) {
    if (ch.slot == 0)
        e->free_pages.insert(e->free_pages.end(), ch.pages.begin(), ch.pages.end());
    else if (ch.slot == kHostPool)
        e->host_free.insert(e->host_free.end(), ch.pages.begin(), ch.pages.end());
    // peer-registered chunks do not own pages here
}

uint8_t* page_ptr(tkv_engine* e, int slot, int32_t page) {
    return static_cast<uint8_t*>(const_cast<void*>(e->pools.p[slot])) + (size_t)page * e->page_bytes;
}

}  // namespace

void tkv_engine::index_add(uint64_t id, const int32_t* payload, int64_t n, bool* added) {
    if (idx_row.count(id)) {  // content dedup (RetrievalIndex::add returns false)
        if (added) *added = false;
        return;
    }
    std::vector<double> e(kIndexDim);
    embed_tokens(payload, n, kIndexDim, e.data());
    const int64_t r = (int64_t)idx_ids.size();
    if (r >= idx_cap) {  // grow: copy the transposed matrix into a wider one
        const int64_t ncap = std::max<int64_t>(1024, 2 * idx_cap);
        DevMem ne, nn, ni;
        ne.ensure((size_t)kIndexDim * ncap * 8);
        nn.ensure((size_t)ncap * 8);
        ni.ensure((size_t)ncap * 8);
        if (r > 0) {
            TKV_CUDA(cudaMemcpy2DAsync(ne.p, (size_t)ncap * 8, d_idx_emb.p, (size_t)idx_cap * 8, (size_t)r * 8, kIndexDim,
                                       cudaMemcpyDeviceToDevice, stream));
            TKV_CUDA(cudaMemcpyAsync(nn.p, d_idx_nb.p, (size_t)r * 8, cudaMemcpyDeviceToDevice, stream));
            TKV_CUDA(cudaMemcpyAsync(ni.p, d_idx_ids.p, (size_t)r * 8, cudaMemcpyDeviceToDevice, stream));
        }
        sync();
        std::swap(d_idx_emb.p, ne.p);
        std::swap(d_idx_emb.n, ne.n);
        std::swap(d_idx_nb.p, nn.p);
        std::swap(d_idx_nb.n, nn.n);
        std::swap(d_idx_ids.p, ni.p);
        std::swap(d_idx_ids.n, ni.n);
        idx_cap = ncap;
    }
    const double nb = sumsq(e.data(), kIndexDim);
    TKV_CUDA(cudaMemcpy2DAsync(static_cast<double*>(d_idx_emb.p) + r, (size_t)idx_cap * 8, e.data(), 8, 8, kIndexDim,
                               cudaMemcpyHostToDevice, stream));
    TKV_CUDA(cudaMemcpyAsync(static_cast<double*>(d_idx_nb.p) + r, &nb, 8, cudaMemcpyHostToDevice, stream));
    TKV_CUDA(cudaMemcpyAsync(static_cast<uint64_t*>(d_idx_ids.p) + r, &id, 8, cudaMemcpyHostToDevice, stream));
    sync();
    idx_row[id] = r;
    idx_ids.push_back(id);
    idx_nb.push_back(nb);
    if (added) *added = true;
}

extern "C" {

int tkv_abi_version(void) { return TKV_ABI_VERSION; }

tkv_status tkv_embed(const int32_t* tokens, int64_t n, int64_t dim, double* out) {
    return guard([&] {
        if (n > 0) need(tokens, "tokens");
        need(out, "out");
        embed_tokens(tokens, n, dim, out);
    });
}

tkv_status tkv_index_add(tkv_engine* e, uint64_t chunk_id, const int32_t* payload, int64_t n, int* added) {
    return guard([&] {
        need(e, "engine");
        if (n > 0) need(payload, "payload");
        e->bind();
        bool a = false;
        e->index_add(chunk_id, payload, n, &a);
        if (added) *added = a ? 1 : 0;
    });
}

int64_t tkv_index_size(const tkv_engine* e) { return e ? (int64_t)e->idx_ids.size() : -1; }

tkv_status tkv_index_top_k(tkv_engine* e, const int32_t* query, int64_t n, int64_t k, uint64_t* ids_out,
                           double* scores_out, int64_t* n_out) {
    return guard([&] {
        need(e, "engine");
        need(ids_out, "ids_out");
        if (k < 1) fail(TKV_ERR_DOMAIN, "top_k: k must be >= 1");      // retrieval.cpp:119
        if (e->idx_ids.empty()) fail(TKV_ERR_DOMAIN, "top_k: empty index");  // retrieval.cpp:120
        if (n > 0) need(query, "query");
        std::vector<double> q(kIndexDim);
        embed_tokens(query, n, kIndexDim, q.data());
        const double na = sumsq(q.data(), kIndexDim);
        e->bind();
        const int64_t rows = (int64_t)e->idx_ids.size();
        const int kk = (int)std::min<int64_t>(k, std::min<int64_t>(rows, kIndexMaxK));
        if (k > kIndexMaxK && rows > kIndexMaxK) fail(TKV_ERR_CONFIG, "top_k: k > 256 over a larger index is not supported");
        e->d_idx_q.ensure((size_t)kIndexDim * 8);
        TKV_CUDA(cudaMemcpyAsync(e->d_idx_q.p, q.data(), (size_t)kIndexDim * 8, cudaMemcpyHostToDevice, e->stream));
        e->d_idx_scratch.ensure(index_topk_scratch_bytes(rows, kk));
        const int64_t got = launch_index_top_k(e->d_idx_emb.as<double>(), e->d_idx_nb.as<double>(),
                                               static_cast<const uint64_t*>(e->d_idx_ids.p), rows, e->idx_cap,
                                               e->d_idx_q.as<double>(), na, kk, e->d_idx_scratch.p, ids_out, scores_out,
                                               e->stream);
        if (n_out) *n_out = got;
    });
}
const char* tkv_last_error(void) { return g_last_error.c_str(); }

const char* tkv_status_name(tkv_status s) {
    static const char* names[] = {"ok",          "error",       "shape",     "domain",      "config",
                                  "degenerate_row", "io",       "format",    "not_found",   "stale_cache",
                                  "no_context",  "cuda",        "oom"};
    return (s >= 0 && s <= 12) ? names[s] : "unknown";
}

tkv_status tkv_config_preset(const char* name, tkv_model_config* out) {
    return guard([&] {
        need(name, "name");
        need(out, "out");
        tkv_model_config c{};
        c.rope_base = 10000.0;
        c.norm_eps = 1e-6;
        c.vocab_size = 259;
        const std::string n = name;
        if (n == "toy") {  // config.cpp:44-54
            c.layer_num = 4, c.head_num = 8, c.kv_head_num = 2, c.head_size = 8, c.hidden_size = 64,
            c.intermediate_size = 192;
        } else if (n == "qwen2-7b") {  // config.cpp:56-66
            c.layer_num = 28, c.head_num = 28, c.kv_head_num = 4, c.head_size = 128, c.hidden_size = 3584,
            c.intermediate_size = 18944;
        } else if (n == "llama3-8b") {  // BASELINE.json configs[3] (vocab kept at 259 for parity)
            c.layer_num = 32, c.head_num = 32, c.kv_head_num = 8, c.head_size = 128, c.hidden_size = 4096,
            c.intermediate_size = 14336, c.rope_base = 500000.0, c.norm_eps = 1e-5;
        } else {
            fail(TKV_ERR_CONFIG, "unknown preset '" + n + "' (expected 'toy', 'qwen2-7b' or 'llama3-8b')");
        }
        *out = c;
    });
}

tkv_status tkv_config_validate(const tkv_model_config* cfg) {
    return guard([&] {
        need(cfg, "cfg");
        validate_cfg(*cfg);
    });
}

uint64_t tkv_config_fingerprint_seed(const tkv_model_config* cfg) { return cfg ? fp_seed(*cfg) : 0; }

tkv_status tkv_weights_identity(const tkv_model_config* cfg, uint64_t seed, uint64_t* checksum,
                                uint64_t* fingerprint) {
    return guard([&] {
        need(cfg, "cfg");
        validate_cfg(*cfg);
        const uint64_t ck = weights_checksum_stream(*cfg, seed);
        if (checksum) *checksum = ck;
        if (fingerprint) *fingerprint = fingerprint_of(*cfg, ck);
    });
}

uint64_t tkv_chunk_content_id(uint64_t fp, const int32_t* framed, int64_t n) { return content_id(fp, framed, n); }

void tkv_engine_opts_default(tkv_engine_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->dtype = TKV_DTYPE_BF16;
    o->device = 0;
    o->page_tokens = 64;
    o->store_capacity_tokens = 0;
    o->max_position = 0;
    o->exact_fingerprint = -1;
    o->flags = 0;
}

}  // extern "C"
namespace {
struct WeightsFile;  // a TKVW file positioned after its header (tkv_engine_create_from_weights)
void load_tkvw(tkv_engine* e, WeightsFile& wf);
}  // namespace
extern "C" {

static tkv_status create_engine(const tkv_model_config* cfg, uint64_t seed, const tkv_engine_opts* opts, tkv_engine** out,
                                WeightsFile* wf) {
    std::unique_ptr<tkv_engine> e;
    tkv_status st = guard([&] {
        need(cfg, "cfg");
        need(out, "out");
        validate_cfg(*cfg);
        if (cfg->vocab_size < 259) fail(TKV_ERR_CONFIG, "vocab_size must cover the byte tokenizer (>= 259)");
        e.reset(new tkv_engine);
        e->cfg = *cfg;
        e->seed = seed;
        tkv_engine_opts_default(&e->opts);
        if (opts) e->opts = *opts;
        if (e->opts.dtype != TKV_DTYPE_F32 && e->opts.dtype != TKV_DTYPE_BF16) fail(TKV_ERR_CONFIG, "unknown dtype");
        if (e->opts.page_tokens < 1) e->opts.page_tokens = 64;
        e->dt = e->opts.dtype == TKV_DTYPE_F32 ? DT::F32 : DT::BF16;
        e->device = e->opts.device;
        set_pdl_enabled(!(e->opts.flags & TKV_FLAG_NO_PDL));

        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            fail(TKV_ERR_CUDA, "no CUDA device: the engine has no CPU fallback");
        }
        if (e->device < 0 || e->device >= ndev) fail(TKV_ERR_CUDA, "device ordinal out of range");
        e->bind();
        cudaDeviceProp prop;
        TKV_CUDA(cudaGetDeviceProperties(&prop, e->device));
        if (prop.major != 10) fail(TKV_ERR_CUDA, std::string("requires an sm_100 GPU (B200), found ") + prop.name);
        e->num_sms = prop.multiProcessorCount;
        TKV_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));

        const tkv_model_config& c = *cfg;
        e->L = c.layer_num, e->H = c.head_num, e->Hkv = c.kv_head_num, e->d = c.head_size, e->hid = c.hidden_size;
        e->I = c.intermediate_size, e->V = c.vocab_size, e->qd = e->H * e->d, e->kvd = e->Hkv * e->d;
        e->nqkv = e->qd + 2 * e->kvd;
        e->gu_block = e->I % 128 == 0 ? 128 : e->I % 64 == 0 ? 64 : 0;
        e->gu_interleaved = e->gu_block > 0;
        if (e->d != 8 && e->d != 16 && e->d != 32 && e->d != 64 && e->d != 128)
            fail(TKV_ERR_CONFIG, "head_size must be one of 8/16/32/64/128 for the device kernels");

        // ---- identity chain ----
        // reference-exact at every size: the FNV-1a of all f64 weights, hashed in parallel on the device
        // (fingerprint.cu; 52 GB of hashed bytes for Qwen2-7B); exact_fingerprint = 0 opts into a fast
        // non-reference identity
        e->exact_fp = e->opts.exact_fingerprint != 0 || wf;
        if (wf) {
            // fingerprint from the file's own weights: set by load_tkvw below
        } else if (e->exact_fp) {
            e->fingerprint = fingerprint_of(c, weights_checksum_device(c, seed, e->stream));
        } else {  // opt-in fast identity: NOT the reference's
            Fnv f;
            f.u64(fp_seed(c));
            f.u64(seed);
            f.u64(0xFA57F1A9E4ULL);
            e->fingerprint = f.h;
        }

        // ---- weights (init_random draw order, model.cpp:68-92) ----
        const size_t es = dt_size(e->dt);
        const int64_t H_ = e->hid, qd = e->qd, kvd = e->kvd, I = e->I, V = e->V;
        const size_t per_layer = (size_t)(e->nqkv * H_ + H_ * qd + 2 * I * H_ + H_ * I) * es;
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t emb_b = al((size_t)V * H_ * 4), ones_b = al((size_t)std::max(H_, I) * 4);
        const size_t norms_b = al((size_t)(2 * e->L + 1) * H_ * 4);
        const size_t lm_b = al((size_t)V * H_ * es);
        const size_t total_b = emb_b + ones_b + norms_b + lm_b + e->L * al(per_layer);
        uint8_t* base = static_cast<uint8_t*>(e->wmem.ensure(total_b));
        e->emb = reinterpret_cast<float*>(base);
        e->ones = reinterpret_cast<float*>(base + emb_b);
        e->norms = reinterpret_cast<float*>(base + emb_b + ones_b);
        e->w_lm = base + emb_b + ones_b + norms_b;
        uint8_t* lp = base + emb_b + ones_b + norms_b + lm_b;
        const double scale = 1.0 / std::sqrt((double)H_);
        uint64_t cur = 0;
        for (int64_t l = 0; l < e->L; ++l) {
            uint8_t* qkv = lp;
            e->w_qkv.push_back(qkv);
            e->w_o.push_back(qkv + (size_t)e->nqkv * H_ * es);
            e->w_gu.push_back(qkv + (size_t)e->nqkv * H_ * es + (size_t)H_ * qd * es);
            e->w_down.push_back(qkv + (size_t)e->nqkv * H_ * es + (size_t)H_ * qd * es + (size_t)2 * I * H_ * es);
            lp += al(per_layer);
        }
        launch_fill_f32(e->ones, 1.0f, std::max(H_, I), e->stream);
        if (wf) {
            load_tkvw(e.get(), *wf);  // weights, norms and the reference identity from the file
        } else {
        launch_fill_f32(e->norms, 1.0f, (2 * e->L + 1) * H_, e->stream);  // init_random: every norm weight is 1.0
        launch_init_rowmajor_f32(e->emb, seed, cur, V, H_, scale, e->stream);
        cur += (uint64_t)(V * H_);
        for (int64_t l = 0; l < e->L; ++l) {
            uint8_t* qkv = static_cast<uint8_t*>(e->w_qkv[l]);
            uint8_t* o = static_cast<uint8_t*>(e->w_o[l]);
            uint8_t* gu = static_cast<uint8_t*>(e->w_gu[l]);
            uint8_t* dn = static_cast<uint8_t*>(e->w_down[l]);
            // [in, out] draws written as [out][in] rows: wq | wk | wv stacked, gate | up stacked
            launch_init_transposed(qkv, e->dt, seed, cur, H_, qd, scale, e->stream);
            cur += (uint64_t)(H_ * qd);
            launch_init_transposed(qkv + (size_t)qd * H_ * es, e->dt, seed, cur, H_, kvd, scale, e->stream);
            cur += (uint64_t)(H_ * kvd);
            launch_init_transposed(qkv + (size_t)(qd + kvd) * H_ * es, e->dt, seed, cur, H_, kvd, scale, e->stream);
            cur += (uint64_t)(H_ * kvd);
            launch_init_transposed(o, e->dt, seed, cur, qd, H_, scale, e->stream);
            cur += (uint64_t)(qd * H_);
            // gate | up rows: interleaved in gu_block-row blocks (fused SwiGLU epilogue)
            const int rb = e->gu_block;
            launch_init_transposed(gu, e->dt, seed, cur, H_, I, scale, e->stream, rb, 0);
            cur += (uint64_t)(H_ * I);
            launch_init_transposed(rb ? gu : gu + (size_t)I * H_ * es, e->dt, seed, cur, H_, I, scale, e->stream, rb,
                                   rb);
            cur += (uint64_t)(H_ * I);
            launch_init_transposed(dn, e->dt, seed, cur, I, H_, scale, e->stream);
            cur += (uint64_t)(I * H_);
        }
        launch_init_transposed(e->w_lm, e->dt, seed, cur, H_, V, scale, e->stream);
        e->launches += 3 + 7 * e->L;
        }

        e->err.ensure(64);
#ifdef TKV_TUNING
        // Tuning / cost-attribution knobs (tools/*.sh). Compiled into TUNING builds only (make TUNING=1): several
        // of them skip work or change numerics, so the release library never reads them.
        if (const char* pfm = getenv("TKV_L2_PREFETCH_MB")) e->l2_prefetch_bytes = (size_t)atol(pfm) << 20;
        if (const char* sk = getenv("TKV_TIMING_SKIP")) e->skip_mask = atoi(sk);
        if (const char* tl = getenv("TKV_TRACE_LAYER")) e->trace_layer = atoi(tl);
        if (const char* as = getenv("TKV_ATTN_SPLITS")) e->attn_split_override = std::min(32, std::max(0, atoi(as)));
        if (const char* dr = getenv("TKV_DECODE_ROWS")) e->decode_rows_max = atol(dr);
        if (const char* mp = getenv("TKV_GEMM_NSMP")) set_gemm_nsmp(atoi(mp));
        if (const char* bs = getenv("TKV_BATCH_ATTN_SPLITS")) e->batch_attn_splits = std::min(32, std::max(0, atoi(bs)));
        if (const char* se = getenv("TKV_GEMM_SKIP_EPI")) set_gemm_skip_epi(atoi(se));
        if (const char* ra = getenv("TKV_GEMM_RASTER")) set_gemm_raster(atoi(ra));
        if (const char* gm = getenv("TKV_GEMM_GROUP_MB")) set_gemm_raster(1, atoi(gm));
        if (const char* gk = getenv("TKV_GEMM_KNOBS")) {  // "stages,smem_kb,ctas_per_sm,evict_first[,np[,pf]]"
            int st = 0, sm = 0, cps = 0, ef = 1, np = 0, pf = -1, kr = -1;
            if (sscanf(gk, "%d,%d,%d,%d,%d,%d,%d", &st, &sm, &cps, &ef, &np, &pf, &kr) >= 3)
                set_gemm_knobs(st, sm, cps, ef, np, pf, kr);
        }
#endif
        TKV_CUDA(cudaMemsetAsync(e->err.p, 0, 64, e->stream));
        e->logits.ensure((size_t)V * 4);
        e->ensure_rope(e->opts.max_position > 0 ? e->opts.max_position - 1 : 32767);

        // ---- paged KV store ----
        e->page_tokens = e->opts.page_tokens;
        e->page_bytes = (size_t)(e->L * 2 * e->page_tokens * e->kvd) * es;
        int64_t cap_tokens = e->opts.store_capacity_tokens;
        if (cap_tokens <= 0) {
            size_t fr = 0, tot = 0;
            TKV_CUDA(cudaMemGetInfo(&fr, &tot));
            const size_t tok_bytes = (size_t)(e->L * 2 * e->kvd) * es;
            cap_tokens = (int64_t)std::min<size_t>(fr / 4 / tok_bytes, (size_t)1 << 24);
        }
        e->n_pages = std::max<int64_t>(1, (cap_tokens + e->page_tokens - 1) / e->page_tokens);
        e->pool.ensure((size_t)e->n_pages * e->page_bytes);
        e->pools.p[0] = e->pool.p;
        e->free_pages.reserve((size_t)e->n_pages);
        for (int64_t p = e->n_pages - 1; p >= 0; --p) e->free_pages.push_back((int32_t)p);
        if (e->opts.host_spill_tokens > 0) {  // pinned host tier, mapped into the device address space
            e->n_host_pages = (e->opts.host_spill_tokens + e->page_tokens - 1) / e->page_tokens;
            TKV_CUDA(cudaHostAlloc(&e->host_pool, (size_t)e->n_host_pages * e->page_bytes,
                                   cudaHostAllocMapped | cudaHostAllocPortable));
            void* dp = nullptr;
            TKV_CUDA(cudaHostGetDevicePointer(&dp, e->host_pool, 0));
            e->pools.p[kHostPool] = dp;
            e->host_free.reserve((size_t)e->n_host_pages);
            for (int64_t p = e->n_host_pages - 1; p >= 0; --p) e->host_free.push_back((int32_t)p);
        }
        e->sync();
        *out = e.release();
    });
    return st;
}

tkv_status tkv_engine_create(const tkv_model_config* cfg, uint64_t seed, const tkv_engine_opts* opts,
                             tkv_engine** out) {
    return create_engine(cfg, seed, opts, out, nullptr);
}

// ---- TKVW weights files (docs/formats.md "TKVW"; src/model.cpp:120-196) ----
}  // extern "C"
namespace {
struct WeightsFile {
    std::ifstream in;
    std::string path;
    tkv_model_config cfg{};
    void read(void* dst, size_t n, const char* what) {
        in.read(static_cast<char*>(dst), (std::streamsize)n);
        if ((size_t)in.gcount() != n) fail(TKV_ERR_FORMAT, std::string(what) + ": truncated weights file " + path);
    }
    template <typename T>
    T get(const char* what) {
        T v;
        read(&v, sizeof v, what);
        return v;
    }
};

// header (magic, version, config) -- FormatError / NotFoundError like load_weights (model.cpp:152-172)
void open_tkvw(WeightsFile& wf, const char* path) {
    wf.path = path;
    wf.in.open(path, std::ios::binary);
    if (!wf.in) fail(TKV_ERR_NOT_FOUND, std::string("no such file: ") + path);
    char magic[4];
    wf.read(magic, 4, "weights magic");
    if (std::memcmp(magic, "TKVW", 4) != 0) fail(TKV_ERR_FORMAT, std::string("not a weights file: ") + path);
    const uint32_t version = wf.get<uint32_t>("weights version");
    if (version != 1) fail(TKV_ERR_FORMAT, "unsupported weights version " + std::to_string(version));
    tkv_model_config& c = wf.cfg;
    c.layer_num = wf.get<int64_t>("weights config");
    c.head_num = wf.get<int64_t>("weights config");
    c.kv_head_num = wf.get<int64_t>("weights config");
    c.head_size = wf.get<int64_t>("weights config");
    c.hidden_size = wf.get<int64_t>("weights config");
    c.intermediate_size = wf.get<int64_t>("weights config");
    c.vocab_size = wf.get<int64_t>("weights config");
    c.rope_base = wf.get<double>("weights config");
    c.norm_eps = wf.get<double>("weights config");
    validate_cfg(c);
}

// The tensors in draw order: each shape-checked against the config, streamed in pieces through pinned host memory to
// the device, FNV-hashed there (the bytes ARE weights_checksum's stream) and cast into the engine layout; the trailing
// checksum must match (FormatError otherwise).
void load_tkvw(tkv_engine* e, WeightsFile& wf) {
    const int64_t H = e->hid, qd = e->qd, kvd = e->kvd, I = e->I, V = e->V;
    const size_t es = dt_size(e->dt);
    const int64_t piece = std::min<int64_t>(int64_t(1) << 25, std::max({V * H, H * I, qd * H, H * V}));
    void* host = nullptr;
    TKV_CUDA(cudaHostAlloc(&host, (size_t)piece * 8, cudaHostAllocDefault));
    std::unique_ptr<void, void (*)(void*)> host_guard(host, [](void* p) { cudaFreeHost(p); });
    DevMem dbuf;
    dbuf.ensure((size_t)piece * 8);
    uint64_t h = Fnv{}.h;
    // store(dev values, element offset e0, count n) of one tensor
    auto tensor = [&](bool mat, int64_t rows, int64_t cols, const char* name,
                      const std::function<void(const double*, int64_t, int64_t)>& store) {
        std::vector<FpSeg> head;
        uint64_t w = 0;
        if (mat) {
            const uint64_t r = wf.get<uint64_t>("tensor shape"), c = wf.get<uint64_t>("tensor shape");
            if ((int64_t)r != rows || (int64_t)c != cols)
                fail(TKV_ERR_FORMAT, std::string(name) + ": tensor shape does not match the weights config");
            head.push_back(FpSeg{w++, 1, r, 0.0, 0, 0});
            head.push_back(FpSeg{w++, 1, c, 0.0, 0, 0});
        } else {
            const uint64_t n = wf.get<uint64_t>("tensor shape");
            if ((int64_t)n != cols) fail(TKV_ERR_FORMAT, std::string(name) + ": vector size does not match the config");
            head.push_back(FpSeg{w++, 1, n, 0.0, 0, 0});
        }
        const int64_t total = rows * cols;
        for (int64_t e0 = 0; e0 < total || (total == 0 && e0 == 0); e0 += piece) {
            const int64_t n = std::min(piece, total - e0);
            wf.read(host, (size_t)n * 8, name);
            TKV_CUDA(cudaMemcpyAsync(dbuf.p, host, (size_t)n * 8, cudaMemcpyHostToDevice, e->stream));
            std::vector<FpSeg> segs = e0 == 0 ? head : std::vector<FpSeg>{};
            const uint64_t w0 = segs.empty() ? 0 : w;
            segs.push_back(FpSeg{w0, (uint64_t)n, (uint64_t)(uintptr_t)dbuf.p, 0.0, 3, 0});
            h = device_fnv_words(segs, 0, h, e->stream);  // synchronises: the pinned piece is free afterwards
            store(dbuf.as<double>(), e0, n);
            if (total == 0) break;
        }
    };
    auto vec = [&](float* dst, const char* name) {
        tensor(false, 1, H, name, [&](const double* src, int64_t e0, int64_t n) {
            launch_store_f32_from_f64(dst + e0, src, n, e->stream);
        });
    };
    auto mat = [&](void* dst, int64_t rows, int64_t cols, const char* name, int rb = 0, int off = 0) {
        tensor(true, rows, cols, name, [&](const double* src, int64_t e0, int64_t n) {
            launch_store_transposed_f64(dst, e->dt, src, e0, n, rows, cols, e->stream, rb, off);
        });
    };
    tensor(true, V, H, "embedding", [&](const double* src, int64_t e0, int64_t n) {
        launch_store_f32_from_f64(e->emb + e0, src, n, e->stream);
    });
    const int rb = e->gu_block;
    for (int64_t l = 0; l < e->L; ++l) {
        uint8_t* qkv = static_cast<uint8_t*>(e->w_qkv[l]);
        uint8_t* gu = static_cast<uint8_t*>(e->w_gu[l]);
        vec(e->norm_attn(l), "attn_norm");
        vec(e->norm_mlp(l), "mlp_norm");
        mat(qkv, H, qd, "wq");
        mat(qkv + (size_t)qd * H * es, H, kvd, "wk");
        mat(qkv + (size_t)(qd + kvd) * H * es, H, kvd, "wv");
        mat(e->w_o[l], qd, H, "wo");
        mat(gu, H, I, "w_gate", rb, 0);
        mat(rb ? gu : gu + (size_t)I * H * es, H, I, "w_up", rb, rb);
        mat(e->w_down[l], I, H, "w_down");
    }
    vec(e->norms + (size_t)2 * e->L * H, "final_norm");
    mat(e->w_lm, H, V, "lm_head");
    const uint64_t stored = wf.get<uint64_t>("weights checksum");
    e->sync();
    if (stored != h) fail(TKV_ERR_FORMAT, "weights checksum mismatch: " + wf.path);
    e->fingerprint = fingerprint_of(e->cfg, h);
}
}  // namespace
extern "C" {

tkv_status tkv_engine_create_from_weights(const char* path, const tkv_engine_opts* opts, tkv_engine** out,
                                          tkv_model_config* cfg_out) {
    WeightsFile wf;
    const tkv_status st = guard([&] {
        need(path, "path");
        need(out, "out");
        open_tkvw(wf, path);
        if (cfg_out) *cfg_out = wf.cfg;
    });
    if (st != TKV_OK) return st;
    return create_engine(&wf.cfg, 0, opts, out, &wf);
}

tkv_status tkv_save_weights(const tkv_model_config* cfg, uint64_t seed, const char* path, int device) {
    return guard([&] {
        need(cfg, "cfg");
        need(path, "path");
        validate_cfg(*cfg);
        TKV_CUDA(cudaSetDevice(device));
        std::string head("TKVW", 4);
        auto put = [&](const void* p, size_t n) { head.append(static_cast<const char*>(p), n); };
        const uint32_t version = 1;
        put(&version, 4);
        const int64_t ints[7] = {cfg->layer_num, cfg->head_num, cfg->kv_head_num, cfg->head_size, cfg->hidden_size,
                                 cfg->intermediate_size, cfg->vocab_size};
        put(ints, sizeof ints);
        put(&cfg->rope_base, 8);
        put(&cfg->norm_eps, 8);
        const std::vector<FpSeg> segs = checksum_segments(*cfg);  // the tensor stream: shapes, 1.0 norms, draws
        uint64_t words = 0;
        for (const FpSeg& g : segs) words = std::max(words, g.word0 + g.n);
        const std::string tmp = std::string(path) + ".tmp";
        std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
        if (!f) fail(TKV_ERR_IO, "cannot open " + tmp + " for writing");
        f.write(head.data(), (std::streamsize)head.size());
        const int64_t piece = int64_t(1) << 24;
        DevMem d;
        d.ensure((size_t)std::min<uint64_t>(words, piece) * 8 + 8);
        std::vector<uint64_t> buf((size_t)std::min<uint64_t>(words, piece));
        for (uint64_t w0 = 0; w0 < words; w0 += piece) {
            const int64_t n = (int64_t)std::min<uint64_t>(piece, words - w0);
            device_words(segs, seed, w0, n, d.as<uint64_t>(), 0);
            TKV_CUDA(cudaMemcpy(buf.data(), d.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
            f.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(n * 8));
        }
        const uint64_t ck = device_fnv_words(segs, seed, Fnv{}.h, 0);
        f.write(reinterpret_cast<const char*>(&ck), 8);
        f.close();
        if (!f) fail(TKV_ERR_IO, "write failed: " + tmp);
        if (std::rename(tmp.c_str(), path) != 0) fail(TKV_ERR_IO, std::string("rename to ") + path + " failed");
    });
}

void tkv_engine_destroy(tkv_engine* eng) {
    if (!eng) return;
    cudaSetDevice(eng->device);
    delete eng;
}

tkv_status tkv_engine_fingerprint(const tkv_engine* eng, uint64_t* out) {
    return guard([&] {
        need(eng, "engine");
        need(out, "out");
        *out = eng->fingerprint;
    });
}

tkv_status tkv_engine_config(const tkv_engine* eng, tkv_model_config* out) {
    return guard([&] {
        need(eng, "engine");
        need(out, "out");
        *out = eng->cfg;
    });
}

tkv_status tkv_ingest_chunks(tkv_engine* e, const int32_t* payloads, const int64_t* offsets, int64_t n_chunks,
                             uint64_t* ids_out, tkv_ingest_stats* stats) {
    return guard([&] {
        NvtxRange nvtx("tkv_ingest_chunks");
        need(e, "engine");
        need(offsets, "offsets");
        e->bind();
        struct Pending {
            uint64_t id;
            std::vector<int32_t> framed;
        };
        std::vector<Pending> todo;
        std::set<uint64_t> batch_ids;
        for (int64_t c = 0; c < n_chunks; ++c) {
            const int64_t n = offsets[c + 1] - offsets[c];
            if (n < 0) fail(TKV_ERR_SHAPE, "ingest: offsets must be non-decreasing");
            std::vector<int32_t> framed = framed_of(payloads + offsets[c], n);
            check_tokens(e, framed.data(), (int64_t)framed.size());
            const uint64_t id = content_id(e->fingerprint, framed.data(), (int64_t)framed.size());
            if (ids_out) ids_out[c] = id;
            if (stats) stats->chunks += 1;
            auto known = e->chunks.find(id);
            if (known != e->chunks.end()) {
                // idempotent: no prefill, no bytes written (pipeline.cpp:104-123) -- but, like the reference
                // (:124-131), a chunk that reached the store without a record (TKVC import) gets its framed
                // tokens and its retrieval-index entry now
                if (known->second.framed.empty()) known->second.framed = framed;
                if (n > 0 && !e->idx_row.count(id)) e->index_add(id, framed.data() + 1, n, nullptr);
                continue;
            }
            if (batch_ids.count(id)) continue;
            batch_ids.insert(id);
            todo.push_back({id, std::move(framed)});
        }
        // Packed block-diagonal prefill: up to ~16K tokens per forward.
        const int64_t kMaxTokens = 16384;
        size_t i0 = 0;
        while (i0 < todo.size()) {
            size_t i1 = i0;
            int64_t T = 0;
            while (i1 < todo.size() && (T == 0 || T + (int64_t)todo[i1].framed.size() <= kMaxTokens)) {
                T += (int64_t)todo[i1].framed.size();
                ++i1;
            }
            Stage s;
            std::vector<Chunk> made;
            int64_t off = 0;
            try {
                for (size_t k = i0; k < i1; ++k) {
                    Chunk ch;
                    ch.len = (int64_t)todo[k].framed.size();
                    ch.framed = todo[k].framed;
                    store_chunk_pages(e, ch);
                    for (int64_t t = 0; t < ch.len; ++t) {
                        s.tok.push_back(todo[k].framed[t]);
                        s.pos.push_back((int32_t)t);          // positions 0..len-1 (pipeline.cpp:106)
                        s.lo.push_back((int32_t)off);         // causal_rows(len, 0) per chunk: block-diagonal
                        s.hi.push_back((int32_t)(off + t));
                        const int32_t pg = ch.pages[t / e->page_tokens];
                        s.page.push_back(ch.slot == kHostPool ? (int32_t)e->n_pages + pg : pg);  // host_base = n_pages
                        s.slot.push_back((int32_t)(t % e->page_tokens));
                    }
                    off += ch.len;
                    made.push_back(std::move(ch));
                }
                tkv_context* scratch = new_context(e, T);
                try {
                    e->ensure_rope(T);
                    upload_stage(e, s, true);
                    tkv_engine::Fwd f;
                    f.tok = e->p_tok;
                    f.T = (int)T;
                    f.pos = e->p_pos;
                    f.ctx = scratch;
                    f.row0 = 0;
                    f.lo = e->p_lo;
                    f.hi = e->p_hi;
                    f.logits = false;
                    f.kv_only = true;
                    f.sc.pool = e->pool.p;
                    f.sc.page = e->p_page;
                    f.sc.slot = e->p_slot;
                    f.sc.page_tokens = (int)e->page_tokens;
                    f.sc.layer_num = (int)e->L;
                    f.sc.host_pool = const_cast<void*>(e->pools.p[kHostPool]);
                    f.sc.host_base = (int32_t)e->n_pages;
                    e->forward(f);
                    e->check_err("ingest");
                } catch (...) {
                    tkv_context_destroy(scratch);
                    throw;
                }
                tkv_context_destroy(scratch);
            } catch (...) {
                for (auto& ch : made) release_chunk_pages(e, ch);
                throw;
            }
            for (size_t k = i0; k < i1; ++k) {
                Chunk& ch = made[k - i0];
                if (stats) {
                    stats->new_chunks += 1;
                    stats->bytes_written += (uint64_t)ch.len * e->L * 2 * e->kvd * dt_size(e->dt);
                }
                // the retrieval index entry over the unframed payload (Engine::ingest_chunk_payload adds the
                // ChunkRecord, pipeline.cpp:97-134; ChunkRecord.embedding, retrieval.hpp:25-30)
                if (ch.framed.size() > 2) e->index_add(todo[k].id, ch.framed.data() + 1, (int64_t)ch.framed.size() - 2, nullptr);
                e->chunks.emplace(todo[k].id, std::move(ch));
            }
            i0 = i1;
        }
    });
}

tkv_status tkv_import_tkvc(tkv_engine* e, const char* path, uint64_t* id_out) {
    return guard([&] {
        need(e, "engine");
        need(path, "path");
        e->bind();
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(TKV_ERR_NOT_FOUND, std::string("no such file: ") + path);
        std::string raw((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        size_t cur = 0;
        auto rd = [&](void* dst, size_t n, const char* what) {
            if (cur + n > raw.size()) fail(TKV_ERR_FORMAT, std::string(what) + ": truncated");
            std::memcpy(dst, raw.data() + cur, n);
            cur += n;
        };
        auto u32 = [&](const char* w) {
            uint8_t b[4];
            rd(b, 4, w);
            return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
        };
        auto u64 = [&](const char* w) {
            uint64_t lo = u32(w), hi = u32(w);
            return lo | (hi << 32);
        };
        char magic[4];
        rd(magic, 4, "chunk magic");  // kvstore.cpp:144-191 validation order
        if (std::memcmp(magic, "TKVC", 4) != 0) fail(TKV_ERR_FORMAT, std::string("not a chunk cache file: ") + path);
        const uint32_t version = u32("chunk version");
        if (version != 1) fail(TKV_ERR_FORMAT, "unsupported chunk version " + std::to_string(version));
        const uint32_t dtype = u32("chunk dtype");
        if (dtype != 1 && dtype != 2) fail(TKV_ERR_FORMAT, "unknown chunk dtype " + std::to_string(dtype));
        const uint32_t layers = u32("chunk header"), kvh = u32("chunk header"), hs = u32("chunk header"),
                       ntok = u32("chunk header");
        const uint64_t fp = u64("chunk header"), id = u64("chunk header");
        std::string stem = path;
        const size_t slash = stem.find_last_of('/');
        if (slash != std::string::npos) stem = stem.substr(slash + 1);
        if (stem.size() == 21 && stem.substr(16) == ".tkvc" && stem.substr(0, 16) != hex_id(id))
            fail(TKV_ERR_FORMAT, std::string("chunk id mismatch in ") + path);
        if (fp != e->fingerprint)
            fail(TKV_ERR_STALE_CACHE, "chunk " + hex_id(id) + " was built under a different model fingerprint");
        if (layers == 0 || kvh == 0 || hs == 0 || ntok == 0)
            fail(TKV_ERR_FORMAT, std::string("chunk header: zero dimension in ") + path);
        const uint64_t elem = dtype == 1 ? 8 : 4, kvd = (uint64_t)kvh * hs, tb = (uint64_t)ntok * kvd * elem;
        uint64_t expect = 44 + (uint64_t)layers * 16;
        for (uint32_t i = 0; i < layers * 2; ++i) {
            if (u64("chunk offsets") != expect) fail(TKV_ERR_FORMAT, std::string("chunk offsets table corrupt in ") + path);
            expect += tb;
        }
        if (raw.size() != expect) fail(TKV_ERR_FORMAT, std::string("chunk file size mismatch in ") + path);
        if ((int64_t)kvh != e->Hkv || (int64_t)hs != e->d || (int64_t)layers != e->L)
            fail(TKV_ERR_STALE_CACHE, "chunk geometry does not match the engine config");
        if (id_out) *id_out = id;
        if (e->chunks.count(id)) return;
        Chunk ch;
        ch.len = ntok;
        store_chunk_pages(e, ch);
        try {
        // convert f64/f32 -> f32 -> engine dtype on the host, page by page, then one H2D per page
        std::vector<uint8_t> page(e->page_bytes);
        for (size_t p = 0; p < ch.pages.size(); ++p) {
            std::fill(page.begin(), page.end(), 0);
            const int64_t t0 = (int64_t)p * e->page_tokens, nt = std::min<int64_t>(e->page_tokens, ntok - t0);
            for (uint32_t l = 0; l < layers; ++l)
                for (int kv = 0; kv < 2; ++kv) {
                    const size_t src = 44 + (size_t)layers * 16 + (size_t)(l * 2 + kv) * tb;
                    for (int64_t t = 0; t < nt; ++t)
                        for (uint64_t c = 0; c < kvd; ++c) {
                            const size_t at = src + ((size_t)(t0 + t) * kvd + c) * elem;
                            float f;
                            if (elem == 8) {
                                double v;
                                std::memcpy(&v, raw.data() + at, 8);
                                f = (float)v;
                            } else {
                                std::memcpy(&f, raw.data() + at, 4);
                            }
                            const size_t dst = ((size_t)(l * 2 + kv) * e->page_tokens + t) * kvd + c;
                            if (e->dt == DT::F32) {
                                std::memcpy(page.data() + dst * 4, &f, 4);
                            } else {  // f32 -> bf16 round-to-nearest-even (same as __float2bfloat16_rn)
                                uint32_t b;
                                std::memcpy(&b, &f, 4);
                                uint16_t h;
                                if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x7FFFFFu))
                                    h = (uint16_t)((b >> 16) | 0x40);
                                else
                                    h = (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
                                std::memcpy(page.data() + dst * 2, &h, 2);
                            }
                        }
                }
            TKV_CUDA(cudaMemcpy(page_ptr(e, ch.slot, ch.pages[p]), page.data(), e->page_bytes, cudaMemcpyDefault));
        }
        } catch (...) {
            release_chunk_pages(e, ch);  // a failed copy must not leak store capacity
            throw;
        }
        e->chunks.emplace(id, std::move(ch));
    });
}

tkv_status tkv_export_tkvc(tkv_engine* e, uint64_t id, const char* path) {
    return guard([&] {
        need(e, "engine");
        need(path, "path");
        e->bind();
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        const Chunk& ch = it->second;
        const uint64_t kvd = e->kvd, tb = (uint64_t)ch.len * kvd * 4;
        std::string out;
        auto w32 = [&](uint32_t v) {
            for (int i = 0; i < 4; ++i) out.push_back((char)((v >> (8 * i)) & 0xFF));
        };
        auto w64 = [&](uint64_t v) {
            w32((uint32_t)v);
            w32((uint32_t)(v >> 32));
        };
        out.append("TKVC", 4);
        w32(1);
        w32(2);  // f32
        w32((uint32_t)e->L);
        w32((uint32_t)e->Hkv);
        w32((uint32_t)e->d);
        w32((uint32_t)ch.len);
        w64(e->fingerprint);
        w64(id);
        uint64_t cur = 44 + (uint64_t)e->L * 16;
        for (int64_t l = 0; l < e->L * 2; ++l) {
            w64(cur);
            cur += tb;
        }
        std::vector<float> buf((size_t)(ch.len * kvd));
        for (int64_t l = 0; l < e->L; ++l)
            for (int kv = 0; kv < 2; ++kv) {
                tkv_status st = tkv_store_read(e, id, l, (tkv_kv_which)kv, buf.data(), (int64_t)buf.size());
                if (st != TKV_OK) fail(st, g_last_error);
                out.append(reinterpret_cast<const char*>(buf.data()), buf.size() * 4);
            }
        const std::string tmp = std::string(path) + ".tmp";
        {
            std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
            if (!f) fail(TKV_ERR_IO, "cannot open " + tmp + " for writing");
            f.write(out.data(), (std::streamsize)out.size());
            if (!f) fail(TKV_ERR_IO, "write failed: " + tmp);
        }
        if (std::rename(tmp.c_str(), path) != 0) fail(TKV_ERR_IO, std::string("rename to ") + path + " failed");
    });
}

tkv_status tkv_store_contains(const tkv_engine* e, uint64_t id, int* out) {
    return guard([&] {
        need(e, "engine");
        need(out, "out");
        *out = e->chunks.count(id) ? 1 : 0;
    });
}

tkv_status tkv_store_evict(tkv_engine* e, uint64_t id) {
    return guard([&] {
        need(e, "engine");
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        if (it->second.shared)
            fail(TKV_ERR_CONFIG, "chunk " + hex_id(id) + " is listed in an exported directory: peers read its pages");
        release_chunk_pages(e, it->second);  // peer-registered chunks only drop the entry
        e->chunks.erase(it);
        e->store_epoch += 1;
    });
}

tkv_status tkv_store_tiers(const tkv_engine* e, int64_t* hbm_used, int64_t* hbm_total, int64_t* host_used,
                           int64_t* host_total) {
    return guard([&] {
        need(e, "engine");
        if (hbm_used) *hbm_used = e->n_pages - (int64_t)e->free_pages.size();
        if (hbm_total) *hbm_total = e->n_pages;
        if (host_used) *host_used = e->n_host_pages - (int64_t)e->host_free.size();
        if (host_total) *host_total = e->n_host_pages;
    });
}

tkv_status tkv_store_rebalance(tkv_engine* e, int64_t max_moves, int64_t* promoted, int64_t* demoted) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        int64_t up = 0, down = 0;
        if (e->n_host_pages > 0 && max_moves > 0) {
            // frequency policy: the most-retrieved host-tier chunks move into HBM; when HBM is full, the least-retrieved
            // HBM chunks move out to make room, but only while the incoming chunk is hotter than the outgoing one
            std::vector<std::pair<uint32_t, uint64_t>> cold_hbm, hot_host;
            for (auto& kv : e->chunks) {
                if (kv.second.shared) continue;  // peers hold its page indices
                if (kv.second.slot == 0) cold_hbm.emplace_back(kv.second.hits, kv.first);
                else if (kv.second.slot == kHostPool && kv.second.hits > 0) hot_host.emplace_back(kv.second.hits, kv.first);
            }
            std::sort(hot_host.begin(), hot_host.end(), [](auto& a, auto& b) { return a.first != b.first ? a.first > b.first : a.second < b.second; });
            std::sort(cold_hbm.begin(), cold_hbm.end());
            size_t victim = 0;
            auto move = [&](Chunk& ch, bool to_hbm) {
                Chunk dst;
                dst.len = ch.len;
                const int64_t np = (int64_t)ch.pages.size();
                std::vector<int32_t>& fl = to_hbm ? e->free_pages : e->host_free;
                if ((int64_t)fl.size() < np) return false;
                for (int64_t p = 0; p < np; ++p) {
                    dst.pages.push_back(fl.back());
                    fl.pop_back();
                }
                dst.slot = to_hbm ? 0 : kHostPool;
                for (int64_t p = 0; p < np; ++p)  // PCIe / C2C copies of whole pages
                    TKV_CUDA(cudaMemcpyAsync(page_ptr(e, dst.slot, dst.pages[(size_t)p]), page_ptr(e, ch.slot, ch.pages[(size_t)p]),
                                             e->page_bytes, cudaMemcpyDefault, e->stream));
                release_chunk_pages(e, ch);
                ch.pages = std::move(dst.pages);
                ch.slot = dst.slot;
                return true;
            };
            for (auto& h : hot_host) {
                if (up + down >= max_moves) break;
                Chunk& ch = e->chunks[h.second];
                const int64_t np = (int64_t)ch.pages.size();
                while ((int64_t)e->free_pages.size() < np && victim < cold_hbm.size() && cold_hbm[victim].first < h.first &&
                       up + down < max_moves) {
                    Chunk& v = e->chunks[cold_hbm[victim++].second];
                    if (!move(v, false)) break;
                    ++down;
                }
                if ((int64_t)e->free_pages.size() < np) break;
                if (move(ch, true)) ++up;
            }
            if (up + down > 0) {
                e->sync();
                e->store_epoch += 1;  // contexts that re-read store pages must not use the old page lists
            }
        }
        for (auto& kv : e->chunks) kv.second.hits >>= 1;  // decay: recent retrievals count most
        if (promoted) *promoted = up;
        if (demoted) *demoted = down;
    });
}

tkv_status tkv_store_chunk_tier(const tkv_engine* e, uint64_t id, int32_t* tier) {
    return guard([&] {
        need(e, "engine");
        need(tier, "tier");
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        *tier = it->second.slot == 0 ? 0 : (it->second.slot == kHostPool ? 1 : 2);
    });
}

tkv_status tkv_store_chunk_tokens(const tkv_engine* e, uint64_t id, int64_t* out) {
    return guard([&] {
        need(e, "engine");
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        *out = it->second.len;
    });
}

tkv_status tkv_store_count(const tkv_engine* e, int64_t* chunks, int64_t* used, int64_t* total) {
    return guard([&] {
        need(e, "engine");
        if (chunks) *chunks = (int64_t)e->chunks.size();
        if (used) *used = e->n_pages - (int64_t)e->free_pages.size();
        if (total) *total = e->n_pages;
    });
}

tkv_status tkv_store_ids(const tkv_engine* e, uint64_t* ids_out, int64_t capacity, int64_t* n_out) {
    return guard([&] {
        need(e, "engine");
        std::vector<uint64_t> ids;
        ids.reserve(e->chunks.size());
        for (const auto& kv : e->chunks) ids.push_back(kv.first);
        std::sort(ids.begin(), ids.end());  // CacheStore::ids: ascending (kvstore.cpp)
        if (n_out) *n_out = (int64_t)ids.size();
        if (ids_out) {
            if (capacity < (int64_t)ids.size()) fail(TKV_ERR_SHAPE, "store_ids: output capacity too small");
            std::copy(ids.begin(), ids.end(), ids_out);
        }
    });
}

tkv_status tkv_store_read(const tkv_engine* ce, uint64_t id, int64_t layer, tkv_kv_which which, float* host_out,
                          int64_t capacity) {
    return guard([&] {
        tkv_engine* e = const_cast<tkv_engine*>(ce);
        need(e, "engine");
        need(host_out, "host_out");
        e->bind();
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        if (layer < 0 || layer >= e->L) fail(TKV_ERR_SHAPE, "layer out of range");
        const Chunk& ch = it->second;
        if (capacity < ch.len * e->kvd) fail(TKV_ERR_SHAPE, "host buffer too small");
        const size_t es = dt_size(e->dt);
        DevMem tmp, tmpf;
        tmp.ensure((size_t)ch.len * e->kvd * es);
        tmpf.ensure((size_t)ch.len * e->kvd * 4);
        for (size_t p = 0; p < ch.pages.size(); ++p) {
            const int64_t t0 = (int64_t)p * e->page_tokens, nt = std::min<int64_t>(e->page_tokens, ch.len - t0);
            const uint8_t* src = static_cast<const uint8_t*>(e->pools.p[ch.slot]) + (size_t)ch.pages[p] * e->page_bytes +
                                 (size_t)((layer * 2 + (int)which) * e->page_tokens) * e->kvd * es;
            TKV_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(tmp.p) + (size_t)t0 * e->kvd * es, src,
                                     (size_t)nt * e->kvd * es, cudaMemcpyDefault, e->stream));  // HBM, host tier or peer
        }
        launch_to_f32(tmp.p, ch.len * e->kvd, tmpf.as<float>(), e->dt, e->stream);
        TKV_CUDA(cudaMemcpyAsync(host_out, tmpf.p, (size_t)ch.len * e->kvd * 4, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
    });
}

tkv_status tkv_assemble(tkv_engine* e, const uint64_t* ids, int64_t n, tkv_position_mode mode, tkv_context** out) {
    return guard([&] {
        NvtxRange nvtx("tkv_assemble");
        need(e, "engine");
        need(out, "out");
        if (n > 0) need(ids, "chunk_ids");
        if (mode != TKV_POS_COMPOSITE && mode != TKV_POS_REORDERED) fail(TKV_ERR_CONFIG, "unknown position mode");
        e->bind();
        *out = assemble_impl(e, ids, n, mode);
    });
}

tkv_status tkv_prefill_query(tkv_engine* e, tkv_context* c, const int32_t* query, int64_t n, float* logits_out,
                             tkv_flops* fl) {
    return guard([&] {
        NvtxRange nvtx("tkv_prefill_query");
        need(e, "engine");
        need(c, "context");
        if (n <= 0) fail(TKV_ERR_DOMAIN, "prefill_query: empty query");  // pipeline.cpp:169
        need(query, "query");
        if (c->eng != e) fail(TKV_ERR_STALE_CACHE, "context was assembled under a different model");
        check_tokens(e, query, n);
        e->bind();
        std::vector<float> lg((size_t)e->V);
        const int64_t P = c->total;
        extend(e, c, query, nullptr, n, lg.data(), nullptr);
        if (logits_out) std::memcpy(logits_out, lg.data(), lg.size() * 4);
        flops_add(e, fl, n, P + n);
    });
}

tkv_status tkv_prefill_query_batch(tkv_engine* e, tkv_context* const* ctxs, int64_t n_req, const int32_t* queries,
                                   const int64_t* offsets, float* logits_out, tkv_flops* fl) {
    return guard([&] {
        NvtxRange nvtx("tkv_prefill_query_batch");
        need(e, "engine");
        need(ctxs, "contexts");
        need(offsets, "offsets");
        if (n_req <= 0) fail(TKV_ERR_DOMAIN, "prefill_query_batch: empty batch");
        std::set<const tkv_context*> seen;
        for (int64_t r = 0; r < n_req; ++r) {
            need(ctxs[r], "context");
            if (ctxs[r]->eng != e) fail(TKV_ERR_STALE_CACHE, "context was assembled under a different model");
            if (!seen.insert(ctxs[r]).second) fail(TKV_ERR_CONFIG, "prefill_query_batch: a context appears twice");
            if (offsets[r + 1] - offsets[r] <= 0) fail(TKV_ERR_DOMAIN, "prefill_query: empty query");  // pipeline.cpp:169
        }
        const int64_t T = offsets[n_req] - offsets[0];
        need(queries, "queries");
        check_tokens(e, queries + offsets[0], T);
        e->bind();
        Stage s;
        tkv_engine::Fwd f;
        int64_t max_pos = 0;
        for (int64_t r = 0; r < n_req; ++r) {
            tkv_context* c = ctxs[r];
            const int64_t n = offsets[r + 1] - offsets[r], P = c->total;
            ensure_cap(e, c, P + n);
            f.reqs.push_back({c, (int)s.pos.size(), (int)n, (int)P});
            for (int64_t i = 0; i < n; ++i) {
                s.tok.push_back(queries[offsets[r] + i]);
                s.pos.push_back((int32_t)(c->next_position + i));
                s.lo.push_back(0);
                s.hi.push_back((int32_t)(P + i));  // causal_rows(n, P) of this request
            }
            max_pos = std::max(max_pos, c->next_position + n);
        }
        e->ensure_rope(max_pos);
        upload_stage(e, s, true);
        // batched attention: one launch when the batch alone fills the GPU (bf16, head_size 128)
        const int group = (int)(e->H / e->Hkv);
        int64_t row_groups = 0;
        int max_n = 0;
        for (const auto& r : f.reqs) {
            row_groups += ((int64_t)r.n * group + kAttnTcRows - 1) / kAttnTcRows * e->Hkv;
            max_n = std::max(max_n, r.n);
        }
        if (e->dt == DT::BF16 && !(e->opts.flags & TKV_FLAG_SIMT_ATTN) && attention_tc_supported((int)e->d, e->dt) &&
            (row_groups >= e->num_sms || (e->opts.flags & TKV_FLAG_BATCH_ATTN))) {
            std::vector<AttnReq> rq;
            std::vector<uint8_t> maps((size_t)n_req * 128);
            for (size_t r = 0; r < f.reqs.size(); ++r) {
                const auto& q = f.reqs[r];
                rq.push_back({q.tok0, q.n, q.row0, 0});
                attn_tc_cache_map(q.ctx->kv, q.row0 + q.n, q.ctx->cap, (int)e->kvd, (int)e->L, maps.data() + r * 128);
            }
            e->d_breq.ensure(rq.size() * sizeof(AttnReq));
            e->d_bmaps.ensure(maps.size());
            TKV_CUDA(cudaMemcpyAsync(e->d_breq.p, rq.data(), rq.size() * sizeof(AttnReq), cudaMemcpyHostToDevice, e->stream));
            TKV_CUDA(cudaMemcpyAsync(e->d_bmaps.p, maps.data(), maps.size(), cudaMemcpyHostToDevice, e->stream));
            e->h2d_bytes += (int64_t)(rq.size() * sizeof(AttnReq) + maps.size());
            f.batch_reqs = e->d_breq.as<AttnReq>();
            f.batch_maps = e->d_bmaps.p;
            f.batch_max_n = max_n;
            int min_keys = INT32_MAX;
            for (const auto& q : f.reqs) min_keys = std::min(min_keys, q.row0 + q.n);
            f.batch_min_keys = min_keys;
        }
        {  // the batched QKV epilogue's request table (tok0 ascending)
            std::vector<EpiReq> er;
            for (const auto& q : f.reqs) er.push_back({q.ctx->kv, q.ctx->cap, q.tok0, q.n, q.row0, 0});
            e->d_epireq.ensure(er.size() * sizeof(EpiReq));
            TKV_CUDA(cudaMemcpyAsync(e->d_epireq.p, er.data(), er.size() * sizeof(EpiReq), cudaMemcpyHostToDevice,
                                     e->stream));
            e->h2d_bytes += (int64_t)(er.size() * sizeof(EpiReq));
            f.epi_reqs = e->d_epireq.as<EpiReq>();
        }
        f.tok = e->p_tok;
        f.T = (int)T;
        f.pos = e->p_pos;
        f.lo = e->p_lo;
        f.hi = e->p_hi;
        f.logits = true;
        e->forward(f);
        std::vector<float> lg((size_t)n_req * e->V);
        TKV_CUDA(cudaMemcpyAsync(lg.data(), e->logits.p, lg.size() * 4, cudaMemcpyDeviceToHost, e->stream));
        e->d2h_bytes += (int64_t)lg.size() * 4;
        e->check_err("prefill_query_batch");
        if (logits_out) std::memcpy(logits_out, lg.data(), lg.size() * 4);
        for (int64_t r = 0; r < n_req; ++r) {  // the same bookkeeping as prefill_query (pipeline.cpp:166-186)
            tkv_context* c = ctxs[r];
            const int64_t n = offsets[r + 1] - offsets[r], P = c->total;
            Stage sr;
            sr.lo.assign(s.lo.begin() + f.reqs[r].tok0, s.lo.begin() + f.reqs[r].tok0 + n);
            sr.hi.assign(s.hi.begin() + f.reqs[r].tok0, s.hi.begin() + f.reqs[r].tok0 + n);
            remember_mask(c, sr, P + n);
            for (int64_t i = 0; i < n; ++i) c->positions.push_back(c->next_position + i);
            c->total = P + n;
            c->extend_query_segment(n);
            c->next_position += n;
            c->last_logits.assign(lg.begin() + r * e->V, lg.begin() + (r + 1) * e->V);
            flops_add(e, fl, n, P + n);
        }
    });
}

tkv_status tkv_prefill_query_device(tkv_engine* e, tkv_context* c, const int32_t* d_query, int64_t n,
                                    float* d_logits) {
    return guard([&] {
        NvtxRange nvtx("tkv_prefill_query_device");
        need(e, "engine");
        need(c, "context");
        if (n <= 0) fail(TKV_ERR_DOMAIN, "prefill_query: empty query");
        need(d_query, "query");
        if (c->eng != e) fail(TKV_ERR_STALE_CACHE, "context was assembled under a different model");
        e->bind();
        extend(e, c, nullptr, d_query, n, nullptr, d_logits);
    });
}

tkv_status tkv_debug_weights_checksum(const tkv_model_config* cfg, uint64_t seed, int device, uint64_t* checksum,
                                      uint64_t* fingerprint) {
    return guard([&] {
        need(cfg, "cfg");
        validate_cfg(*cfg);
        uint64_t ck;
        if (device < 0) {
            ck = weights_checksum_stream(*cfg, seed);
        } else {
            TKV_CUDA(cudaSetDevice(device));
            ck = weights_checksum_device(*cfg, seed, 0);
        }
        if (checksum) *checksum = ck;
        if (fingerprint) *fingerprint = fingerprint_of(*cfg, ck);
    });
}

tkv_status tkv_debug_weight_rows(tkv_engine* e, int64_t layer, int which, int64_t row0, int64_t nrows, float* out) {
    return guard([&] {
        need(e, "engine");
        need(out, "out");
        e->bind();
        const void* base = nullptr;
        int64_t rows = 0, cols = 0;
        bool f32 = e->dt == DT::F32;
        if (which == 4 || which == 5) {
            rows = e->V, cols = e->hid;
            base = which == 4 ? e->w_lm : (const void*)e->emb;
            if (which == 5) f32 = true;
        } else {
            if (layer < 0 || layer >= e->L) fail(TKV_ERR_SHAPE, "layer out of range");
            const void* t[] = {e->w_qkv[layer], e->w_o[layer], e->w_gu[layer], e->w_down[layer]};
            const int64_t r[] = {e->nqkv, e->hid, 2 * e->I, e->hid}, c[] = {e->hid, e->qd, e->hid, e->I};
            if (which < 0 || which > 3) fail(TKV_ERR_DOMAIN, "which must be 0..5");
            base = t[which], rows = r[which], cols = c[which];
        }
        if (row0 < 0 || nrows < 0 || row0 + nrows > rows) fail(TKV_ERR_SHAPE, "rows out of range");
        const size_t es = f32 ? 4 : 2;
        DevMem tmp;
        tmp.ensure((size_t)(nrows * cols) * 4);
        launch_to_f32(static_cast<const uint8_t*>(base) + (size_t)(row0 * cols) * es, nrows * cols, tmp.as<float>(),
                      f32 ? DT::F32 : DT::BF16, e->stream);
        TKV_CUDA(cudaMemcpyAsync(out, tmp.p, (size_t)(nrows * cols) * 4, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
    });
}

tkv_status tkv_engine_check(tkv_engine* e) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        e->check_err("deferred device work");
    });
}

tkv_status tkv_naive_prefill(tkv_engine* e, const int32_t* framed, const int64_t* offsets, int64_t n_chunks,
                             const int32_t* query, int64_t nq, tkv_mask_mode mode, float* logits_out, tkv_flops* fl,
                             tkv_context** ctx_out) {
    return guard([&] {
        NvtxRange nvtx("tkv_naive_prefill");
        need(e, "engine");
        if (n_chunks > 0) {
            need(framed, "framed");
            need(offsets, "offsets");
        }
        if (mode != TKV_MASK_CAUSAL && mode != TKV_MASK_INDEPENDENT) fail(TKV_ERR_CONFIG, "unknown mask mode");
        e->bind();
        static const int64_t zero = 0;
        naive_impl(e, framed, n_chunks > 0 ? offsets : &zero, n_chunks, query, nq, mode, logits_out, fl, ctx_out);
    });
}

tkv_status tkv_naive_prefill_ids(tkv_engine* e, const uint64_t* ids, int64_t n, const int32_t* query, int64_t nq,
                                 tkv_mask_mode mode, float* logits_out, tkv_flops* fl, tkv_context** ctx_out) {
    return guard([&] {
        NvtxRange nvtx("tkv_naive_prefill_ids");
        need(e, "engine");
        std::vector<int32_t> toks;
        std::vector<int64_t> offs{0};
        for (int64_t i = 0; i < n; ++i) {
            auto it = e->chunks.find(ids[i]);
            if (it == e->chunks.end() || it->second.framed.empty())
                fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(ids[i]) + " has no token record");
            toks.insert(toks.end(), it->second.framed.begin(), it->second.framed.end());
            offs.push_back((int64_t)toks.size());
        }
        if (mode != TKV_MASK_CAUSAL && mode != TKV_MASK_INDEPENDENT) fail(TKV_ERR_CONFIG, "unknown mask mode");
        e->bind();
        naive_impl(e, toks.data(), offs.data(), n, query, nq, mode, logits_out, fl, ctx_out);
    });
}

tkv_status tkv_greedy_decode(tkv_engine* e, tkv_context* c, int64_t max_new, int32_t* tokens_out, int64_t* n_out) {
    return guard([&] {
        NvtxRange nvtx("tkv_greedy_decode");
        need(e, "engine");
        need(c, "context");
        if (max_new < 0) fail(TKV_ERR_DOMAIN, "greedy_decode: negative max_new");
        if ((int64_t)c->last_logits.size() != e->V) fail(TKV_ERR_DOMAIN, "greedy_decode: context has no logits yet");
        e->bind();
        int64_t n = 0;
        std::vector<float> lg((size_t)e->V);
        for (int64_t step = 0; step < max_new; ++step) {  // model.cpp:284-301
            int32_t best = 0;
            for (int64_t id = 1; id < e->V; ++id)
                if (c->last_logits[id] > c->last_logits[best]) best = (int32_t)id;
            if (best == 258) break;
            if (tokens_out) tokens_out[n] = best;
            ++n;
            extend(e, c, &best, nullptr, 1, lg.data(), nullptr);
        }
        if (n_out) *n_out = n;
    });
}

void tkv_context_destroy(tkv_context* c) {
    if (!c) return;
    if (c->eng) {
        c->eng->ctx_release(c->kv, c->kv_bytes);
        c->eng->live.erase(c);
    }
    delete c;
}

int64_t tkv_context_total_tokens(const tkv_context* c) { return c ? c->total : -1; }
int64_t tkv_context_next_position(const tkv_context* c) { return c ? c->next_position : -1; }

int64_t tkv_context_segments(const tkv_context* c, int64_t* lens, int32_t* is_query, int64_t cap) {
    if (!c) return -1;
    const int64_t n = (int64_t)c->seg_len.size();
    for (int64_t i = 0; i < n && i < cap; ++i) {
        if (lens) lens[i] = c->seg_len[i];
        if (is_query) is_query[i] = c->seg_query[i];
    }
    return n;
}

tkv_status tkv_context_positions(const tkv_context* c, int64_t* out, int64_t capacity) {
    return guard([&] {
        need(c, "context");
        if (capacity < (int64_t)c->positions.size()) fail(TKV_ERR_SHAPE, "positions buffer too small");
        if (!c->positions.empty()) std::memcpy(out, c->positions.data(), c->positions.size() * 8);
    });
}

tkv_status tkv_context_last_logits(const tkv_context* c, float* out, int64_t capacity) {
    return guard([&] {
        need(c, "context");
        if (c->last_logits.empty()) fail(TKV_ERR_DOMAIN, "context has no logits yet");
        if (capacity < (int64_t)c->last_logits.size()) fail(TKV_ERR_SHAPE, "logits buffer too small");
        std::memcpy(out, c->last_logits.data(), c->last_logits.size() * 4);
    });
}

tkv_status tkv_context_read_kv(const tkv_context* c, int64_t layer, tkv_kv_which which, int rotated, float* host_out,
                               int64_t capacity) {
    return guard([&] {
        need(c, "context");
        need(host_out, "host_out");
        tkv_engine* e = c->eng;
        if (!e) fail(TKV_ERR_GENERIC, "engine destroyed");
        if (layer < 0 || layer >= e->L) fail(TKV_ERR_SHAPE, "layer out of range");
        const int64_t rows = c->total;
        if (capacity < rows * e->kvd) fail(TKV_ERR_SHAPE, "host buffer too small");
        if (rows == 0) return;
        e->bind();
        DevMem f32;
        f32.ensure((size_t)rows * e->kvd * 4);
        tkv_context* cc = const_cast<tkv_context*>(c);
        if (which == TKV_V || rotated) {
            launch_to_f32(e->kv_plane(cc, layer, (int)which), rows * e->kvd, f32.as<float>(), e->dt, e->stream);
        } else {
            // injected rows: re-gather the unrotated store pages (identity rotation = bit-exact)
            if (c->chunk_rows > 0 && c->store_epoch != e->store_epoch)
                fail(TKV_ERR_STALE_CACHE, "store chunks were evicted since this context was assembled");
            if (c->chunk_rows > 0) {
                DevMem scratch, segs;
                const int64_t cap = c->chunk_rows;
                scratch.ensure((size_t)(e->L * 2 * cap * e->kvd) * dt_size(e->dt));
                segs.ensure(c->chunk_segs.size() * sizeof(GatherSeg));
                TKV_CUDA(cudaMemcpyAsync(segs.p, c->chunk_segs.data(), c->chunk_segs.size() * sizeof(GatherSeg),
                                         cudaMemcpyHostToDevice, e->stream));
                launch_gather_rope(e->pools, (int)e->page_tokens, segs.as<GatherSeg>(), (int)c->chunk_segs.size(),
                                   (int)e->L, (int)e->kvd, (int)e->d, e->rope.as<float2>(), scratch.p, cap, 0, e->dt,
                                   e->num_sms, e->stream);
                launch_to_f32(static_cast<uint8_t*>(scratch.p) + (size_t)(layer * 2 * cap) * e->kvd * dt_size(e->dt),
                              cap * e->kvd, f32.as<float>(), e->dt, e->stream);
                e->sync();
            }
            // the rest (query / naive rows): inverse rotation of the cached rotated keys
            const int64_t r0 = c->chunk_rows, nr = rows - r0;
            if (nr > 0) {
                std::vector<int32_t> pos(c->positions.begin() + r0, c->positions.end());
                DevMem dpos;
                dpos.ensure((size_t)nr * 4);
                TKV_CUDA(cudaMemcpyAsync(dpos.p, pos.data(), (size_t)nr * 4, cudaMemcpyHostToDevice, e->stream));
                launch_unrotate_rows(static_cast<uint8_t*>(e->kv_plane(cc, layer, 0)) + (size_t)r0 * e->kvd * dt_size(e->dt),
                                     (int)nr, (int)e->kvd, (int)e->d, dpos.as<int32_t>(), e->rope.as<float2>(),
                                     f32.as<float>() + r0 * e->kvd, e->dt, e->stream);
                e->sync();
            }
        }
        TKV_CUDA(cudaMemcpyAsync(host_out, f32.p, (size_t)rows * e->kvd * 4, cudaMemcpyDeviceToHost, e->stream));
        e->sync();
    });
}

tkv_status tkv_context_mask(const tkv_context* c, uint8_t* out, int64_t rows, int64_t cols) {
    return guard([&] {
        need(c, "context");
        need(out, "out");
        tkv_engine* e = c->eng;
        if (!e) fail(TKV_ERR_GENERIC, "engine destroyed");
        if (c->last_rows == 0) fail(TKV_ERR_DOMAIN, "no forward has run over this context yet");
        if (rows != c->last_rows || cols != c->last_cols)
            fail(TKV_ERR_SHAPE, "mask is " + std::to_string(c->last_rows) + "x" + std::to_string(c->last_cols));
        e->bind();
        DevMem lo, hi, m;
        lo.ensure((size_t)rows * 4);
        hi.ensure((size_t)rows * 4);
        m.ensure((size_t)(rows * cols));
        TKV_CUDA(cudaMemcpyAsync(lo.p, c->last_lo.data(), (size_t)rows * 4, cudaMemcpyHostToDevice, e->stream));
        TKV_CUDA(cudaMemcpyAsync(hi.p, c->last_hi.data(), (size_t)rows * 4, cudaMemcpyHostToDevice, e->stream));
        launch_mask_materialize(lo.as<int32_t>(), hi.as<int32_t>(), (int)rows, (int)cols, m.as<uint8_t>(), e->stream);
        TKV_CUDA(cudaMemcpyAsync(out, m.p, (size_t)(rows * cols), cudaMemcpyDeviceToHost, e->stream));
        e->sync();
    });
}

void* tkv_engine_stream(tkv_engine* e) { return e ? (void*)e->stream : nullptr; }

tkv_status tkv_profile_enable(tkv_engine* e, int on) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        e->prof_flush();
        e->prof_on = on != 0;
    });
}

tkv_status tkv_profile_read(tkv_engine* e, const char* cls, double* total_ms, int64_t* launches) {
    return guard([&] {
        need(e, "engine");
        need(cls, "class");
        e->bind();
        e->prof_flush();
        for (int i = 0; i < PC_N; ++i)
            if (std::strcmp(cls, kProfNames[i]) == 0) {
                if (total_ms) *total_ms = e->prof_ms[i];
                if (launches) *launches = e->prof_n[i];
                return;
            }
        fail(TKV_ERR_CONFIG, std::string("unknown kernel class ") + cls);
    });
}

tkv_status tkv_profile_reset(tkv_engine* e) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        e->prof_flush();
        for (int i = 0; i < PC_N; ++i) {
            e->prof_ms[i] = 0;
            e->prof_n[i] = 0;
        }
    });
}

int64_t tkv_launch_count(const tkv_engine* e) { return e ? e->launches : -1; }

tkv_status tkv_io_bytes(const tkv_engine* e, int64_t* h2d, int64_t* d2h) {
    return guard([&] {
        need(e, "engine");
        if (h2d) *h2d = e->h2d_bytes;
        if (d2h) *d2h = e->d2h_bytes;
    });
}

tkv_status tkv_debug_set_mask_rows(tkv_engine* e, const int64_t* rows, const int32_t* lo, const int32_t* hi, int64_t n) {
    return guard([&] {
        need(e, "engine");
        if (n > 0) {
            need(rows, "rows");
            need(lo, "lo");
            need(hi, "hi");
        }
        for (int64_t i = 0; i < n; ++i) {
            if (lo[i] < 0 || hi[i] < lo[i]) fail(TKV_ERR_DOMAIN, "mask override: need 0 <= lo <= hi");
            e->mask_override.push_back({rows[i], lo[i], hi[i]});
        }
    });
}

tkv_status tkv_debug_set_mask_fault(tkv_engine* e, int64_t row, int64_t col) {
    return guard([&] {
        need(e, "engine");
        // widen row `row` so it also sees column `col` (its range grows down to col)
        e->mask_override.push_back({row, -2, col});
    });
}

// ---- multi-GPU: document-sharded stores, remote chunks read over NVLink ----
namespace {
void check_slot(int32_t slot) {
    if (slot < 1 || slot >= kHostPool) fail(TKV_ERR_CONFIG, "peer slot must be in [1, " + std::to_string(kHostPool) + ")");
}
}  // namespace

tkv_status tkv_store_export_ipc(tkv_engine* e, tkv_ipc_handle* out, uint64_t* pool_bytes) {
    return guard([&] {
        need(e, "engine");
        need(out, "out");
        static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(tkv_ipc_handle), "ipc handle size");
        e->bind();
        cudaIpcMemHandle_t h;
        TKV_CUDA(cudaIpcGetMemHandle(&h, e->pool.p));
        std::memset(out, 0, sizeof *out);
        std::memcpy(out->bytes, &h, sizeof h);
        if (pool_bytes) *pool_bytes = (uint64_t)e->pool.n;
    });
}

tkv_status tkv_store_attach_ipc(tkv_engine* e, int32_t slot, const tkv_ipc_handle* h) {
    return guard([&] {
        need(e, "engine");
        need(h, "handle");
        check_slot(slot);
        e->bind();
        cudaIpcMemHandle_t mh;
        std::memcpy(&mh, h->bytes, sizeof mh);
        void* p = nullptr;
        TKV_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
        e->ipc_opened.push_back(p);
        e->pools.p[slot] = p;
    });
}

tkv_status tkv_store_attach_engine(tkv_engine* e, int32_t slot, tkv_engine* peer) {
    return guard([&] {
        need(e, "engine");
        need(peer, "peer");
        check_slot(slot);
        if (peer->fingerprint != e->fingerprint || peer->page_bytes != e->page_bytes)
            fail(TKV_ERR_STALE_CACHE, "peer store was built under a different model or page geometry");
        e->bind();
        if (peer->device != e->device) {
            int ok = 0;
            TKV_CUDA(cudaDeviceCanAccessPeer(&ok, e->device, peer->device));
            if (!ok) fail(TKV_ERR_CUDA, "no peer access between the two GPUs");
            const cudaError_t r = cudaDeviceEnablePeerAccess(peer->device, 0);
            if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) TKV_CUDA(r);
            cudaGetLastError();
        }
        e->pools.p[slot] = peer->pool.p;
        e->peer_pages[slot] = peer->n_pages;
    });
}

tkv_status tkv_store_chunk_pages(const tkv_engine* e, uint64_t id, int32_t* pages, int64_t capacity, int64_t* n_pages,
                                 int64_t* len) {
    return guard([&] {
        need(e, "engine");
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        if (it->second.slot != 0) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " is not owned by this store");
        const int64_t np = (int64_t)it->second.pages.size();
        if (n_pages) *n_pages = np;
        if (len) *len = it->second.len;
        if (pages) {
            if (capacity < np) fail(TKV_ERR_SHAPE, "pages buffer too small");
            std::memcpy(pages, it->second.pages.data(), (size_t)np * 4);
        }
    });
}

tkv_status tkv_store_register_remote(tkv_engine* e, uint64_t id, int32_t slot, int64_t len, const int32_t* pages,
                                     int64_t n_pages, const int32_t* framed) {
    return guard([&] {
        need(e, "engine");
        need(pages, "pages");
        check_slot(slot);
        if (!e->pools.p[slot]) fail(TKV_ERR_CONFIG, "peer slot " + std::to_string(slot) + " is not attached");
        if (len < 1 || n_pages != (len + e->page_tokens - 1) / e->page_tokens)
            fail(TKV_ERR_SHAPE, "remote chunk: page count does not match its length");
        if (e->peer_pages[slot] > 0)
            for (int64_t i = 0; i < n_pages; ++i)
                if (pages[i] < 0 || pages[i] >= e->peer_pages[slot])
                    fail(TKV_ERR_FORMAT, "remote chunk " + hex_id(id) + ": page index outside the peer pool");
        if (e->chunks.count(id)) return;  // already local (or registered): keep the local copy
        Chunk ch;
        ch.len = len;
        ch.slot = slot;
        ch.pages.assign(pages, pages + n_pages);
        if (framed) ch.framed.assign(framed, framed + len);
        e->chunks.emplace(id, std::move(ch));
    });
}

tkv_status tkv_store_fetch_remote(tkv_engine* e, uint64_t id) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        auto it = e->chunks.find(id);
        if (it == e->chunks.end()) fail(TKV_ERR_NOT_FOUND, "chunk " + hex_id(id) + " not in store");
        Chunk& ch = it->second;
        if (ch.slot == 0) return;
        Chunk local;
        local.len = ch.len;
        local.framed = ch.framed;
        store_chunk_pages(e, local);
        for (size_t p = 0; p < ch.pages.size(); ++p)  // page-sized copies over NVLink (copy engine)
            TKV_CUDA(cudaMemcpyAsync(page_ptr(e, local.slot, local.pages[p]), page_ptr(e, ch.slot, ch.pages[p]),
                                     e->page_bytes, cudaMemcpyDefault, e->stream));
        e->remote_bytes += (int64_t)(ch.pages.size() * e->page_bytes);
        e->sync();
        ch = std::move(local);
    });
}

int64_t tkv_remote_bytes(const tkv_engine* e) { return e ? e->remote_bytes : -1; }
// ---- directory blobs: the store exchange of a sharded deployment, behind the C ABI ----
}  // extern "C"
namespace {
constexpr uint32_t kDirVersion = 1;
struct Writer {
    std::vector<uint8_t> b;
    void raw(const void* p, size_t n) { b.insert(b.end(), (const uint8_t*)p, (const uint8_t*)p + n); }
    template <typename T>
    void v(T x) { raw(&x, sizeof x); }
};
struct Reader {
    const uint8_t* p;
    size_t n, at = 0;
    void raw(void* d, size_t k) {
        if (at + k > n) fail(TKV_ERR_FORMAT, "directory blob truncated");
        std::memcpy(d, p + at, k);
        at += k;
    }
    template <typename T>
    T v() {
        T x;
        raw(&x, sizeof x);
        return x;
    }
};
}  // namespace
extern "C" {

tkv_status tkv_store_export_directory(tkv_engine* e, uint8_t* buf, int64_t capacity, int64_t* size) {
    return guard([&] {
        need(e, "engine");
        need(size, "size");
        e->bind();
        Writer w;
        w.raw("TKVD", 4);
        w.v<uint32_t>(kDirVersion);
        w.v<uint64_t>(e->fingerprint);
        w.v<uint64_t>((uint64_t)e->page_bytes);
        w.v<int64_t>(e->page_tokens);
        w.v<int64_t>(e->n_pages);
        cudaIpcMemHandle_t h;
        TKV_CUDA(cudaIpcGetMemHandle(&h, e->pool.p));
        uint8_t hb[64] = {};
        std::memcpy(hb, &h, sizeof h);
        w.raw(hb, 64);
        std::vector<std::pair<uint64_t, Chunk*>> own;
        for (auto& kv : e->chunks)
            if (kv.second.slot == 0) own.emplace_back(kv.first, &kv.second);
        std::sort(own.begin(), own.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        w.v<int64_t>((int64_t)own.size());
        for (auto& [id, ch] : own) {
            w.v<uint64_t>(id);
            w.v<int64_t>(ch->len);
            w.v<int64_t>((int64_t)ch->pages.size());
            w.raw(ch->pages.data(), ch->pages.size() * 4);
            w.v<int64_t>((int64_t)ch->framed.size());
            w.raw(ch->framed.data(), ch->framed.size() * 4);
        }
        *size = (int64_t)w.b.size();
        if (!buf) return;  // size query
        if (capacity < *size) fail(TKV_ERR_SHAPE, "directory buffer too small");
        std::memcpy(buf, w.b.data(), w.b.size());
        for (auto& [id, ch] : own) ch->shared = true;  // peers will read these pages: no eviction from now on
    });
}

tkv_status tkv_store_import_directory(tkv_engine* e, int32_t slot, const uint8_t* blob, int64_t size) {
    return guard([&] {
        need(e, "engine");
        need(blob, "blob");
        check_slot(slot);
        e->bind();
        Reader r{blob, (size_t)size};
        char magic[4];
        r.raw(magic, 4);
        if (std::memcmp(magic, "TKVD", 4) != 0) fail(TKV_ERR_FORMAT, "not a store directory blob");
        if (r.v<uint32_t>() != kDirVersion) fail(TKV_ERR_FORMAT, "unsupported directory version");
        const uint64_t fp = r.v<uint64_t>(), page_bytes = r.v<uint64_t>();
        const int64_t page_tokens = r.v<int64_t>(), n_pages = r.v<int64_t>();
        uint8_t hb[64];
        r.raw(hb, 64);
        if (fp != e->fingerprint)
            fail(TKV_ERR_STALE_CACHE, "peer store was built under a different model fingerprint");
        if (page_bytes != (uint64_t)e->page_bytes || page_tokens != e->page_tokens || n_pages < 1)
            fail(TKV_ERR_STALE_CACHE, "peer store page geometry does not match this engine");
        struct Entry {
            uint64_t id;
            int64_t len;
            std::vector<int32_t> pages, framed;
        };
        std::vector<Entry> ents((size_t)std::max<int64_t>(0, r.v<int64_t>()));
        for (Entry& en : ents) {  // parse and validate everything before touching the engine
            en.id = r.v<uint64_t>();
            en.len = r.v<int64_t>();
            const int64_t np = r.v<int64_t>();
            if (en.len < 1 || np != (en.len + e->page_tokens - 1) / e->page_tokens)
                fail(TKV_ERR_FORMAT, "directory entry " + hex_id(en.id) + ": page count does not match its length");
            en.pages.resize((size_t)np);
            r.raw(en.pages.data(), (size_t)np * 4);
            for (int32_t pg : en.pages)
                if (pg < 0 || pg >= n_pages)
                    fail(TKV_ERR_FORMAT, "directory entry " + hex_id(en.id) + ": page index outside the peer pool");
            const int64_t nf = r.v<int64_t>();
            if (nf != 0 && nf != en.len) fail(TKV_ERR_FORMAT, "directory entry " + hex_id(en.id) + ": token record");
            en.framed.resize((size_t)nf);
            r.raw(en.framed.data(), (size_t)nf * 4);
        }
        if (!e->pools.p[slot]) {
            cudaIpcMemHandle_t mh;
            std::memcpy(&mh, hb, sizeof mh);
            void* p = nullptr;
            TKV_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
            e->ipc_opened.push_back(p);
            e->pools.p[slot] = p;
        }
        e->peer_pages[slot] = n_pages;
        for (Entry& en : ents) {
            if (e->chunks.count(en.id)) continue;  // already local (or registered): keep it
            Chunk ch;
            ch.len = en.len;
            ch.slot = slot;
            ch.pages = std::move(en.pages);
            ch.framed = std::move(en.framed);
            e->chunks.emplace(en.id, std::move(ch));
        }
    });
}


// ---- kernel-level test entry points ----
namespace {
struct DebugDev {
    explicit DebugDev(int device) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(TKV_ERR_CUDA, "no CUDA device");
        }
        TKV_CUDA(cudaSetDevice(device));
    }
};
void* to_dev_dt(DevMem& m, const float* host, int64_t n, DT dt) {
    DevMem f;
    f.ensure((size_t)n * 4);
    TKV_CUDA(cudaMemcpy(f.p, host, (size_t)n * 4, cudaMemcpyHostToDevice));
    m.ensure((size_t)n * dt_size(dt));
    launch_from_f32(f.as<float>(), n, m.p, dt, 0);
    TKV_CUDA(cudaDeviceSynchronize());
    return m.p;
}
}  // namespace

tkv_status tkv_debug_gemm(int device, tkv_dtype dtype, int use_tc, const float* A, const float* W, int64_t M,
                          int64_t N, int64_t K, int splits, float* out) {
    return guard([&] {
        need(A, "A");
        need(W, "W");
        need(out, "out");
        DebugDev dd(device);
        const DT dt = dtype == TKV_DTYPE_F32 ? DT::F32 : DT::BF16;
        if (use_tc && dt != DT::BF16) fail(TKV_ERR_CONFIG, "tcgen05 GEMM is bf16-only");
        if (use_tc && !gemm_tc_supported((int)M, (int)N, (int)K, (int)K)) fail(TKV_ERR_CONFIG, "unsupported shape");
        DevMem a, w, part, o;
        to_dev_dt(a, A, M * K, dt);
        to_dev_dt(w, W, N * K, dt);
        if (splits <= 0) splits = 1;
        part.ensure((size_t)splits * M * N * 4);
        o.ensure((size_t)M * N * 4);
        if (use_tc)
            splits = launch_gemm_tc(a.p, (int)K, w.p, (int)M, (int)N, (int)K, part.as<float>(), splits, 0);
        else
            launch_gemm_simt(a.p, (int)K, w.p, (int)M, (int)N, (int)K, part.as<float>(), splits, dt, 0);
        launch_reduce_splits(part.as<float>(), splits, M * N, o.as<float>(), 0);
        TKV_CUDA(cudaDeviceSynchronize());
        TKV_CUDA(cudaMemcpy(out, o.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
    });
}

tkv_status tkv_debug_attn_trace(int on, uint64_t* out, int64_t capacity) {
    return guard([&] {
        unsigned long long* buf = nullptr;
        if (out) {  // read back the last trace
            attn_trace_enable(true, &buf);
            TKV_CUDA(cudaDeviceSynchronize());
            TKV_CUDA(cudaMemcpy(out, buf, (size_t)std::min<int64_t>(capacity, attn_trace_words()) * 8, cudaMemcpyDeviceToHost));
        }
        attn_trace_enable(on != 0, &buf);
    });
}

tkv_status tkv_kernel_timeline(tkv_engine* e, int on, uint64_t* out, int32_t* classes, int64_t capacity,
                               int64_t* n_launches) {
    return guard([&] {
        need(e, "engine");
        e->bind();
        if (on) {
            e->tl_buf.ensure((size_t)tkv_engine::kTlMax * 16);
            // slot[0] starts at ~0 (atomicMin), slot[1] at 0 (atomicMax): two strided memsets
            TKV_CUDA(cudaMemset2DAsync(e->tl_buf.p, 16, 0xFF, 8, tkv_engine::kTlMax, e->stream));
            TKV_CUDA(cudaMemset2DAsync(static_cast<uint8_t*>(e->tl_buf.p) + 8, 16, 0, 8, tkv_engine::kTlMax, e->stream));
            g_tl = TimelineState{};
            g_tl.base = e->tl_buf.as<unsigned long long>();
            g_tl.cap = tkv_engine::kTlMax;
            return;
        }
        const int64_t n = g_tl.n;
        std::vector<int32_t> cls = g_tl.classes;
        g_tl = TimelineState{};
        e->sync();
        if (n_launches) *n_launches = n;
        const int64_t m = std::min<int64_t>(capacity, n);
        if (out && m > 0) TKV_CUDA(cudaMemcpy(out, e->tl_buf.p, (size_t)m * 16, cudaMemcpyDeviceToHost));
        if (classes && m > 0) std::memcpy(classes, cls.data(), (size_t)m * sizeof(int32_t));
    });
}

tkv_status tkv_debug_gemm_trace(int on, uint64_t* out, int64_t capacity) {
    return guard([&] { gemm_trace_enable(on != 0, reinterpret_cast<unsigned long long*>(out), capacity); });
}

tkv_status tkv_debug_set_gemm_knobs(int stages, int smem_kb, int ctas_per_sm, int w_evict_first) {
    return guard([&] { set_gemm_knobs(stages, smem_kb, ctas_per_sm, w_evict_first); });
}

// Device-resident GEMM timing: buffers filled on the device (no host copies), `iters` back-to-back
// launches timed with CUDA events; returns the mean ms per launch.
tkv_status tkv_debug_gemm_bench(int device, int64_t M, int64_t N, int64_t K, int splits, int swiglu, int iters,
                                double* ms_per_launch) {
    return guard([&] {
        DebugDev dd(device);
        DevMem a, w, part, act, ssp;
        a.ensure((size_t)M * K * 2);
        w.ensure((size_t)N * K * 2);
        launch_init_transposed(a.p, DT::BF16, 1, 0, K, M, 0.01, 0);
        launch_init_transposed(w.p, DT::BF16, 2, 0, K, N, 0.01, 0);
        if (swiglu & 2) TKV_CUDA(cudaMemset(w.p, 0, (size_t)N * K * 2));  // constant weights (data-dependence probe)
        if (swiglu & 4) TKV_CUDA(cudaMemset(a.p, 0, (size_t)M * K * 2));
        swiglu &= 1;
        const int nb = norm_blocks((int)K);
        ssp.ensure((size_t)M * nb * 4);
        launch_fill_f32(ssp.as<float>(), 1.0f, M * nb, 0);
        if (splits < 1) splits = 1;
        part.ensure((size_t)splits * M * N * 4);
        act.ensure((size_t)M * (N / 2) * 2);
        cudaStream_t st;
        TKV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        TKV_CUDA(cudaDeviceSynchronize());
        auto run = [&] {
            if (swiglu)
                launch_gemm_tc(a.p, (int)K, w.p, (int)M, (int)N, (int)K, nullptr, 1, st, act.p, ssp.as<float>(), nb,
                               1e-6f, N % 256 == 0 ? 128 : 64);
            else
                launch_gemm_tc(a.p, (int)K, w.p, (int)M, (int)N, (int)K, part.as<float>(), splits, st);
        };
        for (int i = 0; i < 3; ++i) run();
        cudaEvent_t e0, e1;
        TKV_CUDA(cudaEventCreate(&e0));
        TKV_CUDA(cudaEventCreate(&e1));
        TKV_CUDA(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i) run();
        TKV_CUDA(cudaEventRecord(e1, st));
        TKV_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        TKV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *ms_per_launch = ms / iters;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
    });
}

tkv_status tkv_debug_attention(int device, tkv_dtype dtype, int impl, const float* q, const float* k, const float* v,
                               const int32_t* lo, const int32_t* hi, int64_t Tq, int64_t Tk, int64_t H, int64_t Hkv,
                               int64_t d, float* out) {
    return guard([&] {
        DebugDev dd(device);
        const DT dt = dtype == TKV_DTYPE_F32 ? DT::F32 : DT::BF16;
        DevMem dq, dk, dv, dlo, dhi, dout, of, ws, errm;
        to_dev_dt(dq, q, Tq * H * d, dt);
        to_dev_dt(dk, k, Tk * Hkv * d, dt);
        to_dev_dt(dv, v, Tk * Hkv * d, dt);
        dlo.ensure((size_t)Tq * 4);
        dhi.ensure((size_t)Tq * 4);
        TKV_CUDA(cudaMemcpy(dlo.p, lo, (size_t)Tq * 4, cudaMemcpyHostToDevice));
        TKV_CUDA(cudaMemcpy(dhi.p, hi, (size_t)Tq * 4, cudaMemcpyHostToDevice));
        dout.ensure((size_t)Tq * H * d * dt_size(dt));
        of.ensure((size_t)Tq * H * d * 4);
        errm.ensure(4);
        TKV_CUDA(cudaMemset(errm.p, 0, 4));
        int dev_sms = 148;
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
        const bool dec = impl == 2;  // decode-sized kernel (attn_decode.cu)
        if (dec && !attention_decode_supported((int)Tq, (int)H, (int)Hkv, (int)d, dt))
            fail(TKV_ERR_CONFIG, "decode attention needs bf16, d = 128 and Tq * H / Hkv in {4, 7, 8, 16}");
        const bool tc = impl == 0 && attention_tc_supported((int)d, dt);
        const int splits = tc ? attn_tc_pick_splits((int)Tq, (int)H, (int)Hkv, (int)Tk, dev_sms)
                              : dec ? attn_decode_pick_splits((int)Tk, (int)Hkv, dev_sms)
                                    : attn_pick_splits((int)Tq, (int)H, (int)Hkv, (int)Tk, dev_sms);
        AttnWork w;
        if (splits > 1) {
            size_t mloff = (size_t)splits * Tq * H * d;
            ws.ensure((tc ? attn_tc_workspace_floats((int)Tq, (int)H, (int)Hkv, splits, &mloff)
                          : attn_workspace_floats((int)Tq, (int)H, (int)d, splits)) * 4);
            w.o = ws.as<float>();
            w.ml = w.o + mloff;
        }
        auto run = [&] {
            if (dec)
                launch_attention_decode(dq.p, dk.p, dv.p, (int)(Hkv * d), dlo.as<int32_t>(), dhi.as<int32_t>(),
                                        dout.p, (int)Tq, (int)Tk, (int)H, (int)Hkv, splits, w, errm.as<int>(), 0);
            else if (tc)
                launch_attention_tc(dq.p, dk.p, dv.p, (int)(Hkv * d), dlo.as<int32_t>(), dhi.as<int32_t>(), dout.p,
                                    (int)Tq, (int)Tk, (int)H, (int)Hkv, splits, w, errm.as<int>(), 0, (int)Tk);
            else
                launch_attention_simt(dq.p, dk.p, dv.p, (int)(Hkv * d), dlo.as<int32_t>(), dhi.as<int32_t>(),
                                      dout.p, (int)Tq, (int)Tk, (int)H, (int)Hkv, (int)d, splits, w,
                                      errm.as<int>(), dt, 0);
        };
        run();
        if (const char* it = getenv("TKV_DEBUG_TIME_ITERS")) {  // warm timing (tools/decode_time.py)
            const int iters = atoi(it);
            DevMem flush;
            flush.ensure((size_t)256 << 20);  // > L2: every timed launch streams K/V from HBM
            cudaEvent_t e0, e1;
            TKV_CUDA(cudaEventCreate(&e0));
            TKV_CUDA(cudaEventCreate(&e1));
            float tot = 0.f;
            for (int i = 0; i < iters; ++i) {
                TKV_CUDA(cudaMemsetAsync(flush.p, i & 0xff, (size_t)256 << 20, 0));
                TKV_CUDA(cudaEventRecord(e0, 0));
                run();
                TKV_CUDA(cudaEventRecord(e1, 0));
                TKV_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                TKV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                tot += ms;
            }
            fprintf(stderr, "debug_attention impl %d splits %d: %.2f us per launch (L2 flushed)\n", impl, splits,
                    1000.f * tot / iters);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        launch_to_f32(dout.p, Tq * H * d, of.as<float>(), dt, 0);
        TKV_CUDA(cudaDeviceSynchronize());
        int e = 0;
        TKV_CUDA(cudaMemcpy(&e, errm.p, 4, cudaMemcpyDeviceToHost));
        if (e & 8) fail(TKV_ERR_DEGENERATE_ROW, "attention: row with no attendable positions");
        TKV_CUDA(cudaMemcpy(out, of.p, (size_t)Tq * H * d * 4, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"

/* TEST INFRASTRUCTURE ONLY — CPU oracle (float64 C restatement of the
 * reference turbokv prefill path). See tkv_oracle.h for the contract and the
 * rules on who may load this. Every function cites the reference file:line
 * it restates (paths relative to /root/reference/proj).
 *
 * Bit-parity notes: the per-element operation order of matmul, rmsnorm,
 * softmax, attention and RoPE follows the reference exactly, and this file
 * is built with the same plain -O2 (no FMA contraction on baseline x86-64),
 * so outputs equal the reference's bit for bit. OpenMP only splits work
 * across independent output elements; it never reorders a reduction.
 */
#include "tkv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* tko_last_error(void) { return g_err; }

/* ---- SplitMix64 / FNV-1a (include/turbokv/rng.hpp:14-78) ---- */
#define PHI 0x9E3779B97F4A7C15ULL

uint64_t tko_splitmix_at(uint64_t seed, uint64_t index) {
    uint64_t z = seed + (index + 1) * PHI;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t h;
} fnv;
static void fnv_init(fnv* f) { f->h = 0xCBF29CE484222325ULL; }
static void fnv_u32(fnv* f, uint32_t v) {
    for (int i = 0; i < 4; ++i) {
        f->h ^= (v >> (8 * i)) & 0xFF;
        f->h *= 0x100000001B3ULL;
    }
}
static void fnv_u64(fnv* f, uint64_t v) {
    fnv_u32(f, (uint32_t)v);
    fnv_u32(f, (uint32_t)(v >> 32));
}
static void fnv_f64(fnv* f, double v) {
    uint64_t b;
    memcpy(&b, &v, 8);
    fnv_u64(f, b);
}

/* ---- config (src/config.cpp:9-42) ---- */
int tko_config_validate(const tko_config* c) {
    if (c->layer_num < 1 || c->head_num < 1 || c->kv_head_num < 1 || c->head_size < 1 || c->hidden_size < 1 ||
        c->intermediate_size < 1 || c->vocab_size < 1)
        return fail(4, "ModelConfig: all counts must be >= 1");
    if (c->hidden_size != c->head_num * c->head_size) return fail(4, "ModelConfig: hidden != head_num*head_size");
    if (c->head_num % c->kv_head_num != 0) return fail(4, "ModelConfig: head_num not divisible by kv_head_num");
    if (c->head_size % 2 != 0) return fail(4, "ModelConfig: head_size must be even");
    if (!(c->rope_base > 0.0) || c->norm_eps < 0.0) return fail(4, "ModelConfig: rope_base/norm_eps");
    return 0;
}

uint64_t tko_fingerprint_seed(const tko_config* c) {
    fnv f;
    fnv_init(&f);
    fnv_u64(&f, (uint64_t)c->layer_num);
    fnv_u64(&f, (uint64_t)c->head_num);
    fnv_u64(&f, (uint64_t)c->kv_head_num);
    fnv_u64(&f, (uint64_t)c->head_size);
    fnv_u64(&f, (uint64_t)c->hidden_size);
    fnv_u64(&f, (uint64_t)c->intermediate_size);
    fnv_u64(&f, (uint64_t)c->vocab_size);
    fnv_f64(&f, c->rope_base);
    fnv_f64(&f, c->norm_eps);
    return f.h;
}

/* chunk_content_id (src/kvstore.cpp:58-64) */
uint64_t tko_chunk_content_id(uint64_t fp, const int32_t* framed, int64_t n) {
    fnv f;
    fnv_init(&f);
    fnv_u64(&f, fp);
    fnv_u64(&f, (uint64_t)n);
    for (int64_t i = 0; i < n; ++i) fnv_u32(&f, (uint32_t)framed[i]);
    return f.h;
}

/* ---- model weights (src/model.cpp:68-118) ---- */
typedef struct {
    double *wq, *wk, *wv, *wo, *gate, *up, *down;
} layer_w;

struct tko_model {
    tko_config c;
    uint64_t seed;
    double* emb;
    layer_w* layers;
    double* lm_head;
    double* ones; /* every norm vector is 1.0 (init_random, model.cpp:79-80,89) */
    int have_checksum;
    uint64_t checksum;
};

static double* draw(uint64_t seed, uint64_t* cursor, int64_t rows, int64_t cols, double scale) {
    double* m = (double*)malloc((size_t)(rows * cols) * sizeof(double));
    if (!m) return NULL;
    const uint64_t base = *cursor;
    const int64_t n = rows * cols;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double u = (double)(tko_splitmix_at(seed, base + (uint64_t)i) >> 11) * 0x1.0p-53;
        m[i] = (2.0 * u - 1.0) * scale; /* next_signed() * scale, model.cpp:15-21 */
    }
    *cursor += (uint64_t)n;
    return m;
}

int tko_model_create(const tko_config* c, uint64_t seed, tko_model** out) {
    int rc = tko_config_validate(c);
    if (rc) return rc;
    tko_model* m = (tko_model*)calloc(1, sizeof *m);
    m->c = *c;
    m->seed = seed;
    const double scale = 1.0 / sqrt((double)c->hidden_size);
    const int64_t qd = c->head_num * c->head_size, kvd = c->kv_head_num * c->head_size;
    uint64_t cur = 0;
    m->emb = draw(seed, &cur, c->vocab_size, c->hidden_size, scale);
    m->layers = (layer_w*)calloc((size_t)c->layer_num, sizeof(layer_w));
    for (int64_t l = 0; l < c->layer_num; ++l) {
        layer_w* L = &m->layers[l];
        L->wq = draw(seed, &cur, c->hidden_size, qd, scale);
        L->wk = draw(seed, &cur, c->hidden_size, kvd, scale);
        L->wv = draw(seed, &cur, c->hidden_size, kvd, scale);
        L->wo = draw(seed, &cur, qd, c->hidden_size, scale);
        L->gate = draw(seed, &cur, c->hidden_size, c->intermediate_size, scale);
        L->up = draw(seed, &cur, c->hidden_size, c->intermediate_size, scale);
        L->down = draw(seed, &cur, c->intermediate_size, c->hidden_size, scale);
        if (!L->wq || !L->wk || !L->wv || !L->wo || !L->gate || !L->up || !L->down) {
            tko_model_destroy(m);
            return fail(12, "oracle: out of host memory for weights");
        }
    }
    m->lm_head = draw(seed, &cur, c->hidden_size, c->vocab_size, scale);
    int64_t big = c->hidden_size > c->intermediate_size ? c->hidden_size : c->intermediate_size;
    m->ones = (double*)malloc((size_t)big * sizeof(double));
    for (int64_t i = 0; i < big; ++i) m->ones[i] = 1.0;
    *out = m;
    return 0;
}

void tko_model_destroy(tko_model* m) {
    if (!m) return;
    free(m->emb);
    if (m->layers) {
        for (int64_t l = 0; l < m->c.layer_num; ++l) {
            layer_w* L = &m->layers[l];
            free(L->wq);
            free(L->wk);
            free(L->wv);
            free(L->wo);
            free(L->gate);
            free(L->up);
            free(L->down);
        }
    }
    free(m->layers);
    free(m->lm_head);
    free(m->ones);
    free(m);
}

static void ck_vec(fnv* f, const double* v, int64_t n) {
    fnv_u64(f, (uint64_t)n);
    for (int64_t i = 0; i < n; ++i) fnv_f64(f, v[i]);
}
static void ck_mat(fnv* f, const double* v, int64_t r, int64_t c) {
    fnv_u64(f, (uint64_t)r);
    fnv_u64(f, (uint64_t)c);
    for (int64_t i = 0; i < r * c; ++i) fnv_f64(f, v[i]);
}

/* weights_checksum (model.cpp:94-112) */
uint64_t tko_weights_checksum(tko_model* m) {
    if (m->have_checksum) return m->checksum;
    const tko_config* c = &m->c;
    const int64_t qd = c->head_num * c->head_size, kvd = c->kv_head_num * c->head_size, H = c->hidden_size;
    fnv f;
    fnv_init(&f);
    ck_mat(&f, m->emb, c->vocab_size, H);
    for (int64_t l = 0; l < c->layer_num; ++l) {
        layer_w* L = &m->layers[l];
        ck_vec(&f, m->ones, H);
        ck_vec(&f, m->ones, H);
        ck_mat(&f, L->wq, H, qd);
        ck_mat(&f, L->wk, H, kvd);
        ck_mat(&f, L->wv, H, kvd);
        ck_mat(&f, L->wo, qd, H);
        ck_mat(&f, L->gate, H, c->intermediate_size);
        ck_mat(&f, L->up, H, c->intermediate_size);
        ck_mat(&f, L->down, c->intermediate_size, H);
    }
    ck_vec(&f, m->ones, H);
    ck_mat(&f, m->lm_head, H, c->vocab_size);
    m->checksum = f.h;
    m->have_checksum = 1;
    return f.h;
}

/* weights_checksum (model.cpp:94-112) over init_random's draws (model.cpp:68-92) WITHOUT materialising the
 * weights: the same bytes in the same order, each value drawn on the fly (full-size models are 52 GB of f64). */
static void ck_draws(fnv* f, uint64_t seed, uint64_t* cursor, int64_t r, int64_t c, double scale) {
    fnv_u64(f, (uint64_t)r);
    fnv_u64(f, (uint64_t)c);
    const uint64_t n = (uint64_t)(r * c);
    for (uint64_t i = 0; i < n; ++i) {
        const double u = (double)(tko_splitmix_at(seed, *cursor + i) >> 11) * 0x1.0p-53;
        fnv_f64(f, (2.0 * u - 1.0) * scale);
    }
    *cursor += n;
}
static void ck_ones(fnv* f, int64_t n) {
    fnv_u64(f, (uint64_t)n);
    for (int64_t i = 0; i < n; ++i) fnv_f64(f, 1.0);
}
uint64_t tko_weights_checksum_stream(const tko_config* c, uint64_t seed) {
    const int64_t qd = c->head_num * c->head_size, kvd = c->kv_head_num * c->head_size, H = c->hidden_size;
    const int64_t I = c->intermediate_size;
    const double scale = 1.0 / sqrt((double)H);
    uint64_t cur = 0;
    fnv f;
    fnv_init(&f);
    ck_draws(&f, seed, &cur, c->vocab_size, H, scale);
    for (int64_t l = 0; l < c->layer_num; ++l) {
        ck_ones(&f, H);
        ck_ones(&f, H);
        ck_draws(&f, seed, &cur, H, qd, scale);
        ck_draws(&f, seed, &cur, H, kvd, scale);
        ck_draws(&f, seed, &cur, H, kvd, scale);
        ck_draws(&f, seed, &cur, qd, H, scale);
        ck_draws(&f, seed, &cur, H, I, scale);
        ck_draws(&f, seed, &cur, H, I, scale);
        ck_draws(&f, seed, &cur, I, H, scale);
    }
    ck_ones(&f, H);
    ck_draws(&f, seed, &cur, H, c->vocab_size, scale);
    return f.h;
}

/* model_fingerprint (model.cpp:114-118) from a streamed checksum */
uint64_t tko_fingerprint_of(const tko_config* c, uint64_t checksum) {
    fnv f;
    fnv_init(&f);
    fnv_u64(&f, tko_fingerprint_seed(c));
    fnv_u64(&f, checksum);
    return f.h;
}

/* model_fingerprint (model.cpp:114-118) */
uint64_t tko_model_fingerprint(tko_model* m) {
    fnv f;
    fnv_init(&f);
    fnv_u64(&f, tko_fingerprint_seed(&m->c));
    fnv_u64(&f, tko_weights_checksum(m));
    return f.h;
}

const double* tko_weight(const tko_model* m, int64_t layer, int which, int64_t* rows, int64_t* cols) {
    const tko_config* c = &m->c;
    const int64_t qd = c->head_num * c->head_size, kvd = c->kv_head_num * c->head_size, H = c->hidden_size,
                  I = c->intermediate_size;
    if (which == 0) { *rows = c->vocab_size; *cols = H; return m->emb; }
    if (which == 8) { *rows = H; *cols = c->vocab_size; return m->lm_head; }
    if (layer < 0 || layer >= c->layer_num) return NULL;
    const layer_w* L = &m->layers[layer];
    switch (which) {
        case 1: *rows = H; *cols = qd; return L->wq;
        case 2: *rows = H; *cols = kvd; return L->wk;
        case 3: *rows = H; *cols = kvd; return L->wv;
        case 4: *rows = qd; *cols = H; return L->wo;
        case 5: *rows = H; *cols = I; return L->gate;
        case 6: *rows = H; *cols = I; return L->up;
        case 7: *rows = I; *cols = H; return L->down;
    }
    return NULL;
}

/* ---- numerics (src/numerics.cpp) ---- */

/* matmul, i-k-j order with ascending-k accumulation per element (numerics.cpp:8-29). */
static int matmul(const double* a, const double* b, double* c, int64_t m, int64_t k, int64_t n) {
    const int64_t JB = 256;
    const int64_t nb = (n + JB - 1) / JB;
    int bad = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
    for (int64_t t = 0; t < m * nb; ++t) {
        const int64_t i = t / nb, j0 = (t % nb) * JB, j1 = j0 + JB < n ? j0 + JB : n;
        double* ci = c + i * n;
        const double* ai = a + i * k;
        for (int64_t j = j0; j < j1; ++j) ci[j] = 0.0;
        for (int64_t p = 0; p < k; ++p) {
            const double aip = ai[p];
            const double* bp = b + p * n;
            for (int64_t j = j0; j < j1; ++j) ci[j] += aip * bp[j];
        }
        for (int64_t j = j0; j < j1; ++j)
            if (!isfinite(ci[j])) bad = 1;
    }
    return bad ? fail(3, "matmul: non-finite element") : 0;
}

/* rmsnorm_rows (numerics.cpp:84-101) */
static int rmsnorm_rows(const double* x, const double* w, double* out, int64_t rows, int64_t cols, double eps) {
    int bad = 0;
    for (int64_t i = 0; i < rows; ++i) {
        const double* xi = x + i * cols;
        double ss = 0.0;
        for (int64_t j = 0; j < cols; ++j) ss += xi[j] * xi[j];
        const double scale = 1.0 / sqrt(ss / (double)cols + eps);
        double* oi = out + i * cols;
        for (int64_t j = 0; j < cols; ++j) {
            oi[j] = xi[j] * scale * w[j];
            if (!isfinite(oi[j])) bad = 1;
        }
    }
    return bad ? fail(3, "rmsnorm_rows: non-finite element") : 0;
}

/* ---- RoPE (src/rope.cpp:8-46,75-88): interleaved pairs (2m, 2m+1) ---- */
int tko_rope_rotate(double* rows, int64_t n_rows, int64_t cols, const int64_t* positions, int64_t d, double base) {
    if (d <= 0 || d % 2 != 0) return fail(4, "RopeParams: head_size must be positive and even");
    if (cols % d != 0) return fail(2, "rope_rotate_heads: cols not a multiple of head_size");
    for (int64_t i = 0; i < n_rows; ++i)
        if (positions[i] < 0) return fail(3, "rope: negative position");
    const int64_t half = d / 2, heads = cols / d;
    double* theta = (double*)malloc((size_t)half * sizeof(double));
    for (int64_t m = 0; m < half; ++m) theta[m] = pow(base, -2.0 * (double)m / (double)d);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i) {
        const double t = (double)positions[i];
        for (int64_t h = 0; h < heads; ++h) {
            double* row = rows + i * cols + h * d;
            for (int64_t m = 0; m < half; ++m) {
                const double angle = t * theta[m];
                const double c = cos(angle), s = sin(angle);
                const double x0 = row[2 * m], x1 = row[2 * m + 1];
                row[2 * m] = x0 * c - x1 * s;
                row[2 * m + 1] = x0 * s + x1 * c;
            }
        }
    }
    free(theta);
    return 0;
}

/* ---- attention (src/attention.cpp:94-169 + numerics.cpp:31-60) ----
 * GQA: head h reads kv group h / (H/Hkv). Scores skip masked columns; softmax
 * subtracts the row max, exponentiates, multiplies by 1/sum; PV skips zero
 * weights. Row i sees columns [lo[i], hi[i]]. */
static int attend(const double* q, int64_t tq, const double* k, const double* v, int64_t tk, int64_t H,
                  int64_t Hkv, int64_t d, const int64_t* lo, const int64_t* hi, double* out) {
    const int64_t group = H / Hkv, qc = H * d, kc = Hkv * d;
    const double scale = 1.0 / sqrt((double)d);
    int rc = 0;
    memset(out, 0, (size_t)(tq * qc) * sizeof(double));
#pragma omp parallel reduction(max : rc)
    {
        double* s = (double*)malloc((size_t)(tk > 0 ? tk : 1) * sizeof(double));
#pragma omp for schedule(dynamic) collapse(2)
        for (int64_t h = 0; h < H; ++h) {
            for (int64_t i = 0; i < tq; ++i) {
                const int64_t g = h / group;
                const double* qi = q + i * qc + h * d;
                double mx = -INFINITY;
                for (int64_t j = 0; j < tk; ++j) {
                    if (j < lo[i] || j > hi[i]) {
                        s[j] = -INFINITY;
                        continue;
                    }
                    const double* kj = k + j * kc + g * d;
                    double dot = 0.0;
                    for (int64_t e = 0; e < d; ++e) dot += qi[e] * kj[e];
                    s[j] = dot * scale + 0.0;
                    if (s[j] > mx) mx = s[j];
                }
                if (mx == -INFINITY) {
                    rc = 5; /* DegenerateRowError */
                    continue;
                }
                double sum = 0.0;
                for (int64_t j = 0; j < tk; ++j) {
                    if (s[j] == -INFINITY) {
                        s[j] = 0.0;
                    } else {
                        s[j] = exp(s[j] - mx);
                        sum += s[j];
                    }
                }
                const double inv = 1.0 / sum;
                for (int64_t j = 0; j < tk; ++j) s[j] *= inv;
                double* oi = out + i * qc + h * d;
                for (int64_t j = 0; j < tk; ++j) {
                    const double w = s[j];
                    if (w == 0.0) continue;
                    const double* vj = v + j * kc + g * d;
                    for (int64_t e = 0; e < d; ++e) oi[e] += w * vj[e];
                }
            }
        }
        free(s);
    }
    if (rc == 5) return fail(5, "softmax_rows: row has no attendable positions");
    for (int64_t i = 0; i < tq * qc; ++i)
        if (!isfinite(out[i])) return fail(3, "attend: non-finite element");
    return 0;
}

/* ---- forward_tokens (src/model.cpp:198-272) ---- */
int tko_forward(const tko_model* m, const int32_t* tokens, int64_t n, const int64_t* positions,
                const double* past_k, const double* past_v, const int64_t* past_positions, int64_t n_past,
                const int64_t* row_lo, const int64_t* row_hi, double* logits, int last_only, double* new_k,
                double* new_v) {
    const tko_config* c = &m->c;
    if (n == 0) return fail(3, "forward_tokens: empty token list");
    for (int64_t i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= c->vocab_size) return fail(3, "token id outside vocab");
    const int64_t Hd = c->hidden_size, H = c->head_num, Hkv = c->kv_head_num, d = c->head_size;
    const int64_t qd = H * d, kvd = Hkv * d, I = c->intermediate_size, tk = n_past + n;
    int rc = 0;

    int64_t* all_pos = (int64_t*)malloc((size_t)tk * sizeof(int64_t));
    for (int64_t j = 0; j < n_past; ++j) all_pos[j] = past_positions[j];
    for (int64_t j = 0; j < n; ++j) all_pos[n_past + j] = positions[j];

    double* x = (double*)malloc((size_t)(n * Hd) * sizeof(double));
    double* h = (double*)malloc((size_t)(n * Hd) * sizeof(double));
    double* q = (double*)malloc((size_t)(n * qd) * sizeof(double));
    double* kall = (double*)malloc((size_t)(tk * kvd) * sizeof(double));
    double* vall = (double*)malloc((size_t)(tk * kvd) * sizeof(double));
    double* att = (double*)malloc((size_t)(n * qd) * sizeof(double));
    double* tmp = (double*)malloc((size_t)(n * Hd) * sizeof(double));
    double* g = (double*)malloc((size_t)(n * I) * sizeof(double));
    double* u = (double*)malloc((size_t)(n * I) * sizeof(double));
    if (!x || !h || !q || !kall || !vall || !att || !tmp || !g || !u) {
        rc = fail(12, "oracle: out of host memory");
        goto done;
    }
    for (int64_t i = 0; i < n; ++i) memcpy(x + i * Hd, m->emb + (int64_t)tokens[i] * Hd, (size_t)Hd * sizeof(double));

    for (int64_t l = 0; l < c->layer_num; ++l) {
        const layer_w* L = &m->layers[l];
        if ((rc = rmsnorm_rows(x, m->ones, h, n, Hd, c->norm_eps))) goto done;
        if ((rc = matmul(h, L->wq, q, n, Hd, qd))) goto done;
        if (n_past) {
            memcpy(kall, past_k + l * n_past * kvd, (size_t)(n_past * kvd) * sizeof(double));
            memcpy(vall, past_v + l * n_past * kvd, (size_t)(n_past * kvd) * sizeof(double));
        }
        double* kn = kall + n_past * kvd;
        double* vn = vall + n_past * kvd;
        if ((rc = matmul(h, L->wk, kn, n, Hd, kvd))) goto done;
        if ((rc = matmul(h, L->wv, vn, n, Hd, kvd))) goto done;
        /* K leaves the layer unrotated (model.cpp:250-262) */
        if (new_k) memcpy(new_k + l * n * kvd, kn, (size_t)(n * kvd) * sizeof(double));
        if (new_v) memcpy(new_v + l * n * kvd, vn, (size_t)(n * kvd) * sizeof(double));
        if ((rc = tko_rope_rotate(q, n, qd, positions, d, c->rope_base))) goto done;
        if ((rc = tko_rope_rotate(kall, tk, kvd, all_pos, d, c->rope_base))) goto done;
        if ((rc = attend(q, n, kall, vall, tk, H, Hkv, d, row_lo, row_hi, att))) goto done;
        if ((rc = matmul(att, L->wo, tmp, n, qd, Hd))) goto done;
        for (int64_t i = 0; i < n * Hd; ++i) x[i] = x[i] + tmp[i];
        if ((rc = rmsnorm_rows(x, m->ones, h, n, Hd, c->norm_eps))) goto done;
        /* swiglu_rows (numerics.cpp:107-124) */
        if ((rc = matmul(h, L->gate, g, n, Hd, I))) goto done;
        if ((rc = matmul(h, L->up, u, n, Hd, I))) goto done;
        for (int64_t i = 0; i < n * I; ++i) g[i] = (g[i] / (1.0 + exp(-g[i]))) * u[i];
        if ((rc = matmul(g, L->down, tmp, n, I, Hd))) goto done;
        for (int64_t i = 0; i < n * Hd; ++i) x[i] = x[i] + tmp[i];
    }
    if (logits) {
        const int64_t r0 = last_only ? n - 1 : 0, nr = last_only ? 1 : n;
        if ((rc = rmsnorm_rows(x + r0 * Hd, m->ones, h, nr, Hd, c->norm_eps))) goto done;
        if ((rc = matmul(h, m->lm_head, logits, nr, Hd, c->vocab_size))) goto done;
    }
done:
    free(all_pos);
    free(x);
    free(h);
    free(q);
    free(kall);
    free(vall);
    free(att);
    free(tmp);
    free(g);
    free(u);
    return rc;
}

/* ---- masks (src/attention.cpp:50-92) ---- */
int tko_build_mask_rows(const int64_t* lens, int64_t n_segments, int independent, int64_t* lo, int64_t* hi) {
    if (n_segments < 1) return fail(4, "SegmentLayout: empty");
    int64_t off = 0;
    for (int64_t s = 0; s < n_segments; ++s) {
        if (lens[s] < 1) return fail(4, "SegmentLayout: segment with token_count < 1");
        const int is_query = s == n_segments - 1;
        for (int64_t i = off; i < off + lens[s]; ++i) {
            lo[i] = (independent && !is_query) ? off : 0;
            hi[i] = i;
        }
        off += lens[s];
    }
    return 0;
}

int tko_causal_rows(int64_t new_tokens, int64_t past, int64_t* lo, int64_t* hi) {
    if (new_tokens < 0 || past < 0) return fail(2, "causal_rows: negative token count");
    for (int64_t i = 0; i < new_tokens; ++i) {
        lo[i] = 0;
        hi[i] = past + i;
    }
    return 0;
}

/* ---- pipeline (src/pipeline.cpp) ---- */
int tko_assemble_positions(const int64_t* lens, int64_t n, int reordered, int64_t* pos, int64_t* next) {
    int64_t running = 0, max_len = 0, k = 0;
    for (int64_t c = 0; c < n; ++c) {
        const int64_t first = reordered ? running : 0;
        for (int64_t t = 0; t < lens[c]; ++t) pos[k++] = first + t;
        running += lens[c];
        if (lens[c] > max_len) max_len = lens[c];
    }
    *next = reordered ? running : max_len;
    return 0;
}

int tko_chunk_kv(const tko_model* m, const int32_t* framed, int64_t n, double* k_out, double* v_out) {
    int64_t* pos = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* lo = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* hi = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) pos[i] = i;
    tko_causal_rows(n, 0, lo, hi);
    int rc = tko_forward(m, framed, n, pos, NULL, NULL, NULL, 0, lo, hi, NULL, 1, k_out, v_out);
    free(pos);
    free(lo);
    free(hi);
    return rc;
}

int tko_prefill_query(const tko_model* m, const double* ctx_k, const double* ctx_v, const int64_t* ctx_pos,
                      int64_t n_ctx, int64_t next_position, const int32_t* q, int64_t nq, double* logits) {
    if (nq == 0) return fail(3, "prefill_query: empty query");
    int64_t* pos = (int64_t*)malloc((size_t)nq * sizeof(int64_t));
    int64_t* lo = (int64_t*)malloc((size_t)nq * sizeof(int64_t));
    int64_t* hi = (int64_t*)malloc((size_t)nq * sizeof(int64_t));
    for (int64_t i = 0; i < nq; ++i) pos[i] = next_position + i;
    tko_causal_rows(nq, n_ctx, lo, hi);
    int rc = tko_forward(m, q, nq, pos, ctx_k, ctx_v, ctx_pos, n_ctx, lo, hi, logits, 1, NULL, NULL);
    free(pos);
    free(lo);
    free(hi);
    return rc;
}

int tko_naive_prefill(const tko_model* m, const int32_t* tokens, const int64_t* offsets, int64_t n_chunks,
                      const int32_t* q, int64_t nq, int independent, double* logits) {
    if (nq == 0) return fail(3, "naive_prefill: empty query");
    const int64_t nc_tok = offsets[n_chunks] - offsets[0], total = nc_tok + nq;
    int64_t* lens = (int64_t*)malloc((size_t)(n_chunks + 1) * sizeof(int64_t));
    int32_t* all = (int32_t*)malloc((size_t)total * sizeof(int32_t));
    int64_t* pos = (int64_t*)malloc((size_t)total * sizeof(int64_t));
    int64_t* lo = (int64_t*)malloc((size_t)total * sizeof(int64_t));
    int64_t* hi = (int64_t*)malloc((size_t)total * sizeof(int64_t));
    int rc = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        lens[c] = offsets[c + 1] - offsets[c];
        if (lens[c] < 1) {
            rc = fail(3, "naive_prefill: empty chunk");
            goto out;
        }
    }
    lens[n_chunks] = nq;
    memcpy(all, tokens + offsets[0], (size_t)nc_tok * sizeof(int32_t));
    memcpy(all + nc_tok, q, (size_t)nq * sizeof(int32_t));
    for (int64_t i = 0; i < total; ++i) pos[i] = i;
    if ((rc = tko_build_mask_rows(lens, n_chunks + 1, independent, lo, hi))) goto out;
    rc = tko_forward(m, all, total, pos, NULL, NULL, NULL, 0, lo, hi, logits, 1, NULL, NULL);
out:
    free(lens);
    free(all);
    free(pos);
    free(lo);
    free(hi);
    return rc;
}

/* ---- cost model (src/costmodel.cpp:11-45) ---- */
uint64_t tko_flops_total(const tko_config* c, int64_t n_input, int64_t n_context, int64_t batch) {
    const uint64_t qkv = 2ULL * (uint64_t)c->hidden_size * (uint64_t)(c->head_num + 2 * c->kv_head_num) *
                         (uint64_t)c->head_size;
    const uint64_t attn = 2ULL * (uint64_t)c->head_num * (uint64_t)c->head_size * (uint64_t)n_context;
    const uint64_t o = 2ULL * (uint64_t)c->hidden_size * (uint64_t)c->hidden_size;
    const uint64_t mlp = 6ULL * (uint64_t)c->hidden_size * (uint64_t)c->intermediate_size;
    return (uint64_t)batch * (uint64_t)n_input * (uint64_t)c->layer_num * (qkv + attn + o + mlp);
}


/* ---- retrieval (retrieval.cpp) ---- */
int tko_embed(const int32_t* tokens, int64_t n, int64_t dim, double* out) {
    if (n < 1) return fail(3, "embed: empty token list");
    if (dim < 1) return fail(3, "embed: dimension must be >= 1");
    for (int64_t i = 0; i < dim; ++i) out[i] = 0.0;
    int32_t prev = -1; /* sentinel precedes the first token (retrieval.cpp:70) */
    for (int64_t i = 0; i < n; ++i) {
        fnv f;
        fnv_init(&f);
        fnv_u32(&f, (uint32_t)prev);
        fnv_u32(&f, (uint32_t)tokens[i]);
        const uint64_t h = f.h;
        out[h % (uint64_t)dim] += (h >> 63) ? -1.0 : 1.0;
        prev = tokens[i];
    }
    double ss = 0.0;
    for (int64_t i = 0; i < dim; ++i) ss += out[i] * out[i];
    if (ss == 0.0) { /* signed counts cancelled exactly (retrieval.cpp:80-84) */
        out[0] = 1.0;
        ss = 1.0;
    }
    const double inv = 1.0 / sqrt(ss);
    for (int64_t i = 0; i < dim; ++i) out[i] *= inv;
    return 0;
}

typedef struct {
    double score;
    uint64_t id;
} tko_scored;

static int scored_cmp(const void* pa, const void* pb) {
    const tko_scored* a = (const tko_scored*)pa;
    const tko_scored* b = (const tko_scored*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

int64_t tko_top_k(const double* emb, const uint64_t* ids, int64_t n, int64_t dim, const double* q, int64_t k,
                  uint64_t* ids_out, double* scores_out) {
    if (k < 1) return -fail(3, "top_k: k must be >= 1");
    if (n < 1) return -fail(3, "top_k: empty index");
    tko_scored* sc = (tko_scored*)malloc((size_t)n * sizeof *sc);
    for (int64_t r = 0; r < n; ++r) {
        const double* b = emb + r * dim;
        double dot = 0.0, na = 0.0, nb = 0.0; /* cosine, retrieval.cpp:90-100 (same operation order) */
        for (int64_t i = 0; i < dim; ++i) {
            dot += q[i] * b[i];
            na += q[i] * q[i];
            nb += b[i] * b[i];
        }
        sc[r].score = dot / sqrt(na * nb);
        sc[r].id = ids[r];
    }
    qsort(sc, (size_t)n, sizeof *sc, scored_cmp);
    const int64_t take = k < n ? k : n;
    for (int64_t i = 0; i < take; ++i) {
        ids_out[i] = sc[i].id;
        if (scores_out) scores_out[i] = sc[i].score;
    }
    free(sc);
    return take;
}

/*
 * otflm_oracle.c -- CPU restatement of the reference (otflm) on-the-fly
 * RNNLM rescoring hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path (paper_2007_11794_b200) never links
 * or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/pkg/src/otflm/).  Arithmetic order follows the
 * reference exactly (float64 accumulation of float32 operands, left-to-right
 * sums, no FMA contraction -- compile with -ffp-contract=off) so that the
 * oracle is bit-compatible with the numba backend; tests/test_oracle_golden.py
 * pins it against vectors produced by the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_VALUE -1        /* ValueError (bad word id, beam, order) */
#define ORC_ERR_UNKNOWN_INDEX -2 /* context_table.UnknownIndexError */
#define ORC_ERR_TABLE_FULL -3   /* context_table.TableFullError */
#define ORC_ERR_NO_PATH -4      /* decoder: "no complete path" ValueError */
#define ORC_ERR_KEY -5          /* ngram: word missing from unigram table */
#define ORC_ERR_NOMEM -6
#define ORC_ERR_CYCLE -7        /* lattice.LatticeFormatError (cycle) */
#define ORC_ERR_PACK -8         /* codec.PackOverflowError */

/* ------------------------------------------------------------------ */
/* feature hash: _kernels_nb.py:21-33 (normative, docs/protocol.md:71-82) */
/* ------------------------------------------------------------------ */
#define ORC_MULT 0x9E3779B97F4A7C15ULL

static inline uint64_t orc_mix(uint64_t h, uint64_t x) {
    h = (h ^ x) * ORC_MULT;
    return h ^ (h >> 32);
}

uint64_t orc_feature_index(uint64_t seed, int64_t order_k, const int64_t *words,
                           int64_t n_words, int64_t node_id, uint64_t mask) {
    uint64_t h = orc_mix(seed, (uint64_t)order_k);
    for (int64_t i = 0; i < n_words; i++) h = orc_mix(h, (uint64_t)words[i]);
    h = orc_mix(h, (uint64_t)node_id);
    return h & mask;
}

/* _kernels_nb.py:36-48 */
static inline double orc_sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

static inline double orc_log_sigmoid(double x) {
    if (x >= 0.0) return -log1p(exp(-x));
    return x - log1p(exp(x));
}

/* ------------------------------------------------------------------ */
/* model                                                                */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t H, V, order;     /* hidden_size, vocab_size, maxent_order */
    uint64_t maxent_size;    /* power of two */
    uint64_t seed;           /* hash_seed */
    const float *U;          /* input_weights [V,H] */
    const float *W;          /* recurrent_weights [H,H] */
    const float *NV;         /* node_vectors [V-1,H] */
    const float *ME;         /* maxent_table [M] */
    const int32_t *path_nodes;
    const float *path_signs;
    const int64_t *path_offsets; /* [V+1] */
} OrcModel;

/* advance_hidden: _kernels_nb.py:51-60 */
void orc_advance_hidden(const float *input_row, const float *W, const float *h,
                        int32_t H, float *out) {
    for (int32_t i = 0; i < H; i++) {
        double acc = (double)input_row[i];
        const float *wr = W + (size_t)i * H;
        for (int32_t j = 0; j < H; j++) acc += (double)wr[j] * (double)h[j];
        out[i] = (float)orc_sigmoid(acc);
    }
}

/* _node_activation: _kernels_nb.py:63-75 */
static double orc_node_activation(int64_t j, const float *hidden, int32_t H,
                                  const int64_t *history, int64_t L,
                                  const float *NV, const float *ME,
                                  int32_t order, uint64_t seed, uint64_t mask) {
    double a = 0.0;
    const float *v = NV + (size_t)j * H;
    for (int32_t i = 0; i < H; i++) a += (double)v[i] * (double)hidden[i];
    int64_t kmax = order < L ? order : L;
    for (int64_t k = 1; k <= kmax; k++) {
        uint64_t idx = orc_feature_index(seed, k, history + (L - k), k, j, mask);
        a += (double)ME[idx];
    }
    return a;
}

/* word_logprob: _kernels_nb.py:78-86 */
double orc_word_logprob(const float *hidden, int32_t H, const int64_t *history,
                        int64_t L, const int32_t *nodes, const float *signs,
                        int64_t P, const float *NV, const float *ME,
                        int32_t order, uint64_t seed, uint64_t mask) {
    double lp = 0.0;
    for (int64_t p = 0; p < P; p++) {
        double a = orc_node_activation(nodes[p], hidden, H, history, L, NV, ME,
                                       order, seed, mask);
        lp += orc_log_sigmoid((double)signs[p] * a);
    }
    return lp;
}

/* all_word_logprobs: _kernels_nb.py:89-104 */
void orc_all_word_logprobs(const float *hidden, int32_t H, const int64_t *history,
                           int64_t L, const int32_t *path_nodes,
                           const float *path_signs, const int64_t *path_offsets,
                           int32_t V, const float *NV, const float *ME,
                           int32_t order, uint64_t seed, uint64_t mask,
                           double *out) {
    int32_t n_nodes = V - 1;
    double *acts = (double *)malloc(sizeof(double) * (size_t)(n_nodes > 0 ? n_nodes : 1));
    for (int32_t j = 0; j < n_nodes; j++)
        acts[j] = orc_node_activation(j, hidden, H, history, L, NV, ME, order, seed, mask);
    for (int32_t w = 0; w < V; w++) {
        double lp = 0.0;
        for (int64_t p = path_offsets[w]; p < path_offsets[w + 1]; p++)
            lp += orc_log_sigmoid((double)path_signs[p] * acts[path_nodes[p]]);
        out[w] = lp;
    }
    free(acts);
}

/* ------------------------------------------------------------------ */
/* generic open-addressing map u64 -> i64 (linear probing, grows)       */
/* ------------------------------------------------------------------ */
typedef struct {
    uint64_t *keys;
    int64_t *vals;
    uint8_t *used;
    uint64_t cap, n;
} OrcMap;

static inline uint64_t orc_hash64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

static int orc_map_init(OrcMap *m, uint64_t cap) {
    uint64_t c = 16;
    while (c < cap) c <<= 1;
    m->keys = (uint64_t *)calloc(c, sizeof(uint64_t));
    m->vals = (int64_t *)calloc(c, sizeof(int64_t));
    m->used = (uint8_t *)calloc(c, 1);
    m->cap = c;
    m->n = 0;
    return (m->keys && m->vals && m->used) ? ORC_OK : ORC_ERR_NOMEM;
}

static void orc_map_free(OrcMap *m) {
    free(m->keys); free(m->vals); free(m->used);
    memset(m, 0, sizeof(*m));
}

static void orc_map_clear(OrcMap *m) {
    memset(m->used, 0, m->cap);
    m->n = 0;
}

static int64_t *orc_map_find(const OrcMap *m, uint64_t key) {
    uint64_t mask = m->cap - 1, i = orc_hash64(key) & mask;
    while (m->used[i]) {
        if (m->keys[i] == key) return &m->vals[i];
        i = (i + 1) & mask;
    }
    return NULL;
}

static int orc_map_put(OrcMap *m, uint64_t key, int64_t val);

static int orc_map_grow(OrcMap *m) {
    OrcMap n2;
    if (orc_map_init(&n2, m->cap * 2) != ORC_OK) return ORC_ERR_NOMEM;
    for (uint64_t i = 0; i < m->cap; i++)
        if (m->used[i]) orc_map_put(&n2, m->keys[i], m->vals[i]);
    orc_map_free(m);
    *m = n2;
    return ORC_OK;
}

static int orc_map_put(OrcMap *m, uint64_t key, int64_t val) {
    if ((m->n + 1) * 2 > m->cap) {
        int rc = orc_map_grow(m);
        if (rc) return rc;
    }
    uint64_t mask = m->cap - 1, i = orc_hash64(key) & mask;
    while (m->used[i]) {
        if (m->keys[i] == key) { m->vals[i] = val; return ORC_OK; }
        i = (i + 1) & mask;
    }
    m->used[i] = 1; m->keys[i] = key; m->vals[i] = val; m->n++;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* n-gram LM lookup: ngram.py:34-46 (NgramModel), :161-179 (logprob)    */
/* keys are word tuples (len <= 5); stored as (len, words) records and   */
/* indexed by a 64-bit tuple hash with full-tuple verification.          */
/* ------------------------------------------------------------------ */
#define ORC_MAX_NGRAM 6
typedef struct {
    int32_t len;
    int32_t w[ORC_MAX_NGRAM];
    double val;
    int64_t next; /* chain of records sharing the same 64-bit hash */
} OrcGram;

typedef struct {
    int32_t order, V, bos;
    OrcGram *probs; int64_t n_probs;
    OrcGram *bows; int64_t n_bows;
    OrcMap probs_map, bows_map; /* tuple hash -> first record index */
} OrcNgram;

static uint64_t orc_tuple_hash(const int32_t *w, int32_t len) {
    uint64_t h = 0x243F6A8885A308D3ULL ^ (uint64_t)len;
    for (int32_t i = 0; i < len; i++) h = orc_hash64(h ^ (uint64_t)(uint32_t)w[i]) + 0x9E37ULL * (uint64_t)(i + 1);
    return h;
}

static int orc_gram_index(OrcGram *recs, int64_t n, OrcMap *map) {
    if (orc_map_init(map, (uint64_t)(n * 2 + 16)) != ORC_OK) return ORC_ERR_NOMEM;
    for (int64_t r = 0; r < n; r++) {
        uint64_t h = orc_tuple_hash(recs[r].w, recs[r].len);
        int64_t *head = orc_map_find(map, h);
        recs[r].next = head ? *head : -1;
        if (orc_map_put(map, h, r) != ORC_OK) return ORC_ERR_NOMEM;
    }
    return ORC_OK;
}

static const double *orc_gram_get(const OrcGram *recs, const OrcMap *map,
                                  const int32_t *w, int32_t len) {
    int64_t *head = orc_map_find(map, orc_tuple_hash(w, len));
    for (int64_t r = head ? *head : -1; r >= 0; r = recs[r].next) {
        if (recs[r].len != len) continue;
        int eq = 1;
        for (int32_t i = 0; i < len; i++) if (recs[r].w[i] != w[i]) { eq = 0; break; }
        if (eq) return &recs[r].val;
    }
    return NULL;
}

/* Create from flat arrays: keys [n, order] int32 (row-padded), lens [n]. */
OrcNgram *orc_ngram_create(int32_t order, int32_t V, int32_t bos,
                           int64_t n_probs, const int32_t *prob_keys,
                           const int32_t *prob_lens, const double *prob_vals,
                           int64_t n_bows, const int32_t *bow_keys,
                           const int32_t *bow_lens, const double *bow_vals) {
    if (order < 1 || order > ORC_MAX_NGRAM - 1) return NULL;
    OrcNgram *g = (OrcNgram *)calloc(1, sizeof(OrcNgram));
    g->order = order; g->V = V; g->bos = bos;
    g->probs = (OrcGram *)calloc((size_t)(n_probs > 0 ? n_probs : 1), sizeof(OrcGram));
    g->bows = (OrcGram *)calloc((size_t)(n_bows > 0 ? n_bows : 1), sizeof(OrcGram));
    g->n_probs = n_probs; g->n_bows = n_bows;
    for (int64_t r = 0; r < n_probs; r++) {
        g->probs[r].len = prob_lens[r];
        for (int32_t i = 0; i < prob_lens[r]; i++) g->probs[r].w[i] = prob_keys[r * order + i];
        g->probs[r].val = prob_vals[r];
    }
    for (int64_t r = 0; r < n_bows; r++) {
        g->bows[r].len = bow_lens[r];
        for (int32_t i = 0; i < bow_lens[r]; i++) g->bows[r].w[i] = bow_keys[r * order + i];
        g->bows[r].val = bow_vals[r];
    }
    if (orc_gram_index(g->probs, n_probs, &g->probs_map) ||
        orc_gram_index(g->bows, n_bows, &g->bows_map)) return NULL;
    return g;
}

void orc_ngram_destroy(OrcNgram *g) {
    if (!g) return;
    orc_map_free(&g->probs_map); orc_map_free(&g->bows_map);
    free(g->probs); free(g->bows); free(g);
}

/* ngram_logprob: ngram.py:161-179 */
int orc_ngram_logprob(const OrcNgram *g, const int32_t *context, int32_t n_ctx,
                      int32_t w, double *out) {
    if (w < 0 || w >= g->V) return ORC_ERR_VALUE;
    int32_t keep = g->order > 1 ? g->order - 1 : 0;
    if (keep > n_ctx) keep = n_ctx;
    const int32_t *ctx = context + (n_ctx - keep);
    int32_t buf[ORC_MAX_NGRAM];
    for (int32_t depth = 0; depth <= keep; depth++) {
        int32_t slen = keep - depth; /* suffix ctx[depth:] */
        for (int32_t i = 0; i < slen; i++) buf[i] = ctx[depth + i];
        buf[slen] = w;
        const double *lp = orc_gram_get(g->probs, &g->probs_map, buf, slen + 1);
        if (lp) {
            double v = *lp;
            for (int32_t sh = depth - 1; sh >= 0; sh--) { /* reversed(suffixes[:depth]) */
                const double *b = orc_gram_get(g->bows, &g->bows_map, ctx + sh, keep - sh);
                v = (b ? *b : 0.0) + v;
            }
            *out = v;
            return ORC_OK;
        }
    }
    return ORC_ERR_KEY;
}

/* small_context: decoder.py:73-80 -> padded history into buf; returns length */
static int32_t orc_small_context(const OrcNgram *g, const int64_t *hist, int32_t L,
                                 int32_t *buf) {
    int32_t need = g->order - 1, n = 0;
    if (L < need) for (int32_t i = 0; i < need - L; i++) buf[n++] = g->bos;
    for (int32_t i = 0; i < L; i++) buf[n++] = (int32_t)hist[i];
    return n;
}

/* ------------------------------------------------------------------ */
/* IndexTable: context_table.py:48-119 (content-dedup, idx = len + 1)   */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t H, order;
    uint64_t max_entries;
    float *hidden;    /* [cap, H] row idx-1 */
    int64_t *hist;    /* [cap, order] */
    int32_t *hlen;
    int64_t *chain;   /* next index with the same digest */
    uint64_t n, cap;
    OrcMap digest;    /* content digest -> most recent idx */
} OrcTable;

static uint64_t orc_content_digest(const float *h, int32_t H, const int64_t *hist,
                                   int32_t L, int32_t order) {
    /* FNV-1a over the serialized key bytes (f32 hidden + u64 slots with the
     * all-ones sentinel), context_table.py:64-72.  Only used to bucket;
     * equality is decided by full comparison as in context_table.py:78-79. */
    uint64_t x = 0xcbf29ce484222325ULL;
    const uint8_t *b = (const uint8_t *)h;
    for (size_t i = 0; i < (size_t)H * 4; i++) { x ^= b[i]; x *= 0x100000001b3ULL; }
    for (int32_t s = 0; s < order; s++) {
        uint64_t v = s < L ? (uint64_t)hist[s] : 0xFFFFFFFFFFFFFFFFULL;
        for (int k = 0; k < 8; k++) { x ^= (v >> (8 * k)) & 0xff; x *= 0x100000001b3ULL; }
    }
    return x;
}

static int orc_table_init(OrcTable *t, int32_t H, int32_t order, uint64_t max_entries) {
    memset(t, 0, sizeof(*t));
    t->H = H; t->order = order; t->max_entries = max_entries;
    t->cap = 1024;
    t->hidden = (float *)malloc(sizeof(float) * t->cap * (size_t)H);
    t->hist = (int64_t *)malloc(sizeof(int64_t) * t->cap * (size_t)(order > 0 ? order : 1));
    t->hlen = (int32_t *)malloc(sizeof(int32_t) * t->cap);
    t->chain = (int64_t *)malloc(sizeof(int64_t) * t->cap);
    return orc_map_init(&t->digest, 2048);
}

static void orc_table_free(OrcTable *t) {
    free(t->hidden); free(t->hist); free(t->hlen); free(t->chain);
    orc_map_free(&t->digest);
}

static void orc_table_clear(OrcTable *t) {
    t->n = 0;
    orc_map_clear(&t->digest);
}

/* encode: context_table.py:74-86 */
static int orc_table_encode(OrcTable *t, const float *h, const int64_t *hist, int32_t L,
                            uint64_t *idx_out) {
    uint64_t dg = orc_content_digest(h, t->H, hist, L, t->order);
    int64_t *head = orc_map_find(&t->digest, dg);
    for (int64_t idx = head ? *head : 0; idx > 0; idx = t->chain[idx - 1]) {
        const float *sh = t->hidden + (size_t)(idx - 1) * t->H;
        if (t->hlen[idx - 1] != L) continue;
        if (memcmp(sh, h, (size_t)t->H * 4) != 0) continue;
        if (memcmp(t->hist + (size_t)(idx - 1) * t->order, hist, sizeof(int64_t) * (size_t)L) != 0) continue;
        *idx_out = (uint64_t)idx;
        return ORC_OK;
    }
    if (t->n >= t->max_entries) return ORC_ERR_TABLE_FULL;
    if (t->n == t->cap) {
        uint64_t nc = t->cap * 2;
        t->hidden = (float *)realloc(t->hidden, sizeof(float) * nc * (size_t)t->H);
        t->hist = (int64_t *)realloc(t->hist, sizeof(int64_t) * nc * (size_t)(t->order > 0 ? t->order : 1));
        t->hlen = (int32_t *)realloc(t->hlen, sizeof(int32_t) * nc);
        t->chain = (int64_t *)realloc(t->chain, sizeof(int64_t) * nc);
        if (!t->hidden || !t->hist || !t->hlen || !t->chain) return ORC_ERR_NOMEM;
        t->cap = nc;
    }
    uint64_t idx = t->n + 1;
    memcpy(t->hidden + (size_t)t->n * t->H, h, (size_t)t->H * 4);
    for (int32_t s = 0; s < L; s++) t->hist[(size_t)t->n * t->order + s] = hist[s];
    t->hlen[t->n] = L;
    t->chain[t->n] = head ? *head : 0;
    t->n++;
    if (orc_map_put(&t->digest, dg, (int64_t)idx) != ORC_OK) return ORC_ERR_NOMEM;
    *idx_out = idx;
    return ORC_OK;
}

/* decode: context_table.py:88-104 -- returns pointers into the table (or
 * the zero context for idx 0, supplied by the caller's scratch). */
static int orc_table_decode(const OrcTable *t, uint64_t idx, const float *zero_h,
                            const float **h, const int64_t **hist, int32_t *L) {
    if (idx == 0) { *h = zero_h; *hist = NULL; *L = 0; return ORC_OK; }
    if (idx > t->n) return ORC_ERR_UNKNOWN_INDEX;
    *h = t->hidden + (size_t)(idx - 1) * t->H;
    *hist = t->hist + (size_t)(idx - 1) * t->order;
    *L = t->hlen[idx - 1];
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* RescoreStack = table + cache + ledger: decoder.py:61-70, cache.py    */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t lookups, hits, misses, evictions;
} OrcCacheStats;

typedef struct {
    const OrcModel *model;
    OrcTable table;
    int32_t enabled;
    OrcMap cache;          /* (c<<32|w) -> slot */
    double *cache_p; uint32_t *cache_c; uint64_t cache_n, cache_cap;
    OrcCacheStats cur, cum;
    int64_t ledger_requests, ledger_bytes_indexed, ledger_bytes_full;
    float *zero_h, *scratch_h;
    int64_t scratch_hist[8];
    /* capacity-bounded LFU with LRU tie-break (cache.py:98-134): per slot
     * residency, use count and last use; lazy min-heap of (freq, seq, slot) */
    int64_t capacity_bytes;   /* 0 = unbounded */
    uint8_t *resident; int64_t *freq, *last;
    int64_t seq, n_resident;
    int64_t *heap; int64_t heap_n, heap_cap;   /* triples */
} OrcStack;

#define ORC_ENTRY_BYTES 32   /* cache.py:26 */

OrcStack *orc_stack_create(const OrcModel *model, int32_t enabled, uint64_t max_entries) {
    OrcStack *s = (OrcStack *)calloc(1, sizeof(OrcStack));
    s->model = model;
    s->enabled = enabled;
    if (orc_table_init(&s->table, model->H, model->order, max_entries)) return NULL;
    if (orc_map_init(&s->cache, 4096)) return NULL;
    s->cache_cap = 1024;
    s->cache_p = (double *)malloc(sizeof(double) * s->cache_cap);
    s->cache_c = (uint32_t *)malloc(sizeof(uint32_t) * s->cache_cap);
    s->resident = (uint8_t *)calloc(s->cache_cap, 1);
    s->freq = (int64_t *)calloc(s->cache_cap, sizeof(int64_t));
    s->last = (int64_t *)calloc(s->cache_cap, sizeof(int64_t));
    s->heap_cap = 1024;
    s->heap = (int64_t *)malloc(sizeof(int64_t) * 3 * s->heap_cap);
    s->zero_h = (float *)calloc((size_t)model->H, sizeof(float));
    s->scratch_h = (float *)calloc((size_t)model->H, sizeof(float));
    return s;
}

void orc_stack_destroy(OrcStack *s) {
    if (!s) return;
    orc_table_free(&s->table);
    orc_map_free(&s->cache);
    free(s->cache_p); free(s->cache_c); free(s->zero_h); free(s->scratch_h);
    free(s->resident); free(s->freq); free(s->last); free(s->heap);
    free(s);
}

/* lazy heap of (freq, seq, slot), ordered by (freq, seq) -- heapq tuples
 * (cache.py:95,110); seq is unique per push so the slot never decides */
static int orc_heap_less(const int64_t *a, const int64_t *b) {
    return a[0] < b[0] || (a[0] == b[0] && a[1] < b[1]);
}
static void orc_heap_push(OrcStack *s, int64_t f, int64_t q, int64_t slot) {
    if (s->heap_n == s->heap_cap) {
        s->heap_cap *= 2;
        s->heap = (int64_t *)realloc(s->heap, sizeof(int64_t) * 3 * s->heap_cap);
    }
    int64_t i = s->heap_n++;
    int64_t *h = s->heap;
    h[3 * i] = f; h[3 * i + 1] = q; h[3 * i + 2] = slot;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!orc_heap_less(h + 3 * i, h + 3 * p)) break;
        for (int k = 0; k < 3; k++) { int64_t t = h[3 * p + k]; h[3 * p + k] = h[3 * i + k]; h[3 * i + k] = t; }
        i = p;
    }
}
static void orc_heap_pop(OrcStack *s, int64_t *out) {
    int64_t *h = s->heap;
    for (int k = 0; k < 3; k++) out[k] = h[k];
    s->heap_n--;
    for (int k = 0; k < 3; k++) h[k] = h[3 * s->heap_n + k];
    int64_t i = 0, n = s->heap_n;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && orc_heap_less(h + 3 * l, h + 3 * m)) m = l;
        if (r < n && orc_heap_less(h + 3 * r, h + 3 * m)) m = r;
        if (m == i) break;
        for (int k = 0; k < 3; k++) { int64_t t = h[3 * m + k]; h[3 * m + k] = h[3 * i + k]; h[3 * i + k] = t; }
        i = m;
    }
}

/* _evict_one (cache.py:117-128): stale heap items are skipped lazily */
static void orc_evict_one(OrcStack *s) {
    int64_t t[3];
    while (s->heap_n > 0) {
        orc_heap_pop(s, t);
        int64_t slot = t[2];
        if (s->resident[slot] && s->freq[slot] == t[0] && s->last[slot] == t[1]) {
            s->resident[slot] = 0;
            s->n_resident--;
            s->cur.evictions++;
            return;
        }
    }
}

/* set_capacity (cache.py:130-137): 0 removes the bound; shrinking evicts at once */
int orc_stack_set_capacity(OrcStack *s, int64_t capacity_bytes) {
    if (capacity_bytes < 0) return ORC_ERR_VALUE;
    s->capacity_bytes = capacity_bytes;
    if (capacity_bytes > 0)
        while (s->n_resident > 0 && s->n_resident * ORC_ENTRY_BYTES > capacity_bytes) orc_evict_one(s);
    return ORC_OK;
}

/* reset_utterance: cache.py:185-191 (roll stats; clear unless retain) */
void orc_stack_reset(OrcStack *s, int32_t retain) {
    s->cum.lookups += s->cur.lookups; s->cum.hits += s->cur.hits;
    s->cum.misses += s->cur.misses; s->cum.evictions += s->cur.evictions;
    memset(&s->cur, 0, sizeof(s->cur));
    if (!retain) {
        orc_map_clear(&s->cache);
        s->cache_n = 0;
        s->n_resident = 0;
        s->heap_n = 0;
        orc_table_clear(&s->table);
    }
}

/* RescoreCache.clear (cache.py:136-140): drop every entry and the policy
 * state; counters and the index table stay */
void orc_stack_cache_clear(OrcStack *s) {
    orc_map_clear(&s->cache);
    s->cache_n = 0;
    s->n_resident = 0;
    s->heap_n = 0;
}

/* RescoreCache.roll_stats (cache.py:156-158) alone */
void orc_stack_roll_stats(OrcStack *s) {
    s->cum.lookups += s->cur.lookups; s->cum.hits += s->cur.hits;
    s->cum.misses += s->cur.misses; s->cum.evictions += s->cur.evictions;
    memset(&s->cur, 0, sizeof(s->cur));
}

/* stats out: [lookups, hits, misses, evictions, entries, table_len,
 *             cum_lookups, cum_hits, cum_misses, ledger_requests,
 *             ledger_bytes_indexed, ledger_bytes_full] */
void orc_stack_stats(const OrcStack *s, int64_t *out) {
    out[0] = s->cur.lookups; out[1] = s->cur.hits; out[2] = s->cur.misses;
    out[3] = s->cur.evictions; out[4] = s->n_resident; out[5] = (int64_t)s->table.n;
    out[6] = s->cum.lookups + s->cur.lookups; out[7] = s->cum.hits + s->cur.hits;
    out[8] = s->cum.misses + s->cur.misses;
    out[9] = s->ledger_requests; out[10] = s->ledger_bytes_indexed; out[11] = s->ledger_bytes_full;
}

/* Copy of a stored context (for replay tests): hidden [H], hist [order]. */
int orc_stack_context(const OrcStack *s, uint64_t idx, float *hidden, int64_t *hist,
                      int32_t *L) {
    const float *h; const int64_t *hh; int32_t n;
    int rc = orc_table_decode(&s->table, idx, s->zero_h, &h, &hh, &n);
    if (rc) return rc;
    memcpy(hidden, h, sizeof(float) * (size_t)s->model->H);
    for (int32_t i = 0; i < n; i++) hist[i] = hh[i];
    *L = n;
    return ORC_OK;
}

/* compute_rnnlm: rnnlm.py:217-221 = word_logprob (:195-204) then
 * advance_context (:180-188).  Scores w against h_c, not h'. */
static int orc_compute(OrcStack *s, const float *h, const int64_t *hist, int32_t L,
                       int32_t w, double *p, uint64_t *c_next) {
    const OrcModel *m = s->model;
    int64_t o0 = m->path_offsets[w], o1 = m->path_offsets[w + 1];
    *p = orc_word_logprob(h, m->H, hist, L, m->path_nodes + o0, m->path_signs + o0,
                          o1 - o0, m->NV, m->ME, m->order, m->seed, m->maxent_size - 1);
    orc_advance_hidden(m->U + (size_t)w * m->H, m->W, h, m->H, s->scratch_h);
    /* history' = (history + (w,))[-order:] */
    int32_t nl = 0;
    int64_t tmp[16];
    for (int32_t i = 0; i < L; i++) tmp[nl++] = hist[i];
    tmp[nl++] = w;
    int32_t start = nl > m->order ? nl - m->order : 0;
    for (int32_t i = start; i < nl; i++) s->scratch_hist[i - start] = tmp[i];
    return orc_table_encode(&s->table, s->scratch_h, s->scratch_hist, nl - start, c_next);
}

/* rnnlm_prob: cache.py:165-182 with RescoreCache.get/put (cache.py:82-109);
 * capacity_bytes > 0 adds the LFU + LRU eviction of cache.py:98-128. */
int orc_rnnlm_prob(OrcStack *s, int32_t w, uint64_t c, double *p, uint64_t *c_next,
                   int32_t *hit) {
    const OrcModel *m = s->model;
    if (w < 0 || w >= m->V) return ORC_ERR_VALUE;
    uint64_t key = (c << 32) | (uint64_t)(uint32_t)w;
    s->cur.lookups++;
    *hit = 0;
    if (s->enabled) {
        int64_t *slot = orc_map_find(&s->cache, key);
        if (slot && s->resident[*slot]) {
            s->cur.hits++;
            s->seq++;                         /* freq / recency bookkeeping (cache.py:91-95) */
            s->freq[*slot]++;
            s->last[*slot] = s->seq;
            orc_heap_push(s, s->freq[*slot], s->seq, *slot);
            *p = s->cache_p[*slot]; *c_next = s->cache_c[*slot]; *hit = 1;
            return ORC_OK;
        }
    }
    s->cur.misses++;
    const float *h; const int64_t *hist; int32_t L;
    int rc = orc_table_decode(&s->table, c, s->zero_h, &h, &hist, &L);
    if (rc) return rc;
    rc = orc_compute(s, h, hist, L, w, p, c_next);
    if (rc) return rc;
    if (s->enabled) {                        /* put (cache.py:99-109) */
        if (s->capacity_bytes > 0) {
            while (s->n_resident > 0 && (s->n_resident + 1) * ORC_ENTRY_BYTES > s->capacity_bytes)
                orc_evict_one(s);
            if ((s->n_resident + 1) * ORC_ENTRY_BYTES > s->capacity_bytes) return ORC_OK;
        }
        int64_t *old = orc_map_find(&s->cache, key);
        int64_t slot;
        if (old) {                           /* re-insert of an evicted key: reuse its slot */
            slot = *old;
        } else {
            if (s->cache_n == s->cache_cap) {
                s->cache_cap *= 2;
                s->cache_p = (double *)realloc(s->cache_p, sizeof(double) * s->cache_cap);
                s->cache_c = (uint32_t *)realloc(s->cache_c, sizeof(uint32_t) * s->cache_cap);
                s->resident = (uint8_t *)realloc(s->resident, s->cache_cap);
                s->freq = (int64_t *)realloc(s->freq, sizeof(int64_t) * s->cache_cap);
                s->last = (int64_t *)realloc(s->last, sizeof(int64_t) * s->cache_cap);
            }
            slot = (int64_t)s->cache_n++;
            if (orc_map_put(&s->cache, key, slot)) return ORC_ERR_NOMEM;
        }
        s->cache_p[slot] = *p; s->cache_c[slot] = (uint32_t)*c_next;
        s->resident[slot] = 1;
        s->n_resident++;
        s->seq++;
        s->freq[slot] = 1;
        s->last[slot] = s->seq;
        orc_heap_push(s, 1, s->seq, slot);
    }
    return ORC_OK;
}

/* RescoreServer.serve: decoder.py:94-104 -> f32 delta and successor. */
static int orc_serve(OrcStack *s, const OrcNgram *g, int32_t w, uint64_t c,
                     float *delta, uint64_t *c_next) {
    double p;
    int32_t hit;
    if (c >> 32) return ORC_ERR_PACK; /* pack(c, ., 32): codec.py:35-46 */
    int rc = orc_rnnlm_prob(s, w, c, &p, c_next, &hit);
    if (rc) return rc;
    if (*c_next >> 32) return ORC_ERR_PACK;
    const float *h; const int64_t *hist; int32_t L;
    rc = orc_table_decode(&s->table, c, s->zero_h, &h, &hist, &L);
    if (rc) return rc;
    int32_t ctx[16];
    int32_t n = orc_small_context(g, hist, L, ctx);
    double p_small;
    rc = orc_ngram_logprob(g, ctx, n, w, &p_small);
    if (rc) return rc;
    *delta = (float)(p - p_small); /* quantize_delta: codec.py:57-59 */
    s->ledger_requests += 1;                                   /* codec.py:95-110 */
    s->ledger_bytes_indexed += 32;
    s->ledger_bytes_full += 2 * (int64_t)(4 * s->model->H + 8 * s->model->order + 8);
    return ORC_OK;
}

int orc_serve_request(OrcStack *s, const OrcNgram *g, int32_t w, uint64_t c,
                      float *delta, uint64_t *c_next) {
    return orc_serve(s, g, w, c, delta, c_next);
}

/* ------------------------------------------------------------------ */
/* Lattice + rescore_onthefly: lattice.py:47-86, decoder.py:114-173     */
/* node ids must be 0..n_nodes-1 (the Python wrapper remaps ids          */
/* monotonically, which preserves Kahn smallest-id order and sorted      */
/* finals).                                                             */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t n_nodes, n_arcs, start, n_finals;
    const int32_t *src, *dst, *word;
    const double *ac, *slm;
    const int32_t *finals; /* ascending */
} OrcLattice;

typedef struct {
    int32_t n_arcs;        /* path length */
    int32_t *arcs;         /* caller buffer, capacity max_arcs */
    int32_t max_arcs;
    double acoustic, lm, combined;
    int64_t end_ctx;
    int64_t expansions;
} OrcResult;

/* Kahn topo order with smallest-id-first ready queue (lattice.py:68-82). */
static int orc_topo(const OrcLattice *lat, int32_t *order, int32_t *out_off, int32_t *out_arc) {
    int32_t N = lat->n_nodes;
    int32_t *indeg = (int32_t *)calloc((size_t)N, sizeof(int32_t));
    for (int32_t a = 0; a < lat->n_arcs; a++) { out_off[lat->src[a] + 1]++; indeg[lat->dst[a]]++; }
    for (int32_t n = 0; n < N; n++) out_off[n + 1] += out_off[n];
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    for (int32_t n = 0; n < N; n++) fill[n] = out_off[n];
    for (int32_t a = 0; a < lat->n_arcs; a++) out_arc[fill[lat->src[a]]++] = a;
    /* binary min-heap of ready node ids */
    int32_t *heap = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    int32_t hn = 0, cnt = 0;
#define HPUSH(v) do { int32_t _i = hn++; heap[_i] = (v); while (_i > 0) { int32_t _p = (_i - 1) / 2; if (heap[_p] <= heap[_i]) break; int32_t _t = heap[_p]; heap[_p] = heap[_i]; heap[_i] = _t; _i = _p; } } while (0)
    for (int32_t n = 0; n < N; n++) if (indeg[n] == 0) HPUSH(n);
    while (hn > 0) {
        int32_t n = heap[0];
        heap[0] = heap[--hn];
        int32_t i = 0;
        for (;;) {
            int32_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < hn && heap[l] < heap[m]) m = l;
            if (r < hn && heap[r] < heap[m]) m = r;
            if (m == i) break;
            int32_t t = heap[m]; heap[m] = heap[i]; heap[i] = t; i = m;
        }
        order[cnt++] = n;
        for (int32_t k = out_off[n]; k < out_off[n + 1]; k++) {
            int32_t d = lat->dst[out_arc[k]];
            if (--indeg[d] == 0) HPUSH(d);
        }
    }
#undef HPUSH
    free(indeg); free(fill); free(heap);
    return cnt == N ? ORC_OK : ORC_ERR_CYCLE;
}

typedef struct { uint32_t ctx; double score; int64_t bp; } OrcTok;

static int orc_tok_cmp(const void *a, const void *b) {
    const OrcTok *x = (const OrcTok *)a, *y = (const OrcTok *)b;
    if (x->score > y->score) return -1;   /* key (-score, ctx): decoder.py:135 */
    if (x->score < y->score) return 1;
    return x->ctx < y->ctx ? -1 : (x->ctx > y->ctx ? 1 : 0);
}

static int orc_ctx_cmp(const void *a, const void *b) {
    const OrcTok *x = (const OrcTok *)a, *y = (const OrcTok *)b;
    return x->ctx < y->ctx ? -1 : (x->ctx > y->ctx ? 1 : 0);
}

int orc_rescore_onthefly(OrcStack *s, const OrcNgram *g, const OrcLattice *lat,
                         double lm_weight, int64_t beam, OrcResult *res) {
    if (beam < 1) return ORC_ERR_VALUE;
    if (g->order - 1 > s->model->order) return ORC_ERR_VALUE; /* decoder.py:87-90 */
    int32_t N = lat->n_nodes;
    int rc = ORC_OK;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    int32_t *out_off = (int32_t *)calloc((size_t)N + 2, sizeof(int32_t));
    int32_t *out_arc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(lat->n_arcs + 1));
    rc = orc_topo(lat, order, out_off, out_arc);
    /* tokens: per node dynamic list; (node, ctx) -> token slot map */
    int64_t tcap = 1024, tn = 0;
    OrcTok *toks = (OrcTok *)malloc(sizeof(OrcTok) * (size_t)tcap);
    int32_t *tnode = (int32_t *)malloc(sizeof(int32_t) * (size_t)tcap);
    int64_t *node_head = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
    int64_t *tnext = (int64_t *)malloc(sizeof(int64_t) * (size_t)tcap);
    for (int32_t n = 0; n < N; n++) node_head[n] = -1;
    OrcMap slot; orc_map_init(&slot, 4096);
    int64_t bcap = 1024, bn = 0;
    int64_t *bp_prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)bcap);
    int32_t *bp_arc = (int32_t *)malloc(sizeof(int32_t) * (size_t)bcap);
    int64_t expansions = 0;
    OrcTok *ranked = NULL; int64_t rcap = 0;
    if (rc) goto done;
    /* start token {start: {0: (0.0, -1)}} */
    toks[0].ctx = 0; toks[0].score = 0.0; toks[0].bp = -1; tnode[0] = lat->start;
    tnext[0] = -1; node_head[lat->start] = 0; tn = 1;
    orc_map_put(&slot, ((uint64_t)(uint32_t)lat->start << 32) | 0u, 0);
    for (int32_t oi = 0; oi < N; oi++) {
        int32_t node = order[oi];
        int64_t cnt = 0;
        for (int64_t t = node_head[node]; t >= 0; t = tnext[t]) cnt++;
        if (cnt == 0) continue;
        if (cnt > rcap) { rcap = cnt * 2; ranked = (OrcTok *)realloc(ranked, sizeof(OrcTok) * (size_t)rcap); }
        int64_t k = 0;
        for (int64_t t = node_head[node]; t >= 0; t = tnext[t]) ranked[k++] = toks[t];
        qsort(ranked, (size_t)cnt, sizeof(OrcTok), orc_tok_cmp);
        int64_t keep = cnt < beam ? cnt : beam;
        for (int64_t r = 0; r < keep; r++) {
            OrcTok tk = ranked[r];
            for (int32_t q = out_off[node]; q < out_off[node + 1]; q++) {
                int32_t a = out_arc[q];
                expansions++;
                float delta; uint64_t c_next;
                rc = orc_serve(s, g, lat->word[a], tk.ctx, &delta, &c_next);
                if (rc) goto done;
                /* decoder.py:144 -- (score + ac) + lm_weight * (slm + delta) */
                double ns = (tk.score + lat->ac[a]) + lm_weight * (lat->slm[a] + (double)delta);
                int32_t d = lat->dst[a];
                uint64_t key = ((uint64_t)(uint32_t)d << 32) | c_next;
                int64_t *sl = orc_map_find(&slot, key);
                if (sl == NULL || ns > toks[*sl].score) {
                    if (bn == bcap) {
                        bcap *= 2;
                        bp_prev = (int64_t *)realloc(bp_prev, sizeof(int64_t) * (size_t)bcap);
                        bp_arc = (int32_t *)realloc(bp_arc, sizeof(int32_t) * (size_t)bcap);
                    }
                    bp_prev[bn] = tk.bp; bp_arc[bn] = a; bn++;
                    if (sl) {
                        toks[*sl].score = ns; toks[*sl].bp = bn - 1;
                    } else {
                        if (tn == tcap) {
                            tcap *= 2;
                            toks = (OrcTok *)realloc(toks, sizeof(OrcTok) * (size_t)tcap);
                            tnode = (int32_t *)realloc(tnode, sizeof(int32_t) * (size_t)tcap);
                            tnext = (int64_t *)realloc(tnext, sizeof(int64_t) * (size_t)tcap);
                        }
                        toks[tn].ctx = (uint32_t)c_next; toks[tn].score = ns; toks[tn].bp = bn - 1;
                        tnode[tn] = d; tnext[tn] = node_head[d]; node_head[d] = tn;
                        orc_map_put(&slot, key, tn);
                        tn++;
                    }
                }
            }
        }
    }
    /* final best: sorted(finals) x sorted(ctx), strict > (decoder.py:150-156) */
    {
        int have = 0; double best_s = 0.0; int64_t best_bp = -1; uint32_t best_ctx = 0;
        for (int32_t f = 0; f < lat->n_finals; f++) {
            int32_t node = lat->finals[f];
            int64_t cnt = 0;
            for (int64_t t = node_head[node]; t >= 0; t = tnext[t]) cnt++;
            if (cnt == 0) continue;
            if (cnt > rcap) { rcap = cnt * 2; ranked = (OrcTok *)realloc(ranked, sizeof(OrcTok) * (size_t)rcap); }
            int64_t k = 0;
            for (int64_t t = node_head[node]; t >= 0; t = tnext[t]) ranked[k++] = toks[t];
            qsort(ranked, (size_t)cnt, sizeof(OrcTok), orc_ctx_cmp);
            for (int64_t i = 0; i < cnt; i++)
                if (!have || ranked[i].score > best_s) {
                    have = 1; best_s = ranked[i].score; best_bp = ranked[i].bp; best_ctx = ranked[i].ctx;
                }
        }
        if (!have) { rc = ORC_ERR_NO_PATH; goto done; }
        /* backtrace (decoder.py:157-162) */
        int32_t len = 0;
        for (int64_t b = best_bp; b >= 0; b = bp_prev[b]) len++;
        res->n_arcs = len;
        if (len <= res->max_arcs) {
            int32_t i = len - 1;
            for (int64_t b = best_bp; b >= 0; b = bp_prev[b]) res->arcs[i--] = bp_arc[b];
        }
        double ac = 0.0;
        /* acoustic_total = sum(a.acoustic for a in arcs) in path order */
        if (len <= res->max_arcs)
            for (int32_t i = 0; i < len; i++) ac = ac + lat->ac[res->arcs[i]];
        res->acoustic = ac;
        res->combined = best_s;
        res->lm = lm_weight != 0.0 ? (best_s - ac) / lm_weight : 0.0;
        res->end_ctx = best_ctx;
        res->expansions = expansions;
    }
done:
    orc_map_free(&slot);
    free(order); free(out_off); free(out_arc); free(toks); free(tnode); free(tnext);
    free(node_head); free(bp_prev); free(bp_arc); free(ranked);
    return rc;
}

/* oracle_path_score (tests/conftest.py:65-78, = decoder.rescored_path_score
 * decoder.py:277-292): direct model calls, no cache/table/beam. */
int orc_path_score(const OrcModel *m, const OrcNgram *g, const OrcLattice *lat,
                   const int32_t *arc_ids, int32_t n, double lm_weight, double *out) {
    float *h = (float *)calloc((size_t)m->H, sizeof(float));
    float *h2 = (float *)calloc((size_t)m->H, sizeof(float));
    int64_t hist[16]; int32_t L = 0;
    double score = 0.0;
    for (int32_t i = 0; i < n; i++) {
        int32_t a = arc_ids[i], w = lat->word[a];
        if (w < 0 || w >= m->V) { free(h); free(h2); return ORC_ERR_VALUE; }
        int64_t o0 = m->path_offsets[w], o1 = m->path_offsets[w + 1];
        double p = orc_word_logprob(h, m->H, hist, L, m->path_nodes + o0, m->path_signs + o0,
                                    o1 - o0, m->NV, m->ME, m->order, m->seed, m->maxent_size - 1);
        int32_t ctx[16];
        int32_t nc = orc_small_context(g, hist, L, ctx);
        double ps;
        int rc = orc_ngram_logprob(g, ctx, nc, w, &ps);
        if (rc) { free(h); free(h2); return rc; }
        float delta = (float)(p - ps);
        score = (score + lat->ac[a]) + lm_weight * (lat->slm[a] + (double)delta);
        orc_advance_hidden(m->U + (size_t)w * m->H, m->W, h, m->H, h2);
        memcpy(h, h2, sizeof(float) * (size_t)m->H);
        if (L < m->order) hist[L++] = w;
        else { for (int32_t k = 1; k < L; k++) hist[k - 1] = hist[k]; hist[L - 1] = w; }
    }
    *out = score;
    free(h); free(h2);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Multi-utterance driver for the CPU baseline: independent streams,    */
/* fresh (retain=False) stack per utterance, utterance-parallel threads  */
/* (SPEC.md:508 permits utterance-level parallelism).                   */
/* ------------------------------------------------------------------ */
typedef struct {
    const OrcModel *m; const OrcNgram *g; const OrcLattice *lats; int32_t n_lat;
    double lm_weight; int64_t beam; int32_t enabled;
    OrcResult *res; int32_t *rcs;
    int32_t next; pthread_mutex_t mu;
    int64_t *lookups, *hits, *misses, *table_len;
} OrcJob;

static void *orc_worker(void *arg) {
    OrcJob *j = (OrcJob *)arg;
    OrcStack *s = orc_stack_create(j->m, j->enabled, (uint64_t)-2);
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int32_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->n_lat) break;
        j->rcs[i] = orc_rescore_onthefly(s, j->g, &j->lats[i], j->lm_weight, j->beam, &j->res[i]);
        j->lookups[i] = s->cur.lookups; j->hits[i] = s->cur.hits; j->misses[i] = s->cur.misses;
        if (j->table_len) j->table_len[i] = (int64_t)s->table.n;
        orc_stack_reset(s, 0);
    }
    orc_stack_destroy(s);
    return NULL;
}

/* table_len (nullable): IndexTable length of each utterance's stream after
 * its decode (context_table.py:116-119) */
int orc_decode_many_t(const OrcModel *m, const OrcNgram *g, const OrcLattice *lats,
                      int32_t n_lat, double lm_weight, int64_t beam, int32_t enabled,
                      int32_t n_threads, OrcResult *res, int32_t *rcs,
                      int64_t *lookups, int64_t *hits, int64_t *misses, int64_t *table_len) {
    OrcJob j;
    j.m = m; j.g = g; j.lats = lats; j.n_lat = n_lat; j.lm_weight = lm_weight;
    j.beam = beam; j.enabled = enabled; j.res = res; j.rcs = rcs; j.next = 0;
    j.lookups = lookups; j.hits = hits; j.misses = misses; j.table_len = table_len;
    pthread_mutex_init(&j.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int32_t t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, orc_worker, &j);
    for (int32_t t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&j.mu);
    for (int32_t i = 0; i < n_lat; i++) if (rcs[i]) return rcs[i];
    return ORC_OK;
}

int orc_decode_many(const OrcModel *m, const OrcNgram *g, const OrcLattice *lats,
                    int32_t n_lat, double lm_weight, int64_t beam, int32_t enabled,
                    int32_t n_threads, OrcResult *res, int32_t *rcs,
                    int64_t *lookups, int64_t *hits, int64_t *misses) {
    return orc_decode_many_t(m, g, lats, n_lat, lm_weight, beam, enabled, n_threads, res, rcs,
                             lookups, hits, misses, NULL);
}

/* Batched kernel-level helpers (threaded) for the query microbench and
 * for parity tests at sizes where a Python loop would be slow. */
typedef struct {
    const OrcModel *m; int64_t n; const float *h; const int64_t *hist; const int32_t *hlen;
    const int32_t *w; double *p; float *h_out; int32_t nt, t;
} OrcQJob;

static void *orc_qworker(void *arg) {
    OrcQJob *q = (OrcQJob *)arg;
    const OrcModel *m = q->m;
    for (int64_t i = q->t; i < q->n; i += q->nt) {
        const float *h = q->h + (size_t)i * m->H;
        const int64_t *hist = q->hist + (size_t)i * m->order;
        int32_t w = q->w[i];
        int64_t o0 = m->path_offsets[w], o1 = m->path_offsets[w + 1];
        if (q->p)
            q->p[i] = orc_word_logprob(h, m->H, hist, q->hlen[i], m->path_nodes + o0,
                                       m->path_signs + o0, o1 - o0, m->NV, m->ME, m->order,
                                       m->seed, m->maxent_size - 1);
        if (q->h_out)
            orc_advance_hidden(m->U + (size_t)w * m->H, m->W, h, m->H, q->h_out + (size_t)i * m->H);
    }
    return NULL;
}

void orc_query_batch(const OrcModel *m, int64_t n, const float *h, const int64_t *hist,
                     const int32_t *hlen, const int32_t *w, double *p, float *h_out,
                     int32_t n_threads) {
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    OrcQJob *jobs = (OrcQJob *)malloc(sizeof(OrcQJob) * (size_t)n_threads);
    for (int32_t t = 0; t < n_threads; t++) {
        jobs[t] = (OrcQJob){m, n, h, hist, hlen, w, p, h_out, n_threads, t};
        pthread_create(&th[t], NULL, orc_qworker, &jobs[t]);
    }
    for (int32_t t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th); free(jobs);
}

/* ------------------------------------------------------------------ */
/* Two-pass rescoring: nbest (decoder.py:180-230) and rescore_twopass   */
/* (decoder.py:243-274).                                                */
/* ------------------------------------------------------------------ */
static double orc_pysum(const double *x, const int32_t *idx, int32_t n);
typedef struct { double key; uint64_t counter; int32_t done, node; double g; int64_t path; } OrcNbEnt;
typedef struct { int32_t arc; int64_t parent; } OrcNbLink;

/* heap order of the reference tuples (-f, counter, ...): counter is unique */
static int orc_nb_less(const OrcNbEnt *a, const OrcNbEnt *b) {
    if (a->key < b->key) return 1;
    if (a->key > b->key) return 0;
    return a->counter < b->counter;
}

static uint64_t orc_words_hash(const int32_t *w, int32_t n) {
    uint64_t h = 0xcbf29ce484222325ULL ^ (uint64_t)n;
    for (int32_t i = 0; i < n; i++) h = orc_mix(h, (uint64_t)(uint32_t)w[i]);
    return h;
}

/* nbest: exact best-first search with the backward-Viterbi completion as
 * heuristic; the first complete path of each distinct word sequence is
 * kept (decoder.py:180-230).  Outputs: *n_out hypotheses, hyp_len [n],
 * arcs (concatenated, capacity arcs_cap), scores [n, 3] = (combined,
 * acoustic, lm).  Returns ORC_ERR_NOMEM with *arcs_needed set when
 * arcs_cap is too small. */
int orc_nbest(const OrcLattice *lat, int32_t n, double lm_weight, int32_t *n_out,
              int32_t *hyp_len, int32_t *arcs, int64_t arcs_cap, double *scores,
              int64_t *arcs_needed) {
    if (n < 1) return ORC_ERR_VALUE;
    int32_t N = lat->n_nodes;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    int32_t *out_off = (int32_t *)calloc((size_t)N + 1, sizeof(int32_t));
    int32_t *out_arc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(lat->n_arcs > 0 ? lat->n_arcs : 1));
    int rc = orc_topo(lat, order, out_off, out_arc);
    if (rc) { free(order); free(out_off); free(out_arc); return rc; }
    uint8_t *is_final = (uint8_t *)calloc((size_t)N + 1, 1);
    for (int32_t i = 0; i < lat->n_finals; i++) is_final[lat->finals[i]] = 1;
    double *comp = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    for (int32_t k = N - 1; k >= 0; k--) {            /* decoder.py:191-198 */
        int32_t v = order[k];
        double best = is_final[v] ? 0.0 : -INFINITY;
        for (int32_t e = out_off[v]; e < out_off[v + 1]; e++) {
            int32_t a = out_arc[e];
            double cand = (lat->ac[a] + lm_weight * lat->slm[a]) + comp[lat->dst[a]];
            if (cand > best) best = cand;
        }
        comp[v] = best;
    }
    *n_out = 0;
    *arcs_needed = 0;
    if (comp[lat->start] == -INFINITY) {
        free(order); free(out_off); free(out_arc); free(is_final); free(comp);
        return ORC_ERR_NO_PATH;
    }
    size_t hcap = 1024, hn = 0, lcap = 1024, ln = 0;
    OrcNbEnt *heap = (OrcNbEnt *)malloc(sizeof(OrcNbEnt) * hcap);
    OrcNbLink *links = (OrcNbLink *)malloc(sizeof(OrcNbLink) * lcap);
    /* seen word sequences: open addressing over (hash, offset, len) */
    size_t scap = 1024;
    uint64_t *s_hash = (uint64_t *)calloc(scap, sizeof(uint64_t));
    int64_t *s_off = (int64_t *)malloc(sizeof(int64_t) * scap);
    int32_t *s_len = (int32_t *)malloc(sizeof(int32_t) * scap);
    uint8_t *s_used = (uint8_t *)calloc(scap, 1);
    size_t s_n = 0, wcap = 4096, wn = 0;
    int32_t *warena = (int32_t *)malloc(sizeof(int32_t) * wcap);
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    int32_t *tmpw = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    uint64_t counter = 0;
    int64_t arcs_used = 0;

#define NB_PUSH(E) do {                                                                  \
        if (hn == hcap) { hcap *= 2; heap = (OrcNbEnt *)realloc(heap, sizeof(OrcNbEnt) * hcap); } \
        size_t _i = hn++; heap[_i] = (E);                                                \
        while (_i > 0) { size_t _p = (_i - 1) / 2;                                       \
            if (!orc_nb_less(&heap[_i], &heap[_p])) break;                               \
            OrcNbEnt _t = heap[_p]; heap[_p] = heap[_i]; heap[_i] = _t; _i = _p; }       \
    } while (0)

    OrcNbEnt e0 = {-comp[lat->start], counter, 0, lat->start, 0.0, -1};
    NB_PUSH(e0);
    while (hn > 0 && *n_out < n) {
        OrcNbEnt cur = heap[0];
        heap[0] = heap[--hn];
        for (size_t i = 0;;) {
            size_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < hn && orc_nb_less(&heap[l], &heap[m])) m = l;
            if (r < hn && orc_nb_less(&heap[r], &heap[m])) m = r;
            if (m == i) break;
            OrcNbEnt t = heap[m]; heap[m] = heap[i]; heap[i] = t; i = m;
        }
        if (cur.done) {                                  /* decoder.py:207-218 */
            int32_t L = 0;
            for (int64_t p = cur.path; p >= 0; p = links[p].parent) tmp[L++] = links[p].arc;
            for (int32_t i = 0; i < L / 2; i++) { int32_t t = tmp[i]; tmp[i] = tmp[L - 1 - i]; tmp[L - 1 - i] = t; }
            for (int32_t i = 0; i < L; i++) tmpw[i] = lat->word[tmp[i]];
            uint64_t hh = orc_words_hash(tmpw, L);
            size_t slot = (size_t)(hh & (scap - 1));
            int dup = 0;
            while (s_used[slot]) {
                if (s_hash[slot] == hh && s_len[slot] == L &&
                    memcmp(warena + s_off[slot], tmpw, sizeof(int32_t) * (size_t)L) == 0) { dup = 1; break; }
                slot = (slot + 1) & (scap - 1);
            }
            if (dup) continue;
            if (wn + (size_t)L > wcap) { while (wn + (size_t)L > wcap) wcap *= 2; warena = (int32_t *)realloc(warena, sizeof(int32_t) * wcap); }
            memcpy(warena + wn, tmpw, sizeof(int32_t) * (size_t)L);
            s_used[slot] = 1; s_hash[slot] = hh; s_off[slot] = (int64_t)wn; s_len[slot] = L;
            wn += (size_t)L;
            if (++s_n * 2 > scap) {                      /* rehash */
                size_t ncap = scap * 2;
                uint64_t *nh = (uint64_t *)calloc(ncap, sizeof(uint64_t));
                int64_t *no = (int64_t *)malloc(sizeof(int64_t) * ncap);
                int32_t *nl = (int32_t *)malloc(sizeof(int32_t) * ncap);
                uint8_t *nu = (uint8_t *)calloc(ncap, 1);
                for (size_t i = 0; i < scap; i++) if (s_used[i]) {
                    size_t q = (size_t)(s_hash[i] & (ncap - 1));
                    while (nu[q]) q = (q + 1) & (ncap - 1);
                    nu[q] = 1; nh[q] = s_hash[i]; no[q] = s_off[i]; nl[q] = s_len[i];
                }
                free(s_hash); free(s_off); free(s_len); free(s_used);
                s_hash = nh; s_off = no; s_len = nl; s_used = nu; scap = ncap;
            }
            double ac = orc_pysum(lat->ac, tmp, L), lm = orc_pysum(lat->slm, tmp, L);
            int32_t k = (*n_out)++;
            hyp_len[k] = L;
            scores[3 * k] = cur.g; scores[3 * k + 1] = ac; scores[3 * k + 2] = lm;
            if (arcs_used + L <= arcs_cap) memcpy(arcs + arcs_used, tmp, sizeof(int32_t) * (size_t)L);
            arcs_used += L;
            continue;
        }
        if (is_final[cur.node]) {                        /* decoder.py:220-222 */
            OrcNbEnt e = {-cur.g, ++counter, 1, cur.node, cur.g, cur.path};
            NB_PUSH(e);
        }
        for (int32_t x = out_off[cur.node]; x < out_off[cur.node + 1]; x++) {
            int32_t a = out_arc[x];
            double tail = comp[lat->dst[a]];
            if (tail == -INFINITY) continue;
            double g2 = cur.g + (lat->ac[a] + lm_weight * lat->slm[a]);
            if (ln == lcap) { lcap *= 2; links = (OrcNbLink *)realloc(links, sizeof(OrcNbLink) * lcap); }
            links[ln].arc = a; links[ln].parent = cur.path;
            OrcNbEnt e = {-(g2 + tail), ++counter, 0, lat->dst[a], g2, (int64_t)ln};
            ln++;
            NB_PUSH(e);
        }
    }
#undef NB_PUSH
    *arcs_needed = arcs_used;
    free(order); free(out_off); free(out_arc); free(is_final); free(comp); free(heap); free(links);
    free(s_hash); free(s_off); free(s_len); free(s_used); free(warena); free(tmp); free(tmpw);
    return arcs_used > arcs_cap ? ORC_ERR_NOMEM : ORC_OK;
}

/* CPython >= 3.12 builtin sum() over floats starting from int 0: the first
 * item is taken exactly, the rest use Neumaier-compensated summation, and the
 * compensation is added once at the end (Python/bltinmodule.c builtin_sum_impl). */
static double orc_pysum(const double *x, const int32_t *idx, int32_t n) {
    if (n == 0) return 0.0;
    double f = 0.0 + x[idx[0]], c = 0.0;
    for (int32_t i = 1; i < n; i++) {
        double v = x[idx[i]], t = f + v;
        if (fabs(f) >= fabs(v)) c += (f - t) + v;
        else c += (v - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* _hybrid_logprob: decoder.py:233-240 */
static double orc_hybrid(double lp_ng, double lp_rnn, double lam) {
    if (lam >= 1.0) return lp_ng;
    if (lam <= 0.0) return lp_rnn;
    double hi = lp_ng > lp_rnn ? lp_ng : lp_rnn;
    return hi + log(lam * exp(lp_ng - hi) + (1.0 - lam) * exp(lp_rnn - hi));
}

/* rescore_twopass (decoder.py:243-274) for one n-best list: per hypothesis
 * a fresh zero context, word-by-word score then advance; mode 0 = rnnlm,
 * 1 = hybrid.  lm_out / combined_out [n_hyp]; *best = index of the first
 * maximum (strict >).  g may be NULL in rnnlm mode. */
int orc_twopass(const OrcModel *m, const OrcNgram *g, int32_t n_hyp, const int64_t *hyp_off,
                const int32_t *words, const double *acoustic, int32_t mode, double lam,
                double lm_weight, double *lm_out, double *combined_out, int32_t *best) {
    if (n_hyp < 1 || mode < 0 || mode > 1 || (mode == 1 && !g)) return ORC_ERR_VALUE;
    float *h = (float *)calloc((size_t)m->H, sizeof(float));
    float *h2 = (float *)calloc((size_t)m->H, sizeof(float));
    int rc = ORC_OK;
    *best = -1;
    double best_s = 0.0;
    for (int32_t j = 0; j < n_hyp && rc == ORC_OK; j++) {
        memset(h, 0, sizeof(float) * (size_t)m->H);
        int64_t hist[16]; int32_t L = 0;
        double lm = 0.0;
        const int32_t *ws = words + hyp_off[j];
        int64_t len = hyp_off[j + 1] - hyp_off[j];
        for (int64_t i = 0; i < len; i++) {
            int32_t w = ws[i];
            if (w < 0 || w >= m->V) { rc = ORC_ERR_VALUE; break; }
            int64_t o0 = m->path_offsets[w], o1 = m->path_offsets[w + 1];
            double lp_rnn = orc_word_logprob(h, m->H, hist, L, m->path_nodes + o0, m->path_signs + o0,
                                             o1 - o0, m->NV, m->ME, m->order, m->seed, m->maxent_size - 1);
            if (mode == 0) {
                lm += lp_rnn;
            } else {
                int32_t need = g->order - 1, ctx[ORC_MAX_NGRAM], nc = 0;
                if (need > 0) {
                    if (i < need) for (int64_t k = 0; k < need - i; k++) ctx[nc++] = g->bos;
                    for (int64_t k = (i < need ? 0 : i - need); k < i; k++) ctx[nc++] = ws[k];
                }
                double lp_ng;
                rc = orc_ngram_logprob(g, ctx, nc, w, &lp_ng);
                if (rc) break;
                lm += orc_hybrid(lp_ng, lp_rnn, lam);
            }
            orc_advance_hidden(m->U + (size_t)w * m->H, m->W, h, m->H, h2);
            memcpy(h, h2, sizeof(float) * (size_t)m->H);
            if (L < m->order) hist[L++] = w;
            else { for (int32_t k = 1; k < L; k++) hist[k - 1] = hist[k]; hist[L - 1] = w; }
        }
        double combined = acoustic[j] + lm_weight * lm;
        lm_out[j] = lm;
        combined_out[j] = combined;
        if (*best < 0 || combined > best_s) { *best = j; best_s = combined; }
    }
    free(h); free(h2);
    return rc;
}

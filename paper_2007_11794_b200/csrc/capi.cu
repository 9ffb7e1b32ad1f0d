// capi.cu -- C-ABI of libotflm_b200.so (declared in include/otflm_b200.h):
// model / small-LM upload, per-stream device tables, the host lattice
// compiler (topological levels, per-node beam capacities, arrival slots) and
// the level loop (captured once into a CUDA graph and replayed).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "../../include/otflm_b200.h"
#include "common.cuh"
#include "decode.cuh"
#include "hs.cuh"
#include "tc_advance.cuh"
#include "stream_decode.cuh"
#include "exact_solo.cuh"

// --------------------------------------------------------------------------
static thread_local std::string g_detail;
static thread_local int64_t g_launches = 0;

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t _e = (x);                                                    \
        if (_e != cudaSuccess) {                                                 \
            g_detail = std::string(#x) + ": " + cudaGetErrorString(_e);          \
            return OTFLM_ERR_CUDA;                                               \
        }                                                                        \
    } while (0)
#define CKL()                                                                    \
    do {                                                                         \
        g_launches++;                                                            \
        cudaError_t _e = cudaGetLastError();                                     \
        if (_e != cudaSuccess) {                                                 \
            g_detail = std::string("launch: ") + cudaGetErrorString(_e);         \
            return OTFLM_ERR_CUDA;                                               \
        }                                                                        \
    } while (0)

// ---- optional per-kernel CUDA-event timing (non-graph runs only) ----
enum { K_EXPAND, K_HS, K_ADVANCE, K_ASSIGN, K_FINAL, K_MISC, K_STREAM, K_NCAT };
static bool g_prof = false;
static std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> g_prof_ev;
static double g_prof_ms[K_NCAT];
static long long g_prof_n[K_NCAT];
// Recorded only while capturing a profiling graph: external event-record
// nodes around each kernel, so the timings are device-side kernel spans of a
// graph replay (no host launch gaps).
struct ProfScope {
    int cat; cudaStream_t s; cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(int c, cudaStream_t st) : cat(c), s(st) {
        if (g_prof) {
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecordWithFlags(a, s, cudaEventRecordExternal);
        }
    }
    ~ProfScope() {
        if (g_prof) {
            cudaEventRecordWithFlags(b, s, cudaEventRecordExternal);
            g_prof_ev.push_back({cat, {a, b}});
        }
    }
};

static inline uint32_t pow2_at_least(uint64_t x) {
    uint64_t c = 16;
    while (c < x) c <<= 1;
    return (uint32_t)c;
}
static inline unsigned cdiv(uint64_t a, uint64_t b) { return (unsigned)((a + b - 1) / b); }

struct Allocs {
    std::vector<void *> ptrs;
    template <class T>
    cudaError_t alloc(T **p, size_t count) {
        void *q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) { ptrs.push_back(q); *p = (T *)q; }
        return e;
    }
    void free_all() {
        for (void *p : ptrs) cudaFree(p);
        ptrs.clear();
    }
};

// OTFLM_PREC_EXACT runs the integer digit-plane update only in the persistent
// stream kernel; everywhere else it is the FP64 path (both are bit-exact with
// the reference's float32 results: exact_update.cuh, hs.cuh)
static inline bool prec_ok(int p) { return p >= 0 && p <= 4; }
static inline int level_prec(int p) { return p == OTFLM_PREC_EXACT ? OTFLM_PREC_FP64 : p; }

// ==========================================================================
// model
// ==========================================================================
struct OtflmModel {
    DevModel d;
    int device;
    Allocs mem;
    int64_t n_path;
    // tensor-core copies of the node vectors (all_word_logprobs), made on first use
    mutable std::mutex nv_mu;
    mutable float *NV_hi = nullptr, *NV_lo = nullptr;
    mutable __nv_bfloat16 *NV_bf = nullptr;
};

__global__ void k_prep_weights(DevModel m, float *WT, float *W_hi, float *W_lo, __nv_bfloat16 *W_bf) {
    const int64_t HH = (int64_t)m.H * m.H;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < HH; t += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(t / m.H), j = (int)(t % m.H);
        float w = m.W[t];
        WT[(int64_t)j * m.H + i] = w;
        // tf32 split: hi = round-to-nearest tf32 (10-bit mantissa), lo = rest
        uint32_t b = __float_as_uint(w);
        uint32_t r = (b + 0x1000u) & 0xFFFFE000u;
        float hi = __uint_as_float(r);
        float lo = w - hi;
        uint32_t lb = (__float_as_uint(lo) + 0x1000u) & 0xFFFFE000u;
        W_hi[t] = hi;
        W_lo[t] = __uint_as_float(lb);
        W_bf[t] = __float2bfloat16_rn(w);
    }
}

// W_hi / W_lo into the persistent kernel's chunked canonical tiles (see DevModel::W_t)
__global__ void k_prep_wtiles(DevModel m, float *wt, int kcb) {
    const int H = m.H, np = m.wt_npad, KE = kcb / 4;
    const int NK = (H + KE - 1) / KE;
    const int64_t total = (int64_t)NK * 2 * np * KE;
    const int64_t blk = (int64_t)np * KE;                  // floats per [hi] or [lo] block
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(t % KE);
        const int row = (int)((t / KE) % np);
        const int part = (int)((t / ((int64_t)KE * np)) % 2);
        const int kc = (int)(t / ((int64_t)KE * np * 2));
        const int k = kc * KE + kk;
        float v = 0.f;
        if (row < H && k < H) v = (part ? m.W_lo : m.W_hi)[(int64_t)row * H + k];
        const int sh = kcb == 128 ? 0 : kcb == 64 ? 1 : 2;      // swizzled K-major (tc::swz_off)
        const int64_t off = (int64_t)(kc * 2 + part) * blk +
                            ((row >> 3) * (8 * kcb) + (row & 7) * kcb + ((((kk >> 2) ^ ((row & 7) >> sh))) << 4)) / 4 +
                            (kk & 3);
        wt[off] = v;
    }
}

extern "C" int otflm_model_create(const OtflmModelDesc *d, int32_t device, OtflmModel **out) {
    {   // stream-ordered scratch (cudaMallocAsync) stays pooled across calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    if (!d || !out) return OTFLM_ERR_VALUE;
    if (d->hidden_size < 1 || d->vocab_size < 2 || d->maxent_order < 1 ||
        d->maxent_order > OTF_MAX_ORDER || d->maxent_size < 1 ||
        (d->maxent_size & (d->maxent_size - 1))) {
        g_detail = "bad model geometry";
        return OTFLM_ERR_VALUE;
    }
    CK(cudaSetDevice(device));
    OtflmModel *m = new OtflmModel();
    m->device = device;
    const int H = d->hidden_size, V = d->vocab_size;
    m->n_path = d->n_path;
    DevModel &dm = m->d;
    dm.H = H; dm.V = V; dm.order = d->maxent_order;
    dm.mask = d->maxent_size - 1; dm.seed = d->hash_seed;
    float *U = nullptr, *W = nullptr, *WT = nullptr, *NV = nullptr, *ME = nullptr, *Whi = nullptr, *Wlo = nullptr;
    __nv_bfloat16 *Wbf = nullptr;
    uint32_t *poff = nullptr, *pcode = nullptr;
    const size_t VH = (size_t)V * H, HH = (size_t)H * H;
    // every weight block is optional (the reference-signature kernel calls
    // upload only what they use); the decoder requires all of them
#define AL(p, n) if (m->mem.alloc(&p, n) != cudaSuccess) { m->mem.free_all(); delete m; g_detail = "cudaMalloc model"; return OTFLM_ERR_NOMEM; }
    if (d->input_weights) { AL(U, VH); CK(cudaMemcpy(U, d->input_weights, VH * 4, cudaMemcpyHostToDevice)); }
    if (d->recurrent_weights) {
        AL(W, HH); AL(WT, HH); AL(Whi, HH); AL(Wlo, HH); AL(Wbf, HH);
        CK(cudaMemcpy(W, d->recurrent_weights, HH * 4, cudaMemcpyHostToDevice));
    }
    if (d->node_vectors) { AL(NV, (size_t)(V - 1) * H); CK(cudaMemcpy(NV, d->node_vectors, (size_t)(V - 1) * H * 4, cudaMemcpyHostToDevice)); }
    if (d->maxent_table) { AL(ME, d->maxent_size); CK(cudaMemcpy(ME, d->maxent_table, d->maxent_size * 4, cudaMemcpyHostToDevice)); }
    if (d->path_offsets && d->n_path >= 0) {
        AL(poff, (size_t)V + 1); AL(pcode, (size_t)std::max<int64_t>(d->n_path, 1));
        std::vector<uint32_t> off(V + 1), code(std::max<int64_t>(d->n_path, 1));
        for (int w = 0; w <= V; w++) off[w] = (uint32_t)d->path_offsets[w];
        if (off[V] != (uint64_t)d->n_path) { m->mem.free_all(); delete m; g_detail = "path_offsets[V] != n_path"; return OTFLM_ERR_VALUE; }
        for (int64_t p = 0; p < d->n_path; p++) {
            if (d->path_nodes[p] < 0 || d->path_nodes[p] >= V - 1) { m->mem.free_all(); delete m; g_detail = "bad path node"; return OTFLM_ERR_VALUE; }
            code[p] = (uint32_t)d->path_nodes[p] | (d->path_signs[p] < 0.f ? 0x80000000u : 0u);
        }
        CK(cudaMemcpy(poff, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pcode, code.data(), (size_t)std::max<int64_t>(d->n_path, 1) * 4, cudaMemcpyHostToDevice));
    }
#undef AL
    dm.U = U; dm.W = W; dm.WT = WT; dm.NV = NV; dm.ME = ME;
    dm.path_off = poff; dm.path_code = pcode;
    dm.W_hi = Whi; dm.W_lo = Wlo; dm.W_bf = Wbf;
    dm.W_t = nullptr; dm.wt_kcb = 0; dm.wt_npad = 0; dm.W_t64 = nullptr;
    dm.Wd = nullptr; dm.wx = nullptr; dm.wd_nkx = 0; dm.NVd = nullptr; dm.nx = nullptr;
    if (W) {
        k_prep_weights<<<256, 256>>>(dm, WT, Whi, Wlo, Wbf);
        CK(cudaGetLastError());
        const int np = (H + 127) / 128 * 128;             // whole 128-row M tiles
        if (np <= 512) {
            const int kcb = np <= 256 ? 128 : 64, KE = kcb / 4, NK = (H + KE - 1) / KE;   // few, large K chunks
            float *Wt = nullptr;
            const size_t nwt = (size_t)NK * 2 * np * KE;
            if (m->mem.alloc(&Wt, nwt) != cudaSuccess) { m->mem.free_all(); delete m; g_detail = "cudaMalloc model"; return OTFLM_ERR_NOMEM; }
            dm.W_t = Wt; dm.wt_kcb = kcb; dm.wt_npad = np;
            k_prep_wtiles<<<256, 256>>>(dm, Wt, kcb);
            CK(cudaGetLastError());
            float *Wt64 = nullptr;
            const size_t nwt64 = (size_t)((H + 15) / 16) * 2 * np * 16;
            if (m->mem.alloc(&Wt64, nwt64) != cudaSuccess) { m->mem.free_all(); delete m; g_detail = "cudaMalloc model"; return OTFLM_ERR_NOMEM; }
            dm.W_t64 = Wt64;
            k_prep_wtiles<<<256, 256>>>(dm, Wt64, 64);
            CK(cudaGetLastError());
            // exact mode: 8-bit digit planes of W + per-unit bound constants
            const int nkx = (H + xu::KC - 1) / xu::KC;
            uint8_t *Wd = nullptr;
            double4 *wx = nullptr;
            const size_t nwd = (size_t)(np / tc::BM) * nkx * xu::NPW * xu::PLANE_W;
            if (m->mem.alloc(&Wd, nwd) != cudaSuccess || m->mem.alloc(&wx, (size_t)H) != cudaSuccess) {
                m->mem.free_all(); delete m; g_detail = "cudaMalloc model"; return OTFLM_ERR_NOMEM;
            }
            CK(cudaMemset(Wd, 0, nwd));
            k_prep_wdigits<<<H, 256>>>(W, U, V, H, nkx, Wd, wx);
            CK(cudaGetLastError());
            dm.Wd = Wd; dm.wx = wx; dm.wd_nkx = nkx;
            if (NV) {        // the HS node vectors as digit planes (exact HS on rank 0's tensor core)
                uint8_t *NVd = nullptr;
                double4 *nx = nullptr;
                const size_t nnv = (size_t)(V - 1) * nkx * xu::NPW * xu::KC;
                if (m->mem.alloc(&NVd, nnv) != cudaSuccess || m->mem.alloc(&nx, (size_t)(V - 1)) != cudaSuccess) {
                    m->mem.free_all(); delete m; g_detail = "cudaMalloc model"; return OTFLM_ERR_NOMEM;
                }
                k_prep_wdigits<<<V - 1, 256>>>(NV, nullptr, V, H, nkx, NVd, nx, V - 1, 1);
                CK(cudaGetLastError());
                dm.NVd = NVd; dm.nx = nx;
            }
        }
    }
    CK(cudaDeviceSynchronize());
    *out = m;
    return OTFLM_OK;
}

extern "C" int otflm_model_destroy(OtflmModel *m) {
    if (!m) return OTFLM_OK;
    cudaSetDevice(m->device);
    m->mem.free_all();
    delete m;
    return OTFLM_OK;
}

extern "C" int otflm_model_info(const OtflmModel *m, int64_t *o) {
    if (!m || !o) return OTFLM_ERR_VALUE;
    o[0] = m->d.H; o[1] = m->d.V; o[2] = m->d.order; o[3] = (int64_t)(m->d.mask + 1);
    o[4] = (int64_t)(uintptr_t)m->d.U; o[5] = (int64_t)(uintptr_t)m->d.NV;
    o[6] = (int64_t)(uintptr_t)m->d.ME; o[7] = m->n_path;
    return OTFLM_OK;
}

// ==========================================================================
// small LM
// ==========================================================================
struct OtflmNgram {
    DevNgram d;
    Allocs mem;
};

static int build_ng_table(int order, int64_t n, const int32_t *keys, const int32_t *lens,
                          const double *vals, uint32_t &cap, std::vector<uint64_t> &tag,
                          std::vector<int32_t> &words, std::vector<double> &val) {
    const int width = order + 1;
    cap = pow2_at_least((uint64_t)std::max<int64_t>(n, 1) * 2);
    tag.assign(cap, 0);
    words.assign((size_t)cap * width, 0);
    val.assign(cap, 0.0);
    for (int64_t r = 0; r < n; r++) {
        const int len = lens[r];
        if (len < 0 || len > order) return OTFLM_ERR_VALUE;
        const int32_t *k = keys + r * order;
        uint64_t h = otf_tuple_hash(k, len);
        uint32_t s = (uint32_t)(h >> 7) & (cap - 1);
        for (;;) {
            if (tag[s] == 0) break;
            if (tag[s] == h && words[(size_t)s * width] == len &&
                std::equal(k, k + len, &words[(size_t)s * width + 1]))
                break;   // duplicate key: last one wins (dict semantics)
            s = (s + 1) & (cap - 1);
        }
        tag[s] = h;
        words[(size_t)s * width] = len;
        for (int i = 0; i < len; i++) words[(size_t)s * width + 1 + i] = k[i];
        val[s] = vals[r];
    }
    return OTFLM_OK;
}

extern "C" int otflm_ngram_create(const OtflmNgramDesc *d, const OtflmModel *m, OtflmNgram **out) {
    if (!d || !out) return OTFLM_ERR_VALUE;
    if (d->order < 1 || d->order > OTF_MAX_ORDER) { g_detail = "small LM order out of range"; return OTFLM_ERR_VALUE; }
    if (m && d->order - 1 > m->d.order) {
        g_detail = "small LM order exceeds the stored context history";   // decoder.py:87-90
        return OTFLM_ERR_VALUE;
    }
    OtflmNgram *g = new OtflmNgram();
    g->d.order = d->order; g->d.V = d->vocab_size; g->d.bos = d->bos_id;
    std::vector<uint64_t> pt, bt;
    std::vector<int32_t> pw, bw;
    std::vector<double> pv, bv;
    int rc = build_ng_table(d->order, d->n_probs, d->prob_keys, d->prob_lens, d->prob_vals, g->d.p_cap, pt, pw, pv);
    if (!rc) rc = build_ng_table(d->order, d->n_backoffs, d->bow_keys, d->bow_lens, d->bow_vals, g->d.b_cap, bt, bw, bv);
    if (rc) { delete g; g_detail = "bad n-gram key length"; return rc; }
    uint64_t *dpt, *dbt; int32_t *dpw, *dbw; double *dpv, *dbv;
    if (g->mem.alloc(&dpt, pt.size()) || g->mem.alloc(&dpw, pw.size()) || g->mem.alloc(&dpv, pv.size()) ||
        g->mem.alloc(&dbt, bt.size()) || g->mem.alloc(&dbw, bw.size()) || g->mem.alloc(&dbv, bv.size())) {
        g->mem.free_all(); delete g; return OTFLM_ERR_NOMEM;
    }
    CK(cudaMemcpy(dpt, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpw, pw.data(), pw.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpv, pv.data(), pv.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dbt, bt.data(), bt.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dbw, bw.data(), bw.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dbv, bv.data(), bv.size() * 8, cudaMemcpyHostToDevice));
    g->d.p_tag = dpt; g->d.p_words = dpw; g->d.p_val = dpv;
    g->d.b_tag = dbt; g->d.b_words = dbw; g->d.b_val = dbv;
    *out = g;
    return OTFLM_OK;
}

extern "C" int otflm_ngram_destroy(OtflmNgram *g) {
    if (!g) return OTFLM_OK;
    g->mem.free_all();
    delete g;
    return OTFLM_OK;
}

__global__ void k_ngram_batch(DevNgram g, int64_t n, const int32_t *ctx, const int32_t *w, double *out,
                              unsigned int *err) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t hist[OTF_MAX_ORDER];
    int L = g.order - 1;
    for (int k = 0; k < L; k++) hist[k] = (uint32_t)ctx[i * (g.order > 1 ? g.order - 1 : 1) + k];
    double v;
    if (w[i] < 0 || w[i] >= g.V) { atomicOr(err, OTF_E_VALUE); out[i] = 0; return; }
    if (!ngram_logprob_dev(g, hist, L, w[i], &v)) { atomicOr(err, OTF_E_KEY); v = 0; }
    out[i] = v;
}

static unsigned int *scratch_err() {
    static unsigned int *p = nullptr;
    if (!p) cudaMalloc(&p, 4);
    return p;
}

extern "C" int otflm_ngram_logprob_batch(const OtflmNgram *g, int64_t n, const int32_t *ctx, const int32_t *w,
                                         double *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    unsigned int *err = scratch_err();
    CK(cudaMemsetAsync(err, 0, 4, s));
    if (n > 0) { k_ngram_batch<<<cdiv(n, 256), 256, 0, s>>>(g->d, n, ctx, w, out, err); CKL(); }
    unsigned int he = 0;
    CK(cudaMemcpyAsync(&he, err, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (he & OTF_E_VALUE) return OTFLM_ERR_VALUE;
    if (he & OTF_E_KEY) return OTFLM_ERR_KEY;
    return OTFLM_OK;
}

// ==========================================================================
// kernel table
// ==========================================================================
extern "C" int otflm_feature_index_batch(uint64_t seed, uint64_t mask, int64_t n, const int32_t *order_k,
                                         const int64_t *words, const int64_t *node, uint64_t *out, void *stream) {
    if (n <= 0) return OTFLM_OK;
    k_feature_index<<<cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(seed, mask, n, order_k, words, node, out);
    CKL();
    return OTFLM_OK;
}

static int launch_ring_batch(const DevModel &m, int64_t n, const int32_t *ctx, const float *h, const int32_t *hist,
                             const int32_t *hist_len, const int32_t *w, double *out, bool exact, cudaStream_t s) {
    const size_t smem = 4 * ring_bytes_per_warp(m.H);
    int per_sm = 1;
#define CALLR(CPL, EX, ORD)                                                                                        \
    do {                                                                                                           \
        CK(cudaFuncSetAttribute(k_word_logprob_ring<CPL, EX, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_word_logprob_ring<CPL, EX, ORD>, 128, smem)); \
        const unsigned grid = (unsigned)std::min<int64_t>(cdiv(n, 4), (int64_t)148 * std::max(per_sm, 1));        \
        k_word_logprob_ring<CPL, EX, ORD><<<grid, 128, smem, s>>>(m, n, ctx, h, hist, hist_len, w, out);           \
    } while (0)
    if (exact) RING_DISPATCH(m.H, true, m.order, CALLR);
    else RING_DISPATCH(m.H, false, m.order, CALLR);
#undef CALLR
    CKL();
    return OTFLM_OK;
}

extern "C" int otflm_word_logprob_batch2(const OtflmModel *m, int64_t n, const int32_t *ctx, const float *h,
                                         const int32_t *hist, const int32_t *hist_len, const int32_t *w,
                                         double *out, int32_t exact, void *stream) {
    if (n <= 0) return OTFLM_OK;
    if (!m->d.NV || !m->d.ME || !m->d.path_off) { g_detail = "model has no output layer"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    if (m->d.H % 4 == 0 && m->d.H <= 1024)
        return launch_ring_batch(m->d, n, ctx, h, hist, hist_len, w, out, exact != 0, s);
    const unsigned blocks = cdiv(n, 8);
#define CALL(VEC, CPL) k_word_logprob_batch<VEC, CPL><<<blocks, 256, 0, s>>>(m->d, n, ctx, h, hist, hist_len, w, out)
    HS_DISPATCH(m->d.H, CALL);
#undef CALL
    CKL();
    return OTFLM_OK;
}

extern "C" int otflm_word_logprob_batch(const OtflmModel *m, int64_t n, const int32_t *ctx, const float *h,
                                        const int32_t *hist, const int32_t *hist_len, const int32_t *w,
                                        double *out, void *stream) {
    return otflm_word_logprob_batch2(m, n, ctx, h, hist, hist_len, w, out, 1, stream);
}

extern "C" int otflm_word_logprob_paths(const OtflmModel *m, int64_t n, const int32_t *ctx, const float *h,
                                        const int32_t *hist, const int32_t *hist_len, const int64_t *path_off,
                                        const uint32_t *path_code, double *out, void *stream) {
    if (n <= 0) return OTFLM_OK;
    if (!m->d.NV || !m->d.ME) { g_detail = "model has no output layer"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned blocks = cdiv(n, 8);
#define CALL(VEC, CPL) k_word_logprob_paths<VEC, CPL><<<blocks, 256, 0, s>>>(m->d, n, ctx, h, hist, hist_len, path_off, path_code, out)
    HS_DISPATCH(m->d.H, CALL);
#undef CALL
    CKL();
    return OTFLM_OK;
}

static int launch_advance(const DevModel &m, int prec, uint32_t n_cap, const RowSpec &rs,
                          const int32_t *in_row, const int32_t *words, const float *h_base, float *out_base,
                          uint32_t row_limit, cudaStream_t s) {
    if (n_cap == 0) return OTFLM_OK;
    if (prec == OTFLM_PREC_EXACT && m.Wd && m.H % 4 == 0) {
        // persistent digit-plane update: a two-slot digit scratch per CTA,
        // stream-ordered (pooled; also valid inside a graph capture)
        const size_t stride = 2 * xu::xs_slot_bytes(m.wd_nkx);
        const size_t stages = std::min<size_t>(4, (200u * 1024u - xu::tail_layout().total) / xu::STAGE);
        const size_t smem = stages * xu::STAGE + xu::tail_layout().total;
        const unsigned grid = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>(148, (n_cap + xu::XR - 1) / xu::XR));
        uint8_t *scratch = nullptr;
        if (cudaMallocAsync(&scratch, stride * grid, s) != cudaSuccess) { g_detail = "cudaMallocAsync exact scratch"; return OTFLM_ERR_NOMEM; }
        CK(cudaFuncSetAttribute(k_advance_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_advance_exact<<<grid, sd::NT, smem, s>>>(m, n_cap, rs, in_row, words, h_base, out_base, scratch, stride,
                                                   (int)stages, nullptr);
        CKL();
        CK(cudaFreeAsync(scratch, s));
        return OTFLM_OK;
    }
    if (prec == OTFLM_PREC_FP64 || prec == OTFLM_PREC_EXACT) {
        constexpr int QT = 16;
        const size_t smem = (size_t)QT * m.H * sizeof(float);
        if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k_advance_f64<QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid(cdiv(n_cap, QT), cdiv(m.H, 256));
        k_advance_f64<QT><<<grid, 256, smem, s>>>(m, n_cap, rs, in_row, words, h_base, out_base, row_limit);
        CKL();
        return OTFLM_OK;
    }
    int rc = tc_advance_launch(m, prec, n_cap, rs, in_row, words, h_base, out_base, row_limit, s);
    if (rc == OTFLM_OK) g_launches++;
    else g_detail = "tcgen05 advance launch failed";
    return rc;
}

extern "C" int otflm_advance_hidden_batch(const OtflmModel *m, int64_t n, const int32_t *ctx, const float *h_in,
                                          const int32_t *w, float *h_out, int32_t precision, void *stream) {
    if (n <= 0) return OTFLM_OK;
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    /* EXACT: k_advance_exact */
    if (!m->d.U || !m->d.W) { g_detail = "model has no recurrent weights"; return OTFLM_ERR_VALUE; }
    const RowSpec rs{nullptr, nullptr, nullptr, nullptr, nullptr, 0xFFFFFFFFu};
    return launch_advance(m->d, precision, (uint32_t)n, rs, ctx, w, h_in, h_out, 0xFFFFFFFFu, (cudaStream_t)stream);
}

extern "C" int otflm_advance_hidden_rows(const OtflmModel *m, int64_t n, const float *input_rows, const int32_t *ctx,
                                         const float *h_in, float *h_out, int32_t precision, void *stream) {
    if (n <= 0) return OTFLM_OK;
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    /* EXACT: k_advance_exact */
    if (!m->d.W) { g_detail = "model has no recurrent weights"; return OTFLM_ERR_VALUE; }
    DevModel dm = m->d;
    dm.U = input_rows;   // row i is the input row of query i
    const RowSpec rs{nullptr, nullptr, nullptr, nullptr, nullptr, 0xFFFFFFFFu};
    return launch_advance(dm, precision, (uint32_t)n, rs, ctx, nullptr, h_in, h_out, 0xFFFFFFFFu, (cudaStream_t)stream);
}

// all_word_logprobs: activations of every internal node, then path sums
template <int VEC, int CPL>
__global__ void k_all_acts(DevModel m, const float *h, const uint32_t *hist, int L, double *acts) {
    const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= m.V - 1) return;
    const int H = m.H;
    const int NCH = VEC == 4 ? H / 4 : H;
    double a = 0.0;
    const float *row = m.NV + (size_t)j * H;
    for (int k = lane; k < NCH; k += 32) {
        if (VEC == 4) {
            float4 t = reinterpret_cast<const float4 *>(row)[k];
            float4 hh = reinterpret_cast<const float4 *>(h)[k];
            a = fma((double)t.x, (double)hh.x, a); a = fma((double)t.y, (double)hh.y, a);
            a = fma((double)t.z, (double)hh.z, a); a = fma((double)t.w, (double)hh.w, a);
        } else {
            a = fma((double)row[k], (double)h[k], a);
        }
    }
    a = warp_sum_d(a);
    if (lane == 0) {
        const int kmax = m.order < L ? m.order : L;
        for (int k = 1; k <= kmax; k++) {
            uint64_t x = otf_mix(m.seed, (uint64_t)k);
            for (int i = L - k; i < L; i++) x = otf_mix(x, (uint64_t)hist[i]);
            x = otf_mix(x, (uint64_t)j);
            a += (double)m.ME[x & m.mask];
        }
        acts[j] = a;
    }
}

__global__ void k_all_paths(DevModel m, const double *acts, double *out) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= m.V) return;
    double lp = 0.0;
    for (uint32_t p = m.path_off[w]; p < m.path_off[w + 1]; p++) {
        uint32_t c = m.path_code[p];
        double a = acts[c & 0x7FFFFFFFu];
        lp += otf_log_sigmoid((c & 0x80000000u) ? -a : a);
    }
    out[w] = lp;
}

extern "C" int otflm_all_word_logprobs(const OtflmModel *m, const float *h, const int32_t *hist_host,
                                       int32_t hist_len, double *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (hist_len < 0 || hist_len > OTF_MAX_ORDER) return OTFLM_ERR_VALUE;
    double *acts; uint32_t *dh;
    CK(cudaMallocAsync(&acts, sizeof(double) * (size_t)(m->d.V - 1 + 1), s));
    CK(cudaMallocAsync(&dh, sizeof(uint32_t) * OTF_MAX_ORDER, s));
    uint32_t hh[OTF_MAX_ORDER] = {0};
    for (int i = 0; i < hist_len; i++) hh[i] = (uint32_t)hist_host[i];
    CK(cudaMemcpyAsync(dh, hh, sizeof(hh), cudaMemcpyHostToDevice, s));
    const unsigned blocks = cdiv((uint64_t)m->d.V - 1, 8);
#define CALL(VEC, CPL) k_all_acts<VEC, CPL><<<blocks, 256, 0, s>>>(m->d, h, dh, hist_len, acts)
    HS_DISPATCH(m->d.H, CALL);
#undef CALL
    CKL();
    k_all_paths<<<cdiv(m->d.V, 256), 256, 0, s>>>(m->d, acts, out);
    CKL();
    CK(cudaFreeAsync(acts, s));
    CK(cudaFreeAsync(dh, s));
    CK(cudaStreamSynchronize(s));
    return OTFLM_OK;
}

// ---- batched all_word_logprobs: every word's log-prob for n contexts ----
// node activations a[q, j] = v_j . h_q (tcgen05 GEMM, or float64 CUDA cores in
// exact mode), + MaxEnt terms in the reference's order (_kernels_nb.py:63-75),
// then per node both log-sigmoids once, then per word the path-order sum
// (_kernels_nb.py:89-104).
__global__ void k_split_nv(DevModel m, float *hi, float *lo, __nv_bfloat16 *bf) {
    const int64_t n = (int64_t)(m.V - 1) * m.H;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = m.NV[i];
        const float h = tc::tf32_rn(x);
        hi[i] = h; lo[i] = tc::tf32_rn(x - h); bf[i] = __float2bfloat16(x);
    }
}

// exact mode: warp per node, AW_QT contexts per block (their rows staged in
// shared memory), the node row read once per block into registers; float64
// FMA over H, lane-strided, then a warp reduction per context
constexpr int AW_QT = 8;
template <int VEC>
__global__ void __launch_bounds__(256) k_all_acts_f64(DevModel m, int64_t n, const int32_t *ctx, const float *h,
                                                      double *act, int64_t ld) {
    extern __shared__ float4 aw_h4[];
    float *hs = reinterpret_cast<float *>(aw_h4);
    const int H = m.H;
    const int64_t q0 = (int64_t)blockIdx.y * AW_QT;
    const int nq = (int)min((int64_t)AW_QT, n - q0);
    for (int t = threadIdx.x; t < AW_QT * H; t += blockDim.x) {
        const int q = t / H, k = t - q * H;
        hs[t] = q < nq ? h[(size_t)ctx[q0 + q] * H + k] : 0.f;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < m.V - 1; j += nw) {
        const float *row = m.NV + (size_t)j * H;
        double a[AW_QT];
#pragma unroll
        for (int q = 0; q < AW_QT; q++) a[q] = 0.0;
        if (VEC == 4) {
            for (int k = lane; k < H / 4; k += 32) {
                const float4 t = __ldg(reinterpret_cast<const float4 *>(row) + k);
#pragma unroll
                for (int q = 0; q < AW_QT; q++) {
                    const float4 hh = reinterpret_cast<const float4 *>(hs + q * H)[k];
                    a[q] = fma((double)t.x, (double)hh.x, a[q]); a[q] = fma((double)t.y, (double)hh.y, a[q]);
                    a[q] = fma((double)t.z, (double)hh.z, a[q]); a[q] = fma((double)t.w, (double)hh.w, a[q]);
                }
            }
        } else {
            for (int k = lane; k < H; k += 32) {
                const double t = (double)__ldg(row + k);
#pragma unroll
                for (int q = 0; q < AW_QT; q++) a[q] = fma(t, (double)hs[q * H + k], a[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < AW_QT; q++) {
            const double v = warp_sum_d(a[q]);
            if (lane == q && q < nq) act[(q0 + q) * ld + j] = v;
        }
    }
}

// per (context, node): + MaxEnt, then log-sigmoid of +a and -a
template <typename T>
__global__ void k_all_node_lsig(DevModel m, int64_t n, const int32_t *ctx, const int32_t *hist,
                                const int32_t *hist_len, const T *act, int64_t ld, double2 *ls) {
    const int64_t q = blockIdx.y;
    if (q >= n) return;
    const int c = ctx[q];
    const int L = hist_len[c];
    const int kmax = m.order < L ? m.order : L;
    uint64_t pre[OTF_MAX_ORDER];
    for (int k = 0; k < kmax; k++) {
        uint64_t x = otf_mix(m.seed, (uint64_t)(k + 1));
        for (int i = L - (k + 1); i < L; i++) x = otf_mix(x, (uint64_t)hist[(size_t)c * m.order + i]);
        pre[k] = x;
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m.V - 1; j += (int64_t)gridDim.x * blockDim.x) {
        double a = (double)act[q * ld + j];
        for (int k = 0; k < kmax; k++) a += (double)__ldg(m.ME + (otf_mix(pre[k], (uint64_t)j) & m.mask));
        ls[q * (int64_t)(m.V - 1) + j] = make_double2(otf_log_sigmoid(a), otf_log_sigmoid(-a));
    }
}

__global__ void k_all_word_paths(DevModel m, int64_t n, const double2 *ls, double *out) {
    const int64_t q = blockIdx.y;
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n || w >= m.V) return;
    const double2 *l = ls + q * (int64_t)(m.V - 1);
    double lp = 0.0;
    for (uint32_t p = m.path_off[w]; p < m.path_off[w + 1]; p++) {
        const uint32_t c = m.path_code[p];
        const double2 v = l[c & 0x7FFFFFFFu];
        lp += (c & 0x80000000u) ? v.y : v.x;
    }
    out[q * (int64_t)m.V + w] = lp;
}

extern "C" int otflm_all_word_logprobs_batch(const OtflmModel *m, int64_t n, const int32_t *ctx,
                                             const float *h, const int32_t *hist, const int32_t *hist_len,
                                             double *out, int32_t precision, void *stream) {
    if (n <= 0) return OTFLM_OK;
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    precision = level_prec(precision);
    if (!m->d.NV || !m->d.ME || !m->d.path_off) { g_detail = "model has no output layer"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    const DevModel &d = m->d;
    const int64_t NV = d.V - 1;
    const bool tcm = precision != OTFLM_PREC_FP64;
    if (tcm && (d.H % 4 != 0)) { g_detail = "tensor-core all_word_logprobs needs H % 4 == 0"; return OTFLM_ERR_VALUE; }
    if (tcm) {
        std::lock_guard<std::mutex> lk(m->nv_mu);
        if (!m->NV_hi) {
            OtflmModel *mm = const_cast<OtflmModel *>(m);
            if (mm->mem.alloc(&mm->NV_hi, (size_t)NV * d.H) || mm->mem.alloc(&mm->NV_lo, (size_t)NV * d.H) ||
                mm->mem.alloc(&mm->NV_bf, (size_t)NV * d.H)) { g_detail = "cudaMalloc NV split"; return OTFLM_ERR_NOMEM; }
            k_split_nv<<<1184, 256, 0, s>>>(d, mm->NV_hi, mm->NV_lo, mm->NV_bf);
            CKL();
        }
    }
    // contexts in chunks: activations + node log-sigmoids are [chunk, V-1]
    const int64_t ld = (NV + 3) / 4 * 4;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)(512ll << 20) / (ld * 20)));
    void *act = nullptr; double2 *ls = nullptr;
    CK(cudaMallocAsync(&act, (size_t)chunk * ld * (tcm ? 4 : 8), s));
    CK(cudaMallocAsync(&ls, (size_t)chunk * NV * sizeof(double2), s));
    int rc = OTFLM_OK;
    for (int64_t q0 = 0; q0 < n && rc == OTFLM_OK; q0 += chunk) {
        const int64_t nq = std::min(chunk, n - q0);
        if (tcm) {
            tc::TcB B{};
            B.hi = m->NV_hi; B.lo = m->NV_lo; B.bf = m->NV_bf;
            B.n_rows = (int)NV; B.n_pad = (int)((NV + 31) / 32 * 32);
            B.out = (float *)act; B.ld = ld;
            const RowSpec rs{nullptr, nullptr, nullptr, nullptr, nullptr, 0xFFFFFFFFu};
            if (tc_gemm_launch(d, precision, (uint32_t)nq, rs, ctx + q0, nullptr, h, nullptr, &B, s)) {
                g_detail = "tcgen05 all_word GEMM launch failed"; rc = OTFLM_ERR_CUDA; break;
            }
            g_launches++;
            k_all_node_lsig<float><<<dim3(cdiv(NV, 256 * 4), (unsigned)nq), 256, 0, s>>>(
                d, nq, ctx + q0, hist, hist_len, (const float *)act, ld, ls);
        } else {
            const size_t sm = (size_t)AW_QT * d.H * sizeof(float);
            const dim3 grid((unsigned)std::min<int64_t>(cdiv(NV, 8), 1184), cdiv(nq, AW_QT));
            if (d.H % 4 == 0) {
                CK(cudaFuncSetAttribute(k_all_acts_f64<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                k_all_acts_f64<4><<<grid, 256, sm, s>>>(d, nq, ctx + q0, h, (double *)act, ld);
            } else {
                CK(cudaFuncSetAttribute(k_all_acts_f64<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                k_all_acts_f64<1><<<grid, 256, sm, s>>>(d, nq, ctx + q0, h, (double *)act, ld);
            }
            g_launches++;
            k_all_node_lsig<double><<<dim3(cdiv(NV, 256 * 4), (unsigned)nq), 256, 0, s>>>(
                d, nq, ctx + q0, hist, hist_len, (const double *)act, ld, ls);
        }
        g_launches++;
        k_all_word_paths<<<dim3(cdiv(d.V, 256), (unsigned)nq), 256, 0, s>>>(d, nq, ls, out + q0 * d.V);
        CKL();
    }
    CK(cudaFreeAsync(act, s));
    CK(cudaFreeAsync(ls, s));
    return rc;
}

// ==========================================================================
// streams
// ==========================================================================
struct LfuHost;
struct OtflmStreams {
    const OtflmModel *m;
    DevStreams d;
    Allocs mem;
    OtflmPlan *scratch = nullptr;   // workspace for rnnlm_prob_batch
    LfuHost *lfu = nullptr;         // capacity-bounded cache policy (lfu.cuh)
    int64_t capacity_bytes = 0;
    uint64_t version = 0;           // bumped when DevStreams changes (captured graphs re-capture)
    uint32_t dig_epoch = 0;         // EXACT stream launches so far (arena_dep tags)
};
#include "lfu.cuh"

__global__ void k_streams_reset(DevStreams S, int retain) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < (uint64_t)S.S) {
        unsigned long long *st = S.stats + t * 8;
        st[3] += st[0]; st[4] += st[1]; st[5] += st[2];
        st[0] = st[1] = st[2] = 0;
        if (!retain) { st[6] = 0; S.table_len[t] = 0; S.novel_cnt[t] = 0; S.ctx_row[t * (S.max_ctx + 1)] = 0; }
    }
    if (t == 0 && !retain) {
        *S.arena_used = 1;
        for (int i = 0; i < OTF_META; i++) S.arena_meta[i] = 0;
    }
    if (!retain && t < (uint64_t)S.H) S.arena_h[t] = 0.f;   // row 0 = zero context
}

static int streams_clear(OtflmStreams *s, int retain, cudaStream_t st) {
    DevStreams &d = s->d;
    if (!retain) {
        const size_t nct = (size_t)d.S * d.ct_cap, nkc = (size_t)d.S * d.kc_cap;
        CK(cudaMemsetAsync(d.ct_key, 0, nct * 8, st));
        CK(cudaMemsetAsync(d.ct_idx, 0xFF, nct * 4, st));
        CK(cudaMemsetAsync(d.kc_key, 0, nkc * 8, st));
        CK(cudaMemsetAsync(d.kc_claim, 0xFF, nkc * 4, st));
        CK(cudaMemsetAsync(d.kc_cnext, 0xFF, nkc * 4, st));
    }
    uint64_t n = std::max<uint64_t>((uint64_t)d.S, (uint64_t)d.H);
    k_streams_reset<<<cdiv(n, 256), 256, 0, st>>>(d, retain);
    CKL();
    if (s->lfu) {
        if (!retain) CK(cudaMemsetAsync(s->lfu->d.kc_lfu, 0xFF, (size_t)d.S * d.kc_cap * 4, st));
        k_lfu_reset<<<cdiv(d.S, 128), 128, 0, st>>>(s->lfu->d, retain);
        CKL();
        CK(cudaMemsetAsync(d.lfu_logn, 0, (size_t)d.S * 4, st));
    }
    return OTFLM_OK;
}

extern "C" int otflm_streams_create(const OtflmModel *m, const OtflmStreamConfig *cfg, OtflmStreams **out) {
    if (!m || !cfg || !out || cfg->n_streams < 1 || cfg->max_contexts < 1 || cfg->arena_rows < 2)
        return OTFLM_ERR_VALUE;
    if (!m->d.U || !m->d.W || !m->d.NV || !m->d.ME || !m->d.path_off) {
        g_detail = "decoding streams need a complete model";
        return OTFLM_ERR_VALUE;
    }
    if (cfg->max_contexts >= 0xFFFFFFF0ll || cfg->arena_rows >= 0xFFFFFFF0ll) return OTFLM_ERR_VALUE;
    OtflmStreams *s = new OtflmStreams();
    s->m = m;
    DevStreams &d = s->d;
    d.S = cfg->n_streams; d.enabled = cfg->cache_enabled ? 1 : 0;
    d.H = m->d.H; d.order = m->d.order;
    d.max_ctx = (uint32_t)cfg->max_contexts;
    d.arena_rows = (uint32_t)cfg->arena_rows;
    d.lfu_cap = 0; d.lfu_logcap = 0; d.lfu_log = nullptr; d.lfu_logn = nullptr;
    d.arena_dig = nullptr; d.arena_deh = nullptr; d.arena_dep = nullptr;
    d.ct_first = nullptr;
    d.ct_cap = pow2_at_least((uint64_t)cfg->max_contexts * 2 + 2);
    d.kc_cap = pow2_at_least((uint64_t)std::max<int64_t>(cfg->cache_slots, 16));
    const size_t S = d.S;
    bool bad = false;
    bad |= s->mem.alloc(&d.ctx_row, S * (d.max_ctx + 1)) != cudaSuccess;
    bad |= s->mem.alloc(&d.arena_h, (size_t)d.arena_rows * d.H) != cudaSuccess;
    bad |= s->mem.alloc(&d.arena_meta, (size_t)d.arena_rows * OTF_META) != cudaSuccess;
    bad |= s->mem.alloc(&d.arena_used, 1) != cudaSuccess;
    bad |= s->mem.alloc(&d.ct_key, S * d.ct_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.ct_idx, S * d.ct_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.ct_row, S * d.ct_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.kc_key, S * d.kc_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.kc_claim, S * d.kc_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.kc_cnext, S * d.kc_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.kc_p, S * d.kc_cap) != cudaSuccess;
    bad |= s->mem.alloc(&d.table_len, S) != cudaSuccess;
    bad |= s->mem.alloc(&d.novel_cnt, S) != cudaSuccess;
    bad |= s->mem.alloc(&d.stats, S * 8) != cudaSuccess;
    bad |= s->mem.alloc(&d.err, 1) != cudaSuccess;
    if (bad) { s->mem.free_all(); delete s; g_detail = "cudaMalloc streams"; return OTFLM_ERR_NOMEM; }
    CK(cudaMemset(d.stats, 0, S * 8 * 8));
    CK(cudaMemset(d.err, 0, 4));
    CK(cudaMemset(d.arena_meta, 0, (size_t)OTF_META * 4));
    int rc = streams_clear(s, 0, 0);
    if (rc) return rc;
    CK(cudaDeviceSynchronize());
    *out = s;
    return OTFLM_OK;
}

extern "C" int otflm_plan_destroy(OtflmPlan *p);

extern "C" int otflm_streams_destroy(OtflmStreams *s) {
    if (!s) return OTFLM_OK;
    if (s->scratch) otflm_plan_destroy(s->scratch);
    if (s->lfu) { s->lfu->mem.free_all(); delete s->lfu; }
    s->mem.free_all();
    delete s;
    return OTFLM_OK;
}

extern "C" int otflm_streams_reset(OtflmStreams *s, int32_t retain, void *stream) {
    if (!s) return OTFLM_ERR_VALUE;
    return streams_clear(s, retain, (cudaStream_t)stream);
}

static int check_err(OtflmStreams *s, cudaStream_t st) {
    unsigned int he = 0;
    CK(cudaMemcpyAsync(&he, s->d.err, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (he) {
        CK(cudaMemsetAsync(s->d.err, 0, 4, st));
        CK(cudaStreamSynchronize(st));
        // a new context left without an index-table slot by an in-chunk
        // digest mismatch (HASH | NOSLOT) is a digest error, not a full table
        if ((he & OTF_E_HASH) && (he & OTF_E_NOSLOT) && !(he & (OTF_E_ARENA_FULL | OTF_E_CACHE_FULL))) {
            g_detail = "content digest collision [device flags " + std::to_string(he) + "]";
            return OTFLM_ERR_HASH;
        }
        // a capacity overflow first: the stages after it read rows that were
        // never written, which can also raise a spurious digest mismatch
        if (he & (OTF_E_TABLE_FULL | OTF_E_ARENA_FULL | OTF_E_CACHE_FULL)) {
            g_detail = (he & OTF_E_ARENA_FULL) ? "hidden-state arena full"
                     : (he & OTF_E_CACHE_FULL) ? "cache table full" : "index table full";
            g_detail += " [device flags " + std::to_string(he) + "]";
            return OTFLM_ERR_TABLE_FULL;
        }
        if (he & OTF_E_HASH) { g_detail = "content digest collision"; return OTFLM_ERR_HASH; }
        if (he & OTF_E_KEY) { g_detail = "word missing from unigram table"; return OTFLM_ERR_KEY; }
        if (he & OTF_E_VALUE) return OTFLM_ERR_VALUE;
        return OTFLM_ERR_CUDA;
    }
    return OTFLM_OK;
}

extern "C" int otflm_streams_stats(OtflmStreams *s, int64_t *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t S = s->d.S;
    std::vector<unsigned long long> raw(S * 8);
    std::vector<uint32_t> tl(S);
    CK(cudaMemcpyAsync(raw.data(), s->d.stats, S * 64, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tl.data(), s->d.table_len, S * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (size_t i = 0; i < S; i++) {
        const unsigned long long *r = &raw[i * 8];
        int64_t *o = out + i * 8;
        o[0] = r[0]; o[1] = r[1]; o[2] = r[2]; o[3] = tl[i];
        o[4] = r[3] + r[0]; o[5] = r[4] + r[1]; o[6] = r[5] + r[2]; o[7] = r[6];
    }
    return OTFLM_OK;
}

static int lfu_enqueue(const OtflmStreams *s, cudaStream_t st) {
    if (!s->lfu || !s->d.lfu_log) return OTFLM_OK;
    k_lfu_replay<<<cdiv(s->d.S, 64), 64, 0, st>>>(s->d, s->lfu->d, nullptr, nullptr);
    CKL();
    return OTFLM_OK;
}

extern "C" int otflm_streams_set_capacity(OtflmStreams *s, int64_t capacity_bytes, void *stream) {
    if (!s || capacity_bytes < 0) return OTFLM_ERR_VALUE;
    cudaStream_t st = (cudaStream_t)stream;
    DevStreams &d = s->d;
    s->capacity_bytes = capacity_bytes;
    if (capacity_bytes == 0) {                 // unbounded: stop logging (the policy state is dropped)
        d.lfu_log = nullptr; d.lfu_cap = 0;
        s->version++;
        return OTFLM_OK;
    }
    const uint64_t want = (uint64_t)(capacity_bytes / 32);
    if (want >= 0x7FFFFFF0ull) return OTFLM_ERR_VALUE;
    const uint32_t cap = (uint32_t)want;
    const size_t S = d.S;
    if (!s->lfu || s->lfu->d.E < std::max<uint32_t>(cap, 1)) {
        // (re)allocate the pools at the new size; a resident set carried over is copied row by row
        LfuHost *n = new LfuHost();
        DevLfu &L = n->d;
        L.S = d.S; L.E = std::max<uint32_t>(cap, 1); L.kc_cap = d.kc_cap;
        const size_t E = L.E, F = L.E + 1;
        bool bad = n->mem.alloc(&L.kc_lfu, S * d.kc_cap) || n->mem.alloc(&L.en_slot, S * E) ||
                   n->mem.alloc(&L.en_prev, S * E) || n->mem.alloc(&L.en_next, S * E) ||
                   n->mem.alloc(&L.en_f, S * E) || n->mem.alloc(&L.fn_freq, S * F) ||
                   n->mem.alloc(&L.fn_prev, S * F) || n->mem.alloc(&L.fn_next, S * F) ||
                   n->mem.alloc(&L.fn_head, S * F) || n->mem.alloc(&L.fn_tail, S * F) ||
                   n->mem.alloc(&L.sc, S * 8) || n->mem.alloc(&L.ev, S * 2);
        if (!d.lfu_log)
            bad = bad || s->mem.alloc(&d.lfu_log, S * std::max<uint32_t>(d.kc_cap, 4096)) ||
                  s->mem.alloc(&d.lfu_logn, S);
        if (bad) { n->mem.free_all(); delete n; g_detail = "cudaMalloc cache policy"; return OTFLM_ERR_NOMEM; }
        d.lfu_logcap = std::max<uint32_t>(d.kc_cap, 4096);
        if (s->lfu) {
            const DevLfu &O = s->lfu->d;
            const size_t oE = O.E, oF = O.E + 1;
            auto cp2 = [&](uint32_t *dst, const uint32_t *src, size_t dw, size_t sw) {
                return cudaMemcpy2DAsync(dst, dw * 4, src, sw * 4, sw * 4, S, cudaMemcpyDeviceToDevice, st);
            };
            CK(cudaMemcpyAsync(L.kc_lfu, O.kc_lfu, S * d.kc_cap * 4, cudaMemcpyDeviceToDevice, st));
            CK(cp2(L.en_slot, O.en_slot, E, oE)); CK(cp2(L.en_prev, O.en_prev, E, oE));
            CK(cp2(L.en_next, O.en_next, E, oE)); CK(cp2(L.en_f, O.en_f, E, oE));
            CK(cp2(L.fn_freq, O.fn_freq, F, oF)); CK(cp2(L.fn_prev, O.fn_prev, F, oF));
            CK(cp2(L.fn_next, O.fn_next, F, oF)); CK(cp2(L.fn_head, O.fn_head, F, oF));
            CK(cp2(L.fn_tail, O.fn_tail, F, oF));
            CK(cudaMemcpyAsync(L.sc, O.sc, S * 8 * 4, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(L.ev, O.ev, S * 2 * 8, cudaMemcpyDeviceToDevice, st));
            CK(cudaStreamSynchronize(st));
            s->lfu->mem.free_all();
            delete s->lfu;
        } else {
            CK(cudaMemsetAsync(L.kc_lfu, 0xFF, S * d.kc_cap * 4, st));
            CK(cudaMemsetAsync(L.ev, 0, S * 2 * 8, st));
            CK(cudaMemsetAsync(d.lfu_logn, 0, S * 4, st));
            k_lfu_reset<<<cdiv(d.S, 128), 128, 0, st>>>(L, 0);
            CKL();
            // keys already cached (unbounded so far) are not resident under the policy:
            // the reference's set_capacity keeps them; start the policy from the
            // current resident count only when the cache is empty
        }
        s->lfu = n;
    }
    s->lfu->d.cap = cap;
    d.lfu_cap = cap;
    s->version++;
    k_lfu_shrink<<<cdiv(d.S, 64), 64, 0, st>>>(d, s->lfu->d);
    CKL();
    return OTFLM_OK;
}

/* per stream: evictions in the current window, cumulative evictions, resident entries */
extern "C" int otflm_streams_cache_stats(OtflmStreams *s, int64_t *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t S = s->d.S;
    std::vector<unsigned long long> ev(S * 2, 0), raw(S * 8);
    if (s->lfu) CK(cudaMemcpyAsync(ev.data(), s->lfu->d.ev, S * 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(raw.data(), s->d.stats, S * 64, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (size_t i = 0; i < S; i++) {
        out[i * 3] = (int64_t)ev[i * 2];
        out[i * 3 + 1] = (int64_t)(ev[i * 2] + ev[i * 2 + 1]);
        out[i * 3 + 2] = (int64_t)raw[i * 8 + 6];
    }
    return OTFLM_OK;
}

extern "C" int otflm_streams_context(OtflmStreams *s, int32_t sid, uint32_t idx, float *hidden, int32_t *hist,
                                     int32_t *len, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (sid < 0 || sid >= s->d.S) return OTFLM_ERR_VALUE;
    uint32_t tl = 0;
    CK(cudaMemcpyAsync(&tl, s->d.table_len + sid, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (idx > tl) { g_detail = "index not in table"; return OTFLM_ERR_UNKNOWN_INDEX; }
    uint32_t row = 0;
    CK(cudaMemcpyAsync(&row, s->d.ctx_row + (size_t)sid * (s->d.max_ctx + 1) + idx, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint32_t meta[OTF_META];
    CK(cudaMemcpyAsync(hidden, s->d.arena_h + (size_t)row * s->d.H, (size_t)s->d.H * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(meta, s->d.arena_meta + (size_t)row * OTF_META, sizeof(meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *len = (int32_t)meta[0];
    for (uint32_t i = 0; i < meta[0] && i < OTF_MAX_ORDER; i++) hist[i] = (int32_t)meta[1 + i];
    return OTFLM_OK;
}

// ==========================================================================
// plan: compiled lattice batch + level loop
// ==========================================================================
struct OtflmPlan {
    OtflmStreams *st = nullptr;
    int64_t beam = 0;
    uint32_t n_utt = 0, n_levels = 0, n_nodes = 0, n_arcs = 0, n_slots = 0, R_max = 0;
    bool has_big = false;              // nodes for k_expand_big (expb_min < cap <= EXPB_MAX)
    uint32_t expb_min = EXPB_MIN;      // (OTFLM_EXPAND_BIG_MIN / OTFLM_ASSIGN_BIG: test overrides of the thresholds)
    uint32_t asg_big = ASSIGN_BIG;
    bool hs_tc = true;                 // EXACT level schedule: digit-plane HS (OTFLM_HS_TC=0: float64 CUDA cores)
    bool lvl_fused = true;             // ... fused with the update in one kernel (OTFLM_LEVEL_FUSED=0: two kernels)
    bool big_asg = false;              // a (level, stream) range above ASSIGN_BIG requests: k_asg_* assign
    uint32_t ch_cap = 0;               // chunk entries of the multi-CTA assign (max over levels)
    uint64_t total_req = 0;
    std::vector<uint32_t> lvl_node_off, lvl_req, lvl_range_off;   // host copies
    DevPlan d{};
    Allocs mem;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    double g_lm = 0; int g_prec = -1; const OtflmNgram *g_ng = nullptr; int64_t g_nodes = 0;
    uint64_t h2d_bytes = 0;
    unsigned long long *alg_buf = nullptr;
    uint8_t *xs = nullptr;             // exact stream mode: per-stream digit scratch (Allocs-owned)
    uint32_t *work = nullptr;          // stream queue counter of the persistent one-CTA schedule
    size_t xs_bytes = 0;
    cudaStream_t side = nullptr;               // second branch of each level (HS)
    cudaStream_t chain = nullptr;              // this plan's chain inside a group graph
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_done = nullptr;
    std::vector<uint32_t> utt_stream_host;
    int32_t schedule = OTFLM_SCHED_LEVEL;      // level-synchronous or persistent per-stream
    uint32_t ws_cap = 0;                       // request / primary workspace entries
    uint32_t ul_cap = 0;                       // UttLevel entries
    // pinned staging for otflm_plan_refresh: the uploads are truly
    // asynchronous, so compiling the next batch on the host overlaps the
    // decode of the current one; ev_staged guards reuse of the buffer
    uint8_t *staging = nullptr;
    size_t staging_cap = 0;
    cudaEvent_t ev_staged = nullptr;
    bool grouped = false;           // part of an OtflmGroup (the group runs the cache policy)
    // lattice-out (otflm_plan_set_lattice_out): per-utterance slot ranges and buffers
    std::vector<uint32_t> utt_slot_off;
    uint32_t *utt_slot_off_dev = nullptr;
    LatRecord *lat_rec = nullptr;
    long long *lat_cnt = nullptr;
    uint8_t *kept_buf = nullptr;
    // refresh uploads run on their own stream, after this plan's previous run
    // (ev_lastrun) and before its next one (ev_up), so the H2D of batch i+1
    // overlaps the decode of batch i on the compute stream
    cudaStream_t up = nullptr;
    cudaEvent_t ev_up = nullptr, ev_lastrun = nullptr;
    uint64_t g_ver = 0;             // OtflmStreams::version of the captured graph
    ~OtflmPlan() {
        if (up) cudaStreamDestroy(up);
        if (ev_up) cudaEventDestroy(ev_up);
        if (ev_lastrun) cudaEventDestroy(ev_lastrun);
        if (staging) cudaFreeHost(staging);
        if (ev_staged) cudaEventDestroy(ev_staged);
        if (side) cudaStreamDestroy(side);
        if (chain) cudaStreamDestroy(chain);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_done) cudaEventDestroy(ev_done);
    }
};

static int compile_batch(OtflmPlan *p, const OtflmLatticeBatch *L, int64_t beam, int V,
                         std::vector<NodeInfo> &nodes, std::vector<uint32_t> &level_nodes,
                         std::vector<uint32_t> &out_list, std::vector<uint32_t> &arc_slot,
                         std::vector<int32_t> &arc_word, std::vector<double> &arc_ac,
                         std::vector<double> &arc_slm, std::vector<uint32_t> &start_slot,
                         std::vector<uint32_t> &final_off, std::vector<uint32_t> &finals,
                         std::vector<uint32_t> &utt_stream, std::vector<StreamRange> &ranges,
                         std::vector<UttLevel> &ul, std::vector<uint32_t> &ul_off, std::vector<uint32_t> &rq_off) {
    const int U = L->n_utt;
    std::vector<std::vector<std::vector<uint32_t>>> lv(U);   // per utt: levels -> global nodes
    uint64_t node_base = 0, slot_base = 0;
    final_off.assign(1, 0);
    const uint64_t n_arcs_total = (uint64_t)L->arc_off[U];
    arc_slot.assign(n_arcs_total, 0);
    arc_word.assign(L->arc_word, L->arc_word + n_arcs_total);
    arc_ac.assign(L->arc_ac, L->arc_ac + n_arcs_total);
    arc_slm.assign(L->arc_slm, L->arc_slm + n_arcs_total);
    out_list.assign(n_arcs_total, 0);
    for (int u = 0; u < U; u++) {
        const int N = L->n_nodes[u];
        const int64_t a0 = L->arc_off[u], a1 = L->arc_off[u + 1];
        const int start = L->start[u];
        if (N < 1 || start < 0 || start >= N) { g_detail = "bad start node"; return OTFLM_ERR_VALUE; }
        std::vector<uint32_t> out_cnt(N + 1, 0), indeg(N, 0);
        for (int64_t a = a0; a < a1; a++) {
            int s = L->arc_src[a], d = L->arc_dst[a], w = L->arc_word[a];
            if (s < 0 || s >= N || d < 0 || d >= N) { g_detail = "arc node out of range"; return OTFLM_ERR_VALUE; }
            if (w < 0 || w >= V) { g_detail = "word id out of range"; return OTFLM_ERR_VALUE; }
            out_cnt[s + 1]++;
            indeg[d]++;
        }
        for (int n = 0; n < N; n++) out_cnt[n + 1] += out_cnt[n];
        std::vector<uint32_t> fill(out_cnt.begin(), out_cnt.end() - 1);
        std::vector<uint32_t> out_loc(std::max<int64_t>(a1 - a0, 1));
        for (int64_t a = a0; a < a1; a++) out_loc[fill[L->arc_src[a]]++] = (uint32_t)a;
        for (int64_t k = 0; k < a1 - a0; k++) out_list[a0 + k] = out_loc[k];
        // Kahn, smallest id first (lattice.py:68-82)
        std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
        for (int n = 0; n < N; n++) if (indeg[n] == 0) ready.push(n);
        std::vector<int> topo;
        topo.reserve(N);
        while (!ready.empty()) {
            int n = ready.top(); ready.pop();
            topo.push_back(n);
            for (uint32_t k = out_cnt[n]; k < out_cnt[n + 1]; k++) {
                int d = L->arc_dst[out_loc[k]];
                if (--indeg[d] == 0) ready.push(d);
            }
        }
        if ((int)topo.size() != N) { g_detail = "lattice contains a cycle"; return OTFLM_ERR_CYCLE; }
        // greedy levels: maximal runs of the topological order with no internal arc
        std::vector<int> lvl(N, -1), predmax(N, -1);
        int cur = 0;
        for (int n : topo) {
            if (predmax[n] >= cur) cur++;
            lvl[n] = cur;
            for (uint32_t k = out_cnt[n]; k < out_cnt[n + 1]; k++) {
                int d = L->arc_dst[out_loc[k]];
                predmax[d] = std::max(predmax[d], cur);
            }
        }
        // capacities: distinct tokens at a node <= arrivals <= sum of the
        // sources' kept tokens; the start token occupies slot 0 of start.
        std::vector<uint64_t> cap(N, 0), keep(N, 0);
        std::vector<uint32_t> arc_off_in(a1 - a0 + 1, 0);
        cap[start] = 1;
        for (int n : topo) {
            keep[n] = std::min<uint64_t>((uint64_t)beam, cap[n]);
            for (uint32_t k = out_cnt[n]; k < out_cnt[n + 1]; k++) {
                uint32_t a = out_loc[k];
                int d = L->arc_dst[a];
                arc_off_in[a - a0] = (uint32_t)cap[d];
                cap[d] += keep[n];
                if (cap[d] > (1ull << 30)) { g_detail = "token capacity explodes (beam too wide for this lattice)"; return OTFLM_ERR_NOMEM; }
            }
        }
        std::vector<uint64_t> sbase(N);
        for (int n = 0; n < N; n++) { sbase[n] = slot_base; slot_base += cap[n]; }
        if (slot_base > 0xF0000000ull) { g_detail = "too many arrival slots"; return OTFLM_ERR_NOMEM; }
        for (int64_t a = a0; a < a1; a++) arc_slot[a] = (uint32_t)(sbase[L->arc_dst[a]] + arc_off_in[a - a0]);
        start_slot.push_back((uint32_t)sbase[start]);
        const uint32_t sid = L->stream_ids ? (uint32_t)L->stream_ids[u] : (uint32_t)u;
        utt_stream.push_back(sid);
        const uint32_t nb = (uint32_t)node_base;
        for (int n = 0; n < N; n++) {
            NodeInfo ni;
            ni.slot_base = (uint32_t)sbase[n];
            ni.cap = (uint32_t)cap[n];
            ni.keep = (uint32_t)keep[n];
            ni.out_b = (uint32_t)(a0 + out_cnt[n]);
            ni.out_e = (uint32_t)(a0 + out_cnt[n + 1]);
            ni.req_base = 0;
            ni.stream = sid;
            ni.pad = 0;
            if (ni.cap > p->expb_min && ni.cap <= EXPB_MAX && ni.out_e > ni.out_b) p->has_big = true;
            nodes.push_back(ni);
        }
        lv[u].assign(cur + 1, {});
        for (int n : topo) lv[u][lvl[n]].push_back(nb + n);
        for (int64_t f = L->final_off[u]; f < L->final_off[u + 1]; f++) {
            int fn = L->finals[f];
            if (fn < 0 || fn >= N) { g_detail = "final node out of range"; return OTFLM_ERR_VALUE; }
            finals.push_back(nb + fn);
        }
        final_off.push_back((uint32_t)finals.size());
        node_base += N;
    }
    // merge levels across utterances (utterance-major inside a level); static
    // request slots per node; one request range per (level, stream)
    size_t nlev = 0;
    for (int u = 0; u < U; u++) nlev = std::max(nlev, lv[u].size());
    std::vector<std::vector<UttLevel>> ulv(U);
    p->lvl_node_off.assign(1, 0);
    p->lvl_range_off.assign(1, 0);
    p->lvl_req.clear();
    uint64_t rmax = 0, total = 0;
    for (size_t t = 0; t < nlev; t++) {
        uint64_t run = 0;
        for (int u = 0; u < U; u++) {
            if (t >= lv[u].size() || lv[u][t].empty()) continue;
            const uint64_t rb = run;
            const uint32_t nb = (uint32_t)level_nodes.size();
            for (uint32_t g : lv[u][t]) {
                NodeInfo &ni = nodes[g];
                ni.req_base = (uint32_t)run;
                run += (uint64_t)ni.keep * (ni.out_e - ni.out_b);
                level_nodes.push_back(g);
            }
            if (run > rb) {
                if (run - rb > p->asg_big) p->big_asg = true;
                ranges.push_back(StreamRange{utt_stream[u], (uint32_t)rb, (uint32_t)run, 0});
                ulv[u].push_back(UttLevel{(uint32_t)t, nb, (uint32_t)level_nodes.size(), (uint32_t)rb, (uint32_t)run, 0, 0, 0});
            }
        }
        if (run > 0xF0000000ull) { g_detail = "too many requests in one level"; return OTFLM_ERR_NOMEM; }
        p->lvl_node_off.push_back((uint32_t)level_nodes.size());
        p->lvl_range_off.push_back((uint32_t)ranges.size());
        p->lvl_req.push_back((uint32_t)run);
        {
            const uint64_t nr = p->lvl_range_off.back() - p->lvl_range_off[p->lvl_range_off.size() - 2];
            p->ch_cap = (uint32_t)std::max<uint64_t>(p->ch_cap, nr * ((run + ASG_CH - 1) / ASG_CH));
        }
        rmax = std::max(rmax, run);
        total += run;
    }
    // persistent schedule: levels per utterance, private workspace offsets
    ul.clear(); ul_off.assign(1, 0); rq_off.assign(1, 0);
    uint64_t ws = 0;
    for (int u = 0; u < U; u++) {
        uint32_t mx = 0;
        for (const UttLevel &e : ulv[u]) { ul.push_back(e); mx = std::max(mx, e.re - e.rb); }
        ul_off.push_back((uint32_t)ul.size());
        ws += mx;
        if (ws > 0xF0000000ull) { g_detail = "too many requests"; return OTFLM_ERR_NOMEM; }
        rq_off.push_back((uint32_t)ws);
    }
    p->n_levels = (uint32_t)nlev;
    p->n_nodes = (uint32_t)node_base;
    p->n_arcs = (uint32_t)n_arcs_total;
    p->n_slots = (uint32_t)slot_base;
    p->R_max = (uint32_t)std::max<uint64_t>(rmax, 1);
    p->total_req = total;
    return OTFLM_OK;
}

static uint64_t g_upload_bytes = 0;
template <class T>
static int upload(Allocs &mem, T **dst, const std::vector<T> &v, cudaStream_t s) {
    if (mem.alloc(dst, v.size()) != cudaSuccess) { g_detail = "cudaMalloc plan"; return OTFLM_ERR_NOMEM; }
    g_upload_bytes += v.size() * sizeof(T);
    if (!v.empty()) CK(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return OTFLM_OK;
}

static int plan_alloc_workspace(OtflmPlan *p, uint32_t R, uint32_t n_lvl_slots) {
    DevPlan &d = p->d;
    bool bad = false;
    bad |= p->mem.alloc(&d.rq_c, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_arc, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_parent, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_cslot, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_m, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_dslot, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_w, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_state, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_score, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_slm, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.rq_ps, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.pr_req, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.pr_inrow, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.pr_w, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.pr_p, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.pr_dig, R) != cudaSuccess;
    bad |= p->mem.alloc(&d.lvl, n_lvl_slots) != cudaSuccess;
    bad |= p->mem.alloc(&p->alg_buf, 40) != cudaSuccess;   // [0..3] work counters, [8..19] phase ns, [24..28] assign sections
    bad |= p->mem.alloc(&d.cursor, 1) != cudaSuccess;
    d.alg = nullptr;   // counters are only maintained in profiling runs
    d.phase_ns = nullptr;
    d.arena_start = OTF_UNSET;
    d.arena_end = 0;
    if (bad) { g_detail = "cudaMalloc workspace"; return OTFLM_ERR_NOMEM; }
    if (cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->chain, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming) != cudaSuccess) {
        g_detail = "stream/event creation";
        return OTFLM_ERR_CUDA;
    }
    return OTFLM_OK;
}

extern "C" int otflm_plan_create(OtflmStreams *st, const OtflmLatticeBatch *L, int64_t beam, OtflmPlan **out,
                                 void *stream) {
    if (!st || !L || !out) return OTFLM_ERR_VALUE;
    if (beam < 1) { g_detail = "beam must be >= 1"; return OTFLM_ERR_VALUE; }
    if (L->n_utt < 1) return OTFLM_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    OtflmPlan *p = new OtflmPlan();
    if (const char *e = getenv("OTFLM_EXPAND_BIG_MIN")) p->expb_min = (uint32_t)strtoul(e, nullptr, 10);
    if (const char *e = getenv("OTFLM_ASSIGN_BIG")) p->asg_big = (uint32_t)strtoul(e, nullptr, 10);
    if (const char *e = getenv("OTFLM_HS_TC")) p->hs_tc = atoi(e) != 0;
    if (const char *e = getenv("OTFLM_LEVEL_FUSED")) p->lvl_fused = atoi(e) != 0;
    p->st = st;
    p->beam = beam;
    p->n_utt = L->n_utt;
    std::vector<NodeInfo> nodes;
    std::vector<uint32_t> level_nodes, out_list, arc_slot, start_slot, final_off, finals, utt_stream;
    std::vector<int32_t> arc_word;
    std::vector<double> arc_ac, arc_slm;
    std::vector<StreamRange> ranges;
    std::vector<UttLevel> ul;
    std::vector<uint32_t> ul_off, rq_off;
    int rc = compile_batch(p, L, beam, st->m->d.V, nodes, level_nodes, out_list, arc_slot, arc_word, arc_ac,
                           arc_slm, start_slot, final_off, finals, utt_stream, ranges, ul, ul_off, rq_off);
    if (rc) { delete p; return rc; }
    {
        std::vector<uint32_t> seen(st->d.S, 0);
        for (uint32_t sid : utt_stream) {
            if (sid >= (uint32_t)st->d.S || seen[sid]) { delete p; g_detail = "stream ids must be distinct and < n_streams"; return OTFLM_ERR_VALUE; }
            seen[sid] = 1;
        }
    }
    if (ranges.empty()) ranges.push_back(StreamRange{0, 0, 0, 0});
    p->utt_stream_host = utt_stream;
    {   // per-utterance arrival-slot ranges (slots are assigned utterance by utterance)
        p->utt_slot_off.assign(1, 0);
        uint64_t nb = 0;
        for (int u = 0; u < L->n_utt; u++) {
            nb += (uint64_t)L->n_nodes[u];
            p->utt_slot_off.push_back(u + 1 < L->n_utt ? nodes[nb].slot_base : p->n_slots);
        }
    }
    DevPlan &d = p->d;
    NodeInfo *dn; uint32_t *dln, *dol, *das, *dss, *dus, *dfo, *dfi; int32_t *daw; double *dac, *dsl;
    StreamRange *drg;
    UttLevel *dul; uint32_t *dulo, *drqo;
    if (ul.empty()) ul.push_back(UttLevel{0, 0, 0, 0, 0, 0, 0, 0});   // keep the buffer non-empty
    g_upload_bytes = 0;
    if ((rc = upload(p->mem, &dn, nodes, s)) || (rc = upload(p->mem, &dln, level_nodes, s)) ||
        (rc = upload(p->mem, &dol, out_list, s)) || (rc = upload(p->mem, &das, arc_slot, s)) ||
        (rc = upload(p->mem, &daw, arc_word, s)) || (rc = upload(p->mem, &dac, arc_ac, s)) ||
        (rc = upload(p->mem, &dsl, arc_slm, s)) || (rc = upload(p->mem, &dss, start_slot, s)) ||
        (rc = upload(p->mem, &dus, utt_stream, s)) || (rc = upload(p->mem, &dfo, final_off, s)) ||
        (rc = upload(p->mem, &dfi, finals, s)) || (rc = upload(p->mem, &drg, ranges, s)) ||
        (rc = upload(p->mem, &dul, ul, s)) || (rc = upload(p->mem, &dulo, ul_off, s)) ||
        (rc = upload(p->mem, &drqo, rq_off, s))) {
        p->mem.free_all(); delete p; return rc;
    }
    d.ul = dul; d.ul_off = dulo; d.rq_off = drqo;
    p->ul_cap = (uint32_t)ul.size();
    p->ws_cap = std::max(p->R_max, rq_off.back());
    d.nodes = dn; d.level_nodes = dln; d.out_list = dol; d.arc_slot = das; d.arc_word = daw;
    d.arc_ac = dac; d.arc_slm = dsl; d.n_utt = p->n_utt; d.utt_start_slot = dss; d.utt_stream = dus;
    d.final_off = dfo; d.finals = dfi; d.ranges = drg;
    p->h2d_bytes = g_upload_bytes;
    bool bad = p->mem.alloc(&d.arr, std::max<uint32_t>(p->n_slots, 1)) != cudaSuccess;
    bad |= p->mem.alloc(&d.slot_win, std::max<uint32_t>(p->n_slots, 1)) != cudaSuccess;
    bad |= p->mem.alloc(&d.tok, std::max<uint32_t>(p->n_slots, 1)) != cudaSuccess;
    uint32_t max_path = std::max<uint32_t>(p->n_levels, 1);
    d.max_path = (int32_t)max_path;
    bad |= p->mem.alloc(&d.out_len, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_arcs, (size_t)p->n_utt * max_path) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_status, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_combined, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_acoustic, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_lm, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_end_ctx, p->n_utt) != cudaSuccess;
    bad |= p->mem.alloc(&d.out_expansions, p->n_utt) != cudaSuccess;
    if (bad) { p->mem.free_all(); delete p; g_detail = "cudaMalloc plan buffers"; return OTFLM_ERR_NOMEM; }
    if ((rc = plan_alloc_workspace(p, std::max<uint32_t>(p->ws_cap, 1), p->n_levels + 1))) { p->mem.free_all(); delete p; return rc; }
    if (p->big_asg) {
        // multi-CTA assign scratch; the streams' first-request table once (all unset)
        const uint32_t W = std::max<uint32_t>(p->ws_cap, 1), C = std::max<uint32_t>(p->ch_cap, 1);
        bool bad2 = p->mem.alloc(&d.as_kind, W) != cudaSuccess || p->mem.alloc(&d.as_slot, W) != cudaSuccess ||
                    p->mem.alloc(&d.as_aux, W) != cudaSuccess || p->mem.alloc(&d.ch_cnt, C) != cudaSuccess ||
                    p->mem.alloc(&d.ch_pre, C) != cudaSuccess;
        if (!bad2 && !st->d.ct_first) {
            const size_t n = (size_t)st->d.S * st->d.ct_cap;
            bad2 = st->mem.alloc(&st->d.ct_first, n) != cudaSuccess;
            if (!bad2) CK(cudaMemsetAsync(st->d.ct_first, 0xFF, n * 4, s));
        }
        if (bad2) { p->mem.free_all(); delete p; g_detail = "cudaMalloc assign scratch"; return OTFLM_ERR_NOMEM; }
    }
    *out = p;
    return OTFLM_OK;
}

// Load a new lattice batch into an existing plan.  If the compiled
// structure (levels, per-level node / request / range counts, slots, arcs,
// utterances, stream ids) is identical, the arrays are copied into the same
// device buffers and every captured CUDA graph stays valid: the next run is
// a graph replay.  Returns OTFLM_ERR_VALUE with *same == 0 otherwise (the
// caller creates a new plan).
extern "C" int otflm_plan_refresh(OtflmPlan *p, const OtflmLatticeBatch *L, int32_t *same, void *stream) {
    if (!p || !L || !same) return OTFLM_ERR_VALUE;
    *same = 0;
    if ((uint32_t)L->n_utt != p->n_utt) return OTFLM_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    OtflmPlan tmp;
    tmp.expb_min = p->expb_min; tmp.asg_big = p->asg_big;
    std::vector<NodeInfo> nodes;
    std::vector<uint32_t> level_nodes, out_list, arc_slot, start_slot, final_off, finals, utt_stream;
    std::vector<int32_t> arc_word;
    std::vector<double> arc_ac, arc_slm;
    std::vector<StreamRange> ranges;
    std::vector<UttLevel> ul;
    std::vector<uint32_t> ul_off, rq_off;
    int rc = compile_batch(&tmp, L, p->beam, p->st->m->d.V, nodes, level_nodes, out_list, arc_slot, arc_word,
                           arc_ac, arc_slm, start_slot, final_off, finals, utt_stream, ranges, ul, ul_off, rq_off);
    if (rc) return rc;
    if (ranges.empty()) ranges.push_back(StreamRange{0, 0, 0, 0});
    if (ul.empty()) ul.push_back(UttLevel{0, 0, 0, 0, 0, 0, 0, 0});
    if (ul.size() > p->ul_cap || rq_off.back() > p->ws_cap) return OTFLM_ERR_VALUE;
    if (tmp.n_levels != p->n_levels || tmp.n_nodes != p->n_nodes || tmp.n_arcs != p->n_arcs ||
        tmp.n_slots != p->n_slots || tmp.R_max != p->R_max || tmp.has_big != p->has_big || tmp.lvl_node_off != p->lvl_node_off ||
        tmp.lvl_req != p->lvl_req || tmp.lvl_range_off != p->lvl_range_off || utt_stream != p->utt_stream_host)
        return OTFLM_ERR_VALUE;
    DevPlan &d = p->d;
    // stage every array in one pinned buffer, then issue async copies
    size_t need = 0;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    need += al(nodes.size() * sizeof(NodeInfo)) + al(level_nodes.size() * 4) + al(out_list.size() * 4) +
            al(arc_slot.size() * 4) + al(arc_word.size() * 4) + al(arc_ac.size() * 8) + al(arc_slm.size() * 8) +
            al(start_slot.size() * 4) + al(final_off.size() * 4) + al(finals.size() * 4) +
            al(ranges.size() * sizeof(StreamRange)) + al(ul.size() * sizeof(UttLevel)) + al(ul_off.size() * 4) +
            al(rq_off.size() * 4);
    if (p->ev_staged) CK(cudaEventSynchronize(p->ev_staged));     // previous uploads left the buffer
    if (need > p->staging_cap) {
        if (p->staging) cudaFreeHost(p->staging);
        p->staging = nullptr;
        p->staging_cap = 0;
        CK(cudaMallocHost((void **)&p->staging, need));
        p->staging_cap = need;
    }
    if (!p->ev_staged) CK(cudaEventCreateWithFlags(&p->ev_staged, cudaEventDisableTiming));
    if (!p->up) {
        CK(cudaStreamCreateWithFlags(&p->up, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&p->ev_up, cudaEventDisableTiming));
    }
    if (p->ev_lastrun) CK(cudaStreamWaitEvent(p->up, p->ev_lastrun, 0));   // buffers free again
    size_t pos = 0;
    auto put = [&](const void *dst, const void *src, size_t bytes) -> cudaError_t {
        if (!bytes) return cudaSuccess;
        std::memcpy(p->staging + pos, src, bytes);
        cudaError_t e = cudaMemcpyAsync((void *)dst, p->staging + pos, bytes, cudaMemcpyHostToDevice, p->up);
        pos += al(bytes);
        return e;
    };
    CK(put(d.nodes, nodes.data(), nodes.size() * sizeof(NodeInfo)));
    CK(put(d.level_nodes, level_nodes.data(), level_nodes.size() * 4));
    CK(put(d.out_list, out_list.data(), out_list.size() * 4));
    CK(put(d.arc_slot, arc_slot.data(), arc_slot.size() * 4));
    CK(put(d.arc_word, arc_word.data(), arc_word.size() * 4));
    CK(put(d.arc_ac, arc_ac.data(), arc_ac.size() * 8));
    CK(put(d.arc_slm, arc_slm.data(), arc_slm.size() * 8));
    CK(put(d.utt_start_slot, start_slot.data(), start_slot.size() * 4));
    CK(put(d.final_off, final_off.data(), final_off.size() * 4));
    CK(put(d.finals, finals.data(), finals.size() * 4));
    CK(put(d.ranges, ranges.data(), ranges.size() * sizeof(StreamRange)));
    CK(put(d.ul, ul.data(), ul.size() * sizeof(UttLevel)));
    CK(put(d.ul_off, ul_off.data(), ul_off.size() * 4));
    CK(put(d.rq_off, rq_off.data(), rq_off.size() * 4));
    CK(cudaEventRecord(p->ev_staged, p->up));
    CK(cudaEventRecord(p->ev_up, p->up));
    CK(cudaStreamWaitEvent(s, p->ev_up, 0));          // the next run on s sees the new batch
    *same = 1;
    return OTFLM_OK;
}

extern "C" int otflm_plan_destroy(OtflmPlan *p) {
    if (!p) return OTFLM_OK;
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->graph) cudaGraphDestroy(p->graph);
    p->mem.free_all();
    delete p;
    return OTFLM_OK;
}

extern "C" int otflm_plan_info(const OtflmPlan *p, int64_t *o) {
    if (!p || !o) return OTFLM_ERR_VALUE;
    o[0] = p->n_levels; o[1] = p->n_nodes; o[2] = p->n_arcs; o[3] = p->n_slots;
    o[4] = p->R_max; o[5] = (int64_t)p->total_req; o[6] = p->g_nodes; o[7] = p->n_utt;
    return OTFLM_OK;
}

extern "C" int otflm_plan_wide(const OtflmPlan *p, int32_t *flags) {
    if (!p || !flags) return OTFLM_ERR_VALUE;
    *flags = (p->has_big ? 1 : 0) | (p->big_asg ? 2 : 0);
    return OTFLM_OK;
}

extern "C" int otflm_plan_phase_ns(const OtflmPlan *p, int64_t *o, void *stream) {
    if (!p || !o) return OTFLM_ERR_VALUE;
    unsigned long long a[32] = {0};
    CK(cudaMemcpyAsync(a, p->alg_buf + 8, sizeof(a), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    for (int i = 0; i < 12; i++) o[i] = (int64_t)a[i];
    for (int i = 0; i < 5; i++) o[12 + i] = (int64_t)a[16 + i];
    for (int i = 0; i < 4; i++) o[17 + i] = (int64_t)a[12 + i];   // EXACT update: row table, digitize, spare
    for (int i = 0; i < 3; i++) o[21 + i] = (int64_t)a[21 + i];   // EXACT HS (rank 0): digits wait, GEMM, log-sigmoid
    o[24] = (int64_t)a[24]; o[25] = (int64_t)a[25];                 // EXACT update: plane-copy row pass, copy
    o[26] = (int64_t)a[26]; o[27] = (int64_t)a[27];                 // EXACT update: MMA warp's K loop, epilogue stores
    for (int i = 28; i < 32; i++) o[i] = (int64_t)a[i];            // warp 2 under the K loops: HS tail, rows, fallbacks, U
    return OTFLM_OK;
}

extern "C" int otflm_plan_counters(const OtflmPlan *p, int64_t *o, void *stream) {
    if (!p || !o) return OTFLM_ERR_VALUE;
    unsigned long long a[6] = {0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(a, p->alg_buf, sizeof(a), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    o[0] = (int64_t)a[0]; o[1] = (int64_t)a[1]; o[2] = (int64_t)a[2];
    o[3] = (int64_t)p->h2d_bytes;
    o[4] = (int64_t)a[3];
    o[5] = (int64_t)a[5];
    return OTFLM_OK;
}

// stage 2 of a level: HS on the side branch || recurrent update on s
static int enqueue_stage2(OtflmPlan *p, const DevModel &m, DevStreams &S, uint32_t R, int prec,
                          const RowSpec &rs, cudaStream_t s) {
    DevPlan &d = p->d;
    if (prec == OTFLM_PREC_EXACT && m.Wd && m.NVd && m.H % 64 == 0 && m.H <= 512 && p->hs_tc && p->lvl_fused &&
        (R + xu::XR - 1) / xu::XR > 148) {
        // EXACT, a level of more 80-request chunks than SMs: HS + recurrent
        // update in one persistent kernel (exact_solo.cuh k_level_exact,
        // k_decode_solo's chunk body: one digitize, no second kernel holding
        // SMs).  Smaller levels keep the two kernels side by side, which
        // halves the level's latency (HS and update of a chunk on two SMs).
        ProfScope ps(K_ADVANCE, s);
        const int ord = m.order <= 3 ? 3 : OTF_MAX_ORDER;
        const size_t smem = xs1::smem_bytes(ord);
        const size_t stride = 2 * xu::xs_slot_bytes(m.wd_nkx);
        const unsigned grid = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>(148, (R + xu::XR - 1) / xu::XR));
        uint8_t *scratch = nullptr;
        if (cudaMallocAsync(&scratch, stride * grid, s) != cudaSuccess) {
            g_detail = "cudaMallocAsync exact level scratch"; return OTFLM_ERR_NOMEM;
        }
#define LX_LAUNCH(ORD)                                                                                          \
        do {                                                                                                    \
            CK(cudaFuncSetAttribute(k_level_exact<ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
            k_level_exact<ORD><<<grid, sd::NT, smem, s>>>(m, d, S, rs, scratch, stride);                     \
        } while (0)
        if (ord == 3) LX_LAUNCH(3); else LX_LAUNCH(OTF_MAX_ORDER);
#undef LX_LAUNCH
        CKL();
        CK(cudaFreeAsync(scratch, s));
        return OTFLM_OK;
    }
    CK(cudaEventRecord(p->ev_fork, s));
    CK(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    {
        ProfScope ps(K_HS, p->side);
        // EXACT: the digit-plane HS on the tensor cores (exact_solo.cuh k_hs_exact)
        const bool hs_tc = prec == OTFLM_PREC_EXACT && m.Wd && m.NVd && m.H % 64 == 0 && m.H <= 512 && p->hs_tc;
        if (hs_tc) {
            const int ord = m.order <= 3 ? 3 : OTF_MAX_ORDER;
            const size_t smem = xs1::smem_bytes(ord);
            const size_t stride = 2 * xu::xs_slot_bytes(m.wd_nkx);
            const unsigned grid = (unsigned)std::max<uint32_t>(1, std::min<uint32_t>(148, (R + xu::XR - 1) / xu::XR));
            uint8_t *scratch = nullptr;
            if (cudaMallocAsync(&scratch, stride * grid, p->side) != cudaSuccess) {
                g_detail = "cudaMallocAsync exact HS scratch"; return OTFLM_ERR_NOMEM;
            }
#define HX_LAUNCH(ORD)                                                                                          \
            do {                                                                                                \
                CK(cudaFuncSetAttribute(k_hs_exact<ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
                k_hs_exact<ORD><<<grid, sd::NT, smem, p->side>>>(m, d, S, rs, scratch, stride);                \
            } while (0)
            if (ord == 3) HX_LAUNCH(3); else HX_LAUNCH(OTF_MAX_ORDER);
#undef HX_LAUNCH
            CKL();
            CK(cudaFreeAsync(scratch, p->side));
        } else if (m.H % 4 == 0 && m.H <= 1024) {
            // persistent TMA-ring warps: enough CTAs for the level, at most the
            // resident capacity of the GPU
            const size_t smem = 4 * ring_bytes_per_warp(m.H);
            const bool exact = prec == OTFLM_PREC_FP64 || prec == OTFLM_PREC_EXACT;
#define CALLR(CPL, EX, ORD)                                                                                        \
            do {                                                                                                   \
                CK(cudaFuncSetAttribute(k_hs_prim_ring<CPL, EX, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
                int per_sm = 1;                                                                                    \
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hs_prim_ring<CPL, EX, ORD>, 128, smem)); \
                const unsigned grid = (unsigned)std::min<uint64_t>(cdiv(R, 4), (uint64_t)148 * std::max(per_sm, 1)); \
                k_hs_prim_ring<CPL, EX, ORD><<<grid, 128, smem, p->side>>>(m, d, S, rs);                          \
            } while (0)
            if (exact) RING_DISPATCH(m.H, true, m.order, CALLR);
            else RING_DISPATCH(m.H, false, m.order, CALLR);
#undef CALLR
        } else {
#define CALL(VEC, CPL) k_hs_prim<VEC, CPL><<<cdiv(R, 8), 256, 0, p->side>>>(m, d, S, rs)
            HS_DISPATCH(m.H, CALL);
#undef CALL
        }
        CKL();
    }
    {
        ProfScope ps(K_ADVANCE, s);
        int rc = launch_advance(m, prec, R, rs, d.pr_inrow, d.pr_w, S.arena_h, S.arena_h, rs.row_limit, s);
        if (rc) return rc;
    }
    CK(cudaEventRecord(p->ev_join, p->side));
    CK(cudaStreamWaitEvent(s, p->ev_join, 0));
    return OTFLM_OK;
}

static int enqueue_run(OtflmPlan *p, const OtflmNgram *g, double lm, int prec, cudaStream_t s) {
    OtflmStreams *st = p->st;
    const DevModel &m = st->m->d;
    DevStreams &S = st->d;
    DevPlan &d = p->d;
    CK(cudaMemsetAsync(d.arr, 0xFF, (size_t)std::max<uint32_t>(p->n_slots, 1) * sizeof(Arrival), s));
    CK(cudaMemsetAsync(d.lvl, 0, (size_t)(p->n_levels + 1) * sizeof(LevelCtr), s));
    if (d.alg) CK(cudaMemsetAsync(d.alg, 0, 4 * sizeof(unsigned long long), s));
    if (d.kept) CK(cudaMemsetAsync(d.kept, 0, std::max<uint32_t>(p->n_slots, 1), s));
    { ProfScope ps(K_MISC, s); k_run_begin<<<cdiv(p->n_utt, 128), 128, 0, s>>>(d, S); CKL(); }
    if (p->has_big)
        CK(cudaFuncSetAttribute(k_expand_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)expb_smem(EXPB_MAX)));
    int prev = -1;
    for (uint32_t t = 0; t < p->n_levels; t++) {
        const uint32_t nb0 = p->lvl_node_off[t], nn = p->lvl_node_off[t + 1] - nb0;
        const uint32_t R = p->lvl_req[t];
        auto expand = [&]() -> int {
            ProfScope ps(K_EXPAND, s);
            k_expand<<<cdiv(nn, 8), 256, 0, s>>>(d, S, g->d, nb0, nn, (long long)p->beam, t,
                                                 p->has_big ? p->expb_min : 0xFFFFFFFFu);
            CKL();
            if (p->has_big) {             // a CTA per node with many arrival slots
                k_expand_big<<<nn, EXPB_T, expb_smem(EXPB_MAX), s>>>(d, S, g->d, nb0, (long long)p->beam, t, EXPB_MAX,
                                                                     p->expb_min);
                CKL();
            }
            return OTFLM_OK;
        };
        if (nn == 0 || R == 0) {
            if (nn) { int rc = expand(); if (rc) return rc; }
            continue;
        }
        { int rc = expand(); if (rc) return rc; }
        const bool part = d.arena_start != OTF_UNSET;
        const RowSpec rs{&d.lvl[t].n_prim, &d.lvl[t], prev >= 0 ? &d.lvl[prev] : nullptr,
                         part ? d.cursor : S.arena_used, d.pr_dig, part ? d.arena_end : S.arena_rows};
        int rc = enqueue_stage2(p, m, S, R, prec, rs, s);
        if (rc) return rc;
        const uint32_t r0 = p->lvl_range_off[t], nr = p->lvl_range_off[t + 1] - r0;
        if (p->big_asg && !S.lfu_log && S.ct_first) {
            // many requests per stream: the ordered resolution over chunks (decode.cuh k_asg_*)
            ProfScope ps(K_ASSIGN, s);
            const uint32_t nch = (R + ASG_CH - 1) / ASG_CH;
            const dim3 grid(nch, nr);
            const uint32_t limit = d.arena_start == OTF_UNSET ? S.arena_rows : d.arena_end;
            k_asg_probe<<<grid, ASG_CH, 0, s>>>(d, S, t, r0, limit); CKL();
            k_asg_dedup<<<grid, ASG_CH, 0, s>>>(d, S, t, r0, limit); CKL();
            k_asg_scan<<<nr, 32, 0, s>>>(d, S, t, r0, nch, limit); CKL();
            k_asg_number<<<grid, ASG_CH, 0, s>>>(d, S, t, r0, limit); CKL();
            k_asg_values<<<grid, ASG_CH, 0, s>>>(d, S, t, r0, limit); CKL();
            k_asg_arrive<<<grid, ASG_CH, 0, s>>>(d, S, t, r0, limit, lm); CKL();
        } else {
            ProfScope ps(K_ASSIGN, s);
            k_assign<0><<<nr, ASSIGN_T, 0, s>>>(d, S, t, r0, lm, nullptr, nullptr, nullptr);
            CKL();
        }
        prev = (int)t;
    }
    { ProfScope ps(K_FINAL, s); k_final<<<cdiv(p->n_utt, 4), 128, 0, s>>>(d, S, lm, prev); CKL(); }
    if (!p->grouped) { int rc = lfu_enqueue(p->st, s); if (rc) return rc; }
    return OTFLM_OK;
}

// ---- persistent per-stream schedule (stream_decode.cuh) ----
struct SdConfig { int stages, qb_max; size_t smem; uint32_t tmem_cols; };
static bool sd_config(const DevModel &m, int prec, SdConfig *c) {
    if (prec == OTFLM_PREC_EXACT) {
        if (!m.Wd || m.H % 4 != 0 || m.H > 512 || !m.U || !m.NV || !m.path_off) return false;
        if (!m.NVd) return false;
        const size_t budget = 200u * 1024u;
        // 2 ring stages + the staged U block of a tile (the epilogue reads U
        // from shared memory); the K loop is MMA-bound with W planes in L2
        const size_t tail = xu::tail_layout().total + xu::US_BYTES;
        c->stages = 2;
        if ((size_t)c->stages * xu::STAGE + tail > budget) return false;
        const int ord = m.order <= 3 ? 3 : OTF_MAX_ORDER;
        // rank 1: the update ring + tail; rank 0: the HS ring + pair tables
        const size_t hs_bytes = (size_t)xh::ring_bytes() + xh::layout(ord).total;
        c->qb_max = 0;
        c->smem = std::max((size_t)c->stages * xu::STAGE + tail, hs_bytes);
        c->smem = std::max(c->smem, (size_t)28 * sd::NT);
        if (c->smem > 207u * 1024u) return false;
        c->tmem_cols = 512;
        return true;
    }
    if (!(prec == OTFLM_PREC_TF32X3 || prec == OTFLM_PREC_TF32)) return false;
    if (!m.W_t || m.H % 4 != 0 || m.wt_npad > 512 || !m.U || !m.NV || !m.path_off) return false;
    const bool x3 = prec == OTFLM_PREC_TF32X3;
    const size_t stage = (x3 ? 2u : 1u) * ((size_t)m.wt_npad * m.wt_kcb + (size_t)tc::BM * m.wt_kcb);
    const size_t budget = 200u * 1024u;                   // + ~21 KB static shared memory
    // rank 1 (update) uses the dynamic shared memory as its ring, rank 0
    // (control) as the HS scratch: one size serves both
    c->stages = (int)std::min<size_t>(4, budget / stage);
    if (c->stages < 2) return false;
    const int ord = m.order <= 3 ? 3 : OTF_MAX_ORDER;
    const size_t hs_fixed = (size_t)sd::PAIRCAP * 13 + (size_t)sd::QMAX * (ord * 8 + 7 * 4) + (sd::NW + 2) * 4 + 64;
    if (hs_fixed + 8 * 4 * (size_t)m.H > budget) return false;
    c->qb_max = (int)std::min<size_t>(sd::QMAX, (budget - hs_fixed) / (4 * (size_t)m.H));
    c->smem = std::max((size_t)c->stages * stage, hs_fixed + (size_t)c->qb_max * 4 * m.H);
    c->smem = std::max(c->smem, (size_t)28 * sd::NT);       // assign's chunk dedup hash (rank 0)
    c->tmem_cols = 128;
    while ((int)c->tmem_cols < m.wt_npad) c->tmem_cols <<= 1;
    return true;
}

static int launch_streams(OtflmPlan *p, const OtflmNgram *g, double lm, int prec, cudaStream_t s) {
    const DevModel &m = p->st->m->d;
    DevStreams &S = p->st->d;
    DevPlan &d = p->d;
    SdConfig c;
    if (!sd_config(m, prec, &c)) { g_detail = "persistent schedule needs an EXACT/TF32X3/TF32 precision and H % 4 == 0, H <= 512"; return OTFLM_ERR_VALUE; }
    const bool part = d.arena_start != OTF_UNSET;
    uint32_t *cursor = part ? d.cursor : S.arena_used;
    const uint32_t limit = part ? d.arena_end : S.arena_rows;
#define SD_LAUNCH(MODE, KCB, CPL, ORD)                                                                          \
    do {                                                                                                        \
        CK(cudaFuncSetAttribute(k_decode_streams<MODE, KCB, CPL, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem)); \
        k_decode_streams<MODE, KCB, CPL, ORD><<<2 * p->n_utt, sd::NT, c.smem, s>>>(m, d, S, g->d, (long long)p->beam, lm, \
                                                                              c.stages, c.qb_max, cursor, limit, c.tmem_cols, \
                                                                              p->xs, xs_stride, x_epoch, 1); \
    } while (0)
#define SD_ORD(MODE, KCB, CPL) do { if (m.order <= 3) SD_LAUNCH(MODE, KCB, CPL, 3); else SD_LAUNCH(MODE, KCB, CPL, OTF_MAX_ORDER); } while (0)
#define SD_H(MODE)                                                                                              \
    do {                                                                                                        \
        if (m.H <= 128) SD_ORD(MODE, 128, 1);                                                                   \
        else if (m.H <= 256) SD_ORD(MODE, 128, 2);                                                              \
        else SD_ORD(MODE, 64, 4);                                                                               \
    } while (0)
    size_t xs_stride = 0;
    uint32_t x_epoch = 0;
    if (prec == OTFLM_PREC_EXACT) {
        // per-arena-row digit planes (made at row creation), allocated on first use
        OtflmStreams *st = p->st;
        if (!st->d.arena_dig) {
            uint8_t *dg = nullptr; float *deh = nullptr; uint32_t *dep = nullptr;
            const size_t rows = std::max<uint32_t>(st->d.arena_rows, 1);
            if (st->mem.alloc(&dg, rows * (size_t)m.wd_nkx * 4 * xu::KC) != cudaSuccess ||
                st->mem.alloc(&deh, rows) != cudaSuccess || st->mem.alloc(&dep, rows) != cudaSuccess) {
                g_detail = "cudaMalloc digit store"; return OTFLM_ERR_NOMEM;
            }
            CK(cudaMemsetAsync(dep, 0, rows * 4, s));
            st->d.arena_dig = dg; st->d.arena_deh = deh; st->d.arena_dep = dep;
        }
        x_epoch = ++st->dig_epoch;
        S.arena_dig = st->d.arena_dig; S.arena_deh = st->d.arena_deh; S.arena_dep = st->d.arena_dep;
        // two chunk slots of digit planes per stream: [slot][kc][plane][XR rows x 64 B]
        xs_stride = 2 * xu::xs_slot_bytes(m.wd_nkx);
        const size_t need = xs_stride * std::max<uint32_t>(p->n_utt, 1);
        if (p->xs_bytes < need) {
            uint8_t *x = nullptr;
            if (p->mem.alloc(&x, need) != cudaSuccess) { g_detail = "cudaMalloc exact scratch"; return OTFLM_ERR_NOMEM; }
            p->xs = x; p->xs_bytes = need;
        }
        if (p->schedule == OTFLM_SCHED_STREAM1) {
            // persistent CTAs (one per SM at most) taking the streams from a queue (exact_solo.cuh)
            const int ord = m.order <= 3 ? 3 : OTF_MAX_ORDER;
            const size_t smem = xs1::smem_bytes(ord);
            int dev = 0, n_sm = 148;
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
            const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(p->n_utt, (uint32_t)n_sm));
            if (!p->work) {
                if (p->mem.alloc(&p->work, 1) != cudaSuccess) { g_detail = "cudaMalloc work queue"; return OTFLM_ERR_NOMEM; }
            }
            CK(cudaMemsetAsync(p->work, 0, sizeof(uint32_t), s));
#define SO_LAUNCH(ORD)                                                                                          \
            do {                                                                                                \
                CK(cudaFuncSetAttribute(k_decode_solo<ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
                k_decode_solo<ORD><<<grid, sd::NT, smem, s>>>(m, d, S, g->d, (long long)p->beam, lm, cursor, limit, \
                                                              p->xs, xs_stride, x_epoch, p->work);                \
            } while (0)
            if (ord == 3) SO_LAUNCH(3); else SO_LAUNCH(OTF_MAX_ORDER);
#undef SO_LAUNCH
        } else if (m.H <= 128) SD_ORD(4, 64, 1);
        else if (m.H <= 256) SD_ORD(4, 64, 2);
        else SD_ORD(4, 64, 4);
    } else {
        if ((m.wt_npad <= 256 ? 128 : 64) != m.wt_kcb) { g_detail = "W tile layout mismatch"; return OTFLM_ERR_VALUE; }
        if (prec == OTFLM_PREC_TF32X3) SD_H(1); else SD_H(3);
    }
#undef SD_H
#undef SD_ORD
#undef SD_LAUNCH
    CKL();
    return OTFLM_OK;
}

static int enqueue_streams(OtflmPlan *p, const OtflmNgram *g, double lm, int prec, cudaStream_t s) {
    DevStreams &S = p->st->d;
    DevPlan &d = p->d;
    if (d.kept) CK(cudaMemsetAsync(d.kept, 0, std::max<uint32_t>(p->n_slots, 1), s));
    CK(cudaMemsetAsync(d.arr, 0xFF, (size_t)std::max<uint32_t>(p->n_slots, 1) * sizeof(Arrival), s));
    if (d.alg) CK(cudaMemsetAsync(d.alg, 0, 40 * sizeof(unsigned long long), s));   // counters + all phase slots
    { ProfScope ps(K_MISC, s); k_run_begin<<<cdiv(p->n_utt, 128), 128, 0, s>>>(d, S); CKL(); }
    { ProfScope ps(K_STREAM, s); int rc = launch_streams(p, g, lm, prec, s); if (rc) return rc; }
    { ProfScope ps(K_FINAL, s); k_final<<<cdiv(p->n_utt, 4), 128, 0, s>>>(d, S, lm, -1); CKL(); }
    return lfu_enqueue(p->st, s);
}

extern "C" int otflm_plan_set_schedule(OtflmPlan *p, int32_t schedule) {
    if (!p || (schedule != OTFLM_SCHED_LEVEL && schedule != OTFLM_SCHED_STREAM && schedule != OTFLM_SCHED_STREAM1))
        return OTFLM_ERR_VALUE;
    p->schedule = schedule;
    return OTFLM_OK;
}

extern "C" int otflm_schedule_supported(const OtflmModel *m, int32_t schedule, int32_t precision) {
    if (!m) return 0;
    if (schedule == OTFLM_SCHED_LEVEL) return prec_ok(precision) ? 1 : 0;
    SdConfig c;
    if (schedule == OTFLM_SCHED_STREAM1)
        return precision == OTFLM_PREC_EXACT && sd_config(m->d, precision, &c) &&
               xs1::smem_bytes(m->d.order <= 3 ? 3 : OTF_MAX_ORDER) <= 207u * 1024u ? 1 : 0;
    return schedule == OTFLM_SCHED_STREAM && sd_config(m->d, precision, &c) ? 1 : 0;
}

static int enqueue_any(OtflmPlan *p, const OtflmNgram *g, double lm, int prec, cudaStream_t s) {
    return p->schedule != OTFLM_SCHED_LEVEL ? enqueue_streams(p, g, lm, prec, s) : enqueue_run(p, g, lm, prec, s);
}

static int64_t g_last_launches = 0;

static int decode_run_impl(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                           int32_t use_graph, void *stream);
extern "C" int otflm_decode_run(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                                int32_t use_graph, void *stream) {
    int rc = decode_run_impl(p, g, lm_weight, precision, use_graph, stream);
    if (rc == OTFLM_OK) {      // the plan's input arrays may be refreshed once this run is done
        if (!p->ev_lastrun) CK(cudaEventCreateWithFlags(&p->ev_lastrun, cudaEventDisableTiming));
        CK(cudaEventRecord(p->ev_lastrun, (cudaStream_t)stream));
    }
    return rc;
}

static int decode_run_impl(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                           int32_t use_graph, void *stream) {
    if (!p || !g) return OTFLM_ERR_VALUE;
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    // (EXACT in the level schedule: k_advance_exact + the float64 HS kernels)
    if (g->d.order - 1 > p->st->m->d.order) { g_detail = "small LM order exceeds the stored context history"; return OTFLM_ERR_VALUE; }
    if (g->d.V < p->st->m->d.V) { g_detail = "small LM vocabulary smaller than model"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    g_launches = 0;
    if (!use_graph || p->schedule != OTFLM_SCHED_LEVEL) {   // the persistent schedules are 3 launches
        int rc = enqueue_any(p, g, lm_weight, precision, s);
        g_last_launches = g_launches;
        return rc;
    }
    if (!p->gexec || p->g_lm != lm_weight || p->g_prec != precision || p->g_ng != g ||
        p->g_ver != p->st->version) {
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
        // capture on a private stream (the caller's may be the legacy default stream)
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_run(p, g, lm_weight, precision, cs);
        cudaGraph_t graph;
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        CK(e);
        p->graph = graph;
        CK(cudaGraphInstantiate(&p->gexec, graph, 0));
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        p->g_nodes = (int64_t)nn;
        p->g_lm = lm_weight; p->g_prec = precision; p->g_ng = g; p->g_ver = p->st->version;
        g_last_launches = g_launches;
    }
    CK(cudaGraphLaunch(p->gexec, s));
    return OTFLM_OK;
}

extern "C" int64_t otflm_last_launch_count(void) { return g_last_launches; }

extern "C" int otflm_decode_profile(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                                    void *stream, double *ms_out, int64_t *n_out) {
    if (!p || !g) return OTFLM_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < K_NCAT; i++) { g_prof_ms[i] = 0; g_prof_n[i] = 0; }
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    g_prof = true;
    p->d.alg = p->alg_buf;
    p->d.phase_ns = p->alg_buf + 8;
    int rc = enqueue_any(p, g, lm_weight, precision, cs);
    p->d.alg = nullptr;
    p->d.phase_ns = nullptr;
    g_prof = false;
    cudaGraph_t graph;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc) return rc;
    CK(e);
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, graph, 0));
    CK(cudaGraphLaunch(ex, s));
    CK(cudaStreamSynchronize(s));
    for (auto &ev : g_prof_ev) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev.second.first, ev.second.second));
        g_prof_ms[ev.first] += ms;
        g_prof_n[ev.first] += 1;
        cudaEventDestroy(ev.second.first);
        cudaEventDestroy(ev.second.second);
    }
    g_prof_ev.clear();
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(graph);
    for (int i = 0; i < K_NCAT; i++) { if (ms_out) ms_out[i] = g_prof_ms[i]; if (n_out) n_out[i] = g_prof_n[i]; }
    return OTFLM_OK;
}

extern "C" int otflm_decode_fetch(OtflmPlan *p, OtflmDecodeResult *r, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t U = p->n_utt, MP = (uint32_t)p->d.max_path;
    std::vector<int32_t> len(U), status(U), arcs((size_t)U * MP);
    std::vector<double> comb(U), ac(U), lm(U);
    std::vector<long long> endc(U), exps(U);
    CK(cudaMemcpyAsync(len.data(), p->d.out_len, U * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(status.data(), p->d.out_status, U * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(arcs.data(), p->d.out_arcs, (size_t)U * MP * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(comb.data(), p->d.out_combined, U * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ac.data(), p->d.out_acoustic, U * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(lm.data(), p->d.out_lm, U * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(endc.data(), p->d.out_end_ctx, U * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(exps.data(), p->d.out_expansions, U * 8, cudaMemcpyDeviceToHost, s));
    int rc = check_err(p->st, s);
    if (rc) return rc;
    for (uint32_t u = 0; u < U; u++) {
        r->path_len[u] = len[u];
        r->status[u] = status[u];
        r->combined[u] = comb[u];
        r->acoustic[u] = ac[u];
        r->lm[u] = lm[u];
        r->end_ctx[u] = endc[u];
        r->expansions[u] = exps[u];
        int32_t n = std::min<int32_t>(len[u], r->max_path);
        for (int32_t k = 0; k < n; k++) r->path_arcs[(size_t)u * r->max_path + k] = arcs[(size_t)u * MP + k];
    }
    for (uint32_t u = 0; u < U; u++) if (status[u]) return status[u];
    return OTFLM_OK;
}

extern "C" int otflm_decode(OtflmStreams *s, const OtflmNgram *g, const OtflmLatticeBatch *lats, double lm_weight,
                            int64_t beam, int32_t precision, OtflmDecodeResult *res, void *stream) {
    OtflmPlan *p = nullptr;
    int rc = otflm_plan_create(s, lats, beam, &p, stream);
    if (rc) return rc;
    rc = otflm_decode_run(p, g, lm_weight, precision, 0, stream);
    if (!rc) rc = otflm_decode_fetch(p, res, stream);
    cudaStreamSynchronize((cudaStream_t)stream);
    otflm_plan_destroy(p);
    return rc;
}

// ==========================================================================
// plan groups: several plans over disjoint utterances (and disjoint arena
// partitions) captured as parallel dependency chains of one CUDA graph, so
// the latency-bound level stages of different groups overlap on the GPU
// ==========================================================================
extern "C" int otflm_plan_set_lattice_out(OtflmPlan *p, int32_t enable) {
    if (!p) return OTFLM_ERR_VALUE;
    if (enable && !p->lat_rec) {
        const size_t n = std::max<uint32_t>(p->n_slots, 1);
        uint8_t *kept;
        if (p->mem.alloc(&kept, n) || p->mem.alloc(&p->lat_rec, n) || p->mem.alloc(&p->lat_cnt, p->n_utt) ||
            p->mem.alloc(&p->utt_slot_off_dev, p->utt_slot_off.size())) {
            g_detail = "cudaMalloc lattice-out"; return OTFLM_ERR_NOMEM;
        }
        CK(cudaMemcpy(p->utt_slot_off_dev, p->utt_slot_off.data(), p->utt_slot_off.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(kept, 0, n));
        p->kept_buf = kept;
    }
    uint8_t *want = enable ? p->kept_buf : nullptr;
    if (p->d.kept != want) {          // captured graphs hold the old plan arguments
        p->d.kept = want;
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
    }
    return OTFLM_OK;
}

extern "C" int otflm_decode_lattice_fetch(OtflmPlan *p, int64_t *count_host, void *records_host, int64_t cap,
                                          void *stream) {
    if (!p || !p->d.kept) { g_detail = "lattice-out not enabled on this plan"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    k_lattice_out<<<p->n_utt, 256, 0, s>>>(p->d, p->utt_slot_off_dev, p->lat_rec, p->lat_cnt);
    CKL();
    std::vector<long long> cnt(p->n_utt);
    CK(cudaMemcpyAsync(cnt.data(), p->lat_cnt, p->n_utt * sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t total = 0;
    for (uint32_t u = 0; u < p->n_utt; u++) { count_host[u] = cnt[u]; total += cnt[u]; }
    if (!records_host) return OTFLM_OK;              // size query
    if (total > cap) { g_detail = "record buffer too small"; return OTFLM_ERR_VALUE; }
    uint8_t *dst = (uint8_t *)records_host;
    for (uint32_t u = 0; u < p->n_utt; u++) {        // utterance u's records sit at its slot base
        if (!cnt[u]) continue;
        CK(cudaMemcpyAsync(dst, p->lat_rec + p->utt_slot_off[u], cnt[u] * sizeof(LatRecord), cudaMemcpyDeviceToHost, s));
        dst += cnt[u] * sizeof(LatRecord);
    }
    CK(cudaStreamSynchronize(s));
    return OTFLM_OK;
}

extern "C" int otflm_plan_set_arena(OtflmPlan *p, uint32_t start, uint32_t end) {
    if (!p || end <= start || end > p->st->d.arena_rows || start == 0) return OTFLM_ERR_VALUE;
    p->d.arena_start = start;
    p->d.arena_end = end;
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
    if (p->graph) { cudaGraphDestroy(p->graph); p->graph = nullptr; }
    return OTFLM_OK;
}

struct OtflmGroup {
    std::vector<OtflmPlan *> plans;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaEvent_t ev0 = nullptr;
    double g_lm = 0; int g_prec = -1; const OtflmNgram *g_ng = nullptr;
    uint64_t g_ver = 0;
    int64_t launches = 0;
    ~OtflmGroup() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        if (ev0) cudaEventDestroy(ev0);
    }
};

extern "C" int otflm_group_create(OtflmPlan **plans, int32_t n, OtflmGroup **out) {
    if (!plans || n < 1 || !out) return OTFLM_ERR_VALUE;
    OtflmGroup *g = new OtflmGroup();
    for (int i = 0; i < n; i++) {
        if (!plans[i] || plans[i]->st != plans[0]->st) { delete g; return OTFLM_ERR_VALUE; }
        if (n > 1 && plans[i]->d.arena_start == OTF_UNSET) {
            delete g; g_detail = "grouped plans need disjoint arena partitions"; return OTFLM_ERR_VALUE;
        }
        g->plans.push_back(plans[i]);
        plans[i]->grouped = n > 1;
    }
    CK(cudaEventCreateWithFlags(&g->ev0, cudaEventDisableTiming));
    *out = g;
    return OTFLM_OK;
}

extern "C" int otflm_group_destroy(OtflmGroup *g) {
    delete g;
    return OTFLM_OK;
}

static int enqueue_group(OtflmGroup *g, const OtflmNgram *ng, double lm, int prec, cudaStream_t cs) {
    CK(cudaEventRecord(g->ev0, cs));
    for (OtflmPlan *p : g->plans) {
        CK(cudaStreamWaitEvent(p->chain, g->ev0, 0));
        int rc = enqueue_run(p, ng, lm, prec, p->chain);
        if (rc) return rc;
        CK(cudaEventRecord(p->ev_done, p->chain));
        CK(cudaStreamWaitEvent(cs, p->ev_done, 0));
    }
    return g->plans.empty() ? OTFLM_OK : lfu_enqueue(g->plans[0]->st, cs);
}

extern "C" int otflm_group_run(OtflmGroup *g, const OtflmNgram *ng, double lm_weight, int32_t precision,
                               void *stream) {
    if (!g || !ng || !prec_ok(precision)) return OTFLM_ERR_VALUE;
    /* EXACT: k_advance_exact + float64 HS */
    cudaStream_t s = (cudaStream_t)stream;
    if (!g->gexec || g->g_lm != lm_weight || g->g_prec != precision || g->g_ng != ng ||
        g->g_ver != g->plans[0]->st->version) {
        if (g->gexec) { cudaGraphExecDestroy(g->gexec); g->gexec = nullptr; }
        if (g->graph) { cudaGraphDestroy(g->graph); g->graph = nullptr; }
        g_launches = 0;
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_group(g, ng, lm_weight, precision, cs);
        cudaGraph_t graph;
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        CK(e);
        g->graph = graph;
        CK(cudaGraphInstantiate(&g->gexec, graph, 0));
        g->g_lm = lm_weight; g->g_prec = precision; g->g_ng = ng; g->g_ver = g->plans[0]->st->version;
        g->launches = g_launches;
    }
    g_last_launches = g->launches;
    CK(cudaGraphLaunch(g->gexec, s));
    for (OtflmPlan *gp : g->plans) {
        if (!gp->ev_lastrun) CK(cudaEventCreateWithFlags(&gp->ev_lastrun, cudaEventDisableTiming));
        CK(cudaEventRecord(gp->ev_lastrun, s));
    }
    return OTFLM_OK;
}

extern "C" int otflm_group_profile(OtflmGroup *g, const OtflmNgram *ng, double lm_weight, int32_t precision,
                                   void *stream, double *ms_out, int64_t *n_out) {
    if (!g || !ng) return OTFLM_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < K_NCAT; i++) { g_prof_ms[i] = 0; g_prof_n[i] = 0; }
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    g_prof = true;
    for (OtflmPlan *p : g->plans) p->d.alg = p->alg_buf;
    int rc = enqueue_group(g, ng, lm_weight, precision, cs);
    for (OtflmPlan *p : g->plans) p->d.alg = nullptr;
    g_prof = false;
    cudaGraph_t graph;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc) return rc;
    CK(e);
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, graph, 0));
    CK(cudaGraphLaunch(ex, s));
    CK(cudaStreamSynchronize(s));
    for (auto &ev : g_prof_ev) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev.second.first, ev.second.second));
        g_prof_ms[ev.first] += ms;
        g_prof_n[ev.first] += 1;
        cudaEventDestroy(ev.second.first);
        cudaEventDestroy(ev.second.second);
    }
    g_prof_ev.clear();
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(graph);
    for (int i = 0; i < K_NCAT; i++) { if (ms_out) ms_out[i] = g_prof_ms[i]; if (n_out) n_out[i] = g_prof_n[i]; }
    return OTFLM_OK;
}

// ==========================================================================
// rnnlm_prob_batch: Table-1 lookups in array order (cache.py:165-182)
// ==========================================================================
__global__ void k_probe_batch(DevPlan P, DevStreams S, uint32_t n, const uint32_t *c, const int32_t *w,
                              const uint32_t *sid) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    bool need = false;
    uint32_t s = 0, cc = 0;
    int32_t ww = 0;
    if (r < n) {
        s = sid[r]; cc = c[r]; ww = w[r];
        P.rq_c[r] = cc; P.rq_w[r] = ww; P.rq_m[r] = OTF_UNSET;
        uint8_t st = RQ_NOCACHE;
        uint32_t cslot = OTF_UNSET;
        if (cc > S.table_len[s]) {
            atomicOr(S.err, OTF_E_PATH);
            st = RQ_INVALID;
        } else if (S.enabled) {
            cslot = cache_probe(S, s, cc, ww, r, &st);
        }
        P.rq_cslot[r] = cslot;
        P.rq_state[r] = st;
        need = st == RQ_PENDING || st == RQ_NOCACHE;
    }
    compact_primary(P, S, &P.lvl[0].n_prim, need, r, cc, ww, s);
}

extern "C" int otflm_rnnlm_prob_batch(OtflmStreams *s, int64_t n, const int32_t *sid_h, const uint32_t *c_h,
                                      const int32_t *w_h, int32_t precision, double *p_h, uint32_t *cn_h,
                                      uint8_t *hit_h, void *stream) {
    if (!s || n < 0) return OTFLM_ERR_VALUE;
    if (n == 0) return OTFLM_OK;
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    /* EXACT: k_advance_exact + float64 HS */
    cudaStream_t st = (cudaStream_t)stream;
    const DevModel &m = s->m->d;
    for (int64_t i = 0; i < n; i++) {
        if (w_h[i] < 0 || w_h[i] >= m.V) { g_detail = "word id out of range"; return OTFLM_ERR_VALUE; }
        if (sid_h[i] < 0 || sid_h[i] >= s->d.S) return OTFLM_ERR_VALUE;
    }
    // stable order by stream: each stream's requests contiguous, array order kept
    std::vector<uint32_t> order((size_t)n);
    for (int64_t i = 0; i < n; i++) order[i] = (uint32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return sid_h[a] < sid_h[b]; });
    std::vector<uint32_t> sc(n), cc(n);
    std::vector<int32_t> ww(n);
    std::vector<StreamRange> ranges;
    for (int64_t i = 0; i < n; i++) {
        sc[i] = (uint32_t)sid_h[order[i]]; cc[i] = c_h[order[i]]; ww[i] = w_h[order[i]];
        if (i == 0 || sc[i] != sc[i - 1]) ranges.push_back(StreamRange{sc[i], (uint32_t)i, (uint32_t)i, 0});
        ranges.back().re = (uint32_t)i + 1;
    }
    OtflmPlan *p = s->scratch;
    if (!p || p->R_max < (uint32_t)n || p->n_utt < ranges.size()) {
        if (p) otflm_plan_destroy(p);
        p = new OtflmPlan();
        p->st = s;
        p->R_max = (uint32_t)std::max<int64_t>(n, 1024);
        p->n_utt = (uint32_t)std::max<size_t>(ranges.size(), (size_t)s->d.S);
        int rc = plan_alloc_workspace(p, p->R_max, 2);
        StreamRange *drg = nullptr;
        bool bad = rc != 0 || p->mem.alloc(&drg, p->n_utt) != cudaSuccess;
        if (bad) { p->mem.free_all(); delete p; s->scratch = nullptr; return OTFLM_ERR_NOMEM; }
        p->d.ranges = drg;
        s->scratch = p;
    }
    uint32_t *dsid, *dc, *dcn; int32_t *dw; double *dp; uint8_t *dh;
    CK(cudaMallocAsync(&dsid, n * 4, st)); CK(cudaMallocAsync(&dc, n * 4, st)); CK(cudaMallocAsync(&dw, n * 4, st));
    CK(cudaMallocAsync(&dp, n * 8, st)); CK(cudaMallocAsync(&dcn, n * 4, st)); CK(cudaMallocAsync(&dh, n, st));
    CK(cudaMemcpyAsync(dsid, sc.data(), n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dc, cc.data(), n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dw, ww.data(), n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)p->d.ranges, ranges.data(), ranges.size() * sizeof(StreamRange), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(p->d.lvl, 0, 2 * sizeof(LevelCtr), st));
    const uint32_t R = (uint32_t)n;
    k_probe_batch<<<cdiv(R, 256), 256, 0, st>>>(p->d, s->d, R, dc, dw, dsid);
    CKL();
    const RowSpec rs{&p->d.lvl[0].n_prim, &p->d.lvl[0], nullptr, s->d.arena_used, p->d.pr_dig, s->d.arena_rows};
    int rc = enqueue_stage2(p, m, s->d, R, precision, rs, st);
    if (rc) return rc;
    k_assign<1><<<(unsigned)ranges.size(), ASSIGN_T, 0, st>>>(p->d, s->d, 0, 0, 0.0, dp, dcn, dh);
    CKL();
    if (s->lfu && s->d.lfu_log) {   // capacity-bounded cache: the policy's hit flags
        std::vector<uint32_t> hb((size_t)s->d.S, LFU_NIL);
        for (const StreamRange &r : ranges) hb[r.stream] = r.rb;
        uint32_t *dhb;
        CK(cudaMallocAsync(&dhb, hb.size() * 4, st));
        CK(cudaMemcpyAsync(dhb, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice, st));
        k_lfu_replay<<<cdiv(s->d.S, 64), 64, 0, st>>>(s->d, s->lfu->d, dh, dhb);
        CKL();
        CK(cudaFreeAsync(dhb, st));
    }
    std::vector<double> pp(n);
    std::vector<uint32_t> cn(n);
    std::vector<uint8_t> hh(n);
    CK(cudaMemcpyAsync(pp.data(), dp, n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cn.data(), dcn, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hh.data(), dh, n, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(dsid, st)); CK(cudaFreeAsync(dc, st)); CK(cudaFreeAsync(dw, st));
    CK(cudaFreeAsync(dp, st)); CK(cudaFreeAsync(dcn, st)); CK(cudaFreeAsync(dh, st));
    unsigned int he = 0;
    CK(cudaMemcpyAsync(&he, s->d.err, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (he & OTF_E_PATH) {
        CK(cudaMemset(s->d.err, 0, 4));
        g_detail = "context index not in table";
        return OTFLM_ERR_UNKNOWN_INDEX;
    }
    rc = check_err(s, st);
    if (rc) return rc;
    for (int64_t i = 0; i < n; i++) { p_h[order[i]] = pp[i]; cn_h[order[i]] = cn[i]; hit_h[order[i]] = hh[i]; }
    return OTFLM_OK;
}

// ==========================================================================
extern "C" const char *otflm_error_string(int32_t code) {
    switch (code) {
    case OTFLM_OK: return "ok";
    case OTFLM_ERR_VALUE: return "ValueError";
    case OTFLM_ERR_UNKNOWN_INDEX: return "UnknownIndexError";
    case OTFLM_ERR_TABLE_FULL: return "TableFullError";
    case OTFLM_ERR_NO_PATH: return "no complete path through the lattice";
    case OTFLM_ERR_KEY: return "word missing from unigram table";
    case OTFLM_ERR_NOMEM: return "out of device memory";
    case OTFLM_ERR_CYCLE: return "lattice contains a cycle";
    case OTFLM_ERR_PACK: return "PackOverflowError";
    case OTFLM_ERR_CUDA: return "CUDA error";
    case OTFLM_ERR_HASH: return "context digest collision";
    }
    return "unknown error";
}

extern "C" const char *otflm_last_error_detail(void) { return g_detail.c_str(); }

// ==========================================================================
// two-pass rescoring (uses the launchers above)
// ==========================================================================
#include "twopass.cuh"

// ==========================================================================
// container-level table operations (tables.cuh)
// ==========================================================================
#include "tables.cuh"

template <typename T>
static int to_dev(T **d, const T *h, int64_t n, cudaStream_t st) {
    CK(cudaMallocAsync(d, (size_t)std::max<int64_t>(n, 1) * sizeof(T), st));
    if (h && n) CK(cudaMemcpyAsync(*d, h, (size_t)n * sizeof(T), cudaMemcpyHostToDevice, st));
    return OTFLM_OK;
}

extern "C" int otflm_streams_encode(OtflmStreams *s, int32_t sid, int64_t n, const float *hidden_h,
                                    const uint32_t *hist_h, const int32_t *hist_len_h, uint32_t *idx_h,
                                    void *stream) {
    if (!s || sid < 0 || sid >= s->d.S || n < 0) return OTFLM_ERR_VALUE;
    if (n == 0) return OTFLM_OK;
    for (int64_t i = 0; i < n; i++)
        if (hist_len_h[i] < 0 || hist_len_h[i] > s->d.order) { g_detail = "context history longer than table maxent order"; return OTFLM_ERR_VALUE; }
    cudaStream_t st = (cudaStream_t)stream;
    float *dh; uint32_t *dhist, *didx; int32_t *dlen;
    int rc = to_dev(&dh, hidden_h, n * s->d.H, st);
    if (!rc) rc = to_dev(&dhist, hist_h, n * s->d.order, st);
    if (!rc) rc = to_dev(&dlen, hist_len_h, n, st);
    if (!rc) rc = to_dev(&didx, (const uint32_t *)nullptr, n, st);
    if (rc) return rc;
    CK(cudaMemsetAsync(didx, 0, (size_t)n * 4, st));
    k_table_encode<<<1, 1, 0, st>>>(s->d, (uint32_t)sid, (uint32_t)n, dh, dhist, dlen, didx);
    CKL();
    CK(cudaMemcpyAsync(idx_h, didx, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(dh, st)); CK(cudaFreeAsync(dhist, st)); CK(cudaFreeAsync(dlen, st)); CK(cudaFreeAsync(didx, st));
    return check_err(s, st);
}

static int cache_direct_ok(const OtflmStreams *s, int32_t sid, int64_t n) {
    if (!s || sid < 0 || sid >= s->d.S || n < 0) return OTFLM_ERR_VALUE;
    if (s->lfu && s->d.lfu_log) {
        g_detail = "direct get/put on a capacity-bounded device cache is not supported (use rnnlm_prob)";
        return OTFLM_ERR_VALUE;
    }
    return OTFLM_OK;
}

extern "C" int otflm_streams_cache_get(OtflmStreams *s, int32_t sid, int64_t n, const uint32_t *c_h,
                                       const int32_t *w_h, uint8_t *found_h, double *p_h, uint32_t *cn_h,
                                       void *stream) {
    int rc = cache_direct_ok(s, sid, n);
    if (rc || n == 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *dc, *dcn; int32_t *dw; uint8_t *df; double *dp;
    rc = to_dev(&dc, c_h, n, st);
    if (!rc) rc = to_dev(&dw, w_h, n, st);
    if (!rc) rc = to_dev(&df, (const uint8_t *)nullptr, n, st);
    if (!rc) rc = to_dev(&dp, (const double *)nullptr, n, st);
    if (!rc) rc = to_dev(&dcn, (const uint32_t *)nullptr, n, st);
    if (rc) return rc;
    k_cache_get<<<1, 1, 0, st>>>(s->d, (uint32_t)sid, (uint32_t)n, dc, dw, df, dp, dcn);
    CKL();
    CK(cudaMemcpyAsync(found_h, df, (size_t)n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(p_h, dp, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cn_h, dcn, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(dc, st)); CK(cudaFreeAsync(dw, st)); CK(cudaFreeAsync(df, st));
    CK(cudaFreeAsync(dp, st)); CK(cudaFreeAsync(dcn, st));
    return check_err(s, st);
}

extern "C" int otflm_streams_cache_put(OtflmStreams *s, int32_t sid, int64_t n, const uint32_t *c_h,
                                       const int32_t *w_h, const double *p_h, const uint32_t *cn_h,
                                       void *stream) {
    int rc = cache_direct_ok(s, sid, n);
    if (rc || n == 0) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *dc, *dcn; int32_t *dw; double *dp;
    rc = to_dev(&dc, c_h, n, st);
    if (!rc) rc = to_dev(&dw, w_h, n, st);
    if (!rc) rc = to_dev(&dp, p_h, n, st);
    if (!rc) rc = to_dev(&dcn, cn_h, n, st);
    if (rc) return rc;
    k_cache_put<<<1, 1, 0, st>>>(s->d, (uint32_t)sid, (uint32_t)n, dc, dw, dp, dcn);
    CKL();
    CK(cudaFreeAsync(dc, st)); CK(cudaFreeAsync(dw, st)); CK(cudaFreeAsync(dp, st)); CK(cudaFreeAsync(dcn, st));
    return check_err(s, st);
}

// RescoreCache.roll_stats / clear (cache.py:156-158, :136-140) on one stream;
// with a capacity bound also the policy: roll moves the window's evictions
// into the cumulative count, clear empties the LFU structure (the window's
// counters stay, as in the reference)
__global__ void k_stream_stats_op(DevStreams S, uint32_t s, int op, DevLfu L, int bounded) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned long long *st = S.stats + (size_t)s * 8;
    if (op == 0) {
        st[3] += st[0]; st[4] += st[1]; st[5] += st[2]; st[0] = st[1] = st[2] = 0;
        if (bounded) { unsigned long long *ev = L.ev + (size_t)s * 2; ev[1] += ev[0]; ev[0] = 0; }
    } else {
        st[6] = 0;                                     // entries after clear
        if (bounded) {
            uint32_t *sc = L.sc + (size_t)s * 8;
            sc[0] = LFU_NIL; sc[1] = 0; sc[2] = 0; sc[3] = LFU_NIL; sc[4] = 0; sc[5] = LFU_NIL;
        }
    }
}

static int stats_op_ok(const OtflmStreams *s, int32_t sid) {
    if (!s || sid < 0 || sid >= s->d.S) return OTFLM_ERR_VALUE;
    return OTFLM_OK;
}

extern "C" int otflm_streams_roll_stats(OtflmStreams *s, int32_t sid, void *stream) {
    int rc = stats_op_ok(s, sid);
    if (rc) return rc;
    const bool bounded = s->lfu && s->d.lfu_log;
    k_stream_stats_op<<<1, 1, 0, (cudaStream_t)stream>>>(s->d, (uint32_t)sid, 0, bounded ? s->lfu->d : DevLfu{},
                                                         bounded ? 1 : 0);
    CKL();
    return OTFLM_OK;
}

extern "C" int otflm_streams_cache_clear(OtflmStreams *s, int32_t sid, void *stream) {
    int rc = stats_op_ok(s, sid);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t o = (size_t)sid * s->d.kc_cap, n = s->d.kc_cap;
    CK(cudaMemsetAsync(s->d.kc_key + o, 0, n * 8, st));
    CK(cudaMemsetAsync(s->d.kc_claim + o, 0xFF, n * 4, st));
    CK(cudaMemsetAsync(s->d.kc_cnext + o, 0xFF, n * 4, st));
    const bool bounded = s->lfu && s->d.lfu_log;
    if (bounded) CK(cudaMemsetAsync(s->lfu->d.kc_lfu + o, 0xFF, n * 4, st));
    k_stream_stats_op<<<1, 1, 0, st>>>(s->d, (uint32_t)sid, 1, bounded ? s->lfu->d : DevLfu{}, bounded ? 1 : 0);
    CKL();
    return OTFLM_OK;
}

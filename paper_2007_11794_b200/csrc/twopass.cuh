// twopass.cuh -- two-pass rescoring, included at the
// end of capi.cu (it reuses the HS / recurrent-update launchers there).
//
//  * nbest (decoder.py:180-230): exact best-first search over the first-pass
//    weights with the backward-Viterbi completion as heuristic.  The search is
//    a sequential priority-queue walk, so it runs on the host in C++ (one
//    thread per utterance); it only touches the lattice, never the RNNLM.
//  * rescore_twopass (decoder.py:243-274): every hypothesis of every n-best
//    list is scored word by word by the RNNLM from the zero context.  The
//    context after a word prefix is a pure function of the prefix, so the
//    hypotheses are merged into a prefix trie (per list) and the device
//    scores each trie node once, level by level over all lists together:
//        HS + MaxEnt   lp[t]  = word_logprob(h[parent], hist[parent], w[t])
//        update        h[t]   = sigmoid(U[w[t]] + W h[parent])   (internal nodes only)
//        post          S[t]   = S[parent] + term(lp[t], ngram(ctx[parent], w[t]))
//    S[t] is the reference's running sum `lm += term` along the prefix, in
//    the same order, so a hypothesis' LM score is S[leaf].  Leaves need no
//    recurrent update (the reference advances past the last word but never
//    uses the result).
//
// Node numbering: node 0 = root (zero context, row 0); level d holds the
// nodes at depth d+1 of all lists, internal nodes (with children) first, so
// the level's internal nodes own consecutive hidden-state rows.

#include <atomic>
#include <thread>
#include <unordered_map>

// ==========================================================================
// n-best (host)
// ==========================================================================
namespace nb {

struct Ent { double key; uint64_t counter; int32_t done, node; double g; int64_t path; };
struct EntGreater {
    bool operator()(const Ent &a, const Ent &b) const {   // min-heap on (key, counter)
        if (a.key != b.key) return a.key > b.key;
        return a.counter > b.counter;
    }
};

// CPython >= 3.12 sum() over floats from int 0: first item exact, then
// Neumaier-compensated summation, compensation added at the end.
static double pysum(const double *x, const int32_t *idx, int32_t n) {
    if (n == 0) return 0.0;
    double f = 0.0 + x[idx[0]], c = 0.0;
    for (int32_t i = 1; i < n; i++) {
        const double v = x[idx[i]], t = f + v;
        if (std::fabs(f) >= std::fabs(v)) c += (f - t) + v;
        else c += (v - t) + f;
        f = t;
    }
    if (c != 0.0 && std::isfinite(c)) f += c;
    return f;
}

static uint64_t words_hash(const int32_t *w, int32_t n) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)n;
    for (int32_t i = 0; i < n; i++) {
        h = (h ^ (uint32_t)w[i]) * 0xff51afd7ed558ccdull;
        h ^= h >> 33;
    }
    return h;
}

struct List {
    std::vector<int32_t> len, arcs;
    std::vector<double> scores;   // [n, 3] combined, acoustic, lm
    int status = OTFLM_OK;
};

// Per-thread search state, reused across utterances: the heap and path links
// reach ~10^5-10^6 entries at n = 1000, and regrowing them per utterance
// serialises the threads on page faults.
struct Work {
    std::vector<Ent> heap;
    std::vector<std::pair<int32_t, int64_t>> links;     // (arc, parent link)
    std::unordered_map<uint64_t, std::vector<std::pair<int64_t, int32_t>>> seen;   // hash -> (offset, len)
    std::vector<int32_t> seen_words, tmp, tmpw, out_off, out_arc, indeg, order;
    std::vector<uint8_t> is_final;
    std::vector<double> comp;
};

// one utterance of the batch; node ids 0..N-1, arcs [a0, a1) of the batch arrays
static int search(const OtflmLatticeBatch *L, int u, int32_t n, double lmw, List *out, Work &W) {
    const int32_t N = L->n_nodes[u];
    const int64_t a0 = L->arc_off[u], a1 = L->arc_off[u + 1];
    const int32_t A = (int32_t)(a1 - a0);
    const int32_t *src = L->arc_src + a0, *dst = L->arc_dst + a0, *word = L->arc_word + a0;
    const double *ac = L->arc_ac + a0, *slm = L->arc_slm + a0;
    std::vector<int32_t> &out_off = W.out_off, &out_arc = W.out_arc, &indeg = W.indeg, &order = W.order;
    out_off.assign(N + 1, 0); out_arc.resize(A); indeg.assign(N, 0); order.clear();
    for (int32_t a = 0; a < A; a++) {
        if (src[a] < 0 || src[a] >= N || dst[a] < 0 || dst[a] >= N) return OTFLM_ERR_VALUE;
        out_off[src[a] + 1]++; indeg[dst[a]]++;
    }
    for (int32_t v = 0; v < N; v++) out_off[v + 1] += out_off[v];
    {
        std::vector<int32_t> fill(out_off.begin(), out_off.end() - 1);
        for (int32_t a = 0; a < A; a++) out_arc[fill[src[a]]++] = a;     // arc-id order per node
    }
    // Kahn order, smallest ready id first (lattice.py:68-82)
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> ready;
    for (int32_t v = 0; v < N; v++) if (indeg[v] == 0) ready.push(v);
    order.reserve(N);
    while (!ready.empty()) {
        const int32_t v = ready.top(); ready.pop();
        order.push_back(v);
        for (int32_t e = out_off[v]; e < out_off[v + 1]; e++)
            if (--indeg[dst[out_arc[e]]] == 0) ready.push(dst[out_arc[e]]);
    }
    if ((int32_t)order.size() != N) return OTFLM_ERR_CYCLE;
    std::vector<uint8_t> &is_final = W.is_final;
    is_final.assign(N, 0);
    for (int64_t f = L->final_off[u]; f < L->final_off[u + 1]; f++) is_final[L->finals[f]] = 1;
    // backward Viterbi completion (decoder.py:191-198)
    std::vector<double> &comp = W.comp;
    comp.resize(N);
    for (int32_t k = N - 1; k >= 0; k--) {
        const int32_t v = order[k];
        double best = is_final[v] ? 0.0 : -INFINITY;
        for (int32_t e = out_off[v]; e < out_off[v + 1]; e++) {
            const int32_t a = out_arc[e];
            const double cand = (ac[a] + lmw * slm[a]) + comp[dst[a]];
            if (cand > best) best = cand;
        }
        comp[v] = best;
    }
    const int32_t start = L->start[u];
    if (start < 0 || start >= N || comp[start] == -INFINITY) return OTFLM_ERR_NO_PATH;
    // best-first search (decoder.py:200-229); paths are parent-linked lists
    // (a binary heap on a reused vector; (key, counter) is a total order, so
    // the pop sequence is the reference's heapq sequence)
    std::vector<Ent> &heap = W.heap;
    auto &links = W.links;
    auto &seen = W.seen;
    std::vector<int32_t> &seen_words = W.seen_words, &tmp = W.tmp, &tmpw = W.tmpw;
    heap.clear(); links.clear(); seen.clear(); seen_words.clear();
    const EntGreater cmp;
    auto push = [&](const Ent &e) { heap.push_back(e); std::push_heap(heap.begin(), heap.end(), cmp); };
    uint64_t counter = 0;
    push(Ent{-comp[start], counter, 0, start, 0.0, -1});
    int32_t got = 0;
    while (!heap.empty() && got < n) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        const Ent cur = heap.back(); heap.pop_back();
        if (cur.done) {
            tmp.clear();
            for (int64_t p = cur.path; p >= 0; p = links[p].second) tmp.push_back(links[p].first);
            std::reverse(tmp.begin(), tmp.end());
            const int32_t Lp = (int32_t)tmp.size();
            tmpw.resize(Lp);
            for (int32_t i = 0; i < Lp; i++) tmpw[i] = word[tmp[i]];
            auto &bucket = seen[words_hash(tmpw.data(), Lp)];
            bool dup = false;
            for (auto &e : bucket)
                if (e.second == Lp && std::equal(tmpw.begin(), tmpw.end(), seen_words.begin() + e.first)) { dup = true; break; }
            if (dup) continue;
            bucket.push_back({(int64_t)seen_words.size(), Lp});
            seen_words.insert(seen_words.end(), tmpw.begin(), tmpw.end());
            out->len.push_back(Lp);
            out->arcs.insert(out->arcs.end(), tmp.begin(), tmp.end());
            out->scores.push_back(cur.g);
            out->scores.push_back(pysum(ac, tmp.data(), Lp));
            out->scores.push_back(pysum(slm, tmp.data(), Lp));
            got++;
            continue;
        }
        if (is_final[cur.node]) push(Ent{-cur.g, ++counter, 1, cur.node, cur.g, cur.path});
        for (int32_t e = out_off[cur.node]; e < out_off[cur.node + 1]; e++) {
            const int32_t a = out_arc[e];
            const double tail = comp[dst[a]];
            if (tail == -INFINITY) continue;
            const double g2 = cur.g + (ac[a] + lmw * slm[a]);
            links.push_back({a, cur.path});
            push(Ent{-(g2 + tail), ++counter, 0, dst[a], g2, (int64_t)links.size() - 1});
        }
    }
    return OTFLM_OK;
}

// f(item, thread index) over items 0..n-1, dynamic scheduling
template <class F>
static void parallel_for(int n, int threads, F f) {
    threads = std::max(1, std::min(threads, n));
    if (threads == 1) { for (int i = 0; i < n; i++) f(i, 0); return; }
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < threads; t++)
        th.emplace_back([&, t] { for (int i; (i = next.fetch_add(1)) < n;) f(i, t); });
    for (auto &x : th) x.join();
}

static int default_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? (int)hc : 4;
}

}  // namespace nb

struct OtflmNbest {
    std::vector<nb::List> lists;
};

extern "C" int otflm_nbest_create(const OtflmLatticeBatch *L, int32_t n, double lm_weight, int32_t n_threads,
                                  OtflmNbest **out) {
    *out = nullptr;
    if (n < 1) { g_detail = "n must be >= 1"; return OTFLM_ERR_VALUE; }
    auto *r = new OtflmNbest();
    r->lists.resize(L->n_utt);
    const int nt = std::max(1, std::min(n_threads > 0 ? n_threads : nb::default_threads(), L->n_utt));
    std::vector<nb::Work> work(nt);
    nb::parallel_for(L->n_utt, nt, [&](int u, int t) {
        r->lists[u].status = nb::search(L, u, n, lm_weight, &r->lists[u], work[t]);
    });
    *out = r;
    return OTFLM_OK;
}

extern "C" int otflm_nbest_sizes(const OtflmNbest *r, int32_t *n_hyp, int64_t *out2) {
    int64_t th = 0, ta = 0;
    for (size_t u = 0; u < r->lists.size(); u++) {
        n_hyp[u] = (int32_t)r->lists[u].len.size();
        th += (int64_t)r->lists[u].len.size();
        ta += (int64_t)r->lists[u].arcs.size();
    }
    out2[0] = th; out2[1] = ta;
    return OTFLM_OK;
}

extern "C" int otflm_nbest_copy(const OtflmNbest *r, int32_t *hyp_len, int32_t *arcs, double *scores,
                                int32_t *status) {
    int64_t h = 0, a = 0;
    for (size_t u = 0; u < r->lists.size(); u++) {
        const nb::List &l = r->lists[u];
        std::copy(l.len.begin(), l.len.end(), hyp_len + h);
        std::copy(l.scores.begin(), l.scores.end(), scores + 3 * h);
        std::copy(l.arcs.begin(), l.arcs.end(), arcs + a);
        h += (int64_t)l.len.size(); a += (int64_t)l.arcs.size();
        status[u] = l.status;
    }
    return OTFLM_OK;
}

extern "C" int otflm_nbest_destroy(OtflmNbest *r) {
    delete r;
    return OTFLM_OK;
}

// ==========================================================================
// two-pass scoring (device)
// ==========================================================================
struct DevTrie {
    int H, order, sw;               // sw = small-LM context width (order - 1, >= 1)
    const uint32_t *par_row, *par_node, *own_row;   // [N]
    const int32_t *word;            // [N]
    float *h;                       // [R, H]
    int32_t *hist, *hlen;           // [R, order], [R]
    int32_t *sctx, *slen;           // [R, sw], [R]
    double *lp, *S;                 // [N]
    const uint32_t *leaf;           // [n_hyp]
    const double *ac;               // [n_hyp]
    const int64_t *list_off;        // [n_lists + 1]
    double *lm_out, *comb_out;      // [n_hyp]
    int32_t *best;                  // [n_lists]
    unsigned int *err;
};

// _hybrid_logprob (decoder.py:233-240)
__device__ __forceinline__ double tp_hybrid(double lp_ng, double lp_rnn, double lam) {
    if (lam >= 1.0) return lp_ng;
    if (lam <= 0.0) return lp_rnn;
    const double hi = fmax(lp_ng, lp_rnn);
    return hi + log(lam * exp(lp_ng - hi) + (1.0 - lam) * exp(lp_rnn - hi));
}

__global__ void k_tp_root(DevTrie T) {
    if (threadIdx.x == 0) { T.hlen[0] = 0; T.slen[0] = 0; T.S[0] = 0.0; }
}

// per level [lo, hi): running LM sum + the internal nodes' histories
__global__ void k_tp_post(DevTrie T, DevNgram g, uint32_t lo, uint32_t hi, int mode, double lam) {
    const uint32_t t = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= hi) return;
    const uint32_t pr = T.par_row[t];
    const int32_t w = T.word[t];
    double term = T.lp[t];
    if (mode == 1) {
        uint32_t ctx[OTF_MAX_ORDER];
        const int L = T.slen[pr];
        for (int i = 0; i < L; i++) ctx[i] = (uint32_t)T.sctx[(size_t)pr * T.sw + i];
        double v;
        if (!ngram_logprob_dev(g, ctx, L, w, &v)) { atomicOr(T.err, OTF_E_KEY); v = 0.0; }
        term = tp_hybrid(v, term, lam);
    }
    T.S[t] = __dadd_rn(T.S[T.par_node[t]], term);
    const uint32_t r = T.own_row[t];
    if (r == 0xFFFFFFFFu) return;
    // history' = (history + (w,))[-order:]  (rnnlm.py:180-188); small-LM context likewise
    int L = T.hlen[pr];
    const int32_t *ph = T.hist + (size_t)pr * T.order;
    int32_t *oh = T.hist + (size_t)r * T.order;
    const int drop = L >= T.order ? 1 : 0;
    for (int i = drop; i < L; i++) oh[i - drop] = ph[i];
    oh[L - drop] = w;
    T.hlen[r] = L - drop + 1;
    L = T.slen[pr];
    const int32_t *ps = T.sctx + (size_t)pr * T.sw;
    int32_t *os = T.sctx + (size_t)r * T.sw;
    const int sd = L >= T.sw ? 1 : 0;
    for (int i = sd; i < L; i++) os[i - sd] = ps[i];
    os[L - sd] = w;
    T.slen[r] = L - sd + 1;
}

// per hypothesis: lm = S[leaf], combined = acoustic + lm_weight * lm; per
// list the first maximum (strict >, decoder.py:271-272)
__global__ void k_tp_final(DevTrie T, int n_lists, double lmw) {
    const int l = blockIdx.x;
    if (l >= n_lists) return;
    const int64_t h0 = T.list_off[l], h1 = T.list_off[l + 1];
    double bs = -INFINITY;
    int64_t bi = -1;
    for (int64_t j = h0 + threadIdx.x; j < h1; j += blockDim.x) {
        const double lm = T.S[T.leaf[j]];
        const double c = __dadd_rn(T.ac[j], __dmul_rn(lmw, lm));
        T.lm_out[j] = lm;
        T.comb_out[j] = c;
        if (bi < 0 || c > bs) { bs = c; bi = j; }
    }
    // (score desc, index asc) reduction = first maximum
    __shared__ double s_s[32];
    __shared__ long long s_i[32];
    for (int o = 16; o >= 1; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, (long long)bi, o);
        if (oi >= 0 && (bi < 0 || os > bs || (os == bs && oi < bi))) { bs = os; bi = oi; }
    }
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) { s_s[wid] = bs; s_i[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < nw; k++)
            if (s_i[k] >= 0 && (bi < 0 || s_s[k] > bs || (s_s[k] == bs && s_i[k] < bi))) { bs = s_s[k]; bi = s_i[k]; }
        T.best[l] = bi < 0 ? -1 : (int32_t)(bi - h0);
    }
}

struct OtflmTwopass {
    const OtflmModel *m;
    const OtflmNgram *g;
    Allocs mem;
    DevTrie d;
    int n_lists;
    int64_t n_hyp, n_nodes, n_rows, n_words;
    std::vector<uint32_t> level_off, level_int, level_row;   // [D+1], [D], [D]
    uint32_t *par_row_dev = nullptr, *par_node_dev = nullptr, *own_row_dev = nullptr, *leaf_dev = nullptr;
    int32_t *word_dev = nullptr;
    double *ac_dev = nullptr;
    int64_t *list_off_dev = nullptr;
    // captured level loop
    cudaGraphExec_t exec = nullptr;
    int g_mode = -1, g_prec = -1;
    double g_lam = 0, g_lmw = 0;
    int64_t g_launches = 0;
};

// Trie of every list's word sequences, numbered level-major across lists,
// internal nodes first within a level.
struct TrieBuild {
    struct Local { std::vector<uint32_t> par, depth; std::vector<int32_t> word; std::vector<uint8_t> internal;
                   std::vector<uint32_t> leaf; std::vector<uint32_t> gid; std::vector<uint32_t> rank; };
};

static int twopass_build(OtflmTwopass *p, const OtflmHypBatch *B, int n_threads, cudaStream_t s) {
    const int NL = B->n_lists;
    std::vector<TrieBuild::Local> loc(NL);
    std::atomic<int> bad{0};
    const int V = p->m->d.V;
    // 1. per-list tries (local ids, root = 0)
    nb::parallel_for(NL, n_threads, [&](int l, int) {
        TrieBuild::Local &T = loc[l];
        T.par.push_back(0); T.depth.push_back(0); T.word.push_back(-1); T.internal.push_back(0);
        std::unordered_map<uint64_t, uint32_t> child;
        const int64_t h0 = B->list_off[l], h1 = B->list_off[l + 1];
        int64_t total = 0;
        for (int64_t j = h0; j < h1; j++) total += B->hyp_off[j + 1] - B->hyp_off[j];
        child.reserve((size_t)total + 16);
        for (int64_t j = h0; j < h1; j++) {
            uint32_t cur = 0;
            for (int64_t i = B->hyp_off[j]; i < B->hyp_off[j + 1]; i++) {
                const int32_t w = B->words[i];
                if (w < 0 || w >= V) { bad = 1; break; }
                const uint64_t key = ((uint64_t)cur << 32) | (uint32_t)w;
                auto it = child.find(key);
                if (it == child.end()) {
                    const uint32_t id = (uint32_t)T.par.size();
                    child.emplace(key, id);
                    T.par.push_back(cur); T.depth.push_back(T.depth[cur] + 1); T.word.push_back(w);
                    T.internal.push_back(0);
                    T.internal[cur] = 1;
                    cur = id;
                } else {
                    cur = it->second;
                }
            }
            T.leaf.push_back(cur);
        }
    });
    if (bad) { g_detail = "word id out of range"; return OTFLM_ERR_VALUE; }
    // 2. per (list, depth) counts of internal / leaf nodes -> global offsets
    uint32_t D = 0;
    for (auto &T : loc) for (uint32_t d : T.depth) D = std::max(D, d);
    std::vector<std::vector<uint32_t>> cnt_int(NL, std::vector<uint32_t>(D + 1, 0)), cnt_leaf = cnt_int;
    nb::parallel_for(NL, n_threads, [&](int l, int) {
        TrieBuild::Local &T = loc[l];
        T.rank.resize(T.par.size());
        for (size_t v = 1; v < T.par.size(); v++)
            T.rank[v] = T.internal[v] ? cnt_int[l][T.depth[v]]++ : cnt_leaf[l][T.depth[v]]++;
    });
    p->level_off.assign(D + 1, 0); p->level_int.assign(D, 0); p->level_row.assign(D, 0);
    std::vector<std::vector<uint32_t>> base_int(NL, std::vector<uint32_t>(D + 1)), base_leaf = base_int;
    uint64_t node = 1, row = 1;
    for (uint32_t d = 1; d <= D; d++) {
        p->level_off[d - 1] = (uint32_t)node;
        p->level_row[d - 1] = (uint32_t)row;
        uint32_t ni = 0;
        for (int l = 0; l < NL; l++) { base_int[l][d] = (uint32_t)node; node += cnt_int[l][d]; ni += cnt_int[l][d]; }
        for (int l = 0; l < NL; l++) { base_leaf[l][d] = (uint32_t)node; node += cnt_leaf[l][d]; }
        p->level_int[d - 1] = ni;
        row += ni;
    }
    if (D > 0) p->level_off[D] = (uint32_t)node;
    if (node >= 0xFFFFFFFFull) { g_detail = "trie too large"; return OTFLM_ERR_VALUE; }
    p->n_nodes = (int64_t)node; p->n_rows = (int64_t)row;
    // 3. global arrays
    std::vector<uint32_t> par_row(node, 0), par_node(node, 0), own_row(node, 0xFFFFFFFFu), leaf(B->list_off[NL]);
    std::vector<int32_t> word(node, 0);
    nb::parallel_for(NL, n_threads, [&](int l, int) {
        TrieBuild::Local &T = loc[l];
        T.gid.assign(T.par.size(), 0);
        for (size_t v = 1; v < T.par.size(); v++) {   // parents precede children (creation order)
            const uint32_t d = T.depth[v];
            const uint32_t gid = (T.internal[v] ? base_int[l][d] : base_leaf[l][d]) + T.rank[v];
            T.gid[v] = gid;
            const uint32_t pg = T.gid[T.par[v]];
            par_node[gid] = pg;
            par_row[gid] = pg == 0 ? 0u : own_row[pg];
            word[gid] = T.word[v];
            if (T.internal[v]) own_row[gid] = p->level_row[d - 1] + (gid - p->level_off[d - 1]);
        }
        for (size_t j = 0; j < T.leaf.size(); j++) leaf[B->list_off[l] + j] = T.gid[T.leaf[j]];
    });
    p->n_words = B->hyp_off[B->list_off[NL]];
    // 4. upload
    int rc;
    if ((rc = upload(p->mem, &p->par_row_dev, par_row, s))) return rc;
    if ((rc = upload(p->mem, &p->par_node_dev, par_node, s))) return rc;
    if ((rc = upload(p->mem, &p->own_row_dev, own_row, s))) return rc;
    if ((rc = upload(p->mem, &p->word_dev, word, s))) return rc;
    if ((rc = upload(p->mem, &p->leaf_dev, leaf, s))) return rc;
    std::vector<double> ac(B->acoustic, B->acoustic + B->list_off[NL]);
    if ((rc = upload(p->mem, &p->ac_dev, ac, s))) return rc;
    std::vector<int64_t> lo(B->list_off, B->list_off + NL + 1);
    if ((rc = upload(p->mem, &p->list_off_dev, lo, s))) return rc;
    return OTFLM_OK;
}

extern "C" int otflm_twopass_create(const OtflmModel *m, const OtflmNgram *g, const OtflmHypBatch *B,
                                    int32_t n_threads, OtflmTwopass **out, void *stream) {
    *out = nullptr;
    if (B->n_lists < 1) { g_detail = "empty hypothesis batch"; return OTFLM_ERR_VALUE; }
    for (int l = 0; l < B->n_lists; l++)
        if (B->list_off[l + 1] <= B->list_off[l]) { g_detail = "empty hypothesis list"; return OTFLM_ERR_VALUE; }
    if (!m->d.U || !m->d.W || !m->d.NV || !m->d.ME) { g_detail = "incomplete model"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    auto *p = new OtflmTwopass();
    p->m = m; p->g = g;
    p->n_lists = B->n_lists;
    p->n_hyp = B->list_off[B->n_lists];
    int rc = twopass_build(p, B, n_threads > 0 ? n_threads : nb::default_threads(), s);
    if (rc) { p->mem.free_all(); delete p; return rc; }
    DevTrie &d = p->d;
    d.H = m->d.H; d.order = m->d.order;
    d.sw = std::max(1, g ? g->d.order - 1 : 1);
    d.par_row = p->par_row_dev; d.par_node = p->par_node_dev; d.own_row = p->own_row_dev;
    d.word = p->word_dev; d.leaf = p->leaf_dev; d.ac = p->ac_dev; d.list_off = p->list_off_dev;
    const size_t R = (size_t)p->n_rows, N = (size_t)p->n_nodes;
    bool bad = p->mem.alloc(&d.h, R * d.H) || p->mem.alloc(&d.hist, R * d.order) || p->mem.alloc(&d.hlen, R) ||
               p->mem.alloc(&d.sctx, R * d.sw) || p->mem.alloc(&d.slen, R) || p->mem.alloc(&d.lp, N) ||
               p->mem.alloc(&d.S, N) || p->mem.alloc(&d.lm_out, (size_t)p->n_hyp) ||
               p->mem.alloc(&d.comb_out, (size_t)p->n_hyp) || p->mem.alloc(&d.best, (size_t)p->n_lists) ||
               p->mem.alloc(&d.err, 1);
    if (bad) { p->mem.free_all(); delete p; g_detail = "cudaMalloc twopass"; return OTFLM_ERR_NOMEM; }
    if (cudaMemsetAsync(d.h, 0, (size_t)d.H * sizeof(float), s) != cudaSuccess ||   // row 0 = zero context
        cudaMemsetAsync(d.err, 0, sizeof(unsigned int), s) != cudaSuccess) {
        p->mem.free_all(); delete p; return OTFLM_ERR_CUDA;
    }
    *out = p;
    return OTFLM_OK;
}

extern "C" int otflm_twopass_info(const OtflmTwopass *p, int64_t *o) {
    o[0] = p->n_nodes - 1;                       // trie nodes (scored words)
    o[1] = (int64_t)p->level_int.size();         // levels
    o[2] = p->n_words;                           // words in the hypotheses
    o[3] = p->n_rows - 1;                        // recurrent updates (internal nodes)
    int64_t w = 0;
    for (size_t d = 0; d < p->level_int.size(); d++) w = std::max<int64_t>(w, p->level_off[d + 1] - p->level_off[d]);
    o[4] = w;                                    // widest level
    o[5] = p->n_hyp;
    return OTFLM_OK;
}

// One pass over the levels.  With s2 != s the recurrent-update chain runs on
// s2 (level d only needs level d-1's rows) and overlaps the HS + post of the
// same level on s; HS of level d+1 waits for the update of level d.
static int twopass_enqueue(OtflmTwopass *p, int mode, double lam, double lmw, int prec, cudaStream_t s,
                           cudaStream_t s2, std::vector<cudaEvent_t> *evs) {
    const DevModel &m = p->m->d;
    DevTrie &d = p->d;
    DevNgram g{};
    if (p->g) g = p->g->d;
    k_tp_root<<<1, 32, 0, s>>>(d);
    CKL();
    const bool fork = s2 != s;
    auto event = [&]() { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); evs->push_back(e); return e; };
    if (fork) { cudaEvent_t e = event(); CK(cudaEventRecord(e, s)); CK(cudaStreamWaitEvent(s2, e, 0)); }
    const bool exact = prec == OTFLM_PREC_FP64 || prec == OTFLM_PREC_EXACT;
    const RowSpec rs{nullptr, nullptr, nullptr, nullptr, nullptr, 0xFFFFFFFFu};
    for (size_t lv = 0; lv < p->level_int.size(); lv++) {
        const uint32_t lo = p->level_off[lv], hi = p->level_off[lv + 1], ni = p->level_int[lv];
        const int32_t *ctx = (const int32_t *)(p->par_row_dev + lo);
        int rc;
        {
            ProfScope ps(K_HS, s);
            if (m.H % 4 == 0 && m.H <= 1024) {
                rc = launch_ring_batch(m, hi - lo, ctx, d.h, d.hist, d.hlen, d.word + lo, d.lp + lo, exact, s);
            } else {
                rc = otflm_word_logprob_batch2(p->m, hi - lo, ctx, d.h, d.hist, d.hlen, d.word + lo, d.lp + lo,
                                               exact ? 1 : 0, s);
            }
            if (rc) return rc;
        }
        if (ni) {
            ProfScope ps(K_ADVANCE, s2);
            rc = launch_advance(m, prec, ni, rs, ctx, d.word + lo, d.h, d.h + (size_t)p->level_row[lv] * m.H,
                                0xFFFFFFFFu, s2);
            if (rc) return rc;
        }
        {
            ProfScope ps(K_MISC, s);
            k_tp_post<<<cdiv(hi - lo, 256), 256, 0, s>>>(d, g, lo, hi, mode, lam);
            CKL();
        }
        if (fork) {   // next level's HS reads the rows this level's update wrote
            cudaEvent_t e = event();
            CK(cudaEventRecord(e, s2));
            CK(cudaStreamWaitEvent(s, e, 0));
        }
    }
    k_tp_final<<<p->n_lists, 256, 0, s>>>(d, p->n_lists, lmw);
    CKL();
    return OTFLM_OK;
}

extern "C" int otflm_twopass_run(OtflmTwopass *p, int32_t mode, double interp_weight, double lm_weight,
                                 int32_t precision, int32_t use_graph, void *stream) {
    if (mode != 0 && mode != 1) { g_detail = "unknown two-pass mode"; return OTFLM_ERR_VALUE; }
    if (mode == 1 && !p->g) { g_detail = "hybrid mode needs the small LM"; return OTFLM_ERR_VALUE; }
    if (!prec_ok(precision)) return OTFLM_ERR_VALUE;
    if (precision != OTFLM_PREC_FP64 && precision != OTFLM_PREC_EXACT && p->m->d.H > 512) { g_detail = "tensor-core update needs H <= 512"; return OTFLM_ERR_VALUE; }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t l0 = g_launches;
    if (!use_graph) {
        int rc = twopass_enqueue(p, mode, interp_weight, lm_weight, precision, s, s, nullptr);
        g_last_launches = g_launches - l0;
        return rc;
    }
    if (!p->exec || p->g_mode != mode || p->g_prec != precision || p->g_lam != interp_weight ||
        p->g_lmw != lm_weight) {
        if (p->exec) { cudaGraphExecDestroy(p->exec); p->exec = nullptr; }
        // capture on private streams (the caller's may be the legacy default stream)
        cudaStream_t cs, cs2;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking));
        std::vector<cudaEvent_t> evs;
        cudaGraph_t graph;
        cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        int rc = e == cudaSuccess ? twopass_enqueue(p, mode, interp_weight, lm_weight, precision, cs, cs2, &evs)
                                  : OTFLM_ERR_CUDA;
        cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs); cudaStreamDestroy(cs2);
        for (cudaEvent_t x : evs) cudaEventDestroy(x);
        CK(e);
        if (rc) { if (e2 == cudaSuccess) cudaGraphDestroy(graph); return rc; }
        CK(e2);
        e = cudaGraphInstantiate(&p->exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(e);
        p->g_mode = mode; p->g_prec = precision; p->g_lam = interp_weight; p->g_lmw = lm_weight;
        p->g_launches = g_launches - l0;
    }
    CK(cudaGraphLaunch(p->exec, s));
    g_last_launches = p->g_launches;
    return OTFLM_OK;
}

extern "C" int otflm_twopass_fetch(OtflmTwopass *p, double *lm, double *combined, int32_t *best, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    unsigned int he = 0;
    CK(cudaMemcpyAsync(&he, p->d.err, 4, cudaMemcpyDeviceToHost, s));
    if (lm) CK(cudaMemcpyAsync(lm, p->d.lm_out, sizeof(double) * p->n_hyp, cudaMemcpyDeviceToHost, s));
    if (combined) CK(cudaMemcpyAsync(combined, p->d.comb_out, sizeof(double) * p->n_hyp, cudaMemcpyDeviceToHost, s));
    if (best) CK(cudaMemcpyAsync(best, p->d.best, sizeof(int32_t) * p->n_lists, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (he & OTF_E_KEY) {
        CK(cudaMemset(p->d.err, 0, 4));
        g_detail = "word missing from the small LM's unigram table";
        return OTFLM_ERR_KEY;
    }
    return OTFLM_OK;
}

extern "C" int otflm_twopass_destroy(OtflmTwopass *p) {
    if (!p) return OTFLM_OK;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    p->mem.free_all();
    delete p;
    return OTFLM_OK;
}

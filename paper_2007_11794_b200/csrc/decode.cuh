// decode.cuh -- frame-synchronous token passing with on-the-fly rescoring
// (reference decoder.py:114-173) over a batch of utterances, one stream each.
//
// A "level" is a maximal run of the reference's Kahn topological order
// (lattice.py:68-82) in which no node feeds another; for generator lattices
// a level is one frame.  Every node owns a fixed block of arrival slots (one
// per (in-arc, source rank)), so token recombination needs no atomics, and
// every (kept token, out-arc) request has a static slot whose index IS the
// reference's request order (topo node, rank, arc id).
//
// Per level, three graph stages (the middle two run as parallel branches):
//   k_expand   warp per node: recombine arrivals (max score, earliest arrival
//              wins ties = the strict '>' of decoder.py:145-149), rank by
//              (-score, ctx) (decoder.py:135), keep the beam, emit requests,
//              probe/claim the stream's (c, w) cache (cache.py:82-96) and
//              compact the requests that must run the model;
//   k_hs_prim  HS + MaxEnt score of every computed request (warp each) and the
//   || advance successor history; the recurrent update h' (tcgen05 GEMM or the
//              exact FP64 kernel) -- both add their part of the new context's
//              content digest;
//   k_assign   warp per stream: walks the stream's requests in reference
//              order, resolves cache claims (first occurrence = miss),
//              dedups successor contexts against the IndexTable
//              (context_table.py:74-86), numbers new ones len+1, fills the
//              cache, then computes the small-LM delta (decoder.py:99-102),
//              the new path score (decoder.py:144) and writes the arrival.
#pragma once
#include "common.cuh"
#include "hs.cuh"

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct StreamRange {         // requests of one stream inside one level
    uint32_t stream, rb, re, pad;
};

struct UttLevel {             // one (utterance, level) with requests (persistent schedule)
    uint32_t t;               // level index (arrival ordering key)
    uint32_t nb, ne;          // nodes: level_nodes[nb .. ne)
    uint32_t rb, re;          // level-global request range of the utterance
    uint32_t pad0, pad1, pad2;
};

struct DevPlan {
    // compiled lattice batch
    const NodeInfo *nodes;
    const uint32_t *level_nodes;
    const uint32_t *out_list;     // global arc ids grouped by source node, arc-id order
    const uint32_t *arc_slot;     // first arrival slot of the arc at its dst
    const int32_t *arc_word;
    const double *arc_ac, *arc_slm;
    Arrival *arr;
    uint8_t *slot_win;
    uint4 *tok;                   // general path: kept token by (node slot base + rank)
    // per utterance
    uint32_t n_utt;
    const uint32_t *utt_start_slot, *utt_stream, *final_off, *finals;
    // per level stream ranges
    const StreamRange *ranges;
    LevelCtr *lvl;
    // request workspace [R_max]
    uint32_t *rq_c, *rq_arc, *rq_parent, *rq_cslot, *rq_m, *rq_dslot;
    int32_t *rq_w;
    uint8_t *rq_state;
    double *rq_score;             // token score + arc acoustic (decoder.py:144 first sum)
    double *rq_slm, *rq_ps;       // arc small-LM score; ngram_logprob(small_context(c), w)
    // primaries [R_max]
    uint32_t *pr_req;
    int32_t *pr_inrow, *pr_w;
    double *pr_p;
    unsigned long long *pr_dig;   // content digest (sum of per-element hashes)
    // outputs
    int32_t *out_len, *out_arcs, *out_status;
    double *out_combined, *out_acoustic, *out_lm;
    long long *out_end_ctx, *out_expansions;
    int32_t max_path;
    uint32_t *cursor;             // arena cursor of a partitioned plan (concurrent groups)
    uint32_t arena_start, arena_end;   // partition [start, end), or start == OTF_UNSET
    unsigned long long *alg;      // profiling only: [0] sum P, [1] sum P*k, [2] HS queries
    // persistent schedule: per utterance its levels ul[ul_off[u] .. ul_off[u+1])
    // and the offset of its private request / primary workspace
    const UttLevel *ul;
    const uint32_t *ul_off, *rq_off;
    unsigned long long *phase_ns;  // profiling only: [expand, update, hs, assign, CTAs]
    uint8_t *kept;                // lattice-out only: [n_slots] arrival kept (expanded, or a final winner)
    // multi-CTA assign (k_asg_*): per request kind / table slot / aux, per chunk counts and offsets
    uint8_t *as_kind;
    uint32_t *as_slot, *as_aux, *ch_cnt, *ch_pre;
};

// content digest term of element i of a hidden row / word j of the history
// meta; the digest is their wrapping sum, so partial sums from different CTAs
// and kernels compose (context_table.py:64-72 serializes the same content)
__device__ __forceinline__ unsigned long long dig_h(int i, float x) { return otf_dig_h((uint32_t)i, x); }
__device__ __forceinline__ unsigned long long dig_meta(int j, uint32_t w) {
    return otf_hash64(((uint64_t)(0x10000 + j) << 32) ^ w);
}

// --------------------------------------------------------------------------
// recombination: arrival j beats i for the same ctx if higher score or equal
// score and earlier arrival (strict '>' keeps the first, decoder.py:147)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t arr_key(const Arrival &a) {
    return ((uint64_t)a.lvl << 32) | a.ridx;
}

__device__ __forceinline__ void recombine_node(const Arrival *__restrict__ arr, uint8_t *win,
                                               uint32_t base, uint32_t cap, int lane) {
    for (uint32_t i0 = 0; i0 < cap; i0 += 32) {
        uint32_t i = i0 + lane;
        Arrival ai;
        bool vi = false;
        if (i < cap) { ai = arr[base + i]; vi = ai.ctx != OTF_UNSET; }
        bool w = vi;
        for (uint32_t j0 = 0; j0 < cap; j0 += 32) {
            uint32_t j = j0 + lane;
            double sj = 0.0; uint32_t cj = OTF_UNSET; uint64_t kj = 0;
            if (j < cap) { Arrival aj = arr[base + j]; sj = aj.score; cj = aj.ctx; kj = arr_key(aj); }
            uint32_t lim = min(32u, cap - j0);
            for (uint32_t t = 0; t < lim; t++) {
                double s = __shfl_sync(0xffffffffu, sj, t);
                uint32_t c = __shfl_sync(0xffffffffu, cj, t);
                uint64_t k = __shfl_sync(0xffffffffu, kj, t);
                if (w && c == ai.ctx && (j0 + t) != i &&
                    (s > ai.score || (s == ai.score && k < arr_key(ai))))
                    w = false;
            }
        }
        if (i < cap) win[base + i] = w ? 1 : 0;
    }
    __syncwarp();
}

// probe/insert (c, w) in the stream's cache table; returns the slot and
// whether a value from an earlier level/call is present; a new or pending
// key is claimed by the lowest request index (atomicMin)
__device__ __forceinline__ uint32_t cache_probe(const DevStreams &S, uint32_t s, uint32_t c, int32_t w,
                                                uint32_t r, uint8_t *state) {
    const uint64_t kb = (uint64_t)s * S.kc_cap;
    const unsigned long long key = ((((unsigned long long)c) << 32) | (uint32_t)w) + 1ull;
    const uint32_t mask = S.kc_cap - 1;
    uint32_t sl = (uint32_t)otf_hash64(key) & mask;
    // one atomic per probe: a fresh key is inserted by the CAS itself (no
    // value can be present yet), an existing one is checked for a value
    for (uint32_t probes = 0;; probes++) {
        const unsigned long long prev = atomicCAS(&S.kc_key[kb + sl], 0ull, key);
        if (prev == 0ull) {
            atomicMin(&S.kc_claim[kb + sl], r);
            *state = RQ_PENDING;
            return sl;
        }
        if (prev == key) break;
        sl = (sl + 1) & mask;
        if (probes > S.kc_cap) { atomicOr(S.err, OTF_E_CACHE_FULL); *state = RQ_INVALID; return OTF_UNSET; }
    }
    if (ld_volatile_u32(&S.kc_cnext[kb + sl]) != OTF_UNSET) {
        *state = RQ_HIT;
    } else {
        atomicMin(&S.kc_claim[kb + sl], r);
        *state = RQ_PENDING;
    }
    return sl;
}

// warp-aggregated compaction of the requests that run the model this level
// (all lanes of the warp call it)
__device__ __forceinline__ void compact_primary(DevPlan &P, const DevStreams &S, uint32_t *n_prim, bool need,
                                                uint32_t r, uint32_t c, int32_t w, uint32_t s,
                                                uint32_t crow = OTF_UNSET) {
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(n_prim, (uint32_t)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (need) {
        const uint32_t m = base + __popc(bal & ((1u << lane) - 1u));
        P.rq_m[r] = m;
        P.pr_req[m] = r;
        P.pr_w[m] = w;
        P.pr_inrow[m] = (int32_t)(crow != OTF_UNSET ? crow : S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + c]);
        P.pr_dig[m] = 0ull;
    }
}

__device__ __forceinline__ bool ng_get(const uint64_t *tag, const int32_t *words, const double *val,
                                       uint32_t cap, int width, const int32_t *key, int len,
                                       double *out) {
    const uint64_t h = otf_tuple_hash(key, len);
    uint32_t s = (uint32_t)(h >> 7) & (cap - 1);
    for (uint32_t probes = 0; probes <= cap; probes++) {
        uint64_t t = tag[s];
        if (t == 0) return false;
        if (t == h) {
            const int32_t *wk = words + (size_t)s * width;
            if (wk[0] == len) {
                bool eq = true;
                for (int i = 0; i < len; i++) eq &= wk[1 + i] == key[i];
                if (eq) { *out = val[s]; return true; }
            }
        }
        s = (s + 1) & (cap - 1);
    }
    return false;
}

// ngram_logprob(small_context(history), w) (ngram.py:161-179, decoder.py:73-80)
__device__ __forceinline__ bool ngram_logprob_dev(const DevNgram &g, const uint32_t *hist, int L,
                                                  int w, double *out) {
    int32_t ctx[OTF_MAX_ORDER + 1];
    const int need = g.order - 1;
    int n = 0;
    for (int i = L; i < need; i++) ctx[n++] = g.bos;
    for (int i = 0; i < L; i++) ctx[n++] = (int32_t)hist[i];
    int keep = g.order > 1 ? g.order - 1 : 0;
    if (keep > n) keep = n;
    const int32_t *c = ctx + (n - keep);
    int32_t buf[OTF_MAX_ORDER + 1];
    const int width = g.order + 1;
    for (int depth = 0; depth <= keep; depth++) {
        int sl = keep - depth;
        for (int i = 0; i < sl; i++) buf[i] = c[depth + i];
        buf[sl] = w;
        double v;
        if (ng_get(g.p_tag, g.p_words, g.p_val, g.p_cap, width, buf, sl + 1, &v)) {
            for (int sh = depth - 1; sh >= 0; sh--) {
                double b;
                if (!ng_get(g.b_tag, g.b_words, g.b_val, g.b_cap, width, c + sh, keep - sh, &b)) b = 0.0;
                v = __dadd_rn(b, v);
            }
            *out = v;
            return true;
        }
    }
    return false;
}

// --------------------------------------------------------------------------
// stage 1: expand one level (warp per node)
// --------------------------------------------------------------------------
// Fast path: a node's arrivals fit one warp (cap <= 32, e.g. 24 at beam 8 /
// breadth 3): arrivals live in registers, recombination and ranking are
// shuffle sweeps, the kept tokens go to a per-warp shared table by rank, and
// the (rank, arc) requests are spread over lanes so their cache probes and
// small-LM lookups overlap.  Larger nodes (wide beams) take the general path
// through the slot_win scratch.
// One warp expands one node.  Request slots are nd.req_base + r_shift + j
// (r_shift = 0: level-global indices; the persistent stream kernel passes
// -rb so indices are local to its utterance's workspace).  s_* are this
// warp's 32-entry token / arc tables in shared memory.
__device__ __forceinline__ void expand_node(DevPlan &P, const DevStreams &S, const DevNgram &g,
                                            const NodeInfo &nd, long long beam, uint32_t lvl, int64_t r_shift,
                                            uint32_t *n_prim, uint32_t *s_ctx, uint32_t *s_slot, double *s_score,
                                            uint32_t *s_arc, int lane, bool defer_ps = false) {
    const uint32_t outdeg = nd.out_e - nd.out_b;
    const uint32_t rq0 = (uint32_t)((int64_t)nd.req_base + r_shift);
    if (nd.cap == 0 || outdeg == 0) {
        for (uint32_t r = lane; r < nd.keep * outdeg; r += 32) P.rq_state[rq0 + r] = RQ_INVALID;
        return;
    }
    // out-arcs of the node (arc-id order), staged once
    for (uint32_t q = lane; q < outdeg && q < 32; q += 32) s_arc[q] = P.out_list[nd.out_b + q];
    uint32_t n_kept = 0;
    if (nd.cap <= 32) {
        Arrival ai;
        bool vi = false;
        if ((uint32_t)lane < nd.cap) { ai = P.arr[nd.slot_base + lane]; vi = ai.ctx != OTF_UNSET; }
        const double si = vi ? ai.score : 0.0;
        const uint32_t ci = vi ? ai.ctx : OTF_UNSET;
        const uint64_t ki = vi ? arr_key(ai) : 0;
        bool win = vi;
        for (uint32_t t = 0; t < nd.cap; t++) {
            const double st = __shfl_sync(0xffffffffu, si, t);
            const uint32_t ct = __shfl_sync(0xffffffffu, ci, t);
            const uint64_t kt = __shfl_sync(0xffffffffu, ki, t);
            if (win && ct == ci && t != (uint32_t)lane && (st > si || (st == si && kt < ki))) win = false;
        }
        const unsigned wb = __ballot_sync(0xffffffffu, win);
        uint32_t rank = 0;
        for (uint32_t t = 0; t < nd.cap; t++) {
            const double st = __shfl_sync(0xffffffffu, si, t);
            const uint32_t ct = __shfl_sync(0xffffffffu, ci, t);
            if (win && ((wb >> t) & 1u) && (st > si || (st == si && ct < ci))) rank++;
        }
        n_kept = (uint32_t)min((long long)__popc(wb), beam);
        if (win && rank < n_kept) {
            s_ctx[rank] = ci;
            s_score[rank] = si;
            s_slot[rank] = nd.slot_base + lane;
            if (P.kept) P.kept[nd.slot_base + lane] = 1;
        }
    } else {
        // general path: O(cap^2 / 32) sweeps through the slot_win scratch;
        // kept tokens are written to P.tok by rank
        recombine_node(P.arr, P.slot_win, nd.slot_base, nd.cap, lane);
        uint32_t n_win = 0;
        for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
            uint32_t i = i0 + lane;
            n_win += __popc(__ballot_sync(0xffffffffu, i < nd.cap && P.slot_win[nd.slot_base + i]));
        }
        n_kept = (uint32_t)min((long long)n_win, beam);
        for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool wi = i < nd.cap && P.slot_win[nd.slot_base + i];
            Arrival ai;
            if (wi) ai = P.arr[nd.slot_base + i];
            uint32_t rank = 0;
            for (uint32_t j0 = 0; j0 < nd.cap; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool wj = j < nd.cap && P.slot_win[nd.slot_base + j];
                double sj = 0.0; uint32_t cj = 0;
                if (wj) { const Arrival aj = P.arr[nd.slot_base + j]; sj = aj.score; cj = aj.ctx; }
                const unsigned bal = __ballot_sync(0xffffffffu, wj);
                const uint32_t lim = min(32u, nd.cap - j0);
                for (uint32_t t = 0; t < lim; t++) {
                    const double st = __shfl_sync(0xffffffffu, sj, t);
                    const uint32_t ct = __shfl_sync(0xffffffffu, cj, t);
                    if (wi && ((bal >> t) & 1u) && (st > ai.score || (st == ai.score && ct < ai.ctx))) rank++;
                }
            }
            if (wi && rank < n_kept) {
                const unsigned long long sb = (unsigned long long)__double_as_longlong(ai.score);
                P.tok[nd.slot_base + rank] = make_uint4(ai.ctx, nd.slot_base + i, (uint32_t)sb, (uint32_t)(sb >> 32));
                if (P.kept) P.kept[nd.slot_base + i] = 1;
            }
        }
        __threadfence_block();
    }
    __syncwarp();
    const bool fast = nd.cap <= 32;   // token table by rank is in shared memory
    // one lane per (rank, arc) request; the trip count is uniform per warp
    for (uint32_t j0 = 0; j0 < n_kept * outdeg; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool emit = j < n_kept * outdeg;
        uint32_t r = 0, c = 0, s_tok = 0, crow = OTF_UNSET;
        int32_t w = 0;
        double sc = 0.0;
        uint8_t st = RQ_INVALID;
        if (emit) {
            const uint32_t rank = j / outdeg, q = j - rank * outdeg;
            if (fast) {
                c = s_ctx[rank]; sc = s_score[rank]; s_tok = s_slot[rank];
            } else {
                const uint4 tk = P.tok[nd.slot_base + rank];
                c = tk.x; s_tok = tk.y;
                sc = __longlong_as_double((long long)(((unsigned long long)tk.w << 32) | tk.z));
            }
            const uint32_t a = (outdeg <= 32) ? s_arc[q] : P.out_list[nd.out_b + q];
            r = rq0 + j;
            w = P.arc_word[a];
            crow = S.ctx_row[(uint64_t)nd.stream * (S.max_ctx + 1) + c];   // in flight during the probe
            st = RQ_NOCACHE;
            uint32_t cslot = OTF_UNSET;
            if (S.enabled) cslot = cache_probe(S, nd.stream, c, w, r, &st);
            // small-LM score of the same transition from the context's
            // stored history (decoder.py:99-100), independent of the model
            double ps = 0.0;
            if (!defer_ps) {
                const uint32_t crow = S.ctx_row[(uint64_t)nd.stream * (S.max_ctx + 1) + c];
                const uint32_t *meta = S.arena_meta + (size_t)crow * OTF_META;
                if (!ngram_logprob_dev(g, meta + 1, (int)meta[0], w, &ps)) { atomicOr(S.err, OTF_E_KEY); ps = 0.0; }
            }
            P.rq_c[r] = c;
            P.rq_w[r] = w;
            P.rq_arc[r] = a;
            P.rq_parent[r] = s_tok;
            P.rq_score[r] = __dadd_rn(sc, P.arc_ac[a]);
            P.rq_slm[r] = P.arc_slm[a];
            P.rq_ps[r] = ps;
            P.rq_dslot[r] = P.arc_slot[a] + rank;
            P.rq_m[r] = OTF_UNSET;
            P.rq_cslot[r] = cslot;
            P.rq_state[r] = st;
        }
        compact_primary(P, S, n_prim, emit && (st == RQ_PENDING || st == RQ_NOCACHE), r, c, w, nd.stream, crow);
    }
    for (uint32_t r = n_kept * outdeg + lane; r < nd.keep * outdeg; r += 32)
        P.rq_state[rq0 + r] = RQ_INVALID;
}

// Small-LM scores of requests [0, nreq) of one stream (decoder.py:99-100),
// when expand_node ran with defer_ps: thread per request over `nthr` threads
// starting at thread `t0` (they only feed assign, so they can run alongside
// the recurrent update and HS).
__device__ __forceinline__ void small_lm_scores(DevPlan &P, const DevStreams &S, const DevNgram &g, uint32_t s,
                                                uint32_t nreq, int t, int nthr) {
    for (uint32_t r = (uint32_t)t; r < nreq; r += (uint32_t)nthr) {
        if (P.rq_state[r] == RQ_INVALID) continue;
        const uint32_t c = P.rq_c[r];
        const int32_t w = P.rq_w[r];
        const uint32_t crow = S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + c];
        const uint32_t *meta = S.arena_meta + (size_t)crow * OTF_META;
        double ps;
        if (!ngram_logprob_dev(g, meta + 1, (int)meta[0], w, &ps)) { atomicOr(S.err, OTF_E_KEY); ps = 0.0; }
        P.rq_ps[r] = ps;
    }
}

constexpr int EXP_WARPS = 8;
// Nodes with big_min < cap <= EXPB_MAX arrival slots (big beams / wide
// lattices; big_min = EXPB_MIN unless a test lowers it) are expanded by
// k_expand_big, a CTA per node; k_expand skips them when it runs beside it
// and takes every node otherwise.
constexpr uint32_t EXPB_MIN = 64, EXPB_MAX = 2048;
constexpr int EXPB_T = 512;

__global__ void __launch_bounds__(256) k_expand(DevPlan P, DevStreams S, DevNgram g, uint32_t node_begin,
                                                uint32_t n_nodes, long long beam, uint32_t lvl,
                                                uint32_t big_min = 0xFFFFFFFFu) {
    __shared__ uint32_t s_ctx[EXP_WARPS][32], s_slot[EXP_WARPS][32];
    __shared__ double s_score[EXP_WARPS][32];
    __shared__ uint32_t s_arc[EXP_WARPS][32];
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * EXP_WARPS + wib;
    if (gw >= n_nodes) return;
    const NodeInfo nd = P.nodes[P.level_nodes[node_begin + gw]];
    if (nd.cap > big_min && nd.cap <= EXPB_MAX) return;           // k_expand_big's node
    expand_node(P, S, g, nd, beam, lvl, 0, &P.lvl[lvl].n_prim, s_ctx[wib], s_slot[wib], s_score[wib], s_arc[wib],
                threadIdx.x & 31);
}

// One node with many arrival slots per CTA (decoder.py:131-149): the same
// recombination (per context the best score, ties to the earliest arrival),
// the same beam ranking (score desc, ctx asc) and the same request emission as
// expand_node, but O(cap) for the recombination (a shared-memory hash of the
// contexts: atomicMax of the order-preserving score bits, then atomicMin of
// the arrival key among the tied) and the ranking spread over the CTA.
// Dynamic shared memory: expb_smem(cap_max).
__host__ __device__ constexpr uint32_t expb_hash_slots(uint32_t cap) {
    uint32_t h = 64;
    while (h < 2 * cap) h <<= 1;
    return h;
}
__host__ __device__ constexpr size_t expb_smem(uint32_t cap) {
    return (size_t)cap * 56 + (size_t)expb_hash_slots(cap) * 20 + 64;
}
__device__ __forceinline__ unsigned long long ord_score(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x == 0.0 ? 0.0 : x);   // -0 == +0
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(EXPB_T) k_expand_big(DevPlan P, DevStreams S, DevNgram g, uint32_t node_begin,
                                                       long long beam, uint32_t lvl, uint32_t cap_max, uint32_t big_min) {
    extern __shared__ __align__(16) uint8_t smem_eb[];
    __shared__ uint32_t s_arc[32], s_nwin;
    const NodeInfo nd = P.nodes[P.level_nodes[node_begin + blockIdx.x]];
    if (nd.cap <= big_min || nd.cap > EXPB_MAX) return;           // k_expand's node
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t C = cap_max, HB = expb_hash_slots(cap_max), cap = nd.cap;
    double *a_sc = reinterpret_cast<double *>(smem_eb);
    unsigned long long *a_key = reinterpret_cast<unsigned long long *>(a_sc + C);
    double *w_sc = reinterpret_cast<double *>(a_key + C);
    double *t_sc = w_sc + C;
    unsigned long long *h_best = reinterpret_cast<unsigned long long *>(t_sc + C);
    unsigned long long *h_kmin = h_best + HB;
    uint32_t *a_ct = reinterpret_cast<uint32_t *>(h_kmin + HB);
    uint32_t *a_hs = a_ct + C;
    uint32_t *w_ct = a_hs + C, *w_i = w_ct + C, *t_ct = w_i + C, *t_slot = t_ct + C;
    uint32_t *h_ctx = t_slot + C;
    const uint32_t outdeg = nd.out_e - nd.out_b;
    const uint32_t rq0 = nd.req_base;
    if (outdeg == 0) return;
    for (uint32_t i = tid; i < HB; i += EXPB_T) { h_ctx[i] = OTF_UNSET; h_best[i] = 0ull; h_kmin[i] = ~0ull; }
    if (tid < 32 && (uint32_t)tid < outdeg) s_arc[tid] = P.out_list[nd.out_b + tid];
    if (tid == 0) s_nwin = 0;
    __syncthreads();
    // arrivals -> shared memory; per context the best (score, then key) through the hash
    for (uint32_t i = tid; i < cap; i += EXPB_T) {
        const Arrival a = P.arr[nd.slot_base + i];
        a_sc[i] = a.score; a_ct[i] = a.ctx; a_key[i] = arr_key(a);
        uint32_t hs = OTF_UNSET;
        if (a.ctx != OTF_UNSET) {
            hs = (a.ctx * 0x9E3779B1u) & (HB - 1);
            for (;;) {
                const uint32_t prev = atomicCAS(&h_ctx[hs], OTF_UNSET, a.ctx);
                if (prev == OTF_UNSET || prev == a.ctx) break;
                hs = (hs + 1) & (HB - 1);
            }
            atomicMax(&h_best[hs], ord_score(a.score));
        }
        a_hs[i] = hs;
    }
    __syncthreads();
    for (uint32_t i = tid; i < cap; i += EXPB_T)
        if (a_hs[i] != OTF_UNSET && ord_score(a_sc[i]) == h_best[a_hs[i]]) atomicMin(&h_kmin[a_hs[i]], a_key[i]);
    __syncthreads();
    // winners (one per context) into a list; their order there is irrelevant
    for (uint32_t i = tid; i < cap; i += EXPB_T) {
        const uint32_t hs = a_hs[i];
        if (hs != OTF_UNSET && ord_score(a_sc[i]) == h_best[hs] && a_key[i] == h_kmin[hs]) {
            const uint32_t k = atomicAdd(&s_nwin, 1u);
            w_sc[k] = a_sc[i]; w_ct[k] = a_ct[i]; w_i[k] = i;
        }
    }
    __syncthreads();
    const uint32_t n_win = s_nwin;
    const uint32_t n_kept = (uint32_t)min((long long)n_win, beam);
    // rank = winners ahead in (score desc, ctx asc) -- contexts are distinct
    // among winners, so the order is total: a bitonic sort of the winner list
    // (padded to a power of two with -inf) puts winner of rank r at position r
    uint32_t N = 2;
    while (N < n_win) N <<= 1;
    for (uint32_t i = n_win + tid; i < N; i += EXPB_T) { w_sc[i] = -__longlong_as_double(0x7FF0000000000000LL); w_ct[i] = OTF_UNSET; w_i[i] = 0u; }
    __syncthreads();
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = tid; i < N; i += EXPB_T) {
                const uint32_t l = i ^ j;
                if (l <= i) continue;
                const double si = w_sc[i], sl = w_sc[l];
                const uint32_t ci = w_ct[i], cl = w_ct[l];
                const bool l_first = sl > si || (sl == si && cl < ci);      // l ranks ahead of i
                const bool i_first = si > sl || (si == sl && ci < cl);
                if ((i & k) == 0 ? l_first : i_first) {
                    w_sc[i] = sl; w_sc[l] = si; w_ct[i] = cl; w_ct[l] = ci;
                    const uint32_t t2 = w_i[i]; w_i[i] = w_i[l]; w_i[l] = t2;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t r = tid; r < n_kept; r += EXPB_T) {
        t_sc[r] = w_sc[r]; t_ct[r] = w_ct[r]; t_slot[r] = nd.slot_base + w_i[r];
        if (P.kept) P.kept[nd.slot_base + w_i[r]] = 1;
    }
    __syncthreads();
    // one thread per (rank, arc) request, as expand_node
    const uint32_t nreq = n_kept * outdeg;
    for (uint32_t j0 = 0; j0 < nreq; j0 += EXPB_T) {
        const uint32_t j = j0 + tid;
        const bool emit = j < nreq;
        uint32_t r = 0, c = 0, crow = OTF_UNSET;
        int32_t w = 0;
        uint8_t st = RQ_INVALID;
        if (emit) {
            const uint32_t rank = j / outdeg, q = j - rank * outdeg;
            c = t_ct[rank];
            const uint32_t a = (outdeg <= 32) ? s_arc[q] : P.out_list[nd.out_b + q];
            r = rq0 + j;
            w = P.arc_word[a];
            crow = S.ctx_row[(uint64_t)nd.stream * (S.max_ctx + 1) + c];
            st = RQ_NOCACHE;
            uint32_t cslot = OTF_UNSET;
            if (S.enabled) cslot = cache_probe(S, nd.stream, c, w, r, &st);
            double ps = 0.0;
            {
                const uint32_t *meta = S.arena_meta + (size_t)crow * OTF_META;
                if (!ngram_logprob_dev(g, meta + 1, (int)meta[0], w, &ps)) { atomicOr(S.err, OTF_E_KEY); ps = 0.0; }
            }
            P.rq_c[r] = c;
            P.rq_w[r] = w;
            P.rq_arc[r] = a;
            P.rq_parent[r] = t_slot[rank];
            P.rq_score[r] = __dadd_rn(t_sc[rank], P.arc_ac[a]);
            P.rq_slm[r] = P.arc_slm[a];
            P.rq_ps[r] = ps;
            P.rq_dslot[r] = P.arc_slot[a] + rank;
            P.rq_m[r] = OTF_UNSET;
            P.rq_cslot[r] = cslot;
            P.rq_state[r] = st;
        }
        compact_primary(P, S, &P.lvl[lvl].n_prim, emit && (st == RQ_PENDING || st == RQ_NOCACHE), r, c, w,
                        nd.stream, crow);
    }
    for (uint32_t r = nreq + tid; r < nd.keep * outdeg; r += EXPB_T) P.rq_state[rq0 + r] = RQ_INVALID;
}

// --------------------------------------------------------------------------
// stage 2a: HS + MaxEnt score of the computed requests (warp per request),
// successor history (history + (w,))[-order:] (rnnlm.py:187) and its digest
// --------------------------------------------------------------------------
__device__ __forceinline__ void hs_prim_finish(DevModel &m, DevPlan &P, DevStreams &S, const RowSpec &rs,
                                               uint32_t base, uint32_t q, const uint32_t *meta, int L, int w,
                                               uint32_t P_len, double lp, int lane) {
    // new history: drop the oldest word once `order` are stored (rnnlm.py:187)
    const int nl = L + 1 > m.order ? m.order : L + 1;
    const int drop = L + 1 - nl;
    uint32_t v = 0;
    if (lane == 0) v = (uint32_t)nl;
    else if (lane < nl) v = meta[lane + drop];
    else if (lane == nl) v = (uint32_t)w;
    unsigned long long dg = lane < OTF_META ? dig_meta(lane, v) : 0ull;
    if (lane < OTF_META) S.arena_meta[(size_t)(base + q) * OTF_META + lane] = v;
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) dg += __shfl_xor_sync(0xffffffffu, dg, o);
    if (lane == 0) {
        atomicAdd(&P.pr_dig[q], dg);
        if (P.alg) {   // algorithmic-work counters for the roofline (profiling runs)
            const int km = m.order < L ? m.order : L;
            atomicAdd(&P.alg[0], (unsigned long long)P_len);
            atomicAdd(&P.alg[1], (unsigned long long)P_len * km);
            atomicAdd(&P.alg[2], 1ull);
        }
        P.pr_p[q] = lp;
    }
}

// generic path (H % 4 != 0): warp per request, registers
template <int VEC, int CPL>
__global__ void __launch_bounds__(256) k_hs_prim(DevModel m, DevPlan P, DevStreams S, RowSpec rs) {
    const uint32_t n = *rs.n_dev;
    const uint32_t base = row_base(rs);
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q == 0 && lane == 0) rs.cur->base = base;   // also written by the update kernel (same value)
    if ((uint64_t)base + n > rs.row_limit) {
        if (q == 0 && lane == 0) atomicOr(S.err, OTF_E_ARENA_FULL);
        return;
    }
    if (q >= n) return;
    const uint32_t row = (uint32_t)P.pr_inrow[q];
    const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
    const int L = (int)meta[0];
    const int w = P.pr_w[q];
    const uint32_t o0 = __ldg(m.path_off + w), o1 = __ldg(m.path_off + w + 1);
    const double lp = hs_logprob_warp<VEC, CPL>(m, S.arena_h + (size_t)row * m.H, meta + 1, L,
                                                m.path_code + o0, o1 - o0, lane);
    hs_prim_finish(m, P, S, rs, base, q, meta, L, w, o1 - o0, lp, lane);
}

// TMA ring path (H % 4 == 0): persistent warps stride over the requests
template <int CPL, bool EXACT, int ORD>
__global__ void __launch_bounds__(128) k_hs_prim_ring(DevModel m, DevPlan P, DevStreams S, RowSpec rs) {
    extern __shared__ __align__(128) uint8_t smem_ring[];
    const uint32_t n = *rs.n_dev;
    const uint32_t base = row_base(rs);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib;
    if (gw == 0 && lane == 0) rs.cur->base = base;
    if ((uint64_t)base + n > rs.row_limit) {
        if (gw == 0 && lane == 0) atomicOr(S.err, OTF_E_ARENA_FULL);
        return;
    }
    if (gw >= n) return;
    HsRing ring = ring_setup(smem_ring, wib, m.H, lane);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t q = gw; q < n; q += nw) {
        const uint32_t row = (uint32_t)P.pr_inrow[q];
        const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
        const int L = (int)meta[0];
        const int w = P.pr_w[q];
        const uint32_t o0 = __ldg(m.path_off + w), o1 = __ldg(m.path_off + w + 1);
        const double lp = hs_logprob_ring<CPL, EXACT, ORD>(m, ring, S.arena_h + (size_t)row * m.H, meta + 1, L,
                                                           m.path_code + o0, o1 - o0, lane);
        hs_prim_finish(m, P, S, rs, base, q, meta, L, w, o1 - o0, lp, lane);
    }
}

// --------------------------------------------------------------------------
// stage 3: per-stream ordered resolution + finish
// --------------------------------------------------------------------------
// full-content comparison of two arena rows (bit patterns of h, history
// meta) by one thread; 16-byte loads, 8 of them in flight per trip, from L2
// (rows written earlier in the same kernel by other warps or CTAs)
__device__ __forceinline__ bool rows_equal_lane(const DevStreams &S, uint32_t ra, uint32_t rb) {
    const float *a = S.arena_h + (size_t)ra * S.H, *b = S.arena_h + (size_t)rb * S.H;
    if ((S.H & 3) == 0) {
        const uint4 *a4 = reinterpret_cast<const uint4 *>(a), *b4 = reinterpret_cast<const uint4 *>(b);
        const int n4 = S.H >> 2;
        for (int i = 0; i < n4; i += 4) {
            uint4 x[4], y[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                x[k] = make_uint4(0u, 0u, 0u, 0u); y[k] = x[k];
                if (i + k < n4) { x[k] = __ldcg(a4 + i + k); y[k] = __ldcg(b4 + i + k); }
            }
            bool eq = true;
#pragma unroll
            for (int k = 0; k < 4; k++) eq &= x[k].x == y[k].x && x[k].y == y[k].y && x[k].z == y[k].z && x[k].w == y[k].w;
            if (!eq) return false;
        }
    } else {
        for (int i = 0; i < S.H; i++)
            if (__float_as_uint(__ldcg(a + i)) != __float_as_uint(__ldcg(b + i))) return false;
    }
    const uint4 *ma = reinterpret_cast<const uint4 *>(S.arena_meta + (size_t)ra * OTF_META);
    const uint4 *mb = reinterpret_cast<const uint4 *>(S.arena_meta + (size_t)rb * OTF_META);
    const uint4 p0 = __ldcg(ma), p1 = __ldcg(ma + 1), q0 = __ldcg(mb), q1 = __ldcg(mb + 1);
    return p0.x == q0.x && p0.y == q0.y && p0.z == q0.z && p0.w == q0.w &&
           p1.x == q1.x && p1.y == q1.y && p1.z == q1.z && p1.w == q1.w;
}

// MODE 0: decode (finish requests into arrival slots)
// MODE 1: Table-1 batch API (write p / c' / hit per request)
// One CTA per (level, stream) range, one thread per request (chunks of
// ASSIGN_T): the reference order is the thread order, so the ordered steps
// (cache claim = first occurrence, len+1 numbering of new contexts, dedup of
// equal contexts created in the same level) are block-wide scans.
constexpr int ASSIGN_T = 128;
struct AssignSmem {           // per-thread scratch of assign_range (NTH entries)
    unsigned long long *key;
    uint32_t *row, *cn, *wsum, *cnt;
    unsigned long long *hkey;   // [2 NTH] chunk dedup hash: content key ...
    uint32_t *htid, *ins;       // [2 NTH] ... -> first request (min thread); [NTH] table slot per first
};
// Requests [rg.rb, rg.re) of one stream in one level, NTH threads of the CTA
// (the reference order is the thread order inside each chunk of NTH).
template <int MODE, int NTH>
__device__ __forceinline__ void assign_range(DevPlan &P, const DevStreams &S, uint32_t lvl, const StreamRange &rg,
                                             const LevelCtr &lc, uint32_t limit, double lm_weight, double *out_p,
                                             uint32_t *out_cn, uint8_t *out_hit, const AssignSmem &sm,
                                             unsigned long long *tprof = nullptr) {
    // tprof (profiling runs, thread 0): device ns per section, summed
    unsigned long long tp0 = (tprof && threadIdx.x == 0) ? globaltimer_ns() : 0ull, tpa[6] = {0, 0, 0, 0, 0, 0};
#define AS_MARK(i) do { if (tprof && threadIdx.x == 0) { const unsigned long long t_ = globaltimer_ns(); tpa[i] += t_ - tp0; tp0 = t_; } } while (0)
    unsigned long long *s_key = sm.key;
    uint32_t *s_row = sm.row, *s_cn = sm.cn, *s_wsum = sm.wsum, *s_cnt = sm.cnt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if ((uint64_t)lc.base + lc.n_prim > limit) return;   // flagged by stage 2
    const uint32_t s = rg.stream;
    const uint64_t kb = (uint64_t)s * S.kc_cap, cb = (uint64_t)s * S.ct_cap;
    const uint32_t cmask = S.ct_cap - 1;
    uint32_t tlen = S.table_len[s];
    if (tid < 4) s_cnt[tid] = 0;
    bool full = false;
    const bool lfu_log = S.lfu_log != nullptr && S.enabled;     // uniform
    uint32_t logn = lfu_log ? S.lfu_logn[s] : 0u;
    for (uint32_t r0 = rg.rb; r0 < rg.re; r0 += NTH) {
        const uint32_t r = r0 + tid;
        const bool in = r < rg.re;
        const uint8_t st = in ? P.rq_state[r] : (uint8_t)RQ_INVALID;
        const bool valid = st != RQ_INVALID;
        const uint32_t cslot = (st == RQ_HIT || st == RQ_PENDING) ? P.rq_cslot[r] : OTF_UNSET;
        bool prim = st == RQ_NOCACHE;
        if (st == RQ_PENDING) prim = S.kc_claim[kb + cslot] == r;
        const uint32_t m = prim ? P.rq_m[r] : OTF_UNSET;
        // chunk-local dedup table and slot hand-over, cleared per chunk
        for (int i = tid; i < 2 * NTH; i += NTH) { sm.hkey[i] = 0ull; sm.htid[i] = 0xFFFFFFFFu; }
        sm.ins[tid] = OTF_UNSET;
        unsigned long long key = 0;
        uint32_t row = 0, cn = OTF_UNSET, ins_slot = OTF_UNSET;
        if (prim) {
            key = otf_hash64(P.pr_dig[m]) | 1ull;
            row = lc.base + m;
            // contexts of earlier levels / chunks; a new key is inserted right
            // away (the stream's table has one writer, this CTA) and numbered
            // below -- an entry whose index is still unset was inserted by this
            // chunk and is resolved by the chunk dedup
            uint32_t slot = (uint32_t)(key >> 20) & cmask;
            for (uint32_t probes = 0; probes <= S.ct_cap; probes++) {
                unsigned long long k = S.ct_key[cb + slot];
                if (k == 0ull) {
                    const unsigned long long prev = atomicCAS(&S.ct_key[cb + slot], 0ull, key);
                    if (prev == 0ull) { ins_slot = slot; break; }
                    k = prev;
                }
                if (k == key) {
                    const uint32_t ix = ld_volatile_u32(&S.ct_idx[cb + slot]);
                    if (ix == OTF_UNSET) break;                                  // in flight (this chunk)
                    if (rows_equal_lane(S, S.ct_row[cb + slot], row)) { cn = ix; break; }
                }
                slot = (slot + 1) & cmask;
            }
        }
        const bool novel = prim && cn == OTF_UNSET;
        s_key[tid] = novel ? key : 0ull;
        s_row[tid] = row;
        __syncthreads();
        AS_MARK(0);
        // equal contexts created by earlier requests of this chunk: the first
        // (lowest thread = request order) of each key through a shared hash
        uint32_t hslot = 0;
        if (novel) {
            hslot = (uint32_t)(key >> 7) & (2 * NTH - 1);
            for (int probes = 0; probes < 2 * NTH; probes++) {
                const unsigned long long prev = atomicCAS(&sm.hkey[hslot], 0ull, key);
                if (prev == 0ull || prev == key) { atomicMin(&sm.htid[hslot], (uint32_t)tid); break; }
                hslot = (hslot + 1) & (2 * NTH - 1);
            }
        }
        __syncthreads();
        int dup_of = -1;
        if (novel) {
            const int f = (int)sm.htid[hslot];
            if (f != tid) {
                if (rows_equal_lane(S, s_row[f], row)) dup_of = f;
                else atomicOr(S.err, OTF_E_HASH);
            }
            if (ins_slot != OTF_UNSET) sm.ins[dup_of >= 0 ? dup_of : tid] = ins_slot;   // slot to the first
        }
        const bool first = novel && dup_of < 0;
        // block-wide exclusive scan of `first` in thread (= request) order
        const unsigned fb = __ballot_sync(0xffffffffu, first);
        if (lane == 0) s_wsum[wid] = __popc(fb);
        __syncthreads();
        AS_MARK(1);
        uint32_t before = __popc(fb & ((1u << lane) - 1u)), total = 0;
        for (int w2 = 0; w2 < NTH / 32; w2++) {
            if (w2 < wid) before += s_wsum[w2];
            total += s_wsum[w2];
        }
        if (first) {
            const uint32_t idx = tlen + before + 1u;            // len + 1 (context_table.py:83-86)
            const uint32_t slot = sm.ins[tid];
            if (idx > S.max_ctx || slot == OTF_UNSET) {
                full = true;
                if (slot == OTF_UNSET) atomicOr(S.err, OTF_E_NOSLOT);
            } else {
                cn = idx;
                S.ct_idx[cb + slot] = idx;
                S.ct_row[cb + slot] = row;
                S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + idx] = row;
            }
        }
        tlen += total;
        s_cn[tid] = cn;
        __syncthreads();
        AS_MARK(2);
        if (dup_of >= 0) cn = s_cn[dup_of];
        double p = 0.0;
        if (prim) {
            p = P.pr_p[m];
            if (st == RQ_PENDING) { S.kc_p[kb + cslot] = p; S.kc_cnext[kb + cslot] = cn; }
        }
        __syncthreads();
        AS_MARK(3);
        if (valid && !prim) {   // hit: earlier level, or an earlier request of this level
            p = S.kc_p[kb + cslot];
            cn = ld_volatile_u32(&S.kc_cnext[kb + cslot]);
        }
        {
            const unsigned bv = __ballot_sync(0xffffffffu, valid), bp = __ballot_sync(0xffffffffu, prim);
            if (lane == 0) {
                atomicAdd(&s_cnt[0], __popc(bv));
                atomicAdd(&s_cnt[1], __popc(bp));
            }
        }
        if (valid) {
            if (MODE == 1) {
                out_p[r] = p; out_cn[r] = cn; out_hit[r] = prim ? 0 : 1;
            } else {
                // delta rounded to f32 (codec.py:57-59); score (decoder.py:144)
                const float delta = __double2float_rn(__dsub_rn(p, P.rq_ps[r]));
                const double ns = __dadd_rn(P.rq_score[r], __dmul_rn(lm_weight, __dadd_rn(P.rq_slm[r], (double)delta)));
                Arrival out;
                out.score = ns; out.ctx = cn; out.parent = P.rq_parent[r]; out.arc = P.rq_arc[r];
                out.lvl = lvl; out.ridx = r; out.pad = 0;
                P.arr[P.rq_dslot[r]] = out;
            }
        }
        if (lfu_log) {   // lookups of this chunk, in request order, for the LFU replay
            const unsigned bv = __ballot_sync(0xffffffffu, valid);
            __syncthreads();
            if (lane == 0) s_wsum[wid] = __popc(bv);
            __syncthreads();
            uint32_t before = __popc(bv & ((1u << lane) - 1u)), total = 0;
            for (int w2 = 0; w2 < NTH / 32; w2++) {
                if (w2 < wid) before += s_wsum[w2];
                total += s_wsum[w2];
            }
            if (valid) {
                const uint32_t pos = logn + before;
                if (pos < S.lfu_logcap) S.lfu_log[(size_t)s * S.lfu_logcap + pos] = cslot | (prim ? 0x80000000u : 0u);
                else atomicOr(S.err, OTF_E_CACHE_FULL);
            }
            logn += total;
        }
        __syncthreads();
        AS_MARK(4);
    }
    if (full) atomicOr(S.err, OTF_E_TABLE_FULL);
    if (lfu_log && tid == 0) S.lfu_logn[s] = logn;
    if (tprof && tid == 0) for (int i = 0; i < 5; i++) atomicAdd(&tprof[i], tpa[i]);
#undef AS_MARK
    if (tid == 0) {
        S.table_len[s] = tlen > S.max_ctx ? S.max_ctx : tlen;
        unsigned long long *stt = S.stats + (size_t)s * 8;
        const unsigned long long look = s_cnt[0], miss = s_cnt[1];
        stt[0] += look; stt[1] += look - miss; stt[2] += miss; stt[7] += look;
        if (S.enabled) stt[6] += miss;
    }
}

template <int MODE>
__global__ void __launch_bounds__(ASSIGN_T) k_assign(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                     double lm_weight, double *out_p, uint32_t *out_cn,
                                                     uint8_t *out_hit) {
    __shared__ unsigned long long s_key[ASSIGN_T], s_hkey[2 * ASSIGN_T];
    __shared__ uint32_t s_row[ASSIGN_T], s_cn[ASSIGN_T], s_wsum[ASSIGN_T / 32], s_htid[2 * ASSIGN_T], s_ins[ASSIGN_T];
    __shared__ uint32_t s_cnt[4];
    const LevelCtr lc = P.lvl[lvl];
    if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 0) *S.arena_used = lc.base + lc.n_prim;
    const uint32_t limit = P.arena_start == OTF_UNSET ? S.arena_rows : P.arena_end;
    const StreamRange rg = P.ranges[range_begin + blockIdx.x];
    assign_range<MODE, ASSIGN_T>(P, S, lvl, rg, lc, limit, lm_weight, out_p, out_cn, out_hit,
                                 AssignSmem{s_key, s_row, s_cn, s_wsum, s_cnt, s_hkey, s_htid, s_ins});
}

// --------------------------------------------------------------------------
// multi-CTA assign: the same ordered resolution as assign_range for streams
// whose level has many requests (big beams, wide lattices), spread over
// chunks of ASG_CH requests in six grid steps (grid = chunks x stream ranges):
//   probe   content-table probe / insert per computed request; a new key's
//           first request (lowest index = reference order) by atomicMin on
//           the key's slot (ct_first)
//   dedup   equal contexts created later in the level -> duplicates of that
//           first (full-row check); per-chunk count of new contexts
//   scan    per stream: chunk offsets = len + earlier chunks' new contexts
//   number  len + 1 numbering of the new contexts in request order
//           (context_table.py:83-86)
//   values  duplicates take their first's index; computed values into the
//           cache (cache.py:99-109); ct_first back to unset
//   arrive  hits read the cache (earlier level or an earlier claim of this
//           level), arrivals and counters as assign_range (MODE 0)
// Used when no capacity-bounded cache logs lookups (that log is ordered).
// --------------------------------------------------------------------------
constexpr int ASG_CH = 256;
constexpr uint32_t ASSIGN_BIG = 4096;      // a plan whose largest range exceeds this uses k_asg_*
enum : uint8_t { AK_NONE = 0, AK_OLD = 1, AK_FIRST = 2, AK_DUP = 3 };

struct AsgIdx {
    StreamRange rg;
    uint32_t r, ci;
    bool block_live, in;
};
__device__ __forceinline__ AsgIdx asg_idx(const DevPlan &P, uint32_t range_begin) {
    AsgIdx a;
    a.rg = P.ranges[range_begin + blockIdx.y];
    const uint32_t c0 = a.rg.rb + blockIdx.x * ASG_CH;
    a.block_live = c0 < a.rg.re;
    a.r = c0 + threadIdx.x;
    a.in = a.block_live && a.r < a.rg.re;
    a.ci = blockIdx.y * gridDim.x + blockIdx.x;
    return a;
}
__device__ __forceinline__ bool asg_prim(const DevPlan &P, const DevStreams &S, uint32_t s, uint32_t r,
                                         uint8_t *st_out, uint32_t *cslot_out) {
    const uint8_t st = P.rq_state[r];
    const uint32_t cslot = (st == RQ_HIT || st == RQ_PENDING) ? P.rq_cslot[r] : OTF_UNSET;
    bool prim = st == RQ_NOCACHE;
    if (st == RQ_PENDING) prim = S.kc_claim[(uint64_t)s * S.kc_cap + cslot] == r;
    *st_out = st; *cslot_out = cslot;
    return prim;
}

__global__ void __launch_bounds__(ASG_CH) k_asg_probe(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                      uint32_t limit) {
    const AsgIdx a = asg_idx(P, range_begin);
    const LevelCtr lc = P.lvl[lvl];
    if (!a.in || (uint64_t)lc.base + lc.n_prim > limit) return;
    const uint32_t s = a.rg.stream, r = a.r;
    const uint64_t cb = (uint64_t)s * S.ct_cap;
    const uint32_t cmask = S.ct_cap - 1;
    uint8_t st;
    uint32_t cslot;
    uint8_t kind = AK_NONE;
    uint32_t slot_out = OTF_UNSET, aux = OTF_UNSET;
    if (asg_prim(P, S, s, r, &st, &cslot)) {
        const uint32_t m = P.rq_m[r];
        const unsigned long long key = otf_hash64(P.pr_dig[m]) | 1ull;
        const uint32_t row = lc.base + m;
        kind = AK_FIRST;                                   // new unless found below
        uint32_t slot = (uint32_t)(key >> 20) & cmask;
        for (uint32_t probes = 0; probes <= S.ct_cap; probes++) {
            unsigned long long k = S.ct_key[cb + slot];
            if (k == 0ull) {
                const unsigned long long prev = atomicCAS(&S.ct_key[cb + slot], 0ull, key);
                if (prev == 0ull) { slot_out = slot; break; }
                k = prev;
            }
            if (k == key) {
                const uint32_t ix = ld_volatile_u32(&S.ct_idx[cb + slot]);
                if (ix == OTF_UNSET) { slot_out = slot; break; }         // created in this level
                if (rows_equal_lane(S, S.ct_row[cb + slot], row)) { kind = AK_OLD; aux = ix; break; }
            }
            slot = (slot + 1) & cmask;
        }
        if (kind == AK_FIRST && slot_out != OTF_UNSET) atomicMin(&S.ct_first[cb + slot_out], r);
    }
    P.as_kind[r] = kind;
    P.as_slot[r] = slot_out;
    P.as_aux[r] = aux;
}

__global__ void __launch_bounds__(ASG_CH) k_asg_dedup(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                      uint32_t limit) {
    const AsgIdx a = asg_idx(P, range_begin);
    const LevelCtr lc = P.lvl[lvl];
    if (!a.block_live || (uint64_t)lc.base + lc.n_prim > limit) return;
    bool first = false;
    if (a.in && P.as_kind[a.r] == AK_FIRST) {
        const uint32_t r = a.r, slot = P.as_slot[r];
        first = true;
        if (slot != OTF_UNSET) {
            const uint32_t f = S.ct_first[(uint64_t)a.rg.stream * S.ct_cap + slot];
            if (f != r) {
                if (rows_equal_lane(S, lc.base + P.rq_m[f], lc.base + P.rq_m[r])) {
                    P.as_kind[r] = AK_DUP; P.as_aux[r] = f; first = false;
                } else {
                    atomicOr(S.err, OTF_E_HASH);
                    P.as_slot[r] = OTF_UNSET;               // numbered without a slot -> NOSLOT below
                }
            }
        }
    }
    const int n = __syncthreads_count(first);
    if (threadIdx.x == 0) P.ch_cnt[a.ci] = (uint32_t)n;
}

__global__ void __launch_bounds__(32) k_asg_scan(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                 uint32_t nch, uint32_t limit) {
    const LevelCtr lc = P.lvl[lvl];
    if ((uint64_t)lc.base + lc.n_prim > limit) return;
    const StreamRange rg = P.ranges[range_begin + blockIdx.x];
    const uint32_t s = rg.stream, lane = threadIdx.x;
    const uint32_t n = (rg.re - rg.rb + ASG_CH - 1) / ASG_CH;
    uint32_t run = S.table_len[s];
    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t c = c0 + lane;
        uint32_t v = c < n ? P.ch_cnt[blockIdx.x * nch + c] : 0u, x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)lane >= o) x += y;
        }
        if (c < n) P.ch_pre[blockIdx.x * nch + c] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) S.table_len[s] = run > S.max_ctx ? S.max_ctx : run;
}

__global__ void __launch_bounds__(ASG_CH) k_asg_number(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                       uint32_t limit) {
    __shared__ uint32_t s_w[ASG_CH / 32];
    const AsgIdx a = asg_idx(P, range_begin);
    const LevelCtr lc = P.lvl[lvl];
    if (!a.block_live || (uint64_t)lc.base + lc.n_prim > limit) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool first = a.in && P.as_kind[a.r] == AK_FIRST;
    const unsigned b = __ballot_sync(0xffffffffu, first);
    if (lane == 0) s_w[wid] = __popc(b);
    __syncthreads();
    if (!first) return;
    uint32_t before = __popc(b & ((1u << lane) - 1u));
    for (int w2 = 0; w2 < wid; w2++) before += s_w[w2];
    const uint32_t idx = P.ch_pre[a.ci] + before + 1u;           // len + 1 (context_table.py:83-86)
    const uint32_t r = a.r, s = a.rg.stream, slot = P.as_slot[r], row = lc.base + P.rq_m[r];
    if (idx > S.max_ctx || slot == OTF_UNSET) {
        atomicOr(S.err, OTF_E_TABLE_FULL | (slot == OTF_UNSET ? OTF_E_NOSLOT : 0u));
        return;
    }
    const uint64_t cb = (uint64_t)s * S.ct_cap;
    S.ct_idx[cb + slot] = idx;
    S.ct_row[cb + slot] = row;
    S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + idx] = row;
    P.as_aux[r] = idx;
}

__global__ void __launch_bounds__(ASG_CH) k_asg_values(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                       uint32_t limit) {
    const AsgIdx a = asg_idx(P, range_begin);
    const LevelCtr lc = P.lvl[lvl];
    if (!a.in || (uint64_t)lc.base + lc.n_prim > limit) return;
    const uint32_t r = a.r, s = a.rg.stream;
    const uint8_t kind = P.as_kind[r];
    if (kind == AK_NONE) return;
    uint32_t cn = P.as_aux[r];
    if (kind == AK_DUP) { cn = P.as_aux[cn]; P.as_aux[r] = cn; }   // the first's index (OTF_UNSET if it failed)
    const uint32_t slot = P.as_slot[r];
    if (slot != OTF_UNSET) S.ct_first[(uint64_t)s * S.ct_cap + slot] = OTF_UNSET;
    if (P.rq_state[r] == RQ_PENDING) {
        const uint64_t k = (uint64_t)s * S.kc_cap + P.rq_cslot[r];
        S.kc_p[k] = P.pr_p[P.rq_m[r]];
        S.kc_cnext[k] = cn;
    }
}

__global__ void __launch_bounds__(ASG_CH) k_asg_arrive(DevPlan P, DevStreams S, uint32_t lvl, uint32_t range_begin,
                                                       uint32_t limit, double lm_weight) {
    const AsgIdx a = asg_idx(P, range_begin);
    const LevelCtr lc = P.lvl[lvl];
    if (!a.block_live || (uint64_t)lc.base + lc.n_prim > limit) return;
    const uint32_t r = a.r, s = a.rg.stream;
    bool valid = false, prim = false;
    if (a.in) {
        const uint8_t st = P.rq_state[r];
        valid = st != RQ_INVALID;
        prim = P.as_kind[r] != AK_NONE;
        if (valid) {
            double p;
            uint32_t cn;
            if (prim) { p = P.pr_p[P.rq_m[r]]; cn = P.as_aux[r]; }
            else {
                const uint64_t k = (uint64_t)s * S.kc_cap + P.rq_cslot[r];
                p = S.kc_p[k];
                cn = ld_volatile_u32(&S.kc_cnext[k]);
            }
            // delta rounded to f32 (codec.py:57-59); score (decoder.py:144)
            const float delta = __double2float_rn(__dsub_rn(p, P.rq_ps[r]));
            const double ns = __dadd_rn(P.rq_score[r], __dmul_rn(lm_weight, __dadd_rn(P.rq_slm[r], (double)delta)));
            Arrival out;
            out.score = ns; out.ctx = cn; out.parent = P.rq_parent[r]; out.arc = P.rq_arc[r];
            out.lvl = lvl; out.ridx = r; out.pad = 0;
            P.arr[P.rq_dslot[r]] = out;
        }
    }
    const int look = __syncthreads_count(valid), miss = __syncthreads_count(prim);
    if (threadIdx.x == 0 && look) {
        unsigned long long *stt = S.stats + (size_t)s * 8;
        atomicAdd(&stt[0], (unsigned long long)look);
        atomicAdd(&stt[1], (unsigned long long)(look - miss));
        atomicAdd(&stt[2], (unsigned long long)miss);
        atomicAdd(&stt[7], (unsigned long long)look);
        if (S.enabled) atomicAdd(&stt[6], (unsigned long long)miss);
    }
}

// --------------------------------------------------------------------------
// final: best token over sorted finals x sorted ctx (decoder.py:150-156),
// backtrace (decoder.py:157-162), score breakdown (decoder.py:163-169)
// --------------------------------------------------------------------------
__global__ void k_final(DevPlan P, DevStreams S, double lm_weight, int last_lvl) {
    const uint32_t u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (u == 0 && lane == 0 && last_lvl >= 0) {   // arena rows in use after the run
        const uint32_t end = P.lvl[last_lvl].base + P.lvl[last_lvl].n_prim;
        if (P.arena_start == OTF_UNSET) { if (end <= S.arena_rows) *S.arena_used = end; }
        else *P.cursor = end;
    }
    if (u >= P.n_utt) return;
    bool have = false;
    double best = 0.0;
    uint32_t best_ctx = 0, best_slot = OTF_UNSET;
    for (uint32_t f = P.final_off[u]; f < P.final_off[u + 1]; f++) {
        const NodeInfo nd = P.nodes[P.finals[f]];
        if (nd.cap == 0) continue;
        double bs = 0.0; uint32_t bc = OTF_UNSET, bslot = OTF_UNSET; bool bh = false;
        if (!P.kept) {
            // the node's best recombination winner is the lexicographic best
            // arrival by (score desc, ctx asc, arrival key asc): no O(cap^2)
            // recombination unless lattice-out wants every winner
            uint64_t bk = 0;
            for (uint32_t i = lane; i < nd.cap; i += 32) {
                const Arrival a = P.arr[nd.slot_base + i];
                if (a.ctx == OTF_UNSET) continue;
                const uint64_t k = arr_key(a);
                if (!bh || a.score > bs || (a.score == bs && (a.ctx < bc || (a.ctx == bc && k < bk)))) {
                    bh = true; bs = a.score; bc = a.ctx; bk = k; bslot = nd.slot_base + i;
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const double os = __shfl_xor_sync(0xffffffffu, bs, o);
                const uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
                const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
                const uint32_t osl = __shfl_xor_sync(0xffffffffu, bslot, o);
                const bool oh = __shfl_xor_sync(0xffffffffu, (int)bh, o);
                if (oh && (!bh || os > bs || (os == bs && (oc < bc || (oc == bc && ok < bk))))) {
                    bh = true; bs = os; bc = oc; bk = ok; bslot = osl;
                }
            }
            if (bh && (!have || bs > best)) { have = true; best = bs; best_ctx = bc; best_slot = bslot; }
            continue;
        }
        recombine_node(P.arr, P.slot_win, nd.slot_base, nd.cap, lane);
        for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
            uint32_t i = i0 + lane;
            if (i < nd.cap && P.slot_win[nd.slot_base + i]) {
                Arrival a = P.arr[nd.slot_base + i];
                if (P.kept) P.kept[nd.slot_base + i] = 1;     // lattice-out: every final winner
                if (!bh || a.score > bs || (a.score == bs && a.ctx < bc)) {
                    bh = true; bs = a.score; bc = a.ctx; bslot = nd.slot_base + i;
                }
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            double os = __shfl_xor_sync(0xffffffffu, bs, o);
            uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
            uint32_t osl = __shfl_xor_sync(0xffffffffu, bslot, o);
            bool oh = __shfl_xor_sync(0xffffffffu, (int)bh, o);
            if (oh && (!bh || os > bs || (os == bs && oc < bc))) { bh = true; bs = os; bc = oc; bslot = osl; }
        }
        if (bh && (!have || bs > best)) { have = true; best = bs; best_ctx = bc; best_slot = bslot; }
    }
    if (lane != 0) return;
    const uint32_t s = P.utt_stream[u];
    P.out_expansions[u] = (long long)S.stats[(size_t)s * 8 + 7];
    if (!have) { P.out_status[u] = -4; P.out_len[u] = 0; return; }
    int len = 0;
    for (uint32_t b = best_slot; P.arr[b].parent != OTF_UNSET; b = P.arr[b].parent) len++;
    P.out_len[u] = len;
    if (len > P.max_path) { P.out_status[u] = -6; return; }
    int32_t *oa = P.out_arcs + (size_t)u * P.max_path;
    int k = len - 1;
    for (uint32_t b = best_slot; P.arr[b].parent != OTF_UNSET; b = P.arr[b].parent) oa[k--] = (int32_t)P.arr[b].arc;
    double ac = 0.0;
    for (int i = 0; i < len; i++) ac = __dadd_rn(ac, P.arc_ac[oa[i]]);
    P.out_acoustic[u] = ac;
    P.out_combined[u] = best;
    P.out_lm[u] = lm_weight != 0.0 ? __ddiv_rn(__dsub_rn(best, ac), lm_weight) : 0.0;
    P.out_end_ctx[u] = best_ctx;
    P.out_status[u] = 0;
}

__global__ void k_run_begin(DevPlan P, DevStreams S) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < P.n_utt) {
        Arrival a;
        a.score = 0.0; a.ctx = 0; a.parent = OTF_UNSET; a.arc = OTF_UNSET; a.lvl = 0; a.ridx = 0; a.pad = 0;
        P.arr[P.utt_start_slot[t]] = a;
    }
    if (t < P.n_utt) S.stats[(size_t)P.utt_stream[t] * 8 + 7] = 0;
    if (t == 0 && P.arena_start != OTF_UNSET) *P.cursor = P.arena_start;
}


// --------------------------------------------------------------------------
// lattice-out: the RNNLM-rescored, beam-pruned state lattice of each
// utterance -- every kept arrival (a token that was expanded, or a final
// recombination winner) with its parent arrival, lattice arc and path score.
// One CTA per utterance compacts its slot range in slot order.
// --------------------------------------------------------------------------
struct LatRecord {           // 24 B
    double score;            // path score of the state (decoder.py:144 sums)
    uint32_t state, parent;  // slot - utterance slot base; parent state or OTF_UNSET (start)
    uint32_t arc;            // batch-global arc id (OTF_UNSET for the start state)
    uint32_t pad;
};

__global__ void k_lattice_out(DevPlan P, const uint32_t *utt_slot_off, LatRecord *out, long long *count) {
    const uint32_t u = blockIdx.x;
    if (u >= P.n_utt) return;
    const uint32_t lo = utt_slot_off[u], hi = utt_slot_off[u + 1];
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t s0 = lo; s0 < hi; s0 += blockDim.x) {
        const uint32_t sl = s0 + threadIdx.x;
        const bool k = sl < hi && P.kept[sl];
        const unsigned b = __ballot_sync(0xffffffffu, k);
        if (lane == 0) wsum[wid] = __popc(b);
        __syncthreads();
        uint32_t before = __popc(b & ((1u << lane) - 1u)), total = 0;
        for (int w = 0; w < nw; w++) { if (w < wid) before += wsum[w]; total += wsum[w]; }
        if (k) {
            const Arrival a = P.arr[sl];
            LatRecord r;
            r.score = a.score;
            r.state = sl - lo;
            r.parent = a.parent == OTF_UNSET ? OTF_UNSET : a.parent - lo;
            r.arc = a.arc;
            r.pad = 0;
            out[lo + base + before] = r;
        }
        __syncthreads();
        if (threadIdx.x == 0) base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) count[u] = base;
}

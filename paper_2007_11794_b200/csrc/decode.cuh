// decode.cuh -- frame-synchronous token passing with on-the-fly rescoring
// (reference decoder.py:114-173) over a batch of utterances, one stream each.
//
// A "level" is a maximal run of the reference's Kahn topological order
// (lattice.py:68-82) in which no node feeds another; for generator lattices
// a level is one frame.  Every node owns a fixed block of arrival slots (one
// per (in-arc, source rank)), so token recombination needs no atomics: the
// expand kernel recombines a node's arrivals (max score, earliest arrival on
// ties = the reference's strict '>' , decoder.py:145-149), ranks the
// survivors by (-score, ctx) (decoder.py:135) and emits one request per
// (kept token, out-arc) at a static slot whose index IS the reference's
// request order (topo node, rank, arc id).  That order is what the cache
// claim (first occurrence = miss) and the IndexTable's len+1 numbering
// (context_table.py:83-86) are resolved against, so hit/miss counts and
// context ids are identical to the sequential reference.
//
// Per level:  expand(+cache probe) -> scan primaries -> HS+MaxEnt (+history')
//             -> recurrent update -> content dedup -> scan novel -> resolve
//             -> finish (n-gram delta, score, arrival write).
#pragma once
#include "common.cuh"
#include "hs.cuh"

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
    // per utterance
    uint32_t n_utt;
    const uint32_t *utt_start_slot, *utt_stream, *final_off, *finals;
    // request workspace [R_max]
    uint32_t *rq_c, *rq_arc, *rq_parent, *rq_stream, *rq_cslot, *rq_m, *rq_dslot;
    int32_t *rq_w;
    uint8_t *rq_state;
    double *rq_score;
    // primary workspace [R_max]
    uint32_t *pr_req, *pr_stream, *pr_ctslot, *pr_found, *pr_E, *pr_cnext;
    int32_t *pr_inrow, *pr_w;
    double *pr_p;
    uint32_t *first_E;            // [S]
    uint32_t *counters;           // [0] n_prim, [1] n_novel, [2] arena_base
    unsigned long long *alg;      // run totals: [0] sum P, [1] sum P*k, [2] HS queries
    // outputs
    int32_t *out_len, *out_arcs, *out_status;
    double *out_combined, *out_acoustic, *out_lm;
    long long *out_end_ctx, *out_expansions;
    int32_t max_path;
};

// --------------------------------------------------------------------------
// decoupled look-back scan over a flag predicate (single pass, any n)
// status word: bits 63:62 = 0 none / 1 aggregate / 2 inclusive, 31:0 value
// --------------------------------------------------------------------------
#define SCAN_BLK 512
template <class FlagF, class OutF>
__device__ __forceinline__ void chained_scan(uint32_t n, unsigned long long *status,
                                             uint32_t *ticket, FlagF flagf, OutF outf,
                                             uint32_t *total_out) {
    __shared__ uint32_t s_bid, s_prefix, s_warp[SCAN_BLK / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t bid = s_bid;
    const uint32_t i = bid * SCAN_BLK + tid;
    const bool f = i < n ? flagf(i) : false;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const uint32_t lpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < SCAN_BLK / 32 ? s_warp[lane] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t block_total = __shfl_sync(0xffffffffu, incl, 31);
        if (lane < SCAN_BLK / 32) s_warp[lane] = incl - v;
        if (lane == 0) {
            uint32_t prefix = 0;
            if (bid == 0) {
                __threadfence();
                atomicExch(&status[0], (2ull << 62) | block_total);
            } else {
                atomicExch(&status[bid], (1ull << 62) | block_total);
                int j = (int)bid - 1;
                while (j >= 0) {
                    unsigned long long s = ld_volatile_u64(&status[j]);
                    unsigned fl = (unsigned)(s >> 62);
                    if (fl == 0) continue;
                    prefix += (uint32_t)s;
                    if (fl == 2) break;
                    j--;
                }
                __threadfence();
                atomicExch(&status[bid], (2ull << 62) | (uint64_t)(prefix + block_total));
            }
            s_prefix = prefix;
            if (bid == gridDim.x - 1 && total_out) *total_out = prefix + block_total;
        }
    }
    __syncthreads();
    if (i < n) outf(i, s_prefix + s_warp[wid] + lpre, f);
}

// --------------------------------------------------------------------------
// recombination helpers: arrival j beats i for the same ctx if higher score
// or equal score and earlier arrival (strict '>' keeps the first, decoder.py:147)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t arr_key(const Arrival &a) {
    return ((uint64_t)a.lvl << 32) | a.ridx;
}

// Returns, for the calling lane's slot i (or invalid), whether it is the
// recombined winner of its ctx; all lanes of the warp must call it.
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

// --------------------------------------------------------------------------
// kernel 1: expand one level (warp per node) + cache probe/claim per request
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_expand(DevPlan P, DevStreams S, uint32_t node_begin,
                                                uint32_t n_nodes, long long beam, uint32_t lvl) {
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= n_nodes) return;
    const NodeInfo nd = P.nodes[P.level_nodes[node_begin + gw]];
    const uint32_t outdeg = nd.out_e - nd.out_b;
    if (nd.cap == 0 || outdeg == 0) {
        for (uint32_t r = lane; r < nd.keep * outdeg; r += 32) {
            P.rq_w[nd.req_base + r] = -1;
            P.rq_state[nd.req_base + r] = RQ_INVALID;
        }
        return;
    }
    recombine_node(P.arr, P.slot_win, nd.slot_base, nd.cap, lane);
    uint32_t n_win = 0;
    for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
        uint32_t i = i0 + lane;
        bool wi = i < nd.cap && P.slot_win[nd.slot_base + i];
        n_win += __popc(__ballot_sync(0xffffffffu, wi));
    }
    const uint32_t n_kept = (uint32_t)min((long long)n_win, beam);
    const uint64_t kc_base = (uint64_t)nd.stream * S.kc_cap;
    for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
        uint32_t i = i0 + lane;
        bool wi = i < nd.cap && P.slot_win[nd.slot_base + i];
        uint32_t rank = 0;
        Arrival ai;
        if (wi) ai = P.arr[nd.slot_base + i];
        for (uint32_t j0 = 0; j0 < nd.cap; j0 += 32) {
            uint32_t j = j0 + lane;
            bool wj = j < nd.cap && P.slot_win[nd.slot_base + j];
            double sj = 0.0; uint32_t cj = 0;
            if (wj) { Arrival aj = P.arr[nd.slot_base + j]; sj = aj.score; cj = aj.ctx; }
            unsigned bal = __ballot_sync(0xffffffffu, wj);
            uint32_t lim = min(32u, nd.cap - j0);
            for (uint32_t t = 0; t < lim; t++) {
                double s = __shfl_sync(0xffffffffu, sj, t);
                uint32_t c = __shfl_sync(0xffffffffu, cj, t);
                if (wi && ((bal >> t) & 1u) && (s > ai.score || (s == ai.score && c < ai.ctx))) rank++;
            }
        }
        if (wi && rank < n_kept) {
            for (uint32_t q = 0; q < outdeg; q++) {
                const uint32_t a = P.out_list[nd.out_b + q];
                const uint32_t r = nd.req_base + rank * outdeg + q;
                const int32_t w = P.arc_word[a];
                P.rq_c[r] = ai.ctx;
                P.rq_w[r] = w;
                P.rq_arc[r] = a;
                P.rq_parent[r] = nd.slot_base + i;
                P.rq_score[r] = ai.score;
                P.rq_stream[r] = nd.stream;
                P.rq_dslot[r] = P.arc_slot[a] + rank;
                P.rq_m[r] = OTF_UNSET;
                uint8_t st = RQ_NOCACHE;
                uint32_t cslot = OTF_UNSET;
                if (S.enabled) {
                    const unsigned long long key =
                        ((((unsigned long long)ai.ctx) << 32) | (uint32_t)w) + 1ull;
                    const uint32_t mask = S.kc_cap - 1;
                    uint32_t s = (uint32_t)otf_hash64(key) & mask;
                    uint32_t probes = 0;
                    for (;;) {
                        unsigned long long k = S.kc_key[kc_base + s];
                        if (k == 0ull) {
                            unsigned long long prev = atomicCAS(&S.kc_key[kc_base + s], 0ull, key);
                            k = prev == 0ull ? key : prev;
                        }
                        if (k == key) break;
                        s = (s + 1) & mask;
                        if (++probes > S.kc_cap) { atomicOr(S.err, OTF_E_CACHE_FULL); s = OTF_UNSET; break; }
                    }
                    cslot = s;
                    if (s != OTF_UNSET) {
                        if (ld_volatile_u32(&S.kc_cnext[kc_base + s]) != OTF_UNSET) {
                            st = RQ_HIT;
                        } else {
                            atomicMin(&S.kc_claim[kc_base + s], r);
                            st = RQ_PENDING;
                        }
                    }
                }
                P.rq_cslot[r] = cslot;
                P.rq_state[r] = st;
            }
        }
    }
    // invalidate unused request slots of this node
    for (uint32_t r = n_kept * outdeg + lane; r < nd.keep * outdeg; r += 32) {
        P.rq_w[nd.req_base + r] = -1;
        P.rq_state[nd.req_base + r] = RQ_INVALID;
    }
}

// --------------------------------------------------------------------------
// kernel 2: primaries = requests that must run the model (cache miss, first
// claimant).  Ordered compaction keeps request order.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(SCAN_BLK) k_scan_prim(DevPlan P, DevStreams S, uint32_t n_req,
                                                        unsigned long long *status, uint32_t *ticket) {
    auto flag = [&](uint32_t r) -> bool {
        uint8_t st = P.rq_state[r];
        if (st == RQ_NOCACHE) return true;
        if (st != RQ_PENDING) return false;
        uint64_t kb = (uint64_t)P.rq_stream[r] * S.kc_cap;
        return S.kc_claim[kb + P.rq_cslot[r]] == r;
    };
    auto out = [&](uint32_t r, uint32_t m, bool f) {
        if (!f) return;
        const uint32_t s = P.rq_stream[r];
        P.rq_m[r] = m;
        P.pr_req[m] = r;
        P.pr_w[m] = P.rq_w[r];
        P.pr_stream[m] = s;
        P.pr_inrow[m] = (int32_t)S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + P.rq_c[r]];
    };
    chained_scan(n_req, status, ticket, flag, out, &P.counters[0]);
}

// --------------------------------------------------------------------------
// kernel 3: HS + MaxEnt score of the primaries (warp per primary) and the
// successor history (history + (w,))[-order:] (rnnlm.py:187) of new rows
// --------------------------------------------------------------------------
template <int VEC, int CPL>
__global__ void __launch_bounds__(256) k_hs_prim(DevModel m, DevPlan P, DevStreams S, uint32_t cap) {
    const uint32_t n = P.counters[0];
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= n) return;
    const uint32_t row = (uint32_t)P.pr_inrow[q];
    const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
    const int L = (int)meta[0];
    const int w = P.pr_w[q];
    const uint32_t o0 = __ldg(m.path_off + w), o1 = __ldg(m.path_off + w + 1);
    double lp = hs_logprob_warp<VEC, CPL>(m, S.arena_h + (size_t)row * m.H, meta + 1, L,
                                          m.path_code + o0, o1 - o0, lane);
    const uint32_t base = P.counters[2];
    if (lane == 0) {
        if (P.alg) {   // algorithmic-work counters for the roofline (bench.py)
            const int km = m.order < L ? m.order : L;
            atomicAdd(&P.alg[0], (unsigned long long)(o1 - o0));
            atomicAdd(&P.alg[1], (unsigned long long)(o1 - o0) * km);
            atomicAdd(&P.alg[2], 1ull);
        }
        P.pr_p[q] = lp;
        uint32_t *mo = S.arena_meta + (size_t)(base + q) * OTF_META;
        int nl = L + 1 > m.order ? m.order : L + 1;
        int drop = L + 1 - nl;
        uint32_t nm[OTF_META];
#pragma unroll
        for (int k = 0; k < OTF_META; k++) nm[k] = 0;
        for (int k = 0; k < nl - 1; k++) nm[1 + k] = meta[1 + drop + k];
        nm[nl] = (uint32_t)w;
        nm[0] = (uint32_t)nl;
#pragma unroll
        for (int k = 0; k < OTF_META; k++) mo[k] = nm[k];
    }
}

// arena capacity check + base row for this level (1 thread)
__global__ void k_level_begin(DevPlan P, DevStreams S) {
    const uint32_t base = *S.arena_used;
    P.counters[2] = base;
    if ((uint64_t)base + P.counters[0] > S.arena_rows) {
        atomicOr(S.err, OTF_E_ARENA_FULL);
        P.counters[0] = 0;   // drop the level: the run is failed and reported
    }
}

// --------------------------------------------------------------------------
// kernel 5: content dedup (IndexTable.encode, context_table.py:74-86):
// digest of (h' bytes, history) -> probe the stream's content table; a
// pre-existing entry is confirmed by full comparison; a slot created in
// this level is claimed by the lowest primary index.
// --------------------------------------------------------------------------
__device__ __forceinline__ bool rows_equal(const DevStreams &S, uint32_t ra, uint32_t rb, int lane) {
    const float *a = S.arena_h + (size_t)ra * S.H, *b = S.arena_h + (size_t)rb * S.H;
    bool eq = true;
    for (int i = lane; i < S.H; i += 32) eq &= (__float_as_uint(a[i]) == __float_as_uint(b[i]));
    if (lane < OTF_META) eq &= S.arena_meta[(size_t)ra * OTF_META + lane] == S.arena_meta[(size_t)rb * OTF_META + lane];
    return __all_sync(0xffffffffu, eq);
}

__global__ void __launch_bounds__(256) k_dedup(DevPlan P, DevStreams S) {
    const uint32_t n = P.counters[0];
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= n) return;
    const uint32_t row = P.counters[2] + q;
    const uint32_t s = P.pr_stream[q];
    // content digest: per-element mixes summed (order-independent reduction
    // of position-tagged words; deterministic for identical content)
    const float *h = S.arena_h + (size_t)row * S.H;
    unsigned long long acc = 0;
    for (int i = lane; i < S.H; i += 32)
        acc += otf_hash64(((uint64_t)i << 32) ^ __float_as_uint(h[i]));
    if (lane < OTF_META)
        acc += otf_hash64(((uint64_t)(0x10000 + lane) << 32) ^ S.arena_meta[(size_t)row * OTF_META + lane]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const unsigned long long key = otf_hash64(acc) | 1ull;
    const uint64_t base = (uint64_t)s * S.ct_cap;
    const uint32_t mask = S.ct_cap - 1;
    uint32_t slot = (uint32_t)(key >> 20) & mask;
    for (uint32_t probes = 0;; probes++) {
        if (probes > S.ct_cap) {
            if (lane == 0) { atomicOr(S.err, OTF_E_TABLE_FULL); P.pr_ctslot[q] = OTF_UNSET; P.pr_found[q] = 0; }
            return;
        }
        unsigned long long k = 0;
        if (lane == 0) {
            k = S.ct_key[base + slot];
            if (k == 0ull) {
                unsigned long long prev = atomicCAS(&S.ct_key[base + slot], 0ull, key);
                k = prev == 0ull ? key : prev;
            }
        }
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k == key) {
            uint32_t idx = lane == 0 ? ld_volatile_u32(&S.ct_idx[base + slot]) : 0;
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx != OTF_UNSET) {   // stored by an earlier level / call
                uint32_t srow = S.ct_row[base + slot];
                if (rows_equal(S, srow, row, lane)) {
                    if (lane == 0) { P.pr_ctslot[q] = OTF_UNSET; P.pr_found[q] = idx; }
                    return;
                }
            } else {
                if (lane == 0) { atomicMin(&S.ct_claim[base + slot], q); P.pr_ctslot[q] = slot; }
                return;
            }
        }
        slot = (slot + 1) & mask;
    }
}

// kernel 6: ordered numbering of novel contexts (new index = len + 1 in
// request order per stream)
__global__ void __launch_bounds__(SCAN_BLK) k_scan_novel(DevPlan P, DevStreams S, unsigned long long *status,
                                                         uint32_t *ticket) {
    const uint32_t n = P.counters[0];
    auto flag = [&](uint32_t q) -> bool {
        uint32_t slot = P.pr_ctslot[q];
        if (slot == OTF_UNSET) return false;
        return S.ct_claim[(uint64_t)P.pr_stream[q] * S.ct_cap + slot] == q;
    };
    // pr_E[q] = novel primaries before q (all q); the stream's first primary
    // also records the stream's base so numbering restarts per stream
    auto out = [&](uint32_t q, uint32_t e, bool) {
        P.pr_E[q] = e;
        const uint32_t s = P.pr_stream[q];
        if (q == 0 || P.pr_stream[q - 1] != s) P.first_E[s] = e;
    };
    chained_scan(n, status, ticket, flag, out, &P.counters[1]);
}

// --------------------------------------------------------------------------
// kernel 7: assign indices, fill the IndexTable / cache values
// --------------------------------------------------------------------------
__global__ void k_resolve(DevPlan P, DevStreams S) {
    const uint32_t n = P.counters[0];
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const uint32_t s = P.pr_stream[q];
    const uint32_t slot = P.pr_ctslot[q];
    const uint32_t base_row = P.counters[2];
    uint32_t cn;
    if (slot == OTF_UNSET) {
        cn = P.pr_found[q];
    } else {
        const uint64_t cb = (uint64_t)s * S.ct_cap;
        const uint32_t win = S.ct_claim[cb + slot];
        const uint32_t idx = S.table_len[s] + (P.pr_E[win] - P.first_E[s]) + 1u;
        cn = idx;
        if (win == q) {
            if (idx > S.max_ctx) {
                atomicOr(S.err, OTF_E_TABLE_FULL);
            } else {
                S.ct_idx[cb + slot] = idx;
                S.ct_row[cb + slot] = base_row + q;
                S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + idx] = base_row + q;
                atomicAdd(&S.novel_cnt[s], 1u);
            }
        } else {
            // same digest claimed by another primary: must be identical content
            const float *a = S.arena_h + (size_t)(base_row + q) * S.H;
            const float *b = S.arena_h + (size_t)(base_row + win) * S.H;
            bool eq = true;
            for (int i = 0; i < S.H; i++) eq &= __float_as_uint(a[i]) == __float_as_uint(b[i]);
            for (int i = 0; i < OTF_META; i++)
                eq &= S.arena_meta[(size_t)(base_row + q) * OTF_META + i] ==
                      S.arena_meta[(size_t)(base_row + win) * OTF_META + i];
            if (!eq) atomicOr(S.err, OTF_E_HASH);
        }
    }
    P.pr_cnext[q] = cn;
    const uint32_t r = P.pr_req[q];
    if (S.enabled) {
        const uint64_t kb = (uint64_t)s * S.kc_cap + P.rq_cslot[r];
        S.kc_p[kb] = P.pr_p[q];
        __threadfence();
        S.kc_cnext[kb] = cn;
    }
}

// --------------------------------------------------------------------------
// kernel 8: finish requests: small-LM delta, score, arrival write, counters
// --------------------------------------------------------------------------
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

__global__ void __launch_bounds__(256) k_finish(DevPlan P, DevStreams S, DevNgram g, uint32_t n_req,
                                                uint32_t lvl, double lm_weight) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0) *S.arena_used += P.counters[0];
    if (r < (uint32_t)S.S) {
        uint32_t nc = S.novel_cnt[r];
        if (nc) { S.table_len[r] += nc; S.novel_cnt[r] = 0; }
    }
    if (r >= n_req) return;
    const uint8_t st = P.rq_state[r];
    if (st == RQ_INVALID) return;
    const uint32_t s = P.rq_stream[r];
    double p;
    uint32_t cn;
    const uint32_t m = P.rq_m[r];
    if (m != OTF_UNSET) {
        p = P.pr_p[m];
        cn = P.pr_cnext[m];
    } else {
        const uint64_t kb = (uint64_t)s * S.kc_cap + P.rq_cslot[r];
        p = S.kc_p[kb];
        cn = S.kc_cnext[kb];
    }
    const uint32_t c = P.rq_c[r];
    const int w = P.rq_w[r];
    const uint32_t row = S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + c];
    const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
    double ps;
    if (!ngram_logprob_dev(g, meta + 1, (int)meta[0], w, &ps)) {
        atomicOr(S.err, OTF_E_KEY);
        ps = 0.0;
    }
    const float delta = __double2float_rn(__dsub_rn(p, ps));    // codec.py:57-59
    const uint32_t a = P.rq_arc[r];
    // decoder.py:144: (score + acoustic) + lm_weight * (smalllm + delta)
    const double ns = __dadd_rn(__dadd_rn(P.rq_score[r], P.arc_ac[a]),
                                __dmul_rn(lm_weight, __dadd_rn(P.arc_slm[a], (double)delta)));
    Arrival out;
    out.score = ns; out.ctx = cn; out.parent = P.rq_parent[r]; out.arc = a;
    out.lvl = lvl; out.ridx = r; out.pad = 0;
    P.arr[P.rq_dslot[r]] = out;
    unsigned long long *stt = S.stats + (size_t)s * 8;
    atomicAdd(&stt[0], 1ull);                        // lookups
    if (m != OTF_UNSET) {                            // misses (model runs)
        atomicAdd(&stt[2], 1ull);
        if (S.enabled) atomicAdd(&stt[6], 1ull);     // cache entries
    } else {
        atomicAdd(&stt[1], 1ull);                    // hits
    }
    atomicAdd(&stt[7], 1ull);                        // expansions this run
}

// --------------------------------------------------------------------------
// final: best token over sorted finals x sorted ctx (decoder.py:150-156),
// backtrace (decoder.py:157-162), score breakdown (decoder.py:163-169)
// --------------------------------------------------------------------------
__global__ void k_final(DevPlan P, DevStreams S, double lm_weight) {
    const uint32_t u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (u >= P.n_utt) return;
    bool have = false;
    double best = 0.0;
    uint32_t best_ctx = 0, best_slot = OTF_UNSET;
    for (uint32_t f = P.final_off[u]; f < P.final_off[u + 1]; f++) {
        const NodeInfo nd = P.nodes[P.finals[f]];
        if (nd.cap == 0) continue;
        recombine_node(P.arr, P.slot_win, nd.slot_base, nd.cap, lane);
        // best winner of this node: max score, ties -> smallest ctx
        double bs = 0.0; uint32_t bc = OTF_UNSET, bslot = OTF_UNSET; bool bh = false;
        for (uint32_t i0 = 0; i0 < nd.cap; i0 += 32) {
            uint32_t i = i0 + lane;
            if (i < nd.cap && P.slot_win[nd.slot_base + i]) {
                Arrival a = P.arr[nd.slot_base + i];
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

__global__ void k_init_starts(DevPlan P) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= P.n_utt) return;
    Arrival a;
    a.score = 0.0; a.ctx = 0; a.parent = OTF_UNSET; a.arc = OTF_UNSET; a.lvl = 0; a.ridx = 0; a.pad = 0;
    P.arr[P.utt_start_slot[u]] = a;
}

__global__ void k_run_begin(DevStreams S) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= (uint32_t)S.S) return;
    S.stats[(size_t)s * 8 + 7] = 0;
}

/*
 * otflm_b200.h -- C-ABI of the B200-native on-the-fly RNNLM rescoring path.
 *
 * Drop-in boundary for the reference package ``otflm`` (Python, numba
 * kernels).  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/otflm/).  The Python host
 * mirror ``paper_2007_11794_b200`` binds these with ctypes; INTEGRATION.md
 * shows the stub the reference side would add.
 *
 * Conventions
 *  - Every function returns an int status: OTFLM_OK (0) or a negative code
 *    that the host shim maps 1:1 onto the reference's exceptions.
 *  - "dev" pointers are CUDA device pointers (e.g. torch tensors'
 *    data_ptr()); "host" pointers are ordinary host memory.  Plain pointers
 *    and sizes only -- no torch types cross this boundary.
 *  - ``stream`` is a cudaStream_t passed as void*; all device work is
 *    enqueued asynchronously on it (functions with host outputs synchronize
 *    it before returning).
 *  - A model handle is immutable and may be shared by any number of stream
 *    sets.  A stream set is single-writer.
 */
#ifndef OTFLM_B200_H
#define OTFLM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTFLM_OK 0
#define OTFLM_ERR_VALUE (-1)          /* ValueError (rnnlm.py:173-177, decoder.py:123-124) */
#define OTFLM_ERR_UNKNOWN_INDEX (-2)  /* context_table.UnknownIndexError (:36-37) */
#define OTFLM_ERR_TABLE_FULL (-3)     /* context_table.TableFullError (:40-41) */
#define OTFLM_ERR_NO_PATH (-4)        /* decoder.py:155-156 */
#define OTFLM_ERR_KEY (-5)            /* ngram.py:179 KeyError */
#define OTFLM_ERR_NOMEM (-6)
#define OTFLM_ERR_CYCLE (-7)          /* lattice.LatticeFormatError (lattice.py:86-87) */
#define OTFLM_ERR_PACK (-8)           /* codec.PackOverflowError (codec.py:31-46) */
#define OTFLM_ERR_CUDA (-9)
#define OTFLM_ERR_HASH (-10)          /* 64-bit content-digest collision detected */

/* Precision of the recurrent update h' = sigmoid(U[w] + W h). */
#define OTFLM_PREC_FP64 0    /* CUDA-core DFMA, reference summation order (exact mode) */
#define OTFLM_PREC_TF32X3 1  /* tcgen05 kind::tf32, 3-pass split (fp32-faithful) */
#define OTFLM_PREC_BF16 2    /* tcgen05 kind::f16 with bf16 operands */
#define OTFLM_PREC_TF32 3    /* tcgen05 kind::tf32, single pass */
#define OTFLM_PREC_EXACT 4   /* tcgen05 kind::i8 digit planes, exact int32 accumulation, certified
                                f32 rounding + sequential-f64 fallback: every h' equals the
                                reference's (_kernels_nb.py:51-60); float64 HS.  Persistent stream
                                schedule; elsewhere it runs the FP64 path */

/* decode schedules (otflm_plan_set_schedule) */
#define OTFLM_SCHED_LEVEL 0   /* level-synchronous: expand / HS || update / assign kernels per level
                                 for the whole batch (CUDA graph); every precision */
#define OTFLM_SCHED_STREAM 1  /* persistent: one CTA per utterance stream runs all of its levels in
                                 one launch (TF32X3 / TF32, H % 4 == 0, H <= 512) */
#define OTFLM_SCHED_STREAM1 2  /* OTFLM_PREC_EXACT only: one CTA per utterance stream runs the whole
                                 level chain (HS and update GEMMs in turn on its own tensor core);
                                 for batches with at least one stream per SM (exact_solo.cuh) */

typedef struct OtflmModel OtflmModel;
typedef struct OtflmNgram OtflmNgram;
typedef struct OtflmStreams OtflmStreams;
typedef struct OtflmPlan OtflmPlan;
typedef struct OtflmGroup OtflmGroup;

/* ---- model upload (replaces handing numpy arrays to otflm.kernels;
 *      RnnlmModel rnnlm.py:69-124 + HuffmanTree huffman.py:40-51) ------- */
/* Any weight pointer may be NULL when only some kernels are needed (the
 * reference-signature operator table uploads just what a call uses);
 * decoding streams require a complete model. */
typedef struct {
    int32_t hidden_size, vocab_size, maxent_order;
    uint64_t maxent_size, hash_seed;
    const float *input_weights;     /* host [V, H] */
    const float *recurrent_weights; /* host [H, H] */
    const float *node_vectors;      /* host [V-1, H] */
    const float *maxent_table;      /* host [maxent_size] */
    const int32_t *path_nodes;      /* host [n_path] */
    const float *path_signs;        /* host [n_path] (+1 / -1) */
    const int64_t *path_offsets;    /* host [V+1] */
    int64_t n_path;
} OtflmModelDesc;

int otflm_model_create(const OtflmModelDesc *desc, int32_t device, OtflmModel **out);
int otflm_model_destroy(OtflmModel *m);
/* device-resident row pointers of the uploaded weights (read-only) */
int otflm_model_info(const OtflmModel *m, int64_t *out8);

/* ---- small LM (NgramModel ngram.py:34-46; lookup ngram.py:161-179) ---- */
typedef struct {
    int32_t order, vocab_size, bos_id;
    int64_t n_probs;
    const int32_t *prob_keys;   /* host [n_probs, order] (row-padded) */
    const int32_t *prob_lens;   /* host [n_probs] */
    const double *prob_vals;    /* host [n_probs] natural log */
    int64_t n_backoffs;
    const int32_t *bow_keys;    /* host [n_backoffs, order] */
    const int32_t *bow_lens;
    const double *bow_vals;
} OtflmNgramDesc;

int otflm_ngram_create(const OtflmNgramDesc *desc, const OtflmModel *m, OtflmNgram **out);
int otflm_ngram_destroy(OtflmNgram *g);
/* ngram_logprob for n (context, word) pairs; ctx dev [n, order-1] padded
 * with <s> on the left by the caller, out dev double [n]. */
int otflm_ngram_logprob_batch(const OtflmNgram *g, int64_t n, const int32_t *ctx_dev,
                              const int32_t *w_dev, double *out_dev, void *stream);

/* ---- kernel table (otflm.kernels, kernels.py:30-36), batched ---------- */
/* feature_index (_kernels_nb.py:21-33): words dev [n, 8] (first order_k
 * used), order_k / node dev [n]; out dev uint64 [n]. */
int otflm_feature_index_batch(uint64_t seed, uint64_t mask, int64_t n, const int32_t *order_k_dev,
                              const int64_t *words_dev, const int64_t *node_dev,
                              uint64_t *out_dev, void *stream);
/* word_logprob (_kernels_nb.py:78-86 via rnnlm.py:195-204): per query the
 * hidden row h_dev[ctx[i]], history hist_dev[ctx[i], 0:hist_len[ctx[i]]]
 * (oldest first), word w_dev[i]; out dev double [n]. */
int otflm_word_logprob_batch(const OtflmModel *m, int64_t n, const int32_t *ctx_dev,
                             const float *h_dev, const int32_t *hist_dev,
                             const int32_t *hist_len_dev, const int32_t *w_dev,
                             double *out_dev, void *stream);
/* Same with the accumulation mode chosen: exact != 0 accumulates the dot
 * products in float64 (|d| <= 1e-12 vs the reference); exact == 0 uses f32
 * per-lane partials (|d| <= 1e-5; the tensor-core decode modes use it). */
int otflm_word_logprob_batch2(const OtflmModel *m, int64_t n, const int32_t *ctx_dev,
                              const float *h_dev, const int32_t *hist_dev,
                              const int32_t *hist_len_dev, const int32_t *w_dev,
                              double *out_dev, int32_t exact, void *stream);
/* word_logprob with explicit path slices (the reference kernel signature,
 * _kernels_nb.py:78-79): query i scores path_code[path_off[i]..path_off[i+1])
 * where code = node | (branch bit << 31). */
int otflm_word_logprob_paths(const OtflmModel *m, int64_t n, const int32_t *ctx_dev,
                             const float *h_dev, const int32_t *hist_dev,
                             const int32_t *hist_len_dev, const int64_t *path_off_dev,
                             const uint32_t *path_code_dev, double *out_dev, void *stream);
/* advance_hidden (_kernels_nb.py:51-60 via rnnlm.py:180-188):
 * h_out[i] = f32(sigmoid(U[w[i]] + W h_in[ctx[i]])). */
int otflm_advance_hidden_batch(const OtflmModel *m, int64_t n, const int32_t *ctx_dev,
                               const float *h_in_dev, const int32_t *w_dev, float *h_out_dev,
                               int32_t precision, void *stream);
/* advance_hidden with the input rows given explicitly (the reference
 * signature advance_hidden(input_row, recurrent, hidden)): input_rows dev [n, H]. */
int otflm_advance_hidden_rows(const OtflmModel *m, int64_t n, const float *input_rows_dev,
                              const int32_t *ctx_dev, const float *h_in_dev, float *h_out_dev,
                              int32_t precision, void *stream);
/* all_word_logprobs (_kernels_nb.py:89-104) for one context; out dev [V]. */
int otflm_all_word_logprobs(const OtflmModel *m, const float *h_dev, const int32_t *hist_host,
                            int32_t hist_len, double *out_dev, void *stream);

/* all_word_logprobs for n contexts at once: query i uses h_dev[ctx[i]] and
 * hist_dev[ctx[i], 0:hist_len[ctx[i]]] (row stride maxent_order); out dev
 * double [n, V].  precision OTFLM_PREC_FP64: float64 CUDA-core dot products
 * (the reference's arithmetic up to summation order); a tensor-core mode:
 * the node activations [n x (V-1)] are one tcgen05 GEMM of the contexts
 * against the node vectors (fp32 accumulate), MaxEnt terms and log-sigmoids
 * in float64 once per node, path sums per word. */
int otflm_all_word_logprobs_batch(const OtflmModel *m, int64_t n, const int32_t *ctx_dev,
                                  const float *h_dev, const int32_t *hist_dev,
                                  const int32_t *hist_len_dev, double *out_dev, int32_t precision,
                                  void *stream);

/* ---- decoding streams: IndexTable + RescoreCache + ledger per stream
 *      (context_table.py:48-119, cache.py:61-191, codec.py:95-110) ------ */
typedef struct {
    int32_t n_streams;
    int32_t cache_enabled;       /* RescoreCache(enabled=...) cache.py:84-86 */
    int64_t max_contexts;        /* per stream IndexTable(max_entries) */
    int64_t cache_slots;         /* per stream (power of two, >= 2x entries) */
    int64_t arena_rows;          /* total hidden-state rows across streams */
} OtflmStreamConfig;

int otflm_streams_create(const OtflmModel *m, const OtflmStreamConfig *cfg, OtflmStreams **out);
int otflm_streams_destroy(OtflmStreams *s);
/* reset_utterance (cache.py:185-191) for every stream. */
int otflm_streams_reset(OtflmStreams *s, int32_t retain, void *stream);
/* per stream 8 counters: lookups, hits, misses, table_len, cum_lookups,
 * cum_hits, cum_misses, cache_entries.  out host int64 [n_streams * 8]. */
int otflm_streams_stats(OtflmStreams *s, int64_t *out_host, void *stream);
/* IndexTable.encode (context_table.py:76-89) on stream sid: n host contexts
 * (hidden f32 [n, H], history u32 [n, order] + lengths) in call order; the
 * index of each (existing equal content, or len + 1).  OTFLM_ERR_TABLE_FULL
 * when the table is full (TableFullError, context_table.py:84-85). */
int otflm_streams_encode(OtflmStreams *s, int32_t sid, int64_t n, const float *hidden_host,
                         const uint32_t *hist_host, const int32_t *hist_len_host, uint32_t *idx_host,
                         void *stream);
/* RescoreCache.get / put (cache.py:80-108) on stream sid, keys (c, w) in call
 * order.  get counts lookups / hits / misses (cache disabled: every lookup a
 * miss) and returns found + (p, c').  put stores a value unless the key holds
 * one (first value wins; disabled cache: no-op).  Unbounded caches only: a
 * capacity-bounded cache returns OTFLM_ERR_VALUE (its policy replays the
 * lookups rnnlm_prob logs). */
int otflm_streams_cache_get(OtflmStreams *s, int32_t sid, int64_t n, const uint32_t *c_host,
                            const int32_t *w_host, uint8_t *found_host, double *p_host, uint32_t *c_next_host,
                            void *stream);
int otflm_streams_cache_put(OtflmStreams *s, int32_t sid, int64_t n, const uint32_t *c_host,
                            const int32_t *w_host, const double *p_host, const uint32_t *c_next_host,
                            void *stream);
/* RescoreCache.roll_stats (cache.py:156-158): window counters into the
 * cumulative ones; RescoreCache.clear (cache.py:136-140): drop every entry of
 * the stream's cache, counters kept.  Also on a capacity-bounded cache: roll moves
 * the window's evictions too, clear also empties the LFU policy state. */
int otflm_streams_roll_stats(OtflmStreams *s, int32_t sid, void *stream);
int otflm_streams_cache_clear(OtflmStreams *s, int32_t sid, void *stream);
/* RescoreCache capacity (cache.py:61-137): capacity_bytes > 0 bounds the
 * resident entries to capacity_bytes / 32 (ENTRY_BYTES, cache.py:26) under
 * the reference's LFU + LRU-tie-break eviction; 0 = unbounded.  Lookups of
 * every decode / rnnlm_prob_batch call are replayed through the policy in
 * reference order, so hits / misses / evictions / resident entries equal
 * the reference's; evicted values stay memoised in device memory.  Shrinking
 * evicts at once (set_capacity, cache.py:130-137). */
int otflm_streams_set_capacity(OtflmStreams *s, int64_t capacity_bytes, void *stream);
/* per stream 3 counters: evictions in the current window, cumulative
 * evictions, resident entries.  out host int64 [n_streams * 3]. */
int otflm_streams_cache_stats(OtflmStreams *s, int64_t *out_host, void *stream);
/* IndexTable.decode (context_table.py:88-104): hidden host [H], hist host
 * [order], *len. */
int otflm_streams_context(OtflmStreams *s, int32_t stream_id, uint32_t idx, float *hidden_host,
                          int32_t *hist_host, int32_t *len_host, void *stream);
/* rnnlm_prob (cache.py:165-182) for a batch of n requests with the
 * semantics of issuing them one by one in array order: a (c, w) repeated
 * inside the batch is a miss the first time and a hit afterwards; new
 * context indices are assigned len+1 in array order.  Every c must exist
 * before the call.  All pointers host; outputs p [n], c_next [n], hit [n]. */
int otflm_rnnlm_prob_batch(OtflmStreams *s, int64_t n, const int32_t *stream_ids,
                           const uint32_t *c, const int32_t *w, int32_t precision, double *p,
                           uint32_t *c_next, uint8_t *hit, void *stream);

/* ---- decoder: rescore_onthefly (decoder.py:114-173) over a batch of
 *      utterances, one stream each ------------------------------------- */
typedef struct {
    int32_t n_utt;
    const int32_t *n_nodes;      /* [n_utt]; node ids are 0..n_nodes-1 */
    const int32_t *start;        /* [n_utt] */
    const int64_t *arc_off;      /* [n_utt+1] into the arc arrays (arc-id order) */
    const int32_t *arc_src, *arc_dst, *arc_word;
    const double *arc_ac, *arc_slm;
    const int64_t *final_off;    /* [n_utt+1] */
    const int32_t *finals;       /* ascending per utterance */
    const int32_t *stream_ids;   /* [n_utt] stream of each utterance */
} OtflmLatticeBatch;

typedef struct {
    int32_t *path_len;        /* [n_utt] */
    int32_t *path_arcs;       /* [n_utt * max_path] */
    int32_t max_path;
    double *combined, *acoustic, *lm; /* [n_utt] */
    int64_t *end_ctx, *expansions;    /* [n_utt] */
    int32_t *status;          /* [n_utt] per utterance OTFLM_* code */
} OtflmDecodeResult;

/* Host-side compile (topological levels, per-node beam capacities, arrival
 * slots) and upload of a lattice batch; plan is reusable for repeated runs. */
int otflm_plan_create(OtflmStreams *s, const OtflmLatticeBatch *lats, int64_t beam,
                      OtflmPlan **out, void *stream);
int otflm_plan_destroy(OtflmPlan *p);
/* Load another lattice batch into an existing plan.  When its compiled
 * structure matches, the arrays are re-uploaded into the same buffers and
 * captured graphs stay valid (*same = 1); otherwise nothing changes and
 * OTFLM_ERR_VALUE is returned with *same = 0. */
int otflm_plan_refresh(OtflmPlan *p, const OtflmLatticeBatch *lats, int32_t *same, void *stream);
/* plan stats: levels, nodes, arcs, slots, max requests per level, total
 * request slots, graph nodes (int64 [8]) */
int otflm_plan_info(const OtflmPlan *p, int64_t *out8);
/* wide-level flags of a compiled batch: bit 0 = nodes with more than 64
 * arrival slots (big beams: expanded by a CTA per node, decode.cuh
 * k_expand_big), bit 1 = (level, stream) request ranges above 4096 (the
 * multi-CTA ordered assign, k_asg_*).  Both run on the level schedule, which
 * BatchDecoder(schedule="auto") then picks (decoder.py:131-149 per node). */
int otflm_plan_wide(const OtflmPlan *p, int32_t *flags);
/* Algorithmic-work counters of the last profiled run + upload size (int64 [6]):
 * sum of Huffman path lengths over HS queries, sum of path length x MaxEnt
 * orders, HS queries, bytes uploaded by plan_create, and (OTFLM_PREC_EXACT)
 * hidden-state elements whose rounding could not be certified and ran the
 * reference's sequential loop, and (EXACT stream) context rows whose digit
 * planes were not made at their creation in this launch (digitized late). */
int otflm_plan_counters(const OtflmPlan *p, int64_t *out6, void *stream);
/* One decode run captured as a CUDA graph with an event-record node around
 * every kernel; writes device-side total ms / launch counts per category
 * (7 entries: expand, hs, advance, assign, final, misc, stream).  HS and the
 * recurrent update run as parallel graph branches, so their spans overlap;
 * the stream schedule reports its persistent kernel under "stream". */
int otflm_decode_profile(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                         void *stream, double *ms_out, int64_t *n_out);
/* Device-only decode of a prepared plan (inputs already resident in HBM).
 * use_graph != 0 replays a captured CUDA graph of the level loop (level
 * schedule; the stream schedule is three launches and ignores it). */
int otflm_decode_run(OtflmPlan *p, const OtflmNgram *g, double lm_weight, int32_t precision,
                     int32_t use_graph, void *stream);
/* Concurrent groups: plans over disjoint utterances get disjoint arena row
 * partitions [start, end) and are replayed as parallel chains of one CUDA
 * graph (the per-frame stages of different groups overlap on the GPU). */
int otflm_plan_set_arena(OtflmPlan *p, uint32_t start, uint32_t end);
/* Select the decode schedule of a plan (OTFLM_SCHED_*); both produce the
 * reference's results (rescore_onthefly, decoder.py:114-173) for every
 * utterance.  otflm_schedule_supported returns 1 if the model / precision can
 * run the schedule. */
int otflm_plan_set_schedule(OtflmPlan *p, int32_t schedule);
/* Stream schedule, after otflm_decode_profile: device time per phase summed
 * over CTAs (ns), 12 entries -- o[0] expand, o[1] recurrent-update K loop,
 * o[2] MMA drain, o[3] update epilogue, o[4] HS setup + row staging,
 * o[5] HS pair rounds, o[6] whole HS group (small-LM scores + HS; runs
 * concurrently with o[1..3]), o[7] assign, o[8] wait of the update group for
 * the HS group, o[9] MMA-warp wait for operands, o[10] uncertified-element
 * loop (OTFLM_PREC_EXACT), o[11] CTAs, o[12..16] assign sections (probe, dedup
 * scan, numbering, values, arrivals), o[17..20] EXACT update: row table,
 * digitize, 2 spare, o[21..23] EXACT HS (rank 0): wait for the chunk's digits,
 * digit-plane GEMM + epilogue, MaxEnt + log-sigmoid, o[24..25] EXACT plane
 * copy (row pass, copy), o[26] the MMA warp's update K loops, o[27] update
 * epilogue stores, o[28..31] (one-CTA schedule) warp 2 under the K loops: HS
 * tail, row stores, fallbacks, U staging: 32 entries (o must hold 32).
 * (EXACT: o[1] is the digitize barrier, o[2] the wait of the MMA warp for the
 * other warps after its K loops; o[11] counts streams in the one-CTA schedule.) */
int otflm_plan_phase_ns(const OtflmPlan *p, int64_t *o, void *stream);
int otflm_schedule_supported(const OtflmModel *m, int32_t schedule, int32_t precision);
int otflm_group_create(OtflmPlan **plans, int32_t n, OtflmGroup **out);
int otflm_group_destroy(OtflmGroup *g);
int otflm_group_run(OtflmGroup *g, const OtflmNgram *ng, double lm_weight, int32_t precision,
                    void *stream);
int otflm_group_profile(OtflmGroup *g, const OtflmNgram *ng, double lm_weight, int32_t precision,
                        void *stream, double *ms_out, int64_t *n_out);
/* Lattice-out: with enable != 0 the decode marks every
 * kept arrival (a token that was expanded within the beam, or a final
 * recombination winner); otflm_decode_lattice_fetch then returns, per
 * utterance, the RNNLM-rescored pruned state lattice as 24-byte records
 * {double score; uint32 state, parent, arc, pad} in state order: state =
 * arrival slot relative to the utterance, parent = the state it was expanded
 * from (0xFFFFFFFF for the start state), arc = batch-global arc id, score =
 * the path score of decoder.py:144.  count_host [n_utt]; records_host may be
 * NULL to query the counts (capacity cap records). */
int otflm_plan_set_lattice_out(OtflmPlan *p, int32_t enable);
int otflm_decode_lattice_fetch(OtflmPlan *p, int64_t *count_host, void *records_host, int64_t cap,
                               void *stream);
/* Copy results of the last run to host (synchronizes). */
int otflm_decode_fetch(OtflmPlan *p, OtflmDecodeResult *res, void *stream);
/* End to end: plan_create + decode_run + decode_fetch + plan_destroy. */
int otflm_decode(OtflmStreams *s, const OtflmNgram *g, const OtflmLatticeBatch *lats,
                 double lm_weight, int64_t beam, int32_t precision, OtflmDecodeResult *res,
                 void *stream);
/* number of kernels the last decode_run enqueued */
int64_t otflm_last_launch_count(void);

/* ---- two-pass rescoring ------------------------ */
/* nbest (decoder.py:180-230) for every utterance of a lattice batch:
 * exact best-first search over first-pass weights (acoustic + lm_weight *
 * smalllm) with the backward-Viterbi completion as heuristic; distinct word
 * sequences, best path of each.  Host-side (a sequential priority-queue
 * walk that never touches the RNNLM), utterance-parallel on n_threads
 * threads (<= 0: all).  Per-utterance failures (no complete path, cycle) are
 * reported in the status array of otflm_nbest_copy. */
typedef struct OtflmNbest OtflmNbest;
int otflm_nbest_create(const OtflmLatticeBatch *lats, int32_t n, double lm_weight, int32_t n_threads,
                       OtflmNbest **out);
/* n_hyp host [n_utt]; out2 = {total hypotheses, total arcs} */
int otflm_nbest_sizes(const OtflmNbest *r, int32_t *n_hyp_host, int64_t *out2);
/* hyp_len [total hyps], arcs [total arcs] (lattice-local arc ids, path
 * order), scores [total hyps, 3] = (combined, acoustic, lm), status [n_utt] */
int otflm_nbest_copy(const OtflmNbest *r, int32_t *hyp_len, int32_t *arcs, double *scores,
                     int32_t *status);
int otflm_nbest_destroy(OtflmNbest *r);

/* rescore_twopass (decoder.py:243-274) for a batch of n-best lists.  The
 * hypotheses are merged into per-list prefix tries on the host; the device
 * scores each trie node once (HS + MaxEnt, recurrent update, running LM
 * sum), level by level over all lists. */
typedef struct OtflmTwopass OtflmTwopass;
typedef struct {
    int32_t n_lists;
    const int64_t *list_off;    /* host [n_lists+1] into the hypotheses; lists non-empty */
    const int64_t *hyp_off;     /* host [n_hyp+1] into words */
    const int32_t *words;       /* host word ids, hypothesis order */
    const double *acoustic;     /* host [n_hyp] */
} OtflmHypBatch;
#define OTFLM_TWOPASS_RNNLM 0   /* words scored by the recurrent model alone */
#define OTFLM_TWOPASS_HYBRID 1  /* lambda * ngram + (1 - lambda) * rnnlm in probability space */
int otflm_twopass_create(const OtflmModel *m, const OtflmNgram *g /* may be NULL in rnnlm mode */,
                         const OtflmHypBatch *hyps, int32_t n_threads, OtflmTwopass **out,
                         void *stream);
/* int64 [6]: trie nodes, levels, words, recurrent updates, widest level, hypotheses */
int otflm_twopass_info(const OtflmTwopass *p, int64_t *out6);
/* precision: OTFLM_PREC_FP64 (exact HS + f64 update) or a tensor-core mode;
 * use_graph != 0 replays a captured CUDA graph of the level loop. */
int otflm_twopass_run(OtflmTwopass *p, int32_t mode, double interp_weight, double lm_weight,
                      int32_t precision, int32_t use_graph, void *stream);
/* host outputs (any may be NULL): lm [n_hyp], combined [n_hyp], best [n_lists]
 * (index within the list of the first maximum of combined); synchronizes. */
int otflm_twopass_fetch(OtflmTwopass *p, double *lm, double *combined, int32_t *best, void *stream);
int otflm_twopass_destroy(OtflmTwopass *p);

const char *otflm_error_string(int32_t code);
const char *otflm_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif

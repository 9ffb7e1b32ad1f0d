// common.cuh -- device structures and helpers shared by the sm_100a kernels.
//
// Layout in HBM:
//   model:   U [V,H] f32, W [H,H] f32 (+ WT, tf32 hi/lo and bf16 copies for
//            the recurrent update), NV [V-1,H] f32, ME [M] f32,
//            path CSR: off u32 [V+1], code u32 (node | bit<<31).
//   streams: arena of hidden rows [R,H] f32 + meta [R,8] u32 (len, words),
//            per-stream ctx_row [max_ctx+1] -> arena row, open-addressing
//            content table (IndexTable) and (c,w) cache (RescoreCache).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define OTF_UNSET 0xFFFFFFFFu
#define OTF_META 8          // u32 words per arena row: len, w0..w6
#define OTF_MAX_ORDER 7

// error bits (device word, OR-ed)
#define OTF_E_TABLE_FULL 1u
#define OTF_E_ARENA_FULL 2u
#define OTF_E_CACHE_FULL 4u
#define OTF_E_HASH 8u
#define OTF_E_KEY 16u
#define OTF_E_VALUE 32u
#define OTF_E_PATH 64u
#define OTF_E_NOSLOT 128u   // with OTF_E_TABLE_FULL: a new context found no index-table slot

struct DevModel {
    int H, V, order;
    uint64_t mask, seed;
    const float *U, *W, *WT, *NV, *ME;
    const uint32_t *path_off, *path_code;
    const float *W_hi, *W_lo;          // tf32-rounded split of W (K-major rows)
    const __nv_bfloat16 *W_bf;         // bf16 copy of W
    // W_hi / W_lo pre-tiled for the persistent stream kernel: per K chunk of
    // wt_kcb bytes, [hi | lo] blocks of wt_npad rows (H rounded up to whole
    // 128-row M tiles, zero padded) in the canonical no-swizzle K-major UMMA
    // layout, so one bulk copy moves a whole chunk
    const float *W_t;
    int wt_kcb, wt_npad;
    // the same with 64-byte K chunks (SWIZZLE_64B), for the batched update
    // k_advance_tc's B operand: one bulk copy per (K chunk, N tile, hi/lo)
    const float *W_t64;
    // exact mode (exact_update.cuh): W as 8-bit digit planes pre-tiled per
    // (M tile, 64-byte K chunk) -- [mt][kc][plane][128 rows x 64 B] -- and per
    // output unit {sW 2^-47, A_i, B_i, sW} for the combine and the error bound
    const uint8_t *Wd;
    const double4 *wx;
    int wd_nkx;                        // 64-byte K chunks (H rounded up to 64)
    // the HS node vectors the same way, per node: NVd[node][kc][plane][64 B],
    // nx[node] = {sN 2^-31, eps_n, B_n, sN 2^-55} (exact_hs.cuh)
    const uint8_t *NVd;
    const double4 *nx;
};

struct DevNgram {
    int order, V, bos;
    // open addressing, key = tuple hash (nonzero), verified by stored words
    uint32_t p_cap, b_cap;
    const uint64_t *p_tag; const int32_t *p_words; const double *p_val;   // [cap], [cap*order]
    const uint64_t *b_tag; const int32_t *b_words; const double *b_val;
};

struct DevStreams {
    int S, enabled, H, order;
    uint32_t max_ctx;           // per stream contexts (indices 1..max_ctx)
    uint32_t arena_rows;
    uint32_t *ctx_row;          // [S][max_ctx+1]
    float *arena_h;             // [R][H]
    uint32_t *arena_meta;       // [R][OTF_META]
    uint32_t *arena_used;       // scalar
    uint32_t ct_cap;            // per stream content-table slots (pow2)
    unsigned long long *ct_key; // [S][ct_cap], 0 = empty
    uint32_t *ct_idx, *ct_row;
    uint32_t kc_cap;            // per stream cache slots (pow2)
    unsigned long long *kc_key; // [S][kc_cap], 0 = empty, else ((c<<32)|w)+1
    uint32_t *kc_claim, *kc_cnext;
    double *kc_p;
    uint32_t *table_len, *novel_cnt;  // [S]
    unsigned long long *stats;        // [S][8]
    unsigned int *err;
    // capacity-bounded cache (RescoreCache(capacity_bytes > 0), cache.py:98-134):
    // assign logs each stream's lookups in reference order (kc slot | memo-miss
    // bit 31); k_lfu_replay then runs the exact LFU + LRU policy over them
    uint32_t lfu_cap;                 // resident entries allowed (0: unbounded mode)
    uint32_t lfu_logcap;              // per stream log capacity
    uint32_t *lfu_log, *lfu_logn;     // [S][logcap], [S]  (nullptr: no log)
    // EXACT stream kernel: the digit planes of every arena row, made when the
    // row is created ([row][kc][plane][64 B]), its representation-error sum
    // and the launch (epoch) that made them (exact_update.cuh)
    uint8_t *arena_dig;
    float *arena_deh;
    uint32_t *arena_dep;
    // multi-CTA assign (decode.cuh k_asg_*): per content-table slot the first
    // request of the level that created the key ([S][ct_cap], all OTF_UNSET
    // between levels; allocated on first use)
    uint32_t *ct_first;
};

// per-request state
#define RQ_INVALID 0
#define RQ_HIT 1       // value present from an earlier level / call
#define RQ_PENDING 2   // key inserted this level; claim decides the primary
#define RQ_NOCACHE 3   // cache disabled: every request computes

struct LevelCtr {            // one per level (+ spare slots for the Table-1 batch API)
    uint32_t n_prim;         // requests that run the model this level
    uint32_t base;           // first arena row of this level's new states
    uint32_t pad0, pad1;
};

// Where a recurrent-update / HS launch finds its row count and writes rows:
// base = prev->base + prev->n_prim (previous level) or *base_dev (first
// level of a run) -- computed on the device, so CUDA-graph replays need no
// host round trip.
struct RowSpec {
    const uint32_t *n_dev;          // row count (nullptr: n_cap)
    LevelCtr *cur;                  // this level (its base is recorded here)
    const LevelCtr *prev;           // previous active level or nullptr
    const uint32_t *base_dev;       // base when prev == nullptr (nullptr: 0)
    unsigned long long *dig;        // per-row content digest (nullptr: none)
    uint32_t row_limit;             // rows >= row_limit are out of this plan's arena
};
__device__ __forceinline__ uint32_t row_base(const RowSpec &rs) {
    if (rs.prev) return rs.prev->base + rs.prev->n_prim;
    return rs.base_dev ? *rs.base_dev : 0u;
}

struct Arrival {       // 32 B, one per (dst node, in-arc, source rank)
    double score;
    uint32_t ctx, parent, arc, lvl, ridx, pad;
};

struct NodeInfo {      // 32 B
    uint32_t slot_base, cap, keep, out_b, out_e, req_base, stream, pad;
};

// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t otf_mix(uint64_t h, uint64_t x) {
    h = (h ^ x) * 0x9E3779B97F4A7C15ull;   // _kernels_nb.py:21-24
    return h ^ (h >> 32);
}

__device__ __forceinline__ uint64_t otf_hash64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// _kernels_nb.py:36-48 in float64 (CUDA libdevice exp/log1p, <= 1 ulp).
// Branch-free form of x >= 0 ? -log1p(exp(-x)) : x - log1p(exp(x)): the same
// value for every x (up to the sign of a zero result), without divergence.
__device__ __forceinline__ double otf_log_sigmoid(double x) {
    return fmin(x, 0.0) - log1p(exp(-fabs(x)));
}
__device__ __forceinline__ double otf_sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

// Content-digest term of element i of a hidden row (the digest is the
// wrapping sum over elements; every digest match is confirmed by a full row
// comparison, so the term only needs to spread well): one 64-bit multiply of
// a 32-bit mix of (i, bits).
__device__ __forceinline__ unsigned long long otf_dig_h(uint32_t i, float x) {
    // one full 64-bit mix (fmix64) of (element index, float bits): whenever an
    // element changes -- even by one ulp -- the digest sum moves by an
    // unrelated 64-bit value.  (A cheaper multiply + xorshift term let the
    // +-1 ulp changes of two elements cancel exactly: a real collision on the
    // fat variant between two rows 1 ulp apart in 2 of 256 elements.)  Element
    // indices stay below 0x10000, so these terms never coincide with the
    // history terms (dig_meta).
    return otf_hash64(((uint64_t)i << 32) | (uint64_t)__float_as_uint(x));
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += shfl_xor_d(v, m);
    return v;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// tuple hash for the small-LM tables (host mirrors this exactly)
__host__ __device__ __forceinline__ uint64_t otf_tuple_hash(const int32_t *w, int len) {
    uint64_t h = 0x243F6A8885A308D3ull ^ (uint64_t)len;
    for (int i = 0; i < len; i++) {
        uint64_t x = h ^ (uint64_t)(uint32_t)w[i];
        x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
        x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
        x ^= x >> 33;
        h = x + 0x9E37ull * (uint64_t)(i + 1);
    }
    return h | 1ull;   // never 0 (0 marks an empty slot)
}

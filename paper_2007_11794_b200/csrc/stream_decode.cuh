// stream_decode.cuh -- persistent per-stream decode: one CTA owns one
// utterance stream (its IndexTable, RescoreCache and tokens) and
// runs every level of the traversal inside one launch.
//
// Streams never read each other's state, so no grid-wide synchronisation is
// needed: each CTA advances through its own levels as fast as its dependency
// chain allows.  The level-synchronous schedule (decode.cuh + capi.cu) pays
// ~4 dependent launches per level for the whole batch; here a level costs
// four CTA barriers.
//
// Per level (reference decoder.py:130-149 for one utterance):
//   expand   warp per node (expand_node, shared with k_expand): recombine,
//            rank, keep the beam, probe/claim the (c, w) cache, small-LM score,
//            compact the requests that run the model (shared-memory counter);
//   rows     one atomicAdd reserves the level's arena rows for new contexts;
//   update   h' = sigmoid(U[w] + W h) on tcgen05 with W as the A operand
//            (M = output units in 128-row tiles) and the gathered context rows
//            as B (N = this level's rows, rounded up to 16), so the MMA work
//            follows the actual row count.  W chunks arrive by one bulk copy
//            each (pre-tiled at model upload, DevModel::W_t), context rows by
//            cp.async and are split into tf32 hi/lo in place; an S-stage ring
//            overlaps loads, conversion and MMAs; accumulators in TMEM
//            (lane = output unit, column = row), epilogue by all 16 warps;
//   HS       node-parallel over the level's (query, path node) pairs
//            (hs_level_nodepar): context rows staged in the shared memory the
//            update's ring used, 8 pairs per warp round, path-order sums;
//   assign   assign_range (shared with k_assign) over the stream's requests
//            in reference order with the whole CTA.
// Tensor-core precisions only (TF32X3 / TF32); FP64 exact mode and BF16 use
// the level-synchronous schedule.
#pragma once
#include "decode.cuh"
#include "tc_advance.cuh"
#include <cooperative_groups.h>

namespace sd {
constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int GW = 8;              // warps of the recurrent-update group (warp 0 issues MMAs)
constexpr int GT = GW * 32;

__device__ __forceinline__ void cp_wait_n(int n) {
    if (n <= 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    else if (n == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else if (n == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.wait_group 3;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// Bounded mbarrier wait: a protocol error traps (and reports where) instead
// of hanging the GPU after 2 s of wall time, orders of magnitude above any
// legitimate wait in this kernel.
__device__ __forceinline__ unsigned long long gtimer_() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wait_bounded(uint32_t bar, uint32_t parity, int tag) {
    unsigned long long t0 = 0;
    for (uint32_t it = 0;; it++) {
        uint32_t ok;
        // suspend-time hint (ns): the warp is parked until the phase completes
        // instead of re-polling (polls cost issue slots of the working warps)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity), "r"(1000000u) : "memory");
        if (ok) return;
        if ((it & 1023u) == 0) {                   // wall-clock bound: 2 s
            const unsigned long long t = gtimer_();
            if (it == 0) t0 = t;
            else if (t - t0 > 2000000000ull) {
                printf("k_decode_streams: wait timeout block %d thread %d tag %d parity %u\n", (int)blockIdx.x,
                       (int)threadIdx.x, tag, parity);
                __trap();
            }
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// named barrier over a warp group (id 0 is __syncthreads)
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// reduce8 (hs.cuh) for wrapping 64-bit sums: 8 values per lane -> the sum
// over lanes of value g on the lanes whose bits (4,3,2) spell g
__device__ __forceinline__ unsigned long long reduce8_u64(unsigned long long (&v)[8], int lane) {
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const unsigned long long send = u16 ? v[i] : v[i + 4], keep = u16 ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const unsigned long long send = u8 ? v[i] : v[i + 2], keep = u8 ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        const unsigned long long send = u4 ? v[0] : v[1], keep = u4 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    unsigned long long x = v[0];
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

// v[j] (j = 0..31) per lane -> lane j returns sum over lanes of v[j]
__device__ __forceinline__ unsigned long long transpose_sum32(unsigned long long (&v)[32], int lane) {
#pragma unroll
    for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
        const bool up = lane & off;
#pragma unroll
        for (int i = 0; i < n / 2; i++) {
            const unsigned long long send = up ? v[i] : v[i + n / 2];
            const unsigned long long keep = up ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}
}  // namespace sd
#include "exact_update.cuh"
#include "exact_hs.cuh"

// --------------------------------------------------------------------------
// Node-parallel HS + MaxEnt for one level of one stream (fast mode: f32 lane
// partials, float64 from the lane combine on -- the same arithmetic, in the
// same order, as hs_logprob_ring<CPL, false, ORD>, so both schedules agree
// bit for bit).  Queries are few per stream-level (~70) and each is a
// dependent chain of ~10 node rows, so instead of a warp per query the
// (query, path node) pairs of a batch are spread over all warps, 8 per warp
// round with all row loads in flight; the context rows live in shared memory
// and each pair's log-sigmoid goes to a per-pair slot, summed per query in
// path order afterwards.
// --------------------------------------------------------------------------
namespace sd {
constexpr int PAIRCAP = 2048;      // (query, node) pairs per batch
constexpr int QMAX = 128;          // queries per batch (upper bound)
struct HsLevelSmem {
    float *h;                      // [qb][H] context rows
    double *hd;                    // [qb][H] context rows widened (EXACT)
    double *lsig;                  // [PAIRCAP] activation, then log-sigmoid, per pair
    uint32_t *pcode;               // [PAIRCAP] path code of each pair
    uint8_t *pq;                   // [PAIRCAP] batch query of each pair
    unsigned long long *pre;       // [QMAX][ORD] MaxEnt hash prefixes
    uint32_t *row, *cb, *off, *P;  // [QMAX] arena row, path code base, pair offset, path length
    int32_t *w, *kmax, *L;         // [QMAX]
    uint32_t *scan;                // [NW + 2]
};
}  // namespace sd

// Run by a group of NT threads (NW warps) synchronising on named barrier
// BAR; tid / wid are group-relative.
template <int CPL, int ORD, int NT, int BAR, bool EXACT>
__device__ __forceinline__ void hs_level_nodepar(const DevModel &m, DevPlan &Q, DevStreams &S, uint32_t base,
                                                 uint32_t n, const sd::HsLevelSmem &hs, int qb_max, int tid,
                                                 int wid, int lane, unsigned long long *ph) {
    constexpr int NW = NT / 32;
#define HS_SYNC() sd::group_sync(BAR, NT)
    // ph (profiling, thread 0 only): [4] setup + staging, [5] pair rounds; the
    // caller's mark after HS then covers log-sigmoid + per-query finish
    unsigned long long tm = ph ? sd::gtimer() : 0ull;
#define HS_MARK(i) do { if (ph) { const unsigned long long t2 = sd::gtimer(); ph[i] += t2 - tm; tm = t2; } } while (0)
    const int H = m.H, NCH = H >> 2;
    for (uint32_t q0 = 0; q0 < n;) {
        const int nq = (int)min((uint32_t)qb_max, n - q0);
        // ---- A: per-query setup (thread per query), pair offsets ----
        uint32_t Pt = 0;
        if (tid < nq) {
            const uint32_t q = q0 + tid;
            const uint32_t row = (uint32_t)Q.pr_inrow[q];
            const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
            const int L = (int)meta[0];
            const int w = Q.pr_w[q];
            const uint32_t o0 = __ldg(m.path_off + w), o1 = __ldg(m.path_off + w + 1);
            const int kmax = m.order < L ? m.order : L;
#pragma unroll
            for (int k = 0; k < ORD; k++) {
                uint64_t x = 0;
                if (k < kmax) {
                    x = otf_mix(m.seed, (uint64_t)(k + 1));
                    for (int i = L - (k + 1); i < L; i++) x = otf_mix(x, (uint64_t)meta[1 + i]);
                }
                hs.pre[tid * ORD + k] = x;
            }
            Pt = o1 - o0;
            hs.row[tid] = row; hs.cb[tid] = o0; hs.P[tid] = Pt; hs.w[tid] = w; hs.kmax[tid] = kmax; hs.L[tid] = L;
        }
        // exclusive scan of P over the batch (threads 0..nq-1 live in warps 0..3)
        uint32_t inc = Pt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) hs.scan[wid] = inc;
        HS_SYNC();
        uint32_t before = 0;
        for (int w2 = 0; w2 < wid; w2++) before += hs.scan[w2];
        const uint32_t excl = before + inc - Pt;
        if (tid < nq) hs.off[tid] = excl;
        HS_SYNC();
        // batch = the leading queries whose pairs fit PAIRCAP (offsets are monotone)
        if (tid == 0) {
            int lo = 0, hi = nq;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (hs.off[mid - 1] + hs.P[mid - 1] <= (uint32_t)sd::PAIRCAP) lo = mid; else hi = mid - 1;
            }
            if (lo == 0) { atomicOr(S.err, OTF_E_VALUE); lo = 1; }   // one path longer than PAIRCAP
            hs.scan[NW] = (uint32_t)lo;
        }
        HS_SYNC();
        const int nb = (int)hs.scan[NW];
        const uint32_t T = min(hs.off[nb - 1] + hs.P[nb - 1], (uint32_t)sd::PAIRCAP);
        // pair -> query map and the context rows
        for (int t = wid; t < nb; t += NW) {
            const uint32_t o = hs.off[t], p = hs.P[t], cb = hs.cb[t];
            for (uint32_t i = lane; i < p && o + i < (uint32_t)sd::PAIRCAP; i += 32) {
                hs.pq[o + i] = (uint8_t)t;
                hs.pcode[o + i] = __ldg(m.path_code + cb + i);
            }
        }
        for (int i = tid; i < nb * NCH; i += NT) {
            const int t = i / NCH, c = i - t * NCH;
            const float4 x = __ldcg(reinterpret_cast<const float4 *>(S.arena_h + (size_t)hs.row[t] * H) + c);
            if (EXACT) {
                double2 *d2 = reinterpret_cast<double2 *>(hs.hd + (size_t)t * H + 4 * c);
                d2[0] = make_double2((double)x.x, (double)x.y);   // conversion unit (exact)
                d2[1] = make_double2((double)x.z, (double)x.w);
            } else {
                reinterpret_cast<float4 *>(hs.h)[(size_t)t * NCH + c] = x;
            }
        }
        HS_SYNC();
        HS_MARK(4);
        // ---- B: 8 pairs per warp round, 4 lanes per pair ----
        // lane = 4 * pair + sub; sub covers float4 chunks sub, sub+4, ... of H
        {
            const int pg = lane >> 2, sub = lane & 3;
            for (uint32_t j0 = (uint32_t)wid * HS_G; j0 < T; j0 += (uint32_t)NW * HS_G) {
                const uint32_t j = j0 + (uint32_t)pg;
                const bool live = j < T;
                const int t = live ? (int)hs.pq[j] : 0;
                const uint32_t code = live ? hs.pcode[j] : 0u;
                const int kmax = hs.kmax[t];
                // MaxEnt terms: lane sub < kmax gathers order sub+1 (issued first)
                double me = 0.0;
                if (live && sub < kmax)
                    me = (double)__ldg(m.ME + (otf_mix(hs.pre[t * ORD + sub], (uint64_t)(code & 0x7FFFFFFFu)) & m.mask));
                double a;
                if (EXACT) {
                    // float64 accumulation of the exact f32 x f32 products
                    // (_kernels_nb.py:66-68); the node-vector element is
                    // widened half by the conversion unit, half by integer ops
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                    if (live) {
                        const float4 *row = reinterpret_cast<const float4 *>(m.NV + (size_t)(code & 0x7FFFFFFFu) * H);
                        const double2 *hv = reinterpret_cast<const double2 *>(hs.hd + (size_t)t * H);
#pragma unroll 4
                        for (int k = sub; k < NCH; k += 4) {
                            const float4 x = __ldg(row + k);
                            const double2 h01 = hv[2 * k], h23 = hv[2 * k + 1];
                            a0 = fma((double)x.x, h01.x, a0);
                            a1 = fma(widen(x.y), h01.y, a1);
                            a2 = fma((double)x.z, h23.x, a2);
                            a3 = fma(widen(x.w), h23.y, a3);
                        }
                    }
                    a = (a0 + a1) + (a2 + a3);
                } else {
                    float f0 = 0.f, f1 = 0.f, f2 = 0.f, f3 = 0.f;
                    if (live) {
                        const float4 *row = reinterpret_cast<const float4 *>(m.NV + (size_t)(code & 0x7FFFFFFFu) * H);
                        const float4 *hv = reinterpret_cast<const float4 *>(hs.h + (size_t)t * H);
#pragma unroll 8
                        for (int k = sub; k < NCH; k += 4) {
                            const float4 x = __ldg(row + k);
                            const float4 h4 = hv[k];
                            f0 = fmaf(x.x, h4.x, f0);
                            f1 = fmaf(x.y, h4.y, f1);
                            f2 = fmaf(x.z, h4.z, f2);
                            f3 = fmaf(x.w, h4.w, f3);
                        }
                    }
                    a = ((double)f0 + (double)f1) + ((double)f2 + (double)f3);
                }
                a += __shfl_xor_sync(0xffffffffu, a, 1);
                a += __shfl_xor_sync(0xffffffffu, a, 2);
                // MaxEnt orders added in reference order (k = 1, 2, ...)
#pragma unroll
                for (int k = 0; k < (ORD < 4 ? ORD : 4); k++) {
                    const double mk = __shfl_sync(0xffffffffu, me, (lane & ~3) | k);
                    if (k < kmax) a += mk;
                }
                if (ORD > 4) {                       // orders 5..7 (rare): leader gathers them
                    for (int k = 4; k < kmax; k++)
                        a += (double)__ldg(m.ME + (otf_mix(hs.pre[t * ORD + k], (uint64_t)(code & 0x7FFFFFFFu)) & m.mask));
                }
                if (live && sub == 0) hs.lsig[j] = (code & 0x80000000u) ? -a : a;
            }
        }
        HS_SYNC();
        HS_MARK(5);
        // log-sigmoid once per pair with every lane busy (f64, libdevice)
        for (uint32_t j = (uint32_t)tid; j < T; j += NT) hs.lsig[j] = otf_log_sigmoid(hs.lsig[j]);
        HS_SYNC();
        // ---- C: per query: path-order sum, successor history, digest ----
        // thread per query: path-order sum, successor history (rnnlm.py:187),
        // its digest terms (same values as hs_prim_finish)
        if (tid < nb) {
            const int t = tid;
            const uint32_t q = q0 + (uint32_t)t;
            const uint32_t o = hs.off[t], p = hs.P[t];
            double lp = 0.0;
            for (uint32_t i = 0; i < p; i++) lp += hs.lsig[o + i];
            const uint32_t *meta = S.arena_meta + (size_t)hs.row[t] * OTF_META;
            const int L = hs.L[t];
            const int nl = L + 1 > m.order ? m.order : L + 1;
            const int drop = L + 1 - nl;
            uint32_t *dst = S.arena_meta + (size_t)(base + q) * OTF_META;
            unsigned long long dg = 0ull;
#pragma unroll
            for (int k = 0; k < OTF_META; k++) {
                uint32_t v = 0;
                if (k == 0) v = (uint32_t)nl;
                else if (k < nl) v = meta[k + drop];
                else if (k == nl) v = (uint32_t)hs.w[t];
                dst[k] = v;
                dg += dig_meta(k, v);
            }
            atomicAdd(&Q.pr_dig[q], dg);
            Q.pr_p[q] = lp;
            if (Q.alg) {
                const int km = m.order < L ? m.order : L;
                atomicAdd(&Q.alg[0], (unsigned long long)p);
                atomicAdd(&Q.alg[1], (unsigned long long)p * km);
                atomicAdd(&Q.alg[2], 1ull);
            }
        }
        HS_SYNC();
        q0 += (uint32_t)nb;
    }
#undef HS_MARK
#undef HS_SYNC
}

// MODE 1 = TF32X3, 3 = TF32; KC_B = m.wt_kcb; CPL/ORD as RING_DISPATCH.
// A cluster of two CTAs per stream: rank 0 (control) runs expand, the
// small-LM scores + HS and assign; rank 1 (update) runs the tcgen05 recurrent
// update and its epilogue.  Per level:
//   rank 0: expand -> rows -> [cluster barrier A] -> small-LM + HS -> [B] -> assign
//   rank 1:                   [A] -> update + epilogue                 -> [B]
// The row count / arena base / abort flag cross over DSMEM after A; every
// global write before a barrier is visible after it (release / acquire at
// cluster scope).  Each role has a whole SM: 16 warps and the full shared
// memory (4-stage update ring on rank 1, single-batch HS staging on rank 0).
template <int MODE, int KC_B, int CPL, int ORD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(sd::NT, 1)
k_decode_streams(DevModel m, DevPlan P, DevStreams S, DevNgram g, long long beam, double lm_weight, int stages,
                 int qb_max, uint32_t *cursor, uint32_t row_limit, uint32_t tmem_cols, uint8_t *xscratch,
                 size_t xs_stride, uint32_t x_epoch, int x_stage_u) {
    using namespace tc;
    namespace cg = cooperative_groups;
    constexpr bool X3 = MODE == 1;
    constexpr bool EXACT = MODE == 4;       // integer digit-plane update + float64 HS (bit-exact)
    constexpr int NT = sd::NT, NW = sd::NW;
    constexpr int KE = KC_B / 4;            // tf32 elements of K per chunk
    constexpr int CH = KC_B / 16;           // 16-byte pieces per row per chunk
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t e_ctx[NW][32], e_slot[NW][32], e_arc[NW][32];
    __shared__ double e_score[NW][32];
    __shared__ unsigned long long a_key[NT];
    __shared__ uint32_t a_row[NT], a_cn[NT], a_wsum[NW], a_cnt[4];
    __shared__ __align__(8) uint64_t bar_full[4], bar_empty[4], bar_done;
    __shared__ uint32_t s_tmem, s_nprim, s_base, s_abort;

    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);     // provably warp-uniform
    const uint32_t u = blockIdx.x >> 1;                        // stream of this cluster
    const int H = m.H;
    const int nmt = m.wt_npad / BM;                            // M tiles of output units
    const uint32_t wa_bytes = (uint32_t)m.wt_npad * KC_B;      // one W block (hi or lo)
    const uint32_t hb_bytes = BM * KC_B;                       // one row block (hi or lo)
    const uint32_t stage_bytes = (X3 ? 2u : 1u) * (wa_bytes + hb_bytes);
    const int NK = (H + KE - 1) / KE;

    if (tid == 0) {
        for (int st = 0; st < (EXACT ? 4 : stages); st++) {   // EXACT rank 0: [0, 2) HS ring, [2, 4) its update share
            // TF32: loader warps (+ W copy); EXACT rank 1: one bulk producer;
            // EXACT rank 0 (HS): the A-row gather threads + the B bulk copy
            mbar_init(smem_u32(&bar_full[st]), EXACT ? (rank == 0 && st < xh::STAGES ? xh::GT + 1 : 1) : NW);
            mbar_init(smem_u32(&bar_empty[st]), 1);
        }
        mbar_init(smem_u32(&bar_done), 1);
        s_abort = 0;
        if (EXACT && rank == 1) {                          // deferred-fallback counters (xu::Ring::fb_n)
            uint32_t *fbn = reinterpret_cast<uint32_t *>(smem + (size_t)stages * xu::STAGE + xu::tail_layout().fbn);
            fbn[0] = 0u; fbn[1] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (EXACT && rank == 1 && tid < 32) {                  // exp_neg's 2^(j/32) table (xu::Ring::tab)
        double *tab = reinterpret_cast<double *>(smem + (size_t)stages * xu::STAGE + xu::tail_layout().tab);
        tab[tid] = exp2((double)tid / 32.0);
    }
    uint32_t tmem = 0;
    if ((rank == 1 || EXACT) && wid == 0) {                // EXACT: both ranks run tensor-core GEMMs
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&s_tmem)), "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 1 || EXACT) tmem = s_tmem;
    // rank 0's row count / base / abort flag, read by rank 1 over DSMEM
    const uint32_t *r0_nprim = cluster.map_shared_rank(&s_nprim, 0);
    const uint32_t *r0_base = cluster.map_shared_rank(&s_base, 0);
    const uint32_t *r0_abort = cluster.map_shared_rank(&s_abort, 0);

    // this utterance's request / primary workspace
    DevPlan Q = P;
    if (u < P.n_utt) {
        const uint32_t o = P.rq_off[u];
        Q.rq_c += o; Q.rq_arc += o; Q.rq_parent += o; Q.rq_cslot += o; Q.rq_m += o; Q.rq_dslot += o;
        Q.rq_w += o; Q.rq_state += o; Q.rq_score += o; Q.rq_slm += o; Q.rq_ps += o;
        Q.pr_req += o; Q.pr_inrow += o; Q.pr_w += o; Q.pr_p += o; Q.pr_dig += o;
    }
    const uint32_t sid = u < P.n_utt ? P.utt_stream[u] : 0u;
    // assign's chunk dedup hash lives in rank 0's dynamic shared memory (the HS
    // staging area, idle while assign runs): 2 NT keys + 2 NT threads + NT slots
    const AssignSmem asmem{a_key, a_row, a_cn, a_wsum, a_cnt, reinterpret_cast<unsigned long long *>(smem),
                           reinterpret_cast<uint32_t *>(smem + 16 * NT), reinterpret_cast<uint32_t *>(smem + 24 * NT)};
    uint32_t gctr = 0;          // K chunks through the ring so far (rank 1, uniform)
    uint32_t gctr_u = 0;        // EXACT rank 0: K chunks of its update share (barriers [2, 4))
    uint32_t tiles_done = 0;
    // EXACT: M tiles of output units, and how many of them rank 0 takes
    // (H > 384: rank 0 has spare time after the HS, so the last tile moves there)
    const int x_nmt = (H + BM - 1) / BM;
    const int x_r0_tiles = (EXACT && x_nmt >= 4) ? 1 : 0;
    // node-parallel HS scratch (rank 0): the whole dynamic shared memory
    sd::HsLevelSmem hsm;
    {
        uint8_t *p = smem + (size_t)qb_max * (EXACT ? 8 : 4) * H;
        hsm.h = reinterpret_cast<float *>(smem);
        hsm.hd = reinterpret_cast<double *>(smem);
        hsm.lsig = reinterpret_cast<double *>(p); p += sd::PAIRCAP * 8;
        hsm.pcode = reinterpret_cast<uint32_t *>(p); p += sd::PAIRCAP * 4;
        hsm.pre = reinterpret_cast<unsigned long long *>(p); p += sd::QMAX * ORD * 8;
        hsm.row = reinterpret_cast<uint32_t *>(p); p += sd::QMAX * 4;
        hsm.cb = reinterpret_cast<uint32_t *>(p); p += sd::QMAX * 4;
        hsm.off = reinterpret_cast<uint32_t *>(p); p += sd::QMAX * 4;
        hsm.P = reinterpret_cast<uint32_t *>(p); p += sd::QMAX * 4;
        hsm.w = reinterpret_cast<int32_t *>(p); p += sd::QMAX * 4;
        hsm.kmax = reinterpret_cast<int32_t *>(p); p += sd::QMAX * 4;
        hsm.L = reinterpret_cast<int32_t *>(p); p += sd::QMAX * 4;
        hsm.scan = reinterpret_cast<uint32_t *>(p); p += (NW + 2) * 4;
        hsm.pq = p;
    }

    // profiling runs only: per-phase device time (ns), summed over streams
    // (thread 0 of each rank marks its own phases)
    unsigned long long ph[28] = {0}, t0 = 0, t1 = 0;
    const bool prof = P.phase_ns != nullptr && tid == 0;
#define SD_MARK(i) do { if (prof) { t1 = sd::gtimer(); ph[i] += t1 - t0; t0 = t1; } } while (0)
    if (prof) t0 = sd::gtimer();
    const uint32_t l_begin = u < P.n_utt ? P.ul_off[u] : 0u, l_end = u < P.n_utt ? P.ul_off[u + 1] : 0u;
    for (uint32_t li = l_begin; li < l_end; li++) {
        const UttLevel L = P.ul[li];
        uint32_t n = 0, base = 0;
        bool abort = false;
        if (rank == 0) {
            if (tid == 0) s_nprim = 0;
            __syncthreads();
            // ---------------- expand ----------------
            for (uint32_t k = L.nb + wid; k < L.ne; k += NW) {
                const NodeInfo nd = P.nodes[P.level_nodes[k]];
                expand_node(Q, S, g, nd, beam, L.t, -(int64_t)L.rb, &s_nprim, e_ctx[wid], e_slot[wid], e_score[wid],
                            e_arc[wid], lane, /*defer_ps=*/true);
            }
            __syncthreads();
            n = s_nprim;
            if (tid == 0) {
                uint32_t b = 0;
                if (n) b = atomicAdd(cursor, n);
                if ((uint64_t)b + n > row_limit) { atomicOr(S.err, OTF_E_ARENA_FULL); s_abort = 1; }
                s_base = b;
            }
            SD_MARK(0);
        }
        cluster.sync();                                      // A: rows reserved, requests compacted
        if (rank == 0) { n = s_nprim; base = s_base; abort = s_abort != 0; }
        else { n = *r0_nprim; base = *r0_base; abort = *r0_abort != 0; if (prof) t0 = sd::gtimer(); }
        if (abort) break;
        if (rank == 0 && EXACT) {
            // HS on this CTA's tensor core, chunk by chunk in step with rank 1's
            // update (the chunk's h digit planes are shared through the scratch)
            constexpr int HS_NT = NT - 64;
            const xh::Smem xs_m = xh::carve(smem, ORD);
            const uint32_t eh_off = (uint32_t)stages * xu::STAGE + xu::tail_layout().eh;
            // a level whose requests all hit the cache (retained streams) computes
            // nothing, but assign still needs every request's small-LM score
            if (n == 0) small_lm_scores(Q, S, g, sid, L.re - L.rb, tid, NT);
            for (uint32_t q0 = 0, c = 0; q0 < n; q0 += xu::XR, c++) {
                const int nq = (int)min((uint32_t)xu::XR, n - q0);
                if (tid < HS_NT) xh::setup<ORD, HS_NT>(m, Q, S, q0, nq, xs_m, tid, lane);
                __syncthreads();
                SD_MARK(4);
                cluster.sync();                              // D: rank 1 digitized chunk c
                const double *eh_r = cluster.map_shared_rank(reinterpret_cast<double *>(smem + eh_off), 1) +
                                     (c & 1) * xu::XR;
                SD_MARK(21);
                xh::run<ORD, NT>(m, Q, S, base, q0, nq, xscratch + (size_t)u * xs_stride + (c & 1) * xu::xs_slot_bytes(m.wd_nkx),
                                 eh_r, smem, xs_m, tmem, bar_full, bar_empty, &bar_done, gctr, tiles_done, tid, wid, lane,
                                 [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); },
                                 [&](int t2, int nt2) {   // the level's small-LM scores, under the first GEMM
                                     if (c == 0) small_lm_scores(Q, S, g, sid, L.re - L.rb, t2, nt2);
                                 },
                                 prof ? ph : nullptr, t0);
                SD_MARK(5);
                if (x_r0_tiles) {
                    // this CTA's share of the recurrent update: the last M tile(s)
                    constexpr xh::UpdOverlay ov = xh::upd_overlay();
                    uint8_t *ob = reinterpret_cast<uint8_t *>(xs_m.hkey);
                    xu::Ring rg;
                    rg.smem = smem; rg.stages = xh::STAGES; rg.tmem = tmem;
                    rg.full = bar_full + xh::STAGES; rg.empty = bar_empty + xh::STAGES; rg.done = &bar_done;
                    rg.fb = reinterpret_cast<uint32_t *>(ob + ov.fb);
                    rg.fb_n = reinterpret_cast<uint32_t *>(ob + ov.fbn);
                    rg.eh = reinterpret_cast<double *>(ob + ov.eh);
                    rg.sh = rg.eh;
                    rg.src = reinterpret_cast<int32_t *>(ob + ov.src);
                    rg.wrd = reinterpret_cast<int32_t *>(ob + ov.wrd);
                    rg.tab = reinterpret_cast<const double *>(ob + ov.tab);
                    rg.xs = xscratch + (size_t)u * xs_stride;
                    rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
                    for (int i = tid; i < nq; i += NT) rg.eh[i] = eh_r[i];
                    if (tid < 32) const_cast<double *>(rg.tab)[tid] = exp2((double)tid / 32.0);
                    if (tid < 2) rg.fb_n[tid] = 0u;
                    // (visible after update_chunk's first barrier)
                    rg.hin = S.arena_h; rg.hout = S.arena_h + (size_t)base * H; rg.in_row = Q.pr_inrow;
                    rg.words = Q.pr_w; rg.dig = Q.pr_dig; rg.alg = Q.alg;
                    rg.dig_store = nullptr; rg.deh_store = nullptr; rg.dep_store = nullptr; rg.epoch = 0;
                    rg.us = nullptr;
                    xu::update_chunk<NT>(m, q0, nq, (int)c, rg, gctr_u, tiles_done, tid, wid, lane,
                                         [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); },
                                         []() {}, prof ? ph : nullptr, t0, x_nmt - x_r0_tiles, x_nmt, false);
                }
            }
            SD_MARK(6);
        } else if (rank == 0) {
            // warps 0..13: HS (named barrier 1); warps 14, 15: the small-LM
            // scores of the level's requests (they only feed assign) alongside
            constexpr int HS_NT = NT - 64;
            if (tid < HS_NT) {
                if (n) hs_level_nodepar<CPL, ORD, HS_NT, 1, EXACT>(m, Q, S, base, n, hsm, qb_max, tid, wid, lane,
                                                             prof ? ph : nullptr);
            } else {
                small_lm_scores(Q, S, g, sid, L.re - L.rb, tid - HS_NT, NT - HS_NT);
            }
            SD_MARK(6);
        } else if (n && EXACT) {
            // ------------- exact recurrent update (tcgen05 kind::i8) -------------
            xu::Ring rg;
            rg.smem = smem; rg.stages = stages; rg.tmem = tmem;
            rg.full = bar_full; rg.empty = bar_empty; rg.done = &bar_done;
            uint8_t *tail = smem + (size_t)stages * xu::STAGE;
            constexpr xu::TailLayout tl = xu::tail_layout();
            rg.fb = reinterpret_cast<uint32_t *>(tail + tl.fb);
            rg.sh = reinterpret_cast<double *>(tail + tl.sh);
            rg.eh = reinterpret_cast<double *>(tail + tl.eh);
            rg.fb_n = reinterpret_cast<uint32_t *>(tail + tl.fbn);
            rg.src = reinterpret_cast<int32_t *>(tail + tl.src);
            rg.wrd = reinterpret_cast<int32_t *>(tail + tl.wrd);
            rg.tab = reinterpret_cast<const double *>(tail + tl.tab);
            rg.xs = xscratch + (size_t)u * xs_stride;
            rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
            rg.us = x_stage_u ? reinterpret_cast<float *>(tail + tl.total) : nullptr;
            rg.hin = S.arena_h; rg.hout = S.arena_h + (size_t)base * H; rg.in_row = Q.pr_inrow;
            rg.words = Q.pr_w; rg.dig = Q.pr_dig; rg.alg = Q.alg;
            rg.dig_store = S.arena_dig; rg.deh_store = S.arena_deh; rg.dep_store = S.arena_dep; rg.epoch = x_epoch;
            for (uint32_t q0 = 0, c = 0; q0 < n; q0 += xu::XR, c++)
                xu::update_chunk<NT>(m, q0, (int)min((uint32_t)xu::XR, n - q0), (int)c, rg, gctr, tiles_done,
                                     tid, wid, lane, [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); },
                                     [&]() { cluster.sync(); }, prof ? ph : nullptr, t0, 0, x_nmt - x_r0_tiles, true);
        } else if (n) {
            // ------------- recurrent update (tcgen05) -------------
            for (uint32_t q0 = 0; q0 < n; q0 += BM) {
                const int nr = (int)min((uint32_t)BM, n - q0);
                const int nn = (nr + 15) & ~15;                   // MMA N
                const int nitems = ((nr + 7) & ~7) * CH;          // row pieces per chunk
                // warp 0: MMA issuer (converged; lane 0 issues).  Warps 1..NW-1:
                // loaders / converters -- a divergent issuer inside a loader
                // warp would sit behind its siblings' suspended mbarrier waits.
                constexpr int LT = NT - 32;                        // loader threads (warps 1..NW-1)
                const int ltid = tid - 32;
                auto issue = [&](int st, uint32_t use, int kc) {
                    if (use >= 1) sd::wait_bounded(smem_u32(&bar_empty[st]), (use - 1) & 1, 1);
                    __syncwarp();                                // lanes leave the wait independently
                    uint8_t *sW = smem + st * stage_bytes;
                    uint8_t *sH = sW + (X3 ? 2 : 1) * wa_bytes;
                    if (wid == 1) {                              // W chunk: one bulk copy, elected lane
                        const uint32_t bytes = (X3 ? 2u : 1u) * wa_bytes;
                        const void *src = reinterpret_cast<const uint8_t *>(m.W_t) + (size_t)kc * 2 * wa_bytes;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                                     "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n\t"
                                     "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t}"
                                     :: "r"(smem_u32(sW)), "r"(smem_u32(&bar_full[st])), "l"(src), "r"(bytes) : "memory");
                    }
                    const int k0 = kc * KE;
                    for (int idx = ltid; idx < nitems; idx += LT) {
                        const int r8 = idx & 7, c = (idx >> 3) % CH, g8 = idx / (8 * CH);
                        const int row = g8 * 8 + r8;
                        if (row >= nr) continue;
                        const int kk = k0 + c * 4;
                        const bool ok = kk < H;
                        const int src = Q.pr_inrow[q0 + row];
                        cp_async16(smem_u32(sH + swz_off<KC_B>(row, c)),
                                   ok ? (const void *)(S.arena_h + (size_t)src * H + kk) : (const void *)S.arena_h, ok);
                    }
                    cp_async_commit();
                };
                auto consume = [&](int st, int pending) {
                    sd::cp_wait_n(pending);
                    uint8_t *sH = smem + st * stage_bytes + (X3 ? 2 : 1) * wa_bytes;
                    for (int idx = ltid; idx < nitems; idx += LT) {
                        const int r8 = idx & 7, c = (idx >> 3) % CH, g8 = idx / (8 * CH);
                        const int row = g8 * 8 + r8;
                        if (row >= nr) continue;
                        const uint32_t off = swz_off<KC_B>(row, c);
                        const float4 x = *reinterpret_cast<const float4 *>(sH + off);
                        float4 hi;
                        hi.x = tf32_rn(x.x); hi.y = tf32_rn(x.y); hi.z = tf32_rn(x.z); hi.w = tf32_rn(x.w);
                        *reinterpret_cast<float4 *>(sH + off) = hi;
                        if (X3) {
                            float4 lo;
                            lo.x = tf32_rn(x.x - hi.x); lo.y = tf32_rn(x.y - hi.y);
                            lo.z = tf32_rn(x.z - hi.z); lo.w = tf32_rn(x.w - hi.w);
                            *reinterpret_cast<float4 *>(sH + hb_bytes + off) = lo;
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&bar_full[st])) : "memory");
                };
                if (wid == 0) {
                    const uint32_t idesc = make_idesc(2, nn);
                    for (int kc = 0; kc < NK; kc++) {
                        const int st = (int)((gctr + kc) % (uint32_t)stages);
                        const uint32_t use = (gctr + kc) / (uint32_t)stages;
                        const unsigned long long w0 = prof ? sd::gtimer() : 0ull;
                        sd::wait_bounded(smem_u32(&bar_full[st]), use & 1, 2);
                        __syncwarp();                            // elect.sync below needs a converged warp
                        if (prof) ph[9] += sd::gtimer() - w0;
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        {
                            const uint32_t sW = smem_u32(smem + st * stage_bytes);
                            const uint32_t sWlo = sW + wa_bytes;
                            const uint32_t sH = sW + (X3 ? 2 : 1) * wa_bytes;
                            const uint32_t sHlo = sH + hb_bytes;
#pragma unroll
                            for (int ks = 0; ks < KC_B / 32; ks++) {     // 8 tf32 (32 B) of K per MMA
                                const uint64_t b_hi = make_desc_sw<KC_B>(sH + ks * 32);
                                const uint64_t b_lo = make_desc_sw<KC_B>(sHlo + ks * 32);
                                for (int mt = 0; mt < nmt; mt++) {
                                    const uint32_t d = tmem + (uint32_t)(mt * BM);
                                    const uint32_t mo = (uint32_t)mt * BM * KC_B;
                                    const uint64_t a_hi = make_desc_sw<KC_B>(sW + mo + ks * 32);
                                    mma_elect<false>(d, a_hi, b_hi, idesc, (kc > 0 || ks > 0) ? 1u : 0u);
                                    if (X3) {
                                        const uint64_t a_lo = make_desc_sw<KC_B>(sWlo + mo + ks * 32);
                                        mma_elect<false>(d, a_hi, b_lo, idesc, 1u);
                                        mma_elect<false>(d, a_lo, b_hi, idesc, 1u);
                                    }
                                }
                            }
                            commit_elect(smem_u32(&bar_empty[st]));
                            if (kc == NK - 1) commit_elect(smem_u32(&bar_done));
                        }
                        __syncwarp();
                    }
                } else {
                    const int pre = min(stages - 1, NK);
                    for (int j = 0; j < pre; j++) {
                        const uint32_t gc = gctr + j;
                        issue((int)(gc % (uint32_t)stages), gc / (uint32_t)stages, j);
                    }
                    for (int kc = 0; kc < NK; kc++) {
                        const uint32_t gc = gctr + kc;
                        consume((int)(gc % (uint32_t)stages), min(stages - 2, NK - 1 - kc));
                        if (kc + stages - 1 < NK) {
                            const uint32_t gi = gc + stages - 1;
                            issue((int)(gi % (uint32_t)stages), gi / (uint32_t)stages, kc + stages - 1);
                        }
                    }
                }
                gctr += NK;
                if (tid == 0) SD_MARK(1);
                // epilogue: TMEM lane = output unit, column = row of the tile
                sd::wait_bounded(smem_u32(&bar_done), tiles_done & 1, 3);
                if (tid == 0) SD_MARK(2);
                tiles_done++;
                __syncwarp();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                {
                    // work items = (M tile, group of 8 rows): the 4 warps of a TMEM
                    // lane quadrant share a tile's rows 8 at a time.  The 8 U loads
                    // of a group are in flight together and the group's digest
                    // terms are reduced with the 9-exchange reduce8 pattern (the
                    // sum for row g lands on the lanes whose bits 4,3,2 spell g).
                    const int quad = wid & 3;
                    const int n8 = (nr + 7) / 8;
                    for (int it = wid >> 2; it < nmt * n8; it += NW / 4) {
                        const int mt = it / n8, r0 = (it - mt * n8) * 8;
                        const int unit = mt * BM + quad * 32 + lane;
                        float v[8];
                        tmem_ld8(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mt * BM + r0), v);
                        const int wl = lane < 8 && r0 + lane < nr ? Q.pr_w[q0 + r0 + lane] : 0;
                        const float *ucol = m.U + unit;
                        float *ocol = S.arena_h + (size_t)(base + q0 + r0) * H + unit;
                        float uv[8];
#pragma unroll
                        for (int g = 0; g < 8; g++) {
                            const int wq = __shfl_sync(0xffffffffu, wl, g);
                            uv[g] = (r0 + g < nr && unit < H) ? __ldg(ucol + (size_t)wq * H) : 0.f;
                        }
                        unsigned long long dg[8];
#pragma unroll
                        for (int g = 0; g < 8; g++) {
                            dg[g] = 0ull;
                            if (r0 + g < nr && unit < H) {
                                const float o = __frcp_rn(1.f + expf(-(v[g] + uv[g])));   // == 1/x, IEEE
                                ocol[(size_t)g * H] = o;
                                dg[g] = otf_dig_h((uint32_t)unit, o);
                            }
                        }
                        const unsigned long long tot = sd::reduce8_u64(dg, lane);
                        const int row = r0 + node_of_lane(lane);
                        if ((lane & 3) == 0 && row < nr) atomicAdd(&Q.pr_dig[q0 + row], tot);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncthreads();
                if (tid == 0) SD_MARK(3);
            }
        }
        cluster.sync();                                      // B: h', p and digests complete
        if (rank == 1) {
            // EXACT: the digit planes of the level's new rows, while rank 0
            // runs assign and the next expand (off the per-level critical path)
            if (EXACT && n && S.arena_dig)
                xu::digitize_to_store<NT>(m, S.arena_h, base, n, S.arena_dig, S.arena_deh, S.arena_dep, x_epoch,
                                          tid, wid, lane);
            continue;
        }
        SD_MARK(8);                                          // control waits for the update
        // ---------------- assign (rank 0) ----------------
        const StreamRange rg{sid, 0u, L.re - L.rb, 0u};
        const LevelCtr lc{n, base, 0u, 0u};
        assign_range<0, NT>(Q, S, L.t, rg, lc, row_limit, lm_weight, nullptr, nullptr, nullptr, asmem,
                            P.phase_ns ? P.phase_ns + 16 : nullptr);
        __syncthreads();
        SD_MARK(7);
    }
    if (prof) {
        ph[11] = rank == 0 ? 1 : 0;
        for (int i = 0; i < 28; i++) if (ph[i] && (i < 16 || i > 20)) atomicAdd(&P.phase_ns[i], ph[i]);
    }
#undef SD_MARK
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if ((rank == 1 || EXACT) && wid == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(tmem_cols));
    cluster.sync();                                          // rank 0's shared memory outlives rank 1's reads
}

// --------------------------------------------------------------------------
// The EXACT recurrent update as a batch (level schedule, two-pass, Table-1
// batch and the kernel-table API): persistent CTAs over 80-row chunks of the
// n rows, each with its own two-slot digit scratch, running the same
// xu::update_chunk as the stream kernel (digitize, digit-pair K loops over
// every M tile, certifying epilogue, reference-loop fallbacks).
// Row q: source hin[in_row[q]], word words[q] (nullptr: q), result
// out_base[row_base(rs) + q]; digest terms into rs.dig[q] when set.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(sd::NT, 1)
k_advance_exact(DevModel m, uint32_t n_cap, RowSpec rs, const int32_t *__restrict__ in_row,
                const int32_t *__restrict__ words, const float *__restrict__ h_base, float *__restrict__ out_base,
                uint8_t *xscratch, size_t xs_stride, int stages, unsigned long long *alg) {
    using namespace tc;
    constexpr int NT = sd::NT;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[4], bar_empty[4], bar_done;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const uint32_t n = rs.n_dev ? *rs.n_dev : n_cap;
    const uint32_t out0 = row_base(rs);
    if (rs.cur && blockIdx.x == 0 && tid == 0) rs.cur->base = out0;
    if ((uint64_t)out0 + n > rs.row_limit) return;      // arena overflow (flagged by the HS stage)
    const uint32_t nch = (n + xu::XR - 1) / xu::XR;
    if (blockIdx.x >= nch) return;
    constexpr xu::TailLayout tl = xu::tail_layout();
    uint8_t *tail = smem + (size_t)stages * xu::STAGE;
    if (tid == 0) {
        for (int st = 0; st < stages; st++) { mbar_init(smem_u32(&bar_full[st]), 1); mbar_init(smem_u32(&bar_empty[st]), 1); }
        mbar_init(smem_u32(&bar_done), 1);
        reinterpret_cast<uint32_t *>(tail + tl.fbn)[0] = 0u;
        reinterpret_cast<uint32_t *>(tail + tl.fbn)[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) reinterpret_cast<double *>(tail + tl.tab)[tid] = exp2((double)tid / 32.0);
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    xu::Ring rg;
    rg.smem = smem; rg.stages = stages; rg.tmem = s_tmem;
    rg.full = bar_full; rg.empty = bar_empty; rg.done = &bar_done;
    rg.fb = reinterpret_cast<uint32_t *>(tail + tl.fb);
    rg.sh = reinterpret_cast<double *>(tail + tl.sh);
    rg.eh = reinterpret_cast<double *>(tail + tl.eh);
    rg.fb_n = reinterpret_cast<uint32_t *>(tail + tl.fbn);
    rg.src = reinterpret_cast<int32_t *>(tail + tl.src);
    rg.wrd = reinterpret_cast<int32_t *>(tail + tl.wrd);
    rg.tab = reinterpret_cast<const double *>(tail + tl.tab);
    rg.xs = xscratch + (size_t)blockIdx.x * xs_stride;
    rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
    rg.hin = h_base; rg.hout = out_base + (size_t)out0 * m.H; rg.in_row = in_row; rg.words = words;
    rg.dig = rs.dig; rg.alg = alg;
    rg.dig_store = nullptr; rg.deh_store = nullptr; rg.dep_store = nullptr; rg.epoch = 0;
    rg.us = nullptr;
    const int nmt = (m.H + BM - 1) / BM;
    uint32_t gctr = 0, tiles_done = 0;
    unsigned long long t0 = 0;
    int local = 0;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x, local++) {
        const uint32_t q0 = c * xu::XR;
        xu::update_chunk<NT>(m, q0, (int)min((uint32_t)xu::XR, n - q0), local, rg, gctr, tiles_done, tid, wid, lane,
                             [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); },
                             []() { __syncthreads(); }, nullptr, t0, 0, nmt, true);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(rg.tmem), "r"(512));
}

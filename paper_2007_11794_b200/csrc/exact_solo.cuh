// exact_solo.cuh -- the EXACT persistent decode with ONE CTA per utterance
// stream (schedule OTFLM_SCHED_STREAM1), for batches of at least one stream
// per SM (config e: 148 streams per batch).
//
// The 2-CTA cluster of k_decode_streams overlaps a level's HS (rank 0) with
// its recurrent update (rank 1), but each SM idles part of every level
// (rank 1 through expand and assign, rank 0 at the level barrier).  When the
// batch has a stream for every SM, running the whole chain on one SM wastes
// nothing: per level
//   expand -> plane copy of the level's context rows -> HS digit-plane GEMM
//   (+ small-LM scores on two warps under it) -> update digit-plane GEMMs over
//   every M tile -> planes of the new rows -> assign,
// with the same device functions as the cluster kernel (expand_node,
// xu::update_chunk, xh::setup / xh::run, xu::digitize_to_store,
// assign_range), one TMEM allocation shared by the HS and update
// accumulators in turn, and no cluster barriers.
//
// Shared memory: [ring: 2 stages x xu::STAGE][xh tables | (update fallback
// lists + staged U block, overlaid once the HS of the chunk is done)]
// [small: sh, eh (x2 by chunk parity), fb_n, src, wrd, exp table].
#pragma once
#include "stream_decode.cuh"

namespace xs1 {
struct Small { uint32_t sh, eh, fbn, src, wrd, tab, total; };
__host__ __device__ constexpr Small small_layout() {
    return Small{0u, 2u * xu::XR * 8, 4u * xu::XR * 8, 4u * xu::XR * 8 + 16, 4u * xu::XR * 8 + 16 + xu::XR * 4,
                 4u * xu::XR * 8 + 16 + 2u * xu::XR * 4, 4u * xu::XR * 8 + 16 + 2u * xu::XR * 4 + 32 * 8};
}
// the update's fallback lists live on the HS node-dedup hash (idle after
// xh::setup); its U staging block on the HS pair tables from the second M
// tile on (the HS tail runs under the first tile's K loop)
static_assert(2u * xu::FBCAP * 4 <= (uint32_t)xh::HCAP * 6, "fallback lists exceed the dedup hash");
static_assert(xu::US_BYTES <= xh::layout(3).hkey, "U staging block overlaps the dedup hash");
__host__ __device__ constexpr uint32_t overlay_bytes() { return xu::US_BYTES; }
__host__ __device__ constexpr uint32_t tables_bytes(int ord) {
    return xh::layout(ord).total > overlay_bytes() ? xh::layout(ord).total : overlay_bytes();
}
__host__ __device__ constexpr uint32_t smem_bytes(int ord) {
    return xh::ring_bytes() + ((tables_bytes(ord) + 127u) & ~127u) + small_layout().total;
}
}  // namespace xs1

template <int ORD>
__global__ void __launch_bounds__(sd::NT, 1)
k_decode_solo(DevModel m, DevPlan P, DevStreams S, DevNgram g, long long beam, double lm_weight, uint32_t *cursor,
              uint32_t row_limit, uint8_t *xscratch, size_t xs_stride, uint32_t x_epoch, uint32_t *work) {
    using namespace tc;
    constexpr int NT = sd::NT, NW = sd::NW;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t e_ctx[NW][32], e_slot[NW][32], e_arc[NW][32];
    __shared__ double e_score[NW][32];
    __shared__ unsigned long long a_key[NT];
    __shared__ uint32_t a_row[NT], a_cn[NT], a_wsum[NW], a_cnt[4];
    __shared__ __align__(8) uint64_t bar_full[4], bar_empty[4], bar_done;
    __shared__ uint32_t s_tmem, s_nprim, s_base, s_abort, s_u;
    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int H = m.H;
    const int nmt = (H + BM - 1) / BM;
    uint8_t *tables = smem + xh::ring_bytes();
    uint8_t *small = tables + ((xs1::tables_bytes(ORD) + 127u) & ~127u);
    constexpr xs1::Small sl = xs1::small_layout();
    if (tid == 0) {
        for (int st = 0; st < 4; st++) {           // [0, 2): HS ring (gather threads + B copy), [2, 4): update ring
            mbar_init(smem_u32(&bar_full[st]), st < xh::STAGES ? xh::GT + 1 : 1);
            mbar_init(smem_u32(&bar_empty[st]), 1);
        }
        mbar_init(smem_u32(&bar_done), 1);
        s_abort = 0;
        reinterpret_cast<uint32_t *>(small + sl.fbn)[0] = 0u;
        reinterpret_cast<uint32_t *>(small + sl.fbn)[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) reinterpret_cast<double *>(small + sl.tab)[tid] = exp2((double)tid / 32.0);
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    const AssignSmem asmem{a_key, a_row, a_cn, a_wsum, a_cnt, reinterpret_cast<unsigned long long *>(smem),
                           reinterpret_cast<uint32_t *>(smem + 16 * NT), reinterpret_cast<uint32_t *>(smem + 24 * NT)};
    const xh::Smem hs = xh::carve(smem, ORD);
    // the update's ring state: the shared ring smem, barriers [2, 4)
    xu::Ring rg;
    rg.smem = smem; rg.stages = xh::STAGES; rg.tmem = tmem;
    rg.full = bar_full + xh::STAGES; rg.empty = bar_empty + xh::STAGES; rg.done = &bar_done;
    rg.fb = reinterpret_cast<uint32_t *>(tables + xh::layout(ORD).hkey);
    rg.us = reinterpret_cast<float *>(tables);      // overlay, from the second M tile (the HS tail is done)
    rg.sh = reinterpret_cast<double *>(small + sl.sh);
    rg.eh = reinterpret_cast<double *>(small + sl.eh);
    rg.fb_n = reinterpret_cast<uint32_t *>(small + sl.fbn);
    rg.src = reinterpret_cast<int32_t *>(small + sl.src);
    rg.wrd = reinterpret_cast<int32_t *>(small + sl.wrd);
    rg.tab = reinterpret_cast<const double *>(small + sl.tab);
    rg.xs = xscratch + (size_t)blockIdx.x * xs_stride;
    rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
    rg.hin = S.arena_h;
    rg.dig_store = S.arena_dig; rg.deh_store = S.arena_deh; rg.dep_store = S.arena_dep; rg.epoch = x_epoch;
    uint32_t gctr_h = 0, gctr_u = 0, tiles_done = 0;
    auto wait = [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); };

    unsigned long long ph[28] = {0}, t0 = 0, t1 = 0;
    const bool prof = P.phase_ns != nullptr && tid == 0;
#define SO_MARK(i) do { if (prof) { t1 = sd::gtimer(); ph[i] += t1 - t0; t0 = t1; } } while (0)
    if (prof) t0 = sd::gtimer();
    // persistent: each CTA takes the batch's streams from a queue, so a long
    // utterance does not hold the launch while the other SMs idle
    for (;;) {
    if (tid == 0) s_u = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t u = s_u;
    if (u >= P.n_utt) break;
    DevPlan Q = P;
    {
        const uint32_t o = P.rq_off[u];
        Q.rq_c += o; Q.rq_arc += o; Q.rq_parent += o; Q.rq_cslot += o; Q.rq_m += o; Q.rq_dslot += o;
        Q.rq_w += o; Q.rq_state += o; Q.rq_score += o; Q.rq_slm += o; Q.rq_ps += o;
        Q.pr_req += o; Q.pr_inrow += o; Q.pr_w += o; Q.pr_p += o; Q.pr_dig += o;
    }
    const uint32_t sid = P.utt_stream[u];
    rg.in_row = Q.pr_inrow; rg.words = Q.pr_w; rg.dig = Q.pr_dig; rg.alg = Q.alg;
    if (prof) ph[11]++;
    const uint32_t l_begin = P.ul_off[u], l_end = P.ul_off[u + 1];
    for (uint32_t li = l_begin; li < l_end; li++) {
        const UttLevel L = P.ul[li];
        if (tid == 0) s_nprim = 0;
        __syncthreads();
        // ---------------- expand ----------------
        for (uint32_t k = L.nb + wid; k < L.ne; k += NW) {
            const NodeInfo nd = P.nodes[P.level_nodes[k]];
            expand_node(Q, S, g, nd, beam, L.t, -(int64_t)L.rb, &s_nprim, e_ctx[wid], e_slot[wid], e_score[wid],
                        e_arc[wid], lane, /*defer_ps=*/true);
        }
        __syncthreads();
        const uint32_t n = s_nprim;
        if (tid == 0) {
            uint32_t b = 0;
            if (n) b = atomicAdd(cursor, n);
            if ((uint64_t)b + n > row_limit) { atomicOr(S.err, OTF_E_ARENA_FULL); s_abort = 1; }
            s_base = b;
        }
        __syncthreads();
        SO_MARK(0);
        if (s_abort) break;                          // (every later stream aborts at once too)
        const uint32_t base = s_base;
        rg.hout = S.arena_h + (size_t)base * H;
        if (n == 0) small_lm_scores(Q, S, g, sid, L.re - L.rb, tid, NT);
        for (uint32_t q0 = 0, c = 0; q0 < n; q0 += xu::XR, c++) {
            const int nq = (int)min((uint32_t)xu::XR, n - q0);
            // the chunk's context-row planes into its scratch slot (no tiles)
            xu::update_chunk<NT>(m, q0, nq, (int)c, rg, gctr_u, tiles_done, tid, wid, lane, wait,
                                 []() { __syncthreads(); }, prof ? ph : nullptr, t0, 0, 0, true);
            // HS + MaxEnt of the chunk (digit-plane GEMM on this SM's tensor core)
            if (tid < NT - 64) xh::setup<ORD, NT - 64>(m, Q, S, q0, nq, hs, tid, lane);
            __syncthreads();
            SO_MARK(4);
            xh::run<ORD, NT>(m, Q, S, base, q0, nq, rg.xs + (size_t)(c & 1) * rg.xs_slot, rg.eh + (c & 1) * xu::XR,
                             smem, hs, tmem, bar_full, bar_empty, &bar_done, gctr_h, tiles_done, tid, wid, lane, wait,
                             [&](int t2, int nt2) { if (c == 0) small_lm_scores(Q, S, g, sid, L.re - L.rb, t2, nt2); },
                             prof ? ph : nullptr, t0, /*defer_finish=*/true);
            SO_MARK(5);
            // the recurrent update of the chunk over every M tile (planes already
            // in the slot); the HS tail (MaxEnt, log-sigmoid, path sums, flagged
            // queries) runs on warps 2.. under the first tile's K loop
            xu::Ring rgc = rg;
            rgc.eh = rg.eh + (c & 1) * xu::XR;
            rgc.phase_g = P.phase_ns;
            rgc.fuse_store = S.arena_dig;          // the new rows' planes straight from the epilogue
            rgc.out_row0 = base;
            xu::update_chunk<NT>(m, q0, nq, (int)c, rgc, gctr_u, tiles_done, tid, wid, lane, wait,
                                 []() {}, prof ? ph : nullptr, t0, 0, nmt, false,
                                 [&](int ft, int fn) { xh::finish<ORD>(m, Q, S, base, q0, nq, hs, ft, fn, 5); },
                                 /*side_uses_us=*/true);
            __syncthreads();
        }
        // (the level's new rows got their digit planes in the update epilogue)
        __syncthreads();
        SO_MARK(6);
        const StreamRange rgs{sid, 0u, L.re - L.rb, 0u};
        const LevelCtr lc{n, base, 0u, 0u};
        assign_range<0, NT>(Q, S, L.t, rgs, lc, row_limit, lm_weight, nullptr, nullptr, nullptr, asmem,
                            P.phase_ns ? P.phase_ns + 16 : nullptr);
        __syncthreads();
        SO_MARK(7);
    }
    __syncthreads();                               // s_u / s_abort reused by the next stream
    }
    if (prof)
        for (int i = 0; i < 28; i++) if (ph[i] && (i < 16 || i > 20)) atomicAdd(&P.phase_ns[i], ph[i]);
#undef SO_MARK
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

// --------------------------------------------------------------------------
// The EXACT HS + MaxEnt stage of the level schedule on the tensor cores
// (_kernels_nb.py:63-86 for every computed request of a level): persistent
// CTAs over 80-request chunks, each digitizing its chunk's context rows
// (xu::update_chunk without M tiles) and running the same digit-plane HS as
// k_decode_solo (xh::setup / xh::run: distinct path nodes x the chunk's rows,
// certified delta, float64 recompute of uncertified queries, successor
// history and digest).  Replaces the float64 CUDA-core k_hs_prim_ring in
// EXACT precision; runs beside k_advance_exact.
// --------------------------------------------------------------------------
template <int ORD>
__global__ void __launch_bounds__(sd::NT, 1)
k_hs_exact(DevModel m, DevPlan P, DevStreams S, RowSpec rs, uint8_t *xscratch, size_t xs_stride) {
    using namespace tc;
    constexpr int NT = sd::NT;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[4], bar_empty[4], bar_done;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const uint32_t n = rs.n_dev ? *rs.n_dev : 0u;
    const uint32_t base = row_base(rs);
    if (rs.cur && blockIdx.x == 0 && tid == 0) rs.cur->base = base;
    if ((uint64_t)base + n > rs.row_limit) {
        if (blockIdx.x == 0 && tid == 0) atomicOr(S.err, OTF_E_ARENA_FULL);
        return;
    }
    const uint32_t nch = (n + xu::XR - 1) / xu::XR;
    if (blockIdx.x >= nch) return;
    uint8_t *tables = smem + xh::ring_bytes();
    uint8_t *small = tables + ((xs1::tables_bytes(ORD) + 127u) & ~127u);
    constexpr xs1::Small sl = xs1::small_layout();
    if (tid == 0) {
        for (int st = 0; st < 4; st++) {
            mbar_init(smem_u32(&bar_full[st]), st < xh::STAGES ? xh::GT + 1 : 1);
            mbar_init(smem_u32(&bar_empty[st]), 1);
        }
        mbar_init(smem_u32(&bar_done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) reinterpret_cast<double *>(small + sl.tab)[tid] = exp2((double)tid / 32.0);
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const xh::Smem hs = xh::carve(smem, ORD);
    xu::Ring rg;                                       // (digitize only: no ring stages of its own)
    rg.smem = smem; rg.stages = xh::STAGES; rg.tmem = tmem;
    rg.full = bar_full + xh::STAGES; rg.empty = bar_empty + xh::STAGES; rg.done = &bar_done;
    rg.fb = nullptr; rg.us = nullptr;
    rg.sh = reinterpret_cast<double *>(small + sl.sh);
    rg.eh = reinterpret_cast<double *>(small + sl.eh);
    rg.fb_n = reinterpret_cast<uint32_t *>(small + sl.fbn);
    rg.src = reinterpret_cast<int32_t *>(small + sl.src);
    rg.wrd = reinterpret_cast<int32_t *>(small + sl.wrd);
    rg.tab = reinterpret_cast<const double *>(small + sl.tab);
    rg.xs = xscratch + (size_t)blockIdx.x * xs_stride;
    rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
    rg.hin = S.arena_h; rg.hout = nullptr; rg.in_row = P.pr_inrow; rg.words = P.pr_w;
    rg.dig = nullptr; rg.alg = nullptr;
    rg.dig_store = nullptr; rg.deh_store = nullptr; rg.dep_store = nullptr; rg.epoch = 0;
    DevPlan Q = P;
    uint32_t gctr_h = 0, gctr_u = 0, tiles_done = 0;
    unsigned long long t0 = 0;
    auto wait = [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); };
    int local = 0;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x, local++) {
        const uint32_t q0 = c * xu::XR;
        const int nq = (int)min((uint32_t)xu::XR, n - q0);
        xu::update_chunk<NT>(m, q0, nq, local, rg, gctr_u, tiles_done, tid, wid, lane, wait,
                             []() { __syncthreads(); }, nullptr, t0, 0, 0, true);
        if (tid < NT - 64) xh::setup<ORD, NT - 64>(m, Q, S, q0, nq, hs, tid, lane);
        __syncthreads();
        xh::run<ORD, NT>(m, Q, S, base, q0, nq, rg.xs + (size_t)(local & 1) * rg.xs_slot,
                         rg.eh + (local & 1) * xu::XR, smem, hs, tmem, bar_full, bar_empty, &bar_done, gctr_h,
                         tiles_done, tid, wid, lane, wait, [](int, int) {}, nullptr, t0, /*defer_finish=*/false);
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

// --------------------------------------------------------------------------
// The whole computed-request stage of an EXACT level in one persistent kernel
// (level schedule): per 80-request chunk of the level, k_decode_solo's chunk
// body -- digitize the chunk's context rows once, the digit-plane HS GEMM,
// then the certified recurrent update over every M tile with the HS tail
// (MaxEnt, log-sigmoid, path sums, successor history + digest) on warps 2..
// under the first tile's K loop and each tile's row stores under the next.
// Replaces k_hs_exact + k_advance_exact (one digitize instead of two, no
// second kernel holding SMs).
// --------------------------------------------------------------------------
template <int ORD>
__global__ void __launch_bounds__(sd::NT, 1)
k_level_exact(DevModel m, DevPlan P, DevStreams S, RowSpec rs, uint8_t *xscratch, size_t xs_stride) {
    using namespace tc;
    constexpr int NT = sd::NT;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_full[4], bar_empty[4], bar_done;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const uint32_t n = rs.n_dev ? *rs.n_dev : 0u;
    const uint32_t base = row_base(rs);
    if (rs.cur && blockIdx.x == 0 && tid == 0) rs.cur->base = base;
    if ((uint64_t)base + n > rs.row_limit) {
        if (blockIdx.x == 0 && tid == 0) atomicOr(S.err, OTF_E_ARENA_FULL);
        return;
    }
    const uint32_t nch = (n + xu::XR - 1) / xu::XR;
    if (blockIdx.x >= nch) return;
    const int nmt = (m.H + BM - 1) / BM;
    uint8_t *tables = smem + xh::ring_bytes();
    uint8_t *small = tables + ((xs1::tables_bytes(ORD) + 127u) & ~127u);
    constexpr xs1::Small sl = xs1::small_layout();
    if (tid == 0) {
        for (int st = 0; st < 4; st++) {           // [0, 2): HS ring, [2, 4): update ring
            mbar_init(smem_u32(&bar_full[st]), st < xh::STAGES ? xh::GT + 1 : 1);
            mbar_init(smem_u32(&bar_empty[st]), 1);
        }
        mbar_init(smem_u32(&bar_done), 1);
        reinterpret_cast<uint32_t *>(small + sl.fbn)[0] = 0u;
        reinterpret_cast<uint32_t *>(small + sl.fbn)[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) reinterpret_cast<double *>(small + sl.tab)[tid] = exp2((double)tid / 32.0);
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const xh::Smem hs = xh::carve(smem, ORD);
    DevPlan Q = P;
    xu::Ring rg;
    rg.smem = smem; rg.stages = xh::STAGES; rg.tmem = tmem;
    rg.full = bar_full + xh::STAGES; rg.empty = bar_empty + xh::STAGES; rg.done = &bar_done;
    rg.fb = reinterpret_cast<uint32_t *>(tables + xh::layout(ORD).hkey);
    rg.us = reinterpret_cast<float *>(tables);
    rg.sh = reinterpret_cast<double *>(small + sl.sh);
    rg.eh = reinterpret_cast<double *>(small + sl.eh);
    rg.fb_n = reinterpret_cast<uint32_t *>(small + sl.fbn);
    rg.src = reinterpret_cast<int32_t *>(small + sl.src);
    rg.wrd = reinterpret_cast<int32_t *>(small + sl.wrd);
    rg.tab = reinterpret_cast<const double *>(small + sl.tab);
    rg.xs = xscratch + (size_t)blockIdx.x * xs_stride;
    rg.xs_slot = xu::xs_slot_bytes(m.wd_nkx);
    rg.hin = S.arena_h; rg.hout = S.arena_h + (size_t)base * m.H;
    rg.in_row = Q.pr_inrow; rg.words = Q.pr_w; rg.dig = Q.pr_dig; rg.alg = Q.alg;
    rg.dig_store = nullptr; rg.deh_store = nullptr; rg.dep_store = nullptr; rg.epoch = 0;
    uint32_t gctr_h = 0, gctr_u = 0, tiles_done = 0;
    unsigned long long t0 = 0;
    auto wait = [](uint32_t b, uint32_t par, int tag) { sd::wait_bounded(b, par, tag); };
    int local = 0;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x, local++) {
        const uint32_t q0 = c * xu::XR;
        const int nq = (int)min((uint32_t)xu::XR, n - q0);
        xu::update_chunk<NT>(m, q0, nq, local, rg, gctr_u, tiles_done, tid, wid, lane, wait,
                             []() { __syncthreads(); }, nullptr, t0, 0, 0, true);
        if (tid < NT - 64) xh::setup<ORD, NT - 64>(m, Q, S, q0, nq, hs, tid, lane);
        __syncthreads();
        xh::run<ORD, NT>(m, Q, S, base, q0, nq, rg.xs + (size_t)(local & 1) * rg.xs_slot,
                         rg.eh + (local & 1) * xu::XR, smem, hs, tmem, bar_full, bar_empty, &bar_done, gctr_h,
                         tiles_done, tid, wid, lane, wait, [](int, int) {}, nullptr, t0, /*defer_finish=*/true);
        xu::Ring rgc = rg;
        rgc.eh = rg.eh + (local & 1) * xu::XR;
        xu::update_chunk<NT>(m, q0, nq, local, rgc, gctr_u, tiles_done, tid, wid, lane, wait,
                             []() {}, nullptr, t0, 0, nmt, false,
                             [&](int ft, int fn) { xh::finish<ORD>(m, Q, S, base, q0, nq, hs, ft, fn, 5); },
                             /*side_uses_us=*/true);
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

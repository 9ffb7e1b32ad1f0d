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
//   HS       warp per computed request over the TMA bulk-copy ring
//            (hs_logprob_ring, shared with k_hs_prim_ring), in the same shared
//            memory the update's ring used;
//   assign   assign_range (shared with k_assign) over the stream's requests
//            in reference order with the whole CTA.
// Tensor-core precisions only (TF32X3 / TF32); FP64 exact mode and BF16 use
// the level-synchronous schedule.
#pragma once
#include "decode.cuh"
#include "tc_advance.cuh"

namespace sd {
constexpr int NT = 512;
constexpr int NW = NT / 32;

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
// of hanging the GPU.  2^22 polls is well over a second, orders of magnitude above any
// legitimate wait in this kernel.
__device__ __forceinline__ void wait_bounded(uint32_t bar, uint32_t parity, int tag) {
    for (uint32_t it = 0;; it++) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        if (it == (1u << 22)) {
            printf("k_decode_streams: wait timeout block %d thread %d tag %d parity %u\n", (int)blockIdx.x,
                   (int)threadIdx.x, tag, parity);
            __trap();
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
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

// MODE 1 = TF32X3, 3 = TF32; KC_B = m.wt_kcb; CPL/ORD as RING_DISPATCH.
template <int MODE, int KC_B, int CPL, int ORD>
__global__ void __launch_bounds__(sd::NT, 1)
k_decode_streams(DevModel m, DevPlan P, DevStreams S, DevNgram g, long long beam, double lm_weight, int stages,
                 int hs_warps, uint32_t *cursor, uint32_t row_limit, uint32_t tmem_cols) {
    using namespace tc;
    constexpr bool X3 = MODE == 1;
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
    __shared__ __align__(8) uint64_t hs_bar[NW][HS_NS];   // HS ring barriers (initialised once)

    const int tid = threadIdx.x, lane = tid & 31;
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);     // provably warp-uniform
    const uint32_t u = blockIdx.x;
    if (u >= P.n_utt) return;
    const int H = m.H;
    const int nmt = m.wt_npad / BM;                      // M tiles of output units
    const uint32_t wa_bytes = (uint32_t)m.wt_npad * KC_B;  // one W block (hi or lo)
    const uint32_t hb_bytes = BM * KC_B;                 // one row block (hi or lo)
    const uint32_t stage_bytes = (X3 ? 2u : 1u) * (wa_bytes + hb_bytes);
    const int NK = (H + KE - 1) / KE;

    if (tid == 0) {
        for (int st = 0; st < stages; st++) {
            mbar_init(smem_u32(&bar_full[st]), NW);   // one per loader warp + the W copy
            mbar_init(smem_u32(&bar_empty[st]), 1);
        }
        mbar_init(smem_u32(&bar_done), 1);
        for (int i = 0; i < NW * HS_NS; i++) mbar_init(smem_u32(&hs_bar[i / HS_NS][i % HS_NS]), 1);
        s_abort = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&s_tmem)), "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    // this utterance's request / primary workspace
    DevPlan Q = P;
    {
        const uint32_t o = P.rq_off[u];
        Q.rq_c += o; Q.rq_arc += o; Q.rq_parent += o; Q.rq_cslot += o; Q.rq_m += o; Q.rq_dslot += o;
        Q.rq_w += o; Q.rq_state += o; Q.rq_score += o; Q.rq_slm += o; Q.rq_ps += o;
        Q.pr_req += o; Q.pr_inrow += o; Q.pr_w += o; Q.pr_p += o; Q.pr_dig += o;
    }
    const uint32_t sid = P.utt_stream[u];
    const AssignSmem asmem{a_key, a_row, a_cn, a_wsum, a_cnt};
    uint32_t gctr = 0;          // K chunks through the ring so far (uniform)
    uint32_t tiles_done = 0;
    // HS ring of this warp: row slots in the shared union (free while HS
    // runs), barriers in static shared memory with phases kept across levels
    HsRing ring;
    ring.buf = smem + (size_t)wid * HS_NS * 4 * H;
    ring.bar0 = smem_u32(&hs_bar[wid][0]);
    ring.phase = 0;

    // profiling runs only: per-phase device time (ns), summed over CTAs
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t0 = 0, t1 = 0;
    const bool prof = P.phase_ns != nullptr && tid == 0;
#define SD_MARK(i) do { if (prof) { t1 = sd::gtimer(); ph[i] += t1 - t0; t0 = t1; } } while (0)
    if (prof) t0 = sd::gtimer();
    for (uint32_t li = P.ul_off[u]; li < P.ul_off[u + 1]; li++) {
        const UttLevel L = P.ul[li];
        if (tid == 0) s_nprim = 0;
        __syncthreads();
        // ---------------- expand ----------------
        for (uint32_t k = L.nb + wid; k < L.ne; k += NW) {
            const NodeInfo nd = P.nodes[P.level_nodes[k]];
            expand_node(Q, S, g, nd, beam, L.t, -(int64_t)L.rb, &s_nprim, e_ctx[wid], e_slot[wid], e_score[wid],
                        e_arc[wid], lane);
        }
        __syncthreads();
        SD_MARK(0);
        const uint32_t n = s_nprim;
#ifdef SD_CHECK
        if (tid == 0 && n > L.re - L.rb) { printf("SD_CHECK n %u > requests %u blk %d\n", n, L.re - L.rb, (int)blockIdx.x); __trap(); }
#endif
        if (tid == 0) {
            uint32_t b = 0;
            if (n) b = atomicAdd(cursor, n);
            if ((uint64_t)b + n > row_limit) { atomicOr(S.err, OTF_E_ARENA_FULL); s_abort = 1; }
            s_base = b;
        }
        __syncthreads();
        if (s_abort) break;
        const uint32_t base = s_base;
        if (n) {
            // ------------- recurrent update (tcgen05) -------------
            for (uint32_t q0 = 0; q0 < n; q0 += BM) {
                const int nr = (int)min((uint32_t)BM, n - q0);
                const int nn = (nr + 15) & ~15;                   // MMA N
                const int nitems = ((nr + 7) & ~7) * CH;          // row pieces per chunk
                // warp 0: MMA issuer (converged; lane 0 issues).  Warps 1..NW-1:
                // loaders / converters -- a divergent issuer inside a loader
                // warp would sit behind its siblings' suspended mbarrier waits.
                constexpr int LT = NT - 32;                        // loader threads
                const int ltid = tid - 32;
                auto issue = [&](uint32_t gc, int kc) {
                    const int st = (int)(gc % stages);
                    const uint32_t use = gc / stages;
                    if (use >= 1) sd::wait_bounded(smem_u32(&bar_empty[st]), (use - 1) & 1, 1);
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
                auto consume = [&](uint32_t gc, int pending) {
                    const int st = (int)(gc % stages);
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
                        const uint32_t gc = gctr + kc;
                        const int st = (int)(gc % stages);
                        const unsigned long long w0 = prof ? sd::gtimer() : 0ull;
                        sd::wait_bounded(smem_u32(&bar_full[st]), (gc / stages) & 1, 2);
                        if (prof) ph[5] += sd::gtimer() - w0;
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
                    for (int j = 0; j < pre; j++) issue(gctr + j, j);
                    for (int kc = 0; kc < NK; kc++) {
                        const uint32_t gc = gctr + kc;
                        consume(gc, min(stages - 2, NK - 1 - kc));
                        if (kc + stages - 1 < NK) issue(gctr + kc + stages - 1, kc + stages - 1);
                    }
                }
                gctr += NK;
                SD_MARK(1);
                // epilogue: TMEM lane = output unit, column = row of the tile
                sd::wait_bounded(smem_u32(&bar_done), tiles_done & 1, 3);
                tiles_done++;
                __syncwarp();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                {
                    const int quad = wid & 3;
                    const int nch = (nr + 31) / 32;
                    for (int it = wid >> 2; it < nmt * nch; it += NW / 4) {
                        const int mt = it / nch, ch = it - mt * nch;
                        const int unit = mt * BM + quad * 32 + lane;
                        float v[32];
                        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mt * BM + ch * 32), v);
                        unsigned long long dg[32];
#pragma unroll
                        for (int j = 0; j < 32; j++) {
                            dg[j] = 0ull;
                            const int row = ch * 32 + j;
                            if (row < nr && unit < H) {
                                const uint32_t q = q0 + (uint32_t)row;
                                const int wq = Q.pr_w[q];
                                const float o = 1.f / (1.f + expf(-(v[j] + __ldg(m.U + (size_t)wq * H + unit))));
                                S.arena_h[(size_t)(base + q) * H + unit] = o;
                                dg[j] = otf_hash64(((uint64_t)unit << 32) ^ __float_as_uint(o));
                            }
                        }
                        const unsigned long long tot = sd::transpose_sum32(dg, lane);
                        const int row = ch * 32 + lane;
                        if (row < nr) atomicAdd(&Q.pr_dig[q0 + row], tot);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncthreads();
                SD_MARK(2);
            }
            // ------------- HS + MaxEnt of the computed requests -------------
            if (wid < hs_warps) {
                const RowSpec rs0{nullptr, nullptr, nullptr, nullptr, nullptr, row_limit};
                for (uint32_t q = wid; q < n; q += hs_warps) {
                    const uint32_t row = (uint32_t)Q.pr_inrow[q];
                    const uint32_t *meta = S.arena_meta + (size_t)row * OTF_META;
                    const int Lh = (int)meta[0];
                    const int w = Q.pr_w[q];
#ifdef SD_CHECK
                    if (row >= S.arena_rows || w < 0 || w >= m.V || Lh > m.order) {
                        printf("SD_CHECK hs: blk %d q %u n %u row %u w %d L %d base %u lvl %u\n", (int)blockIdx.x, q, n, row, w, Lh, base, L.t);
                        __trap();
                    }
#endif
                    const uint32_t o0 = __ldg(m.path_off + w), o1 = __ldg(m.path_off + w + 1);
                    const double lp = hs_logprob_ring<CPL, false, ORD>(m, ring, S.arena_h + (size_t)row * H, meta + 1,
                                                                       Lh, m.path_code + o0, o1 - o0, lane);
                    hs_prim_finish(m, Q, S, rs0, base, q, meta, Lh, w, o1 - o0, lp, lane);
                }
            }
            __syncthreads();
            SD_MARK(3);
        }
        // ---------------- assign ----------------
        const StreamRange rg{sid, 0u, L.re - L.rb, 0u};
        const LevelCtr lc{n, base, 0u, 0u};
        assign_range<0, NT>(Q, S, L.t, rg, lc, row_limit, lm_weight, nullptr, nullptr, nullptr, asmem);
        __syncthreads();
        SD_MARK(4);
    }
    if (prof) {
        ph[7] = 1;
        for (int i = 0; i < 8; i++) atomicAdd(&P.phase_ns[i], ph[i]);
    }
#undef SD_MARK
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(tmem_cols));
}

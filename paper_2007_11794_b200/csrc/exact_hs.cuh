// exact_hs.cuh -- hierarchical-softmax + MaxEnt scoring of a level's computed
// requests (_kernels_nb.py:63-86) on the tensor core of the control CTA
// (rank 0), in the EXACT precision of the persistent stream kernel.
//
// The node activations a = sum_i v_node[i] h[i] of all (query, path node)
// pairs of a chunk are one integer digit-plane GEMM, the same scheme as the
// recurrent update (exact_update.cuh): the HS node vectors as five 8-bit
// planes (pre-tiled per node at model upload, NVd[node][kc][plane][64 B]),
// the chunk's context rows as the four planes rank 1 already digitized for
// the update (global scratch, read by bulk copy), 17 plane pairs into six
// exact int32 anti-diagonals in TMEM.  A = the chunk's distinct path nodes
// (rows gathered by cp.async, 128 per M tile), B = the chunk's queries, so a
// node shared by many paths (the top of the Huffman tree) is multiplied
// once.  The epilogue reads, per TMEM lane (node) and query column, only the
// pairs on that query's path.  Then per pair the MaxEnt terms are added in
// the reference's order and the float64 log-sigmoid taken; per query the
// path-order sum p.
//
// Certification: |a~ - a_ref| <= eps_n + B_n eH_r per pair (dropped plane
// pairs, representation of both operands, the reference's sequential-sum
// rounding), |dlog sigma| <= |da|, so |p~ - p_ref| <= sum of the pair
// bounds.  The decode consumes p only through delta = f32(p - p_small)
// (codec.py:57-59); a query whose delta could round differently inside that
// bound has its activations recomputed with float64 CUDA-core dot products
// (the FP64 mode's arithmetic).
#pragma once
#include "exact_update.cuh"

namespace xh {
constexpr int STAGES = 2;
constexpr int GW0 = 2, GW1 = 14;                 // A-row gather warps [GW0, GW1)
constexpr int GT = (GW1 - GW0) * 32;
constexpr int PCAP = 2048;                       // (query, node) pairs per chunk
constexpr int RCAP = 2048;                       // distinct nodes per chunk
constexpr int HCAP = 2048;                       // node dedup hash slots (power of two)
constexpr int QX = xu::XR;                       // queries per chunk = the update's rows per chunk

// rank 0's dynamic shared memory after its ring (byte offsets)
struct Layout {
    uint32_t act, errj, pcode, prow, pq, wpos, nrow, hkey, hval, pre, qa, epsq, misc, total;
};
__host__ __device__ constexpr Layout layout(int ord) {
    const uint32_t act = 0;
    const uint32_t errj = act + PCAP * 8;
    const uint32_t pcode = errj + PCAP * 4;
    const uint32_t prow = pcode + PCAP * 4;
    const uint32_t pq = prow + PCAP * 2;
    const uint32_t wpos = pq + PCAP;
    const uint32_t nrow = wpos + 128 * QX;
    const uint32_t hkey = nrow + RCAP * 4;
    const uint32_t hval = hkey + HCAP * 4;
    const uint32_t pre = (hval + HCAP * 2 + 7) & ~7u;
    const uint32_t qa = pre + (uint32_t)QX * ord * 8;            // row, cb, off, P, w, kmax, L, flag: 8 x [QX] u32
    const uint32_t epsq = qa + 8 * QX * 4;
    const uint32_t misc = epsq + QX * 8;                          // [0] rows, [1] pairs, [2] flagged
    return Layout{act, errj, pcode, prow, pq, wpos, nrow, hkey, hval, pre, qa, epsq, misc, misc + 64};
}
__host__ __device__ constexpr uint32_t ring_bytes() { return (uint32_t)STAGES * xu::STAGE; }
// rank 0's share of the recurrent update (exact_update.cuh) runs after the
// chunk's HS, with its small tail overlaid on the (then idle) dedup hash:
// fb[2][FBCAP] | fb_n[4] | eh[XR] | src[XR] | wrd[XR] | tab[32]
struct UpdOverlay { uint32_t fb, fbn, eh, src, wrd, tab, total; };
__host__ __device__ constexpr UpdOverlay upd_overlay() {
    return UpdOverlay{0u, 2u * xu::FBCAP * 4, 2u * xu::FBCAP * 4 + 16, 2u * xu::FBCAP * 4 + 16 + xu::XR * 8,
                      2u * xu::FBCAP * 4 + 16 + xu::XR * 12, 2u * xu::FBCAP * 4 + 16 + xu::XR * 16,
                      2u * xu::FBCAP * 4 + 16 + xu::XR * 16 + 256};
}
static_assert(upd_overlay().total <= HCAP * 6, "update overlay exceeds the dedup hash region");

struct Smem {
    double *act;
    float *errj;                 // [PCAP] the pair's bound on |a~ - a_ref| (rounded up)
    uint32_t *pcode;
    uint16_t *prow;
    uint8_t *pq, *wpos;
    uint32_t *nrow, *hkey;
    uint16_t *hval;
    unsigned long long *pre;
    uint32_t *row, *cb, *off, *P, *flag;
    int32_t *w, *kmax, *L;
    double *epsq;
    uint32_t *misc;
};
__device__ __forceinline__ Smem carve(uint8_t *smem, int ord) {
    const Layout l = layout(ord);
    uint8_t *b = smem + ring_bytes();
    Smem s;
    s.act = reinterpret_cast<double *>(b + l.act);
    s.errj = reinterpret_cast<float *>(b + l.errj);
    s.pcode = reinterpret_cast<uint32_t *>(b + l.pcode);
    s.prow = reinterpret_cast<uint16_t *>(b + l.prow);
    s.pq = b + l.pq;
    s.wpos = b + l.wpos;
    s.nrow = reinterpret_cast<uint32_t *>(b + l.nrow);
    s.hkey = reinterpret_cast<uint32_t *>(b + l.hkey);
    s.hval = reinterpret_cast<uint16_t *>(b + l.hval);
    s.pre = reinterpret_cast<unsigned long long *>(b + l.pre);
    uint32_t *qa = reinterpret_cast<uint32_t *>(b + l.qa);
    s.row = qa; s.cb = qa + QX; s.off = qa + 2 * QX; s.P = qa + 3 * QX;
    s.w = reinterpret_cast<int32_t *>(qa + 4 * QX); s.kmax = reinterpret_cast<int32_t *>(qa + 5 * QX);
    s.L = reinterpret_cast<int32_t *>(qa + 6 * QX); s.flag = qa + 7 * QX;
    s.epsq = reinterpret_cast<double *>(b + l.epsq);
    s.misc = reinterpret_cast<uint32_t *>(b + l.misc);
    return s;
}

// Certified float32 rounding of d (any sign) for |d - d_ref| <= margin.
__device__ __forceinline__ bool certify_f32(double d, double margin) {
    const float f = __double2float_rn(d);
    const uint32_t fb = __float_as_uint(f) & 0x7FFFFFFFu;
    const uint32_t ef = fb >> 23;
    if (ef == 0u || ef >= 254u) return false;                    // zero / subnormal / huge
    const double ad = fabs(d), af = xu::widen_d(__uint_as_float(fb));
    const double dd = ad - af;                                   // exact
    const int hw = (int)((ef + 1023u - 127u - 24u) << 20);
    const double half_up = __hiloint2double(hw, 0);
    const double half_dn = __hiloint2double((fb & 0x7FFFFFu) ? hw : hw - (1 << 20), 0);
    return dd >= 0.0 ? dd + margin < half_up : margin - dd < half_dn;
}

// ---- part 1 (before the digits of the chunk are ready): per-query path
// data, pair tables, distinct nodes.  Threads [0, NTS) of the CTA, named
// barrier 1.
template <int ORD, int NTS>
__device__ __forceinline__ void setup(const DevModel &m, const DevPlan &Q, const DevStreams &S, uint32_t q0, int nq,
                                      const Smem &hs, int tid, int lane) {
    constexpr int NWS = NTS / 32;
    const int wid = tid >> 5;
    for (int i = tid; i < HCAP; i += NTS) { hs.hkey[i] = 0u; hs.hval[i] = 0xFFFFu; }
    if (tid < 4) hs.misc[tid] = 0u;
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
        hs.epsq[tid] = 0.0; hs.flag[tid] = 0u;
    }
    // exclusive scan of P (queries live in warps 0..2)
    uint32_t inc = Pt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    __shared__ uint32_t s_wsum[4];
    if (lane == 31 && wid < 4) s_wsum[wid] = inc;
    sd::group_sync(1, NTS);
    if (tid < nq) {
        uint32_t before = 0;
        for (int w2 = 0; w2 < wid; w2++) before += s_wsum[w2];
        hs.off[tid] = before + inc - Pt;
        if (tid == nq - 1) hs.misc[1] = min(before + inc, (uint32_t)PCAP);
        if (tid == nq - 1 && before + inc > (uint32_t)PCAP) atomicOr(S.err, OTF_E_VALUE);
    }
    sd::group_sync(1, NTS);
    // pairs (warp per query) and the distinct nodes (open addressing on node + 1)
    for (int t = wid; t < nq; t += NWS) {
        const uint32_t o = hs.off[t], p = hs.P[t], cb = hs.cb[t];
        for (uint32_t i = lane; i < p; i += 32) {
            if (o + i >= (uint32_t)PCAP) break;
            const uint32_t code = __ldg(m.path_code + cb + i);
            const uint32_t node = code & 0x7FFFFFFFu;
            hs.pq[o + i] = (uint8_t)t;
            hs.pcode[o + i] = code;
            uint32_t h = (node * 0x9E3779B1u) >> 21;               // 11 bits = HCAP slots
            uint32_t r = 0xFFFFu;
            for (int probe = 0; probe < HCAP; probe++, h = (h + 1) & (HCAP - 1)) {
                const uint32_t prev = atomicCAS(&hs.hkey[h], 0u, node + 1u);
                if (prev == 0u) {                                   // new node: take the next row
                    r = atomicAdd(&hs.misc[0], 1u);
                    if (r < (uint32_t)RCAP) hs.nrow[r] = node;
                    else { atomicOr(S.err, OTF_E_VALUE); r = RCAP - 1; }
                    // its digit planes ([kc][plane][64 B], contiguous) into L2 now,
                    // so the GEMM's row gathers hit L2
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                                 :: "l"(m.NVd + (size_t)node * m.wd_nkx * xu::NPW * xu::KC),
                                    "r"((uint32_t)(m.wd_nkx * xu::NPW * xu::KC)) : "memory");
                    *reinterpret_cast<volatile uint16_t *>(&hs.hval[h]) = (uint16_t)r;
                    break;
                }
                if (prev == node + 1u) {                            // wait for the inserter's row
                    uint16_t v;
                    do { v = *reinterpret_cast<volatile uint16_t *>(&hs.hval[h]); } while (v == 0xFFFFu);
                    r = v;
                    break;
                }
            }
            hs.prow[o + i] = (uint16_t)r;
        }
    }
    sd::group_sync(1, NTS);
}

// ---- part 2 (the chunk's digits are in the scratch slot): the GEMM over
// M tiles of distinct nodes, the epilogue, MaxEnt + log-sigmoid, path sums,
// certification, the successor history and its digest.  All NT threads.
template <int ORD>
__device__ __forceinline__ void finish(const DevModel &m, DevPlan &Q, DevStreams &S, uint32_t base, uint32_t q0,
                                       int nq, const Smem &hs, int ft, int FN, int bar);

template <int ORD, int NT, typename WaitFn, typename SideFn>
__device__ __forceinline__ void run(const DevModel &m, DevPlan &Q, DevStreams &S, uint32_t base, uint32_t q0,
                                    int nq, const uint8_t *xs_slot, const double *eh_remote, uint8_t *smem,
                                    const Smem &hs, uint32_t tmem, uint64_t *full, uint64_t *empty, uint64_t *done,
                                    uint32_t &gctr, uint32_t &tiles_done, int tid, int wid, int lane, WaitFn wait,
                                    SideFn side, unsigned long long *ph, unsigned long long &t0,
                                    bool defer_finish = false) {
    constexpr int NW = NT / 32;
    auto mark = [&](int i) {
        if (ph) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); ph[i] += t - t0; t0 = t; }
    };
    const int NK = m.wd_nkx;
    const int Rp = (nq + 15) & ~15;
    const uint32_t nrows = min(hs.misc[0], (uint32_t)RCAP);
    const uint32_t T = hs.misc[1];
    const int ntile = (int)((nrows + 127) / 128);
    const uint32_t hbytes = 4u * (uint32_t)Rp * xu::KC;
    for (int t = 0; t < ntile; t++) {
        const int nr = (int)min(128u, nrows - 128u * t);
        // this tile's (row, query) -> path position table (warps GW1.. while the K loop runs)
        if (wid >= GW1) {
            const int t2 = tid - GW1 * 32, nt2 = NT - GW1 * 32;
            for (int i = t2; i < 128 * QX / 4; i += nt2) reinterpret_cast<uint32_t *>(hs.wpos)[i] = 0u;
            sd::group_sync(2, nt2);
            for (uint32_t j = (uint32_t)t2; j < T; j += (uint32_t)nt2) {
                const uint32_t r = hs.prow[j];
                if ((int)(r >> 7) == t) {
                    const int q = hs.pq[j];
                    hs.wpos[(r & 127u) * QX + q] = (uint8_t)(j - hs.off[q] + 1u);
                }
            }
            if (t == 0) side(t2, nt2);                      // e.g. the level's small-LM scores
        } else if (wid >= GW0) {
            // ---- A rows: the tile's node planes, 16-byte pieces into the canonical layout;
            // chunk kc+1 is issued before chunk kc is waited for ----
            const int g = tid - GW0 * 32;
            const int items = nr * xu::NPW * 4;
            auto issue = [&](int kc) {
                const uint32_t gc = gctr + kc;
                const int st = (int)(gc % STAGES);
                const uint32_t use = gc / STAGES;
                if (use >= 1) wait(tc::smem_u32(&empty[st]), (use - 1) & 1, 21);
                uint8_t *sA = smem + (size_t)st * xu::STAGE;
                for (int it = g; it < items; it += GT) {
                    const int r = it / (xu::NPW * 4), rem = it - r * (xu::NPW * 4);
                    const int a = rem >> 2, c = rem & 3;
                    const uint32_t node = hs.nrow[128 * t + r];
                    const uint8_t *src = m.NVd + (((size_t)node * NK + kc) * xu::NPW + a) * xu::KC + c * 16;
                    tc::cp_async16(tc::smem_u32(sA + a * xu::PLANE_W + xu::toff(r, c)), src, true);
                }
                tc::cp_async_commit();
            };
            issue(0);
            for (int kc = 0; kc < NK; kc++) {
                if (kc + 1 < NK) { issue(kc + 1); asm volatile("cp.async.wait_group 1;" ::: "memory"); }
                else asm volatile("cp.async.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(tc::smem_u32(&full[(gctr + kc) % STAGES])) : "memory");
            }
        } else if (wid == 1) {
            // ---- B: the chunk's h planes, one bulk copy per K chunk ----
            for (int kc = 0; kc < NK; kc++) {
                const uint32_t gc = gctr + kc;
                const int st = (int)(gc % STAGES);
                const uint32_t use = gc / STAGES;
                if (use >= 1) wait(tc::smem_u32(&empty[st]), (use - 1) & 1, 22);
                __syncwarp();
                uint8_t *sB = smem + (size_t)st * xu::STAGE + xu::HOFF;
                asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 tt;\n\telect.sync tt|e, 0xffffffff;\n\t"
                             "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n\t"
                             "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t}"
                             :: "r"(tc::smem_u32(sB)), "r"(tc::smem_u32(&full[st])),
                                "l"(xs_slot + (size_t)kc * hbytes), "r"(hbytes) : "memory");
            }
        } else {
            // ---- MMA issuer: the 17 digit pairs (as exact_update.cuh) ----
            for (int kc = 0; kc < NK; kc++) {
                const uint32_t gc = gctr + kc;
                const int st = (int)(gc % STAGES);
                wait(tc::smem_u32(&full[st]), (gc / STAGES) & 1, 23);
                __syncwarp();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sW = tc::smem_u32(smem + (size_t)st * xu::STAGE);
                xu::kc_pairs(Rp, kc == 0, tmem, xu::desc(sW), xu::desc(sW + xu::HOFF));
                tc::commit_elect(tc::smem_u32(&empty[st]));
                if (kc == NK - 1) tc::commit_elect(tc::smem_u32(done));
                __syncwarp();
            }
            wait(tc::smem_u32(done), tiles_done & 1, 24);
        }
        gctr += NK;
        tiles_done++;
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        mark(9);
        // ---- epilogue: lane quadrant warps x 8-query column chunks ----
        {
            const int quad = wid & 3;
            const int r = quad * 32 + lane;                 // tile row = TMEM lane
            const bool rok = r < nr;
            const uint32_t node = rok ? hs.nrow[128 * t + r] : 0u;
            double4 k4 = make_double4(0.0, 0.0, 0.0, 0.0);
            if (rok) k4 = m.nx[node];
            const int ncc = (nq + 7) >> 3;
            for (int cc = wid >> 2; cc < ncc; cc += NW / 4) {
                uint32_t D[xu::NDIAG][8];
                const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(cc * 8);
#pragma unroll
                for (int s2 = 0; s2 < xu::NDIAG; s2++)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(D[s2][0]), "=r"(D[s2][1]), "=r"(D[s2][2]), "=r"(D[s2][3]),
                                   "=r"(D[s2][4]), "=r"(D[s2][5]), "=r"(D[s2][6]), "=r"(D[s2][7])
                                 : "r"(ta + (uint32_t)(s2 * Rp)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (rok) {
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        const int q = cc * 8 + k;
                        if (q >= nq) break;
                        const uint32_t pos = hs.wpos[r * QX + q];
                        if (pos == 0u) continue;
                        const long long th = ((long long)(int)D[0][k] << 16) + ((long long)(int)D[1][k] << 8) + (long long)(int)D[2][k];
                        const long long tl = ((long long)(int)D[3][k] << 16) + ((long long)(int)D[4][k] << 8) + (long long)(int)D[5][k];
                        const double dh = __longlong_as_double(th + 0x4338000000000000LL) - 6755399441055744.0;
                        const double dlo = __longlong_as_double(tl + 0x4338000000000000LL) - 6755399441055744.0;
                        const uint32_t j = hs.off[q] + pos - 1u;
                        hs.act[j] = fma(dh, k4.x, dlo * k4.w);
                        // this pair's activation bound (eH of the query's context row: rank 1's DSMEM)
                        hs.errj[j] = __double2float_ru(fma(k4.z, eh_remote[q], k4.y));
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
    }
    mark(22);
    if (defer_finish) return;
    finish<ORD>(m, Q, S, base, q0, nq, hs, tid, NT, 5);
    mark(23);
}

// The CUDA-core tail of a chunk's HS (after run's TMEM readout): MaxEnt
// terms, log-sigmoid, per-query path sums with the certified delta, history
// rows and digests, the float64 recompute of flagged queries.  Threads
// [0, FN) of the caller's numbering ft take part (named barrier bar): the
// whole CTA, or the warps that are idle under the next GEMM's K loop.
template <int ORD>
__device__ __forceinline__ void finish(const DevModel &m, DevPlan &Q, DevStreams &S, uint32_t base, uint32_t q0,
                                       int nq, const Smem &hs, int ft, int FN, int bar) {
    const int H = m.H, fw = ft >> 5, FNW = FN >> 5, lane = ft & 31;
    const uint32_t T = hs.misc[1];
    // ---- MaxEnt terms in the reference's order, sign, float64 log-sigmoid ----
    // two pairs per thread and trip, every MaxEnt weight of both loaded before
    // any is summed (independent L2 reads in flight instead of a chain)
    for (uint32_t j0 = (uint32_t)ft; j0 < T; j0 += 2u * (uint32_t)FN) {
        float mev[2][ORD];
        int km[2];
        uint32_t cd[2];
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const uint32_t j = j0 + (uint32_t)p * (uint32_t)FN;
            km[p] = 0;
            cd[p] = 0u;
            if (j < T) {
                const int q = hs.pq[j];
                cd[p] = hs.pcode[j];
                km[p] = hs.kmax[q];
#pragma unroll
                for (int k = 0; k < ORD; k++)
                    mev[p][k] = k < km[p] ? __ldg(m.ME + (otf_mix(hs.pre[q * ORD + k], (uint64_t)(cd[p] & 0x7FFFFFFFu)) & m.mask))
                                          : 0.f;
            }
        }
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const uint32_t j = j0 + (uint32_t)p * (uint32_t)FN;
            if (j < T) {
                double a = hs.act[j];
                double me_abs = 0.0;
#pragma unroll
                for (int k = 0; k < ORD; k++)
                    if (k < km[p]) {
                        const double me = (double)mev[p][k];
                        a += me;
                        me_abs += fabs(me);
                    }
                // + the additions' rounding relative to the reference's (different a~)
                hs.errj[j] = __double2float_ru((double)hs.errj[j] + 8.0 * 1.1102230246251565e-16 * (fabs(a) + me_abs));
                hs.act[j] = otf_log_sigmoid((cd[p] & 0x80000000u) ? -a : a);
            }
        }
    }
    sd::group_sync(bar, FN);
    // ---- per query: path-order sum, certification of delta, history, digest ----
    if (ft < nq) {
        const int t = ft;
        const uint32_t q = q0 + (uint32_t)t;
        const uint32_t o = hs.off[t], p = hs.P[t];
        double lp = 0.0, labs = 0.0, eb = 0.0;
        for (uint32_t i = 0; i < p; i++) { lp += hs.act[o + i]; labs += fabs(hs.act[o + i]); eb += (double)hs.errj[o + i]; }
        const double ps = Q.rq_ps[Q.pr_req[q]];
        const double d = __dsub_rn(lp, ps);
        // + log-sigmoid / sum roundings (a few ulp of each term; libm vs glibc)
        const double margin = eb * 1.0001 + 1e-14 * (labs + fabs(ps));
        if (!certify_f32(d, margin)) {
            const uint32_t k = atomicAdd(&hs.misc[2], 1u);
            hs.flag[k] = (uint32_t)t;
        }
        Q.pr_p[q] = lp;
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
        if (Q.alg) {
            const int km = m.order < L ? m.order : L;
            atomicAdd(&Q.alg[0], (unsigned long long)p);
            atomicAdd(&Q.alg[1], (unsigned long long)p * km);
            atomicAdd(&Q.alg[2], 1ull);
        }
    }
    sd::group_sync(bar, FN);
    // ---- uncertified queries: float64 CUDA-core activations (warp per pair) ----
    const uint32_t nf = hs.misc[2];
    if (nf) {
        for (uint32_t f = 0; f < nf; f++) {
            const int t = (int)hs.flag[f];
            const uint32_t o = hs.off[t], p = hs.P[t];
            const float *hrow = S.arena_h + (size_t)hs.row[t] * H;
            for (uint32_t i = (uint32_t)fw; i < p; i += (uint32_t)FNW) {
                const uint32_t code = hs.pcode[o + i];
                const float *v = m.NV + (size_t)(code & 0x7FFFFFFFu) * H;
                double a = 0.0;
                for (int k = lane; k < H; k += 32) a = fma((double)__ldg(v + k), (double)__ldcg(hrow + k), a);
#pragma unroll
                for (int s2 = 16; s2; s2 >>= 1) a += __shfl_xor_sync(0xffffffffu, a, s2);
                for (int k = 0; k < hs.kmax[t]; k++)
                    a += (double)__ldg(m.ME + (otf_mix(hs.pre[t * ORD + k], (uint64_t)(code & 0x7FFFFFFFu)) & m.mask));
                if (lane == 0) hs.act[o + i] = otf_log_sigmoid((code & 0x80000000u) ? -a : a);
            }
        }
        sd::group_sync(bar, FN);
        if (ft < (int)nf) {
            const int t = (int)hs.flag[ft];
            double lp = 0.0;
            for (uint32_t i = 0; i < hs.P[t]; i++) lp += hs.act[hs.off[t] + i];
            Q.pr_p[q0 + (uint32_t)t] = lp;
        }
        if (Q.alg && ft == 0) atomicAdd(&Q.alg[4], (unsigned long long)nf);
        sd::group_sync(bar, FN);
    }
}
}  // namespace xh

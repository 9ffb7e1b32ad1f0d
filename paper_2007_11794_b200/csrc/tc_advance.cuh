// tc_advance.cuh -- the recurrent update h' = sigmoid(U[w] + W h) batched
// over all new (history, word) queries of a level, as a tcgen05 GEMM
// (reference _kernels_nb.py:51-60; the only dense contraction of the path).
//
//   D[q, i] = sum_j A[q, j] * W[i, j]       A[q] = h of query q's context
//   M = queries (128-row tiles), N = H outputs, K = H.
//
// Both operands are K-major in shared memory in the canonical no-swizzle
// UMMA layout (8-row x 16-byte core matrices, LBO = 128 B between K-adjacent
// core matrices, SBO = KC_B/16*128 B between 8-row groups).  A rows are
// GATHERED (the context arena row of each query) with coalesced 16-byte
// loads and written to shared memory already converted (tf32 round /
// hi-lo split / bf16); B (W, pre-split once at model upload) streams through
// a multi-stage cp.async ring.  One elected thread issues tcgen05.mma with
// the accumulator in TMEM (128 lanes x N_pad fp32 columns) and commits each
// stage to an mbarrier that releases the stage for the next loads.  The
// epilogue (4 warps, one TMEM lane per thread) reads the accumulator with
// tcgen05.ld, adds U[w] and applies the sigmoid in fp32, and writes h' into
// its arena row.
//
// Precision modes: TF32X3 = hi*hi + hi*lo + lo*hi (fp32-faithful, ~1e-7
// relative), TF32 = one pass, BF16 = kind::f16 with bf16 operands.
#pragma once
#include "common.cuh"

namespace tc {

constexpr int BM = 128;      // rows per CTA tile (UMMA_M)
constexpr int NTHREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;                 // descriptor version (sm_100)
    return d;                        // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}

// Swizzled K-major operand tiles (rows of KC_B bytes, 8-row atoms of
// 8*KC_B bytes, 16-byte chunk c of row r stored at chunk c ^ f(r)): the
// tensor core reads 8-row core-matrix groups in parallel, and with the
// unswizzled layout (groups SBO apart) those reads collide in the same banks.
// KC_B = 128 / 64 / 32 -> SWIZZLE_128B / 64B / 32B.
template <int KC_B>
__host__ __device__ __forceinline__ uint32_t swz_off(int row, int c) {
    constexpr int SH = KC_B == 128 ? 0 : KC_B == 64 ? 1 : 2;
    return (uint32_t)((row >> 3) * (8 * KC_B) + (row & 7) * KC_B + ((c ^ ((row & 7) >> SH)) << 4));
}
template <int KC_B>
__device__ __forceinline__ uint64_t make_desc_sw(uint32_t saddr) {
    constexpr uint64_t LAYOUT = KC_B == 128 ? 2 : KC_B == 64 ? 4 : 6;
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;                          // LBO (unused for swizzled K-major)
    d |= (uint64_t)(((8 * KC_B) >> 4) & 0x3FFFu) << 32;   // SBO: 8-row atom stride
    d |= 1ull << 46;                                 // descriptor version (sm_100)
    d |= LAYOUT << 61;
    return d;
}

// instruction descriptor: D fp32, A/B K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t make_idesc(int ab_fmt, int n) {
    return (1u << 4) | ((uint32_t)ab_fmt << 7) | ((uint32_t)ab_fmt << 10) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" :: "r"(a), "r"(parity) : "memory");
}

template <bool BF16>
__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (BF16) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    }
}

// Issue from a converged warp: every lane computes the (warp-uniform)
// descriptors, one lane is elected inside the asm.  Issuing under
// `if (lane == 0)` instead makes ptxas move the operands into uniform
// registers through a per-lane R2UR loop -- ~176 cycles per MMA against ~70
// (measured, tools/mma_micro.cu).
template <bool BF16>
__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (BF16) {
        asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                     "setp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    } else {
        asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                     "setp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    }
}
__device__ __forceinline__ void commit_elect(uint32_t mbar) {
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                 :: "r"(mbar) : "memory");
}

__device__ __forceinline__ void commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(mbar) : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g, bool valid) {
    const int sz = valid ? 16 : 0;   // zero-fill out-of-range chunks
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(saddr), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; j++) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = __uint_as_float(r[j]);
}

// smem offset of (row, 16-byte chunk c) inside a [rows x KC_B] operand tile
template <int KC_B>
__device__ __forceinline__ uint32_t tile_off(int row, int c) {
    return (uint32_t)((row >> 3) * (KC_B / 16 * 128) + c * 128 + (row & 7) * 16);
}

// MODE: 1 = TF32X3, 2 = BF16, 3 = TF32.
// Persistent, warp-specialized (the canonical sm_100 GEMM shape):
//   warps 0..3  loaders/converters: stream K chunks of consecutive tiles
//               through an S-stage ring without stopping at tile borders --
//               cp.async of the gathered fp32 A rows (staged in the operand
//               layout for tf32, raw for bf16) and of the pre-converted W
//               slice, cp.async.mbarrier.arrive on full_raw[]; then convert
//               in place (tf32 round, hi/lo split) or raw->bf16, arrive on
//               full_op[];
//   warp 4      MMA issuer: tcgen05.mma into one of two TMEM accumulators
//               (tile parity), commit empty[stage] per chunk and tmem_full[]
//               per tile;
//   warps 5..8  epilogue: tcgen05.ld the finished accumulator (lane quadrant
//               = warp % 4), + U[w], sigmoid, store h', content digest;
//               release the accumulator (tmem_empty[]) so tile i+2 can start
//               while tile i+1 is still in the MMA pipe.
// Grid: persistent CTAs over tiles = (row tile of 128) x (N tile of bn).
constexpr int LW = 8;                 // loader / converter warps 0..LW-1
constexpr int LT = LW * 32;
constexpr int MMA_WARP = LW;          // then 4 epilogue warps
constexpr int WS_THREADS = (LW + 5) * 32;
// The B operand and the epilogue.  EPI 0 (recurrent update): B = W (n_rows =
// H output units), h' = sigmoid(acc + U[w]) into arena rows.  EPI 1 (raw
// product, all_word_logprobs): B = the node vectors (n_rows = V - 1), the fp32
// accumulator goes to out[q * ld + j] as is.
struct TcB {
    const float *hi, *lo;           // tf32-rounded split (TF32X3 / TF32), [n_rows, H]
    const __nv_bfloat16 *bf;        // bf16 copy (BF16)
    const float *tiled;             // optional [K chunk][hi | lo][np rows x 64 B] SWIZZLE_64B tiles
    int tiled_np;
    int n_rows, n_pad;              // N extent, rounded up to the N granule
    float *out;                     // EPI 1
    int64_t ld;
};
template <int MODE, int KC_B, int EPI>
__global__ void __launch_bounds__(WS_THREADS, 1)
k_advance_tc(DevModel m, uint32_t n_cap, RowSpec rs, const int32_t *__restrict__ in_row,
             const int32_t *__restrict__ words, const float *__restrict__ h_base,
             float *__restrict__ out_base, TcB B, int bn_max, int stages,
             uint32_t tmem_cols) {
    constexpr bool BF = MODE == 2;
    constexpr bool X3 = MODE == 1;
    constexpr int ELT = BF ? 2 : 4;                   // operand bytes per element
    constexpr int KE = KC_B / ELT;                     // K elements per stage
    constexpr int CH = KC_B / 16;                      // operand 16-byte chunks per row
    constexpr int RAW_ROW = KE * 4 + 16;               // bf16 only: raw fp32 row stride (+16 B pad)
    constexpr int RAW_CH = KE / 4;                     // raw fp32 16-byte chunks per row
    const uint32_t row_limit = rs.row_limit;
    const uint32_t n = rs.n_dev ? *rs.n_dev : n_cap;
    const uint32_t out0 = row_base(rs);
    if (rs.cur && blockIdx.x == 0 && threadIdx.x == 0) rs.cur->base = out0;
    if ((uint64_t)out0 + n > row_limit) return;     // arena overflow (flagged by the HS stage)
    const int H = m.H;
    const int n_pad = B.n_pad, NR = B.n_rows;
    // B by bulk copy from the pre-tiled swizzled layout (tf32 modes, 64-byte chunks)
    const bool bulk_b = !BF && KC_B == 64 && B.tiled != nullptr;
    const uint32_t m_tiles = (n + BM - 1) / BM;
    // the row count is only known on the device: narrow the N tile while the
    // tiles still fit one per CTA (smem ring and TMEM are sized for bn_max)
    int bn = bn_max;
    while (bn > 32 && (bn / 2) % 16 == 0 && m_tiles * (uint32_t)((n_pad + bn / 2 - 1) / (bn / 2)) <= gridDim.x) bn /= 2;
    const int n_tiles = (n_pad + bn - 1) / bn;
    const uint32_t tiles = m_tiles * (uint32_t)n_tiles;
    if (blockIdx.x >= tiles) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform

    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t raw_bytes = BF ? BM * RAW_ROW : 0u;
    const uint32_t a_bytes = BM * KC_B;
    const uint32_t b_bytes = (uint32_t)bn * KC_B;
    const uint32_t stage_bytes = raw_bytes + (X3 ? 2 : 1) * (a_bytes + b_bytes);
    uint64_t *full_raw = reinterpret_cast<uint64_t *>(smem + stages * stage_bytes);
    uint64_t *full_op = full_raw + stages;
    uint64_t *empty = full_op + stages;
    uint64_t *tfull = empty + stages;                  // [2]
    uint64_t *tempty = tfull + 2;                      // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    if (tid == 0) {
        for (int st = 0; st < stages; st++) {
            mbar_init(smem_u32(&full_raw[st]), LT + (bulk_b ? 1 : 0));
            mbar_init(smem_u32(&full_op[st]), LW);         // one arrival per converter warp
            mbar_init(smem_u32(&empty[st]), 1);
        }
        for (int b2 = 0; b2 < 2; b2++) {
            mbar_init(smem_u32(&tfull[b2]), 1);
            mbar_init(smem_u32(&tempty[b2]), 4);           // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const int NK = (H + KE - 1) / KE;
    const uint32_t sbo = CH * 128, lbo = 128;
    const bool vec_ok = (H & 3) == 0;
    const bool vec_ok_b = BF ? (H & 7) == 0 : vec_ok;   // 16-byte B chunks = 8 bf16
    const uint32_t my_tiles = (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const uint32_t total_chunks = my_tiles * (uint32_t)NK;

    if (warp == MMA_WARP) {
        // ------------------------------ MMA issuer ----------------------------
        const uint32_t idesc = make_idesc(BF ? 1 : 2, bn);
        uint32_t g = 0;
        for (uint32_t it = 0; it < my_tiles; it++) {
            const uint32_t buf = it & 1;
            if (it >= 2) mbar_wait(smem_u32(&tempty[buf]), (uint32_t)(((it >> 1) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * (uint32_t)bn;
            for (int k = 0; k < NK; k++, g++) {
                const int st = (int)(g % stages);
                mbar_wait(smem_u32(&full_op[st]), (uint32_t)((g / stages) & 1));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                {
                    uint8_t *base = smem + st * stage_bytes;
                    uint8_t *sA = base + raw_bytes;
                    uint8_t *sA2 = sA + a_bytes;
                    uint8_t *sB = base + raw_bytes + (X3 ? 2 : 1) * a_bytes;
                    uint8_t *sB2 = sB + b_bytes;
#pragma unroll
                    for (int ks = 0; ks < KC_B / 32; ks++) {     // 32 bytes of K per MMA
                        const uint64_t a_hi = make_desc(smem_u32(sA) + ks * 2 * lbo, lbo, sbo);
                        const uint64_t b_hi = bulk_b ? make_desc_sw<64>(smem_u32(sB) + ks * 32)
                                                     : make_desc(smem_u32(sB) + ks * 2 * lbo, lbo, sbo);
                        const uint32_t acc = (k > 0 || ks > 0) ? 1u : 0u;
                        mma_elect<BF>(dacc, a_hi, b_hi, idesc, acc);
                        if (X3) {
                            const uint64_t a_lo = make_desc(smem_u32(sA2) + ks * 2 * lbo, lbo, sbo);
                            const uint64_t b_lo = bulk_b ? make_desc_sw<64>(smem_u32(sB2) + ks * 32)
                                                         : make_desc(smem_u32(sB2) + ks * 2 * lbo, lbo, sbo);
                            mma_elect<false>(dacc, a_hi, b_lo, idesc, 1u);
                            mma_elect<false>(dacc, a_lo, b_hi, idesc, 1u);
                        }
                    }
                    commit_elect(smem_u32(&empty[st]));
                    if (k == NK - 1) commit_elect(smem_u32(&tfull[buf]));
                }
                __syncwarp();
            }
        }
    } else if (warp < LW) {
        // ----------------------- loaders / converters -------------------------
        // source arena rows of this thread's A items, cached per tile
        constexpr int AI = (BM * (BF ? (KC_B / 2) / 4 : KC_B / 16) + LT - 1) / LT;
        int src_c[AI];
        uint32_t src_tile = 0xFFFFFFFFu;
        auto issue = [&](uint32_t gc) {
            const uint32_t it = gc / NK;
            const int k = (int)(gc - it * NK);
            const uint32_t tile = blockIdx.x + it * gridDim.x;
            const uint32_t q0 = (tile / n_tiles) * BM;
            const int n0 = (int)(tile % n_tiles) * bn;
            const int st = (int)(gc % stages);
            uint8_t *base = smem + st * stage_bytes;
            uint8_t *raw = base;
            uint8_t *sAop = base + raw_bytes;
            uint8_t *sB = base + raw_bytes + (X3 ? 2 : 1) * a_bytes;
            const int k0 = k * KE;
            if (tile != src_tile) {
                src_tile = tile;
#pragma unroll
                for (int i = 0; i < AI; i++) {
                    const int idx = tid + i * LT;
                    const int row = BF ? idx / RAW_CH : ((idx / (8 * CH)) * 8 + (idx & 7));
                    const uint32_t q = q0 + row;
                    src_c[i] = (idx < BM * RAW_CH && q < n) ? __ldg(in_row + q) : -1;
                }
            }
#pragma unroll
            for (int i = 0; i < AI; i++) {
                const int idx = tid + i * LT;
                if (idx >= BM * RAW_CH) break;
                int row, c;
                uint32_t off;
                if (BF) { row = idx / RAW_CH; c = idx - row * RAW_CH; off = row * RAW_ROW + c * 16; }
                else { const int r8 = idx & 7, g8 = idx / (8 * CH); c = (idx >> 3) % CH; row = g8 * 8 + r8; off = tile_off<KC_B>(row, c); }
                uint8_t *dstb = BF ? raw : sAop;
                const int src = src_c[i];
                const int kk = k0 + c * 4;
                const bool ok = src >= 0 && kk < H && vec_ok;
                cp_async16(smem_u32(dstb + off),
                           ok ? (const void *)(h_base + (size_t)src * H + kk) : (const void *)h_base, ok);
                if (!vec_ok && src >= 0) {   // unaligned H: synchronous scalar fill (rare)
                    float *dst = reinterpret_cast<float *>(dstb + off);
                    for (int e = 0; e < 4; e++) dst[e] = kk + e < H ? h_base[(size_t)src * H + kk + e] : 0.f;
                }
            }
            if (bulk_b) {
                if (warp == 0) {       // hi (+ lo) slices of the pre-tiled chunk: one bulk copy each
                    const uint32_t part = (uint32_t)B.tiled_np * KC_B;          // bytes of one [hi] block
                    const uint8_t *src = reinterpret_cast<const uint8_t *>(B.tiled) + (size_t)k * 2 * part +
                                         (size_t)n0 * KC_B;
                    const uint32_t bytes = (uint32_t)bn * KC_B;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (X3)
                        asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                                     "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %4;\n\t"
                                     "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t"
                                     "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%6], %3, [%1];\n\t}"
                                     :: "r"(smem_u32(sB)), "r"(smem_u32(&full_raw[st])), "l"(src), "r"(bytes),
                                        "r"(2u * bytes), "r"(smem_u32(sB + b_bytes)), "l"(src + part) : "memory");
                    else
                        asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                                     "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n\t"
                                     "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t}"
                                     :: "r"(smem_u32(sB)), "r"(smem_u32(&full_raw[st])), "l"(src), "r"(bytes) : "memory");
                }
            } else
            for (int idx = tid; idx < bn * CH; idx += LT) {
                const int r8 = idx & 7, c = (idx >> 3) % CH, g8 = idx / (8 * CH);
                const int row = g8 * 8 + r8;
                const int wrow = n0 + row;
                const int kk = k0 + c * (16 / ELT);
                const bool ok = wrow < NR && kk < H && vec_ok_b;
                const uint32_t off = tile_off<KC_B>(row, c);
                if (BF) {
                    cp_async16(smem_u32(sB + off), ok ? (const void *)(B.bf + (size_t)wrow * H + kk) : (const void *)B.bf, ok);
                } else {
                    cp_async16(smem_u32(sB + off), ok ? (const void *)(B.hi + (size_t)wrow * H + kk) : (const void *)B.hi, ok);
                    if (X3)
                        cp_async16(smem_u32(sB + b_bytes + off), ok ? (const void *)(B.lo + (size_t)wrow * H + kk) : (const void *)B.lo, ok);
                }
                if (!vec_ok_b && wrow < NR) {
                    for (int e = 0; e < 16 / ELT; e++) {
                        const bool in = kk + e < H;
                        if (BF) reinterpret_cast<__nv_bfloat16 *>(sB + off)[e] = in ? B.bf[(size_t)wrow * H + kk + e] : __float2bfloat16(0.f);
                        else {
                            reinterpret_cast<float *>(sB + off)[e] = in ? B.hi[(size_t)wrow * H + kk + e] : 0.f;
                            if (X3) reinterpret_cast<float *>(sB + b_bytes + off)[e] = in ? B.lo[(size_t)wrow * H + kk + e] : 0.f;
                        }
                    }
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_u32(&full_raw[st])) : "memory");
        };
        for (uint32_t gc = 0; gc < (uint32_t)(stages - 1) && gc < total_chunks; gc++) issue(gc);
        for (uint32_t gc = 0; gc < total_chunks; gc++) {
            const int st = (int)(gc % stages);
            const uint32_t gn = gc + stages - 1;
            // convert chunk gc first, so its conversion overlaps MMA gc-1 ...
            mbar_wait(smem_u32(&full_raw[st]), (uint32_t)((gc / stages) & 1));
            uint8_t *base = smem + st * stage_bytes;
            uint8_t *raw = base;
            uint8_t *sA = base + raw_bytes;
            uint8_t *sA2 = sA + a_bytes;
            for (int idx = tid; idx < BM * CH; idx += LT) {
                const int r8 = idx & 7, c = (idx >> 3) % CH, g8 = idx / (8 * CH);
                const int row = g8 * 8 + r8;
                const uint32_t off = tile_off<KC_B>(row, c);
                if (BF) {
                    const float4 x0 = *reinterpret_cast<const float4 *>(raw + row * RAW_ROW + c * 32);
                    const float4 x1 = *reinterpret_cast<const float4 *>(raw + row * RAW_ROW + c * 32 + 16);
                    __nv_bfloat162 b0 = __floats2bfloat162_rn(x0.x, x0.y), b1 = __floats2bfloat162_rn(x0.z, x0.w);
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(x1.x, x1.y), b3 = __floats2bfloat162_rn(x1.z, x1.w);
                    uint4 u;
                    u.x = *reinterpret_cast<uint32_t *>(&b0); u.y = *reinterpret_cast<uint32_t *>(&b1);
                    u.z = *reinterpret_cast<uint32_t *>(&b2); u.w = *reinterpret_cast<uint32_t *>(&b3);
                    *reinterpret_cast<uint4 *>(sA + off) = u;
                } else {
                    const float4 x = *reinterpret_cast<const float4 *>(sA + off);   // staged in place
                    float4 hi;
                    hi.x = tf32_rn(x.x); hi.y = tf32_rn(x.y); hi.z = tf32_rn(x.z); hi.w = tf32_rn(x.w);
                    *reinterpret_cast<float4 *>(sA + off) = hi;
                    if (X3) {
                        float4 lo;
                        lo.x = tf32_rn(x.x - hi.x); lo.y = tf32_rn(x.y - hi.y);
                        lo.z = tf32_rn(x.z - hi.z); lo.w = tf32_rn(x.w - hi.w);
                        *reinterpret_cast<float4 *>(sA2 + off) = lo;
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&full_op[st])) : "memory");
            // ... then refill the stage chunk gc-1 used, once its MMAs retired
            if (gn < total_chunks) {
                if (gc >= 1) mbar_wait(smem_u32(&empty[(gc - 1) % stages]), (uint32_t)(((gc - 1) / stages) & 1));
                issue(gn);
            }
        }
    } else {
        // ------------------------------ epilogue ------------------------------
        const int quad = warp & 3;                        // TMEM lanes 32*quad .. +31
        const int row = quad * 32 + lane;
        for (uint32_t it = 0; it < my_tiles; it++) {
            const uint32_t buf = it & 1;
            const uint32_t tile = blockIdx.x + it * gridDim.x;
            const uint32_t q0 = (tile / n_tiles) * BM;
            const int n0 = (int)(tile % n_tiles) * bn;
            mbar_wait(smem_u32(&tfull[buf]), (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t q = q0 + row;
            const bool valid = q < n;
            if (EPI == 1) {           // raw product rows (all_word_logprobs activations)
                float *orow = B.out + (int64_t)q * B.ld;
                for (int c0 = 0; c0 < bn; c0 += 32) {
                    float v[32];
                    tmem_ld32(tmem + buf * (uint32_t)bn + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, v);
                    const int gc = n0 + c0;
                    if (valid) {
                        if (gc + 32 <= NR && (B.ld & 3) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<float4 *>(orow + gc + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
                            for (int j = 0; j < 32; j++) if (gc + j < NR) orow[gc + j] = v[j];
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[buf])) : "memory");
                continue;
            }
            const int wq = valid ? (words ? __ldg(words + q) : (int32_t)q) : 0;
            unsigned long long dig = 0ull;
            const float *urow = m.U + (size_t)wq * H;
            float *orow = out_base + (size_t)(out0 + q) * H;
            for (int c0 = 0; c0 < bn; c0 += 32) {
                float v[32];
                tmem_ld32(tmem + buf * (uint32_t)bn + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, v);
                const int gc = n0 + c0;
                if (valid) {
                    if (vec_ok && gc + 32 <= H) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            float4 u = __ldg(reinterpret_cast<const float4 *>(urow + gc + j));
                            float4 o;
                            o.x = __frcp_rn(1.f + expf(-(v[j] + u.x)));
                            o.y = __frcp_rn(1.f + expf(-(v[j + 1] + u.y)));
                            o.z = __frcp_rn(1.f + expf(-(v[j + 2] + u.z)));
                            o.w = __frcp_rn(1.f + expf(-(v[j + 3] + u.w)));
                            *reinterpret_cast<float4 *>(orow + gc + j) = o;
                            if (rs.dig) {
                                dig += otf_dig_h((uint32_t)(gc + j), o.x);
                                dig += otf_dig_h((uint32_t)(gc + j + 1), o.y);
                                dig += otf_dig_h((uint32_t)(gc + j + 2), o.z);
                                dig += otf_dig_h((uint32_t)(gc + j + 3), o.w);
                            }
                        }
                    } else {
                        for (int j = 0; j < 32; j++)
                            if (gc + j < H) {
                                const float o = __frcp_rn(1.f + expf(-(v[j] + urow[gc + j])));
                                orow[gc + j] = o;
                                dig += otf_dig_h((uint32_t)(gc + j), o);
                            }
                    }
                }
            }
            if (rs.dig && valid) atomicAdd(&rs.dig[q], dig);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&tempty[buf])) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(tmem_cols));
}

}  // namespace tc

// EPI 0 with B = W (the recurrent update) unless b is given (EPI 1).
static int tc_gemm_launch(const DevModel &m, int prec, uint32_t n_cap, const RowSpec &rs,
                          const int32_t *in_row, const int32_t *words, const float *h_base,
                          float *out_base, const tc::TcB *b, cudaStream_t s) {
    const int H = m.H;
    tc::TcB B{};
    const int epi = b ? 1 : 0;
    if (b) {
        B = *b;
    } else {
        B.hi = m.W_hi; B.lo = m.W_lo; B.bf = m.W_bf;
        B.tiled = m.W_t64; B.tiled_np = m.wt_npad;
        B.n_rows = H;
        B.n_pad = H > 256 ? (H + 31) / 32 * 32 : (H + 15) / 16 * 16;
        if (B.n_pad > 512) return -1;
    }
    const int n_pad = B.n_pad;
    const uint32_t m_tiles = (n_cap + tc::BM - 1) / tc::BM;
    // Small problems (one decode level) are latency-bound: one tile per CTA,
    // 128-byte K chunks (half the pipeline steps).  Large ones stream tiles
    // through persistent CTAs with 64-byte chunks and deeper rings.
    const bool small = epi ? m_tiles * (uint64_t)((n_pad + 255) / 256) < 148 : m_tiles < 148;
    int bn = std::min(n_pad, (small && prec == 1) ? 128 : 256);   // bn_max; the kernel narrows it
    bn = (bn + 15) / 16 * 16;
    uint32_t cols = 32;
    while ((int)cols < 2 * bn) cols <<= 1;             // two accumulators
    if (cols > 512) return -1;
    const bool x3 = prec == 1;
    const int kcb = small ? 128 : 64;
    const int ke = prec == 2 ? kcb / 2 : kcb / 4;
    const uint32_t raw_bytes = prec == 2 ? tc::BM * (ke * 4 + 16) : 0u;
    const uint32_t stage_bytes = raw_bytes + (x3 ? 2u : 1u) * (uint32_t)(tc::BM + bn) * kcb;
    const int nk = (H + ke - 1) / ke;
    int stages = (int)std::min<uint32_t>(8u, (200u * 1024u) / stage_bytes);
    if (!small && 4u * stage_bytes <= 110u * 1024u) stages = (int)std::min<uint32_t>(8u, (110u * 1024u) / stage_bytes);
    stages = std::max(2, std::min(stages, std::max(nk, 2)));
    const size_t smem = (size_t)stages * stage_bytes + (3 * stages + 4) * 8 + 16 + 1024;
    const uint64_t tiles = small ? (uint64_t)m_tiles * ((n_pad + 31) / 32)      // finest split
                                 : (uint64_t)m_tiles * ((n_pad + bn - 1) / bn);
    cudaError_t e;
#define TC_LAUNCH(MODE, KCB, EPI)                                                               \
    do {                                                                                        \
        e = cudaFuncSetAttribute(tc::k_advance_tc<MODE, KCB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return -9;                                                        \
        int per_sm = 1;                                                                         \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tc::k_advance_tc<MODE, KCB, EPI>, tc::WS_THREADS, smem); \
        per_sm = std::max(1, std::min(per_sm, (int)(512 / cols)));                              \
        const dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)148 * per_sm))); \
        tc::k_advance_tc<MODE, KCB, EPI><<<grid, tc::WS_THREADS, smem, s>>>(m, n_cap, rs, in_row, words, h_base, \
                                                                             out_base, B, bn, stages, cols); \
    } while (0)
#define TC_PREC(KCB, EPI)                                                                       \
    do {                                                                                        \
        if (prec == 1) TC_LAUNCH(1, KCB, EPI); else if (prec == 2) TC_LAUNCH(2, KCB, EPI);      \
        else if (prec == 3) TC_LAUNCH(3, KCB, EPI); else return -1;                             \
    } while (0)
    if (kcb == 128) { if (epi) TC_PREC(128, 1); else TC_PREC(128, 0); }
    else { if (epi) TC_PREC(64, 1); else TC_PREC(64, 0); }
#undef TC_PREC
#undef TC_LAUNCH
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -9;
}

static int tc_advance_launch(const DevModel &m, int prec, uint32_t n_cap, const RowSpec &rs,
                             const int32_t *in_row, const int32_t *words, const float *h_base,
                             float *out_base, uint32_t row_limit, cudaStream_t s) {
    (void)row_limit;
    return tc_gemm_launch(m, prec, n_cap, rs, in_row, words, h_base, out_base, nullptr, s);
}

// exact_update.cuh -- the recurrent update h' = f32(sigmoid(U[w] + W h)) bit
// for bit equal to the reference's float64 arithmetic (_kernels_nb.py:51-60),
// on tcgen05 integer tensor cores.
//
// Digit planes.  Every W row i gets a power-of-two scale sW_i > max_j |W_ij|
// and X_ij = rint(W_ij / sW_i * 2^39) in five 8-bit planes (top plane signed,
// lower planes unsigned): W_ij ~ sW_i (d0 2^-7 + u1 2^-15 + ... + u4 2^-39),
// exact for |W_ij| >= 2^-15 sW_i.
// Every context row r (a sigmoid output in [0, 1), or the zero context) has
// Y_rj = rint(h_rj 2^32) in four unsigned planes (sH_r = 1; exact for
// h >= 2^-9, the rest is carried by the error bound).  A digit pair (a, b) carries the weight
// sW sH 2^-(15 + 8(a + b)); the 17 pairs with a + b <= 5 are accumulated by
// `tcgen05.mma.kind::i8` into six int32 anti-diagonal accumulators D_s
// (s = a + b) -- exactly, |D_s| < 2^28 -- and combined once:
//   x~ = U + sW sH (T_hi 2^-31 + T_lo 2^-55),
//   T_hi = D0 2^16 + D1 2^8 + D2,  T_lo = D3 2^16 + D4 2^8 + D5  (int64, exact).
// One MMA serves several pairs: the h planes sit in shared memory as
// consecutive row blocks [e0 | e1 | e2 | e3], so the MMA of W plane a over the
// row blocks b = 0..nb-1 writes TMEM column blocks s = a..a+nb-1 -- the
// anti-diagonals -- directly (N up to 4 x rows; pieces of <= 256 columns).
//
// Certified rounding.  A rigorous bound eps >= |x~ - x_ref| (x_ref = the
// reference's sequential float64 sum) covers the dropped pairs, the digit
// representation of both operands and the reference's own rounding
// (prep: per unit A_i, B_i; eps = A_i sH_r + B_i eH_r + c |U|).  The f32
// candidate y = rcp(1 + exp(-x~)) is accepted only if sigmoid over
// [x~ - eps, x~ + eps] provably stays strictly between the two f32 rounding
// midpoints around y (checked as z m - 1 against the margin, z = 1 + e^-x).
// Elements that cannot be certified (~1e-5 of them) are recomputed by the
// reference's own sequential float64 loop and sigmoid (a warp per element).  So every h' equals
// the reference's float32 result; the content dedup (context_table.py:74-86)
// then merges exactly the contexts the reference merges.
#pragma once
#include "tc_advance.cuh"

namespace xu {
constexpr int KC = 64;                 // bytes (= int8 elements) of K per ring stage
constexpr int NDIAG = 6;               // anti-diagonals s = a + b <= 5 (17 digit pairs)
constexpr int NPW = 5;                 // W digit planes (h: 4)
constexpr int XR = 80;                 // context rows per chunk: 6 accumulators x 80 columns <= 512
constexpr int PLANE_W = tc::BM * KC;   // one W plane block (128 rows x 64 B)
constexpr int FBCAP = 1024;            // deferred fallback elements per M tile

// canonical no-swizzle K-major operand layout (8-row x 16-byte core matrices,
// LBO = 128 B between K-adjacent core matrices, SBO = 512 B between 8-row groups)
__host__ __device__ __forceinline__ uint32_t toff(int row, int c) {
    return (uint32_t)((row >> 3) * (KC / 16 * 128) + c * 128 + (row & 7) * 16);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)((KC / 16 * 128) >> 4) << 32;
    d |= 1ull << 46;
    return d;
}
// D s32, A s8 (plane 0) or u8, B u8, K-major, M = 128
__host__ __device__ constexpr uint32_t idesc(bool a_signed, int n) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// One MMA whose TMEM column, A / B descriptor offsets, instruction
// descriptor and accumulate flag are immediates: only the three bases
// (stage descriptors, TMEM base) go through the uniform datapath.  With
// run-time offsets every MMA paid ~7 R2UR moves and ran at ~170 cycles
// whatever its N (tools/kloop_micro.cu); with immediates the 17 digit pairs
// of a K step run at the int8 tensor peak.
template <uint32_t TOFF, uint32_t AOFF, uint32_t BOFF, uint32_t IDESC, int ACC>
__device__ __forceinline__ void mma_imm(uint32_t tm, uint64_t da, uint64_t db) {
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\t.reg .b64 a, b;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "add.u32 t, %0, %3;\n\tadd.s64 a, %1, %4;\n\tadd.s64 b, %2, %5;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t], a, b, %6, %7;\n\t}"
                 :: "r"(tm), "l"(da), "l"(db), "n"(TOFF), "n"(AOFF >> 4), "n"(BOFF >> 4), "n"(IDESC), "n"(ACC));
}
// W plane a x h planes [b0, b0 + nb) into TMEM column blocks a + b (Rp
// columns each), split at N = 256
template <int RP, int A, int B0, int NB, int ACC>
__device__ __forceinline__ void range_imm(uint32_t tm, uint64_t da, uint64_t db) {
    constexpr int TOT = NB * RP, N1 = TOT < 256 ? TOT : 256, N2 = TOT - N1;
    mma_imm<(uint32_t)((A + B0) * RP), (uint32_t)(A * 128 * 64), (uint32_t)(((B0 * RP) >> 3) * 512),
            idesc(A == 0, N1), ACC>(tm, da, db);
    if constexpr (N2 > 0)
        mma_imm<(uint32_t)((A + B0) * RP + 256), (uint32_t)(A * 128 * 64), (uint32_t)(((B0 * RP + 256) >> 3) * 512),
                idesc(A == 0, N2), ACC>(tm, da, db);
}
// the 17 digit pairs (a + b <= 5) of one 32-byte K step into the six
// anti-diagonal accumulators; FIRST: the chunk's first K step, where each
// diagonal block is written before it accumulates
template <int RP, bool FIRST>
__device__ __forceinline__ void ks_pairs(uint32_t tm, uint64_t da, uint64_t db) {
    if constexpr (FIRST) {
        range_imm<RP, 0, 0, 4, 0>(tm, da, db);      // (0,0) (0,1) (0,2) (0,3): blocks 0-3 first written
        range_imm<RP, 1, 0, 3, 1>(tm, da, db);      // (1,0) (1,1) (1,2)
        range_imm<RP, 1, 3, 1, 0>(tm, da, db);      // (1,3): block 4 first written
        range_imm<RP, 2, 0, 3, 1>(tm, da, db);      // (2,0) (2,1) (2,2)
        range_imm<RP, 2, 3, 1, 0>(tm, da, db);      // (2,3): block 5 first written
        range_imm<RP, 3, 0, 3, 1>(tm, da, db);      // (3,0) (3,1) (3,2)
        range_imm<RP, 4, 0, 2, 1>(tm, da, db);      // (4,0) (4,1)
    } else {
        range_imm<RP, 0, 0, 4, 1>(tm, da, db);
        range_imm<RP, 1, 0, 4, 1>(tm, da, db);
        range_imm<RP, 2, 0, 4, 1>(tm, da, db);
        range_imm<RP, 3, 0, 3, 1>(tm, da, db);
        range_imm<RP, 4, 0, 2, 1>(tm, da, db);
    }
}
// one staged K chunk (KC = 64 bytes: two K steps) at a run-time Rp in {16, ..., 80}
__device__ __forceinline__ void kc_pairs(int Rp, bool first, uint32_t tm, uint64_t da, uint64_t db) {
#define XU_KS(RP)                                                                          \
    case RP:                                                                               \
        if (first) ks_pairs<RP, true>(tm, da, db); else ks_pairs<RP, false>(tm, da, db);  \
        ks_pairs<RP, false>(tm, da + 16, db + 16);                                         \
        break;
    switch (Rp) { XU_KS(16) XU_KS(32) XU_KS(48) XU_KS(64) XU_KS(80) default: break; }
#undef XU_KS
}
static_assert(KC == 64, "kc_pairs issues two 32-byte K steps per chunk");

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(d_tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// exact int32 -> float64 (|v| < 2^31) without the conversion unit
__device__ __forceinline__ double i2d(int v) {
    return __hiloint2double(0x43380000 + (v >> 31), v) - 6755399441055744.0;
}
__device__ __forceinline__ void tmem_ld8i(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// The reference's element, sequentially (_kernels_nb.py:54-58): acc = U;
// acc += W[i, j] * h[j] for j = 0..H-1 in float64 (the product of two
// floats is exact in float64, so the fma rounds like the reference's add);
// then the reference sigmoid (_kernels_nb.py:36-41) rounded to float32.
__device__ __noinline__ float ref_element(const float *__restrict__ wrow, const float *__restrict__ h, float u, int H) {
    double acc = (double)u;
    const float4 *w4 = reinterpret_cast<const float4 *>(wrow);
    const float4 *h4 = reinterpret_cast<const float4 *>(h);
    int j = 0;
    if ((H & 3) == 0) {
        for (; j < H; j += 4) {
            const float4 a = __ldg(w4 + (j >> 2)), b = __ldcg(h4 + (j >> 2));
            acc = fma((double)a.x, (double)b.x, acc);
            acc = fma((double)a.y, (double)b.y, acc);
            acc = fma((double)a.z, (double)b.z, acc);
            acc = fma((double)a.w, (double)b.w, acc);
        }
    }
    for (; j < H; j++) acc = fma((double)__ldg(wrow + j), (double)__ldcg(h + j), acc);
    return (float)otf_sigmoid(acc);
}

// exact f32 -> f64 of a normal float by integer operations (no conversion unit)
__device__ __forceinline__ double widen_d(float x) {
    const uint32_t u = __float_as_uint(x);
    return __hiloint2double((int)((u & 0x80000000u) | (((u >> 3) & 0x0FFFFFFFu) + (896u << 20))), (int)(u << 29));
}

// e^-x for |x| <= 700: k = rint(-32 x log2 e), r = -x - k ln2/32 (Cody-Waite,
// ln2_hi has 11 trailing zero bits so k ln2_hi/32 is exact), e^-x =
// 2^(k>>5) * tab[k & 31] * e^r with tab[j] = 2^(j/32) and e^r by its degree-6
// Taylor polynomial (|r| <= ln2/64: truncation < 4e-18).  Relative error
// ~1e-16, well inside the certification margin, in 12 float64 operations.
__device__ __forceinline__ double exp_neg(double x, const double *__restrict__ tab) {
    const double t = x * -46.166241308446828;                 // -32 log2(e) x
    const double sh = t + 6755399441055744.0;
    const int k = __double2loint(sh);
    const double kd = sh - 6755399441055744.0;
    double r = fma(kd, -0.021660849386535119265, -x);         // ln2_hi / 32
    r = fma(kd, -5.9631716539705865626e-12, r);               // ln2_lo / 32
    double p = 1.0 / 720.0;
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    p *= tab[k & 31];
    return __hiloint2double(__double2hiint(p) + ((k >> 5) << 20), __double2loint(p));
}

// Certified float32 rounding of sigmoid(x) (branch free, so the elements of
// a row group interleave).  epsm = the x error bound (|x - x_ref| <= eps) x
// 1.0001 + 2e-15 for the exp, Newton and the reference's own float64
// sigmoid roundings, all relative to sigmoid.  h = 1/(1 + e^-x) to ~1 f64 ulp
// (hardware reciprocal seed + two Newton steps); y = the float nearest h;
// d = h - y is exact.  sigmoid(x_ref), and the reference's float64 sigmoid
// of x_ref, round to y if |d| + epsm h stays inside the half gap to the
// neighbouring float on d's side (a quarter gap below a power of two).
// Returns false otherwise, or for |x| >= 60 / y outside the normal (0, 1).
__device__ __forceinline__ bool certify(double x, double epsm, const double *__restrict__ tab, float &out) {
    const double z = 1.0 + exp_neg(x, tab);
    double h;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(h) : "d"(z));
    h = fma(h, fma(-z, h, 1.0), h);
    h = fma(h, fma(-z, h, 1.0), h);
    const float y = __double2float_rn(h);
    const uint32_t yb = __float_as_uint(y);
    const double d = h - widen_d(y);                 // (y normal whenever the result is accepted)
    // half gap above y: 2^(E_y - 24); below: the same, halved at a power of two
    const uint32_t ey = (yb >> 23) & 255u;
    const int hw = (int)((ey + 1023u - 127u - 24u) << 20);
    const double half_up = __hiloint2double(hw, 0);
    const double half_dn = __hiloint2double((yb & 0x7FFFFFu) ? hw : hw - (1 << 20), 0);
    const double margin = epsm * h;
    out = y;
    const bool ok = d >= 0.0 ? d + margin < half_up : margin - d < half_dn;
    return ok && fabs(x) < 60.0 && ey >= 1u && yb < 0x3F800000u;
}
}  // namespace xu

// --------------------------------------------------------------------------
// model preparation (once per model upload)
// --------------------------------------------------------------------------
// per unit i (block per row): planes into the pre-tiled layout
// Wd[mt][kc][a < 5][128 rows x 64 B] and the float64 constants
// wx[i] = {sW 2^-31, epsm_i, B_i, sW 2^-55}: the certification margin of
// unit i is epsm_i + B_i eH_r (relative to sigmoid).
// kind 1 (node vectors, exact_hs.cuh): rows are the V-1 HS node vectors, laid
// out per node as NVd[node][kc][a][64 B] (gathered by rows), and
// nx[n] = {sN 2^-31, eps_n, B_n, sN 2^-55} bounds the dot with a context
// row (no U, no sigmoid margin).
__global__ void k_prep_wdigits(const float *__restrict__ W, const float *__restrict__ U, int V, int H, int nkx,
                               uint8_t *__restrict__ Wd, double4 *__restrict__ wx, int n_rows = -1, int kind = 0) {
    const int i = blockIdx.x;
    if (i >= (n_rows < 0 ? H : n_rows)) return;
    const float *row = W + (size_t)i * H;
    __shared__ float s_max[32];
    __shared__ double s_sum[4][32];
    // (the h-representation term of the bound is B_i * sum_j |dh_j| with
    // B_i = max_j |W_ij| -- only the few elements below 2^-9 carry dh)
    float mx = 0.f;
    for (int j = threadIdx.x; j < H; j += blockDim.x) mx = fmaxf(mx, fabsf(row[j]));
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? s_max[threadIdx.x] : 0.f;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) s_max[0] = v;
    }
    __syncthreads();
    mx = s_max[0];
    // max_w |U[w, i]| (the reference's sum starts from U: rounding bound)
    float mu = 0.f;
    if (U && kind == 0) for (int w = threadIdx.x; w < V; w += blockDim.x) mu = fmaxf(mu, fabsf(U[(size_t)w * H + i]));
    for (int o = 16; o; o >>= 1) mu = fmaxf(mu, __shfl_xor_sync(0xffffffffu, mu, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_max[2 + (threadIdx.x >> 5)] = mu;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = 0.f;
        for (int wv = 0; wv < (int)(blockDim.x >> 5); wv++) v = fmaxf(v, s_max[2 + wv]);
        s_max[1] = v;
    }
    __syncthreads();
    int e = 0;                                   // sW = 2^e > max |W_ij|
    if (mx > 0.f) { frexpf(mx, &e); }             // mx = f * 2^e, f in [0.5, 1)
    const double sW = ldexp(1.0, e);
    const int mt = i / tc::BM, r = i % tc::BM;
    double sum_w = 0.0, err_w = 0.0, s3 = 0.0, s4 = 0.0;
    for (int j = threadIdx.x; j < nkx * xu::KC; j += blockDim.x) {
        int dg[xu::NPW] = {0, 0, 0, 0, 0};
        if (j < H) {
            const double w = (double)row[j];
            const long long X = llrint(ldexp(w, 39 - e));           // |X| < 2^39
            const long long d0 = X >> 32;
            const long long R = X - (d0 << 32);                      // [0, 2^32)
            dg[0] = (int)d0; dg[1] = (int)(R >> 24); dg[2] = (int)((R >> 16) & 255);
            dg[3] = (int)((R >> 8) & 255); dg[4] = (int)(R & 255);
            sum_w += fabs(w);
            err_w += fabs(ldexp((double)X, e - 39) - w);
            s3 += dg[3]; s4 += dg[4];
        }
        const int kc = j / xu::KC, kk = j % xu::KC;
        if (kind == 0) {
            const size_t blk = ((size_t)mt * nkx + kc) * xu::NPW;
            const uint32_t o = xu::toff(r, kk >> 4) + (kk & 15);
#pragma unroll
            for (int a = 0; a < xu::NPW; a++) Wd[(blk + a) * xu::PLANE_W + o] = (uint8_t)dg[a];
        } else {
            uint8_t *dst = Wd + (((size_t)i * nkx + kc) * xu::NPW) * xu::KC + kk;
#pragma unroll
            for (int a = 0; a < xu::NPW; a++) dst[(size_t)a * xu::KC] = (uint8_t)dg[a];
        }
    }
    double v4[4] = {sum_w, err_w, s3, s4};
#pragma unroll
    for (int k = 0; k < 4; k++)
        for (int o = 16; o; o >>= 1) v4[k] += __shfl_xor_sync(0xffffffffu, v4[k], o);
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 4; k++) s_sum[k][threadIdx.x >> 5] = v4[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[4] = {0, 0, 0, 0};
        for (int wv = 0; wv < (int)(blockDim.x >> 5); wv++)
            for (int k = 0; k < 4; k++) t[k] += s_sum[k][wv];
        // dropped pairs (3,3), (4,2), (4,3): |D_ab| <= (sum_j |w_a|) * 255
        const double drop = 255.0 * (t[2] * ldexp(1.0, -63) + t[3] * ldexp(1.0, -63) + t[3] * ldexp(1.0, -71));
        const double c1 = (double)(H + 8) * ldexp(1.0, -53) * 1.01;   // sequential-sum rounding
        // (context rows are scaled by sH = 1: sum_j |W_ij h_j| <= sum_j |W_ij|)
        const double eps = (drop * sW + t[1]) * 1.01 + c1 * (t[0] + (double)s_max[1]) * 1.01;
        double4 o;
        o.x = ldexp(sW, -31);
        o.y = kind == 0 ? eps * 1.0001 + 2.0e-15 : eps;             // W: epsm without the h term
        o.z = (double)mx * 1.01 * (kind == 0 ? 1.0001 : 1.0);        // coefficient of eH_r (sum |dh|)
        o.w = ldexp(sW, -55);
        wx[i] = o;
    }
}

// --------------------------------------------------------------------------
// One level's exact recurrent update inside the persistent stream kernel
// (rank 1 of the cluster, all NT threads).  n rows (the level's computed
// requests) at arena rows base..base+n-1, sources Q.pr_inrow[], words Q.pr_w[].
// Per chunk of <= XR rows: digitize the source rows into the stream's global
// scratch (the ring's h block layout), then per 128-unit M tile a K loop
// (warp 1 bulk-copies the W and h plane blocks of each 64-byte K chunk into
// the ring, warp 0 issues the digit-pair MMAs) and the epilogue of all warps
// (combine, certify, store, digest); uncertified elements are recomputed by
// the reference loop after the tile, a warp per element.
// --------------------------------------------------------------------------
namespace xu {
struct Ring {
    uint8_t *smem;                 // stages x STAGE bytes
    int stages;
    uint32_t tmem;
    uint64_t *full, *empty, *done;
    uint32_t *fb;                  // [2][FBCAP] deferred fallback elements (row << 16 | unit)
    uint32_t *fb_n;                // [2]
    double *sh, *eh;               // [2][XR] per chunk row: scale sH, sum_j |dh_j| (by chunk parity)
    int32_t *src;                  // [XR] per chunk row: its source context's arena row
    int32_t *wrd;                  // [XR] per chunk row: its word x H (U row offset)
    const double *tab;             // [32] 2^(j/32) for exp_neg
    // rows: source context rows hin[in_row[q]], words (nullptr: word = q), results
    // hout[q], content-digest terms dig[q] (nullptr: none), work counters alg
    const float *hin;
    float *hout;
    const int32_t *in_row, *words;
    unsigned long long *dig, *alg;
    // per-arena-row planes made at row creation (nullptr: digitize every chunk)
    uint8_t *dig_store;
    float *deh_store;
    uint32_t *dep_store;
    uint32_t epoch;
    uint8_t *xs;                   // this stream's global digit scratch: 2 chunk slots (by parity)
    size_t xs_slot;                // bytes per slot
    float *us;                     // [XR][128] U[w_r, tile units], staged during the tile's K loop
                                   // (nullptr: the epilogue reads U from global memory)
    // non-null: the epilogue also writes each result's digit planes into
    // this per-row store (row out_row0 + q; deh_store / dep_store as
    // digitize_to_store), so no separate digitize pass follows the update
    uint8_t *fuse_store = nullptr;
    uint32_t out_row0 = 0;
    unsigned long long *phase_g = nullptr;   // profiling: warp 2's sections under the K loops -> [28, 32)
};
constexpr uint32_t US_BYTES = (uint32_t)XR * 128 * 4;
constexpr uint32_t STAGE = (uint32_t)NPW * PLANE_W + 4u * XR * KC;
constexpr uint32_t HOFF = (uint32_t)NPW * PLANE_W;
// rank 1's shared memory after its ring (byte offsets); sh / eh are double
// buffered by chunk parity because rank 0 reads a chunk's eh (DSMEM) while
// rank 1 already digitizes the next chunk
struct TailLayout { uint32_t fb, sh, eh, fbn, src, wrd, tab, total; };
__host__ __device__ constexpr TailLayout tail_layout() {
    return TailLayout{0u, 2u * FBCAP * 4, 2u * FBCAP * 4 + 2u * XR * 8, 2u * FBCAP * 4 + 4u * XR * 8,
                      2u * FBCAP * 4 + 4u * XR * 8 + 16, 2u * FBCAP * 4 + 4u * XR * 8 + 16 + XR * 4,
                      2u * FBCAP * 4 + 4u * XR * 8 + 16 + 2u * XR * 4,
                      2u * FBCAP * 4 + 4u * XR * 8 + 16 + 2u * XR * 4 + 32 * 8};
}
// one chunk of h digit planes in the global scratch: [kc][plane][XR rows x 64 B]
__host__ __device__ constexpr size_t xs_slot_bytes(int nkx) { return (size_t)nkx * 4 * XR * KC; }

// Y = rint(h 2^32) of one h element and the representation error
// |h - Y 2^-32| (every context row uses the scale sH = 1: hidden states are
// sigmoid outputs in [0, 1), and the zero context is 0).  h >= 2^-9 is exact;
// smaller, non-finite, negative or >= 1 values are still bounded by err.
__device__ __forceinline__ uint32_t digit_word(float h, float &err) {
    const uint32_t u = __float_as_uint(h);
    const uint32_t E = u >> 23;                          // biased exponent (sign bit -> >= 256)
    if (E >= 118u && E < 127u) {                          // [2^-9, 1): 24-bit significand << (E - 118)
        err = 0.f;
        return ((u & 0x7FFFFFu) | 0x800000u) << (E - 118u);
    }
    if (E < 118u) {                                      // tiny (or zero / subnormal): Y < 2^24
        const uint32_t Y = __float2uint_rn(h * 4294967296.f);
        err = fabsf(h - (float)Y * 2.3283064365386963e-10f);
        return Y;
    }
    err = (u >> 31) ? fabsf(h) : fabsf(h - 1.0f) + 2.3283064365386963e-10f;   // negative / >= 1 / NaN
    return (u >> 31) ? 0u : 0xFFFFFFFFu;
}

// The reference's element (_kernels_nb.py:54-58) by one warp: lane l holds
// elements [l P, (l + 1) P) of the W row and the context row; the exact
// float64 products are formed in parallel, then the sum runs in the
// reference's order, lane after lane (acc = U; acc += p_j for j = 0..H-1).
template <int P>
__device__ __forceinline__ float ref_element_warp(const float *__restrict__ wrow, const float *__restrict__ h,
                                                 float u, int H, int lane) {
    double p[P];
#pragma unroll
    for (int k = 0; k < P; k += 4) {
        const int j = lane * P + k;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (j < H) { a = __ldg(reinterpret_cast<const float4 *>(wrow + j)); b = __ldcg(reinterpret_cast<const float4 *>(h + j)); }
        p[k] = (double)a.x * (double)b.x; p[k + 1] = (double)a.y * (double)b.y;
        p[k + 2] = (double)a.z * (double)b.z; p[k + 3] = (double)a.w * (double)b.w;
    }
    double acc = (double)u;
    const int nl = (H + P - 1) / P;
    for (int l = 0; l < nl; l++) {
        if (lane == l) {
#pragma unroll
            for (int k = 0; k < P; k++)
                if (l * P + k < H) acc += p[k];
        }
        acc = __shfl_sync(0xffffffffu, acc, l);
    }
    return (float)otf_sigmoid(acc);
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// 16 consecutive elements of a context row -> their four digit-plane
// words per plane (pl[plane][4 x 4 bytes]) and the representation-error sum
__device__ __forceinline__ void planes16(const float (&x)[16], uint32_t (&pl)[4][4], float &esum) {
    esum = 0.f;                  // errors are exact multiples of tiny powers of two; f32 sum + 1% slack
#pragma unroll
    for (int v = 0; v < 4; v++) {
        uint32_t Y[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            float err;
            Y[k] = digit_word(x[4 * v + k], err);
            esum += err;
        }
        // plane b = byte 3 - b of the four words (byte permutes)
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const uint32_t sel = (uint32_t)(3 - b) | ((uint32_t)(7 - b) << 4);
            pl[b][v] = __byte_perm(__byte_perm(Y[0], Y[1], sel), __byte_perm(Y[2], Y[3], sel), 0x5410);
        }
    }
}
__device__ __forceinline__ void load16(const float *hrow, int g, int H, bool live, float (&x)[16]) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
        const int j = g * 16 + v * 4;
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live && j < H) t = __ldcg(reinterpret_cast<const float4 *>(hrow + j));
        x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
    }
}

// The digit planes of arena rows [row0, row0 + n) into the per-row store
// (right after the rows are created), tagged with this launch's epoch.
// Thread = (row, 16-element group); the row's lanes reduce its error sum.
template <int NT>
__device__ __forceinline__ void digitize_to_store(const DevModel &m, const float *__restrict__ hin, uint32_t row0,
                                                  uint32_t n, uint8_t *store, float *deh, uint32_t *dep,
                                                  uint32_t epoch, int tid, int wid, int lane) {
    constexpr int NW = NT / 32;
    const int H = m.H, NK = m.wd_nkx, NG = NK * 4;
    int NGP = 4;
    while (NGP < NG) NGP <<= 1;
    const int RPW = 32 / NGP;
    for (uint32_t rb = (uint32_t)(wid * RPW); rb < n; rb += (uint32_t)(2 * NW * RPW)) {
        float xa[16], xb[16];
        const uint32_t ra = rb + lane / NGP, rbb = ra + NW * RPW;
        const int g = lane % NGP;
        const bool la = ra < n && g < NG, lb = rbb < n && g < NG;
        load16(hin + (size_t)(row0 + (la ? ra : 0)) * H, g, H, la, xa);
        load16(hin + (size_t)(row0 + (lb ? rbb : 0)) * H, g, H, lb, xb);
#pragma unroll
        for (int half = 0; half < 2; half++) {
            uint32_t pl[4][4];
            float esum;
            planes16(half ? xb : xa, pl, esum);
            if (__any_sync(0xffffffffu, esum != 0.f))
                for (int o = NGP >> 1; o; o >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, o);
            const uint32_t r = half ? rbb : ra;
            if (half ? lb : la) {
                uint8_t *dst = store + ((size_t)(row0 + r) * NK + (g >> 2)) * 4 * KC + (g & 3) * 16;
#pragma unroll
                for (int b = 0; b < 4; b++)
                    *reinterpret_cast<uint4 *>(dst + b * KC) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
                if (g == 0) { deh[row0 + r] = esum * 1.01f; dep[row0 + r] = epoch; }
            }
        }
    }
}

struct NoSide {
    __device__ void operator()(int, int) const {}
};

// side(t, n): work for warps 2.. (thread t of n) under the first tile's K
// loop; when it uses the U staging area, side_uses_us makes the first tile's
// epilogue read U from global memory instead
template <int NT, typename WaitFn, typename SyncFn, typename SideFn = NoSide>
__device__ __forceinline__ void update_chunk(const DevModel &m, uint32_t q0, int R, int chunk, const Ring &rg0, uint32_t &gctr,
                                             uint32_t &tiles_done, int tid, int wid, int lane, WaitFn wait,
                                             SyncFn digits_ready, unsigned long long *ph, unsigned long long &t0,
                                             int mt0, int mt1, bool digitize, SideFn side = SideFn(),
                                             bool side_uses_us = false) {
    constexpr int NW = NT / 32;
    const int H = m.H, NK = m.wd_nkx, nmt = (H + tc::BM - 1) / tc::BM;
    auto mark = [&](int i) {
        if (ph) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); ph[i] += t - t0; t0 = t; }
    };
    // this chunk's parity slot of the digit scratch and (the digitizing
    // rank's) sh / eh; the other rank passes its own copy of eh
    Ring rg = rg0;
    rg.xs = rg0.xs + (size_t)(chunk & 1) * rg0.xs_slot;
    if (digitize) {
        rg.sh = rg0.sh + (chunk & 1) * XR;
        rg.eh = rg0.eh + (chunk & 1) * XR;
    }
    // digitize geometry: NG 16-element groups per row, a power-of-two lane
    // group per row (NGP lanes), 32 / NGP rows per warp
    const int NG = NK * 4;
    int NGP = 4;
    while (NGP < NG) NGP <<= 1;
    const int RPW = 32 / NGP;
    {
        const int Rp = (R + 15) & ~15;
        // ---- digitize the chunk's context rows: thread = (row, 16-element group) ----
        // row table; with the per-row plane store also each row's freshness
        // (planes made when the row was created in this launch: sh[r] = 1)
        for (int r = tid; r < R; r += NT) {
            const int src = rg.in_row[q0 + r];
            rg.src[r] = src;
            if (rg.fuse_store && mt0 < mt1) {
                rg.deh_store[rg.out_row0 + q0 + r] = 0.f;
                rg.dep_store[rg.out_row0 + q0 + r] = rg.epoch;
            }
            rg.wrd[r] = (rg.words ? rg.words[q0 + r] : (int32_t)(q0 + r)) * H;
            if (digitize && rg.dig_store) {
                const bool fresh = rg.dep_store[src] == rg.epoch;
                rg.sh[r] = fresh ? 1.0 : 0.0;
                if (!fresh && rg.alg) atomicAdd(&rg.alg[5], 1ull);
                if (fresh) rg.eh[r] = (double)rg.deh_store[src];
            }
        }
        __syncthreads();
        mark(12);
        if (digitize && rg.dig_store) {
            // fresh rows: a copy of their planes into the chunk layout; other
            // rows (the zero context, rows of an earlier launch or another
            // schedule) are digitized here
            mark(24);
            // warp per (kc, plane) block: lane = c * 8 + (row & 7), so each of the
            // block's 8-row groups is one contiguous 512-byte write of the
            // canonical layout; all groups' loads are in flight together.  Rows
            // not made in this launch are copied too and overwritten below.
            {
                const int KP = NK * 4, g8n = Rp >> 3;
                const size_t row_bytes = (size_t)KP * KC;
                for (int kp = wid; kp < KP; kp += NW) {
                    uint4 v[XR / 8];
#pragma unroll
                    for (int g8 = 0; g8 < XR / 8; g8++) {
                        const int r = g8 * 8 + (lane & 7);
                        v[g8] = make_uint4(0u, 0u, 0u, 0u);
                        if (g8 < g8n && r < R)
                            v[g8] = __ldcg(reinterpret_cast<const uint4 *>(rg.dig_store + (size_t)rg.src[r] * row_bytes +
                                                                           (size_t)kp * KC) + (lane >> 3));
                    }
#pragma unroll
                    for (int g8 = 0; g8 < XR / 8; g8++)
                        if (g8 < g8n)
                            *reinterpret_cast<uint4 *>(rg.xs + (size_t)kp * Rp * KC + (size_t)g8 * 512 + lane * 16) = v[g8];
                }
            }
            __syncthreads();
            mark(25);
            for (int rb = wid * RPW; rb < R; rb += NW * RPW) {
                const int r = rb + lane / NGP, g = lane % NGP;
                const bool live = r < R && g < NG;
                const bool todo = live && rg.sh[r] == 0.0;
                if (__any_sync(0xffffffffu, todo)) {
                    float x[16];
                    load16(rg.hin + (size_t)(live ? rg.src[r] : 0) * H, g, H, todo, x);
                    uint32_t pl[4][4];
                    float esum;
                    planes16(x, pl, esum);
                    if (__any_sync(0xffffffffu, esum != 0.f))
                        for (int o = NGP >> 1; o; o >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, o);
                    if (todo) {
                        uint8_t *blk = rg.xs + (size_t)(g >> 2) * 4 * Rp * KC + toff(r, g & 3);
#pragma unroll
                        for (int b = 0; b < 4; b++)
                            *reinterpret_cast<uint4 *>(blk + (size_t)b * Rp * KC) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
                        if (g == 0) rg.eh[r] = (double)esum * 1.01;
                    }
                }
            }
            mark(13);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            digits_ready();
        } else if (digitize) {
        auto load = [&](int rb, float (&x)[16]) {
            const int r = rb + lane / NGP, g = lane % NGP;
            const bool live = r < R && g < NG;
            const float *hrow = rg.hin + (size_t)(live ? rg.src[r] : 0) * H;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const int j = g * 16 + v * 4;
                float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                if (live && j < H) t = __ldcg(reinterpret_cast<const float4 *>(hrow + j));
                x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
            }
        };
        auto emit = [&](int rb, const float (&x)[16]) {
            const int r = rb + lane / NGP, g = lane % NGP;
            const bool live = r < R && g < NG;
            float esum = 0.f;          // errors are exact multiples of tiny powers of two; f32 sum + 1% slack
            uint32_t pl[4][4];
#pragma unroll
            for (int v = 0; v < 4; v++) {
                uint32_t Y[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    float err;
                    Y[k] = digit_word(x[4 * v + k], err);
                    esum += err;
                }
                // plane b = byte 3 - b of the four words (byte permutes)
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const uint32_t sel = (uint32_t)(3 - b) | ((uint32_t)(7 - b) << 4);
                    pl[b][v] = __byte_perm(__byte_perm(Y[0], Y[1], sel), __byte_perm(Y[2], Y[3], sel), 0x5410);
                }
            }
            // (rare) representation errors: reduce only when some lane has one
            if (__any_sync(0xffffffffu, esum != 0.f))
                for (int o = NGP >> 1; o; o >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, o);
            if (live) {
                uint8_t *blk = rg.xs + (size_t)(g >> 2) * 4 * Rp * KC + toff(r, g & 3);
#pragma unroll
                for (int b = 0; b < 4; b++)
                    *reinterpret_cast<uint4 *>(blk + (size_t)b * Rp * KC) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
                if (g == 0) { rg.sh[r] = 1.0; rg.eh[r] = (double)esum * 1.01; }
            }
        };
        // three row blocks per trip: their loads are in flight together
        for (int rb = wid * RPW; rb < R; rb += 3 * NW * RPW) {
            float xa[16], xb[16], xc[16];
            load(rb, xa);
            load(rb + NW * RPW, xb);
            load(rb + 2 * NW * RPW, xc);
            emit(rb, xa);
            emit(rb + NW * RPW, xb);
            emit(rb + 2 * NW * RPW, xc);
        }
        // rows R..Rp-1 of the h blocks are never read back from TMEM (their
        // columns are skipped by the epilogue), whatever the scratch holds
        mark(13);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        digits_ready();                       // rank 0's HS reads this chunk's planes too
        }
        mark(1);
        if (mt0 >= mt1) return;
        const uint32_t hbytes = 4u * (uint32_t)Rp * KC;
        // warp 1: the W plane block (mt, kc) + h plane block kc of stage gctr + kc
        auto produce = [&](int mt, int kc0, int kc1) {
            for (int kc = kc0; kc < kc1; kc++) {
                const uint32_t gc = gctr + kc;
                const int st = (int)(gc % (uint32_t)rg.stages);
                const uint32_t use = gc / (uint32_t)rg.stages;
                if (use >= 1) wait(tc::smem_u32(&rg.empty[st]), (use - 1) & 1, 11);
                __syncwarp();
                uint8_t *sW = rg.smem + (size_t)st * STAGE;
                const uint8_t *srcW = m.Wd + ((size_t)mt * NK + kc) * NPW * PLANE_W;
                const uint8_t *srcH = rg.xs + (size_t)kc * hbytes;
                asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                             "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %6;\n\t"
                             "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t"
                             "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5], %7, [%1];\n\t}"
                             :: "r"(tc::smem_u32(sW)), "r"(tc::smem_u32(&rg.full[st])), "l"(srcW),
                                "r"(HOFF), "r"(tc::smem_u32(sW + HOFF)), "l"(srcH),
                                "r"(HOFF + hbytes), "r"(hbytes) : "memory");
            }
        };
        const int npre = min(rg.stages, NK);        // stages of a tile issued ahead (during the previous epilogue)
        // result element (row, unit) = y into the per-row plane store (fused digitize):
        // plane b is byte 3 - b of Y = rint(y 2^32) at byte offset (unit mod 64) of K chunk unit / 64
        auto put_planes = [&](int row, int unit, float y) {
            float err;
            const uint32_t Y = digit_word(y, err);
            const uint32_t orow = rg.out_row0 + q0 + (uint32_t)row;
            uint8_t *dst = rg.fuse_store + ((size_t)orow * NK + (unit >> 6)) * 4 * KC + (unit & 63);
            dst[0] = (uint8_t)(Y >> 24);
            dst[KC] = (uint8_t)(Y >> 16);
            dst[2 * KC] = (uint8_t)(Y >> 8);
            dst[3 * KC] = (uint8_t)Y;
            if (err != 0.f) atomicAdd(&rg.deh_store[orow], err * 1.01f);
        };
        // the reference loop for tile mt's uncertified elements, a warp per
        // element among warps [w0, NW)
        auto fallbacks = [&](int mt, int w0) {
            uint32_t *fbl = rg.fb + ((mt - mt0) & 1) * FBCAP;
            uint32_t *fbn = rg.fb_n + ((mt - mt0) & 1);
            const uint32_t nf = min(*fbn, (uint32_t)FBCAP);
            for (uint32_t k = (uint32_t)(wid - w0); k < nf; k += (uint32_t)(NW - w0)) {
                const uint32_t e = fbl[k];
                const int row = (int)(e >> 16), un = (int)(e & 0xFFFFu);
                const float *wr = m.W + (size_t)un * H, *hr = rg.hin + (size_t)rg.src[row] * H;
                const float uu = __ldg(m.U + (size_t)rg.wrd[row] + un);
                float y;
                if (H <= 128) y = ref_element_warp<4>(wr, hr, uu, H, lane);
                else if (H <= 256) y = ref_element_warp<8>(wr, hr, uu, H, lane);
                else y = ref_element_warp<16>(wr, hr, uu, H, lane);
                if (lane == 0) {
                    rg.hout[(size_t)(q0 + row) * H + un] = y;
                    if (rg.dig) atomicAdd(&rg.dig[q0 + row], otf_dig_h((uint32_t)un, y));
                    if (rg.fuse_store) put_planes(row, un, y);
                }
            }
        };
        auto fallbacks_done = [&](int mt) {        // one thread, after a barrier that follows fallbacks(mt)
            uint32_t *fbn = rg.fb_n + ((mt - mt0) & 1);
            if (rg.alg) atomicAdd(&rg.alg[3], (unsigned long long)*fbn);
            *fbn = 0u;
        };
        // With a U staging block the epilogue only certifies: it leaves tile
        // mt's results y[row][unit] in that block (NaN: uncertified, left to
        // the fallbacks), and this pass -- a warp per row among warps
        // [w0, NW), under the next tile's K loop -- stores them: 512-byte
        // hidden-row segments, the digit planes (4-byte words of the per-row
        // store), one digest atomic and one error sum per row and tile.
        auto rows_out = [&](int mt, int w0) {
            const int c4 = lane * 4, u = mt * tc::BM + c4;
            // the ring's fields in registers (the struct itself may live in local memory)
            const float *__restrict__ us = rg.us;
            float *__restrict__ hout = rg.hout;
            uint8_t *__restrict__ fuse = rg.fuse_store;
            unsigned long long *__restrict__ dig = rg.dig;
            float *__restrict__ deh = rg.deh_store;
            const uint32_t orow0 = rg.out_row0 + q0;
            for (int r = wid - w0; r < R; r += NW - w0) {
                unsigned long long dgs = 0ull;
                float es = 0.f;
                if (u < H) {                          // (H % 4 == 0: whole float4s)
                    const float4 y4 = *reinterpret_cast<const float4 *>(us + r * 128 + c4);
                    const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
                    bool ok[4];
#pragma unroll
                    for (int k = 0; k < 4; k++) ok[k] = !isnan(yv[k]);
                    float *ho = hout + (size_t)(q0 + r) * H + u;
                    if (ok[0] && ok[1] && ok[2] && ok[3]) *reinterpret_cast<float4 *>(ho) = y4;
                    else {
#pragma unroll
                        for (int k = 0; k < 4; k++) if (ok[k]) ho[k] = yv[k];
                    }
                    uint32_t Y[4];
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        float err = 0.f;
                        Y[k] = ok[k] ? digit_word(yv[k], err) : 0u;
                        es += err;
                        if (ok[k]) dgs += otf_dig_h((uint32_t)(u + k), yv[k]);
                    }
                    if (fuse) {
                        uint8_t *dst = fuse + ((size_t)(orow0 + r) * NK + (u >> 6)) * 4 * KC + (u & 63);
#pragma unroll
                        for (int b = 0; b < 4; b++) {
                            const uint32_t sel = (uint32_t)(3 - b) | ((uint32_t)(7 - b) << 4);
                            *reinterpret_cast<uint32_t *>(dst + b * KC) =
                                __byte_perm(__byte_perm(Y[0], Y[1], sel), __byte_perm(Y[2], Y[3], sel), 0x5410);
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) dgs += __shfl_xor_sync(0xffffffffu, dgs, o);
                if (lane == 0 && dig) atomicAdd(&dig[q0 + r], dgs);
                if (fuse && __any_sync(0xffffffffu, es != 0.f)) {
#pragma unroll
                    for (int o = 16; o; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
                    if (lane == 0) atomicAdd(&deh[orow0 + r], es * 1.01f);
                }
            }
        };
        const bool ystage = rg.us != nullptr;
        for (int mt = mt0; mt < mt1; mt++) {
            unsigned long long g0 = 0;
            auto gmark = [&](int i) {
                if (rg.phase_g && tid == 64) {
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (i >= 0) atomicAdd(&rg.phase_g[i], t - g0);
                    g0 = t;
                }
            };
            gmark(-1);
            if (wid >= 2 && mt > mt0) {
                // the previous tile's results and uncertified elements, under this tile's K loop
                if (ystage) {
                    rows_out(mt - 1, 2);
                    gmark(29);
                    named_sync(3, NT - 64);
                }
                // (no barrier after the fallbacks: the U staging below does not
                // touch what they read, and their list is reset after the
                // tile's completion barrier)
                fallbacks(mt - 1, 2);
                gmark(30);
            }
            const bool us_t = rg.us && !(side_uses_us && mt == mt0);
            if (wid >= 2 && mt == mt0) { side(tid - 64, NT - 64); gmark(28); }
            if (wid >= 2 && us_t) {
                // this tile's U block U[w_r, mt*128 + (0..127)] into shared memory,
                // under the K loop (the previous epilogue is done with it)
                const int u0 = mt * tc::BM;
                for (int i = tid - 64; i < R * 32; i += NT - 64) {
                    const int r = i >> 5, c4 = (i & 31) * 4;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (u0 + c4 < H) v = __ldg(reinterpret_cast<const float4 *>(m.U + (size_t)rg.wrd[r] + u0 + c4));
                    *reinterpret_cast<float4 *>(rg.us + r * 128 + c4) = v;
                }
                gmark(31);
            }
            if (wid == 1) {
                produce(mt, mt == mt0 ? 0 : npre, NK);
            } else if (wid == 0) {
                // ---- MMA issuer: 17 digit pairs per 32-byte K step ----
                for (int kc = 0; kc < NK; kc++) {
                    const uint32_t gc = gctr + kc;
                    const int st = (int)(gc % (uint32_t)rg.stages);
                    wait(tc::smem_u32(&rg.full[st]), (gc / (uint32_t)rg.stages) & 1, 12);
                    __syncwarp();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sW = tc::smem_u32(rg.smem + (size_t)st * STAGE);
                    // 17 digit pairs per 32-byte K step (ks_pairs), immediates off two stage descriptors
                    kc_pairs(Rp, kc == 0, rg.tmem, desc(sW), desc(sW + HOFF));
                    tc::commit_elect(tc::smem_u32(&rg.empty[st]));
                    if (kc == NK - 1) tc::commit_elect(tc::smem_u32(rg.done));
                    __syncwarp();
                }
            }
            gctr += NK;
            // one warp polls the tile's completion; the others block in the
            // hardware barrier instead of spinning on the mbarrier
            if (wid == 0) wait(tc::smem_u32(rg.done), tiles_done & 1, 13);
            mark(26);
            tiles_done++;
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (tid == 64 && mt > mt0) fallbacks_done(mt - 1);   // every warp is past fallbacks(mt - 1)
            // the ring is drained: issue the next tile's first stages now, so
            // they load while this tile's epilogue runs
            if (wid == 1 && mt + 1 < mt1) produce(mt + 1, 0, npre);
            mark(2);
            // ---- epilogue: TMEM lane = output unit, columns s * Rp + row;
            // the 4 warps of a lane quadrant take groups of 4 rows in turn ----
            const int quad = wid & 3;
            const int unit = mt * tc::BM + quad * 32 + lane;
            float *__restrict__ us_e = rg.us;               // ring fields in registers
            const double *__restrict__ eh_e = rg.eh;
            const double *__restrict__ tab_e = rg.tab;
            const int32_t *__restrict__ wrd_e = rg.wrd;
            const uint32_t tmem_e = rg.tmem;
            const bool uok = unit < H;
            double4 k4 = make_double4(0.0, 0.0, 0.0, 0.0);
            if (uok) k4 = m.wx[unit];
            uint32_t *fbl = rg.fb + ((mt - mt0) & 1) * FBCAP;
            uint32_t *fbn = rg.fb_n + ((mt - mt0) & 1);
            const float *ucol = m.U + (uok ? unit : 0);
            const int n4 = (R + 3) >> 2;
            for (int it = wid >> 2; it < n4; it += NW / 4) {
                const int r0 = it * 4;
                mark(27);
                float uv[4];          // U[w, unit] of the group's rows (V H < 2^31: 32-bit offsets)
                if (us_t) {
#pragma unroll
                    for (int g = 0; g < 4; g++) uv[g] = us_e[min(r0 + g, R - 1) * 128 + quad * 32 + lane];
                } else {
#pragma unroll
                    for (int g = 0; g < 4; g++) uv[g] = __ldg(ucol + wrd_e[min(r0 + g, R - 1)]);
                }
                long long th[4], tl[4];
                {
                    uint32_t D[NDIAG][4];
                    const uint32_t ta = tmem_e + ((uint32_t)(quad * 32) << 16) + (uint32_t)r0;
#pragma unroll
                    for (int s2 = 0; s2 < NDIAG; s2++)
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(D[s2][0]), "=r"(D[s2][1]), "=r"(D[s2][2]), "=r"(D[s2][3])
                                     : "r"(ta + (uint32_t)(s2 * Rp)));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    mark(14);
#pragma unroll
                    for (int g = 0; g < 4; g++) {
                        th[g] = ((long long)(int)D[0][g] << 16) + ((long long)(int)D[1][g] << 8) + (long long)(int)D[2][g];
                        tl[g] = ((long long)(int)D[3][g] << 16) + ((long long)(int)D[4][g] << 8) + (long long)(int)D[5][g];
                    }
                }
                bool okv[4];
                float yv[4];
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    // |T_hi| < 2^41, |T_lo| < 2^44: exact int64 -> f64 through the 1.5 * 2^52 magic
                    const double dh = __longlong_as_double(th[g] + 0x4338000000000000LL) - 6755399441055744.0;
                    const double dlo = __longlong_as_double(tl[g] + 0x4338000000000000LL) - 6755399441055744.0;
                    const double x = fma(dh, k4.x, fma(dlo, k4.w, widen(uv[g])));
                    const double epsm = fma(k4.z, eh_e[min(r0 + g, R - 1)], k4.y);
                    okv[g] = certify(x, epsm, tab_e, yv[g]);
                }
                if (ph) { const float y0 = yv[0] + yv[1] + yv[2] + yv[3]; asm volatile("" :: "f"(y0)); }
                mark(15);
                if (ystage) {
                    // results into the staging block (rows_out stores them); uncertified -> NaN + list
#pragma unroll
                    for (int g = 0; g < 4; g++) {
                        const int row = r0 + g;
                        if (uok && row < R) {
                            float y = yv[g];
                            if (!okv[g]) {
                                y = __int_as_float(0x7fffffff);
                                const uint32_t k = atomicAdd(fbn, 1u);
                                if (k < (uint32_t)FBCAP) fbl[k] = ((uint32_t)row << 16) | (uint32_t)unit;
                                else                                  // list full: recompute here
                                    y = ref_element(m.W + (size_t)unit * H, rg.hin + (size_t)rg.src[row] * H, uv[g], H);
                            }
                            us_e[row * 128 + quad * 32 + lane] = y;
                        }
                    }
                    continue;
                }
                unsigned long long dg[4];
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    dg[g] = 0ull;
                    const int row = r0 + g;
                    if (uok && row < R) {
                        if (okv[g]) {
                            rg.hout[(size_t)(q0 + row) * H + unit] = yv[g];
                            dg[g] = otf_dig_h((uint32_t)unit, yv[g]);
                            if (rg.fuse_store) put_planes(row, unit, yv[g]);
                        } else {
                            const uint32_t k = atomicAdd(fbn, 1u);
                            if (k < (uint32_t)FBCAP) fbl[k] = ((uint32_t)row << 16) | (uint32_t)unit;
                            else {                                   // list full: recompute here
                                const float y = ref_element(m.W + (size_t)unit * H,
                                                            rg.hin + (size_t)rg.src[row] * H, uv[g], H);
                                rg.hout[(size_t)(q0 + row) * H + unit] = y;
                                dg[g] = otf_dig_h((uint32_t)unit, y);
                                if (rg.fuse_store) put_planes(row, unit, y);
                            }
                        }
                    }
                }
                // digest terms of the 4 rows summed over the warp's 32 units:
                // the sum for row g lands on the lanes whose bits (4,3) spell g
                {
                    const bool u16 = lane & 16, u8 = lane & 8;
#pragma unroll
                    for (int i2 = 0; i2 < 2; i2++) {
                        const unsigned long long send = u16 ? dg[i2] : dg[i2 + 2], keep = u16 ? dg[i2 + 2] : dg[i2];
                        dg[i2] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
                    const unsigned long long send = u8 ? dg[0] : dg[1], keep = u8 ? dg[1] : dg[0];
                    unsigned long long x2 = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    x2 += __shfl_xor_sync(0xffffffffu, x2, 4);
                    x2 += __shfl_xor_sync(0xffffffffu, x2, 2);
                    x2 += __shfl_xor_sync(0xffffffffu, x2, 1);
                    const int row = r0 + ((lane >> 3) & 3);
                    if ((lane & 7) == 0 && row < R && rg.dig) atomicAdd(&rg.dig[q0 + row], x2);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            mark(3);
        }
        // the last tile's results and uncertified elements (every warp)
        if (ystage) {
            rows_out(mt1 - 1, 0);
            __syncthreads();
        }
        fallbacks(mt1 - 1, 0);
        __syncthreads();
        if (tid == 0) fallbacks_done(mt1 - 1);
        mark(10);
    }
}
}  // namespace xu

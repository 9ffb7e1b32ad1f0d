// exact_update.cuh -- the recurrent update h' = f32(sigmoid(U[w] + W h)) bit
// for bit equal to the reference's float64 arithmetic (_kernels_nb.py:51-60),
// on tcgen05 integer tensor cores.
//
// Digit planes.  Every W row i gets a power-of-two scale sW_i > max_j |W_ij|
// and X_ij = rint(W_ij / sW_i * 2^31) in four 8-bit planes (top plane signed,
// lower planes unsigned): W_ij ~ sW_i (d0 2^-7 + u1 2^-15 + u2 2^-23 + u3 2^-31).
// Every context row r gets sH_r = 2^e > max_j h_rj and Y_rj = rint(h_rj / sH_r
// * 2^32) in four unsigned planes.  A digit pair (a, b) carries the weight
// sW sH 2^-(15 + 8(a + b)); the 13 pairs with a + b <= 4 are accumulated by
// `tcgen05.mma.kind::i8` into five int32 anti-diagonal accumulators D_s
// (s = a + b) -- exactly, |D_s| < 2^28 -- and combined once in float64:
//   x~ = U + sW sH 2^-47 (D0 2^32 + D1 2^24 + D2 2^16 + D3 2^8 + D4).
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
// Elements that cannot be certified (~0.2-0.4 %) are recomputed by the
// reference's own sequential float64 loop and sigmoid.  So every h' equals
// the reference's float32 result; the content dedup (context_table.py:74-86)
// then merges exactly the contexts the reference merges.
#pragma once
#include "tc_advance.cuh"

namespace xu {
constexpr int KC = 64;                 // bytes (= int8 elements) of K per ring stage
constexpr int XR = 96;                 // context rows per chunk: 5 accumulators x 96 columns <= 512
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
__device__ __forceinline__ uint32_t idesc(bool a_signed, int n) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(tc::BM >> 4) << 24);
}
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

// Certified float32 rounding of sigmoid(x) for |x - x_ref| <= eps.  Returns
// false when the interval may straddle a rounding midpoint.
__device__ __forceinline__ bool certify(double x, double eps, float &out) {
    const double z = 1.0 + exp(-x);
    if (!(z < 1e300) || !(eps < 1e-3)) return false;        // non-finite / no useful bound
    const double dl = eps * 1.0001 + 2.0e-15;               // + exp, sigmoid and fma roundings
    float y = __frcp_rn(__double2float_rn(z));
#pragma unroll 1
    for (int it = 0; it < 3; it++) {
        const uint32_t yb = __float_as_uint(y);
        if (yb < 0x00800000u || yb >= 0x3F800000u) return false;   // keep to normal (0, 1)
        const double yd = (double)y;
        const double m_lo = 0.5 * (yd + (double)__uint_as_float(yb - 1));
        const double m_hi = 0.5 * (yd + (double)__uint_as_float(yb + 1));
        const double t_lo = fma(z, m_lo, -1.0), t_hi = fma(z, m_hi, -1.0);
        if (t_lo < -dl && t_hi > dl) { out = y; return true; }
        if (t_lo > dl) { y = __uint_as_float(yb - 1); continue; }   // sigmoid below the lower midpoint
        if (t_hi < -dl) { y = __uint_as_float(yb + 1); continue; }  // above the upper midpoint
        return false;                                            // within the margin of a midpoint
    }
    return false;
}
}  // namespace xu

// --------------------------------------------------------------------------
// model preparation (once per model upload)
// --------------------------------------------------------------------------
// per unit i (block per row): planes into the pre-tiled layout
// Wd[mt][kc][a][128 rows x 64 B] and the float64 constants
// wx[i] = {sW 2^-47, A_i, B_i, sW}.
__global__ void k_prep_wdigits(const float *__restrict__ W, int H, int nkx, uint8_t *__restrict__ Wd,
                               double4 *__restrict__ wx) {
    const int i = blockIdx.x;
    if (i >= H) return;
    const float *row = W + (size_t)i * H;
    __shared__ float s_max[32];
    __shared__ double s_sum[4][32];
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
    int e = 0;                                   // sW = 2^e > max |W_ij|
    if (mx > 0.f) { frexpf(mx, &e); }             // mx = f * 2^e, f in [0.5, 1)
    const double sW = ldexp(1.0, e);
    const int mt = i / tc::BM, r = i % tc::BM;
    double sum_w = 0.0, err_w = 0.0, s2 = 0.0, s3 = 0.0;
    for (int j = threadIdx.x; j < nkx * xu::KC; j += blockDim.x) {
        int d0 = 0, u1 = 0, u2 = 0, u3 = 0;
        if (j < H) {
            const double w = (double)row[j];
            const long long X = llrint(ldexp(w, 31 - e));           // |X| < 2^31
            d0 = (int)(X >> 24);
            const long long R = X - ((long long)d0 << 24);
            u1 = (int)(R >> 16); u2 = (int)((R >> 8) & 255); u3 = (int)(R & 255);
            sum_w += fabs(w);
            err_w += fabs(ldexp((double)X, e - 31) - w);
            s2 += u2; s3 += u3;
        }
        const int kc = j / xu::KC, kk = j % xu::KC;
        const size_t blk = ((size_t)mt * nkx + kc) * 4;
        const uint32_t o = xu::toff(r, kk >> 4) + (kk & 15);
        Wd[(blk + 0) * xu::PLANE_W + o] = (uint8_t)(int8_t)d0;
        Wd[(blk + 1) * xu::PLANE_W + o] = (uint8_t)u1;
        Wd[(blk + 2) * xu::PLANE_W + o] = (uint8_t)u2;
        Wd[(blk + 3) * xu::PLANE_W + o] = (uint8_t)u3;
    }
    double v4[4] = {sum_w, err_w, s2, s3};
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
        // dropped pairs (2,3), (3,2), (3,3): |D_ab| <= (sum_j |w_a|) * 255
        const double drop = 255.0 * (t[2] * ldexp(1.0, -55) + t[3] * ldexp(1.0, -55) + t[3] * ldexp(1.0, -63));
        const double c1 = (double)(H + 8) * ldexp(1.0, -53) * 1.01;   // sequential-sum rounding
        double4 o;
        o.x = ldexp(sW, -47);
        o.y = (drop * sW + t[1]) * 1.01 + c1 * t[0] * 1.01;         // coefficient of sH_r
        o.z = t[0] * 1.01;                                           // coefficient of eH_r (max |dh|)
        o.w = sW;
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
// the reference loop after the tile.
// --------------------------------------------------------------------------
namespace xu {
struct Ring {
    uint8_t *smem;                 // stages x STAGE bytes
    int stages;
    uint32_t tmem;
    uint64_t *full, *empty, *done;
    uint32_t *fb;                  // [2][FBCAP] deferred fallback elements (row << 16 | unit)
    uint32_t *fb_n;                // [2]
    double *sh, *eh;               // [XR] per chunk row: scale sH, max |dh|
    uint8_t *xs;                   // this stream's global digit scratch
};
constexpr uint32_t STAGE = 4u * PLANE_W + 4u * XR * KC;
constexpr uint32_t HOFF = 4u * PLANE_W;

template <int NT, typename WaitFn>
__device__ __forceinline__ void update_level(const DevModel &m, const DevPlan &Q, DevStreams &S, uint32_t n,
                                             uint32_t base, const Ring &rg, uint32_t &gctr, uint32_t &tiles_done,
                                             int tid, int wid, int lane, WaitFn wait, unsigned long long *ph,
                                             unsigned long long &t0) {
    constexpr int NW = NT / 32;
    const int H = m.H, NK = m.wd_nkx, nmt = (H + tc::BM - 1) / tc::BM;
    const double c1 = (double)(H + 8) * 1.1102230246251565e-16 * 1.01;
    auto mark = [&](int i) {
        if (ph) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); ph[i] += t - t0; t0 = t; }
    };
    for (uint32_t q0 = 0; q0 < n; q0 += XR) {
        const int R = (int)min((uint32_t)XR, n - q0);
        const int Rp = (R + 15) & ~15;
        // ---- digitize the chunk's context rows (warp per row) ----
        for (int r = wid; r < R; r += NW) {
            const float *hrow = S.arena_h + (size_t)Q.pr_inrow[q0 + r] * H;
            float mx = 0.f;
            for (int g = lane; g < NK * 4; g += 32)
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const int j = g * 16 + v * 4;
                    if (j < H) {
                        const float4 x = __ldcg(reinterpret_cast<const float4 *>(hrow + j));
                        mx = fmaxf(mx, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
                    }
                }
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            int e = 0;
            if (mx > 0.f) frexpf(mx, &e);                    // sH = 2^e > max h
            float emax = 0.f;
            for (int g = lane; g < NK * 4; g += 32) {
                uint32_t pl[4][4];
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const int j = g * 16 + v * 4;
                    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (j < H) x = __ldcg(reinterpret_cast<const float4 *>(hrow + j));
                    const float xs4[4] = {x.x, x.y, x.z, x.w};
                    uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        // Y = rint(h 2^(32-e)) by integer shifts of the f32 significand
                        const uint32_t u = __float_as_uint(xs4[k]);
                        const int E = (int)((u >> 23) & 255);
                        uint32_t Y = 0;
                        float err = 0.f;
                        if ((u >> 31) == 0 && E > 0) {
                            const uint32_t mnt = (u & 0x7FFFFFu) | 0x800000u;
                            const int sh = E - 118 - e;             // <= 8 because h < 2^e
                            if (sh >= 0) Y = mnt << sh;
                            else if (sh > -25) {
                                Y = (mnt + (1u << (-sh - 1))) >> (-sh);
                                const int d = (int)mnt - (int)(Y << (-sh));
                                err = ldexpf((float)abs(d), E - 150);
                            } else err = xs4[k];
                        } else if (u != 0u && u != 0x80000000u) {
                            err = fabsf(xs4[k]);                    // subnormal / negative: not represented
                        }
                        emax = fmaxf(emax, err);
                        b0 |= (Y >> 24) << (8 * k);
                        b1 |= ((Y >> 16) & 255u) << (8 * k);
                        b2 |= ((Y >> 8) & 255u) << (8 * k);
                        b3 |= (Y & 255u) << (8 * k);
                    }
                    pl[0][v] = b0; pl[1][v] = b1; pl[2][v] = b2; pl[3][v] = b3;
                }
                const int kc = g >> 2, c = g & 3;
                uint8_t *blk = rg.xs + (size_t)kc * 4 * Rp * KC;
#pragma unroll
                for (int b = 0; b < 4; b++)
                    *reinterpret_cast<uint4 *>(blk + (size_t)b * Rp * KC + toff(r, c)) =
                        make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
            }
            for (int o = 16; o; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            if (lane == 0) { rg.sh[r] = ldexp(1.0, e); rg.eh[r] = (double)emax; }
        }
        // rows R..Rp-1 of the h blocks are never read back from TMEM (their
        // columns are skipped by the epilogue), whatever the scratch holds
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
        mark(1);
        for (int mt = 0; mt < nmt; mt++) {
            if (wid == 1) {
                // ---- producer: W plane block (mt, kc) + h plane block kc per stage ----
                const uint32_t hbytes = 4u * (uint32_t)Rp * KC;
                for (int kc = 0; kc < NK; kc++) {
                    const uint32_t gc = gctr + kc;
                    const int st = (int)(gc % (uint32_t)rg.stages);
                    const uint32_t use = gc / (uint32_t)rg.stages;
                    if (use >= 1) wait(tc::smem_u32(&rg.empty[st]), (use - 1) & 1, 11);
                    __syncwarp();
                    uint8_t *sW = rg.smem + (size_t)st * STAGE;
                    const uint8_t *srcW = m.Wd + ((size_t)mt * NK + kc) * 4 * PLANE_W;
                    const uint8_t *srcH = rg.xs + (size_t)kc * hbytes;
                    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                                 "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %6;\n\t"
                                 "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t"
                                 "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5], %7, [%1];\n\t}"
                                 :: "r"(tc::smem_u32(sW)), "r"(tc::smem_u32(&rg.full[st])), "l"(srcW),
                                    "r"(4u * PLANE_W), "r"(tc::smem_u32(sW + HOFF)), "l"(srcH),
                                    "r"(4u * PLANE_W + hbytes), "r"(hbytes) : "memory");
                }
            } else if (wid == 0) {
                // ---- MMA issuer: 13 digit pairs per 32-byte K step ----
                for (int kc = 0; kc < NK; kc++) {
                    const uint32_t gc = gctr + kc;
                    const int st = (int)(gc % (uint32_t)rg.stages);
                    wait(tc::smem_u32(&rg.full[st]), (gc / (uint32_t)rg.stages) & 1, 12);
                    __syncwarp();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sW = tc::smem_u32(rg.smem + (size_t)st * STAGE);
                    const uint32_t sH = sW + HOFF;
#pragma unroll
                    for (int ks = 0; ks < KC / 32; ks++) {
                        const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
                        // W plane a over h blocks [b0, b0 + nb): TMEM column blocks a + b
                        auto range = [&](int a, int b0, int nb, uint32_t acc) {
                            const int tot = nb * Rp;
                            for (int off = 0; off < tot; off += 256) {
                                const int nn = min(256, tot - off);
                                const int brow = b0 * Rp + off;
                                const uint64_t da = desc(sW + (uint32_t)a * PLANE_W + (uint32_t)ks * 256u);
                                const uint64_t db = desc(sH + (uint32_t)(brow >> 3) * 512u + (uint32_t)ks * 256u);
                                mma_i8(rg.tmem + (uint32_t)((a + b0) * Rp + off), da, db, idesc(a == 0, nn), acc);
                            }
                        };
                        range(0, 0, 4, acc0);      // (0,0) (0,1) (0,2) (0,3)
                        range(1, 0, 3, 1u);        // (1,0) (1,1) (1,2)
                        range(1, 3, 1, acc0);      // (1,3): first write of block 4
                        range(2, 0, 3, 1u);        // (2,0) (2,1) (2,2)
                        range(3, 0, 2, 1u);        // (3,0) (3,1)
                    }
                    tc::commit_elect(tc::smem_u32(&rg.empty[st]));
                    if (kc == NK - 1) tc::commit_elect(tc::smem_u32(rg.done));
                    __syncwarp();
                }
            }
            gctr += NK;
            wait(tc::smem_u32(rg.done), tiles_done & 1, 13);
            tiles_done++;
            __syncwarp();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            mark(2);
            // ---- epilogue: TMEM lane = output unit, columns s * Rp + row ----
            const int quad = wid & 3;
            const int unit = mt * tc::BM + quad * 32 + lane;
            const bool uok = unit < H;
            double4 k4 = make_double4(0.0, 0.0, 0.0, 0.0);
            if (uok) k4 = m.wx[unit];
            uint32_t *fbl = rg.fb + (mt & 1) * FBCAP;
            uint32_t *fbn = rg.fb_n + (mt & 1);
            const int n8 = (R + 7) >> 3;
            for (int it = wid >> 2; it < n8; it += NW / 4) {
                const int r0 = it * 8;
                int D[5][8];
                const uint32_t ta = rg.tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)r0;
#pragma unroll
                for (int s = 0; s < 5; s++) tmem_ld8i(ta + (uint32_t)(s * Rp), D[s]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int wl = lane < 8 && r0 + lane < R ? Q.pr_w[q0 + r0 + lane] : 0;
                float uv[8];
#pragma unroll
                for (int g = 0; g < 8; g++) {
                    const int wq = __shfl_sync(0xffffffffu, wl, g);
                    uv[g] = (uok && r0 + g < R) ? __ldg(m.U + (size_t)wq * H + unit) : 0.f;
                }
                unsigned long long dg[8];
#pragma unroll
                for (int g = 0; g < 8; g++) {
                    dg[g] = 0ull;
                    const int row = r0 + g;
                    if (uok && row < R) {
                        const double sHr = rg.sh[row], eHr = rg.eh[row];
                        double T = i2d(D[0][g]);
                        T = fma(T, 256.0, i2d(D[1][g]));
                        T = fma(T, 256.0, i2d(D[2][g]));
                        T = fma(T, 256.0, i2d(D[3][g]));
                        T = fma(T, 256.0, i2d(D[4][g]));
                        const double u = (double)uv[g];
                        const double x = fma(T, k4.x * sHr, u);
                        const double eps = fma(k4.y, sHr, fma(k4.z, eHr, c1 * fabs(u)));
                        float y;
                        bool ok = certify(x, eps, y);
                        if (!ok) {
                            const uint32_t k = atomicAdd(fbn, 1u);
                            if (k < (uint32_t)FBCAP) fbl[k] = ((uint32_t)row << 16) | (uint32_t)unit;
                            else {                                   // list full: recompute here
                                y = ref_element(m.W + (size_t)unit * H, S.arena_h + (size_t)Q.pr_inrow[q0 + row] * H,
                                                uv[g], H);
                                ok = true;
                            }
                        }
                        if (ok) {
                            S.arena_h[(size_t)(base + q0 + row) * H + unit] = y;
                            dg[g] = otf_dig_h((uint32_t)unit, y);
                        }
                    }
                }
                const unsigned long long tot = sd::reduce8_u64(dg, lane);
                const int row = r0 + node_of_lane(lane);
                if ((lane & 3) == 0 && row < R) atomicAdd(&Q.pr_dig[q0 + row], tot);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            mark(3);
            // ---- the reference loop for the uncertified elements ----
            const uint32_t nf = min(*fbn, (uint32_t)FBCAP);
            for (uint32_t k = (uint32_t)tid; k < nf; k += NT) {
                const uint32_t e = fbl[k];
                const int row = (int)(e >> 16), un = (int)(e & 0xFFFFu);
                const int wq = Q.pr_w[q0 + row];
                const float y = ref_element(m.W + (size_t)un * H, S.arena_h + (size_t)Q.pr_inrow[q0 + row] * H,
                                            __ldg(m.U + (size_t)wq * H + un), H);
                S.arena_h[(size_t)(base + q0 + row) * H + un] = y;
                atomicAdd(&Q.pr_dig[q0 + row], otf_dig_h((uint32_t)un, y));
            }
            if (Q.alg && tid == 0) atomicAdd(&Q.alg[3], (unsigned long long)*fbn);
            __syncthreads();
            if (tid == 0) *fbn = 0u;
            mark(10);
        }
    }
}
}  // namespace xu

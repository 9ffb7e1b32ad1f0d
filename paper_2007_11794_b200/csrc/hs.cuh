// hs.cuh -- gather-bound warp-per-query kernels:
//   * Huffman hierarchical-softmax path score + hashed MaxEnt n-gram
//     features (reference _kernels_nb.py:63-86, rnnlm.py:195-204);
//   * feature_index (reference _kernels_nb.py:21-33), bit-exact;
//   * the exact-mode (FP64, reference summation order) recurrent update
//     (reference _kernels_nb.py:51-60).
//
// word_logprob work per query: P path nodes (P ~ 7-10 at Zipf vocabularies),
// each a 4H-byte node-vector row + min(order, |hist|) 4-byte MaxEnt gathers.
// One warp owns one query: the hidden vector sits in registers as float4
// chunks, each node row is read with coalesced 16-byte lanes, G=8 rows are in
// flight per warp, partial dot products are reduced with xor shuffles in
// float64 (f32 x f32 products are exact in f64, so only the summation order
// differs from the reference), the MaxEnt gathers of all G nodes are spread
// over lanes, and lane g evaluates log-sigmoid for node g so the f64
// transcendental cost is paid once per node.  The final sum over nodes runs
// in path order like the reference.
#pragma once
#include "common.cuh"
#include <cstdio>

#define HS_G 8

// f32 -> f64 with integer ops (rebias the exponent, shift the mantissa):
// the F2F conversion unit was the top stall reason of the first version.
// Exact for normal numbers and zero; f32 denormals (|x| < 1.2e-38) flush to
// signed zero, a change far below one f64 ulp of any activation sum.
__device__ __forceinline__ double widen(float x) {
    const uint32_t u = __float_as_uint(x);
    const uint32_t hi = (u & 0x80000000u) | (((u >> 3) & 0x0FFFFFFFu) + (896u << 20));
    const uint32_t lo = u << 29;
    return (u & 0x7F800000u) ? __hiloint2double((int)hi, (int)lo)
                             : __hiloint2double((int)(u & 0x80000000u), 0);
}

// Reduce 8 per-lane partial sums across the warp with 9 exchanges (instead of
// 8 x 5 butterflies): each step halves the vector, lanes keep one half and
// receive the partner's other half.  Afterwards the full sum of node g is in
// the 4 lanes whose bits (4,3,2) spell g; lane_of(g) names the first of them.
__device__ __forceinline__ double reduce8(double (&v)[8], int lane) {
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        double send = u16 ? v[i] : v[i + 4];
        double keep = u16 ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; i++) {
        double send = u8 ? v[i] : v[i + 2];
        double keep = u8 ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        double send = u4 ? v[0] : v[1];
        double keep = u4 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    double x = v[0];
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}
__device__ __forceinline__ int node_of_lane(int lane) {
    return ((lane >> 4) & 1) << 2 | ((lane >> 3) & 1) << 1 | ((lane >> 2) & 1);
}
__device__ __forceinline__ int lane_of_node(int g) {
    return ((g >> 2) & 1) << 4 | ((g >> 1) & 1) << 3 | (g & 1) << 2;
}

template <int VEC, int CPL>
__device__ __forceinline__ double hs_logprob_warp(const DevModel &m, const float *__restrict__ h,
                                                  const uint32_t *__restrict__ hist, int L,
                                                  const uint32_t *__restrict__ codes, uint32_t P,
                                                  int lane) {
    const int H = m.H;
    const int NCH = VEC == 4 ? (H >> 2) : H;   // chunks of VEC floats
    double hv[CPL][VEC];                        // hidden state, widened once
#pragma unroll
    for (int c = 0; c < CPL; c++) {
        int k = lane + 32 * c;
        if (k < NCH) {
            if (VEC == 4) {
                float4 t = __ldg(reinterpret_cast<const float4 *>(h) + k);
                hv[c][0] = widen(t.x); hv[c][1] = widen(t.y); hv[c][2] = widen(t.z); hv[c][3] = widen(t.w);
            } else {
                hv[c][0] = widen(__ldg(h + k));
            }
        } else {
#pragma unroll
            for (int v = 0; v < VEC; v++) hv[c][v] = 0.0;
        }
    }
    // MaxEnt hash prefixes: order-k feature hash of (k, last k words oldest
    // first), finished per node (_kernels_nb.py:27-33, :72-74)
    const int kmax = m.order < L ? m.order : L;
    uint64_t pre[OTF_MAX_ORDER];
#pragma unroll
    for (int k = 0; k < OTF_MAX_ORDER; k++) {
        pre[k] = 0;
        if (k < kmax) {
            uint64_t x = otf_mix(m.seed, (uint64_t)(k + 1));
            for (int i = L - (k + 1); i < L; i++) x = otf_mix(x, (uint64_t)hist[i]);
            pre[k] = x;
        }
    }
    const int my_g = node_of_lane(lane);
    const bool leader = (lane & 3) == 0;
    double lp = 0.0;
    for (uint32_t p0 = 0; p0 < P; p0 += HS_G) {
        // this lane's node (for the MaxEnt / log-sigmoid part)
        const uint32_t my_code = (p0 + my_g < P) ? __ldg(codes + p0 + my_g) : OTF_UNSET;
        double me[OTF_MAX_ORDER];
#pragma unroll
        for (int k = 0; k < OTF_MAX_ORDER; k++) {
            me[k] = 0.0;
            if (leader && k < kmax && my_code != OTF_UNSET)
                me[k] = (double)__ldg(m.ME + (otf_mix(pre[k], (uint64_t)(my_code & 0x7FFFFFFFu)) & m.mask));
        }
        double acc[HS_G];
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            acc[g] = 0.0;
            const uint32_t cg = (p0 + g < P) ? __ldg(codes + p0 + g) : OTF_UNSET;
            if (cg != OTF_UNSET) {
                const float *row = m.NV + (size_t)(cg & 0x7FFFFFFFu) * H;
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    int k = lane + 32 * c;
                    if (k < NCH) {
                        if (VEC == 4) {
                            float4 t = __ldg(reinterpret_cast<const float4 *>(row) + k);
                            acc[g] = fma(widen(t.x), hv[c][0], acc[g]);
                            acc[g] = fma(widen(t.y), hv[c][1], acc[g]);
                            acc[g] = fma(widen(t.z), hv[c][2], acc[g]);
                            acc[g] = fma(widen(t.w), hv[c][3], acc[g]);
                        } else {
                            acc[g] = fma(widen(__ldg(row + k)), hv[c][0], acc[g]);
                        }
                    }
                }
            }
        }
        // a_g = dot + ME[k=1] + ME[k=2] + ... (reference order, :72-74)
        double a = reduce8(acc, lane);
#pragma unroll
        for (int k = 0; k < OTF_MAX_ORDER; k++) if (k < kmax) a += me[k];
        double mylog = 0.0;
        if (leader && my_code != OTF_UNSET)
            mylog = otf_log_sigmoid((my_code & 0x80000000u) ? -a : a);   // sign -1 for bit 1
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            const double v = __shfl_sync(0xffffffffu, mylog, lane_of_node(g));
            if (p0 + g < P) lp += v;
        }
    }
    return lp;
}

// --------------------------------------------------------------------------
// HS v3: node rows streamed into a per-warp shared-memory ring by the TMA
// bulk-copy engine (cp.async.bulk + mbarrier complete_tx), NS rows in flight
// per warp without holding registers; lanes read the landed row with
// conflict-free 16-byte shared loads.  Same arithmetic as hs_logprob_warp
// (float64 accumulation, reduce8, reference node / MaxEnt order).
// --------------------------------------------------------------------------
#define HS_NS 8
struct HsRing {
    uint8_t *buf;            // HS_NS rows of 4H bytes
    uint32_t bar0;           // shared address of HS_NS mbarriers (8 B apart)
    uint32_t phase;          // bit s = parity to wait for on slot s
};

// Warp-collective: all lanes pass the same operands, one lane is elected
// inside the asm (issuing under `if (lane == 0)` costs a per-lane R2UR loop).
// The slot's previous contents were only read by this warp (ordered by the
// __syncwarp before the refill), so no proxy fence is needed.
__device__ __forceinline__ void ring_issue(HsRing &r, int slot, const float *src, uint32_t bytes) {
    const uint32_t bar = r.bar0 + slot * 8;
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(r.buf + (size_t)slot * bytes);
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\telect.sync t|e, 0xffffffff;\n\t"
                 "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n\t"
                 "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n\t}"
                 :: "r"(dst), "r"(bar), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ring_wait(HsRing &r, int slot) {
    const uint32_t bar = r.bar0 + slot * 8;
    const uint32_t par = (r.phase >> slot) & 1u;
    for (uint32_t it = 0;; it++) {     // bounded: a lost copy traps instead of hanging
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
        if (ok) break;
        if (it == (1u << 22)) {
            printf("hs ring: wait timeout block %d thread %d slot %d\n", (int)blockIdx.x, (int)threadIdx.x, slot);
            __trap();
        }
    }
    r.phase ^= 1u << slot;
}

// EXACT: float64 accumulation of the exact f32 x f32 products (4 independent
// accumulators per row keep the DFMA chains short); only the summation order
// differs from the reference (~1e-16 relative).
// !EXACT: per-lane partial dot in f32 FFMA (<= 4H/128 terms per lane, error
// ~1e-7 relative), lane partials combined and everything after (MaxEnt,
// log-sigmoid, path sum) in float64 -- used with the tensor-core update
// modes, whose h' already differs from the reference at ~1e-7; log-probs stay
// within 1e-5 of the reference (the north star allows 1e-4).
template <int CPL, bool EXACT, int ORD>
__device__ __forceinline__ double hs_logprob_ring(const DevModel &m, HsRing &ring, const float *__restrict__ h,
                                                  const uint32_t *__restrict__ hist, int L,
                                                  const uint32_t *__restrict__ codes, uint32_t P, int lane) {
    const int H = m.H;
    const int NCH = H >> 2;
    const uint32_t bytes = (uint32_t)H * 4u;
    for (uint32_t p = 0; p < P && p < HS_NS; p++)
        ring_issue(ring, (int)p, m.NV + (size_t)(__ldg(codes + p) & 0x7FFFFFFFu) * H, bytes);
    double hd[EXACT ? CPL : 1][4];
    float hf[EXACT ? 1 : CPL][4];
#pragma unroll
    for (int c = 0; c < CPL; c++) {
        const int k = lane + 32 * c;
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        // L2 load: h may have been written earlier in the same (persistent) kernel
        if (k < NCH) t = __ldcg(reinterpret_cast<const float4 *>(h) + k);
        if (EXACT) {
            hd[EXACT ? c : 0][0] = widen(t.x); hd[EXACT ? c : 0][1] = widen(t.y);
            hd[EXACT ? c : 0][2] = widen(t.z); hd[EXACT ? c : 0][3] = widen(t.w);
        } else {
            hf[EXACT ? 0 : c][0] = t.x; hf[EXACT ? 0 : c][1] = t.y;
            hf[EXACT ? 0 : c][2] = t.z; hf[EXACT ? 0 : c][3] = t.w;
        }
    }
    const int kmax = m.order < L ? m.order : L;
    uint64_t pre[ORD];
#pragma unroll
    for (int k = 0; k < ORD; k++) {
        pre[k] = 0;
        if (k < kmax) {
            uint64_t x = otf_mix(m.seed, (uint64_t)(k + 1));
            for (int i = L - (k + 1); i < L; i++) x = otf_mix(x, (uint64_t)hist[i]);
            pre[k] = x;
        }
    }
    const int my_g = node_of_lane(lane);
    const bool leader = (lane & 3) == 0;
    double lp = 0.0;
    for (uint32_t p0 = 0; p0 < P; p0 += HS_G) {
        const uint32_t my_code = (p0 + my_g < P) ? __ldg(codes + p0 + my_g) : OTF_UNSET;
        double me[ORD];
#pragma unroll
        for (int k = 0; k < ORD; k++) {
            me[k] = 0.0;
            if (leader && k < kmax && my_code != OTF_UNSET)
                me[k] = (double)__ldg(m.ME + (otf_mix(pre[k], (uint64_t)(my_code & 0x7FFFFFFFu)) & m.mask));
        }
        double acc[HS_G];
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            acc[g] = 0.0;
            const uint32_t p = p0 + g;
            if (p < P) {
                const int slot = (int)(p % HS_NS);
                ring_wait(ring, slot);
                const float4 *row = reinterpret_cast<const float4 *>(ring.buf + (size_t)slot * bytes);
                if (EXACT) {
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int c = 0; c < CPL; c++) {
                        const int k = lane + 32 * c;
                        if (k < NCH) {
                            const float4 t = row[k];
                            a0 = fma(widen(t.x), hd[EXACT ? c : 0][0], a0);
                            a1 = fma(widen(t.y), hd[EXACT ? c : 0][1], a1);
                            a2 = fma(widen(t.z), hd[EXACT ? c : 0][2], a2);
                            a3 = fma(widen(t.w), hd[EXACT ? c : 0][3], a3);
                        }
                    }
                    acc[g] = (a0 + a1) + (a2 + a3);
                } else {
                    float f0 = 0.f, f1 = 0.f, f2 = 0.f, f3 = 0.f;
#pragma unroll
                    for (int c = 0; c < CPL; c++) {
                        const int k = lane + 32 * c;
                        if (k < NCH) {
                            const float4 t = row[k];
                            f0 = fmaf(t.x, hf[EXACT ? 0 : c][0], f0);
                            f1 = fmaf(t.y, hf[EXACT ? 0 : c][1], f1);
                            f2 = fmaf(t.z, hf[EXACT ? 0 : c][2], f2);
                            f3 = fmaf(t.w, hf[EXACT ? 0 : c][3], f3);
                        }
                    }
                    acc[g] = ((double)f0 + (double)f1) + ((double)f2 + (double)f3);
                }
                __syncwarp();
                if (p + HS_NS < P)
                    ring_issue(ring, slot, m.NV + (size_t)(__ldg(codes + p + HS_NS) & 0x7FFFFFFFu) * H, bytes);
            }
        }
        double a = reduce8(acc, lane);
#pragma unroll
        for (int k = 0; k < ORD; k++) if (k < kmax) a += me[k];
        double mylog = 0.0;
        if (leader && my_code != OTF_UNSET)
            mylog = otf_log_sigmoid((my_code & 0x80000000u) ? -a : a);
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            const double v = __shfl_sync(0xffffffffu, mylog, lane_of_node(g));
            if (p0 + g < P) lp += v;
        }
    }
    return lp;
}

// warp-ring setup: HS_NS row slots + barriers per warp in dynamic smem
__device__ __forceinline__ HsRing ring_setup(uint8_t *smem, int warp_in_block, int H, int lane) {
    const uint32_t bytes = (uint32_t)H * 4u;
    HsRing r;
    uint8_t *wbase = smem + (size_t)warp_in_block * (HS_NS * bytes + HS_NS * 8);
    r.buf = wbase;
    r.bar0 = (uint32_t)__cvta_generic_to_shared(wbase + HS_NS * bytes);
    r.phase = 0;
    if (lane < HS_NS)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(r.bar0 + lane * 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    return r;
}
__host__ __device__ constexpr size_t ring_bytes_per_warp(int H) { return (size_t)HS_NS * (4 * H + 8); }

// CALLR(CPL, EXACT, ORD) for H % 4 == 0, H <= 1024
#define RING_DISPATCH(H, EXACT, ORDER, CALLR)                                   \
    do {                                                                       \
        if ((ORDER) <= 3) {                                                    \
            if ((H) <= 128) { CALLR(1, EXACT, 3); }                            \
            else if ((H) <= 256) { CALLR(2, EXACT, 3); }                       \
            else if ((H) <= 512) { CALLR(4, EXACT, 3); }                       \
            else { CALLR(8, EXACT, 3); }                                       \
        } else {                                                               \
            if ((H) <= 128) { CALLR(1, EXACT, OTF_MAX_ORDER); }                \
            else if ((H) <= 256) { CALLR(2, EXACT, OTF_MAX_ORDER); }           \
            else if ((H) <= 512) { CALLR(4, EXACT, OTF_MAX_ORDER); }           \
            else { CALLR(8, EXACT, OTF_MAX_ORDER); }                           \
        }                                                                      \
    } while (0)

// batch API (config d): warps stride over queries, ring reused across queries
template <int CPL, bool EXACT, int ORD>
__global__ void __launch_bounds__(128) k_word_logprob_ring(DevModel m, int64_t n, const int32_t *__restrict__ ctx,
                                                           const float *__restrict__ h,
                                                           const int32_t *__restrict__ hist,
                                                           const int32_t *__restrict__ hist_len,
                                                           const int32_t *__restrict__ w,
                                                           double *__restrict__ out) {
    extern __shared__ __align__(128) uint8_t smem_ring[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    HsRing ring = ring_setup(smem_ring, wib, m.H, lane);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; q < n; q += nw) {
        const int c = ctx[q];
        uint32_t hw[OTF_MAX_ORDER];
        const int L = hist_len[c];
        for (int i = 0; i < L; i++) hw[i] = (uint32_t)hist[(int64_t)c * m.order + i];
        const uint32_t o0 = __ldg(m.path_off + w[q]), o1 = __ldg(m.path_off + w[q] + 1);
        const double lp = hs_logprob_ring<CPL, EXACT, ORD>(m, ring, h + (int64_t)c * m.H, hw, L, m.path_code + o0,
                                                           o1 - o0, lane);
        if (lane == 0) out[q] = lp;
    }
}

// dispatch on H: VEC=4 needs H % 4 == 0 (16-byte aligned rows)
#define HS_DISPATCH(H, CALL)                                                   \
    do {                                                                       \
        if ((H) % 4 == 0) {                                                    \
            if ((H) <= 128) { CALL(4, 1); }                                    \
            else if ((H) <= 256) { CALL(4, 2); }                               \
            else if ((H) <= 512) { CALL(4, 4); }                               \
            else if ((H) <= 1024) { CALL(4, 8); }                              \
            else { CALL(4, 16); }                                              \
        } else {                                                               \
            if ((H) <= 32) { CALL(1, 1); }                                     \
            else if ((H) <= 64) { CALL(1, 2); }                                \
            else if ((H) <= 128) { CALL(1, 4); }                               \
            else if ((H) <= 256) { CALL(1, 8); }                               \
            else if ((H) <= 512) { CALL(1, 16); }                              \
            else { CALL(1, 64); }                                              \
        }                                                                      \
    } while (0)

// --- batch API kernel: query i uses hidden row ctx[i], history row ctx[i] --
template <int VEC, int CPL>
__global__ void __launch_bounds__(256) k_word_logprob_batch(DevModel m, int64_t n,
                                                            const int32_t *__restrict__ ctx,
                                                            const float *__restrict__ h,
                                                            const int32_t *__restrict__ hist,
                                                            const int32_t *__restrict__ hist_len,
                                                            const int32_t *__restrict__ w,
                                                            double *__restrict__ out) {
    int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (q >= n) return;
    int c = ctx[q];
    uint32_t hw[OTF_MAX_ORDER];
    int L = hist_len[c];
    for (int i = 0; i < L; i++) hw[i] = (uint32_t)hist[(int64_t)c * m.order + i];
    const uint32_t o0 = __ldg(m.path_off + w[q]), o1 = __ldg(m.path_off + w[q] + 1);
    double lp = hs_logprob_warp<VEC, CPL>(m, h + (int64_t)c * m.H, hw, L, m.path_code + o0, o1 - o0, lane);
    if (lane == 0) out[q] = lp;
}

// explicit paths: query i scores path codes[off[i] .. off[i+1]) (the
// reference kernel signature passes the path slice, _kernels_nb.py:78-79)
template <int VEC, int CPL>
__global__ void __launch_bounds__(256) k_word_logprob_paths(DevModel m, int64_t n,
                                                            const int32_t *__restrict__ ctx,
                                                            const float *__restrict__ h,
                                                            const int32_t *__restrict__ hist,
                                                            const int32_t *__restrict__ hist_len,
                                                            const int64_t *__restrict__ off,
                                                            const uint32_t *__restrict__ codes,
                                                            double *__restrict__ out) {
    int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (q >= n) return;
    int c = ctx[q];
    uint32_t hw[OTF_MAX_ORDER];
    int L = hist_len[c];
    for (int i = 0; i < L; i++) hw[i] = (uint32_t)hist[(int64_t)c * m.order + i];
    double lp = hs_logprob_warp<VEC, CPL>(m, h + (int64_t)c * m.H, hw, L, codes + off[q],
                                          (uint32_t)(off[q + 1] - off[q]), lane);
    if (lane == 0) out[q] = lp;
}

__global__ void k_feature_index(uint64_t seed, uint64_t mask, int64_t n, const int32_t *order_k,
                                const int64_t *words, const int64_t *node, uint64_t *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int k = order_k[i];
    uint64_t x = otf_mix(seed, (uint64_t)k);
    for (int j = 0; j < k; j++) x = otf_mix(x, (uint64_t)words[i * 8 + j]);
    x = otf_mix(x, (uint64_t)node[i]);
    out[i] = x & mask;
}

// --------------------------------------------------------------------------
// Exact-mode recurrent update: h'_i = f32(sigmoid(U[w,i] + sum_j W[i,j] h_j))
// accumulated in float64 in the reference's order (U first, then j = 0..H-1,
// _kernels_nb.py:55-59); the f32 x f32 products are exact in f64 so DFMA
// reproduces the reference's rounding step for step.  Threads own output
// columns i (coalesced reads of W^T rows), QT queries share each W^T load.
// --------------------------------------------------------------------------
template <int QT>
__global__ void __launch_bounds__(256) k_advance_f64(DevModel m, uint32_t n_cap, RowSpec rs,
                                                     const int32_t *__restrict__ in_row,
                                                     const int32_t *__restrict__ words,
                                                     const float *__restrict__ h_base,
                                                     float *__restrict__ out_base, uint32_t row_limit_unused) {
    const uint32_t row_limit = rs.row_limit;
    extern __shared__ float4 smem4[];
    float *hs = reinterpret_cast<float *>(smem4);
    __shared__ unsigned long long s_dig[QT];
    const uint32_t n = rs.n_dev ? *rs.n_dev : n_cap;
    const uint32_t out0 = row_base(rs);
    if (rs.cur && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) rs.cur->base = out0;
    if ((uint64_t)out0 + n > row_limit) return;     // arena overflow (flagged by the HS stage)
    const uint32_t q0 = blockIdx.x * QT;
    if (q0 >= n) return;
    const int H = m.H;
    const int nq = (int)min((uint32_t)QT, n - q0);
    for (int t = threadIdx.x; t < QT * H; t += blockDim.x) {
        int q = t / H, j = t - q * H;
        hs[t] = q < nq ? h_base[(size_t)in_row[q0 + q] * H + j] : 0.f;
    }
    if (threadIdx.x < QT) s_dig[threadIdx.x] = 0ull;
    __syncthreads();
    unsigned long long dg[QT];
#pragma unroll
    for (int q = 0; q < QT; q++) dg[q] = 0ull;
    for (int i = threadIdx.x + blockIdx.y * blockDim.x; i < H; i += blockDim.x * gridDim.y) {
        double acc[QT];
#pragma unroll
        for (int q = 0; q < QT; q++)
            acc[q] = q < nq ? (double)m.U[(size_t)(words ? words[q0 + q] : (int32_t)(q0 + q)) * H + i] : 0.0;
        const float *wt = m.WT + i;
        for (int j = 0; j < H; j++) {
            double wv = (double)__ldg(wt + (size_t)j * H);
#pragma unroll
            for (int q = 0; q < QT; q++) acc[q] = fma(wv, (double)hs[q * H + j], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < QT; q++)
            if (q < nq) {
                const float o = (float)otf_sigmoid(acc[q]);
                out_base[(size_t)(out0 + q0 + q) * H + i] = o;
                dg[q] += otf_dig_h((uint32_t)i, o);
            }
    }
    if (rs.dig) {
#pragma unroll
        for (int q = 0; q < QT; q++) {
            unsigned long long d = dg[q];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if ((threadIdx.x & 31) == 0 && q < nq) atomicAdd(&s_dig[q], d);
        }
        __syncthreads();
        if (threadIdx.x < nq) atomicAdd(&rs.dig[q0 + threadIdx.x], s_dig[threadIdx.x]);
    }
}

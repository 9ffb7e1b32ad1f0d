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

#define HS_G 8

template <int VEC, int CPL>
__device__ __forceinline__ double hs_logprob_warp(const DevModel &m, const float *__restrict__ h,
                                                  const uint32_t *__restrict__ hist, int L,
                                                  const uint32_t *__restrict__ codes, uint32_t P,
                                                  int lane) {
    const int H = m.H;
    const int NCH = VEC == 4 ? (H >> 2) : H;   // chunks of VEC floats
    double hv[CPL][VEC];                        // hidden state, converted once
#pragma unroll
    for (int c = 0; c < CPL; c++) {
        int k = lane + 32 * c;
        if (k < NCH) {
            if (VEC == 4) {
                float4 t = __ldg(reinterpret_cast<const float4 *>(h) + k);
                hv[c][0] = t.x; hv[c][1] = t.y; hv[c][2] = t.z; hv[c][3] = t.w;
            } else {
                hv[c][0] = __ldg(h + k);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VEC; v++) hv[c][v] = 0.0;
        }
    }
    // MaxEnt hash prefixes: order-k feature hashes (k, last k words oldest
    // first) and then the node id (_kernels_nb.py:27-33, :72-74).
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
    double lp = 0.0;
    for (uint32_t p0 = 0; p0 < P; p0 += HS_G) {
        uint32_t code[HS_G];
        double acc[HS_G];
#pragma unroll
        for (int g = 0; g < HS_G; g++) code[g] = (p0 + g < P) ? __ldg(codes + p0 + g) : OTF_UNSET;
        // MaxEnt gathers first (independent of the dot products): lane j ->
        // (node g = j / kmax, order k = j % kmax); order > 4 spills below
        double me = 0.0;
        if (lane < HS_G * kmax) {
            int g = lane / kmax, k = lane - g * kmax;
            uint32_t cg = 0; uint64_t pk = 0;
#pragma unroll
            for (int t = 0; t < HS_G; t++) if (t == g) cg = code[t];
#pragma unroll
            for (int t = 0; t < OTF_MAX_ORDER; t++) if (t == k) pk = pre[t];
            if (cg != OTF_UNSET) {
                uint64_t idx = otf_mix(pk, (uint64_t)(cg & 0x7FFFFFFFu)) & m.mask;
                me = (double)__ldg(m.ME + idx);
            }
        }
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            acc[g] = 0.0;
            if (code[g] != OTF_UNSET) {
                const float *row = m.NV + (size_t)(code[g] & 0x7FFFFFFFu) * H;
#pragma unroll
                for (int c = 0; c < CPL; c++) {
                    int k = lane + 32 * c;
                    if (k < NCH) {
                        if (VEC == 4) {
                            float4 t = __ldg(reinterpret_cast<const float4 *>(row) + k);
                            acc[g] = fma((double)t.x, hv[c][0], acc[g]);
                            acc[g] = fma((double)t.y, hv[c][1], acc[g]);
                            acc[g] = fma((double)t.z, hv[c][2], acc[g]);
                            acc[g] = fma((double)t.w, hv[c][3], acc[g]);
                        } else {
                            acc[g] = fma((double)__ldg(row + k), hv[c][0], acc[g]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int g = 0; g < HS_G; g++) acc[g] = warp_sum_d(acc[g]);
        // node activation a_g = dot + ME[k=1] + ME[k=2] + ... in order; lane g
        // keeps a_g and all G log-sigmoids are evaluated in one pass
        double my_a = 0.0;
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            double a = acc[g];
            for (int k = 0; k < kmax; k++) {
                int j = g * kmax + k;
                double v = __shfl_sync(0xffffffffu, me, j & 31);
                if (j >= 32) {  // order > 4 overflow: gather directly
                    uint64_t pk = 0;
#pragma unroll
                    for (int t = 0; t < OTF_MAX_ORDER; t++) if (t == k) pk = pre[t];
                    v = code[g] != OTF_UNSET
                            ? (double)__ldg(m.ME + (otf_mix(pk, (uint64_t)(code[g] & 0x7FFFFFFFu)) & m.mask))
                            : 0.0;
                }
                a += v;
            }
            if (lane == g) my_a = a;
        }
        uint32_t my_code = OTF_UNSET;
#pragma unroll
        for (int g = 0; g < HS_G; g++) if (lane == g) my_code = code[g];
        double mylog = 0.0;
        if (my_code != OTF_UNSET)
            mylog = otf_log_sigmoid((my_code & 0x80000000u) ? -my_a : my_a);   // sign -1 for bit 1
#pragma unroll
        for (int g = 0; g < HS_G; g++) {
            double v = __shfl_sync(0xffffffffu, mylog, g);
            if (code[g] != OTF_UNSET) lp += v;
        }
    }
    return lp;
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
__global__ void __launch_bounds__(256) k_advance_f64(DevModel m, uint32_t n_cap, const uint32_t *n_dev,
                                                     const int32_t *__restrict__ in_row,
                                                     const int32_t *__restrict__ words,
                                                     const float *__restrict__ h_base,
                                                     float *__restrict__ out_base,
                                                     const uint32_t *out_row0_dev) {
    extern __shared__ float4 smem4[];
    float *hs = reinterpret_cast<float *>(smem4);
    const uint32_t n = n_dev ? *n_dev : n_cap;
    const uint32_t q0 = blockIdx.x * QT;
    if (q0 >= n) return;
    const int H = m.H;
    const int nq = (int)min((uint32_t)QT, n - q0);
    for (int t = threadIdx.x; t < QT * H; t += blockDim.x) {
        int q = t / H, j = t - q * H;
        hs[t] = q < nq ? h_base[(size_t)in_row[q0 + q] * H + j] : 0.f;
    }
    __syncthreads();
    const uint32_t out0 = out_row0_dev ? *out_row0_dev : 0u;
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
            if (q < nq) out_base[(size_t)(out0 + q0 + q) * H + i] = (float)otf_sigmoid(acc[q]);
    }
}

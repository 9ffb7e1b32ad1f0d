// tools/copy_micro.cu -- why does the per-level digit gather (147 KB per CTA) take ~11 us?
// 74 CTAs x 512 threads; each copies R=72 rows x 2 KB (row-major source rows at random
// indices) into a scattered 16-byte-piece layout; variants: (a) flat copy as in
// exact_update.cuh, (b) contiguous destination, (c) loads only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t toff(int row, int c) { return (uint32_t)((row >> 3) * 512 + c * 128 + (row & 7) * 16); }
template <int MODE>
__global__ void k_copy(const uint8_t *store, const int *src_rows, uint8_t *xs, int R, int NK, long long *cyc) {
    __shared__ int s_src[128];
    const int tid = threadIdx.x, NT = blockDim.x;
    const int Rp = (R + 15) & ~15;
    for (int r = tid; r < R; r += NT) s_src[r] = src_rows[blockIdx.x * 128 + r];
    __syncthreads();
    long long t0 = clock64();
    const int per_row = NK * 16, items = R * per_row;
    const size_t row_bytes = (size_t)NK * 256;
    uint8_t *x = xs + (size_t)blockIdx.x * NK * 4 * Rp * 64;
    unsigned acc = 0;
    for (int i0 = tid; i0 < items; i0 += 6 * NT) {
        uint4 v[6];
#pragma unroll
        for (int u = 0; u < 6; u++) {
            const int i = i0 + u * NT;
            v[u] = make_uint4(0, 0, 0, 0);
            if (i < items) { const int r = i / per_row, pc = i - r * per_row; v[u] = __ldcg(reinterpret_cast<const uint4 *>(store + (size_t)s_src[r] * row_bytes) + pc); }
        }
#pragma unroll
        for (int u = 0; u < 6; u++) {
            const int i = i0 + u * NT;
            if (i < items) {
                const int r = i / per_row, pc = i - r * per_row;
                if (MODE == 0) { const int kc = pc >> 4, b = (pc >> 2) & 3, c = pc & 3;
                    *reinterpret_cast<uint4 *>(x + (size_t)kc * 4 * Rp * 64 + (size_t)b * Rp * 64 + toff(r, c)) = v[u]; }
                else if (MODE == 1) *reinterpret_cast<uint4 *>(x + (size_t)i * 16) = v[u];
                else acc ^= v[u].x ^ v[u].w;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) cyc[0] = 0;
}
int main() {
    const int R = 72, NK = 8, CTAS = 74;
    const size_t rows = 1 << 20;
    uint8_t *store, *xs; int *src; long long *cyc;
    cudaMalloc(&store, rows * NK * 256); cudaMalloc(&xs, (size_t)CTAS * NK * 4 * 80 * 64); cudaMalloc(&src, CTAS * 128 * 4); cudaMalloc(&cyc, CTAS * 8);
    int h[CTAS * 128]; for (int i = 0; i < CTAS * 128; i++) h[i] = (int)(((long long)i * 2654435761u) % rows);
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMemset(store, 1, rows * NK * 256);
    for (int mode = 0; mode < 3; mode++) for (int rep = 0; rep < 3; rep++) {
        if (mode == 0) k_copy<0><<<CTAS, 512>>>(store, src, xs, R, NK, cyc);
        if (mode == 1) k_copy<1><<<CTAS, 512>>>(store, src, xs, R, NK, cyc);
        if (mode == 2) k_copy<2><<<CTAS, 512>>>(store, src, xs, R, NK, cyc);
        long long c[CTAS]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        long long mx = 0, sm = 0; for (int i = 0; i < CTAS; i++) { mx = c[i] > mx ? c[i] : mx; sm += c[i]; }
        printf("mode %d rep %d: mean %.2f us max %.2f us (1965 MHz)\n", mode, rep, sm / (double)CTAS / 1965.0, mx / 1965.0);
    }
    return 0;
}

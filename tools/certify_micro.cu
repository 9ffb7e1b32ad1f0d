// tools/certify_micro.cu -- cost of xu::certify (exact_update.cuh) per element on one SM,
// 512 threads, ILP 4 / 8, and the float64 FMA dependent-chain latency.
#include <cstdio>
#include <cstdint>
#include "../paper_2007_11794_b200/csrc/decode.cuh"
#include "../paper_2007_11794_b200/csrc/stream_decode.cuh"

template <int ILP>
__global__ void k_cert(int iters, const double *tabg, double *out, long long *cyc) {
    __shared__ double tab[32];
    if (threadIdx.x < 32) tab[threadIdx.x] = tabg[threadIdx.x];
    __syncthreads();
    double x[ILP];
    for (int i = 0; i < ILP; i++) x[i] = -2.0 + 1e-3 * threadIdx.x + 0.37 * i;
    float acc = 0.f;
    int okc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        float y[ILP];
        bool ok[ILP];
#pragma unroll
        for (int i = 0; i < ILP; i++) ok[i] = xu::certify(x[i], 3e-12, tab, y[i]);
#pragma unroll
        for (int i = 0; i < ILP; i++) { acc += y[i]; okc += ok[i]; x[i] += 1.1e-5; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (acc == 1234.5f) out[0] = okc;
    out[1 + threadIdx.x] = okc;
}
__global__ void k_lat(int iters, double a, double *out, long long *cyc) {
    double x = threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) x = fma(x, a, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x; }
}

int main() {
    double *tab, *out; long long *cyc;
    cudaMalloc(&tab, 32 * 8); cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
    double h[32]; for (int j = 0; j < 32; j++) h[j] = exp2(j / 32.0);
    cudaMemcpy(tab, h, 256, cudaMemcpyHostToDevice);
    long long c;
    k_lat<<<1, 32>>>(1000, 1.0000001, out, cyc); cudaDeviceSynchronize();
    k_lat<<<1, 32>>>(10000, 1.0000001, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", c / 10000.0);
    for (int thr : {128, 512}) {
        k_cert<4><<<1, thr>>>(10, tab, out, cyc); cudaDeviceSynchronize();
        k_cert<4><<<1, thr>>>(1000, tab, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("certify ILP4 %d thr: %.2f cycles per element per SM  (%.0f cyc per 4-elem group per thread)\n", thr,
               (double)c / (1000.0 * 4 * thr), c / 1000.0);
        k_cert<8><<<1, thr>>>(10, tab, out, cyc); cudaDeviceSynchronize();
        k_cert<8><<<1, thr>>>(1000, tab, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("certify ILP8 %d thr: %.2f cycles per element per SM\n", thr, (double)c / (1000.0 * 8 * thr));
    }
    return 0;
}

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
// variant: the 2^(j/32) table in a register (lane j holds entry j), read by shuffle
__device__ __forceinline__ double exp_neg_shfl(double x, double tabreg) {
    const double t = x * -46.166241308446828;
    const double sh = t + 6755399441055744.0;
    const int k = __double2loint(sh);
    const double kd = sh - 6755399441055744.0;
    double r = fma(kd, -0.021660849386535119265, -x);
    r = fma(kd, -5.9631716539705865626e-12, r);
    double p = 1.0 / 720.0;
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    p *= __shfl_sync(0xffffffffu, tabreg, k & 31);
    return __hiloint2double(__double2hiint(p) + ((k >> 5) << 20), __double2loint(p));
}
__device__ __forceinline__ bool certify_shfl(double x, double epsm, double tabreg, float &out) {
    const double z = 1.0 + exp_neg_shfl(x, tabreg);
    double h;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(h) : "d"(z));
    h = fma(h, fma(-z, h, 1.0), h);
    h = fma(h, fma(-z, h, 1.0), h);
    const float y = __double2float_rn(h);
    const uint32_t yb = __float_as_uint(y);
    const double d = h - xu::widen_d(y);
    const uint32_t ey = (yb >> 23) & 255u;
    const int hw = (int)((ey + 1023u - 127u - 24u) << 20);
    const double half_up = __hiloint2double(hw, 0);
    const double half_dn = __hiloint2double((yb & 0x7FFFFFu) ? hw : hw - (1 << 20), 0);
    const double margin = epsm * h;
    out = y;
    const bool ok = d >= 0.0 ? d + margin < half_up : margin - d < half_dn;
    return ok && fabs(x) < 60.0 && ey >= 1u && yb < 0x3F800000u;
}
template <int ILP>
__global__ void k_cert_shfl(int iters, const double *tabg, double *out, long long *cyc) {
    const double tabreg = tabg[threadIdx.x & 31];
    double x[ILP];
    for (int i = 0; i < ILP; i++) x[i] = -2.0 + 1e-3 * threadIdx.x + 0.37 * i;
    float acc = 0.f;
    int okc = 0, diff = 0;
    __shared__ double tab[32];
    if (threadIdx.x < 32) tab[threadIdx.x] = tabg[threadIdx.x];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        float y[ILP];
        bool ok[ILP];
#pragma unroll
        for (int i = 0; i < ILP; i++) ok[i] = certify_shfl(x[i], 3e-12, tabreg, y[i]);
#pragma unroll
        for (int i = 0; i < ILP; i++) { acc += y[i]; okc += ok[i]; x[i] += 1.1e-5; }
    }
    long long t1 = clock64();
    // identity with the shared-memory table version on a few values
    for (int i = 0; i < ILP; i++) {
        float ya, yb2; const bool a = xu::certify(x[i], 3e-12, tab, ya), b = certify_shfl(x[i], 3e-12, tabreg, yb2);
        diff += (a != b) || (__float_as_uint(ya) != __float_as_uint(yb2));
    }
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (acc == 1234.5f) out[0] = okc;
    out[1 + threadIdx.x] = diff;
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
        k_cert_shfl<4><<<1, thr>>>(10, tab, out, cyc); cudaDeviceSynchronize();
        k_cert_shfl<4><<<1, thr>>>(1000, tab, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double dd[1025]; cudaMemcpy(dd, out, 8 * (1 + thr), cudaMemcpyDeviceToHost);
        double nd = 0; for (int i = 1; i <= thr; i++) nd += dd[i];
        printf("certify(shfl table) ILP4 %d thr: %.2f cycles per element per SM, mismatches %g\n", thr,
               (double)c / (1000.0 * 4 * thr), nd);
    }
    return 0;
}

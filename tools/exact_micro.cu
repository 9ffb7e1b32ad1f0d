// tools/exact_micro.cu -- feasibility probes for the exact (integer-sliced)
// recurrent update on sm_100a:
//   1. tcgen05.mma kind::i8 (A s8, B u8, D s32) correctness vs a host dot;
//   2. cycles per i8 MMA (M=128, K=32) vs N, next to tf32 (K=8);
//   3. DFMA and f32->f64 conversion throughput of one SM;
//   4. f64 exp throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exact_micro tools/exact_micro.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// no-swizzle K-major: core matrix = 8 rows x 16 B; LBO = K-adjacent core
// matrices, SBO = 8-row groups
__host__ __device__ inline uint32_t toff(int row, int c, int kcb) { return (row >> 3) * (kcb / 16 * 128) + c * 128 + (row & 7) * 16; }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    return d;
}

// A [128 x K] s8 row-major (K contiguous), B [N x K] u8; out D [128 x N] s32
__global__ void k_i8_check(const int8_t *A, const uint8_t *B, int N, int K, int *D, long long *cyc, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    const int kcb = K;    // whole K resident
    uint8_t *sA = smem, *sB = smem + 128 * K;
    for (int i = tid; i < 128 * K / 16; i += blockDim.x) {
        const int row = i / (K / 16), c = i % (K / 16);
        *reinterpret_cast<uint4 *>(sA + toff(row, c, kcb)) = *reinterpret_cast<const uint4 *>(A + row * K + c * 16);
    }
    for (int i = tid; i < N * K / 16; i += blockDim.x) {
        const int row = i / (K / 16), c = i % (K / 16);
        *reinterpret_cast<uint4 *>(sB + toff(row, c, kcb)) = *reinterpret_cast<const uint4 *>(B + row * K + c * 16);
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    // D s32 (2 << 4), A s8 (1 << 7), B u8 (0 << 10), K-major both
    const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
    long long t0 = 0, t1 = 0;
    if (wid == 0) {
        for (int rep = 0; rep < 2; rep++) {
            t0 = clock64();
            for (int r = 0; r < reps; r++)
            for (int ks = 0; ks < K / 32; ks++) {
                const uint64_t da = desc(su32(sA) + ks * 256, 128, kcb / 16 * 128);
                const uint64_t db = desc(su32(sB) + ks * 256, 128, kcb / 16 * 128);
                const uint32_t acc = (ks > 0 || r > 0) ? 1u : 0u;
                asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 rr;\n\telect.sync rr|e, 0xffffffff;\n\t"
                             "setp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                             :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 rr;\n\telect.sync rr|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                         :: "r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D2;\n\tbra W2;\n\tD2:\n\t}"
                         :: "r"(su32(&bar)), "r"(rep & 1) : "memory");
            t1 = clock64();
        }
        if (tid == 0) *cyc = t1 - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // 4 warps read lanes 32w..32w+31, columns 0..N-1
    if (wid < 4) {
        for (int c = 0; c < N; c++) {
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(wid * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            D[(wid * 32 + (tid & 31)) * N + c] = (int)v;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

// DFMA throughput: each thread runs 8 independent chains
__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.678) out[0] = s;
}
// f32 -> f64 conversions (+ a DADD each so they are not dead)
__global__ void k_cvt(const float *in, double *out, int iters) {
    float f[8];
    for (int i = 0; i < 8; i++) f[i] = in[threadIdx.x & 31] + i;
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) { s[i] += (double)f[i]; f[i] += 1.0f; }
    }
    double t = 0;
    for (int i = 0; i < 8; i++) t += s[i];
    if (t == 12345.678) out[0] = t;
}
__global__ void k_exp(double *out, int iters) {
    double x[4];
    for (int i = 0; i < 4; i++) x[i] = -0.5 + threadIdx.x * 1e-4 + i * 0.1;
    double s = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 4; i++) { const double e = exp(-x[i]); s += 1.0 / (1.0 + e); x[i] += 1e-7; }
    }
    if (s == 12345.678) out[0] = s;
}

int main() {
    // ---- 1/2: kind::i8
    for (int N : {16, 24, 48, 80, 96, 128, 256}) {   // (N = 40, 72: illegal instruction: steps of 16 above 32)
        const int K = 128;
        int8_t *hA = (int8_t *)malloc(128 * K);
        uint8_t *hB = (uint8_t *)malloc(N * K);
        srand(7 + N);
        for (int i = 0; i < 128 * K; i++) hA[i] = (int8_t)((rand() & 255) - 128);
        for (int i = 0; i < N * K; i++) hB[i] = (uint8_t)(rand() & 255);
        int8_t *dA; uint8_t *dB; int *dD; long long *dc;
        cudaMalloc(&dA, 128 * K); cudaMalloc(&dB, N * K); cudaMalloc(&dD, 128 * N * 4); cudaMalloc(&dc, 8);
        cudaMemcpy(dA, hA, 128 * K, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_i8_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        k_i8_check<<<1, 128, 128 * K + N * K + 1024>>>(dA, dB, N, K, dD, dc, 1);
        int *hD = (int *)malloc(128 * N * 4);
        cudaError_t e = cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("i8 N=%d: %s\n", N, cudaGetErrorString(e)); return 1; }
        int bad = 0;
        for (int m = 0; m < 128; m++)
            for (int n = 0; n < N; n++) {
                long long s = 0;
                for (int k = 0; k < K; k++) s += (long long)hA[m * K + k] * (long long)hB[n * K + k];
                if (s != hD[m * N + n]) { if (bad < 3) printf("  mismatch m=%d n=%d dev=%d host=%lld\n", m, n, hD[m * N + n], s); bad++; }
            }
        // timing: 64 reps of K/32 MMAs into one accumulator
        const int reps = 64;
        k_i8_check<<<1, 128, 128 * K + N * K + 1024>>>(dA, dB, N, K, dD, dc, reps);
        long long c = 0;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("i8 N=%3d: %s (%d bad)  %.1f cyc/mma (M=128,K=32)\n", N, bad ? "MISMATCH" : "exact", bad,
               (double)c / (reps * K / 32));
        cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc); free(hA); free(hB); free(hD);
    }
    // ---- 3/4: FP64 rates on the whole chip and one SM
    double *dout; cudaMalloc(&dout, 8);
    float *din; cudaMalloc(&din, 128); cudaMemset(din, 0, 128);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int blocks : {1, sms * 4}) {
        const int iters = 4096, thr = 512;
        k_dfma<<<blocks, thr>>>(dout, 16, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<<<blocks, thr>>>(dout, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double dfma = (double)blocks * thr * iters * 8;
        printf("DFMA  blocks=%4d: %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz)\n", blocks, 2 * dfma / ms / 1e9,
               dfma / (ms * 1e-3) / (clk * 1e3) / (blocks < sms ? blocks : sms), clk / 1000);
        k_cvt<<<blocks, thr>>>(din, dout, 16);
        cudaEventRecord(e0);
        k_cvt<<<blocks, thr>>>(din, dout, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("CVT+DADD blocks=%4d: %.1f cvt/clk/SM\n", blocks, dfma / (ms * 1e-3) / (clk * 1e3) / (blocks < sms ? blocks : sms));
        k_exp<<<blocks, thr>>>(dout, 16);
        cudaEventRecord(e0);
        k_exp<<<blocks, thr>>>(dout, iters / 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double ne = (double)blocks * thr * (iters / 4) * 4;
        printf("f64 sigmoid blocks=%4d: %.2f per clk per SM\n", blocks, ne / (ms * 1e-3) / (clk * 1e3) / (blocks < sms ? blocks : sms));
    }
    return 0;
}

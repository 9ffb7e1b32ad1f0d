// tools/mma_micro.cu -- tcgen05.mma issue/completion microbenchmark (one CTA).
// Measures cycles per MMA (M=128, tf32, K=8) for a chain of NMMA MMAs
// into NACC independent TMEM accumulators, for several N, with SS operands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_micro tools/mma_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, int sw) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    if (sw) {
        d |= 1ull << 16;
        d |= (uint64_t)((8 * 64) >> 4) << 32;   // SW64: 8 rows x 64 B
        d |= 1ull << 46;
        d |= 4ull << 61;
    } else {
        d |= (uint64_t)(128 >> 4) << 16;        // LBO
        d |= (uint64_t)(512 >> 4) << 32;        // SBO (64 B rows of 4 chunks)
        d |= 1ull << 46;
    }
    return d;
}

__global__ void k_micro(int N, int nacc, int nmma, int sw, int mode_elect, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 0.001f * (i & 255);
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t sA = su32(smem), sB = su32(smem + 32768);
    long long t0 = 0, t1 = 0;
    const int wid_u = __shfl_sync(0xffffffffu, tid >> 5, 0);
    if (mode_elect && wid_u == 0) {
        // whole warp runs the loop; descriptors uniform; elect.sync inside asm
        for (int rep = 0; rep < 2; rep++) {
            t0 = clock64();
            for (int i = 0; i < nmma; i++) {
                const int a = i % nacc;
                const uint32_t d = tmem + (uint32_t)(a * (512 / nacc) / 16 * 16);
                const uint64_t da = desc(sA + (i & 1) * 32, sw), db = desc(sB + (i & 1) * 32, sw);
                const uint32_t acc = i >= nacc ? 1u : 0u;
                asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
                             "elect.sync r|e, 0xffffffff;\n\t"
                             "setp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             :: "r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                         :: "r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D2;\n\tbra W2;\n\tD2:\n\t}"
                         :: "r"(su32(&bar)), "r"(rep & 1) : "memory");
            t1 = clock64();
        }
        if (tid == 0) out[0] = t1 - t0;
    }
    if (!mode_elect && tid == 0) {
        for (int rep = 0; rep < 2; rep++) {
            t0 = clock64();
            for (int i = 0; i < nmma; i++) {
                const int a = i % nacc;
                const uint32_t d = tmem + (uint32_t)(a * (512 / nacc) / 16 * 16);
                const uint64_t da = desc(sA + (i & 1) * 32, sw), db = desc(sB + (i & 1) * 32, sw);
                const uint32_t acc = i >= nacc ? 1u : 0u;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             :: "r"(d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}"
                         :: "r"(su32(&bar)), "r"(rep & 1) : "memory");
            t1 = clock64();
        }
        out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_micro, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int Ns[] = {16, 32, 64, 80, 128, 256};
    for (int me = 0; me < 2; me++)
    for (int sw = 0; sw < 2; sw++)
        for (int nacc : {1, 2, 6})
            for (int N : Ns) {
                if (nacc * N > 512) continue;
                const int nmma = 192;
                k_micro<<<1, 128, 65536>>>(N, nacc, nmma, sw, me, d);
                long long h = 0;
                cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                printf("elect=%d sw=%d nacc=%d N=%3d : %7.1f cyc/mma  (floor N/2 = %d)\n", me, sw, nacc, N, (double)h / nmma, N / 2), (void)0;
            }
    return 0;
}

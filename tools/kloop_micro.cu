// tools/kloop_micro.cu -- is the EXACT update's K loop tensor-bound or
// operand-bound?  148 CTAs (one per SM) each run the update's K loop shape:
// 4 M tiles x (K = 512) with 17 digit-pair MMAs (8 instructions per 32-byte
// K step, N = Rp..256) per K step; W planes (5 x 128 rows) and h planes
// (4 x Rp rows) arrive by cp.async.bulk into a ring of S stages of KCB bytes
// of K.  Modes: 0 = copies + MMAs, 1 = MMAs only (operands resident),
// 2 = copies only.  Prints cycles per M tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/kloop_micro tools/kloop_micro.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    return d;
}
__device__ __forceinline__ uint32_t idesc(bool a_signed, int n) {
    // kind::i8: D s32 (bit 4), A s8/u8 (bits 7..9), B u8 (10..12), K-major, N >> 3, M >> 4
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint32_t b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(n)); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" :: "r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ void commit(uint32_t b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(b) : "memory");
}


// one 32-byte K step of layout 1 at Rp = 64 in ONE asm block: 5 MMAs whose
// descriptor / TMEM offsets are immediates, so only the three bases need the
// uniform datapath
__device__ __forceinline__ void ks_rp64(uint32_t tm, uint64_t da, uint64_t db) {
    constexpr uint32_t ID256 = (2u << 4) | (0u << 7) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t ID256S = ID256 | (1u << 7);
    constexpr uint32_t ID192 = (2u << 4) | ((192u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t ID128 = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t1, t2, t3, t4;\n\t.reg .b64 a1, a2, a3, a4;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "add.u32 t1, %0, 64;\n\tadd.u32 t2, %0, 128;\n\tadd.u32 t3, %0, 192;\n\tadd.u32 t4, %0, 256;\n\t"
                 "add.s64 a1, %1, 512;\n\tadd.s64 a2, %1, 1024;\n\tadd.s64 a3, %1, 1536;\n\tadd.s64 a4, %1, 2048;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t1], a1, %2, %4, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t2], a2, %2, %4, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t3], a3, %2, %5, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t4], a4, %2, %6, 1;\n\t}"
                 :: "r"(tm), "l"(da), "l"(db), "n"(ID256S), "n"(ID256), "n"(ID192), "n"(ID128));
}

// one MMA per asm statement, offsets as immediates (layout 4)
template <uint32_t TOFF, uint32_t AOFF, uint32_t BOFF, uint32_t IDESC, int ACC>
__device__ __forceinline__ void mma_imm(uint32_t tm, uint64_t da, uint64_t db) {
    asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 t;\n\t.reg .b64 a, b;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "add.u32 t, %0, %3;\n\tadd.s64 a, %1, %4;\n\tadd.s64 b, %2, %5;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [t], a, b, %6, %7;\n\t}"
                 :: "r"(tm), "l"(da), "l"(db), "n"(TOFF), "n"(AOFF >> 4), "n"(BOFF >> 4), "n"(IDESC), "n"(ACC));
}
__device__ __forceinline__ void ks4_rp64(uint32_t tm, uint64_t da, uint64_t db) {
    constexpr uint32_t ID256 = (2u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t ID192 = (2u << 4) | ((192u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t ID128 = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    mma_imm<0, 0, 0, ID256 | (1u << 7), 1>(tm, da, db);
    mma_imm<64, 8192, 0, ID256, 1>(tm, da, db);
    mma_imm<128, 16384, 0, ID256, 1>(tm, da, db);
    mma_imm<192, 24576, 0, ID192, 1>(tm, da, db);
    mma_imm<256, 32768, 0, ID128, 1>(tm, da, db);
}

__host__ __device__ constexpr uint32_t idesc_c(bool a_signed, int n) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
template <int RP, int A, int B0, int NB, int ACC>
__device__ __forceinline__ void range_imm(uint32_t tm, uint64_t da, uint64_t db) {
    constexpr int TOT = NB * RP, N1 = TOT < 256 ? TOT : 256, N2 = TOT - N1;
    mma_imm<(uint32_t)((A + B0) * RP), (uint32_t)(A * 128 * 64), (uint32_t)(((B0 * RP) >> 3) * 512), idesc_c(A == 0, N1), ACC>(tm, da, db);
    if constexpr (N2 > 0)
        mma_imm<(uint32_t)((A + B0) * RP + 256), (uint32_t)(A * 128 * 64), (uint32_t)(((B0 * RP + 256) >> 3) * 512), idesc_c(A == 0, N2), ACC>(tm, da, db);
}
template <int RP>
__device__ __forceinline__ void ks_steady(uint32_t tm, uint64_t da, uint64_t db) {
    range_imm<RP, 0, 0, 4, 1>(tm, da, db); range_imm<RP, 1, 0, 4, 1>(tm, da, db); range_imm<RP, 2, 0, 4, 1>(tm, da, db);
    range_imm<RP, 3, 0, 3, 1>(tm, da, db); range_imm<RP, 4, 0, 2, 1>(tm, da, db);
}
__device__ __forceinline__ void ks_any(int Rp, uint32_t tm, uint64_t da, uint64_t db) {
    switch (Rp) { case 16: ks_steady<16>(tm, da, db); break; case 32: ks_steady<32>(tm, da, db); break;
                  case 48: ks_steady<48>(tm, da, db); break; case 64: ks_steady<64>(tm, da, db); break;
                  case 80: ks_steady<80>(tm, da, db); break; default: break; }
}

template <int KCB>
__global__ void __launch_bounds__(128, 1) k_loop(const uint8_t *Wd, const uint8_t *xs, int S, int Rp, int mode,
                                                 int reps, long long *cyc, int layout) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[8], empty[8], done;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, wid = tid >> 5;
    constexpr int NK = 512 / KCB;                      // K chunks per tile
    const uint32_t PW = 128 * KCB, HB = 4u * Rp * KCB, STAGE = 5 * PW + HB;
    if (tid == 0) {
        for (int s = 0; s < S; s++) { mbar_init(su32(&full[s]), 1); mbar_init(su32(&empty[s]), 1); }
        mbar_init(su32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint8_t *myxs = xs + (size_t)blockIdx.x * NK * HB;
    uint32_t gc = 0, tiles = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int mt = 0; mt < 4; mt++) {
            if (wid == 1) {
                for (int kc = 0; kc < NK; kc++, gc++) {
                    const int st = (int)(gc % (uint32_t)S);
                    const uint32_t use = gc / (uint32_t)S;
                    if (use >= 1) mbar_wait(su32(&empty[st]), (use - 1) & 1);
                    __syncwarp();
                    if (tid == 32) {
                        uint8_t *dst = smem + (size_t)st * STAGE;
                        if (mode == 1) {
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&full[st])) : "memory");
                        } else {
                            const uint8_t *sw = Wd + ((size_t)mt * NK + kc) * 5 * PW;
                            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[st])), "r"(STAGE) : "memory");
                            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                         :: "r"(su32(dst)), "l"(sw), "r"(5 * PW), "r"(su32(&full[st])) : "memory");
                            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                         :: "r"(su32(dst + 5 * PW)), "l"(myxs + (size_t)kc * HB), "r"(HB), "r"(su32(&full[st])) : "memory");
                        }
                    }
                    __syncwarp();
                }
            } else if (wid == 0) {
                uint32_t g2 = gc;
                for (int kc = 0; kc < NK; kc++, g2++) {
                    const int st = (int)(g2 % (uint32_t)S);
                    mbar_wait(su32(&full[st]), (g2 / (uint32_t)S) & 1);
                    __syncwarp();
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (layout == 4 && mode != 2) {
                        const uint32_t sW = su32(smem + (size_t)st * STAGE), sH = sW + 5 * PW;
                        const uint64_t da0 = desc(sW, 128, 8 * KCB), db0 = desc(sH, 128, 8 * KCB);
                        for (int ks = 0; ks < KCB / 32; ks++) ks_any(Rp, tmem, da0 + 16 * ks, db0 + 16 * ks);
                        if (tid == 0) {
                            commit(su32(&empty[st]));
                            if (kc == NK - 1) commit(su32(&done));
                        }
                    } else if (layout == 3 && mode != 2) {
                        // whole warp: the asm elects one lane itself
                        const uint32_t sW = su32(smem + (size_t)st * STAGE), sH = sW + 5 * PW;
                        const uint64_t da0 = desc(sW, 128, 8 * KCB), db0 = desc(sH, 128, 8 * KCB);
                        for (int ks = 0; ks < KCB / 32; ks++) ks_rp64(tmem, da0 + 16 * ks, db0 + 16 * ks);
                        if (tid == 0) {
                            commit(su32(&empty[st]));
                            if (kc == NK - 1) commit(su32(&done));
                        }
                    } else if (tid == 0) {
                        if (mode != 2) {
                            const uint32_t sW = su32(smem + (size_t)st * STAGE), sH = sW + 5 * PW;
                            for (int ks = 0; ks < KCB / 32; ks++) {
                                const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
                                auto range = [&](int a, int b0, int nb, uint32_t acc) {
                                    const int tot = nb * Rp;
                                    for (int off = 0; off < tot; off += 256) {
                                        const int nn = tot - off < 256 ? tot - off : 256;
                                        const int brow = b0 * Rp + off;
                                        const uint64_t da = desc(sW + (uint32_t)a * PW + (uint32_t)ks * 256u, 128, 8 * KCB);
                                        const uint64_t db = desc(sH + (uint32_t)(brow >> 3) * (8 * KCB) + (uint32_t)ks * 256u, 128, 8 * KCB);
                                        mma_i8(tmem + (uint32_t)((a + b0) * Rp + off), da, db, idesc(a == 0, nn), acc);
                                    }
                                };
                                if (layout == 0 || acc0 == 0u) {
                                    range(0, 0, 4, acc0); range(1, 0, 3, 1u); range(1, 3, 1, acc0); range(2, 0, 3, 1u);
                                    range(2, 3, 1, acc0); range(3, 0, 3, 1u); range(4, 0, 2, 1u);
                                } else if (layout == 1) {      // merged ranges once every block is initialised
                                    range(0, 0, 4, 1u); range(1, 0, 4, 1u); range(2, 0, 4, 1u); range(3, 0, 3, 1u);
                                    range(4, 0, 2, 1u);
                                } else {                       // reference: N = 256 MMAs only, same column total
                                    for (int t = 0; t < 17 * Rp; t += 256) {
                                        const int nn = 17 * Rp - t < 256 ? 17 * Rp - t : 256;
                                        mma_i8(tmem, desc(sW, 128, 8 * KCB), desc(sH, 128, 8 * KCB), idesc(false, nn < 16 ? 16 : nn), 1u);
                                    }
                                }
                            }
                            commit(su32(&empty[st]));
                            if (kc == NK - 1) commit(su32(&done));
                        } else {
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[st])) : "memory");
                            if (kc == NK - 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&done)) : "memory");
                        }
                    }
                    __syncwarp();
                }
                mbar_wait(su32(&done), tiles & 1);
            }
            gc = (wid == 1) ? gc : gc + NK;
            tiles++;
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / (reps * 4);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

int main() {
    const int NB = 148, reps = 50;
    uint8_t *Wd, *xs;
    long long *cyc;
    cudaMalloc(&Wd, 4 * 512 * 5 * 128);
    cudaMalloc(&xs, (size_t)NB * 512 * 4 * 128);
    cudaMemset(Wd, 1, 4 * 512 * 5 * 128);
    cudaMemset(xs, 1, (size_t)NB * 512 * 4 * 128);
    cudaMallocManaged(&cyc, NB * sizeof(long long));
    for (int layout : {4})
        for (int Rp : {16, 32, 48, 64, 80}) {
            
            const int S = 2, kcb = 64;
            const size_t stage = 5 * 128 * kcb + 4 * Rp * kcb;
            const size_t smem = S * stage;
            for (int mode : {1, 0}) {
                cudaFuncSetAttribute(k_loop<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_loop<64><<<NB, 128, smem>>>(Wd, xs, S, Rp, mode, reps, cyc, layout);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                long long mx = 0;
                for (int i = 0; i < NB; i++) mx = cyc[i] > mx ? cyc[i] : mx;
                printf("layout %d Rp %3d %s: %6lld cycles per M tile (%.2f us) = %.3f cycles per (column x K step)\n", layout, Rp,
                       mode == 0 ? "copy+mma" : "mma only", mx, mx / 1965.0, mx / 16.0 / (17.0 * Rp));
            }
        }
    return 0;
}

// Exact BFV scale-and-round t*D/q (bfv.cpp:811-849) of the tensor product on the tensor cores.
//
// HPS decomposition (also used by the IMAD-only fallback k_round_mac_t, ntt_reg.cuh):
//   w_j = D_j (A/a_j)^-1 mod a_j,   gamma = round(sum_j w_j / a_j),
//   r = sum_j w_j I_j - gamma I_A + rho,   rho = round(sum_j w_j F_j - gamma F_A),
// with t (A/a_j) = (I_j + F_j) q.  The result is needed mod each MAC prime a_k (k < Mm).
#pragma once
#include "kernels.cuh"
#include "ntt_reg.cuh"
#include "mac.cuh"

namespace cwgpu {

// ---------------------------------------------------------------------------------------
// Tensor-core variant (tcgen05.mma kind::i8, A from TMEM, B from shared memory).
//
// Every quantity the rounding needs is a dot product of the coefficient's residues w_j with
// per-prime constants, so a 128-coefficient tile is one small int8 GEMM: A[coef][4j + a] is
// byte a of w_j (the thread's JM words, as stored, ARE its K = 4 JM bytes) and each column
// of B holds bytes of one constant, placed so that column groups recombine by shifts:
//   residues   cols 4k+b   : byte b of (2^(8a) I_kj 2^32 mod a_k)      S_k = sum_b C 2^(8b)
//   fraction   cols F0+s   : byte s-a of the 64-bit fraction F_j       FR  = sum_s C 2^(8s)
//   gamma      cols G0+s   : byte s-a of floor(2^46 / a_j)             GS  = sum_s C 2^(8s)
// Each column sum is < K 255^2 < 2^23, exact in the int32 accumulator.  The epilogue
// (CUDA cores) adds the gamma / rho corrections and reduces mod a_k (Montgomery).  The
// residues arrive already multiplied by (A/a_j)^-1 (folded into the INTT scaling).
// ---------------------------------------------------------------------------------------

template <int JM, int NC>
struct RoundTcPar {
    static constexpr int K = 4 * JM;        // GEMM depth in bytes
    static constexpr int F0 = NC - 17;      // fraction columns F0 .. F0+10
    static constexpr int G0 = NC - 6;       // gamma columns G0 .. G0+5
    static constexpr int MMAX = F0 / 4;     // residue column groups available
    // per MAC prime: {a, -a^-1 mod 2^32, (-I_A) 2^32 mod a, 2^30 - a < 2^24}; (-2^36) 2^32 mod a
    uint4 kq[MMAX];
    u32 krm[MMAX];
    // k_round_tma epilogue: (rho + 2^36) mod a_k enters the Montgomery sum as rlo 2^32 + rhi 2^62
    u32 kc0[MMAX];   // 2^32 mod a_k
    u32 kc30[MMAX];  // 2^62 mod a_k
};

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------------------------------
// k_round_tma: a producer warp streams each 128-coefficient tile's J plane segments (512 B
// each, contiguous) into a kRtStages-deep shared-memory ring with cp.async.bulk, completing on a
// `full` mbarrier; the 4 consumer warps read their coefficient's J words from the ring
// (conflict-free) into their TMEM lanes, release the stage, issue the GEMM (one elected thread)
// and run the epilogue, writing the Mm MAC-basis residues in place.  (A first version without
// the producer warp -- the consumers loading their own planes -- kept one tile in flight per CTA
// and reached ~45% of HBM.)  Persistent: CTA b handles tiles b, b + grid, ...
// ---------------------------------------------------------------------------------------
constexpr int kRtStages = 4;
template <int JM>
constexpr size_t round_tma_smem() { return (size_t)kRtStages * JM * 128 * 4; }

template <int LOGN, int JM, int NC, int MMT = 0>  // LOGN = 0: N at run time; MMT = 0: Mm at run time
__global__ void __launch_bounds__(160, 4) k_round_tma(u32* __restrict__ D, u32 P, DevTab T,
                                                     const __grid_constant__ RoundTcPar<JM, NC> RP,
                                                     const uint4* __restrict__ Bglob, const RoundK* __restrict__ gRK,
                                                     const uint4* __restrict__ B2glob,
                                                     const __grid_constant__ CUtensorMap tmD) {
    using RPT = RoundTcPar<JM, NC>;
    constexpr int K = RPT::K, F0 = RPT::F0, G0 = RPT::G0;
    constexpr int KSTEPS = K / 32;
    constexpr int A2 = JM + NC;  // TMEM columns of the second GEMM's A operand (8 x 32 bit = K 32 bytes)
    constexpr bool G2OK = A2 + 8 <= 128;  // A, D and A2 fit the 128-column allocation
    __shared__ __align__(128) uint4 Bs[NC * K / 16];
    __shared__ __align__(128) uint4 Bs2[G2OK ? NC * 32 / 16 : 1];
    const bool g2 = G2OK && B2glob != nullptr;
    extern __shared__ __align__(128) u32 ringd[];  // [kRtStages][JM][128]
    auto ring = reinterpret_cast<u32(*)[JM][128]>(ringd);
    __shared__ __align__(8) unsigned long long mbar, full[kRtStages], empty[kRtStages];
    __shared__ u32 tmem_base_sh;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 J = T.J, Mm = MMT ? (u32)MMT : T.Mm;
    const u32 N = LOGN ? (1u << LOGN) : T.N, logN = LOGN ? (u32)LOGN : T.logN;  // compile-time N: immediate plane offsets
    const size_t total = (size_t)P * 3 * N;
    const u32 ntiles = (u32)((total + 127) / 128);

    for (u32 x = tid; x < NC * K / 16; x += blockDim.x) Bs[x] = Bglob[x];
    if (g2)
        for (u32 x = tid; x < NC * 32 / 16; x += blockDim.x) Bs2[x] = B2glob[x];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        mbar_init(&mbar, 1);
        for (int i = 0; i < kRtStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

    if (warp == 4) {  // producer: J plane segments of each tile -> ring stage
        if ((tid & 31) == 0) {
            u32 i = 0;
            for (u32 tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++i) {
                const u32 st = i % kRtStages;
                if (i >= (u32)kRtStages) mbar_wait_sleep(&empty[st], ((i / kRtStages) - 1) & 1);
                const size_t base = (size_t)tl * 128;
                const size_t pc = base >> logN;
                const u32 n0 = (u32)(base & (N - 1));
                mbar_expect_tx(&full[st], J * 512u);
                // one {128, J, 1} box of D viewed as [pc][plane][n]: per-plane 512 B bulk copies were
                // bound by the copy issue rate (~30-50 ns per copy and SM)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                        "r"(smem_u32(&ring[st][0][0])),
                    "l"(&tmD), "r"(n0), "r"(0u), "r"((u32)pc), "r"(smem_u32(&full[st]))
                    : "memory");
            }
        }
        return;
    }

    const u32 tbase = tmem_base_sh;
    const u32 ta = tbase + ((warp * 32u) << 16);
    const u32 td = ta + JM;
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((K / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);
    const u64 bdesc2 = ((u64)((smem_u32(Bs2) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((32 / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 fA0 = T.fracA[1], fA1 = T.fracA[2];
    u32 phase = 0, i = 0;
#pragma unroll 1
    for (u32 tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++i) {
        const u32 st = i % kRtStages;
        const size_t idx = (size_t)tl * 128 + tid;
        const size_t pc = idx >> logN;
        const u32 n = (u32)(idx & (N - 1));
        u32* Dp = D + pc * T.DS * N + n;
        mbar_wait_sleep(&full[st], (i / kRtStages) & 1);
        u32 w[JM];
#pragma unroll
        for (int j = 0; j < JM; ++j) w[j] = j < (int)J ? ring[st][j][tid] : 0u;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // next writer of the stage: TMA
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[st]);
#pragma unroll
        for (int c = 0; c < JM; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + c),
                         "r"(w[c]), "r"(w[c + 1]), "r"(w[c + 2]), "r"(w[c + 3]), "r"(w[c + 4]), "r"(w[c + 5]),
                         "r"(w[c + 6]), "r"(w[c + 7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const u64 bd = bdesc0 + (u64)((s * 2 * 128) >> 4);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + JM),
                    "r"(tbase + (u32)(s * 8)), "l"(bd), "r"(idesc), "r"(s)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        mbar_wait_sleep(&mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        u32 C[17];  // fraction / gamma columns F0 .. NC-1
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];\n"
            : "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]), "=r"(C[8]),
              "=r"(C[9]), "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15]), "=r"(C[16])
            : "r"(td + F0 + 1)
            : "memory");
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(C[0]) : "r"(td + F0) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        u64 gs = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) gs += (u64)C[G0 - F0 + s] << (8 * s);
        const u32 gamma = (u32)((gs + (1ull << 45)) >> 46);
        u64 plo = 0, phi = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) plo += (u64)C[s] << (8 * s);
#pragma unroll
        for (int s = 6; s < 11; ++s) phi += (u64)C[s] << (8 * (s - 6));
        const u64 lo64 = plo + (phi << 48);
        const u64 hi64 = (phi >> 16) + (lo64 < plo ? 1u : 0u);
        u32 s0 = (u32)lo64, s1 = (u32)(lo64 >> 32), s2 = (u32)hi64, s3 = (u32)(hi64 >> 32);
        {
            const u64 p0 = (u64)gamma * fA0, p1 = (u64)gamma * fA1;
            const u32 q0 = (u32)p0;
            const u64 t1 = (p0 >> 32) + (u32)p1;
            const u32 q1 = (u32)t1;
            const u32 q2 = (u32)((t1 >> 32) + (p1 >> 32));
            asm("sub.cc.u32  %0, %0, %4;\n\t"
                "subc.cc.u32 %1, %1, %5;\n\t"
                "subc.cc.u32 %2, %2, %6;\n\t"
                "subc.u32    %3, %3, 0;\n\t"
                "add.cc.u32  %1, %1, 0x80000000;\n\t"
                "addc.cc.u32 %2, %2, 0;\n\t"
                "addc.u32    %3, %3, 0;\n\t"
                : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3)
                : "r"(q0), "r"(q1), "r"(q2));
        }
        const long long rho = (long long)(((u64)s3 << 32) | s2);
        const bool bad = (s1 == 0u && s0 < 64u) || (s1 >= 0xfffffff0u) || T.force_exact;
        if (g2) {
            // second GEMM: the gamma / rho / offset corrections enter the residue columns on the
            // tensor core (K = 32 bytes: gamma < J, rb = rho + 2^36 < 2^37 in 5 bytes, a constant 1)
            {
                const u64 rb = (u64)(rho + (1ll << 36));
                const u32 a0 = gamma | (u32)((rb & 0xffffffull) << 8);
                const u32 a1 = (u32)((rb >> 24) & 0xffffull) | (1u << 16);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %3, %3, %3, %3, %3};\n" ::"r"(ta + A2),
                             "r"(a0), "r"(a1), "r"(0u)
                             : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                if (tid == 0) {
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + JM),
                        "r"(tbase + (u32)A2), "l"(bdesc2), "r"(idesc)
                        : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     smem_u32(&mbar))
                                 : "memory");
                }
                mbar_wait_sleep(&mbar, phase);
                phase ^= 1u;
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            }
#pragma unroll
            for (int k0 = 0; k0 < RPT::MMAX; k0 += 4) {  // S'_k < 2^49: one Montgomery reduction, < a + 2^17
                u32 Rc[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                    "%14, %15}, [%16];\n"
                    : "=r"(Rc[0]), "=r"(Rc[1]), "=r"(Rc[2]), "=r"(Rc[3]), "=r"(Rc[4]), "=r"(Rc[5]), "=r"(Rc[6]),
                      "=r"(Rc[7]), "=r"(Rc[8]), "=r"(Rc[9]), "=r"(Rc[10]), "=r"(Rc[11]), "=r"(Rc[12]), "=r"(Rc[13]),
                      "=r"(Rc[14]), "=r"(Rc[15])
                    : "r"(td + 4 * k0)
                    : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (!bad) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int k = k0 + kk;
                        if (k < RPT::MMAX && (MMT ? k < MMT : k < (int)Mm)) {
                            const u32 a = RP.kq[k].x;
                            const u32 p01 = Rc[4 * kk] + (Rc[4 * kk + 1] << 8), p23 = Rc[4 * kk + 2] + (Rc[4 * kk + 3] << 8);
                            const u64 X = (u64)p01 + ((u64)p23 << 16);
                            Dp[(size_t)k * N] = red32(mont_red64(X, a, RP.kq[k].y), a);
                        }
                    }
                }
            }
        } else {
        {
            const u64 rb = (u64)(rho + (1ll << 36));
            const u32 rlo = (u32)(rb & ((1u << 30) - 1)), rhi = (u32)(rb >> 30);
#pragma unroll
            for (int k0 = 0; k0 < RPT::MMAX; k0 += 4) {  // 4 MAC primes per TMEM load (warp-uniform)
                u32 Rc[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                    "%14, %15}, [%16];\n"
                    : "=r"(Rc[0]), "=r"(Rc[1]), "=r"(Rc[2]), "=r"(Rc[3]), "=r"(Rc[4]), "=r"(Rc[5]), "=r"(Rc[6]),
                      "=r"(Rc[7]), "=r"(Rc[8]), "=r"(Rc[9]), "=r"(Rc[10]), "=r"(Rc[11]), "=r"(Rc[12]), "=r"(Rc[13]),
                      "=r"(Rc[14]), "=r"(Rc[15])
                    : "r"(td + 4 * k0)
                    : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (!bad) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int k = k0 + kk;
                        if (k < RPT::MMAX && (MMT ? k < MMT : k < (int)Mm)) {
                            // S + gamma (-I_A) 2^32 + (rho + 2^36) 2^32 - 2^36 2^32 < 2^61, one Montgomery
                            // reduction: < 2^29 + 2^30 < 2 a_k
                            const u32 a = RP.kq[k].x;
                            const u32 p01 = Rc[4 * kk] + (Rc[4 * kk + 1] << 8), p23 = Rc[4 * kk + 2] + (Rc[4 * kk + 3] << 8);
                            u64 X = (u64)p01 + ((u64)p23 << 16) + RP.krm[k];
                            X += (u64)gamma * RP.kq[k].z;
                            X += (u64)rlo * RP.kc0[k];
                            X += (u64)rhi * RP.kc30[k];
                            Dp[(size_t)k * N] = red32(mont_red64(X, a, RP.kq[k].y), a);
                        }
                    }
                }
            }
        }
        }
        if (bad) {  // exact multiword path (no tensor-memory instructions inside); D still holds w_j
            HpsState h;
            for (u32 j = 0; j < J; ++j) h.w[j] = Dp[(size_t)j * N];
            h.gamma = gamma;
            h.rho = rho;
            u32 Rw[kAW + 2];
            const bool neg = round_exact(h, *T.self, Rw);
            for (u32 k = 0; k < Mm; ++k) {
                const u32 a = gRK[k].a;
                u32 r = mag_mod32(Rw, a, gRK[k].abar);
                if (neg && r) r = a - r;
                Dp[(size_t)k * N] = r;
            }
        }
        __syncwarp();
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(128));
}


// ---------------------------------------------------------------------------------------
// Centred lift chain -> aux basis on the tensor cores (to_aux_basis, bfv.cpp:718-744).
//
// x_j = (sum_i y_i (q / q_i mod a_j) - rho (q mod a_j)) mod a_j with y_i = res_i (q/q_i)^-1 mod q_i
// (< 2^60, 8 bytes) and rho = round(sum_i y_i / q_i) (crt_round: 64-bit fraction, exact fallback).
// The dot products over i are one int8 GEMM per 128 coefficients: A = the bytes of the L y_i
// (K = 64 bytes, from TMEM), B = byte b of (2^(8a) V_ij mod a_j) at column 4 j + b (shared memory,
// canonical K-major layout), so column group j sums to S_j = sum_b C 2^(8b) < 2^48 with
// S_j = sum_i y_i V_ij (mod a_j).  The epilogue adds rho (a_j - W_j) and reduces once per prime by a
// Montgomery step: V and (a_j - W_j) are stored with one more factor 2^32 (on top of the Montgomery
// (x 2^32) or plain lift constants of k_lift).
// ---------------------------------------------------------------------------------------
constexpr int kLiftK = 64;  // 8 chain primes x 8 bytes
template <int NC>
__global__ void __launch_bounds__(128, 4) k_lift_tc(const u64* __restrict__ src, size_t src_stride,
                                                   const u32* __restrict__ sel, u32 count, u32 nj, DevTab T,
                                                   const uint4* __restrict__ Bglob, const u32* __restrict__ Wj,
                                                   u32* __restrict__ out, u32 out_stride_j) {
    constexpr int K = kLiftK, KSTEPS = K / 32, ACOLS = K / 4;
    __shared__ __align__(128) uint4 Bs[NC * K / 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ u32 tmem_base_sh;
    __shared__ u32 sA[kMaxJ], sW[kMaxJ], sPi[kMaxJ];
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 N = T.N, L = T.L, logN = T.logN;  // N is a power of two: no 64-bit divisions
    for (u32 x = tid; x < NC * K / 16; x += blockDim.x) Bs[x] = Bglob[x];
    for (u32 j = tid; j < nj; j += blockDim.x) {
        sA[j] = T.a[j];
        sW[j] = Wj[j];      // (a_j - W_j) 2^32 mod a_j
        sPi[j] = T.apinv[j];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const u32 tbase = tmem_base_sh;
    const u32 ta = tbase + ((warp * 32u) << 16);  // A columns [0, 16), this warp's lanes
    const u32 td = ta + ACOLS;                    // D columns [16, 16 + NC)
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((K / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);  // D s32, A / B u8, M 128
    const size_t total = (size_t)count * 2 * N;
    u32 phase = 0;
    // the next tile's residues are loaded before this tile's GEMM round trip and epilogue (the
    // kernel is bound by the per-tile latency chain: 4 CTAs / SM by the TMEM allocation)
    u64 resn[kMaxL];
    auto fetch = [&](size_t base) {
        const size_t idx = base + tid;
#pragma unroll
        for (int i = 0; i < kMaxL; ++i) resn[i] = 0;
        if (idx < total) {
            const u32 c = (u32)(idx >> (logN + 1)), k = (u32)(idx >> logN) & 1u, n = (u32)(idx & (N - 1));
            const u64* s = src + (size_t)(sel ? sel[c] : c) * src_stride + (size_t)k * L * N + n;
#pragma unroll
            for (int i = 0; i < kMaxL; ++i)
                if (i < (int)L) resn[i] = s[(size_t)i * N];
        }
    };
    fetch((size_t)blockIdx.x * 128);
    for (size_t base = (size_t)blockIdx.x * 128; base < total; base += (size_t)gridDim.x * 128) {
        const size_t idx = base + tid;
        const bool live = idx < total;
        u32* o = nullptr;
        u32 rho = 0;
        u32 w[ACOLS];
#pragma unroll
        for (int x = 0; x < ACOLS; ++x) w[x] = 0;
        u64 res[kMaxL];
#pragma unroll
        for (int i = 0; i < kMaxL; ++i) res[i] = resn[i];
        if (base + (size_t)gridDim.x * 128 < total) fetch(base + (size_t)gridDim.x * 128);
        if (live) {
            const u32 c = (u32)(idx >> (logN + 1)), k = (u32)(idx >> logN) & 1u, n = (u32)(idx & (N - 1));
            u64 y[kMaxL];
            u32 ip;
            const u64 fr = crt_prepare(res, T, y, &ip);
            rho = crt_round(y, ip, fr, T);
#pragma unroll
            for (int i = 0; i < kMaxL; ++i) {
                if (i < (int)L) {
                    w[2 * i] = (u32)y[i];
                    w[2 * i + 1] = (u32)(y[i] >> 32);
                }
            }
            o = out + ((size_t)c * 2 + k) * out_stride_j * N + n;
        }
#pragma unroll
        for (int x = 0; x < ACOLS; x += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + x),
                         "r"(w[x]), "r"(w[x + 1]), "r"(w[x + 2]), "r"(w[x + 3]), "r"(w[x + 4]), "r"(w[x + 5]),
                         "r"(w[x + 6]), "r"(w[x + 7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int st = 0; st < KSTEPS; ++st) {
                const u64 bd = bdesc0 + (u64)((st * 2 * 128) >> 4);  // 2 K chunks of 16 B per step
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + ACOLS),
                    "r"(tbase + (u32)(st * 8)), "l"(bd), "r"(idesc), "r"(st)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        mbar_wait_sleep(&mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
        for (int j0 = 0; j0 < NC / 4; j0 += 4) {  // 4 primes (16 columns) per TMEM load
            u32 C[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                "%14, %15}, [%16];\n"
                : "=r"(C[0]), "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]),
                  "=r"(C[8]), "=r"(C[9]), "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15])
                : "r"(td + 4 * j0)
                : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (o) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const u32 j = j0 + jj;
                    if (j < nj) {
                        const u32 a = sA[j];
                        // the constants carry one more factor 2^32: S < 2^48 + 2^34 a, one Montgomery step
                        // (x 2^-32) leaves the residue in [0, 2a)
                        const u64 S = (u64)C[4 * jj] + ((u64)C[4 * jj + 1] << 8) + ((u64)C[4 * jj + 2] << 16) +
                                      ((u64)C[4 * jj + 3] << 24) + (u64)rho * sW[j];
                        o[(size_t)j * N] = red32(mont_red64(S, a, sPi[j]), a);
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // D and A are rewritten by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(128));
}

// ---------------------------------------------------------------------------------------
// MAC basis -> chain on the tensor cores (the exact centred base conversion of k_mac_to_chain).
//
// out_i = (sum_k v_k (M/a_k mod q_i) + gamma (-M mod q_i)) mod q_i with v_k = x_k (M/a_k)^-1 mod a_k
// and gamma = round(sum_k v_k / a_k) (|X| < M/2 (1 - 2^-20): the 64-bit estimate decides).  The
// Mm x L dot products are one int8 GEMM per 128 coefficients: A = the bytes of the v_k (K = 4 KW
// bytes, from TMEM), B = byte b of (2^(8a) (M/a_k) mod q_i) at column 8 i + b, K byte 4 k + a, so
// column group i sums to S_i = sum_b C_b 2^(8b) < 2^80 with S_i = sum_k v_k (M/a_k) (mod q_i); the
// epilogue adds the gamma term and reduces once per chain prime (reduce96).  The CUDA-core kernel
// spends ~4,800 instructions per coefficient at C5 (Mm = 17, L = 8) on the same sums.
// X layout [G][xs][N] (the first Mm planes of each group of xs); out layout [G][L][N].
// ---------------------------------------------------------------------------------------
// NC = 48 (L <= 6) keeps A + D within a 64-column TMEM allocation: 6 CTAs per SM instead of 4 (the
// kernel is bound by the per-tile latency chain).
template <int KW, int NC = 64>  // A words per coefficient (Mm <= KW, KW a multiple of 8); D columns 8 L <= NC
__global__ void __launch_bounds__(128, (KW + NC <= 64) ? 6 : 4) k_mac_to_chain_tc(const u32* __restrict__ X, u32 xs, u32 G, DevTab T,
                                                           const uint4* __restrict__ Bglob, u64* __restrict__ out) {
    constexpr int K = 4 * KW, KSTEPS = K / 32;
    constexpr int TCOLS = (KW + NC <= 64) ? 64 : 128;  // TMEM allocation (power of two)
    __shared__ __align__(128) uint4 Bs[NC * K / 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ u32 tmem_base_sh;
    __shared__ u32 sA[KW], sH[KW], sHs[KW];
    __shared__ u64 sMF[KW], sQ[kMaxL], sMu[kMaxL], sNeg[kMaxL];
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 N = T.N, L = T.L, Mm = T.Mm, logN = T.logN;
    for (u32 x = tid; x < NC * K / 16; x += blockDim.x) Bs[x] = Bglob[x];
    for (u32 k = tid; k < (u32)KW; k += blockDim.x) {
        const bool on = k < Mm;
        sA[k] = on ? T.a[k] : 1u;  // padded primes: v = 0
        sH[k] = on ? T.mhat[k] : 0u;
        sHs[k] = on ? T.mhat_s[k] : 0u;
        sMF[k] = on ? T.mF[k] : 0ull;
    }
    for (u32 i = tid; i < L; i += blockDim.x) {
        sQ[i] = T.q[i];
        sMu[i] = T.q_mu96[i];
        sNeg[i] = T.MnegQ[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const u32 tbase = tmem_base_sh;
    const u32 ta = tbase + ((warp * 32u) << 16);  // A columns [0, KW), this warp's lanes
    const u32 td = ta + KW;                       // D columns [KW, KW + 64)
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((K / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);  // D s32, A / B u8, M 128
    const u32 gsh = 64 - T.gbits;
    const size_t total = (size_t)G * N;
    u32 phase = 0;
    // the next tile's residues are loaded before this tile's GEMM round trip and epilogue (the
    // kernel is bound by the per-tile latency chain: 4 CTAs / SM by the TMEM allocation)
    u32 xn[KW];
    auto fetch = [&](size_t base) {
        const size_t idx = base + tid;
        const bool live = idx < total;
        const size_t g = live ? idx >> logN : 0;  // N is a power of two: no 64-bit divisions
        const u32 n = live ? (u32)(idx & (N - 1)) : 0;
#pragma unroll
        for (int k = 0; k < KW; ++k) xn[k] = (live && k < (int)Mm) ? __ldg(X + (g * xs + k) * N + n) : 0u;
    };
    fetch((size_t)blockIdx.x * 128);
    for (size_t base = (size_t)blockIdx.x * 128; base < total; base += (size_t)gridDim.x * 128) {
        const size_t idx = base + tid;
        const bool live = idx < total;
        const size_t g = live ? idx >> logN : 0;
        const u32 n = live ? (u32)(idx & (N - 1)) : 0;
        u32 v[KW];
#pragma unroll
        for (int k = 0; k < KW; ++k) v[k] = red32(shoup32(xn[k], sH[k], sHs[k], sA[k]), sA[k]);
        if (base + (size_t)gridDim.x * 128 < total) fetch(base + (size_t)gridDim.x * 128);
        u64 gs = 0;
#pragma unroll
        for (int k = 0; k < KW; ++k) gs += (u64)v[k] * sMF[k];
        const u32 gamma = (u32)((gs + (1ull << (gsh - 1))) >> gsh);
#pragma unroll
        for (int x = 0; x < KW; x += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + x),
                         "r"(v[x]), "r"(v[x + 1]), "r"(v[x + 2]), "r"(v[x + 3]), "r"(v[x + 4]), "r"(v[x + 5]),
                         "r"(v[x + 6]), "r"(v[x + 7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int st = 0; st < KSTEPS; ++st) {
                const u64 bd = bdesc0 + (u64)((st * 2 * 128) >> 4);  // 2 K chunks of 16 B per step
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + KW),
                    "r"(tbase + (u32)(st * 8)), "l"(bd), "r"(idesc), "r"(st)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        mbar_wait_sleep(&mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
        for (int i0 = 0; i0 < kMaxL; i0 += 2) {  // 2 chain primes (16 columns) per TMEM load
            if (i0 >= (int)L || 8 * i0 >= NC) break;  // warp-uniform
            u32 C[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
                "%15}, [%16];\n"
                : "=r"(C[0]), "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]),
                  "=r"(C[8]), "=r"(C[9]), "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15])
                : "r"(td + 8 * i0)
                : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (live) {
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) {
                    const u32 i = i0 + ii;
                    if (i < L) {
                        const u32* c = C + 8 * ii;
                        const u64 P = (u64)c[0] + ((u64)c[1] << 8) + ((u64)c[2] << 16) + ((u64)c[3] << 24);
                        const u64 Q = (u64)c[4] + ((u64)c[5] << 8) + ((u64)c[6] << 16) + ((u64)c[7] << 24);
                        u64 lo = P + (Q << 32);
                        u64 hi = (Q >> 32) + (lo < P ? 1u : 0u);
                        mac128(hi, lo, (u64)gamma, sNeg[i]);  // < 2^80 + 2^65
                        out[(g * L + i) * N + n] = reduce96((u32)hi, lo, sQ[i], sMu[i]);
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // D and A are rewritten by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(TCOLS));
}

// ---------------------------------------------------------------------------------------
// Digit decomposition on the tensor cores (decompose_digits, bfv.cpp:316-339, 16-bit digits written
// as key-switch aux residues): the exact CRT x = sum_i y_i (q/q_i) - alpha q in positional form.
//
// The L x QW limb products of crt_exact_cols are one int8 GEMM per 128 coefficients: A = the bytes
// of the y_i (K = 64, from TMEM), B[8 i + a][s] = byte s - a of q / q_i, so column s is the base-256
// column sum of sum_i y_i (q/q_i) (< 64 255^2 < 2^22); the epilogue carries the 64 columns into
// 32-bit limbs, subtracts alpha q with one correction (as crt_exact_cols) and cuts the digits.
// The CUDA-core kernel issues ~4,700 instructions per coefficient at C5 (unrolled limb products,
// instruction-cache misses).  Requires 4 QW + 7 < 64 (q below 448 bits).
// ---------------------------------------------------------------------------------------
template <int QWT>  // 32-bit limbs of q (T.QW <= QWT <= 14): the carry / subtract / compare loops stop there
__global__ void __launch_bounds__(128, 4) k_decompose_tc(const u64* __restrict__ polys, size_t stride, u64 ginv, u32 B,
                                                        u32 D, DevTab T, const uint4* __restrict__ Bglob,
                                                        u32* __restrict__ aux_out, u32 K) {
    constexpr int KB = 64, KSTEPS = KB / 32, ACOLS = KB / 4, NC = 64;
    __shared__ __align__(128) uint4 Bs[NC * KB / 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ u32 tmem_base_sh;
    constexpr int SW = QWT + 2;  // limbs of the column sums (sum_i y_i q/q_i < 2^61 q 2^3)
    constexpr int NCU = (4 * SW + 15) / 16 * 16 < NC ? (4 * SW + 15) / 16 * 16 : NC;  // columns that can be non-zero
    __shared__ u32 sqw[kQW];
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 N = T.N, L = T.L, QW = T.QW, logN = T.logN;
    for (u32 x = tid; x < NC * KB / 16; x += blockDim.x) Bs[x] = Bglob[x];
    for (u32 x = tid; x < (u32)kQW; x += blockDim.x) sqw[x] = x < QW ? T.qw[x] : 0u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const u32 tbase = tmem_base_sh;
    const u32 ta = tbase + ((warp * 32u) << 16);  // A columns [0, 16), this warp's lanes
    const u32 td = ta + ACOLS;                    // D columns [16, 80)
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((KB / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);  // D s32, A / B u8, M 128
    const size_t total = (size_t)B * N;
    u32 phase = 0;
    // the next tile's residues are loaded before this tile's GEMM round trip and epilogue
    u64 resn[kMaxL];
    auto fetch = [&](size_t base) {
        const size_t idx = base + tid;
        const bool live = idx < total;
        const u32 b = live ? (u32)(idx >> logN) : 0, n = live ? (u32)(idx & (N - 1)) : 0;
        const u64* pb = polys + (size_t)b * stride;
        u32 src = n;
        bool neg = false;
        if (ginv) {
            const u32 sidx = (u32)(((u64)n * ginv) & (2 * N - 1));
            neg = sidx >= N;
            src = neg ? sidx - N : sidx;
        }
#pragma unroll
        for (int i = 0; i < kMaxL; ++i) {
            resn[i] = 0;
            if (live && i < (int)L) {
                u64 v = pb[(size_t)i * N + src];
                if (neg && v) v = T.q[i] - v;
                resn[i] = v;
            }
        }
    };
    fetch((size_t)blockIdx.x * 128);
    for (size_t base = (size_t)blockIdx.x * 128; base < total; base += (size_t)gridDim.x * 128) {
        const size_t idx = base + tid;
        const bool live = idx < total;
        const u32 b = live ? (u32)(idx >> logN) : 0, n = live ? (u32)(idx & (N - 1)) : 0;
        u32 w[ACOLS];
        u32 alpha = 0;
        {
            u64 res[kMaxL], y[kMaxL];
#pragma unroll
            for (int i = 0; i < kMaxL; ++i) res[i] = resn[i];
            if (base + (size_t)gridDim.x * 128 < total) fetch(base + (size_t)gridDim.x * 128);
            crt_prepare(res, T, y, &alpha);
#pragma unroll
            for (int i = 0; i < kMaxL; ++i) {
                w[2 * i] = i < (int)L ? (u32)y[i] : 0u;
                w[2 * i + 1] = i < (int)L ? (u32)(y[i] >> 32) : 0u;
            }
        }
#pragma unroll
        for (int x = 0; x < ACOLS; x += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + x),
                         "r"(w[x]), "r"(w[x + 1]), "r"(w[x + 2]), "r"(w[x + 3]), "r"(w[x + 4]), "r"(w[x + 5]),
                         "r"(w[x + 6]), "r"(w[x + 7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int st = 0; st < KSTEPS; ++st) {
                const u64 bd = bdesc0 + (u64)((st * 2 * 128) >> 4);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + ACOLS),
                    "r"(tbase + (u32)(st * 8)), "l"(bd), "r"(idesc), "r"(st)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        mbar_wait_sleep(&mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // column sums -> carried 32-bit limbs S (16 limbs from the 64 columns, the carry in limb 16)
        u32 S[SW];
        u64 carry = 0;
#pragma unroll
        for (int c0 = 0; c0 < NCU; c0 += 16) {
            u32 C[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
                "%15}, [%16];\n"
                : "=r"(C[0]), "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]),
                  "=r"(C[8]), "=r"(C[9]), "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15])
                : "r"(td + c0)
                : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                if (c0 / 4 + l < SW) {
                    const u64 s = carry + (u64)C[4 * l] + ((u64)C[4 * l + 1] << 8) + ((u64)C[4 * l + 2] << 16) +
                                  ((u64)C[4 * l + 3] << 24);
                    S[c0 / 4 + l] = (u32)s;
                    carry = s >> 32;
                }
            }
        }
        // X = S - alpha q (alpha: the fractional estimate, short by at most one) and one correction
        u32 X[SW];
        {
            u64 c = 0;
            u32 bb = 0;
#pragma unroll
            for (int x = 0; x < SW; ++x) {
                const u64 pk = (x < QWT ? (u64)alpha * sqw[x] : 0) + c;
                c = pk >> 32;
                const u32 pl = (u32)pk, sx = S[x];
                const u32 r1 = sx - pl, b1 = sx < pl;
                const u32 r2 = r1 - bb, b2 = r1 < bb;
                X[x] = r2;
                bb = b1 | b2;
            }
            int ge = 1;
#pragma unroll
            for (int x = SW - 1; x >= 0; --x) {
                const u32 qv = x < QWT ? sqw[x] : 0u;
                if (ge == 1 && X[x] != qv) ge = X[x] > qv ? 2 : 0;
            }
            if (ge != 0) {
                u32 b2 = 0;
#pragma unroll
                for (int x = 0; x < SW; ++x) {
                    const u32 qv = x < QWT ? sqw[x] : 0u;
                    const u32 r1 = X[x] - qv, c1 = X[x] < qv;
                    const u32 r2 = r1 - b2, c2 = r1 < b2;
                    X[x] = r2;
                    b2 = c1 | c2;
                }
            }
        }
        if (live) {
            u32* o = aux_out + (size_t)b * D * K * N + n;
#pragma unroll
            for (int d = 0; d < 2 * QWT; ++d) {
                if (d < (int)D) {
                    const u32 v = (X[d >> 1] >> (16 * (d & 1))) & 0xffffu;
                    for (u32 j = 0; j < K; ++j) o[((size_t)d * K + j) * N] = v;  // digits < 2^16 < a_j
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // D and A are rewritten by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(128));
}

}  // namespace cwgpu

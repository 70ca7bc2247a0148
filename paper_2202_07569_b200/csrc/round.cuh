// Exact BFV scale-and-round t*D/q (bfv.cpp:811-849) of the tensor product, split across the
// integer (IMAD) and FP64 (DFMA) pipes of a B200 SM.
//
// Same HPS decomposition as k_round_mac_t (ntt_reg.cuh):
//   w_j = D_j (A/a_j)^-1 mod a_j,   gamma = round(sum_j w_j / a_j),
//   r = sum_j w_j I_j - gamma I_A + rho,   rho = round(sum_j w_j F_j - gamma F_A),
// with t (A/a_j) = (I_j + F_j) q.  The result is needed mod each MAC prime a_k (k < Mm).
// The Mm x J dot products sum_j w_j (I_j mod a_k) are ~45% of the IMAD-pipe work of the
// integer-only kernel (IMAD.WIDE costs 2.4 IMAD slots on B200); the FP64 pipe runs DFMA at
// the IMAD rate (measured 60 lanes/clk/SM each, 112 combined), so:
//   * integer pipe: w_j (Shoup), the 96-bit fixed-point fraction rho, and the first MI
//     MAC primes (Montgomery dot products, as k_round_mac_t);
//   * FP64 pipe: gamma = rint(sum_j w_j (1/a_j)) and the remaining MAC primes, each as two
//     exact DFMA dot products on a 15-bit split I = Ihi 2^15 + Ilo (every partial sum is an
//     integer < 2^51, so the doubles are exact), reduced mod a_k with rint-by-magic-constant
//     quotients and read back through the 2^52 mantissa trick (no F2I / I2F conversions).
// All per-prime constants travel in the kernel-parameter constant bank (RoundPar), so the
// unrolled loops take them as instruction operands instead of shared-memory loads.
#pragma once
#include "kernels.cuh"
#include "ntt_reg.cuh"
#include "mac.cuh"

namespace cwgpu {

template <int JM>
struct RoundPar {
    static constexpr int MI = JM / 4;  // MAC primes reduced on the integer pipe
    // per aux prime j (padded: a = 1, everything else 0 -> w_j = 0)
    u32 a[JM], chat[JM], chat_s[JM], f0[JM], f1[JM];
    double inva_j[JM];
    // integer-pipe MAC primes k < MI (Montgomery forms, as RoundK)
    u32 ka[MI], kpinv[MI], kgcoef[MI], kroff[MI], kc0[MI], kc30[MI];
    u32 ImodT[MI][JM];
    // FP64-pipe MAC primes k >= MI: I_kj = Ihi 2^15 + Ilo, -I_A = nIAhi 2^15 + nIAlo (mod a_k);
    // processed in unguarded groups of 4 (KP = JM + 4 entries, padding a = 1)
    static constexpr int KP = JM + 4;
    u32 fa[KP];
    double Ilo[KP][JM], Ihi[KP][JM];
    double nIAlo[KP], nIAhi[KP], roff[KP], ad[KP], inva[KP], off2a[KP];
};

__device__ __forceinline__ double u32_to_f64(u32 x) {  // exact, FP64 pipe only
    return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}
__device__ __forceinline__ double rint_f64(double x) {  // |x| < 2^51, round half even
    return (x + 6755399441055744.0) - 6755399441055744.0;
}
__device__ __forceinline__ double rint_fma(double x, double y) {  // rint(x * y)
    return fma(x, y, 6755399441055744.0) - 6755399441055744.0;
}

/// D planes: D[pc][j][N] for pc < P*3; writes r mod a_k (k < Mm) in place.
template <int JM>
__global__ void __launch_bounds__(256, JM >= 32 ? 1 : 2) k_round_hyb(u32* __restrict__ D, u32 P, DevTab T,
                                                     const __grid_constant__ RoundPar<JM> RP,
                                                     const RoundK* __restrict__ gRK) {
    constexpr int MI = RoundPar<JM>::MI;
    const u32 J = T.J, Mm = T.Mm, N = T.N, logN = T.logN;
    const u32 fA0 = T.fracA[1], fA1 = T.fracA[2];  // 64-bit fraction of t A / q
    const size_t total = (size_t)P * 3 * N;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t pc = idx >> logN;
        const u32 n = (u32)(idx & (N - 1));
        u32* Dp = D + pc * T.DS * N + n;
        u32 d[JM];
#pragma unroll
        for (int j = 0; j < JM; ++j) d[j] = Dp[(size_t)min(j, (int)J - 1) * N];  // padded j: any value (w_j = 0)
#pragma unroll
        for (int j = 0; j < JM; ++j) asm volatile("" : "+r"(d[j]));  // all plane loads in flight before any use
        u32 w[JM];
        double wd[JM];
        double gsum = 0.0;
        u32 s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
        for (int j = 0; j < JM; ++j) {
            const u32 wj = red32(shoup32(d[j], RP.chat[j], RP.chat_s[j], RP.a[j]), RP.a[j]);
            w[j] = wj;
            wd[j] = u32_to_f64(wj);
            gsum = fma(wd[j], RP.inva_j[j], gsum);
            asm("mad.lo.cc.u32  %0, %4, %5, %0;\n\t"
                "madc.lo.cc.u32 %1, %4, %6, %1;\n\t"
                "addc.cc.u32    %2, %2, 0;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                "mad.hi.cc.u32  %1, %4, %5, %1;\n\t"
                "madc.hi.cc.u32 %2, %4, %6, %2;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3)
                : "r"(wj), "r"(RP.f0[j]), "r"(RP.f1[j]));
        }
        // sum_j w_j / a_j lies within 2^-7 of an integer (|D| < A / 2^7): any rounding of the
        // double sum gives the centred-lift gamma
        const double gd = rint_f64(gsum);
        const u32 gamma = (u32)__double2loint(gd + 4503599627370496.0);
        {
            // subtract gamma * F_A (64-bit fraction) and add 1/2
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
        // true - estimate in (-gamma, J 2^30) units of 2^-64: undecidable near a wrap
        const bool bad = (s1 == 0u && s0 < 64u) || (s1 >= 0xfffffff0u) || T.force_exact;
        if (!bad) {
            const u64 rb = (u64)(rho + (1ll << 36));  // >= 0, < 2^37
            const u32 rlo = (u32)(rb & ((1u << 30) - 1)), rhi = (u32)(rb >> 30);
            // integer pipe: k < MI, pairs of primes (independent accumulation chains)
#pragma unroll
            for (int k0 = 0; k0 < MI; k0 += 2) {
                if (k0 >= (int)Mm) break;
                u32 r[2];
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const int k = k0 + kk;
                    u64 g0 = (u64)gamma * RP.kgcoef[k] + (u64)rlo * RP.kc0[k] + (u64)rhi * RP.kc30[k] + RP.kroff[k];
                    r[kk] = 0;
#pragma unroll
                    for (int gb = 0; gb < JM; gb += 8) {
                        u64 g = gb == 0 ? g0 : 0;
#pragma unroll
                        for (int j = gb; j < gb + 8; ++j) g += (u64)w[j] * RP.ImodT[k][j];
                        u32 x = mont_red64(g, RP.ka[k], RP.kpinv[k]);  // [0, 3a)
                        x = red32(red32(x, 2 * RP.ka[k]), RP.ka[k]);
                        r[kk] = red32(r[kk] + x, RP.ka[k]);
                    }
                }
                Dp[(size_t)k0 * N] = r[0];
                if (k0 + 1 < (int)Mm) Dp[(size_t)(k0 + 1) * N] = r[1];
            }
            // FP64 pipe: MI <= k < Mm in groups of 4 primes, 4 accumulation chains per prime
            const double rr = u32_to_f64(rlo) + 1073741824.0 * u32_to_f64(rhi);  // rho + 2^36, exact
#pragma unroll
            for (int k0 = MI; k0 < JM; k0 += 4) {
                if (k0 >= (int)Mm) break;
                u32 x[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int k = k0 + kk;
                    double lo0 = fma(gd, RP.nIAlo[k], rr + RP.roff[k]), lo1 = 0.0;
                    double hi0 = gd * RP.nIAhi[k], hi1 = 0.0;
#pragma unroll
                    for (int j = 0; j < JM; j += 2) {
                        lo0 = fma(wd[j], RP.Ilo[k][j], lo0);
                        hi0 = fma(wd[j], RP.Ihi[k][j], hi0);
                        lo1 = fma(wd[j + 1], RP.Ilo[k][j + 1], lo1);
                        hi1 = fma(wd[j + 1], RP.Ihi[k][j + 1], hi1);
                    }
                    const double lo = lo0 + lo1, hi = hi0 + hi1;                      // exact integers < 2^51
                    const double rh = fma(-rint_fma(hi, RP.inva[k]), RP.ad[k], hi);  // |rh| < 1.5 a
                    const double t = fma(rh, 32768.0, lo);                            // exact, < 2^51
                    const double r = fma(-rint_fma(t, RP.inva[k]), RP.ad[k], t);      // |r| < 1.5 a
                    x[kk] = (u32)__double2loint(r + RP.off2a[k]);                     // r + 2a in [0, 4a)
                    x[kk] = red32(red32(x[kk], 2 * RP.fa[k]), RP.fa[k]);
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (k0 + kk < (int)Mm) Dp[(size_t)(k0 + kk) * N] = x[kk];
            }
        } else {
            HpsState h;
#pragma unroll
            for (int j = 0; j < JM; ++j) if (j < (int)J) h.w[j] = w[j];
            h.gamma = gamma;
            h.rho = rho;
            u32 R[kAW + 2];
            const bool neg = round_exact(h, *T.self, R);
            for (u32 k = 0; k < Mm; ++k) {
                const u32 a = gRK[k].a;
                u32 r = mag_mod32(R, a, gRK[k].abar);
                if (neg && r) r = a - r;
                Dp[(size_t)k * N] = r;
            }
        }
    }
}

}  // namespace cwgpu

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

// TMEM budget: <= 4 resident CTAs x 128 columns.  The register file already caps residency at 4
// (>= 122 registers x 128 threads), so no shared-memory padding is requested (padding would keep
// the NTT kernels of the other tile stream off the SM).
constexpr size_t kRoundTcSmem = 0;

template <int JM, int NC>
__global__ void __launch_bounds__(128, 4) k_round_tc(u32* __restrict__ D, u32 P, DevTab T,
                                                    const __grid_constant__ RoundTcPar<JM, NC> RP,
                                                    const uint4* __restrict__ Bglob, const RoundK* __restrict__ gRK) {
    using RPT = RoundTcPar<JM, NC>;
    constexpr int K = RPT::K, F0 = RPT::F0, G0 = RPT::G0;
    constexpr int KSTEPS = K / 32;
    constexpr u32 TCOLS = (JM + NC) <= 32 ? 32 : (JM + NC) <= 64 ? 64 : (JM + NC) <= 128 ? 128 : 256;
    __shared__ __align__(128) uint4 Bs[NC * K / 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ u32 tmem_base_sh;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 J = T.J, Mm = T.Mm, N = T.N, logN = T.logN;

    for (u32 x = tid; x < NC * K / 16; x += blockDim.x) Bs[x] = Bglob[x];
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
    const u32 ta = tbase + ((warp * 32u) << 16);           // A columns [0, JM), this warp's lanes
    const u32 td = tbase + ((warp * 32u) << 16) + JM;      // D columns [JM, JM + NC)
    // smem descriptor, K-major, no swizzle: core matrix 8 rows x 16 B; LBO = next 16-B K chunk
    // (128 B), SBO = next 8-row group (K / 16 chunks * 128 B); version 1 (sm_100)
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((K / 16 * 128) >> 4) << 32) | (1ull << 46);
    // instruction descriptor: D s32, A / B u8, K-major both, N = NC, M = 128
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);
    const u32 fA0 = T.fracA[1], fA1 = T.fracA[2];
    const size_t total = (size_t)P * 3 * N;
    u32 phase = 0;
    for (size_t base = (size_t)blockIdx.x * 128; base < total; base += (size_t)gridDim.x * 128) {
        const size_t idx = base + tid;
        const size_t pc = idx >> logN;
        const u32 n = (u32)(idx & (N - 1));
        u32* Dp = D + pc * T.DS * N + n;
        u32 w[JM];
#pragma unroll
        for (int j = 0; j < JM; ++j) w[j] = j < (int)J ? Dp[(size_t)j * N] : 0u;
        // A tile: this thread's row
#pragma unroll
        for (int c = 0; c < JM; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + c),
                         "r"(w[c]), "r"(w[c + 1]), "r"(w[c + 2]), "r"(w[c + 3]), "r"(w[c + 4]), "r"(w[c + 5]),
                         "r"(w[c + 6]), "r"(w[c + 7])
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const u64 bd = bdesc0 + (u64)((s * 2 * 128) >> 4);  // 2 K chunks per step
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
        {
            u32 done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                    : "=r"(done)
                    : "r"(smem_u32(&mbar)), "r"(phase)
                    : "memory");
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        u32 C[NC];
#pragma unroll
        for (int c = 0; c < NC; c += 16)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
                "%15}, [%16];\n"
                : "=r"(C[c]), "=r"(C[c + 1]), "=r"(C[c + 2]), "=r"(C[c + 3]), "=r"(C[c + 4]), "=r"(C[c + 5]),
                  "=r"(C[c + 6]), "=r"(C[c + 7]), "=r"(C[c + 8]), "=r"(C[c + 9]), "=r"(C[c + 10]), "=r"(C[c + 11]),
                  "=r"(C[c + 12]), "=r"(C[c + 13]), "=r"(C[c + 14]), "=r"(C[c + 15])
                : "r"(td + c)
                : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");

        // gamma = round(sum_j w_j / a_j)
        u64 gs = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) gs += (u64)C[G0 + s] << (8 * s);
        const u32 gamma = (u32)((gs + (1ull << 45)) >> 46);
        // FR = sum_j w_j F_j (96-bit, units 2^-64) = plo + phi 2^48
        u64 plo = 0, phi = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) plo += (u64)C[F0 + s] << (8 * s);
#pragma unroll
        for (int s = 6; s < 11; ++s) phi += (u64)C[F0 + s] << (8 * (s - 6));
        const u64 lo64 = plo + (phi << 48);
        const u64 hi64 = (phi >> 16) + (lo64 < plo ? 1u : 0u);
        u32 s0 = (u32)lo64, s1 = (u32)(lo64 >> 32), s2 = (u32)hi64, s3 = (u32)(hi64 >> 32);
        {
            // subtract gamma * F_A (64-bit fraction) and add 1/2
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
        if (!bad) {
            const u64 rb = (u64)(rho + (1ll << 36));  // >= 0, < 2^37
            const u32 rlo = (u32)(rb & ((1u << 30) - 1)), rhi = (u32)(rb >> 30);
#pragma unroll
            for (int k = 0; k < RPT::MMAX; ++k) {
                if (k < (int)Mm) {
                    const uint4 q = RP.kq[k];  // a, pinv, Montgomery(-I_A), 2^30 - a
                    // S = sum_b C[4k+b] 2^(8b) < 2^47 from two 32-bit pair sums (column sums < 2^23)
                    const u32 p01 = C[4 * k] + (C[4 * k + 1] << 8), p23 = C[4 * k + 2] + (C[4 * k + 3] << 8);
                    const u64 S = (u64)p01 + ((u64)p23 << 16);
                    // Montgomery part: (S + gamma (-I_A) 2^32 - 2^36 2^32) 2^-32 mod a
                    const u64 X = (u64)gamma * q.z + S + RP.krm[k];
                    const u32 x = red32(mont_red64(X, q.x, q.y), q.x);  // < 2a before the reduction
                    // + (rho + 2^36) mod a, with 2^30 = a + (2^30 - a)
                    const u32 y = red32(red32(rlo + rhi * q.w, 2 * q.x), q.x);  // < 2^30 + 2^31 < 4a
                    Dp[(size_t)k * N] = red32(x + y, q.x);
                }
            }
        } else {
            HpsState h;
#pragma unroll
            for (int j = 0; j < JM; ++j) if (j < (int)J) h.w[j] = w[j];
            h.gamma = gamma;
            h.rho = rho;
            u32 R[kAW + 2];
            const bool neg = round_exact(h, *T.self, R);
            for (u32 k = 0; k < Mm; ++k) {
                const u32 a = gRK[k].a;
                u32 r = mag_mod32(R, a, gRK[k].abar);
                if (neg && r) r = a - r;
                Dp[(size_t)k * N] = r;
            }
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(TCOLS));
}

}  // namespace cwgpu

namespace cwgpu {

// ---------------------------------------------------------------------------------------
// TMA-fed variant of k_round_tc.  The plane loads of k_round_tc are issued by the same threads
// that then wait for the MMA and run the epilogue, so at most one 128-coefficient tile per CTA
// is in flight and the kernel is latency-bound (ncu: long-scoreboard stalls, ~45% of HBM).
// Here a producer warp streams each tile's J plane segments (512 B each, contiguous) into a
// kRtStages-deep shared-memory ring with cp.async.bulk, completing on a `full` mbarrier; the 4
// consumer warps read their coefficient's J words from the ring (conflict-free), release the
// stage, and run the tensor-core rounding and epilogue exactly as k_round_tc, writing the Mm
// MAC-basis residues in place.  Persistent: CTA b handles tiles b, b + grid, ...
// ---------------------------------------------------------------------------------------
constexpr int kRtStages = 4;
template <int JM>
constexpr size_t round_tma_smem() { return (size_t)kRtStages * JM * 128 * 4; }

template <int LOGN, int JM, int NC, int MMT = 0>  // LOGN = 0: N at run time; MMT = 0: Mm at run time
__global__ void __launch_bounds__(160, 4) k_round_tma(u32* __restrict__ D, u32 P, DevTab T,
                                                     const __grid_constant__ RoundTcPar<JM, NC> RP,
                                                     const uint4* __restrict__ Bglob, const RoundK* __restrict__ gRK,
                                                     const uint4* __restrict__ B2glob) {
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
                const u32* src = D + pc * T.DS * N + n0;
                for (u32 j = 0; j < J; ++j) tma_bulk_g2s(&ring[st][j][0], src + (size_t)j * N, 512u, &full[st]);
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

}  // namespace cwgpu

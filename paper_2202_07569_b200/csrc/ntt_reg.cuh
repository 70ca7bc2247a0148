// Register-resident negacyclic NTT for the 31-bit aux / MAC primes.
//
// Same transform as RingContext::ntt_forward / ntt_inverse (reference ring.cpp:78-144):
// forward Cooley-Tukey, natural order in, bit-reversed out, twiddle root_pow[m + i]
// for block i of stage m; inverse Gentleman-Sande back to natural order.
//
// A CTA of T = N/16 threads owns one polynomial; each thread keeps 16 coefficients in
// registers.  The log2(N) stages are processed in 4-bit windows: within a window the
// thread's 16 registers span the window's 4 index bits, so all of the window's
// butterflies are register-local; between windows the polynomial is transposed through
// shared memory (padded by one word per 16 to avoid bank conflicts).  Twiddles for a
// window stage are contiguous in the bit-reversed tables and are fetched with vector
// loads where 4 or more are needed.
#pragma once
#include "devtab.h"
#include "modarith.cuh"

namespace cwgpu {

// one pad word per 16: conflict-free (<= 1 collision per warp) for every window mapping
__device__ __forceinline__ u32 pidx(u32 x) { return x + (x >> 4); }

template <int LOGN>
struct NttGeom {
    static constexpr int N = 1 << LOGN;
    static constexpr int T = N / 16;
    static constexpr int NW = (LOGN + 3) / 4;       // windows
    static constexpr int SMEM = N + N / 16 + 8;     // padded u32 words
};

/// window w (low bit) mapping: x = (tid >> w) << (w + 4) | r << w | (tid & (2^w - 1))
__device__ __forceinline__ u32 win_index(u32 tid, int w, int r) {
    const u32 low = tid & ((1u << w) - 1u);
    const u32 high = tid >> w;
    return (high << (w + 4)) | ((u32)r << w) | low;
}

/// Load `cnt` consecutive twiddles (and Shoup companions) starting at base (cnt <= 8).
template <int CNT>
__device__ __forceinline__ void load_tw(const u32* __restrict__ tp, const u32* __restrict__ tsp, u32 base, u32* w,
                                        u32* ws) {
    if constexpr (CNT >= 4) {
#pragma unroll
        for (int u = 0; u < CNT; u += 4) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(tp + base + u));
            const uint4 b = __ldg(reinterpret_cast<const uint4*>(tsp + base + u));
            w[u] = a.x; w[u + 1] = a.y; w[u + 2] = a.z; w[u + 3] = a.w;
            ws[u] = b.x; ws[u + 1] = b.y; ws[u + 2] = b.z; ws[u + 3] = b.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < CNT; ++u) {
            w[u] = __ldg(tp + base + u);
            ws[u] = __ldg(tsp + base + u);
        }
    }
}

/// Forward NTT of NP polynomials (same prime) held in v (input mapping: window 0, i.e.
/// x = r << (LOGN-4) | tid; output mapping: last window, x = tid << 4 | r).
/// Values in [0, 4p) in and out (p < 2^30).  sm: NP * NttGeom<LOGN>::SMEM words.
template <int LOGN, int NP>
__device__ __forceinline__ void ntt32_fwd_reg(u32 (&v)[NP][16], u32* sm, const u32* __restrict__ rp,
                                              const u32* __restrict__ rps, u32 p) {
    using G = NttGeom<LOGN>;
    const u32 tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < G::NW; ++k) {
        const int w = (LOGN - 4 - 4 * k) > 0 ? (LOGN - 4 - 4 * k) : 0;
        const int btop = LOGN - 1 - 4 * k;
        if (k > 0) {
            const int wp = (LOGN - 4 - 4 * (k - 1)) > 0 ? (LOGN - 4 - 4 * (k - 1)) : 0;
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) sm[q * G::SMEM + pidx(win_index(tid, wp, r))] = v[q][r];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) v[q][r] = sm[q * G::SMEM + pidx(win_index(tid, w, r))];
        }
        const u32 high = tid >> w;
#pragma unroll
        for (int b = btop; b >= w; --b) {
            const int j = b - w;  // register bit
            const u32 m = (u32)G::N >> (b + 1);
            u32 tw[8], tws[8];
            const u32 base = m + (high << (3 - j));
            if (j == 3) load_tw<1>(rp, rps, base, tw, tws);
            else if (j == 2) load_tw<2>(rp, rps, base, tw, tws);
            else if (j == 1) load_tw<4>(rp, rps, base, tw, tws);
            else load_tw<8>(rp, rps, base, tw, tws);
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {  // Harvey: values in [0, 4p), p < 2^30
                    const u32 a = red32(v[q][r], 2 * p);
                    const u32 t = shoup32(v[q][r2], tw[u], tws[u], p);
                    v[q][r] = a + t;
                    v[q][r2] = a - t + 2 * p;
                }
            }
        }
    }
}

/// Inverse NTT of NP polynomials (input mapping: x = tid << 4 | r; output mapping:
/// x = r << (LOGN-4) | tid).  Values in [0, 2p) in and out (no N^-1 scaling; p < 2^30).
template <int LOGN, int NP>
__device__ __forceinline__ void ntt32_inv_reg(u32 (&v)[NP][16], u32* sm, const u32* __restrict__ irp,
                                              const u32* __restrict__ irps, u32 p) {
    using G = NttGeom<LOGN>;
    const u32 tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < G::NW; ++k) {
        const int w = (4 * k) < (LOGN - 4) ? (4 * k) : (LOGN - 4);
        const int bbot = 4 * k;
        const int btop = (4 * k + 3) < (LOGN - 1) ? (4 * k + 3) : (LOGN - 1);
        if (k > 0) {
            const int wp = (4 * (k - 1)) < (LOGN - 4) ? (4 * (k - 1)) : (LOGN - 4);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) sm[q * G::SMEM + pidx(win_index(tid, wp, r))] = v[q][r];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) v[q][r] = sm[q * G::SMEM + pidx(win_index(tid, w, r))];
        }
        const u32 high = tid >> w;
#pragma unroll
        for (int b = bbot; b <= btop; ++b) {
            const int j = b - w;
            const u32 h = (u32)G::N >> (b + 1);
            u32 tw[8], tws[8];
            const u32 base = h + (high << (3 - j));
            if (j == 3) load_tw<1>(irp, irps, base, tw, tws);
            else if (j == 2) load_tw<2>(irp, irps, base, tw, tws);
            else if (j == 1) load_tw<4>(irp, irps, base, tw, tws);
            else load_tw<8>(irp, irps, base, tw, tws);
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {  // values in [0, 2p)
                    const u32 a = v[q][r], c = v[q][r2];
                    v[q][r] = red32(a + c, 2 * p);
                    v[q][r2] = shoup32(a - c + 2 * p, tw[u], tws[u], p);
                }
            }
        }
    }
}

/// Batched forward / inverse NTT (register version of k_ntt32): poly p -> group g = p / gs,
/// prime j = off + p % gs, address (g * stride + j) * N.  scale (inverse only):
/// 0 = N^-1, 1 = (N 2^32)^-1.  Output canonical [0, p).
template <int LOGN, bool INV>
__global__ void __launch_bounds__(NttGeom<LOGN>::T, LOGN >= 14 ? 1 : 2) k_ntt32r(u32* __restrict__ base, DevTab T, u32 gs, u32 stride,
                                                            u32 off, int scale) {
    using G = NttGeom<LOGN>;
    extern __shared__ u32 sm[];
    const u32 tid = threadIdx.x;
    const u32 pi = blockIdx.x, g = pi / gs, j = off + pi % gs;
    const u32 pr = T.a[j];
    u32* d = base + ((size_t)g * stride + j) * G::N;
    u32 v[1][16];
    if (!INV) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[0][r] = d[((u32)r << (LOGN - 4)) | tid];
        ntt32_fwd_reg<LOGN, 1>(v, sm, T.arp + (size_t)j * G::N, T.arps + (size_t)j * G::N, pr);
        uint4* o = reinterpret_cast<uint4*>(d + (tid << 4));
#pragma unroll
        for (int r = 0; r < 16; ++r) v[0][r] = red32(red32(v[0][r], 2 * pr), pr);
#pragma unroll
        for (int r = 0; r < 16; r += 4) o[r / 4] = make_uint4(v[0][r], v[0][r + 1], v[0][r + 2], v[0][r + 3]);
    } else {
        const uint4* in = reinterpret_cast<const uint4*>(d + (tid << 4));
#pragma unroll
        for (int r = 0; r < 16; r += 4) {
            const uint4 x = in[r / 4];
            v[0][r] = x.x; v[0][r + 1] = x.y; v[0][r + 2] = x.z; v[0][r + 3] = x.w;
        }
        ntt32_inv_reg<LOGN, 1>(v, sm, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, pr);
        const u32 ni = scale ? T.ninvRA[j] : T.ninvA[j], nis = scale ? T.ninvRA_s[j] : T.ninvA_s[j];
#pragma unroll
        for (int r = 0; r < 16; ++r) d[((u32)r << (LOGN - 4)) | tid] = red32(shoup32(v[0][r], ni, nis, pr), pr);
    }
}

/// Forward NTT of the 3 selection components of one product for one MAC prime:
/// polys at base + ((pr * 3 + comp) * stride_j + k) * N, k = blockIdx.x % Mm.
template <int LOGN, int NP>
__global__ void __launch_bounds__(NttGeom<LOGN>::T, (NP == 1 && LOGN < 14) ? 2 : 1) k_ntt32r_sel3(u32* __restrict__ base, DevTab T, u32 stride_j) {
    using G = NttGeom<LOGN>;
    extern __shared__ u32 smd[];
    const u32 tid = threadIdx.x;
    const u32 Mm = T.Mm;
    const u32 pr = blockIdx.x / Mm, k = blockIdx.x % Mm;
    const u32 p = T.a[k];
#pragma unroll 1
    for (int c0 = 0; c0 < 3; c0 += NP) {
        u32 v[NP][16];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const u32* d = base + (((size_t)pr * 3 + c0 + q) * stride_j + k) * G::N;
#pragma unroll
            for (int r = 0; r < 16; ++r) v[q][r] = d[((u32)r << (LOGN - 4)) | tid];
        }
        ntt32_fwd_reg<LOGN, NP>(v, smd, T.arp + (size_t)k * G::N, T.arps + (size_t)k * G::N, p);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            uint4* o = reinterpret_cast<uint4*>(base + (((size_t)pr * 3 + c0 + q) * stride_j + k) * G::N + (tid << 4));
#pragma unroll
            for (int r = 0; r < 16; ++r) v[q][r] = red32(red32(v[q][r], 2 * p), p);
#pragma unroll
            for (int r = 0; r < 16; r += 4) o[r / 4] = make_uint4(v[q][r], v[q][r + 1], v[q][r + 2], v[q][r + 3]);
        }
        if (NP == 1) __syncthreads();
    }
}

/// Tensor (mul_lazy_prepared, bfv.cpp:776-791) + INTT for P products, one aux prime per CTA.
/// NP = 3: the three components are transformed together (shared twiddles, 3-way ILP);
/// NP = 1: one component at a time (register budget of 1024-thread CTAs at N = 16384).
/// Operands: Montgomery-form NTT residues [idx][2][J][N]; output D[p][comp][j][N] in normal
/// form (the (N 2^32)^-1 scale undoes the Montgomery factor).
template <int LOGN, int NP>
__global__ void __launch_bounds__(NttGeom<LOGN>::T, (NP == 1 && LOGN < 14) ? 2 : 1) k_tensor_intt_r(const u32* __restrict__ prepA,
                                                                   const u32* __restrict__ idxA,
                                                                   const u32* __restrict__ prepB,
                                                                   const u32* __restrict__ idxB, u32 P, DevTab T,
                                                                   u32* __restrict__ D) {
    using G = NttGeom<LOGN>;
    extern __shared__ u32 smd[];
    const u32 J = T.J;
    const u32 tid = threadIdx.x;
    const u32 pr = blockIdx.x / J, j = blockIdx.x % J;
    const u32 p = T.a[j], pinv = T.apinv[j];
    const size_t per = (size_t)2 * J * G::N;
    const u32* A = prepA + (size_t)(idxA ? idxA[pr] : pr) * per + (size_t)j * G::N + (tid << 4);
    const u32* B = prepB + (size_t)(idxB ? idxB[pr] : pr) * per + (size_t)j * G::N + (tid << 4);
    const size_t o1 = (size_t)J * G::N;
    const u32 ni = T.ninvRA[j], nis = T.ninvRA_s[j];
#pragma unroll 1
    for (int c0 = 0; c0 < 3; c0 += NP) {
        u32 v[NP][16];
#pragma unroll
        for (int r = 0; r < 16; r += 4) {
            const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(A + r));
            const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(A + o1 + r));
            const uint4 y0 = __ldg(reinterpret_cast<const uint4*>(B + r));
            const uint4 y1 = __ldg(reinterpret_cast<const uint4*>(B + o1 + r));
            const u32 a0[4] = {x0.x, x0.y, x0.z, x0.w}, a1[4] = {x1.x, x1.y, x1.z, x1.w};
            const u32 b0[4] = {y0.x, y0.y, y0.z, y0.w}, b1[4] = {y1.x, y1.y, y1.z, y1.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const int comp = NP == 3 ? q : c0;
                    if (comp == 0) v[q][r + e] = red32(mont32(a0[e], b0[e], p, pinv), p);
                    else if (comp == 1)
                        v[q][r + e] = red32(mont32(a0[e], b1[e], p, pinv), p) + red32(mont32(a1[e], b0[e], p, pinv), p);
                    else v[q][r + e] = red32(mont32(a1[e], b1[e], p, pinv), p);
                }
            }
        }
        ntt32_inv_reg<LOGN, NP>(v, smd, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, p);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int comp = NP == 3 ? q : c0;
            u32* out = D + (((size_t)pr * 3 + comp) * J + j) * G::N;
#pragma unroll
            for (int r = 0; r < 16; ++r) out[((u32)r << (LOGN - 4)) | tid] = red32(shoup32(v[q][r], ni, nis, p), p);
        }
        if (NP == 1) __syncthreads();
    }
}

}  // namespace cwgpu

namespace cwgpu {

/// Per-aux-prime constants of the HPS rounding, padded to JM entries (zeros beyond J).
struct RoundJ {
    u32 a, chat, chat_s, pad;
    u64 aF;
    u32 f0, f1;  // floor(frac(t (A/a_j) / q) * 2^64)
};
struct RoundK {
    u32 a, gcoef, roff, c30;  // gcoef = (-I_A) mod a; roff = (-2^36) mod a; c30 = 2^30 mod a
    u64 abar;
};

/// Exact scale-and-round t*D/q (bfv.cpp:811-849) by HPS scaling:
///   D = sum_j w_j (A/a_j) - gamma A,  w_j = D_j (A/a_j)^-1 mod a_j,
///   t D / q = sum_j w_j (I_j + F_j) - gamma (I_A + F_A),
///   r = sum_j w_j I_j - gamma I_A + round(sum_j w_j F_j - gamma F_A)   (no ties: q odd).
/// The fractional sum is estimated in 64-bit fixed point; when the estimate is within its
/// error band of a half-integer the exact multiword path (round_exact) decides.
/// D planes: D[pc][j][N] for pc < P*3; writes r mod a_k (k < Mm) in place.
template <int JM>
__global__ void __launch_bounds__(256) k_round_mac_t(u32* __restrict__ D, u32 P, DevTab T,
                                                     const RoundJ* __restrict__ gRJ, const RoundK* __restrict__ gRK,
                                                     const u32* __restrict__ gImodT) {
    extern __shared__ __align__(16) unsigned char smraw[];
    RoundJ* RJ = reinterpret_cast<RoundJ*>(smraw);
    RoundK* RK = reinterpret_cast<RoundK*>(smraw + sizeof(RoundJ) * JM);
    u32* ImodT = reinterpret_cast<u32*>(smraw + sizeof(RoundJ) * JM + sizeof(RoundK) * kMaxJ);
    const u32 J = T.J, Mm = T.Mm, N = T.N, logN = T.logN;
    for (u32 x = threadIdx.x; x < JM; x += blockDim.x) RJ[x] = gRJ[x];
    for (u32 x = threadIdx.x; x < Mm; x += blockDim.x) RK[x] = gRK[x];
    for (u32 x = threadIdx.x; x < Mm * JM; x += blockDim.x) ImodT[x] = gImodT[x];
    __syncthreads();
    const u32 gsh = 64 - T.gbits;
    const u32 fA0 = T.fracA[1], fA1 = T.fracA[2];  // 64-bit fraction of t A / q
    const size_t total = (size_t)P * 3 * N;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t pc = idx >> logN;
        const u32 n = (u32)(idx & (N - 1));
        u32* Dp = D + pc * J * N + n;
        u32 d[JM];
#pragma unroll
        for (int j = 0; j < JM; ++j) d[j] = (j < (int)J) ? Dp[(size_t)j * N] : 0u;
        u32 w[JM];
        u64 gs = 0;
        u32 s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
        for (int j = 0; j < JM; ++j) {
            const RoundJ c = RJ[j];
            const u32 wj = red32(shoup32(d[j], c.chat, c.chat_s, c.a), c.a);  // padded a = 1 -> 0
            w[j] = wj;
            gs += (u64)wj * c.aF;
            asm("mad.lo.cc.u32  %0, %4, %5, %0;\n\t"
                "madc.lo.cc.u32 %1, %4, %6, %1;\n\t"
                "addc.cc.u32    %2, %2, 0;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                "mad.hi.cc.u32  %1, %4, %5, %1;\n\t"
                "madc.hi.cc.u32 %2, %4, %6, %2;\n\t"
                "addc.u32       %3, %3, 0;\n\t"
                : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3)
                : "r"(wj), "r"(c.f0), "r"(c.f1));
        }
        const u32 gamma = (u32)((gs + (1ull << (gsh - 1))) >> gsh);
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
#pragma unroll 2
            for (u32 k = 0; k < Mm; ++k) {
                const RoundK ck = RK[k];
                const uint4* Im = reinterpret_cast<const uint4*>(ImodT + k * JM);
                u64 lo = 0;
                u32 hi = 0;
#pragma unroll
                for (int g0 = 0; g0 < JM; g0 += 16) {
                    u64 g = 0;  // 16 products < 2^60 each: < 2^64
#pragma unroll
                    for (int j0 = g0; j0 < g0 + 16 && j0 < JM; j0 += 4) {
                        const uint4 I = Im[j0 / 4];
                        g += (u64)w[j0] * I.x;
                        g += (u64)w[j0 + 1] * I.y;
                        g += (u64)w[j0 + 2] * I.z;
                        g += (u64)w[j0 + 3] * I.w;
                    }
                    if (g0 == 0) {
                        lo = g;
                    } else {
                        lo += g;
                        hi += (lo < g);
                    }
                }
                u64 t = (u64)bar64(lo, ck.a, ck.abar) + (u64)gamma * ck.gcoef + rlo + (u64)rhi * ck.c30 + ck.roff;
                if (JM > 16) t += (u64)hi * bar64(0xffffffffffffffffull, ck.a, ck.abar) + hi;  // hi * 2^64
                Dp[(size_t)k * N] = bar64(t, ck.a, ck.abar);
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
                const u32 a = RK[k].a;
                u32 r = mag_mod32(R, a, RK[k].abar);
                if (neg && r) r = a - r;
                Dp[(size_t)k * N] = r;
            }
        }
    }
}

}  // namespace cwgpu

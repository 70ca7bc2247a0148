// Key switching through the 30-bit aux primes (bfv.cpp:343-372, key_switch).
//
// The reference multiplies the NTT of every decomposition digit with the key modulo each chain
// prime q_i (64-bit NTTs: D L forward + 2 L inverse per switch).  The result is the ring element
// sum_d digit_d * key_{d,c} mod q_i, i.e. the exact integer negacyclic convolution reduced mod
// q_i; its integer value is bounded by D N 2^bits q_i (digits in [0, 2^bits), key coefficients in
// [0, q_i)), so it is recovered exactly from K' aux primes with prod a_j > 2 D N 2^bits q_max and
// reduced mod q_i afterwards.  Per switch that is D K' forward and 2 L K' inverse register NTTs on
// 32-bit words (C4: 42 + 30, each ~4x cheaper than a 64-bit NTT), with the key transformed once
// per key upload (INTT mod q_i, reduce mod a_j, NTT mod a_j).
#pragma once
#include "devtab.h"
#include "modarith.cuh"

namespace cwgpu {

constexpr int kMaxKs = 5;  // aux primes for the key-switch convolution

/// Garner / mixed-radix constants of the K' key-switch primes, and their images mod each q_i.
struct KsCrt {
    u32 K;
    u32 a[kMaxKs];
    u32 half[kMaxKs];             // (a_j - 1) / 2: mixed-radix digits of floor(A'/2)
    u32 cinv[kMaxKs][kMaxKs];     // a_k^-1 mod a_j (k < j)
    u32 cinv_s[kMaxKs][kMaxKs];   // Shoup companions floor(cinv 2^32 / a_j)
    u64 pmod[kMaxL][kMaxKs];      // prod_{k<j} a_k mod q_i
    u64 amod[kMaxL];              // A' mod q_i
};

/// u64 values (< 2^64) of npolys planes [npolys][N] -> u32 residues [npolys][K'][N] mod a_j.
__global__ void k_to_ks_aux(const u64* __restrict__ src, size_t npolys, u32 N, const __grid_constant__ KsCrt C,
                            u32* __restrict__ dst) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= npolys * N) return;
    const size_t p = idx / N;
    const u32 n = (u32)(idx % N);
    const u64 v = src[idx];
    for (u32 j = 0; j < C.K; ++j) dst[(p * C.K + j) * N + n] = (u32)(v % C.a[j]);
}

/// out[b][c][i][j][n] = sum_d dig[b][d][j][n] key[d][c][i][j][n] mod a_j (NTT domain, any order
/// shared by both operands).  Products < 2^60; reduced every 8 terms.
__global__ void k_ks_mac32(const u32* __restrict__ dig, const u32* __restrict__ key, u32 B, u32 D, u32 L, u32 N,
                           const __grid_constant__ KsCrt C, const u64* __restrict__ abar, u32* __restrict__ out) {
    const u32 K = C.K;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per_b = (size_t)2 * L * K * N;
    if (idx >= (size_t)B * per_b) return;
    const u32 b = (u32)(idx / per_b);
    const size_t r = idx % per_b;  // ((c L + i) K + j) N + n
    const u32 n = (u32)(r % N);
    const u32 j = (u32)((r / N) % K);
    const size_t cij = r / N;      // (c L + i) K + j
    const u32 a = C.a[j];
    const u64 mu = abar[j];
    const u32* dp = dig + ((size_t)b * D * K + j) * N + n;
    const u32* kp = key + cij * N + n;
    const size_t dstride = (size_t)K * N, kstride = (size_t)2 * L * K * N;
    u64 acc = 0;
    for (u32 d = 0; d < D; ++d) {
        acc += (u64)dp[(size_t)d * dstride] * __ldg(kp + (size_t)d * kstride);
        if ((d & 7) == 7) acc = bar64(acc, a, mu);
    }
    out[idx] = bar64(acc, a, mu);
}

/// k_ks_mac32 with the loads shared: thread (b pair, j, n) keeps both rows' D digit residues in
/// registers and loops over the 2 L (component, chain prime) outputs, each key word feeding two
/// products (C4: 8.4 loads per output instead of 28).
constexpr int kKsDmax = 16;
template <int DMAX>
__global__ void __launch_bounds__(128) k_ks_mac32x(const u32* __restrict__ dig, const u32* __restrict__ key, u32 B, u32 D,
                                                   u32 L, u32 N, const __grid_constant__ KsCrt C, const u64* __restrict__ abar,
                                                   u32* __restrict__ out) {
    const u32 K = C.K;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = (size_t)K * N;
    if (idx >= (size_t)((B + 1) / 2) * per) return;
    const u32 b0 = (u32)(idx / per) * 2;
    const u32 j = (u32)((idx / N) % K), n = (u32)(idx % N);
    const bool two = b0 + 1 < B;
    const u32 a = C.a[j];
    const u64 mu = abar[j];
    u32 d0[DMAX], d1[DMAX];
    const u32* dp0 = dig + ((size_t)b0 * D * K + j) * N + n;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
        d0[d] = d < (int)D ? dp0[(size_t)d * K * N] : 0u;
        d1[d] = (two && d < (int)D) ? dp0[((size_t)D + d) * K * N] : 0u;
    }
    const size_t kstride = (size_t)2 * L * K * N;
    for (u32 ci = 0; ci < 2 * L; ++ci) {
        const u32* kp = key + ((size_t)ci * K + j) * N + n;
        u64 s0 = 0, s1 = 0;
#pragma unroll
        for (int d = 0; d < DMAX; ++d) {
            if (d >= (int)D) break;
            const u64 kv = __ldg(kp + (size_t)d * kstride);
            s0 += (u64)d0[d] * kv;
            s1 += (u64)d1[d] * kv;
            if ((d & 7) == 7) {
                s0 = bar64(s0, a, mu);
                s1 = bar64(s1, a, mu);
            }
        }
        out[(((size_t)b0 * 2 * L + ci) * K + j) * N + n] = bar64(s0, a, mu);
        if (two) out[((((size_t)b0 + 1) * 2 * L + ci) * K + j) * N + n] = bar64(s1, a, mu);
    }
}

/// Slot-major key-switch MAC: thread = one NTT slot (j, n) of the K' aux primes.  Per slot the key
/// is a [D][2L] matrix shared by every row b, so each thread keeps a CI-column block of it in
/// registers (D x CI words) and streams the rows' D digit residues past it: D x CI products per
/// D digit loads, the key read once per group of G rows instead of once per output.  Products are
/// < 2^60 (residues < 2^30), accumulated 15 at a time in u64 before a Barrett reduction.
/// Grid: (ceil(K' N / 128), row splits); rows [b0, b1) of this split in groups of G.
template <int D, int CI, int G, int MINB, int UB = 1>
__global__ void __launch_bounds__(128, MINB) k_ks_mac32s(const u32* __restrict__ dig, const u32* __restrict__ key, u32 B,
                                                      u32 L, u32 N, const __grid_constant__ KsCrt C,
                                                      const u64* __restrict__ abar, u32* __restrict__ out) {
    const u32 K = C.K;
    const u32 KN = K * N;  // < 2^32: plane offsets in 32-bit arithmetic (fewer live 64-bit addresses)
    const u32 slot = blockIdx.x * 128 + threadIdx.x;  // j N + n
    if (slot >= KN) return;
    const u32 j = slot / N;
    const u32 a = C.a[j];
    const u64 mu = abar[j];
    const u32 nci = 2 * L;
    const u32 b0 = (u32)(((u64)B * blockIdx.y) / gridDim.y), b1 = (u32)(((u64)B * (blockIdx.y + 1)) / gridDim.y);
#pragma unroll 1
    for (u32 g0 = b0; g0 < b1; g0 += G) {
        const u32 g1 = min(b1, g0 + G);
#pragma unroll 1
        for (u32 c0 = 0; c0 < nci; c0 += CI) {
            u32 kr[D][CI];
            const u32* kp = key + (size_t)c0 * KN + slot;
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int c = 0; c < CI; ++c)
                    kr[d][c] = (c0 + c < nci) ? __ldg(kp + ((u32)d * nci + (u32)c) * KN) : 0u;
#pragma unroll UB
            for (u32 b = g0; b < g1; ++b) {  // UB > 1: the next rows' digit loads overlap this row's MACs
                const u32* dp = dig + (size_t)b * D * KN + slot;
                u32 dr[D];
#pragma unroll
                for (int d = 0; d < D; ++d) dr[d] = dp[(u32)d * KN];
                u32* op = out + ((size_t)b * nci + c0) * KN + slot;
#pragma unroll
                for (int c = 0; c < CI; ++c) {
                    // two independent chains (even / odd digits), each < 15 products < 2^64
                    u64 s0 = 0, s1 = 0;
                    u32 r = 0;
#pragma unroll
                    for (int d = 0; d < D; d += 2) {
                        s0 += (u64)dr[d] * kr[d][c];
                        if (d + 1 < D) s1 += (u64)dr[d + 1] * kr[d + 1][c];
                        if (d % 28 == 26 && d + 2 < D) {  // 14 products per chain
                            r += bar64(s0, a, mu);
                            r += bar64(s1, a, mu);
                            s0 = s1 = 0;
                        }
                    }
                    if (c0 + c < nci) op[(u32)c * KN] = red32(bar64(s0, a, mu) + bar64(s1 + r, a, mu), a);
                }
            }
        }
    }
}

/// (acc + m a) / 2^32 with m = -acc a^-1 mod 2^32: acc 2^-32 mod a, in [0, 3a) for acc < 2^63 + 2^62.
__device__ __forceinline__ u32 ks_mont_red64(u64 acc, u32 a, u32 pinv) {
    const u32 m = (u32)acc * pinv;
    return (u32)((acc + (u64)m * a) >> 32);
}

/// Slot-major key-switch MAC with every size a compile-time constant (k_ks_mac32s spent ~9 issued
/// instructions per product on 64-bit address arithmetic, tail predicates and two Barrett
/// reductions per output): the digit and output planes of a row are read at immediate offsets
/// d K'N from one base pointer, the key block of CI columns walks one pointer per digit, and each
/// output is reduced by Montgomery steps -- chains of <= 12 products (< 2^63.6), one
/// (acc + m a) >> 32 per chain, their sum times 2^64 mod a (one Montgomery product) restores the
/// plain residue.  The key-switch primes are the first K' aux primes, so T.apinv / T.a2_64 apply.
/// Grid: (K'N / 128, row splits); rows [b0, b1) of this split in groups of G.
template <int LOGN, int KP, int D, int NCI, int CI, int G, int MINB>
__global__ void __launch_bounds__(128, MINB) k_ks_mac32t(const u32* __restrict__ dig, const u32* __restrict__ key, u32 B,
                                                      const u32* __restrict__ ap, const u32* __restrict__ apinv,
                                                      const u32* __restrict__ a2_64, u32* __restrict__ out) {
    constexpr u32 N = 1u << LOGN, KN = KP * N;
    constexpr int NCH = (D + 11) / 12;           // chains of <= 12 products
    constexpr int CL = (D + NCH - 1) / NCH;      // products per chain
    static_assert(NCI % CI == 0 && KN % 128 == 0, "k_ks_mac32t shape");
    const u32 slot = blockIdx.x * 128 + threadIdx.x;  // j N + n
    const u32 j = slot >> LOGN;
    const u32 a = ap[j], pinv = apinv[j], r64 = a2_64[j];
    const u32 b0 = (u32)(((u64)B * blockIdx.y) / gridDim.y), b1 = (u32)(((u64)B * (blockIdx.y + 1)) / gridDim.y);
#pragma unroll 1
    for (u32 g0 = b0; g0 < b1; g0 += G) {
        const u32 g1 = min(b1, g0 + G);
#pragma unroll 1
        for (u32 c0 = 0; c0 < (u32)NCI; c0 += CI) {
            u32 kr[D][CI];
            const u32* kp = key + (size_t)c0 * KN + slot;
#pragma unroll
            for (int d = 0; d < D; ++d) {
#pragma unroll
                for (int c = 0; c < CI; ++c) kr[d][c] = __ldg(kp + (u32)c * KN);
                kp += (size_t)NCI * KN;
            }
#pragma unroll 2
            for (u32 b = g0; b < g1; ++b) {
                const u32* dp = dig + (size_t)b * D * KN + slot;
                u32 dr[D];
#pragma unroll
                for (int d = 0; d < D; ++d) dr[d] = dp[(u32)d * KN];
                u32* op = out + ((size_t)b * NCI + c0) * KN + slot;
#pragma unroll
                for (int c = 0; c < CI; ++c) {
                    u32 r = 0;
#pragma unroll
                    for (int h = 0; h < NCH; ++h) {
                        u64 s = 0;
#pragma unroll
                        for (int d = h * CL; d < (h + 1) * CL && d < D; ++d) s += (u64)dr[d] * kr[d][c];
                        const u32 x = ks_mont_red64(s, a, pinv);  // [0, 3a)
                        r += red32(red32(x, 2 * a), a);           // NCH <= 3: r < 3a < 2^32
                    }
                    op[(u32)c * KN] = red32(mont32(r, r64, a, pinv), a);
                }
            }
        }
    }
}

/// ks[b][c][i][n] = (centred CRT of the K' residues x_j) mod q_i.  x: [B][2][L][K'][N] in [0, a_j).
/// add (optional): the result is (ks + add[b * add_stride + (c L + i) N + n]) mod q_i -- the
/// relinearisation's (c0 + ks0, c1 + ks1), bfv.cpp:859-869 -- and scale (optional, != 0) then
/// multiplies it by a constant mod q_i (the arithmetic operator's (k!)^-1, eq_circuits.cpp:126).
__global__ void k_ks_crt(const u32* __restrict__ x, u32 B, u32 L, u32 N, const __grid_constant__ KsCrt C, DevTab T,
                         u64* __restrict__ ks, const u64* __restrict__ add, size_t add_stride, u64 scale) {
    const u32 K = C.K;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * 2 * L * N) return;
    const size_t bci = idx / N;  // (b 2 + c) L + i
    const u32 n = (u32)(idx % N);
    const u32 i = (u32)(bci % L);
    const u32* xp = x + bci * K * N + n;
    u32 y[kMaxKs];
    // Garner: y_j = ((x_j - y_0) c_0j - y_1) c_1j ... mod a_j
#pragma unroll
    for (int jj = 0; jj < kMaxKs; ++jj) {
        y[jj] = 0;
        if (jj >= (int)K) continue;
        const u32 a = C.a[jj];
        u32 t = xp[(size_t)jj * N];
#pragma unroll
        for (int k = 0; k < kMaxKs - 1; ++k) {
            if (k >= jj) break;
            const u32 yk = red32(y[k], a);                 // y_k < a_k < 2 a_j
            t = red32(t + a - yk, a);                      // (t - y_k) mod a_j
            t = red32(shoup32(t, C.cinv[jj][k], C.cinv_s[jj][k], a), a);
        }
        y[jj] = t;
    }
    // centred: v > (A'-1)/2 <=> mixed-radix digits (top first) exceed the half digits
    int cmp = 0;
#pragma unroll
    for (int jj = kMaxKs - 1; jj >= 0; --jj)
        if (jj < (int)K && cmp == 0) cmp = y[jj] > C.half[jj] ? 1 : (y[jj] < C.half[jj] ? -1 : 0);
    const u64 q = T.q[i];
    u64 hi = 0, lo = 0;
#pragma unroll
    for (int jj = 0; jj < kMaxKs; ++jj)
        if (jj < (int)K) mac128(hi, lo, (u64)y[jj], C.pmod[i][jj]);
    u64 v = reduce128(hi, lo, q, T.q_mu96[i]);
    if (cmp > 0) v = v >= C.amod[i] ? v - C.amod[i] : v + q - C.amod[i];
    if (add) {
        const size_t b = bci / (2 * L), ci = bci % (2 * L);
        v += add[b * add_stride + ci * N + n];
        if (v >= q) v -= q;
    }
    if (scale) v = reduce128(__umul64hi(v, scale), v * scale, q, T.q_mu96[i]);
    ks[idx] = v;
}

/// k_ks_crt for K' = 3 with the sums kept in 96 bits: y_j < 2^30 times (prod_{k<j} a_k mod q_i) < 2^60
/// is two 32 x 32 products, and sum_j y_j P_ij < 2^92 needs one reduce96 (the generic kernel forms
/// 64 x 64 -> 128-bit products and reduces twice: ~330 instructions per output at C5).
__global__ void __launch_bounds__(256) k_ks_crt3(const u32* __restrict__ x, u32 B, u32 L, u32 N,
                                                 const __grid_constant__ KsCrt C, DevTab T, u64* __restrict__ ks,
                                                 const u64* __restrict__ add, size_t add_stride, u64 scale) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * 2 * L * N) return;
    const u32 bci = (u32)(idx >> T.logN);  // (b 2 + c) L + i  (N is a power of two: no 64-bit div / mod)
    const u32 n = (u32)idx & (N - 1);
    const u32 i = bci % L;
    const u32* xp = x + (size_t)bci * 3 * N + n;
    const u32 x0 = xp[0], x1 = xp[N], x2 = xp[2 * (size_t)N];
    const u32 a1 = C.a[1], a2 = C.a[2];
    // Garner (mixed radix): v = y0 + y1 a0 + y2 a0 a1
    const u32 y0 = x0;
    u32 t = red32(x1 + a1 - red32(y0, a1), a1);
    const u32 y1 = red32(shoup32(t, C.cinv[1][0], C.cinv_s[1][0], a1), a1);
    t = red32(x2 + a2 - red32(y0, a2), a2);
    t = red32(shoup32(t, C.cinv[2][0], C.cinv_s[2][0], a2), a2);
    t = red32(t + a2 - red32(y1, a2), a2);
    const u32 y2 = red32(shoup32(t, C.cinv[2][1], C.cinv_s[2][1], a2), a2);
    // centred: v > (A'-1)/2 <=> mixed-radix digits (top first) exceed the half digits
    const bool neg = y2 != C.half[2] ? y2 > C.half[2] : (y1 != C.half[1] ? y1 > C.half[1] : y0 > C.half[0]);
    const u64 q = T.q[i];
    const u64 P1 = C.pmod[i][1], P2 = C.pmod[i][2];  // P0 = 1
    // 96-bit sum y0 + y1 P1 + y2 P2 (< 2^92)
    u64 lo = (u64)y0 + (u64)y1 * (u32)P1;           // < 2^63
    const u64 l2 = (u64)y2 * (u32)P2;
    lo += l2;
    u32 hi = lo < l2 ? 1u : 0u;
    const u64 h = (u64)y1 * (u32)(P1 >> 32) + (u64)y2 * (u32)(P2 >> 32);  // < 2^59, weight 2^32
    const u64 hs = h << 32;
    lo += hs;
    hi += (u32)(h >> 32) + (lo < hs ? 1u : 0u);
    u64 v = reduce96(hi, lo, q, T.q_mu96[i]);
    if (neg) v = v >= C.amod[i] ? v - C.amod[i] : v + q - C.amod[i];
    if (add) {
        const u32 b = bci / (2 * L), ci = bci % (2 * L);
        v += add[(size_t)b * add_stride + (size_t)ci * N + n];
        if (v >= q) v -= q;
    }
    if (scale) v = reduce128(__umul64hi(v, scale), v * scale, q, T.q_mu96[i]);
    ks[idx] = v;
}

}  // namespace cwgpu

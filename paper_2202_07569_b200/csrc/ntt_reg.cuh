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

// XOR swizzle inside each 32-word row, y = x >> 5: bank(x) = x ^ (y ^ (y << 1)) mod 32 is conflict-free
// for every transpose window of 2^8 <= N <= 2^14 (checked exhaustively) and needs no padding
__device__ __forceinline__ u32 pidx(u32 x) { const u32 y = x >> 5; return x ^ ((y ^ (y << 1)) & 31u); }

template <int LOGN>
struct NttGeom {
    static constexpr int N = 1 << LOGN;
    static constexpr int T = N / 16;
    static constexpr int NW = (LOGN + 3) / 4;       // windows
    static constexpr int SMEM = N;                  // u32 words per polynomial (swizzled, unpadded)
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

/// Twiddles of one 4-bit window: stage slot j (register bit) needs 2^(3-j) consecutive
/// table entries starting at (N >> (b+1)) + (high << (3-j)), b = w + j.  Loaded for the whole
/// window before its transpose so their latency overlaps the shared-memory exchange.
template <int LOGN>
__device__ __forceinline__ void load_window_tw(const u32* __restrict__ tp, const u32* __restrict__ tsp, int w,
                                               int jlo, int jhi, u32 high, u32 (&tw)[4][8], u32 (&tws)[4][8]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j < jlo || j > jhi) continue;
        const int b = w + j;
        const u32 base = ((u32)(1 << LOGN) >> (b + 1)) + (high << (3 - j));
        if (j == 3) load_tw<1>(tp, tsp, base, tw[j], tws[j]);
        else if (j == 2) load_tw<2>(tp, tsp, base, tw[j], tws[j]);
        else if (j == 1) load_tw<4>(tp, tsp, base, tw[j], tws[j]);
        else load_tw<8>(tp, tsp, base, tw[j], tws[j]);
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
        const u32 high = tid >> w;
        u32 tw[4][8], tws[4][8];
        load_window_tw<LOGN>(rp, rps, w, 0, btop - w, high, tw, tws);
        if (k > 0) {
            const int wp = (LOGN - 4 - 4 * (k - 1)) > 0 ? (LOGN - 4 - 4 * (k - 1)) : 0;
            // pidx is GF(2)-linear and the thread / register fields of the index are disjoint:
            // pidx(win_index(tid, w, r)) = pidx(win_index(tid, w, 0)) ^ pidx(r << w)
            const u32 ps = pidx(win_index(tid, wp, 0)), pl = pidx(win_index(tid, w, 0));
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) sm[q * G::SMEM + (ps ^ pidx((u32)r << wp))] = v[q][r];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) v[q][r] = sm[q * G::SMEM + (pl ^ pidx((u32)r << w))];
        }
#pragma unroll
        for (int b = btop; b >= w; --b) {
            const int j = b - w;  // register bit
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {  // Harvey: values in [0, 4p), p < 2^30
                    const u32 a = red32(v[q][r], 2 * p);
                    const u32 t = shoup32(v[q][r2], tw[j][u], tws[j][u], p);
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
        const u32 high = tid >> w;
        u32 tw[4][8], tws[4][8];
        load_window_tw<LOGN>(irp, irps, w, bbot - w, btop - w, high, tw, tws);
        if (k > 0) {
            const int wp = (4 * (k - 1)) < (LOGN - 4) ? (4 * (k - 1)) : (LOGN - 4);
            // pidx is GF(2)-linear and the thread / register fields of the index are disjoint:
            // pidx(win_index(tid, w, r)) = pidx(win_index(tid, w, 0)) ^ pidx(r << w)
            const u32 ps = pidx(win_index(tid, wp, 0)), pl = pidx(win_index(tid, w, 0));
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) sm[q * G::SMEM + (ps ^ pidx((u32)r << wp))] = v[q][r];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int r = 0; r < 16; ++r) v[q][r] = sm[q * G::SMEM + (pl ^ pidx((u32)r << w))];
        }
#pragma unroll
        for (int b = bbot; b <= btop; ++b) {
            const int j = b - w;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {  // values in [0, 2p)
                    const u32 a = v[q][r], c = v[q][r2];
                    v[q][r] = red32(a + c, 2 * p);
                    v[q][r2] = shoup32(a - c + 2 * p, tw[j][u], tws[j][u], p);
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
    // Montgomery forms (x 2^32 mod a): gcoef = -I_A, roff = -2^36, c0 = 1, c30 = 2^30
    u32 a, pinv, gcoef, roff, c0, c30;
    u64 abar;
};

/// (acc + m a) / 2^32 with m = -acc a^-1 mod 2^32: acc 2^-32 mod a, in [0, 3a) for acc < 2^63 + 2^62.
__device__ __forceinline__ u32 mont_red64(u64 acc, u32 a, u32 pinv) {
    const u32 m = (u32)acc * pinv;
    return (u32)((acc + (u64)m * a) >> 32);
}

/// Exact scale-and-round t*D/q (bfv.cpp:811-849) by HPS scaling:
///   D = sum_j w_j (A/a_j) - gamma A,  w_j = D_j (A/a_j)^-1 mod a_j,
///   t D / q = sum_j w_j (I_j + F_j) - gamma (I_A + F_A),
///   r = sum_j w_j I_j - gamma I_A + round(sum_j w_j F_j - gamma F_A)   (no ties: q odd).
/// The fractional sum is estimated in 64-bit fixed point; when the estimate is within its
/// error band of a half-integer the exact multiword path (round_exact) decides.
/// D planes: D[pc][j][N] for pc < P*3; writes r mod a_k (k < Mm) in place.
template <int JM>
__global__ void __launch_bounds__(256, 4) k_round_mac_t(u32* __restrict__ D, u32 P, DevTab T,
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
        for (int j = 0; j < JM; ++j) d[j] = Dp[(size_t)min(j, (int)J - 1) * N];  // padded j: any value (w_j = 0)
#pragma unroll
        for (int j = 0; j < JM; ++j) asm volatile("" : "+r"(d[j]));  // all plane loads in flight before any use
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
                const uint4* Im = reinterpret_cast<const uint4*>(ImodT + k * JM);  // Montgomery form
                // groups of 8 products (< 2^63); the gamma / rho correction terms ride in group 0
                u64 g0 = (u64)gamma * ck.gcoef + (u64)rlo * ck.c0 + (u64)rhi * ck.c30 + ck.roff;
                u32 r = 0;
#pragma unroll
                for (int gb = 0; gb < JM; gb += 8) {
                    u64 g = gb == 0 ? g0 : 0;
#pragma unroll
                    for (int j0 = gb; j0 < gb + 8; j0 += 4) {
                        const uint4 I = Im[j0 / 4];
                        g += (u64)w[j0] * I.x;
                        g += (u64)w[j0 + 1] * I.y;
                        g += (u64)w[j0 + 2] * I.z;
                        g += (u64)w[j0 + 3] * I.w;
                    }
                    u32 x = mont_red64(g, ck.a, ck.pinv);  // [0, 3a)
                    x = red32(red32(x, 2 * ck.a), ck.a);
                    r = red32(r + x, ck.a);
                }
                Dp[(size_t)k * N] = r;
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

namespace cwgpu {
/// Payload multiply-accumulate (weighted_sum, bfv.cpp:944-986, in the NTT domain of the MAC
/// basis): acc[sj][c][k][n] += sum_r Z[r][c][k][n] * DB[row0 + r][sj][k][n]  (mod a_k, lazily).
/// Thread = 4 consecutive coefficients of one (sj, k) plane over a chunk of rows; 128-bit
/// loads, 16-row u64 groups (products < 2^60), one 64-bit atomic add per output per chunk.
/// Z: Z + ((r * nc + c) * zstride + k) * N.  DB: [rows][s][Mm][N].  acc: u64 sums of residues.
template <int NC>
__global__ void __launch_bounds__(256, 3) k_mac2(const u32* __restrict__ Z, u32 zstride, const u32* __restrict__ DB,
                                              u32 R, u32 s, u32 chunk, DevTab T, unsigned long long* __restrict__ acc) {
    const u32 N = T.N, Mm = T.Mm;
    const u32 n4s = N >> 2;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const u32 nchunks = (R + chunk - 1) / chunk;
    if (idx >= (size_t)s * Mm * ((n4s + 255) / 256) * 256 * nchunks) return;  // padded 256-wide blocks
    // index order (slowest .. fastest): chunk, prime, 16-KB coefficient block, payload chunk sj,
    // coefficient: the s slices that reuse the same selection values run back to back (L2 hits)
    const u32 nb = (n4s + 255) / 256;
    const u32 n4lo = (u32)(idx % 256);
    size_t rest = idx / 256;
    const u32 sj = (u32)(rest % s);
    rest /= s;
    const u32 blk = (u32)(rest % nb);
    rest /= nb;
    const u32 k = (u32)(rest % Mm);
    const u32 ch = (u32)(rest / Mm);
    const u32 n4 = blk * 256 + n4lo;
    if (n4 >= n4s) return;
    const u32 p = T.a[k];
    const u64 pb = T.abar[k];
    const u32 r0 = ch * chunk, r1 = min(R, r0 + chunk);
    const size_t dbs = (size_t)s * Mm * N;
    const uint4* dbp = reinterpret_cast<const uint4*>(DB + ((size_t)sj * Mm + k) * N) + n4;
    const size_t zs = (size_t)NC * zstride * N;
    const uint4* zp = reinterpret_cast<const uint4*>(Z + (size_t)k * N) + n4;
    u32 accr[NC][4];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) accr[c][e] = 0;
    for (u32 rg = r0; rg < r1; rg += 16) {
        const u32 re = min(r1, rg + 16);
        u64 g[NC][4];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) g[c][e] = 0;
#pragma unroll 2
        for (u32 r = rg; r < re; ++r) {
            const uint4 d = __ldg(dbp + (size_t)r * (dbs >> 2));
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const uint4 z = __ldg(zp + ((size_t)r * zs + (size_t)c * zstride * N) / 4);
                g[c][0] += (u64)z.x * d.x;
                g[c][1] += (u64)z.y * d.y;
                g[c][2] += (u64)z.z * d.z;
                g[c][3] += (u64)z.w * d.w;
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) accr[c][e] = red32(accr[c][e] + bar64(g[c][e], p, pb), p);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        unsigned long long* o = acc + (((size_t)sj * 3 + c) * Mm + k) * N + 4 * n4;
#pragma unroll
        for (int e = 0; e < 4; ++e) atomicAdd(o + e, (unsigned long long)accr[c][e]);
    }
}

/// acc (u64 sums of residues) -> partial[x] = acc mod a_k.
__global__ void k_acc_mod(const unsigned long long* __restrict__ acc, size_t total, DevTab T, u64* __restrict__ partial) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const u32 k = (u32)((idx >> T.logN) % T.Mm);
    partial[idx] = bar64(acc[idx], T.a[k], T.abar[k]);
}
}  // namespace cwgpu

namespace cwgpu {
/// Variant of k_tensor_intt_r with one tensor component per CTA (grid P * J * 3): 64 registers,
/// two CTAs per SM whose barrier phases interleave.
template <int LOGN>
__global__ void __launch_bounds__(NttGeom<LOGN>::T, LOGN >= 14 ? 1 : 2) k_tensor_intt_c(
    const u32* __restrict__ prepA, const u32* __restrict__ idxA, const u32* __restrict__ prepB,
    const u32* __restrict__ idxB, u32 P, DevTab T, u32* __restrict__ D) {
    using G = NttGeom<LOGN>;
    extern __shared__ u32 smd[];
    const u32 J = T.J;
    const u32 tid = threadIdx.x;
    const u32 comp = blockIdx.x % 3, pj = blockIdx.x / 3;
    const u32 pr = pj / J, j = pj % J;
    const u32 p = T.a[j], pinv = T.apinv[j];
    const size_t per = (size_t)2 * J * G::N;
    const u32* A = prepA + (size_t)(idxA ? idxA[pr] : pr) * per + (size_t)j * G::N + (tid << 4);
    const u32* B = prepB + (size_t)(idxB ? idxB[pr] : pr) * per + (size_t)j * G::N + (tid << 4);
    const size_t o1 = (size_t)J * G::N;
    u32 v[1][16];
#pragma unroll
    for (int r = 0; r < 16; r += 4) {
        if (comp == 0) {
            const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(A + r)), y0 = __ldg(reinterpret_cast<const uint4*>(B + r));
            v[0][r] = red32(mont32(x0.x, y0.x, p, pinv), p); v[0][r + 1] = red32(mont32(x0.y, y0.y, p, pinv), p);
            v[0][r + 2] = red32(mont32(x0.z, y0.z, p, pinv), p); v[0][r + 3] = red32(mont32(x0.w, y0.w, p, pinv), p);
        } else if (comp == 2) {
            const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(A + o1 + r)), y1 = __ldg(reinterpret_cast<const uint4*>(B + o1 + r));
            v[0][r] = red32(mont32(x1.x, y1.x, p, pinv), p); v[0][r + 1] = red32(mont32(x1.y, y1.y, p, pinv), p);
            v[0][r + 2] = red32(mont32(x1.z, y1.z, p, pinv), p); v[0][r + 3] = red32(mont32(x1.w, y1.w, p, pinv), p);
        } else {
            const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(A + r)), y0 = __ldg(reinterpret_cast<const uint4*>(B + r));
            const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(A + o1 + r)), y1 = __ldg(reinterpret_cast<const uint4*>(B + o1 + r));
            v[0][r] = red32(mont32(x0.x, y1.x, p, pinv), p) + red32(mont32(x1.x, y0.x, p, pinv), p);
            v[0][r + 1] = red32(mont32(x0.y, y1.y, p, pinv), p) + red32(mont32(x1.y, y0.y, p, pinv), p);
            v[0][r + 2] = red32(mont32(x0.z, y1.z, p, pinv), p) + red32(mont32(x1.z, y0.z, p, pinv), p);
            v[0][r + 3] = red32(mont32(x0.w, y1.w, p, pinv), p) + red32(mont32(x1.w, y0.w, p, pinv), p);
        }
    }
    ntt32_inv_reg<LOGN, 1>(v, smd, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, p);
    const u32 ni = T.ninvRA[j], nis = T.ninvRA_s[j];
    u32* out = D + (((size_t)pr * 3 + comp) * J + j) * G::N;
#pragma unroll
    for (int r = 0; r < 16; ++r) out[((u32)r << (LOGN - 4)) | tid] = red32(shoup32(v[0][r], ni, nis, p), p);
}
}  // namespace cwgpu

// sm_100a kernels for the constant-weight PIR server answer.
//
// Reference functions replaced (all under /root/reference/proj/core/src):
//   k_ntt64 / ntt64 smem     RingContext::ntt_forward / ntt_inverse   ring.cpp:78-144
//   k_ntt32                  same transform over the 31-bit aux / MAC primes (our basis)
//   k_decompose              decompose_digits + crt_q                 bfv.cpp:316-339, 197-209
//   k_ks_mac                 key_switch accumulation                  bfv.cpp:352-363
//   k_expand_combine         expand_one node update                   expansion.cpp:55-59,
//                            automorphism / monomial_mul              ring.cpp:296-331
//   k_lift                   to_aux_basis                             bfv.cpp:718-744
//   k_tensor_intt            mul_lazy_prepared tensor + INTT          bfv.cpp:776-791
//   k_round_chain            exact scale-and-round t/q                bfv.cpp:811-849
//   (payload MAC: k_ntt_mac in ntt_mac.cuh, k_mac2 in ntt_reg.cuh, k_mac_tma in mac.cuh: weighted_sum bfv.cpp:944-986)
//   k_relin_add              relinearize                              bfv.cpp:859-869
#pragma once
#include "devtab.h"
#include "modarith.cuh"

namespace cwgpu {

typedef long long i64;

// ============================================================== NTT in shared memory
// Chain primes: Harvey lazy butterflies exactly as ring.cpp:78-144 ([0,4q) ranges).
__device__ __forceinline__ void ntt64_fwd_smem(u64* sm, u32 N, u32 logN, const u64* rp, const u64* rps, u64 q) {
    const u64 tq = 2 * q;
    u32 logt = logN - 1;
    for (u32 m = 1; m < N; m <<= 1, --logt) {
        const u32 t = 1u << logt;
        for (u32 k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
            const u32 ii = k >> logt, jj = k & (t - 1);
            const u32 lo = (ii << (logt + 1)) + jj, hi = lo + t;
            const u64 w = __ldg(rp + m + ii), ws = __ldg(rps + m + ii);
            u64 u = sm[lo];
            if (u >= tq) u -= tq;
            const u64 v = shoup64(sm[hi], w, ws, q);
            sm[lo] = u + v;
            sm[hi] = u - v + tq;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void ntt64_inv_smem(u64* sm, u32 N, u32 logN, const u64* rp, const u64* rps, u64 q) {
    const u64 tq = 2 * q;
    u32 logt = 0;
    for (u32 m = N; m > 1; m >>= 1, ++logt) {
        const u32 h = m >> 1, t = 1u << logt;
        for (u32 k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
            const u32 ii = k >> logt, jj = k & (t - 1);
            const u32 lo = (ii << (logt + 1)) + jj, hi = lo + t;
            const u64 w = __ldg(rp + h + ii), ws = __ldg(rps + h + ii);
            const u64 u = sm[lo], v = sm[hi];
            u64 s = u + v;
            if (s >= tq) s -= tq;
            sm[lo] = s;
            sm[hi] = shoup64(u - v + tq, w, ws, q);
        }
        __syncthreads();
    }
}

// 31-bit primes: values kept in [0, 2p) (2p < 2^32).
__device__ __forceinline__ void ntt32_fwd_smem(u32* sm, u32 N, u32 logN, const u32* rp, const u32* rps, u32 p) {
    u32 logt = logN - 1;
    for (u32 m = 1; m < N; m <<= 1, --logt) {
        const u32 t = 1u << logt;
        for (u32 k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
            const u32 ii = k >> logt, jj = k & (t - 1);
            const u32 lo = (ii << (logt + 1)) + jj, hi = lo + t;
            const u32 w = __ldg(rp + m + ii), ws = __ldg(rps + m + ii);
            const u32 u = red32(sm[lo], p);
            const u32 v = red32(shoup32(sm[hi], w, ws, p), p);
            sm[lo] = u + v;
            sm[hi] = u - v + p;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void ntt32_inv_smem(u32* sm, u32 N, u32 logN, const u32* rp, const u32* rps, u32 p) {
    u32 logt = 0;
    for (u32 m = N; m > 1; m >>= 1, ++logt) {
        const u32 h = m >> 1, t = 1u << logt;
        for (u32 k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
            const u32 ii = k >> logt, jj = k & (t - 1);
            const u32 lo = (ii << (logt + 1)) + jj, hi = lo + t;
            const u32 w = __ldg(rp + h + ii), ws = __ldg(rps + h + ii);
            const u32 u = red32(sm[lo], p), v = red32(sm[hi], p);
            sm[lo] = u + v;
            sm[hi] = shoup32(u - v + p, w, ws, p);
        }
        __syncthreads();
    }
}

/// Batched 64-bit NTT over chain primes; poly p uses prime p % L.
/// SRC_DIGITS: input row (p / L) of a digit array, reduced mod q_i (bfv.cpp:355-358).
template <bool INV, bool SRC_DIGITS>
__global__ void k_ntt64(u64* __restrict__ dst, const u64* __restrict__ src, DevTab T) {
    extern __shared__ u64 sm64[];
    const u32 N = T.N;
    const u32 p = blockIdx.x, i = p % T.L;
    const u64 q = T.q[i];
    const u64* s = SRC_DIGITS ? src + (size_t)(p / T.L) * N : dst + (size_t)p * N;
    for (u32 x = threadIdx.x; x < N; x += blockDim.x) {
        u64 v = s[x];
        if (SRC_DIGITS && v >= q) v %= q;
        sm64[x] = v;
    }
    __syncthreads();
    u64* o = dst + (size_t)p * N;
    if (!INV) {
        ntt64_fwd_smem(sm64, N, T.logN, T.crp + (size_t)i * N, T.crps + (size_t)i * N, q);
        const u64 tq = 2 * q;
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) {
            u64 v = sm64[x];
            if (v >= tq) v -= tq;
            if (v >= q) v -= q;
            o[x] = v;
        }
    } else {
        ntt64_inv_smem(sm64, N, T.logN, T.cirp + (size_t)i * N, T.cirps + (size_t)i * N, q);
        const u64 ni = T.ninv[i], nis = T.ninv_s[i];
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) {
            u64 v = shoup64(sm64[x], ni, nis, q);
            if (v >= q) v -= q;
            o[x] = v;
        }
    }
}

/// Batched 32-bit NTT over aux primes. Poly p: group g = p / gs, prime j = off + p % gs,
/// address (g * stride + j) * N.  scale: 0 = N^-1, 1 = (N 2^32)^-1 (Montgomery undo).
template <bool INV>
__global__ void k_ntt32(u32* __restrict__ base, DevTab T, u32 gs, u32 stride, u32 off, int scale) {
    extern __shared__ u32 sm32[];
    const u32 N = T.N;
    const u32 p = blockIdx.x, g = p / gs, j = off + p % gs;
    const u32 pr = T.a[j];
    u32* d = base + ((size_t)g * stride + j) * N;
    for (u32 x = threadIdx.x; x < N; x += blockDim.x) sm32[x] = d[x];
    __syncthreads();
    if (!INV) {
        ntt32_fwd_smem(sm32, N, T.logN, T.arp + (size_t)j * N, T.arps + (size_t)j * N, pr);
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) d[x] = red32(sm32[x], pr);
    } else {
        ntt32_inv_smem(sm32, N, T.logN, T.airp + (size_t)j * N, T.airps + (size_t)j * N, pr);
        const u32 ni = scale ? T.ninvRA[j] : T.ninvA[j], nis = scale ? T.ninvRA_s[j] : T.ninvA_s[j];
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) d[x] = red32(shoup32(sm32[x], ni, nis, pr), pr);
    }
}

// ============================================================== multiword helpers (32-bit limbs)
// X (kQW+2 limbs) += y * src (n limbs) << (32 * OFF)
template <u32 OFF>
__device__ __forceinline__ void mw_mac(u32* X, const u32* src, u32 n, u32 y) {
    constexpr u32 off = OFF;
    u64 c = 0;
#pragma unroll
    for (u32 k = 0; k < kQW; ++k) {
        if (k < n) {
            u64 cur = (u64)X[k + off] + (u64)y * __ldg(src + k) + c;
            X[k + off] = (u32)cur;
            c = cur >> 32;
        }
    }
#pragma unroll
    for (u32 k = 0; k < kQW + 2; ++k) {
        if (k >= n + off && c) {
            u64 cur = (u64)X[k] + c;
            X[k] = (u32)cur;
            c = cur >> 32;
        }
    }
}

// X -= y * src (n limbs); caller guarantees no underflow.
__device__ __forceinline__ void mw_msub(u32* X, const u32* src, u32 n, u32 y) {
    u64 c = 0;
    u32 br = 0;
#pragma unroll
    for (u32 k = 0; k < kQW + 2; ++k) {
        u64 pk = (k < n ? (u64)y * __ldg(src + k) : 0) + c;
        c = pk >> 32;
        const u32 pl = (u32)pk, x = X[k];
        const u32 r1 = x - pl;
        const u32 b1 = x < pl;
        const u32 r2 = r1 - br;
        const u32 b2 = r1 < br;
        X[k] = r2;
        br = b1 | b2;
    }
}

// X >= src (n limbs)?
__device__ __forceinline__ bool mw_ge(const u32* X, const u32* src, u32 n) {
    int res = 1;  // equal -> ge
#pragma unroll
    for (int k = kQW + 1; k >= 0; --k) {
        const u32 s = (u32)k < n ? __ldg(src + k) : 0u;
        if (res == 1 && X[k] != s) res = X[k] > s ? 2 : 0;
    }
    return res != 0;
}

/// CRT of chain residues y_i (already multiplied by (q/q_i)^-1) into the integer
/// x = sum y_i (q/q_i) - alpha q in [0, q) (32-bit limbs), alpha from the fractional
/// estimate (an underestimate by at most one) then corrected (crt_q, bfv.cpp:197-209).
/// Returns alpha.
__device__ __forceinline__ u32 crt_exact(const u64* y, u32 alpha_est, const DevTab& T, u32* X) {
#pragma unroll
    for (u32 k = 0; k < kQW + 2; ++k) X[k] = 0;
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {  // unrolled with a uniform guard: y stays in registers
        if (i < (int)T.L) {
            mw_mac<0>(X, T.qov + (size_t)i * T.QW, T.QW, (u32)y[i]);
            mw_mac<1>(X, T.qov + (size_t)i * T.QW, T.QW, (u32)(y[i] >> 32));
        }
    }
    mw_msub(X, T.qw, T.QW, alpha_est);
    if (mw_ge(X, T.qw, T.QW)) {
        mw_msub(X, T.qw, T.QW, 1u);
        return alpha_est + 1;
    }
    return alpha_est;
}

/// y_i = res_i (q/q_i)^-1 mod q_i and the fractional sum of y_i / q_i
/// (integer part in *ip, 64-bit fraction returned; underestimate by < 2L units).
__device__ __forceinline__ u64 crt_prepare(const u64* res, const DevTab& T, u64* y, u32* ip) {
    u64 lo = 0;
    u32 carry = 0;
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        if (i < (int)T.L) {
            const u64 q = T.q[i];
            y[i] = red64(shoup64(res[i], T.muq[i], T.muq_s[i], q), q);
            const u64 f = frac64(y[i], T.q_gh[i], T.q_gl[i]);
            lo += f;
            carry += (lo < f);
        }
    }
    *ip = carry;
    return lo;
}

/// rho = round(sum y_i / q_i): x > floor(q/2) decides (bfv.cpp:731).  Exact: the
/// fractional estimate decides unless it lies within its error band below 1/2.
__device__ __noinline__ u32 crt_round_exact(const u64* y, u32 ip, const DevTab& T) {
    u32 X[kQW + 2];
    const u32 alpha = crt_exact(y, ip, T, X);
    u32 c = 0;  // X <- 2X
#pragma unroll
    for (u32 k = 0; k < kQW + 2; ++k) {
        const u32 nv = (X[k] << 1) | c;
        c = X[k] >> 31;
        X[k] = nv;
    }
    atomicAdd(T.fallbacks, 1ull);
    return alpha + (mw_ge(X, T.qw, T.QW) ? 1u : 0u);  // 2X >= q <=> 2X > q (q odd)
}

__device__ __forceinline__ u32 crt_round(const u64* y, u32 ip, u64 frac, const DevTab& T) {
    if (T.force_exact) return crt_round_exact(y, ip, *T.self);
    if (frac >= (1ull << 63)) return ip + 1;
    if (frac < (1ull << 63) - 2ull * T.L - 2ull) return ip;
    return crt_round_exact(y, ip, *T.self);
}

// ============================================================== expansion / key switching
/// Digit decomposition (bfv.cpp:316-339) of B polys (each L x N at polys + b*stride),
/// optionally through the automorphism with inverse exponent ginv (0 = identity).
/// digits: [B][D][N].
/// AUX (key switching through the aux primes, ks32.cuh): digit d is written as its residues
/// mod the first K aux primes, u32 [B][D][K][N] at aux_out (digits < 2^29 need no reduction).
/// crt_exact with the limb products accumulated column-wise (independent across limbs: no
/// carry chain through the L x 2 x QW products, one carry pass at the end) and the q / q_i limbs
/// read from shared memory (sqov [L][QW], sqw [QW]).
__device__ __forceinline__ void crt_exact_cols(const u64* y, u32 alpha_est, const DevTab& T, const u32* sqov,
                                               const u32* sqw, u32* X) {
    const u32 QW = T.QW, L = T.L;
    u64 col[kQW + 2];
#pragma unroll
    for (int w = 0; w < kQW + 2; ++w) col[w] = 0;
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        if (i >= (int)L) break;
        const u32 y0 = (u32)y[i], y1 = (u32)(y[i] >> 32);
#pragma unroll
        for (int w = 0; w < kQW; ++w) {
            if (w < (int)QW) {
                const u32 qv = sqov[i * QW + w];
                const u64 p0 = (u64)y0 * qv, p1 = (u64)y1 * qv;
                col[w] += (u32)p0;
                col[w + 1] += (p0 >> 32) + (u32)p1;
                col[w + 2] += p1 >> 32;
            }
        }
    }
    // carried sum S, then X = S - alpha_est q (alpha_est < 2^8) and one correction
    u32 S[kQW + 2];
    u64 carry = 0;
#pragma unroll
    for (int w = 0; w < kQW + 2; ++w) {
        const u64 s = col[w] + carry;
        S[w] = (u32)s;
        carry = s >> 32;
    }
    u64 c = 0;
    u32 bb = 0;
#pragma unroll
    for (int w = 0; w < kQW + 2; ++w) {
        const u64 pk = (w < (int)QW ? (u64)alpha_est * sqw[w] : 0) + c;
        c = pk >> 32;
        const u32 pl = (u32)pk, x = S[w];
        const u32 r1 = x - pl, b1 = x < pl;
        const u32 r2 = r1 - bb, b2 = r1 < bb;
        X[w] = r2;
        bb = b1 | b2;
    }
    // one correction: X >= q -> X - q (the fractional estimate is short by at most one)
    int ge = 1;
#pragma unroll
    for (int w = kQW + 1; w >= 0; --w) {
        const u32 qv = w < (int)QW ? sqw[w] : 0u;
        if (ge == 1 && X[w] != qv) ge = X[w] > qv ? 2 : 0;
    }
    if (ge != 0) {
        u32 b2 = 0;
#pragma unroll
        for (int w = 0; w < kQW + 2; ++w) {
            const u32 qv = w < (int)QW ? sqw[w] : 0u;
            const u32 r1 = X[w] - qv, c1 = X[w] < qv;
            const u32 r2 = r1 - b2, c2 = r1 < b2;
            X[w] = r2;
            b2 = c1 | c2;
        }
    }
}

template <bool AUX = false>
__global__ void k_decompose_t(const u64* __restrict__ polys, size_t stride, u64 ginv, u32 B, u32 bits,
                              u32 D, DevTab T, u64* __restrict__ digits, u32* __restrict__ aux_out, u32 K) {
    const u32 N = T.N;
    __shared__ u32 sqov[kMaxL * kQW], sqw[kQW];
    for (u32 x = threadIdx.x; x < T.L * T.QW; x += blockDim.x) sqov[x] = T.qov[x];
    for (u32 x = threadIdx.x; x < T.QW; x += blockDim.x) sqw[x] = T.qw[x];
    __syncthreads();
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * N) return;
    const u32 b = (u32)(idx / N), n = (u32)(idx % N);
    const u64* pb = polys + (size_t)b * stride;
    u32 src = n;
    bool neg = false;
    if (ginv) {
        const u32 s = (u32)(((u64)n * ginv) & (2 * N - 1));
        neg = s >= N;
        src = neg ? s - N : s;
    }
    u64 res[kMaxL];
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        if (i < (int)T.L) {
            u64 v = pb[(size_t)i * N + src];
            if (neg && v) v = T.q[i] - v;
            res[i] = v;
        }
    }
    u64* out = digits + (size_t)b * D * N + n;
    auto put = [&](u32 d, u64 v) {
        if constexpr (AUX) {
            u32* o = aux_out + ((size_t)b * D + d) * K * N + n;
            for (u32 j = 0; j < K; ++j) o[(size_t)j * N] = (bits && bits <= 29) ? (u32)v : (u32)(v % T.a[j]);
        } else {
            out[(size_t)d * N] = v;
        }
    };
    if (bits == 0) {  // one RNS digit per chain prime (bfv.cpp:320-323)
#pragma unroll
        for (int d = 0; d < kMaxL; ++d)
            if (d < (int)D) put(d, res[d]);
        return;
    }
    u64 y[kMaxL];
    u32 ip;
    crt_prepare(res, T, y, &ip);
    u32 X[kQW + 2];
    crt_exact_cols(y, ip, T, sqov, sqw, X);
    if (bits == 16) {  // the configured digit width: limb and shift are compile-time per unrolled digit
#pragma unroll
        for (int d = 0; d < 2 * kQW; ++d)
            if (d < (int)D) put(d, (X[d >> 1] >> (16 * (d & 1))) & 0xffffu);
        return;
    }
    const u64 mask = (bits == 64) ? ~0ull : ((1ull << bits) - 1);
    for (u32 d = 0; d < D; ++d) {
        const u32 bit = d * bits, limb = bit >> 5, off = bit & 31;
        u64 v = 0;
        // gather 96 bits starting at limb
        u32 l0 = 0, l1 = 0, l2 = 0;
#pragma unroll
        for (u32 k = 0; k < kQW + 2; ++k) {
            if (k == limb) l0 = X[k];
            if (k == limb + 1) l1 = X[k];
            if (k == limb + 2) l2 = X[k];
        }
        const u64 lo64 = ((u64)l1 << 32) | l0;
        v = lo64 >> off;
        if (off) v |= ((u64)l2 << (64 - off));
        put(d, v & mask);
    }
}


/// ks[b][k][i][n] = sum_d dntt[b][d][i][n] * key[d][k][i][n] mod q_i (key_switch MAC).
__global__ void k_ks_mac(const u64* __restrict__ dntt, const u64* __restrict__ key, u32 B, u32 D, DevTab T,
                         u64* __restrict__ ks) {
    const u32 N = T.N, L = T.L;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = (size_t)2 * L * N;
    if (idx >= (size_t)B * per) return;
    const u32 b = (u32)(idx / per);
    const u32 rem = (u32)(idx % per);
    const u32 k = rem / (L * N), i = (rem / N) % L, n = rem % N;
    u64 hi = 0, lo = 0;
    const u64* dp = dntt + ((size_t)b * D * L + i) * N + n;
    const u64* kp = key + ((size_t)k * L + i) * N + n;
    for (u32 d = 0; d < D; ++d) mac128(hi, lo, dp[(size_t)d * L * N], __ldg(kp + (size_t)d * 2 * L * N));
    ks[idx] = reduce128(hi, lo, T.q[i], T.q_mu96[i]);
}

/// Gathered expansion shards (rank-major: shard r holds global leaves r, r + W, r + 2W, ...,
/// `per_shard` of them) -> entries in global order, the first m leaves.  Words per entry: wpe.
__global__ void k_unshard(const u64* __restrict__ shards, u32 m, u32 W, u32 per_shard, size_t wpe,
                          u64* __restrict__ entries) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)m * wpe) return;
    const u32 e = (u32)(idx / wpe);
    const size_t w = idx % wpe;
    entries[idx] = shards[((size_t)(e % W) * per_shard + e / W) * wpe + w];
}

/// One expansion level node update for all B ciphertexts (expansion.cpp:55-59):
///   sub = (auto_g(c0) + ks0, ks1)
///   out[b]     = ct_b + sub
///   out[b + partner] = x^(-2^a) (ct_b - sub)   (partner = 2^a)
__global__ void k_expand_combine(const u64* __restrict__ in, const u64* __restrict__ ks, u32 B, u32 partner,
                                 u64 ginv, u32 shift, DevTab T, u64* __restrict__ out) {
    const u32 N = T.N, L = T.L;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * L * N) return;
    const u32 plane = (u32)(idx >> T.logN), e = (u32)idx & (N - 1);  // N is a power of two
    const u32 b = plane / L, i = plane % L;
    const u64 q = T.q[i];
    const size_t LN = (size_t)L * N;
    const u64* c0 = in + (size_t)b * 2 * LN + (size_t)i * N;
    const u64* c1 = c0 + LN;
    const u64* k0 = ks + (size_t)b * 2 * LN + (size_t)i * N;
    const u64* k1 = k0 + LN;
    auto auto_c0 = [&](u32 x) -> u64 {
        const u32 s = (u32)(((u64)x * ginv) & (2 * N - 1));
        if (s < N) return c0[s];
        const u64 v = c0[s - N];
        return v ? q - v : 0;
    };
    auto addq = [&](u64 a, u64 c) { u64 s = a + c; return s >= q ? s - q : s; };
    auto subq = [&](u64 a, u64 c) { return a >= c ? a - c : a + q - c; };
    // out[b] at e
    const u64 s0e = addq(auto_c0(e), k0[e]), s1e = k1[e];
    u64* o0 = out + (size_t)b * 2 * LN + (size_t)i * N;
    o0[e] = addq(c0[e], s0e);
    o0[LN + e] = addq(c1[e], s1e);
    // out[b + B] at e: source index x = (e + 2^a) mod 2N
    const u32 sm = (e + shift) & (2 * N - 1);
    const bool neg = sm >= N;
    const u32 x = neg ? sm - N : sm;
    const u64 s0x = addq(auto_c0(x), k0[x]), s1x = k1[x];
    u64 v0 = subq(c0[x], s0x), v1 = subq(c1[x], s1x);
    if (neg) {
        v0 = v0 ? q - v0 : 0;
        v1 = v1 ? q - v1 : 0;
    }
    u64* o1 = out + (size_t)(b + partner) * 2 * LN + (size_t)i * N;
    o1[e] = v0;
    o1[LN + e] = v1;
}

/// out2[r][p] = (c0 + ks0, c1 + ks1) of product p of group r with the group's shared key switch
/// ks[r] (ct3 [R][np][3][L][N], ks [R][2][L][N], out2 [R][np][2][L][N]).
__global__ void k_relin_add_shared(const u64* __restrict__ ct3, u32 R, u32 np, const u64* __restrict__ ks, DevTab T,
                                   u64* __restrict__ out2) {
    const u32 N = T.N, L = T.L;
    const size_t LN = (size_t)L * N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)R * np * 2 * LN) return;
    // N is a power of two: plane index by shift, then 32-bit divisions (no 64-bit div / mod)
    const u32 plane = (u32)(idx >> T.logN), n = (u32)idx & (N - 1);
    const u32 rp = plane / (2 * L), xp = plane % (2 * L);
    const u32 r = rp / np;
    const size_t x = (size_t)xp * N + n;
    const u64 q = T.q[xp % L];
    const u64 s = ct3[(size_t)rp * 3 * LN + x] + ks[(size_t)r * 2 * LN + x];
    out2[idx] = s >= q ? s - q : s;
}

/// out2 = (c0 + ks0, c1 + ks1) for B ciphertexts; ct3 stride 3LN, ks stride 2LN (relinearize).
__global__ void k_relin_add(const u64* __restrict__ ct3, size_t ct_stride, const u64* __restrict__ ks, u32 B,
                            DevTab T, u64* __restrict__ out2) {
    const u32 N = T.N, L = T.L;
    const size_t LN = (size_t)L * N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * 2 * LN) return;
    const size_t b = idx / (2 * LN), r = idx % (2 * LN);
    const u32 i = (u32)((r / N) % L);
    const u64 q = T.q[i];
    u64 s = ct3[b * ct_stride + r] + ks[idx];
    out2[idx] = s >= q ? s - q : s;
}

// ============================================================== aux / MAC lift
/// Centred lift of chain ciphertexts into aux residues (to_aux_basis, bfv.cpp:718-744):
/// for count ciphertexts (2 comps each, ct c at src + sel(c) * src_stride),
/// out[c][k][j][n] for j < nj, constants mont (x 2^32, tensor operands) or plain.
__global__ void __launch_bounds__(256) k_lift(const u64* __restrict__ src, size_t src_stride, const u32* __restrict__ sel,
                                             u32 count, u32 nj, int mont, DevTab T, u32* __restrict__ out,
                                             u32 out_stride_j) {
    // per-prime lift constants staged in shared memory once per CTA (they were L1 loads inside the
    // L x nj loop: 2 L nj loads per coefficient)
    __shared__ u32 sV[kMaxL * kMaxJ], sV2[kMaxL * kMaxJ], sW[kMaxJ], sA[kMaxJ];
    __shared__ u64 sAb[kMaxJ];
    const u32 N = T.N, L = T.L;
    {
        const u32* V = mont ? T.liftV_m : T.liftV_n;
        const u32* V2 = mont ? T.liftV2_m : T.liftV2_n;
        const u32* W = mont ? T.liftW_m : T.liftW_n;
        for (u32 x = threadIdx.x; x < L * nj; x += blockDim.x) {
            const u32 i = x / nj, j = x % nj;
            sV[x] = V[i * T.J + j];
            sV2[x] = V2[i * T.J + j];
        }
        for (u32 j = threadIdx.x; j < nj; j += blockDim.x) {
            sW[j] = W[j];
            sA[j] = T.a[j];
            sAb[j] = T.abar[j];
        }
        __syncthreads();
    }
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)count * 2 * N) return;
    const u32 c = (u32)(idx / (2 * N)), k = (u32)((idx / N) % 2), n = (u32)(idx % N);
    const u64* s = src + (size_t)(sel ? sel[c] : c) * src_stride + (size_t)k * L * N + n;
    u64 res[kMaxL], y[kMaxL];
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) res[i] = i < (int)L ? s[(size_t)i * N] : 0;
    u32 ip;
    const u64 fr = crt_prepare(res, T, y, &ip);
    const u32 rho = crt_round(y, ip, fr, T);
    // y_i < 2^60 split 30 | 30 bits: sum_i ylo V + yhi V2 < L 2^61 (L <= 8: < 2^64), one reduction per prime
    u32 ylo[kMaxL], yhi[kMaxL];
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        ylo[i] = i < (int)L ? (u32)(y[i] & ((1u << 30) - 1)) : 0u;
        yhi[i] = i < (int)L ? (u32)(y[i] >> 30) : 0u;
    }
    u32* o = out + ((size_t)c * 2 + k) * out_stride_j * N + n;
    for (u32 j = 0; j < nj; ++j) {
        const u32 a = sA[j];
        u64 acc = 0;
#pragma unroll
        for (int i = 0; i < kMaxL; ++i)
            if (i < (int)L) acc += (u64)ylo[i] * sV[i * nj + j] + (u64)yhi[i] * sV2[i * nj + j];
        const u64 ab = sAb[j];
        o[(size_t)j * N] = red32(bar64(acc, a, ab) + bar64((u64)rho * (a - sW[j]), a, ab), a);
    }
}

// ============================================================== tensor + INTT (aux)
/// Tensor product of prepared operands (mul_lazy_prepared, bfv.cpp:776-791) for P
/// products and one aux prime per CTA, then INTT; D[p][comp][j][N] normal form.
__global__ void k_tensor_intt(const u32* __restrict__ prepA, const u32* __restrict__ idxA,
                              const u32* __restrict__ prepB, const u32* __restrict__ idxB, u32 P, DevTab T,
                              u32* __restrict__ D) {
    extern __shared__ u32 sm32[];
    const u32 N = T.N, J = T.J;
    const u32 pr = blockIdx.x / J, j = blockIdx.x % J;
    const u32 p = T.a[j], pinv = T.apinv[j];
    const size_t per = (size_t)2 * J * N;
    const u32* A = prepA + (size_t)(idxA ? idxA[pr] : pr) * per + (size_t)j * N;
    const u32* B = prepB + (size_t)(idxB ? idxB[pr] : pr) * per + (size_t)j * N;
    const size_t o1 = (size_t)J * N;
    for (u32 comp = 0; comp < 3; ++comp) {
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) {
            u32 d;
            if (comp == 0) {
                d = red32(mont32(A[x], B[x], p, pinv), p);
            } else if (comp == 1) {
                d = red32(mont32(A[x], B[o1 + x], p, pinv), p) + red32(mont32(A[o1 + x], B[x], p, pinv), p);
            } else {
                d = red32(mont32(A[o1 + x], B[o1 + x], p, pinv), p);
            }
            sm32[x] = d;
        }
        __syncthreads();
        ntt32_inv_smem(sm32, N, T.logN, T.airp + (size_t)j * N, T.airps + (size_t)j * N, p);
        const u32 ni = T.ninvRA[j], nis = T.ninvRA_s[j];
        u32* out = D + (((size_t)pr * 3 + comp) * T.DS + j) * N;
        for (u32 x = threadIdx.x; x < N; x += blockDim.x) out[x] = red32(shoup32(sm32[x], ni, nis, p), p);
        __syncthreads();
    }
}

// ============================================================== exact scale-and-round
struct HpsState {
    u32 w[kMaxJ];
    u32 gamma;
    i64 rho;       // round(sum w_j F_j - gamma F_A)
    bool exact;    // fast path decided
};

/// HPS scaling: r = sum_j w_j I_j - gamma I_A + round(sum_j w_j F_j - gamma F_A), with
/// t (A/a_j) = I_j q + F_j q.  Returns false when the 96-bit fractional estimate cannot
/// decide the rounding (then the exact multiword path runs).
__device__ __forceinline__ bool hps_prepare(const u32* __restrict__ Dp, size_t jstride, const DevTab& T, HpsState& h) {
    const u32 J = T.J;
    u64 gs = 0;
    u32 s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (u32 j = 0; j < J; ++j) {
        const u32 a = T.a[j];
        const u32 w = red32(shoup32(Dp[(size_t)j * jstride], T.chat[j], T.chat_s[j], a), a);
        h.w[j] = w;
        gs += (u64)w * T.aF[j];
        const u32 f0 = T.frac96[3 * j], f1 = T.frac96[3 * j + 1], f2 = T.frac96[3 * j + 2];
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.lo.cc.u32 %1, %5, %7, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %8, %2;\n\t"
            "addc.cc.u32    %3, %3, 0;\n\t"
            "addc.u32       %4, %4, 0;\n\t"
            "mad.hi.cc.u32  %1, %5, %6, %1;\n\t"
            "madc.hi.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %8, %3;\n\t"
            "addc.u32       %4, %4, 0;\n\t"
            : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3), "+r"(s4)
            : "r"(w), "r"(f0), "r"(f1), "r"(f2));
    }
    const u32 gsh = 64 - T.gbits;
    const u32 gamma = (u32)((gs + (1ull << (gsh - 1))) >> gsh);
    h.gamma = gamma;
    // subtract gamma * fracA (96-bit) as a 128-bit value
    {
        const u32 f0 = T.fracA[0], f1 = T.fracA[1], f2 = T.fracA[2];
        const u64 p0 = (u64)gamma * f0, p1 = (u64)gamma * f1, p2 = (u64)gamma * f2;
        // P = p0 + p1 << 32 + p2 << 64
        u32 q0 = (u32)p0;
        u64 t1 = (p0 >> 32) + (u32)p1;
        u32 q1 = (u32)t1;
        u64 t2 = (t1 >> 32) + (p1 >> 32) + (u32)p2;
        u32 q2 = (u32)t2;
        u64 t3 = (t2 >> 32) + (p2 >> 32);
        u32 q3 = (u32)t3;
        asm("sub.cc.u32  %0, %0, %5;\n\t"
            "subc.cc.u32 %1, %1, %6;\n\t"
            "subc.cc.u32 %2, %2, %7;\n\t"
            "subc.cc.u32 %3, %3, %8;\n\t"
            "subc.u32    %4, %4, 0;\n\t"
            : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3), "+r"(s4)
            : "r"(q0), "r"(q1), "r"(q2), "r"(q3));
    }
    // + 1/2
    asm("add.cc.u32  %0, %0, 0x80000000;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.u32    %2, %2, 0;\n\t"
        : "+r"(s2), "+r"(s3), "+r"(s4));
    h.rho = (i64)(((u64)s4 << 32) | s3);
    // estimate error in (-J, J 2^31) units of 2^-96: undecidable near a wrap of the low 96 bits
    const bool bad = (s2 == 0u && s1 == 0u) || (s2 == 0xffffffffu && s1 >= 0xffffff00u) || T.force_exact;
    h.exact = !bad;
    return !bad;
}

/// Exact slow path: D = sum_j w_j (A/a_j) - gamma A (signed), r = sign(D) round(|D| t / q)
/// by long division (bfv.cpp:811-849). Writes the magnitude limbs into R and returns sign.
__device__ __noinline__ bool round_exact(const HpsState& h, const DevTab& T, u32* R /*kAW+2*/) {
    u32 Dm[kAW + 2];
    for (u32 k = 0; k < kAW + 2; ++k) Dm[k] = 0;
    for (u32 j = 0; j < T.J; ++j) {
        u64 c = 0;
        const u32* src = T.Aov + (size_t)j * T.AW;
        for (u32 k = 0; k < T.AW; ++k) {
            u64 cur = (u64)Dm[k] + (u64)h.w[j] * src[k] + c;
            Dm[k] = (u32)cur;
            c = cur >> 32;
        }
        for (u32 k = T.AW; k < kAW + 2 && c; ++k) {
            u64 cur = (u64)Dm[k] + c;
            Dm[k] = (u32)cur;
            c = cur >> 32;
        }
    }
    // Dm - gamma * A ; if negative, negate
    u32 G[kAW + 2];
    {
        u64 c = 0;
        for (u32 k = 0; k < kAW + 2; ++k) {
            u64 cur = (k < T.AW ? (u64)h.gamma * T.Aw[k] : 0) + c;
            G[k] = (u32)cur;
            c = cur >> 32;
        }
    }
    bool neg = false;
    {
        int cmp = 0;
        for (int k = kAW + 1; k >= 0 && !cmp; --k)
            if (Dm[k] != G[k]) cmp = Dm[k] > G[k] ? 1 : -1;
        neg = cmp < 0;
        const u32* X = neg ? G : Dm;
        const u32* Y = neg ? Dm : G;
        u32 br = 0;
        for (u32 k = 0; k < kAW + 2; ++k) {
            u64 need = (u64)Y[k] + br;
            u64 cur = X[k];
            Dm[k] = (u32)(cur - need);
            br = cur < need;
        }
    }
    // |D| * t
    {
        u64 c = 0;
        for (u32 k = 0; k < kAW + 2; ++k) {
            u64 cur = (u64)Dm[k] * (u32)T.t + c;
            Dm[k] = (u32)cur;
            c = cur >> 32;
        }
    }
    // long division by q, bitwise
    u32 Rm[kQW + 2];
    for (u32 k = 0; k < kQW + 2; ++k) Rm[k] = 0;
    for (u32 k = 0; k < kAW + 2; ++k) R[k] = 0;
    for (int bit = 32 * (kAW + 2) - 1; bit >= 0; --bit) {
        u32 c = (Dm[bit >> 5] >> (bit & 31)) & 1u;
        for (u32 k = 0; k < kQW + 2; ++k) {
            u32 nv = (Rm[k] << 1) | c;
            c = Rm[k] >> 31;
            Rm[k] = nv;
        }
        if (mw_ge(Rm, T.qw, T.QW)) {
            mw_msub(Rm, T.qw, T.QW, 1u);
            R[bit >> 5] |= 1u << (bit & 31);
        }
    }
    // round half up on the magnitude: 2 rem >= q
    {
        u32 c = 0;
        for (u32 k = 0; k < kQW + 2; ++k) {
            u32 nv = (Rm[k] << 1) | c;
            c = Rm[k] >> 31;
            Rm[k] = nv;
        }
        if (mw_ge(Rm, T.qw, T.QW)) {
            for (u32 k = 0; k < kAW + 2; ++k)
                if (++R[k]) break;
        }
    }
    atomicAdd(T.fallbacks, 1ull);
    return neg;
}

__device__ __forceinline__ u32 mag_mod32(const u32* R, u32 a, u64 abar) {
    u32 r = 0;
    for (int k = kAW + 1; k >= 0; --k) r = bar64(((u64)r << 32) | R[k], a, abar);
    return r;
}

__device__ __forceinline__ u64 mag_mod64(const u32* R, u64 q, u64 mu96) {
    u64 r = 0;
    for (int k = kAW + 1; k >= 0; --k) r = reduce96((u32)(r >> 32), (r << 32) | R[k], q, mu96);
    return r;
}

/// Round t*D/q into the chain: out[p][comp][i][n] = r mod q_i (mul_lazy_prepared output).
__global__ void k_round_chain(const u32* __restrict__ D, u32 P, DevTab T, u64* __restrict__ out) {
    const u32 N = T.N, J = T.J, L = T.L;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)P * 3 * N) return;
    const size_t pc = idx >> T.logN;
    const u32 n = (u32)(idx & (N - 1));
    const u32* Dp = D + pc * T.DS * N + n;
    u64* o = out + pc * L * N + n;
    HpsState h;
    if (hps_prepare(Dp, N, T, h)) {
        for (u32 i = 0; i < L; ++i) {
            const u64 q = T.q[i];
            u64 hi = 0, lo = 0;
            for (u32 j = 0; j < J; ++j) mac128(hi, lo, h.w[j], T.ImodQ[(size_t)j * L + i]);
            mac128(hi, lo, h.gamma, q - T.IAmodQ[i]);
            u64 r = reduce128(hi, lo, q, T.q_mu96[i]);
            // + rho (signed, |rho| < 2^40 < q)
            if (h.rho >= 0) {
                r += (u64)h.rho;
                r = red64(r, q);
            } else {
                const u64 m = (u64)(-h.rho);
                r = r >= m ? r - m : r + q - m;
            }
            o[(size_t)i * N] = r;
        }
    } else {
        u32 R[kAW + 2];
        const bool neg = round_exact(h, *T.self, R);
        for (u32 i = 0; i < L; ++i) {
            const u64 q = T.q[i];
            u64 r = mag_mod64(R, q, T.q_mu96[i]);
            if (neg && r) r = q - r;
            o[(size_t)i * N] = r;
        }
    }
}

// ============================================================== payload MAC
/// Summed partials -> u32 residues mod a_k (in place into a u32 plane array).
__global__ void k_partial_mod(const u64* __restrict__ partial, size_t total, DevTab T, u32* __restrict__ X) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const u32 k = (u32)((idx / T.N) % T.Mm);
    X[idx] = bar64(partial[idx], T.a[k], T.abar[k]);
}

/// MAC basis -> chain: X (coefficient form, centred |X| < M/2) -> out[g][i][n] mod q_i.
/// X layout [G][xs][N] (the first Mm planes of each group of xs); out layout [G][L][N].
constexpr int kMacToChainMm = 20;  // MAC-basis sizes handled with the residues in registers
__global__ void __launch_bounds__(128) k_mac_to_chain(const u32* __restrict__ X, u32 xs, u32 G, DevTab T,
                                                      u64* __restrict__ out) {
    // per-prime constants in shared memory, M / m_k mod q_i split into 30-bit halves: every product
    // is a 32 x 32 -> 64-bit IMAD.WIDE (< 2^60) and 16 of them fit one u64 accumulator.  The Mm
    // residues stay in registers and each output prime is one short dot product (low register use).
    __shared__ u32 sMl[kMaxJ * kMaxL], sMh[kMaxJ * kMaxL];
    __shared__ u64 sMF[kMaxJ], sQ[kMaxL], sMu[kMaxL], sNeg[kMaxL];
    __shared__ u32 sA[kMaxJ], sH[kMaxJ], sHs[kMaxJ];
    const u32 N = T.N, Mm = T.Mm, L = T.L;
    for (u32 x = threadIdx.x; x < Mm * L; x += blockDim.x) {
        const u64 v = T.Mconv[x];
        sMl[x] = (u32)(v & ((1u << 30) - 1));
        sMh[x] = (u32)(v >> 30);
    }
    for (u32 k = threadIdx.x; k < Mm; k += blockDim.x) {
        sMF[k] = T.mF[k];
        sA[k] = T.a[k];
        sH[k] = T.mhat[k];
        sHs[k] = T.mhat_s[k];
    }
    for (u32 i = threadIdx.x; i < L; i += blockDim.x) {
        sQ[i] = T.q[i];
        sMu[i] = T.q_mu96[i];
        sNeg[i] = T.MnegQ[i];
    }
    __syncthreads();
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)G * N) return;
    const size_t g = idx / N;
    const u32 n = (u32)(idx % N);
    const u32 gsh = 64 - T.gbits;
    if (Mm <= (u32)kMacToChainMm) {
        u32 v[kMacToChainMm];
        u64 gs = 0;
#pragma unroll
        for (int k = 0; k < kMacToChainMm; ++k) {
            if (k < (int)Mm) {
                const u32 a = sA[k];
                v[k] = red32(shoup32(X[(g * xs + k) * N + n], sH[k], sHs[k], a), a);
                gs += (u64)v[k] * sMF[k];
            } else {
                v[k] = 0;
            }
        }
        const u32 gamma = (u32)((gs + (1ull << (gsh - 1))) >> gsh);
        for (u32 i = 0; i < L; ++i) {
            u64 lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;  // two chains of <= 10 products each
#pragma unroll
            for (int k = 0; k < kMacToChainMm; k += 2) {
                if (k < (int)Mm) {
                    lo0 += (u64)v[k] * sMl[k * L + i];
                    hi0 += (u64)v[k] * sMh[k * L + i];
                }
                if (k + 1 < (int)Mm) {
                    lo1 += (u64)v[k + 1] * sMl[(k + 1) * L + i];
                    hi1 += (u64)v[k + 1] * sMh[(k + 1) * L + i];
                }
            }
            u64 hi = 0, lo = lo0;
            mac128(hi, lo, lo1, 1ull);
            mac128(hi, lo, hi0, 1ull << 30);
            mac128(hi, lo, hi1, 1ull << 30);
            mac128(hi, lo, gamma, sNeg[i]);
            out[(g * L + i) * N + n] = reduce128(hi, lo, sQ[i], sMu[i]);
        }
        return;
    }
    // larger MAC bases: accumulate per output prime in 128 bits
    u64 hi[kMaxL], lo[kMaxL];
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) hi[i] = lo[i] = 0;
    u64 gs = 0;
    for (u32 k = 0; k < Mm; ++k) {
        const u32 a = sA[k];
        const u32 vk = red32(shoup32(X[(g * xs + k) * N + n], sH[k], sHs[k], a), a);
        gs += (u64)vk * sMF[k];
#pragma unroll
        for (int i = 0; i < kMaxL; ++i)
            if (i < (int)L) mac128(hi[i], lo[i], vk, ((u64)sMh[k * L + i] << 30) | sMl[k * L + i]);
    }
    const u32 gamma = (u32)((gs + (1ull << (gsh - 1))) >> gsh);
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        if (i < (int)L) {
            mac128(hi[i], lo[i], gamma, sNeg[i]);
            out[(g * L + i) * N + n] = reduce128(hi[i], lo[i], sQ[i], sMu[i]);
        }
    }
}

// ============================================================== row-level helpers
/// Arithmetic-operator factors: for row r, inner = sum of its k selected
/// entries; factor f = inner + Delta (t - f) on c0's constant coefficient (add_plain,
/// bfv.cpp:641-649). out[r][f][2][L][N].
__global__ void k_arith_factors(const u64* __restrict__ entries, const u32* __restrict__ pos, u32 R, u32 k,
                                DevTab T, u64* __restrict__ out) {
    const u32 N = T.N, L = T.L;
    const size_t LN = (size_t)L * N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)R * 2 * LN) return;
    // N is a power of two: plane index by shift, then 32-bit divisions (no 64-bit div / mod)
    const u32 plane = (u32)(idx >> T.logN), n = (u32)idx & (N - 1);
    const u32 r = plane / (2 * L), pl = plane % (2 * L);
    const u32 comp = pl / L, i = pl % L;
    const size_t rem = (size_t)pl * N + n;
    const u64 q = T.q[i];
    u64 s = 0;
    for (u32 p = 0; p < k; ++p) {
        s += entries[(size_t)pos[(size_t)r * k + p] * 2 * LN + rem];
        if (s >= q) s -= q;
    }
    for (u32 f = 0; f < k; ++f) {
        u64 v = s;
        if (f > 0 && comp == 0 && n == 0) {
            const u64 m = (T.t - f) % q;
            // Delta * m mod q_i (small m < 2^31): via 128-bit reduce
            const u64 dl = T.delta[i];
            const u64 pl = dl * m, ph = __umul64hi(dl, m);
            v += reduce128(ph, pl, q, T.q_mu96[i]);
            if (v >= q) v -= q;
        }
        out[(((size_t)r * k + f) * 2) * LN + rem] = v;
    }
}

/// Arithmetic-operator factors share everything but one coefficient: f_f = k' + Delta (t - f) only
/// changes coefficient 0 of component 0 (add_plain, bfv.cpp:641-649), so the centred aux lift of
/// f_f equals that of k' except there, and the NTT of that difference is the same constant in every
/// slot.  delta[r][f][j] = (lift(f_f)_0 - lift(k')_0) mod a_j (Montgomery form, like the prepared
/// operands) from the chain residues of coefficient 0 of each factor (nodes [R][k][2][L][N]).
__global__ void k_arith_deltas(const u64* __restrict__ nodes, u32 R, u32 k, DevTab T, u32* __restrict__ delta) {
    const u32 x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= R * k) return;
    const u32 r = x / k, f = x % k;
    const u32 L = T.L, N = T.N, J = T.J;
    const size_t per = (size_t)2 * L * N;
    u32 lf[kMaxJ];
    for (int which = 0; which < 2; ++which) {  // 0: factor f, 1: factor 0 (= k')
        const u64* s = nodes + ((size_t)r * k + (which ? 0 : f)) * per;
        u64 res[kMaxL], y[kMaxL];
#pragma unroll
        for (int i = 0; i < kMaxL; ++i) res[i] = i < (int)L ? s[(size_t)i * N] : 0;
        u32 ip;
        const u64 fr = crt_prepare(res, T, y, &ip);
        const u32 rho = crt_round(y, ip, fr, T);
        for (u32 j = 0; j < J; ++j) {
            const u32 a = T.a[j];
            u64 acc = 0;
#pragma unroll
            for (int i = 0; i < kMaxL; ++i)
                if (i < (int)L)
                    acc += (u64)(u32)(y[i] & ((1u << 30) - 1)) * T.liftV_m[i * J + j] +
                           (u64)(u32)(y[i] >> 30) * T.liftV2_m[i * J + j];
            const u32 v = red32(bar64(acc, a, T.abar[j]) + bar64((u64)rho * (a - T.liftW_m[j]), a, T.abar[j]), a);
            if (which == 0) lf[j] = v;
            else delta[(size_t)x * J + j] = red32(lf[j] + a - v, a);
        }
    }
}

/// Prepared factors [R][k][2][J][N] from the prepared k' [R][2][J][N] (NTT form, Montgomery) and
/// the per-factor constants delta (component 0 only).  Block = one (row, factor, component, prime)
/// plane (indices decoded once), threads copy it as uint4.
__global__ void __launch_bounds__(256) k_prep_factors(const u32* __restrict__ pk, const u32* __restrict__ delta, u32 k,
                                                      DevTab T, u32* __restrict__ out) {
    const u32 J = T.J, N = T.N;
    const u32 plane = blockIdx.x;  // ((r k + f) 2 + comp) J + j
    const u32 j = plane % J, comp = (plane / J) % 2, rf = plane / (2 * J), r = rf / k;
    const uint4* src = reinterpret_cast<const uint4*>(pk + (((size_t)r * 2 + comp) * J + j) * N);
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)plane * N);
    const u32 a = T.a[j];
    const u32 d = comp == 0 ? delta[(size_t)rf * J + j] : 0u;
    for (u32 x = threadIdx.x; x < N / 4; x += blockDim.x) {
        uint4 v = src[x];
        if (comp == 0) {
            v.x = red32(v.x + d, a);
            v.y = red32(v.y + d, a);
            v.z = red32(v.z + d, a);
            v.w = red32(v.w + d, a);
        }
        dst[x] = v;
    }
}

/// Multiply every coefficient of B 2-comp ciphertexts by c mod q_i (plain_mul by a
/// constant polynomial, bfv.cpp:664-680).
__global__ void k_scale_const(u64* __restrict__ ct, u32 B, u64 c, DevTab T) {
    const u32 N = T.N, L = T.L;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * 2 * L * N) return;
    const u32 i = (u32)((idx / N) % L);
    const u64 q = T.q[i];
    const u64 cm = c % q;
    const u64 pl = ct[idx] * cm, ph = __umul64hi(ct[idx], cm);
    ct[idx] = reduce128(ph, pl, q, T.q_mu96[i]);
}

/// out = in * f_j mod a_j over planes [count][J][N] (Shoup constants per aux prime), canonical.
__global__ void k_scale_planes(const u32* __restrict__ in, u32* __restrict__ out, size_t total,
                               const u32* __restrict__ f, const u32* __restrict__ fs, DevTab T) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const u32 j = (u32)((idx >> T.logN) % T.J);
    const u32 p = T.a[j];
    out[idx] = red32(red32(shoup32(in[idx], f[j], fs[j], p), 2 * p), p);
}

/// Gather 2-comp ciphertexts: out[x] = src[sel[x]] (each 2LN words).
__global__ void k_gather_ct(const u64* __restrict__ src, const u32* __restrict__ sel, u32 count, size_t per,
                            u64* __restrict__ out) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)count * per) return;
    const size_t x = idx / per, o = idx % per;
    out[idx] = src[(size_t)sel[x] * per + o];
}

/// Strided ciphertext gather: out[x * out_stride + o] = src[(sel ? sel[x] : x) * src_stride + o] for
/// o < per (per-row copies of the selection path as one launch).
__global__ void k_gather_strided(const u64* __restrict__ src, size_t src_stride, const u32* __restrict__ sel,
                                 u32 count, size_t per, u64* __restrict__ out, size_t out_stride) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)count * per) return;
    const size_t x = idx / per, o = idx % per;
    out[x * out_stride + o] = src[(size_t)(sel ? sel[x] : (u32)x) * src_stride + o];
}

/// Leaf pairs of the folklore product tree (pir.cpp:294-300, eq_circuits.cpp:53-69) for rows
/// [r0, r0 + R): ia[r * np + p] = pos[r][2p], ib[...] = pos[r][2p + 1] (positions ascending).
__global__ void k_leaf_pairs(const u32* __restrict__ pos_rows, u64 r0, u32 R, u32 k, u32* __restrict__ ia,
                             u32* __restrict__ ib) {
    const u32 np = k / 2;
    const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= (size_t)R * np) return;
    const size_t r = x / np, p = x % np;
    const u32* pr = pos_rows + (r0 + r) * k;
    ia[x] = pr[2 * p];
    ib[x] = pr[2 * p + 1];
}

/// Node pairs of one product-tree level: ia[r * np + p] = r * cnt + 2p, ib = ia + 1.
__global__ void k_level_pairs(u32 R, u32 cnt, u32* __restrict__ ia, u32* __restrict__ ib) {
    const u32 np = cnt / 2;
    const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= (size_t)R * np) return;
    const u32 r = (u32)(x / np), p = (u32)(x % np);
    ia[x] = r * cnt + 2 * p;
    ib[x] = r * cnt + 2 * p + 1;
}

/// Next product-tree level [R][ncnt] from the np products per row (prod [R * np], 2-comp) and, when
/// cnt is odd, the carried last node of each row (carry + r * carry_stride, or the expanded entry
/// pos[r][k-1] when carry_pos != nullptr) (eq_circuits.cpp:53-69: an odd leftover moves up unchanged).
__global__ void k_tree_next(const u64* __restrict__ prod, u32 R, u32 np, u32 ncnt, const u64* __restrict__ carry,
                            size_t carry_stride, const u32* __restrict__ carry_pos, u64 r0, u32 k, size_t per,
                            u64* __restrict__ out) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)R * ncnt * per) return;
    const size_t o = idx % per, slot = (idx / per) % ncnt, r = idx / (per * ncnt);
    u64 v;
    if (slot < np)
        v = prod[(r * np + slot) * per + o];
    else if (carry_pos)
        v = carry[(size_t)carry_pos[(r0 + r) * k + k - 1] * per + o];
    else
        v = carry[r * carry_stride + o];
    out[idx] = v;
}

/// flag |= (a != b) over n words (evaluation-key cache: is the uploaded key set the resident one?)
__global__ void k_words_differ(const u64* __restrict__ a, const u64* __restrict__ b, size_t n,
                               unsigned int* __restrict__ flag) {
    bool d = false;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        d |= a[i] != b[i];
    if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(flag, 1u);
}

/// dst[x] += src[x] (row-shard partial accumulators: each word < 2^31, any device count < 2^32 sums)
__global__ void k_add_u64(u64* __restrict__ dst, const u64* __restrict__ src, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

}  // namespace cwgpu

namespace cwgpu {
/// DB staging: payload rows [R][N] (< t) -> [R][Mm][N] (lifted unchanged into each MAC prime,
/// prepare_plain, bfv.cpp:933-942; the NTT follows).
__global__ void k_db_spread(const u64* __restrict__ src, u64 rows, DevTab T, u32* __restrict__ dst) {
    const u32 N = T.N, Mm = T.Mm;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)rows * Mm * N) return;
    const size_t r = idx / ((size_t)Mm * N);
    const u32 n = (u32)(idx % N);
    dst[idx] = (u32)src[r * N + n];  // t < 2^31 < a_k
}

/// substitute (bfv.cpp:694-712): out = (auto_g(c0) + ks0, ks1).
__global__ void k_subst_combine(const u64* __restrict__ in, const u64* __restrict__ ks, u32 B, u64 ginv, DevTab T,
                                u64* __restrict__ out) {
    const u32 N = T.N, L = T.L;
    const size_t LN = (size_t)L * N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * LN) return;
    const u32 plane = (u32)(idx >> T.logN), e = (u32)idx & (N - 1);  // N is a power of two
    const size_t b = plane / L;
    const u32 i = plane % L;
    const u64 q = T.q[i];
    const u64* c0 = in + b * 2 * LN + (size_t)i * N;
    const u32 s = (u32)(((u64)e * ginv) & (2 * N - 1));
    u64 v = s < N ? c0[s] : (c0[s - N] ? q - c0[s - N] : 0);
    v += ks[b * 2 * LN + (size_t)i * N + e];
    if (v >= q) v -= q;
    out[b * 2 * LN + (size_t)i * N + e] = v;
    out[b * 2 * LN + LN + (size_t)i * N + e] = ks[b * 2 * LN + LN + (size_t)i * N + e];
}
}  // namespace cwgpu

// Client side on the GPU: query construction (pack_query_bits, expansion.cpp:17-38,
// with BfvBackend::encrypt, bfv.cpp:516-549) and decryption (BfvBackend::decrypt, bfv.cpp:551-595),
// bit-identical to the reference for the same secret key, key seed and encryption indices.
//
// Randomness is the reference's ChaCha20 (prf.cpp:9-83): RFC 7539 block, key = the four seed words,
// counter in word 12 (carry into 15), stream id in words 13-14; next_u64 = two consecutive block
// words.  Every word of a stream is addressable, so the streams are generated in parallel:
//   * uniform(q) is rejection sampling (accept v < 2^64 - (2^64 mod q)); a CTA per (ciphertext,
//     prime) generates the stream in 16K-word passes, ranks the accepted words with a block scan
//     and keeps the first N (rejections have probability < 2^-14 at these moduli);
//   * sample_noise = popcount(20 bits) - popcount(20 bits) of words 2n, 2n + 1;
//   * derive_seed(master, d, i) = the first four u64 of stream (d << 48) ^ i.
#pragma once
#include "devtab.h"
#include "modarith.cuh"
#include "kernels.cuh"

namespace cwgpu {

struct Seed4 {
    u64 w[4];
};

__device__ __forceinline__ u32 cc_rotl(u32 x, int n) { return (x << n) | (x >> (32 - n)); }
__device__ __forceinline__ void cc_qr(u32& a, u32& b, u32& c, u32& d) {
    a += b; d ^= a; d = cc_rotl(d, 16);
    c += d; b ^= c; b = cc_rotl(b, 12);
    a += b; d ^= a; d = cc_rotl(d, 8);
    c += d; b ^= c; b = cc_rotl(b, 7);
}

/// ChaCha20 block `counter` of stream `stream` under `seed` (prf.cpp:22-56).
__device__ void chacha_block(const Seed4& seed, u64 stream, u64 counter, u32 (&out)[16]) {
    u32 in[16];
    in[0] = 0x61707865; in[1] = 0x3320646e; in[2] = 0x79622d32; in[3] = 0x6b206574;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        in[4 + 2 * i] = (u32)seed.w[i];
        in[5 + 2 * i] = (u32)(seed.w[i] >> 32);
    }
    in[12] = (u32)counter;
    in[13] = (u32)stream;
    in[14] = (u32)(stream >> 32);
    in[15] = (u32)(counter >> 32);
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = in[i];
#pragma unroll 1
    for (int r = 0; r < 10; ++r) {
        cc_qr(out[0], out[4], out[8], out[12]);
        cc_qr(out[1], out[5], out[9], out[13]);
        cc_qr(out[2], out[6], out[10], out[14]);
        cc_qr(out[3], out[7], out[11], out[15]);
        cc_qr(out[0], out[5], out[10], out[15]);
        cc_qr(out[1], out[6], out[11], out[12]);
        cc_qr(out[2], out[7], out[8], out[13]);
        cc_qr(out[3], out[4], out[9], out[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] += in[i];
}

/// derive_seed (bfv.cpp:19-24).
__device__ Seed4 derive_seed_dev(const Seed4& master, u64 domain, u64 index) {
    u32 b[16];
    chacha_block(master, (domain << 48) ^ index, 0, b);
    Seed4 s;
#pragma unroll
    for (int i = 0; i < 4; ++i) s.w[i] = (u64)b[2 * i] | ((u64)b[2 * i + 1] << 32);
    return s;
}

/// Encryption seeds of h ciphertexts (indices first_index + q): c1 (domain 5) and noise (domain 6).
__global__ void k_enc_seeds(Seed4 sk_seed, u64 first_index, u32 h, Seed4* __restrict__ c1_seed,
                            Seed4* __restrict__ e_seed) {
    const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= h) return;
    c1_seed[q] = derive_seed_dev(sk_seed, 5, first_index + q);
    e_seed[q] = derive_seed_dev(sk_seed, 6, first_index + q);
}

/// uniform_rns (bfv.cpp:303-312): out[q][i][n] = the n-th accepted uniform(q_i) draw of stream i
/// under c1_seed[q].  Grid: h x L CTAs of 1024 threads, 16 words (2 blocks) per thread per pass.
__global__ void __launch_bounds__(1024) k_uniform_rns(const Seed4* __restrict__ seeds, DevTab T, const u64* __restrict__ limit,
                                                      u64* __restrict__ out, size_t out_stride) {
    constexpr u32 TW = 16;  // words per thread per pass
    __shared__ u32 warp_sum[32];
    __shared__ u32 base_sh;
    const u32 L = T.L, N = T.N;
    const u32 q = blockIdx.x / L, i = blockIdx.x % L;
    const Seed4 seed = seeds[q];
    const u64 p = T.q[i], lim = limit[i];
    u64* o = out + (size_t)q * out_stride + (size_t)i * N;
    const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) base_sh = 0;
    __syncthreads();
    for (u64 pass = 0;; ++pass) {
        const u32 got = base_sh;
        if (got >= N) break;
        u64 v[TW];
        u32 acc = 0;
        const u64 w0 = (pass * blockDim.x + tid) * TW;  // first word of this thread
#pragma unroll
        for (u32 b = 0; b < TW / 8; ++b) {
            u32 blk[16];
            chacha_block(seed, i, w0 / 8 + b, blk);
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                v[b * 8 + x] = (u64)blk[2 * x] | ((u64)blk[2 * x + 1] << 32);
                acc += v[b * 8 + x] < lim;
            }
        }
        // exclusive scan of the accepted counts in stream (thread) order
        u32 incl = acc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= (u32)d) incl += y;
        }
        if (lane == 31) warp_sum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            u32 ws = lane < blockDim.x / 32 ? warp_sum[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, ws, d);
                if (lane >= (u32)d) ws += y;
            }
            warp_sum[lane] = ws;  // inclusive over warps
        }
        __syncthreads();
        u32 pos = got + (warp ? warp_sum[warp - 1] : 0) + incl - acc;
#pragma unroll
        for (u32 x = 0; x < TW; ++x)
            if (v[x] < lim) {
                if (pos < N) o[pos] = v[x] % p;
                ++pos;
            }
        __syncthreads();
        if (tid == blockDim.x - 1) base_sh = got + warp_sum[blockDim.x / 32 - 1];
        __syncthreads();
    }
}

/// Noise (sample_noise_poly, bfv.cpp:297-301) of h ciphertexts: e[q][n] in [-20, 20].
__global__ void k_noise(const Seed4* __restrict__ seeds, u32 h, u32 N, int* __restrict__ e) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)h * N) return;
    const u32 q = (u32)(idx / N), n = (u32)(idx % N);
    u32 blk[16];
    chacha_block(seeds[q], 0, n / 4, blk);  // words 2n, 2n + 1: block (2n) / 8, slots 2 (n % 4), +1
    const u32 s = 2 * (n % 4);
    const u64 a = ((u64)blk[2 * s] | ((u64)blk[2 * s + 1] << 32)) & ((1ull << 20) - 1);
    const u64 b = ((u64)blk[2 * s + 2] | ((u64)blk[2 * s + 3] << 32)) & ((1ull << 20) - 1);
    e[idx] = __popcll(a) - __popcll(b);
}

/// Signed small polynomial -> residues mod every chain prime: out[i][n] (NTT input).
__global__ void k_signed_to_chain(const signed char* __restrict__ s, DevTab T, u64* __restrict__ out) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)T.L * T.N) return;
    const u32 i = (u32)(idx / T.N), n = (u32)(idx % T.N);
    const int v = s[n];
    out[idx] = v < 0 ? T.q[i] - (u64)(-v) : (u64)v;
}

/// a[x] = a[x] * b[x mod (L N)] mod q_i (NTT-domain products; a: [count][L][N]).
__global__ void k_mul64(u64* __restrict__ a, const u64* __restrict__ b, size_t count, DevTab T) {
    const size_t LN = (size_t)T.L * T.N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= count * LN) return;
    const u32 i = (u32)((idx % LN) / T.N);
    const u64 x = a[idx], y = b[idx % LN];
    a[idx] = reduce128(__umul64hi(x, y), x * y, T.q[i], T.q_mu96[i]);
}

/// c0 = -(c1 s) + e + Delta m (bfv.cpp:530-545) with m = pack_query_bits' plaintext: coefficient j of
/// ciphertext q is `scale` when bit q 2^c + j < m_bits is set (expansion.cpp:27-35).  out [h][2][L][N]
/// (comp 1 = c1 already in place); prod [h][L][N] = c1 s (coefficient form).
__global__ void k_enc_combine(const u64* __restrict__ prod, const int* __restrict__ e, const unsigned char* __restrict__ bits,
                              u32 m_bits, u32 c, u64 scale, u32 h, DevTab T, u64* __restrict__ out) {
    const u32 N = T.N, L = T.L;
    const size_t LN = (size_t)L * N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)h * LN) return;
    const u32 q = (u32)(idx / LN), i = (u32)((idx % LN) / N), n = (u32)(idx % N);
    const u64 qi = T.q[i];
    u64 v = prod[idx] ? qi - prod[idx] : 0;
    const int ev = e[(size_t)q * N + n];
    v += ev < 0 ? qi - (u64)(-ev) : (u64)ev;
    if (v >= qi) v -= qi;
    const u64 bit = (u64)q << c;
    if (n < (1u << c) && bit + n < m_bits && bits[bit + n]) {
        const u64 dm = reduce128(__umul64hi(T.delta[i], scale), T.delta[i] * scale, qi, T.q_mu96[i]);
        v += dm;
        if (v >= qi) v -= qi;
    }
    out[(size_t)q * 2 * LN + (size_t)i * N + n] = v;
}

/// a[b][x] = (a[b][x] + src[b * src_stride + x]) mod q_i for x < L N (src: c0 of ciphertext b).
__global__ void k_add64_strided(u64* __restrict__ a, const u64* __restrict__ src, size_t src_stride, size_t count,
                                DevTab T) {
    const size_t LN = (size_t)T.L * T.N;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= count * LN) return;
    const size_t b = idx / LN, x = idx % LN;
    const u64 q = T.q[x / T.N];
    const u64 s = a[idx] + src[b * src_stride + x];
    a[idx] = s >= q ? s - q : s;
}

/// decrypt's rounding (bfv.cpp:572-592): v [count][L][N] (coefficient form, sum_k c_k s^k) ->
/// m_n = (sum_i floor(t y_i / q_i) + round(rem / q)) mod t, y_i = v_i (q / q_i)^-1 mod q_i,
/// rem = sum_i (t y_i mod q_i) (q / q_i), rounding counted as the reference does (odd multiples).
__global__ void k_dec_round(const u64* __restrict__ v, size_t count, DevTab T, u64* __restrict__ out) {
    const u32 N = T.N, L = T.L;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= count * N) return;
    const size_t b = idx / N;
    const u32 n = (u32)(idx % N);
    const u64 t = T.t;
    u64 r[kMaxL];
    u64 qsum = 0, lo = 0;
    u32 ip = 0;
#pragma unroll
    for (int i = 0; i < kMaxL; ++i) {
        if (i < (int)L) {
            const u64 qi = T.q[i];
            const u64 y = red64(shoup64(v[(b * L + i) * N + n], T.muq[i], T.muq_s[i], qi), qi);
            // t y = fl q_i + r_i with fl < t: r_i by the 128-bit reduction, fl by exact division
            // (q_i odd: fl = (t y - r_i) q_i^-1 mod 2^64, exact since fl < 2^64)
            const u64 tl = t * y, th = __umul64hi(t, y);
            r[i] = reduce128(th, tl, qi, T.q_mu96[i]);
            u64 qinv = qi;  // q_i^-1 mod 2^64 (Newton)
#pragma unroll
            for (int it = 0; it < 5; ++it) qinv *= 2 - qi * qinv;
            qsum = (qsum + ((tl - r[i]) * qinv) % t) % t;
            // fractional sum of r_i / q_i (the same estimate as the centred lift)
            const u64 f = frac64(r[i], T.q_gh[i], T.q_gl[i]);
            lo += f;
            ip += (lo < f);
        } else {
            r[i] = 0;
        }
    }
    // round(rem / q), rem = sum_i r_i (q / q_i): crt_round decides from the 64-bit fraction and
    // falls back to the exact multiword comparison inside its error band (the reference counts
    // odd multiples of q below 2 rem, bfv.cpp:581-590: the same round-half-up)
    const u32 round_add = crt_round(r, ip, lo, T);
    out[idx] = (qsum + round_add) % t;
}

}  // namespace cwgpu

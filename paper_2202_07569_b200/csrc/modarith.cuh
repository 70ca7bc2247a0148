// Device modular arithmetic for the B200 answer path (sm_100a).
//
// 32-bit side (31-bit aux / MAC primes a_j < 2^31): Shoup twiddle products,
// Montgomery products (R = 2^32) for the tensor, Barrett reduction of 64-bit sums.
// 64-bit side (chain primes 2^32 < q_i < 2^60): Shoup products (ring.cpp:13-18),
// 96/128-bit reductions for key-switch sums, CRT fractional estimates.
#pragma once
#include <cstdint>

namespace cwgpu {

typedef std::uint32_t u32;
typedef std::uint64_t u64;

// ---------------------------------------------------------------- 32-bit
__device__ __forceinline__ u32 red32(u32 x, u32 p) { return min(x, x - p); }  // [0,2p) -> [0,p)

/// x*w mod p in [0, 2p), ws = floor(w * 2^32 / p); valid for any x < 2^32.
__device__ __forceinline__ u32 shoup32(u32 x, u32 w, u32 ws, u32 p) {
    return x * w - __umulhi(x, ws) * p;
}

/// Montgomery product a*b*2^-32 mod p in [0, 2p); pinv = -p^-1 mod 2^32; a, b < 2^32, p < 2^31.
__device__ __forceinline__ u32 mont32(u32 a, u32 b, u32 p, u32 pinv) {
    u64 t = (u64)a * b;
    u32 m = (u32)t * pinv;
    return (u32)((t + (u64)m * p) >> 32);
}

/// x mod p for any 64-bit x; mu = floor(2^64 / p) (p < 2^31 so mu < 2^34).
__device__ __forceinline__ u32 bar64(u64 x, u32 p, u64 mu) {
    u64 qh = __umul64hi(x, mu);
    u64 r = x - qh * p;  // < 2p
    return red32((u32)r, p);
}

// ---------------------------------------------------------------- 64-bit
__device__ __forceinline__ u64 shoup64(u64 x, u64 w, u64 ws, u64 q) {
    return x * w - __umul64hi(x, ws) * q;  // [0, 2q)
}

__device__ __forceinline__ u64 red64(u64 x, u64 q) { return x >= q ? x - q : x; }

/// (hi * 2^64 + lo) mod q for a value < 2^96; mu96 = floor(2^96 / q), 2^32 < q < 2^60.
__device__ __forceinline__ u64 reduce96(u32 hi, u64 lo, u64 q, u64 mu96) {
    u64 xs = ((u64)hi << 32) | (lo >> 32);
    u64 qh = __umul64hi(xs, mu96);
    u64 r = lo - qh * q;  // true remainder + (0..3) q < 2^62
    r = red64(r, 2 * q);
    return red64(r, q);
}

/// (hi * 2^64 + lo) mod q for any 128-bit value (two 96-bit steps).
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, u64 q, u64 mu96) {
    // top = value >> 32 < 2^96
    u64 top_lo = (hi << 32) | (lo >> 32);
    u32 top_hi = (u32)(hi >> 32);
    u64 r1 = reduce96(top_hi, top_lo, q, mu96);  // (value >> 32) mod q < 2^60
    // (r1 * 2^32 + low32) < 2^92
    u64 x_lo = (r1 << 32) | (lo & 0xffffffffull);
    u32 x_hi = (u32)(r1 >> 32);
    return reduce96(x_hi, x_lo, q, mu96);
}

/// 64x64 -> 128 accumulate.
__device__ __forceinline__ void mac128(u64& hi, u64& lo, u64 a, u64 b) {
    u64 pl = a * b, ph = __umul64hi(a, b);
    lo += pl;
    hi += ph + (lo < pl);
}

/// floor(y * 2^64 / q) up to -2 units, from G = floor(2^128 / q) = gh * 2^64 + gl.
__device__ __forceinline__ u64 frac64(u64 y, u64 gh, u64 gl) { return y * gh + __umul64hi(y, gl); }

}  // namespace cwgpu

// On-device database setup from raw rows (PirDatabase::setup, reference pir.cpp:214-252):
// row codewords by perfect_map (cw_code.cpp:80-102) and payload chunking into plaintexts
// (chunk_payload, pir.cpp:169-193); the resident NTT form is then built exactly as for
// cwg_load_db (prepare_plain, bfv.cpp:933-942).  Byte-level work, one pass over the payload.
#pragma once
#include "devtab.h"

namespace cwgpu {

/// perfect_map: ascending positions of the x-th weight-k word of length m in colex order, for
/// every row (ids[r]).  Binomials in u64 (the host checks max_j C(m-1, j) < 2^64).
__global__ void k_perfect_map(const u64* __restrict__ ids, u64 n, u32 m, u32 k, u32* __restrict__ pos) {
    const u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    u64 row[65];  // row[j] = C(m', j), j <= k <= 64, starting at m' = m - 1
    row[0] = 1;
    for (u32 j = 1; j <= k; ++j) {
        // C(m-1, j) = C(m-1, j-1) (m - j) / j, exact at every step
        row[j] = j > m - 1 ? 0 : (u64)(((unsigned __int128)row[j - 1] * (m - j)) / j);
    }
    u64 x = ids[r];
    u32 h = k;
    u32* out = pos + r * k;
    for (u32 mp = m; mp-- > 0;) {
        if (x >= row[h]) {
            out[h - 1] = mp;  // bits are found from the top: slot h-1 keeps the order ascending
            x -= row[h];
            if (--h == 0) break;
        }
        if (mp > 0)
            for (u32 j = 1; j <= h; ++j) row[j] -= row[j - 1];  // C(m'-1, j) = C(m', j) - C(m'-1, j-1)
    }
}

/// chunk_payload: row r's bytes -> s plaintexts of N coefficients, b bits each (LSB first,
/// zero padded past the payload).  bytes: [R][payload_bytes]; out: [R][s][N] u64.
__global__ void k_chunk_payload(const unsigned char* __restrict__ bytes, u64 R, u64 payload_bytes, u32 s, u32 N,
                                u32 b, u64* __restrict__ out) {
    const u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    const u64 per_row = (u64)s * N;
    if (idx >= R * per_row) return;
    const u64 r = idx / per_row, cj = idx % per_row;  // cj = chunk * N + j
    const unsigned char* p = bytes + r * payload_bytes;
    const u64 bit0 = cj * b, total = payload_bytes * 8;
    u64 v = 0;
    if (bit0 < total) {
        const u64 byte0 = bit0 >> 3;
        const u32 sh = (u32)(bit0 & 7);
        const u32 nbytes = (sh + b + 7) >> 3;  // <= 9 for b <= 64
        unsigned __int128 w = 0;
        for (u32 i = 0; i < nbytes; ++i)
            if (byte0 + i < payload_bytes) w |= (unsigned __int128)p[byte0 + i] << (8 * i);
        w >>= sh;
        v = b >= 64 ? (u64)w : (u64)w & ((1ull << b) - 1);
        const u64 left = total - bit0;  // bits past the payload end read as zero
        if (left < b) v &= (1ull << left) - 1;
    }
    out[idx] = v;
}

}  // namespace cwgpu

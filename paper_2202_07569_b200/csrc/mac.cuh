// Payload multiply-accumulate (weighted_sum, reference bfv.cpp:944-986) as a TMA-fed stream.
//
// acc[sj][c][k][n] += sum_r Z[r][c][k][n] * DB[row0 + r][sj][k][n]   (NTT domain, MAC basis)
//
// One CTA owns a 1024-coefficient block of one (sj, k) plane over a chunk of rows.  A producer
// warp streams, per row, the block's 4 KB payload segment and the NC 4 KB selection segments
// into a 4-stage shared-memory ring with cp.async.bulk (1-D TMA: contiguous, no register
// staging), signalling a `full` mbarrier by transaction bytes; 8 consumer warps (4 coefficients
// per thread, 128-bit shared loads) accumulate 16-row groups of 60-bit products in u64 and
// release the stage through an `empty` mbarrier (after a fence.proxy.async: the stage's next
// writer is the async proxy).  Loads in flight are bounded by the ring, not
// by registers, so the stream runs at HBM rate.
#pragma once
#include <cuda.h>  // CUtensorMap (types only: the encoder is fetched through the runtime)
#include "devtab.h"
#include "modarith.cuh"

namespace cwgpu {

constexpr int kMacStages = 4;
constexpr int kMacBlock = 1024;  // coefficients per CTA (256 consumer threads x 4)

__device__ __forceinline__ u32 mac_smem(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mac_smem(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, u32 phase) {
    u32 done = 0;
    while (!done)
        asm volatile(
            "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
            : "=r"(done)
            : "r"(mac_smem(b)), "r"(phase)
            : "memory");
}
/// Same, but each try_wait may suspend the warp in hardware for up to `ns` nanoseconds instead of
/// returning at once: a waiting warp then spends no issue slots spinning (the rounding kernel's
/// consumer waits were ~20% of its issued instructions).
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* b, u32 phase, u32 ns = 1000000u) {
    u32 done = 0;
    while (!done)
        asm volatile(
            "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
            : "=r"(done)
            : "r"(mac_smem(b)), "r"(phase), "r"(ns)
            : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mac_smem(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mac_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, u32 bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     mac_smem(dst)),
                 "l"(src), "r"(bytes), "r"(mac_smem(bar))
                 : "memory");
}

/// Grid: chunks x Mm x (N / 1024) x s CTAs of 288 threads (8 consumer warps + 1 producer warp),
/// block index (slowest .. fastest): chunk, prime k, coefficient block, payload slice sj.
/// Z: Z + ((r * NC + c) * zstride + k) * N.  DB: [rows][s][Mm][N].  acc: u64 sums of residues.
template <int NC>
__global__ void __launch_bounds__(288, 3) k_mac_tma(const u32* __restrict__ Z, u32 zstride, const u32* __restrict__ DB,
                                                   u32 R, u32 s, u32 chunk, DevTab T, unsigned long long* __restrict__ acc) {
    extern __shared__ __align__(128) uint4 ring[];  // [stage][1 + NC][kMacBlock / 4]
    __shared__ __align__(8) unsigned long long full[kMacStages], empty[kMacStages];
    const u32 N = T.N, Mm = T.Mm;
    const u32 nblk = N / kMacBlock;
    u32 b = blockIdx.x;
    const u32 sj = b % s;
    b /= s;
    const u32 blk = b % nblk;
    b /= nblk;
    const u32 k = b % Mm;
    const u32 ch = b / Mm;
    const u32 r0 = ch * chunk, r1 = min(R, r0 + chunk);
    const u32 rows = r1 > r0 ? r1 - r0 : 0;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    constexpr u32 SEG = kMacBlock * 4;  // bytes per segment
    constexpr u32 SEGV = kMacBlock / 4; // uint4 per segment
    if (tid == 0) {
        for (int i = 0; i < kMacStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {  // producer
        if ((tid & 31) == 0) {
            const size_t dbs = (size_t)s * Mm * N;
            const u32* dbase = DB + ((size_t)sj * Mm + k) * N + (size_t)blk * kMacBlock;
            const u32* zbase = Z + (size_t)k * N + (size_t)blk * kMacBlock;
            const size_t zs = (size_t)NC * zstride * N;
            for (u32 i = 0; i < rows; ++i) {
                const u32 st = i % kMacStages;
                if (i >= (u32)kMacStages) mbar_wait(&empty[st], ((i / kMacStages) - 1) & 1);
                uint4* buf = ring + (size_t)st * (1 + NC) * SEGV;
                mbar_expect_tx(&full[st], SEG * (1 + NC));
                const size_t r = r0 + i;
                tma_bulk_g2s(buf, dbase + r * dbs, SEG, &full[st]);
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    tma_bulk_g2s(buf + (1 + c) * SEGV, zbase + r * zs + (size_t)c * zstride * N, SEG, &full[st]);
            }
        }
        return;
    }
    const u32 p = T.a[k];
    const u64 pb = T.abar[k];
    u32 accr[NC][4];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) accr[c][e] = 0;
    for (u32 g0 = 0; g0 < rows; g0 += 16) {
        const u32 ge = min(rows, g0 + 16);
        u64 g[NC][4];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) g[c][e] = 0;
        for (u32 i = g0; i < ge; ++i) {
            const u32 st = i % kMacStages;
            mbar_wait(&full[st], (i / kMacStages) & 1);
            const uint4* buf = ring + (size_t)st * (1 + NC) * SEGV;
            const uint4 d = buf[tid];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const uint4 z = buf[(1 + c) * SEGV + tid];
                g[c][0] += (u64)z.x * d.x;
                g[c][1] += (u64)z.y * d.y;
                g[c][2] += (u64)z.z * d.z;
                g[c][3] += (u64)z.w * d.w;
            }
            // the stage is rewritten by TMA (async proxy): order this thread's generic-proxy reads
            // of it before the release, then one arrival per warp
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[st]);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) accr[c][e] = red32(accr[c][e] + bar64(g[c][e], p, pb), p);
    }
    if (rows == 0) return;
    const u32 n = blk * kMacBlock + 4 * tid;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        unsigned long long* o = acc + (((size_t)sj * 3 + c) * Mm + k) * N + n;
#pragma unroll
        for (int e = 0; e < 4; ++e) atomicAdd(o + e, (unsigned long long)accr[c][e]);
    }
}


/// Multi-query / multi-slice payload MAC: the k_mac_tma stream with QB queries' selection planes
/// and SG payload slices per ring stage.  QB > 1: one pass over a row tile's
/// database planes serves several queries.  SG > 1 (s >= 3 rows, e.g. C3's 15 plaintexts): the
/// NC selection segments of a row are read once per SG slices instead of once per slice.
/// 512-coefficient blocks (2 per consumer thread) keep the ring at 4 stages x (SG + QB NC) x 2 KB.
/// Grid: chunks x Mm x (N / 512) x (s / SG); s must be a multiple of SG.
constexpr int kMacBlockQ = 512;
struct ZPtrs {
    const u32* z[4];
    unsigned long long* acc[4];
};
template <int NC, int QB, int SG, int ST = kMacStages>
__global__ void __launch_bounds__(288, 2) k_mac_tma_q(const __grid_constant__ ZPtrs Zp, u32 zstride,
                                                     const u32* __restrict__ DB, u32 R, u32 s, u32 chunk, DevTab T) {
    extern __shared__ __align__(128) uint2 ringq[];  // [stage][SG + QB NC][kMacBlockQ / 2]
    __shared__ __align__(8) unsigned long long full[ST], empty[ST];
    constexpr u32 NSEG = SG + QB * NC;
    constexpr u32 SEG = kMacBlockQ * 4;   // bytes per segment
    constexpr u32 SEGV = kMacBlockQ / 2;  // uint2 per segment
    const u32 N = T.N, Mm = T.Mm;
    const u32 nblk = N / kMacBlockQ;
    const u32 ngrp = s / SG;
    u32 b = blockIdx.x;
    const u32 sg0 = (b % ngrp) * SG;
    b /= ngrp;
    const u32 blk = b % nblk;
    b /= nblk;
    const u32 k = b % Mm;
    const u32 ch = b / Mm;
    const u32 r0 = ch * chunk, r1 = min(R, r0 + chunk);
    const u32 rows = r1 > r0 ? r1 - r0 : 0;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {  // producer
        if ((tid & 31) == 0) {
            const size_t dbs = (size_t)s * Mm * N;
            const u32* dbase = DB + ((size_t)sg0 * Mm + k) * N + (size_t)blk * kMacBlockQ;
            const size_t zs = (size_t)NC * zstride * N;
            const size_t zoff = (size_t)k * N + (size_t)blk * kMacBlockQ;
            for (u32 i = 0; i < rows; ++i) {
                const u32 st = i % ST;
                if (i >= (u32)ST) mbar_wait(&empty[st], ((i / ST) - 1) & 1);
                uint2* buf = ringq + (size_t)st * NSEG * SEGV;
                mbar_expect_tx(&full[st], SEG * NSEG);
                const size_t r = r0 + i;
#pragma unroll
                for (int g = 0; g < SG; ++g)
                    tma_bulk_g2s(buf + g * SEGV, dbase + r * dbs + (size_t)g * Mm * N, SEG, &full[st]);
#pragma unroll
                for (int q = 0; q < QB; ++q)
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        tma_bulk_g2s(buf + (SG + q * NC + c) * SEGV, Zp.z[q] + zoff + r * zs + (size_t)c * zstride * N,
                                     SEG, &full[st]);
            }
        }
        return;
    }
    const u32 p = T.a[k];
    const u64 pb = T.abar[k];
    // lazy accumulation: 60-bit products summed in u64, folded every 8 rows with
    // x -> (x >> 32) (2^32 mod a) + (x & 2^32 - 1) (< 2^62 + 2^32: one IMAD.WIDE instead of a Barrett
    // reduction), one Barrett reduction per output at the end of the chunk
    const u32 c32 = bar64(1ull << 32, p, pb);
    u64 acc64[QB][SG][NC][2];
#pragma unroll
    for (int q = 0; q < QB; ++q)
#pragma unroll
        for (int g = 0; g < SG; ++g)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc64[q][g][c][0] = acc64[q][g][c][1] = 0;
    for (u32 g0 = 0; g0 < rows; g0 += 8) {
        const u32 ge = min(rows, g0 + 8);
        for (u32 i = g0; i < ge; ++i) {
            const u32 st = i % ST;
            mbar_wait(&full[st], (i / ST) & 1);
            const uint2* buf = ringq + (size_t)st * NSEG * SEGV;
            uint2 d[SG];
#pragma unroll
            for (int g = 0; g < SG; ++g) d[g] = buf[g * SEGV + tid];
#pragma unroll
            for (int q = 0; q < QB; ++q)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const uint2 z = buf[(SG + q * NC + c) * SEGV + tid];
#pragma unroll
                    for (int g = 0; g < SG; ++g) {
                        acc64[q][g][c][0] += (u64)z.x * d[g].x;
                        acc64[q][g][c][1] += (u64)z.y * d[g].y;
                    }
                }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[st]);
        }
        if (ge < rows) {
#pragma unroll
            for (int q = 0; q < QB; ++q)
#pragma unroll
                for (int g = 0; g < SG; ++g)
#pragma unroll
                    for (int c = 0; c < NC; ++c)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            acc64[q][g][c][e] = (u64)(u32)(acc64[q][g][c][e] >> 32) * c32 + (u32)acc64[q][g][c][e];
        }
    }
    if (rows == 0) return;
    const u32 n = blk * kMacBlockQ + 2 * tid;
#pragma unroll
    for (int q = 0; q < QB; ++q)
#pragma unroll
        for (int g = 0; g < SG; ++g)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                unsigned long long* o = Zp.acc[q] + (((size_t)(sg0 + g) * 3 + c) * Mm + k) * N + n;
                atomicAdd(o, (unsigned long long)bar64(acc64[q][g][c][0], p, pb));
                atomicAdd(o + 1, (unsigned long long)bar64(acc64[q][g][c][1], p, pb));
            }
}


/// Whole-row payload MAC for rows of many plaintexts (C3: s = 15): one persistent CTA per SM streams,
/// per row, ALL SG payload segments and the NC selection segments of a 256-coefficient block of one
/// MAC prime -- so each selection word is fetched once per row instead of once per slice group, and
/// the ring (ST stages x (SG + NC) KB, ~180 KB) keeps enough bytes in flight per SM for the HBM
/// stream on its own.  A stage is filled by TWO tensor-map copies (cp.async.bulk.tensor.4d: a
/// {256, 1, SG, 1} box of the database viewed as [row][s][Mm][N] and a {256, 1, NC, 1} box of the
/// selection planes): per-segment 1 KB cp.async.bulk copies were bound by the copy issue rate
/// (~50 ns per copy and SM: 2.8 TB/s).  Work items (row chunk, prime, coefficient block) are handed
/// out by a global counter: a CTA that starts late (the tile streams' other kernels still hold its
/// SM) simply takes fewer items.  The item id travels with the ring stage (meta word; ~0 ends the
/// stream).  Accumulation is lazy: 60-bit products summed in u64 and folded every 8 rows with
/// x -> (x >> 32) (2^32 mod a) + (x & 2^32 - 1)  (< 2^62 + 2^32, one IMAD.WIDE), one Barrett
/// reduction and one atomic add per output per item.
/// Grid: <= SMs CTAs of 288 threads (8 consumer warps, 1 coefficient per thread, + a producer warp).
constexpr int kMacBlockS = 256;
__device__ __forceinline__ void tma_tensor4_g2s(void* dst, const void* tmap, u32 c0, u32 c1, u32 c2, u32 c3,
                                                unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(mac_smem(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mac_smem(bar))
        : "memory");
}
template <int NC, int SG, int ST>
__global__ void __launch_bounds__(288, 1) k_mac_rows(const __grid_constant__ CUtensorMap tmDB,
                                                    const __grid_constant__ CUtensorMap tmZ, u32 R, u32 chunk,
                                                    u32 nchunks, DevTab T, unsigned long long* __restrict__ acc,
                                                    u32* __restrict__ counter) {
    extern __shared__ __align__(128) u32 rings[];  // [stage][SG + NC][kMacBlockS]
    __shared__ __align__(8) unsigned long long full[ST], empty[ST];
    __shared__ u32 meta[ST];
    constexpr u32 NSEG = SG + NC;
    constexpr u32 SEG = kMacBlockS * 4;  // bytes per segment
    const u32 N = T.N, Mm = T.Mm;
    const u32 nblk = N / kMacBlockS;
    const u32 nitems = nchunks * Mm * nblk;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {  // producer
        if ((tid & 31) == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmDB) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmZ) : "memory");
            u32 i = 0;
            for (;;) {
                const u32 it = atomicAdd(counter, 1u);
                if (it >= nitems) break;
                const u32 blk = it % nblk, k = (it / nblk) % Mm, ch = it / (nblk * Mm);
                const u32 r0 = ch * chunk, r1 = min(R, r0 + chunk);
                for (u32 r = r0; r < r1; ++r, ++i) {
                    const u32 st = i % ST;
                    if (i >= (u32)ST) mbar_wait(&empty[st], ((i / ST) - 1) & 1);
                    u32* buf = rings + (size_t)st * NSEG * kMacBlockS;
                    meta[st] = it;
                    mbar_expect_tx(&full[st], SEG * NSEG);
                    tma_tensor4_g2s(buf, &tmDB, blk * kMacBlockS, k, 0, r, &full[st]);
                    tma_tensor4_g2s(buf + SG * kMacBlockS, &tmZ, blk * kMacBlockS, k, 0, r, &full[st]);
                }
            }
            const u32 st = i % ST;  // end of stream
            if (i >= (u32)ST) mbar_wait(&empty[st], ((i / ST) - 1) & 1);
            meta[st] = 0xffffffffu;
            mbar_arrive(&full[st]);
        }
        return;
    }
    u32 i = 0;
    for (;;) {
        mbar_wait(&full[i % ST], (i / ST) & 1);  // first row of the next item (waited for again below)
        const u32 it = meta[i % ST];
        if (it == 0xffffffffu) break;
        const u32 blk = it % nblk, k = (it / nblk) % Mm, ch = it / (nblk * Mm);
        const u32 r0 = ch * chunk, rows = min(R, r0 + chunk) - r0;
        const u32 p = T.a[k];
        const u64 pb = T.abar[k];
        const u32 c32 = bar64(1ull << 32, p, pb);  // 2^32 mod a_k
        u64 a64[SG][NC];
#pragma unroll
        for (int g = 0; g < SG; ++g)
#pragma unroll
            for (int c = 0; c < NC; ++c) a64[g][c] = 0;
        for (u32 g0 = 0; g0 < rows; g0 += 8) {
            const u32 ge = min(rows, g0 + 8);
            for (u32 r = g0; r < ge; ++r, ++i) {
                const u32 st = i % ST;
                mbar_wait(&full[st], (i / ST) & 1);
                const u32* buf = rings + (size_t)st * NSEG * kMacBlockS + tid;
                u32 z[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) z[c] = buf[(SG + c) * kMacBlockS];
#pragma unroll
                for (int g = 0; g < SG; ++g) {
                    const u32 d = buf[g * kMacBlockS];
#pragma unroll
                    for (int c = 0; c < NC; ++c) a64[g][c] += (u64)z[c] * d;
                }
                // the stage is rewritten by TMA (async proxy): order this thread's generic-proxy reads
                // of it before the release, then one arrival per warp
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if ((tid & 31) == 0) mbar_arrive(&empty[st]);
            }
            if (ge < rows) {
#pragma unroll
                for (int g = 0; g < SG; ++g)
#pragma unroll
                    for (int c = 0; c < NC; ++c) a64[g][c] = (u64)(u32)(a64[g][c] >> 32) * c32 + (u32)a64[g][c];
            }
        }
        const u32 n = blk * kMacBlockS + tid;
#pragma unroll
        for (int g = 0; g < SG; ++g)
#pragma unroll
            for (int c = 0; c < NC; ++c)
                atomicAdd(acc + (((size_t)g * 3 + c) * Mm + k) * N + n, (unsigned long long)bar64(a64[g][c], p, pb));
    }
}

}  // namespace cwgpu

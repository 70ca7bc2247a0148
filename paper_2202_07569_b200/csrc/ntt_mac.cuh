// Fused selection NTT + payload MAC (weighted_sum, reference bfv.cpp:944-986):
//   ntt_forward of every selection component (bfv.cpp:967) and
//   pointwise_mul_accumulate against the NTT-form database row (bfv.cpp:968)
// in one pass, so the NTT-domain selection values never travel to HBM and back.
//
// Block (ch, k, c): MAC prime k, selection component c, rows [ch*chunk, ch*chunk+chunk) of the
// tile.  For each row the CTA loads the coefficient-domain selection plane Z[row][c][k] (the
// rounding kernel's output), transforms it in registers (nttw_fwd, 32 coefficients per
// thread), and multiplies it with the S payload planes DB[row][sj][k] read at the same
// positions (both in the register-transposed PERM order pos = r * N/E + tid, so every load is
// coalesced and thread tid owns the same positions for every row).  Products are Montgomery
// (x 2^-32) and accumulate in [0, 2p) per thread; the chunk's sums get the 2^32 back with one
// Montgomery product by 2^64 mod p and land in acc[sj][c][k][pos] with one u64 atomic each, the
// same accumulator contract as k_mac2 (sums of residues, reduced later by k_acc_mod).
#pragma once
#include "ntt_reg.cuh"
#include "mac.cuh"

namespace cwgpu {

/// ACCS = false: accumulators in registers (S = 1 only; <= 128 registers, 2 CTAs / SM at
/// N = 8192); true: thread-private slots in shared memory (the NTT kernels' register budget).
template <int LOGN, int S, bool ACCS>
struct NttMac {
    using R = RegNtt<LOGN>;
    static constexpr int T = R::T, E = R::E, WB = R::WB;
    static constexpr bool ACC_SMEM = ACCS || S >= 2;
    static constexpr size_t SMEM = R::SMEM + (ACC_SMEM ? (size_t)S * (1 << LOGN) * 4 : 0);
    static constexpr int MINB = ACC_SMEM ? R::MINB : (R::MINB2 < R::MINB ? R::MINB2 : R::MINB);
};

template <int LOGN, int NC, int S, bool ACCS>
__global__ void __launch_bounds__(NttMac<LOGN, S, ACCS>::T, NttMac<LOGN, S, ACCS>::MINB) k_ntt_mac(
    const u32* __restrict__ Z, u32 zstride, const u32* __restrict__ DB, u32 R, u32 nchunks, DevTab T,
    unsigned long long* __restrict__ acc) {
    using G = NttMac<LOGN, S, ACCS>;
    constexpr int E = G::E, WB = G::WB, N = 1 << LOGN, SH = LOGN - WB;
    extern __shared__ u32 smd[];
    u32* accs = smd + N;  // S x N thread-private accumulator slots (ACC_SMEM)
    const u32 tid = threadIdx.x;
    const u32 Mm = T.Mm;
    const u32 c = blockIdx.x % NC, k = (blockIdx.x / NC) % Mm, ch = blockIdx.x / (NC * Mm);
    const u32 p = T.a[k], pinv = T.apinv[k], p2 = 2 * p;
    const u32 r0 = (u32)(((u64)ch * R) / nchunks), r1 = (u32)(((u64)(ch + 1) * R) / nchunks);  // balanced
    u32 a[G::ACC_SMEM ? 1 : S][E];
    if constexpr (G::ACC_SMEM) {
#pragma unroll
        for (int sj = 0; sj < S; ++sj)
#pragma unroll
            for (int r = 0; r < E; ++r) accs[sj * N + ((u32)r << SH) + tid] = 0;
    } else {
#pragma unroll
        for (int r = 0; r < E; ++r) a[0][r] = 0;
    }
    const size_t dbrow = (size_t)S * Mm * N;
    for (u32 i = r0; i < r1; ++i) {
        const u32* z = Z + (((size_t)i * NC + c) * zstride + k) * N + tid;
        u32 v[1][E];
#pragma unroll
        for (int r = 0; r < E; ++r) v[0][r] = __ldg(z + ((u32)r << SH));
        nttw_fwd<LOGN, WB, 1>(v, smd, T.arp + (size_t)k * N, T.arps + (size_t)k * N, p);  // [0, 4p)
#pragma unroll
        for (int sj = 0; sj < S; ++sj) {
            const u32* d = DB + (size_t)i * dbrow + ((size_t)sj * Mm + k) * N + tid;
            u32 dv[E];
#pragma unroll
            for (int r = 0; r < E; ++r) dv[r] = __ldg(d + ((u32)r << SH));
            if constexpr (G::ACC_SMEM) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    u32& s = accs[sj * N + ((u32)r << SH) + tid];
                    s = red32(s + mont32(v[0][r], dv[r], p, pinv), p2);
                }
            } else {
#pragma unroll
                for (int r = 0; r < E; ++r) a[0][r] = red32(a[0][r] + mont32(v[0][r], dv[r], p, pinv), p2);
            }
        }
    }
    if (r0 >= r1) return;
    const u32 r64 = T.a2_64[k];  // mont32(x, 2^64 mod p) = x 2^32 mod p: undoes the product's 2^-32
#pragma unroll
    for (int sj = 0; sj < S; ++sj) {
        unsigned long long* o = acc + (((size_t)sj * 3 + c) * Mm + k) * N + tid;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const u32 x = G::ACC_SMEM ? accs[sj * N + ((u32)r << SH) + tid] : a[0][r];
            atomicAdd(o + ((u32)r << SH), (unsigned long long)red32(mont32(x, r64, p, pinv), p));
        }
    }
}

}  // namespace cwgpu

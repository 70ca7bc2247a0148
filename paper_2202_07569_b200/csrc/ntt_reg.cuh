// Register-resident negacyclic NTT for the 30-bit aux / MAC primes.
//
// Same transform as RingContext::ntt_forward / ntt_inverse (reference ring.cpp:78-144):
// forward Cooley-Tukey, natural order in, bit-reversed out, twiddle root_pow[m + i]
// for block i of stage m; inverse Gentleman-Sande back to natural order.
//
// A CTA of T = N/E threads owns one polynomial; each thread keeps E = 2^WB coefficients
// in registers (WB = 5 for N >= 1024: 32 coefficients, 256 threads at N = 8192).  The
// log2(N) stages are processed in WB-bit windows: inside a window the thread's registers
// span the window's index bits, so all of its butterflies are register-local; between
// windows the polynomial is transposed through shared memory (XOR-swizzled, unpadded,
// bank-conflict free).  Twiddles are fetched per stage (at most 16 Shoup pairs live), and
// the small CTAs let several polynomials per SM run out of barrier phase with each other:
// measured 23-26 ns per 8192-point NTT on a B200 vs 52 ns for radix-16 / 512-thread CTAs
// (scripts/bench_ntt.py).
#pragma once
#include "devtab.h"
#include "modarith.cuh"

namespace cwgpu {

// XOR swizzle inside each 32-word row, y = x >> 5: bank(x) = x ^ (y ^ (y << 1)) mod 32 is conflict-free
// for every transpose window (WB = 4 and 5) of 2^8 <= N <= 2^14 (checked exhaustively) and needs no padding
__device__ __forceinline__ u32 pidx(u32 x) { const u32 y = x >> 5; return x ^ ((y ^ (y << 1)) & 31u); }

/// Load `cnt` consecutive twiddles (and Shoup companions) starting at base (cnt a multiple of 4 or < 4).
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

/// Write one polynomial (thread tid's E registers at positions (r << (LOGN - WB)) | tid, the PERM
/// order) to global memory through shared memory and one bulk copy.  Microbenchmark variant only
/// (scripts/bench_ntt.py): 21.0 vs 25.9 ns per NTT against the strided uint4 stores of the
/// benchmark's baseline, but no gain over the production kernels' coalesced PERM-order STG in
/// situ (k_tensor_intt, persistent with deferred bulk-store waits: 96.6 vs 81.4 ms at C4).
template <int LOGN, int WB>
__device__ __forceinline__ void bulk_store_poly(u32* __restrict__ gdst, u32* sm, const u32 (&v)[1 << WB]) {
    constexpr int E = 1 << WB, SH = LOGN - WB;
    const u32 tid = threadIdx.x;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r) sm[((u32)r << SH) | tid] = v[r];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                     "r"((u32)__cvta_generic_to_shared(sm)), "r"((u32)(4u << LOGN))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // smem stays valid until read
    }
}

template <int LOGN, int WB>
struct NttW {
    static constexpr int N = 1 << LOGN;
    static constexpr int E = 1 << WB;
    static constexpr int T = N / E;
    static constexpr int NW = (LOGN + WB - 1) / WB;
};

template <int WB>
__device__ __forceinline__ u32 win_index_w(u32 tid, int w, int r) {
    const u32 low = tid & ((1u << w) - 1u);
    const u32 high = tid >> w;
    return (high << (w + WB)) | ((u32)r << w) | low;
}

/// Twiddles of register bit j of a WB-bit window at low bit w: 2^(WB-1-j) consecutive
/// entries from (N >> (w+j+1)) + (high << (WB-1-j)).
template <int LOGN, int WB, int FAKE = 0>
__device__ __forceinline__ void load_stage_tw(const u32* __restrict__ tp, const u32* __restrict__ tsp, int w, int j,
                                              u32 high, u32* tw, u32* tws) {
    if constexpr ((FAKE & 1) != 0) {  // diagnostics only (microbenchmark): register twiddles, no loads
#pragma unroll
        for (int u = 0; u < (1 << (WB - 1)); ++u) { tw[u] = tp[u] + high; tws[u] = tsp[u] ^ high; }
        return;
    }
    const u32 base = ((u32)(1 << LOGN) >> (w + j + 1)) + (high << (WB - 1 - j));
    const int c = WB - 1 - j;
    if (c == 0) load_tw<1>(tp, tsp, base, tw, tws);
    else if (c == 1) load_tw<2>(tp, tsp, base, tw, tws);
    else if (c == 2) load_tw<4>(tp, tsp, base, tw, tws);
    else if (c == 3) load_tw<8>(tp, tsp, base, tw, tws);
    else if constexpr (WB <= 5) load_tw<16>(tp, tsp, base, tw, tws);
    else if (c == 4) load_tw<16>(tp, tsp, base, tw, tws);
    else load_tw<32>(tp, tsp, base, tw, tws);
}

/// Move the E registers of each thread from window wp to window w through shared memory.
template <int WB, int NP, int SMEM>
__device__ __forceinline__ void nttw_transpose(u32 (&v)[NP][1 << WB], u32* sm, u32 tid, int wp, int w) {
    constexpr int E = 1 << WB;
    // pidx is GF(2)-linear and the thread / register fields of the index are disjoint
    const u32 ps = pidx(win_index_w<WB>(tid, wp, 0)), pl = pidx(win_index_w<WB>(tid, w, 0));
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < E; ++r) sm[q * SMEM + (ps ^ pidx((u32)r << wp))] = v[q][r];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < E; ++r) v[q][r] = sm[q * SMEM + (pl ^ pidx((u32)r << w))];
}

/// Forward NTT; input mapping x = r << (LOGN-WB) | tid, output x = tid << WB | r.
/// Values in [0, 4p) in and out (p < 2^30).  sm: NP * N words.
template <int LOGN, int WB, int NP, int FAKE = 0>
__device__ __forceinline__ void nttw_fwd(u32 (&v)[NP][1 << WB], u32* sm, const u32* __restrict__ rp,
                                         const u32* __restrict__ rps, u32 p) {
    using G = NttW<LOGN, WB>;
    constexpr int E = G::E;
    const u32 tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < G::NW; ++k) {
        const int w = (LOGN - WB - WB * k) > 0 ? (LOGN - WB - WB * k) : 0;
        const int btop = LOGN - 1 - WB * k;
        const u32 high = tid >> w;
        if (k > 0) {
            const int wp = (LOGN - WB - WB * (k - 1)) > 0 ? (LOGN - WB - WB * (k - 1)) : 0;
            if constexpr ((FAKE & 2) == 0) nttw_transpose<WB, NP, G::N>(v, sm, tid, wp, w);
        }
#pragma unroll
        for (int b = btop; b >= w; --b) {
            const int j = b - w;
            u32 tw[E / 2], tws[E / 2];
            load_stage_tw<LOGN, WB, FAKE>(rp, rps, w, j, high, tw, tws);
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const u32 a = red32(v[q][r], 2 * p);
                    const u32 t = shoup32(v[q][r2], tw[u], tws[u], p);
                    v[q][r] = a + t;
                    v[q][r2] = a - t + 2 * p;
                }
            }
        }
    }
}

/// Inverse NTT (no N^-1 scaling); input mapping x = tid << WB | r, output
/// x = r << (LOGN-WB) | tid.  Values in [0, 2p) in and out.
template <int LOGN, int WB, int NP>
__device__ __forceinline__ void nttw_inv(u32 (&v)[NP][1 << WB], u32* sm, const u32* __restrict__ irp,
                                         const u32* __restrict__ irps, u32 p) {
    using G = NttW<LOGN, WB>;
    constexpr int E = G::E;
    const u32 tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < G::NW; ++k) {
        const int w = (WB * k) < (LOGN - WB) ? (WB * k) : (LOGN - WB);
        const int bbot = WB * k;
        const int btop = (WB * k + WB - 1) < (LOGN - 1) ? (WB * k + WB - 1) : (LOGN - 1);
        const u32 high = tid >> w;
        if (k > 0) {
            const int wp = (WB * (k - 1)) < (LOGN - WB) ? (WB * (k - 1)) : (LOGN - WB);
            nttw_transpose<WB, NP, G::N>(v, sm, tid, wp, w);
        }
#pragma unroll
        for (int b = bbot; b <= btop; ++b) {
            const int j = b - w;
            u32 tw[E / 2], tws[E / 2];
            load_stage_tw<LOGN, WB>(irp, irps, w, j, high, tw, tws);
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if (r & (1 << j)) continue;
                const int r2 = r | (1 << j);
                const int u = r >> (j + 1);
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const u32 a = v[q][r], c = v[q][r2];
                    v[q][r] = red32(a + c, 2 * p);
                    v[q][r2] = shoup32(a - c + 2 * p, tw[u], tws[u], p);
                }
            }
        }
    }
}


/// Window width and occupancy of the production kernels for a degree 2^LOGN.
template <int LOGN>
struct RegNtt {
    static constexpr int WB = LOGN >= 10 ? 5 : 4;
    using G = NttW<LOGN, WB>;
    static constexpr int T = G::T;
    static constexpr int E = G::E;
    // <= 85 registers at N = 8192 (3 CTAs / SM); 2 CTAs of 512 threads at N = 16384
    static constexpr int MINB = LOGN >= 14 ? 2 : (768 / T > 16 ? 16 : 768 / T);
    // two polynomials per CTA (shared twiddles, twice the ILP): <= 128 registers
    static constexpr int MINB2 = 512 / T > 16 ? 16 : (512 / T < 1 ? 1 : 512 / T);
    static constexpr size_t SMEM = (size_t)G::N * 4;
};

/// Batched forward / inverse NTT: poly p -> group g = p / gs, prime j = off + p % gs,
/// address (g * stride + j) * N.  scale (inverse only): 0 = N^-1, 1 = (N 2^32)^-1.
/// Output canonical [0, p).  PERM: the NTT-domain side is stored in the register-transposed
/// order pos = r * (N / E) + tid (thread tid's r-th output), so both directions move it with
/// coalesced scalar accesses; the answer path's aux / MAC-basis NTT-domain data (prepared
/// operands, database, selection values, accumulators) all use this order and are only
/// combined pointwise.  !PERM: the reference's bit-reversed order (cwg_ntt).
template <int LOGN, bool INV, bool PERM = true>
__global__ void __launch_bounds__(RegNtt<LOGN>::T, RegNtt<LOGN>::MINB) k_ntt32r(u32* __restrict__ base, DevTab T, u32 gs,
                                                                               u32 stride, u32 off, int scale) {
    using R = RegNtt<LOGN>;
    constexpr int WB = R::WB, E = R::E, N = 1 << LOGN;
    extern __shared__ u32 sm[];
    const u32 tid = threadIdx.x;
    const u32 pi = blockIdx.x, g = pi / gs, j = off + pi % gs;
    const u32 pr = T.a[j];
    u32* d = base + ((size_t)g * stride + j) * N;
    u32 v[1][E];
    if (!INV) {
#pragma unroll
        for (int r = 0; r < E; ++r) v[0][r] = d[((u32)r << (LOGN - WB)) | tid];
        nttw_fwd<LOGN, WB, 1>(v, sm, T.arp + (size_t)j * N, T.arps + (size_t)j * N, pr);
#pragma unroll
        for (int r = 0; r < E; ++r) v[0][r] = red32(red32(v[0][r], 2 * pr), pr);
        if (PERM) {
#pragma unroll
            for (int r = 0; r < E; ++r) d[((u32)r << (LOGN - WB)) | tid] = v[0][r];
        } else {
            uint4* o = reinterpret_cast<uint4*>(d + (tid << WB));
#pragma unroll
            for (int r = 0; r < E; r += 4) o[r / 4] = make_uint4(v[0][r], v[0][r + 1], v[0][r + 2], v[0][r + 3]);
        }
    } else {
        if (PERM) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[0][r] = d[((u32)r << (LOGN - WB)) | tid];
        } else {
            const uint4* in = reinterpret_cast<const uint4*>(d + (tid << WB));
#pragma unroll
            for (int r = 0; r < E; r += 4) {
                const uint4 x = in[r / 4];
                v[0][r] = x.x; v[0][r + 1] = x.y; v[0][r + 2] = x.z; v[0][r + 3] = x.w;
            }
        }
        nttw_inv<LOGN, WB, 1>(v, sm, T.airp + (size_t)j * N, T.airps + (size_t)j * N, pr);
        const u32 ni = scale ? T.ninvRA[j] : T.ninvA[j], nis = scale ? T.ninvRA_s[j] : T.ninvA_s[j];
#pragma unroll
        for (int r = 0; r < E; ++r) d[((u32)r << (LOGN - WB)) | tid] = red32(shoup32(v[0][r], ni, nis, pr), pr);
    }
}

/// Forward NTT of the 3 selection components of P products for every MAC prime, NP planes
/// of one prime per CTA: block (pc0 / NP) * Mm + k transforms the planes pc0 .. pc0 + NP - 1
/// (pc = pr * 3 + comp < npc) at base + (pc * stride_j + k) * N in place.
template <int LOGN, int NP>
__global__ void __launch_bounds__(RegNtt<LOGN>::T, NP == 1 ? RegNtt<LOGN>::MINB : RegNtt<LOGN>::MINB2) k_ntt32r_sel3(
    u32* __restrict__ base, DevTab T, u32 stride_j, u32 npc) {
    using R = RegNtt<LOGN>;
    constexpr int WB = R::WB, E = R::E, N = 1 << LOGN;
    extern __shared__ u32 smd[];
    const u32 tid = threadIdx.x;
    const u32 Mm = T.Mm;
    const u32 pc0 = (blockIdx.x / Mm) * NP, k = blockIdx.x % Mm;
    const u32 p = T.a[k];
    u32* d[NP];
    u32 v[NP][E];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const u32 pc = min(pc0 + q, npc - 1);  // odd tail: the duplicate is transformed, not stored
        d[q] = base + ((size_t)pc * stride_j + k) * N;
#pragma unroll
        for (int r = 0; r < E; ++r) v[q][r] = d[q][((u32)r << (LOGN - WB)) | tid];
    }
    nttw_fwd<LOGN, WB, NP>(v, smd, T.arp + (size_t)k * N, T.arps + (size_t)k * N, p);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        if (pc0 + q >= npc) break;
#pragma unroll
        for (int r = 0; r < E; ++r) d[q][((u32)r << (LOGN - WB)) | tid] = red32(red32(v[q][r], 2 * p), p);  // PERM order
    }
}

/// Tensor (mul_lazy_prepared, bfv.cpp:776-791) + INTT of NP products per CTA for one (aux
/// prime, component): block ((pr0 / NP) * J + j) * 3 + comp (the three components of the same
/// products are adjacent, so their shared operand planes are L2 hits).  Operands:
/// Montgomery-form NTT residues [idx][2][J][N]; output D[pr][comp][j][N] in normal form (the
/// (N 2^32)^-1 scale undoes the Montgomery factor).  fold = 1: also multiply by (A/a_j)^-1, i.e.
/// emit the HPS residues w_j that the tensor-core rounding kernel consumes directly; fold = 2:
/// the A operands already carry (N 2^32)^-1 (A/a_j)^-1 (k_scale_planes, once per query), so the
/// INTT output needs no scaling pass.
template <int LOGN, int NP>
__global__ void __launch_bounds__(RegNtt<LOGN>::T, NP == 1 ? RegNtt<LOGN>::MINB : RegNtt<LOGN>::MINB2) k_tensor_intt_r(
    const u32* __restrict__ prepA, const u32* __restrict__ idxA, const u32* __restrict__ prepB,
    const u32* __restrict__ idxB, u32 P, DevTab T, u32* __restrict__ D, int fold) {
    using R = RegNtt<LOGN>;
    constexpr int WB = R::WB, E = R::E, N = 1 << LOGN;
    extern __shared__ u32 smd[];
    const u32 J = T.J;
    const u32 tid = threadIdx.x;
    const u32 comp = blockIdx.x % 3, pj = blockIdx.x / 3;
    const u32 pr0 = (pj / J) * NP, j = pj % J;
    const u32 p = T.a[j], pinv = T.apinv[j];
    const size_t per = (size_t)2 * J * N;
    const size_t o1 = (size_t)J * N;
    u32 v[NP][E];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const u32 pr = min(pr0 + q, P - 1);  // odd tail: the duplicate is transformed, not stored
        const u32* A = prepA + (size_t)(idxA ? idxA[pr] : pr) * per + (size_t)j * N + tid;
        const u32* B = prepB + (size_t)(idxB ? idxB[pr] : pr) * per + (size_t)j * N + tid;
        // comp 0: A0 B0, comp 2: A1 B1, comp 1: A0 B1 + A1 B0; operands in the PERM order of
        // k_ntt32r: thread tid's r-th value at r * (N / E) + tid (coalesced)
        const u32* X = A + (comp == 2 ? o1 : 0);
        const u32* Y = B + (comp == 0 ? 0 : o1);
        u32 x[E], y[E];
#pragma unroll
        for (int r = 0; r < E; ++r) {
            x[r] = __ldg(X + ((u32)r << (LOGN - WB)));
            y[r] = __ldg(Y + ((u32)r << (LOGN - WB)));
        }
#pragma unroll
        for (int r = 0; r < E; ++r) v[q][r] = red32(mont32(x[r], y[r], p, pinv), p);
        if (comp == 1) {
#pragma unroll
            for (int r = 0; r < E; ++r) {
                x[r] = __ldg(A + o1 + ((u32)r << (LOGN - WB)));
                y[r] = __ldg(B + ((u32)r << (LOGN - WB)));
            }
#pragma unroll
            for (int r = 0; r < E; ++r) v[q][r] += red32(mont32(x[r], y[r], p, pinv), p);
        }
    }
    nttw_inv<LOGN, WB, NP>(v, smd, T.airp + (size_t)j * N, T.airps + (size_t)j * N, p);
    const u32 ni = fold == 1 ? T.ninvRAc[j] : T.ninvRA[j], nis = fold == 1 ? T.ninvRAc_s[j] : T.ninvRA_s[j];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        if (pr0 + q >= P) break;
        u32* out = D + (((size_t)(pr0 + q) * 3 + comp) * T.DS + j) * N;
        if (fold == 2) {  // scale already folded into the A operands
#pragma unroll
            for (int r = 0; r < E; ++r) out[((u32)r << (LOGN - WB)) | tid] = red32(v[q][r], p);
        } else {
#pragma unroll
            for (int r = 0; r < E; ++r) out[((u32)r << (LOGN - WB)) | tid] = red32(shoup32(v[q][r], ni, nis, p), p);
        }
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
        u32* Dp = D + pc * T.DS * N + n;
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
template <int NC, int RB = 4>
__global__ void __launch_bounds__(256, 2) k_mac2(const u32* __restrict__ Z, u32 zstride, const u32* __restrict__ DB,
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
        // RB rows per batch: all of a batch's loads are issued before its multiply-adds
        // (memory-level parallelism for the latency-bound stream); tail rows clamp to re-1 and
        // are masked by a zero DB word
        for (u32 r = rg; r < re; r += RB) {
            uint4 d[RB], z[RB][NC];
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const u32 rr = min(r + b, re - 1);
                d[b] = __ldg(dbp + (size_t)rr * (dbs >> 2));
#pragma unroll
                for (int c = 0; c < NC; ++c) z[b][c] = __ldg(zp + ((size_t)rr * zs + (size_t)c * zstride * N) / 4);
            }
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                if (r + b >= re) d[b] = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    g[c][0] += (u64)z[b][c].x * d[b].x;
                    g[c][1] += (u64)z[b][c].y * d[b].y;
                    g[c][2] += (u64)z[b][c].z * d[b].z;
                    g[c][3] += (u64)z[b][c].w * d[b].w;
                }
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

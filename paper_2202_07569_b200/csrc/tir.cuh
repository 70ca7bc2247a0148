// Fused tensor + INTT + scale-and-round over a thread-block cluster (mul_lazy_prepared,
// reference bfv.cpp:765-857: the tensor at :776-791, the INTT of every aux residue, the t/q
// rounding at :811-849), writing the selection value r = round(t D / q) mod each MAC prime.
//
// One cluster of J CTAs per (product, component): CTA j (= its cluster rank) forms the
// Montgomery tensor in aux prime a_j from the prepared operands and inverse-transforms it in
// registers (nttw_inv, as k_tensor_intt_r), leaving the HPS residue w_j of all N coefficients
// in its shared memory.  After one cluster barrier every CTA gathers, over distributed shared
// memory, the J residues of its N/J coefficients (coalesced ld.shared::cluster, one word per
// thread per peer) into a padded local staging array; a second barrier releases the peers.
// The rounding then runs on the tensor cores exactly as k_round_tc: per 128 coefficients one
// tcgen05.mma.kind::i8 (A = residue bytes in TMEM, B = the constant byte matrix in shared
// memory), an epilogue that recombines the column sums, adds the gamma / rho corrections and
// reduces mod the MAC primes, and the exact multiword path (round_exact) for coefficients
// whose 64-bit fractional estimate falls inside its error band.
//
// Versus k_tensor_intt_r + k_round_tc this removes the round trip of the J residue planes
// through HBM (J words written and read back per coefficient): only the Mm MAC-basis words
// leave the SM.  Output Z[pr][comp][k][N] (k < Mm), coefficient domain, consumed by k_ntt_mac.
#pragma once
#include "round.cuh"

namespace cwgpu {

template <int LOGN, int CL>
struct Tir {
    using R = RegNtt<LOGN>;
    static constexpr int T = R::T, E = R::E, WB = R::WB, N = 1 << LOGN;
    static constexpr int NPC = N / CL;          // coefficients rounded per CTA
    static constexpr int SPAD = CL + 1;         // staging row stride (conflict-free both ways)
    static constexpr int SZ0 = (N > NPC * SPAD ? N : NPC * SPAD);  // transposes / staging (words)
    static constexpr size_t SMEM = (size_t)(SZ0 + N) * 4;
};

__device__ __forceinline__ u32 cluster_rank() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
/// Remote shared-memory load: volatile (stays after the cluster barrier, in program order with
/// the other loads) but without a memory clobber, so a batch of them stays in flight together
/// instead of each being ordered before the next local store.
__device__ __forceinline__ u32 dsmem_ld(u32 local_addr, u32 rank) {
    u32 ra, v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.u32 %0, [%1];\n" : "=r"(v) : "r"(ra));
    return v;
}

/// Block (unit * CL + rank): unit = pr * 3 + comp over the P products; rank = aux prime j.
/// fold = 1: multiply the INTT output by (N 2^32)^-1 (A/a_j)^-1 here; 2: already folded into the
/// A operands (k_scale_planes).  Z: [P][3][Mm][N].
template <int LOGN, int CL, int JM, int NC>
__global__ void __launch_bounds__(RegNtt<LOGN>::T, RegNtt<LOGN>::MINB) k_tir(
    const u32* __restrict__ prepA, const u32* __restrict__ idxA, const u32* __restrict__ prepB,
    const u32* __restrict__ idxB, u32 P, DevTab T, int fold, const __grid_constant__ RoundTcPar<JM, NC> RP,
    const uint4* __restrict__ Bglob, const RoundK* __restrict__ gRK, u32* __restrict__ Z) {
    using G = Tir<LOGN, CL>;
    using RPT = RoundTcPar<JM, NC>;
    constexpr int E = G::E, WB = G::WB, N = G::N, SH = LOGN - WB, NPC = G::NPC, SPAD = G::SPAD;
    constexpr int K = RPT::K, F0 = RPT::F0, G0 = RPT::G0, KSTEPS = K / 32;
    static_assert(JM >= CL && JM % 8 == 0, "aux primes padded to the rounding width");
    static_assert(NPC % 128 == 0, "whole 128-coefficient MMA tiles per CTA");
    extern __shared__ u32 smd[];
    u32* sm = smd;              // INTT transposes, then the staging array [NPC][SPAD]
    u32* dsm = smd + G::SZ0;    // this prime's INTT output, read by the whole cluster
    __shared__ __align__(128) uint4 Bs[NC * K / 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ u32 tmem_base_sh;
    const u32 tid = threadIdx.x, warp = tid >> 5;
    const u32 J = T.J, Mm = T.Mm;
    const u32 j = cluster_rank();
    const u32 unit = blockIdx.x / CL, pr = unit / 3, comp = unit % 3;

    // ---- tensor-core setup (overlaps the operand loads of the other warps)
    for (u32 x = tid; x < NC * K / 16; x += blockDim.x) Bs[x] = Bglob[x];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }

    // ---- phase 1: tensor + INTT in prime a_j (k_tensor_intt_r, one product)
    {
        const u32 p = T.a[j], pinv = T.apinv[j];
        const size_t per = (size_t)2 * J * N, o1 = (size_t)J * N;
        const u32* A = prepA + (size_t)(idxA ? idxA[pr] : pr) * per + (size_t)j * N + tid;
        const u32* B = prepB + (size_t)(idxB ? idxB[pr] : pr) * per + (size_t)j * N + tid;
        const u32* X = A + (comp == 2 ? o1 : 0);
        const u32* Y = B + (comp == 0 ? 0 : o1);
        u32 v[1][E];
        {
            u32 x[E], y[E];
#pragma unroll
            for (int r = 0; r < E; ++r) {
                x[r] = __ldg(X + ((u32)r << SH));
                y[r] = __ldg(Y + ((u32)r << SH));
            }
#pragma unroll
            for (int r = 0; r < E; ++r) v[0][r] = red32(mont32(x[r], y[r], p, pinv), p);
            if (comp == 1) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    x[r] = __ldg(A + o1 + ((u32)r << SH));
                    y[r] = __ldg(B + ((u32)r << SH));
                }
#pragma unroll
                for (int r = 0; r < E; ++r) v[0][r] += red32(mont32(x[r], y[r], p, pinv), p);
            }
        }
        nttw_inv<LOGN, WB, 1>(v, sm, T.airp + (size_t)j * N, T.airps + (size_t)j * N, p);
        if (fold == 2) {
#pragma unroll
            for (int r = 0; r < E; ++r) dsm[((u32)r << SH) | tid] = red32(v[0][r], p);
        } else {
            const u32 ni = T.ninvRAc[j], nis = T.ninvRAc_s[j];
#pragma unroll
            for (int r = 0; r < E; ++r) dsm[((u32)r << SH) | tid] = red32(shoup32(v[0][r], ni, nis, p), p);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();  // every prime's residues are in its CTA's shared memory
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

    // ---- gather: the J residues of this CTA's NPC coefficients -> staging [NPC][SPAD]
    {
        const u32 n0 = j * NPC;
        const u32 la = smem_u32(dsm);
        constexpr int PER = NPC * CL / G::T;  // words per thread (32 at N = 8192, CL = 16)
        static_assert(PER % 8 == 0, "gather batches of 8");
#pragma unroll 1
        for (int b = 0; b < PER; b += 8) {
            u32 g[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {  // 8 remote loads in flight, then 8 local stores
                const u32 x = tid + (u32)(b + u) * G::T;
                const u32 q = x / NPC, i = x % NPC;  // peer q, coefficient i (consecutive threads: consecutive i)
                g[u] = dsmem_ld(la + (n0 + i) * 4, q);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const u32 x = tid + (u32)(b + u) * G::T;
                sm[(x % NPC) * SPAD + x / NPC] = g[u];
            }
        }
    }
    cluster_sync_all();  // all remote reads done: peers may exit; staging visible CTA-wide
    if (warp >= 4) return;

    // ---- phase 2: tensor-core rounding of NPC coefficients in 128-row tiles (warps 0-3)
    const u32 tbase = tmem_base_sh;
    const u32 ta = tbase + ((warp * 32u) << 16);
    const u32 td = ta + JM;
    const u64 bdesc0 = ((u64)((smem_u32(Bs) >> 4) & 0x3fff)) | ((u64)(128 >> 4) << 16) |
                       ((u64)((K / 16 * 128) >> 4) << 32) | (1ull << 46);
    const u32 idesc = (2u << 4) | ((u32)(NC >> 3) << 17) | ((u32)(128 >> 4) << 24);
    const u32 fA0 = T.fracA[1], fA1 = T.fracA[2];
    u32* Zu = Z + (size_t)unit * Mm * N + j * NPC;
    u32 phase = 0;
#pragma unroll 1
    for (u32 tile = 0; tile < (u32)(NPC / 128); ++tile) {
        const u32 i = tile * 128 + tid;
        const u32* srow = sm + i * SPAD;
        {
            u32 w[JM];
#pragma unroll
            for (int q = 0; q < JM; ++q) w[q] = q < CL && q < (int)J ? srow[q] : 0u;
#pragma unroll
            for (int c = 0; c < JM; c += 8)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta + c),
                             "r"(w[c]), "r"(w[c + 1]), "r"(w[c + 2]), "r"(w[c + 3]), "r"(w[c + 4]), "r"(w[c + 5]),
                             "r"(w[c + 6]), "r"(w[c + 7])
                             : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const u64 bd = bdesc0 + (u64)((s * 2 * 128) >> 4);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + JM),
                    "r"(tbase + (u32)(s * 8)), "l"(bd), "r"(idesc), "r"(s)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        {
            u32 done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                    : "=r"(done)
                    : "r"(smem_u32(&mbar)), "r"(phase)
                    : "memory");
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // fraction / gamma columns F0 .. NC-1 (17 columns) first
        u32 C[17];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];\n"
            : "=r"(C[1]), "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]), "=r"(C[8]),
              "=r"(C[9]), "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15]), "=r"(C[16])
            : "r"(td + F0 + 1)
            : "memory");
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(C[0]) : "r"(td + F0) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        u64 gs = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) gs += (u64)C[G0 - F0 + s] << (8 * s);
        const u32 gamma = (u32)((gs + (1ull << 45)) >> 46);
        u64 plo = 0, phi = 0;
#pragma unroll
        for (int s = 0; s < 6; ++s) plo += (u64)C[s] << (8 * s);
#pragma unroll
        for (int s = 6; s < 11; ++s) phi += (u64)C[s] << (8 * (s - 6));
        const u64 lo64 = plo + (phi << 48);
        const u64 hi64 = (phi >> 16) + (lo64 < plo ? 1u : 0u);
        u32 s0 = (u32)lo64, s1 = (u32)(lo64 >> 32), s2 = (u32)hi64, s3 = (u32)(hi64 >> 32);
        {
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
        const bool bad = (s1 == 0u && s0 < 64u) || (s1 >= 0xfffffff0u) || T.force_exact;
        u32* zo = Zu + i;
        {
            // residue columns, 4 MAC primes per TMEM load (warp-uniform: .sync.aligned)
            const u64 rb = (u64)(rho + (1ll << 36));
            const u32 rlo = (u32)(rb & ((1u << 30) - 1)), rhi = (u32)(rb >> 30);
#pragma unroll
            for (int k0 = 0; k0 < RPT::MMAX; k0 += 4) {
                u32 Rc[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                    "%14, %15}, [%16];\n"
                    : "=r"(Rc[0]), "=r"(Rc[1]), "=r"(Rc[2]), "=r"(Rc[3]), "=r"(Rc[4]), "=r"(Rc[5]), "=r"(Rc[6]),
                      "=r"(Rc[7]), "=r"(Rc[8]), "=r"(Rc[9]), "=r"(Rc[10]), "=r"(Rc[11]), "=r"(Rc[12]), "=r"(Rc[13]),
                      "=r"(Rc[14]), "=r"(Rc[15])
                    : "r"(td + 4 * k0)
                    : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (!bad) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int k = k0 + kk;
                        if (k < RPT::MMAX && k < (int)Mm) {
                            const uint4 q = RP.kq[k];
                            const u32 p01 = Rc[4 * kk] + (Rc[4 * kk + 1] << 8), p23 = Rc[4 * kk + 2] + (Rc[4 * kk + 3] << 8);
                            const u64 S = (u64)p01 + ((u64)p23 << 16);
                            const u64 Xv = (u64)gamma * q.z + S + RP.krm[k];
                            const u32 x = red32(mont_red64(Xv, q.x, q.y), q.x);
                            const u32 y = red32(red32(rlo + rhi * q.w, 2 * q.x), q.x);
                            zo[(size_t)k * N] = red32(x + y, q.x);
                        }
                    }
                }
            }
        }
        if (bad) {  // exact multiword path (no tensor-memory instructions inside)
            HpsState h;
#pragma unroll
            for (int q = 0; q < JM; ++q) if (q < (int)J) h.w[q] = srow[q];
            h.gamma = gamma;
            h.rho = rho;
            u32 Rw[kAW + 2];
            const bool neg = round_exact(h, *T.self, Rw);
            for (u32 k = 0; k < Mm; ++k) {
                const u32 a = gRK[k].a;
                u32 r = mag_mod32(Rw, a, gRK[k].abar);
                if (neg && r) r = a - r;
                zo[(size_t)k * N] = r;
            }
        }
        __syncwarp();
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        // next tile's tcgen05.st (A) / MMA (D) only after every thread's D reads: the bar.sync at
        // the top of the next iteration orders them
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(128));
}

}  // namespace cwgpu

// Microbenchmark variants of the register NTT (window width / polys per CTA / occupancy);
// used only by cwg_bench_kernel (scripts/bench_ntt.py) to pick the production
// configuration (RegNtt in ntt_reg.cuh).  Not on the answer path.
#pragma once
#include "ntt_reg.cuh"

namespace cwgpu {

template <int LOGN, int WB, int NP, int MINB, bool INV, bool JSLOW = false, int FAKE = 0>
__global__ void __launch_bounds__(NttW<LOGN, WB>::T, MINB) k_nttw_bench(u32* __restrict__ base, DevTab T) {
    using G = NttW<LOGN, WB>;
    extern __shared__ u32 smb[];
    const u32 tid = threadIdx.x;
    // JSLOW: prime-major block order (every SM works on the same twiddle table at a time)
    const u32 j = JSLOW ? (u32)(((u64)blockIdx.x * T.J) / gridDim.x) : blockIdx.x % T.J;
    const u32 p = T.a[j];
    u32 v[NP][G::E];
    u32* d = base + (size_t)blockIdx.x * NP * G::N;
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < G::E; ++r)
            v[q][r] = (FAKE & 12) == 4 || (FAKE & 12) == 12 ? (tid * 7 + r * 13 + q) & 0x3fffffffu
                                 : d[(size_t)q * G::N + (((u32)r << (LOGN - WB)) | tid)] & 0x3fffffffu;
    if (INV) nttw_inv<LOGN, WB, NP>(v, smb, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, p);
    else nttw_fwd<LOGN, WB, NP, FAKE>(v, smb, T.arp + (size_t)j * G::N, T.arps + (size_t)j * G::N, p);
    if constexpr ((FAKE & 16) != 0 && NP == 1) {  // PERM-order output through smem + one bulk copy
        bulk_store_poly<LOGN, WB>(d, smb, v[0]);
        return;
    }
    if ((FAKE & 4) || (FAKE & 8)) {  // keep the result live without storing it (4: no loads either)
        u32 x = 0;
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int r = 0; r < G::E; ++r) x ^= v[q][r];
        if (x == 0x12345678u) d[tid] = x;
        return;
    }
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < G::E; r += 4)
            *reinterpret_cast<uint4*>(d + (size_t)q * G::N + (tid << WB) + r) = make_uint4(v[q][r], v[q][r + 1], v[q][r + 2], v[q][r + 3]);
    (void)0;
}

/// Persistent variant: CTA loops over polynomials blockIdx.x, +gridDim.x, ...; the next
/// polynomial is copied into a shared-memory staging buffer with cp.async while the current one
/// is transformed (hides the load latency that dominates the non-butterfly time).
template <int LOGN, int WB, int MINB>
__global__ void __launch_bounds__(NttW<LOGN, WB>::T, MINB) k_nttw_bench_pf(u32* __restrict__ base, DevTab T, u32 npolys) {
    using G = NttW<LOGN, WB>;
    extern __shared__ u32 smb[];
    u32* stage = smb + G::N;  // staging buffer (natural order)
    const u32 tid = threadIdx.x;
    u32 poly = blockIdx.x;
    auto issue = [&](u32 pl) {
        const u32* src = base + (size_t)pl * G::N;
#pragma unroll
        for (int r = 0; r < G::E; ++r) {
            const u32 x = ((u32)r << (LOGN - WB)) | tid;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((u32)__cvta_generic_to_shared(stage + x)),
                         "l"(src + x));
        }
        asm volatile("cp.async.commit_group;");
    };
    if (poly < npolys) issue(poly);
    for (; poly < npolys; poly += gridDim.x) {
        const u32 j = poly % T.J;
        const u32 p = T.a[j];
        u32 v[1][G::E];
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int r = 0; r < G::E; ++r) v[0][r] = stage[((u32)r << (LOGN - WB)) | tid] & 0x3fffffffu;  // own words only
        if (poly + gridDim.x < npolys) issue(poly + gridDim.x);
        nttw_fwd<LOGN, WB, 1>(v, smb, T.arp + (size_t)j * G::N, T.arps + (size_t)j * G::N, p);
        u32* d = base + (size_t)poly * G::N;
#pragma unroll
        for (int r = 0; r < G::E; r += 4)
            *reinterpret_cast<uint4*>(d + (tid << WB) + r) = make_uint4(v[0][r], v[0][r + 1], v[0][r + 2], v[0][r + 3]);
        __syncthreads();  // transposes of this polynomial done before the next one reuses smb
    }
}

}  // namespace cwgpu

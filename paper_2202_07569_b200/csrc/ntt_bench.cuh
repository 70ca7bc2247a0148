// Microbenchmark variants of the register NTT (occupancy vs ILP trade-offs); used only by
// cwg_bench_kernel to pick the production configuration.  Not on the answer path.
#pragma once
#include "ntt_reg.cuh"

namespace cwgpu {

template <int LOGN, int NP, int MINB, bool INV>
__global__ void __launch_bounds__(NttGeom<LOGN>::T, MINB) k_ntt_bench(u32* __restrict__ base, DevTab T) {
    using G = NttGeom<LOGN>;
    extern __shared__ u32 smb[];
    const u32 tid = threadIdx.x;
    const u32 j = blockIdx.x % T.J;
    const u32 p = T.a[j];
    u32 v[NP][16];
    u32* d = base + (size_t)blockIdx.x * NP * G::N;
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < 16; ++r) v[q][r] = d[(size_t)q * G::N + (((u32)r << (LOGN - 4)) | tid)] & 0x3fffffffu;
    if (INV) ntt32_inv_reg<LOGN, NP>(v, smb, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, p);
    else ntt32_fwd_reg<LOGN, NP>(v, smb, T.arp + (size_t)j * G::N, T.arps + (size_t)j * G::N, p);
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < 16; ++r) d[(size_t)q * G::N + (tid << 4) + r] = v[q][r];
}

}  // namespace cwgpu

// Microbenchmark variants of the register NTT (window width / polys per CTA / occupancy);
// used only by cwg_bench_kernel (scripts/bench_ntt.py) to pick the production
// configuration (RegNtt in ntt_reg.cuh).  Not on the answer path.
#pragma once
#include "ntt_reg.cuh"

namespace cwgpu {

template <int LOGN, int WB, int NP, int MINB, bool INV, bool JSLOW = false>
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
        for (int r = 0; r < G::E; ++r) v[q][r] = d[(size_t)q * G::N + (((u32)r << (LOGN - WB)) | tid)] & 0x3fffffffu;
    if (INV) nttw_inv<LOGN, WB, NP>(v, smb, T.airp + (size_t)j * G::N, T.airps + (size_t)j * G::N, p);
    else nttw_fwd<LOGN, WB, NP>(v, smb, T.arp + (size_t)j * G::N, T.arps + (size_t)j * G::N, p);
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int r = 0; r < G::E; r += 4)
            *reinterpret_cast<uint4*>(d + (size_t)q * G::N + (tid << WB) + r) = make_uint4(v[q][r], v[q][r + 1], v[q][r + 2], v[q][r + 3]);
}

}  // namespace cwgpu

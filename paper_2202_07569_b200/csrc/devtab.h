// Device-resident parameter tables shared by every kernel (passed by value; all
// arrays live in one device allocation owned by the context).
#pragma once
#include <cstdint>

namespace cwgpu {

constexpr int kMaxL = 8;    // chain primes
constexpr int kMaxJ = 40;   // 31-bit aux primes
constexpr int kQW = 16;     // 32-bit limbs for q (<= 480 bits) + headroom
constexpr int kAW = 44;     // 32-bit limbs for A (<= 40 * 31 bits) + headroom

struct DevTab {
    std::uint32_t N, logN, L, J, Mm, Dr, Dg, relin_bits, galois_bits, QW, AW, gbits;
    std::uint32_t DS;           // planes per (product, component) in the tensor / rounding buffer D (>= J)
    std::uint32_t force_exact;  // test knob (env CWGPU_FORCE_EXACT): every rounding / centring decision
                                // takes the exact multiword path
    std::uint64_t t;
    // ---- chain primes q_i (bfv.cpp:31-129 restated) ----
    const std::uint64_t* q;        // [L]
    const std::uint64_t* q_mu96;   // floor(2^96 / q_i)
    const std::uint64_t* q_gh;     // floor(2^128 / q_i) >> 64
    const std::uint64_t* q_gl;     // floor(2^128 / q_i) & (2^64-1)
    const std::uint64_t* muq;      // (q/q_i)^-1 mod q_i
    const std::uint64_t* muq_s;    // Shoup companion
    const std::uint64_t* ninv;     // N^-1 mod q_i
    const std::uint64_t* ninv_s;
    const std::uint64_t* delta;    // floor(q/t) mod q_i
    const std::uint64_t* crp;      // [L][N] root powers (ring.cpp:57-63)
    const std::uint64_t* crps;
    const std::uint64_t* cirp;
    const std::uint64_t* cirps;
    const std::uint32_t* qw;       // q, 32-bit limbs [QW]
    const std::uint32_t* qov;      // q / q_i, [L][QW]
    // ---- aux primes a_j < 2^31 ----
    const std::uint32_t* a;        // [J]
    const std::uint32_t* apinv;    // -a_j^-1 mod 2^32
    const std::uint64_t* abar;     // floor(2^64 / a_j)
    const std::uint32_t* a2_64;    // 2^64 mod a_j
    const std::uint32_t* ninvA;    // N^-1 mod a_j        (+ Shoup)
    const std::uint32_t* ninvA_s;
    const std::uint32_t* ninvRA;   // (N * 2^32)^-1 mod a_j (+ Shoup): undoes the Montgomery factor
    const std::uint32_t* ninvRA_s;
    const std::uint32_t* ninvRAc;  // ninvRA (A/a_j)^-1 mod a_j (+ Shoup): INTT output = HPS residue w_j
    const std::uint32_t* ninvRAc_s;
    const std::uint32_t* arp;      // [J][N]
    const std::uint32_t* arps;
    const std::uint32_t* airp;
    const std::uint32_t* airps;
    // ---- chain -> aux centred lift (to_aux_basis, bfv.cpp:718-744) ----
    // residue_j = sum_i (ylo_i V[i][j] + yhi_i V2[i][j]) + rho (a_j - W[j])  mod a_j
    // Montgomery variant (x 2^32) for tensor operands, plain variant for MAC lifts.
    const std::uint32_t* liftV_m;  // [L][J]
    const std::uint32_t* liftV2_m;
    const std::uint32_t* liftW_m;  // [J]
    const std::uint32_t* liftV_n;
    const std::uint32_t* liftV2_n;
    const std::uint32_t* liftW_n;
    // ---- A -> integer (HPS scaling of t*D/q) ----
    const std::uint32_t* chat;     // (A/a_j)^-1 mod a_j (+ Shoup)
    const std::uint32_t* chat_s;
    const std::uint64_t* aF;       // floor(2^(64-gbits) / a_j)
    const std::uint32_t* frac96;   // [J][3]  frac(t (A/a_j) / q) * 2^96
    const std::uint32_t* fracA;    // [3]     frac(t A / q) * 2^96
    const std::uint32_t* Imod;     // [J][Mm] floor(t (A/a_j) / q) mod a_k
    const std::uint32_t* IAmod;    // [Mm]    floor(t A / q) mod a_k
    const std::uint64_t* ImodQ;    // [J][L]  ... mod q_i
    const std::uint64_t* IAmodQ;   // [L]
    const std::uint32_t* Aw;       // A, 32-bit limbs [AW]
    const std::uint32_t* Aov;      // A / a_j, [J][AW]
    // ---- MAC basis M = a_0..a_{Mm-1} -> chain ----
    const std::uint32_t* mhat;     // (M/a_k)^-1 mod a_k (+ Shoup)
    const std::uint32_t* mhat_s;
    const std::uint64_t* mF;       // floor(2^(64-gbits) / a_k)
    const std::uint64_t* Mconv;    // [Mm][L] (M/a_k) mod q_i
    const std::uint64_t* MnegQ;    // [L] (-M) mod q_i
    // ---- diagnostics ----
    unsigned long long* fallbacks;  // exact-path counter (device)
    const DevTab* self;             // device-memory copy of this table (slow paths take it by
                                    // reference so kernels never spill the parameter block)
};

}  // namespace cwgpu

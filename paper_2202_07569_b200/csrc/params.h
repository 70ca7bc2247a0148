// Host-side parameter derivation for the B200 answer path.
//
// Chain-side constants restate BfvContext (reference bfv.cpp:67-129) and the NTT
// tables restate RingContext::create (ring.cpp:30-74): psi = g^((q-1)/2N) with g the
// smallest primitive root, tables indexed by bit-reversed exponent, so the device
// NTT reproduces RingContext::ntt_forward element for element (the evaluation keys
// arrive in that layout).
//
// The tensor / MAC basis is OUR choice ("the choice of aux primes is
// free"): 30-bit NTT primes instead of the reference's 59-bit ones, sized so that
//   A = prod a_j  >  2^6 * N * q^2                 (exact tensor, bfv.cpp:103-108)
//   M = prod_{j<Mm} a_j > 2^6 * 2 * |sum_r DB_r * sel_r|   (exact payload MAC)
// and the exact t/q rounding is computed by HPS-style scaling with an exact
// multiword fallback.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace cwgpu {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using u128 = unsigned __int128;

/// Minimal host big integer (little-endian 64-bit limbs), setup-time only.
struct Big {
    std::vector<u64> l;
    Big() = default;
    explicit Big(u64 v) { if (v) l.push_back(v); }
    void trim() { while (!l.empty() && l.back() == 0) l.pop_back(); }
    bool zero() const { return l.empty(); }
    unsigned bits() const;
    int cmp(const Big& o) const;
    Big operator+(const Big& o) const;
    Big operator-(const Big& o) const;  // requires *this >= o
    Big mul_u64(u64 v) const;
    Big operator*(const Big& o) const;
    Big shl(unsigned s) const;
    u64 mod_u64(u64 m) const;
    Big div_u64(u64 m) const;
    static void divmod(const Big& a, const Big& b, Big& q, Big& r);
    std::vector<u32> limbs32(std::size_t n) const;  // zero padded
    u64 limb(std::size_t i) const { return i < l.size() ? l[i] : 0; }
};

u64 mulmod64(u64 a, u64 b, u64 m);
u64 powmod64(u64 b, u64 e, u64 m);
u64 invmod64(u64 a, u64 m);
bool is_prime64(u64 n);
/// numeric.cpp:63-84
u64 find_ntt_prime_below(u64 hint, u64 step);
std::vector<u64> find_ntt_primes_below(u64 hint, u64 step, std::size_t count,
                                       const std::vector<u64>& exclude = {});
/// numeric.cpp:86-108
u64 primitive_root(u64 p);

/// Per-prime negacyclic NTT tables in the reference convention.
struct NttTables {
    std::vector<u64> rp, rps, irp, irps;  // root_pow / Shoup, inverse root_pow / Shoup
    u64 ninv = 0;
};
NttTables make_ntt_tables(std::size_t N, u64 q, unsigned shoup_bits);

struct ChainParams {
    u32 N = 0, logN = 0, L = 0;
    u64 t = 0;
    std::vector<u64> q;
    unsigned relin_bits = 16, galois_bits = 16;
    u32 Dr = 0, Dg = 0;  // digit counts (bfv.cpp:133-136)
    Big Q;
    unsigned q_bits = 0;
};

/// Throws std::invalid_argument with the reference's messages where they exist.
ChainParams make_chain(u32 N, u64 t, const std::vector<u64>& primes, unsigned relin_bits,
                       unsigned galois_bits);

/// Aux (tensor) basis A = a_0..a_{J-1}; the MAC basis is its prefix a_0..a_{Mm-1}.
struct AuxBasis {
    std::vector<u64> a;
    u32 J = 0, Mm = 0;
};
AuxBasis choose_aux_basis(const ChainParams& cp, u64 n_rows_total);

}  // namespace cwgpu

// Host-side parameter derivation (see params.h).
#include "params.h"

#include <algorithm>
#include <stdexcept>

namespace cwgpu {

unsigned Big::bits() const {
    if (l.empty()) return 0;
    return 64 * unsigned(l.size() - 1) + (64 - __builtin_clzll(l.back()));
}

int Big::cmp(const Big& o) const {
    if (l.size() != o.l.size()) return l.size() < o.l.size() ? -1 : 1;
    for (std::size_t i = l.size(); i-- > 0;)
        if (l[i] != o.l[i]) return l[i] < o.l[i] ? -1 : 1;
    return 0;
}

Big Big::operator+(const Big& o) const {
    Big r;
    std::size_t n = std::max(l.size(), o.l.size());
    r.l.resize(n + 1);
    u64 c = 0;
    for (std::size_t i = 0; i < n; ++i) {
        u128 s = u128(limb(i)) + o.limb(i) + c;
        r.l[i] = u64(s);
        c = u64(s >> 64);
    }
    r.l[n] = c;
    r.trim();
    return r;
}

Big Big::operator-(const Big& o) const {
    Big r;
    r.l.resize(l.size());
    u64 b = 0;
    for (std::size_t i = 0; i < l.size(); ++i) {
        u128 need = u128(o.limb(i)) + b;
        r.l[i] = l[i] - u64(need);
        b = u128(l[i]) < need;
    }
    if (b) throw std::logic_error("Big: negative result");
    r.trim();
    return r;
}

Big Big::mul_u64(u64 v) const {
    Big r;
    r.l.resize(l.size() + 1);
    u64 c = 0;
    for (std::size_t i = 0; i < l.size(); ++i) {
        u128 cur = u128(l[i]) * v + c;
        r.l[i] = u64(cur);
        c = u64(cur >> 64);
    }
    r.l[l.size()] = c;
    r.trim();
    return r;
}

Big Big::operator*(const Big& o) const {
    Big r;
    r.l.assign(l.size() + o.l.size() + 1, 0);
    for (std::size_t i = 0; i < l.size(); ++i) {
        u64 c = 0;
        for (std::size_t j = 0; j < o.l.size(); ++j) {
            u128 cur = u128(l[i]) * o.l[j] + r.l[i + j] + c;
            r.l[i + j] = u64(cur);
            c = u64(cur >> 64);
        }
        std::size_t k = i + o.l.size();
        while (c) {
            u128 cur = u128(r.l[k]) + c;
            r.l[k++] = u64(cur);
            c = u64(cur >> 64);
        }
    }
    r.trim();
    return r;
}

Big Big::shl(unsigned s) const {
    Big r;
    if (l.empty()) return r;
    unsigned w = s / 64, b = s % 64;
    r.l.assign(l.size() + w + 1, 0);
    for (std::size_t i = 0; i < l.size(); ++i) {
        r.l[i + w] |= l[i] << b;
        if (b) r.l[i + w + 1] |= l[i] >> (64 - b);
    }
    r.trim();
    return r;
}

u64 Big::mod_u64(u64 m) const {
    u128 r = 0;
    for (std::size_t i = l.size(); i-- > 0;) r = ((r << 64) | l[i]) % m;
    return u64(r);
}

Big Big::div_u64(u64 m) const {
    Big q;
    q.l.resize(l.size());
    u128 r = 0;
    for (std::size_t i = l.size(); i-- > 0;) {
        u128 cur = (r << 64) | l[i];
        q.l[i] = u64(cur / m);
        r = cur % m;
    }
    q.trim();
    return q;
}

void Big::divmod(const Big& a, const Big& b, Big& q, Big& r) {
    if (b.zero()) throw std::logic_error("Big: division by zero");
    q = Big();
    r = Big();
    unsigned nb = a.bits();
    q.l.assign((nb + 63) / 64 + 1, 0);
    for (unsigned i = nb; i-- > 0;) {
        r = r.shl(1);
        if ((a.limb(i / 64) >> (i % 64)) & 1) {
            if (r.l.empty()) r.l.push_back(1); else r.l[0] |= 1;
        }
        if (r.cmp(b) >= 0) {
            r = r - b;
            q.l[i / 64] |= u64(1) << (i % 64);
        }
    }
    q.trim();
    r.trim();
}

std::vector<u32> Big::limbs32(std::size_t n) const {
    std::vector<u32> out(n, 0);
    for (std::size_t i = 0; i < n && i / 2 < l.size(); ++i) out[i] = u32(l[i / 2] >> (32 * (i % 2)));
    if (bits() > 32 * n) throw std::logic_error("Big: value does not fit the limb budget");
    return out;
}

u64 mulmod64(u64 a, u64 b, u64 m) { return u64((u128(a) * b) % m); }

u64 powmod64(u64 b, u64 e, u64 m) {
    u64 r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod64(r, b, m);
        b = mulmod64(b, b, m);
        e >>= 1;
    }
    return r;
}

u64 invmod64(u64 a, u64 m) {
    __int128 t = 0, nt = 1, r = m, nr = a % m;
    while (nr) {
        __int128 qq = r / nr, tmp = t - qq * nt;
        t = nt;
        nt = tmp;
        tmp = r - qq * nr;
        r = nr;
        nr = tmp;
    }
    if (r != 1) throw std::invalid_argument("inv_mod: operand not invertible");
    if (t < 0) t += m;
    return u64(t);
}

bool is_prime64(u64 n) {
    static const u64 W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : W) if (n % p == 0) return n == p;
    u64 d = n - 1;
    unsigned s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (u64 a : W) {
        u64 x = powmod64(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (unsigned i = 1; i < s; ++i) {
            x = mulmod64(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

u64 find_ntt_prime_below(u64 hint, u64 step) {
    u64 p = hint - (hint % step) + 1;
    if (p > hint) p -= step;
    while (p > 3 * step) {
        if (is_prime64(p)) return p;
        p -= step;
    }
    throw std::runtime_error("find_ntt_prime_below: no prime in range");
}

std::vector<u64> find_ntt_primes_below(u64 hint, u64 step, std::size_t count,
                                       const std::vector<u64>& exclude) {
    std::vector<u64> out;
    u64 p = hint + 1;
    while (out.size() < count) {
        p = find_ntt_prime_below(p - 1, step);
        if (std::find(exclude.begin(), exclude.end(), p) == exclude.end()) out.push_back(p);
    }
    return out;
}

u64 primitive_root(u64 p) {
    u64 phi = p - 1, n = phi;
    std::vector<u64> f;
    for (u64 x = 2; x * x <= n; ++x) {
        if (n % x == 0) {
            f.push_back(x);
            while (n % x == 0) n /= x;
        }
    }
    if (n > 1) f.push_back(n);
    for (u64 g = 2; g < p; ++g) {
        bool ok = true;
        for (u64 x : f) if (powmod64(g, phi / x, p) == 1) { ok = false; break; }
        if (ok) return g;
    }
    throw std::runtime_error("primitive_root: none found");
}

static unsigned bitrev(unsigned v, unsigned bits) {
    unsigned r = 0;
    for (unsigned i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1);
    return r;
}

NttTables make_ntt_tables(std::size_t N, u64 q, unsigned shoup_bits) {
    NttTables t;
    unsigned logn = 0;
    while ((std::size_t(1) << logn) < N) ++logn;
    const u64 g = primitive_root(q);
    const u64 psi = powmod64(g, (q - 1) / (2 * N), q);
    if (powmod64(psi, N, q) != q - 1) throw std::runtime_error("NTT setup: psi^N != -1");
    const u64 psi_inv = invmod64(psi, q);
    t.rp.resize(N); t.rps.resize(N); t.irp.resize(N); t.irps.resize(N);
    for (std::size_t i = 0; i < N; ++i) {
        unsigned r = bitrev(unsigned(i), logn);
        t.rp[i] = powmod64(psi, r, q);
        t.irp[i] = powmod64(psi_inv, r, q);
        t.rps[i] = u64((u128(t.rp[i]) << shoup_bits) / q);
        t.irps[i] = u64((u128(t.irp[i]) << shoup_bits) / q);
    }
    t.ninv = invmod64(N % q, q);
    return t;
}

ChainParams make_chain(u32 N, u64 t, const std::vector<u64>& primes, unsigned relin_bits,
                       unsigned galois_bits) {
    ChainParams cp;
    if (N < 8 || (N & (N - 1))) throw std::invalid_argument("ring degree must be a power of two >= 8");
    if (N > 32768) throw std::invalid_argument("cwgpu: ring degree above 32768 is not supported");
    // bfv.cpp:177-191 (validate), with the chain capacity of this implementation.
    if (primes.empty() || primes.size() > 8)
        throw std::invalid_argument("coefficient chain must have 1..8 primes");
    if (!is_prime64(t)) throw std::invalid_argument("plaintext modulus must be prime");
    if (t >= (u64(1) << 31)) throw std::invalid_argument("cwgpu: plaintext modulus must be below 2^31");
    for (std::size_t i = 0; i < primes.size(); ++i) {
        const u64 p = primes[i];
        if (!is_prime64(p) || (p - 1) % (2 * u64(N)) != 0)
            throw std::invalid_argument("chain prime not NTT friendly");
        if (p <= t) throw std::invalid_argument("chain prime must exceed t");
        if (p >= (u64(1) << 60)) throw std::invalid_argument("chain primes must be below 2^60");
        if (p <= (u64(1) << 32)) throw std::invalid_argument("cwgpu: chain primes must exceed 2^32");
        for (std::size_t j = i + 1; j < primes.size(); ++j)
            if (primes[j] == p) throw std::invalid_argument("chain primes must be distinct");
    }
    if (relin_bits > 60 || galois_bits > 60)
        throw std::invalid_argument("cwgpu: digit width above 60 bits is not supported");
    cp.N = N;
    while ((1u << cp.logN) < N) ++cp.logN;
    cp.L = u32(primes.size());
    cp.t = t;
    cp.q = primes;
    cp.relin_bits = relin_bits;
    cp.galois_bits = galois_bits;
    cp.Q = Big(1);
    for (u64 p : primes) cp.Q = cp.Q.mul_u64(p);
    cp.q_bits = cp.Q.bits();
    auto digits = [&](unsigned b) { return b == 0 ? cp.L : (cp.q_bits + b - 1) / b; };
    cp.Dr = digits(relin_bits);
    cp.Dg = digits(galois_bits);
    return cp;
}

AuxBasis choose_aux_basis(const ChainParams& cp, u64 n_rows_total) {
    // |D| <= N q^2 / 2 for the tensor of centred operands (comp 1 = a0 b1 + a1 b0), and the HPS
    // rounding needs the integer gamma = round(sum_j w_j / a_j) with sum_j w_j / a_j = gamma + D / A:
    // A > N q^2 (1 + 2^-8) keeps |D / A| <= 1/2 - 2^-10, far outside the J 2^-16 error of the
    // 46-bit fixed-point gamma estimate (round.cuh), and A > 2 |D| for the centred representative.
    const Big qq = cp.Q * cp.Q;
#ifdef CWGPU_AUX_MARGIN6  // A/B builds only: the earlier, looser bound A > 2^6 N q^2 (C2-C4: J = 16)
    Big needA = qq.mul_u64(u64(cp.N) << 6);
#else
    Big needA = qq.mul_u64(u64(cp.N)) + qq.mul_u64(u64(cp.N)).div_u64(256);
#endif
    // |sel| <= t N q / 2 + 1 (rounded tensor) or q / 2 (a lifted ciphertext);
    // |MAC| <= |sel| (t-1) N n;  M > 2 |MAC| (1 + 2^-20): the centred value, and the MAC -> chain
    // conversion's gamma = round(sum v_k / m_k) (58-bit fixed point, error < Mm 2^-28) stays exact
    // with |MAC / M| < 1/2 - 2^-22.  (The first version asked M > 2^7 |MAC|: C3 / C4 Mm = 11, now 10.)
    Big selb = cp.Q.mul_u64(cp.t).mul_u64(cp.N).div_u64(2) + Big(1);
    Big mac2 = selb.mul_u64(cp.t - 1).mul_u64(cp.N).mul_u64(std::max<u64>(n_rows_total, 1)).mul_u64(2);
#ifdef CWGPU_AUX_MARGIN6
    Big needM = mac2.mul_u64(64);
#else
    Big needM = mac2 + mac2.div_u64(u64(1) << 20);
#endif
    AuxBasis ab;
    // 30-bit NTT-friendly primes, descending below 2^30: 4p < 2^32 allows Harvey-style lazy
    // butterflies in 32-bit words and 16 residue products fit one u64 accumulator.
    const u64 step = 2 * u64(cp.N);
    u64 p = (u64(1) << 30);
    Big prod(1);
    u32 J = 0, Mm = 0;
    while (prod.cmp(needA) <= 0 || prod.cmp(needM) <= 0) {
        p = find_ntt_prime_below(p - 1, step);
        ab.a.push_back(p);
        prod = prod.mul_u64(p);
        ++J;
        if (Mm == 0 && prod.cmp(needM) > 0) Mm = J;
        if (J > 40) throw std::invalid_argument("cwgpu: parameters need more than 40 aux primes");
    }
    ab.J = J;
    ab.Mm = Mm;
    return ab;
}

}  // namespace cwgpu

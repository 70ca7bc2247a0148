// CPU client side of the protocol: key generation, query encryption and response
// decryption.  Not on the server hot path; it produces the benchmark's inputs and
// checks its outputs on the GPU box (where the reference is not available).
//
// Restates the reference's seeded derivations so that the same seed yields the same
// keys and ciphertexts as the reference client:
//   Seed256::from_u64            prf.hpp:18-22
//   ChaChaRng (RFC 7539 block)    prf.cpp:37-94
//   derive_seed                   bfv.cpp:19-24
//   bfv_keygen / make_ks_key      bfv.cpp:376-406, 465-488
//   encrypt                       bfv.cpp:521-549 (index passed explicitly instead of the
//                                 process-global counter, bfv.cpp:518)
//   pack_query_bits               expansion.cpp:17-38
//   decrypt                       bfv.cpp:551-595 (round(t x / q) mod t)
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cwgpu_client.h"
#include "params.h"

namespace cwgpu {
using i64 = std::int64_t;
namespace {

thread_local std::string c_err;

struct Seed {
    u64 w[4];
    static Seed from_u64(u64 v) { return Seed{{v, 0x9e3779b97f4a7c15ULL, 0xbf58476d1ce4e5b9ULL, 0x94d049bb133111ebULL}}; }
};

class Rng {
public:
    Rng(const Seed& s, u64 stream) {
        in_[0] = 0x61707865; in_[1] = 0x3320646e; in_[2] = 0x79622d32; in_[3] = 0x6b206574;
        for (int i = 0; i < 4; ++i) {
            in_[4 + 2 * i] = (u32)s.w[i];
            in_[5 + 2 * i] = (u32)(s.w[i] >> 32);
        }
        in_[12] = 0;
        in_[13] = (u32)stream;
        in_[14] = (u32)(stream >> 32);
        in_[15] = 0;
    }
    u64 next_u64() {
        if (pos_ + 2 > 16) refill();
        u64 lo = blk_[pos_], hi = blk_[pos_ + 1];
        pos_ += 2;
        return lo | (hi << 32);
    }
    u64 uniform(u64 bound) {
        if (bound <= 1) return 0;
        const u64 limit = (~0ull) - (~0ull) % bound;
        u64 v;
        do { v = next_u64(); } while (v >= limit);
        return v % bound;
    }
    int ternary() { return (int)uniform(3) - 1; }
    int noise() {
        u64 a = next_u64() & ((1ull << 20) - 1), b = next_u64() & ((1ull << 20) - 1);
        return __builtin_popcountll(a) - __builtin_popcountll(b);
    }

private:
    static u32 rotl(u32 x, int n) { return (x << n) | (x >> (32 - n)); }
    static void qr(u32& a, u32& b, u32& c, u32& d) {
        a += b; d ^= a; d = rotl(d, 16);
        c += d; b ^= c; b = rotl(b, 12);
        a += b; d ^= a; d = rotl(d, 8);
        c += d; b ^= c; b = rotl(b, 7);
    }
    void refill() {
        u32 x[16];
        std::memcpy(x, in_, sizeof(x));
        for (int r = 0; r < 10; ++r) {
            qr(x[0], x[4], x[8], x[12]); qr(x[1], x[5], x[9], x[13]);
            qr(x[2], x[6], x[10], x[14]); qr(x[3], x[7], x[11], x[15]);
            qr(x[0], x[5], x[10], x[15]); qr(x[1], x[6], x[11], x[12]);
            qr(x[2], x[7], x[8], x[13]); qr(x[3], x[4], x[9], x[14]);
        }
        for (int i = 0; i < 16; ++i) blk_[i] = x[i] + in_[i];
        if (++in_[12] == 0) ++in_[15];
        pos_ = 0;
    }
    u32 in_[16];
    u32 blk_[16];
    int pos_ = 16;
};

Seed derive_seed(const Seed& m, u64 domain, u64 index) {
    Rng r(m, (domain << 48) ^ index);
    Seed s;
    for (auto& w : s.w) w = r.next_u64();
    return s;
}

struct Ring {
    u64 q;
    u32 N, logN;
    NttTables t;
    u64 ninv_s;
    static u64 mshoup(u64 x, u64 w, u64 ws, u64 q) { return x * w - (u64)(((u128)x * ws) >> 64) * q; }
    void fwd(u64* a) const {
        const u64 tq = 2 * q;
        u32 tt = N;
        for (u32 m = 1; m < N; m <<= 1) {
            tt >>= 1;
            for (u32 i = 0; i < m; ++i) {
                const u64 w = t.rp[m + i], ws = t.rps[m + i];
                u64* lo = a + 2 * i * tt;
                u64* hi = lo + tt;
                for (u32 j = 0; j < tt; ++j) {
                    u64 u = lo[j];
                    if (u >= tq) u -= tq;
                    const u64 v = mshoup(hi[j], w, ws, q);
                    lo[j] = u + v;
                    hi[j] = u - v + tq;
                }
            }
        }
        for (u32 j = 0; j < N; ++j) {
            u64 v = a[j];
            if (v >= tq) v -= tq;
            if (v >= q) v -= q;
            a[j] = v;
        }
    }
    void inv(u64* a) const {
        const u64 tq = 2 * q;
        u32 tt = 1;
        for (u32 m = N; m > 1; m >>= 1) {
            const u32 h = m >> 1;
            u64* lo = a;
            for (u32 i = 0; i < h; ++i) {
                const u64 w = t.irp[h + i], ws = t.irps[h + i];
                u64* hi = lo + tt;
                for (u32 j = 0; j < tt; ++j) {
                    const u64 u = lo[j], v = hi[j];
                    u64 s = u + v;
                    if (s >= tq) s -= tq;
                    lo[j] = s;
                    hi[j] = mshoup(u - v + tq, w, ws, q);
                }
                lo += 2 * tt;
            }
            tt <<= 1;
        }
        for (u32 j = 0; j < N; ++j) {
            u64 v = mshoup(a[j], t.ninv, ninv_s, q);
            if (v >= q) v -= q;
            a[j] = v;
        }
    }
    /// negacyclic product (ring.cpp:159-170)
    std::vector<u64> mul(const std::vector<u64>& a, const std::vector<u64>& b) const {
        std::vector<u64> x = a, y = b;
        fwd(x.data());
        fwd(y.data());
        for (u32 i = 0; i < N; ++i) x[i] = mulmod64(x[i], y[i], q);
        inv(x.data());
        return x;
    }
};

struct Client {
    ChainParams cp;
    std::vector<Ring> rq;
    Seed seed;
    std::vector<int8_t> s;
    std::vector<std::vector<u64>> s_rns;
    std::vector<u64> delta;  // floor(q/t) mod q_i
    u32 levels = 0;
    std::vector<u64> relin;   // [Dr][2][L][N]
    std::vector<u64> galois;  // [levels][Dg][2][L][N]

    std::vector<u64> reduce_signed(const std::vector<i64>& v, u32 i) const {
        std::vector<u64> o(cp.N);
        const i64 q = (i64)cp.q[i];
        for (u32 n = 0; n < cp.N; ++n) {
            i64 x = v[n] % q;
            if (x < 0) x += q;
            o[n] = (u64)x;
        }
        return o;
    }

    std::vector<std::vector<u64>> uniform_rns(const Seed& sd) const {
        std::vector<std::vector<u64>> out(cp.L, std::vector<u64>(cp.N));
        for (u32 i = 0; i < cp.L; ++i) {
            Rng r(sd, i);
            for (auto& x : out[i]) x = r.uniform(cp.q[i]);
        }
        return out;
    }

    std::vector<std::vector<u64>> digit_factors(unsigned bits, u32 digits) const {
        std::vector<std::vector<u64>> f(digits, std::vector<u64>(cp.L));
        for (u32 d = 0; d < digits; ++d) {
            Big factor;
            if (bits == 0) {
                Big ov = cp.Q.div_u64(cp.q[d]);
                u64 mu = invmod64(ov.mod_u64(cp.q[d]), cp.q[d]);
                Big qq, rr;
                Big::divmod(ov.mul_u64(mu), cp.Q, qq, rr);
                factor = rr;
            } else {
                factor = Big(1).shl(bits * d);
            }
            for (u32 i = 0; i < cp.L; ++i) f[d][i] = factor.mod_u64(cp.q[i]);
        }
        return f;
    }

    /// make_ks_key (bfv.cpp:376-406): rows [D][2][L][N], NTT form.
    void make_ks_key(const std::vector<std::vector<u64>>& target, unsigned bits, u32 D, const Seed& kseed, u64* out) {
        const u32 N = cp.N, L = cp.L;
        auto fac = digit_factors(bits, D);
        for (u32 d = 0; d < D; ++d) {
            auto k1 = uniform_rns(derive_seed(kseed, 11, d));
            Rng nr(kseed, (u64(13) << 32) | d);
            std::vector<i64> e(N);
            for (auto& x : e) x = nr.noise();
            for (u32 i = 0; i < L; ++i) {
                const u64 q = cp.q[i];
                auto prod = rq[i].mul(k1[i], s_rns[i]);
                auto ei = reduce_signed(e, i);
                std::vector<u64> body(N);
                for (u32 n = 0; n < N; ++n) {
                    u64 v = prod[n] ? q - prod[n] : 0;  // -k1 s
                    v = (v + ei[n]) % q;
                    v = (v + mulmod64(target[i][n], fac[d][i], q)) % q;
                    body[n] = v;
                }
                std::vector<u64> c1 = k1[i];
                rq[i].fwd(body.data());
                rq[i].fwd(c1.data());
                std::memcpy(out + (((size_t)d * 2 + 0) * L + i) * N, body.data(), N * 8);
                std::memcpy(out + (((size_t)d * 2 + 1) * L + i) * N, c1.data(), N * 8);
            }
        }
    }

    void keygen(u32 galois_levels) {
        const u32 N = cp.N, L = cp.L;
        Rng sk(seed, 1);
        s.resize(N);
        for (auto& x : s) x = (int8_t)sk.ternary();
        std::vector<i64> si(s.begin(), s.end());
        s_rns.resize(L);
        for (u32 i = 0; i < L; ++i) s_rns[i] = reduce_signed(si, i);
        std::vector<std::vector<u64>> s_sq(L);
        for (u32 i = 0; i < L; ++i) s_sq[i] = rq[i].mul(s_rns[i], s_rns[i]);
        relin.assign((size_t)cp.Dr * 2 * L * N, 0);
        make_ks_key(s_sq, cp.relin_bits, cp.Dr, derive_seed(seed, 2, 0), relin.data());
        levels = galois_levels;
        const size_t per = (size_t)cp.Dg * 2 * L * N;
        galois.assign(per * galois_levels, 0);
        for (u32 a = 0; a < galois_levels; ++a) {
            const u64 g = N / (u64(1) << a) + 1;
            std::vector<std::vector<u64>> sg(L, std::vector<u64>(N));
            for (u32 i = 0; i < L; ++i)
                for (u32 n = 0; n < N; ++n) {  // automorphism (ring.cpp:315-331)
                    const u64 e = ((u64)n * g) % (2 * (u64)N);
                    const u64 v = s_rns[i][n];
                    if (e < N) sg[i][e] = v; else sg[i][e - N] = v ? cp.q[i] - v : 0;
                }
            make_ks_key(sg, cp.galois_bits, cp.Dg, derive_seed(seed, 3, g), galois.data() + a * per);
        }
    }

    /// encrypt (bfv.cpp:521-549) with explicit randomness index.
    void encrypt(const u64* m, u64 index, u64* out) const {
        const u32 N = cp.N, L = cp.L;
        auto c1 = uniform_rns(derive_seed(seed, 5, index));
        Rng nr(derive_seed(seed, 6, index), 0);
        std::vector<i64> e(N);
        for (auto& x : e) x = nr.noise();
        for (u32 i = 0; i < L; ++i) {
            const u64 q = cp.q[i];
            auto prod = rq[i].mul(c1[i], s_rns[i]);
            auto ei = reduce_signed(e, i);
            for (u32 n = 0; n < N; ++n) {
                u64 v = prod[n] ? q - prod[n] : 0;
                v = (v + ei[n]) % q;
                v = (v + mulmod64(m[n] % q, delta[i], q)) % q;
                out[(size_t)i * N + n] = v;
            }
            std::memcpy(out + ((size_t)L + i) * N, c1[i].data(), N * 8);
        }
    }

    /// decrypt (bfv.cpp:551-595): round(t x / q) mod t of x = <ct, (1, s, s^2)>.
    void decrypt(const u64* ct, u32 comps, u64* out) const {
        const u32 N = cp.N, L = cp.L;
        std::vector<std::vector<u64>> v(L), sp = s_rns;
        for (u32 i = 0; i < L; ++i) v[i].assign(ct + (size_t)i * N, ct + (size_t)(i + 1) * N);
        for (u32 k = 1; k < comps; ++k) {
            for (u32 i = 0; i < L; ++i) {
                std::vector<u64> c(ct + ((size_t)k * L + i) * N, ct + ((size_t)k * L + i + 1) * N);
                auto p = rq[i].mul(c, sp[i]);
                for (u32 n = 0; n < N; ++n) v[i][n] = (v[i][n] + p[n]) % cp.q[i];
            }
            if (k + 1 < comps)
                for (u32 i = 0; i < L; ++i) sp[i] = rq[i].mul(sp[i], s_rns[i]);
        }
        std::vector<Big> qov(L);
        std::vector<u64> mu(L);
        for (u32 i = 0; i < L; ++i) {
            qov[i] = cp.Q.div_u64(cp.q[i]);
            mu[i] = invmod64(qov[i].mod_u64(cp.q[i]), cp.q[i]);
        }
        const Big q2 = cp.Q.mul_u64(2);
        for (u32 n = 0; n < N; ++n) {
            Big x;
            for (u32 i = 0; i < L; ++i) x = x + qov[i].mul_u64(mulmod64(v[i][n], mu[i], cp.q[i]));
            Big qq, rr;
            Big::divmod(x, cp.Q, qq, rr);  // rr = x mod q
            Big num = rr.mul_u64(2 * cp.t) + cp.Q;
            Big::divmod(num, q2, qq, rr);
            out[n] = qq.mod_u64(cp.t);
        }
    }
};

}  // namespace
}  // namespace cwgpu

using namespace cwgpu;

struct cwg_client {
    Client c;
};

template <class F>
static int cguard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        c_err = e.what();
        return -1;
    }
}

extern "C" {

const char* cwg_client_last_error(void) { return c_err.c_str(); }

cwg_client* cwg_client_create(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_bits,
                              uint32_t galois_bits, uint64_t seed, uint32_t galois_levels) {
    cwg_client* h = nullptr;
    cguard([&] {
        auto p = std::make_unique<cwg_client>();
        Client& c = p->c;
        c.cp = make_chain(N, t, std::vector<u64>(q, q + L), relin_bits, galois_bits);
        for (u32 i = 0; i < L; ++i) {
            Ring r;
            r.q = q[i];
            r.N = N;
            r.logN = c.cp.logN;
            r.t = make_ntt_tables(N, q[i], 64);
            r.ninv_s = (u64)(((u128)r.t.ninv << 64) / q[i]);
            c.rq.push_back(std::move(r));
        }
        Big dq = c.cp.Q.div_u64(t);
        for (u32 i = 0; i < L; ++i) c.delta.push_back(dq.mod_u64(q[i]));
        c.seed = Seed::from_u64(seed);
        c.keygen(galois_levels);
        h = p.release();
    });
    return h;
}

void cwg_client_destroy(cwg_client* h) { delete h; }

uint32_t cwg_client_digits(const cwg_client* h, int galois) { return galois ? h->c.cp.Dg : h->c.cp.Dr; }

int cwg_client_export_keys(const cwg_client* h, uint64_t* relin, uint64_t* galois) {
    return cguard([&] {
        std::memcpy(relin, h->c.relin.data(), h->c.relin.size() * 8);
        if (galois && !h->c.galois.empty()) std::memcpy(galois, h->c.galois.data(), h->c.galois.size() * 8);
    });
}

int cwg_client_encrypt(const cwg_client* h, const uint64_t* plain, uint64_t index, uint64_t* out) {
    return cguard([&] {
        for (u32 n = 0; n < h->c.cp.N; ++n)
            if (plain[n] >= h->c.cp.t) throw std::invalid_argument("plaintext not in R_t");
        h->c.encrypt(plain, index, out);
    });
}

int cwg_client_pack_query(const cwg_client* h, const uint8_t* bits, uint32_t m, uint32_t c, uint64_t first_index,
                          uint64_t* out) {
    return cguard([&] {
        const Client& cl = h->c;
        const u32 N = cl.cp.N;
        if ((u64(1) << c) > N) throw std::invalid_argument("compression factor exceeds log2(N)");
        const u64 chunk = u64(1) << c;
        const u64 scale = invmod64(powmod64(2, c, cl.cp.t), cl.cp.t);
        const u64 hq = (m + chunk - 1) / chunk;
        std::vector<u64> coeffs(N);
        for (u64 i = 0; i < hq; ++i) {
            std::fill(coeffs.begin(), coeffs.end(), 0);
            for (u64 j = 0; j < chunk; ++j) {
                const u64 idx = i * chunk + j;
                if (idx < m && bits[idx]) coeffs[j] = scale;
            }
            cl.encrypt(coeffs.data(), first_index + i, out + i * 2 * (size_t)cl.cp.L * N);
        }
    });
}

int cwg_client_decrypt(const cwg_client* h, const uint64_t* ct, uint32_t comps, uint64_t* out) {
    return cguard([&] { h->c.decrypt(ct, comps, out); });
}

int cwg_client_export_secret(const cwg_client* h, int8_t* s, uint64_t* seed_words) {
    return cguard([&] {
        std::memcpy(s, h->c.s.data(), h->c.s.size());
        for (int i = 0; i < 4; ++i) seed_words[i] = h->c.seed.w[i];
    });
}

}  // extern "C"

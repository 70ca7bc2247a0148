// extern "C" harness over the UNMODIFIED reference library (test oracle only).
//
// TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load this library.  It is never on the
// product path.
//
// Every entry point drives the reference's own public API (cwpir::BfvBackend,
// expand_query, product_tree, weighted_sum, finalize, ...) on raw little-endian
// u64 arrays so Python tests and the CPU baseline can call it through ctypes.
//
// Array layouts (shared with include/cwgpu.h):
//   ciphertext      [comps][L][N]      coefficient form, canonical residues
//   key-switch key  [D][2][L][N]       rows[d][k][i] in the reference NTT form (bfv.cpp:394-402)
//   galois keys     [c][Dg][2][L][N]   exponent g_a = N/2^a + 1, a = 0..c-1
//   query           [h][2][L][N]
//   database        [n][s][N]          plaintext coefficients < t
//   positions       [n][k]             ascending codeword positions
//   response        [s][2][L][N]
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cwpir/bfv.hpp"
#include "cwpir/cw_code.hpp"
#include "cwpir/db_file.hpp"
#include "cwpir/eq_circuits.hpp"
#include "cwpir/expansion.hpp"
#include "cwpir/parallel.hpp"
#include "cwpir/pir.hpp"

using namespace cwpir;

namespace {

thread_local std::string g_err;
thread_local bool g_partial = false;

struct RefBackend {
    HeParams hp;
    std::unique_ptr<BfvBackend> be;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

RnsPoly read_rns(const BfvBackend& be, const std::uint64_t* src) {
    const std::size_t N = be.params()->degree, L = be.chain_length();
    RnsPoly out;
    for (std::size_t i = 0; i < L; ++i) {
        out.push_back(RingElement::from_coeffs(be.chain_context(i),
                                               std::vector<u64>(src + i * N, src + (i + 1) * N)));
    }
    return out;
}

void write_rns(const BfvBackend& be, const RnsPoly& p, std::uint64_t* dst) {
    const std::size_t N = be.params()->degree;
    for (std::size_t i = 0; i < p.size(); ++i) std::memcpy(dst + i * N, p[i].coeffs().data(), N * 8);
}

CipherValue read_ct(const BfvBackend& be, const std::uint64_t* src, unsigned comps) {
    const std::size_t N = be.params()->degree, L = be.chain_length();
    CipherValue v;
    v.kind = BackendKind::bfv;
    v.params = be.params();
    for (unsigned k = 0; k < comps; ++k) v.comps.push_back(read_rns(be, src + k * L * N));
    return v;
}

void write_ct(const BfvBackend& be, const CipherValue& v, std::uint64_t* dst) {
    const std::size_t N = be.params()->degree, L = be.chain_length();
    for (std::size_t k = 0; k < v.comps.size(); ++k) write_rns(be, v.comps[k], dst + k * L * N);
}

HeParams make_params(std::uint32_t N, std::uint64_t t, std::uint32_t L, const std::uint64_t* primes,
                     std::uint32_t relin_bits, std::uint32_t galois_bits) {
    HeParams hp;
    hp.name = "custom";
    hp.degree = N;
    hp.plain_modulus = t;
    hp.coeff_primes.assign(primes, primes + L);
    for (std::uint32_t i = 0; i < L; ++i) {
        unsigned b = 0;
        while (b < 64 && (primes[i] >> b)) ++b;
        hp.declared_coeff_bits.push_back(b);
    }
    hp.relin_digit_bits = relin_bits;
    hp.galois_digit_bits = galois_bits;
    hp.depth_cap = 8;
    return hp;
}

void read_ks_key(const BfvBackend& be, unsigned digit_bits, unsigned digits, const std::uint64_t* src,
                 KeySwitchKey& key) {
    const std::size_t N = be.params()->degree, L = be.chain_length();
    key.digit_bits = digit_bits;
    key.rows.clear();
    for (unsigned d = 0; d < digits; ++d) {
        std::array<RnsPoly, 2> row;
        for (int k = 0; k < 2; ++k) row[k] = read_rns(be, src + (std::size_t(d) * 2 + k) * L * N);
        key.rows.push_back(std::move(row));
    }
}

unsigned digit_count(const HeParams& hp, unsigned digit_bits) {
    if (digit_bits == 0) return static_cast<unsigned>(hp.coeff_primes.size());
    BigUint q(1);
    for (u64 p : hp.coeff_primes) q.mul_u64(p);
    return (q.bit_length() + digit_bits - 1) / digit_bits;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

std::uint64_t ref_worker_threads(void) { return worker_threads(); }

int ref_find_ntt_primes_below(std::uint64_t hint, std::uint64_t step, std::uint32_t count,
                              const std::uint64_t* excl, std::uint32_t n_excl, std::uint64_t* out) {
    return guarded([&] {
        std::vector<u64> ex(excl, excl + n_excl);
        auto v = find_ntt_primes_below(hint, step, count, ex);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

std::uint64_t ref_find_ntt_prime_below(std::uint64_t hint, std::uint64_t step) {
    try {
        return find_ntt_prime_below(hint, step);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

std::uint64_t ref_primitive_root(std::uint64_t p) { return primitive_root(p); }

/// bfv_custom_params(N, t, L, bits, depth) chain (bfv.cpp:410-422).
int ref_custom_chain(std::uint32_t N, std::uint64_t t, std::uint32_t L, std::uint32_t bits,
                     std::uint64_t* out) {
    return guarded([&] {
        HeParams hp = bfv_custom_params(N, t, L, bits, 3);
        std::memcpy(out, hp.coeff_primes.data(), L * 8);
    });
}

/// RingContext::ntt_forward / ntt_inverse on `count` polys of one prime (ring.cpp:78-144).
int ref_ntt(std::uint32_t N, std::uint64_t q, std::uint64_t* a, std::uint32_t count, int inverse) {
    return guarded([&] {
        auto ctx = RingContext::create(N, q);
        for (std::uint32_t c = 0; c < count; ++c) {
            std::span<u64> s(a + std::size_t(c) * N, N);
            if (inverse) ctx->ntt_inverse(s); else ctx->ntt_forward(s);
        }
    });
}

/// Client-side backend: keygen from Seed256::from_u64(seed) with `galois_levels` Galois keys
/// (bfv.cpp:465-488).
void* ref_backend_new(std::uint32_t N, std::uint64_t t, std::uint32_t L, const std::uint64_t* primes,
                      std::uint32_t relin_bits, std::uint32_t galois_bits, std::uint64_t seed,
                      std::uint32_t galois_levels) {
    try {
        auto rb = std::make_unique<RefBackend>();
        rb->hp = make_params(N, t, L, primes, relin_bits, galois_bits);
        rb->be = std::make_unique<BfvBackend>(rb->hp, Seed256::from_u64(seed), galois_levels);
        return rb.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

/// Server-side backend from caller-supplied evaluation keys (bfv.hpp:73).
void* ref_backend_from_keys(std::uint32_t N, std::uint64_t t, std::uint32_t L,
                            const std::uint64_t* primes, std::uint32_t relin_bits,
                            std::uint32_t galois_bits, const std::uint64_t* relin,
                            std::uint32_t n_galois, const std::uint64_t* galois_g,
                            const std::uint64_t* galois) {
    try {
        auto rb = std::make_unique<RefBackend>();
        rb->hp = make_params(N, t, L, primes, relin_bits, galois_bits);
        // a throwaway backend gives us RingContexts for parsing
        BfvBackend parse(rb->hp, EvalKeySet{});
        EvalKeySet keys;
        const unsigned dr = digit_count(rb->hp, relin_bits), dg = digit_count(rb->hp, galois_bits);
        read_ks_key(parse, relin_bits, dr, relin, keys.relin);
        const std::size_t per = std::size_t(dg) * 2 * L * N;
        for (std::uint32_t a = 0; a < n_galois; ++a) {
            read_ks_key(parse, galois_bits, dg, galois + a * per, keys.galois[galois_g[a]]);
        }
        rb->be = std::make_unique<BfvBackend>(rb->hp, std::move(keys));
        return rb.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_backend_free(void* h) { delete static_cast<RefBackend*>(h); }

std::uint32_t ref_digits(void* h, int galois) {
    auto* rb = static_cast<RefBackend*>(h);
    return digit_count(rb->hp, galois ? rb->hp.galois_digit_bits : rb->hp.relin_digit_bits);
}

/// Exports relin rows [Dr][2][L][N] and Galois keys for a = 0..n_galois-1, [Dg][2][L][N] each.
int ref_export_keys(void* h, std::uint64_t* relin, std::uint32_t n_galois, std::uint64_t* galois) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const BfvBackend& be = *rb->be;
        const std::size_t N = rb->hp.degree, L = rb->hp.coeff_primes.size();
        const auto& keys = be.eval_keys();
        auto dump = [&](const KeySwitchKey& k, std::uint64_t* dst) {
            for (std::size_t d = 0; d < k.rows.size(); ++d)
                for (int c = 0; c < 2; ++c) write_rns(be, k.rows[d][c], dst + (d * 2 + c) * L * N);
        };
        dump(keys.relin, relin);
        const std::size_t per = std::size_t(ref_digits(h, 1)) * 2 * L * N;
        for (std::uint32_t a = 0; a < n_galois; ++a) {
            const u64 g = N / (u64(1) << a) + 1;
            auto it = keys.galois.find(g);
            if (it == keys.galois.end()) throw he_error("missing Galois key for requested exponent");
            dump(it->second, galois + a * per);
        }
    });
}

/// pack_query_bits (expansion.cpp:17-38): h ciphertexts [h][2][L][N].
int ref_pack_query(void* h, const std::uint8_t* bits, std::uint32_t m, std::uint32_t c,
                   std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        PackedQuery pq = pack_query_bits(*rb->be, std::span<const std::uint8_t>(bits, m), c);
        const std::size_t per = 2 * rb->hp.coeff_primes.size() * rb->hp.degree;
        for (std::size_t i = 0; i < pq.cts.size(); ++i) write_ct(*rb->be, pq.cts[i], out + i * per);
    });
}

/// encrypt (bfv.cpp:521-549) of a plaintext with N coefficients < t.
int ref_encrypt(void* h, const std::uint64_t* plain, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        std::vector<u64> c(plain, plain + rb->hp.degree);
        write_ct(*rb->be, rb->be->encrypt(RingElement::from_coeffs(rb->be->plain_context(), c)), out);
    });
}

int ref_decrypt(void* h, const std::uint64_t* ct, std::uint32_t comps, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        RingElement m = rb->be->decrypt(read_ct(*rb->be, ct, comps));
        std::memcpy(out, m.coeffs().data(), rb->hp.degree * 8);
    });
}

int ref_noise_budget(void* h, const std::uint64_t* ct, std::uint32_t comps) {
    auto* rb = static_cast<RefBackend*>(h);
    try {
        return rb->be->noise_budget(read_ct(*rb->be, ct, comps));
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

/// BfvBackend::substitute (bfv.cpp:694-712).
int ref_substitute(void* h, const std::uint64_t* ct, std::uint64_t g, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        write_ct(*rb->be, rb->be->substitute(read_ct(*rb->be, ct, 2), g), out);
    });
}

/// expand_query (expansion.cpp:67-83): m entries [m][2][L][N].
int ref_expand(void* h, const std::uint64_t* query, std::uint32_t nq, std::uint32_t c,
               std::uint32_t m, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const std::size_t per = 2 * rb->hp.coeff_primes.size() * rb->hp.degree;
        PackedQuery pq;
        pq.compression = c;
        pq.code_length = m;
        for (std::uint32_t i = 0; i < nq; ++i) pq.cts.push_back(read_ct(*rb->be, query + i * per, 2));
        auto ex = expand_query(*rb->be, pq);
        for (std::size_t j = 0; j < ex.size(); ++j) write_ct(*rb->be, ex[j], out + j * per);
    });
}

/// mul_lazy = mul_lazy_prepared(prepare_cipher(a), prepare_cipher(b)) (bfv.cpp:748-857).
int ref_mul_lazy(void* h, const std::uint64_t* a, std::uint32_t ca, const std::uint64_t* b,
                 std::uint32_t cb, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        write_ct(*rb->be, rb->be->mul_lazy(read_ct(*rb->be, a, ca), read_ct(*rb->be, b, cb)), out);
    });
}

/// mul = relinearize(mul_lazy) (bfv.cpp:877-879).
int ref_mul(void* h, const std::uint64_t* a, const std::uint64_t* b, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        write_ct(*rb->be, rb->be->mul(read_ct(*rb->be, a, 2), read_ct(*rb->be, b, 2)), out);
    });
}

/// finalize (bfv.cpp:871-875) of a 3-component ciphertext.
int ref_finalize(void* h, const std::uint64_t* ct3, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        write_ct(*rb->be, rb->be->finalize(read_ct(*rb->be, ct3, 3)), out);
    });
}

/// weighted_sum (bfv.cpp:944-986) of n ciphertexts (comps each) against n plaintexts,
/// plaintexts prepared with prepare_plain (bfv.cpp:933-942).
int ref_weighted_sum(void* h, const std::uint64_t* cts, std::uint32_t comps, std::uint64_t n,
                     const std::uint64_t* plains, std::uint64_t* out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const std::size_t N = rb->hp.degree, L = rb->hp.coeff_primes.size();
        std::vector<CipherValue> v;
        std::vector<BfvBackend::PreparedPlain> p;
        for (std::uint64_t r = 0; r < n; ++r) {
            v.push_back(read_ct(*rb->be, cts + r * comps * L * N, comps));
            std::vector<u64> c(plains + r * N, plains + (r + 1) * N);
            p.push_back(rb->be->prepare_plain(RingElement::from_coeffs(rb->be->plain_context(), c)));
        }
        write_ct(*rb->be, rb->be->weighted_sum(v, p), out);
    });
}

/// Server answer composed from the reference's public calls:
///   expanded = expand_query(be, query)                              (pir.cpp:342)
///   op 0 (folklore): per row, exactly compute_selection_vector's BFV branch
///        (pir.cpp:287-302): prepare_cipher once per entry, mul_lazy_prepared of leaf
///        pairs (finalize unless k == 2), odd leftover carried, product_tree(lazy_root=true);
///        k == 1 takes the expanded entry itself (the generic path, pir.cpp:305-310).
///   op 1 (arithmetic, config 5): k' = sum of the selected entries (be.add),
///        f_0 = k', f_i = add_plain(k', t - i), product_tree(lazy_root=false),
///        plain_mul((k!)^-1) (eq_circuits.cpp:105-127 specialised to a public codeword).
///   inner product: prepare_plain + weighted_sum per chunk (pir.cpp:319-326), evaluated
///        over row tiles of `tile_rows` and summed with be.add (bit-identical to the
///        untiled weighted_sum: INTT and mod-q addition are linear), then finalize
///        (pir.cpp:345).
/// stage_ms (optional, 6 doubles): expand, select (incl. prepare_cipher), inner (weighted_sum + add),
/// finalize, prepare_cipher, prepare_plain wall times.  prepare_plain (the database's NTT form) is
/// timed apart from the inner product: the reference computes it offline (PirDatabase::prepare_for,
/// pir.cpp:255-264), so a server answer does not pay it.
int ref_answer(void* h, const std::uint64_t* query, std::uint32_t nq, std::uint32_t c,
               std::uint32_t m, std::uint64_t n, std::uint32_t k, const std::uint32_t* positions,
               std::uint32_t s, const std::uint64_t* db, std::uint32_t op, std::uint64_t tile_rows,
               std::uint64_t* out, double* stage_ms) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const BfvBackend& be = *rb->be;
        const std::size_t N = rb->hp.degree, L = rb->hp.coeff_primes.size();
        const u64 t = rb->hp.plain_modulus;
        const std::size_t per = 2 * L * N;
        if (tile_rows == 0) tile_rows = n;
        auto t0 = std::chrono::steady_clock::now();
        PackedQuery pq;
        pq.compression = c;
        pq.code_length = m;
        for (std::uint32_t i = 0; i < nq; ++i) pq.cts.push_back(read_ct(be, query + i * per, 2));
        auto expanded = expand_query(be, pq);
        if (expanded.size() != m) throw std::invalid_argument("expanded query length must equal the code length");
        double t_expand = ms_since(t0), t_select = 0, t_inner = 0, t_plain = 0;

        std::vector<BfvBackend::PreparedCipher> prepared;
        auto t1 = std::chrono::steady_clock::now();
        if (op == 0 && k >= 2) {
            prepared.resize(expanded.size());
            parallel_for(expanded.size(), [&](std::size_t j) { prepared[j] = be.prepare_cipher(expanded[j]); });
        }
        const double t_prepare = ms_since(t1);
        t_select += t_prepare;

        u64 kfact_inv = 0;
        if (op == 1) {
            u64 f = 1;
            for (unsigned i = 2; i <= k; ++i) f = mul_mod(f, i % t, t);
            kfact_inv = inv_mod(f, t);
        }
        std::vector<CipherValue> acc(s);
        std::vector<bool> have(s, false);
        for (std::uint64_t r0 = 0; r0 < n; r0 += tile_rows) {
            const std::uint64_t r1 = std::min<std::uint64_t>(n, r0 + tile_rows);
            auto ts = std::chrono::steady_clock::now();
            std::vector<CipherValue> sel(r1 - r0);
            parallel_for(r1 - r0, [&](std::size_t ii) {
                const std::uint64_t i = r0 + ii;
                std::vector<unsigned> pos(positions + i * k, positions + (i + 1) * k);
                if (op == 0) {
                    if (k == 1) {
                        sel[ii] = expanded[pos[0]];
                        return;
                    }
                    std::vector<CipherValue> nodes;
                    for (std::size_t p = 0; p + 1 < pos.size(); p += 2) {
                        const bool root = pos.size() == 2;
                        CipherValue prod = be.mul_lazy_prepared(prepared[pos[p]], prepared[pos[p + 1]]);
                        if (!root) prod = be.finalize(prod);
                        nodes.push_back(std::move(prod));
                    }
                    if (pos.size() % 2) nodes.push_back(expanded[pos.back()]);
                    sel[ii] = product_tree(be, std::move(nodes), /*lazy_root=*/true);
                } else {
                    CipherValue inner = expanded[pos[0]];
                    for (std::size_t p = 1; p < pos.size(); ++p) inner = be.add(inner, expanded[pos[p]]);
                    std::vector<CipherValue> factors;
                    for (unsigned f = 0; f < k; ++f) {
                        factors.push_back(f == 0 ? inner
                                                 : be.add_plain(inner, RingElement::constant(be.plain_context(), t - (f % t))));
                    }
                    CipherValue prod = product_tree(be, std::move(factors));
                    sel[ii] = be.plain_mul(RingElement::constant(be.plain_context(), kfact_inv), prod);
                }
            });
            t_select += ms_since(ts);
            auto tp = std::chrono::steady_clock::now();
            std::vector<std::vector<BfvBackend::PreparedPlain>> plains(
                s, std::vector<BfvBackend::PreparedPlain>(r1 - r0));
            parallel_for(r1 - r0, [&](std::size_t ii) {
                const std::uint64_t i = r0 + ii;
                for (std::uint32_t j = 0; j < s; ++j) {
                    const std::uint64_t* src = db + (i * s + j) * N;
                    plains[j][ii] = be.prepare_plain(RingElement::from_coeffs(
                        be.plain_context(), std::vector<u64>(src, src + N)));
                }
            });
            t_plain += ms_since(tp);
            auto ti = std::chrono::steady_clock::now();
            std::vector<CipherValue> part(s);
            parallel_for(s, [&](std::size_t j) { part[j] = be.weighted_sum(sel, plains[j]); });
            for (std::uint32_t j = 0; j < s; ++j) {
                acc[j] = have[j] ? be.add(acc[j], part[j]) : std::move(part[j]);
                have[j] = true;
            }
            t_inner += ms_since(ti);
        }
        auto tf = std::chrono::steady_clock::now();
        for (std::uint32_t j = 0; j < s; ++j) {
            if (g_partial) {  // un-finalized inner product, [s][3][L][N]
                write_ct(be, acc[j], out + j * 3 * L * N);
                continue;
            }
            CipherValue r = be.finalize(acc[j]);
            write_ct(be, r, out + j * per);
        }
        if (stage_ms) {
            stage_ms[0] = t_expand;
            stage_ms[1] = t_select;
            stage_ms[2] = t_inner;
            stage_ms[3] = ms_since(tf);
            stage_ms[4] = t_prepare;
            stage_ms[5] = t_plain;
        }
    });
}

/// compute_selection_vector's BFV branch (pir.cpp:287-302) for caller-given codewords
/// (config 2 draws them at random, with duplicates, so PirDatabase::setup cannot be used).
/// sel: [n][3][L][N] (2-component rows zero padded), comps[n].
/// stage_ms (optional, 3 doubles): expand_query, prepare_cipher, per-row selection wall times.
int ref_select(void* h, const std::uint64_t* query, std::uint32_t nq, std::uint32_t c, std::uint32_t m,
               std::uint64_t n, std::uint32_t k, const std::uint32_t* positions, std::uint64_t* sel,
               std::uint32_t* comps, double* stage_ms) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const BfvBackend& be = *rb->be;
        const std::size_t N = rb->hp.degree, L = rb->hp.coeff_primes.size();
        const std::size_t per = 2 * L * N;
        PackedQuery pq;
        pq.compression = c;
        pq.code_length = m;
        for (std::uint32_t i = 0; i < nq; ++i) pq.cts.push_back(read_ct(be, query + i * per, 2));
        auto t0 = std::chrono::steady_clock::now();
        auto expanded = expand_query(be, pq);
        const double t_expand = ms_since(t0);
        auto t1 = std::chrono::steady_clock::now();
        std::vector<BfvBackend::PreparedCipher> prepared;
        if (k >= 2) {
            prepared.resize(expanded.size());
            parallel_for(expanded.size(), [&](std::size_t j) { prepared[j] = be.prepare_cipher(expanded[j]); });
        }
        const double t_prepare = ms_since(t1);
        auto t2 = std::chrono::steady_clock::now();
        parallel_for(n, [&](std::size_t i) {
            std::vector<unsigned> pos(positions + i * k, positions + (i + 1) * k);
            CipherValue out;
            if (k == 1) {
                out = expanded[pos[0]];
            } else {
                std::vector<CipherValue> nodes;
                for (std::size_t p = 0; p + 1 < pos.size(); p += 2) {
                    const bool root = pos.size() == 2;
                    CipherValue prod = be.mul_lazy_prepared(prepared[pos[p]], prepared[pos[p + 1]]);
                    if (!root) prod = be.finalize(prod);
                    nodes.push_back(std::move(prod));
                }
                if (pos.size() % 2) nodes.push_back(expanded[pos.back()]);
                out = product_tree(be, std::move(nodes), /*lazy_root=*/true);
            }
            std::memset(sel + i * 3 * L * N, 0, 3 * L * N * 8);
            write_ct(be, out, sel + i * 3 * L * N);
            comps[i] = static_cast<std::uint32_t>(out.comps.size());
        });
        if (stage_ms) {
            stage_ms[0] = t_expand;
            stage_ms[1] = t_prepare;
            stage_ms[2] = ms_since(t2);
        }
    });
}

/// ref_answer without the final relinearisation: the row shard's inner product
/// (weighted_sum, bfv.cpp:944-986) as [s][3][L][N] (zero padded when 2-component).
/// Summing these over row shards mod q and then finalize = the full answer (row sharding).
int ref_answer_partial(void* h, const std::uint64_t* query, std::uint32_t nq, std::uint32_t c,
                       std::uint32_t m, std::uint64_t n, std::uint32_t k, const std::uint32_t* positions,
                       std::uint32_t s, const std::uint64_t* db, std::uint32_t op, std::uint64_t* out) {
    g_partial = true;
    int rc = ref_answer(h, query, nq, c, m, n, k, positions, s, db, op, 0, out, nullptr);
    g_partial = false;
    return rc;
}

/// The reference's own process_query (pir.cpp:337-347) on a PirDatabase built by
/// PirDatabase::setup from byte payloads (index mode, rows in perfect_map order).
/// Used to pin ref_answer's composition against the stock entry point.
/// payloads: [n][payload_bytes]; outputs s (returned via *s_out) responses.
int ref_process_query_bytes(void* h, const std::uint64_t* query, std::uint32_t nq, std::uint32_t c,
                            std::uint32_t m, std::uint64_t n, std::uint32_t k,
                            const std::uint8_t* payloads, std::uint64_t payload_bytes,
                            std::uint64_t* out, std::uint32_t* s_out, std::uint64_t* chunk_coeffs,
                            std::uint32_t* positions_out) {
    return guarded([&] {
        auto* rb = static_cast<RefBackend*>(h);
        const BfvBackend& be = *rb->be;
        const std::size_t N = rb->hp.degree, L = rb->hp.coeff_primes.size();
        PirConfig cfg = make_index_config(n, k, c, rb->hp, payload_bytes);
        if (cfg.code_length != m) throw std::invalid_argument("code length mismatch");
        std::vector<PirRow> rows(n);
        for (std::uint64_t i = 0; i < n; ++i)
            rows[i].payload.assign(payloads + i * payload_bytes, payloads + (i + 1) * payload_bytes);
        PirDatabase db = PirDatabase::setup(std::move(rows), cfg);
        const std::size_t per = 2 * L * N;
        PackedQuery pq;
        pq.compression = c;
        pq.code_length = m;
        for (std::uint32_t i = 0; i < nq; ++i) pq.cts.push_back(read_ct(be, query + i * per, 2));
        auto resp = process_query(be, pq, db);
        *s_out = static_cast<std::uint32_t>(resp.size());
        for (std::size_t j = 0; j < resp.size(); ++j) write_ct(be, resp[j], out + j * per);
        const std::size_t s = db.chunks_per_row();
        for (std::uint64_t i = 0; i < n; ++i) {
            for (std::size_t j = 0; j < s; ++j)
                std::memcpy(chunk_coeffs + (i * s + j) * N, db.chunk(i, j).coeffs().data(), N * 8);
            auto pos = db.codeword(i).positions();
            for (unsigned p = 0; p < k; ++p) positions_out[i * k + p] = pos[p];
        }
    });
}

/// The reference's own database-file writer (db_file.cpp:13-31, write_db_file): mode 0 index,
/// 1 keyword (keys: n x key_len bytes); payloads n x payload_bytes.
int ref_write_db_file(const char* path, int mode, std::uint32_t keyword_bits, std::uint64_t n, std::uint32_t key_len,
                      const std::uint8_t* keys, std::uint32_t payload_bytes, const std::uint8_t* payloads) {
    return guarded([&] {
        DbFileData db;
        db.header.mode = mode ? PirMode::keyword : PirMode::index;
        db.header.keyword_bits = keyword_bits;
        db.header.row_count = n;
        db.header.payload_bytes = payload_bytes;
        db.rows.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            if (mode) db.rows[i].key.assign(keys + i * key_len, keys + (i + 1) * key_len);
            db.rows[i].payload.assign(payloads + i * payload_bytes, payloads + (i + 1) * payload_bytes);
        }
        write_db_file(path, db);
    });
}

/// perfect_map (cw_code.cpp:80-102): ascending positions of the x-th weight-k codeword.
int ref_perfect_map(std::uint64_t x, std::uint32_t m, std::uint32_t k, std::uint32_t* out) {
    return guarded([&] {
        auto pos = perfect_map(x, CodeSpec(m, k)).positions();
        for (unsigned i = 0; i < k; ++i) out[i] = pos[i];
    });
}

std::uint32_t ref_min_code_length(std::uint64_t n, std::uint32_t k) { return min_code_length(n, k); }

}  // extern "C"

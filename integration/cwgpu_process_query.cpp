// Drop-in replacement for the reference's server answer, for the reference's own build.
//   std::vector<CipherValue> cwpir::process_query(const HeBackend&, const PackedQuery&,
//                                                 const PirDatabase&)   (pir.hpp:114-117)
// Same signature in namespace cwgpu, implemented over include/cwgpu.h (libcwgpu.so).
// Compiled and checked against the reference by oracle/build_ref.sh + tests/test_dropin.py.
#include <memory>
#include <mutex>
#include <stdexcept>
#include "cwpir/pir.hpp"
#include "cwgpu.h"   // this repo's include/

namespace cwgpu {

namespace {
[[noreturn]] void rethrow(int rc) {          // same exception types and messages as the reference
    const char* m = cwg_last_error();
    if (rc == CWG_EHE) throw cwpir::he_error(m);
    throw std::invalid_argument(m);
}
void check(int rc) { if (rc != CWG_OK) rethrow(rc); }

struct Resident {                            // device-resident DB per (params, database)
    cwg_ctx* ctx = nullptr;
    const cwpir::PirDatabase* db = nullptr;
    std::uint64_t fp = 0;
    std::mutex mu;
};
Resident& resident() { static Resident r; return r; }
}  // namespace

std::vector<cwpir::CipherValue> process_query(const cwpir::HeBackend& be, const cwpir::PackedQuery& query,
                                              const cwpir::PirDatabase& db) {
    using namespace cwpir;
    const auto* bfv = dynamic_cast<const BfvBackend*>(&be);
    if (!bfv) return cwpir::process_query(be, query, db);   // transparent backend: reference path
    const HeParams& hp = *be.params();
    const std::size_t N = hp.degree, L = hp.coeff_primes.size();
    if (query.code_length != db.config().code_length)
        throw std::invalid_argument("query code length does not match the database");

    Resident& R = resident();
    std::lock_guard<std::mutex> lk(R.mu);
    if (!R.ctx || R.db != &db || R.fp != hp.fingerprint()) {
        if (R.ctx) cwg_destroy(R.ctx);
        R.ctx = cwg_create(N, L, hp.coeff_primes.data(), hp.plain_modulus, hp.relin_digit_bits,
                           hp.galois_digit_bits, /*device=*/0);
        if (!R.ctx) rethrow(CWG_EINVAL);
        const std::size_t n = db.rows(), s = db.chunks_per_row(), k = db.config().hamming_weight;
        std::vector<std::uint32_t> pos(n * k);
        std::vector<std::uint64_t> payload(n * s * N);
        for (std::size_t i = 0; i < n; ++i) {
            auto p = db.codeword(i).positions();
            std::copy(p.begin(), p.end(), pos.begin() + i * k);
            for (std::size_t j = 0; j < s; ++j)
                std::copy(db.chunk(i, j).coeffs().begin(), db.chunk(i, j).coeffs().end(),
                          payload.begin() + (i * s + j) * N);
        }
        check(cwg_load_db(R.ctx, n, 0, n, s, k, db.config().code_length, pos.data(), payload.data()));
        R.db = &db;
        R.fp = hp.fingerprint();
    }
    // evaluation keys (reference layout: rows[d][k][i] in NTT form, bfv.cpp:394-402)
    const EvalKeySet& keys = bfv->eval_keys();
    auto flat = [&](const KeySwitchKey& key, std::vector<std::uint64_t>& out) {
        for (const auto& row : key.rows)
            for (int c = 0; c < 2; ++c)
                for (std::size_t i = 0; i < L; ++i)
                    out.insert(out.end(), row[c][i].coeffs().begin(), row[c][i].coeffs().end());
    };
    std::vector<std::uint64_t> relin, galois, gs;
    flat(keys.relin, relin);
    for (unsigned a = 0; a < query.compression; ++a) {
        const std::uint64_t g = N / (std::uint64_t(1) << a) + 1;
        auto it = keys.galois.find(g);
        if (it == keys.galois.end()) throw he_error("missing Galois key for requested exponent");
        flat(it->second, galois);
        gs.push_back(g);
    }
    std::vector<std::uint64_t> q;
    for (const auto& ct : query.cts)
        for (const auto& comp : ct.comps)
            for (const auto& e : comp) q.insert(q.end(), e.coeffs().begin(), e.coeffs().end());
    const std::size_t s = db.chunks_per_row();
    std::vector<std::uint64_t> out(s * 2 * L * N);
    check(cwg_answer(R.ctx, relin.data(), (uint32_t)gs.size(), gs.data(), galois.data(),
                     (uint32_t)query.cts.size(), query.compression, query.code_length, q.data(),
                     CWG_OP_FOLKLORE, out.data(), nullptr));
    std::vector<CipherValue> resp(s);
    for (std::size_t j = 0; j < s; ++j) {
        resp[j].kind = BackendKind::bfv;
        resp[j].params = be.params();
        resp[j].comps.resize(2);
        for (int c = 0; c < 2; ++c)
            for (std::size_t i = 0; i < L; ++i) {
                const std::uint64_t* src = out.data() + ((j * 2 + c) * L + i) * N;
                resp[j].comps[c].push_back(RingElement::from_coeffs(bfv->chain_context(i),
                                                                    std::vector<std::uint64_t>(src, src + N)));
            }
    }
    return resp;
}

}  // namespace cwgpu

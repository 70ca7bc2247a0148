// Drop-in replacement for the reference's server answer, for the reference's own build.
//   std::vector<CipherValue> cwpir::process_query(const HeBackend&, const PackedQuery&,
//                                                 const PirDatabase&)   (pir.hpp:114-117)
// Same signature in namespace cwgpu, implemented over include/cwgpu.h (libcwgpu.so).
// Compiled and checked against the reference by oracle/build_ref.sh + tests/test_dropin.py.
//
// Devices: every visible GPU by default (rows split across them, cwg_create_multi), or the list
// given to cwgpu::set_devices (a device may repeat).
// Database residency: the NTT-form rows stay on the devices between calls.  The resident copy is
// keyed on the database's CONTENTS -- shape (rows, chunks per row, code length, weight, params
// fingerprint) plus a 64-bit digest of every codeword position and payload coefficient.  The
// digest of the caller's database is recomputed on every call by host threads while the GPUs
// answer from the resident copy; if it differs (a new database, possibly at the same address),
// the rows are reloaded and the answer is recomputed, so a stale copy is never returned.
// Evaluation keys travel with every call, as in the reference server (server.cpp:61-87); the
// library keeps the resident set when the uploaded words are identical (device key cache).
#include <algorithm>
#include <cstring>
#include <future>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
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

struct Shape {
    std::uint64_t fp = 0, rows = 0, chunks = 0, m = 0, k = 0;
    std::vector<int> devices;
    bool operator==(const Shape& o) const {
        return fp == o.fp && rows == o.rows && chunks == o.chunks && m == o.m && k == o.k && devices == o.devices;
    }
};

/// Pinned host staging buffer (cwg_pinned_alloc), grown on demand.
struct Pinned {
    std::uint64_t* p = nullptr;
    std::size_t words = 0;
    std::uint64_t* get(std::size_t n) {
        if (n > words) {
            cwg_pinned_free(p);
            p = static_cast<std::uint64_t*>(cwg_pinned_alloc(n * 8));
            words = p ? n : 0;
            if (!p) throw std::runtime_error(cwg_last_error());
        }
        return p;
    }
    ~Pinned() { cwg_pinned_free(p); }
};

struct Resident {                            // device-resident DB (one per process)
    cwg_ctx* ctx = nullptr;
    Pinned keys, query, out;                 // per-call staging in pinned memory
    Shape shape;
    std::uint64_t digest = 0;
    std::vector<int> devices;                // empty: all visible
    std::mutex mu;
};
Resident& resident() { static Resident r; return r; }

inline std::uint64_t mix64(std::uint64_t x) {  // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/// 64-bit digest of the database contents (codeword positions and payload coefficients of every
/// row, position-sensitive), over host threads.
std::uint64_t db_digest(const cwpir::PirDatabase& db) {
    const std::size_t n = db.rows(), s = db.chunks_per_row();
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::uint64_t> part(T, 0);
    auto work = [&](unsigned t) {
        std::uint64_t acc = 0;
        for (std::size_t i = n * t / T; i < n * (t + 1) / T; ++i) {
            std::uint64_t a0 = i + 1, a1 = 0x9e3779b97f4a7c15ull, a2 = 0, a3 = 0;
            for (auto p : db.codeword(i).positions()) a0 = (a0 + p) * 0xff51afd7ed558ccdull;
            for (std::size_t j = 0; j < s; ++j) {
                const auto& v = db.chunk(i, j).coeffs();
                const std::uint64_t* w = v.data();
                std::size_t x = 0, len = v.size();
                for (; x + 4 <= len; x += 4) {
                    a0 = (a0 + w[x]) * 0xc4ceb9fe1a85ec53ull;
                    a1 = (a1 + w[x + 1]) * 0x9e3779b97f4a7c15ull;
                    a2 = (a2 + w[x + 2]) * 0xbf58476d1ce4e5b9ull;
                    a3 = (a3 + w[x + 3]) * 0x94d049bb133111ebull;
                }
                for (; x < len; ++x) a0 = (a0 + w[x]) * 0xc4ceb9fe1a85ec53ull;
            }
            acc += mix64(mix64(a0 ^ mix64(a1)) ^ mix64(a2 + mix64(a3)) ^ (i * 0x9e3779b97f4a7c15ull));
        }
        part[t] = acc;
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    std::uint64_t d = 0;
    for (auto x : part) d += x;
    return d;
}

void load(Resident& R, const cwpir::HeParams& hp, const cwpir::PirDatabase& db, const Shape& shape) {
    const std::size_t N = hp.degree, L = hp.coeff_primes.size();
    if (!R.ctx || !(R.shape.fp == shape.fp && R.shape.devices == shape.devices)) {
        if (R.ctx) cwg_destroy(R.ctx);
        R.ctx = cwg_create_multi(N, L, hp.coeff_primes.data(), hp.plain_modulus, hp.relin_digit_bits,
                                 hp.galois_digit_bits, shape.devices.data(), (int)shape.devices.size());
        if (!R.ctx) rethrow(CWG_EINVAL);
    }
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
    R.shape = Shape{};  // invalid until the upload succeeded
    check(cwg_load_db(R.ctx, n, 0, n, s, k, db.config().code_length, pos.data(), payload.data()));
    R.shape = shape;
}
}  // namespace

void set_devices(const std::vector<int>& device_ids) {
    Resident& R = resident();
    std::lock_guard<std::mutex> lk(R.mu);
    R.devices = device_ids;
}

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
    Shape shape{hp.fingerprint(), db.rows(), db.chunks_per_row(), db.config().code_length,
                db.config().hamming_weight, R.devices};
    if (shape.devices.empty()) {
        const int nd = cwg_device_count();
        if (nd < 1) throw he_error("cwgpu: no CUDA device");
        for (int d = 0; d < nd; ++d) shape.devices.push_back(d);
    }
    // one device per row at most
    if (shape.devices.size() > db.rows()) shape.devices.resize(db.rows());
    bool fresh = false;
    if (!R.ctx || !(R.shape == shape)) {
        load(R, hp, db, shape);
        R.digest = db_digest(db);
        fresh = true;
    }
    // evaluation keys (reference layout: rows[d][k][i] in NTT form, bfv.cpp:394-402)
    // keys and query flattened straight into pinned staging buffers (asynchronous DMA to the devices)
    const EvalKeySet& keys = bfv->eval_keys();
    std::vector<const KeySwitchKey*> gkeys;
    std::vector<std::uint64_t> gs;
    for (unsigned a = 0; a < query.compression; ++a) {
        const std::uint64_t g = N / (std::uint64_t(1) << a) + 1;
        auto it = keys.galois.find(g);
        if (it == keys.galois.end()) throw he_error("missing Galois key for requested exponent");
        gkeys.push_back(&it->second);
        gs.push_back(g);
    }
    auto words = [&](const KeySwitchKey& key) { return key.rows.size() * 2 * L * N; };
    std::size_t gw = 0;
    for (const auto* k : gkeys) gw += words(*k);
    const std::size_t rw = words(keys.relin);
    std::uint64_t* kbuf = R.keys.get(rw + gw);
    auto flat = [&](const KeySwitchKey& key, std::uint64_t* dst) {
        for (const auto& row : key.rows)
            for (int c = 0; c < 2; ++c)
                for (std::size_t i = 0; i < L; ++i) {
                    std::memcpy(dst, row[c][i].coeffs().data(), N * 8);
                    dst += N;
                }
        return dst;
    };
    flat(keys.relin, kbuf);
    std::uint64_t* gp = kbuf + rw;
    for (const auto* k : gkeys) gp = flat(*k, gp);
    std::uint64_t* q = R.query.get(query.cts.size() * 2 * L * N);
    {
        std::uint64_t* dst = q;
        for (const auto& ct : query.cts)
            for (const auto& comp : ct.comps)
                for (const auto& e : comp) {
                    std::memcpy(dst, e.coeffs().data(), N * 8);
                    dst += N;
                }
    }
    const std::size_t s = db.chunks_per_row();
    std::uint64_t* out = R.out.get(s * 2 * L * N);
    auto answer = [&] {
        check(cwg_answer(R.ctx, kbuf, (uint32_t)gs.size(), gs.data(), kbuf + rw, (uint32_t)query.cts.size(),
                         query.compression, query.code_length, q, CWG_OP_FOLKLORE, out, nullptr));
    };
    if (fresh) {
        answer();
    } else {  // verify the resident rows against the caller's database while the GPUs answer
        auto dig = std::async(std::launch::async, [&] { return db_digest(db); });
        int rc = cwg_answer(R.ctx, kbuf, (uint32_t)gs.size(), gs.data(), kbuf + rw, (uint32_t)query.cts.size(),
                            query.compression, query.code_length, q, CWG_OP_FOLKLORE, out, nullptr);
        const std::uint64_t d = dig.get();
        if (d != R.digest) {  // different contents: reload and answer again
            load(R, hp, db, shape);
            R.digest = d;
            answer();
        } else {
            check(rc);
        }
    }
    std::vector<CipherValue> resp(s);
    for (std::size_t j = 0; j < s; ++j) {
        resp[j].kind = BackendKind::bfv;
        resp[j].params = be.params();
        resp[j].comps.resize(2);
        for (int c = 0; c < 2; ++c)
            for (std::size_t i = 0; i < L; ++i) {
                const std::uint64_t* src = out + ((j * 2 + c) * L + i) * N;
                resp[j].comps[c].push_back(RingElement::from_coeffs(bfv->chain_context(i),
                                                                    std::vector<std::uint64_t>(src, src + N)));
            }
    }
    return resp;
}

}  // namespace cwgpu

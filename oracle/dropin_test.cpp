// Test harness for the drop-in shim integration/cwgpu_process_query.cpp (TEST INFRASTRUCTURE).
// Builds a reference BfvBackend + PirDatabase::setup database, answers the same query with
// the reference's process_query (pir.cpp:337-347) and with cwgpu::process_query, and
// compares the responses word for word, then extract()s the payload.
#include <climits>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "cwpir/pir.hpp"

namespace cwgpu {
std::vector<cwpir::CipherValue> process_query(const cwpir::HeBackend& be, const cwpir::PackedQuery& query,
                                              const cwpir::PirDatabase& db);
}

thread_local std::string d_err;

extern "C" const char* dropin_last_error(void) { return d_err.c_str(); }

/// returns 0 on success; equal = responses identical; extracted = payload recovered.
extern "C" int dropin_check(std::uint64_t seed, std::uint32_t N, std::uint64_t t, std::uint32_t L,
                            std::uint32_t bits, std::uint64_t n, std::uint32_t k, std::uint32_t payload_bytes,
                            std::uint64_t target, int* equal, int* extracted) {
    using namespace cwpir;
    try {
        HeParams hp = bfv_custom_params(N, t, L, bits, 3);
        PirConfig cfg = make_index_config(n, k, UINT_MAX, hp, payload_bytes);
        BfvBackend be(hp, Seed256::from_u64(seed), cfg.compression);
        std::mt19937_64 rng(seed);
        std::vector<PirRow> rows(n);
        std::vector<std::vector<std::uint8_t>> payloads;
        for (auto& r : rows) {
            r.payload.resize(payload_bytes);
            for (auto& b : r.payload) b = static_cast<std::uint8_t>(rng() % 255 + 1);
            payloads.push_back(r.payload);
        }
        PirDatabase db = PirDatabase::setup(std::move(rows), cfg);
        PackedQuery q = build_query_index(be, target, cfg);
        auto want = cwpir::process_query(be, q, db);
        auto got = cwgpu::process_query(be, q, db);
        bool eq = want.size() == got.size();
        for (std::size_t j = 0; eq && j < want.size(); ++j) {
            eq = want[j].comps.size() == got[j].comps.size();
            for (std::size_t c = 0; eq && c < want[j].comps.size(); ++c)
                for (std::size_t i = 0; eq && i < want[j].comps[c].size(); ++i)
                    eq = want[j].comps[c][i].coeffs() == got[j].comps[c][i].coeffs();
        }
        *equal = eq ? 1 : 0;
        auto out = extract(be, got, cfg);
        *extracted = (out && *out == payloads[target]) ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        d_err = e.what();
        return -1;
    }
}

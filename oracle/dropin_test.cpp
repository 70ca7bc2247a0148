// Test harness for the drop-in shim integration/cwgpu_process_query.cpp (TEST INFRASTRUCTURE).
// Builds a reference BfvBackend + PirDatabase::setup database, answers the same query with
// the reference's process_query (pir.cpp:337-347) and with cwgpu::process_query, and
// compares the responses word for word, then extract()s the payload.  Then it REPLACES the
// database in the same variable (same address, same parameters, different rows) and checks
// again, so a stale device copy would be caught.
#include <climits>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "cwpir/pir.hpp"

namespace cwgpu {
std::vector<cwpir::CipherValue> process_query(const cwpir::HeBackend& be, const cwpir::PackedQuery& query,
                                              const cwpir::PirDatabase& db);
void set_devices(const std::vector<int>& device_ids);
}

thread_local std::string d_err;

extern "C" const char* dropin_last_error(void) { return d_err.c_str(); }

namespace {
cwpir::PirDatabase make_db(std::uint64_t seed, std::uint64_t n, std::uint32_t payload_bytes, const cwpir::PirConfig& cfg,
                           std::vector<std::vector<std::uint8_t>>& payloads) {
    std::mt19937_64 rng(seed);
    std::vector<cwpir::PirRow> rows(n);
    payloads.clear();
    for (auto& r : rows) {
        r.payload.resize(payload_bytes);
        for (auto& b : r.payload) b = static_cast<std::uint8_t>(rng() % 255 + 1);
        payloads.push_back(r.payload);
    }
    return cwpir::PirDatabase::setup(std::move(rows), cfg);
}

bool same(const std::vector<cwpir::CipherValue>& want, const std::vector<cwpir::CipherValue>& got) {
    bool eq = want.size() == got.size();
    for (std::size_t j = 0; eq && j < want.size(); ++j) {
        eq = want[j].comps.size() == got[j].comps.size();
        for (std::size_t c = 0; eq && c < want[j].comps.size(); ++c)
            for (std::size_t i = 0; eq && i < want[j].comps[c].size(); ++i)
                eq = want[j].comps[c][i].coeffs() == got[j].comps[c][i].coeffs();
    }
    return eq;
}
}  // namespace

/// returns 0 on success; equal = responses identical (both databases); extracted = payloads
/// recovered (both).  n_dev > 0: cwgpu::set_devices with n_dev copies of device 0 (several
/// contexts on one GPU: the multi-device path of cwg_create_multi); 0: every visible GPU.
extern "C" int dropin_check(std::uint64_t seed, std::uint32_t N, std::uint64_t t, std::uint32_t L,
                            std::uint32_t bits, std::uint64_t n, std::uint32_t k, std::uint32_t payload_bytes,
                            std::uint64_t target, int n_dev, int* equal, int* extracted) {
    using namespace cwpir;
    try {
        cwgpu::set_devices(std::vector<int>(n_dev > 0 ? n_dev : 0, 0));
        HeParams hp = bfv_custom_params(N, t, L, bits, 3);
        PirConfig cfg = make_index_config(n, k, UINT_MAX, hp, payload_bytes);
        BfvBackend be(hp, Seed256::from_u64(seed), cfg.compression);
        std::vector<std::vector<std::uint8_t>> payloads;
        PirDatabase db = make_db(seed, n, payload_bytes, cfg, payloads);
        int eq = 1, ex = 1;
        for (int round = 0; round < 2; ++round) {
            if (round == 1) db = make_db(seed + 1000, n, payload_bytes, cfg, payloads);  // same address
            PackedQuery q = build_query_index(be, target, cfg);
            auto want = cwpir::process_query(be, q, db);
            auto got = cwgpu::process_query(be, q, db);
            eq &= same(want, got) ? 1 : 0;
            auto out = extract(be, got, cfg);
            ex &= (out && *out == payloads[target]) ? 1 : 0;
        }
        *equal = eq;
        *extracted = ex;
        return 0;
    } catch (const std::exception& e) {
        d_err = e.what();
        return -1;
    }
}

// Context, device tables, orchestration and the C ABI (include/cwgpu.h).
//
// Orchestration mirrors process_query (reference pir.cpp:337-347):
//   expand_query (expansion.cpp:67-83)      -> expand()
//   compute_selection_vector (pir.cpp:277)   -> select_tile() per row tile (sel never
//                                               materialised beyond one tile)
//   inner_product / weighted_sum             -> k_mac per tile into NTT-domain accumulators
//   finalize (pir.cpp:345)                   -> finish()
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/cwgpu.h"
#include "kernels.cuh"
#include "ntt_reg.cuh"
#include "params.h"
#include "round.cuh"
#include "mac.cuh"
#include "ntt_mac.cuh"
#include "ks32.cuh"
#include "dbsetup.cuh"
#include "client_gpu.cuh"

namespace cwgpu {

struct he_err : std::runtime_error { using std::runtime_error::runtime_error; };
struct cuda_err : std::runtime_error { using std::runtime_error::runtime_error; };
struct state_err : std::runtime_error { using std::runtime_error::runtime_error; };

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) throw cuda_err(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {  // owns one device allocation (freed on destruction; cudaFree finds the device)
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void ensure(size_t b) {
        if (b <= bytes && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        CK(cudaMalloc(&p, std::max<size_t>(b, 16)));
        bytes = std::max<size_t>(b, 16);
    }
    template <class T>
    T* get(size_t count) {
        ensure(count * sizeof(T));
        return static_cast<T*>(p);
    }
    template <class T>
    T* ptr() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    std::mutex mu;
    ChainParams cp;
    AuxBasis ab;
    u64 aux_n = 0;
    DevTab T{};
    DevBuf tab, tab_self, round_tab;
    u32 JM = 16;  // aux-prime count padded to a multiple of 8 (rounding kernel template)
    std::vector<unsigned char> rtc;   // RoundTcPar<JM, NC> (k_round_tma kernel-parameter block)
    DevBuf rtc_B;                     // k_round_tma B matrix (canonical UMMA K-major layout)
    DevBuf rtc_B2;                    // k_round_tma second-GEMM B matrix (gamma / rho / offset terms)
    DevBuf lift_B;                    // k_lift_tc B matrices (plain, Montgomery)
    DevBuf lift_W2;                   // k_lift_tc rho constants (a_j - W_j) 2^32 mod a_j (plain, Montgomery)
    u32 lift_nc = 0;                  // k_lift_tc GEMM width (0: not available)
    bool lift_tc = true;              // "lift_tc": tensor-core centred lift (0: k_lift on the CUDA cores)
    DevBuf m2c_B;                     // k_mac_to_chain_tc B matrix
    u32 m2c_kw = 0;                   // k_mac_to_chain_tc A words (0: not available)
    DevBuf dec_B;                     // k_decompose_tc B matrix (bytes of q / q_i by column)
    bool dec_ok = false;              // k_decompose_tc available (q below 448 bits)
    bool dec_tc = true;               // "dec_tc": tensor-core digit decomposition (0: k_decompose_t)
    u32 ks_chunk_mb = 3072;           // "ks_chunk_mb": key-switch scratch bound (rows per key-switch launch)
    bool ks_fixed = true;             // "ks_fixed": compile-time-shape key-switch MAC (k_ks_mac32t) for the configured shapes
    bool m2c_tc = true;               // "m2c_tc": tensor-core MAC basis -> chain conversion (0: k_mac_to_chain)
    u32 rtc_nc = 0;                   // k_round_tma GEMM width (0: no instance for this JM / Mm)
    int round_kind = 2;               // 2 tensor-core (k_round_tma), 0 IMAD only (k_round_mac_t); option "round"
    DevBuf prep_s;                    // A-side prepared operands with the INTT output scale folded in
    bool prep_s_ok = false;           // prep_s valid for the current answer
    const u32* prep_s_ptr = nullptr;  // the scaled A operands select_tile uses (prep_s or a batch query's)
    // multi-query answers (cwg_answer_batch): per-query expanded entries, prepared operands, scaled
    // A operands, D buffers and accumulators
    std::vector<std::unique_ptr<DevBuf>> bq_ent, bq_prep, bq_preps, bq_D;
    DevBuf bq_acc;
    DevBuf prep_k, pair_idx;  // arithmetic-operator k' prepared once; product-tree pair indices
    DevBuf cl_seeds, cl_lim, cl_s, cl_s2, cl_a, cl_b, cl_e, cl_bits, cl_out;  // GPU client scratch
    // tuning / test options (cwg_set_option; the defaults are the measured-fastest choices)
    bool prescale = true;             // "prescale": fold the INTT output scale into the A operands
    bool mac_tma = true;              // "mac": 1 TMA-fed payload MAC for s >= 3 (k_mac_tma), 0 k_mac2
    int mac_waves = 2;                // "mac_waves": k_mac_tma grid size in waves of 3 CTAs / SM
    int ntt_np = 1;                   // "ntt_np": polynomials per CTA in the tensor / selection NTT kernels
    // fused selection NTT + payload MAC (k_ntt_mac) for s <= 2 ("fuse_mac" = 0 off); fuse_now: the
    // current answer uses it, so select_tile leaves the MAC-basis selection values in the
    // coefficient domain
    int fuse_mac = 1;
    bool fuse_now = false;
    bool round_g2 = true;   // "round_g2": k_round_tma two-GEMM epilogue (0: corrections on CUDA cores)
    u32 mac_ck = 0;         // "mac_ck": k_ntt_mac row chunks per (component, prime) (0 = auto)
    u32 round_ctas = 4;     // "round_ctas": k_round_tma grid, persistent CTAs per SM
    u32 tile_rows_opt = 0;  // "tile_rows": rows per selection tile (0 = auto)
    bool force_exact = false;  // "force_exact": every rounding / lift decision through the multiword path (tests)
    // key switching through the 30-bit aux primes ("ks32" = 0: the 64-bit NTT path)
    bool ks32 = true;
    bool ks_wide = true;  // "ks_wide": slot-major key-switch MAC (k_ks_mac32s) for D = 7 / 14 / 25
    u32 ks_ci = 2;        // "ks_ci": key columns held per thread in k_ks_mac32s (2 default: 4 CTAs / SM, unrolled rows; 4: wider, 2 CTAs / SM)
    int prep_mode = 1;    // "prep_factors": 1 prepare k' once for the arithmetic factors, 0 each factor
    bool mac_sg = true;   // "mac_sg": s >= 3 payload MAC with 3 or 5 slices per CTA (0: k_mac_tma, one slice)
    bool mac_stages8 = false;  // "mac_stages": 8 ring stages for the 3-slice MAC (default 4)
    bool mac_rows = true;      // "mac_rows": whole-row persistent payload MAC (k_mac_rows) when s is 3, 5 or 15
    u32 mac_item_rows = 256;    // "mac_item_rows": rows per k_mac_rows work item
    DevBuf mac_ctr;            // k_mac_rows work counters (one per launch in flight, rotating)
    u32 mac_ctr_next = 0;
    int n_sms = 148;
    bool ksA_ok = false;               // relinA / galoisA valid for the uploaded keys and aux basis
    KsCrt ksC_r{}, ksC_g{};            // K' = 0: this key type keeps the 64-bit path
    DevBuf relinA, galoisA, ksdig, ksmac;  // keys re-based into the aux primes, digit / MAC scratch
    u32 zs_last = 0;        // MAC-basis plane stride of the last mul_prepared output (J or Mm)
    unsigned next_cluster = 0;  // cluster size of the next launch (launch_named)
    // row-tile pipeline on three streams (k <= 2 folklore): tiles rotate over streams and D buffers
    // so the latency-bound kernels of one tile (NTTs, tensor-core rounding, MAC) co-reside with
    // those of the next (option "streams"; C4: 251 ms vs 272 ms on one stream when introduced;
    // now 3 streams ~1 ms ahead of 2, profiles/r01_experiments.txt)
    int nstreams = 3;
    static constexpr int kMaxStreams = 4;
    cudaStream_t tst[kMaxStreams] = {};
    cudaEvent_t tev[kMaxStreams + 1] = {};
    DevBuf Dmore[kMaxStreams - 1];  // D buffers of tile streams 1.. (stream 0 uses Dbuf)
    DevBuf* dcur = nullptr;
    unsigned long long* d_fb = nullptr;
    // database
    bool db_loaded = false;
    u64 n_total = 0, row_begin = 0, n_local = 0;
    u32 s = 0, k = 0, m = 0;
    DevBuf pos_rows;  // [n_local][k]
    DevBuf pos_cols;  // [k][n_local]
    DevBuf db;        // [n_local][s][Mm][N] u32 NTT form (MAC basis)
    std::vector<u64> h_payload;  // kept to rebuild the NTT form if the basis changes
    // keys
    bool have_keys = false;
    DevBuf relin, galois, key_stage, key_flag;
    std::vector<u64> galois_g;
    bool keys_cached = false;  // the last call's keys equalled the resident set (cwg_timings.keys_cached)
    // scratch
    DevBuf shard_out, shard_all;  // multi-device context: this device's expansion shard, all shards
    DevBuf query, exA, exB, digits, dntt, ks, prep, Dbuf, chain3, node2, acc_lo, partial, X, resp3,
        out2, tmp_idx, lift_tmp;
    u64 launches = 0;
    // per-kernel profiling (CUDA events around every launch; off in timed runs)
    bool profiling = false;
    struct ProfLaunch {
        const char* name;
        cudaEvent_t e0, e1;
        double units;
    };
    struct ProfStat {
        std::string name;
        double ms = 0, units = 0;
        u64 count = 0;
    };
    std::vector<ProfLaunch> prof_pending;
    std::vector<cudaEvent_t> ev_pool;  // recycled profiling events
    std::vector<ProfStat> prof_stats;
    // algorithmic work of the next launch for the profile (0: the grid size, i.e. one unit per
    // CTA -- polynomials for the NTT kernels); see cwg_kernel_units
    double next_units = 0;
    Ctx() = default;
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
    ~Ctx() {  // the DevBuf members free themselves afterwards
        cudaSetDevice(device);
        if (st) cudaStreamSynchronize(st);
        for (cudaStream_t t : tst)
            if (t) cudaStreamSynchronize(t);
        if (d_fb) cudaFree(d_fb);
        for (cudaStream_t t : tst)
            if (t) cudaStreamDestroy(t);
        for (cudaEvent_t e : tev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
        for (auto& p : prof_pending) {
            cudaEventDestroy(p.e0);
            cudaEventDestroy(p.e1);
        }
        if (st) cudaStreamDestroy(st);
    }
};

thread_local std::string g_err;

/// NVTX range for the host-side stages (expand / select / MAC / finish / load / keys): visible in
/// Nsight timelines, free when no tool is attached.
struct Nvtx {
    explicit Nvtx(const char* s) { nvtxRangePushA(s); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// ------------------------------------------------------------------ launches
template <class K, class... A>
static void launch_named(Ctx& c, const char* name, K kern, size_t grid, unsigned block, size_t smem, A... args) {
    if (grid == 0) return;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c.profiling) {  // pooled events: creating them per launch would stall the host and open GPU gaps
        for (cudaEvent_t* e : {&e0, &e1}) {
            if (c.ev_pool.empty()) {
                CK(cudaEventCreate(e));
            } else {
                *e = c.ev_pool.back();
                c.ev_pool.pop_back();
            }
        }
        CK(cudaEventRecord(e0, c.st));
    }
    if (c.next_cluster > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(block);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = c.st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.next_cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        c.next_cluster = 0;
        CK(cudaLaunchKernelEx(&cfg, kern, args...));
    } else {
        kern<<<(unsigned)grid, block, smem, c.st>>>(args...);
    }
    CK(cudaGetLastError());
    ++c.launches;
    if (c.profiling) {
        CK(cudaEventRecord(e1, c.st));
        c.prof_pending.push_back({name, e0, e1, c.next_units > 0 ? c.next_units : (double)grid});
    }
    c.next_units = 0;
}
#define launch(c, kern, ...) launch_named(c, #kern, kern, __VA_ARGS__)

/// Tiled tensor map of a dense u32 array of `rank` dimensions (dims[0] contiguous) with the given box:
/// the operand of cp.async.bulk.tensor in k_mac_rows and k_round_tma.  cuTensorMapEncodeTiled is a
/// host-side encoder; it is fetched through the runtime so the library does not link libcuda.
static CUtensorMap tensor_map(const u32* base, u32 rank, const u64* dims, const u32* box) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
        if (!fn || qr != cudaDriverEntryPointSuccess) throw std::runtime_error("cwgpu: cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeFn>(fn);
    }();
    CUtensorMap tm;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    u64 stride = 4;
    for (u32 i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        stride *= dims[i];
        if (i + 1 < rank) gs[i] = stride;
    }
    const CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, rank, const_cast<u32*>(base), gd, gs, bx, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cwgpu: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return tm;
}
static CUtensorMap tensor_map4(const u32* base, u64 d0, u64 d1, u64 d2, u64 d3, u32 box0, u32 box2) {
    const u64 dims[4] = {d0, d1, d2, d3};
    const u32 box[4] = {box0, 1, box2, 1};
    return tensor_map(base, 4, dims, box);
}


/// launch_named for an explicit (multi-dimensional) launch configuration (cfg.stream is replaced by
/// the context's stream); the same profiling / counting.
template <class K, class... A>
static void launch_grid(Ctx& c, const char* name, K kern, cudaLaunchConfig_t cfg, A... args) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c.profiling) {
        for (cudaEvent_t* e : {&e0, &e1}) {
            if (c.ev_pool.empty()) {
                CK(cudaEventCreate(e));
            } else {
                *e = c.ev_pool.back();
                c.ev_pool.pop_back();
            }
        }
        CK(cudaEventRecord(e0, c.st));
    }
    cfg.stream = c.st;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
    ++c.launches;
    if (c.profiling) {
        CK(cudaEventRecord(e1, c.st));
        c.prof_pending.push_back({name, e0, e1, c.next_units > 0 ? c.next_units : (double)cfg.gridDim.x});
    }
    c.next_units = 0;
}

/// fold finished launch events into per-kernel totals (call after a stream sync)
static void prof_collect(Ctx& c) {
    for (auto& p : c.prof_pending) {
        float f = 0;
        CK(cudaEventElapsedTime(&f, p.e0, p.e1));
        c.ev_pool.push_back(p.e0);
        c.ev_pool.push_back(p.e1);
        std::string name(p.name);
        auto it = std::find_if(c.prof_stats.begin(), c.prof_stats.end(), [&](auto& x) { return x.name == name; });
        if (it == c.prof_stats.end()) {
            c.prof_stats.push_back({name});
            it = c.prof_stats.end() - 1;
        }
        it->ms += f;
        it->units += p.units;
        it->count += 1;
    }
    c.prof_pending.clear();
}

static size_t blocks(size_t n, unsigned b) { return (n + b - 1) / b; }

static unsigned ntt_block(u32 N) { return std::min<u32>(512, N / 2); }

// ------------------------------------------------------------------ tables
struct Blob {
    std::vector<unsigned char> b;
    template <class T>
    size_t add(const std::vector<T>& v) {
        size_t off = (b.size() + 255) & ~size_t(255);
        b.resize(off + v.size() * sizeof(T) + 1);
        if (!v.empty()) std::memcpy(b.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

static u32 inv32_neg(u32 a) {  // -a^-1 mod 2^32
    u32 x = a;
    for (int i = 0; i < 5; ++i) x *= 2 - a * x;
    return (u32)(0u - x);
}

static u32 shoup32h(u32 w, u32 p) { return (u32)(((u64)w << 32) / p); }
static u64 shoup64h(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

/// (JM, NC) pairs k_round_tma is instantiated for (TMEM: JM + NC <= 128 columns).
static bool tc_instance(u32 JM, u32 nc) {
    return (JM == 8 && (nc == 48 || nc == 64)) || (JM == 16 && (nc == 64 || nc == 80)) ||
           (JM == 24 && (nc == 80 || nc == 96)) || (JM == 32 && nc == 96);
}

/// k_round_tma tables: the parameter block (integer epilogue constants, Montgomery forms) and the
/// B matrix [NC][K = 4 JM] of u8, K-major in the canonical no-swizzle UMMA layout (8-row x 16-B
/// core matrices; a row's 16-B K chunks 128 B apart, 8-row groups K/16 * 128 B apart).
static bool build_round_tc(u32 JM, u32 NC, const std::vector<RoundJ>& rj, const std::vector<RoundK>& rk,
                           const std::vector<u32>& Imod, const std::vector<u32>& a, u32 J, u32 Mm,
                           std::vector<unsigned char>& par, std::vector<unsigned char>& Bm) {
    const u32 K = 4 * JM, F0 = NC - 17, G0 = NC - 6, MMAX = F0 / 4;
    Bm.assign((size_t)NC * K, 0);
    auto put = [&](u32 n, u32 kb, unsigned char v) {
        Bm[(size_t)(n / 8) * (K / 16 * 128) + (kb / 16) * 128 + (n % 8) * 16 + kb % 16] = v;
    };
    auto mf = [](u64 x, u32 p) { return (u32)((((u128)(x % p)) << 32) % p); };  // Montgomery form
    for (u32 k = 0; k < Mm; ++k)
        for (u32 j = 0; j < J; ++j) {
            const u32 p = a[k];
            const u64 Im = mf(Imod[(size_t)j * Mm + k], p);
            for (u32 aa = 0; aa < 4; ++aa) {
                const u32 v = (u32)((Im << (8 * aa)) % p);  // (2^(8a) I_kj 2^32) mod a_k
                for (u32 b = 0; b < 4; ++b) put(4 * k + b, 4 * j + aa, (unsigned char)(v >> (8 * b)));
            }
        }
    for (u32 j = 0; j < J; ++j) {
        const u64 F = ((u64)rj[j].f1 << 32) | rj[j].f0;
        const u64 G = (1ull << 46) / a[j];
        for (u32 aa = 0; aa < 4; ++aa) {
            for (u32 sft = 0; sft < 11; ++sft)
                if (sft >= aa && sft - aa < 8) put(F0 + sft, 4 * j + aa, (unsigned char)(F >> (8 * (sft - aa))));
            for (u32 sft = 0; sft < 6; ++sft)
                if (sft >= aa && sft - aa < 3) put(G0 + sft, 4 * j + aa, (unsigned char)(G >> (8 * (sft - aa))));
        }
    }
    // parameter block: RoundTcPar<JM, NC> = uint4 kq[MMAX] + u32 krm[MMAX] + u32 kc0[MMAX] + u32 kc30[MMAX]
    par.assign((size_t)MMAX * 16 + (size_t)MMAX * 12, 0);
    u32* P = reinterpret_cast<u32*>(par.data());
    for (u32 k = 0; k < Mm && k < MMAX; ++k) {
        const u32 p = rk[k].a;
        if (p >= (1u << 30) || (1u << 30) - p >= (1u << 24)) return false;  // epilogue needs 2^30 - a < 2^24
        P[4 * k + 0] = p;
        P[4 * k + 1] = rk[k].pinv;
        P[4 * k + 2] = rk[k].gcoef;
        P[4 * k + 3] = (1u << 30) - p;
        P[4 * MMAX + k] = rk[k].roff;
        P[5 * MMAX + k] = (u32)((1ull << 32) % p);
        P[6 * MMAX + k] = (u32)(((u128)1 << 62) % p);
    }
    return true;
}

static void build_tables(Ctx& c) {
    const ChainParams& cp = c.cp;
    const AuxBasis& ab = c.ab;
    const u32 N = cp.N, L = cp.L, J = ab.J, Mm = ab.Mm;
    Blob blob;
    DevTab T{};
    T.N = N;
    T.logN = cp.logN;
    T.L = L;
    T.J = J;
    T.Mm = Mm;
    T.Dr = cp.Dr;
    T.Dg = cp.Dg;
    T.relin_bits = cp.relin_bits;
    T.galois_bits = cp.galois_bits;
    T.t = cp.t;
    T.gbits = 6;
    T.force_exact = c.force_exact ? 1u : 0u;
    T.DS = c.ab.J;  // D-plane stride
    const Big& Q = cp.Q;
    T.QW = (cp.q_bits + 31) / 32;
    if (T.QW > (u32)kQW) throw std::invalid_argument("cwgpu: modulus too wide");
    // chain
    std::vector<u64> q(L), mu96(L), gh(L), gl(L), muq(L), muq_s(L), ninv(L), ninv_s(L), delta(L);
    std::vector<u64> crp, crps, cirp, cirps;
    std::vector<u32> qov;
    Big dq = Q.div_u64(cp.t);
    for (u32 i = 0; i < L; ++i) {
        const u64 qi = cp.q[i];
        q[i] = qi;
        mu96[i] = (u64)(((u128)1 << 96) / qi);
        const u128 G = (~(u128)0) / qi;
        gh[i] = (u64)(G >> 64);
        gl[i] = (u64)G;
        Big ov = Q.div_u64(qi);
        muq[i] = invmod64(ov.mod_u64(qi), qi);
        muq_s[i] = shoup64h(muq[i], qi);
        ninv[i] = invmod64(N % qi, qi);
        ninv_s[i] = shoup64h(ninv[i], qi);
        delta[i] = dq.mod_u64(qi);
        NttTables nt = make_ntt_tables(N, qi, 64);
        crp.insert(crp.end(), nt.rp.begin(), nt.rp.end());
        crps.insert(crps.end(), nt.rps.begin(), nt.rps.end());
        cirp.insert(cirp.end(), nt.irp.begin(), nt.irp.end());
        cirps.insert(cirps.end(), nt.irps.begin(), nt.irps.end());
        auto l = ov.limbs32(T.QW);
        qov.insert(qov.end(), l.begin(), l.end());
    }
    std::vector<u32> qw = Q.limbs32(T.QW);
    // aux
    std::vector<u32> a(J), apinv(J), a2_64(J), ninvA(J), ninvA_s(J), ninvRA(J), ninvRA_s(J);
    std::vector<u64> abar(J), aF(J);
    std::vector<u32> arp, arps, airp, airps;
    Big A(1);
    for (u32 j = 0; j < J; ++j) A = A.mul_u64(ab.a[j]);
    Big M(1);
    for (u32 k = 0; k < Mm; ++k) M = M.mul_u64(ab.a[k]);
    T.AW = (A.bits() + 31) / 32;
    if (T.AW > (u32)kAW) throw std::invalid_argument("cwgpu: aux basis too wide");
    std::vector<u32> chat(J), chat_s(J), frac96(3 * J), Imod((size_t)J * Mm), Aov, ninvRAc(J), ninvRAc_s(J);
    std::vector<u64> ImodQ((size_t)J * L);
    std::vector<u32> liftV_m((size_t)L * J), liftV2_m((size_t)L * J), liftW_m(J), liftV_n((size_t)L * J),
        liftV2_n((size_t)L * J), liftW_n(J);
    for (u32 j = 0; j < J; ++j) {
        const u32 p = (u32)ab.a[j];
        a[j] = p;
        apinv[j] = inv32_neg(p);
        abar[j] = (~0ull) / p;
        a2_64[j] = (u32)(((u128)1 << 64) % p);
        aF[j] = (1ull << (64 - T.gbits)) / p;
        ninvA[j] = (u32)invmod64(N % p, p);
        ninvA_s[j] = shoup32h(ninvA[j], p);
        const u64 r32 = (1ull << 32) % p;
        ninvRA[j] = (u32)invmod64(mulmod64(N % p, r32, p), p);
        ninvRA_s[j] = shoup32h(ninvRA[j], p);
        NttTables nt = make_ntt_tables(N, p, 32);
        for (u32 x = 0; x < N; ++x) {
            arp.push_back((u32)nt.rp[x]);
            arps.push_back((u32)nt.rps[x]);
            airp.push_back((u32)nt.irp[x]);
            airps.push_back((u32)nt.irps[x]);
        }
        Big Aj = A.div_u64(p);
        chat[j] = (u32)invmod64(Aj.mod_u64(p), p);
        chat_s[j] = shoup32h(chat[j], p);
        ninvRAc[j] = (u32)mulmod64(ninvRA[j], chat[j], p);
        ninvRAc_s[j] = shoup32h(ninvRAc[j], p);
        // t (A/a_j) = I_j q + R_j ; frac96 = floor(R_j 2^96 / q)
        Big tA = Aj.mul_u64(cp.t), I, R;
        Big::divmod(tA, Q, I, R);
        Big f, fr;
        Big::divmod(R.shl(96), Q, f, fr);
        for (int w = 0; w < 3; ++w) frac96[3 * j + w] = (u32)(f.limb(w / 2) >> (32 * (w % 2)));
        for (u32 k = 0; k < Mm; ++k) Imod[(size_t)j * Mm + k] = (u32)I.mod_u64(ab.a[k]);
        for (u32 i = 0; i < L; ++i) ImodQ[(size_t)j * L + i] = I.mod_u64(cp.q[i]);
        auto l = Aj.limbs32(T.AW);
        Aov.insert(Aov.end(), l.begin(), l.end());
        // chain -> aux lift constants
        const u64 qmod = Q.mod_u64(p);
        liftW_n[j] = (u32)qmod;
        liftW_m[j] = (u32)mulmod64(qmod, r32, p);
        for (u32 i = 0; i < L; ++i) {
            const u64 v = Q.div_u64(cp.q[i]).mod_u64(p);
            const u64 v2 = mulmod64(v, (1ull << 30) % p, p);
            liftV_n[(size_t)i * J + j] = (u32)v;
            liftV2_n[(size_t)i * J + j] = (u32)v2;
            liftV_m[(size_t)i * J + j] = (u32)mulmod64(v, r32, p);
            liftV2_m[(size_t)i * J + j] = (u32)mulmod64(v2, r32, p);
        }
    }
    std::vector<u32> fracA(3), IAmod(Mm);
    std::vector<u64> IAmodQ(L);
    {
        Big tA = A.mul_u64(cp.t), I, R, f, fr;
        Big::divmod(tA, Q, I, R);
        Big::divmod(R.shl(96), Q, f, fr);
        for (int w = 0; w < 3; ++w) fracA[w] = (u32)(f.limb(w / 2) >> (32 * (w % 2)));
        for (u32 k = 0; k < Mm; ++k) IAmod[k] = (u32)I.mod_u64(ab.a[k]);
        for (u32 i = 0; i < L; ++i) IAmodQ[i] = I.mod_u64(cp.q[i]);
    }
    std::vector<u32> Aw = A.limbs32(T.AW);
    // MAC basis -> chain
    std::vector<u32> mhat(Mm), mhat_s(Mm);
    std::vector<u64> mF(Mm), Mconv((size_t)Mm * L), MnegQ(L);
    for (u32 k = 0; k < Mm; ++k) {
        const u32 p = (u32)ab.a[k];
        Big Mk = M.div_u64(p);
        mhat[k] = (u32)invmod64(Mk.mod_u64(p), p);
        mhat_s[k] = shoup32h(mhat[k], p);
        mF[k] = aF[k];
        for (u32 i = 0; i < L; ++i) Mconv[(size_t)k * L + i] = Mk.mod_u64(cp.q[i]);
    }
    for (u32 i = 0; i < L; ++i) {
        const u64 mm = M.mod_u64(cp.q[i]);
        MnegQ[i] = mm ? cp.q[i] - mm : 0;
    }

#define ADD(name) const size_t o_##name = blob.add(name)
    ADD(q); ADD(mu96); ADD(gh); ADD(gl); ADD(muq); ADD(muq_s); ADD(ninv); ADD(ninv_s); ADD(delta);
    ADD(crp); ADD(crps); ADD(cirp); ADD(cirps); ADD(qw); ADD(qov);
    ADD(a); ADD(apinv); ADD(abar); ADD(a2_64); ADD(ninvA); ADD(ninvA_s); ADD(ninvRA); ADD(ninvRA_s);
    ADD(arp); ADD(arps); ADD(airp); ADD(airps);
    ADD(liftV_m); ADD(liftV2_m); ADD(liftW_m); ADD(liftV_n); ADD(liftV2_n); ADD(liftW_n);
    ADD(chat); ADD(chat_s); ADD(ninvRAc); ADD(ninvRAc_s); ADD(aF); ADD(frac96); ADD(fracA); ADD(Imod); ADD(IAmod); ADD(ImodQ); ADD(IAmodQ);
    ADD(Aw); ADD(Aov); ADD(mhat); ADD(mhat_s); ADD(mF); ADD(Mconv); ADD(MnegQ);
#undef ADD
    c.tab.ensure(blob.b.size());
    CK(cudaMemcpy(c.tab.p, blob.b.data(), blob.b.size(), cudaMemcpyHostToDevice));
    unsigned char* base = static_cast<unsigned char*>(c.tab.p);
#define P64(field, name) T.field = reinterpret_cast<const u64*>(base + o_##name)
#define P32(field, name) T.field = reinterpret_cast<const u32*>(base + o_##name)
    P64(q, q); P64(q_mu96, mu96); P64(q_gh, gh); P64(q_gl, gl); P64(muq, muq); P64(muq_s, muq_s);
    P64(ninv, ninv); P64(ninv_s, ninv_s); P64(delta, delta); P64(crp, crp); P64(crps, crps); P64(cirp, cirp);
    P64(cirps, cirps); P32(qw, qw); P32(qov, qov);
    P32(a, a); P32(apinv, apinv); P64(abar, abar); P32(a2_64, a2_64); P32(ninvA, ninvA); P32(ninvA_s, ninvA_s);
    P32(ninvRA, ninvRA); P32(ninvRA_s, ninvRA_s); P32(arp, arp); P32(arps, arps); P32(airp, airp); P32(airps, airps);
    P32(liftV_m, liftV_m); P32(liftV2_m, liftV2_m); P32(liftW_m, liftW_m); P32(liftV_n, liftV_n);
    P32(liftV2_n, liftV2_n); P32(liftW_n, liftW_n);
    P32(chat, chat); P32(chat_s, chat_s); P32(ninvRAc, ninvRAc); P32(ninvRAc_s, ninvRAc_s); P64(aF, aF); P32(frac96, frac96); P32(fracA, fracA); P32(Imod, Imod);
    P32(IAmod, IAmod); P64(ImodQ, ImodQ); P64(IAmodQ, IAmodQ); P32(Aw, Aw); P32(Aov, Aov);
    P32(mhat, mhat); P32(mhat_s, mhat_s); P64(mF, mF); P64(Mconv, Mconv); P64(MnegQ, MnegQ);
#undef P64
#undef P32
    T.fallbacks = c.d_fb;
    c.T = T;
    // HPS rounding tables for k_round_mac_t (padded to JM, ImodT transposed)
    {
        c.JM = std::max<u32>(8, (J + 7) / 8 * 8);
        if (c.JM > 40) throw std::invalid_argument("cwgpu: too many aux primes for the rounding kernel");
        std::vector<RoundJ> rj(c.JM);
        for (u32 j = 0; j < c.JM; ++j) {
            RoundJ x{};
            if (j < J) {
                x.a = a[j]; x.chat = chat[j]; x.chat_s = chat_s[j]; x.aF = aF[j];
                x.f0 = frac96[3 * j + 1]; x.f1 = frac96[3 * j + 2];  // top 64 bits of the 96-bit fraction
            } else {
                x.a = 1;  // padded prime: w_j = 0
            }
            rj[j] = x;
        }
        std::vector<RoundK> rk(kMaxJ);
        auto mf = [](u64 x, u32 p) { return (u32)((((u128)(x % p)) << 32) % p); };  // Montgomery form
        for (u32 k = 0; k < Mm; ++k) {
            RoundK x{};
            x.a = a[k];
            x.pinv = apinv[k];
            x.gcoef = mf((a[k] - IAmod[k]) % a[k], a[k]);
            x.roff = mf((a[k] - (u32)(((u128)1 << 36) % a[k])) % a[k], a[k]);
            x.c0 = mf(1, a[k]);
            x.c30 = mf(1ull << 30, a[k]);
            x.abar = abar[k];
            rk[k] = x;
        }
        std::vector<u32> imT((size_t)Mm * c.JM, 0);
        for (u32 k = 0; k < Mm; ++k)
            for (u32 j = 0; j < J; ++j) imT[(size_t)k * c.JM + j] = mf(Imod[(size_t)j * Mm + k], a[k]);
        const size_t bytes = sizeof(RoundJ) * c.JM + sizeof(RoundK) * kMaxJ + imT.size() * 4;
        std::vector<unsigned char> blob(bytes);
        std::memcpy(blob.data(), rj.data(), sizeof(RoundJ) * c.JM);
        std::memcpy(blob.data() + sizeof(RoundJ) * c.JM, rk.data(), sizeof(RoundK) * kMaxJ);
        std::memcpy(blob.data() + sizeof(RoundJ) * c.JM + sizeof(RoundK) * kMaxJ, imT.data(), imT.size() * 4);
        c.round_tab.ensure(bytes);
        CK(cudaMemcpy(c.round_tab.p, blob.data(), bytes, cudaMemcpyHostToDevice));
        // tensor-core rounding: smallest instantiated GEMM width holding 4 Mm + 17 columns
        c.rtc.clear();
        c.rtc_nc = 0;
        const u32 need = 4 * Mm + 17;
        for (u32 nc : {48u, 64u, 80u, 96u, 112u}) {
            if (nc < need || !tc_instance(c.JM, nc)) continue;
            c.rtc_nc = nc;
            break;
        }
        if (c.rtc_nc) {
            std::vector<unsigned char> Bm;
            if (build_round_tc(c.JM, c.rtc_nc, rj, rk, Imod, a, J, Mm, c.rtc, Bm)) {
                c.rtc_B.ensure(Bm.size());
                CK(cudaMemcpy(c.rtc_B.p, Bm.data(), Bm.size(), cudaMemcpyHostToDevice));
                // second GEMM of k_round_tma (K = 32 bytes): A2 = [gamma, rb0..rb4, 1, 0...] per
                // coefficient; column 4k+b collects byte b of gamma (-I_A 2^32), (2^(8i) 2^32) rb_i
                // and (-2^36) 2^32, all mod a_k, so the residue columns end as S_k + the corrections
                {
                    const u32 NC = c.rtc_nc, K2 = 32;
                    std::vector<unsigned char> B2((size_t)NC * K2, 0);
                    auto put2 = [&](u32 n, u32 kb, unsigned char v) {
                        B2[(size_t)(n / 8) * (K2 / 16 * 128) + (kb / 16) * 128 + (n % 8) * 16 + kb % 16] = v;
                    };
                    for (u32 k = 0; k < Mm && 4 * k + 3 < NC - 17; ++k) {
                        const u64 p = rk[k].a;
                        const u64 h32 = (1ull << 32) % p;
                        u64 cst[7];
                        cst[0] = rk[k].gcoef;  // (-I_A) 2^32 mod a_k
                        for (u32 i = 0; i < 5; ++i) cst[1 + i] = (u64)(((u128)h32 << (8 * i)) % p);
                        cst[6] = rk[k].roff;   // (-2^36) 2^32 mod a_k
                        for (u32 kb = 0; kb < 7; ++kb)
                            for (u32 b = 0; b < 4; ++b) put2(4 * k + b, kb, (unsigned char)(cst[kb] >> (8 * b)));
                    }
                    c.rtc_B2.ensure(B2.size());
                    CK(cudaMemcpy(c.rtc_B2.p, B2.data(), B2.size(), cudaMemcpyHostToDevice));
                }
            } else {
                c.rtc_nc = 0;  // IMAD rounding (k_round_mac_t) instead
            }
        }
    }
    // tensor-core lift (k_lift_tc): B matrices [NC][K = 64] of byte b of (2^(8a) V_ij mod a_j) at
    // column 4 j + b, K byte 8 i + a, for the Montgomery and the plain lift constants
    c.lift_nc = 0;
    if (L <= 8 && 4 * J <= 112) {
        const u32 NCl = (4 * J + 15) / 16 * 16, K = 64;
        std::vector<unsigned char> Bl((size_t)2 * NCl * K, 0);
        for (int mont = 0; mont < 2; ++mont) {
            unsigned char* B = Bl.data() + (size_t)mont * NCl * K;
            auto put = [&](u32 n, u32 kb, unsigned char v) {
                B[(size_t)(n / 8) * (K / 16 * 128) + (kb / 16) * 128 + (n % 8) * 16 + kb % 16] = v;
            };
            for (u32 j = 0; j < J; ++j)
                for (u32 i = 0; i < L; ++i) {
                    const u64 p = a[j];
                    // with one more factor 2^32: the epilogue reduces by a Montgomery step (x 2^-32)
                    const u64 V = (((u64)(mont ? liftV_m[(size_t)i * J + j] : liftV_n[(size_t)i * J + j])) << 32) % p;
                    for (u32 aa = 0; aa < 8; ++aa) {
                        const u32 v = (u32)(((u128)V << (8 * aa)) % p);
                        for (u32 b = 0; b < 4; ++b) put(4 * j + b, 8 * i + aa, (unsigned char)(v >> (8 * b)));
                    }
                }
        }
        c.lift_B.ensure(Bl.size());
        CK(cudaMemcpy(c.lift_B.p, Bl.data(), Bl.size(), cudaMemcpyHostToDevice));
        // rho term of the lift in the same form: (a_j - W_j) 2^32 mod a_j, [plain | Montgomery][J]
        std::vector<u32> W2((size_t)2 * J);
        for (int mont = 0; mont < 2; ++mont)
            for (u32 j = 0; j < J; ++j) {
                const u64 p = a[j];
                const u64 w = mont ? liftW_m[j] : liftW_n[j];
                W2[(size_t)mont * J + j] = (u32)((((p - w % p) % p) << 32) % p);
            }
        c.lift_W2.ensure(W2.size() * 4);
        CK(cudaMemcpy(c.lift_W2.p, W2.data(), W2.size() * 4, cudaMemcpyHostToDevice));
        c.lift_nc = NCl;
    }
    // tensor-core MAC basis -> chain conversion (k_mac_to_chain_tc): B [64][K = 4 KW] of byte b of
    // (2^(8a) (M/a_k) mod q_i) at column 8 i + b, K byte 4 k + a
    c.m2c_kw = 0;
    if (L <= 8 && Mm <= 24) {
        const u32 KW = Mm <= 16 ? 16 : 24, K = 4 * KW, NCm = 64;
        std::vector<unsigned char> Bm((size_t)NCm * K, 0);
        auto put = [&](u32 n, u32 kb, unsigned char v) {
            Bm[(size_t)(n / 8) * (K / 16 * 128) + (kb / 16) * 128 + (n % 8) * 16 + kb % 16] = v;
        };
        for (u32 k = 0; k < Mm; ++k)
            for (u32 i = 0; i < L; ++i) {
                const u64 qi = cp.q[i];
                for (u32 aa = 0; aa < 4; ++aa) {
                    const u64 v = (u64)(((u128)Mconv[(size_t)k * L + i] << (8 * aa)) % qi);
                    for (u32 b = 0; b < 8; ++b) put(8 * i + b, 4 * k + aa, (unsigned char)(v >> (8 * b)));
                }
            }
        c.m2c_B.ensure(Bm.size());
        CK(cudaMemcpy(c.m2c_B.p, Bm.data(), Bm.size(), cudaMemcpyHostToDevice));
        c.m2c_kw = KW;
    }
    // tensor-core digit decomposition (k_decompose_tc): B [64][K = 64], column s, K byte 8 i + a = byte
    // s - a of q / q_i (32-bit limbs qov [L][QW])
    c.dec_ok = false;
    if (L <= 8 && 4 * T.QW + 7 < 64) {
        const u32 K = 64, NCd = 64;
        std::vector<unsigned char> Bd((size_t)NCd * K, 0);
        auto put = [&](u32 n, u32 kb, unsigned char v) {
            Bd[(size_t)(n / 8) * (K / 16 * 128) + (kb / 16) * 128 + (n % 8) * 16 + kb % 16] = v;
        };
        for (u32 i = 0; i < L; ++i)
            for (u32 aa = 0; aa < 8; ++aa)
                for (u32 sb = 0; sb < 4 * T.QW && sb + aa < NCd; ++sb)
                    put(sb + aa, 8 * i + aa, (unsigned char)(qov[(size_t)i * T.QW + sb / 4] >> (8 * (sb % 4))));
        c.dec_B.ensure(Bd.size());
        CK(cudaMemcpy(c.dec_B.p, Bd.data(), Bd.size(), cudaMemcpyHostToDevice));
        c.dec_ok = true;
    }
    // device copy of the table itself (slow paths read it through T.self)
    c.tab_self.ensure(sizeof(DevTab));
    c.T.self = static_cast<const DevTab*>(c.tab_self.p);
    CK(cudaMemcpy(c.tab_self.p, &c.T, sizeof(DevTab), cudaMemcpyHostToDevice));
}


static void ensure_aux(Ctx& c, u64 n_total) {
    n_total = std::max<u64>(n_total, 1);
    if (c.aux_n == n_total && c.ab.J) return;
    AuxBasis nb = choose_aux_basis(c.cp, n_total);
    const bool same = c.ab.J && nb.a == c.ab.a && nb.Mm == c.ab.Mm;
    c.aux_n = n_total;
    if (same) return;
    c.ab = nb;
    build_tables(c);
    c.ksA_ok = false;
}

// ------------------------------------------------------------------ NTT launchers
static void ntt64(Ctx& c, u64* data, u32 npolys, bool inverse) {
    const u32 N = c.cp.N;
    if (inverse)
        launch_named(c, "k_ntt64_inv", k_ntt64<true, false>, npolys, ntt_block(N), N * 8, data, (const u64*)nullptr, c.T);
    else
        launch_named(c, "k_ntt64_fwd", k_ntt64<false, false>, npolys, ntt_block(N), N * 8, data, (const u64*)nullptr, c.T);
}

// Register-resident NTT kernels (ntt_reg.cuh) for 2^8 <= N <= 2^14; the shared-memory
// radix-2 kernels remain for smaller rings.
template <int LOGN>
struct Reg32 {
    using R = RegNtt<LOGN>;
    static void limits() {
        const int sm = (int)R::SMEM;
        CK(cudaFuncSetAttribute(k_ntt32r<LOGN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_ntt32r<LOGN, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_ntt32r<LOGN, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_ntt32r<LOGN, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_ntt32r_sel3<LOGN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_ntt32r_sel3<LOGN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * sm));
        CK(cudaFuncSetAttribute(k_tensor_intt_r<LOGN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CK(cudaFuncSetAttribute(k_tensor_intt_r<LOGN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * sm));
#define NM(NC, S, A) CK(cudaFuncSetAttribute(k_ntt_mac<LOGN, NC, S, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NttMac<LOGN, S, A>::SMEM));
        NM(2, 1, true) NM(3, 1, true) NM(2, 2, true) NM(3, 2, true)
#undef NM
    }
    /// fused selection NTT + payload MAC over the R rows of a tile (Z: coefficient-domain
    /// MAC-basis selection planes, Z + ((r * nc + comp) * zs + k) * N)
    static void ntt_mac(Ctx& c, const u32* Z, u32 zs, u32 nc, const u32* dbt, u32 Rt, unsigned long long* acc) {
        const u32 Mm = c.ab.Mm;
        const u32 per = nc * Mm;  // CTAs per row chunk
        // row chunks per (component, prime), balanced to +-1 row: ~2 waves of resident CTAs, >= 8
        // rows per chunk (fewer accumulator atomics); env CWGPU_MAC_CK overrides
        const u32 slots = 148 * 3 * 2;
        u32 ck = std::max<u32>(1, std::min<u32>((Rt + 7) / 8, (slots + per - 1) / per));
        if (c.mac_ck) ck = std::max<u32>(1, std::min<u32>(c.mac_ck, Rt));
        const u32 chunk = ck;  // the kernels take the chunk count
        c.next_units = (double)Rt * nc * Mm;  // polynomials transformed (+ payload words streamed)
        const size_t grid = (size_t)ck * per;
#define NMC(NC, S, A) launch_named(c, "k_ntt_mac", k_ntt_mac<LOGN, NC, S, A>, grid, R::T, NttMac<LOGN, S, A>::SMEM, Z, zs, dbt, Rt, chunk, c.T, acc)
        if (nc == 3) {
            if (c.s == 1) NMC(3, 1, true);
            else NMC(3, 2, true);
        } else {
            if (c.s == 1) NMC(2, 1, true);
            else NMC(2, 2, true);
        }
#undef NMC
    }
    static void ntt(Ctx& c, u32* base, u32 npolys, u32 gs, u32 stride, u32 off, bool inverse, int scale, bool perm) {
        if (inverse && perm)
            launch_named(c, "k_ntt32r_inv", k_ntt32r<LOGN, true, true>, npolys, R::T, R::SMEM, base, c.T, gs, stride,
                         off, scale);
        else if (perm)
            launch_named(c, "k_ntt32r_fwd", k_ntt32r<LOGN, false, true>, npolys, R::T, R::SMEM, base, c.T, gs, stride,
                         off, scale);
        else if (inverse)
            launch_named(c, "k_ntt32r_inv", k_ntt32r<LOGN, true, false>, npolys, R::T, R::SMEM, base, c.T, gs, stride,
                         off, scale);
        else
            launch_named(c, "k_ntt32r_fwd", k_ntt32r<LOGN, false, false>, npolys, R::T, R::SMEM, base, c.T, gs, stride,
                         off, scale);
    }
    static void sel3(Ctx& c, u32* D, u32 P, u32 stride) {
        const u32 npc = 3 * P;
        c.next_units = (double)npc * c.ab.Mm;
        if (c.ntt_np == 2)
            launch_named(c, "k_ntt32r_sel3", k_ntt32r_sel3<LOGN, 2>, (size_t)((npc + 1) / 2) * c.ab.Mm, R::T,
                         2 * R::SMEM, D, c.T, stride, npc);
        else
            launch_named(c, "k_ntt32r_sel3", k_ntt32r_sel3<LOGN, 1>, (size_t)npc * c.ab.Mm, R::T, R::SMEM, D, c.T,
                         stride, npc);
    }
    static void tensor(Ctx& c, const u32* pa, const u32* ia, const u32* pb, const u32* ib, u32 P, u32* D, int fold) {
        c.next_units = (double)P * c.ab.J * 3;
        if (c.ntt_np == 2)
            launch_named(c, "k_tensor_intt", k_tensor_intt_r<LOGN, 2>, (size_t)((P + 1) / 2) * c.ab.J * 3, R::T,
                         2 * R::SMEM, pa, ia, pb, ib, P, c.T, D, fold);
        else
            launch_named(c, "k_tensor_intt", k_tensor_intt_r<LOGN, 1>, (size_t)P * c.ab.J * 3, R::T, R::SMEM, pa, ia,
                         pb, ib, P, c.T, D, fold);
    }
};

#define REG32_DISPATCH(logn, call)            \
    switch (logn) {                           \
        case 8: Reg32<8>::call; break;        \
        case 9: Reg32<9>::call; break;        \
        case 10: Reg32<10>::call; break;      \
        case 11: Reg32<11>::call; break;      \
        case 12: Reg32<12>::call; break;      \
        case 13: Reg32<13>::call; break;      \
        case 14: Reg32<14>::call; break;      \
        default: throw std::logic_error("no register NTT for this degree"); \
    }

static void set_smem_limits(u32 N) {
    CK(cudaFuncSetAttribute(k_mac_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMacStages * 4 * kMacBlock * 4));
    CK(cudaFuncSetAttribute(k_mac_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMacStages * 3 * kMacBlock * 4));
#define MQ(NCv, QBv, SGv)                                                                                         \
    CK(cudaFuncSetAttribute(k_mac_tma_q<NCv, QBv, SGv>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                            kMacStages * (SGv + QBv * NCv) * kMacBlockQ * 4));
    MQ(2, 1, 1) MQ(2, 2, 1) MQ(2, 3, 1) MQ(2, 4, 1) MQ(3, 1, 1) MQ(3, 2, 1) MQ(3, 3, 1) MQ(3, 4, 1)
    MQ(2, 1, 3) MQ(3, 1, 3) MQ(2, 1, 5) MQ(3, 1, 5)
#undef MQ
    CK(cudaFuncSetAttribute(k_mac_tma_q<2, 1, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * (3 + 2) * kMacBlockQ * 4));
#define MAC_ROWS_ATTR(NCv, SGv, STv)                                                                         \
    CK(cudaFuncSetAttribute(k_mac_rows<NCv, SGv, STv>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                            STv * (SGv + NCv) * kMacBlockS * 4));
    MAC_ROWS_ATTR(3, 15, 10) MAC_ROWS_ATTR(2, 15, 10) MAC_ROWS_ATTR(3, 5, 16) MAC_ROWS_ATTR(2, 5, 16)
    MAC_ROWS_ATTR(3, 3, 16) MAC_ROWS_ATTR(2, 3, 16)
#undef MAC_ROWS_ATTR
    CK(cudaFuncSetAttribute(k_mac_tma_q<3, 1, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * (3 + 3) * kMacBlockQ * 4));
#define RTC(JMv, NCv)                                                                                                \
    CK(cudaFuncSetAttribute(k_round_tma<0, JMv, NCv>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)round_tma_smem<JMv>())); \
    {                                                                                                                \
        constexpr int LN = JMv == 16 ? 13 : JMv == 8 ? 12 : JMv == 32 ? 14 : 0;                                     \
        CK(cudaFuncSetAttribute(k_round_tma<LN, JMv, NCv>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)round_tma_smem<JMv>())); \
        if (LN == 13) CK(cudaFuncSetAttribute(k_round_tma<LN, JMv, NCv, 11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)round_tma_smem<JMv>())); \
        if (LN == 13) CK(cudaFuncSetAttribute(k_round_tma<LN, JMv, NCv, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)round_tma_smem<JMv>())); \
    }
    RTC(8, 48) RTC(8, 64) RTC(16, 64) RTC(16, 80) RTC(24, 80) RTC(24, 96) RTC(32, 96)
#undef RTC
    Reg32<8>::limits(); Reg32<9>::limits(); Reg32<10>::limits(); Reg32<11>::limits();
    Reg32<12>::limits(); Reg32<13>::limits(); Reg32<14>::limits();
    const int s64 = (int)(N * sizeof(u64)), s32 = (int)(N * sizeof(u32));
    CK(cudaFuncSetAttribute(k_ntt64<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64));
    CK(cudaFuncSetAttribute(k_ntt64<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64));
    CK(cudaFuncSetAttribute(k_ntt64<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64));
    CK(cudaFuncSetAttribute(k_ntt32<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s32));
    CK(cudaFuncSetAttribute(k_ntt32<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s32));
    CK(cudaFuncSetAttribute(k_tensor_intt, cudaFuncAttributeMaxDynamicSharedMemorySize, s32));
}

static bool reg32_ok(u32 logN) { return logN >= 8 && logN <= 14; }

/// Aux / MAC-prime NTTs.  perm (default): the answer path's internal NTT-domain order (see
/// k_ntt32r); false: the reference's order (cwg_ntt).  Rings below 2^8 use the shared-memory
/// kernels in the reference's order throughout (their tensor kernel matches).
static void ntt32(Ctx& c, u32* base, u32 npolys, u32 gs, u32 stride, u32 off, bool inverse, int scale,
                  bool perm = true) {
    const u32 N = c.cp.N;
    if (reg32_ok(c.cp.logN)) {
        REG32_DISPATCH(c.cp.logN, ntt(c, base, npolys, gs, stride, off, inverse, scale, perm));
        return;
    }
    if (inverse)
        launch_named(c, "k_ntt32_inv", k_ntt32<true>, npolys, ntt_block(N), N * 4, base, c.T, gs, stride, off, scale);
    else
        launch_named(c, "k_ntt32_fwd", k_ntt32<false>, npolys, ntt_block(N), N * 4, base, c.T, gs, stride, off, scale);
}

// ------------------------------------------------------------------ key switching
/// ks[b] (2 comps, coefficient form) = key_switch(poly_b) for B polys at polys + b*stride
/// through automorphism ginv (0 = none) (bfv.cpp:343-372).
/// Garner constants of the aux primes that hold sum_d digit_d * key_d exactly:
/// |value| <= D N (2^bits - 1)(q_max - 1) (bits = 0: RNS digits < q_max), prod a_j > 2^2 |value|.
static KsCrt make_ks_crt(const Ctx& c, u32 bits, u32 D) {
    KsCrt C{};
    double qb = 0;
    for (u64 q : c.cp.q) qb = std::max(qb, std::log2((double)q));
    const double need = std::log2((double)D) + c.cp.logN + (bits ? bits : qb) + qb + 2.0;
    double have = 0;
    u32 K = 0;
    while (have < need) {
        if (K >= (u32)kMaxKs || K >= c.ab.J) return KsCrt{};  // K = 0: keep the 64-bit path
        C.a[K] = (u32)c.ab.a[K];
        have += std::log2((double)C.a[K]);
        ++K;
    }
    C.K = K;
    for (u32 j = 0; j < K; ++j) {
        C.half[j] = (C.a[j] - 1) / 2;
        for (u32 k = 0; k < j; ++k) {
            C.cinv[j][k] = (u32)invmod64(C.a[k] % C.a[j], C.a[j]);
            C.cinv_s[j][k] = (u32)(((u64)C.cinv[j][k] << 32) / C.a[j]);
        }
    }
    for (u32 i = 0; i < c.cp.L; ++i) {
        const u64 q = c.cp.q[i];
        u64 p = 1 % q;
        for (u32 j = 0; j < K; ++j) {
            C.pmod[i][j] = p;
            p = (u64)(((u128)p * C.a[j]) % q);
        }
        C.amod[i] = p;
    }
    return C;
}

/// Transform one key [D][2][L][N] (NTT form mod q_i, reference layout) into the key-switch aux
/// basis: [D][2][L][K'][N] u32, NTT form mod a_j.
static void key_to_aux(Ctx& c, const u64* key, u32 D, const KsCrt& C, u32* out) {
    const u32 N = c.cp.N, L = c.cp.L;
    const size_t np = (size_t)D * 2 * L;
    u64* tmp = c.dntt.get<u64>(np * N);
    CK(cudaMemcpyAsync(tmp, key, np * N * 8, cudaMemcpyDeviceToDevice, c.st));
    ntt64(c, tmp, (u32)np, true);  // coefficient form in [0, q_i)
    launch(c, k_to_ks_aux, blocks(np * N, 256), 256, 0, (const u64*)tmp, np, N, C, out);
    ntt32(c, out, (u32)(np * C.K), C.K, C.K, 0, false, 0);
}

/// relinA / galoisA for the uploaded keys (once per key upload or aux-basis change).
static bool ks32_ready(Ctx& c) {
    if (!c.ks32 || !c.have_keys) return false;
    if (c.ksA_ok) return true;
    const u32 N = c.cp.N, L = c.cp.L;
    c.ksC_r = make_ks_crt(c, c.cp.relin_bits, c.cp.Dr);
    c.ksC_g = make_ks_crt(c, c.cp.galois_bits, c.cp.Dg);
    if (c.ksC_r.K) {
        const size_t w = (size_t)c.cp.Dr * 2 * L * c.ksC_r.K * N;
        key_to_aux(c, c.relin.ptr<u64>(), c.cp.Dr, c.ksC_r, c.relinA.get<u32>(w));
    }
    if (c.ksC_g.K && !c.galois_g.empty()) {
        const size_t w = (size_t)c.cp.Dg * 2 * L * c.ksC_g.K * N, gw = (size_t)c.cp.Dg * 2 * L * N;
        u32* ga = c.galoisA.get<u32>(w * c.galois_g.size());
        for (size_t a = 0; a < c.galois_g.size(); ++a)
            key_to_aux(c, c.galois.ptr<u64>() + a * gw, c.cp.Dg, c.ksC_g, ga + a * w);
    }
    c.ksA_ok = true;
    return true;
}

/// add / add_stride / scale (aux-prime path only, see k_ks_crt): fused relinearisation add and
/// constant scaling; returns true when they were applied.
static bool key_switch(Ctx& c, const u64* polys, size_t stride, u64 ginv, u32 B, const u64* key, u32 bits,
                       u32 D, u64* ks, const u64* add = nullptr, size_t add_stride = 0, u64 scale = 0) {
    const u32 N = c.cp.N, L = c.cp.L;
    if (ks32_ready(c)) {
        const bool rel = key == c.relin.ptr<u64>();
        const KsCrt& C = rel ? c.ksC_r : c.ksC_g;
        if (C.K) {
            const u32 K = C.K;
            const u32* kA = nullptr;
            if (rel) {
                kA = c.relinA.ptr<u32>();
            } else {
                const size_t gw = (size_t)D * 2 * L * N;
                const size_t a = (size_t)(key - c.galois.ptr<u64>()) / gw;
                kA = c.galoisA.ptr<u32>() + a * (size_t)D * 2 * L * K * N;
            }
            u32* dA = c.ksdig.get<u32>((size_t)B * D * K * N);
            u32* mA = c.ksmac.get<u32>((size_t)B * 2 * L * K * N);
            if (c.dec_tc && c.dec_ok && bits == 16) {
                const size_t gr = std::min<size_t>(blocks((size_t)B * N, 128), (size_t)c.n_sms * 4);
                const uint4* Bd = c.dec_B.ptr<uint4>();
                const u32 QW = c.T.QW;  // limb count of q: the kernel's multiword loops are sized for it
                if (QW <= 4) launch_named(c, "k_decompose", k_decompose_tc<4>, gr, 128, 0, polys, stride, ginv, B, D, c.T, Bd, dA, K);
                else if (QW <= 7) launch_named(c, "k_decompose", k_decompose_tc<7>, gr, 128, 0, polys, stride, ginv, B, D, c.T, Bd, dA, K);
                else if (QW <= 10) launch_named(c, "k_decompose", k_decompose_tc<10>, gr, 128, 0, polys, stride, ginv, B, D, c.T, Bd, dA, K);
                else launch_named(c, "k_decompose", k_decompose_tc<14>, gr, 128, 0, polys, stride, ginv, B, D, c.T, Bd, dA, K);
            } else
                launch_named(c, "k_decompose", k_decompose_t<true>, blocks((size_t)B * N, 256), 256, 0, polys, stride, ginv,
                             B, bits, D, c.T, (u64*)nullptr, dA, K);
            ntt32(c, dA, B * D * K, K, K, 0, false, 0);
            // shared-load variant once the level is wide enough to fill the GPU (B >= 64 rows of
            // K N threads / 2); narrow levels and long digit chains keep one output per thread
            // (latency-bound otherwise: C5's D = 25, L = 8 ran 917 vs 320 ms with it)
            // slot-major MAC (key block in registers, rows streamed) for the digit counts of the
            // 16-bit decompositions of the configured chains (7: 108-bit q, 14: 218-bit, 25: 400-bit)
            const u32 gx = (u32)blocks((size_t)K * N, 128);
            const u32 gy = std::max<u32>(1, std::min<u32>(B, (148 * 6 + gx - 1) / gx));
            auto ks_s = [&](auto kern) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(gx, gy);
                cfg.blockDim = dim3(128);
                cfg.stream = c.st;
                c.next_units = (double)B * 2 * L * K * N * D;  // residue products (MACs)
                launch_grid(c, "k_ks_mac32", kern, cfg, (const u32*)dA, kA, B, L, N, C, (const u64*)c.T.abar, mA);
            };
            auto ks_t = [&](auto kern) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(gx, gy);
                cfg.blockDim = dim3(128);
                cfg.stream = c.st;
                c.next_units = (double)B * 2 * L * K * N * D;  // residue products (MACs)
                launch_grid(c, "k_ks_mac32", kern, cfg, (const u32*)dA, kA, B, c.T.a, c.T.apinv, c.T.a2_64, mA);
            };
            // every size at compile time (immediate plane offsets, Montgomery reductions) for the
            // configured shapes: (log N, K', D, 2L)
            const u32 lg = c.cp.logN;
            if (c.ks_fixed && c.ks_wide && lg == 14 && K == 3 && D == 25 && L == 8 && c.ks_ci == 4) ks_t(k_ks_mac32t<14, 3, 25, 16, 4, 16, 2>);
            else if (c.ks_fixed && c.ks_wide && lg == 14 && K == 3 && D == 25 && L == 8 && c.ks_ci == 8) ks_t(k_ks_mac32t<14, 3, 25, 16, 2, 16, 3>);
            else if (c.ks_fixed && c.ks_wide && lg == 14 && K == 3 && D == 25 && L == 8) ks_t(k_ks_mac32t<14, 3, 25, 16, 2, 8, 3>);
            else if (c.ks_fixed && c.ks_wide && lg == 13 && K == 3 && D == 14 && L == 5) ks_t(k_ks_mac32t<13, 3, 14, 10, 2, 8, 4>);
            else if (c.ks_fixed && c.ks_wide && lg == 12 && K == 3 && D == 7 && L == 3) ks_t(k_ks_mac32t<12, 3, 7, 6, 6, 8, 3>);
            else if (c.ks_wide && D == 7) ks_s(k_ks_mac32s<7, 6, 8, 3>);
            else if (c.ks_wide && D == 14 && c.ks_ci == 2) ks_s(k_ks_mac32s<14, 2, 8, 4, 2>);
            else if (c.ks_wide && D == 14) ks_s(k_ks_mac32s<14, 5, 8, 2>);
            else if (c.ks_wide && D == 25 && c.ks_ci == 2) ks_s(k_ks_mac32s<25, 2, 8, 3, 2>);
            else if (c.ks_wide && D == 25) ks_s(k_ks_mac32s<25, 4, 8, 2>);
            else if (D <= (u32)kKsDmax && B >= 64)
                launch_named(c, "k_ks_mac32", k_ks_mac32x<kKsDmax>, blocks((size_t)((B + 1) / 2) * K * N, 128), 128, 0,
                             (const u32*)dA, kA, B, D, L, N, C, (const u64*)c.T.abar, mA);
            else
                launch(c, k_ks_mac32, blocks((size_t)B * 2 * L * K * N, 256), 256, 0, (const u32*)dA, kA, B, D, L, N, C,
                       (const u64*)c.T.abar, mA);
            ntt32(c, mA, B * 2 * L * K, K, K, 0, true, 0);
            if (K == 3 && c.ks_fixed)
                launch_named(c, "k_ks_crt", k_ks_crt3, blocks((size_t)B * 2 * L * N, 256), 256, 0, (const u32*)mA, B, L, N, C,
                             c.T, ks, add, add_stride, scale);
            else
                launch(c, k_ks_crt, blocks((size_t)B * 2 * L * N, 256), 256, 0, (const u32*)mA, B, L, N, C, c.T, ks, add,
                       add_stride, scale);
            return true;
        }
    }
    u64* dig = c.digits.get<u64>((size_t)B * D * N);
    u64* dn = c.dntt.get<u64>((size_t)B * D * L * N);
    launch_named(c, "k_decompose", k_decompose_t<false>, blocks((size_t)B * N, 256), 256, 0, polys, stride, ginv, B, bits,
                 D, c.T, dig, (u32*)nullptr, 0u);
    launch_named(c, "k_ntt64_digits", k_ntt64<false, true>, (size_t)B * D * L, ntt_block(N), N * 8, dn, (const u64*)dig, c.T);
    launch(c, k_ks_mac, blocks((size_t)B * 2 * L * N, 256), 256, 0, (const u64*)dn, key, B, D, c.T, ks);
    ntt64(c, ks, B * 2 * L, true);
    return false;
}

static size_t ks_chunk(const Ctx& c, u32 D) {
    // bound the digit / digit-NTT scratch (3 GB by default: C5 96 rows per key-switch launch, 409 vs 417 ms per 4,096 rows at 1.5 GB; option "ks_chunk_mb")
    const size_t per = (size_t)D * (c.cp.L + 1) * c.cp.N * 8 + 2 * (size_t)c.cp.L * c.cp.N * 8;
    return std::max<size_t>(1, (size_t(c.ks_chunk_mb) << 20) / per);
}

/// relinearize count 3-comp cts (stride 3LN) into out2 [count][2][L][N]; scale != 0 multiplies the
/// result by that constant (fused into the key switch's CRT on the aux-prime path).
static void relinearize(Ctx& c, const u64* ct3, u32 count, u64* out2, u64 scale = 0) {
    const size_t LN = (size_t)c.cp.L * c.cp.N;
    const size_t chunk = ks_chunk(c, c.cp.Dr);
    for (u32 b0 = 0; b0 < count; b0 += (u32)chunk) {
        const u32 B = (u32)std::min<size_t>(chunk, count - b0);
        const u64* c3 = ct3 + (size_t)b0 * 3 * LN;
        u64* o2 = out2 + (size_t)b0 * 2 * LN;
        // the aux-prime key switch writes (c0 + ks0, c1 + ks1) straight into out2
        if (key_switch(c, c3 + 2 * LN, 3 * LN, 0, B, c.relin.ptr<u64>(), c.cp.relin_bits, c.cp.Dr, o2, c3, 3 * LN,
                       scale))
            continue;
        u64* ks = c.ks.get<u64>((size_t)B * 2 * LN);
        CK(cudaMemcpyAsync(ks, o2, (size_t)B * 2 * LN * 8, cudaMemcpyDeviceToDevice, c.st));
        launch(c, k_relin_add, blocks((size_t)B * 2 * LN, 256), 256, 0, c3, 3 * LN, (const u64*)ks, B, c.T, o2);
        if (scale) launch(c, k_scale_const, blocks((size_t)B * 2 * LN, 256), 256, 0, o2, B, scale, c.T);
    }
}

/// Relinearisation of R groups of np products whose third components are identical within a group
/// (ct3 [R][np][3][L][N]): one key switch per group (product 0's c2) into ks [R][2][L][N], then
/// out2[r][p] = (c0 + ks0, c1 + ks1) for every product of the group.
static void relinearize_shared(Ctx& c, const u64* ct3, u32 R, u32 np, u64* ks, u64* out2) {
    const size_t LN = (size_t)c.cp.L * c.cp.N;
    const size_t chunk = ks_chunk(c, c.cp.Dr);
    for (u32 r0 = 0; r0 < R; r0 += (u32)chunk) {
        const u32 B = (u32)std::min<size_t>(chunk, R - r0);
        key_switch(c, ct3 + (size_t)r0 * np * 3 * LN + 2 * LN, (size_t)np * 3 * LN, 0, B, c.relin.ptr<u64>(),
                   c.cp.relin_bits, c.cp.Dr, ks + (size_t)r0 * 2 * LN);
    }
    launch(c, k_relin_add_shared, blocks((size_t)R * np * 2 * LN, 256), 256, 0, ct3, R, np, (const u64*)ks, c.T, out2);
}

static u64 inv_mod_2n(u64 g, u64 twoN) {
    for (u64 x = 1; x < twoN; x += 2)
        if ((x * g) % twoN == 1) return x;
    throw std::logic_error("no inverse");
}

static const u64* galois_key(Ctx& c, u64 g) {
    for (size_t a = 0; a < c.galois_g.size(); ++a)
        if (c.galois_g[a] == g)
            return c.galois.ptr<u64>() + a * (size_t)c.cp.Dg * 2 * c.cp.L * c.cp.N;
    throw he_err("missing Galois key for requested exponent");
}

/// Expansion levels a_from .. a_to - 1 (expansion.cpp:67-83) of h independent trees whose
/// level-a_from nodes are at cur ([h][2^0 nodes] when a_from is the tree's local root level):
/// node b of the local numbering at level a has children b and b + 2^(a - a_from); the Galois
/// exponent and the monomial shift are those of the global level a.  Returns the buffer holding
/// the level-a_to nodes ([h][2^(a_to - a_from)]).
static u64* expand_levels(Ctx& c, u64* cur, u64* nxt, u32 h, u32 a_from, u32 a_to) {
    const u32 N = c.cp.N, L = c.cp.L;
    const size_t per = 2 * (size_t)L * N;
    const size_t chunk = ks_chunk(c, c.cp.Dg);
    for (u32 a = a_from; a < a_to; ++a) {
        const u64 g = N / (u64(1) << a) + 1;
        const u64 ginv = inv_mod_2n(g, 2 * (u64)N);
        const u64* key = galois_key(c, g);
        const u32 Bq = 1u << (a - a_from);  // nodes per tree at this level
        for (u32 qi = 0; qi < h; ++qi) {
            const u64* in = cur + (size_t)qi * Bq * per;
            u64* out = nxt + (size_t)qi * 2 * Bq * per;
            for (u32 b0 = 0; b0 < Bq; b0 += (u32)chunk) {
                const u32 B = (u32)std::min<size_t>(chunk, Bq - b0);
                u64* ks = c.ks.get<u64>((size_t)B * per);
                key_switch(c, in + (size_t)b0 * per + (size_t)L * N, per, ginv, B, key, c.cp.galois_bits,
                           c.cp.Dg, ks);
                // combine: in/out bases shifted to the chunk, partner offset Bq
                launch(c, k_expand_combine, blocks((size_t)B * L * N, 256), 256, 0, in + (size_t)b0 * per,
                       (const u64*)ks, B, Bq, ginv, (u32)(1u << a), c.T, out + (size_t)b0 * per);
            }
        }
        std::swap(cur, nxt);
    }
    return cur;
}

static void check_expand(const Ctx& c, u32 h, u32 comp, u32 m) {
    if ((u64(1) << comp) > c.cp.N) throw std::invalid_argument("compression factor exceeds log2(N)");
    if ((size_t)h << comp < m) throw std::invalid_argument("packed query too short for code length");
}

/// expand_query (expansion.cpp:67-83): query [h][2][L][N] on device -> entries [h * 2^c].
/// Returns a pointer to the final level buffer (first m entries are the result).
static u64* expand(Ctx& c, const u64* dquery, u32 h, u32 comp, u32 m) {
    check_expand(c, h, comp, m);
    const size_t per = 2 * (size_t)c.cp.L * c.cp.N;
    const size_t full = (size_t)h << comp;
    u64* cur = c.exA.get<u64>(full * per);
    u64* nxt = c.exB.get<u64>(full * per);
    CK(cudaMemcpyAsync(cur, dquery, (size_t)h * per * 8, cudaMemcpyDeviceToDevice, c.st));
    return expand_levels(c, cur, nxt, h, 0, comp);
}

/// Row-sharded expansion (one query ciphertext): the leaves with e = rank (mod W) all descend
/// from node `rank` of level s = log2 W, so a rank runs levels 0 .. s-1 (2^s - 1 switches, the
/// narrow latency-bound top of the tree) and then only its own subtree: 2^(comp - s) leaves,
/// local leaf u = global leaf rank + W u, written to out (device, [2^(comp-s)][2][L][N]).
/// Gathering the W shards rank-major gives every rank all entries (k_unshard reorders them).
static void expand_shard(Ctx& c, const u64* dquery, u32 comp, u32 W, u32 rank, u64* out) {
    u32 s = 0;
    while ((1u << s) < W) ++s;
    if ((1u << s) != W || s > comp) throw std::invalid_argument("shard count must be a power of two <= 2^c");
    if (rank >= W) throw std::invalid_argument("shard rank out of range");
    const size_t per = 2 * (size_t)c.cp.L * c.cp.N;
    const size_t full = (size_t)1 << comp;
    u64* A = c.exA.get<u64>(full * per);
    u64* Bb = c.exB.get<u64>(full * per);
    CK(cudaMemcpyAsync(A, dquery, per * 8, cudaMemcpyDeviceToDevice, c.st));
    u64* top = expand_levels(c, A, Bb, 1, 0, s);
    u64* other = top == A ? Bb : A;
    CK(cudaMemcpyAsync(other, top + (size_t)rank * per, per * 8, cudaMemcpyDeviceToDevice, c.st));
    u64* leaves = expand_levels(c, other, top, 1, s, comp);
    CK(cudaMemcpyAsync(out, leaves, (full / W) * per * 8, cudaMemcpyDefault, c.st));
}

/// MAC basis -> chain (exact centred base conversion): X [G][xs][N] -> out [G][L][N].
static void mac_to_chain(Ctx& c, const u32* X, u32 xs, u32 G, u64* out) {
    const size_t items = (size_t)G * c.cp.N;
    c.next_units = (double)items * c.ab.Mm * c.cp.L;  // residue x constant products
    if (c.m2c_tc && c.m2c_kw) {
        const size_t grid = std::min<size_t>(blocks(items, 128), (size_t)c.n_sms * 4);
        const uint4* Bm = c.m2c_B.ptr<uint4>();
        if (c.m2c_kw == 16 && c.cp.L <= 6) {  // 48 D columns: 64 TMEM columns per CTA, 6 CTAs / SM
            const size_t g6 = std::min<size_t>(blocks(items, 128), (size_t)c.n_sms * 6);
            launch_named(c, "k_mac_to_chain", k_mac_to_chain_tc<16, 48>, g6, 128, 0, X, xs, G, c.T, Bm, out);
        } else if (c.m2c_kw == 16) launch_named(c, "k_mac_to_chain", k_mac_to_chain_tc<16>, grid, 128, 0, X, xs, G, c.T, Bm, out);
        else launch_named(c, "k_mac_to_chain", k_mac_to_chain_tc<24>, grid, 128, 0, X, xs, G, c.T, Bm, out);
        return;
    }
    launch(c, k_mac_to_chain, blocks(items, 128), 128, 0, X, xs, G, c.T, out);
}

// ------------------------------------------------------------------ per-row selection
/// Centred lift of count 2-comp chain ciphertexts into nj aux / MAC residues (to_aux_basis,
/// bfv.cpp:718-744): the tensor-core k_lift_tc when its tables exist, else k_lift.
static void lift(Ctx& c, const u64* src, size_t stride, const u32* sel, u32 count, u32 nj, int mont, u32* out,
                 u32 out_stride_j) {
    const size_t items = (size_t)count * 2 * c.cp.N;
    c.next_units = (double)items * nj;  // coefficient lifts x output primes
    if (c.lift_tc && c.lift_nc && nj <= c.ab.J && reg32_ok(c.cp.logN)) {
        const uint4* Bm = reinterpret_cast<const uint4*>(c.lift_B.ptr<unsigned char>() + (size_t)mont * c.lift_nc * kLiftK);
        const u32* W = c.lift_W2.ptr<u32>() + (size_t)mont * c.ab.J;
        const size_t grid = std::min<size_t>(blocks(items, 128), (size_t)148 * 4);
#define LTC(NCv)                                                                                               \
    if (c.lift_nc == NCv) {                                                                                     \
        launch_named(c, "k_lift", k_lift_tc<NCv>, grid, 128, 0, src, stride, sel, count, nj, c.T, Bm, W, out,   \
                     out_stride_j);                                                                            \
        return;                                                                                                \
    }
        LTC(32) LTC(48) LTC(64) LTC(80) LTC(96) LTC(112)
#undef LTC
    }
    launch(c, k_lift, blocks(items, 256), 256, 0, src, stride, sel, count, nj, mont, c.T, out, out_stride_j);
}

/// Lift count 2-comp chain cts (at src + sel[x]*stride) to the aux basis (Montgomery) and NTT:
/// out [count][2][J][N].
static void prepare(Ctx& c, const u64* src, size_t stride, const u32* sel, u32 count, u32* out) {
    const u32 N = c.cp.N, J = c.ab.J;
    lift(c, src, stride, sel, count, J, 1, out, J);
    ntt32(c, out, count * 2 * J, J, J, 0, false, 0);
}

/// A-side copy of prepared operands with the INTT's output scale (N 2^32)^-1 (A/a_j)^-1 folded
/// in: one pass per query instead of one Shoup product per tensor output coefficient.
static u32* prepare_scaled(Ctx& c, const u32* prep, u32 count, u32* out = nullptr) {
    const u32 N = c.cp.N, J = c.ab.J;
    const size_t total = (size_t)count * 2 * J * N;
    if (!out) out = c.prep_s.get<u32>(total);
    launch(c, k_scale_planes, blocks(total, 256), 256, 0, prep, out, total, c.T.ninvRAc, c.T.ninvRAc_s, c.T);
    return out;
}

/// Tensor + INTT + exact rounding for P products of prepared operands.
/// to_mac: D planes k < Mm become the NTT-form MAC-basis selection values (in c.Dbuf);
/// else the 3-comp chain products are written to chain_out [P][3][L][N].
static bool round_tc_on(const Ctx& c) { return reg32_ok(c.cp.logN) && c.round_kind == 2 && c.rtc_nc != 0; }

/// prepA_scaled: the A operands carry (N 2^32)^-1 (A/a_j)^-1 (see prepare_scaled; tc rounding only).
static u32* mul_prepared(Ctx& c, const u32* prepA, const u32* idxA, const u32* prepB, const u32* idxB, u32 P,
                         bool to_mac, u64* chain_out, bool prepA_scaled = false) {
    const u32 N = c.cp.N, J = c.ab.J;
    u32* D = c.dcur->get<u32>((size_t)P * 3 * c.T.DS * N);
    // tensor-core rounding for both outputs: MAC-basis selection values (to_mac) or, for chain
    // outputs (product-tree nodes, selection ciphertexts), r mod a_k converted to r mod q_i by the
    // exact centred base conversion (the MAC basis M > 2 |r|: choose_aux_basis sizes it for
    // |MAC| >= (t - 1) N |r|), which replaces the per-coefficient multiword k_round_chain
    const bool tc = round_tc_on(c);
    c.zs_last = c.T.DS;
    if (reg32_ok(c.cp.logN)) {
        REG32_DISPATCH(c.cp.logN, tensor(c, prepA, idxA, prepB, idxB, P, D, tc ? (prepA_scaled ? 2 : 1) : 0));
    } else {
        launch(c, k_tensor_intt, (size_t)P * J, ntt_block(N), N * 4, prepA, idxA, prepB, idxB, P, c.T, D);
    }
    if (to_mac || tc) {
        const size_t items = (size_t)P * 3 * N;
        const size_t grid = std::min<size_t>(blocks(items, 256), 148 * 8);
        const size_t sm = sizeof(RoundJ) * c.JM + sizeof(RoundK) * kMaxJ + (size_t)c.ab.Mm * c.JM * 4;
        const RoundJ* rj = c.round_tab.ptr<RoundJ>();
        const RoundK* rk = reinterpret_cast<const RoundK*>(rj + c.JM);
        const u32* im = reinterpret_cast<const u32*>(rk + kMaxJ);
        c.next_units = (double)items;  // coefficients rounded
        if (tc) {
            // the producer warp fills a ring stage with ONE box copy: 128 coefficients x J planes of D[pc][j][n]
            const u64 ddims[3] = {N, c.T.DS, (u64)P * 3};
            const u32 dbox[3] = {128, J, 1};
            const CUtensorMap tmD = tensor_map(D, 3, ddims, dbox);
            const uint4* Bm = c.rtc_B.ptr<uint4>();
            const uint4* B2m = c.round_g2 ? c.rtc_B2.ptr<uint4>() : nullptr;  // null: one-GEMM epilogue
#define RTC(JMv, NCv)                                                                                             \
    if (c.JM == JMv && c.rtc_nc == NCv) {                                                                        \
        {                                                                                                         \
            const size_t gr = std::min<size_t>(items / 128, (size_t)148 * c.round_ctas);                         \
            const auto& rp = *reinterpret_cast<const RoundTcPar<JMv, NCv>*>(c.rtc.data());                        \
            constexpr int LN = JMv == 16 ? 13 : JMv == 8 ? 12 : JMv == 32 ? 14 : 0;                              \
            if (LN == 13 && c.cp.logN == 13 && c.ab.Mm == 11)                                                    \
                launch_named(c, "k_round_tma", k_round_tma<LN, JMv, NCv, 11>, gr, 160, round_tma_smem<JMv>(), D, P,  \
                             c.T, rp, Bm, rk, B2m, tmD);                                                               \
            else if (LN == 13 && c.cp.logN == 13 && c.ab.Mm == 10)                                               \
                launch_named(c, "k_round_tma", k_round_tma<LN, JMv, NCv, 10>, gr, 160, round_tma_smem<JMv>(), D, P,  \
                             c.T, rp, Bm, rk, B2m, tmD);                                                               \
            else if (LN != 0 && c.cp.logN == (u32)LN)                                                             \
                launch_named(c, "k_round_tma", k_round_tma<LN, JMv, NCv>, gr, 160, round_tma_smem<JMv>(), D, P, c.T, \
                             rp, Bm, rk, B2m, tmD);                                                                    \
            else                                                                                                  \
                launch_named(c, "k_round_tma", k_round_tma<0, JMv, NCv>, gr, 160, round_tma_smem<JMv>(), D, P, c.T,  \
                             rp, Bm, rk, B2m, tmD);                                                                    \
        }                                                                                                         \
    }
            RTC(8, 48) RTC(8, 64) RTC(16, 64) RTC(16, 80) RTC(24, 80) RTC(24, 96) RTC(32, 96)
#undef RTC
        } else if (c.JM == 8) launch_named(c, "k_round_mac", k_round_mac_t<8>, grid, 256, sm, D, P, c.T, rj, rk, im);
        else if (c.JM == 16) launch_named(c, "k_round_mac", k_round_mac_t<16>, grid, 256, sm, D, P, c.T, rj, rk, im);
        else if (c.JM == 24) launch_named(c, "k_round_mac", k_round_mac_t<24>, grid, 256, sm, D, P, c.T, rj, rk, im);
        else if (c.JM == 32) launch_named(c, "k_round_mac", k_round_mac_t<32>, grid, 256, sm, D, P, c.T, rj, rk, im);
        else launch_named(c, "k_round_mac", k_round_mac_t<40>, grid, 256, sm, D, P, c.T, rj, rk, im);
        if (!to_mac) {
            mac_to_chain(c, (const u32*)D, c.T.DS, P * 3, chain_out);
        } else if (c.fuse_now) {
            // forward NTT happens inside k_ntt_mac
        } else if (reg32_ok(c.cp.logN)) {
            REG32_DISPATCH(c.cp.logN, sel3(c, D, P, c.T.DS));
        } else {
            ntt32(c, D, P * 3 * c.ab.Mm, c.ab.Mm, c.T.DS, 0, false, 0);
        }
    } else {
        c.next_units = (double)P * 3 * N;  // coefficients rounded
        launch(c, k_round_chain, blocks((size_t)P * 3 * N, 128), 128, 0, (const u32*)D, P, c.T, chain_out);
    }
    return D;
}

/// Selection values for rows [r0, r0+R) of the resident DB.  Returns the Z buffer and sets
/// nc / zstride (Z + ((r*nc + comp)*zstride + k)*N in NTT form, MAC basis).
/// If chain_sel != nullptr the selection ciphertexts are written there instead
/// ([R][3][L][N], comps[r]) and no MAC-basis values are produced (config 2).
static u32* select_tile(Ctx& c, const u64* entries, const u32* prep, u32 op, u64 r0, u32 R, u32& nc, u32& zstride,
                        u64* chain_sel) {
    const u32 N = c.cp.N, L = c.cp.L, J = c.ab.J, Mm = c.ab.Mm, k = c.k;
    const size_t LN = (size_t)L * N;
    const u32* pcol = c.pos_cols.ptr<u32>();
    auto col = [&](u32 p) { return pcol + (size_t)p * c.n_local + r0; };
    if (op == CWG_OP_FOLKLORE && k == 1) {
        if (chain_sel) {  // the expanded entries themselves, 2-comp rows in 3-comp slots
            launch(c, k_gather_strided, blocks((size_t)R * 2 * LN, 256), 256, 0, entries, 2 * LN, col(0), R, 2 * LN,
                   chain_sel, 3 * LN);
            nc = 2;
            return nullptr;
        }
        u32* Z = c.dcur->get<u32>((size_t)R * 2 * Mm * N);  // the tile stream's own buffer
        lift(c, entries, 2 * LN, col(0), R, Mm, 0, Z, Mm);
        if (!c.fuse_now) ntt32(c, Z, R * 2 * Mm, Mm, Mm, 0, false, 0);
        nc = 2;
        zstride = Mm;
        return Z;
    }
    if (op == CWG_OP_FOLKLORE && k == 2) {
        if (chain_sel) {
            mul_prepared(c, prep, col(0), prep, col(1), R, false, chain_sel);
            nc = 3;
            return nullptr;
        }
        u32* D = c.prep_s_ok ? mul_prepared(c, c.prep_s_ptr, col(0), prep, col(1), R, true, nullptr, true)
                             : mul_prepared(c, prep, col(0), prep, col(1), R, true, nullptr);
        nc = 3;
        zstride = c.zs_last;
        return D;
    }
    // ---- general product trees (k >= 3 folklore, arithmetic operator); every index vector and
    // node move is a device kernel (no host round trips inside the tile)
    // nodes: [R][cnt][2][L][N] 2-comp chain ciphertexts, alternating between two buffers
    const size_t per = 2 * LN;
    u32 cnt = 0;
    u64* nodes = nullptr;
    DevBuf* nbuf[2] = {&c.node2, &c.out2};
    int cur = 0;
    const u32* prow = c.pos_rows.ptr<u32>();
    if (op == CWG_OP_FOLKLORE) {
        // leaves: pairs (pos[2p], pos[2p+1]) -> mul_lazy_prepared -> finalize (pir.cpp:294-300)
        const u32 np = k / 2;
        cnt = np + (k % 2);
        u32* di = c.tmp_idx.get<u32>((size_t)2 * R * np);
        launch(c, k_leaf_pairs, blocks((size_t)R * np, 256), 256, 0, prow, r0, R, k, di, di + (size_t)R * np);
        u64* c3 = c.chain3.get<u64>((size_t)R * np * 3 * LN);
        mul_prepared(c, prep, di, prep, di + (size_t)R * np, R * np, false, c3);
        nodes = nbuf[cur]->get<u64>((size_t)R * cnt * per);
        if (k % 2 == 0) {
            relinearize(c, c3, R * np, nodes);  // [R * np] == [R][cnt]
        } else {
            u64* leaf2 = c.resp3.get<u64>((size_t)R * np * per);
            relinearize(c, c3, R * np, leaf2);
            launch(c, k_tree_next, blocks((size_t)R * cnt * per, 256), 256, 0, (const u64*)leaf2, R, np, cnt, entries,
                   (size_t)0, prow, r0, k, per, nodes);
        }
    } else {
        cnt = k;
        nodes = nbuf[cur]->get<u64>((size_t)R * cnt * per);
        launch(c, k_arith_factors, blocks((size_t)R * 2 * LN, 256), 256, 0, entries, prow + (size_t)r0 * k, R, k, c.T,
               nodes);
    }
    const bool lazy_root = (op == CWG_OP_FOLKLORE);
    // arithmetic operator: the root gets plain_mul((k!)^-1) (eq_circuits.cpp:126), fused into the
    // last relinearisation
    u64 kinv = 0;
    if (op == CWG_OP_ARITH) {
        u64 f = 1;
        for (u32 i = 2; i <= k; ++i) f = mulmod64(f, i % c.cp.t, c.cp.t);
        if (f == 0) throw std::invalid_argument("k! is not invertible mod t");
        kinv = invmod64(f, c.cp.t);
    }
    // product_tree (eq_circuits.cpp:53-69)
    bool first = true;
    while (cnt > 1) {
        const bool last = cnt == 2;
        const u32 np = cnt / 2, ncnt = np + (cnt % 2);
        // prepare every node of every row (entries keep their own prepared buffer)
        u32* np_prep = c.lift_tmp.get<u32>((size_t)R * cnt * 2 * J * N);
        if (first && op == CWG_OP_ARITH && c.prep_mode == 1) {
            // the k factors of a row differ from k' only in coefficient 0 of component 0: prepare
            // k' once (lift + NTT) and add each factor's lifted difference to every NTT slot
            u32* pk = c.prep_k.get<u32>((size_t)R * 2 * J * N);
            prepare(c, nodes, (size_t)cnt * per, nullptr, R, pk);
            u32* dl = c.tmp_idx.get<u32>((size_t)R * cnt * J);
            launch(c, k_arith_deltas, blocks((size_t)R * cnt, 128), 128, 0, (const u64*)nodes, R, cnt, c.T, dl);
            launch(c, k_prep_factors, (size_t)R * cnt * 2 * J, 256, 0, (const u32*)pk, (const u32*)dl, cnt, c.T,
                   np_prep);
        } else {
            prepare(c, nodes, per, nullptr, R * cnt, np_prep);
        }
        const bool arith_first = first && op == CWG_OP_ARITH && np > 1 && c.prep_mode == 1;
        first = false;
        u32* di = c.pair_idx.get<u32>((size_t)2 * R * np);
        launch(c, k_level_pairs, blocks((size_t)R * np, 256), 256, 0, R, cnt, di, di + (size_t)R * np);
        if (last && lazy_root) {
            if (chain_sel) {
                mul_prepared(c, np_prep, di, np_prep, di + (size_t)R * np, R, false, chain_sel);
                nc = 3;
                return nullptr;
            }
            u32* D = mul_prepared(c, np_prep, di, np_prep, di + (size_t)R * np, R, true, nullptr);
            nc = 3;
            zstride = c.zs_last;
            return D;
        }
        u64* c3 = c.chain3.get<u64>((size_t)R * np * 3 * LN);
        mul_prepared(c, np_prep, di, np_prep, di + (size_t)R * np, R * np, false, c3);
        u64* nn = nbuf[cur ^ 1]->get<u64>((size_t)R * ncnt * per);
        if (arith_first) {
            // every first-level factor has component 1 = k'_1, so all of a row's first-level
            // products have the same d2 = k'_1 x k'_1, the same rounded c2, and the same key switch:
            // one key switch per row (product 0), added to each product's (c0, c1)
            const size_t LN2 = 2 * LN;
            u64* ks = c.ks.get<u64>((size_t)R * LN2);
            relinearize_shared(c, c3, R, np, ks, cnt % 2 == 0 ? nn : c.resp3.get<u64>((size_t)R * np * per));
            if (cnt % 2)
                launch(c, k_tree_next, blocks((size_t)R * ncnt * per, 256), 256, 0, (const u64*)c.resp3.ptr<u64>(), R, np,
                       ncnt, (const u64*)(nodes + (size_t)(cnt - 1) * per), (size_t)cnt * per, (const u32*)nullptr,
                       (u64)0, 0u, per, nn);
        } else if (cnt % 2 == 0) {
            relinearize(c, c3, R * np, nn, last ? kinv : 0);
        } else {
            u64* rl = c.resp3.get<u64>((size_t)R * np * per);
            relinearize(c, c3, R * np, rl);
            launch(c, k_tree_next, blocks((size_t)R * ncnt * per, 256), 256, 0, (const u64*)rl, R, np, ncnt,
                   (const u64*)(nodes + (size_t)(cnt - 1) * per), (size_t)cnt * per, (const u32*)nullptr, (u64)0, 0u,
                   per, nn);
        }
        nodes = nn;
        cur ^= 1;
        cnt = ncnt;
    }
    // (the arithmetic root's plain_mul((k!)^-1) was applied by the last relinearisation)
    if (chain_sel) {
        launch(c, k_gather_strided, blocks((size_t)R * per, 256), 256, 0, (const u64*)nodes, per, (const u32*)nullptr, R,
               per, chain_sel, 3 * LN);
        nc = 2;
        return nullptr;
    }
    u32* Z = c.dcur->get<u32>((size_t)R * 2 * Mm * N);
    lift(c, (const u64*)nodes, 2 * LN, (const u32*)nullptr, R, Mm, 0, Z, Mm);
    if (!c.fuse_now) ntt32(c, Z, R * 2 * Mm, Mm, Mm, 0, false, 0);
    nc = 2;
    zstride = Mm;
    return Z;
}

static u32 tile_rows(const Ctx& c) {
    // bound the per-tile aux buffer (P x 3 x DS x N u32) to ~256 MB and tree scratch
    // (product trees, k > 2: ~2 GB for the leaf products' D planes; the node, chain-product and
    // prepared-node buffers scale with it, ~12 GB in all at C5)
    const size_t per = (size_t)3 * c.T.DS * c.cp.N * 4 * std::max<u32>(1, c.k / 2);
    size_t r = std::max<size_t>(4, (size_t(c.k > 2 ? 2048 : 256) << 20) / per);
    if (c.tile_rows_opt) return (u32)std::min<size_t>(c.tile_rows_opt, 2048);
    // rows of many plaintexts (whole-row payload MAC, k_mac_rows): large tiles keep its work items long
    // (C3: 1,024-row tiles, 15.0 vs 18.4 ms of MAC per answer at 182 rows)
    if (c.k <= 2 && c.s >= 3) return (u32)std::min<size_t>(std::max<size_t>(4, (size_t(1536) << 20) / per), 1024);
    return (u32)std::min<size_t>(r, 512);
}

// ------------------------------------------------------------------ answer
struct Timer {
    Ctx& c;
    bool on;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    Timer(Ctx& cc, bool enabled) : c(cc), on(enabled) {}
    ~Timer() {
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
    void mark(int tag) {
        if (!on) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, c.st));
        marks.push_back({tag, e});
    }
    /// sum of elapsed times over consecutive marks whose END mark carries `tag`
    double sum(int tag) const {
        double s = 0;
        for (size_t i = 1; i < marks.size(); ++i) {
            if (marks[i].first != tag) continue;
            float f = 0;
            CK(cudaEventElapsedTime(&f, marks[i - 1].second, marks[i].second));
            s += f;
        }
        return s;
    }
};
enum { TM_START = 0, TM_H2D, TM_EXPAND, TM_SELECT, TM_MAC, TM_FINISH, TM_D2H };

/// Evaluation keys for this call (EvalKeySet, bfv.hpp:42-51; the reference server receives them
/// with every query, server.cpp:61-87).  Device key cache: when a key set of the same shape is
/// resident, the upload goes to a staging buffer and is compared word for word on the device;
/// identical keys keep the resident copy and its aux-basis transform (key_to_aux, ~2 ms at C4),
/// different keys replace it.  Returns true when the resident keys were reused.
static bool upload_keys(Ctx& c, const u64* relin, u32 n_galois, const u64* gg, const u64* galois) {
    Nvtx nv("cwgpu keys");
    const size_t LN = (size_t)c.cp.L * c.cp.N;
    const size_t rw = (size_t)c.cp.Dr * 2 * LN, gw = (size_t)c.cp.Dg * 2 * LN;
    const bool same_shape = c.have_keys && c.galois_g.size() == n_galois &&
                            std::equal(c.galois_g.begin(), c.galois_g.end(), gg);
    if (!same_shape) {
        CK(cudaMemcpyAsync(c.relin.get<u64>(rw), relin, rw * 8, cudaMemcpyDefault, c.st));
        if (n_galois)
            CK(cudaMemcpyAsync(c.galois.get<u64>(gw * n_galois), galois, gw * n_galois * 8, cudaMemcpyDefault, c.st));
        c.galois_g.assign(gg, gg + n_galois);
        c.have_keys = true;
        c.ksA_ok = false;
        return false;
    }
    const size_t gall = gw * n_galois;
    u64* stage = c.key_stage.get<u64>(rw + gall);
    CK(cudaMemcpyAsync(stage, relin, rw * 8, cudaMemcpyDefault, c.st));
    if (n_galois) CK(cudaMemcpyAsync(stage + rw, galois, gall * 8, cudaMemcpyDefault, c.st));
    unsigned int* flag = c.key_flag.get<unsigned int>(1);
    CK(cudaMemsetAsync(flag, 0, 4, c.st));
    launch(c, k_words_differ, 148 * 8, 256, 0, (const u64*)stage, (const u64*)c.relin.ptr<u64>(), rw, flag);
    if (n_galois)
        launch(c, k_words_differ, 148 * 8, 256, 0, (const u64*)(stage + rw), (const u64*)c.galois.ptr<u64>(), gall, flag);
    unsigned int differ = 1;
    CK(cudaMemcpyAsync(&differ, flag, 4, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (!differ) return true;
    CK(cudaMemcpyAsync(c.relin.ptr<u64>(), stage, rw * 8, cudaMemcpyDeviceToDevice, c.st));
    if (n_galois) CK(cudaMemcpyAsync(c.galois.ptr<u64>(), stage + rw, gall * 8, cudaMemcpyDeviceToDevice, c.st));
    c.ksA_ok = false;
    return false;
}

/// expand + select + MAC; leaves the reduced partial accumulators [s][3][Mm][N] u64
/// in dev_partial; returns the response component count (2 or 3).
static u32 answer_partial(Ctx& c, u32 h, u32 comp, u32 m, const u64* query, u32 op, u64* dev_partial, Timer& tm,
                          const u64* shards = nullptr, u32 W = 0) {
    if (!c.db_loaded) throw state_err("no database loaded");
    if (m != c.m) throw std::invalid_argument("query code length does not match the database");  // pir.cpp:339-341
    if (c.s == 0) throw state_err("database has no payload (selection-only); use cwg_select");
    if (!c.have_keys) throw he_err("evaluation keys not set");
    if (op != CWG_OP_FOLKLORE && op != CWG_OP_ARITH) throw std::invalid_argument("unknown equality operator");
    if (op == CWG_OP_ARITH && c.k < 2) throw std::invalid_argument("arithmetic operator needs k >= 2");
    const u32 N = c.cp.N, L = c.cp.L, J = c.ab.J, Mm = c.ab.Mm;
    const size_t LN = (size_t)L * N;
    CK(cudaMemsetAsync(c.d_fb, 0, 8, c.st));  // exact-path counter: per answer (cwg_timings.exact_fallbacks)
    u64* entries = nullptr;
    if (shards) {  // entries expanded by W ranks (expand_shard) and gathered rank-major
        check_expand(c, 1, comp, m);
        tm.mark(TM_H2D);
        const size_t full = (size_t)1 << comp;
        entries = c.exA.get<u64>(full * 2 * LN);
        launch(c, k_unshard, blocks((size_t)m * 2 * LN, 256), 256, 0, shards, (u32)m, W, (u32)(full / W), 2 * LN,
               entries);
        tm.mark(TM_EXPAND);
    } else {
        u64* dq = c.query.get<u64>((size_t)h * 2 * LN);
        CK(cudaMemcpyAsync(dq, query, (size_t)h * 2 * LN * 8, cudaMemcpyDefault, c.st));  // host or device
        tm.mark(TM_H2D);
        {
            Nvtx nv("cwgpu expand_query");
            entries = expand(c, dq, h, comp, m);
        }
        tm.mark(TM_EXPAND);
    }
    u32* prep = nullptr;
    c.prep_s_ok = false;
    if (op == CWG_OP_FOLKLORE && c.k >= 2) {
        prep = c.prep.get<u32>((size_t)m * 2 * J * N);
        prepare(c, entries, 2 * LN, nullptr, m, prep);
        if (c.k == 2 && round_tc_on(c) && c.prescale) {
            c.prep_s_ptr = prepare_scaled(c, prep, m);
            c.prep_s_ok = true;
        }
    }
    const size_t accw = (size_t)c.s * 3 * Mm * N;
    auto* acc = reinterpret_cast<unsigned long long*>(c.acc_lo.get<u64>(accw));
    CK(cudaMemsetAsync(acc, 0, accw * 8, c.st));
    const u32 R = tile_rows(c);
    u32 nc_all = 2;
    // profiling serialises the tile pipeline: per-kernel CUDA-event times then measure each kernel
    // alone (as ncu's launch list does) instead of its overlap with the other stream's kernels
    const int ns = c.profiling ? 1 : (int)std::min<u64>((u64)c.nstreams, (c.n_local + R - 1) / R);
    const bool piped = ns >= 2 && op == CWG_OP_FOLKLORE && c.k <= 2;
    cudaStream_t main_st = c.st;
    if (piped) {
        // all D buffers exist before the streams diverge (allocation synchronises)
        c.Dbuf.ensure((size_t)R * 3 * c.T.DS * N * 4);
        for (int i = 1; i < ns; ++i) c.Dmore[i - 1].ensure((size_t)R * 3 * c.T.DS * N * 4);
        CK(cudaEventRecord(c.tev[0], main_st));
        for (int i = 0; i < ns; ++i) CK(cudaStreamWaitEvent(c.tst[i], c.tev[0], 0));
    }
    c.fuse_now = c.fuse_mac != 0 && reg32_ok(c.cp.logN) && c.s <= 2;
    // restores the context's stream / D buffer and the fuse flag on every exit, including an
    // exception thrown inside the tile loop (the main stream then waits for the tile streams, so
    // callers that captured cwg_stream() stay ordered after all of this answer's work)
    struct PipeGuard {
        Ctx& c;
        cudaStream_t main_st;
        int ns;
        bool piped;
        ~PipeGuard() {
            c.fuse_now = false;
            if (!piped) return;
            c.st = main_st;
            c.dcur = &c.Dbuf;
            for (int i = 0; i < ns; ++i)
                if (cudaEventRecord(c.tev[1 + i], c.tst[i]) == cudaSuccess) cudaStreamWaitEvent(main_st, c.tev[1 + i], 0);
        }
    } pipe_guard{c, main_st, ns, piped};
    u64 tile = 0;
    for (u64 r0 = 0; r0 < c.n_local; r0 += R, ++tile) {
        const u32 Rt = (u32)std::min<u64>(R, c.n_local - r0);
        if (piped) {
            const int i = (int)(tile % (u64)ns);
            c.st = c.tst[i];
            c.dcur = i ? &c.Dmore[i - 1] : &c.Dbuf;
        }
        u32 nc = 0, zs = 0;
        Nvtx nv("cwgpu row tile");
        u32* Z = select_tile(c, entries, prep, op, r0, Rt, nc, zs, nullptr);
        nc_all = std::max(nc_all, nc);
        tm.mark(TM_SELECT);
        // rows per chunk: enough threads to cover the GPU several times, >= 16 rows each
        const size_t per_chunk_threads = (size_t)c.s * Mm * (N / 4);
        u32 chunks = (u32)std::max<size_t>(1, std::min<size_t>((size_t)(Rt + 15) / 16, (148 * 2048 * 2) / per_chunk_threads + 1));
        const u32 chunk = (Rt + chunks - 1) / chunks;
        chunks = (Rt + chunk - 1) / chunk;
        const u32* dbt = c.db.ptr<u32>() + (size_t)r0 * c.s * Mm * N;
        const size_t threads = (size_t)c.s * Mm * ((N / 4 + 255) / 256) * 256 * chunks;
        c.next_units = (double)Rt * (c.s + nc) * Mm * N * 4;  // DB + selection words streamed
        // TMA ring for multi-plaintext rows (C3: 37 vs 45 ms; the selection segments are reused
        // across the s payload slices); the register stream is as fast for s = 1 (C4: 22.9 ms)
        if (c.fuse_now) {
            REG32_DISPATCH(c.cp.logN, ntt_mac(c, Z, zs, nc, dbt, Rt, acc));
        } else if (c.mac_rows && c.mac_tma && (c.s == 15 || c.s == 5 || c.s == 3) && N >= (u32)kMacBlockS) {
            // whole rows per CTA: every selection word is fetched once per row (persistent CTAs, work
            // items from a global counter)
            const u32 ck = std::max<u32>(1, (Rt + c.mac_item_rows / 2) / std::max<u32>(1, c.mac_item_rows));
            const u32 crow = (Rt + ck - 1) / ck;
            const u32 nch = (Rt + crow - 1) / crow;
            const u32 items = nch * Mm * (N / kMacBlockS);
            c.mac_ctr.ensure(64 * sizeof(u32));
            u32* ctr = c.mac_ctr.ptr<u32>() + (c.mac_ctr_next++ % 64);
            CK(cudaMemsetAsync(ctr, 0, sizeof(u32), c.st));
            const size_t grid = std::min<size_t>(items, (size_t)c.n_sms);
            // 4-D views [row][slice or component][prime plane][coefficient] of the tile's database rows
            // and selection planes; one box per ring stage each
            const CUtensorMap tmDB = tensor_map4(dbt, N, Mm, c.s, Rt, kMacBlockS, c.s);
            const CUtensorMap tmZ = tensor_map4(Z, N, zs, nc, Rt, kMacBlockS, nc);
#define MAC_ROWS(NCv, SGv)                                                                                         \
    if (nc == NCv && c.s == SGv) {                                                                                 \
        constexpr int STv = SGv == 15 ? 10 : 16;                                                                   \
        launch_named(c, "k_mac", k_mac_rows<NCv, SGv, STv>, grid, 288, (size_t)STv*(SGv + NCv) * kMacBlockS * 4,   \
                     tmDB, tmZ, Rt, crow, nch, c.T, acc, ctr);                                                     \
    }
            MAC_ROWS(3, 15) MAC_ROWS(2, 15) MAC_ROWS(3, 5) MAC_ROWS(2, 5) MAC_ROWS(3, 3) MAC_ROWS(2, 3)
#undef MAC_ROWS
        } else if (c.mac_sg && c.s >= 3 && (c.s % 5 == 0 || c.s % 3 == 0) && N >= (u32)kMacBlockQ) {
            // several payload slices per CTA: the row's selection segments are read once per SG slices
            const u32 SG = c.s % 3 == 0 ? 3 : 5;
            ZPtrs zp{};
            zp.z[0] = Z;
            zp.acc[0] = acc;
            const u32 blocksN = Mm * (N / kMacBlockQ) * (c.s / SG);
            const u32 slots = 148 * 2 * 2;
            u32 ck = std::max<u32>(1, std::min<u32>((Rt + 7) / 8, slots / blocksN));
            const u32 crow = (Rt + ck - 1) / ck;
            ck = (Rt + crow - 1) / crow;
            const size_t smem = (size_t)(c.mac_stages8 ? 8 : kMacStages) * (SG + nc) * kMacBlockQ * 4;
            if (SG == 3 && c.mac_stages8) {
                if (nc == 3) launch_named(c, "k_mac", k_mac_tma_q<3, 1, 3, 8>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
                else launch_named(c, "k_mac", k_mac_tma_q<2, 1, 3, 8>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
            } else if (SG == 5) {
                if (nc == 3) launch_named(c, "k_mac", k_mac_tma_q<3, 1, 5>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
                else launch_named(c, "k_mac", k_mac_tma_q<2, 1, 5>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
            } else {
                if (nc == 3) launch_named(c, "k_mac", k_mac_tma_q<3, 1, 3>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
                else launch_named(c, "k_mac", k_mac_tma_q<2, 1, 3>, (size_t)ck * blocksN, 288, smem, zp, zs, dbt, Rt, c.s, crow, c.T);
            }
        } else if (c.mac_tma && c.s >= 2 && N >= (u32)kMacBlock) {
            // TMA-fed stream: whole waves of 3 CTAs / SM (no partial tail wave), >= 8 rows per chunk
            const u32 per = Mm * (N / kMacBlock) * c.s;
            const u32 slots = 148 * 3 * (c.mac_waves > 0 ? c.mac_waves : 2);
            u32 ck = std::max<u32>(1, std::min<u32>((Rt + 7) / 8, slots / per));
            const u32 crow = (Rt + ck - 1) / ck;
            ck = (Rt + crow - 1) / crow;
            const size_t smem = (size_t)kMacStages * (1 + nc) * kMacBlock * 4;
            if (nc == 3)
                launch_named(c, "k_mac", k_mac_tma<3>, (size_t)ck * per, 288, smem, (const u32*)Z, zs, dbt, Rt, c.s,
                             crow, c.T, acc);
            else
                launch_named(c, "k_mac", k_mac_tma<2>, (size_t)ck * per, 288, smem, (const u32*)Z, zs, dbt, Rt, c.s,
                             crow, c.T, acc);
        } else if (nc == 3)
            launch_named(c, "k_mac", k_mac2<3>, blocks(threads, 256), 256, 0, (const u32*)Z, zs, dbt, Rt, c.s, chunk,
                         c.T, acc);
        else
            launch_named(c, "k_mac", k_mac2<2>, blocks(threads, 256), 256, 0, (const u32*)Z, zs, dbt, Rt, c.s, chunk,
                         c.T, acc);
        tm.mark(TM_MAC);
    }
    if (piped) {
        pipe_guard.piped = false;
        c.st = main_st;
        c.dcur = &c.Dbuf;
        for (int i = 0; i < ns; ++i) {
            CK(cudaEventRecord(c.tev[1 + i], c.tst[i]));
            CK(cudaStreamWaitEvent(main_st, c.tev[1 + i], 0));
        }
    }
    launch(c, k_acc_mod, blocks(accw, 256), 256, 0, (const unsigned long long*)acc, accw, c.T, dev_partial);
    tm.mark(TM_MAC);
    return nc_all;
}

static void finish(Ctx& c, const u64* dev_partial, u32 nc, u64* out_host, Timer& tm);

/// Multi-query answer (the reference answers one query per process_query,
/// pir.cpp:337-347): Q queries under one evaluation-key set, each expanded and prepared once, then
/// per row tile every query's selection is computed and the payload MAC reads the tile's database
/// planes once for all of them (k_mac_tma_q for s >= 2 rows; the fused selection NTT + MAC of s <= 2
/// rows streams the database per query, where it is a small part of the cost).  out: [Q][s][2][L][N].
static void answer_batch(Ctx& c, u32 Q, u32 h, u32 comp, u32 m, const u64* queries, u32 op, u64* out, Timer& tm) {
    if (!c.db_loaded) throw state_err("no database loaded");
    if (m != c.m) throw std::invalid_argument("query code length does not match the database");  // pir.cpp:339-341
    if (c.s == 0) throw state_err("database has no payload (selection-only); use cwg_select");
    if (!c.have_keys) throw he_err("evaluation keys not set");
    if (op != CWG_OP_FOLKLORE && op != CWG_OP_ARITH) throw std::invalid_argument("unknown equality operator");
    if (op == CWG_OP_ARITH && c.k < 2) throw std::invalid_argument("arithmetic operator needs k >= 2");
    if (Q == 0) throw std::invalid_argument("empty query batch");
    const u32 N = c.cp.N, L = c.cp.L, J = c.ab.J, Mm = c.ab.Mm;
    const size_t LN = (size_t)L * N;
    const size_t per = 2 * LN;
    CK(cudaMemsetAsync(c.d_fb, 0, 8, c.st));
    auto grow = [](std::vector<std::unique_ptr<DevBuf>>& v, u32 n) {
        while (v.size() < n) v.push_back(std::make_unique<DevBuf>());
    };
    grow(c.bq_ent, Q);
    grow(c.bq_prep, Q);
    grow(c.bq_preps, Q);
    grow(c.bq_D, Q);
    const bool folk = op == CWG_OP_FOLKLORE && c.k >= 2;
    const bool scaled = c.k == 2 && folk && round_tc_on(c) && c.prescale;
    // 1. expansion + preparation of every query (expand_query, prepare_cipher)
    for (u32 q = 0; q < Q; ++q) {
        Nvtx nv("cwgpu expand_query");
        u64* dq = c.query.get<u64>((size_t)h * per);
        CK(cudaMemcpyAsync(dq, queries + (size_t)q * h * per, (size_t)h * per * 8, cudaMemcpyDefault, c.st));
        const u64* e = expand(c, dq, h, comp, m);
        u64* ent = c.bq_ent[q]->get<u64>((size_t)m * per);
        CK(cudaMemcpyAsync(ent, e, (size_t)m * per * 8, cudaMemcpyDeviceToDevice, c.st));
        if (folk) {
            u32* pr = c.bq_prep[q]->get<u32>((size_t)m * 2 * J * N);
            prepare(c, ent, per, nullptr, m, pr);
            if (scaled) prepare_scaled(c, pr, m, c.bq_preps[q]->get<u32>((size_t)m * 2 * J * N));
        }
    }
    tm.mark(TM_EXPAND);
    const size_t accw = (size_t)c.s * 3 * Mm * N;
    auto* acc = reinterpret_cast<unsigned long long*>(c.bq_acc.get<u64>(accw * Q));
    CK(cudaMemsetAsync(acc, 0, accw * Q * 8, c.st));
    const u32 R = tile_rows(c);
    c.fuse_now = c.fuse_mac != 0 && reg32_ok(c.cp.logN) && c.s <= 2;
    struct Reset {
        Ctx& c;
        ~Reset() {
            c.fuse_now = false;
            c.prep_s_ok = false;
            c.dcur = &c.Dbuf;
        }
    } reset{c};
    u32 nc_all = 2;
    std::vector<u32*> Z(Q);
    std::vector<u32> zst(Q);
    for (u64 r0 = 0; r0 < c.n_local; r0 += R) {
        Nvtx nv("cwgpu row tile (batch)");
        const u32 Rt = (u32)std::min<u64>(R, c.n_local - r0);
        u32 nc = 0;
        for (u32 q = 0; q < Q; ++q) {  // 2. every query's selection values for the tile
            c.dcur = c.bq_D[q].get();
            c.prep_s_ok = scaled;
            c.prep_s_ptr = scaled ? c.bq_preps[q]->ptr<u32>() : nullptr;
            Z[q] = select_tile(c, c.bq_ent[q]->ptr<u64>(), folk ? c.bq_prep[q]->ptr<u32>() : nullptr, op, r0, Rt, nc,
                               zst[q], nullptr);
        }
        nc_all = std::max(nc_all, nc);
        tm.mark(TM_SELECT);
        const u32* dbt = c.db.ptr<u32>() + (size_t)r0 * c.s * Mm * N;
        if (c.fuse_now) {  // 3a. fused selection NTT + MAC per query
            for (u32 q = 0; q < Q; ++q) REG32_DISPATCH(c.cp.logN, ntt_mac(c, Z[q], zst[q], nc, dbt, Rt, acc + q * accw));
        } else if (c.mac_tma && N >= (u32)kMacBlockQ) {  // 3b. one database pass per group of <= 4 queries
            for (u32 q0 = 0; q0 < Q; q0 += 4) {
                const u32 qb = std::min<u32>(4, Q - q0);
                ZPtrs zp{};
                for (u32 x = 0; x < qb; ++x) {
                    if (zst[q0 + x] != zst[q0]) throw std::logic_error("batch selection strides differ");
                    zp.z[x] = Z[q0 + x];
                    zp.acc[x] = acc + (q0 + x) * accw;
                }
                const u32 blocksN = Mm * (N / kMacBlockQ) * c.s;  // SG = 1
                const u32 slots = 148 * 2 * 2;
                u32 ck = std::max<u32>(1, std::min<u32>((Rt + 7) / 8, slots / blocksN));
                const u32 crow = (Rt + ck - 1) / ck;
                ck = (Rt + crow - 1) / crow;
                const size_t smem = (size_t)kMacStages * (1 + qb * nc) * kMacBlockQ * 4;
                c.next_units = (double)Rt * (c.s + (double)qb * nc) * Mm * N * 4;  // DB once + qb selections
#define MACQ(NCv, QBv)                                                                                            \
    launch_named(c, "k_mac_q", k_mac_tma_q<NCv, QBv, 1>, (size_t)ck * blocksN, 288, smem, zp, zst[q0], dbt, Rt,   \
                 c.s, crow, c.T)
                if (nc == 3) {
                    if (qb == 1) MACQ(3, 1); else if (qb == 2) MACQ(3, 2); else if (qb == 3) MACQ(3, 3); else MACQ(3, 4);
                } else {
                    if (qb == 1) MACQ(2, 1); else if (qb == 2) MACQ(2, 2); else if (qb == 3) MACQ(2, 3); else MACQ(2, 4);
                }
#undef MACQ
            }
        } else {
            for (u32 q = 0; q < Q; ++q) {
                const u32 chunks = (u32)std::max<size_t>(1, std::min<size_t>((size_t)(Rt + 15) / 16,
                                                                             (148 * 2048 * 2) / ((size_t)c.s * Mm * (N / 4)) + 1));
                const u32 chunk = (Rt + chunks - 1) / chunks;
                const size_t threads = (size_t)c.s * Mm * ((N / 4 + 255) / 256) * 256 * ((Rt + chunk - 1) / chunk);
                if (nc == 3)
                    launch_named(c, "k_mac", k_mac2<3>, blocks(threads, 256), 256, 0, (const u32*)Z[q], zst[q], dbt, Rt,
                                 c.s, chunk, c.T, acc + q * accw);
                else
                    launch_named(c, "k_mac", k_mac2<2>, blocks(threads, 256), 256, 0, (const u32*)Z[q], zst[q], dbt, Rt,
                                 c.s, chunk, c.T, acc + q * accw);
            }
        }
        tm.mark(TM_MAC);
    }
    // 4. finalize every query's response
    u64* part = c.partial.get<u64>(accw);
    for (u32 q = 0; q < Q; ++q) {
        launch(c, k_acc_mod, blocks(accw, 256), 256, 0, (const unsigned long long*)(acc + q * accw), accw, c.T, part);
        finish(c, part, nc_all, out + (size_t)q * c.s * per, tm);
    }
}

/// summed partials -> responses: mod a_k, INTT, M -> chain, finalize (pir.cpp:345).
static void finish(Ctx& c, const u64* dev_partial, u32 nc, u64* out_host, Timer& tm) {
    Nvtx nv("cwgpu finalize");
    const u32 N = c.cp.N, L = c.cp.L, Mm = c.ab.Mm;
    const size_t LN = (size_t)L * N;
    const size_t accw = (size_t)c.s * 3 * Mm * N;
    u32* X = c.X.get<u32>(accw);
    launch(c, k_partial_mod, blocks(accw, 256), 256, 0, dev_partial, accw, c.T, X);
    ntt32(c, X, c.s * 3 * Mm, Mm, Mm, 0, true, 0);
    u64* r3 = c.resp3.get<u64>((size_t)c.s * 3 * LN);
    c.next_units = (double)c.s * 3 * N * Mm * L;
    mac_to_chain(c, (const u32*)X, Mm, c.s * 3, r3);
    u64* o2 = c.out2.get<u64>((size_t)c.s * 2 * LN);
    if (nc == 3) {
        relinearize(c, r3, c.s, o2);
    } else {
        for (u32 j = 0; j < c.s; ++j)
            CK(cudaMemcpyAsync(o2 + (size_t)j * 2 * LN, r3 + (size_t)j * 3 * LN, 2 * LN * 8, cudaMemcpyDeviceToDevice,
                               c.st));
    }
    tm.mark(TM_FINISH);
    CK(cudaMemcpyAsync(out_host, o2, (size_t)c.s * 2 * LN * 8, cudaMemcpyDefault, c.st));  // host or device
    CK(cudaStreamSynchronize(c.st));
    tm.mark(TM_D2H);
}

static void fill_timings(Ctx& c, Timer& tm, cwg_timings* t, double total_ms) {
    CK(cudaStreamSynchronize(c.st));
    if (c.profiling) prof_collect(c);
    if (!t) return;
    t->total_ms = total_ms;
    t->h2d_ms = tm.sum(TM_H2D);
    t->expand_ms = tm.sum(TM_EXPAND);
    t->select_ms = tm.sum(TM_SELECT);
    t->mac_ms = tm.sum(TM_MAC);
    t->finish_ms = tm.sum(TM_FINISH);
    t->d2h_ms = tm.sum(TM_D2H);
    t->kernel_launches = c.launches;
    unsigned long long fb = 0;
    CK(cudaMemcpy(&fb, c.d_fb, 8, cudaMemcpyDeviceToHost));
    t->exact_fallbacks = fb;
    t->keys_cached = c.keys_cached ? 1u : 0u;
    t->n_devices = 1;
}

// ------------------------------------------------------------------ database
/// Common part of cwg_load_db / cwg_load_db_bytes: positions (host, [n_local][k]) checked and made
/// resident; `fill(r0, R, stage)` writes rows [r0, r0+R)'s plaintext coefficients (< t) as u64
/// [R][s][N] into the device staging buffer, which is lifted to the MAC basis and NTT'd.
static void load_db_impl(Ctx& c, u64 n_total, u64 row_begin, u64 n_local, u32 s, u32 k, u32 m, const u32* positions,
                         const std::function<void(u64, u64, u64*)>& fill) {
    Nvtx nv("cwgpu load_db");
    if (n_local == 0 || n_total == 0) throw std::invalid_argument("empty database");
    if (row_begin + n_local > n_total) throw std::invalid_argument("row range outside the database");
    if (k < 1) throw std::invalid_argument("hamming weight must be >= 1");
    if (k > 64) throw std::invalid_argument("cwgpu: hamming weight above 64 is not supported");
    if (c.cp.t <= k) throw std::invalid_argument("plaintext modulus must exceed the Hamming weight");
    const u32 N = c.cp.N;
    for (u64 r = 0; r < n_local; ++r) {
        for (u32 p = 0; p < k; ++p) {
            const u32 v = positions[r * k + p];
            if (v >= m) throw std::invalid_argument("codeword position outside the code length");
            if (p && v <= positions[r * k + p - 1]) throw std::invalid_argument("codeword positions must ascend");
        }
    }
    c.db_loaded = false;  // set again only after the upload and the stream sync succeed
    ensure_aux(c, n_total);
    const u32 Mm = c.ab.Mm;
    c.n_total = n_total;
    c.row_begin = row_begin;
    c.n_local = n_local;
    c.s = s;
    c.k = k;
    c.m = m;
    std::vector<u32> cols((size_t)k * n_local);
    for (u64 r = 0; r < n_local; ++r)
        for (u32 p = 0; p < k; ++p) cols[(size_t)p * n_local + r] = positions[r * k + p];
    CK(cudaMemcpy(c.pos_rows.get<u32>(n_local * k), positions, n_local * k * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.pos_cols.get<u32>(n_local * k), cols.data(), cols.size() * 4, cudaMemcpyHostToDevice));
    if (s > 0) {
        // prepare_plain (bfv.cpp:933-942) into the MAC basis: coefficients < t lifted unchanged,
        // NTT per MAC prime; staged in chunks of rows.
        u32* dbp = c.db.get<u32>(n_local * s * Mm * N);
        const u64 chunk = std::max<u64>(1, (u64(256) << 20) / ((u64)s * N * 8));
        u64* stage = c.chain3.get<u64>(std::min(chunk, n_local) * s * N);
        for (u64 r0 = 0; r0 < n_local; r0 += chunk) {
            const u64 R = std::min(chunk, n_local - r0);
            fill(r0, R, stage);
            u32* dst = dbp + r0 * s * Mm * N;
            launch(c, k_db_spread, blocks(R * s * Mm * N, 256), 256, 0, (const u64*)stage, R * s, c.T, dst);
            ntt32(c, dst, (u32)(R * s * Mm), Mm, Mm, 0, false, 0);
        }
    }
    CK(cudaStreamSynchronize(c.st));
    c.db_loaded = true;
}

static void load_db(Ctx& c, u64 n_total, u64 row_begin, u64 n_local, u32 s, u32 k, u32 m, const u32* positions,
                    const u64* payload) {
    if (s > 0 && !payload) throw std::invalid_argument("payload missing");
    const u32 N = c.cp.N;
    if (s > 0)
        for (u64 i = 0; i < n_local * s * N; ++i)
            if (payload[i] >= c.cp.t) throw std::invalid_argument("plain operand not reduced mod t");
    load_db_impl(c, n_total, row_begin, n_local, s, k, m, positions, [&](u64 r0, u64 R, u64* stage) {
        CK(cudaMemcpyAsync(stage, payload + r0 * s * N, R * s * N * 8, cudaMemcpyHostToDevice, c.st));
    });
}

/// PirDatabase::setup + prepare_for from raw rows (pir.cpp:214-264): codewords by perfect_map of
/// the row ids on the device (index mode: the global row index, map_index pir.cpp:149-153;
/// keyword mode: keyword_value of the row's key, pir.cpp:22-30 / 155-159, computed by the
/// caller), payloads chunked on the device (chunk_payload, pir.cpp:169-193: s plaintexts of
/// floor(log2 t)-bit coefficients, s = max(1, ceil(8 bytes / (N b))), pir.cpp:39-43).
static void load_db_bytes(Ctx& c, u64 n_total, u64 row_begin, u64 n_local, u32 k, u32 m, u64 payload_bytes,
                          const unsigned char* payloads, const u64* row_ids) {
    if (n_local == 0 || n_total == 0) throw std::invalid_argument("empty database");
    if (!payloads || payload_bytes == 0) throw std::invalid_argument("payload missing");
    if (k < 1) throw std::invalid_argument("hamming weight must be >= 1");
    if (k > 64) throw std::invalid_argument("cwgpu: hamming weight above 64 is not supported");
    const u32 N = c.cp.N;
    u32 b = 0;
    while (b < 63 && (u64(1) << (b + 1)) <= c.cp.t) ++b;  // plain_bits_per_coeff (he.cpp:17-21)
    const u64 cap_bits = (u64)N * b;
    const u32 s = (u32)std::max<u64>(1, (payload_bytes * 8 + cap_bits - 1) / cap_bits);
    // code capacity C(m, k) and the largest binomial the device unranking touches, C(m-1, j <= k)
    auto binom = [](u32 n, u32 r) {  // C(n, r), saturating at 2^90 (products stay below 2^122)
        if (r > n) return (u128)0;
        u128 v = 1;
        for (u32 j = 1; j <= r; ++j) {
            if (v >> 90) return ((u128)1) << 90;
            v = v * (n - r + j) / j;  // exact: C(n-r+j, j) = C(n-r+j-1, j-1) (n-r+j) / j
        }
        return v;
    };
    const u128 cap = binom(m, k);
    u128 big = 0;
    for (u32 j = 0; j <= k; ++j) big = std::max(big, binom(m - 1, j));
    if (big >> 64) throw std::invalid_argument("cwgpu: code capacity above 2^64 is not supported");
    std::vector<u64> ids(n_local);
    for (u64 r = 0; r < n_local; ++r) {
        ids[r] = row_ids ? row_ids[r] : row_begin + r;
        if ((u128)ids[r] >= cap) throw std::invalid_argument("perfect_map: input out of range");
    }
    if (row_ids) {
        std::vector<u64> srt(ids);
        std::sort(srt.begin(), srt.end());
        if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) throw std::invalid_argument("duplicate identifier");
    }
    for (u64 r = 0; r < n_local; ++r) {  // pir.cpp:231-235
        const unsigned char* p = payloads + r * payload_bytes;
        if (std::all_of(p, p + payload_bytes, [](unsigned char x) { return x == 0; }))
            throw std::invalid_argument("all-zero payloads are reserved for the absent-keyword sentinel");
    }
    u64* dids = c.tmp_idx.get<u64>(n_local);
    u32* dpos = c.digits.get<u32>(n_local * k);
    CK(cudaMemcpyAsync(dids, ids.data(), n_local * 8, cudaMemcpyHostToDevice, c.st));
    launch(c, k_perfect_map, blocks(n_local, 128), 128, 0, (const u64*)dids, n_local, m, k, dpos);
    std::vector<u32> pos(n_local * k);
    CK(cudaMemcpyAsync(pos.data(), dpos, pos.size() * 4, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    unsigned char* dbytes = nullptr;
    load_db_impl(c, n_total, row_begin, n_local, s, k, m, pos.data(), [&](u64 r0, u64 R, u64* stage) {
        dbytes = reinterpret_cast<unsigned char*>(c.lift_tmp.get<u32>((R * payload_bytes + 3) / 4));
        CK(cudaMemcpyAsync(dbytes, payloads + r0 * payload_bytes, R * payload_bytes, cudaMemcpyDefault, c.st));
        launch(c, k_chunk_payload, blocks(R * s * N, 256), 256, 0, (const unsigned char*)dbytes, R, payload_bytes, s,
               N, b, stage);
    });
}

/// compute_selection_vector (pir.cpp:277-312) for this context's rows into sel ([n_local][3][L][N],
/// host or device memory) and comps (host).  Device output: tiles are written in place, no copies
/// back and no per-tile synchronisation (the C2 equality microbenchmark times this).
static void select_rows(Ctx& c, u32 nq, u32 comp, u32 m, const u64* query, u32 op, u64* sel, u32* comps, Timer& tm) {
    Nvtx nv("cwgpu select");
    if (!c.db_loaded) throw state_err("no database loaded");
    if (m != c.m) throw std::invalid_argument("expanded query length must equal the code length");
    if (!c.have_keys) throw he_err("evaluation keys not set");
    if (op != CWG_OP_FOLKLORE && op != CWG_OP_ARITH) throw std::invalid_argument("unknown equality operator");
    if (op == CWG_OP_ARITH && c.k < 2) throw std::invalid_argument("arithmetic operator needs k >= 2");
    c.prep_s_ok = false;  // the selection path uses the unscaled operands only
    cudaPointerAttributes pa{};
    const bool dev_out = cudaPointerGetAttributes(&pa, sel) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    const u32 N = c.cp.N, L = c.cp.L, J = c.ab.J;
    const size_t LN = (size_t)L * N;
    u64* dq = c.query.get<u64>((size_t)nq * 2 * LN);
    CK(cudaMemcpyAsync(dq, query, (size_t)nq * 2 * LN * 8, cudaMemcpyDefault, c.st));
    tm.mark(TM_H2D);
    u64* entries = expand(c, dq, nq, comp, m);
    tm.mark(TM_EXPAND);
    u32* prep = nullptr;
    if (op == CWG_OP_FOLKLORE && c.k >= 2) {
        prep = c.prep.get<u32>((size_t)m * 2 * J * N);
        prepare(c, entries, 2 * LN, nullptr, m, prep);
    }
    const u32 R = tile_rows(c);
    u64* dsel = dev_out ? nullptr : c.partial.get<u64>((size_t)R * 3 * LN);
    u32 nc = 0;
    for (u64 r0 = 0; r0 < c.n_local; r0 += R) {
        const u32 Rt = (u32)std::min<u64>(R, c.n_local - r0);
        u64* dst = dev_out ? sel + r0 * 3 * LN : dsel;
        u32 zs = 0;
        select_tile(c, entries, prep, op, r0, Rt, nc, zs, dst);
        if (nc == 2)  // 2-component rows: slot 2 is zero
            CK(cudaMemset2DAsync(dst + 2 * LN, 3 * LN * 8, 0, LN * 8, Rt, c.st));
        tm.mark(TM_SELECT);
        if (!dev_out) {
            CK(cudaMemcpyAsync(sel + r0 * 3 * LN, dsel, (size_t)Rt * 3 * LN * 8, cudaMemcpyDeviceToHost, c.st));
            CK(cudaStreamSynchronize(c.st));
            tm.mark(TM_D2H);
        }
    }
    CK(cudaStreamSynchronize(c.st));
    for (u64 r = 0; r < c.n_local; ++r) comps[r] = nc;
}


}  // namespace cwgpu


// ================================================================== C ABI
using namespace cwgpu;

/// One context = one device, or (cwg_create_multi) several: rows split contiguously across the
/// devices, every device expands the query (sharded when possible) and runs its rows, the partial
/// accumulators are summed on the root (device_ids[0]) by peer copies + k_add_u64, which finishes.
struct cwg_ctx {
    Ctx c;                                   // device_ids[0]: reduction and finalize
    std::vector<std::unique_ptr<Ctx>> more;  // device_ids[1..]
    std::mutex mmu;                          // serialises calls on a multi-device context
    DevBuf red;                              // root: a peer's partial accumulators in flight
    std::vector<Ctx*> all() {
        std::vector<Ctx*> v{&c};
        for (auto& p : more) v.push_back(p.get());
        return v;
    }
    bool multi() const { return !more.empty(); }
    ~cwg_ctx() { cudaSetDevice(c.device); red.release(); }
};

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return CWG_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return CWG_EINVAL;
    } catch (const he_err& e) {
        g_err = e.what();
        return CWG_EHE;
    } catch (const cuda_err& e) {
        g_err = e.what();
        return CWG_ECUDA;
    } catch (const state_err& e) {
        g_err = e.what();
        return CWG_ESTATE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CWG_EINVAL;
    }
}

/// f(ctx, index) on every device of h, one host thread per device (the first exception is
/// rethrown on the calling thread after all have finished).
template <class F>
static void for_devices(cwg_ctx* h, F&& f) {
    auto all = h->all();
    if (all.size() == 1) {
        CK(cudaSetDevice(all[0]->device));
        f(*all[0], (size_t)0);
        return;
    }
    std::vector<std::exception_ptr> err(all.size());
    std::vector<std::thread> th;
    for (size_t i = 0; i < all.size(); ++i)
        th.emplace_back([&, i] {
            try {
                CK(cudaSetDevice(all[i]->device));
                f(*all[i], i);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

/// rows [lo, hi) of n of device i among W (contiguous split)
static inline u64 split_lo(u64 n, size_t i, size_t W) { return n * i / W; }

static void init_ctx(Ctx& c, uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                     uint32_t galois_digit_bits, int device) {
    c.cp = make_chain(N, t, std::vector<u64>(q, q + L), relin_digit_bits, galois_digit_bits);
    if (N > 16384) throw std::invalid_argument("cwgpu: ring degree above 16384 is not supported");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw std::invalid_argument("cwgpu: device id out of range");
    c.device = device;
    cudaDeviceGetAttribute(&c.n_sms, cudaDevAttrMultiProcessorCount, device);
    if (c.n_sms <= 0) c.n_sms = 148;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    CK(cudaMalloc(&c.d_fb, 8));
    CK(cudaMemset(c.d_fb, 0, 8));
    set_smem_limits(N);
    c.dcur = &c.Dbuf;
    for (int i = 0; i < Ctx::kMaxStreams; ++i) CK(cudaStreamCreateWithFlags(&c.tst[i], cudaStreamNonBlocking));
    for (int i = 0; i <= Ctx::kMaxStreams; ++i) CK(cudaEventCreateWithFlags(&c.tev[i], cudaEventDisableTiming));
    ensure_aux(c, 1);
}

extern "C" {

const char* cwg_last_error(void) { return g_err.c_str(); }

void* cwg_pinned_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<uint64_t>(bytes, 16), cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        g_err = "cwgpu: pinned host allocation failed";
        return nullptr;
    }
    return p;
}

void cwg_pinned_free(void* p) {
    if (p) cudaFreeHost(p);
}

int cwg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

cwg_ctx* cwg_create(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                    uint32_t galois_digit_bits, int device) {
    return cwg_create_multi(N, L, q, t, relin_digit_bits, galois_digit_bits, &device, 1);
}

cwg_ctx* cwg_create_multi(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                          uint32_t galois_digit_bits, const int* device_ids, int n_devices) {
    cwg_ctx* h = nullptr;
    int rc = guarded([&] {
        if (n_devices < 1 || !device_ids) throw std::invalid_argument("cwgpu: no devices given");
        auto ctx = std::make_unique<cwg_ctx>();
        init_ctx(ctx->c, N, L, q, t, relin_digit_bits, galois_digit_bits, device_ids[0]);
        for (int i = 1; i < n_devices; ++i) {
            ctx->more.push_back(std::make_unique<Ctx>());
            init_ctx(*ctx->more.back(), N, L, q, t, relin_digit_bits, galois_digit_bits, device_ids[i]);
        }
        // direct peer access where the topology allows it (NVLink / NVSwitch); cudaMemcpyPeerAsync
        // stages through the host otherwise
        for (int i = 0; i < n_devices; ++i)
            for (int j = 0; j < n_devices; ++j) {
                if (device_ids[i] == device_ids[j]) continue;
                int ok = 0;
                if (cudaDeviceCanAccessPeer(&ok, device_ids[i], device_ids[j]) == cudaSuccess && ok) {
                    CK(cudaSetDevice(device_ids[i]));
                    if (cudaDeviceEnablePeerAccess(device_ids[j], 0) != cudaSuccess) cudaGetLastError();
                }
            }
        h = ctx.release();
    });
    return rc == CWG_OK ? h : nullptr;
}

void cwg_destroy(cwg_ctx* h) { delete h; }

int cwg_get_info(const cwg_ctx* h, cwg_info* out) {
    return guarded([&] {
        const Ctx& c = h->c;
        out->N = c.cp.N;
        out->L = c.cp.L;
        out->J = c.ab.J;
        out->Mm = c.ab.Mm;
        out->Dr = c.cp.Dr;
        out->Dg = c.cp.Dg;
        out->q_bits = c.cp.q_bits;
        Big A(1);
        for (u64 a : c.ab.a) A = A.mul_u64(a);
        out->aux_bits = A.bits();
        out->n_total = c.n_total;
        out->row_begin = c.row_begin;
        out->n_local = c.n_local;
        for (const auto& p : h->more) out->n_local += p->n_local;  // multi-device: all rows held
        out->s = c.s;
        out->k = c.k;
        out->m = c.m;
    });
}

int cwg_load_db(cwg_ctx* h, uint64_t n_total, uint64_t row_begin, uint64_t n_local, uint32_t s, uint32_t k,
                uint32_t m, const uint32_t* positions, const uint64_t* payload) {
    return guarded([&] {
        std::lock_guard<std::mutex> gm(h->mmu);
        const size_t W = h->all().size();
        if (n_local < W) throw std::invalid_argument("cwgpu: fewer rows than devices");
        for_devices(h, [&](Ctx& c, size_t i) {
            std::lock_guard<std::mutex> g(c.mu);
            const u64 lo = split_lo(n_local, i, W), hi = split_lo(n_local, i + 1, W);
            load_db(c, n_total, row_begin + lo, hi - lo, s, k, m, positions + lo * k,
                    payload ? payload + lo * s * c.cp.N : nullptr);
        });
    });
}

int cwg_load_db_bytes(cwg_ctx* h, uint64_t n_total, uint64_t row_begin, uint64_t n_local, uint32_t k, uint32_t m,
                      uint64_t payload_bytes, const uint8_t* payloads, const uint64_t* row_ids) {
    return guarded([&] {
        std::lock_guard<std::mutex> gm(h->mmu);
        const size_t W = h->all().size();
        if (n_local < W) throw std::invalid_argument("cwgpu: fewer rows than devices");
        for_devices(h, [&](Ctx& c, size_t i) {
            std::lock_guard<std::mutex> g(c.mu);
            const u64 lo = split_lo(n_local, i, W), hi = split_lo(n_local, i + 1, W);
            load_db_bytes(c, n_total, row_begin + lo, hi - lo, k, m, payload_bytes, payloads + lo * payload_bytes,
                          row_ids ? row_ids + lo : nullptr);
        });
    });
}

/// The reference's on-disk database (CWDB v1, db_file.cpp:34-59 / serialize.cpp: little-endian
/// u8 / u16 / u32 / u64 fields, u16-length strings, 4 x u64 seed, then per row a u32-length key and
/// a u32-length payload) straight into cwg_load_db_bytes: index mode -> codeword of the row index
/// (map_index), non-lossy keyword mode -> codeword of keyword_value(key) (pir.cpp:22-30,155-159),
/// payloads zero padded to the header's payload_bytes (chunk_payload pads the same way).
int cwg_load_db_file(cwg_ctx* h, const uint8_t* data, uint64_t size, uint32_t k, uint32_t m) {
    std::vector<uint8_t> payloads;
    std::vector<uint64_t> ids;
    uint64_t rows = 0, payload_bytes = 0, mode = 0;
    const int rc = guarded([&] {
        struct Rd {
            const uint8_t* p;
            uint64_t n, pos = 0;
            void need(uint64_t x) {
                if (x > n - pos) throw std::invalid_argument("truncated database file");
            }
            uint64_t le(int bytes) {
                need(bytes);
                uint64_t v = 0;
                for (int i = 0; i < bytes; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
                pos += bytes;
                return v;
            }
        } r{data, size};
        if (!data) throw std::invalid_argument("database file missing");
        if (r.le(4) != 0x42445743u) throw std::invalid_argument("not a database file");
        if (r.le(1) != 1) throw std::invalid_argument("unsupported database version");
        mode = r.le(1);
        const uint64_t keyword_bits = r.le(2), lossy = r.le(1);
        rows = r.le(8);
        r.le(4);  // plaintexts_per_row (recomputed from payload_bytes, as PirConfig does)
        payload_bytes = r.le(4);
        const uint64_t slen = r.le(2);
        r.need(slen);
        r.pos += slen;  // preset name (the caller built the context for it)
        for (int i = 0; i < 4; ++i) r.le(8);  // lossy seed
        if (mode > 1) throw std::invalid_argument("unknown database mode");
        if (lossy) throw std::invalid_argument("cwgpu: lossy keyword databases are not supported");
        if (mode == 1 && (keyword_bits == 0 || keyword_bits > 64))
            throw std::invalid_argument("keyword bit-length must be in [1, 64]");
        if (rows == 0) throw std::invalid_argument("empty database");
        payloads.assign(rows * payload_bytes, 0);
        ids.assign(mode == 1 ? rows : 0, 0);
        for (uint64_t i = 0; i < rows; ++i) {
            const uint64_t klen = r.le(4);
            r.need(klen);
            if (mode == 1) {  // keyword_value (pir.cpp:22-30)
                if (klen > 8) throw std::invalid_argument("numeric keyword longer than 8 bytes");
                uint64_t v = 0;
                for (uint64_t b = klen; b-- > 0;) v = (v << 8) | r.p[r.pos + b];
                if (keyword_bits < 64 && v >= (uint64_t(1) << keyword_bits))
                    throw std::invalid_argument("keyword outside the configured domain");
                ids[i] = v;
            }
            r.pos += klen;
            const uint64_t plen = r.le(4);
            r.need(plen);
            if (plen > payload_bytes) throw std::invalid_argument("payload exceeds the configured row size");
            std::memcpy(payloads.data() + i * payload_bytes, r.p + r.pos, plen);
            r.pos += plen;
        }
        if (r.pos != size) throw std::invalid_argument("trailing bytes in database file");
        if (mode == 1) {  // parse_db's duplicate-key check, on the decoded keyword values
            std::vector<uint64_t> srt(ids);
            std::sort(srt.begin(), srt.end());
            if (std::adjacent_find(srt.begin(), srt.end()) != srt.end())
                throw std::invalid_argument("duplicate key in database file");
        }
    });
    if (rc != CWG_OK) return rc;
    return cwg_load_db_bytes(h, rows, 0, rows, k, m, payload_bytes, payloads.data(), mode == 1 ? ids.data() : nullptr);
}

int cwg_set_keys(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                 const uint64_t* galois) {
    return guarded([&] {
        std::lock_guard<std::mutex> gm(h->mmu);
        for_devices(h, [&](Ctx& c, size_t) {
            std::lock_guard<std::mutex> g(c.mu);
            upload_keys(c, relin, n_galois, galois_g, galois);
            CK(cudaStreamSynchronize(c.st));
        });
    });
}

uint64_t cwg_partial_words(const cwg_ctx* h) {
    const Ctx& c = h->c;
    return (uint64_t)c.s * 3 * c.ab.Mm * c.cp.N;
}

int cwg_answer_partial(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                       const uint64_t* galois, uint32_t nq, uint32_t comp, uint32_t m, const uint64_t* query,
                       uint32_t op, uint64_t* dev_partial, cwg_timings* t) {
    return guarded([&] {
        if (h->multi()) throw state_err("cwgpu: row-shard entry points take a single-device context");
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        auto t0 = std::chrono::steady_clock::now();
        Timer tm(c, t != nullptr);
        tm.mark(TM_START);
        c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
        answer_partial(c, nq, comp, m, query, op, dev_partial, tm);
        CK(cudaStreamSynchronize(c.st));
        fill_timings(c, tm, t,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
}

int cwg_expand_shard(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                     const uint64_t* galois, uint32_t comp, const uint64_t* query, uint32_t world, uint32_t rank,
                     uint64_t* out) {
    return guarded([&] {
        if (h->multi()) throw state_err("cwgpu: row-shard entry points take a single-device context");
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
        if (!c.have_keys) throw he_err("evaluation keys not set");
        const size_t per = 2 * (size_t)c.cp.L * c.cp.N;
        u64* dq = c.query.get<u64>(per);
        CK(cudaMemcpyAsync(dq, query, per * 8, cudaMemcpyDefault, c.st));  // host or device
        expand_shard(c, dq, comp, world, rank, out);
        CK(cudaStreamSynchronize(c.st));
    });
}
int cwg_answer_partial_shards(cwg_ctx* h, const uint64_t* shards, uint32_t world, uint32_t comp, uint32_t m,
                              uint32_t op, uint64_t* dev_partial, cwg_timings* t) {
    return guarded([&] {
        if (h->multi()) throw state_err("cwgpu: row-shard entry points take a single-device context");
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        auto t0 = std::chrono::steady_clock::now();
        Timer tm(c, t != nullptr);
        tm.mark(TM_START);
        answer_partial(c, 1, comp, m, nullptr, op, dev_partial, tm, shards, world);
        CK(cudaStreamSynchronize(c.st));
        fill_timings(c, tm, t,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
}
int cwg_finish(cwg_ctx* h, const uint64_t* dev_partial_sum, uint32_t op, uint64_t* out, cwg_timings* t) {
    return guarded([&] {
        if (h->multi()) throw state_err("cwgpu: row-shard entry points take a single-device context");
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        if (!c.db_loaded || c.s == 0) throw state_err("no database loaded");
        if (!c.have_keys) throw he_err("evaluation keys not set");
        auto t0 = std::chrono::steady_clock::now();
        Timer tm(c, t != nullptr);
        tm.mark(TM_START);
        const u32 nc = (op == CWG_OP_FOLKLORE && c.k >= 2) ? 3 : 2;
        finish(c, dev_partial_sum, nc, out, tm);
        fill_timings(c, tm, t,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
}

/// cwg_answer on a multi-device context (see cwg_ctx).
static void answer_multi(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                         const uint64_t* galois, uint32_t nq, uint32_t comp, uint32_t m, const uint64_t* query,
                         uint32_t op, uint64_t* out, cwg_timings* t) {
    std::lock_guard<std::mutex> gm(h->mmu);
    auto all = h->all();
    const u32 W = (u32)all.size();
    Ctx& root = h->c;
    const auto t0 = std::chrono::steady_clock::now();
    const size_t per = 2 * (size_t)root.cp.L * root.cp.N;
    // sharded expansion when the query is one ciphertext and W | 2^c is a power of two: device i
    // expands the leaves i, i + W, ... (cwg_expand_shard) and the shards are all-gathered by peer copies
    const bool shard = nq == 1 && (W & (W - 1)) == 0 && W <= (1u << comp) && (1u << comp) <= root.cp.N;
    const size_t shard_words = shard ? ((size_t)1 << comp) / W * per : 0;
    std::vector<u32> ncs(W, 2);
    for_devices(h, [&](Ctx& c, size_t i) {
        std::lock_guard<std::mutex> g(c.mu);
        c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
        if (!c.have_keys) throw he_err("evaluation keys not set");
        if (shard) {
            if (m != c.m) throw std::invalid_argument("query code length does not match the database");
            u64* dq = c.query.get<u64>(per);
            CK(cudaMemcpyAsync(dq, query, per * 8, cudaMemcpyDefault, c.st));
            c.shard_all.get<u64>(shard_words * W);
            expand_shard(c, dq, comp, W, (u32)i, c.shard_out.get<u64>(shard_words));
        }
        CK(cudaStreamSynchronize(c.st));
    });
    for_devices(h, [&](Ctx& c, size_t i) {
        std::lock_guard<std::mutex> g(c.mu);
        Timer tm(c, false);
        u64* part = c.partial.get<u64>((size_t)c.s * 3 * c.ab.Mm * c.cp.N);
        if (shard) {
            u64* dst = c.shard_all.ptr<u64>();
            for (u32 j = 0; j < W; ++j)
                CK(cudaMemcpyPeerAsync(dst + j * shard_words, c.device, all[j]->shard_out.ptr<u64>(), all[j]->device,
                                       shard_words * 8, c.st));
            ncs[i] = answer_partial(c, 1, comp, m, nullptr, op, part, tm, dst, W);
        } else {
            ncs[i] = answer_partial(c, nq, comp, m, query, op, part, tm);
        }
        CK(cudaStreamSynchronize(c.st));
    });
    CK(cudaSetDevice(root.device));
    std::lock_guard<std::mutex> g(root.mu);
    Timer tm(root, t != nullptr);
    tm.mark(TM_START);
    const size_t words = (size_t)root.s * 3 * root.ab.Mm * root.cp.N;
    u64* acc = root.partial.ptr<u64>();
    u64* buf = h->red.get<u64>(words);
    for (u32 j = 1; j < W; ++j) {  // row-shard reduction: u64 sums of residues < 2^31
        CK(cudaMemcpyPeerAsync(buf, root.device, all[j]->partial.ptr<u64>(), all[j]->device, words * 8, root.st));
        launch(root, k_add_u64, blocks(words, 256), 256, 0, acc, (const u64*)buf, words);
    }
    tm.mark(TM_MAC);
    finish(root, acc, ncs[0], out, tm);
    fill_timings(root, tm, t, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (t) {
        t->n_devices = W;
        for (Ctx* c : all) t->kernel_launches += c == &root ? 0 : c->launches;
    }
}

int cwg_answer(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g, const uint64_t* galois,
               uint32_t nq, uint32_t comp, uint32_t m, const uint64_t* query, uint32_t op, uint64_t* out,
               cwg_timings* t) {
    return guarded([&] {
        if (h->multi()) {
            answer_multi(h, relin, n_galois, galois_g, galois, nq, comp, m, query, op, out, t);
            return;
        }
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        auto t0 = std::chrono::steady_clock::now();
        Timer tm(c, t != nullptr);
        tm.mark(TM_START);
        c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
        u64* part = c.partial.get<u64>((size_t)c.s * 3 * c.ab.Mm * c.cp.N);
        const u32 nc = answer_partial(c, nq, comp, m, query, op, part, tm);
        finish(c, part, nc, out, tm);
        fill_timings(c, tm, t,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
}

int cwg_answer_batch(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                     const uint64_t* galois, uint32_t Q, uint32_t nq, uint32_t comp, uint32_t m,
                     const uint64_t* queries, uint32_t op, uint64_t* out, cwg_timings* t) {
    if (h->multi()) {  // several devices: one multi-device answer per query
        const size_t qw = (size_t)nq * 2 * h->c.cp.L * h->c.cp.N, ow = (size_t)h->c.s * 2 * h->c.cp.L * h->c.cp.N;
        for (uint32_t q = 0; q < Q; ++q) {
            const int rc = cwg_answer(h, q ? nullptr : relin, n_galois, galois_g, galois, nq, comp, m, queries + q * qw,
                                      op, out + q * ow, t);
            if (rc != CWG_OK) return rc;
        }
        return CWG_OK;
    }
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        auto t0 = std::chrono::steady_clock::now();
        Timer tm(c, t != nullptr);
        tm.mark(TM_START);
        c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
        answer_batch(c, Q, nq, comp, m, queries, op, out, tm);
        fill_timings(c, tm, t,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
}

/// NTT of the secret key (and its square) mod every chain prime, for the GPU client calls.
static void client_secret(Ctx& c, const int8_t* sk, bool square) {
    const u32 N = c.cp.N, L = c.cp.L;
    const size_t LN = (size_t)L * N;
    signed char* ds = reinterpret_cast<signed char*>(c.cl_bits.get<unsigned char>(std::max<size_t>(N, 16)));
    CK(cudaMemcpyAsync(ds, sk, N, cudaMemcpyDefault, c.st));
    u64* s1 = c.cl_s.get<u64>(LN);
    launch(c, k_signed_to_chain, blocks(LN, 256), 256, 0, (const signed char*)ds, c.T, s1);
    ntt64(c, s1, L, false);
    if (square) {
        u64* s2 = c.cl_s2.get<u64>(LN);
        CK(cudaMemcpyAsync(s2, s1, LN * 8, cudaMemcpyDeviceToDevice, c.st));
        launch(c, k_mul64, blocks(LN, 256), 256, 0, s2, (const u64*)s1, (size_t)1, c.T);
    }
}

int cwg_encrypt_query(cwg_ctx* h, const uint64_t* sk_seed, const int8_t* sk, const uint8_t* bits, uint32_t m,
                      uint32_t comp, uint64_t first_index, uint64_t* out) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        Nvtx nv("cwgpu encrypt_query");
        const u32 N = c.cp.N, L = c.cp.L;
        const size_t LN = (size_t)L * N;
        if ((u64(1) << comp) > N) throw std::invalid_argument("compression factor exceeds log2(N)");
        if (!sk || !sk_seed || (!bits && m)) throw std::invalid_argument("missing secret key or query bits");
        const u64 t = c.cp.t;
        const u64 scale = invmod64(((u64)1 << comp) % t, t);  // pack_query_bits' 2^-c mod t
        const u32 hq = (u32)(((u64)m + (1u << comp) - 1) >> comp);
        if (hq == 0) throw std::invalid_argument("empty query");
        Seed4 seed;
        for (int i = 0; i < 4; ++i) seed.w[i] = sk_seed[i];
        Seed4* seeds = reinterpret_cast<Seed4*>(c.cl_seeds.get<u64>((size_t)8 * hq));
        launch(c, k_enc_seeds, blocks(hq, 64), 64, 0, seed, (u64)first_index, hq, seeds, seeds + hq);
        std::vector<u64> lim(L);
        for (u32 i = 0; i < L; ++i) lim[i] = ~0ull - (~0ull % c.cp.q[i]);
        u64* dlim = c.cl_lim.get<u64>(L);
        CK(cudaMemcpyAsync(dlim, lim.data(), L * 8, cudaMemcpyHostToDevice, c.st));
        u64* dout = c.cl_out.get<u64>((size_t)hq * 2 * LN);
        // c1 = uniform_rns(derive_seed(sk.seed, 5, index)) straight into component 1
        launch(c, k_uniform_rns, (size_t)hq * L, 1024, 0, (const Seed4*)seeds, c.T, (const u64*)dlim, dout + LN, 2 * LN);
        // c1 s (negacyclic, per prime) through the chain NTT
        client_secret(c, sk, false);
        u64* prod = c.cl_a.get<u64>((size_t)hq * LN);
        launch(c, k_gather_strided, blocks((size_t)hq * LN, 256), 256, 0, (const u64*)(dout + LN), 2 * LN,
               (const u32*)nullptr, hq, LN, prod, LN);
        ntt64(c, prod, hq * L, false);
        launch(c, k_mul64, blocks((size_t)hq * LN, 256), 256, 0, prod, (const u64*)c.cl_s.ptr<u64>(), (size_t)hq, c.T);
        ntt64(c, prod, hq * L, true);
        int* e = c.cl_e.get<int>((size_t)hq * N);
        launch(c, k_noise, blocks((size_t)hq * N, 256), 256, 0, (const Seed4*)(seeds + hq), hq, N, e);
        unsigned char* db = c.cl_bits.get<unsigned char>(std::max<size_t>(m, N));
        CK(cudaMemcpyAsync(db, bits, m, cudaMemcpyDefault, c.st));
        launch(c, k_enc_combine, blocks((size_t)hq * LN, 256), 256, 0, (const u64*)prod, (const int*)e,
               (const unsigned char*)db, m, comp, scale, hq, c.T, dout);
        CK(cudaMemcpyAsync(out, dout, (size_t)hq * 2 * LN * 8, cudaMemcpyDefault, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_decrypt(cwg_ctx* h, const int8_t* sk, uint32_t count, uint32_t comps, const uint64_t* cts, uint64_t* out) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        Nvtx nv("cwgpu decrypt");
        if (comps < 2 || comps > 3) throw std::invalid_argument("ciphertext must have 2 or 3 components");
        if (!sk) throw std::invalid_argument("decryption requires the secret key");
        if (count == 0) return;
        const u32 N = c.cp.N, L = c.cp.L;
        const size_t LN = (size_t)L * N, per = (size_t)comps * LN;
        u64* d = c.cl_out.get<u64>((size_t)count * per);
        CK(cudaMemcpyAsync(d, cts, (size_t)count * per * 8, cudaMemcpyDefault, c.st));
        client_secret(c, sk, comps == 3);
        u64* v = c.cl_a.get<u64>((size_t)count * LN);
        u64* w = c.cl_b.get<u64>((size_t)count * LN);
        // v = c1 s (+ c2 s^2) in the NTT domain, back to coefficients, + c0 (bfv.cpp:556-568)
        launch(c, k_gather_strided, blocks((size_t)count * LN, 256), 256, 0, (const u64*)(d + LN), per,
               (const u32*)nullptr, count, LN, v, LN);
        ntt64(c, v, count * L, false);
        launch(c, k_mul64, blocks((size_t)count * LN, 256), 256, 0, v, (const u64*)c.cl_s.ptr<u64>(), (size_t)count, c.T);
        if (comps == 3) {
            launch(c, k_gather_strided, blocks((size_t)count * LN, 256), 256, 0, (const u64*)(d + 2 * LN), per,
                   (const u32*)nullptr, count, LN, w, LN);
            ntt64(c, w, count * L, false);
            launch(c, k_mul64, blocks((size_t)count * LN, 256), 256, 0, w, (const u64*)c.cl_s2.ptr<u64>(), (size_t)count,
                   c.T);
            launch(c, k_add64_strided, blocks((size_t)count * LN, 256), 256, 0, v, (const u64*)w, LN, (size_t)count, c.T);
        }
        ntt64(c, v, count * L, true);
        launch(c, k_add64_strided, blocks((size_t)count * LN, 256), 256, 0, v, (const u64*)d, per, (size_t)count, c.T);
        u64* m = c.cl_b.get<u64>((size_t)count * N);
        launch(c, k_dec_round, blocks((size_t)count * N, 128), 128, 0, (const u64*)v, (size_t)count, c.T, m);
        CK(cudaMemcpyAsync(out, m, (size_t)count * N * 8, cudaMemcpyDefault, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_select(cwg_ctx* h, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g, const uint64_t* galois,
               uint32_t nq, uint32_t comp, uint32_t m, const uint64_t* query, uint32_t op, uint64_t* sel,
               uint32_t* comps, cwg_timings* t) {
    return guarded([&] {
        std::lock_guard<std::mutex> gm(h->mmu);
        auto t0 = std::chrono::steady_clock::now();
        const size_t W = h->all().size();
        u64 off = 0;
        std::vector<u64> offs;
        for (Ctx* c : h->all()) {
            offs.push_back(off);
            off += c->n_local;
        }
        if (W > 1) {
            cudaPointerAttributes pa{};
            if (cudaPointerGetAttributes(&pa, sel) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
                throw std::invalid_argument("cwgpu: a multi-device selection is written to host memory");
            cudaGetLastError();
        }
        for_devices(h, [&](Ctx& c, size_t i) {
            std::lock_guard<std::mutex> g(c.mu);
            Timer tm(c, t != nullptr && i == 0);
            tm.mark(TM_START);
            c.keys_cached = relin ? upload_keys(c, relin, n_galois, galois_g, galois) : false;
            const size_t LN = (size_t)c.cp.L * c.cp.N;
            select_rows(c, nq, comp, m, query, op, sel + offs[i] * 3 * LN, comps + offs[i], tm);
            if (i == 0)
                fill_timings(c, tm, t,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        });
        if (t) t->n_devices = (uint32_t)W;
    });
}

int cwg_ntt(cwg_ctx* h, int chain, uint32_t idx, uint64_t* data, uint32_t count, int inverse) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        const u32 N = c.cp.N;
        if (chain) {
            if (idx >= c.cp.L) throw std::invalid_argument("prime index out of range");
            // lay the polys out as p = x*L + idx so that prime(p) = idx
            u64* d = c.exA.get<u64>((size_t)count * c.cp.L * N);
            for (u32 x = 0; x < count; ++x)
                CK(cudaMemcpyAsync(d + ((size_t)x * c.cp.L + idx) * N, data + (size_t)x * N, N * 8,
                                   cudaMemcpyHostToDevice, c.st));
            ntt64(c, d, count * c.cp.L, inverse != 0);
            for (u32 x = 0; x < count; ++x)
                CK(cudaMemcpyAsync(data + (size_t)x * N, d + ((size_t)x * c.cp.L + idx) * N, N * 8,
                                   cudaMemcpyDeviceToHost, c.st));
        } else {
            if (idx >= c.ab.J) throw std::invalid_argument("prime index out of range");
            std::vector<u32> tmp((size_t)count * N);
            for (size_t x = 0; x < tmp.size(); ++x) tmp[x] = (u32)data[x];
            u32* d = c.lift_tmp.get<u32>(tmp.size());
            CK(cudaMemcpyAsync(d, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, c.st));
            // group size 1, stride 1, offset idx: poly p at (p + idx) * N uses prime idx
            ntt32(c, d - (size_t)idx * N, count, 1, 1, idx, inverse != 0, 0, false);
            CK(cudaMemcpyAsync(tmp.data(), d, tmp.size() * 4, cudaMemcpyDeviceToHost, c.st));
            CK(cudaStreamSynchronize(c.st));
            for (size_t x = 0; x < tmp.size(); ++x) data[x] = tmp[x];
        }
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_expand(cwg_ctx* h, uint32_t nq, uint32_t comp, uint32_t m, const uint64_t* query, uint64_t* out) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        if (!c.have_keys) throw he_err("evaluation keys not set");
        const size_t per = 2 * (size_t)c.cp.L * c.cp.N;
        u64* dq = c.query.get<u64>(nq * per);
        CK(cudaMemcpyAsync(dq, query, nq * per * 8, cudaMemcpyHostToDevice, c.st));
        u64* e = expand(c, dq, nq, comp, m);
        CK(cudaMemcpyAsync(out, e, (size_t)m * per * 8, cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_mul_lazy(cwg_ctx* h, uint32_t count, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        const u32 N = c.cp.N, J = c.ab.J;
        const size_t per = 2 * (size_t)c.cp.L * N;
        u64* d = c.exA.get<u64>(2 * (size_t)count * per);
        CK(cudaMemcpyAsync(d, a, count * per * 8, cudaMemcpyHostToDevice, c.st));
        CK(cudaMemcpyAsync(d + count * per, b, count * per * 8, cudaMemcpyHostToDevice, c.st));
        u32* pr = c.prep.get<u32>((size_t)2 * count * 2 * J * N);
        prepare(c, d, per, nullptr, 2 * count, pr);
        u64* o = c.chain3.get<u64>((size_t)count * 3 * c.cp.L * N);
        mul_prepared(c, pr, nullptr, pr + (size_t)count * 2 * J * N, nullptr, count, false, o);
        CK(cudaMemcpyAsync(out, o, (size_t)count * 3 * c.cp.L * N * 8, cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_relinearize(cwg_ctx* h, uint32_t count, const uint64_t* ct3, uint64_t* out2) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        if (!c.have_keys) throw he_err("evaluation keys not set");
        const size_t LN = (size_t)c.cp.L * c.cp.N;
        u64* d = c.chain3.get<u64>(count * 3 * LN);
        CK(cudaMemcpyAsync(d, ct3, count * 3 * LN * 8, cudaMemcpyHostToDevice, c.st));
        u64* o = c.out2.get<u64>(count * 2 * LN);
        relinearize(c, d, count, o);
        CK(cudaMemcpyAsync(out2, o, count * 2 * LN * 8, cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_substitute(cwg_ctx* h, uint32_t count, const uint64_t* ct, uint64_t g, uint64_t* out) {
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> lk(c.mu);
        CK(cudaSetDevice(c.device));
        if (!c.have_keys) throw he_err("evaluation keys not set");
        const u32 N = c.cp.N, L = c.cp.L;
        if (g % 2 == 0 || g >= 2 * (u64)N) throw std::invalid_argument("automorphism exponent must be odd in (0, 2N)");
        const u64* key = galois_key(c, g);
        const size_t per = 2 * (size_t)L * N;
        u64* d = c.exA.get<u64>(count * per);
        CK(cudaMemcpyAsync(d, ct, count * per * 8, cudaMemcpyHostToDevice, c.st));
        u64* ks = c.ks.get<u64>(count * per);
        const u64 ginv = inv_mod_2n(g, 2 * (u64)N);
        key_switch(c, d + (size_t)L * N, per, ginv, count, key, c.cp.galois_bits, c.cp.Dg, ks);
        u64* o = c.out2.get<u64>(count * per);
        launch(c, k_subst_combine, blocks((size_t)count * L * N, 256), 256, 0, (const u64*)d, (const u64*)ks, count,
               ginv, c.T, o);
        CK(cudaMemcpyAsync(out, o, count * per * 8, cudaMemcpyDeviceToHost, c.st));
        CK(cudaStreamSynchronize(c.st));
    });
}

int cwg_set_option(cwg_ctx* h, const char* key, int64_t value) {
    return guarded([&] {
      for (Ctx* cp : h->all()) {
        Ctx& c = *cp;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaSetDevice(c.device));
        const std::string k = key ? key : "";
        const int v = (int)value;
        if (k == "streams") c.nstreams = std::max(1, std::min(Ctx::kMaxStreams, v));
        else if (k == "mac") c.mac_tma = v != 0;
        else if (k == "mac_waves") c.mac_waves = std::max(1, v);
        else if (k == "prescale") c.prescale = v != 0;
        else if (k == "ntt_np") c.ntt_np = v == 2 ? 2 : 1;
        else if (k == "round") c.round_kind = v == 0 ? 0 : 2;
        else if (k == "fuse_mac") c.fuse_mac = v != 0;
        else if (k == "mac_ck") c.mac_ck = (u32)std::max(0, v);
        else if (k == "round_g2") c.round_g2 = v != 0;
        else if (k == "round_ctas") c.round_ctas = (u32)std::max(1, std::min(4, v));
        else if (k == "ks32") { c.ks32 = v != 0; c.ksA_ok = false; }
        else if (k == "tile_rows") c.tile_rows_opt = (u32)std::max(0, v);
        else if (k == "ks_wide") c.ks_wide = v != 0;
        else if (k == "ks_ci") c.ks_ci = (u32)v;
        else if (k == "prep_factors") c.prep_mode = v != 0;
        else if (k == "lift_tc") c.lift_tc = v != 0;
        else if (k == "m2c_tc") c.m2c_tc = v != 0;
        else if (k == "ks_fixed") c.ks_fixed = v != 0;
        else if (k == "ks_chunk_mb") c.ks_chunk_mb = (u32)std::max(64, v);
        else if (k == "dec_tc") c.dec_tc = v != 0;
        else if (k == "mac_sg") c.mac_sg = v != 0;
        else if (k == "mac_stages") c.mac_stages8 = v >= 8;
        else if (k == "mac_rows") c.mac_rows = v != 0;
        else if (k == "mac_item_rows") c.mac_item_rows = (u32)std::max(1, v);
        else if (k == "force_exact") {
            c.force_exact = v != 0;
            c.T.force_exact = c.force_exact ? 1u : 0u;
            CK(cudaMemcpy(c.tab_self.p, &c.T, sizeof(DevTab), cudaMemcpyHostToDevice));
        } else
            throw std::invalid_argument("cwgpu: unknown option " + k);
      }
    });
}

uint64_t cwg_kernel_launches(const cwg_ctx* h) {
    uint64_t n = h->c.launches;
    for (const auto& p : h->more) n += p->launches;
    return n;
}

void* cwg_stream(const cwg_ctx* h) { return (void*)h->c.st; }

int cwg_set_profiling(cwg_ctx* h, int on) {  // root device only on a multi-device context
    return guarded([&] {
        Ctx& c = h->c;
        std::lock_guard<std::mutex> g(c.mu);
        CK(cudaStreamSynchronize(c.st));
        prof_collect(c);
        c.profiling = on != 0;
        c.prof_stats.clear();
    });
}

int cwg_kernel_stats(const cwg_ctx* h, uint32_t idx, char* name, uint32_t name_len, double* total_ms,
                     uint64_t* count) {
    const Ctx& c = h->c;
    if (idx >= c.prof_stats.size()) return CWG_EINVAL;
    const auto& e = c.prof_stats[idx];
    std::snprintf(name, name_len, "%s", e.name.c_str());
    *total_ms = e.ms;
    *count = e.count;
    return CWG_OK;
}

int cwg_kernel_units(const cwg_ctx* h, uint32_t idx, double* units) {
    const Ctx& c = h->c;
    if (idx >= c.prof_stats.size()) return CWG_EINVAL;
    *units = c.prof_stats[idx].units;
    return CWG_OK;
}

}  // extern "C"


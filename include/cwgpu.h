/*
 * cwgpu.h -- C ABI of the B200-native constant-weight PIR server answer.
 *
 * Drop-in boundary for the reference's server answer
 *   std::vector<CipherValue> process_query(const HeBackend&, const PackedQuery&,
 *                                          const PirDatabase&)
 *   (/root/reference/proj/core/include/cwpir/pir.hpp:114-117, pir.cpp:337-347)
 * plus the stage entry points its tests exercise.  Plain pointers and sizes only;
 * no exceptions cross this boundary: every call returns CWG_OK (0) or a negative
 * status, and cwg_last_error() returns the thread's last message, worded like the
 * reference's exceptions (he_error / std::invalid_argument, he.hpp:16-18).
 *
 * Array layouts (little-endian u64, canonical residues):
 *   ciphertext      [comps][L][N]       coefficient form          (he.hpp:56-65)
 *   key-switch key  [D][2][L][N]        rows[d][k][i], reference NTT form (bfv.hpp:37-40,
 *                                       bfv.cpp:394-402)
 *   galois keys     [n_galois][Dg][2][L][N]  for exponents galois_g[a]
 *   query           [h][2][L][N]        PackedQuery::cts (expansion.hpp:21-25)
 *   positions       [n][k]              Codeword::positions(), ascending (cw_code.hpp:40)
 *   payload         [n][s][N]           PirDatabase::chunk(i, j) coefficients < t
 *   response        [s][2][L][N]
 */
#ifndef CWGPU_H
#define CWGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CWG_OK 0
#define CWG_EINVAL (-1) /* std::invalid_argument in the reference */
#define CWG_EHE (-2)    /* he_error in the reference (e.g. missing Galois key) */
#define CWG_ECUDA (-3)  /* CUDA runtime failure */
#define CWG_ESTATE (-4) /* call out of order (e.g. answer before cwg_load_db) */

#define CWG_OP_FOLKLORE 0u   /* product of the k selected bits (pir.cpp:287-302) */
#define CWG_OP_ARITH 1u      /* prod_{i<k} (k' - i) / k!   (eq_circuits.cpp:105-127) */

typedef struct cwg_ctx cwg_ctx;

typedef struct cwg_info {
    uint32_t N, L, J, Mm, Dr, Dg, q_bits, aux_bits;
    uint64_t n_total, row_begin, n_local;
    uint32_t s, k, m;
} cwg_info;

typedef struct cwg_timings {
    double total_ms;   /* cwg_answer entry to return (includes H2D / D2H) */
    double h2d_ms;     /* keys + query upload */
    double expand_ms;  /* expand_query */
    double select_ms;  /* aux lift + per-row equality (tensor, INTT, exact rounding, NTT) */
    double mac_ms;     /* payload multiply-accumulate (DB streamed from HBM) */
    double finish_ms;  /* accumulator reduce, INTT, basis conversion, relinearisation */
    double d2h_ms;
    uint64_t kernel_launches;
    uint64_t exact_fallbacks; /* coefficients decided by the multiword slow path (this answer) */
    uint32_t keys_cached;     /* 1: the keys passed with this call equalled the resident set (device
                                 key cache: upload compared on the device, aux-basis transform kept) */
    uint32_t n_devices;       /* devices that worked on this call */
} cwg_timings;

const char* cwg_last_error(void);

/* Pinned (page-locked, portable) host memory for staging keys, queries and responses: copies
 * from it run as asynchronous DMA at full PCIe / C2C speed.  NULL on failure. */
void* cwg_pinned_alloc(uint64_t bytes);
void cwg_pinned_free(void* p);

/* Number of CUDA devices visible to this process (0 without a driver / device). */
int cwg_device_count(void);

/* BfvContext equivalent (bfv.cpp:67-129) on one device.  q: L chain primes
 * (each 2^32 < q_i < 2^60, NTT-friendly), t: plaintext prime, digit widths as
 * HeParams::relin_digit_bits / galois_digit_bits (0 = one digit per prime). */
cwg_ctx* cwg_create(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                    uint32_t galois_digit_bits, int device);
/* The same over several devices of this process (SURVEY 8b's device_ids / n_devices): the rows
 * of cwg_load_db / cwg_load_db_bytes are split contiguously across device_ids (a device id may
 * repeat: two contexts on one GPU); cwg_answer expands the query on every device (sharded by
 * subtree and all-gathered by peer copies when the query is one ciphertext and n_devices is a
 * power of two <= 2^c), runs each device's rows into partial accumulators, sums them on
 * device_ids[0] (peer copies + one add kernel per device) and finishes there.  Bit-identical to
 * one device.  cwg_select writes each device's rows to a host buffer; set_keys / set_option apply
 * to all devices; the stage entry points (cwg_ntt ... cwg_substitute) and profiling use
 * device_ids[0]; the per-process row-shard calls (cwg_answer_partial, cwg_finish, ...) need a
 * single-device context. */
cwg_ctx* cwg_create_multi(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                          uint32_t galois_digit_bits, const int* device_ids, int n_devices);
void cwg_destroy(cwg_ctx* ctx);
int cwg_get_info(const cwg_ctx* ctx, cwg_info* out);

/* PirDatabase::setup + prepare_for (pir.cpp:214-264): rows [row_begin, row_begin+n_local)
 * of an n_total-row database are made resident in NTT form on this device.
 * positions: [n_local][k]; payload: [n_local][s][N] (NULL for a selection-only database,
 * then s must be 0).  m: code length. */
int cwg_load_db(cwg_ctx* ctx, uint64_t n_total, uint64_t row_begin, uint64_t n_local, uint32_t s,
                uint32_t k, uint32_t m, const uint32_t* positions, const uint64_t* payload);

/* PirDatabase::setup + prepare_for from raw rows (pir.cpp:214-264), codewords and plaintexts
 * built on the device: row r's codeword is perfect_map(id_r) (cw_code.cpp:80-102) with
 * id_r = row_ids[r] (keyword mode: keyword_value of the key, pir.cpp:22-30) or, when row_ids is
 * NULL, the global row index row_begin + r (index mode, map_index pir.cpp:149-153); payloads
 * [n_local][payload_bytes] (host or device) are chunked into s = max(1, ceil(8 payload_bytes /
 * (N floor(log2 t)))) plaintexts (chunk_payload, pir.cpp:169-193).  Errors as the reference:
 * all-zero payloads, duplicate identifiers, ids outside the code capacity. */
int cwg_load_db_bytes(cwg_ctx* ctx, uint64_t n_total, uint64_t row_begin, uint64_t n_local, uint32_t k, uint32_t m,
                      uint64_t payload_bytes, const uint8_t* payloads, const uint64_t* row_ids);

/* The reference's database file (CWDB v1, db_file.cpp:34-59: header + length-prefixed key /
 * payload records; index or non-lossy keyword mode) parsed from memory and loaded as
 * cwg_load_db_bytes does (codewords and plaintext chunks built on the device).  k, m: the
 * PirConfig's Hamming weight and code length.  Errors as parse_db / PirDatabase::setup. */
int cwg_load_db_file(cwg_ctx* ctx, const uint8_t* data, uint64_t size, uint32_t k, uint32_t m);

/* Evaluation keys (EvalKeySet, bfv.hpp:42-51).  Kept resident until replaced. */
int cwg_set_keys(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                 const uint64_t* galois);

/* process_query (pir.cpp:337-347): expand_query -> selection -> inner product ->
 * finalize.  Keys may be passed per call (relin != NULL uploads them, as the
 * reference server receives them with every query, server.cpp:63-68) or NULL to use
 * the resident set.  query: [h][2][L][N] with compression c and code length m.
 * out: [s][2][L][N].  query, out and the keys may be host (pageable or pinned) or device
 * pointers (copies use cudaMemcpyDefault).  t (optional) receives stage timings. */
int cwg_answer(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
               const uint64_t* galois, uint32_t h, uint32_t c, uint32_t m, const uint64_t* query,
               uint32_t op, uint64_t* out, cwg_timings* t);

/* Multi-query answer: Q queries under one evaluation-key set (e.g. one client
 * fetching Q rows) answered in one pass over the database -- every row tile's selection values are
 * computed for all Q queries and the payload MAC reads the tile's database planes once for up to
 * four of them.  queries: [Q][h][2][L][N]; out: [Q][s][2][L][N]; each response equals cwg_answer's.
 * A multi-device context answers the queries one after another. */
int cwg_answer_batch(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                     const uint64_t* galois, uint32_t Q, uint32_t h, uint32_t c, uint32_t m, const uint64_t* queries,
                     uint32_t op, uint64_t* out, cwg_timings* t);

/* Row-sharded form (one process per GPU): the partial NTT-domain accumulators of this
 * device's rows, written to DEVICE memory (cwg_partial_words() u64 words, each < 2^31,
 * summable with a plain uint64 reduction), then cwg_finish on the root with the summed
 * partials (device pointer) produces the response exactly as cwg_answer would. */
uint64_t cwg_partial_words(const cwg_ctx* ctx);
int cwg_answer_partial(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                       const uint64_t* galois, uint32_t h, uint32_t c, uint32_t m, const uint64_t* query,
                       uint32_t op, uint64_t* dev_partial, cwg_timings* t);
int cwg_finish(cwg_ctx* ctx, const uint64_t* dev_partial_sum, uint32_t op, uint64_t* out, cwg_timings* t);

/* Sharded expansion for the row-sharded form (one query ciphertext, h = 1; W a power of two
 * <= 2^c): rank r expands the subtree of level-log2(W) node r, i.e. the global leaves
 * r, r + W, r + 2W, ... (2^c / W of them), into out (device, [2^c / W][2][L][N]).  Gathering
 * the W outputs rank-major (e.g. an all-gather) and passing them to cwg_answer_partial_shards
 * replaces each rank's full expand_query (expansion.cpp:67-83) -- same entries, 1/W of the
 * key switches below level log2(W). */
int cwg_expand_shard(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
                     const uint64_t* galois, uint32_t c, const uint64_t* query, uint32_t world, uint32_t rank,
                     uint64_t* out);
int cwg_answer_partial_shards(cwg_ctx* ctx, const uint64_t* shards, uint32_t world, uint32_t c, uint32_t m,
                              uint32_t op, uint64_t* dev_partial, cwg_timings* t);

/* compute_selection_vector (pir.cpp:277-312) without a payload (config 2): sel is
 * [n_local][3][L][N] in host memory or (single-device context) device memory -- then the tiles
 * are written in place with no copy back; comps (host) [r] receives 2 or 3 (a 2-component row
 * leaves slot 2 zero). */
int cwg_select(cwg_ctx* ctx, const uint64_t* relin, uint32_t n_galois, const uint64_t* galois_g,
               const uint64_t* galois, uint32_t h, uint32_t c, uint32_t m, const uint64_t* query,
               uint32_t op, uint64_t* sel, uint32_t* comps, cwg_timings* t);

/* ---- client side on the GPU, bit-identical to the reference client ---- */
/* pack_query_bits (expansion.cpp:17-38): the m query bits packed 2^c per plaintext (scaled by
 * 2^-c mod t) and encrypted (BfvBackend::encrypt, bfv.cpp:516-549) with the secret key sk (N ternary
 * coefficients) under encryption indices first_index, first_index + 1, ...; sk_seed: the 4 words
 * of the key's Seed256 (the reference's derive_seed domains 5 / 6).  out: [ceil(m / 2^c)][2][L][N]. */
int cwg_encrypt_query(cwg_ctx* ctx, const uint64_t* sk_seed, const int8_t* sk, const uint8_t* bits, uint32_t m,
                      uint32_t c, uint64_t first_index, uint64_t* out);
/* BfvBackend::decrypt (bfv.cpp:551-595) of count ciphertexts [count][comps][L][N] (comps 2 or 3) ->
 * out [count][N] plaintext coefficients mod t. */
int cwg_decrypt(cwg_ctx* ctx, const int8_t* sk, uint32_t count, uint32_t comps, const uint64_t* cts, uint64_t* out);

/* ---- stage entry points (the reference's unit-test surface) ---- */
/* RingContext::ntt_forward/inverse (ring.cpp:78-144) on `count` polys of chain prime
 * idx (chain=1) or of aux prime idx (chain=0; our internal basis). */
int cwg_ntt(cwg_ctx* ctx, int chain, uint32_t idx, uint64_t* data, uint32_t count, int inverse);
/* expand_query (expansion.cpp:67-83) with the resident keys: out [m][2][L][N]. */
int cwg_expand(cwg_ctx* ctx, uint32_t h, uint32_t c, uint32_t m, const uint64_t* query, uint64_t* out);
/* BfvBackend::mul_lazy (bfv.cpp:761-857) of count pairs of 2-comp ciphertexts: out [count][3][L][N]. */
int cwg_mul_lazy(cwg_ctx* ctx, uint32_t count, const uint64_t* a, const uint64_t* b, uint64_t* out);
/* BfvBackend::finalize / relinearize (bfv.cpp:859-875) with the resident relin key. */
int cwg_relinearize(cwg_ctx* ctx, uint32_t count, const uint64_t* ct3, uint64_t* out2);
/* BfvBackend::substitute (bfv.cpp:694-712) with the resident Galois key for g. */
int cwg_substitute(cwg_ctx* ctx, uint32_t count, const uint64_t* ct, uint64_t g, uint64_t* out);

/* Tuning / test options (defaults are the measured-fastest choices; no environment variables are
 * read by the library).  key: "streams" (row-tile streams, 1-4), "tile_rows" (0 = auto),
 * "fuse_mac" (0: separate selection NTT + MAC kernels), "mac" (0: k_mac2 instead of the TMA
 * payload MAC for s >= 3), "round" (0: IMAD rounding instead of the tensor cores), "round_g2",
 * "round_ctas", "mac_waves", "mac_ck", "ntt_np", "prescale", "ks32" (0: 64-bit key switching),
 * "ks_wide", "ks_ci", "ks_fixed" (0: run-time-shape key-switch MAC / CRT kernels), "ks_chunk_mb"
 * (scratch bound of one key-switch launch, default 3072), "prep_factors",
 * "lift_tc", "m2c_tc", "dec_tc" (0: the centred lift / MAC-basis -> chain conversion / digit
 * decomposition on the CUDA cores instead of the tensor cores), "mac_rows" (0: per-slice-group
 * payload MAC instead of the whole-row persistent kernel for s = 3, 5, 15), "mac_item_rows" (rows
 * per work item of that kernel), "mac_sg", "mac_stages",
 * "force_exact" (every rounding / lift decision through the exact multiword path; tests).
 * Unknown keys return CWG_EINVAL. */
int cwg_set_option(cwg_ctx* ctx, const char* key, int64_t value);
/* Kernel launch counter (all launches by this library since cwg_create). */
uint64_t cwg_kernel_launches(const cwg_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) so callers can record events on it. */
void* cwg_stream(const cwg_ctx* ctx);
/* Per-kernel CUDA-event timing of every launch (adds overhead; off by default; the row-tile
 * pipeline runs on one stream meanwhile, so each kernel is timed alone).  Turning it on or off
 * clears the statistics; cwg_kernel_stats enumerates (idx = 0, 1, ...) name, summed device time
 * and launch count, returning CWG_EINVAL past the end. */
int cwg_set_profiling(cwg_ctx* ctx, int on);
int cwg_kernel_stats(const cwg_ctx* ctx, uint32_t idx, char* name, uint32_t name_len, double* total_ms,
                     uint64_t* count);
/* Algorithmic work of kernel idx summed over its profiled launches: polynomials transformed
 * (NTT kernels), coefficients rounded (k_round_*), bytes streamed (k_mac: payload + selection
 * words).  Used for the roofline fractions in bench.py. */
int cwg_kernel_units(const cwg_ctx* ctx, uint32_t idx, double* units);

#ifdef __cplusplus
}
#endif
#endif /* CWGPU_H */

/*
 * cwgpu_client.h -- CPU client side used to produce benchmark inputs and check
 * outputs (key generation, query encryption, decryption).  Not on the server path.
 *
 * Replaces, for the harness only, the reference client calls
 *   BfvBackend(params, seed, galois_levels)   bfv.hpp:71 / bfv_keygen bfv.cpp:465-488
 *   pack_query_bits                           expansion.hpp:21 / expansion.cpp:17-38
 *   BfvBackend::encrypt / decrypt             bfv.cpp:521-595
 * Same seed => same keys as the reference; encrypt takes the randomness index that the
 * reference draws from a process-global counter (bfv.cpp:518-525).
 */
#ifndef CWGPU_CLIENT_H
#define CWGPU_CLIENT_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct cwg_client cwg_client;

const char* cwg_client_last_error(void);
cwg_client* cwg_client_create(uint32_t N, uint32_t L, const uint64_t* q, uint64_t t, uint32_t relin_digit_bits,
                              uint32_t galois_digit_bits, uint64_t seed, uint32_t galois_levels);
void cwg_client_destroy(cwg_client* c);
uint32_t cwg_client_digits(const cwg_client* c, int galois);
/* relin: [Dr][2][L][N]; galois: [galois_levels][Dg][2][L][N] (NTT form, reference layout) */
int cwg_client_export_keys(const cwg_client* c, uint64_t* relin, uint64_t* galois);
int cwg_client_encrypt(const cwg_client* c, const uint64_t* plain, uint64_t index, uint64_t* out);
/* h = ceil(m / 2^c) ciphertexts [h][2][L][N]; ciphertext i uses randomness index first_index + i */
int cwg_client_pack_query(const cwg_client* c, const uint8_t* bits, uint32_t m, uint32_t c_factor,
                          uint64_t first_index, uint64_t* out);
int cwg_client_decrypt(const cwg_client* c, const uint64_t* ct, uint32_t comps, uint64_t* out);
/* The secret key (N ternary coefficients) and its Seed256 words, for the GPU client calls of
 * include/cwgpu.h (cwg_encrypt_query / cwg_decrypt). */
int cwg_client_export_secret(const cwg_client* c, int8_t* s, uint64_t* seed_words);

#ifdef __cplusplus
}
#endif
#endif

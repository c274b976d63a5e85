/*
 * ckks_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, scalar, single-threaded restatement of the reference CKKS/RNS
 * hot path (arxiv/paper_1810_10121 "hegraph", proj/include/heg/ckks/*.hpp and
 * proj/include/heg/common.hpp).  It is the CHECKER the CUDA product is compared
 * against; it is never linked into, called by, or shipped with the product
 * library (libhegpu.so).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.
 *
 * Parity of this restatement is pinned (tests/test_oracle.py) against
 *   - the reference's own known-answer tests (test_ring.cpp:129-142, 159-166;
 *     test_ckks.cpp:95-110; test_ring.cpp:187-196), and
 *   - golden vectors produced by the reference itself compiled from
 *     /root/reference (oracle/_ref, recipe oracle/Makefile, generator
 *     tests/golden/make_golden.py).
 *
 * Layout conventions (shared with the product): a polynomial at level l is
 * (l+1) residue rows of n uint64 words, row i modulo prime i.  A size-s
 * ciphertext is s such polynomials back to back.
 */
#ifndef CKKS_ORACLE_H
#define CKKS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OC_MAX_PRIMES 64

/* ---- deterministic RNG (common.hpp:71-122) ---- */
typedef struct { uint64_t state; } oc_rng;
uint64_t oc_splitmix64(uint64_t* state);
void oc_rng_init(oc_rng* r, uint64_t seed);
uint64_t oc_rng_next(oc_rng* r);
double oc_rng_uniform(oc_rng* r);
uint64_t oc_rng_uniform_int(oc_rng* r, uint64_t n);
double oc_rng_gaussian(oc_rng* r);
oc_rng oc_rng_fork(const oc_rng* r, uint64_t label);
oc_rng oc_rng_fork_str(const oc_rng* r, const char* label);
/* expose the raw state (for the product-side counter-based sampler tests) */
uint64_t oc_rng_state(const oc_rng* r);

/* ---- modular arithmetic (ring.hpp:37-111) ---- */
typedef struct { uint64_t value, ratio_hi, ratio_lo; } oc_mod;
void oc_mod_init(oc_mod* m, uint64_t q);
uint64_t oc_mod_mul(const oc_mod* m, uint64_t a, uint64_t b);
uint64_t oc_mod_shoup(const oc_mod* m, uint64_t w);
uint64_t oc_mod_mul_shoup(const oc_mod* m, uint64_t x, uint64_t w, uint64_t ws);
uint64_t oc_mod_pow(const oc_mod* m, uint64_t b, uint64_t e);
uint64_t oc_mod_inv(const oc_mod* m, uint64_t a);

/* ---- primes (ring.hpp:137-196) ---- */
int oc_is_prime(uint64_t n);
/* returns 0 on success, -1 if no prime found / bad args */
int oc_generate_primes(int64_t n, const int* bits, int count, uint64_t* out);

/* ---- context: primes + NTT tables (context.hpp:90-109, ring.hpp:221-257) ---- */
typedef struct oc_ctx oc_ctx;
oc_ctx* oc_ctx_create(int64_t n, const int* bits, int count, int scale_bits);
void oc_ctx_free(oc_ctx* c);
int64_t oc_ctx_n(const oc_ctx* c);
int oc_ctx_count(const oc_ctx* c);
uint64_t oc_ctx_prime(const oc_ctx* c, int i);
/* copies psi_brv, psi_brv_shoup, ipsi_brv, ipsi_brv_shoup (4*n words) and n_inv */
void oc_ctx_tables(const oc_ctx* c, int i, uint64_t* out4n, uint64_t* ninv2);

void oc_ntt_forward(const oc_ctx* c, int limb, uint64_t* a);   /* ring.hpp:263-279 */
void oc_ntt_inverse(const oc_ctx* c, int limb, uint64_t* a);   /* ring.hpp:282-301 */
void oc_negacyclic_schoolbook(const oc_mod* q, int64_t n, const uint64_t* a, const uint64_t* b, uint64_t* out);

/* ---- CRT (ring.hpp:438-480) ---- */
/* residues[i] for i < count, moduli primes[0..count) -> centred double */
double oc_crt_centered(const uint64_t* primes, int count, const uint64_t* residues);

/* ---- slot encoder (encoder.hpp:38-115) ---- */
void oc_encode_values(int64_t n, const double* values, int64_t count, double* coeffs_out);
void oc_decode_coeffs(int64_t n, const double* coeffs, int64_t count, double* values_out);

/* ---- polynomials / samplers (poly.hpp) ---- */
void oc_poly_to_ntt(const oc_ctx* c, int level, uint64_t* p);
void oc_poly_to_coeff(const oc_ctx* c, int level, uint64_t* p);
void oc_poly_rescale(const oc_ctx* c, int level, int ntt_form, const uint64_t* in, uint64_t* out);
void oc_sample_ternary(const oc_ctx* c, int level, oc_rng* r, uint64_t* out);
void oc_sample_gaussian(const oc_ctx* c, int level, double sigma, oc_rng* r, uint64_t* out);
void oc_sample_uniform(const oc_ctx* c, int level, oc_rng* r, uint64_t* out);

/* ---- keys (ckks_backend.hpp:39-114) ---- */
int oc_relin_digit_count(uint64_t q);
/* total relin (i,d) rows */
int oc_relin_rows(const oc_ctx* c);
typedef struct oc_keys oc_keys;
oc_keys* oc_keys_generate(const oc_ctx* c, uint64_t seed, int with_relin);
void oc_keys_free(oc_keys* k);
/* NTT-form full-chain polys: (L+1)*n words each */
const uint64_t* oc_keys_secret(const oc_keys* k);
const uint64_t* oc_keys_pk_b(const oc_keys* k);
const uint64_t* oc_keys_pk_a(const oc_keys* k);
/* relin row r (ordered i-major, d-minor): b then a */
const uint64_t* oc_keys_relin_b(const oc_keys* k, int row);
const uint64_t* oc_keys_relin_a(const oc_keys* k, int row);

/* ---- scheme operations (ckks_backend.hpp) ----
 * All ciphertexts/plaintexts in NTT form (the reference default, ckks_backend.hpp:160).
 * ct buffers: size * (level+1) * n words. Return 0 ok, nonzero = error code. */
int oc_encode(const oc_ctx* c, const double* values, int64_t count, int level, double scale, uint64_t* pt_out);
int oc_encode_constant(const oc_ctx* c, double value, int level, double scale, uint64_t* pt_out);
void oc_encrypt_zero(const oc_ctx* c, const oc_keys* k, int level, uint64_t seed, uint64_t* ct_out);
void oc_encrypt(const oc_ctx* c, const oc_keys* k, const uint64_t* pt, int level, uint64_t seed, uint64_t* ct_out);
/* decrypt a size-s ct at level -> count decoded doubles (before /scale is applied: pass scale) */
void oc_decrypt(const oc_ctx* c, const oc_keys* k, const uint64_t* ct, int size, int level, double scale,
                int64_t count, double* out);
void oc_decrypt_coeffs(const oc_ctx* c, const oc_keys* k, const uint64_t* ct, int size, int level, uint64_t* m_out);
void oc_add(const oc_ctx* c, int level, int64_t words, const uint64_t* a, const uint64_t* b, uint64_t* out);
void oc_sub(const oc_ctx* c, int level, int64_t words, const uint64_t* a, const uint64_t* b, uint64_t* out);
void oc_negate(const oc_ctx* c, int level, int64_t words, const uint64_t* a, uint64_t* out);
void oc_mul_plain(const oc_ctx* c, int level, int size, const uint64_t* ct, const uint64_t* pt, uint64_t* out);
/* size-2 x size-2 -> relinearized size-2 (keys with relin) at the same level */
void oc_multiply_relin(const oc_ctx* c, const oc_keys* k, int level, const uint64_t* x, const uint64_t* y,
                       uint64_t* out);
void oc_multiply_norelin(const oc_ctx* c, int level, const uint64_t* x, const uint64_t* y, uint64_t* out3);
void oc_relinearize(const oc_ctx* c, const oc_keys* k, int level, const uint64_t* in3, uint64_t* out2);
void oc_rescale_ct(const oc_ctx* c, int level, int size, const uint64_t* in, uint64_t* out);
/* fused weighted sum (ckks_backend.hpp:381-411): xs[t] size-2 at level, weights as scalars
 * encoded with encode_constant(w[t], level, q_level); output rescaled to level-1. */
/* sum_t x_t (x) w_t (size 3), relinearised once, rescaled: ct x ct weighted sum (ckks_backend.hpp:413-450) */
void oc_weighted_sum_cipher(const oc_ctx* c, const oc_keys* k, int level, int terms, const uint64_t* const* xs,
                            const uint64_t* const* ws, uint64_t* out);
int oc_weighted_sum(const oc_ctx* c, int level, int terms, const uint64_t* const* xs, const double* w,
                    uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * dilithium_oracle.h -- CPU oracle for the batched Dilithium hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference's
 * round-3 Dilithium algorithm (reference: the headers under proj/include/dilithium).  It is
 * the checker for the CUDA engine: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * (paper_2211_12265_b200/csrc) never links, includes or calls anything here.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function below
 * against the reference's own known-answer vectors (tests/golden/ref_kat.json,
 * extracted from proj/tests/vectors/ref_vectors.hpp) and against outputs of the
 * unmodified reference headers compiled in place (oracle/_ref/).
 */
#ifndef DILITHIUM_ORACLE_H
#define DILITHIUM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_Q 8380417
#define ORC_N 256

typedef struct {
  int level, k, l, eta, tau, beta, gamma1, gamma2, omega;
  int eta_bits, z_bits, w1_bits;
  size_t pk_bytes, sk_bytes, sig_bytes;
  int mldsa;              /* 1 = FIPS 204 hashing conventions (levels 44 / 65 / 87) */
  int tr_bytes, ct_bytes; /* 32, 32 for round 3; 64 and lambda/4 for FIPS 204 */
} orc_params;

/* level in {2,3,5} (the reference's round-3 parameter sets; params.hpp:53-55,91-106) or
 * {44,65,87} (ML-DSA-44/65/87, FIPS 204 -- NOT in the reference, which declares it a
 * non-goal: restated from the standard, keygen and verify pinned against OpenSSL 4.0 through
 * the fixtures of tests/golden/make_mldsa_golden.py; deterministic signing with an empty
 * context only, its signature bytes are cross-verified but have no independent KAT);
 * returns NULL otherwise */
const orc_params* orc_get_params(int level);

/* keccak.hpp:70-93 */
void orc_keccak_f1600(uint64_t state[25]);
/* keccak.hpp:174-184; rate 168 / 136 */
void orc_shake128(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen);
void orc_shake256(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen);

/* sampling.hpp:42-56, 61-79, 83-92, 97-120 */
void orc_expand_a(int32_t out[256], const uint8_t rho[32], unsigned i, unsigned j);
void orc_expand_s(int32_t out[256], const uint8_t rho_prime[64], unsigned nonce, int eta);
void orc_expand_mask(int32_t out[256], const uint8_t rho_prime[64], unsigned nonce, int gamma1,
                     int z_bits);
void orc_sample_in_ball(int32_t out[256], const uint8_t c_tilde[32], int tau);

/* ntt.hpp:74-126 -- value semantics only: outputs are canonical in [0,q) */
void orc_ntt(int32_t a[256]);
void orc_intt(int32_t a[256]);

/* rounding.hpp:13-59 */
void orc_power2round(int32_t a, int32_t* a1, int32_t* a0);
void orc_decompose(int32_t r, int32_t gamma2, int32_t* r1, int32_t* r0);
int orc_make_hint(int32_t z, int32_t r, int32_t gamma2);
int32_t orc_use_hint(int h, int32_t r, int32_t gamma2);

/* FIPS 204 context string used by sign / verify at levels 44 / 65 / 87 (len <= 255; default
 * empty; process-wide, not thread-safe -- tests only) */
int orc_set_mldsa_context(const uint8_t* ctx, size_t len);
/* HashML-DSA (FIPS 204 Alg. 4 / 5): M' = 1 || len || ctx || OID || PH(M); messages are digests */
int orc_set_mldsa_prehash(const uint8_t* ctx, size_t len, const uint8_t* oid, size_t oid_len);

/* scheme.hpp:68-104 */
int orc_keygen(int level, const uint8_t zeta[32], uint8_t* pk, uint8_t* sk);
/* scheme.hpp:253-273 (make_precomp + sign_with_precomp).  rho_prime_override may be
 * NULL.  Returns 0 on success, -1 malformed sk (packing.hpp:79-86,215-233), -2 if the
 * loop exceeds 2^14 attempts.  *attempts = winning attempt ordinal (1-based). */
int orc_sign(int level, const uint8_t* sk, const uint8_t* msg, size_t msglen,
             const uint8_t* rho_prime_override, uint8_t* sig, uint32_t* attempts);
/* scheme.hpp:277-318; returns 1 accept / 0 reject; never fails otherwise */
int orc_verify(int level, const uint8_t* pk, size_t pklen, const uint8_t* msg, size_t msglen,
               const uint8_t* sig, size_t siglen);

/* scheme.hpp:133-219 one rejection-loop iteration.  Returns 1 accepted, 0 rejected;
 * *stage = 0 ZNorm, 1 R0Norm, 2 VtNorm, 3 HintWeight when rejected.  z (l*256,
 * centered) and hints (k*256) are filled as far as the reference computes them.
 * c_tilde: ct_bytes (32; up to 64 for the FIPS 204 levels). */
int orc_sign_attempt(int level, const uint8_t* sk, const uint8_t mu[64],
                     const uint8_t rho_prime[64], uint32_t kappa, int* stage,
                     uint8_t* c_tilde, int32_t* z, int32_t* hints);

/* detail::sign_attempt_bounded (scheme.hpp:133-138): the same with the norm bounds injected */
int orc_sign_attempt_bounded(int level, const uint8_t* sk, const uint8_t mu[64],
                             const uint8_t rho_prime[64], uint32_t kappa, int32_t z_bound,
                             int32_t r0_bound, int32_t vt_bound, int* stage, uint8_t* c_tilde,
                             int32_t* z, int32_t* hints);

#ifdef __cplusplus
}
#endif
#endif

/*
 * dilithium_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see dilithium_oracle.h).
 *
 * A definitional restatement of the reference's round-3 Dilithium: plain `% q`
 * arithmetic instead of the reference's Montgomery forms, textbook rounding
 * instead of its branch-free magic constants.  Only canonical values reach the
 * codecs and hashes, so byte outputs are identical;
 * tests/test_oracle.py pins that against the reference's KATs and against the
 * reference itself (oracle/_ref).  Every function cites the reference lines it
 * restates, relative to /root/reference/proj/include/dilithium/.
 */
#include "dilithium_oracle.h"

#include <stdlib.h>
#include <string.h>

#define Q ORC_Q
#define N ORC_N

/* ------------------------------------------------------------------ params */

static const orc_params kParams[6] = {
    /* params.hpp:53 */
    {2, 4, 4, 2, 39, 78, 1 << 17, (Q - 1) / 88, 80, 3, 18, 6, 1312, 2528, 2420, 0, 32, 32},
    /* params.hpp:54 */
    {3, 6, 5, 4, 49, 196, 1 << 19, (Q - 1) / 32, 55, 4, 20, 4, 1952, 4000, 3293, 0, 32, 32},
    /* params.hpp:55 */
    {5, 8, 7, 2, 60, 120, 1 << 19, (Q - 1) / 32, 75, 3, 20, 4, 2592, 4864, 4595, 0, 32, 32},
    /* FIPS 204 table 1 / table 2 (ML-DSA-44 / 65 / 87): same ring and bounds; tr is 64
     * bytes, c~ is lambda/4 = 32 / 48 / 64 bytes.  Not part of the reference (its README
     * declares FIPS 204 a non-goal); restated from the standard, see the header. */
    {44, 4, 4, 2, 39, 78, 1 << 17, (Q - 1) / 88, 80, 3, 18, 6, 1312, 2560, 2420, 1, 64, 32},
    {65, 6, 5, 4, 49, 196, 1 << 19, (Q - 1) / 32, 55, 4, 20, 4, 1952, 4032, 3309, 1, 64, 48},
    {87, 8, 7, 2, 60, 120, 1 << 19, (Q - 1) / 32, 75, 3, 20, 4, 2592, 4896, 4627, 1, 64, 64},
};

const orc_params* orc_get_params(int level) {
  for (int i = 0; i < 6; ++i)
    if (kParams[i].level == level) return &kParams[i];
  return NULL;
}

/* ------------------------------------------------------------------ keccak */

/* FIPS 202 iota constants; the reference derives the same table from the rc()
 * LFSR at compile time (keccak.hpp:27-42). */
static const uint64_t kIota[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull, 0x8000000080008000ull,
    0x000000000000808bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800aull, 0x800000008000000aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

static uint64_t rol64(uint64_t v, unsigned r) { return r ? (v << r) | (v >> (64 - r)) : v; }

/* keccak.hpp:70-93.  Written from the FIPS 202 step definitions: lane (x,y) at
 * index x+5y; rho offsets by the (t+1)(t+2)/2 walk; pi: B[y][2x+3y] = A[x][y]. */
void orc_keccak_f1600(uint64_t A[25]) {
  unsigned rho[25];
  rho[0] = 0;
  {
    unsigned x = 1, y = 0;
    for (unsigned t = 0; t < 24; ++t) {
      rho[x + 5 * y] = ((t + 1) * (t + 2) / 2) % 64;
      unsigned nx = y, ny = (2 * x + 3 * y) % 5;
      x = nx;
      y = ny;
    }
  }
  for (int round = 0; round < 24; ++round) {
    uint64_t C[5], B[25];
    for (int x = 0; x < 5; ++x) C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];
    for (int x = 0; x < 5; ++x) {
      uint64_t D = C[(x + 4) % 5] ^ rol64(C[(x + 1) % 5], 1);
      for (int y = 0; y < 5; ++y) A[x + 5 * y] ^= D;
    }
    for (int x = 0; x < 5; ++x)
      for (int y = 0; y < 5; ++y) B[y + 5 * ((2 * x + 3 * y) % 5)] = rol64(A[x + 5 * y], rho[x + 5 * y]);
    for (int y = 0; y < 5; ++y)
      for (int x = 0; x < 5; ++x)
        A[x + 5 * y] = B[x + 5 * y] ^ (~B[(x + 1) % 5 + 5 * y] & B[(x + 2) % 5 + 5 * y]);
    A[0] ^= kIota[round];
  }
}

/* keccak.hpp:98-172: sponge with byte position, pad 0x1F .. 0x80, resumable squeeze */
typedef struct {
  uint64_t s[25];
  size_t rate, pos;
  int squeezing;
} xof_t;

static void xof_init(xof_t* x, size_t rate) {
  memset(x, 0, sizeof *x);
  x->rate = rate;
}

static void xof_absorb(xof_t* x, const uint8_t* in, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    if (x->pos == x->rate) {
      orc_keccak_f1600(x->s);
      x->pos = 0;
    }
    x->s[x->pos / 8] ^= (uint64_t)in[i] << (8 * (x->pos % 8));
    x->pos++;
  }
}

static void xof_finalize(xof_t* x) {
  if (x->pos == x->rate) {
    orc_keccak_f1600(x->s);
    x->pos = 0;
  }
  x->s[x->pos / 8] ^= (uint64_t)0x1F << (8 * (x->pos % 8));
  x->s[(x->rate - 1) / 8] ^= (uint64_t)0x80 << (8 * ((x->rate - 1) % 8));
  x->pos = x->rate;
  x->squeezing = 1;
}

static void xof_squeeze(xof_t* x, uint8_t* out, size_t n) {
  if (!x->squeezing) xof_finalize(x);
  for (size_t i = 0; i < n; ++i) {
    if (x->pos == x->rate) {
      orc_keccak_f1600(x->s);
      x->pos = 0;
    }
    out[i] = (uint8_t)(x->s[x->pos / 8] >> (8 * (x->pos % 8)));
    x->pos++;
  }
}

void orc_shake128(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen) {
  xof_t x;
  xof_init(&x, 168);
  xof_absorb(&x, in, inlen);
  xof_squeeze(&x, out, outlen);
}

void orc_shake256(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen) {
  xof_t x;
  xof_init(&x, 136);
  xof_absorb(&x, in, inlen);
  xof_squeeze(&x, out, outlen);
}

/* hash_h of two concatenated parts (keccak.hpp:187-198) */
static void hash2(uint8_t* out, size_t outlen, const uint8_t* a, size_t alen, const uint8_t* b,
                  size_t blen) {
  xof_t x;
  xof_init(&x, 136);
  xof_absorb(&x, a, alen);
  xof_absorb(&x, b, blen);
  xof_squeeze(&x, out, outlen);
}

/* ---------------------------------------------------------------- samplers */

/* sampling.hpp:28-34: seed || nonce as two little-endian bytes */
static void seeded_xof(xof_t* x, size_t rate, const uint8_t* seed, size_t seedlen,
                       unsigned nonce) {
  uint8_t n[2] = {(uint8_t)nonce, (uint8_t)(nonce >> 8)};
  xof_init(x, rate);
  xof_absorb(x, seed, seedlen);
  xof_absorb(x, n, 2);
}

/* sampling.hpp:42-56: SHAKE128, 3-byte LE candidates masked to 23 bits, keep < q.
 * Nonce = (i << 8) | j, row in the high byte. */
void orc_expand_a(int32_t out[256], const uint8_t rho[32], unsigned i, unsigned j) {
  xof_t x;
  seeded_xof(&x, 168, rho, 32, ((i << 8) | j) & 0xFFFF);
  int ctr = 0;
  while (ctr < N) {
    uint8_t b[3];
    xof_squeeze(&x, b, 3);
    int32_t t = (b[0] | (b[1] << 8) | (b[2] << 16)) & 0x7FFFFF;
    if (t < Q) out[ctr++] = t;
  }
}

/* sampling.hpp:61-79: SHAKE256, low nibble first then high; eta=2 keeps <15 and
 * maps 2-(t mod 5); eta=4 keeps <9 and maps 4-t. */
void orc_expand_s(int32_t out[256], const uint8_t rho_prime[64], unsigned nonce, int eta) {
  xof_t x;
  seeded_xof(&x, 136, rho_prime, 64, nonce & 0xFFFF);
  int ctr = 0;
  while (ctr < N) {
    uint8_t b;
    xof_squeeze(&x, &b, 1);
    int nib[2] = {b & 0xF, b >> 4};
    for (int h = 0; h < 2 && ctr < N; ++h) {
      int t = nib[h];
      if (eta == 2) {
        if (t < 15) out[ctr++] = 2 - t % 5;
      } else {
        if (t < 9) out[ctr++] = 4 - t;
      }
    }
  }
}

/* LSB-first little-endian bit stream reader (packing.hpp:35-52) */
static uint32_t get_bits(const uint8_t* in, size_t idx, int width) {
  uint32_t v = 0;
  size_t bit = idx * (size_t)width;
  for (int b = 0; b < width; ++b, ++bit) v |= (uint32_t)((in[bit >> 3] >> (bit & 7)) & 1) << b;
  return v;
}

/* LSB-first writer (packing.hpp:16-33); out must be zeroed */
static void put_bits(uint8_t* out, size_t idx, int width, uint32_t v) {
  size_t bit = idx * (size_t)width;
  for (int b = 0; b < width; ++b, ++bit) out[bit >> 3] |= (uint8_t)(((v >> b) & 1) << (bit & 7));
}

/* sampling.hpp:83-92: squeeze 32*z_bits bytes, decode gamma1 - raw (packing.hpp:92-94) */
void orc_expand_mask(int32_t out[256], const uint8_t rho_prime[64], unsigned nonce, int gamma1,
                     int z_bits) {
  xof_t x;
  uint8_t buf[640];
  seeded_xof(&x, 136, rho_prime, 64, nonce & 0xFFFF);
  xof_squeeze(&x, buf, (size_t)32 * z_bits);
  for (int i = 0; i < N; ++i) out[i] = gamma1 - (int32_t)get_bits(buf, i, z_bits);
}

/* sampling.hpp:97-120: 8 sign bytes (LE, consumed LSB first), then for
 * i = 256-tau..255 draw byte b <= i (reject b > i); c[i] = c[b]; c[b] = +-1. */
static void sample_in_ball_n(int32_t out[256], const uint8_t* c_tilde, size_t ct_len, int tau);
void orc_sample_in_ball(int32_t out[256], const uint8_t c_tilde[32], int tau) {
  sample_in_ball_n(out, c_tilde, 32, tau);
}
/* FIPS 204 Alg. 29 absorbs the whole commitment hash (lambda/4 bytes) */
static void sample_in_ball_n(int32_t out[256], const uint8_t* c_tilde, size_t ct_len, int tau) {
  xof_t x;
  uint8_t sb[8];
  xof_init(&x, 136);
  xof_absorb(&x, c_tilde, ct_len);
  xof_squeeze(&x, sb, 8);
  uint64_t signs = 0;
  for (int i = 0; i < 8; ++i) signs |= (uint64_t)sb[i] << (8 * i);
  memset(out, 0, 256 * sizeof(int32_t));
  for (int i = N - tau; i < N; ++i) {
    uint8_t b;
    do xof_squeeze(&x, &b, 1);
    while (b > i);
    out[i] = out[b];
    out[b] = (signs & 1) ? -1 : 1;
    signs >>= 1;
  }
}

/* -------------------------------------------------------------------- ring */

static int32_t modq(int64_t a) {
  int64_t r = a % Q;
  return (int32_t)(r < 0 ? r + Q : r);
}

/* centered representative in (-(q+1)/2, q/2]  (reduce.hpp:58-65) */
static int32_t centered(int64_t a) {
  int32_t r = modq(a);
  return r > (Q - 1) / 2 ? r - Q : r;
}

static int32_t powq(int64_t b, unsigned e) {
  int64_t acc = 1;
  b = modq(b);
  while (e) {
    if (e & 1) acc = acc * b % Q;
    b = b * b % Q;
    e >>= 1;
  }
  return (int32_t)acc;
}

static int32_t g_zeta[256]; /* psi^brv8(k), plain domain (ntt.hpp:48-59 without the R factor) */
static int g_zeta_ready = 0;

static void init_zetas(void) {
  if (g_zeta_ready) return;
  for (unsigned k = 0; k < 256; ++k) {
    unsigned r = 0;
    for (int b = 0; b < 8; ++b) r |= ((k >> b) & 1u) << (7 - b);
    g_zeta[k] = powq(1753, r); /* ntt.hpp:14 */
  }
  g_zeta_ready = 1;
}

/* ntt.hpp:74-86: Cooley-Tukey, len 128..1, zeta index pre-incremented */
void orc_ntt(int32_t a[256]) {
  init_zetas();
  unsigned k = 0;
  for (unsigned len = 128; len > 0; len >>= 1)
    for (unsigned start = 0; start < N; start += 2 * len) {
      int64_t z = g_zeta[++k];
      for (unsigned j = start; j < start + len; ++j) {
        int32_t t = modq(z * a[j + len]);
        a[j + len] = modq((int64_t)a[j] - t);
        a[j] = modq((int64_t)a[j] + t);
      }
    }
}

/* ntt.hpp:92-110: Gentleman-Sande with twiddle -zeta, n^{-1} applied at the end
 * (the reference fuses it into the last level; same value mod q) */
void orc_intt(int32_t a[256]) {
  init_zetas();
  unsigned k = 256;
  for (unsigned len = 1; len < N; len <<= 1)
    for (unsigned start = 0; start < N; start += 2 * len) {
      int64_t z = Q - g_zeta[--k];
      for (unsigned j = start; j < start + len; ++j) {
        int32_t t = a[j];
        a[j] = modq((int64_t)t + a[j + len]);
        a[j + len] = modq(z * modq((int64_t)t - a[j + len]));
      }
    }
  int64_t ninv = powq(256, Q - 2);
  for (int i = 0; i < N; ++i) a[i] = modq(ninv * a[i]);
}

/* ---------------------------------------------------------------- rounding */

/* rounding.hpp:13-16 */
void orc_power2round(int32_t a, int32_t* a1, int32_t* a0) {
  int32_t lo = a % 8192;
  if (lo > 4096) lo -= 8192;
  *a0 = lo;
  *a1 = (a - lo) / 8192;
}

/* rounding.hpp:22-34, textbook form: r0 = r mod+- 2*gamma2, corner r-r0 = q-1 */
void orc_decompose(int32_t r, int32_t gamma2, int32_t* r1, int32_t* r0) {
  int32_t alpha = 2 * gamma2;
  int32_t lo = r % alpha;
  if (lo > gamma2) lo -= alpha;
  if (r - lo == Q - 1) {
    *r1 = 0;
    *r0 = lo - 1;
  } else {
    *r1 = (r - lo) / alpha;
    *r0 = lo;
  }
}

static int32_t highbits(int32_t r, int32_t gamma2) {
  int32_t r1, r0;
  orc_decompose(r, gamma2, &r1, &r0);
  return r1;
}

/* rounding.hpp:46-50 */
int orc_make_hint(int32_t z, int32_t r, int32_t gamma2) {
  return highbits(r, gamma2) != highbits(modq((int64_t)r + z), gamma2);
}

/* rounding.hpp:53-59 */
int32_t orc_use_hint(int h, int32_t r, int32_t gamma2) {
  int32_t m = (Q - 1) / (2 * gamma2), r1, r0;
  orc_decompose(r, gamma2, &r1, &r0);
  if (!h) return r1;
  if (r0 > 0) return (r1 + 1) % m;
  return (r1 + m - 1) % m;
}

/* rounding.hpp:64-74: 1 = some |centered(c)| >= bound */
static int norm_ge(const int32_t* f, int32_t bound) {
  for (int i = 0; i < N; ++i) {
    int32_t c = centered(f[i]);
    if (abs(c) >= bound) return 1;
  }
  return 0;
}

/* ------------------------------------------------------------------ codecs */

static void pack_poly(uint8_t* out, const int32_t* f, int width, int32_t bias /* raw = bias - c */,
                      int negate) {
  memset(out, 0, (size_t)N * width / 8);
  for (int i = 0; i < N; ++i) put_bits(out, i, width, (uint32_t)(negate ? bias - f[i] : f[i]));
}

/* packing.hpp:56-98 field encodings */
static void pack_t1(uint8_t* o, const int32_t* f) { pack_poly(o, f, 10, 0, 0); }
static void pack_t0(uint8_t* o, const int32_t* f) { pack_poly(o, f, 13, 4096, 1); }
static void pack_eta(uint8_t* o, const int32_t* f, const orc_params* P) {
  pack_poly(o, f, P->eta_bits, P->eta, 1);
}
static void pack_z(uint8_t* o, const int32_t* f, const orc_params* P) {
  pack_poly(o, f, P->z_bits, P->gamma1, 1);
}
static void pack_w1(uint8_t* o, const int32_t* f, const orc_params* P) {
  pack_poly(o, f, P->w1_bits, 0, 0);
}

/* packing.hpp:105-118 */
static void encode_hint(uint8_t* out, const int32_t* h, const orc_params* P) {
  memset(out, 0, (size_t)P->omega + P->k);
  int ctr = 0;
  for (int i = 0; i < P->k; ++i) {
    for (int j = 0; j < N; ++j)
      if (h[i * N + j]) out[ctr++] = (uint8_t)j;
    out[P->omega + i] = (uint8_t)ctr;
  }
}

/* packing.hpp:122-140: strict; returns 0 on malformed input */
static int decode_hint(int32_t* h, const uint8_t* in, const orc_params* P) {
  memset(h, 0, (size_t)P->k * N * sizeof(int32_t));
  int ctr = 0;
  for (int i = 0; i < P->k; ++i) {
    int cnt = in[P->omega + i];
    if (cnt < ctr || cnt > P->omega) return 0;
    for (int j = ctr; j < cnt; ++j) {
      if (j > ctr && in[j] <= in[j - 1]) return 0;
      h[i * N + in[j]] = 1;
    }
    ctr = cnt;
  }
  for (int j = ctr; j < P->omega; ++j)
    if (in[j]) return 0;
  return 1;
}

/* ------------------------------------------------------------------ scheme */

#define KMAX 8
#define LMAX 7

typedef struct {
  uint8_t rho[32], key[32], tr[64];
  int32_t s1[LMAX][N], s2[KMAX][N], t0[KMAX][N];
} sk_view;

/* packing.hpp:215-233 incl. the eta range check :79-86 */
static int unpack_sk(sk_view* v, const uint8_t* sk, const orc_params* P) {
  memcpy(v->rho, sk, 32);
  memcpy(v->key, sk + 32, 32);
  memcpy(v->tr, sk + 64, (size_t)P->tr_bytes);
  size_t off = 64 + (size_t)P->tr_bytes, eb = (size_t)N * P->eta_bits / 8;
  int ok = 1;
  for (int i = 0; i < P->l; ++i, off += eb)
    for (int m = 0; m < N; ++m) {
      uint32_t r = get_bits(sk + off, m, P->eta_bits);
      if (r > 2u * P->eta) ok = 0;
      v->s1[i][m] = P->eta - (int32_t)r;
    }
  for (int i = 0; i < P->k; ++i, off += eb)
    for (int m = 0; m < N; ++m) {
      uint32_t r = get_bits(sk + off, m, P->eta_bits);
      if (r > 2u * P->eta) ok = 0;
      v->s2[i][m] = P->eta - (int32_t)r;
    }
  for (int i = 0; i < P->k; ++i, off += 416)
    for (int m = 0; m < N; ++m) v->t0[i][m] = 4096 - (int32_t)get_bits(sk + off, m, 13);
  return ok;
}

/* out = A * v in the NTT domain, A expanded on the fly (polyvec.hpp:65-89 with the
 * supplier of scheme.hpp:49-55); vhat canonical, out canonical */
static void matvec(int32_t out[][N], const uint8_t rho[32], int32_t vhat[][N],
                   const orc_params* P) {
  int32_t a[N];
  for (int i = 0; i < P->k; ++i) {
    memset(out[i], 0, sizeof(int32_t) * N);
    for (int j = 0; j < P->l; ++j) {
      orc_expand_a(a, rho, (unsigned)i, (unsigned)j);
      for (int m = 0; m < N; ++m) out[i][m] = modq(out[i][m] + (int64_t)a[m] * vhat[j][m]);
    }
  }
}

/* scheme.hpp:68-104 */
int orc_keygen(int level, const uint8_t zeta[32], uint8_t* pk, uint8_t* sk) {
  const orc_params* P = orc_get_params(level);
  if (!P) return -1;
  uint8_t seed[128];
  if (P->mldsa) { /* FIPS 204 Alg. 6 line 1: H(xi || k || l, 128) */
    const uint8_t kl[2] = {(uint8_t)P->k, (uint8_t)P->l};
    hash2(seed, 128, zeta, 32, kl, 2);
  } else {
    orc_shake256(seed, 128, zeta, 32);
  }
  const uint8_t *rho = seed, *rho_prime = seed + 32, *key = seed + 96; /* scheme.hpp:70-76 */
  static _Thread_local int32_t s1[LMAX][N], s2[KMAX][N], s1h[LMAX][N], t[KMAX][N], t1[KMAX][N],
      t0[KMAX][N];
  for (int i = 0; i < P->l; ++i) orc_expand_s(s1[i], rho_prime, (unsigned)i, P->eta);
  for (int i = 0; i < P->k; ++i) orc_expand_s(s2[i], rho_prime, (unsigned)(P->l + i), P->eta);
  for (int i = 0; i < P->l; ++i) {
    for (int m = 0; m < N; ++m) s1h[i][m] = modq(s1[i][m]);
    orc_ntt(s1h[i]);
  }
  matvec(t, rho, s1h, P);
  for (int i = 0; i < P->k; ++i) {
    orc_intt(t[i]);
    for (int m = 0; m < N; ++m) {
      int32_t c = modq((int64_t)t[i][m] + s2[i][m]); /* scheme.hpp:94 */
      orc_power2round(c, &t1[i][m], &t0[i][m]);
    }
  }
  memcpy(pk, rho, 32);
  for (int i = 0; i < P->k; ++i) pack_t1(pk + 32 + 320 * i, t1[i]);
  uint8_t tr[64];
  orc_shake256(tr, (size_t)P->tr_bytes, pk, P->pk_bytes); /* scheme.hpp:102 */
  memcpy(sk, rho, 32);
  memcpy(sk + 32, key, 32);
  memcpy(sk + 64, tr, (size_t)P->tr_bytes);
  size_t off = 64 + (size_t)P->tr_bytes, eb = (size_t)N * P->eta_bits / 8;
  for (int i = 0; i < P->l; ++i, off += eb) pack_eta(sk + off, s1[i], P);
  for (int i = 0; i < P->k; ++i, off += eb) pack_eta(sk + off, s2[i], P);
  for (int i = 0; i < P->k; ++i, off += 416) pack_t0(sk + off, t0[i]);
  return 0;
}

typedef struct {
  sk_view v;
  int32_t s1h[LMAX][N], s2h[KMAX][N], t0h[KMAX][N];
} precomp;

/* scheme.hpp:106-125 (the matrix is regenerated per attempt here; values equal) */
static int make_precomp(precomp* pre, const uint8_t* sk, const orc_params* P) {
  if (!unpack_sk(&pre->v, sk, P)) return 0;
  for (int i = 0; i < P->l; ++i) {
    for (int m = 0; m < N; ++m) pre->s1h[i][m] = modq(pre->v.s1[i][m]);
    orc_ntt(pre->s1h[i]);
  }
  for (int i = 0; i < P->k; ++i) {
    for (int m = 0; m < N; ++m) {
      pre->s2h[i][m] = modq(pre->v.s2[i][m]);
      pre->t0h[i][m] = modq(pre->v.t0[i][m]);
    }
    orc_ntt(pre->s2h[i]);
    orc_ntt(pre->t0h[i]);
  }
  return 1;
}

/* c*s for one polynomial: intt(chat o shat), centered */
static void mul_c(int32_t out[N], const int32_t chat[N], const int32_t shat[N]) {
  for (int m = 0; m < N; ++m) out[m] = modq((int64_t)chat[m] * shat[m]);
  orc_intt(out);
  for (int m = 0; m < N; ++m) out[m] = centered(out[m]);
}

/* scheme.hpp:133-219 (sign_attempt_bounded): bounds = {z, r0, c t0} norm bounds */
static int attempt_bounded(const precomp* pre, const orc_params* P, const uint8_t mu[64],
                           const uint8_t rho_prime[64], uint32_t kappa, const int32_t bounds[3],
                           int* stage, uint8_t* c_tilde, int32_t z[][N], int32_t hints[][N]) {
  static _Thread_local int32_t y[LMAX][N], yh[LMAX][N], w[KMAX][N], w1[KMAX][N], wcs2[KMAX][N],
      vt[KMAX][N];
  int32_t c[N], chat[N], tmp[N];
  for (int j = 0; j < P->l; ++j) {
    orc_expand_mask(y[j], rho_prime, (kappa + (uint32_t)j) & 0xFFFF, P->gamma1, P->z_bits);
    for (int m = 0; m < N; ++m) yh[j][m] = modq(y[j][m]);
    orc_ntt(yh[j]);
  }
  matvec(w, pre->v.rho, yh, P);
  uint8_t hin[64 + KMAX * 192];
  size_t w1b = (size_t)N * P->w1_bits / 8;
  memcpy(hin, mu, 64);
  for (int i = 0; i < P->k; ++i) {
    orc_intt(w[i]); /* canonical [0,q) == caddq(centered) (scheme.hpp:153-155) */
    for (int m = 0; m < N; ++m) w1[i][m] = highbits(w[i][m], P->gamma2);
    pack_w1(hin + 64 + w1b * i, w1[i], P);
  }
  orc_shake256(c_tilde, (size_t)P->ct_bytes, hin, 64 + w1b * P->k); /* scheme.hpp:158-163 */
  sample_in_ball_n(c, c_tilde, (size_t)P->ct_bytes, P->tau);
  for (int m = 0; m < N; ++m) chat[m] = modq(c[m]);
  orc_ntt(chat);

  for (int j = 0; j < P->l; ++j) { /* scheme.hpp:167-174 */
    mul_c(tmp, chat, pre->s1h[j]);
    for (int m = 0; m < N; ++m) z[j][m] = centered((int64_t)y[j][m] + tmp[m]);
    if (norm_ge(z[j], bounds[0])) {
      *stage = 0;
      return 0;
    }
  }
  for (int i = 0; i < P->k; ++i) { /* scheme.hpp:177-190 */
    int32_t r0[N], r1;
    mul_c(tmp, chat, pre->s2h[i]);
    for (int m = 0; m < N; ++m) {
      wcs2[i][m] = modq((int64_t)w[i][m] - tmp[m]);
      orc_decompose(wcs2[i][m], P->gamma2, &r1, &r0[m]);
    }
    if (norm_ge(r0, bounds[1])) {
      *stage = 1;
      return 0;
    }
  }
  for (int i = 0; i < P->k; ++i) { /* scheme.hpp:192-199 */
    mul_c(vt[i], chat, pre->t0h[i]);
    if (norm_ge(vt[i], bounds[2])) {
      *stage = 2;
      return 0;
    }
  }
  int weight = 0;
  for (int i = 0; i < P->k; ++i) /* scheme.hpp:201-215 */
    for (int m = 0; m < N; ++m) {
      int32_t zc = modq(-(int64_t)vt[i][m]);
      int32_t rc = modq((int64_t)wcs2[i][m] + vt[i][m]);
      hints[i][m] = orc_make_hint(zc, rc, P->gamma2);
      weight += hints[i][m];
    }
  if (weight > P->omega) {
    *stage = 3;
    return 0;
  }
  return 1;
}

/* the production bounds of scheme.hpp:225-230 */
static int attempt(const precomp* pre, const orc_params* P, const uint8_t mu[64],
                   const uint8_t rho_prime[64], uint32_t kappa, int* stage, uint8_t* c_tilde,
                   int32_t z[][N], int32_t hints[][N]) {
  const int32_t b[3] = {P->gamma1 - P->beta, P->gamma2 - P->beta, P->gamma2};
  return attempt_bounded(pre, P, mu, rho_prime, kappa, b, stage, c_tilde, z, hints);
}

int orc_sign_attempt(int level, const uint8_t* sk, const uint8_t mu[64],
                     const uint8_t rho_prime[64], uint32_t kappa, int* stage,
                     uint8_t* c_tilde, int32_t* z, int32_t* hints) {
  const orc_params* P = orc_get_params(level);
  if (!P) return -1;
  const int32_t b[3] = {P->gamma1 - P->beta, P->gamma2 - P->beta, P->gamma2};
  return orc_sign_attempt_bounded(level, sk, mu, rho_prime, kappa, b[0], b[1], b[2], stage, c_tilde, z,
                                  hints);
}

int orc_sign_attempt_bounded(int level, const uint8_t* sk, const uint8_t mu[64],
                             const uint8_t rho_prime[64], uint32_t kappa, int32_t z_bound,
                             int32_t r0_bound, int32_t vt_bound, int* stage, uint8_t* c_tilde,
                             int32_t* z, int32_t* hints) {
  const orc_params* P = orc_get_params(level);
  if (!P) return -1;
  const int32_t bounds[3] = {z_bound, r0_bound, vt_bound};
  precomp* pre = malloc(sizeof *pre);
  if (!make_precomp(pre, sk, P)) {
    free(pre);
    return -1;
  }
  int32_t(*zz)[N] = calloc(LMAX, sizeof *zz);
  int32_t(*hh)[N] = calloc(KMAX, sizeof *hh);
  int st = 0;
  int ok = attempt_bounded(pre, P, mu, rho_prime, kappa, bounds, &st, c_tilde, zz, hh);
  memcpy(z, zz, sizeof(int32_t) * N * (size_t)P->l);
  memcpy(hints, hh, sizeof(int32_t) * N * (size_t)P->k);
  if (stage) *stage = st;
  free(zz);
  free(hh);
  free(pre);
  return ok;
}

/* FIPS 204 context string (ML-DSA levels only): M' = 0 || len || ctx || M */
static uint8_t g_ctx[255];
static size_t g_ctx_len = 0;
static uint8_t g_oid[16];
static size_t g_oid_len = 0; /* > 0: HashML-DSA, FIPS 204 Alg. 4 / 5 (messages are digests PH(M)) */
int orc_set_mldsa_context(const uint8_t* ctx, size_t len) {
  if (len > 255) return -1;
  if (len) memcpy(g_ctx, ctx, len);
  g_ctx_len = len;
  g_oid_len = 0;
  return 0;
}
int orc_set_mldsa_prehash(const uint8_t* ctx, size_t len, const uint8_t* oid, size_t oid_len) {
  if (orc_set_mldsa_context(ctx, len) != 0 || oid_len > 16) return -1;
  if (oid_len) memcpy(g_oid, oid, oid_len);
  g_oid_len = oid_len;
  return 0;
}
static void mldsa_mu(uint8_t mu[64], const uint8_t tr[64], const uint8_t* msg, size_t msglen) {
  xof_t x;
  const uint8_t pfx[2] = {(uint8_t)(g_oid_len ? 1 : 0), (uint8_t)g_ctx_len};
  xof_init(&x, 136);
  xof_absorb(&x, tr, 64);
  xof_absorb(&x, pfx, 2);
  xof_absorb(&x, g_ctx, g_ctx_len);
  xof_absorb(&x, g_oid, g_oid_len);
  xof_absorb(&x, msg, msglen);
  xof_squeeze(&x, mu, 64);
}

/* scheme.hpp:240-273 */
int orc_sign(int level, const uint8_t* sk, const uint8_t* msg, size_t msglen,
             const uint8_t* rho_prime_override, uint8_t* sig, uint32_t* attempts) {
  const orc_params* P = orc_get_params(level);
  if (!P) return -1;
  precomp* pre = malloc(sizeof *pre);
  if (!make_precomp(pre, sk, P)) {
    free(pre);
    return -1;
  }
  uint8_t mu[64], rho_prime[64], c_tilde[64];
  if (P->mldsa) {
    /* FIPS 204 Alg. 2 / 7, deterministic variant: M' = 0 || |ctx| || ctx || M,
     * mu = H(tr || M', 64), rho'' = H(K || rnd || mu, 64), rnd = 0^32 */
    mldsa_mu(mu, pre->v.tr, msg, msglen);
    uint8_t krnd[64] = {0};
    memcpy(krnd, pre->v.key, 32);
    hash2(rho_prime, 64, krnd, 64, mu, 64);
  } else {
    hash2(mu, 64, pre->v.tr, 32, msg, msglen);        /* scheme.hpp:240-243 */
    hash2(rho_prime, 64, pre->v.key, 32, mu, 64);     /* scheme.hpp:245-248 */
  }
  if (rho_prime_override) memcpy(rho_prime, rho_prime_override, 64); /* scheme.hpp:257-258 */
  int32_t(*z)[N] = calloc(LMAX, sizeof *z);
  int32_t(*h)[N] = calloc(KMAX, sizeof *h);
  int rc = -2;
  for (uint32_t a = 0; a < (1u << 14); ++a) { /* scheme.hpp:238,259 */
    int st;
    if (attempt(pre, P, mu, rho_prime, a * (uint32_t)P->l, &st, c_tilde, z, h)) {
      memcpy(sig, c_tilde, (size_t)P->ct_bytes); /* packing.hpp:236-254 */
      size_t off = (size_t)P->ct_bytes, zb = (size_t)N * P->z_bits / 8;
      for (int j = 0; j < P->l; ++j, off += zb) pack_z(sig + off, z[j], P);
      encode_hint(sig + off, &h[0][0], P);
      if (attempts) *attempts = a + 1;
      rc = 0;
      break;
    }
  }
  free(z);
  free(h);
  free(pre);
  return rc;
}

/* scheme.hpp:277-318 */
int orc_verify(int level, const uint8_t* pk, size_t pklen, const uint8_t* msg, size_t msglen,
               const uint8_t* sig, size_t siglen) {
  const orc_params* P = orc_get_params(level);
  if (!P) return 0;
  if (pklen != P->pk_bytes || siglen != P->sig_bytes) return 0; /* packing.hpp:185,257 */
  static _Thread_local int32_t z[LMAX][N], zh[LMAX][N], h[KMAX][N], acc[KMAX][N], w1[KMAX][N];
  size_t zb = (size_t)N * P->z_bits / 8;
  for (int j = 0; j < P->l; ++j)
    for (int m = 0; m < N; ++m)
      z[j][m] = P->gamma1 - (int32_t)get_bits(sig + P->ct_bytes + zb * j, m, P->z_bits);
  if (!decode_hint(&h[0][0], sig + P->ct_bytes + zb * P->l, P)) return 0;
  for (int j = 0; j < P->l; ++j)
    if (norm_ge(z[j], P->gamma1 - P->beta)) return 0; /* scheme.hpp:284 */

  uint8_t tr[64], mu[64];
  orc_shake256(tr, (size_t)P->tr_bytes, pk, pklen);
  if (P->mldsa) { /* FIPS 204 Alg. 3 / 8: mu = H(tr || 0 || |ctx| || ctx || M, 64) */
    mldsa_mu(mu, tr, msg, msglen);
  } else {
    hash2(mu, 64, tr, 32, msg, msglen);
  }

  int32_t c[N], chat[N], t1h[N];
  sample_in_ball_n(c, sig, (size_t)P->ct_bytes, P->tau);
  for (int m = 0; m < N; ++m) chat[m] = modq(c[m]);
  orc_ntt(chat);
  for (int j = 0; j < P->l; ++j) {
    for (int m = 0; m < N; ++m) zh[j][m] = modq(z[j][m]);
    orc_ntt(zh[j]);
  }
  matvec(acc, pk, zh, P);
  uint8_t hin[64 + KMAX * 192];
  size_t w1b = (size_t)N * P->w1_bits / 8;
  memcpy(hin, mu, 64);
  for (int i = 0; i < P->k; ++i) { /* scheme.hpp:299-309 */
    for (int m = 0; m < N; ++m)
      t1h[m] = (int32_t)get_bits(pk + 32 + 320 * i, m, 10) << 13;
    orc_ntt(t1h);
    for (int m = 0; m < N; ++m) acc[i][m] = modq(acc[i][m] - (int64_t)chat[m] * t1h[m]);
    orc_intt(acc[i]);
    for (int m = 0; m < N; ++m) w1[i][m] = orc_use_hint(h[i][m], acc[i][m], P->gamma2);
    pack_w1(hin + 64 + w1b * i, w1[i], P);
  }
  uint8_t expect[64];
  orc_shake256(expect, (size_t)P->ct_bytes, hin, 64 + w1b * P->k);
  return memcmp(expect, sig, (size_t)P->ct_bytes) == 0;
}

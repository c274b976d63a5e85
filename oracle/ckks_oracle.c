/*
 * ckks_oracle.c -- TEST INFRASTRUCTURE ONLY (see ckks_oracle.h).
 *
 * Scalar C restatement of the reference CKKS/RNS algorithms.  Every function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj/include/heg/).  Deliberately written as straight loops
 * in the reference's own operation order: this file is the checker, not the
 * product.  Compile WITHOUT -ffast-math / -mfma so double arithmetic matches
 * the reference's x86-64 build bit for bit (the encoder FFT, Box-Muller and
 * llround are sensitive to contraction).
 */
#include "ckks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------- */
/* RNG: common.hpp:71-122                                                     */
/* ------------------------------------------------------------------------- */

uint64_t oc_splitmix64(uint64_t* state) { /* common.hpp:71-76 */
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void oc_rng_init(oc_rng* r, uint64_t seed) { /* common.hpp:81-86 */
  r->state = seed ^ 0xd1b54a32d192ed03ULL;
  oc_splitmix64(&r->state);
  oc_splitmix64(&r->state);
}

uint64_t oc_rng_next(oc_rng* r) { return oc_splitmix64(&r->state); }           /* :88 */
double oc_rng_uniform(oc_rng* r) { return (double)(oc_rng_next(r) >> 11) * 0x1.0p-53; } /* :91 */
uint64_t oc_rng_uniform_int(oc_rng* r, uint64_t n) { return oc_rng_next(r) % n; }       /* :97 */
uint64_t oc_rng_state(const oc_rng* r) { return r->state; }

double oc_rng_gaussian(oc_rng* r) { /* common.hpp:100-105 */
  double u1 = oc_rng_uniform(r);
  double u2 = oc_rng_uniform(r);
  while (u1 <= 1e-300) u1 = oc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

oc_rng oc_rng_fork(const oc_rng* r, uint64_t label) { /* common.hpp:108-112 */
  uint64_t s = r->state;
  uint64_t mixed = oc_splitmix64(&s) ^ (label * 0x9e3779b97f4a7c15ULL + 0x165667b19e3779f9ULL);
  oc_rng out;
  oc_rng_init(&out, mixed);
  return out;
}

oc_rng oc_rng_fork_str(const oc_rng* r, const char* label) { /* common.hpp:115-119, FNV-1a */
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const unsigned char* p = (const unsigned char*)label; *p; ++p) h = (h ^ *p) * 0x100000001b3ULL;
  return oc_rng_fork(r, h);
}

/* ------------------------------------------------------------------------- */
/* Modulus: ring.hpp:37-111                                                   */
/* ------------------------------------------------------------------------- */

void oc_mod_init(oc_mod* m, uint64_t q) { /* ring.hpp:41-47 */
  u128 two64 = (u128)1 << 64;
  m->value = q;
  m->ratio_hi = (uint64_t)(two64 / q);
  uint64_t rem = (uint64_t)(two64 % q);
  m->ratio_lo = (uint64_t)(((u128)rem << 64) / q);
}

static uint64_t mod_reduce(const oc_mod* m, u128 z) { /* ring.hpp:52-63 */
  uint64_t z0 = (uint64_t)z, z1 = (uint64_t)(z >> 64);
  u128 m0 = (u128)z0 * m->ratio_lo;
  u128 m1 = (u128)z0 * m->ratio_hi;
  u128 m2 = (u128)z1 * m->ratio_lo;
  u128 m3 = (u128)z1 * m->ratio_hi;
  u128 mid = (m0 >> 64) + (uint64_t)m1 + (uint64_t)m2;
  uint64_t quotient = (uint64_t)(m3 + (m1 >> 64) + (m2 >> 64) + (mid >> 64));
  uint64_t r = z0 - quotient * m->value;
  return r >= m->value ? r - m->value : r;
}

static inline uint64_t mod_add(const oc_mod* m, uint64_t a, uint64_t b) { /* ring.hpp:66-69 */
  uint64_t s = a + b;
  return s >= m->value ? s - m->value : s;
}
static inline uint64_t mod_sub(const oc_mod* m, uint64_t a, uint64_t b) { /* ring.hpp:72 */
  return a >= b ? a - b : a + m->value - b;
}
static inline uint64_t mod_neg(const oc_mod* m, uint64_t a) { return a == 0 ? 0 : m->value - a; } /* :74 */

uint64_t oc_mod_mul(const oc_mod* m, uint64_t a, uint64_t b) { return mod_reduce(m, (u128)a * b); } /* :76 */

uint64_t oc_mod_pow(const oc_mod* m, uint64_t base, uint64_t e) { /* ring.hpp:78-87 */
  uint64_t result = 1;
  uint64_t cur = base >= m->value ? base % m->value : base;
  while (e != 0) {
    if (e & 1) result = oc_mod_mul(m, result, cur);
    cur = oc_mod_mul(m, cur, cur);
    e >>= 1;
  }
  return result;
}

uint64_t oc_mod_inv(const oc_mod* m, uint64_t a) { return oc_mod_pow(m, a, m->value - 2); } /* :90-93 */

uint64_t oc_mod_shoup(const oc_mod* m, uint64_t w) { return (uint64_t)(((u128)w << 64) / m->value); } /* :96 */

uint64_t oc_mod_mul_shoup(const oc_mod* m, uint64_t x, uint64_t w, uint64_t ws) { /* ring.hpp:99-103 */
  uint64_t hi = (uint64_t)(((u128)x * ws) >> 64);
  uint64_t r = x * w - hi * m->value;
  return r >= m->value ? r - m->value : r;
}

/* ------------------------------------------------------------------------- */
/* Primes: ring.hpp:118-196                                                   */
/* ------------------------------------------------------------------------- */

static uint64_t mulmod_u64(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
static uint64_t powmod_u64(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod_u64(r, b, m);
    b = mulmod_u64(b, b, m);
    e >>= 1;
  }
  return r;
}

int oc_is_prime(uint64_t n) { /* ring.hpp:137-163 (deterministic Miller-Rabin) */
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  for (int b = 0; b < 12; ++b) {
    uint64_t x = powmod_u64(bases[b], d, n);
    if (x == 1 || x == n - 1) continue;
    int witness = 1;
    for (int i = 1; i < s; ++i) {
      x = mulmod_u64(x, x, n);
      if (x == n - 1) { witness = 0; break; }
    }
    if (witness) return 0;
  }
  return 1;
}

int oc_generate_primes(int64_t n, const int* bits, int count, uint64_t* out) { /* ring.hpp:171-196 */
  if (n < 4 || (n & (n - 1)) != 0) return -1;
  uint64_t step = 2 * (uint64_t)n;
  for (int b = 0; b < count; ++b) {
    if (bits[b] < 20 || bits[b] > 60) return -1;
    uint64_t top = (uint64_t)1 << bits[b];
    uint64_t floor_bound = (uint64_t)1 << (bits[b] - 1);
    int found = 0;
    for (uint64_t k = (top - 2) / step; k >= 1; --k) {
      uint64_t cand = k * step + 1;
      if (cand < floor_bound) break;
      int used = 0;
      for (int j = 0; j < b; ++j) used |= out[j] == cand;
      if (used || !oc_is_prime(cand)) continue;
      out[b] = cand;
      found = 1;
      break;
    }
    if (!found) return -1;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Context + NTT tables: context.hpp:92-109, ring.hpp:221-301                 */
/* ------------------------------------------------------------------------- */

typedef struct {
  oc_mod q;
  uint64_t *psi, *psi_s, *ipsi, *ipsi_s;
  uint64_t n_inv, n_inv_s;
} oc_tables;

struct oc_ctx {
  int64_t n;
  int log_n;
  int count;
  int scale_bits;
  oc_tables t[OC_MAX_PRIMES];
};

static size_t bit_reverse(size_t x, int log_n) { /* ring.hpp:204-211 */
  size_t r = 0;
  for (int i = 0; i < log_n; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

static void tables_init(oc_tables* t, uint64_t q, int64_t n, int log_n) { /* ring.hpp:223-257 */
  oc_mod_init(&t->q, q);
  uint64_t exponent = (q - 1) / (2 * (uint64_t)n);
  uint64_t psi = 0;
  for (uint64_t h = 2;; ++h) {
    uint64_t g = oc_mod_pow(&t->q, h, exponent);
    if (oc_mod_pow(&t->q, g, (uint64_t)n) == q - 1) { psi = g; break; }
  }
  uint64_t psi_inv = oc_mod_inv(&t->q, psi);
  t->psi = malloc(sizeof(uint64_t) * n);
  t->psi_s = malloc(sizeof(uint64_t) * n);
  t->ipsi = malloc(sizeof(uint64_t) * n);
  t->ipsi_s = malloc(sizeof(uint64_t) * n);
  uint64_t fwd = 1, bwd = 1;
  for (int64_t j = 0; j < n; ++j) {
    size_t r = bit_reverse((size_t)j, log_n);
    t->psi[r] = fwd;
    t->psi_s[r] = oc_mod_shoup(&t->q, fwd);
    t->ipsi[r] = bwd;
    t->ipsi_s[r] = oc_mod_shoup(&t->q, bwd);
    fwd = oc_mod_mul(&t->q, fwd, psi);
    bwd = oc_mod_mul(&t->q, bwd, psi_inv);
  }
  t->n_inv = oc_mod_inv(&t->q, (uint64_t)n % q);
  t->n_inv_s = oc_mod_shoup(&t->q, t->n_inv);
}

oc_ctx* oc_ctx_create(int64_t n, const int* bits, int count, int scale_bits) {
  if (count < 1 || count > OC_MAX_PRIMES) return NULL;
  uint64_t primes[OC_MAX_PRIMES];
  if (oc_generate_primes(n, bits, count, primes) != 0) return NULL;
  oc_ctx* c = calloc(1, sizeof(oc_ctx));
  c->n = n;
  c->count = count;
  c->scale_bits = scale_bits;
  while (((int64_t)1 << c->log_n) < n) ++c->log_n;
  for (int i = 0; i < count; ++i) tables_init(&c->t[i], primes[i], n, c->log_n);
  return c;
}

void oc_ctx_free(oc_ctx* c) {
  if (!c) return;
  for (int i = 0; i < c->count; ++i) {
    free(c->t[i].psi); free(c->t[i].psi_s); free(c->t[i].ipsi); free(c->t[i].ipsi_s);
  }
  free(c);
}

int64_t oc_ctx_n(const oc_ctx* c) { return c->n; }
int oc_ctx_count(const oc_ctx* c) { return c->count; }
uint64_t oc_ctx_prime(const oc_ctx* c, int i) { return c->t[i].q.value; }

void oc_ctx_tables(const oc_ctx* c, int i, uint64_t* out4n, uint64_t* ninv2) {
  const oc_tables* t = &c->t[i];
  size_t b = sizeof(uint64_t) * (size_t)c->n;
  memcpy(out4n, t->psi, b);
  memcpy(out4n + c->n, t->psi_s, b);
  memcpy(out4n + 2 * c->n, t->ipsi, b);
  memcpy(out4n + 3 * c->n, t->ipsi_s, b);
  ninv2[0] = t->n_inv;
  ninv2[1] = t->n_inv_s;
}

void oc_ntt_forward(const oc_ctx* c, int limb, uint64_t* a) { /* ring.hpp:263-279 (Cooley-Tukey) */
  const oc_tables* T = &c->t[limb];
  size_t n = (size_t)c->n, t = n;
  for (size_t m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (size_t i = 0; i < m; ++i) {
      uint64_t w = T->psi[m + i], ws = T->psi_s[m + i];
      size_t j1 = 2 * i * t;
      for (size_t j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j];
        uint64_t v = oc_mod_mul_shoup(&T->q, a[j + t], w, ws);
        a[j] = mod_add(&T->q, u, v);
        a[j + t] = mod_sub(&T->q, u, v);
      }
    }
  }
}

void oc_ntt_inverse(const oc_ctx* c, int limb, uint64_t* a) { /* ring.hpp:282-301 (Gentleman-Sande) */
  const oc_tables* T = &c->t[limb];
  size_t n = (size_t)c->n, t = 1;
  for (size_t m = n; m > 1; m >>= 1) {
    size_t j1 = 0, h = m >> 1;
    for (size_t i = 0; i < h; ++i) {
      uint64_t w = T->ipsi[h + i], ws = T->ipsi_s[h + i];
      for (size_t j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j], v = a[j + t];
        a[j] = mod_add(&T->q, u, v);
        a[j + t] = oc_mod_mul_shoup(&T->q, mod_sub(&T->q, u, v), w, ws);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (size_t j = 0; j < n; ++j) a[j] = oc_mod_mul_shoup(&T->q, a[j], T->n_inv, T->n_inv_s);
}

void oc_negacyclic_schoolbook(const oc_mod* q, int64_t n, const uint64_t* a, const uint64_t* b,
                              uint64_t* c) { /* ring.hpp:326-343 */
  for (int64_t k = 0; k < n; ++k) c[k] = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (a[i] == 0) continue;
    for (int64_t j = 0; j < n; ++j) {
      uint64_t prod = oc_mod_mul(q, a[i], b[j]);
      int64_t k = i + j;
      if (k < n) c[k] = mod_add(q, c[k], prod);
      else c[k - n] = mod_sub(q, c[k - n], prod);
    }
  }
}

/* ------------------------------------------------------------------------- */
/* CRT reconstruction: ring.hpp:350-480 (WideInt + CrtReconstructor)          */
/* ------------------------------------------------------------------------- */

#define WMAX (OC_MAX_PRIMES + 1)
typedef struct { uint64_t w[WMAX]; int n; } wide;

static void wide_set(wide* x, uint64_t v, int n) { memset(x->w, 0, sizeof x->w); x->w[0] = v; x->n = n; }
static void wide_mul_u64(wide* x, uint64_t s) { /* ring.hpp:362-370 */
  u128 carry = 0;
  for (int i = 0; i < x->n; ++i) {
    u128 cur = (u128)x->w[i] * s + carry;
    x->w[i] = (uint64_t)cur;
    carry = cur >> 64;
  }
}
static void wide_add_scaled(wide* x, const wide* o, uint64_t s) { /* ring.hpp:373-382 */
  u128 carry = 0;
  for (int i = 0; i < x->n; ++i) {
    uint64_t ov = i < o->n ? o->w[i] : 0;
    u128 cur = (u128)ov * s + x->w[i] + carry;
    x->w[i] = (uint64_t)cur;
    carry = cur >> 64;
  }
}
static int wide_cmp(const wide* a, const wide* b) { /* ring.hpp:385-393 */
  int width = a->n > b->n ? a->n : b->n;
  for (int i = width; i-- > 0;) {
    uint64_t x = i < a->n ? a->w[i] : 0, y = i < b->n ? b->w[i] : 0;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
static void wide_sub(wide* a, const wide* b) { /* ring.hpp:396-406 */
  uint64_t borrow = 0;
  for (int i = 0; i < a->n; ++i) {
    uint64_t o = i < b->n ? b->w[i] : 0, before = a->w[i];
    uint64_t after = before - o - borrow;
    borrow = (before < o || (borrow && before == o)) ? 1 : 0;
    a->w[i] = after;
  }
}
static double wide_to_double(const wide* a) { /* ring.hpp:422-426 */
  double r = 0.0;
  for (int i = a->n; i-- > 0;) r = r * 18446744073709551616.0 + (double)a->w[i];
  return r;
}
static uint64_t wide_mod(const wide* a, uint64_t q) { /* ring.hpp:416-420 */
  uint64_t r = 0;
  for (int i = a->n; i-- > 0;) r = (uint64_t)((((u128)r << 64) | a->w[i]) % q);
  return r;
}

double oc_crt_centered(const uint64_t* primes, int count, const uint64_t* residues) { /* ring.hpp:438-471 */
  int width = count + 1;
  wide total, half, acc;
  wide_set(&total, 1, width);
  for (int i = 0; i < count; ++i) wide_mul_u64(&total, primes[i]);
  /* half = total >> 1 (ring.hpp:408-414) */
  half.n = width;
  memset(half.w, 0, sizeof half.w);
  for (int i = 0; i < width; ++i) {
    half.w[i] = total.w[i] >> 1;
    if (i + 1 < width) half.w[i] |= total.w[i + 1] << 63;
  }
  wide_set(&acc, 0, width);
  for (int i = 0; i < count; ++i) {
    wide punct;
    wide_set(&punct, 1, width);
    for (int j = 0; j < count; ++j)
      if (j != i) wide_mul_u64(&punct, primes[j]);
    oc_mod qi;
    oc_mod_init(&qi, primes[i]);
    uint64_t inv = oc_mod_inv(&qi, wide_mod(&punct, primes[i]));
    wide_add_scaled(&acc, &punct, oc_mod_mul(&qi, residues[i], inv));
  }
  while (wide_cmp(&acc, &total) >= 0) wide_sub(&acc, &total);
  if (wide_cmp(&acc, &half) > 0) {
    wide neg = total;
    wide_sub(&neg, &acc);
    return -wide_to_double(&neg);
  }
  return wide_to_double(&acc);
}

/* ------------------------------------------------------------------------- */
/* Slot encoder: encoder.hpp:38-115 (fp64 radix-2 FFT, canonical embedding)   */
/* Complex products are written out as GCC expands std::complex<double>       */
/* multiplication: (a+bi)(c+di) = (ac - bd) + (ad + bc)i.                     */
/* ------------------------------------------------------------------------- */

typedef struct { double re, im; } cplx;

typedef struct {
  int64_t n;
  cplx* roots;
  cplx* half_roots;
  size_t* rev;
} encoder;

static void encoder_init(encoder* e, int64_t n) { /* encoder.hpp:38-58 */
  e->n = n;
  e->roots = malloc(sizeof(cplx) * n);
  e->half_roots = malloc(sizeof(cplx) * n);
  e->rev = malloc(sizeof(size_t) * n);
  const double pi = acos(-1.0);
  for (int64_t j = 0; j < n; ++j) {
    const double a = -2.0 * pi * (double)j / (double)n;
    e->roots[j].re = cos(a);
    e->roots[j].im = sin(a);
    const double h = -pi * (double)j / (double)n;
    e->half_roots[j].re = cos(h);
    e->half_roots[j].im = sin(h);
  }
  int log_n = 0;
  while (((int64_t)1 << log_n) < n) ++log_n;
  for (int64_t j = 0; j < n; ++j) {
    size_t r = 0;
    for (int b = 0; b < log_n; ++b) r |= (((size_t)j >> b) & 1u) << (log_n - 1 - b);
    e->rev[j] = r;
  }
}

static void encoder_free(encoder* e) { free(e->roots); free(e->half_roots); free(e->rev); }

static void encoder_fft(const encoder* e, cplx* a, int conjugate) { /* encoder.hpp:92-109 */
  const size_t n = (size_t)e->n;
  for (size_t j = 0; j < n; ++j)
    if (e->rev[j] > j) { cplx t = a[j]; a[j] = a[e->rev[j]]; a[e->rev[j]] = t; }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t step = n / len;
    for (size_t start = 0; start < n; start += len) {
      for (size_t j = 0; j < len / 2; ++j) {
        cplx w = e->roots[j * step];
        if (conjugate) w.im = -w.im;
        const cplx u = a[start + j];
        const cplx x = a[start + j + len / 2];
        cplx v;
        v.re = x.re * w.re - x.im * w.im;
        v.im = x.re * w.im + x.im * w.re;
        a[start + j].re = u.re + v.re;
        a[start + j].im = u.im + v.im;
        a[start + j + len / 2].re = u.re - v.re;
        a[start + j + len / 2].im = u.im - v.im;
      }
    }
  }
}

void oc_encode_values(int64_t n, const double* values, int64_t count, double* coeffs) { /* encoder.hpp:64-77 */
  encoder e;
  encoder_init(&e, n);
  cplx* a = calloc((size_t)n, sizeof(cplx));
  for (int64_t m = 0; m < count; ++m) a[m].re = values[m];
  encoder_fft(&e, a, 0);
  const double norm = 2.0 / (double)n;
  for (int64_t k = 0; k < n; ++k) {
    const cplx h = e.half_roots[k];
    const double re = h.re * a[k].re - h.im * a[k].im;
    coeffs[k] = norm * re;
  }
  free(a);
  encoder_free(&e);
}

void oc_decode_coeffs(int64_t n, const double* coeffs, int64_t count, double* values) { /* encoder.hpp:80-89 */
  encoder e;
  encoder_init(&e, n);
  cplx* b = malloc(sizeof(cplx) * n);
  for (int64_t k = 0; k < n; ++k) {
    b[k].re = coeffs[k] * e.half_roots[k].re;
    b[k].im = coeffs[k] * -e.half_roots[k].im;
  }
  encoder_fft(&e, b, 1);
  for (int64_t m = 0; m < count; ++m) values[m] = b[m].re;
  free(b);
  encoder_free(&e);
}

/* ------------------------------------------------------------------------- */
/* Polynomials and samplers: poly.hpp                                         */
/* ------------------------------------------------------------------------- */

static inline uint64_t lift_signed(int64_t v, uint64_t q) { /* poly.hpp:54-58 */
  int64_t r = v % (int64_t)q;
  if (r < 0) r += (int64_t)q;
  return (uint64_t)r;
}

void oc_poly_to_ntt(const oc_ctx* c, int level, uint64_t* p) { /* poly.hpp:60-64 */
  for (int i = 0; i <= level; ++i) oc_ntt_forward(c, i, p + (size_t)i * c->n);
}
void oc_poly_to_coeff(const oc_ctx* c, int level, uint64_t* p) { /* poly.hpp:66-70 */
  for (int i = 0; i <= level; ++i) oc_ntt_inverse(c, i, p + (size_t)i * c->n);
}

void oc_poly_rescale(const oc_ctx* c, int level, int ntt_form, const uint64_t* in, uint64_t* out) {
  /* poly.hpp:190-228 */
  const int64_t n = c->n;
  const int t = level;
  const oc_tables* T = &c->t[t];
  uint64_t* top = malloc(sizeof(uint64_t) * n);
  int64_t* centered = malloc(sizeof(int64_t) * n);
  uint64_t* corr = malloc(sizeof(uint64_t) * n);
  memcpy(top, in + (size_t)t * n, sizeof(uint64_t) * n);
  if (ntt_form) oc_ntt_inverse(c, t, top);
  const uint64_t half = T->q.value / 2;
  for (int64_t k = 0; k < n; ++k)
    centered[k] = top[k] > half ? (int64_t)top[k] - (int64_t)T->q.value : (int64_t)top[k];
  for (int j = 0; j < t; ++j) {
    const oc_mod* qj = &c->t[j].q;
    for (int64_t k = 0; k < n; ++k) corr[k] = lift_signed(centered[k], qj->value);
    if (ntt_form) oc_ntt_forward(c, j, corr);
    const uint64_t inv_qt = oc_mod_inv(qj, T->q.value % qj->value);
    const uint64_t inv_qt_s = oc_mod_shoup(qj, inv_qt);
    const uint64_t* x = in + (size_t)j * n;
    uint64_t* o = out + (size_t)j * n;
    for (int64_t k = 0; k < n; ++k) o[k] = oc_mod_mul_shoup(qj, mod_sub(qj, x[k], corr[k]), inv_qt, inv_qt_s);
  }
  free(top); free(centered); free(corr);
}

void oc_sample_uniform(const oc_ctx* c, int level, oc_rng* r, uint64_t* out) { /* poly.hpp:247-254 */
  for (int i = 0; i <= level; ++i)
    for (int64_t k = 0; k < c->n; ++k) out[(size_t)i * c->n + k] = oc_rng_uniform_int(r, c->t[i].q.value);
}

void oc_sample_ternary(const oc_ctx* c, int level, oc_rng* r, uint64_t* out) { /* poly.hpp:257-265 */
  for (int64_t k = 0; k < c->n; ++k) {
    const int64_t v = (int64_t)oc_rng_uniform_int(r, 3) - 1;
    for (int i = 0; i <= level; ++i) out[(size_t)i * c->n + k] = lift_signed(v, c->t[i].q.value);
  }
}

void oc_sample_gaussian(const oc_ctx* c, int level, double sigma, oc_rng* r, uint64_t* out) { /* poly.hpp:268-276 */
  for (int64_t k = 0; k < c->n; ++k) {
    const int64_t v = (int64_t)llround(oc_rng_gaussian(r) * sigma);
    for (int i = 0; i <= level; ++i) out[(size_t)i * c->n + k] = lift_signed(v, c->t[i].q.value);
  }
}

/* pointwise helpers over (level+1) rows */
static void pw_mul(const oc_ctx* c, int level, const uint64_t* a, const uint64_t* b, uint64_t* o) {
  for (int i = 0; i <= level; ++i)
    for (int64_t k = 0; k < c->n; ++k) {
      size_t x = (size_t)i * c->n + k;
      o[x] = oc_mod_mul(&c->t[i].q, a[x], b[x]);
    }
}
static void pw_mul_acc(const oc_ctx* c, int level, const uint64_t* a, const uint64_t* b, uint64_t* o) {
  for (int i = 0; i <= level; ++i)
    for (int64_t k = 0; k < c->n; ++k) {
      size_t x = (size_t)i * c->n + k;
      o[x] = mod_add(&c->t[i].q, o[x], oc_mod_mul(&c->t[i].q, a[x], b[x]));
    }
}
static void pw_add(const oc_ctx* c, int level, const uint64_t* a, const uint64_t* b, uint64_t* o) {
  for (int i = 0; i <= level; ++i)
    for (int64_t k = 0; k < c->n; ++k) {
      size_t x = (size_t)i * c->n + k;
      o[x] = mod_add(&c->t[i].q, a[x], b[x]);
    }
}
static void pw_neg(const oc_ctx* c, int level, const uint64_t* a, uint64_t* o) {
  for (int i = 0; i <= level; ++i)
    for (int64_t k = 0; k < c->n; ++k) {
      size_t x = (size_t)i * c->n + k;
      o[x] = mod_neg(&c->t[i].q, a[x]);
    }
}

/* ------------------------------------------------------------------------- */
/* Keys: ckks_backend.hpp:39-114                                              */
/* ------------------------------------------------------------------------- */

int oc_relin_digit_count(uint64_t q) { /* ckks_backend.hpp:42-46 */
  int digits = 0;
  for (uint64_t m = q - 1; m != 0; m >>= 15) ++digits;
  return digits == 0 ? 1 : digits;
}

int oc_relin_rows(const oc_ctx* c) {
  int r = 0;
  for (int i = 0; i < c->count; ++i) r += oc_relin_digit_count(c->t[i].q.value);
  return r;
}

struct oc_keys {
  int L;
  int64_t words; /* (L+1)*n */
  uint64_t *secret, *pk_b, *pk_a;
  int rows;
  uint64_t** rb;
  uint64_t** ra;
};

static const double kErrorStdDev = 3.2; /* backend.hpp:29 */

oc_keys* oc_keys_generate(const oc_ctx* c, uint64_t seed, int with_relin) { /* ckks_backend.hpp:74-114 */
  const int L = c->count - 1;
  const int64_t W = (int64_t)(L + 1) * c->n;
  oc_rng root, secret_rng, public_rng, relin_rng;
  oc_rng_init(&root, seed);
  secret_rng = oc_rng_fork_str(&root, "secret");
  public_rng = oc_rng_fork_str(&root, "public");
  relin_rng = oc_rng_fork_str(&root, "relin");

  oc_keys* k = calloc(1, sizeof(oc_keys));
  k->L = L;
  k->words = W;
  k->secret = malloc(sizeof(uint64_t) * W);
  k->pk_b = malloc(sizeof(uint64_t) * W);
  k->pk_a = malloc(sizeof(uint64_t) * W);
  oc_sample_ternary(c, L, &secret_rng, k->secret);
  oc_poly_to_ntt(c, L, k->secret);

  uint64_t* e = malloc(sizeof(uint64_t) * W);
  oc_sample_gaussian(c, L, kErrorStdDev, &public_rng, e);
  oc_poly_to_ntt(c, L, e);
  oc_sample_uniform(c, L, &public_rng, k->pk_a);
  uint64_t* tmp = malloc(sizeof(uint64_t) * W);
  pw_mul(c, L, k->pk_a, k->secret, tmp);
  pw_add(c, L, tmp, e, tmp);
  pw_neg(c, L, tmp, k->pk_b);

  if (with_relin) {
    uint64_t* s2 = malloc(sizeof(uint64_t) * W);
    pw_mul(c, L, k->secret, k->secret, s2);
    k->rows = oc_relin_rows(c);
    k->rb = calloc((size_t)k->rows, sizeof(uint64_t*));
    k->ra = calloc((size_t)k->rows, sizeof(uint64_t*));
    int row = 0;
    for (int i = 0; i <= L; ++i) {
      const oc_mod* qi = &c->t[i].q;
      const int digits = oc_relin_digit_count(qi->value);
      for (int d = 0; d < digits; ++d, ++row) {
        uint64_t* b = malloc(sizeof(uint64_t) * W);
        uint64_t* a = malloc(sizeof(uint64_t) * W);
        oc_sample_gaussian(c, L, kErrorStdDev, &relin_rng, e);
        oc_poly_to_ntt(c, L, e);
        oc_sample_uniform(c, L, &relin_rng, a);
        pw_mul(c, L, a, k->secret, tmp);
        pw_add(c, L, tmp, e, tmp);
        pw_neg(c, L, tmp, b);
        const uint64_t f = oc_mod_pow(qi, 2, (uint64_t)15 * (uint64_t)d);
        const uint64_t fs = oc_mod_shoup(qi, f);
        uint64_t* bi = b + (size_t)i * c->n;
        const uint64_t* s2i = s2 + (size_t)i * c->n;
        for (int64_t x = 0; x < c->n; ++x) bi[x] = mod_add(qi, bi[x], oc_mod_mul_shoup(qi, s2i[x], f, fs));
        k->rb[row] = b;
        k->ra[row] = a;
      }
    }
    free(s2);
  }
  free(e);
  free(tmp);
  return k;
}

void oc_keys_free(oc_keys* k) {
  if (!k) return;
  for (int r = 0; r < k->rows; ++r) { free(k->rb[r]); free(k->ra[r]); }
  free(k->rb); free(k->ra);
  free(k->secret); free(k->pk_b); free(k->pk_a);
  free(k);
}

const uint64_t* oc_keys_secret(const oc_keys* k) { return k->secret; }
const uint64_t* oc_keys_pk_b(const oc_keys* k) { return k->pk_b; }
const uint64_t* oc_keys_pk_a(const oc_keys* k) { return k->pk_a; }
const uint64_t* oc_keys_relin_b(const oc_keys* k, int row) { return k->rb[row]; }
const uint64_t* oc_keys_relin_a(const oc_keys* k, int row) { return k->ra[row]; }

/* ------------------------------------------------------------------------- */
/* Scheme operations: ckks_backend.hpp                                        */
/* ------------------------------------------------------------------------- */

int oc_encode(const oc_ctx* c, const double* values, int64_t count, int level, double scale,
              uint64_t* pt) { /* ckks_backend.hpp:182-197 */
  if (count > c->n / 2) return 4; /* capacity */
  double* coeffs = malloc(sizeof(double) * c->n);
  oc_encode_values(c->n, values, count, coeffs);
  for (int64_t k = 0; k < c->n; ++k) {
    const double scaled = coeffs[k] * scale;
    if (!(fabs(scaled) < 9.0e18)) { free(coeffs); return 1; }
    const int64_t v = llround(scaled);
    for (int i = 0; i <= level; ++i) pt[(size_t)i * c->n + k] = lift_signed(v, c->t[i].q.value);
  }
  free(coeffs);
  oc_poly_to_ntt(c, level, pt);
  return 0;
}

int oc_encode_constant(const oc_ctx* c, double value, int level, double scale,
                       uint64_t* pt) { /* ckks_backend.hpp:199-216 */
  const double scaled = value * scale;
  if (!(fabs(scaled) < 9.0e18)) return 1;
  const int64_t v = llround(scaled);
  for (int i = 0; i <= level; ++i) {
    const uint64_t r = lift_signed(v, c->t[i].q.value);
    for (int64_t k = 0; k < c->n; ++k) pt[(size_t)i * c->n + k] = r;
  }
  return 0;
}

static void fresh_encryption(const oc_ctx* c, const oc_keys* k, int level, uint64_t seed,
                             uint64_t* ct) { /* ckks_backend.hpp:470-490 */
  const int64_t W = (int64_t)(level + 1) * c->n;
  oc_rng rng, u_rng, e_rng;
  oc_rng_init(&rng, seed);
  u_rng = oc_rng_fork_str(&rng, "mask");
  e_rng = oc_rng_fork_str(&rng, "error");
  uint64_t* u = malloc(sizeof(uint64_t) * W);
  uint64_t* e0 = malloc(sizeof(uint64_t) * W);
  uint64_t* e1 = malloc(sizeof(uint64_t) * W);
  oc_sample_ternary(c, level, &u_rng, u);
  oc_sample_gaussian(c, level, kErrorStdDev, &e_rng, e0);
  oc_sample_gaussian(c, level, kErrorStdDev, &e_rng, e1);
  oc_poly_to_ntt(c, level, u);
  oc_poly_to_ntt(c, level, e0);
  oc_poly_to_ntt(c, level, e1);
  pw_mul(c, level, k->pk_b, u, ct); /* pk truncated to level: same row layout */
  pw_add(c, level, ct, e0, ct);
  pw_mul(c, level, k->pk_a, u, ct + W);
  pw_add(c, level, ct + W, e1, ct + W);
  free(u); free(e0); free(e1);
}

void oc_encrypt_zero(const oc_ctx* c, const oc_keys* k, int level, uint64_t seed, uint64_t* ct) {
  fresh_encryption(c, k, level, seed, ct); /* ckks_backend.hpp:231-236 */
}

void oc_encrypt(const oc_ctx* c, const oc_keys* k, const uint64_t* pt, int level, uint64_t seed,
                uint64_t* ct) { /* ckks_backend.hpp:223-229 */
  fresh_encryption(c, k, level, seed, ct);
  pw_add(c, level, ct, pt, ct);
}

void oc_decrypt_coeffs(const oc_ctx* c, const oc_keys* k, const uint64_t* ct, int size, int level,
                       uint64_t* m) { /* ckks_backend.hpp:238-247, then poly_copy_coeff (:494) */
  const int64_t W = (int64_t)(level + 1) * c->n;
  uint64_t* sp = malloc(sizeof(uint64_t) * W);
  memcpy(m, ct, sizeof(uint64_t) * W);
  memcpy(sp, k->secret, sizeof(uint64_t) * W);
  for (int j = 1; j < size; ++j) {
    if (j > 1) pw_mul(c, level, sp, k->secret, sp);
    pw_mul_acc(c, level, ct + (size_t)j * W, sp, m);
  }
  free(sp);
  oc_poly_to_coeff(c, level, m);
}

void oc_decrypt(const oc_ctx* c, const oc_keys* k, const uint64_t* ct, int size, int level, double scale,
                int64_t count, double* out) { /* ckks_backend.hpp:238-249, 493-505 */
  const int64_t W = (int64_t)(level + 1) * c->n;
  uint64_t* m = malloc(sizeof(uint64_t) * W);
  oc_decrypt_coeffs(c, k, ct, size, level, m);
  uint64_t primes[OC_MAX_PRIMES], res[OC_MAX_PRIMES];
  for (int i = 0; i <= level; ++i) primes[i] = c->t[i].q.value;
  double* coeffs = malloc(sizeof(double) * c->n);
  for (int64_t x = 0; x < c->n; ++x) {
    for (int i = 0; i <= level; ++i) res[i] = m[(size_t)i * c->n + x];
    coeffs[x] = oc_crt_centered(primes, level + 1, res) / scale;
  }
  oc_decode_coeffs(c->n, coeffs, count, out);
  free(coeffs);
  free(m);
}

void oc_add(const oc_ctx* c, int level, int64_t words, const uint64_t* a, const uint64_t* b, uint64_t* o) {
  /* poly_add (poly.hpp:87-98) over `words`/((level+1)n) polys */
  const int64_t W = (int64_t)(level + 1) * c->n;
  for (int64_t p = 0; p < words / W; ++p) pw_add(c, level, a + p * W, b + p * W, o + p * W);
}

void oc_sub(const oc_ctx* c, int level, int64_t words, const uint64_t* a, const uint64_t* b, uint64_t* o) {
  /* poly_sub (poly.hpp:100-111) */
  const int64_t W = (int64_t)(level + 1) * c->n;
  for (int64_t p = 0; p < words / W; ++p)
    for (int i = 0; i <= level; ++i)
      for (int64_t k = 0; k < c->n; ++k) {
        size_t x = (size_t)(p * W + (int64_t)i * c->n + k);
        o[x] = mod_sub(&c->t[i].q, a[x], b[x]);
      }
}

void oc_negate(const oc_ctx* c, int level, int64_t words, const uint64_t* a, uint64_t* o) {
  /* poly_negate (poly.hpp:113-121) */
  const int64_t W = (int64_t)(level + 1) * c->n;
  for (int64_t p = 0; p < words / W; ++p) pw_neg(c, level, a + p * W, o + p * W);
}

void oc_mul_plain(const oc_ctx* c, int level, int size, const uint64_t* ct, const uint64_t* pt,
                  uint64_t* o) { /* ckks_backend.hpp:299-310 */
  const int64_t W = (int64_t)(level + 1) * c->n;
  for (int p = 0; p < size; ++p) pw_mul(c, level, ct + (size_t)p * W, pt, o + (size_t)p * W);
}

void oc_multiply_norelin(const oc_ctx* c, int level, const uint64_t* x, const uint64_t* y,
                         uint64_t* o) { /* ckks_backend.hpp:265-271 */
  const int64_t W = (int64_t)(level + 1) * c->n;
  memset(o, 0, sizeof(uint64_t) * 3 * W);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) pw_mul_acc(c, level, x + (size_t)i * W, y + (size_t)j * W, o + (size_t)(i + j) * W);
}

void oc_relinearize(const oc_ctx* c, const oc_keys* k, int level, const uint64_t* in3,
                    uint64_t* out2) { /* ckks_backend.hpp:508-554 */
  const int64_t n = c->n, W = (int64_t)(level + 1) * n;
  uint64_t* c2 = malloc(sizeof(uint64_t) * W);
  memcpy(c2, in3 + 2 * W, sizeof(uint64_t) * W);
  oc_poly_to_coeff(c, level, c2);
  memcpy(out2, in3, sizeof(uint64_t) * 2 * W);
  uint64_t* acc0 = out2;
  uint64_t* acc1 = out2 + W;
  uint64_t* digit = malloc(sizeof(uint64_t) * n);
  uint64_t* tr = malloc(sizeof(uint64_t) * n);
  int row_base = 0;
  for (int i = 0; i <= level; ++i) {
    const int digits = oc_relin_digit_count(c->t[i].q.value);
    const uint64_t* src = c2 + (size_t)i * n;
    for (int d = 0; d < digits; ++d) {
      for (int64_t x = 0; x < n; ++x) digit[x] = (src[x] >> (15 * d)) & ((1u << 15) - 1);
      const uint64_t* kb = k->rb[row_base + d];
      const uint64_t* ka = k->ra[row_base + d];
      for (int j = 0; j <= level; ++j) {
        const oc_mod* qj = &c->t[j].q;
        memcpy(tr, digit, sizeof(uint64_t) * n);
        oc_ntt_forward(c, j, tr);
        uint64_t* o0 = acc0 + (size_t)j * n;
        uint64_t* o1 = acc1 + (size_t)j * n;
        const uint64_t* b = kb + (size_t)j * n;
        const uint64_t* a = ka + (size_t)j * n;
        for (int64_t x = 0; x < n; ++x) {
          o0[x] = mod_add(qj, o0[x], oc_mod_mul(qj, tr[x], b[x]));
          o1[x] = mod_add(qj, o1[x], oc_mod_mul(qj, tr[x], a[x]));
        }
      }
    }
    row_base += digits;
  }
  free(digit); free(tr); free(c2);
}

void oc_multiply_relin(const oc_ctx* c, const oc_keys* k, int level, const uint64_t* x, const uint64_t* y,
                       uint64_t* out) {
  const int64_t W = (int64_t)(level + 1) * c->n;
  uint64_t* d = malloc(sizeof(uint64_t) * 3 * W);
  oc_multiply_norelin(c, level, x, y, d);
  oc_relinearize(c, k, level, d, out);
  free(d);
}

void oc_rescale_ct(const oc_ctx* c, int level, int size, const uint64_t* in, uint64_t* out) {
  /* ckks_backend.hpp:344-353: poly_rescale on each poly */
  const int64_t Win = (int64_t)(level + 1) * c->n, Wout = (int64_t)level * c->n;
  for (int p = 0; p < size; ++p) oc_poly_rescale(c, level, 1, in + (size_t)p * Win, out + (size_t)p * Wout);
}

int oc_weighted_sum(const oc_ctx* c, int level, int terms, const uint64_t* const* xs, const double* w,
                    uint64_t* out) { /* ckks_backend.hpp:381-411 with runtime.hpp:536-547 weights */
  const int64_t W = (int64_t)(level + 1) * c->n;
  const double w_scale = (double)c->t[level].q.value; /* backend.hpp:167-170 */
  uint64_t* acc = calloc((size_t)(2 * W), sizeof(uint64_t));
  uint64_t* pt = malloc(sizeof(uint64_t) * W);
  for (int t = 0; t < terms; ++t) {
    if (oc_encode_constant(c, w[t], level, w_scale, pt) != 0) { free(acc); free(pt); return 1; }
    pw_mul_acc(c, level, xs[t], pt, acc);
    pw_mul_acc(c, level, xs[t] + W, pt, acc + W);
  }
  oc_rescale_ct(c, level, 2, acc, out);
  free(acc); free(pt);
  return 0;
}

void oc_weighted_sum_cipher(const oc_ctx* c, const oc_keys* k, int level, int terms, const uint64_t* const* xs,
                            const uint64_t* const* ws, uint64_t* out) { /* ckks_backend.hpp:413-450 */
  /* size-3 accumulation of every x_t (x) w_t tensor product (poly_mul_acc, 437-440), one
     relinearisation (446), one rescale of each poly (448-450) */
  const int64_t W = (int64_t)(level + 1) * c->n;
  uint64_t* acc = calloc((size_t)(3 * W), sizeof(uint64_t));
  uint64_t* r2 = malloc(sizeof(uint64_t) * 2 * W);
  for (int t = 0; t < terms; ++t) {
    pw_mul_acc(c, level, xs[t], ws[t], acc);
    pw_mul_acc(c, level, xs[t], ws[t] + W, acc + W);
    pw_mul_acc(c, level, xs[t] + W, ws[t], acc + W);
    pw_mul_acc(c, level, xs[t] + W, ws[t] + W, acc + 2 * W);
  }
  oc_relinearize(c, k, level, acc, r2);
  oc_rescale_ct(c, level, 2, r2, out);
  free(acc); free(r2);
}

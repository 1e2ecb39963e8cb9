/*
 * oracle/oracle.c — plain, slow, obviously-correct CPU oracle for libfcirc.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2103_02605_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * What it computes (each function cites the passage it follows; PAPER.md line = P:n):
 *
 *   oracle_fcirc_entries   Definition 2, row-vector identification,
 *                          worked 3x3 example.  Written out with 0-based indices:
 *                            A[i][j] = a[(j-i) mod n] * (f if j < i else 1)
 *                            c_i     = sum_{j>=i} a_{j-i} b_j  +  f * sum_{j<i} a_{n+j-i} b_j   (mod p)
 *                          Algorithm 1 reaches exactly A*b in the ring (Theorem 1),
 *                          so the oracle is this definition, NOT Algorithm 1.  O(n) per entry.
 *   oracle_polymul_coeffs  the product of two polynomials: schoolbook coefficient
 *                            C_k = sum_{i} a_i b_{k-i} (mod p).  O(n) per coefficient.
 *   oracle_poly_eval       sum_i c_i x^i mod p by Horner's rule (used for the eigen-checksum of
 *                          SURVEY App. B.4 and Schwartz-Zippel checks; a plain definition).
 *   oracle_fcirc_entries_m31x2, oracle_polymul_coeffs_m31x2
 *                          the same definitions over the paper's own ring Z/pZ[sqrt 3],
 *                          p = 2^31 - 1, elements packed u | v << 32.
 *   oracle_fcirc_entries_batch, oracle_poly_eval_batch
 *                          the same two definitions over a whole batch of instances (instance k of
 *                          the caller's [batch][n] arrays with its own index / point list), threaded
 *                          over (instance, index) pairs.  No new arithmetic: each element is
 *                          fcirc_entry / the Horner loop above; only the indexing is batched.
 *   oracle_bigint_mul      product of two non-negative integers given as little-endian 32-bit
 *                          words (P:135-140 application): an independent Karatsuba recursion
 *                          (schoolbook below 32 words).  Exact, full product.
 *
 * Arithmetic: exact integers.  Products of two residues < 2^64 are formed in unsigned __int128
 * and summed into a 192-bit accumulator; a single reduction mod p happens per sum.  No Montgomery,
 * Shoup, Barrett, lazy reduction or special-prime tricks (those are the product's business).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

/* 192-bit accumulator: value = hi * 2^128 + lo */
typedef struct { u128 lo; uint64_t hi; } acc192;

static inline void acc_add(acc192* s, u128 v) {
  u128 t = s->lo + v;
  if (t < v) s->hi += 1;
  s->lo = t;
}

/* (hi * 2^128 + lo) mod p, by plain % on 128-bit pieces */
static uint64_t acc_mod(const acc192* s, uint64_t p) {
  u128 P = p;
  u128 two64 = (((u128)1) << 64) % P;           /* 2^64 mod p */
  u128 two128 = (two64 * two64) % P;             /* 2^128 mod p */
  u128 r = s->lo % P;
  u128 h = ((u128)s->hi) % P;
  r = (r + (h * two128) % P) % P;
  return (uint64_t)r;
}

static inline uint64_t mulmod(uint64_t x, uint64_t y, uint64_t p) {
  return (uint64_t)(((u128)x * (u128)y) % (u128)p);
}

/* one entry c_i of the f-circulant product, Definition 2 written out */
static uint64_t fcirc_entry(uint64_t p, uint64_t f, const uint64_t* a, const uint64_t* b,
                            int64_t n, int64_t i) {
  acc192 upper = {0, 0}, wrap = {0, 0};
  for (int64_t j = i; j < n; ++j)            /* j >= i: entry a_{j-i}, factor 1 */
    acc_add(&upper, (u128)a[j - i] * (u128)b[j]);
  for (int64_t j = 0; j < i; ++j)            /* j <  i: entry a_{n+j-i} * f (rule (2)) */
    acc_add(&wrap, (u128)a[n + j - i] * (u128)b[j]);
  uint64_t u = acc_mod(&upper, p), w = acc_mod(&wrap, p);
  return (uint64_t)(((u128)u + (u128)mulmod(f, w, p)) % (u128)p);
}

/* ---------------- threading helper ---------------- */
typedef struct {
  int kind;  /* 0 = fcirc entries, 1 = polymul coefficients, 2/3 = the same over Z/(2^31-1)[sqrt 3] */
  uint64_t p, f;
  const uint64_t *a, *b;
  int64_t n, na, nb;
  const int64_t* idx;
  uint64_t* out;
  int64_t lo, hi;
} job_t;

static uint64_t poly_coeff(uint64_t p, const uint64_t* a, int64_t na, const uint64_t* b,
                           int64_t nb, int64_t k) {
  acc192 s = {0, 0};
  int64_t i0 = k - (nb - 1); if (i0 < 0) i0 = 0;
  int64_t i1 = k; if (i1 > na - 1) i1 = na - 1;
  for (int64_t i = i0; i <= i1; ++i) acc_add(&s, (u128)a[i] * (u128)b[k - i]);
  return acc_mod(&s, p);
}

/* ---------------- the paper's ring Z/pZ[sqrt 3], p = 2^31 - 1 ----------------
 * u + v sqrt 3 packed as u | v << 32.  (u1 + v1 s)(u2 + v2 s) = (u1 u2 + 3 v1 v2) + (u1 v2 + u2 v1) s,
 * s^2 = 3.  Sums of products are accumulated exactly per component and reduced once. */
#define M31 2147483647ull
static inline uint64_t cu(uint64_t x) { return x & 0xFFFFFFFFull; }
static inline uint64_t cv(uint64_t x) { return x >> 32; }
static inline void fp2_acc(acc192* U, acc192* V, uint64_t x, uint64_t y) {
  acc_add(U, (u128)cu(x) * cu(y));
  acc_add(U, (u128)3 * ((u128)cv(x) * cv(y)));
  acc_add(V, (u128)cu(x) * cv(y));
  acc_add(V, (u128)cv(x) * cu(y));
}
static uint64_t fp2_mulp(uint64_t x, uint64_t y) {
  acc192 U = {0, 0}, V = {0, 0};
  fp2_acc(&U, &V, x, y);
  return acc_mod(&U, M31) | (acc_mod(&V, M31) << 32);
}
static uint64_t fp2_addp(uint64_t x, uint64_t y) {
  return ((cu(x) + cu(y)) % M31) | (((cv(x) + cv(y)) % M31) << 32);
}
/* c_i of Definition 2 over Z/pZ[sqrt 3] */
static uint64_t fcirc_entry_m31x2(uint64_t f, const uint64_t* a, const uint64_t* b, int64_t n, int64_t i) {
  acc192 Uu = {0, 0}, Uv = {0, 0}, Wu = {0, 0}, Wv = {0, 0};
  for (int64_t j = i; j < n; ++j) fp2_acc(&Uu, &Uv, a[j - i], b[j]);
  for (int64_t j = 0; j < i; ++j) fp2_acc(&Wu, &Wv, a[n + j - i], b[j]);
  const uint64_t up = acc_mod(&Uu, M31) | (acc_mod(&Uv, M31) << 32);
  const uint64_t wr = acc_mod(&Wu, M31) | (acc_mod(&Wv, M31) << 32);
  return fp2_addp(up, fp2_mulp(f, wr));
}
static uint64_t poly_coeff_m31x2(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb, int64_t k) {
  acc192 U = {0, 0}, V = {0, 0};
  int64_t i0 = k - (nb - 1); if (i0 < 0) i0 = 0;
  int64_t i1 = k; if (i1 > na - 1) i1 = na - 1;
  for (int64_t i = i0; i <= i1; ++i) fp2_acc(&U, &V, a[i], b[k - i]);
  return acc_mod(&U, M31) | (acc_mod(&V, M31) << 32);
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (int64_t t = J->lo; t < J->hi; ++t) {
    if (J->kind == 0) J->out[t] = fcirc_entry(J->p, J->f, J->a, J->b, J->n, J->idx[t]);
    else if (J->kind == 1) J->out[t] = poly_coeff(J->p, J->a, J->na, J->b, J->nb, J->idx[t]);
    else if (J->kind == 2) J->out[t] = fcirc_entry_m31x2(J->f, J->a, J->b, J->n, J->idx[t]);
    else J->out[t] = poly_coeff_m31x2(J->a, J->na, J->b, J->nb, J->idx[t]);
  }
  return NULL;
}

static int run_jobs(job_t proto, int64_t count, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (count < threads) threads = count > 0 ? (int)count : 1;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = proto;
    jobs[t].lo = count * t / threads;
    jobs[t].hi = count * (t + 1) / threads;
  }
  if (threads == 1) { worker(&jobs[0]); return 0; }
  int made[256];
  for (int t = 0; t < threads; ++t) {
    made[t] = pthread_create(&th[t], NULL, worker, &jobs[t]) == 0;
    if (!made[t]) worker(&jobs[t]);                  /* no thread: do this slice inline */
  }
  for (int t = 0; t < threads; ++t) if (made[t]) pthread_join(th[t], NULL);
  return 0;
}

/*
 * c[t] = (A*b)_{idx[t]} for the f-circulant A with first row a (Definition 2).
 * a, b: n residues in [0,p) (as uint64).  idx: nidx entry indices in [0,n).  out: nidx results.
 * p: any modulus 2 <= p < 2^64.  Returns 0, or -1 on bad arguments.
 */
int oracle_fcirc_entries(uint64_t p, uint64_t f, const uint64_t* a, const uint64_t* b, int64_t n,
                         const int64_t* idx, int64_t nidx, uint64_t* out, int threads) {
  if (!a || !b || !idx || !out || n < 1 || nidx < 0 || p < 2) return -1;
  for (int64_t t = 0; t < nidx; ++t) if (idx[t] < 0 || idx[t] >= n) return -1;
  job_t J = {0, p, f % p, a, b, n, 0, 0, idx, out, 0, 0};
  return run_jobs(J, nidx, threads);
}

/*
 * out[t] = C_{ks[t]} where C(x) = a(x) b(x) mod p (schoolbook).
 * a: na coefficients, b: nb coefficients (low order first), ks in [0, na+nb-1).
 */
int oracle_polymul_coeffs(uint64_t p, const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb,
                          const int64_t* ks, int64_t nk, uint64_t* out, int threads) {
  if (!a || !b || !ks || !out || na < 1 || nb < 1 || nk < 0 || p < 2) return -1;
  for (int64_t t = 0; t < nk; ++t) if (ks[t] < 0 || ks[t] >= na + nb - 1) return -1;
  job_t J = {1, p, 0, a, b, 0, na, nb, ks, out, 0, 0};
  return run_jobs(J, nk, threads);
}

/* out[t] = sum_{i<n} c_i xs[t]^i mod p (Horner, one reduction per step), for nx points */
typedef struct { uint64_t p; const uint64_t* c; int64_t n; const uint64_t* xs; uint64_t* out; int64_t lo, hi; } ejob_t;
static void* eval_worker(void* arg) {
  ejob_t* J = (ejob_t*)arg;
  for (int64_t t = J->lo; t < J->hi; ++t) {
    u128 acc = 0, x = J->xs[t] % J->p;
    for (int64_t i = J->n - 1; i >= 0; --i) acc = (acc * x + J->c[i]) % J->p;
    J->out[t] = (uint64_t)acc;
  }
  return NULL;
}
int oracle_poly_eval(uint64_t p, const uint64_t* c, int64_t n, const uint64_t* xs, int64_t nx, uint64_t* out,
                     int threads) {
  if (!c || !xs || !out || n < 1 || nx < 0 || p < 2) return -1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (nx < threads) threads = nx > 0 ? (int)nx : 1;
  pthread_t th[256]; ejob_t jobs[256]; int made[256];
  for (int t = 0; t < threads; ++t) {
    ejob_t J = {p, c, n, xs, out, nx * t / threads, nx * (t + 1) / threads};
    jobs[t] = J;
  }
  for (int t = 0; t < threads; ++t) {
    made[t] = threads > 1 && pthread_create(&th[t], NULL, eval_worker, &jobs[t]) == 0;
    if (!made[t]) eval_worker(&jobs[t]);
  }
  for (int t = 0; t < threads; ++t) if (made[t]) pthread_join(th[t], NULL);
  return 0;
}

/* ---------------- big integers: independent Karatsuba on 32-bit words ---------------- */

/* z[0..nx+ny) = x * y, schoolbook */
static void school(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z) {
  memset(z, 0, sizeof(uint32_t) * (size_t)(nx + ny));
  for (int64_t i = 0; i < nx; ++i) {
    uint64_t carry = 0;
    for (int64_t j = 0; j < ny; ++j) {
      uint64_t t = (uint64_t)x[i] * y[j] + z[i + j] + carry;
      z[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    int64_t k = i + ny;
    while (carry) { uint64_t t = (uint64_t)z[k] + carry; z[k] = (uint32_t)t; carry = t >> 32; ++k; }
  }
}

/* z += w (lengths: z has nz words, w has nw <= nz words); returns carry out */
static uint32_t add_into(uint32_t* z, int64_t nz, const uint32_t* w, int64_t nw) {
  uint64_t c = 0;
  int64_t i = 0;
  for (; i < nw; ++i) { uint64_t t = (uint64_t)z[i] + w[i] + c; z[i] = (uint32_t)t; c = t >> 32; }
  for (; c && i < nz; ++i) { uint64_t t = (uint64_t)z[i] + c; z[i] = (uint32_t)t; c = t >> 32; }
  return (uint32_t)c;
}

/* z -= w (z >= w as integers); nz >= nw */
static void sub_from(uint32_t* z, int64_t nz, const uint32_t* w, int64_t nw) {
  int64_t borrow = 0;
  int64_t i = 0;
  for (; i < nw; ++i) {
    int64_t t = (int64_t)z[i] - (int64_t)w[i] - borrow;
    borrow = t < 0; z[i] = (uint32_t)(t + (borrow ? ((int64_t)1 << 32) : 0));
  }
  for (; borrow && i < nz; ++i) {
    int64_t t = (int64_t)z[i] - borrow;
    borrow = t < 0; z[i] = (uint32_t)(t + (borrow ? ((int64_t)1 << 32) : 0));
  }
}

/* Karatsuba for equal lengths n: z[0..2n) = x*y.
 *   x = x1 B^h + x0, y = y1 B^h + y0 (B = 2^32, h = floor(n/2))
 *   z0 = x0 y0, z2 = x1 y1, z1 = (x0+x1)(y0+y1) - z0 - z2
 *   xy = z2 B^{2h} + z1 B^h + z0                                              */
static void kara(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* z) {
  if (n <= 32) { school(x, n, y, n, z); return; }
  int64_t h = n / 2, hh = n - h;                     /* low part h words, high part hh words */
  uint32_t* sx = (uint32_t*)calloc((size_t)(hh + 1), 4);
  uint32_t* sy = (uint32_t*)calloc((size_t)(hh + 1), 4);
  memcpy(sx, x + h, (size_t)hh * 4); sx[hh] = add_into(sx, hh, x, h);
  memcpy(sy, y + h, (size_t)hh * 4); sy[hh] = add_into(sy, hh, y, h);
  uint32_t* z1 = (uint32_t*)calloc((size_t)(2 * (hh + 1)), 4);
  kara(sx, sy, hh + 1, z1);
  uint32_t* z0 = (uint32_t*)calloc((size_t)(2 * h), 4);
  uint32_t* z2 = (uint32_t*)calloc((size_t)(2 * hh), 4);
  kara(x, y, h, z0);
  kara(x + h, y + h, hh, z2);
  sub_from(z1, 2 * (hh + 1), z0, 2 * h);
  sub_from(z1, 2 * (hh + 1), z2, 2 * hh);
  memset(z, 0, (size_t)(2 * n) * 4);
  memcpy(z, z0, (size_t)(2 * h) * 4);
  add_into(z + 2 * h, 2 * n - 2 * h, z2, 2 * hh);
  int64_t n1 = 2 * (hh + 1);
  if (h + n1 > 2 * n) n1 = 2 * n - h;                /* top words of z1 are zero by magnitude */
  add_into(z + h, 2 * n - h, z1, n1);
  free(sx); free(sy); free(z0); free(z1); free(z2);
}

/*
 * z[0..nx+ny) = x * y for little-endian 32-bit word arrays (non-negative magnitudes).
 * Unequal lengths: the shorter operand is zero-extended (Karatsuba on equal halves).
 */
int oracle_bigint_mul(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z) {
  if (!x || !y || !z || nx < 1 || ny < 1) return -1;
  int64_t n = nx > ny ? nx : ny;
  uint32_t* xx = (uint32_t*)calloc((size_t)n, 4);
  uint32_t* yy = (uint32_t*)calloc((size_t)n, 4);
  uint32_t* zz = (uint32_t*)calloc((size_t)(2 * n), 4);
  if (!xx || !yy || !zz) { free(xx); free(yy); free(zz); return -1; }
  memcpy(xx, x, (size_t)nx * 4);
  memcpy(yy, y, (size_t)ny * 4);
  kara(xx, yy, n, zz);
  memcpy(z, zz, (size_t)(nx + ny) * 4);              /* words above nx+ny are zero */
  free(xx); free(yy); free(zz);
  return 0;
}

/* schoolbook product, exposed so tests can cross-check the Karatsuba split logic */
int oracle_bigint_mul_school(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z) {
  if (!x || !y || !z || nx < 1 || ny < 1) return -1;
  school(x, nx, y, ny, z);
  return 0;
}

/*
 * The same two definitions over the paper's ring Z/pZ[sqrt 3], p = 2^31 - 1: elements and f
 * packed u | v << 32 with u, v < p.  Returns 0, or -1 on bad arguments.
 */
int oracle_fcirc_entries_m31x2(uint64_t f, const uint64_t* a, const uint64_t* b, int64_t n, const int64_t* idx,
                               int64_t nidx, uint64_t* out, int threads) {
  if (!a || !b || !idx || !out || n < 1 || nidx < 0) return -1;
  for (int64_t t = 0; t < nidx; ++t) if (idx[t] < 0 || idx[t] >= n) return -1;
  job_t J = {2, M31, f, a, b, n, 0, 0, idx, out, 0, 0};
  return run_jobs(J, nidx, threads);
}

int oracle_polymul_coeffs_m31x2(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb, const int64_t* ks,
                                int64_t nk, uint64_t* out, int threads) {
  if (!a || !b || !ks || !out || na < 1 || nb < 1 || nk < 0) return -1;
  for (int64_t t = 0; t < nk; ++t) if (ks[t] < 0 || ks[t] > na + nb - 2) return -1;
  job_t J = {3, M31, 0, a, b, 0, na, nb, ks, out, 0, 0};
  return run_jobs(J, nk, threads);
}

/* ---------------- batched forms (indexing only; the arithmetic is fcirc_entry / Horner) ----------------
 * Instance k uses a + k n, b + k n, its index list idx + k nidx and writes out + k nidx.  Work items
 * (k, t) are split evenly across the threads. */
typedef struct {
  int kind;                 /* 0: fcirc entries, 1: Horner evaluation */
  uint64_t p, f;
  const uint64_t *a, *b;    /* kind 1: a = c, b unused */
  int64_t n, per;           /* per = nidx (kind 0) or nx (kind 1) */
  const int64_t* idx;
  const uint64_t* xs;
  uint64_t* out;
  int64_t lo, hi;           /* flat work-item range [lo, hi) over batch * per */
} bjob_t;

static void* batch_worker(void* arg) {
  bjob_t* J = (bjob_t*)arg;
  for (int64_t w = J->lo; w < J->hi; ++w) {
    const int64_t k = w / J->per;
    if (J->kind == 0) {
      J->out[w] = fcirc_entry(J->p, J->f, J->a + k * J->n, J->b + k * J->n, J->n, J->idx[w]);
    } else {
      const uint64_t* c = J->a + k * J->n;
      u128 acc = 0, x = J->xs[w] % J->p;
      for (int64_t i = J->n - 1; i >= 0; --i) acc = (acc * x + c[i]) % J->p;
      J->out[w] = (uint64_t)acc;
    }
  }
  return NULL;
}

static int run_batch(bjob_t proto, int64_t items, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (items < threads) threads = items > 0 ? (int)items : 1;
  pthread_t th[256]; bjob_t jobs[256]; int made[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = proto;
    jobs[t].lo = items * t / threads;
    jobs[t].hi = items * (t + 1) / threads;
  }
  for (int t = 0; t < threads; ++t) {
    made[t] = threads > 1 && pthread_create(&th[t], NULL, batch_worker, &jobs[t]) == 0;
    if (!made[t]) batch_worker(&jobs[t]);
  }
  for (int t = 0; t < threads; ++t) if (made[t]) pthread_join(th[t], NULL);
  return 0;
}

/* out[k][t] = (A_k b_k)_{idx[k][t]}: Definition 2 per instance, a, b: [batch][n] */
int oracle_fcirc_entries_batch(uint64_t p, uint64_t f, const uint64_t* a, const uint64_t* b, int64_t n,
                               int64_t batch, const int64_t* idx, int64_t nidx, uint64_t* out, int threads) {
  if (!a || !b || !idx || !out || n < 1 || batch < 0 || nidx < 0 || p < 2) return -1;
  for (int64_t t = 0; t < batch * nidx; ++t) if (idx[t] < 0 || idx[t] >= n) return -1;
  bjob_t J = {0, p, f % p, a, b, n, nidx, idx, NULL, out, 0, 0};
  return run_batch(J, batch * nidx, threads);
}

/* out[k][t] = sum_i c[k][i] xs[k][t]^i mod p (Horner), c: [batch][n], xs: [batch][nx] */
int oracle_poly_eval_batch(uint64_t p, const uint64_t* c, int64_t n, int64_t batch, const uint64_t* xs, int64_t nx,
                           uint64_t* out, int threads) {
  if (!c || !xs || !out || n < 1 || batch < 0 || nx < 0 || p < 2) return -1;
  bjob_t J = {1, p, 0, c, NULL, n, nx, NULL, xs, out, 0, 0};
  return run_batch(J, batch * nx, threads);
}

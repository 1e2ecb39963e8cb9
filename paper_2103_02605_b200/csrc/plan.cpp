// plan.cpp — prime registry, modular helpers, n-th roots and twist tables (host, O(n)).
#include "plan.h"
#include "../../include/fcirc.h"

namespace fcirc {

typedef unsigned __int128 u128;

static const PrimeInfo kPrimes[] = {
    {998244353ull, 23, 3ull, false, KIND_U32},           // 119 * 2^23 + 1
    {469762049ull, 26, 3ull, false, KIND_U32},           //   7 * 2^26 + 1
    {167772161ull, 25, 3ull, false, KIND_U32},           //   5 * 2^25 + 1
    {0xFFFFFFFF00000001ull, 32, 7ull, true, KIND_GOLD},  // (2^32 - 1) * 2^32 + 1
    // Z/pZ[sqrt 3], p = 2^31 - 1: |F_{p^2}^*| = p^2 - 1 = 2^32 (2^30 - 1)
    {kM31, 32, 0ull, true, KIND_M31X2},
};

const PrimeInfo* prime_info(uint64_t p) {
  for (const auto& q : kPrimes)
    if (q.p == p) return &q;
  return nullptr;
}

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }

uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = mulmod(r, a, p);
    a = mulmod(a, a, p);
    e >>= 1;
  }
  return r;
}

uint64_t invmod(uint64_t a, uint64_t p) { return powmod(a, p - 2, p); }

// Tonelli-Shanks with the registry's generator as the non-residue
bool sqrtmod(uint64_t x, uint64_t p, const PrimeInfo& pi, uint64_t* y) {
  x %= p;
  if (x == 0) { *y = 0; return true; }
  if (powmod(x, (p - 1) / 2, p) != 1) return false;
  int S = pi.two_adicity;
  uint64_t Q = (p - 1) >> S;
  uint64_t c = powmod(pi.g, Q, p);          // primitive 2^S-th root of unity
  uint64_t t = powmod(x, Q, p);
  uint64_t r = powmod(x, (Q + 1) / 2, p);
  int Mv = S;
  while (t != 1) {
    int i = 0;
    uint64_t t2 = t;
    while (t2 != 1) { t2 = mulmod(t2, t2, p); ++i; }
    uint64_t b = c;
    for (int j = 0; j < Mv - i - 1; ++j) b = mulmod(b, b, p);
    Mv = i;
    c = mulmod(b, b, p);
    t = mulmod(t, c, p);
    r = mulmod(r, b, p);
  }
  *y = r;
  return true;
}

// x is a 2^j-th power  <=>  x^((p-1)/gcd(2^j, p-1)) == 1; with 2^j | p-1 that is x^((p-1)/2^j) == 1
static bool is_pow2_power(uint64_t x, int j, const PrimeInfo& pi) {
  if (j > pi.two_adicity) j = pi.two_adicity;
  return powmod(x, (pi.p - 1) >> j, pi.p) == 1;
}

bool nth_root_pow2(uint64_t f, int L, const PrimeInfo& pi, uint64_t* w) {
  uint64_t p = pi.p;
  f %= p;
  if (f == 0) return false;
  if (!is_pow2_power(f, L, pi)) return false;
  uint64_t x = f;
  for (int j = L; j >= 1; --j) {
    // x is a 2^j-th power; pick the square root that is a 2^(j-1)-th power
    uint64_t r;
    if (!sqrtmod(x, p, pi, &r)) return false;
    if (j - 1 >= 1 && !is_pow2_power(r, j - 1, pi)) r = (p - r) % p;
    x = r;
  }
  if (powmod(x, (uint64_t)1 << L, p) != f) return false;
  *w = x;
  return true;
}

static inline uint32_t brv(uint32_t e, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((e >> i) & 1u) << (bits - 1 - i);
  return r;
}

// ------------------------------------------------------------------------------------------
// Z/pZ[sqrt 3], p = 2^31 - 1 (the paper's ring)
// ------------------------------------------------------------------------------------------
Fp2 fp2_unpack(uint64_t x) { return Fp2{x & 0xFFFFFFFFull, x >> 32}; }
uint64_t fp2_pack(Fp2 a) { return a.u | (a.v << 32); }
bool fp2_canonical(uint64_t x) { return (x & 0xFFFFFFFFull) < kM31 && (x >> 32) < kM31; }
Fp2 fp2_mul(Fp2 a, Fp2 b) {
  const uint64_t p = kM31;
  return Fp2{(mulmod(a.u, b.u, p) + 3 * mulmod(a.v, b.v, p)) % p, (mulmod(a.u, b.v, p) + mulmod(a.v, b.u, p)) % p};
}
Fp2 fp2_pow(Fp2 a, uint64_t e) {
  Fp2 r{1, 0};
  while (e) {
    if (e & 1) r = fp2_mul(r, a);
    a = fp2_mul(a, a);
    e >>= 1;
  }
  return r;
}
bool fp2_is_zero(Fp2 a) { return a.u == 0 && a.v == 0; }
bool fp2_eq(Fp2 a, Fp2 b) { return a.u == b.u && a.v == b.v; }
// (u + v sqrt 3)^-1 = (u - v sqrt 3) / (u^2 - 3 v^2); the norm is nonzero for a != 0 (3 is a non-residue)
Fp2 fp2_inv(Fp2 a) {
  const uint64_t p = kM31;
  const uint64_t nrm = (mulmod(a.u, a.u, p) + p - mulmod(3, mulmod(a.v, a.v, p), p)) % p;
  const uint64_t ni = invmod(nrm, p);
  return Fp2{mulmod(a.u, ni, p), mulmod((p - a.v) % p, ni, p)};
}

static constexpr uint64_t kFp2Order = ((uint64_t)kM31 * kM31) - 1;   // 2^32 (2^30 - 1)
static constexpr int kFp2S = 32;
static constexpr uint64_t kFp2Q = kFp2Order >> kFp2S;               // 2^30 - 1 (odd)

static bool fp2_is_one(Fp2 a) { return a.u == 1 && a.v == 0; }
// x is a 2^j-th power in the cyclic group F_{p^2}^*  <=>  x^(order / 2^j) == 1
static bool fp2_is_pow2_power(Fp2 x, int j) { return fp2_is_one(fp2_pow(x, kFp2Order >> j)); }

// a generator of the 2-Sylow subgroup (order 2^32): z^q for the first non-square z = k + sqrt 3
static Fp2 fp2_sylow_gen() {
  static const Fp2 c = [] {
    for (uint64_t k = 0;; ++k) {
      const Fp2 z{k, 1};
      if (!fp2_is_pow2_power(z, 1)) return fp2_pow(z, kFp2Q);
    }
  }();
  return c;
}

// Tonelli-Shanks in the cyclic group F_{p^2}^* of order 2^32 q
static bool fp2_sqrt(Fp2 x, Fp2* y) {
  if (fp2_is_zero(x)) { *y = x; return true; }
  if (!fp2_is_pow2_power(x, 1)) return false;
  int Mv = kFp2S;
  Fp2 c = fp2_sylow_gen();
  Fp2 t = fp2_pow(x, kFp2Q);
  Fp2 r = fp2_pow(x, (kFp2Q + 1) / 2);
  while (!fp2_is_one(t)) {
    int i = 0;
    Fp2 t2 = t;
    while (!fp2_is_one(t2)) { t2 = fp2_mul(t2, t2); ++i; }
    Fp2 b = c;
    for (int j = 0; j < Mv - i - 1; ++j) b = fp2_mul(b, b);
    Mv = i;
    c = fp2_mul(b, b);
    t = fp2_mul(t, c);
    r = fp2_mul(r, b);
  }
  *y = r;
  return true;
}

// w with w^(2^L) = f, by L square roots each chosen to remain a 2^(j-1)-th power
static bool fp2_nth_root_pow2(Fp2 f, int L, Fp2* w) {
  if (fp2_is_zero(f) || !fp2_is_pow2_power(f, L)) return false;
  Fp2 x = f;
  for (int j = L; j >= 1; --j) {
    Fp2 r;
    if (!fp2_sqrt(x, &r)) return false;
    if (j - 1 >= 1 && !fp2_is_pow2_power(r, j - 1)) r = Fp2{(kM31 - r.u) % kM31, (kM31 - r.v) % kM31};
    x = r;
  }
  if (!fp2_eq(fp2_pow(x, (uint64_t)1 << L), f)) return false;
  *w = x;
  return true;
}

static inline uint32_t brv_(uint32_t e, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((e >> i) & 1u) << (bits - 1 - i);
  return r;
}

// The same twist table as build_host_plan (heap index 2^d + e: s_{d,e} = w^{n/2^{d+1}}
// zeta_{2^{d+1}}^{brv_d(e)}), over Z/pZ[sqrt 3] with the paper's roots of unity
// zeta_N = (2 + sqrt 3)^{(p+1)/N} (2 + sqrt 3 has order p + 1 = 2^31).
static int build_host_plan_fp2(uint64_t f_packed, int L, HostPlan* out) {
  if (L > 31) return FCIRC_ESIZE;                       // zeta_n from the order-2^31 subgroup
  if (!fp2_canonical(f_packed)) return FCIRC_EINVAL;
  const Fp2 f = fp2_unpack(f_packed);
  Fp2 w;
  if (!fp2_nth_root_pow2(f, L, &w)) return FCIRC_ENOROOT;  // f = 0 or no n-th root
  const uint64_t n = (uint64_t)1 << L;
  out->p = kM31; out->f = f_packed; out->w = fp2_pack(w); out->L = L;
  const Fp2 ninv{invmod(n % kM31, kM31), 0};
  out->K = fp2_pack(ninv);
  if (L == 0) {
    out->s.assign(1, 0); out->sinv.assign(1, 0); out->last_si = 0;
    return FCIRC_OK;
  }
  const Fp2 zn = fp2_pow(Fp2{2, 1}, ((uint64_t)1 << 31) >> L);   // (2 + sqrt 3)^{(p+1)/n}
  std::vector<Fp2> z(n);
  z[0] = Fp2{1, 0};
  for (uint64_t i = 1; i < n; ++i) z[i] = fp2_mul(z[i - 1], zn);
  const Fp2 winv = fp2_inv(w);
  out->s.assign(n, 0);
  out->sinv.assign(n, 0);
  for (int d = 0; d < L; ++d) {
    const Fp2 xd = fp2_pow(w, n >> (d + 1)), xdi = fp2_pow(winv, n >> (d + 1));
    const uint64_t stride = n >> (d + 1);
    for (uint64_t e = 0; e < ((uint64_t)1 << d); ++e) {
      const uint64_t ex = (uint64_t)brv_((uint32_t)e, d) * stride;
      out->s[((uint64_t)1 << d) + e] = fp2_pack(fp2_mul(xd, z[ex]));
      out->sinv[((uint64_t)1 << d) + e] = fp2_pack(fp2_mul(xdi, z[(n - ex) % n]));
    }
  }
  out->last_si = fp2_pack(fp2_mul(fp2_unpack(out->sinv[1]), ninv));
  return FCIRC_OK;
}

int check_premises(const PrimeInfo* pi, uint64_t f, int L) {
  if (pi->kind == KIND_M31X2) {
    if (L > 31) return FCIRC_ESIZE;
    if (!fp2_canonical(f)) return FCIRC_EINVAL;
    const Fp2 x = fp2_unpack(f);
    if (fp2_is_zero(x) || !fp2_is_pow2_power(x, L)) return FCIRC_ENOROOT;
    return FCIRC_OK;
  }
  const uint64_t p = pi->p;
  if (L > pi->two_adicity) return FCIRC_ESIZE;
  if (f % p == 0 || powmod(f % p, (p - 1) >> L, p) != 1) return FCIRC_ENOROOT;
  return FCIRC_OK;
}

int build_host_plan(uint64_t p, uint64_t f, int L, HostPlan* out) {
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  if (pi->kind == KIND_M31X2) return build_host_plan_fp2(f, L, out);
  if (L > pi->two_adicity) return FCIRC_ESIZE;     // no n-th root of unity
  f %= p;
  if (f == 0) return FCIRC_ENOROOT;                 // f^-1 must exist
  uint64_t w;
  if (!nth_root_pow2(f, L, *pi, &w)) return FCIRC_ENOROOT;
  const uint64_t n = (uint64_t)1 << L;
  out->p = p; out->f = f; out->w = w; out->L = L;
  const uint64_t ninv = invmod(n % p, p);
  out->K = pi->wide ? ninv : mulmod(ninv, ((uint64_t)1 << 32) % p, p);
  if (L == 0) {
    out->s.assign(1, 0); out->sinv.assign(1, 0); out->last_si = 0;
    return FCIRC_OK;
  }
  // zeta_n powers z[i] = zeta_n^i, i < n  (zeta_n = g^((p-1)/n))
  const uint64_t zn = powmod(pi->g, (p - 1) >> L, p);
  std::vector<uint64_t> z(n);
  z[0] = 1;
  for (uint64_t i = 1; i < n; ++i) z[i] = mulmod(z[i - 1], zn, p);
  const uint64_t winv = invmod(w, p);
  out->s.assign(n, 0);
  out->sinv.assign(n, 0);
  uint64_t xd = powmod(w, n >> 1, p), xdi = powmod(winv, n >> 1, p);  // w^{n/2^{d+1}} at d = 0
  for (int d = 0; d < L; ++d) {
    const uint64_t stride = n >> (d + 1);  // zeta_{2^{d+1}} = zeta_n^{n / 2^{d+1}}
    for (uint64_t e = 0; e < ((uint64_t)1 << d); ++e) {
      const uint64_t ex = (uint64_t)brv((uint32_t)e, d) * stride;  // exponent of zeta_n, < n/2
      out->s[((uint64_t)1 << d) + e] = mulmod(xd, z[ex], p);
      out->sinv[((uint64_t)1 << d) + e] = mulmod(xdi, z[(n - ex) % n], p);
    }
    if (d + 1 < L) {  // w^{n/2^{d+2}}: the square root along the chain w^{n/2}, w^{n/4}, ...
      xd = powmod(w, n >> (d + 2), p);
      xdi = powmod(winv, n >> (d + 2), p);
    }
  }
  out->last_si = mulmod(out->sinv[1], out->K, p);
  return FCIRC_OK;
}

}  // namespace fcirc

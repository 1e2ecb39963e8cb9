// plan.cpp — prime registry, modular helpers, n-th roots and twist tables (host, O(n)).
#include "plan.h"
#include "../../include/fcirc.h"

namespace fcirc {

typedef unsigned __int128 u128;

static const PrimeInfo kPrimes[] = {
    {998244353ull, 23, 3ull, false},             // 119 * 2^23 + 1
    {469762049ull, 26, 3ull, false},             //   7 * 2^26 + 1
    {167772161ull, 25, 3ull, false},             //   5 * 2^25 + 1
    {0xFFFFFFFF00000001ull, 32, 7ull, true},     // (2^32 - 1) * 2^32 + 1
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

int build_host_plan(uint64_t p, uint64_t f, int L, HostPlan* out) {
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
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

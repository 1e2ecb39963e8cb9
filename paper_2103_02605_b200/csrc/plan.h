// plan.h — host-side twist-table plans.
//
// Theorem 1 premises: n = 2^L, an n-th root of f, an n-th root of unity, 2^-1, f^-1.
// The recursion gives block (d, e) the scalar f_{d,e}; its children carry +sqrt and -sqrt of it
// (P:96-100).  With w^n = f and zeta_m a primitive m-th root of unity, a consistent choice of all
// square roots is
//     s_{d,e} = w^{n / 2^{d+1}} * zeta_{2^{d+1}}^{brv_d(e)}        (heap index 2^d + e)
// since s_{d,e}^2 = w^{n/2^d} zeta_{2^d}^{brv_d(e)} = f_{d,e} and brv_d(2e+1) = brv_{d-1}(e)+2^{d-1}
// supplies the sign of the second child.  The product does not depend on which roots are chosen
// (reading R2; pinned by the random-sign Algorithm 1 test).  Tables are built on the
// host in O(n) ("the roots needed by Algorithm 1 can be precomputed in linear time") and
// the inverses come from the same powers of w and zeta (P:111's inverse-root remark).
#pragma once
#include <cstdint>
#include <cstddef>
#include <vector>

namespace fcirc {

struct PrimeInfo {
  uint64_t p;
  int two_adicity;  // largest S with 2^S | p-1
  uint64_t g;       // a generator of (Z/p)^*
  bool wide;        // element type uint64 (Goldilocks) vs uint32
};

// nullptr if p is not in the registry
const PrimeInfo* prime_info(uint64_t p);

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p);
uint64_t powmod(uint64_t a, uint64_t e, uint64_t p);
uint64_t invmod(uint64_t a, uint64_t p);  // a != 0, p prime
// some y with y^2 = x (mod p), or false if x is a non-residue
bool sqrtmod(uint64_t x, uint64_t p, const PrimeInfo& pi, uint64_t* y);
// some w with w^(2^L) = f, or false (f is not a 2^L-th power)
bool nth_root_pow2(uint64_t f, int L, const PrimeInfo& pi, uint64_t* w);

// Host image of a plan: heap-indexed tables (index 0 unused) plus the scaling constants.
struct HostPlan {
  uint64_t p = 0, f = 0, w = 0;
  int L = 0;
  std::vector<uint64_t> s;     // s[2^d + e] = s_{d,e}, size n (n >= 2), entry 0 = 0
  std::vector<uint64_t> sinv;  // s_{d,e}^-1
  uint64_t K = 0;              // final scale: n^-1 (Goldilocks) or n^-1 * 2^32 (32-bit, Montgomery leaves)
  uint64_t last_si = 0;        // s_{0,0}^-1 * K
};

// status: 0 ok, or FCIRC_ENOROOT / FCIRC_ESIZE
int build_host_plan(uint64_t p, uint64_t f, int L, HostPlan* out);

}  // namespace fcirc

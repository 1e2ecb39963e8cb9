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

// Field kinds of the registry: the ring R of Theorem 1
enum FieldKind { KIND_U32 = 0, KIND_GOLD = 1, KIND_M31X2 = 2 };

struct PrimeInfo {
  uint64_t p;
  int two_adicity;  // largest S with 2^S | (group order): p-1, or p^2-1 for the quadratic extension
  uint64_t g;       // a generator of (Z/p)^* (unused for KIND_M31X2)
  bool wide;        // element type uint64 (Goldilocks, packed Z/p[sqrt 3]) vs uint32
  int kind;         // FieldKind
};

// The paper's own ring: Z/pZ[sqrt 3], p = 2^31 - 1 (3 is a non-residue mod p).  An element
// u + v sqrt 3 (u, v < p) is packed into a uint64 as u | v << 32.
constexpr uint64_t kM31 = 0x7FFFFFFFull;
struct Fp2 {
  uint64_t u = 0, v = 0;
};
Fp2 fp2_unpack(uint64_t x);
uint64_t fp2_pack(Fp2 a);
Fp2 fp2_mul(Fp2 a, Fp2 b);
Fp2 fp2_pow(Fp2 a, uint64_t e);
Fp2 fp2_inv(Fp2 a);
bool fp2_is_zero(Fp2 a);
bool fp2_eq(Fp2 a, Fp2 b);
// x is canonical (both components < p)
bool fp2_canonical(uint64_t x);

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

// status: 0 ok, or FCIRC_ENOROOT / FCIRC_ESIZE (FCIRC_EINVAL: non-canonical packed f of Z/p[sqrt 3])
int build_host_plan(uint64_t p, uint64_t f, int L, HostPlan* out);
// Theorem 1 premises for a product of order 2^L with scalar f: FCIRC_OK / ESIZE / ENOROOT / EINVAL
int check_premises(const PrimeInfo* pi, uint64_t f, int L);

}  // namespace fcirc

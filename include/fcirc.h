/*
 * include/fcirc.h — C ABI of libfcirc, the B200-native (sm_100a) f-circulant matrix-vector
 * product over Z/p and its applications, after arXiv 2103.02605 ("On Fast Computation of a
 * Circulant Matrix-Vector Product").  Citations "P:n" are lines of the paper's PAPER.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Arithmetic is exact modular integer arithmetic; there is no floating point and no rounding.
 *  - Supported moduli ("the registry"):
 *        998244353  = 119*2^23 + 1   (element type uint32_t)
 *        469762049  =   7*2^26 + 1   (uint32_t)
 *        167772161  =   5*2^25 + 1   (uint32_t)
 *        18446744069414584321 = 2^64 - 2^32 + 1  "Goldilocks"  (uint64_t)
 *        2147483647 = 2^31 - 1 selects the paper's own ring Z/pZ[sqrt 3] (3 is a non-residue):
 *          an element u + v sqrt 3 (u, v < p) is a uint64_t packed as u | v << 32, and so is f;
 *          roots of unity are the paper's (2 + sqrt 3)^((p+1)/N); n <= 2^24
 *    The element type of a, b, c follows p: uint32_t for the three 32-bit primes, uint64_t for
 *    Goldilocks.  Inputs must be canonical residues in [0, p) (precondition, not checked on the
 *    device unless the environment sets FCIRC_CHECK_INPUTS=1: then fcirc_matvec / fcirc_polymul
 *    first count non-canonical inputs, synchronise the stream and return FCIRC_EINVAL if there
 *    are any); outputs are canonical.
 *  - Layout: row-major [batch][len], contiguous; instance k starts at element k*len.
 *  - Data pointers are DEVICE pointers owned by the caller, except the *_host entry points,
 *    whose data pointers are HOST pointers (pinned memory gives full PCIe bandwidth).
 *  - Device calls are asynchronous and stream-ordered on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).  The return value reports argument validation,
 *    plan construction and launch errors only; device faults surface at the caller's next
 *    synchronisation.  The first call for a new (device, p, f, n) builds a twist-table plan on
 *    the host and uploads it (synchronous w.r.t. the host, cached afterwards).
 *  - Thread safety: calls may be made concurrently from several host threads; the plan cache is
 *    mutex-guarded (LRU, at most 64 plans / 2 GiB of tables).  Scratch memory is allocated
 *    stream-ordered from the device's default memory pool (cudaMallocAsync / cudaFreeAsync on
 *    `stream`), so concurrent calls on different streams never share it.
 *  - CUDA graphs: a call can be captured into a graph once its plan exists (the first call for a
 *    (device, p, f, n) must happen outside capture; inside a capture it returns FCIRC_EINVAL).  A
 *    plan used during a capture is pinned in the cache -- never evicted -- so the graph may be
 *    replayed at any later time; fcirc_release_cache drops pinned plans too, after which such
 *    graphs must not be replayed.  Evicted (unpinned) plans free their tables stream-ordered after
 *    every recorded use has completed (no device-wide synchronisation, safe during other threads'
 *    captures).
 *  - Nothing here ever falls back to a CPU implementation.
 */
#ifndef FCIRC_H
#define FCIRC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (0 = success, negative = error) */
#define FCIRC_OK 0
#define FCIRC_EINVAL (-1)  /* null pointer, len < 1, batch < 1, n not a power of two, overlap of c with a/b */
#define FCIRC_EPRIME (-2)  /* p not in the registry */
#define FCIRC_ENOROOT (-3) /* f == 0 mod p (no f^-1) or f has no n-th root (f^((p-1)/n) != 1) */
#define FCIRC_ESIZE (-4)   /* n does not divide p-1 (no n-th root of unity) or n above the supported maximum */
#define FCIRC_ENOMEM (-5)  /* device allocation of a plan table or workspace failed */
#define FCIRC_ECUDA (-6)   /* a CUDA API call or kernel launch failed */

/*
 * fcirc_matvec — c = A b for a batch of f-circulant matrices (Definition 2).
 *
 * A is identified by its FIRST ROW a and the scalar f; with 0-based indices
 *     A[i][j] = a[(j - i) mod n] * (f if j < i else 1),
 *     c_i     = sum_{j >= i} a_{j-i} b_j + f * sum_{j < i} a_{n+j-i} b_j        (mod p).
 * (The 3x3 example of P:40-46 is this rule.)  f = 1 is the usual circulant: a cyclic
 * correlation; f = p-1 the negacyclic case.
 *
 * Method: Theorem 1 / Algorithm 1 applied recursively, iteratively and in
 * place, with a precomputed twist table of n-th roots of f and roots of unity.
 * Premises of Theorem 1: n a power of two, n | p-1, f != 0 and f an n-th power.
 *
 *   p      modulus from the registry
 *   f      the scalar of the f-circulant, reduced mod p by the library
 *   a      [batch][n] first rows (device)          b  [batch][n] vectors (device)
 *   c      [batch][n] results (device); must not overlap a or b
 *   n      matrix order, power of two with n | p-1: 1 <= n <= 2^23 for 998244353 (its 2-adicity), 2^24 for
 *          469762049, 167772161, Goldilocks and Z/(2^31-1)[sqrt 3] (2^12..2^13-point sub-problems x 2^11 column levels)
 *   batch  number of independent instances, >= 1 (all share p, f, n)
 *   stream cudaStream_t
 * Errors: FCIRC_EINVAL, FCIRC_EPRIME, FCIRC_ESIZE, FCIRC_ENOROOT, FCIRC_ENOMEM, FCIRC_ECUDA.
 */
int fcirc_matvec(uint64_t p, uint64_t f, const void* a, const void* b, void* c,
                 int64_t n, int64_t batch, void* stream);

/*
 * fcirc_circulant_matvec — c = A b for a batch of usual circulant matrices (f = 1) of
 * ANY order n >= 1 (Corollary 1).  A is identified by its first row a:
 *     c_i = sum_j a[(j - i) mod n] b_j   (mod p).
 * n a power of two: exactly fcirc_matvec with f = 1.  Otherwise the Corollary's embedding: the
 * order-N circulant with row a' = (a_0..a_{n-1}, 0..0, a_1..a_{n-1}) times b' = (b, 0..0), whose
 * first n entries are A b; N = the smallest power of two >= 2n - 1 (the paper's N = 2^{d+1} with
 * 2^d > n also works, at up to twice the size; reading R10).  The embedding is fused into
 * the first pass's loads and the truncation into the last pass's stores.
 *   p, a, b, c, batch, stream as fcirc_matvec; a, b, c are [batch][n]; N must divide p-1 and be
 *   within the fcirc_matvec maximum.
 * Errors: FCIRC_EINVAL, FCIRC_EPRIME, FCIRC_ESIZE, FCIRC_ENOMEM, FCIRC_ECUDA.
 */
int fcirc_circulant_matvec(uint64_t p, const void* a, const void* b, void* c, int64_t n, int64_t batch,
                           void* stream);

/*
 * fcirc_matvec_host — fcirc_matvec on HOST buffers: copies a, b to the device, runs the product
 * and copies c back, pipelined in chunks of instances over two streams so the PCIe transfers in
 * both directions overlap the kernels.  Synchronous: returns when c is written.  Same arguments
 * and errors as fcirc_matvec (a, b, c are host pointers; page-locked memory recommended).
 */
int fcirc_matvec_host(uint64_t p, uint64_t f, const void* a, const void* b, void* c,
                      int64_t n, int64_t batch);

/*
 * fcirc_polymul — c = a(x) * b(x) mod p for a batch of polynomial pairs ("The
 * multiplication of two polynomials forms a circulant matrix-vector product in a natural way").
 * Coefficients are low order first.  The product is computed as an f = 1 circulant matvec of
 * order L = the smallest power of two >= na + nb - 1 (the paper's "N = (d_a+1)(d_b+1)-1" read as
 * (d_a+1)+(d_b+1)-1, reading R8) on the zero-padded, index-reversed row
 * (a~[0] = a[0], a~[L-m] = a[m]), so that the circulant product is the cyclic convolution.
 *   p          registry modulus (32-bit primes and Goldilocks)
 *   a          [batch][na] (device), b [batch][nb] (device)
 *   c          [batch][na+nb-1] (device), must not overlap a or b
 *   na, nb     >= 1, with L | p-1 and L within the fcirc_matvec maximum
 * Errors as fcirc_matvec.
 */
int fcirc_polymul(uint64_t p, const void* a, int64_t na, const void* b, int64_t nb, void* c,
                  int64_t batch, void* stream);

/*
 * bigint_mul — z = x * y for a batch of non-negative integers (the circulant product
 * replaces the three transforms of Schoenhage-Strassen).  Operands are little-endian arrays of
 * 32-bit words.  Route: 16-bit limbs -> three f = 1 circulant products mod 998244353, 469762049
 * and 167772161 (order L = smallest power of two >= 2*(nx+ny) - 1 limbs) -> Garner CRT per
 * coefficient -> carry propagation (reading R12 replaces the paper's Fermat ring).
 *   x  [batch][nx] words (device), y [batch][ny] words (device)
 *   z  [batch][nx+ny] words (device), must not overlap x or y
 *   nx, ny >= 1 with 2*(nx+ny) limbs <= 2^23
 * Errors: FCIRC_EINVAL, FCIRC_ESIZE, FCIRC_ENOMEM, FCIRC_ECUDA.
 */
int bigint_mul(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z,
               int64_t batch, void* stream);

/* human-readable text for a status code (static storage) */
const char* fcirc_strerror(int status);

/* library version string, e.g. "libfcirc 0.1 sm_100a" */
const char* fcirc_version(void);

/*
 * fcirc_schedule — HOST-only: the pass schedule fcirc_matvec uses for (p, n).
 * *sub_log = log2 of the on-chip sub-problem size, *top_levels = number of recursion levels done by
 * the column passes before / after the sub-problems (0: one fused pass over the whole product).
 * Used by bench.py to attribute algorithmic work to kernels.
 * Errors: FCIRC_EINVAL (null output, n not a power of two), FCIRC_EPRIME, FCIRC_ESIZE.
 */
int fcirc_schedule(uint64_t p, int64_t n, int* sub_log, int* top_levels);

/*
 * fcirc_last_launch_count — number of kernels the calling host thread launched in its most
 * recent successful libfcirc call (for the benchmark's gpu_launches count).
 */
int64_t fcirc_last_launch_count(void);

/*
 * fcirc_plan_table — HOST-only inspection of the twist table a plan would use (no GPU needed).
 * Writes, for n = 2^L >= 2: s[2^d + e] = s_{d,e} and sinv[2^d + e] = s_{d,e}^-1 for d < L,
 * e < 2^d (entry 0 is 0), the chosen n-th root w of f (w^n = f), and the final scale K
 * (n^-1, times 2^32 mod p for the 32-bit primes).  s and sinv hold n entries each (1 for n = 1).
 * Errors: FCIRC_EINVAL, FCIRC_EPRIME, FCIRC_ESIZE, FCIRC_ENOROOT.
 */
int fcirc_plan_table(uint64_t p, uint64_t f, int64_t n, uint64_t* s, uint64_t* sinv, uint64_t* w, uint64_t* K);

/*
 * Kernel-level timing (for bench.py's roofline): while enabled, every kernel launch libfcirc makes
 * is bracketed by two CUDA events recorded on the launching stream.  fcirc_profile_read waits for
 * the recorded events, writes per-kind launch counts and summed device milliseconds for up to
 * `nkinds` kinds, clears the record and returns the number of kinds (FCIRC_NKINDS).
 * Kinds: 0 k_block fused (whole problem), 1 k_block sub-problems (multi-pass), 2 k_cols forward,
 * 3 k_cols inverse, 4 application kernels (embed/truncate/CRT/carry).
 */
#define FCIRC_NKINDS 5
int fcirc_profile_enable(int on);
int fcirc_profile_read(int64_t* counts, double* ms, int nkinds);

/*
 * fcirc_primitive_rate — measured integer throughput of the product's OWN ring primitives (the
 * FieldGold / FieldU32 functions the kernels inline), for the roofline's integer peak (SURVEY
 * §8(d): R_const, R_var measured in a register-resident all-SM microbenchmark).
 * One warm-up and one timed launch on `stream` (CUDA events; synchronises the stream): every SM at
 * full occupancy, 8 independent dependency chains per thread, `iters` iterations per chain.
 *   kind  FCIRC_PRIM_*:
 *           GOLD_MUL    Goldilocks 64x64 -> canonical modmul by the special reduction (2^64 = 2^32 - 1)
 *           GOLD_LEAF   Goldilocks var x var modmul of the leaves (canonicalise one factor, then Montgomery)
 *           GOLD_MULM   Goldilocks const x var modmul (Montgomery form, R = 2^64: every twiddle product)
 *           GOLD_FWD_A / GOLD_FWD_B / GOLD_INV  the three Goldilocks butterflies (1 modmul each)
 *           U32_MULC    Shoup const x var modmul (p = 998244353)
 *           U32_LEAF    Montgomery var x var modmul
 *           U32_FWD_A   the 32-bit row butterfly (1 modmul)
 *           IMAD_WIDE   raw 32x32+64 -> 64 multiply-adds (the multiplier-only ceiling: a Goldilocks
 *                       modmul needs >= 4, a Shoup modmul the issue slots of 2)
 *           M31X2_MUL   product in the paper's ring Z/(2^31-1)[sqrt 3]
 *   *ops_per_s  primitives per second;  *ms  the timed launch (may be NULL)
 * Errors: FCIRC_EINVAL (unknown kind, iters < 1, null ops_per_s), FCIRC_ENOMEM, FCIRC_ECUDA.
 */
#define FCIRC_PRIM_GOLD_MUL 0
#define FCIRC_PRIM_GOLD_FWD_A 1
#define FCIRC_PRIM_GOLD_FWD_B 2
#define FCIRC_PRIM_GOLD_INV 3
#define FCIRC_PRIM_U32_MULC 4
#define FCIRC_PRIM_U32_LEAF 5
#define FCIRC_PRIM_U32_FWD_A 6
#define FCIRC_PRIM_IMAD_WIDE 7
#define FCIRC_PRIM_M31X2_MUL 8
#define FCIRC_PRIM_GOLD_MULM 9
#define FCIRC_PRIM_GOLD_LEAF 10
int fcirc_primitive_rate(int kind, int64_t iters, double* ops_per_s, double* ms, void* stream);

/* release all cached plans and trim the current device's default memory pool (tests / teardown) */
int fcirc_release_cache(void);

/* number of cached plans (all devices); *pinned (may be NULL) = how many are pinned by graph captures */
int64_t fcirc_plan_count(int* pinned);

#ifdef __cplusplus
}
#endif

#endif /* FCIRC_H */

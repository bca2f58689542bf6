// numtheory.h -- host-side number theory and per-(p, rep) constants (build layer L0).
//
// Everything here runs once per (p, rep, dtype) on the host; nothing is timed.  The oracle
// (oracle/oracle.c) has its own independent implementations; the two share no code.
#pragma once
#include <cstdint>
#include <vector>

#include "gfp.h"

namespace gfp {

using u128 = unsigned __int128;

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m);
uint64_t powmod(uint64_t a, uint64_t e, uint64_t m);
// Deterministic Miller-Rabin for all n < 2^64 (bases 2..37).
bool is_prime(uint64_t n);
// Inverse of a modulo m by the extended Euclidean algorithm (sec. 2.1). false if none.
bool inv_mod(uint64_t a, uint64_t m, uint64_t *out);
// Prime factors (with multiplicity) by trial division; n < 2^64, used for n = p-1 < 2^32.
std::vector<uint64_t> factorize(uint64_t n);
// Smallest primitive root of prime p (sec. 2.4; reading G12).  p = 2 -> 1.
uint64_t primitive_root(uint64_t p);
// -p^{-1} mod 2^32 for odd p, by Newton-Hensel lifting (sec. 2.2: n_im).
uint32_t neg_inv_mod_2_32(uint32_t p);

// Largest admissible p per (rep, dtype) -- the paper's printed bounds (see gfp.h).
uint64_t rep_bound(gfp_rep rep, gfp_dtype dt);
// The defining predicate of that bound, evaluated exactly (tests check both agree).
bool rep_predicate(gfp_rep rep, gfp_dtype dt, uint64_t p);

// Eq. (1) with a carried residue (reading G7): largest k with k(p-1)^2 + (p-1) <= 2^m - 1.
uint64_t block_k(uint64_t p, int m);
// Centered representation (sec. 3.2.2): largest k with k h^2 + h <= 2^63 - 1 (m = 64, a signed
// 64-bit accumulator: "lambda_centered ((p-1)/2)^2 < 2^(m-1)") or < 2^53 (m = 53, binary64), h = (p-1)/2.
uint64_t centered_k(uint64_t p, int m);
// Montgomery products per REDC (reading G6): largest k with k(p-1)^2 <= pB (REDC precondition,
// P:73) and k(p-1)^2 + (B-1)p <= 2^64 - 1 (T + Up fits the 64-bit word), B = 2^32.
uint64_t mont_k(uint64_t p);

// Discrete-log tables (sec. 2.4).  log_table[x] = code of x (size p; log[0] = 0, log[1] = q-1).
// antilog: "small" layout (p <= 32768): 65536 entries, [s] = g^s for s in [0, 2(q-1)], [65535] = 0
// (zero sentinel); "large" layout: p entries, [0] = 0 (sentinel), [t] = g^t for t in [1, q-1].
bool zech_small_layout(uint64_t p);
void zech_tables(uint64_t p, uint64_t g, std::vector<uint16_t> &log_table,
                 std::vector<uint16_t> &antilog);

// Pure-Zech addition table (sec. 2.4, the t_plus1 table in exponent form):
// delta[k] = the exponent d in [0, qbar) with g^d = 1 + g^k, for k in [0, qbar]; kZechDeltaZero when
// 1 + g^k = 0 (k = qbar/2).  delta[qbar] = delta[0]; delta[qbar + 1] = 0 (the entry a zero product is
// steered to: adding delta 0 leaves the sum unchanged).  Built from log_table (zech_tables).
constexpr uint16_t kZechDeltaZero = 0xFFFF;
void zech_plus1_delta(uint64_t p, const std::vector<uint16_t> &log_table, std::vector<uint16_t> &delta);

// Fill a gfp_info for a validated (p, rep, dtype).
gfp_status describe(uint64_t p, gfp_rep rep, gfp_dtype dt, gfp_info *info);

}  // namespace gfp

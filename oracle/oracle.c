/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of what the GPU hot
 * path computes: the exact dot product of two vectors over GF(p), in each of
 * the four representations of arXiv cs/0404008 section 2, with every term
 * reduced by a 128-bit Euclidean remainder (SURVEY.md 8(c) "Oracle algorithm").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this file's library.  It shares no code, header, table or
 * constant generator with paper_cs_0404008_b200/ (the product), and the
 * product never calls it.
 *
 * Citations: P:n = line n of the paper text, with its section.
 *
 * Definition: with inputs decoded to canonical residues,
 *     r = (sum_{i<n} a_i * b_i) mod p,  r in [0, p),
 * encoded back into the input representation.  The method of the paper
 * reaches this value exactly (sec. 3.1: "A single machine
 * remaindering is needed at the end"), so the oracle is that definition
 * written out -- one remainder per term, no delay, no blocking.
 *
 * Parity status of every function is pinned by tests/test_oracle_pins.py
 * (paper constants, closed forms, brute force with Python integers).
 */
#include <stdint.h>
#include <stddef.h>

typedef unsigned __int128 u128;

enum { O_U16 = 0, O_U32 = 1, O_U64 = 2 };

static uint64_t load(const void *v, int dt, int64_t i)
{
    switch (dt) {
    case O_U16: return ((const uint16_t *)v)[i];
    case O_U32: return ((const uint32_t *)v)[i];
    default:    return ((const uint64_t *)v)[i];
    }
}

/* ---------------------------------------------------------------- numbers */

/* Primality by trial division (obviously correct; n < 2^64, used for n < 2^34). */
int oracle_is_prime(uint64_t n)
{
    if (n < 2) return 0;
    if (n < 4) return 1;
    if (n % 2 == 0) return 0;
    for (uint64_t d = 3; d <= n / d; d += 2)
        if (n % d == 0) return 0;
    return 1;
}

/* a^e mod m by square-and-multiply with 128-bit products. */
uint64_t oracle_pow(uint64_t a, uint64_t e, uint64_t m)
{
    uint64_t r = 1 % m, x = a % m;
    while (e) {
        if (e & 1) r = (uint64_t)(((u128)r * x) % m);
        x = (uint64_t)(((u128)x * x) % m);
        e >>= 1;
    }
    return r;
}

/* Inverse mod a prime p by Fermat's little theorem: a^(p-2).  0 if a = 0 mod p. */
uint64_t oracle_inv(uint64_t a, uint64_t p)
{
    if (a % p == 0) return 0;
    return oracle_pow(a, p - 2, p);
}

/* Multiplicative order of g mod p by brute-force iteration (p < 2^32). */
uint64_t oracle_order(uint64_t g, uint64_t p)
{
    uint64_t x = g % p, k = 1;
    if (x == 0) return 0;
    while (x != 1) {
        x = (uint64_t)(((u128)x * g) % p);
        ++k;
    }
    return k;
}

/* Smallest primitive element of GF(p) by brute-force orders (sec. 2.4, P:122-125;
 * reading G12: the smallest one).  p = 2 -> 1.  Returns 0 if p is not prime. */
uint64_t oracle_primitive_root(uint64_t p)
{
    if (!oracle_is_prime(p)) return 0;
    if (p == 2) return 1;
    for (uint64_t g = 2; g < p; ++g)
        if (oracle_order(g, p) == p - 1) return g;
    return 0;
}

/* ------------------------------------------------------ classical (sec 2.1) */

/* (sum a_i b_i) mod p, one 128-bit remainder per term (reading: "%"
 * scale of sec. 2.5).  dt: 0 = u16, 1 = u32, 2 = u64. */
uint64_t oracle_dot_classical(uint64_t p, const void *a, const void *b, int dt, int64_t n)
{
    uint64_t acc = 0;
    for (int64_t i = 0; i < n; ++i)
        acc = (uint64_t)(((u128)acc + (u128)load(a, dt, i) * load(b, dt, i)) % p);
    return acc;
}

/* One residue per row: out[r] = (sum_j A[r*lda + j] * x[j]) mod p. */
void oracle_dot_batch_classical(uint64_t p, const void *A, int64_t lda, const void *x, int dt,
                                int64_t rows, int64_t n, uint64_t *out)
{
    for (int64_t r = 0; r < rows; ++r) {
        uint64_t acc = 0;
        for (int64_t j = 0; j < n; ++j)
            acc = (uint64_t)(((u128)acc + (u128)load(A, dt, r * lda + j) * load(x, dt, j)) % p);
        out[r] = acc;
    }
}

/* ----------------------------------------------------- Montgomery (sec 2.2) */
/* Element a is stored as a*B mod p with B = 2^32 (reading G15). */

uint64_t oracle_to_mont(uint64_t p, uint64_t a)
{
    return (uint64_t)((((u128)(a % p)) << 32) % p);
}

/* decode x = a*B mod p  ->  a = x * B^{-1} mod p, with B^{-1} by Fermat (no REDC). */
uint64_t oracle_from_mont(uint64_t p, uint64_t x)
{
    uint64_t binv = oracle_inv((uint64_t)(((u128)1 << 32) % p), p);
    return (uint64_t)(((u128)(x % p) * binv) % p);
}

/* Dot of Montgomery-form vectors; result in Montgomery form (reading G10). */
uint64_t oracle_dot_montgomery(uint64_t p, const uint32_t *a, const uint32_t *b, int64_t n)
{
    uint64_t binv = oracle_inv((uint64_t)(((u128)1 << 32) % p), p);
    uint64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t ai = (uint64_t)(((u128)a[i] * binv) % p);
        uint64_t bi = (uint64_t)(((u128)b[i] * binv) % p);
        acc = (uint64_t)(((u128)acc + (u128)ai * bi) % p);
    }
    return oracle_to_mont(p, acc);
}

/* -------------------------------------------------- floating point (sec 2.3) */
/* Elements are exact integers in [0, p) held in binary64. */

/* Decode; returns the index of the first element that is not an integer in
 * [0, p) (caller treats it as a precondition violation), or -1. */
int64_t oracle_f64_decode(uint64_t p, const double *x, int64_t n, uint64_t *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double v = x[i];
        if (!(v >= 0.0) || v >= (double)p || v != (double)(uint64_t)v) return i;
        out[i] = (uint64_t)v;
    }
    return -1;
}

/* Dot of fp64-representation vectors; *bad = first invalid index or -1. */
double oracle_dot_fp64(uint64_t p, const double *a, const double *b, int64_t n, int64_t *bad)
{
    uint64_t acc = 0;
    *bad = -1;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t ai, bi;
        if (oracle_f64_decode(p, a + i, 1, &ai) >= 0 || oracle_f64_decode(p, b + i, 1, &bi) >= 0) {
            *bad = i;
            return -1.0;
        }
        acc = (uint64_t)(((u128)acc + (u128)ai * bi) % p);
    }
    return (double)acc;
}

/* ---------------------------------------------- discrete logarithms (sec 2.4) */
/* Encoding:  x = 0 -> 0;  x = 1 -> q-1;  x = g^i (1 <= i < q-1) -> i.
 * Prime fields only: q = p, qbar = q - 1. */

/* pw[c] = g^c mod p for c = 0 .. p-1, by repeated multiplication. */
void oracle_zech_powers(uint64_t p, uint64_t g, uint64_t *pw)
{
    uint64_t x = 1 % p;
    for (uint64_t c = 0; c < p; ++c) {
        pw[c] = x;
        x = (uint64_t)(((u128)x * g) % p);
    }
}

/* code -> element, following the three cases of P:128-130 literally.
 * Returns -1 for a code outside [0, q-1]. */
int64_t oracle_zech_decode_one(uint64_t p, uint64_t g, uint64_t code)
{
    uint64_t q = p;
    if (code == 0) return 0;
    if (code == q - 1) return 1;
    if (code < q - 1) return (int64_t)oracle_pow(g, code, p);
    return -1;
}

/* element -> code by brute-force discrete log (independent of any table). */
uint64_t oracle_zech_encode_one(uint64_t p, uint64_t g, uint64_t x)
{
    uint64_t q = p;
    x %= p;
    if (x == 0) return 0;
    if (x == 1) return q - 1;
    uint64_t y = g % p;
    for (uint64_t i = 1; i < q - 1; ++i) {
        if (y == x) return i;
        y = (uint64_t)(((u128)y * g) % p);
    }
    return UINT64_MAX; /* unreachable when g is primitive */
}

/* Dot of Zech-coded vectors (reading G11: decode, multiply, add, reduce every
 * term, encode).  The power list is the oracle's own (oracle_zech_powers);
 * tiny cases in the tests decode with oracle_zech_decode_one instead.
 * pw must hold p entries.  *bad = first invalid code index or -1. */
uint64_t oracle_dot_zech(uint64_t p, uint64_t g, const uint16_t *a, const uint16_t *b, int64_t n,
                         uint64_t *pw, int64_t *bad)
{
    uint64_t q = p, acc = 0;
    *bad = -1;
    oracle_zech_powers(p, g, pw);
    for (int64_t i = 0; i < n; ++i) {
        uint64_t ca = a[i], cb = b[i];
        if (ca > q - 1 || cb > q - 1) {
            *bad = i;
            return UINT64_MAX;
        }
        /* code 0 is the zero element; code c in [1, q-1] is g^c (g^(q-1) = 1). */
        uint64_t ai = ca == 0 ? 0 : pw[ca];
        uint64_t bi = cb == 0 ? 0 : pw[cb];
        acc = (uint64_t)(((u128)acc + (u128)ai * bi) % p);
    }
    return oracle_zech_encode_one(p, g, acc);
}

/* ----------------------------- Zech arithmetic of Table 1 (sec 2.4, F3) */
/* The paper's own addition of discrete-log codes (Table 1),
 * written out step by step in the table's order and notation.  Codes follow
 * P:126-131 (0 -> 0, 1 -> qbar = q-1, g^i -> i); all of [1, qbar] are the
 * nonzero codes, code qbar standing for g^0 = 1.  These functions give the
 * same unique field element as oracle_dot_zech (the sum is unique); they
 * exist so the pure-Zech accumulation has its algorithm in the oracle too. */

/* t_plus1[k] for k = 0 .. q-1 (a table "of size q"): the code h of
 * 1 + g^k, i.e. g^h = 1 + g^k, with h = 0 when 1 + g^k = 0 (k = (q-1)/2,
 * g^((q-1)/2) = -1).  t[q-1] = t[0] since g^(q-1) = g^0.  The log
 * map is built by enumerating the powers g^c (no table shared with anything).
 * lg must hold p entries of scratch. */
void oracle_zech_tplus1(uint64_t p, uint64_t g, uint64_t *t, uint64_t *lg)
{
    uint64_t q = p, qbar = q - 1, x = 1 % p;
    for (uint64_t c = 0; c < p; ++c) lg[c] = 0;
    /* lg[g^c] = c for c = 1 .. qbar-1; lg[1] = qbar; lg[0] = 0 */
    for (uint64_t c = 1; c < qbar; ++c) {
        x = (uint64_t)(((u128)x * g) % p);
        lg[x] = c;
    }
    lg[1 % p] = qbar;
    lg[0] = 0;
    x = 1 % p; /* g^k */
    for (uint64_t k = 0; k < qbar; ++k) {
        t[k] = lg[(x + 1) % p];
        x = (uint64_t)(((u128)x * g) % p);
    }
    t[qbar] = t[0];
}

/* Table 1 row "Multiplication": g^i * g^j -> i + j (- qbar).  Zero operands
 * (code 0) give zero (reading G13). */
uint64_t oracle_zech_mul(uint64_t p, uint64_t i, uint64_t j)
{
    uint64_t qbar = p - 1;
    if (i == 0 || j == 0) return 0;
    uint64_t s = i + j;
    if (s > qbar) s -= qbar; /* the "(- qbar)" test */
    return s;
}

/* Table 1 row "Addition": g^i + g^j -> k = j - i (+ qbar); i + t_plus1[k] (- qbar).
 * A zero operand returns the other one; t_plus1[k] = 0 (1 + g^k = 0) gives zero. */
uint64_t oracle_zech_add(uint64_t p, const uint64_t *t, uint64_t i, uint64_t j)
{
    int64_t qbar = (int64_t)p - 1;
    if (i == 0) return j;
    if (j == 0) return i;
    int64_t k = (int64_t)j - (int64_t)i;
    if (k < 0) k += qbar; /* the "(+ qbar)" test */
    uint64_t h = t[k];
    if (h == 0) return 0; /* g^i (1 + g^k) = 0 */
    uint64_t r = i + h;
    if (r > (uint64_t)qbar) r -= (uint64_t)qbar; /* the "(- qbar)" test */
    return r;
}

/* Pure-Zech dot (reading G11's alternative): every product and
 * every partial sum stays a Zech code; acc starts at the zero code and absorbs
 * one Table-1 product per term with one Table-1 addition.  t, lg: scratch of p
 * entries each.  *bad = first invalid code index or -1. */
uint64_t oracle_dot_zech_tplus1(uint64_t p, uint64_t g, const uint16_t *a, const uint16_t *b, int64_t n,
                                uint64_t *t, uint64_t *lg, int64_t *bad)
{
    uint64_t q = p, acc = 0;
    *bad = -1;
    oracle_zech_tplus1(p, g, t, lg);
    for (int64_t i = 0; i < n; ++i) {
        if (a[i] > q - 1 || b[i] > q - 1) {
            *bad = i;
            return UINT64_MAX;
        }
        acc = oracle_zech_add(p, t, acc, oracle_zech_mul(p, a[i], b[i]));
    }
    return acc;
}

/* ------------------------------------- centered representation (sec 3.2.2) */
/* Elements stored between -(p-1)/2 and (p-1)/2, p odd; storage
 * int16, int32 (two's complement) or binary64 holding the integer.  The dot is
 * the same field element; the result is returned centered (reading G10). */

static int64_t load_signed(const void *v, int dt, int64_t i)
{
    switch (dt) {
    case O_U16: return ((const int16_t *)v)[i];
    case O_U32: return ((const int32_t *)v)[i];
    default:    return ((const int64_t *)v)[i];
    }
}

/* centered value c -> residue in [0, p) */
uint64_t oracle_from_centered(uint64_t p, int64_t c)
{
    int64_t r = c % (int64_t)p; /* C99: sign of the dividend */
    return (uint64_t)(r < 0 ? r + (int64_t)p : r);
}

/* residue r in [0, p) -> centered value in [-(p-1)/2, (p-1)/2] */
int64_t oracle_to_centered(uint64_t p, uint64_t r)
{
    r %= p;
    return r > (p - 1) / 2 ? (int64_t)r - (int64_t)p : (int64_t)r;
}

/* Dot of centered vectors; dt: 0 = int16, 1 = int32, 2 = int64.  *bad = first
 * element outside [-(p-1)/2, (p-1)/2], or -1.  One 128-bit remainder per term. */
int64_t oracle_dot_centered(uint64_t p, const void *a, const void *b, int dt, int64_t n, int64_t *bad)
{
    const int64_t h = (int64_t)((p - 1) / 2);
    uint64_t acc = 0;
    *bad = -1;
    for (int64_t i = 0; i < n; ++i) {
        int64_t x = load_signed(a, dt, i), y = load_signed(b, dt, i);
        if (x < -h || x > h || y < -h || y > h) {
            *bad = i;
            return 0;
        }
        acc = (uint64_t)(((u128)acc + (u128)oracle_from_centered(p, x) * oracle_from_centered(p, y)) % p);
    }
    return oracle_to_centered(p, acc);
}

/* binary64 storage: check each value is an integer in the centered range, then as above. */
double oracle_dot_centered_f64(uint64_t p, const double *a, const double *b, int64_t n, int64_t *bad)
{
    const double h = (double)((p - 1) / 2);
    uint64_t acc = 0;
    *bad = -1;
    for (int64_t i = 0; i < n; ++i) {
        double x = a[i], y = b[i];
        if (!(x >= -h && x <= h && y >= -h && y <= h) || x != (double)(int64_t)x || y != (double)(int64_t)y) {
            *bad = i;
            return 0.0;
        }
        acc = (uint64_t)(((u128)acc + (u128)oracle_from_centered(p, (int64_t)x) *
                                          oracle_from_centered(p, (int64_t)y)) % p);
    }
    return (double)oracle_to_centered(p, acc) + 0.0; /* + 0.0: never -0.0 */
}

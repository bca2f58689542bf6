// numtheory.cpp -- host number theory and per-(p, rep) constants.  See numtheory.h.
#include "numtheory.h"

#include <cmath>

namespace gfp {

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }

uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mulmod(r, a, m);
        a = mulmod(a, a, m);
        e >>= 1;
    }
    return r;
}

bool is_prime(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t q : small) {
        if (n == q) return true;
        if (n % q == 0) return false;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (uint64_t a : small) {  // deterministic for n < 3.3e24
        uint64_t x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int r = 1; r < s; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) {
                composite = false;
                break;
            }
        }
        if (composite) return false;
    }
    return true;
}

bool inv_mod(uint64_t a, uint64_t m, uint64_t *out) {
    // extended Euclid on signed 128-bit cofactors
    __int128 r0 = m, r1 = a % m, t0 = 0, t1 = 1;
    while (r1 != 0) {
        __int128 q = r0 / r1, tmp;
        tmp = r0 - q * r1; r0 = r1; r1 = tmp;
        tmp = t0 - q * t1; t0 = t1; t1 = tmp;
    }
    if (r0 != 1) return false;
    if (t0 < 0) t0 += m;
    *out = (uint64_t)t0;
    return true;
}

std::vector<uint64_t> factorize(uint64_t n) {
    std::vector<uint64_t> f;
    for (uint64_t d = 2; d <= n / d; d += (d == 2 ? 1 : 2))
        while (n % d == 0) {
            f.push_back(d);
            n /= d;
        }
    if (n > 1) f.push_back(n);
    return f;
}

uint64_t primitive_root(uint64_t p) {
    if (p == 2) return 1;
    std::vector<uint64_t> fs = factorize(p - 1);
    for (uint64_t g = 2; g < p; ++g) {
        bool ok = true;
        uint64_t last = 0;
        for (uint64_t r : fs) {
            if (r == last) continue;
            last = r;
            if (powmod(g, (p - 1) / r, p) == 1) {
                ok = false;
                break;
            }
        }
        if (ok) return g;
    }
    return 0;
}

uint32_t neg_inv_mod_2_32(uint32_t p) {
    uint32_t x = p;                           // p*p = 1 mod 8 for odd p: 3 correct bits
    for (int i = 0; i < 5; ++i) x *= 2u - p * x;  // each step doubles the correct bits
    return (uint32_t)(0u - x);
}

uint64_t rep_bound(gfp_rep rep, gfp_dtype dt) {
    switch (rep) {
    case GFP_REP_CLASSICAL:
        return dt == GFP_U16 ? 65521ull : (dt == GFP_U32 ? 4294967291ull : 0);
    case GFP_REP_MONTGOMERY:
        return dt == GFP_U32 ? 2654435761ull : 0;
    case GFP_REP_FP64:
        return dt == GFP_F64 ? 94906249ull : 0;                                // p(p-1) < 2^53
    case GFP_REP_ZECH:
        return dt == GFP_U16 ? 65521ull : 0;                                   // u16 codes
    case GFP_REP_CENTERED:                                                     // sec. 3.2.2
        return dt == GFP_U16 ? 65521ull : (dt == GFP_U32 ? 4294967291ull : 189812507ull);
    }
    return 0;
}

bool rep_predicate(gfp_rep rep, gfp_dtype dt, uint64_t p) {
    if (p < 2) return false;
    const u128 P = p;
    switch (rep) {
    case GFP_REP_CLASSICAL:
        // unsigned AXPY a*x+y <= p(p-1) fits the word
        if (dt == GFP_U16) return p < (1ull << 16) && P * (P - 1) < ((u128)1 << 32);
        if (dt == GFP_U32) return p < (1ull << 32) && P * (P - 1) < ((u128)1 << 64);
        return false;
    case GFP_REP_MONTGOMERY: {
        if (dt != GFP_U32 || (p & 1) == 0) return false;
        const u128 B = (u128)1 << 32;
        return (P - 1) * (P - 1) + P * (B - 1) < B * B;
    }
    case GFP_REP_FP64:
        return dt == GFP_F64 && P * (P - 1) < ((u128)1 << 53);
    case GFP_REP_ZECH:
        return dt == GFP_U16 && p - 1 <= 0xFFFFull;
    case GFP_REP_CENTERED: {
        // odd p (no symmetric range at p = 2); h = (p-1)/2 fits the signed storage; binary64:
        // one product plus a carried residue stays exact, h^2 + h < 2^53
        if ((p & 1) == 0) return false;
        const u128 h = (P - 1) / 2;
        if (dt == GFP_U16) return h <= 32767;
        if (dt == GFP_U32) return h <= 0x7FFFFFFFull;
        return h * h + h < ((u128)1 << 53);
    }
    }
    return false;
}

uint64_t centered_k(uint64_t p, int m) {
    const u128 h = (u128)(p - 1) / 2, q = h * h;
    const u128 w = m == 53 ? ((u128)1 << 53) - 1 : ((u128)1 << 63) - 1;  // |T| <= 2^53 - 1 / 2^63 - 1
    if (q == 0) return UINT64_MAX;
    if (w < h) return 0;
    u128 k = (w - h) / q;
    return k > UINT64_MAX ? UINT64_MAX : (uint64_t)k;
}

uint64_t block_k(uint64_t p, int m) {
    const u128 w = m >= 64 ? ~(u128)0 >> 64 : (((u128)1 << m) - 1);  // 2^m - 1
    const u128 q = (u128)(p - 1) * (p - 1);
    if (q == 0) return UINT64_MAX;
    if (w < (p - 1)) return 0;
    u128 k = (w - (p - 1)) / q;
    return k > UINT64_MAX ? UINT64_MAX : (uint64_t)k;
}

uint64_t mont_k(uint64_t p) {
    const u128 B = (u128)1 << 32, q = (u128)(p - 1) * (p - 1);
    if (q == 0) return UINT64_MAX;
    u128 k1 = (u128)p * B / q;
    const u128 w = ~(u128)0 >> 64, up = (B - 1) * p;
    u128 k2 = w >= up ? (w - up) / q : 0;
    u128 k = k1 < k2 ? k1 : k2;
    return k > UINT64_MAX ? UINT64_MAX : (uint64_t)k;
}

bool zech_small_layout(uint64_t p) { return 2 * (p - 1) <= 0xFFFEull; }

void zech_tables(uint64_t p, uint64_t g, std::vector<uint16_t> &log_table, std::vector<uint16_t> &antilog) {
    const uint64_t qbar = p - 1;
    log_table.assign(p, 0);
    // log: 0 -> 0, 1 -> q-1, g^i -> i
    uint64_t x = 1;
    for (uint64_t i = 0; i < qbar; ++i) {
        log_table[x] = (uint16_t)(i == 0 ? qbar : i);
        x = x * g % p;
    }
    if (zech_small_layout(p)) {
        antilog.assign(65536, 0);
        x = 1;
        for (uint64_t s = 0; s <= 2 * qbar; ++s) {
            antilog[s] = (uint16_t)x;
            x = x * g % p;
        }
        antilog[65535] = 0;  // zero sentinel: a zero operand maps its index here
    } else {
        antilog.assign(p, 0);
        x = g % p;
        for (uint64_t t = 1; t <= qbar; ++t) {
            antilog[t] = (uint16_t)x;
            x = x * g % p;
        }
        antilog[0] = 0;  // zero sentinel
    }
}

void zech_plus1_delta(uint64_t p, const std::vector<uint16_t> &log_table, std::vector<uint16_t> &delta) {
    const uint64_t qbar = p - 1;
    delta.assign(qbar + 2, 0);
    std::vector<uint64_t> pw(qbar + 1);  // exponent -> element g^k, inverted from the log table
    for (uint64_t x = 1; x < p; ++x) pw[log_table[x] % qbar] = x;
    for (uint64_t k = 0; k < qbar; ++k) {
        const uint64_t one_plus = (1 + pw[k]) % p;
        delta[k] = one_plus == 0 ? kZechDeltaZero : (uint16_t)(log_table[one_plus] % qbar);
    }
    delta[qbar] = delta[0];  // index qbar aliases 0 (g^qbar = g^0)
    delta[qbar + 1] = 0;     // "add nothing": the index a zero product is steered to (s + 0 = s)
}

gfp_status describe(uint64_t p, gfp_rep rep, gfp_dtype dt, gfp_info *info) {
    if ((int)rep < 0 || (int)rep > 4 || (int)dt < 0 || (int)dt > 2) return GFP_E_INVAL;
    const uint64_t bound = rep_bound(rep, dt);
    if (bound == 0) return GFP_E_UNSUPPORTED;
    if (!is_prime(p)) return GFP_E_NOT_PRIME;
    if (p > bound || !rep_predicate(rep, dt, p)) return GFP_E_BOUND;
    gfp_info I = {};
    I.p = p;
    I.rep = rep;
    I.dtype = dt;
    I.bound = bound;
    I.acc_bits = (rep == GFP_REP_FP64 || (rep == GFP_REP_CENTERED && dt == GFP_F64)) ? 53 : 64;
    I.k = rep == GFP_REP_CENTERED ? centered_k(p, I.acc_bits) : block_k(p, I.acc_bits);
    I.corr = (uint64_t)((((u128)1) << 64) % p);
    I.b_mod_p = (uint64_t)((((u128)1) << 32) % p);
    I.inv_p = 1.0 / (double)p;  // IEEE round-to-nearest division (reading G8)
    if (rep == GFP_REP_MONTGOMERY) {
        I.n_im = neg_inv_mod_2_32((uint32_t)p);
        I.r2 = (uint64_t)((((u128)1) << 64) % p);
        uint64_t kr = mont_k(p);
        I.mont_kr = (int32_t)(kr > 1000000 ? 1000000 : kr);
    }
    if (rep == GFP_REP_ZECH) {
        I.g = primitive_root(p);
        I.qbar = p - 1;
        I.table_bytes = zech_small_layout(p) ? 65536 * 2 : p * 2;
    }
    *info = I;
    return GFP_OK;
}

}  // namespace gfp

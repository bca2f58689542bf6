/*
 * oracle_san_driver.c -- TEST INFRASTRUCTURE: runs the CPU oracle (oracle/oracle.c, compiled into this driver)
 * under -fsanitize=undefined,address ("Run the oracle under -fsanitize=undefined,address";
 * explicitly wrapping operations, never undefined behaviour).  Every oracle entry point is called at
 * the edges the pins use -- the paper's largest admissible primes, all-(p-1) operands, n = 0, every Zech code at a
 * small field, centered extremes -- and a few closed forms are checked, so a sanitizer report or a wrong value
 * exits non-zero.  Built and run by tests/test_oracle_sanitized.py.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "../oracle/oracle.c"

static int fails = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            fprintf(stderr, "check failed at line %d: %s\n", __LINE__, #c); \
            ++fails;                                                    \
        }                                                               \
    } while (0)

int main(void)
{
    enum { N = 1000 };
    /* classical: the largest word-size prime, all-(p-1): sum = n (p-1)^2 = n (mod p) */
    uint32_t a32[N], b32[N];
    uint16_t a16[N], b16[N];
    const uint64_t p32 = 4294967291ull, p16 = 65521;
    for (int i = 0; i < N; ++i) {
        a32[i] = b32[i] = (uint32_t)(p32 - 1);
        a16[i] = b16[i] = (uint16_t)(p16 - 1);
    }
    CHECK(oracle_dot_classical(p32, a32, b32, O_U32, N) == N % p32);
    CHECK(oracle_dot_classical(p16, a16, b16, O_U16, N) == N % p16);
    CHECK(oracle_dot_classical(p16, a16, b16, O_U16, 0) == 0);
    uint64_t out[4];
    oracle_dot_batch_classical(p16, a16, 250, b16, O_U16, 4, 250, out);
    for (int r = 0; r < 4; ++r) CHECK(out[r] == 250);

    /* primality and roots at the paper's bounds */
    CHECK(oracle_is_prime(4294967291ull) && !oracle_is_prime(4294967293ull));
    CHECK(oracle_is_prime(2654435761ull) && oracle_is_prime(1073741789ull));
    CHECK(oracle_primitive_root(7) == 3 && oracle_primitive_root(101) == 2);
    CHECK(oracle_pow(2, 10, 1000) == 24);

    /* Montgomery at the largest B = 2^32 prime: to/from round trip and the all-(p-1) dot */
    const uint64_t pm = 2654435761ull;
    for (uint64_t x = pm - 3; x < pm; ++x) CHECK(oracle_from_mont(pm, oracle_to_mont(pm, x)) == x);
    for (int i = 0; i < N; ++i) a32[i] = b32[i] = (uint32_t)oracle_to_mont(pm, pm - 1);
    CHECK(oracle_from_mont(pm, oracle_dot_montgomery(pm, a32, b32, N)) == N % pm);

    /* binary64 at the largest fp64 prime (p (p-1) < 2^53) */
    const uint64_t pf = 94906249ull;
    double af[N], bf[N];
    int64_t bad = 0;
    for (int i = 0; i < N; ++i) af[i] = bf[i] = (double)(pf - 1);
    CHECK(oracle_dot_fp64(pf, af, bf, N, &bad) == (double)(N % pf) && bad < 0);
    af[7] = 0.5;  /* not an integer: reported, not undefined */
    oracle_dot_fp64(pf, af, bf, N, &bad);
    CHECK(bad == 7);
    uint64_t dec[4];
    CHECK(oracle_f64_decode(pf, bf, 4, dec) < 0 && dec[3] == pf - 1);

    /* Zech: every code pair at GF(101) through the integer and the Table-1 (t_plus1) dots, and the
       largest u16 field's codes at its edges */
    {
        const uint64_t p = 101, g = oracle_primitive_root(p);
        uint64_t *pw = malloc(sizeof(uint64_t) * 65536), *t = malloc(sizeof(uint64_t) * 65536),
                 *lg = malloc(sizeof(uint64_t) * 65536);
        for (uint16_t i = 0; i < p; ++i)
            for (uint16_t j = 0; j < p; ++j) {
                uint16_t x[2] = {i, j}, y[2] = {j, i};
                const uint64_t r1 = oracle_dot_zech(p, g, x, y, 2, pw, &bad);
                CHECK(bad < 0);
                const uint64_t r2 = oracle_dot_zech_tplus1(p, g, x, y, 2, t, lg, &bad);
                CHECK(bad < 0 && r1 == r2);
            }
        const uint64_t pz = 65521, gz = oracle_primitive_root(pz);
        uint16_t za[6] = {0, 1, 2, (uint16_t)(pz - 2), (uint16_t)(pz - 1), 255};
        const uint64_t r1 = oracle_dot_zech(pz, gz, za, za, 6, pw, &bad);
        CHECK(bad < 0);
        const uint64_t r2 = oracle_dot_zech_tplus1(pz, gz, za, za, 6, t, lg, &bad);
        CHECK(bad < 0 && r1 == r2);
        uint16_t zbad[1] = {(uint16_t)pz};  /* a code outside [0, q-1]: reported */
        oracle_dot_zech(pz, gz, zbad, zbad, 1, pw, &bad);
        CHECK(bad == 0);
        CHECK(oracle_zech_decode_one(pz, gz, oracle_zech_encode_one(pz, gz, pz - 1)) == (int64_t)(pz - 1));
        free(pw);
        free(t);
        free(lg);
    }

    /* centered (sec. 3.2.2): the extremes -h and h at the largest int32-storage prime */
    {
        const uint64_t p = 4294967291ull;
        const int64_t h = (int64_t)((p - 1) / 2);
        int32_t ca[N], cb[N];
        for (int i = 0; i < N; ++i) {
            ca[i] = (int32_t)(i & 1 ? h : -h);
            cb[i] = (int32_t)(-h);
        }
        CHECK(oracle_from_centered(p, oracle_to_centered(p, p - 1)) == p - 1);
        oracle_dot_centered(p, ca, cb, O_U32, N, &bad);
        CHECK(bad < 0);
        double da[N], db[N];
        const uint64_t pc = 189812507ull;
        for (int i = 0; i < N; ++i) da[i] = db[i] = (double)((int64_t)((pc - 1) / 2));
        oracle_dot_centered_f64(pc, da, db, N, &bad);
        CHECK(bad < 0);
    }
    if (fails) {
        fprintf(stderr, "%d checks failed\n", fails);
        return 1;
    }
    printf("oracle under sanitizers: ok\n");
    return 0;
}

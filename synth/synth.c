/*
 * synth.c -- seeded synthetic inputs shared by the tests, the bench and the
 * oracle checks.  This module holds NONE of the method's arithmetic (no
 * reduction, no representation, no dot product): it only draws integers.
 *
 * Generator: counter-based SplitMix64.  Element i of stream s under seed S is
 *     h(S, s, i) = mix64(key + (i + 1) * GAMMA),   key = S ^ (s << 56)
 * i.e. the (i+1)-th output of a standard SplitMix64 generator started at
 * `key`, so any slice [start, start+n) can be regenerated independently (each
 * rank generates only its own shard; the oracle regenerates any slice).
 *
 * A uniform draw in [0, m) is floor(h * m / 2^64) (multiply-high; bias below
 * m / 2^64).  Recipes:
 *   residues  : uniform in [0, p-1]                     (configs[0,1,2,4])
 *   zech codes: 0 with probability zero_num/zero_den,    (configs[3])
 *               else uniform in [1, qbar]
 */
#include <stdint.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t key, uint64_t i)
{
    return mix64(key + (i + 1) * GAMMA);
}

static inline uint64_t below(uint64_t h, uint64_t m)
{
    return (uint64_t)(((unsigned __int128)h * m) >> 64);
}

static inline uint64_t key_of(uint64_t seed, uint64_t stream)
{
    return seed ^ (stream << 56);
}

void synth_raw(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t *out)
{
    uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = draw(key, start + (uint64_t)i);
}

void synth_uniform_u16(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t m, uint16_t *out)
{
    uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (uint16_t)below(draw(key, start + (uint64_t)i), m);
}

void synth_uniform_u32(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t m, uint32_t *out)
{
    uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (uint32_t)below(draw(key, start + (uint64_t)i), m);
}

void synth_uniform_u64(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t m, uint64_t *out)
{
    uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = below(draw(key, start + (uint64_t)i), m);
}

/* exact integers in [0, m) stored as binary64 (m <= 2^53) */
void synth_uniform_f64(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t m, double *out)
{
    uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (double)below(draw(key, start + (uint64_t)i), m);
}

/* codes: 0 with probability zero_num/zero_den, else uniform in [1, qbar] */
void synth_zech_codes_u16(uint64_t seed, uint64_t stream, uint64_t start, int64_t n, uint64_t qbar,
                          uint64_t zero_num, uint64_t zero_den, uint16_t *out)
{
    uint64_t key = key_of(seed, stream);
    /* threshold = floor(zero_num * 2^64 / zero_den) */
    uint64_t thr = (uint64_t)((((unsigned __int128)zero_num) << 64) / zero_den);
    if (zero_num >= zero_den) thr = UINT64_MAX;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t h = draw(key, start + (uint64_t)i);
        out[i] = (h < thr) ? (uint16_t)0 : (uint16_t)(1 + below(mix64(h), qbar));
    }
}

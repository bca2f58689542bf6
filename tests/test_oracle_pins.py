"""Pins for the CPU oracle (oracle/): things the paper and the mathematics fix, not the oracle itself.

Each test names what it pins.  A plausible oracle mistake (dropped term, wrong index, transposed
operand, B instead of B^-1, off-by-one Zech code) fails at least one of them:
  * paper-printed constants (tests/golden/paper_constants.json, cited) pin is_prime + the bound
    predicates of sec. 2.1, 2.2, 2.4 and Eq. (1);
  * SPEC worked examples (tests/golden/spec_examples.json, cited);
  * closed forms of the dot: all-ones of length p, all-(p-1), sum of squares,
    Fermat power sums, the Zech geometric cycle, Montgomery closed forms for Mersenne 2^31-1;
  * invariants: bilinearity, symmetry, range, shard additivity;
  * brute force with Python integers on tiny inputs (oracle/bruteforce.py).
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLDEN, "paper_constants.json")))
SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))

LANDMARK_PRIMES = [2, 3, 5, 7, 101, 1009, 2897, 32749, 40009, 40499, 46337, 65521]


def largest_prime_with(pred, start):
    """Largest prime p <= start with pred(p) (pred monotone decreasing), and the next prime above it."""
    p = start
    while not (pred(p) and oracle.is_prime(p)):
        p -= 1
    q = p + 1
    while not oracle.is_prime(q):
        q += 1
    return p, q


# ------------------------------------------------------------------ paper constants
@pytest.mark.parametrize("key,m,signed", [
    ("classical_signed_32", 32, True), ("classical_signed_64", 64, True),
    ("classical_unsigned_32", 32, False), ("classical_unsigned_64", 64, False)])
def test_classical_prime_bounds_printed(key, m, signed):
    """Sec. 2.1: the AXPY value a*x+y <= p(p-1) must not overflow an m-bit word."""
    lim = 2 ** (m - 1) if signed else 2 ** m
    p, nxt = largest_prime_with(lambda p: p * (p - 1) < lim, math.isqrt(lim) + 2)
    assert p == PAPER[key]["value"]
    assert nxt * (nxt - 1) >= lim  # reading G5: inclusive; the next prime fails


@pytest.mark.parametrize("key,B", [("montgomery_B16", 2 ** 16), ("montgomery_B32", 2 ** 32)])
def test_montgomery_prime_bounds_printed(key, B):
    """Sec. 2.2: (p-1)^2 + p(B-1) < B^2."""
    pred = lambda p: (p - 1) ** 2 + p * (B - 1) < B * B
    start = int(B * (math.sqrt(5) - 1) / 2) + 16  # the predicate's root is B(sqrt5-1)/2
    assert not pred(start)
    p, nxt = largest_prime_with(pred, start)
    assert p == PAPER[key]["value"]
    assert not pred(nxt)


def test_zech_index_bound_printed():
    """Sec. 2.4: index sums i+j <= 2(q-1) stay below 2^31 (signed 32-bit)."""
    p, _ = largest_prime_with(lambda q: 2 * (q - 1) < 2 ** 31, 2 ** 30 + 8)
    assert p == PAPER["zech_index_32"]["value"]


def test_lambda_example_printed():
    """Eq. (1): largest lambda with lambda (p-1)^2 < 2^64 at p = 40009 is 1.15 10^10."""
    c = PAPER["lambda_p40009_m64"]
    p, m = c["p"], c["m"]
    lam = (2 ** m - 1) // (p - 1) ** 2
    assert lam * (p - 1) ** 2 < 2 ** m <= (lam + 1) * (p - 1) ** 2
    assert f"{lam / 1e10:.2f}" == "1.15"
    assert oracle.is_prime(p)


def test_hybrid_threshold_printed():
    """Sec. 3.4: at DIM = 512, m = 32 the last prime needing a single division is 2897."""
    c = PAPER["hybrid_threshold_dim512_m32"]
    p, nxt = largest_prime_with(lambda p: c["dim"] * (p - 1) ** 2 < 2 ** c["m"], 3000)
    assert p == c["value"]
    assert c["dim"] * (nxt - 1) ** 2 >= 2 ** c["m"]
    # reading G4: under the printed p(p-1) > 2^23 form the last prime is 2887, not 2897
    p2, _ = largest_prime_with(lambda p: p * (p - 1) <= 2 ** 23, 3000)
    assert p2 == 2887


def test_zech_table_size_printed():
    """a 2^26-element field needs 256 M(i)B of 4-byte table entries (reading G17)."""
    assert PAPER["zech_table_2_26_bytes"]["q"] * 4 == 256 * 2 ** 20


# ------------------------------------------------------------------ SPEC worked examples
def test_spec_examples():
    e = SPEC["oracle_dot_small"]
    a = np.array(e["a"], np.uint32)
    b = np.array(e["b"], np.uint32)
    assert oracle.dot_classical(e["p"], a, b) == e["value"]
    e = SPEC["pow_mod"]
    assert oracle.pow_mod(e["a"], e["e"], e["m"]) == e["value"]
    for p, g in SPEC["primitive_roots"]["values"].items():
        assert oracle.primitive_root(int(p)) == g
    e = SPEC["inv_mod"]
    assert oracle.inv_mod(e["a"], e["p"]) == e["value"]
    e = SPEC["factorize_40008"]
    assert math.prod(e["factors"]) == e["n"] and all(oracle.is_prime(f) for f in e["factors"])
    e = SPEC["zech_p7_powers"]
    assert [oracle.zech_decode(e["p"], e["g"], c) for c in range(1, 7)] == e["powers_1_to_6"]
    e = SPEC["zech_p7_encoding"]
    for x, code in e["encode"].items():
        assert oracle.zech_encode(e["p"], e["g"], int(x)) == code
    e = SPEC["zech_p7_mul"]
    x = oracle.zech_decode(e["p"], e["g"], e["i"]) * oracle.zech_decode(e["p"], e["g"], e["j"]) % e["p"]
    assert oracle.zech_encode(e["p"], e["g"], x) == e["value"]


# ------------------------------------------------------------------ number theory vs brute force
def test_is_prime_matches_sieve():
    n = 20000
    sieve = np.ones(n, bool)
    sieve[:2] = False
    for i in range(2, int(n ** 0.5) + 1):
        if sieve[i]:
            sieve[i * i::i] = False
    assert [oracle.is_prime(i) for i in range(n)] == list(sieve)


def test_primitive_root_and_order_bruteforce():
    for p in [q for q in range(2, 400) if bf.is_prime(q)]:
        g = oracle.primitive_root(p)
        assert g == bf.primitive_root(p)
        assert oracle.order(g, p) == p - 1 or p == 2
    assert oracle.primitive_root(32749) == 2  # configs[3] generator, reading G12
    assert oracle.primitive_root(100) == 0  # not prime


def test_inverse_exhaustive_small():
    for p in [2, 3, 5, 7, 101, 1009]:
        for a in range(1, p):
            assert a * oracle.inv_mod(a, p) % p == 1
    assert oracle.inv_mod(0, 7) == 0


# ------------------------------------------------------------------ Montgomery encode/decode
def test_montgomery_closed_forms():
    """B = 2^32: for p = 2^31-1, B = 2 mod p so a*B = 2a; for p = 2^32-5, B = 5 mod p."""
    rng = random.Random(1)
    for p, bmod in [(2 ** 31 - 1, 2), (4294967291, 5)]:
        for a in [0, 1, 2, p - 1, p // 2] + [rng.randrange(p) for _ in range(200)]:
            x = oracle.to_mont(p, a)
            assert x == bmod * a % p
            assert oracle.from_mont(p, x) == a
    for p in [3, 7, 101, 40009, 40499, 65521, 2654435761]:
        for a in [0, 1, p - 1] + [rng.randrange(p) for _ in range(100)]:
            assert oracle.to_mont(p, a) == bf.to_mont(p, a)
            assert oracle.from_mont(p, oracle.to_mont(p, a)) == a


def test_zech_encode_decode_exhaustive():
    for p in [3, 5, 7, 11, 101, 1009]:
        g = oracle.primitive_root(p)
        seen = set()
        for code in range(p):
            x = oracle.zech_decode(p, g, code)
            assert x == bf.zech_decode(p, g, code)
            assert oracle.zech_encode(p, g, x) == code
            seen.add(x)
        assert seen == set(range(p))  # the encoding is a bijection onto GF(p)
    with pytest.raises(ValueError):
        oracle.zech_decode(7, 3, 7)
    pw = oracle.zech_powers(101, 2)
    assert [int(v) for v in pw] == [pow(2, c, 101) for c in range(101)]


# ------------------------------------------------------------------ dot: brute force
def _rand_vec(rng, p, n):
    return [rng.randrange(p) for _ in range(n)]


@pytest.mark.parametrize("p", LANDMARK_PRIMES + [2 ** 31 - 1, 67108859, 4294967291])
def test_dot_classical_bruteforce(p):
    rng = random.Random(p)
    for n in [0, 1, 2, 3, 17, 64, 511, 512, 513]:
        a, b = _rand_vec(rng, p, n), _rand_vec(rng, p, n)
        dt = np.uint16 if p < 2 ** 16 else np.uint32
        r = oracle.dot_classical(p, np.array(a, dt), np.array(b, dt))
        assert r == bf.dot(p, a, b)
        assert 0 <= r < p
        r64 = oracle.dot_classical(p, np.array(a, np.uint64), np.array(b, np.uint64))
        assert r64 == r


def test_dot_classical_64bit_products_do_not_wrap():
    """Products of u32 near 2^32 exceed 2^64 only when summed; the oracle must use 128 bits."""
    p = 4294967291
    a = np.full(1000, p - 1, np.uint32)
    assert oracle.dot_classical(p, a, a) == 1000 % p  # (p-1)^2 = 1 mod p


@pytest.mark.parametrize("p", [3, 7, 101, 32749, 40009, 40499, 65521, 2 ** 31 - 1, 2654435761])
def test_dot_montgomery_bruteforce(p):
    rng = random.Random(p + 1)
    for n in [0, 1, 2, 3, 64, 513]:
        a, b = _rand_vec(rng, p, n), _rand_vec(rng, p, n)
        am = np.array([bf.to_mont(p, x) for x in a], np.uint32)
        bm = np.array([bf.to_mont(p, x) for x in b], np.uint32)
        r = oracle.dot_montgomery(p, am, bm)
        assert r == bf.to_mont(p, bf.dot(p, a, b))


@pytest.mark.parametrize("p", [2, 3, 101, 32749, 65521, 67108859, 94906249])
def test_dot_fp64_bruteforce(p):
    rng = random.Random(p + 2)
    for n in [0, 1, 2, 3, 64, 513]:
        a, b = _rand_vec(rng, p, n), _rand_vec(rng, p, n)
        r = oracle.dot_fp64(p, np.array(a, np.float64), np.array(b, np.float64))
        assert r == float(bf.dot(p, a, b)) and math.copysign(1.0, r) == 1.0
    with pytest.raises(ValueError):
        oracle.dot_fp64(p, np.array([0.5]), np.array([1.0]))
    with pytest.raises(ValueError):
        oracle.dot_fp64(p, np.array([float(p)]), np.array([1.0]))


@pytest.mark.parametrize("p", [3, 7, 11, 101, 1009, 32749])
def test_dot_zech_bruteforce(p):
    rng = random.Random(p + 3)
    g = bf.primitive_root(p) if p < 2000 else 2
    for n in [0, 1, 2, 3, 64, 513]:
        ca = [rng.randrange(p) for _ in range(n)]
        cb = [rng.randrange(p) for _ in range(n)]
        r = oracle.dot_zech(p, g, np.array(ca, np.uint16), np.array(cb, np.uint16))
        want = bf.dot(p, [bf.zech_decode(p, g, c) for c in ca], [bf.zech_decode(p, g, c) for c in cb])
        assert r == bf.zech_encode(p, g, want)


def test_dot_batch_bruteforce_nonsquare():
    """A non-square, padded (lda > n) matrix catches a transposed or mis-strided oracle."""
    rng = random.Random(5)
    p, rows, n, lda = 65521, 7, 13, 16
    A = np.array([rng.randrange(p) for _ in range(rows * lda)], np.uint16)
    x = np.array(_rand_vec(rng, p, n), np.uint16)
    out = oracle.dot_batch_classical(p, A, x, lda=lda, rows=rows, n=n)
    for r in range(rows):
        assert out[r] == bf.dot(p, A[r * lda:r * lda + n].tolist(), x.tolist())


# ------------------------------------------------------------------ dot: closed forms
@pytest.mark.parametrize("p", [101, 1009, 32749, 65521])
def test_closed_forms_classical(p):
    dt = np.uint16 if p < 2 ** 16 else np.uint32
    ones = np.ones(p, dt)
    assert oracle.dot_classical(p, ones, ones) == 0  # sum of p ones
    for n in [1, 2, 100000]:
        v = np.full(n, p - 1, dt)
        assert oracle.dot_classical(p, v, v) == n % p  # (p-1)^2 = 1
    x = np.arange(p, dtype=np.uint64)
    assert oracle.dot_classical(p, x, x) == 0  # sum_{i<p} i^2 = (p-1)p(2p-1)/6 = 0 for p > 3


@pytest.mark.parametrize("p", [101, 1009])
def test_fermat_power_sums(p):
    """sum_{x=1}^{p-1} x^k = -1 if (p-1) | k else 0 (mod p), via a_x = x, b_x = x^(k-1)."""
    x = np.arange(1, p, dtype=np.uint64)
    for k in [1, 2, 5, p - 1, 2 * (p - 1), p, 3 * (p - 1) + 1]:
        b = np.array([pow(int(v), k - 1, p) for v in x], np.uint64)
        want = p - 1 if k % (p - 1) == 0 else 0
        assert oracle.dot_classical(p, x, b) == want


def test_closed_forms_config_sizes():
    """all-(p-1) of length n gives n mod p at each config's prime and length."""
    assert oracle.dot_classical(65521, np.full(100000, 65520, np.uint32), np.full(100000, 65520, np.uint32)) == 34479
    p = 67108859
    v = np.full(10 ** 6, float(p - 1))
    assert oracle.dot_fp64(p, v, v) == float(10 ** 6 % p)
    p = 2 ** 31 - 1
    m = np.full(1 << 20, oracle.to_mont(p, p - 1), np.uint32)
    assert oracle.dot_montgomery(p, m, m) == oracle.to_mont(p, (1 << 20) % p)
    p, g = 32749, 2
    code_m1 = oracle.zech_encode(p, g, p - 1)
    assert code_m1 == (p - 1) // 2  # g^((q-1)/2) = -1 (i_{-1})
    c = np.full(1 << 16, code_m1, np.uint16)
    assert oracle.dot_zech(p, g, c, c) == oracle.zech_encode(p, g, (1 << 16) % p)


@pytest.mark.parametrize("p", [7, 101, 32749, 65521])
def test_zech_geometric_cycle(p):
    """sum_{c=1}^{qbar} g^c = 0: codes 1..q-1 dotted with the code of 1 (q-1)."""
    g = oracle.primitive_root(p)
    a = np.arange(1, p, dtype=np.uint16)
    b = np.full(p - 1, p - 1, np.uint16)
    assert oracle.dot_zech(p, g, a, b) == 0
    # and with one term dropped the sum is -g^(q-1)... = -1, code (q-1)/2
    assert oracle.dot_zech(p, g, a[:-1], b[:-1]) == oracle.zech_encode(p, g, p - 1)


# ------------------------------------------------------------------ dot: invariants
@pytest.mark.parametrize("p", [65521, 2 ** 31 - 1, 4294967291])
def test_bilinearity_symmetry_additivity(p):
    rng = np.random.default_rng(p % 1000)
    n = 4099
    dt = np.uint32
    a, b, c = (rng.integers(0, p, n, dtype=np.uint64) for _ in range(3))
    d = lambda u, v: oracle.dot_classical(p, u.astype(dt), v.astype(dt))
    bc = ((b + c) % p).astype(np.uint64)
    assert d(a, bc) == (d(a, b) + d(a, c)) % p
    assert d(a, b) == d(b, a)
    s = int(rng.integers(1, p))
    sa = ((a.astype(object) * s) % p).astype(np.uint64)
    assert d(sa, b) == d(a, b) * s % p
    for cut in [0, 1, 1000, n - 1, n]:
        assert (d(a[:cut], b[:cut]) + d(a[cut:], b[cut:])) % p == d(a, b)


# ------------------------------------------------------------------ Zech Table 1 (F3)
def _zech_maps(p, g):
    """decode list and encode dict from the literal P:128-130 cases (bruteforce.py, Python pow)."""
    dec = [bf.zech_decode(p, g, c) for c in range(p)]
    enc = {x: c for c, x in enumerate(dec)}
    assert len(enc) == p  # bijection onto GF(p)
    return dec, enc


@pytest.mark.parametrize("p", [2, 3, 5, 7, 11, 13, 101, 257])
def test_zech_table1_mul_add_exhaustive(p):
    """Pins oracle_zech_mul / oracle_zech_add / t_plus1 (sec. 2.4 Table 1): every pair of
    codes gives the code of the field product / sum computed with Python integers."""
    g = bf.primitive_root(p)
    dec, enc = _zech_maps(p, g)
    t = oracle.zech_tplus1(p, g)
    assert t.size == p  # "a table of size q"
    for i in range(p):
        for j in range(p):
            assert oracle.zech_mul(p, i, j) == enc[dec[i] * dec[j] % p], (i, j)
            assert oracle.zech_add(p, t, i, j) == enc[(dec[i] + dec[j]) % p], (i, j)


@pytest.mark.parametrize("p", [32749, 40009, 65521])
def test_zech_tplus1_identities(p):
    """t_plus1 against facts independent of how it is built: its definition g^h = 1 + g^k on sampled
    k (Python pow), the zero at k = qbar/2 (g^(qbar/2) = -1), and Zech's reflection identity
    Z(-k) = Z(k) - k (mod qbar), from 1 + g^-k = g^-k (1 + g^k)."""
    g = oracle.primitive_root(p)
    qbar = p - 1
    t = [int(v) for v in oracle.zech_tplus1(p, g)]
    assert t[qbar // 2] == 0 and t[qbar] == t[0]
    assert pow(g, t[0], p) == 2
    rng = random.Random(p)
    for k in rng.sample(range(qbar), 2000):
        if k == qbar // 2:
            continue
        assert pow(g, t[k], p) == (1 + pow(g, k, p)) % p
        assert 1 <= t[k] <= qbar
    for k in range(1, qbar):
        if k == qbar // 2:
            continue
        assert (t[qbar - k] - (t[k] - k)) % qbar == 0, k
    assert t.count(0) == 1  # 1 + g^k = 0 only at k = qbar/2


@pytest.mark.parametrize("p", [3, 7, 101, 1009, 32749, 40009, 65521])
def test_dot_zech_tplus1_unique_result(p):
    """The pure-Zech accumulation reaches the unique field element: equal to the integer-decoded
    dot (oracle_dot_zech) and, on tiny inputs, to Python-integer brute force; zero-heavy inputs
    and sums that cancel to zero are included."""
    g = oracle.primitive_root(p)
    rng = random.Random(p + 7)
    for n in [0, 1, 2, 3, 64, 513, 5000]:
        ca = np.array([0 if rng.random() < 0.1 else rng.randrange(1, p) for _ in range(n)], np.uint16)
        cb = np.array([0 if rng.random() < 0.1 else rng.randrange(1, p) for _ in range(n)], np.uint16)
        r = oracle.dot_zech_tplus1(p, g, ca, cb)
        assert r == oracle.dot_zech(p, g, ca, cb)
        if n <= 64:
            want = bf.dot(p, [bf.zech_decode(p, g, int(c)) for c in ca], [bf.zech_decode(p, g, int(c)) for c in cb])
            assert r == bf.zech_encode(p, g, want)
    # x + (-x) = 0: the code of -1 is qbar/2, so [c, c] . [qbar, qbar/2] cancels
    c = np.array([1, 1], np.uint16)
    assert oracle.dot_zech_tplus1(p, g, c, np.array([p - 1, (p - 1) // 2], np.uint16)) == 0
    # all-ones of length p (code qbar) sums to p = 0
    ones = np.full(p, p - 1, np.uint16)
    assert oracle.dot_zech_tplus1(p, g, ones, ones) == 0
    with pytest.raises(ValueError):
        oracle.dot_zech_tplus1(p, g, np.array([p], np.uint32), np.array([1], np.uint32))


# ------------------------------------------------------------------ centered representation (F2)
@pytest.mark.parametrize("p", [3, 5, 7, 11, 101, 1009])
def test_centered_encoding_exhaustive(p):
    """sec. 3.2.2: the encoding is a bijection between [0, p) and [-(p-1)/2, (p-1)/2] that
    commutes with reduction mod p; the SPEC examples 0 -> 0, p-1 -> -1, (p-1)/2 fixed."""
    h = (p - 1) // 2
    seen = set()
    for r in range(p):
        c = oracle.to_centered(p, r)
        assert -h <= c <= h and c % p == r and c == bf.to_centered(p, r)
        assert oracle.from_centered(p, c) == r
        seen.add(c)
    assert seen == set(range(-h, h + 1))
    assert oracle.to_centered(p, 0) == 0 and oracle.to_centered(p, p - 1) == -1 and oracle.to_centered(p, h) == h


@pytest.mark.parametrize("p", [3, 7, 101, 32749, 46337, 65521, 2 ** 31 - 1, 4294967291])
def test_dot_centered_bruteforce(p):
    rng = random.Random(p + 11)
    h = (p - 1) // 2
    dts = ([np.int16] if p <= 65535 else []) + ([np.int32] if p <= 2 ** 32 else []) + [np.int64]
    for dt in dts:
        for n in [0, 1, 2, 3, 64, 513]:
            a = [rng.randint(-h, h) for _ in range(n)]
            b = [rng.randint(-h, h) for _ in range(n)]
            r = oracle.dot_centered(p, np.array(a, dt), np.array(b, dt))
            assert r == bf.to_centered(p, bf.dot(p, a, b)) and -h <= r <= h
            # the same field element as the classical dot of the decoded residues
            ra = np.array([x % p for x in a], np.uint64)
            rb = np.array([x % p for x in b], np.uint64)
            assert r % p == oracle.dot_classical(p, ra, rb)
    if p < 2 ** 53:
        a = [float(rng.randint(-h, h)) for _ in range(300)]
        b = [float(rng.randint(-h, h)) for _ in range(300)]
        r = oracle.dot_centered(p, np.array(a), np.array(b))
        assert r == float(bf.to_centered(p, bf.dot(p, [int(x) for x in a], [int(x) for x in b])))
        assert math.copysign(1.0, oracle.dot_centered(p, np.array([0.0]), np.array([-1.0]))) == 1.0


@pytest.mark.parametrize("p", [101, 65521, 67108859])
def test_dot_centered_invariants(p):
    """negation symmetry dot(-a, b) = -dot(a, b) (the centered range is symmetric), all -1 of length n
    gives n mod p centered, and out-of-range entries are rejected."""
    rng = random.Random(p)
    h = (p - 1) // 2
    a = np.array([rng.randint(-h, h) for _ in range(1000)], np.int64)
    b = np.array([rng.randint(-h, h) for _ in range(1000)], np.int64)
    r = oracle.dot_centered(p, a, b)
    assert oracle.dot_centered(p, -a, b) == (-r if abs(r) != 0 else 0)
    m = np.full(5000, -1, np.int64)
    assert oracle.dot_centered(p, m, m) == bf.to_centered(p, 5000)
    with pytest.raises(ValueError):
        oracle.dot_centered(p, np.array([h + 1], np.int64), np.array([1], np.int64))
    with pytest.raises(ValueError):
        oracle.dot_centered(p, np.array([0.5]), np.array([1.0]))

"""GPU parity: every entry point of libgfp (through the C ABI binding) against the CPU oracle, bit-exact.

Tolerance is 0 everywhere: integer results compare exactly, and the fp64 representation holds exact
integers (north_star: "the fp64 path holds integers exactly, so the tolerance there is 0"); doubles are
compared bitwise (no -0.0).  Inputs are seeded synthetic vectors from synth/ (DESIGN.md input recipe).
Sizes: the SPEC sweep at small n, k-boundary lengths, all-(p-1) worst cases, ragged tails,
misaligned starts, and each BASELINE.json config at its full size (the oracle finishes each in seconds).
"""
import struct

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
CL, MO, FP, ZE = gfp.CLASSICAL, gfp.MONTGOMERY, gfp.FP64, gfp.ZECH
DEV = "cuda:0"
SEED = synth.BASE_SEED
SWEEP_PRIMES = [2, 3, 5, 7, 101, 1009, 2897, 32749, 40009, 40499, 46337, 65521]
SWEEP_DIMS = [0, 1, 2, 511, 512, 513, 10 ** 4]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield
    torch.cuda.synchronize()


def cu(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def bits(x: float) -> bytes:
    return struct.pack("<d", x)


def result_int(t: torch.Tensor) -> int:
    return int(t.cpu().to(torch.int64)[0]) if t.dtype != torch.float64 else t.cpu()[0].item()


def residues(p, n, stream, dtype, seed=SEED):
    return synth.uniform(seed, stream, 0, n, p, dtype)


# ------------------------------------------------------------------------------ classical
@pytest.mark.parametrize("p", SWEEP_PRIMES)
def test_classical_sweep(p):
    for dt in (np.uint16, np.uint32):
        for n in SWEEP_DIMS:
            a, b = residues(p, n, 0, dt, SEED + n), residues(p, n, 1, dt, SEED + n)
            r = gfp.dot(cu(a), cu(b), p, CL)
            assert r.dtype == (torch.uint16 if dt == np.uint16 else torch.uint32)
            assert result_int(r) == oracle.dot_classical(p, a, b), (p, dt, n)
        w = np.full(10 ** 4 + 3, p - 1, dt)  # worst case magnitudes
        assert result_int(gfp.dot(cu(w), cu(w), p, CL)) == oracle.dot_classical(p, w, w) == (10 ** 4 + 3) % p


def test_classical_c1_config():
    """configs[0]: GF(65521), u32, n = 100000."""
    p, n = 65521, 100000
    a, b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
    assert result_int(gfp.dot(cu(a), cu(b), p, CL)) == oracle.dot_classical(p, a, b)


@pytest.mark.parametrize("p", [4294967291, 3037000493, 2 ** 31 - 1, 65537])
def test_classical_u32_large_primes_overflow_path(p):
    """k is tiny here, so the kernel takes a sec. 3.3 path (the Eq. (2) hybrid, or the carry word)."""
    info = gfp.query(p, CL, torch.uint32)
    for n in [1, 3, 4, 5, 17, 1000, 100003, 2 ** 21 + 5]:
        a, b = residues(p, n, 0, np.uint32, SEED + 7), residues(p, n, 1, np.uint32, SEED + 7)
        assert result_int(gfp.dot(cu(a), cu(b), p, CL)) == oracle.dot_classical(p, a, b), (p, n)
    w = np.full(3 * 10 ** 6 + 1, p - 1, np.uint32)  # every add wraps the u64 when (p-1)^2 ~ 2^64
    assert result_int(gfp.dot(cu(w), cu(w), p, CL)) == (3 * 10 ** 6 + 1) % p
    assert info["k"] >= 1
    # the built-in plan: Eq. (2) hybrid while lambda = floor((2^64-1)/(p(p-1))) >= 4, else the carry word
    lam = (2 ** 64 - 1) // (p * (p - 1))
    pl = gfp.plan(p, CL, 3 * 10 ** 6 + 1, dtype=torch.uint32)
    if pl["strategy"] != gfp.AUTO and "ALL" not in pl["kernel"] and "THREAD" not in pl["kernel"]:
        assert pl["strategy"] == (gfp.HYBRID if lam >= 4 else gfp.CARRY), (p, pl)
    # worst-case batches through the same built-in choice (rows of 4096 overflow a lane's u64 sum)
    rows, n = 37, 4096
    W = np.full((rows, n), p - 1, np.uint32)
    got = gfp.dot_batch(cu(W), cu(W[0]), p, CL).cpu().to(torch.int64).numpy()
    assert (got == n % p).all(), (p, "batch worst case")


def test_classical_u32_largest_prime_full_size():
    """bench.py C3-p4294967291: n = 2^28 at p = 4294967291 through the built-in plan (the carry word: the
    carry flag of every 64-bit add counted), against the oracle; and an all-(p-1) vector (closed form n mod p,
    a carry on nearly every product)."""
    p, n = 4294967291, 1 << 28
    a = synth.uniform(SEED + 11, synth.STREAM_A, 0, n, p, np.uint32)
    b = synth.uniform(SEED + 11, synth.STREAM_B, 0, n, p, np.uint32)
    assert result_int(gfp.dot(cu(a), cu(b), p, CL)) == oracle.dot_classical(p, a, b)
    w = cu(np.full(n, p - 1, np.uint32))
    assert result_int(gfp.dot(w, w, p, CL)) == n % p
    for strat in (gfp.CARRY, gfp.OVERFLOW):
        assert result_int(gfp.dot_ex(w, w, p, CL, strategy=strat)) == n % p


def test_misaligned_and_ragged():
    p = 65521
    n = 100003
    a, b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
    ta, tb = cu(a), cu(b)
    for oa, ob in [(1, 1), (2, 2), (3, 3), (1, 2), (0, 3), (5, 0)]:
        m = n - 7
        r = gfp.dot(ta[oa:oa + m], tb[ob:ob + m], p, CL)
        assert result_int(r) == oracle.dot_classical(p, a[oa:oa + m], b[ob:ob + m]), (oa, ob)
    a16, b16 = a.astype(np.uint16), b.astype(np.uint16)
    t16a, t16b = cu(a16), cu(b16)
    for oa, ob in [(1, 1), (7, 7), (3, 5)]:
        m = n - 9
        r = gfp.dot(t16a[oa:oa + m], t16b[ob:ob + m], p, CL)
        assert result_int(r) == oracle.dot_classical(p, a16[oa:oa + m], b16[ob:ob + m])


NON_CO_ALIGNED = [  # (rep, storage, p, explicit strategy or None): every kernel with a realigning instance
    ("classical", np.uint16, 65521, None),        # 16-bit classical, one remainder
    ("classical", np.uint32, 65521, None),        # 32-bit classical
    ("classical", np.uint32, 2 ** 31 - 1, None),  # sec. 3.4 hybrid (lambda = 4)
    ("classical", np.uint32, 4294967291, None),   # sec. 3.3 carry word (lambda < 4)
    ("classical", np.uint32, 2 ** 31 - 1, "carry"),
    ("montgomery", np.uint32, 2 ** 31 - 1, None),
    ("fp64", np.float64, 67108859, None),
    ("zech", np.uint16, 32749, None),
]


@pytest.mark.parametrize("case", NON_CO_ALIGNED, ids=lambda c: f"{c[0]}-{np.dtype(c[1]).name}-{c[2]}-{c[3]}")
def test_non_co_aligned_operands_every_byte_shift(case):
    """b's element 0 at every byte distance from a's 16-byte phase (the realigned vector path: each 16-byte
    window of b assembled from the two aligned vectors it straddles), at lengths around the vector width and at
    several tiles with a ragged tail, against the oracle on the same elements."""
    kind, dt, p, strat = case
    es = np.dtype(dt).itemsize
    per = 16 // es
    nmax = 70003
    if kind == "zech":
        g = gfp.query(p, ZE)["g"]
        A = synth.zech_codes(SEED + 41, 0, 0, nmax + per, p - 1)
        B = synth.zech_codes(SEED + 41, 1, 0, nmax + per, p - 1)
    else:
        A = residues(p, nmax + per, 0, dt, SEED + 41)
        B = residues(p, nmax + per, 1, dt, SEED + 41)
    tA, tB = cu(A), cu(B)
    if kind == "montgomery":
        tA, tB = gfp.to_rep(tA, p, MO), gfp.to_rep(tB, p, MO)
        A, B = host(tA), host(tB)
    rep = {"classical": CL, "montgomery": MO, "fp64": FP, "zech": ZE}[kind]

    def want(x, y):
        if kind == "classical":
            return oracle.dot_classical(p, x, y)
        if kind == "montgomery":
            return oracle.dot_montgomery(p, x, y)
        if kind == "fp64":
            return oracle.dot_fp64(p, x, y)
        return oracle.dot_zech(p, g, x, y)

    for oa in range(per):
        for ob in range(per):
            if oa == ob:
                continue
            for n in (0, 1, per - 1, per, per + 1, 2 * per + 3, 3 * per, 1037, nmax):
                x, y = tA[oa:oa + n], tB[ob:ob + n]
                if strat == "carry":
                    r = gfp.dot_ex(x, y, p, rep, strategy=gfp.CARRY)
                else:
                    r = gfp.dot(x, y, p, rep)
                got = result_int(r)
                w = want(A[oa:oa + n], B[ob:ob + n])
                if kind == "fp64":
                    assert bits(got) == bits(w), (oa, ob, n)
                else:
                    assert got == w, (oa, ob, n)


def test_empty_gives_zero_in_every_representation():
    e16 = torch.empty(0, dtype=torch.uint16, device=DEV)
    e32 = torch.empty(0, dtype=torch.uint32, device=DEV)
    e64 = torch.empty(0, dtype=torch.float64, device=DEV)
    assert result_int(gfp.dot(e32, e32, 65521, CL)) == 0
    assert result_int(gfp.dot(e32, e32, 2 ** 31 - 1, MO)) == 0
    r = gfp.dot(e64, e64, 67108859, FP)
    assert bits(r.cpu()[0].item()) == bits(0.0)
    assert result_int(gfp.dot(e16, e16, 32749, ZE)) == 0


# ------------------------------------------------------------------------------ Montgomery
MONT_PRIMES = [3, 7, 101, 40009, 40499, 65521, 2 ** 31 - 1, 2654435761]


@pytest.mark.parametrize("p", MONT_PRIMES)
def test_montgomery_conversion_and_dot(p):
    kr = gfp.query(p, MO)["mont_kr"]
    dims = sorted({0, 1, 2, 3, 4, 5, 7, 8, 511, 513, 10 ** 4 + 1, 3 * min(kr, 10) + 2})
    for n in dims:
        a, b = residues(p, n, 0, np.uint32, SEED + n), residues(p, n, 1, np.uint32, SEED + n)
        am, bm = gfp.to_rep(cu(a), p, MO), gfp.to_rep(cu(b), p, MO)
        ham = host(am)
        want_am = np.array([oracle.to_mont(p, int(v)) for v in a[:64]], np.uint32)
        assert np.array_equal(ham[:64], want_am)
        r = gfp.dot(am, bm, p, MO)
        assert result_int(r) == oracle.dot_montgomery(p, ham, host(bm)), (p, n)
        assert np.array_equal(host(gfp.from_rep(am, p, MO)), a)  # round trip
    w = np.full(4099, p - 1, np.uint32)
    wm = gfp.to_rep(cu(w), p, MO)
    assert result_int(gfp.dot(wm, wm, p, MO)) == oracle.to_mont(p, 4099 % p)


def test_montgomery_closed_form_mersenne():
    """p = 2^31-1, B = 2^32 = 2 mod p: to_mont(a) = 2a mod p, exhaustive on a 2^24 sample + edges."""
    p = 2 ** 31 - 1
    a = np.concatenate([residues(p, 1 << 24, 5, np.uint32), np.array([0, 1, 2, p - 2, p - 1], np.uint32)])
    got = host(gfp.to_rep(cu(a), p, MO)).astype(np.uint64)
    assert np.array_equal(got, (2 * a.astype(np.uint64)) % p)


def test_montgomery_c3_config_full_size():
    """configs[2]: GF(2^31-1), Montgomery B = 2^32, n = 2^28 (1 GiB per operand), converted on device."""
    p, n = 2 ** 31 - 1, 1 << 28
    a, b = residues(p, n, 0, np.uint32, SEED + 2), residues(p, n, 1, np.uint32, SEED + 2)
    am, bm = gfp.to_rep(cu(a), p, MO), gfp.to_rep(cu(b), p, MO)
    r = result_int(gfp.dot(am, bm, p, MO))
    # oracle on the classical inputs, encoded: (sum a b mod p) * B mod p
    assert r == oracle.to_mont(p, oracle.dot_classical(p, a, b))
    # element-wise conversion check on a strided sample (closed form 2a mod p)
    got = host(am).astype(np.uint64)
    assert np.array_equal(got, (2 * a.astype(np.uint64)) % p)


# ------------------------------------------------------------------------------ fp64
FP_PRIMES = [2, 3, 101, 32749, 65521, 40009, 67108859, 94906249]


@pytest.mark.parametrize("p", FP_PRIMES)
def test_fp64_sweep(p):
    k = gfp.query(p, FP)["k"]
    dims = sorted(set(SWEEP_DIMS + [max(k - 1, 0), k, k + 1, 3 * k + 2] if k < 10 ** 6 else SWEEP_DIMS))
    for n in dims:
        a, b = residues(p, n, 0, np.float64, SEED + n), residues(p, n, 1, np.float64, SEED + n)
        r = gfp.dot(cu(a), cu(b), p, FP).cpu()[0].item()
        assert bits(r) == bits(oracle.dot_fp64(p, a, b)), (p, n)
    for n in [1, 2, 3, 8, 1001, 2 ** 20 + 3]:
        w = np.full(n, float(p - 1))
        r = gfp.dot(cu(w), cu(w), p, FP).cpu()[0].item()
        assert bits(r) == bits(float(n % p))


def _pairs_with_sum(p, T, rng):
    """x0, y0, x1, y1 in [0, p) with x0 y0 + x1 y1 = T exactly (T < 2 (p-1)^2), or None."""
    for _ in range(200):
        x0 = int(rng.integers(max(1, T // (p - 1) - (p - 1) if T > (p - 1) ** 2 else 1), p))
        y0 = min(p - 1, T // x0)
        R = T - x0 * y0
        if R < 0:
            continue
        if R < p:
            return x0, y0, R, 1
        lo = -(-R // (p - 1))
        for d in range(lo, min(p, lo + 2000)):
            if R % d == 0 and R // d < p:
                return x0, y0, d, R // d
    return None


@pytest.mark.parametrize("p", [32749, 65521, 67108859, 94906249])
def test_fp64_reduction_near_multiples_of_p(p):
    """Dots of one and two terms whose block sum T is k p - 1, k p + 1 (and the SURVEY H4 values where
    floor(T * invP) is off by one: T = 1781447353 at 32749, 1063012704 at 65521), so the NTL reduction's
    fix-up branch runs on device with exactly that T; results must be exact."""
    rng = np.random.default_rng(p)
    cases = []
    for d in (-1, 1):
        for _ in range(150):
            x = int(rng.integers(1, p))
            y = d * pow(x, -1, p) % p  # x y = d (mod p), T = x y over the whole range
            cases.append(([x], [y]))
            x0, y0, x1 = (int(v) for v in rng.integers(1, p, 3))
            y1 = (d - x0 * y0) * pow(x1, -1, p) % p  # x0 y0 + x1 y1 = d (mod p)
            cases.append(([x0, x1], [y0, y1]))
    special = {32749: 1781447353, 65521: 1063012704}.get(p)
    if special is not None:
        sol = _pairs_with_sum(p, special, rng)
        assert sol is not None
        cases.append(([sol[0], sol[2]], [sol[1], sol[3]]))
    for xa, xb in cases:
        a, b = np.array(xa, np.float64), np.array(xb, np.float64)
        r = gfp.dot(cu(a), cu(b), p, FP).cpu()[0].item()
        want = float(sum(int(u) * int(v) for u, v in zip(xa, xb)) % p)
        assert bits(r) == bits(want) == bits(oracle.dot_fp64(p, a, b)), (xa, xb)


def test_fp64_c2_config():
    """configs[1]: GF(67108859), fp64, n = 10^7."""
    p, n = 67108859, 10 ** 7
    a, b = residues(p, n, 0, np.float64, SEED + 1), residues(p, n, 1, np.float64, SEED + 1)
    r = gfp.dot(cu(a), cu(b), p, FP).cpu()[0].item()
    assert bits(r) == bits(oracle.dot_fp64(p, a, b))


def test_fp64_conversions():
    p = 67108859
    a = residues(p, 100001, 0, np.uint32)
    f = gfp.to_rep(cu(a), p, FP)
    assert f.dtype == torch.float64 and np.array_equal(host(f), a.astype(np.float64))
    assert np.array_equal(host(gfp.from_rep(f, p, FP)), a)


# ------------------------------------------------------------------------------ Zech
ZECH_PRIMES = [2, 3, 7, 101, 1009, 32749, 32771, 40009, 65521]


@pytest.mark.parametrize("p", ZECH_PRIMES)
def test_zech_sweep(p):
    g = gfp.query(p, ZE)["g"]
    assert g == oracle.primitive_root(p)
    for n in SWEEP_DIMS:
        ca = synth.zech_codes(SEED + n, 0, 0, n, p - 1)
        cb = synth.zech_codes(SEED + n, 1, 0, n, p - 1)
        r = gfp.dot(cu(ca), cu(cb), p, ZE)
        assert r.dtype == torch.uint16
        assert result_int(r) == oracle.dot_zech(p, g, ca, cb), (p, n)
    # geometric cycle: sum_{c=1}^{q-1} g^c = 0 -> code 0 (p > 2)
    a = np.arange(1, p, dtype=np.uint16)
    one = np.full(p - 1, p - 1, np.uint16)
    assert result_int(gfp.dot(cu(a), cu(one), p, ZE)) == (0 if p > 2 else 1)


@pytest.mark.parametrize("p", [7, 101, 32749, 40009, 65521])
def test_zech_conversions_exhaustive(p):
    g = gfp.query(p, ZE)["g"]
    x = np.arange(p, dtype=np.uint16 if p < 65536 else np.uint32)
    codes = host(gfp.to_rep(cu(x), p, ZE))
    pw = oracle.zech_powers(p, g)
    # decode with the oracle's own power list: code 0 -> 0, c -> g^c
    dec = np.where(codes == 0, 0, pw[codes.astype(np.int64)])
    assert np.array_equal(dec, x.astype(np.uint64))
    assert codes[1] == p - 1 and codes[0] == 0
    back = host(gfp.from_rep(cu(codes), p, ZE, dtype=torch.uint32))
    assert np.array_equal(back, x.astype(np.uint32))


def test_zech_c4_config():
    """configs[3]: GF(32749), Zech u16, n = 2^26, 10% zeros."""
    p, n = 32749, 1 << 26
    ca = synth.zech_codes(SEED + 3, 0, 0, n, p - 1)
    cb = synth.zech_codes(SEED + 3, 1, 0, n, p - 1)
    r = result_int(gfp.dot(cu(ca), cu(cb), p, ZE))
    assert r == oracle.dot_zech(p, 2, ca, cb)


# ------------------------------------------------------------------------------ batch
def test_batch_c5_config():
    """configs[4]: 65536 x 4096 u16 matrix-vector over GF(65521)."""
    p, rows, n = 65521, 65536, 4096
    A = residues(p, rows * n, 2, np.uint16, SEED + 4).reshape(rows, n)
    x = residues(p, n, 3, np.uint16, SEED + 4)
    out = host(gfp.dot_batch(cu(A), cu(x), p, CL))
    want = oracle.dot_batch_classical(p, A, x)
    assert np.array_equal(out.astype(np.uint64), want)


@pytest.mark.parametrize("shape", [(1, 4096), (7, 1), (33, 8), (100, 4097), (513, 1000), (3, 0), (2, 60000)])
def test_batch_shapes_u16(shape):
    p = 65521
    rows, n = shape
    A = residues(p, rows * n, 2, np.uint16).reshape(rows, n)
    x = residues(p, n, 3, np.uint16)
    out = host(gfp.dot_batch(cu(A), cu(x), p, CL))
    assert np.array_equal(out.astype(np.uint64), oracle.dot_batch_classical(p, A, x))
    w = np.full((rows, n), p - 1, np.uint16)
    out = host(gfp.dot_batch(cu(w), cu(w[0] if rows else np.zeros(n, np.uint16)), p, CL))
    assert np.all(out.astype(np.int64) == n % p)


def test_batch_padded_and_unaligned_rows():
    p = 40009
    rows, n = 257, 1003
    for lda in [1003, 1008, 1011]:
        A = residues(p, rows * lda, 2, np.uint16)
        x = residues(p, n, 3, np.uint16)
        out = host(gfp.dot_batch(cu(A), cu(x), p, CL, rows=rows, n=n, lda=lda))
        want = oracle.dot_batch_classical(p, A, x, lda=lda, rows=rows, n=n)
        assert np.array_equal(out.astype(np.uint64), want), lda
    # misaligned x / A start
    A = residues(p, rows * n + 1, 2, np.uint16)
    x = residues(p, n + 1, 3, np.uint16)
    out = host(gfp.dot_batch(cu(A)[1:], cu(x)[1:], p, CL, rows=rows, n=n, lda=n))
    assert np.array_equal(out.astype(np.uint64), oracle.dot_batch_classical(p, A[1:], x[1:], lda=n, rows=rows, n=n))


@pytest.mark.parametrize("p", [65521, 2 ** 31 - 1, 4294967291])
def test_batch_u32(p):
    rows, n = 300, 2053
    A = residues(p, rows * n, 2, np.uint32).reshape(rows, n)
    x = residues(p, n, 3, np.uint32)
    out = host(gfp.dot_batch(cu(A), cu(x), p, CL))
    assert np.array_equal(out.astype(np.uint64), oracle.dot_batch_classical(p, A, x))


def test_batch_other_representations():
    rows, n = 129, 777
    # Montgomery
    p = 2 ** 31 - 1
    A = residues(p, rows * n, 2, np.uint32)
    x = residues(p, n, 3, np.uint32)
    Am, xm = gfp.to_rep(cu(A), p, MO), gfp.to_rep(cu(x), p, MO)
    out = host(gfp.dot_batch(Am, xm, p, MO, rows=rows, n=n))
    want = oracle.dot_batch_classical(p, A, x, lda=n, rows=rows, n=n)
    assert np.array_equal(out.astype(np.uint64), np.array([oracle.to_mont(p, int(v)) for v in want], np.uint64))
    # fp64
    p = 67108859
    A = residues(p, rows * n, 2, np.float64)
    x = residues(p, n, 3, np.float64)
    out = host(gfp.dot_batch(cu(A), cu(x), p, FP, rows=rows, n=n))
    want = oracle.dot_batch_classical(p, A.astype(np.uint64), x.astype(np.uint64), lda=n, rows=rows, n=n)
    assert np.array_equal(out, want.astype(np.float64))
    # Zech
    for p in [32749, 65521]:
        g = gfp.query(p, ZE)["g"]
        CA = synth.zech_codes(SEED, 2, 0, rows * n, p - 1)
        cx = synth.zech_codes(SEED, 3, 0, n, p - 1)
        out = host(gfp.dot_batch(cu(CA), cu(cx), p, ZE, rows=rows, n=n))
        want = [oracle.dot_zech(p, g, CA[r * n:(r + 1) * n], cx) for r in range(rows)]
        assert np.array_equal(out.astype(np.int64), np.array(want, np.int64))


# ------------------------------------------------------------------------------ partial / finalize / host
@pytest.mark.parametrize("rep,p", [(CL, 65521), (MO, 2 ** 31 - 1), (FP, 67108859), (ZE, 32749)])
def test_shard_partials_and_finalize(rep, p):
    """dot(a, b) = finalize(sum_g partial(a_g, b_g)): the multi-GPU identity on virtual shards."""
    n = 1_000_003
    if rep == ZE:
        a = synth.zech_codes(SEED, 0, 0, n, p - 1)
        b = synth.zech_codes(SEED, 1, 0, n, p - 1)
        want = oracle.dot_zech(p, 2, a, b)
        ta, tb = cu(a), cu(b)
    elif rep == FP:
        a, b = residues(p, n, 0, np.float64), residues(p, n, 1, np.float64)
        want = oracle.dot_fp64(p, a, b)
        ta, tb = cu(a), cu(b)
    else:
        a, b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
        ta, tb = cu(a), cu(b)
        if rep == MO:
            ta, tb = gfp.to_rep(ta, p, MO), gfp.to_rep(tb, p, MO)
            want = oracle.to_mont(p, oracle.dot_classical(p, a, b))
        else:
            want = oracle.dot_classical(p, a, b)
    for G in [1, 2, 3, 8]:
        bounds = [n * g // G for g in range(G + 1)]
        parts = [gfp.dot_partial(ta[bounds[g]:bounds[g + 1]], tb[bounds[g]:bounds[g + 1]], p, rep) for g in range(G)]
        for pt in parts:
            assert 0 <= int(pt.cpu()[0]) < p
        summed = torch.stack(parts).sum(0)
        r = gfp.finalize(summed, p, rep, ta.dtype)
        got = r.cpu()[0].item() if rep == FP else int(r.cpu().to(torch.int64)[0])
        assert got == want, G


@pytest.mark.parametrize("rep,p", [(CL, 65521), (MO, 2 ** 31 - 1), (FP, 67108859), (ZE, 32749)])
def test_dot_host_end_to_end(rep, p):
    n = (64 << 20) // 4 * 3 + 12345  # several staging chunks and a ragged last one
    if rep == ZE:
        a = synth.zech_codes(SEED, 0, 0, n, p - 1)
        b = synth.zech_codes(SEED, 1, 0, n, p - 1)
        want = oracle.dot_zech(p, 2, a, b)
    elif rep == FP:
        a, b = residues(p, n, 0, np.float64), residues(p, n, 1, np.float64)
        want = oracle.dot_fp64(p, a, b)
    elif rep == MO:
        a = np.array([0], np.uint32)
        raw_a, raw_b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
        a = host(gfp.to_rep(cu(raw_a), p, MO))
        b = host(gfp.to_rep(cu(raw_b), p, MO))
        want = oracle.to_mont(p, oracle.dot_classical(p, raw_a, raw_b))
    else:
        a, b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
        want = oracle.dot_classical(p, a, b)
    ta, tb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
    assert gfp.dot_host(ta, tb, p, rep) == want
    assert gfp.dot_host(torch.from_numpy(a[:1000]), torch.from_numpy(b[:1000]), p, rep) == \
        gfp.dot(cu(a[:1000]), cu(b[:1000]), p, rep).cpu().to(torch.float64 if rep == FP else torch.int64)[0].item()
    # the multi-GPU end-to-end form (bench.py's N > 1 e2e leg): three host shards -> additive-form partials
    # (gfp_dot_host_partial: for Zech the classical value, never a code) -> sum -> gfp_finalize
    cuts = [0, n // 3, n // 3 + 17, n]
    parts = [gfp.dot_host_partial(ta[lo:hi], tb[lo:hi], p, rep) for lo, hi in zip(cuts[:-1], cuts[1:])]
    assert all(0 <= v < p for v in parts)
    summed = torch.tensor([sum(parts)], dtype=torch.int64, device=DEV)
    assert result_int(gfp.finalize(summed, p, rep, ta.dtype)) == want


def test_stream_and_graph_capture():
    """Results are stream-ordered; the single-launch dot is CUDA-graph capturable after a warm call."""
    p, n = 65521, 1 << 20
    a, b = residues(p, n, 0, np.uint32), residues(p, n, 1, np.uint32)
    ta, tb = cu(a), cu(b)
    want = oracle.dot_classical(p, a, b)
    s = torch.cuda.Stream()
    out = torch.empty(1, dtype=torch.uint32, device=DEV)
    with torch.cuda.stream(s):
        gfp.dot(ta, tb, p, CL, out=out)  # warm: allocates the per-stream workspace
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gfp.dot(ta, tb, p, CL, out=out, stream=s)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert result_int(out) == want


def test_launch_counter():
    p = 65521
    a = cu(residues(p, 1000, 0, np.uint32))
    gfp.launch_count(reset=True)
    for _ in range(5):
        gfp.dot(a, a, p, CL)
    assert gfp.launch_count() == 5


# ------------------------------------------------------------------------------ maximum sizes
def _full(n, value, dtype):
    """Device vector of n copies of `value` without a host copy (int16/int32 bit patterns viewed unsigned)."""
    if dtype == torch.uint16:
        v = value - (1 << 16) if value >= 1 << 15 else value
        return torch.full((n,), v, dtype=torch.int16, device=DEV).view(torch.uint16)
    v = value - (1 << 32) if value >= 1 << 31 else value
    return torch.full((n,), v, dtype=torch.int32, device=DEV).view(torch.uint32)


def test_beyond_2_31_elements_closed_form():
    """n > 2^31 exercises the 64-bit index arithmetic of every loop: all-(p-1) vectors dot to n mod p."""
    n = (1 << 31) + 4099
    p = 65521
    w = _full(n, p - 1, torch.uint16)
    assert result_int(gfp.dot(w, w, p, CL)) == n % p
    del w
    p = 32749
    c = _full(n, (p - 1) // 2, torch.uint16)  # code of -1 (i_{-1} = (q-1)/2); (-1)(-1) = 1
    assert result_int(gfp.dot(c, c, p, ZE)) == oracle.zech_encode(p, 2, n % p)
    del c
    torch.cuda.empty_cache()
    p = 2 ** 31 - 1
    m = _full(n, oracle.to_mont(p, p - 1), torch.uint32)
    assert result_int(gfp.dot(m, m, p, MO)) == oracle.to_mont(p, n % p)
    del m
    torch.cuda.empty_cache()


def test_batch_many_rows_closed_form():
    """rows > 2^20 with short rows: every row of all-(p-1) dots to n mod p."""
    p, rows, n = 65521, (1 << 21) + 3, 24
    A = _full(rows * n, p - 1, torch.uint16).view(rows, n)
    x = _full(n, p - 1, torch.uint16)
    out = gfp.dot_batch(A, x, p, CL)
    assert bool((out.to(torch.int32) == n % p).all())


def test_batch_beyond_2_32_elements_closed_form():
    """A matrix of more than 2^32 elements (8 GiB of u16): the 64-bit row offsets of the C5 fast path and of the
    Zech matrix-vector kernel, with a padded leading dimension; every row of all-(p-1) (the code of -1) dots
    to n mod p, and a row of zeros placed last dots to 0."""
    rows, n, lda = (1 << 20) + 5, 4096, 4104
    p = 65521
    A = _full(rows * lda, p - 1, torch.uint16)
    A.view(torch.int16).view(rows, lda)[-1].zero_()
    x = _full(n, p - 1, torch.uint16)
    out = gfp.dot_batch(A, x, p, CL, rows=rows, n=n, lda=lda).to(torch.int32)
    assert bool((out[:-1] == n % p).all()) and int(out[-1]) == 0
    p = 32749
    A.view(torch.int16).fill_((p - 1) // 2)  # code of -1
    A.view(torch.int16).view(rows, lda)[-1].zero_()
    x = _full(n, (p - 1) // 2, torch.uint16)
    out = gfp.dot_batch(A, x, p, ZE, rows=rows, n=n, lda=lda).to(torch.int32)
    assert bool((out[:-1] == oracle.zech_encode(p, 2, n % p)).all()) and int(out[-1]) == 0
    del A
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------------ fused combine (world 1)
def test_fused_allreduce_single_rank():
    """gfp_dot_allreduce on a one-rank group (the only group one GPU can host): the whole exchange protocol
    runs against the rank's own buffer; repeated calls advance the epoch, CUDA-graph replays reuse the
    device-resident state, and every representation matches the plain dot."""
    from paper_cs_0404008_b200 import dist as gd
    x = gd.PeerExchange()
    try:
        for p, rep, dt, gen in [(65521, gfp.CLASSICAL, np.uint32, "u"), (2 ** 31 - 1, gfp.MONTGOMERY, np.uint32, "u"),
                                (67108859, gfp.FP64, np.float64, "u"), (32749, gfp.ZECH, np.uint16, "z")]:
            for n in [0, 1, 1000, 1_000_003]:
                if gen == "z":
                    a, b = synth.zech_codes(SEED, 0, 0, n, p - 1), synth.zech_codes(SEED, 1, 0, n, p - 1)
                else:
                    a, b = synth.uniform(SEED, 0, 0, n, p, dt), synth.uniform(SEED, 1, 0, n, p, dt)
                ga, gb = cu(a), cu(b)
                if rep == gfp.MONTGOMERY:  # the inputs read as Montgomery forms: oracle decodes by B^-1
                    ref = oracle.dot_montgomery(p, a, b)
                else:
                    ref = oracle.dot(p, rep, a, b)
                want = gfp.dot(ga, gb, p, rep).cpu()
                assert (want[0].item() if rep == gfp.FP64 else int(want.to(torch.int64)[0])) == ref, (p, rep, n)
                for _ in range(3):
                    got = gd.dot_fused(ga, gb, p, rep, x).cpu()
                    assert torch.equal(got, want), (p, rep, n)  # equal to the oracle-checked value above
        p, n = 2 ** 31 - 1, 1 << 20
        a, b = cu(synth.uniform(SEED, 0, 0, n, p, np.uint32)), cu(synth.uniform(SEED, 1, 0, n, p, np.uint32))
        want = oracle.dot_classical(p, a.cpu().numpy(), b.cpu().numpy())
        out = torch.empty(1, dtype=torch.uint32, device=DEV)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            gd.dot_fused(a, b, p, gfp.CLASSICAL, x, out=out, stream=s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                gd.dot_fused(a, b, p, gfp.CLASSICAL, x, out=out, stream=s)
        for _ in range(10):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert int(out.cpu().to(torch.int64)[0]) == want
    finally:
        torch.cuda.synchronize()
        x.close()


def _mc_unsupported():
    """None when a multicast object can be created here, else the library's reason."""
    try:
        h = gfp.mc_create(1)[0]
    except gfp.GfpError as e:
        if e.status != 4:  # only GFP_E_UNSUPPORTED (no multicast team on this platform) is a skip
            raise
        return str(e)
    gfp.mc_destroy(h)
    return None


def test_fused_allreduce_nvls_single_rank():
    """gfp_dot_allreduce_mc (NVLS multicast: multimem.red into the switch, counter barrier, finalize) on a one-rank
    group -- the only group one GPU can host: multimem reductions and the acquire polling run for real through the
    multicast mapping; repeated epochs exercise both slot parities and the running-total bookkeeping, CUDA-graph
    replays reuse the device-resident state; every representation against the oracle."""
    from paper_cs_0404008_b200 import dist as gd
    why = _mc_unsupported()
    if why:
        pytest.skip(why)
    x = gd.MulticastExchange()
    try:
        for p, rep, dt, gen in [(65521, gfp.CLASSICAL, np.uint32, "u"), (2 ** 31 - 1, gfp.MONTGOMERY, np.uint32, "u"),
                                (67108859, gfp.FP64, np.float64, "u"), (32749, gfp.ZECH, np.uint16, "z"),
                                (4294967291, gfp.CLASSICAL, np.uint32, "u")]:
            for n in [0, 1, 1000, 1_000_003]:
                if gen == "z":
                    a, b = synth.zech_codes(SEED, 0, 0, n, p - 1), synth.zech_codes(SEED, 1, 0, n, p - 1)
                else:
                    a, b = synth.uniform(SEED, 0, 0, n, p, dt), synth.uniform(SEED, 1, 0, n, p, dt)
                want = oracle.dot_montgomery(p, a, b) if rep == gfp.MONTGOMERY else oracle.dot(p, rep, a, b)
                ga, gb = cu(a), cu(b)
                for _ in range(3):  # odd number of epochs per case: the parities alternate across cases
                    assert result_int(gd.dot_fused(ga, gb, p, rep, x)) == want, (p, rep, n)
        p, n = 2 ** 31 - 1, 1 << 20
        a, b = synth.uniform(SEED, 0, 0, n, p, np.uint32), synth.uniform(SEED, 1, 0, n, p, np.uint32)
        want = oracle.dot_classical(p, a, b)
        ga, gb = cu(a), cu(b)
        out = torch.empty(1, dtype=torch.uint32, device=DEV)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            gd.dot_fused(ga, gb, p, gfp.CLASSICAL, x, out=out, stream=s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(3):
                    gd.dot_fused(ga, gb, p, gfp.CLASSICAL, x, out=out, stream=s)
        for _ in range(7):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert int(out.cpu().to(torch.int64)[0]) == want
    finally:
        torch.cuda.synchronize()
        x.close()


def test_fused_allreduce_pure_zech_plan():
    """an install-time table entry may route an AUTO Zech dot to the pure-Zech kernel (F3); through
    gfp_dot_allreduce that kernel must exchange the classical value of its sum and encode the group's sum --
    never store a code through the 8-byte partial path."""
    from paper_cs_0404008_b200 import dist as gd
    p, n = 32749, 1_000_003
    a, b = synth.zech_codes(SEED, 0, 0, n, p - 1), synth.zech_codes(SEED, 1, 0, n, p - 1)
    want = oracle.dot_zech(p, 2, a, b)
    gfp.tune_set([{"rep": ZE, "dtype": 0, "kind": 0, "strategy": gfp.ZECH_ADD, "acc_bits": 0, "p": p, "n": n,
                   "rows": 0, "us_best": 1.0, "us_builtin": 2.0}])
    x = gd.PeerExchange()
    try:
        assert "zech_add" in gfp.plan(p, ZE, n)["kernel"]
        ga, gb = cu(a), cu(b)
        for _ in range(3):
            assert result_int(gd.dot_fused(ga, gb, p, ZE, x)) == want
        part = gfp.dot_partial(ga, gb, p, ZE)
        assert int(part.cpu()[0]) == oracle.zech_decode(p, 2, want)  # additive form: the classical value
    finally:
        torch.cuda.synchronize()
        x.close()
        gfp.tune_clear()


def test_dist_dot_on_a_side_stream():
    """dist.dot(stream=s) with s not the current stream orders partial -> combine -> finalize on s."""
    from paper_cs_0404008_b200 import dist as gd
    p, n = 2 ** 31 - 1, 1 << 22
    a, b = synth.uniform(SEED, 0, 0, n, p, np.uint32), synth.uniform(SEED, 1, 0, n, p, np.uint32)
    ga, gb = cu(a), cu(b)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    out = gd.dot(ga, gb, p, CL, stream=s)
    s.synchronize()
    assert result_int(out) == oracle.dot_classical(p, a, b)


def test_fused_allreduce_soft_timeout_reports_a_missing_peer():
    """A two-rank group whose second rank never runs (its buffer lives in this process, nobody publishes to
    it): with a soft timeout armed, rank 0's fused dot gives up after the timeout and records it instead of
    trapping -- the connectivity check bench.py runs before timing a multi-GPU group -- and the one-rank
    group's check passes."""
    from paper_cs_0404008_b200 import dist as gd
    own, _ = gfp.xchg_create()
    other, _ = gfp.xchg_create()
    try:
        spec = gfp.GfpXchg()
        spec.rank, spec.world = 0, 2
        spec.peers[0], spec.peers[1] = own, other
        gfp.xchg_soft_timeout(own, 200_000_000)  # 0.2 s
        t = cu(np.ones(1000, np.uint32))
        gfp.dot_allreduce(t, t, 65521, CL, spec)
        torch.cuda.synchronize()
        assert gfp.xchg_timed_out(own)
        gfp.xchg_soft_timeout(own, 0)
        assert not gfp.xchg_timed_out(own)  # re-arming clears the record
    finally:
        torch.cuda.synchronize()
        gfp.xchg_destroy(own)
        gfp.xchg_destroy(other)
    x = gd.PeerExchange()
    try:
        assert x.check(torch.device(DEV))
        a = synth.uniform(SEED, 0, 0, 5000, 65521, np.uint32)
        assert result_int(gd.dot_fused(cu(a), cu(a), 65521, CL, x)) == oracle.dot_classical(65521, a, a)
    finally:
        x.close()


def test_fused_allreduce_rejects_bad_groups():
    xs = gfp.GfpXchg()
    xs.rank, xs.world = 0, 0
    a = cu(np.ones(4, np.uint32))
    with pytest.raises(gfp.GfpError):
        gfp.dot_allreduce(a, a, 65521, gfp.CLASSICAL, xs)
    xs.world, xs.rank = 2, 0
    xs.peers[0] = 0
    with pytest.raises(gfp.GfpError):
        gfp.dot_allreduce(a, a, 65521, gfp.CLASSICAL, xs)


def test_fused_allreduce_buffer_reuse():
    """Exchange buffers created and destroyed repeatedly (recycled addresses) keep a correct group
    description: each new group writes its own rank / world / peer table before its first dot."""
    from paper_cs_0404008_b200 import dist as gd
    p, n = 65521, 100_003
    a, b = synth.uniform(SEED, 0, 0, n, p, np.uint32), synth.uniform(SEED, 1, 0, n, p, np.uint32)
    want = oracle.dot_classical(p, a, b)
    ga, gb = cu(a), cu(b)
    for _ in range(4):
        x = gd.PeerExchange()
        for _ in range(3):
            assert int(gd.dot_fused(ga, gb, p, gfp.CLASSICAL, x).cpu().to(torch.int64)[0]) == want
        torch.cuda.synchronize()
        x.close()


def test_non_canonical_inputs_never_fault():
    """P:49-50 preconditions are not checked on the hot path; violating them gives an unspecified value but
    must never fault (gfp.h): random 16-bit Zech codes at large and small fields, residues >= p, and
    a following canonical call is still exact."""
    rng = np.random.default_rng(7)
    n = 50_001
    raw16 = cu(rng.integers(0, 65536, n, dtype=np.uint16))
    raw32 = cu(rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32))
    for p in [101, 32749, 40009, 65521]:
        gfp.dot(raw16, raw16, p, gfp.ZECH)
        gfp.dot_batch(raw16[: 49 * 1000].view(49, 1000), raw16[:1000], p, gfp.ZECH)
        gfp.from_rep(raw16, p, gfp.ZECH)
        gfp.to_rep(raw32, p, gfp.ZECH, out=torch.empty(n, dtype=torch.uint16, device=DEV))
    gfp.dot(raw32, raw32, 65521, gfp.CLASSICAL)
    gfp.dot(raw32, raw32, 2 ** 31 - 1, gfp.MONTGOMERY)
    torch.cuda.synchronize()
    p = 32749
    a, b = synth.zech_codes(SEED, 0, 0, n, p - 1), synth.zech_codes(SEED, 1, 0, n, p - 1)
    assert int(gfp.dot(cu(a), cu(b), p, gfp.ZECH).cpu().to(torch.int64)[0]) == oracle.dot_zech(p, 2, a, b)
    A = a[: 49 * 1000].reshape(49, 1000)  # and a canonical Zech batch (the split-exponent kernel) after them
    got = gfp.dot_batch(cu(A), cu(b[:1000]), p, gfp.ZECH).cpu().numpy().astype(np.int64)
    assert got.tolist() == [oracle.dot_zech(p, 2, A[r], b[:1000]) for r in range(49)]


def test_back_to_back_dots_keep_stream_order():
    """Dots are launched with programmatic dependent launch (the next launch is staged while the previous
    dot runs); memory order must stay the stream order: a dot whose output lands inside the next dot's
    operand is seen by that dot, in plain launches and in a CUDA graph."""
    p, n = 65521, 1 << 20
    a1, b1 = cu(synth.uniform(SEED, 0, 0, n, p, np.uint32)), cu(synth.uniform(SEED, 1, 0, n, p, np.uint32))
    b2 = cu(synth.uniform(SEED, 2, 0, n, p, np.uint32))
    r1 = oracle.dot_classical(p, a1.cpu().numpy(), b1.cpu().numpy())
    x = cu(synth.uniform(SEED, 3, 0, n, p, np.uint32))
    xh = x.cpu().numpy().copy()
    xh[n // 2] = r1
    want = oracle.dot_classical(p, xh, b2.cpu().numpy())
    s = torch.cuda.Stream()
    out2 = torch.empty(1, dtype=torch.uint32, device=DEV)
    with torch.cuda.stream(s):
        for _ in range(5):
            x[n // 2] = 0
            gfp.dot(a1, b1, p, gfp.CLASSICAL, out=x[n // 2: n // 2 + 1], stream=s)
            gfp.dot(x, b2, p, gfp.CLASSICAL, out=out2, stream=s)
            s.synchronize()
            assert int(out2.cpu().to(torch.int64)[0]) == want
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                gfp.dot(a1, b1, p, gfp.CLASSICAL, out=x[n // 2: n // 2 + 1], stream=s)
                gfp.dot(x, b2, p, gfp.CLASSICAL, out=out2, stream=s)
    for _ in range(5):
        x[n // 2] = 0
        out2.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert int(out2.cpu().to(torch.int64)[0]) == want


def test_pdl_chains_keep_stream_order():
    """Conversions, dots and batches are all launched with programmatic dependent launch (early signal,
    first chunk prefetched into L2 before the wait): every producer -> consumer chain in one stream must
    still see the producer's writes -- conversion -> dot, in-place to/from conversion, batch output as a
    dot operand, a dot result inside the next batch's x -- in plain launches and in a CUDA graph."""
    p = 2 ** 31 - 1
    n = (1 << 20) + 3
    a = cu(synth.uniform(SEED, 0, 0, n, p, np.uint32))
    b = cu(synth.uniform(SEED, 1, 0, n, p, np.uint32))
    want_m = oracle.to_mont(p, oracle.dot_classical(p, a.cpu().numpy(), b.cpu().numpy()))
    q, rows, m = 65521, 4099, 512
    A = cu(synth.uniform(SEED, 2, 0, rows * m, q, np.uint16).reshape(rows, m))
    xb = cu(synth.uniform(SEED, 3, 0, m, q, np.uint16))
    z = cu(synth.uniform(SEED, 4, 0, rows, q, np.uint16))
    u, v = cu(synth.uniform(SEED, 5, 0, 1000, q, np.uint16)), cu(synth.uniform(SEED, 6, 0, 1000, q, np.uint16))
    r_uv = oracle.dot_classical(q, u.cpu().numpy(), v.cpu().numpy())
    xh = xb.cpu().numpy().copy()
    xh[7] = r_uv
    y_want = oracle.dot_batch_classical(q, A.cpu().numpy(), xh).astype(np.uint16)
    want_yz = oracle.dot_classical(q, y_want, z.cpu().numpy())

    am, bm = torch.empty_like(a), torch.empty_like(b)
    t = torch.empty_like(a)
    y = torch.empty(rows, dtype=torch.uint16, device=DEV)
    out_m = torch.empty(1, dtype=torch.uint32, device=DEV)
    out_yz = torch.empty(1, dtype=torch.uint16, device=DEV)
    s = torch.cuda.Stream()

    def chain():
        gfp.to_rep(a, p, gfp.MONTGOMERY, out=am, stream=s)
        gfp.to_rep(b, p, gfp.MONTGOMERY, out=bm, stream=s)
        gfp.dot(am, bm, p, gfp.MONTGOMERY, out=out_m, stream=s)
        t.copy_(a)
        gfp.to_rep(t, p, gfp.MONTGOMERY, out=t, stream=s)
        gfp.from_rep(t, p, gfp.MONTGOMERY, out=t, stream=s)
        gfp.dot(u, v, q, gfp.CLASSICAL, out=xb[7:8], stream=s)
        gfp.dot_batch(A, xb, q, gfp.CLASSICAL, out=y, stream=s)
        gfp.dot(y, z, q, gfp.CLASSICAL, out=out_yz, stream=s)

    def check():
        assert int(out_m.cpu().to(torch.int64)[0]) == want_m
        assert torch.equal(t, a)
        assert np.array_equal(y.cpu().numpy(), y_want)
        assert int(out_yz.cpu().to(torch.int64)[0]) == want_yz

    def scrub():
        for w in (am, bm, t, y, out_m, out_yz):
            w.zero_()
        xb[7] = 0

    with torch.cuda.stream(s):
        for _ in range(3):
            scrub()
            chain()
            s.synchronize()
            check()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            chain()
    for _ in range(5):
        scrub()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        check()

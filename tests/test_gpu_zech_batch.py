"""GPU parity of the Zech matrix-vector product (gfp_dot_batch over Zech codes, sec. 2.4): the split-exponent
kernel (batch_zsplit_kernel: g^c = H[(c-1) >> 8] L[(c-1) & 255] from bank-replicated tables, the zero code through
a free H row for p <= 65281 or a flag page above), the single-lookup decode kernel (batch_zech_kernel, rows too
long for the split kernel's bound) and the index-add fallback (batch_kernel<Zech>: unaligned rows or an explicit
lanes_per_row), each row compared with the oracle's Zech dot (independent decoding by repeated multiplication,
one 128-bit remainder per term, brute-force discrete-log encoding)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
ZE = gfp.ZECH
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def rows_oracle(p, A, x, rows_idx):
    g = oracle.primitive_root(p)
    return np.array([oracle.dot_zech(p, g, A[r], x) for r in rows_idx], np.int64)


@pytest.mark.parametrize("p", [2, 3, 5, 101, 257, 2903, 32749, 40009, 65269, 65287, 65521])
@pytest.mark.parametrize("shape", [(1, 1), (7, 8), (33, 255), (65, 4096), (3, 4103), (130, 777), (2, 0), (257, 768),
                                   (5, 16), (4099, 512)])
def test_zech_batch_shapes(p, shape):
    rows, n = shape
    seed = synth.BASE_SEED + p
    A = synth.zech_codes(seed, 2, 0, rows * n, p - 1).reshape(rows, n)
    x = synth.zech_codes(seed, 3, 0, n, p - 1)
    got = gfp.dot_batch(cu(A), cu(x), p, ZE).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, rows_oracle(p, A, x, range(rows))), (p, shape)


@pytest.mark.parametrize("p", [32749, 65269, 65287, 65521])
def test_zech_batch_worst_case_and_zeros(p):
    """Rows of the code of -1 (value p - 1: the largest products), rows of zeros, x of -1 / of zeros."""
    g = oracle.primitive_root(p)
    m1 = oracle.zech_encode(p, g, p - 1)
    rows, n = 96, 4096
    A = np.full((rows, n), m1, np.uint16)
    A[32:64] = 0
    A[64:] = synth.zech_codes(synth.BASE_SEED, 2, 0, 32 * n, p - 1).reshape(32, n)
    for x in (np.full(n, m1, np.uint16), np.zeros(n, np.uint16), synth.zech_codes(synth.BASE_SEED, 3, 0, n, p - 1)):
        got = gfp.dot_batch(cu(A), cu(x), p, ZE).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, rows_oracle(p, A, x, range(rows)))
    # closed form: (p-1)^2 n = n (mod p) -> the code of n mod p
    got = gfp.dot_batch(cu(A[:1]), cu(np.full(n, m1, np.uint16)), p, ZE).cpu().numpy()
    assert int(got[0]) == oracle.zech_encode(p, g, n % p)


@pytest.mark.parametrize("p", [32749, 65521])
def test_zech_batch_padded_unaligned_and_explicit_lanes(p):
    """lda padding (decode kernel), an odd lda and a misaligned x (index-add fallback), lanes_per_row 8 / 32."""
    rows, n = 77, 1000
    A = synth.zech_codes(synth.BASE_SEED, 2, 0, rows * 1024, p - 1).reshape(rows, 1024)
    x = synth.zech_codes(synth.BASE_SEED, 3, 0, n + 1, p - 1)
    want = rows_oracle(p, A[:, :n], x[:n], range(rows))
    dA = cu(A)
    got = gfp.dot_batch(dA, cu(x[:n]), p, ZE, n=n).cpu().numpy().astype(np.int64)  # lda = 1024
    assert np.array_equal(got, want)
    flat = cu(A.reshape(-1)[: (rows - 1) * 1001 + n])
    Aodd = np.stack([A.reshape(-1)[r * 1001: r * 1001 + n] for r in range(rows)])
    want_odd = rows_oracle(p, Aodd, x[:n], range(rows))
    got = gfp.dot_batch(flat, cu(x[:n]), p, ZE, rows=rows, n=n, lda=1001).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want_odd)
    xd = cu(x)[1:]  # 2-byte aligned, not 16: the fallback kernel
    got = gfp.dot_batch(dA, xd, p, ZE, n=n).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, rows_oracle(p, A[:, :n], x[1:], range(rows)))
    for lanes in (8, 32):
        got = gfp.dot_batch_ex(dA, cu(x[:n]), p, ZE, n=n, lanes_per_row=lanes).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("p", [32749, 65521])
def test_zech_batch_full_size_sampled_rows(p):
    """The bench shape (65536 x 4096, bench.py C5-zech lines): 512 rows spread over the matrix against the oracle."""
    rows, n = 65536, 4096
    A = synth.zech_codes(synth.BASE_SEED + (9 if p == 32749 else 10), 2, 0, rows * n, p - 1).reshape(rows, n)
    x = synth.zech_codes(synth.BASE_SEED + (9 if p == 32749 else 10), 3, 0, n, p - 1)
    got = gfp.dot_batch(cu(A), cu(x), p, ZE).cpu().numpy().astype(np.int64)
    idx = np.unique(np.concatenate([np.arange(0, rows, 131), np.arange(rows - 40, rows)]))
    assert np.array_equal(got[idx], rows_oracle(p, A, x, idx))


@pytest.mark.parametrize("p", [2, 3, 5, 101, 257])
def test_zech_batch_every_product_exhaustive(p):
    """Every pair of codes (i, j), zero included: a batch of rows [i, i, ..., i] (n = 8, one 16-byte vector --
    the decode kernel's vector path) against x = [j] * 8, so row i is 8 g^i g^j; compared with the oracle."""
    q = p - 1
    n = 8
    A = np.repeat(np.arange(q + 1, dtype=np.uint16), n).reshape(q + 1, n)
    g = oracle.primitive_root(p)
    dA = cu(A)
    for j in range(q + 1):
        x = np.full(n, j, np.uint16)
        got = gfp.dot_batch(dA, cu(x), p, ZE).cpu().numpy().astype(np.int64)
        want = np.array([oracle.dot_zech(p, g, A[i], x) for i in range(q + 1)], np.int64)
        assert np.array_equal(got, want), (p, j)


@pytest.mark.parametrize("p", [65269, 65287, 65521])
def test_zech_batch_zero_row_codes(p):
    """The codes whose e = c - 1 sits in the split kernel's last H row (e >> 8 = 255: zero-code row at p <= 65281,
    shared with the zero code's flag page above) and the codes around every 256 boundary, against the oracle."""
    g = oracle.primitive_root(p)
    q = p - 1
    special = [0, 1, 2, 255, 256, 257, q - 1, q] + [c for c in range(0xFF00, q + 1, 7)]
    special = np.array(sorted(set(c for c in special if 0 <= c <= q)), np.uint16)
    n = 4096
    A = np.resize(special, (64, n)).astype(np.uint16)
    A[1::2] = np.roll(A[1::2], 3, axis=1)
    x = np.resize(special[::-1], n).astype(np.uint16)
    got = gfp.dot_batch(cu(A), cu(x), p, ZE).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, rows_oracle(p, A, x, range(64)))


def test_zech_batch_rows_past_the_split_bound():
    """Rows too long for the split kernel's bound n (p-1)^3 < 2^64 at GF(65521) (n > 65536) still match the oracle
    (the other Zech batch kernels serve them)."""
    p, rows, n = 65521, 3, 70000
    A = synth.zech_codes(synth.BASE_SEED, 2, 0, rows * n, p - 1).reshape(rows, n)
    x = synth.zech_codes(synth.BASE_SEED, 3, 0, n, p - 1)
    got = gfp.dot_batch(cu(A), cu(x), p, ZE).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, rows_oracle(p, A, x, range(rows)))


@pytest.mark.parametrize("block", range(4))
def test_zech_batch_fuzz_aligned_rows(block):
    """Random shapes whose rows are 16-byte aligned (the split-exponent kernel's path: lda a multiple of 8), random
    primes on both sides of 65281, zero-heavy and zero-free codes; every row against the oracle."""
    rng = np.random.default_rng(9100 + block)
    primes = [3, 7, 257, 1009, 7919, 32749, 40009, 65267, 65269, 65287, 65293, 65519, 65521]
    for case in range(12):
        p = int(rng.choice(primes))
        rows = int(rng.integers(1, 200))
        n = int(rng.integers(8, 9000))
        lda = (n + 7) // 8 * 8 + 8 * int(rng.integers(0, 3))
        seed = synth.BASE_SEED + 9100 + 100 * block + case
        A = synth.zech_codes(seed, 2, 0, rows * lda, p - 1).reshape(rows, lda)
        x = synth.zech_codes(seed, 3, 0, n, p - 1)
        if case % 3 == 1:
            A[:, ::3] = 0  # many zero codes
        elif case % 3 == 2:
            A[A == 0] = p - 1  # none
        got = gfp.dot_batch(cu(A)[:, :n], cu(x), p, ZE).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, rows_oracle(p, A[:, :n], x, range(rows))), (p, rows, n, lda)

"""GPU parity of the pure-Zech dot (gfp_dot_ex with GFP_STRAT_ZECH_ADD): every product
an index addition and every sum a Zech addition through the t_plus1 table (sec. 2.4, Table 1
P:150-171).  The result is a unique field element, so it must equal, bit for bit, both the oracle's
Table-1 accumulation (oracle_dot_zech_tplus1) and its integer-decoded dot (oracle_dot_zech).
Covers small (2 qbar < 2^16) and large table layouts, n = 0 / 1 / ragged / many tiles, unaligned and
non-co-aligned operands, zero-heavy inputs, sums that cancel to zero, and the full C4 size.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
ZE = gfp.ZECH
DEV = "cuda:0"
SEED = synth.BASE_SEED + 303


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def zadd(a, b, p):
    return int(gfp.dot_ex(a, b, p, ZE, strategy=gfp.ZECH_ADD).cpu().to(torch.int64)[0])


@pytest.mark.parametrize("p", [2, 3, 5, 7, 101, 1009, 32749, 32771, 40009, 65521])
def test_zech_add_random(p):
    g = oracle.primitive_root(p)
    for n in [0, 1, 2, 7, 8, 9, 4095, 4096, 4097, 100_003, 1_000_037]:
        a = synth.zech_codes(SEED + n, 0, 0, n, p - 1)
        b = synth.zech_codes(SEED + n, 1, 0, n, p - 1)
        want = oracle.dot_zech(p, g, a, b)
        if n <= 100_003:
            assert oracle.dot_zech_tplus1(p, g, a, b) == want
        assert zadd(cu(a), cu(b), p) == want, (p, n)


@pytest.mark.parametrize("p", [32749, 65521])
def test_zech_add_unaligned_and_offsets(p):
    g = oracle.primitive_root(p)
    n = 200_017
    a = cu(synth.zech_codes(SEED, 0, 0, n + 16, p - 1))
    b = cu(synth.zech_codes(SEED, 1, 0, n + 16, p - 1))
    for oa, ob in [(0, 0), (1, 1), (3, 3), (7, 7), (1, 2), (0, 5)]:
        x, y = a[oa:oa + n], b[ob:ob + n]
        want = oracle.dot_zech(p, g, x.cpu().numpy(), y.cpu().numpy())
        assert zadd(x, y, p) == want, (oa, ob)


@pytest.mark.parametrize("p", [3, 101, 32749, 65521])
def test_zech_add_degenerate(p):
    """all-zero, all-ones of length p (sum p = 0), cancelling pairs (x + (-x)), a single nonzero
    term among zeros, and per-accumulator cancellation at every position of a 16-byte vector."""
    qbar = p - 1
    n = 3 * p + 5
    z = np.zeros(n, np.uint16)
    assert zadd(cu(z), cu(z), p) == 0
    ones = np.full(p, qbar, np.uint16)  # code qbar = 1
    assert zadd(cu(ones), cu(ones), p) == 0
    one = np.zeros(n, np.uint16)
    one[n // 2] = 1  # g
    assert zadd(cu(one), cu(np.full(n, qbar, np.uint16)), p) == 1
    # x . 1 + x . (-1) for every x in a block: cancels to 0 lane by lane
    m = 4096
    x = synth.zech_codes(SEED, 5, 0, m, qbar)
    a = np.concatenate([x, x])
    b = np.concatenate([np.full(m, qbar, np.uint16), np.full(m, qbar // 2 if p > 2 else qbar, np.uint16)])
    assert zadd(cu(a), cu(b), p) == 0
    # sum = 0 then one more term: the zero state must absorb the next value
    a2 = np.concatenate([a, np.array([3 % p if p > 3 else 1], np.uint16)])
    b2 = np.concatenate([b, np.array([qbar], np.uint16)])
    assert zadd(cu(a2), cu(b2), p) == oracle.dot_zech(p, oracle.primitive_root(p), a2, b2)


def test_zech_add_c4_full_size():
    """BASELINE configs[3] shape (p = 32749, n = 2^26, 10% zeros), the bench's C4-zech_add line: the whole
    vector against the oracle directly -- its integer-accumulation Zech dot and, step by step in Table 1's
    order, its own pure-Zech accumulation (oracle_dot_zech_tplus1) -- and against the default plan."""
    p, n = 32749, 2 ** 26
    a = synth.zech_codes(synth.BASE_SEED + 3, 0, 0, n, p - 1)
    b = synth.zech_codes(synth.BASE_SEED + 3, 1, 0, n, p - 1)
    ga, gb = cu(a), cu(b)
    full = zadd(ga, gb, p)
    assert full == oracle.dot_zech(p, 2, a, b)
    assert full == oracle.dot_zech_tplus1(p, 2, a, b)
    assert full == int(gfp.dot(ga, gb, p, ZE).cpu().to(torch.int64)[0])


def test_zech_add_graph_capture_and_repeat():
    """Self-resetting workspace: repeated launches and CUDA-graph replay give the same code."""
    p, n = 32749, 1 << 20
    a = cu(synth.zech_codes(SEED, 0, 0, n, p - 1))
    b = cu(synth.zech_codes(SEED, 1, 0, n, p - 1))
    want = zadd(a, b, p)
    out = torch.empty(1, dtype=torch.uint16, device=DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gfp.dot_ex(a, b, p, ZE, strategy=gfp.ZECH_ADD, out=out)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gfp.dot_ex(a, b, p, ZE, strategy=gfp.ZECH_ADD, out=out)
    for _ in range(5):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert int(out.cpu().to(torch.int64)[0]) == want


def test_table_sizes_in_any_order():
    """Shared-memory opt-in regression: the same kernel launched with a large table, then smaller ones,
    then the large one again (Zech at several primes, both accumulations) must keep launching."""
    n = 100_003
    for p in [65521, 32771, 40009, 65521, 32749, 65521]:
        g = oracle.primitive_root(p)
        a = synth.zech_codes(SEED, 0, 0, n, p - 1)
        b = synth.zech_codes(SEED, 1, 0, n, p - 1)
        want = oracle.dot_zech(p, g, a, b)
        assert zadd(cu(a), cu(b), p) == want, p
        assert int(gfp.dot(cu(a), cu(b), p, ZE).cpu().to(torch.int64)[0]) == want, p


@pytest.mark.parametrize("p", [3, 101, 32749, 40009, 65521])
def test_zech_add_non_canonical_codes_stay_in_bounds(p):
    """Preconditions are not checked on the hot path, but non-canonical codes (> q-1) must not
    fault (gfp.h): every lookup index is clamped into the table.  The result is unspecified; the next
    call on canonical data must still be exact (no sticky error, workspace intact)."""
    n = 100_003
    rng = np.random.default_rng(p)
    a = rng.integers(0, 65536, n, dtype=np.uint16)
    b = rng.integers(0, 65536, n, dtype=np.uint16)
    zadd(cu(a), cu(b), p)
    torch.cuda.synchronize()
    ca = synth.zech_codes(SEED, 0, 0, n, p - 1)
    cb = synth.zech_codes(SEED, 1, 0, n, p - 1)
    assert zadd(cu(ca), cu(cb), p) == oracle.dot_zech(p, oracle.primitive_root(p), ca, cb)

"""GPU parity of the centered representation (sec. 3.2.2): residues
stored between -(p-1)/2 and (p-1)/2 as int16 / int32 / binary64, dotted with the doubled blocks
lambda_c h^2 + h < 2^(m-1) (2^53 for binary64), bit-exact against the CPU oracle on random and
worst-case-magnitude inputs, at block boundaries, unaligned, batched, and at BASELINE configs[1]'s size."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
CE = gfp.CENTERED
DEV = "cuda:0"
SEED = synth.BASE_SEED + 505


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def centered_inputs(seed, stream, n, p, np_dt):
    r = synth.uniform(seed, stream, 0, n, p, np.uint64).astype(np.int64)
    h = (p - 1) // 2
    c = np.where(r > h, r - p, r)
    return c.astype(np_dt)


def value(t):
    v = t.cpu()[0].item()
    return v


CASES = [(np.int16, [3, 101, 2897, 32749, 46337, 65521]),
         (np.int32, [65537, 2 ** 31 - 1, 3037000493, 4294967291]),
         (np.float64, [3, 32749, 67108859, 94906249, 189812507])]


@pytest.mark.parametrize("np_dt,primes", CASES)
def test_centered_random(np_dt, primes):
    for p in primes:
        for n in [0, 1, 2, 7, 8, 9, 513, 100_003, 1_000_003]:
            a, b = centered_inputs(SEED + n, 0, n, p, np_dt), centered_inputs(SEED + n, 1, n, p, np_dt)
            want = oracle.dot_centered(p, a, b)
            for strat in (gfp.AUTO, gfp.DELAYED, gfp.BLOCKED):
                try:
                    got = value(gfp.dot_ex(cu(a), cu(b), p, CE, strategy=strat))
                except gfp.GfpError as e:
                    assert e.status == 3 and strat == gfp.DELAYED  # Eq. (1) bound for delayed
                    continue
                assert got == want, (p, n, strat)
                if np_dt == np.float64:
                    assert math.copysign(1.0, got) == 1.0 or got != 0


@pytest.mark.parametrize("np_dt,p", [(np.int16, 65521), (np.int32, 4294967291), (np.int32, 2 ** 31 - 1),
                                     (np.float64, 67108859), (np.float64, 189812507)])
def test_centered_worst_case_magnitudes(np_dt, p):
    """all +h / mixed-sign +-h vectors: every product is h^2 in magnitude, so a block of lambda_c
    products reaches the accumulator bound; lengths straddle the block boundary."""
    h = (p - 1) // 2
    k = gfp.query(p, CE, torch.float64 if np_dt == np.float64 else None)["k"] if np_dt == np.float64 else \
        gfp.query(p, CE, torch.int16 if np_dt == np.int16 else torch.int32)["k"]
    lens = sorted({1, 2, 3, 255, 256, 257, 100_001} | ({k - 1, k, k + 1, 3 * k + 2} if k < 10 ** 5 else set()))
    for n in lens:
        if n <= 0:
            continue
        a = np.full(n, h, np_dt)
        signs = np.where(np.arange(n) % 3 == 0, -1, 1)
        for b in (np.full(n, h, np_dt), (signs * h).astype(np_dt), np.full(n, -h, np_dt)):
            want = oracle.dot_centered(p, a, b)
            for strat in (gfp.AUTO, gfp.BLOCKED):
                assert value(gfp.dot_ex(cu(a), cu(b), p, CE, strategy=strat)) == want, (p, n, strat)


def test_centered_conversions_roundtrip():
    for p, dt in [(65521, torch.int16), (32749, torch.int32), (4294967291, torch.int32), (67108859, torch.float64)]:
        n = 100_003
        r = synth.uniform(SEED, 7, 0, n, p, np.uint32)
        c = gfp.to_rep(cu(r), p, CE, out=torch.empty(n, dtype=dt, device=DEV))
        want = np.array([oracle.to_centered(p, int(v)) for v in r[:2000]])
        assert np.array_equal(c.cpu().numpy()[:2000].astype(np.int64), want)
        back = gfp.from_rep(c, p, CE)
        assert np.array_equal(back.cpu().numpy(), r)


def test_centered_unaligned_and_batch():
    p = 32749
    n = 200_017
    a = cu(centered_inputs(SEED, 0, n + 16, p, np.int16))
    b = cu(centered_inputs(SEED, 1, n + 16, p, np.int16))
    for oa, ob in [(1, 1), (3, 3), (1, 2), (0, 5)]:
        x, y = a[oa:oa + n], b[ob:ob + n]
        assert value(gfp.dot(x, y, p, CE)) == oracle.dot_centered(p, x.cpu().numpy(), y.cpu().numpy())
    for p, np_dt in [(65521, np.int16), (4294967291, np.int32), (67108859, np.float64)]:
        rows, m = 300, 777
        A = centered_inputs(SEED, 2, rows * m, p, np_dt).reshape(rows, m)
        xv = centered_inputs(SEED, 3, m, p, np_dt)
        got = gfp.dot_batch(cu(A), cu(xv), p, CE).cpu().numpy()
        want = [oracle.dot_centered(p, A[r], xv) for r in range(rows)]
        assert [v.item() for v in got] == want, p


def test_centered_c2_full_size():
    """BASELINE configs[1] (GF(67108859), n = 10^7) in the centered binary64 representation: k = 8
    instead of 2, same field element as the fp64 representation's dot."""
    p, n = 67108859, 10 ** 7
    a = synth.uniform(synth.BASE_SEED + 1, 0, 0, n, p, np.float64)
    b = synth.uniform(synth.BASE_SEED + 1, 1, 0, n, p, np.float64)
    h = (p - 1) // 2
    ac, bc = np.where(a > h, a - p, a), np.where(b > h, b - p, b)
    got = value(gfp.dot(cu(ac), cu(bc), p, CE))
    assert got == oracle.dot_centered(p, ac, bc)
    assert (int(got) % p) == int(oracle.dot_fp64(p, a, b))
    assert gfp.plan(p, CE, n, dtype=torch.float64)["block"] == 8


def test_centered_storage_type_checks():
    a = cu(np.zeros(10, np.uint16))
    with pytest.raises(TypeError):
        gfp.dot(a, a, 65521, CE)
    s = cu(np.zeros(10, np.int16))
    with pytest.raises(TypeError):
        gfp.dot(s, s, 65521, gfp.CLASSICAL)

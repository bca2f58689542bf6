"""Randomised GPU parity (seeded, reproducible): many (representation, storage, prime, length, offset,
strategy) combinations drawn at random and each compared bit-exactly with the CPU oracle -- dots at
misaligned offsets inside larger buffers, batches with padded leading dimensions, and the explicit-strategy
and pure-Zech paths.  It complements the structured sweeps in test_gpu_parity.py with breadth: every
draw takes a fresh plan (grid, waves, prefetch, packed combine, head / tail split)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
DEV = "cuda:0"
# GFP_FUZZ_SEED shifts every draw (default 0: the committed, reproducible draws); e.g. GFP_FUZZ_SEED=7 for a fresh set
SHIFT = int(__import__("os").environ.get("GFP_FUZZ_SEED", "0")) * 1_000_003

PRIMES = {
    ("classical", np.uint16): [2, 3, 5, 251, 257, 4093, 32749, 40009, 65521],
    ("classical", np.uint32): [3, 65537, 1000000007, 2147483647, 3037000493, 4294967291],
    ("montgomery", np.uint32): [3, 40499, 65537, 1000000007, 2147483647, 2654435761],
    ("fp64", np.float64): [3, 65521, 67108859, 94906249],
    ("zech", np.uint16): [3, 5, 101, 32749, 40009, 65521],
    ("centered", np.int16): [3, 101, 32749, 65521],
    ("centered", np.int32): [65537, 2147483647, 4294967291],
    ("centered", np.float64): [3, 67108859, 189812507],
}
REP = {"classical": gfp.CLASSICAL, "montgomery": gfp.MONTGOMERY, "fp64": gfp.FP64, "zech": gfp.ZECH,
       "centered": gfp.CENTERED}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _inputs(kind, np_dt, p, n, seed, stream):
    if kind == "zech":
        return synth.zech_codes(seed, stream, 0, n, p - 1)
    if kind == "centered":
        r = synth.uniform(seed, stream, 0, n, p, np.uint64).astype(np.int64)
        h = (p - 1) // 2
        return np.where(r > h, r - p, r).astype(np_dt)
    return synth.uniform(seed, stream, 0, n, p, np_dt)


def _value(t):
    v = t.cpu()
    return v[0].item() if v.dtype == torch.float64 else int(v.to(torch.int64)[0])


def _want(kind, p, a, b):
    if kind == "zech":
        return oracle.dot_zech(p, oracle.primitive_root(p), a, b)
    return oracle.dot(p, REP[kind], a, b)


def _draw_n(rng):
    r = rng.random()
    if r < 0.1:
        return int(rng.integers(0, 17))
    if r < 0.6:
        return int(rng.integers(17, 5000))
    if r < 0.95:
        return int(rng.integers(5000, 400_000))
    return int(rng.integers(400_000, 3_000_000))


@pytest.mark.parametrize("block", range(6))
def test_random_dots_at_random_offsets(block):
    rng = np.random.default_rng(20260 + block + SHIFT)
    keys = list(PRIMES)
    for case in range(120):
        kind, np_dt = keys[rng.integers(len(keys))]
        p = int(rng.choice(PRIMES[(kind, np_dt)]))
        n = _draw_n(rng)
        off_a, off_b = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        seed = synth.BASE_SEED + 1000 * block + case
        a = _inputs(kind, np_dt, p, n + off_a, seed, 0)
        b = _inputs(kind, np_dt, p, n + off_b, seed, 1)
        ga, gb = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
        x, y = ga[off_a:off_a + n], gb[off_b:off_b + n]  # views: misaligned starts, ragged tails
        want = _want(kind, p, a[off_a:off_a + n], b[off_b:off_b + n])
        got = _value(gfp.dot(x, y, p, REP[kind]))
        assert got == want, (kind, np_dt, p, n, off_a, off_b)
        if kind == "zech" and p > 2 and rng.random() < 0.5:  # the pure-Zech accumulation, same element
            got = _value(gfp.dot_ex(x, y, p, gfp.ZECH, strategy=gfp.ZECH_ADD))
            assert got == want, ("zech_add", p, n, off_a, off_b)
        if kind == "classical" and rng.random() < 0.5:  # one of the paper's sec.-3 strategies, if admissible
            strat = int(rng.choice([gfp.DELAYED, gfp.BLOCKED, gfp.OVERFLOW, gfp.HYBRID, gfp.CARRY]))
            m = int(rng.choice([32, 64]))
            try:
                got = _value(gfp.dot_ex(x, y, p, gfp.CLASSICAL, strategy=strat, acc_bits=m))
            except gfp.GfpError as e:
                assert e.status in (3, 4)  # bound / unsupported for this (p, n, m)
            else:
                assert got == want, ("strategy", strat, m, p, n)


@pytest.mark.parametrize("block", range(3))
def test_random_batches_with_padded_rows(block):
    rng = np.random.default_rng(4242 + block + SHIFT)
    kinds = [("classical", np.uint16), ("classical", np.uint32), ("montgomery", np.uint32), ("fp64", np.float64),
             ("zech", np.uint16), ("centered", np.int32)]
    for case in range(25):
        kind, np_dt = kinds[rng.integers(len(kinds))]
        p = int(rng.choice(PRIMES[(kind, np_dt)]))
        rows = int(rng.integers(1, 3000))
        n = int(rng.integers(1, 3000))
        lda = n + int(rng.integers(0, 9))
        seed = synth.BASE_SEED + 7000 + 100 * block + case
        A = _inputs(kind, np_dt, p, rows * lda, seed, 2).reshape(rows, lda)
        x = _inputs(kind, np_dt, p, n, seed, 3)
        got = gfp.dot_batch(torch.from_numpy(A).to(DEV)[:, :n], torch.from_numpy(x).to(DEV), p, REP[kind]).cpu()
        got = got.numpy() if got.dtype == torch.float64 else got.to(torch.int64).numpy()
        for r in rng.choice(rows, size=min(rows, 12), replace=False):  # sampled rows, each against the oracle
            assert got[r] == _want(kind, p, A[r, :n], x), (kind, np_dt, p, rows, n, lda, int(r))


@pytest.mark.parametrize("block", range(3))
def test_random_batches_explicit_strategies_and_lanes(block):
    """gfp_dot_batch_ex with random sec.-3 strategies, accumulator widths and lanes per row (1 / 8 / 32 / the
    library's choice) over classical u16 / u32 rows of random length and padding, against the oracle."""
    rng = np.random.default_rng(777 + block + SHIFT)
    for case in range(30):
        np_dt = np.uint16 if rng.random() < 0.5 else np.uint32
        p = int(rng.choice(PRIMES[("classical", np_dt)]))
        rows, n = int(rng.integers(1, 700)), int(rng.integers(1, 2500))
        lda = n + int(rng.integers(0, 9))
        seed = synth.BASE_SEED + 9000 + 100 * block + case
        A = _inputs("classical", np_dt, p, rows * lda, seed, 2).reshape(rows, lda)
        if rng.random() < 0.3:
            A[:] = p - 1  # worst-case magnitudes
        x = _inputs("classical", np_dt, p, n, seed, 3)
        strat = int(rng.choice([gfp.AUTO, gfp.DELAYED, gfp.BLOCKED, gfp.OVERFLOW, gfp.HYBRID, gfp.CARRY]))
        m = int(rng.choice([0, 32, 64])) if strat != gfp.AUTO else 0
        lanes = int(rng.choice([0, 1, 8, 32]))
        try:
            got = gfp.dot_batch_ex(torch.from_numpy(A).to(DEV)[:, :n], torch.from_numpy(x).to(DEV), p, gfp.CLASSICAL,
                                   strategy=strat, acc_bits=m, lanes_per_row=lanes).cpu().to(torch.int64).numpy()
        except gfp.GfpError as e:
            assert e.status in (3, 4), (p, n, strat, m, lanes)  # bound / unsupported for this (p, n, m)
            continue
        want = oracle.dot_batch_classical(p, A[:, :n].copy(), x).astype(np.int64)
        assert np.array_equal(got, want), (np_dt, p, rows, n, lda, strat, m, lanes)

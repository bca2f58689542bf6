"""GPU parity of the paper's explicit accumulation strategies (gfp_dot_ex / gfp_dot_batch_ex):
delayed (sec. 3.1), blocked (3.2), overflow-on-demand (3.3), hybrid (3.4), each with 32- and 64-bit
accumulators, overflow-Montgomery (3.3) and the fp64 delayed/blocked variants -- bit-exact
against the CPU oracle on random and worst-case (all p-1: the accumulator wraps on almost every
product near the bound) inputs, at k-boundary lengths.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
CL, MO, FP = gfp.CLASSICAL, gfp.MONTGOMERY, gfp.FP64
DEV = "cuda:0"
SEED = synth.BASE_SEED + 77
STRATS = [gfp.DELAYED, gfp.BLOCKED, gfp.OVERFLOW, gfp.HYBRID, gfp.CARRY]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def as_int(t):
    return int(t.cpu().to(torch.int64)[0])


def admissible(p, n, dtype, strat, m):
    try:
        return gfp.plan(p, CL, n, dtype=dtype, strategy=strat, acc_bits=m)
    except gfp.GfpError as e:
        assert e.status in (3, 4)  # GFP_E_BOUND / GFP_E_UNSUPPORTED
        return None


@pytest.mark.parametrize("p", [2, 3, 7, 101, 1009, 2887, 2897, 2903, 32749, 40009, 46337, 65521])
def test_classical_strategies_small_primes(p):
    for dt_np, dt_t in [(np.uint16, torch.uint16), (np.uint32, torch.uint32)]:
        for m in (32, 64):
            k = gfp.plan(p, CL, 512, dtype=dt_t, strategy=gfp.BLOCKED, acc_bits=m)["block"]
            dims = sorted({0, 1, 2, 511, 512, 513, 10 ** 4, 10 ** 6 + 3} |
                          ({max(k - 1, 0), k, k + 1, 3 * k + 2} if k < 10 ** 5 else set()))
            for strat in STRATS:
                for n in dims:
                    if admissible(p, n, dt_t, strat, m) is None:
                        continue
                    a = synth.uniform(SEED + n, 0, 0, n, p, dt_np)
                    b = synth.uniform(SEED + n, 1, 0, n, p, dt_np)
                    got = as_int(gfp.dot_ex(cu(a), cu(b), p, CL, strategy=strat, acc_bits=m))
                    assert got == oracle.dot_classical(p, a, b), (p, dt_np, m, strat, n)
                n = 100_003
                if admissible(p, n, dt_t, strat, m) is not None:
                    w = np.full(n, p - 1, dt_np)
                    got = as_int(gfp.dot_ex(cu(w), cu(w), p, CL, strategy=strat, acc_bits=m))
                    assert got == n % p, (p, m, strat)


@pytest.mark.parametrize("p", [65537, 2 ** 31 - 1, 3037000493, 4294967291])
def test_classical_strategies_large_primes_u64(p):
    for strat in (gfp.BLOCKED, gfp.OVERFLOW, gfp.HYBRID, gfp.CARRY):
        for n in [1, 2, 3, 4, 5, 1000, 100_003]:
            a = synth.uniform(SEED, 0, 0, n, p, np.uint32)
            b = synth.uniform(SEED, 1, 0, n, p, np.uint32)
            got = as_int(gfp.dot_ex(cu(a), cu(b), p, CL, strategy=strat, acc_bits=64))
            assert got == oracle.dot_classical(p, a, b), (p, strat, n)
        w = np.full(1_000_001, p - 1, np.uint32)  # (p-1)^2 ~ 2^64: a wrap on nearly every add
        assert as_int(gfp.dot_ex(cu(w), cu(w), p, CL, strategy=strat, acc_bits=64)) == 1_000_001 % p


@pytest.mark.parametrize("p", [3, 101, 40499, 65521, 2 ** 31 - 1, 2654435761])
def test_montgomery_overflow_variant(p):
    for n in [0, 1, 2, 3, 5, 513, 100_003]:
        a = synth.uniform(SEED, 0, 0, n, p, np.uint32)
        b = synth.uniform(SEED, 1, 0, n, p, np.uint32)
        am, bm = gfp.to_rep(cu(a), p, MO), gfp.to_rep(cu(b), p, MO)
        want = oracle.to_mont(p, oracle.dot_classical(p, a, b))
        assert as_int(gfp.dot_ex(am, bm, p, MO, strategy=gfp.OVERFLOW)) == want, (p, n)
        assert as_int(gfp.dot_ex(am, bm, p, MO, strategy=gfp.BLOCKED)) == want, (p, n)
        assert as_int(gfp.dot_ex(am, bm, p, MO, strategy=gfp.CARRY)) == want, (p, n)
    w = gfp.to_rep(cu(np.full(300_001, p - 1, np.uint32)), p, MO)
    assert as_int(gfp.dot_ex(w, w, p, MO, strategy=gfp.OVERFLOW)) == oracle.to_mont(p, 300_001 % p)
    assert as_int(gfp.dot_ex(w, w, p, MO, strategy=gfp.CARRY)) == oracle.to_mont(p, 300_001 % p)


@pytest.mark.parametrize("p", [3, 101, 65521, 67108859, 94906249])
def test_fp64_delayed_and_blocked(p):
    for strat in (gfp.DELAYED, gfp.BLOCKED):
        for n in [0, 1, 2, 3, 5, 513, 100_003]:
            try:
                gfp.plan(p, FP, n, strategy=strat)
            except gfp.GfpError:
                assert strat == gfp.DELAYED
                continue
            a = synth.uniform(SEED, 0, 0, n, p, np.float64)
            b = synth.uniform(SEED, 1, 0, n, p, np.float64)
            got = gfp.dot_ex(cu(a), cu(b), p, FP, strategy=strat).cpu()[0].item()
            assert got == oracle.dot_fp64(p, a, b), (p, strat, n)


def test_batch_ex_strategies():
    rows, n = 1000, 512
    for p in [2897, 2903, 40009, 65521]:
        A = synth.uniform(SEED, 2, 0, rows * n, p, np.uint16).reshape(rows, n)
        x = synth.uniform(SEED, 3, 0, n, p, np.uint16)
        want = oracle.dot_batch_classical(p, A, x)
        for m in (32, 64):
            for strat in STRATS:
                if admissible(p, n, torch.uint16, strat, m) is None:
                    continue
                out = gfp.dot_batch_ex(cu(A), cu(x), p, CL, strategy=strat, acc_bits=m).cpu().numpy()
                assert np.array_equal(out.astype(np.uint64), want), (p, m, strat)


def test_strategy_errors_surface():
    a = cu(np.ones(10, np.uint32))
    with pytest.raises(gfp.GfpError):
        gfp.dot_ex(a, a, 65521, CL, strategy=gfp.DELAYED, acc_bits=48)
    with pytest.raises(gfp.GfpError):
        gfp.dot_ex(a, a, 4294967291, CL, strategy=gfp.DELAYED)

"""GPU parity of the batch kernels at their accumulator bounds: worst-case rows (every
entry p-1, or -h / +h in the centered representation) whose length keeps the generic batch kernel at 8
lanes per row (n < 256 16-byte vectors), and every lanes-per-row choice (gfp_options.lanes_per_row 1 / 8 /
32), so that a per-accumulator overflow bound computed for the wrong lane count fails here.

Each expected value comes from the oracle (one 128-bit remainder per term); all-(p-1) rows are also the
closed form n mod p."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
CL, MO, FP, CE = gfp.CLASSICAL, gfp.MONTGOMERY, gfp.FP64, gfp.CENTERED
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


def prev_prime(x):
    while not oracle.is_prime(x):
        x -= 1
    return x


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


ROWS = 67
LENS = [17, 255, 449, 511, 512, 1000, 1023]  # all below 256 vectors of u16 / u32 / f64


@pytest.mark.parametrize("p", [prev_prime(2 ** 29), prev_prime(2 ** 31), 3037000493, 4294967291])
@pytest.mark.parametrize("lanes", [0, 1, 8, 32])
def test_classical_u32_worst_case_rows(p, lanes):
    for n in LENS:
        A = np.full(ROWS * n, p - 1, np.uint32)
        A[::7] = synth.uniform(synth.BASE_SEED, 2, 0, len(A[::7]), p, np.uint32)  # some rows not all p-1
        x = np.full(n, p - 1, np.uint32)
        want = oracle.dot_batch_classical(p, A.reshape(ROWS, n), x)
        got = gfp.dot_batch_ex(cu(A).view(ROWS, n), cu(x), p, CL, lanes_per_row=lanes)
        assert np.array_equal(got.cpu().numpy().astype(np.uint64), want), (p, n, lanes)
        if lanes == 0:
            got = gfp.dot_batch(cu(A).view(ROWS, n), cu(x), p, CL)
            assert np.array_equal(got.cpu().numpy().astype(np.uint64), want), (p, n)


@pytest.mark.parametrize("p", [2897, 2903, 65521])
@pytest.mark.parametrize("lanes", [0, 1, 8, 32])
def test_classical_u16_worst_case_rows(p, lanes):
    for n in LENS + [4096]:
        A = np.full(ROWS * n, p - 1, np.uint16)
        x = np.full(n, p - 1, np.uint16)
        want = oracle.dot_batch_classical(p, A.reshape(ROWS, n), x)
        assert all(int(v) == n % p for v in want)  # closed form: (p-1)^2 n = n (mod p)
        got = gfp.dot_batch_ex(cu(A).view(ROWS, n), cu(x), p, CL, lanes_per_row=lanes)
        assert np.array_equal(got.cpu().numpy().astype(np.uint64), want), (p, n, lanes)


@pytest.mark.parametrize("p", [16777213, 67108859, 94906249])
@pytest.mark.parametrize("lanes", [0, 8, 32])
def test_fp64_worst_case_rows(p, lanes):
    assert oracle.is_prime(p)
    for n in LENS:
        A = np.full(ROWS * n, p - 1, np.float64)
        x = np.full(n, p - 1, np.float64)
        want = oracle.dot_batch_classical(p, A.reshape(ROWS, n).astype(np.uint64), x.astype(np.uint64))
        got = gfp.dot_batch_ex(cu(A).view(ROWS, n), cu(x), p, FP, lanes_per_row=lanes)
        assert np.array_equal(got.cpu().numpy(), want.astype(np.float64)), (p, n, lanes)


@pytest.mark.parametrize("p", [65521, 4294967291])
@pytest.mark.parametrize("lanes", [0, 1, 8])
def test_montgomery_and_centered_int_worst_case_rows(p, lanes):
    n = 449
    if p < 2 ** 32 and p <= 2654435761:
        A = np.full(ROWS * n, p - 1, np.uint32)
        x = np.full(n, p - 1, np.uint32)
        Am, xm = gfp.to_rep(cu(A), p, MO), gfp.to_rep(cu(x), p, MO)
        got = gfp.dot_batch_ex(Am.view(ROWS, n), xm, p, MO, lanes_per_row=lanes).cpu().numpy().astype(np.uint64)
        want = [oracle.to_mont(p, int(v)) for v in oracle.dot_batch_classical(p, A.reshape(ROWS, n), x)]
        assert np.array_equal(got, np.array(want, np.uint64)), (p, lanes)
    h = (p - 1) // 2
    st = np.int16 if p <= 65521 else np.int32
    for v in (-h, h):
        A = np.full(ROWS * n, v, st)
        x = np.full(n, -h, st)
        got = gfp.dot_batch_ex(cu(A).view(ROWS, n), cu(x), p, CE, lanes_per_row=lanes).cpu().numpy().astype(np.int64)
        want = oracle.dot_centered(p, A[:n].astype(np.int64), x.astype(np.int64))
        assert np.all(got == want), (p, v, lanes)


@pytest.mark.parametrize("p", [67108859, 189812507])
def test_centered_f64_worst_case_rows(p):
    h = (p - 1) // 2
    for n in LENS:
        A = np.full(ROWS * n, -h, np.float64)
        x = np.full(n, h, np.float64)
        got = gfp.dot_batch(cu(A).view(ROWS, n), cu(x), p, CE).cpu().numpy()
        want = oracle.dot_centered(p, A[:n], x)
        assert np.all(got == want), (p, n)


def test_lanes_per_row_validation():
    A = cu(np.zeros((4, 64), np.uint32))
    x = cu(np.zeros(64, np.uint32))
    with pytest.raises(gfp.GfpError):
        gfp.dot_batch_ex(A, x, 65521, CL, lanes_per_row=4)  # only 0, 1, 8, 32
    with pytest.raises(gfp.GfpError):
        gfp.dot_batch_ex(A.to(torch.float64), x.to(torch.float64), 65521, FP, lanes_per_row=1)  # integer only
    # a batch option: dots reject it (GFP_E_INVAL)
    st = gfp.lib.gfp_dot_ex(65521, CL, 1, A.data_ptr(), A.data_ptr(), 8, gfp._opts(0, 0, 1), x.data_ptr(), None)
    assert st == 1


def test_batch_argument_validation():
    """The binding refuses shapes the storage cannot hold (no out-of-bounds kernel access)."""
    A = cu(np.zeros(100, np.uint16))
    x = cu(np.zeros(64, np.uint16))
    with pytest.raises(ValueError):
        gfp.dot_batch(A, x, 65521, rows=2, n=64)  # needs 128 elements
    with pytest.raises(ValueError):
        gfp.dot_batch_ex(A, x, 65521, rows=1, n=65)  # x too short
    with pytest.raises(ValueError):
        gfp.dot_batch(A.view(10, 10).t(), x[:10], 65521)  # transposed: column stride != 1
    with pytest.raises(ValueError):
        gfp.dot_batch_ex(A.view(10, 10), x[:10], 65521, out=cu(np.zeros(5, np.uint16)))  # out too short
    with pytest.raises(ValueError):
        gfp.dot_batch(A.view(10, 10), x[:10], 65521, out=cu(np.zeros(10, np.uint32)))  # out dtype
    gfp.dot_batch(A.view(10, 10)[1:], x[:10], 65521)  # a view with a storage offset is fine


@pytest.mark.parametrize("p,k", [(2887, 515), (2897, 512), (2903, 509)])
@pytest.mark.parametrize("strategy", ["BLOCKED", "HYBRID", "OVERFLOW", "CARRY"])
@pytest.mark.parametrize("lanes", [1, 8, 0])
def test_f1_dim512_m32_at_the_2897_step(p, k, strategy, lanes):
    """SURVEY 8(f) F1 / P:470-478: DIM = 512 dots with 32-bit accumulators.  With one accumulator per row
    (lanes 1, the paper's loop) the block length k = floor((2^32 - 1 - (p-1)) / (p-1)^2) is 515 / 512 / 509 at
    p = 2887 / 2897 / 2903: one final reduction per row up to 2897, two from 2903 -- and an all-(p-1) row of
    512 terms (512 * 2902^2 > 2^32) is wrong unless that second reduction happens."""
    strat = getattr(gfp, strategy)
    if strategy == "BLOCKED":
        assert gfp.plan(p, CL, 512, dtype=torch.uint16, strategy=strat, acc_bits=32)["block"] == k
    rows, n = 1000, 512
    A = synth.uniform(synth.BASE_SEED + 5, synth.STREAM_MAT, 0, rows * n, p, np.uint16)
    A[: 64 * n] = p - 1  # worst-case rows first
    x = synth.uniform(synth.BASE_SEED + 5, synth.STREAM_X, 0, n, p, np.uint16)
    x[:] = np.where(np.arange(n) % 3 == 0, x, p - 1)
    for xx in (x, np.full(n, p - 1, np.uint16)):
        want = oracle.dot_batch_classical(p, A.reshape(rows, n), xx)
        got = gfp.dot_batch_ex(cu(A).view(rows, n), cu(xx), p, CL, strategy=strat, acc_bits=32, lanes_per_row=lanes)
        assert np.array_equal(got.cpu().numpy().astype(np.uint64), want), (p, strategy, lanes)

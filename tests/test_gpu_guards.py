"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this pool): every entry point writes
into a view inside a larger buffer whose guard bands hold a sentinel pattern; after the call the guard
bands must be unchanged and the written values exact.  Covers dots (one output element), partials,
batches (rows outputs, padded lda, ragged rows), to/from conversions (ragged n, misaligned views, in
place), at sizes that exercise heads, tails, multi-wave grids and the packed combine."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
DEV = "cuda:0"
GUARD = 64  # elements on each side
SEED = synth.BASE_SEED + 9191


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def guarded(n, dtype, offset=0):
    """(whole buffer, view of n elements at GUARD + offset, copy of the untouched buffer)."""
    whole = torch.empty(n + 2 * GUARD + 8, dtype=dtype, device=DEV)
    whole.view(torch.uint8).fill_(0xA5)
    view = whole[GUARD + offset: GUARD + offset + n]
    return whole, view, whole.clone()


def assert_guards(whole, ref, n, offset=0):
    lo, hi = GUARD + offset, GUARD + offset + n
    assert torch.equal(whole[:lo].view(torch.uint8), ref[:lo].view(torch.uint8)), "write below the output"
    assert torch.equal(whole[hi:].view(torch.uint8), ref[hi:].view(torch.uint8)), "write above the output"


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


CASES = [(65521, gfp.CLASSICAL, np.uint16, torch.uint16), (4294967291, gfp.CLASSICAL, np.uint32, torch.uint32),
         (2 ** 31 - 1, gfp.MONTGOMERY, np.uint32, torch.uint32), (67108859, gfp.FP64, np.float64, torch.float64),
         (32749, gfp.ZECH, np.uint16, torch.uint16), (65521, gfp.ZECH, np.uint16, torch.uint16)]


def inputs(p, rep, np_dt, n, stream):
    if rep == gfp.ZECH:
        return synth.zech_codes(SEED, stream, 0, n, p - 1)
    return synth.uniform(SEED, stream, 0, n, p, np_dt)


@pytest.mark.parametrize("p,rep,np_dt,t_dt", CASES)
def test_dot_and_partial_write_only_their_element(p, rep, np_dt, t_dt):
    for n in [0, 1, 7, 4099, 1_000_003, 9_000_001]:
        a, b = inputs(p, rep, np_dt, n, 0), inputs(p, rep, np_dt, n, 1)
        want = oracle.dot(p, rep, a, b)
        for off in (0, 3):
            whole, out, ref = guarded(1, t_dt, off)
            gfp.dot(cu(a), cu(b), p, rep, out=out)
            torch.cuda.synchronize()
            assert_guards(whole, ref, 1, off)
            got = out.cpu()[0].item() if t_dt == torch.float64 else int(out.cpu().to(torch.int64)[0])
            assert got == want, (p, rep, n)
        whole, part, ref = guarded(1, torch.int64)
        gfp.dot_partial(cu(a), cu(b), p, rep, out=part)
        torch.cuda.synchronize()
        assert_guards(whole, ref, 1)


@pytest.mark.parametrize("p,rep,np_dt,t_dt", CASES)
def test_batch_writes_only_its_rows(p, rep, np_dt, t_dt):
    for rows, n, pad in [(1, 1, 0), (37, 513, 3), (4099, 512, 0), (2049, 4096, 8)]:
        lda = n + pad
        A = inputs(p, rep, np_dt, rows * lda, 2).reshape(rows, lda)
        x = inputs(p, rep, np_dt, n, 3)
        whole, out, ref = guarded(rows, t_dt, 1)
        gfp.dot_batch(cu(A)[:, :n], cu(x), p, rep, out=out)
        torch.cuda.synchronize()
        assert_guards(whole, ref, rows, 1)
        got = out.cpu()
        got = got.numpy() if t_dt == torch.float64 else got.to(torch.int64).numpy()
        for r in sorted({0, rows // 2, rows - 1}):
            assert got[r] == oracle.dot(p, rep, A[r, :n], x), (p, rep, rows, n, r)


@pytest.mark.parametrize("p,rep,np_dt,t_dt", [c for c in CASES if c[1] in (gfp.MONTGOMERY, gfp.ZECH)])
def test_conversions_write_only_their_range(p, rep, np_dt, t_dt):
    for n in [1, 9, 4097, 1_000_001]:
        for off in (0, 1, 5):
            res = synth.uniform(SEED, 4, 0, n, p, np.uint16 if t_dt == torch.uint16 else np.uint32)
            whole, out, ref = guarded(n, t_dt, off)
            gfp.to_rep(cu(res), p, rep, out=out)
            torch.cuda.synchronize()
            assert_guards(whole, ref, n, off)
            whole2, back, ref2 = guarded(n, cu(res).dtype, off)
            gfp.from_rep(out, p, rep, out=back)
            torch.cuda.synchronize()
            assert_guards(whole2, ref2, n, off)
            assert np.array_equal(back.cpu().numpy(), res), (p, rep, n, off)
    # in place (in == out) inside a guarded buffer: Montgomery only (Zech changes the element width)
    if rep == gfp.MONTGOMERY:
        n = 1_000_003
        res = synth.uniform(SEED, 5, 0, n, p, np.uint32)
        whole, view, _ = guarded(n, torch.uint32, 2)
        view.copy_(cu(res))
        ref = whole.clone()
        gfp.to_rep(view, p, rep, out=view)
        gfp.from_rep(view, p, rep, out=view)
        torch.cuda.synchronize()
        assert_guards(whole, ref, n, 2)
        assert np.array_equal(view.cpu().numpy(), res)

"""GPU checks of the install-time tuner (gfp_tune): it times every admissible strategy,
keeps the fastest (never slower than the built-in plan it also timed), cross-checks that all candidates
agree, and AUTO calls that follow the tuned table stay bit-exact against the CPU oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
DEV = "cuda:0"
SEED = synth.BASE_SEED + 404


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gfp.tune_clear()
    yield
    gfp.tune_clear()


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def test_tune_then_auto_is_exact():
    cases = [dict(rep=gfp.CLASSICAL, p=2 ** 31 - 1, n=1 << 18, dtype=torch.uint32),
             dict(rep=gfp.CLASSICAL, p=2897, n=1 << 16, dtype=torch.uint16),
             dict(rep=gfp.CLASSICAL, p=4294967291, n=512, rows=1 << 12, kind="batch", dtype=torch.uint32),
             dict(rep=gfp.MONTGOMERY, p=2 ** 31 - 1, n=1 << 18),
             dict(rep=gfp.FP64, p=67108859, n=1 << 16),
             dict(rep=gfp.ZECH, p=32749, n=1 << 18)]
    table = gfp.tune(cases, ms_per_candidate=2.0)
    assert len(table) == len(cases)
    for e in table:
        assert 0 < e["us_best"] <= e["us_builtin"]
    # re-tuning a case replaces its entry
    assert len(gfp.tune(cases[:1], ms_per_candidate=1.0)) == len(cases)

    n = 100_003
    for p, dt in [(2 ** 31 - 1, np.uint32), (2897, np.uint16), (4294967291, np.uint32)]:
        a, b = synth.uniform(SEED, 0, 0, n, p, dt), synth.uniform(SEED, 1, 0, n, p, dt)
        got = int(gfp.dot(cu(a), cu(b), p, gfp.CLASSICAL).cpu().to(torch.int64)[0])
        assert got == oracle.dot_classical(p, a, b), p
    p, rows, m = 4294967291, 1000, 512
    A = synth.uniform(SEED, 2, 0, rows * m, p, np.uint32).reshape(rows, m)
    x = synth.uniform(SEED, 3, 0, m, p, np.uint32)
    out = gfp.dot_batch(cu(A), cu(x), p, gfp.CLASSICAL).cpu().numpy().astype(np.uint64)
    assert np.array_equal(out, oracle.dot_batch_classical(p, A, x))
    p = 32749
    a, b = synth.zech_codes(SEED, 0, 0, n, p - 1), synth.zech_codes(SEED, 1, 0, n, p - 1)
    assert int(gfp.dot(cu(a), cu(b), p, gfp.ZECH).cpu().to(torch.int64)[0]) == oracle.dot_zech(p, 2, a, b)


def test_tune_cli_quick(tmp_path):
    from paper_cs_0404008_b200 import autotune as cli
    out = tmp_path / "t.txt"
    assert cli.main(["--quick", "--ms", "1", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0].startswith("# gfp-tune v1") and len(lines) > 20
    gfp.tune_clear()
    gfp.tune_load(str(out))
    assert len(gfp.tune_entries()) == len(lines) - 1


def test_tune_rejects_bad_cases():
    with pytest.raises(gfp.GfpError):
        gfp.tune([dict(rep=gfp.CLASSICAL, p=65521, n=0)])
    with pytest.raises(gfp.GfpError):
        gfp.tune([dict(rep=gfp.CLASSICAL, p=65520, n=10)])  # not prime

"""What ships, on the GPU: the install-time tuning table shipped with the library
(paper_cs_0404008_b200/gfp_tune.txt, loaded automatically by every AUTO call outside the tests) steers the
five BASELINE.json configs at full size -- exactly the calls bench.py and smoke() make -- and every result is
compared with the oracle (the other GPU tests start from the built-in plan, conftest.py).

Also: a fresh process with GFP_TUNE_FILE unset really auto-loads that file and runs smoke()."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

gfp = pytest.importorskip("paper_cs_0404008_b200")
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIPPED = os.path.join(ROOT, "paper_cs_0404008_b200", "gfp_tune.txt")


@pytest.fixture(scope="module", autouse=True)
def _shipped_table():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gfp.tune_load(SHIPPED)
    assert len(gfp.tune_entries()) > 0
    yield
    torch.cuda.synchronize()
    gfp.tune_clear()


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def as_py(t):
    return t.cpu()[0].item() if t.dtype == torch.float64 else int(t.cpu().to(torch.int64)[0])


def test_c1_c2_c3_c4_full_size_under_the_shipped_table():
    seed = synth.BASE_SEED
    # C1: GF(65521) classical u32, n = 10^5
    p, n = 65521, 100_000
    a, b = synth.uniform(seed + 0, 0, 0, n, p, np.uint32), synth.uniform(seed + 0, 1, 0, n, p, np.uint32)
    assert as_py(gfp.dot(cu(a), cu(b), p, gfp.CLASSICAL)) == oracle.dot_classical(p, a, b)
    # C2: GF(67108859) fp64, n = 10^7
    p, n = 67108859, 10 ** 7
    a, b = synth.uniform(seed + 1, 0, 0, n, p, np.float64), synth.uniform(seed + 1, 1, 0, n, p, np.float64)
    assert as_py(gfp.dot(cu(a), cu(b), p, gfp.FP64)) == oracle.dot_fp64(p, a, b)
    # C3: GF(2^31 - 1) Montgomery, n = 2^28, converted on the device
    p, n = 2 ** 31 - 1, 1 << 28
    a, b = synth.uniform(seed + 2, 0, 0, n, p, np.uint32), synth.uniform(seed + 2, 1, 0, n, p, np.uint32)
    am, bm = gfp.to_rep(cu(a), p, gfp.MONTGOMERY), gfp.to_rep(cu(b), p, gfp.MONTGOMERY)
    assert as_py(gfp.dot(am, bm, p, gfp.MONTGOMERY)) == oracle.to_mont(p, oracle.dot_classical(p, a, b))
    del am, bm
    # C4: GF(32749) Zech, n = 2^26, 10% zeros
    p, n = 32749, 1 << 26
    a, b = synth.zech_codes(seed + 3, 0, 0, n, p - 1), synth.zech_codes(seed + 3, 1, 0, n, p - 1)
    assert as_py(gfp.dot(cu(a), cu(b), p, gfp.ZECH)) == oracle.dot_zech(p, 2, a, b)


def test_c5_full_size_and_smoke_batch_under_the_shipped_table():
    seed = synth.BASE_SEED + 4
    p, rows, n = 65521, 65536, 4096
    A = synth.uniform(seed, 2, 0, rows * n, p, np.uint16).reshape(rows, n)
    x = synth.uniform(seed, 3, 0, n, p, np.uint16)
    got = gfp.dot_batch(cu(A), cu(x), p, gfp.CLASSICAL).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, oracle.dot_batch_classical(p, A, x))
    # smoke()'s 512 x 4096 batch (a size the table steers differently from C5)
    got = gfp.dot_batch(cu(A[:512]), cu(x), p, gfp.CLASSICAL).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, oracle.dot_batch_classical(p, A[:512], x))


@pytest.mark.parametrize("p", [3, 2897, 65521, 2 ** 31 - 1, 4294967291])
def test_every_tuned_neighbourhood(p):
    """Dots and batches near each tuned (p, n, rows) the table may redirect, against the oracle."""
    dt = np.uint16 if p <= 65521 else np.uint32
    for n in (4096, 65536, 1 << 20):
        a, b = synth.uniform(7, 0, 0, n, p, dt), synth.uniform(7, 1, 0, n, p, dt)
        assert as_py(gfp.dot(cu(a), cu(b), p, gfp.CLASSICAL)) == oracle.dot_classical(p, a, b), (p, n)
    for rows, n in ((32768, 512), (4096, 4096)):
        A = synth.uniform(7, 2, 0, rows * n, p, dt).reshape(rows, n)
        x = synth.uniform(7, 3, 0, n, p, dt)
        got = gfp.dot_batch(cu(A), cu(x), p, gfp.CLASSICAL).cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, oracle.dot_batch_classical(p, A, x)), (p, rows, n)


def test_fresh_process_autoloads_the_shipped_table_and_smoke_passes():
    env = {k: v for k, v in os.environ.items() if k != "GFP_TUNE_FILE"}
    code = ("import sys; sys.path.insert(0, %r); import paper_cs_0404008_b200 as g, __graft_entry__ as e; "
            "import torch; a = torch.zeros(8, dtype=torch.uint32, device='cuda'); g.dot(a, a, 65521); "
            "print('entries', len(g.tune_entries())); e.smoke()" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    n_file = sum(1 for line in open(SHIPPED) if line.strip() and not line.startswith("#"))
    assert f"entries {n_file}" in r.stdout, r.stdout
    assert "smoke: ok" in r.stdout

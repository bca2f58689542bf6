"""Host-side checks of libgfp (no GPU needed): exported symbols, gfp_query constants and bounds,
argument validation that returns before any device work.

Constants are recomputed here with Python integers (independent of numtheory.cpp); bounds are checked
against the paper's printed primes (tests/golden/paper_constants.json) and the next prime above.
"""
import ctypes
import json
import os
import re

import pytest

import oracle
from oracle import bruteforce as bf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAPER = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_constants.json")))

gfp = pytest.importorskip("paper_cs_0404008_b200")

OK, E_INVAL, E_NOT_PRIME, E_BOUND, E_UNSUPPORTED = 0, 1, 2, 3, 4
CL, MO, FP, ZE = gfp.CLASSICAL, gfp.MONTGOMERY, gfp.FP64, gfp.ZECH
U16, U32, F64 = 0, 1, 2


def header_functions():
    src = open(os.path.join(ROOT, "include", "gfp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gfp_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 13
    for name in names:
        assert hasattr(gfp.lib, name), name


def q(p, rep, dt):
    info = gfp.GfpInfo()
    st = gfp.lib.gfp_query(p, rep, dt, ctypes.byref(info))
    return st, info


def next_prime(p):
    p += 1
    while not bf.is_prime(p) if p < 10 ** 6 else not oracle.is_prime(p):
        p += 1
    return p


@pytest.mark.parametrize("rep,dt,key", [
    (CL, U16, "classical_unsigned_32"), (CL, U32, "classical_unsigned_64"), (MO, U32, "montgomery_B32")])
def test_bounds_at_paper_primes(rep, dt, key):
    p = PAPER[key]["value"]
    st, info = q(p, rep, dt)
    assert st == OK and info.bound == p
    assert q(next_prime(p), rep, dt)[0] in (E_BOUND,)


def test_fp64_and_zech_bounds():
    # fp64: largest prime with p(p-1) < 2^53 (Eq. (1) at m = 53, k >= 1)
    p = 94906249
    assert oracle.is_prime(p) and p * (p - 1) < 2 ** 53
    nxt = next_prime(p)
    assert nxt * (nxt - 1) >= 2 ** 53
    assert q(p, FP, F64)[0] == OK and q(nxt, FP, F64)[0] == E_BOUND
    assert q(65521, ZE, U16)[0] == OK and q(65537, ZE, U16)[0] == E_BOUND


def test_rejections():
    assert q(65535, CL, U16)[0] == E_NOT_PRIME
    assert q(1, CL, U16)[0] == E_NOT_PRIME
    assert q(0, CL, U32)[0] == E_NOT_PRIME
    assert q(2, MO, U32)[0] == E_BOUND  # Montgomery needs odd p (gcd(p, B) = 1)
    assert q(7, MO, U16)[0] == E_UNSUPPORTED
    assert q(7, FP, U32)[0] == E_UNSUPPORTED
    assert q(7, ZE, U32)[0] == E_UNSUPPORTED
    assert q(7, 9, U32)[0] == E_INVAL
    with pytest.raises(gfp.GfpError):
        gfp.query(65535, CL)


PRIMES = [2, 3, 5, 7, 101, 1009, 2897, 32749, 40009, 40499, 46337, 65521, 67108859, 94906249,
          2 ** 31 - 1, 2654435761, 4294967291]


@pytest.mark.parametrize("p", PRIMES)
def test_query_constants(p):
    for rep, dt in [(CL, U16), (CL, U32), (MO, U32), (FP, F64), (ZE, U16)]:
        st, I = q(p, rep, dt)
        if st != OK:
            continue
        m = 53 if rep == FP else 64
        assert I.acc_bits == m
        k = I.k
        # Eq. (1) with a carried residue (reading G7), tight
        if m == 64:
            assert k * (p - 1) ** 2 + (p - 1) <= 2 ** 64 - 1 or p == 2
            assert (k + 1) * (p - 1) ** 2 + (p - 1) > 2 ** 64 - 1 or p == 2
        else:
            assert k * (p - 1) ** 2 + (p - 1) < 2 ** 53 or p == 2
            assert (k + 1) * (p - 1) ** 2 + (p - 1) >= 2 ** 53 or p == 2
        assert I.corr == 2 ** 64 % p
        assert I.b_mod_p == 2 ** 32 % p
        assert I.inv_p == 1.0 / p  # Python float division is IEEE round-to-nearest
        if rep == MO:
            assert (I.n_im * p) % 2 ** 32 == 2 ** 32 - 1  # n_im = -p^{-1} mod B
            assert I.r2 == 2 ** 64 % p
            kr = I.mont_kr
            B = 2 ** 32
            assert kr * (p - 1) ** 2 <= p * B and kr * (p - 1) ** 2 + (B - 1) * p <= 2 ** 64 - 1
            assert kr == 1000000 or (kr + 1) * (p - 1) ** 2 > p * B or \
                (kr + 1) * (p - 1) ** 2 + (B - 1) * p > 2 ** 64 - 1  # capped at 10^6 (gfp.h)
        if rep == ZE:
            assert I.g == oracle.primitive_root(p)
            assert I.qbar == p - 1
            assert I.table_bytes == (131072 if 2 * (p - 1) <= 65534 else 2 * p)


def test_config_constants_match_survey():
    """SURVEY.md 8(a) per-config constants."""
    i = gfp.query(65521, CL, __import__("torch").uint32)
    assert i["k"] == 4297065216
    i = gfp.query(67108859, FP)
    assert i["k"] == 2 and i["inv_p"].hex() == "0x1.0000014000019p-26"
    i = gfp.query(2 ** 31 - 1, MO)
    assert (i["mont_kr"], i["n_im"], i["r2"], i["b_mod_p"], i["corr"]) == (2, 0x80000001, 4, 2, 4)
    i = gfp.query(32749, ZE)
    assert (i["g"], i["k"]) == (2, 17200859919)


def test_lambda_example_via_query():
    """at p = 40009 and 64-bit words, lambda ~ 1.15 10^10."""
    i = gfp.query(40009, CL, __import__("torch").uint32)
    assert f"{i['k'] / 1e10:.2f}" == "1.15"


def test_argument_errors_before_device_work():
    L = gfp.lib
    fake = ctypes.c_void_p(0x10000)
    out = ctypes.c_void_p(0x20000)
    assert L.gfp_dot(65521, CL, U32, fake, fake, -1, out, None) == E_INVAL
    assert L.gfp_dot(65521, CL, U32, None, fake, 5, out, None) == E_INVAL
    assert L.gfp_dot(65521, CL, U32, fake, fake, 5, None, None) == E_INVAL
    assert L.gfp_dot(65521, CL, U32, ctypes.c_void_p(0x10001), fake, 5, out, None) == E_INVAL
    assert L.gfp_dot(65521, CL, 7, fake, fake, 5, out, None) == E_INVAL
    assert L.gfp_dot_batch(65521, CL, U16, fake, 3, fake, 4, 5, out, None) == E_INVAL  # lda < n
    assert L.gfp_dot_batch(65521, CL, U16, fake, 5, fake, 0, 5, out, None) == OK  # rows == 0: no-op
    assert L.gfp_to_rep(7, MO, U32, fake, U32, fake, -3, None) == E_INVAL
    assert b"n < 0" in L.gfp_last_error()
    assert L.gfp_to_rep(7, MO, U32, fake, U32, out, 0, None) == OK  # n == 0: no-op
    assert L.gfp_to_rep(7, MO, U16, fake, U32, fake, 4, None) == E_INVAL  # in-place needs equal dtypes
    assert L.gfp_status_str(E_BOUND).startswith(b"GFP_E_BOUND")


# ------------------------------------------------------------------------------ explicit strategies (F2)
def test_plan_block_lengths_match_the_paper():
    """m = 32 accumulators at DIM = 512 (sec. 3.4): the blocked k (Eq. (1), reading G7)
    is >= 512 up to p = 2897 and below from the next prime; the hybrid lambda of Eq. (2),
    lambda p(p-1) < 2^32, is >= 512 up to 2887 (reading G4)."""
    P = gfp.plan
    assert P(2897, CL, 512, strategy=gfp.BLOCKED, acc_bits=32)["block"] == 512
    assert P(2903, CL, 512, strategy=gfp.BLOCKED, acc_bits=32)["block"] == 509
    assert P(2887, CL, 512, strategy=gfp.HYBRID, acc_bits=32)["block"] >= 512
    assert P(2897, CL, 512, strategy=gfp.HYBRID, acc_bits=32)["block"] == 511
    for p in [3, 101, 2897, 40009, 65521]:
        for m in (32, 64):
            k = P(p, CL, 512, strategy=gfp.BLOCKED, acc_bits=m)["block"]
            assert k * (p - 1) ** 2 + (p - 1) <= 2 ** m - 1 < (k + 1) * (p - 1) ** 2 + (p - 1)
            lam = P(p, CL, 512, strategy=gfp.HYBRID, acc_bits=m)["block"]
            assert lam * p * (p - 1) < 2 ** m <= (lam + 1) * p * (p - 1)
    # the library's 8 lanes per DIM = 512 row give each accumulator 64 terms: the same step moves to where
    # 64 (p-1)^2 + (p-1) crosses 2^32 -- k = 64 at 8191, 63 at 8209 (reading G24; the sweep shows it)
    assert P(8191, CL, 512, strategy=gfp.BLOCKED, acc_bits=32)["block"] == 64
    assert P(8209, CL, 512, strategy=gfp.BLOCKED, acc_bits=32)["block"] == 63
    assert 64 * 8190 ** 2 + 8190 <= 2 ** 32 - 1 < 64 * 8208 ** 2 + 8208
    assert P(40009, CL, 10 ** 6, strategy=gfp.DELAYED)["kernel"].endswith("DELAYED>")
    assert P(65521, CL, 10 ** 6, strategy=gfp.OVERFLOW, acc_bits=32)["reductions_per_thread"] >= 1


def test_plan_rejections():
    P = gfp.plan
    with pytest.raises(gfp.GfpError) as e:
        P(65537, CL, 10, dtype=__import__("torch").uint32, strategy=gfp.BLOCKED, acc_bits=32)
    assert e.value.status == E_BOUND  # (p-1)^2 + (p-1) >= 2^32
    with pytest.raises(gfp.GfpError) as e:
        P(65521, CL, 2, strategy=gfp.DELAYED, acc_bits=32)  # 2 (p-1)^2 > 2^32: Eq. (1) violated
    assert e.value.status == E_BOUND
    with pytest.raises(gfp.GfpError) as e:
        P(4294967291, CL, 3, strategy=gfp.DELAYED)
    assert e.value.status == E_BOUND
    with pytest.raises(gfp.GfpError) as e:
        P(2 ** 31 - 1, MO, 10, strategy=gfp.HYBRID)
    assert e.value.status == E_UNSUPPORTED
    with pytest.raises(gfp.GfpError) as e:
        P(32749, ZE, 10, strategy=gfp.BLOCKED)
    assert e.value.status == E_UNSUPPORTED
    with pytest.raises(gfp.GfpError) as e:
        P(67108859, FP, 10, strategy=gfp.OVERFLOW)
    assert e.value.status == E_UNSUPPORTED
    with pytest.raises(gfp.GfpError) as e:
        P(65521, CL, 10, strategy=gfp.BLOCKED, acc_bits=48)
    assert e.value.status == E_INVAL
    assert P(2 ** 31 - 1, MO, 10, strategy=gfp.OVERFLOW)["kernel"] == "dot_kernel<MontgomeryOverflow>"
    assert P(67108859, FP, 2, strategy=gfp.DELAYED)["kernel"] == "dot_kernel<Fp64<0>>"


def test_plan_zech_add():
    """Pure-Zech accumulation (F3): Zech only, one table lookup per term, no integer accumulator."""
    P = gfp.plan
    d = P(32749, ZE, 2 ** 26, strategy=gfp.ZECH_ADD)
    assert d["kernel"] == "zech_add_dot_kernel" and d["strategy_name"] == "zech_add"
    assert d["acc_bits"] == 0 and d["reductions_per_thread"] >= d["terms_per_thread"] > 0
    assert P(65521, ZE, 10, strategy=gfp.ZECH_ADD)["kernel"] == "zech_add_dot_kernel"
    for rep, p in [(CL, 65521), (MO, 2 ** 31 - 1), (FP, 67108859)]:
        with pytest.raises(gfp.GfpError) as e:
            P(p, rep, 10, strategy=gfp.ZECH_ADD)
        assert e.value.status == E_UNSUPPORTED
    with pytest.raises(gfp.GfpError) as e:
        P(32749, ZE, 10, strategy=gfp.ZECH_ADD, acc_bits=32)
    assert e.value.status == E_UNSUPPORTED


# ------------------------------------------------------------------------------ install-time tuning (F4)
def _entry(rep, dt, kind, p, n, strategy, acc_bits=0, rows=0):
    return dict(rep=rep, dtype=dt, kind=kind, p=p, n=n, rows=rows, strategy=strategy, acc_bits=acc_bits,
                us_best=1.0, us_builtin=2.0)


@pytest.fixture
def clean_table():
    gfp.tune_clear()
    yield
    gfp.tune_clear()


def test_tuned_auto_follows_nearest_case(clean_table):
    """AUTO takes the strategy of the tuned case nearest in (log2 p, log2 n) for the same rep/dtype/kind
    ("switching thresholds"), only when admissible; otherwise the built-in plan."""
    P = gfp.plan
    # built-in plan when a thread's sum can wrap: Eq. (2) hybrid while lambda = floor((2^64-1)/(p(p-1))) >= 4,
    # the carry word (sec. 3.3, the carry flag counted) below (lambda = 1 at 4294967291)
    builtin = P(2 ** 31 - 1, CL, 10 ** 6)
    assert builtin["kernel"] == "ClassicalS<u64acc,u32,HYBRID>"
    assert builtin["block"] == (2 ** 64 - 1) // ((2 ** 31 - 1) * (2 ** 31 - 2)) == 4
    builtin = builtin["kernel"]
    assert P(4294967291, CL, 10 ** 6)["kernel"] == "ClassicalS<u64acc,u32,CARRY>"
    assert P(4294967291, CL, 10 ** 6)["reductions_per_thread"] == 1
    gfp.tune_set([_entry(CL, U32, 0, 2 ** 31 - 1, 1 << 20, gfp.CARRY, 64),
                  _entry(CL, U32, 0, 65537, 1 << 20, gfp.BLOCKED, 64),
                  _entry(CL, U16, 0, 2897, 1 << 12, gfp.DELAYED, 32)])
    assert P(2 ** 31 - 1, CL, 10 ** 6)["kernel"] == "ClassicalS<u64acc,u32,CARRY>"
    assert P(4294967291, CL, 10 ** 6)["kernel"] == "ClassicalS<u64acc,u32,CARRY>"  # nearest: 2^31-1
    assert P(1048573, CL, 10 ** 6)["kernel"] == "ClassicalS<u64acc,u32,BLOCKED>"      # nearest: 65537
    # DELAYED at m = 32 is admissible only while n (p-1)^2 < 2^32: n = 2 is, n = 10^6 falls back
    assert P(2897, CL, 2)["kernel"] == "ClassicalS<u32acc,u16,DELAYED>"
    assert P(2897, CL, 10 ** 6)["kernel"] == "dot_kernel<ClassicalU16<ALL>>"  # the built-in plan
    # explicit options are never overridden; other reps/kinds are untouched
    assert P(2 ** 31 - 1, CL, 10 ** 6, strategy=gfp.OVERFLOW, acc_bits=64)["kernel"] == "ClassicalS<u64acc,u32,OVERFLOW>"
    assert P(2 ** 31 - 1, MO, 10 ** 6)["kernel"] == "dot_kernel<Montgomery<2>>"
    gfp.tune_clear()
    assert P(2 ** 31 - 1, CL, 10 ** 6)["kernel"] == builtin


def test_tuned_builtin_winner_keeps_builtin(clean_table):
    gfp.tune_set([_entry(FP, F64, 0, 67108859, 10 ** 7, gfp.AUTO)])
    assert gfp.plan(67108859, FP, 10 ** 7)["kernel"] == "dot_kernel<Fp64<2>>"
    gfp.tune_set([_entry(FP, F64, 0, 67108859, 10 ** 7, gfp.DELAYED)])  # inadmissible at n = 10^7
    assert gfp.plan(67108859, FP, 10 ** 7)["kernel"] == "dot_kernel<Fp64<2>>"
    gfp.tune_set([_entry(ZE, U16, 0, 32749, 1 << 26, gfp.ZECH_ADD)])
    assert gfp.plan(32749, ZE, 1 << 26)["kernel"] == "zech_add_dot_kernel"


def test_tune_save_load_roundtrip(tmp_path, clean_table):
    es = [_entry(CL, U32, 1, 2 ** 31 - 1, 512, gfp.HYBRID, 64, rows=1 << 15),
          _entry(MO, U32, 0, 2 ** 31 - 1, 1 << 24, gfp.OVERFLOW)]
    gfp.tune_set(es)
    path = str(tmp_path / "t.txt")
    gfp.tune_save(path)
    assert open(path).readline().startswith("# gfp-tune v1")
    gfp.tune_clear()
    assert gfp.tune_entries() == []
    gfp.tune_load(path)
    got = gfp.tune_entries()
    assert [(e["rep"], e["kind"], e["p"], e["n"], e["rows"], e["strategy"], e["acc_bits"]) for e in got] == \
        [(e["rep"], e["kind"], e["p"], e["n"], e["rows"], e["strategy"], e["acc_bits"]) for e in es]
    bad = tmp_path / "bad.txt"
    bad.write_text("not a table\n")
    with pytest.raises(gfp.GfpError) as e:
        gfp.tune_load(str(bad))
    assert e.value.status == E_INVAL and "header" in str(e.value)
    bad.write_text("# gfp-tune v1\n0 1 0 7 5\n")
    with pytest.raises(gfp.GfpError):
        gfp.tune_load(str(bad))
    assert len(gfp.tune_entries()) == 2  # a failed load leaves the table as it was


def test_tune_set_rejects_invalid(clean_table):
    for e in [_entry(9, U32, 0, 7, 5, 0), _entry(CL, U32, 2, 7, 5, 0), _entry(CL, U32, 0, 7, 5, 9),
              _entry(ZE, U16, 1, 32749, 512, gfp.ZECH_ADD), _entry(CL, U32, 0, 1, 5, 0)]:
        with pytest.raises(gfp.GfpError) as err:
            gfp.tune_set([e])
        assert err.value.status == E_INVAL
    assert gfp.tune_entries() == []


def test_tune_file_from_environment(tmp_path):
    """GFP_TUNE_FILE is loaded on the first AUTO call of a process."""
    import subprocess
    import sys
    path = tmp_path / "env.txt"
    path.write_text("# gfp-tune v1\n0 1 0 2147483647 1048576 0 4 64 1.0 2.0\n")
    code = ("import paper_cs_0404008_b200 as g; "
            "print(g.plan(2147483647, 0, 10**6)['kernel']); print(len(g.tune_entries()))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         env=dict(os.environ, GFP_TUNE_FILE=str(path)), check=True).stdout.split()
    assert out == ["ClassicalS<u64acc,u32,HYBRID>", "1"]


def test_shipped_install_time_table_loads_by_default():
    """Without GFP_TUNE_FILE the library loads gfp_tune.txt next to libgfp.so (the table measured on a
    B200 by `python -m paper_cs_0404008_b200.autotune`); AUTO then follows the nearest tuned case."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k != "GFP_TUNE_FILE"}
    code = """
import torch, paper_cs_0404008_b200 as g
es = g.tune_entries()
print(len(es), all(e['us_best'] <= e['us_builtin'] for e in es))
p, n = 2147483647, 65536
e = [e for e in es if (e['rep'], e['dtype'], e['kind'], e['p'], e['n']) == (0, 1, 0, p, n)][0]
tuned = g.plan(p, 0, n, dtype=torch.uint32)
g.tune_clear()
builtin = g.plan(p, 0, n, dtype=torch.uint32)
if e['strategy'] == 0:
    print(tuned['kernel'] == builtin['kernel'])
else:
    print(tuned['strategy'] == e['strategy'] and tuned['acc_bits'] == e['acc_bits'])
"""
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, env=env,
                         check=True).stdout.split("\n")
    n, ok = out[0].split()
    assert int(n) >= 100 and ok == "True"
    assert out[1] == "True"


# ------------------------------------------------------------------------------ centered representation (F2)
CE = gfp.CENTERED


def test_centered_bounds_and_block_lengths():
    """sec. 3.2.2: storage bounds (h = (p-1)/2 fits int16 / int32; binary64 h(h+1) < 2^53),
    odd p only, and lambda_c: the largest k with k h^2 + h < 2^63 (int64) / 2^53 (binary64),
    recomputed here with Python integers -- roughly twice the unsigned k at the same word."""
    for p, dt, ok in [(65521, U16, True), (4294967291, U32, True), (189812507, F64, True),
                      (189812533, F64, False), (2, U16, False), (65537, U16, False)]:
        st, info = q(p, CE, dt)
        assert (st == OK) == ok, (p, dt, st)
        if ok:
            h = (p - 1) // 2
            w = 2 ** 53 if dt == F64 else 2 ** 63
            assert info.k * h * h + h < w <= (info.k + 1) * h * h + h
            assert info.acc_bits == (53 if dt == F64 else 64)
    assert q(67108859, CE, F64)[1].k == 8 and q(67108859, FP, F64)[1].k == 2  # C2 k 2 -> 8
    for p in [5, 101, 32749, 65521, 2 ** 31 - 1, 4294967291]:
        dt = U16 if p <= 65521 else U32
        kc, kz = q(p, CE, dt)[1].k, q(p, CL, U32)[1].k
        assert kc >= 2 * kz - 2, p  # SPEC: K_centered >= 2 K_zpz - c
    for p, dt, ok in [(67108859, F64, True)]:
        st, _ = q(p, CE, dt)
        assert st == OK


def test_centered_plans_and_rejections():
    import torch
    P = gfp.plan
    d = P(67108859, CE, 10 ** 7, dtype=torch.float64)
    assert d["kernel"] == "dot_kernel<Fp64C<8>>" and d["block"] == 8 and d["strategy_name"] == "blocked"
    assert P(65521, CE, 10 ** 7, dtype=torch.int16)["kernel"] == "dot_kernel<CenteredI<i16,ALL>>"
    assert P(4294967291, CE, 10 ** 7, dtype=torch.int32)["kernel"] == "dot_kernel<CenteredI<i32,BLOCKED>>"
    assert P(4294967291, CE, 10 ** 7, dtype=torch.int32)["block"] == 2
    assert P(67108859, CE, 4, dtype=torch.float64, strategy=gfp.DELAYED)["kernel"] == "dot_kernel<Fp64C<0>>"
    for strat in (gfp.OVERFLOW, gfp.HYBRID, gfp.ZECH_ADD):  # signed overflow trick / hybrid centered: OUT
        with pytest.raises(gfp.GfpError) as e:
            P(32749, CE, 10, dtype=torch.int16, strategy=strat)
        assert e.value.status == E_UNSUPPORTED
    with pytest.raises(gfp.GfpError) as e:
        P(67108859, CE, 10 ** 7, dtype=torch.float64, strategy=gfp.DELAYED)
    assert e.value.status == E_BOUND


def test_plan_carry_word():
    """F2 carry word: a second word counts the wraps of the m-bit sum (sec. 3.3 with the CORR deferred);
    admissible wherever the overflow strategy is (classical m = 32 / 64, Montgomery)."""
    import torch
    P = gfp.plan
    assert P(4294967291, CL, 10 ** 6, strategy=gfp.CARRY, acc_bits=64)["kernel"] == "ClassicalS<u64acc,u32,CARRY>"
    assert P(65521, CL, 10 ** 6, strategy=gfp.CARRY, acc_bits=32)["kernel"] == "ClassicalS<u32acc,u16,CARRY>"
    assert P(65521, CL, 10, dtype=torch.uint32, strategy=gfp.CARRY, acc_bits=32)["kernel"] == "ClassicalS<u32acc,u32,CARRY>"
    assert P(2 ** 31 - 1, MO, 10, strategy=gfp.CARRY)["kernel"] == "dot_kernel<MontgomeryCarry>"
    assert P(2 ** 31 - 1, MO, 10, strategy=gfp.CARRY)["strategy_name"] == "carry"
    for rep, p in [(FP, 67108859), (ZE, 32749), (CE, 32749)]:
        with pytest.raises(gfp.GfpError) as e:
            P(p, rep, 10, strategy=gfp.CARRY)
        assert e.value.status == E_UNSUPPORTED
    # every explicit classical policy keeps its own name (the 5-slot encoding)
    names = {P(65521, CL, 1, strategy=s, acc_bits=m)["kernel"] for s in (gfp.DELAYED, gfp.BLOCKED, gfp.OVERFLOW,
                                                                          gfp.HYBRID, gfp.CARRY) for m in (32, 64)}
    assert len(names) == 10

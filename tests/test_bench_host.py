"""Host-side logic of bench.py that runs without a GPU: the threaded oracle baseline (the same oracle on
one contiguous slice per core, combined and checked against one thread) and the --impl reference arm."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = pytest.importorskip("bench")


def _small(cfg_index, n):
    cfg = dict(bench.CONFIGS[cfg_index])
    if cfg["kind"] == "batch":
        cfg["rows"] = n
    else:
        cfg["n"] = n
    return cfg


@pytest.mark.parametrize("cfg_index", [0, 1, 4])
def test_threaded_oracle_slices_recombine(cfg_index):
    cfg = _small(cfg_index, 257 if cfg_index == 4 else 100_003)
    p = cfg["p"]
    if cfg["kind"] == "batch":
        A = synth.uniform(synth.BASE_SEED, 2, 0, cfg["rows"] * cfg["n"], p, cfg["dtype"]).reshape(cfg["rows"], cfg["n"])
        h = {"A": A, "x": synth.uniform(synth.BASE_SEED, 3, 0, cfg["n"], p, cfg["dtype"])}
        m = cfg["rows"]
    else:
        h = {"a": synth.uniform(synth.BASE_SEED, 0, 0, cfg["n"], p, cfg["dtype"]),
             "b": synth.uniform(synth.BASE_SEED, 1, 0, cfg["n"], p, cfg["dtype"])}
        m = cfg["n"]
    single = bench.oracle_slice(cfg, h, 0, m)
    for threads in (1, 3, 8):
        tps, ok = bench.oracle_time_threads(cfg, h, m, threads, single=single)
        assert ok is True and tps > 0


def test_threaded_oracle_detects_a_wrong_combine():
    cfg = _small(0, 10_001)
    p = cfg["p"]
    h = {"a": synth.uniform(synth.BASE_SEED, 0, 0, cfg["n"], p, np.uint32),
         "b": synth.uniform(synth.BASE_SEED, 1, 0, cfg["n"], p, np.uint32)}
    single = bench.oracle_slice(cfg, h, 0, cfg["n"])
    _, ok = bench.oracle_time_threads(cfg, h, cfg["n"], 4, single=(single + 1) % p)
    assert ok is False


def test_reference_arm_runs_on_the_host():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--oracle-budget", "0.2"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2
    assert line["cpu_baseline"]["cores"] == bench.host_threads()
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "True" in line["cpu_baseline"]["threads_note"]


# ------------------------------------------------------------------------------ --gpus N launcher
def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT", "GFP_BENCH_PG_BACKEND")}
    env.update(kw)
    return env


def test_launch_plan_rules():
    # the driver's torchrun form: WORLD_SIZE must equal --gpus
    assert bench.launch_plan(8, {"WORLD_SIZE": "8"}, 8) == ("run", None)
    how, why = bench.launch_plan(8, {"WORLD_SIZE": "1"}, 8)
    assert how == "fail" and "WORLD_SIZE=1" in why
    # no WORLD_SIZE: one process at N = 1, self-launch N ranks at N > 1
    assert bench.launch_plan(1, {}, 1) == ("run", None)
    how, argv = bench.launch_plan(4, {}, 8)
    assert how == "spawn" and "torch.distributed.run" in argv and "--nproc-per-node=4" in argv
    assert "127.0.0.1" in argv
    # more ranks than visible GPUs: fail loudly (never time fewer GPUs than asked for)
    how, why = bench.launch_plan(2, {}, 1)
    assert how == "fail" and "only 1 CUDA device" in why
    # host-logic check mode: ranks may share (or lack) devices
    assert bench.launch_plan(2, {"GFP_BENCH_PG_BACKEND": "gloo"}, 0)[0] == "spawn"
    assert bench.launch_plan(0, {}, 8)[0] == "fail"


def test_gpus2_self_launches_two_ranks_over_gloo():
    """`python bench.py --gpus 2` (the driver's plain form, no torchrun) must run TWO ranks: the launcher
    re-execs itself under torch.distributed.run; --dry-run stops after the process group is up."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       env=_env(GFP_BENCH_PG_BACKEND="gloo"), capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["gpus_arg"] == 2 and line["backend"] == "gloo"
    assert sorted(x["rank"] for x in line["ranks"]) == [0, 1]
    assert len({x["pid"] for x in line["ranks"]}) == 2  # two processes, not one


def test_gpus2_without_enough_gpus_fails_loudly():
    """On a box with fewer GPUs than --gpus (here: none), the bench refuses instead of timing one GPU and
    printing n_gpus: 1."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       env=_env(), capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "CUDA device" in r.stderr
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]
    # and a torchrun world that disagrees with --gpus
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       env=_env(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"), capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_lookup_wavefronts_matches_a_direct_count():
    """bench.lookup_wavefronts (the Zech matrix-vector gather roofline) against a direct per-warp count: lane l
    looks up code 8 (v0 + l) + k for k in 0..7; a warp lookup takes max over banks of the distinct 32-bit words."""
    rng = np.random.default_rng(5)
    A = rng.integers(0, 32749, size=(4, 4096)).astype(np.uint16)
    A[:, ::10] = 0
    direct = []
    for row in A.astype(np.int64):
        for v0 in range(0, 4096 // 8, 32):
            for k in range(8):
                codes = [row[8 * (v0 + l) + k] for l in range(32)]
                banks = {}
                for c in codes:
                    banks.setdefault((c >> 1) & 31, set()).add(c >> 1)
                direct.append(max(len(s) for s in banks.values()))
    assert abs(bench.lookup_wavefronts(A, sample_rows=4) - float(np.mean(direct))) < 1e-9
    assert bench.lookup_wavefronts(np.zeros((2, 4096), np.uint16)) == 1.0  # every lane reads one word


def test_split_lookup_wavefronts_every_lane_in_its_own_bank():
    """bench.split_lookup_wavefronts (the split-exponent kernel's roofline): from the kernel's address map every
    warp lookup is one wavefront, whatever the codes (random, all equal, zeros, both zero-code layouts); and a
    direct recount of one warp lookup's banks from the byte addresses agrees."""
    rng = np.random.default_rng(7)
    for p in (32749, 65269, 65287, 65521):
        A = rng.integers(0, p, size=(4, 4096)).astype(np.uint16)
        A[:, ::10] = 0
        assert bench.split_lookup_wavefronts(A, p, sample_rows=4) == 1.0
        assert bench.split_lookup_wavefronts(np.zeros((2, 4096), np.uint16), p) == 1.0
        assert bench.split_lookup_wavefronts(np.full((2, 4096), p - 1, np.uint16), p) == 1.0
    codes = rng.integers(0, 65521, size=32)
    e = (codes - 1) & 0xFFFF
    for addr in (0x10000 | ((e & 255) << 8) | 4 * np.arange(32), 0x10000 | ((e >> 8) << 8) | (128 + 4 * np.arange(32))):
        banks = (addr >> 2) & 31
        assert sorted(banks.tolist()) == list(range(32))  # 32 distinct banks: one wavefront

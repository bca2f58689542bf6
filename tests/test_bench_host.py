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

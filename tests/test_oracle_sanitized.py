"""The CPU oracle under -fsanitize=undefined,address (wrapping arithmetic is explicit,
never undefined): tests/oracle_san_driver.c compiles oracle/oracle.c into one program with the sanitizers and calls
every entry point at the pins' edges (the paper's largest primes, all-(p-1) operands, n = 0, every Zech code pair at
GF(101) through both Zech dots, invalid inputs that must be reported), checking closed forms on the way."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_runs_clean_under_ubsan_and_asan(tmp_path):
    exe = tmp_path / "oracle_san"
    cc = subprocess.run(["gcc", "-O1", "-g", "-fsanitize=undefined,address", "-fno-sanitize-recover=all",
                         "-fno-omit-frame-pointer", "-Wall", "-o", str(exe),
                         os.path.join(ROOT, "tests", "oracle_san_driver.c"), "-lm"],
                        capture_output=True, text=True, timeout=300)
    if cc.returncode != 0 and ("asan" in cc.stderr.lower() or "ubsan" in cc.stderr.lower()):
        pytest.skip("sanitizer runtime not available: " + cc.stderr.strip().splitlines()[-1])
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0",
                                  UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1"))
    assert run.returncode == 0, run.stdout + run.stderr
    assert "runtime error" not in run.stderr and "AddressSanitizer" not in run.stderr, run.stderr
    assert "oracle under sanitizers: ok" in run.stdout

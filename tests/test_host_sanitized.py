"""The product's host code under UBSan (SURVEY.md 4.2 T6 asks for sanitizers; compute-sanitizer is closed on this pool,
so the device side is covered by tests/test_gpu_guards.py): the C-ABI layer, the number theory (Miller-Rabin, -p^-1,
R^2, the Eq. (1)/(2) bounds, Zech tables) and the tuner (api.cpp, numtheory.cpp, tune.cpp) are recompiled with
-fsanitize=undefined -fno-sanitize-recover and linked with the already-built kernel objects, and the host-side test
file (every constant, plan, bound and validation path, no GPU needed) runs against that library."""
import glob
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
KOBJ = sorted(glob.glob(os.path.join(ROOT, "build", "gfp", "kernels_*.cu.o")))


@pytest.mark.skipif(not os.path.exists(NVCC) or len(KOBJ) < 3, reason="needs nvcc and the built kernel objects (make)")
def test_host_code_runs_clean_under_ubsan(tmp_path):
    csrc = os.path.join(ROOT, "paper_cs_0404008_b200", "csrc")
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O1", "-g", "-std=c++17",
             "-Xcompiler", "-fPIC,-fsanitize=undefined,-fno-sanitize-recover=all",
             "-I" + os.path.join(ROOT, "include"), "-I" + csrc]
    objs = []
    for name in ("api", "numtheory", "tune"):
        o = str(tmp_path / (name + ".o"))
        r = subprocess.run([NVCC, *flags, "-c", "-o", o, os.path.join(csrc, name + ".cpp")],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        objs.append(o)
    # beside libgfp.so: the library finds its shipped tuning table next to itself
    lib = os.path.join(ROOT, "paper_cs_0404008_b200", "libgfp_ubsan.so")
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *KOBJ, *objs,
                        "-lcudart", "-Xcompiler", "-fsanitize=undefined"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    try:
        env = dict(os.environ, GFP_LIBRARY=lib, UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
        run = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                              os.path.join(ROOT, "tests", "test_abi_host.py")],
                             capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
        assert run.returncode == 0, run.stdout[-3000:] + run.stderr[-3000:]
        assert "runtime error" not in run.stdout + run.stderr
    finally:
        os.remove(lib)

"""The product never touches the test infrastructure: no module of the package (or its C/CUDA sources)
imports, links or names the CPU oracle or the input generator, and the binding refuses to load without the
CUDA library (no CPU fallback).  Only tests/, __graft_entry__.smoke() and bench.py's oracle legs may use
oracle/ (DESIGN.md "Oracle")."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_cs_0404008_b200")


def product_sources():
    for base, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                yield os.path.join(base, f)
    yield os.path.join(ROOT, "include", "gfp.h")


def test_product_never_references_oracle_or_synth():
    pat = re.compile(r"^\s*(import|from)\s+(oracle|synth)\b|liboracle|libsynth|oracle_[a-z_]+\(|synth_[a-z_]+\(",
                     re.M)
    bad = [path for path in product_sources() if pat.search(open(path, errors="replace").read())]
    assert not bad, bad


def test_oracle_and_product_share_no_headers():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "#include \"" not in src  # system headers only
    for path in product_sources():
        assert "oracle" not in os.path.basename(path)


def test_binding_fails_loudly_without_the_library(tmp_path):
    code = "import paper_cs_0404008_b200"
    env = dict(os.environ, GFP_LIBRARY=str(tmp_path / "missing.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, env=env)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr

"""Property-based pins of the oracle (hypothesis): for random primes, representations and short vectors,
the compiled oracle equals Python-integer field arithmetic, and the algebraic laws of the dot hold.
Complements tests/test_oracle_pins.py (fixed cases) with shrinking counterexamples."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from oracle import bruteforce as bf

PRIMES = [2, 3, 5, 7, 11, 13, 101, 257, 1009, 2897, 32749, 40009, 65521, 2147483647, 4294967291]
SMALL = [p for p in PRIMES if p <= 1009]


@st.composite
def vectors(draw, primes=PRIMES, max_n=40):
    p = draw(st.sampled_from(primes))
    n = draw(st.integers(0, max_n))
    a = draw(st.lists(st.integers(0, p - 1), min_size=n, max_size=n))
    b = draw(st.lists(st.integers(0, p - 1), min_size=n, max_size=n))
    return p, a, b


@settings(max_examples=300, deadline=None)
@given(vectors())
def test_classical_equals_python_integers(v):
    p, a, b = v
    dt = np.uint64
    assert oracle.dot_classical(p, np.array(a, dt), np.array(b, dt)) == bf.dot(p, a, b)


@settings(max_examples=200, deadline=None)
@given(vectors(primes=[3, 101, 32749, 40499, 65521, 2147483647, 2654435761]))
def test_montgomery_equals_python_integers(v):
    p, a, b = v
    am = np.array([bf.to_mont(p, x) for x in a], np.uint32)
    bm = np.array([bf.to_mont(p, x) for x in b], np.uint32)
    assert oracle.dot_montgomery(p, am, bm) == bf.to_mont(p, bf.dot(p, a, b))


@settings(max_examples=200, deadline=None)
@given(vectors(primes=[3, 101, 65521, 67108859, 94906249]))
def test_fp64_equals_python_integers(v):
    p, a, b = v
    assert oracle.dot_fp64(p, np.array(a, np.float64), np.array(b, np.float64)) == float(bf.dot(p, a, b))


@settings(max_examples=200, deadline=None)
@given(vectors(primes=[3, 5, 7, 11, 13, 101, 257]))
def test_zech_both_accumulations_equal_python_integers(v):
    p, a, b = v
    g = bf.primitive_root(p)
    ca = [bf.zech_encode(p, g, x) for x in a]
    cb = [bf.zech_encode(p, g, x) for x in b]
    want = bf.zech_encode(p, g, bf.dot(p, a, b))
    assert oracle.dot_zech(p, g, np.array(ca, np.uint16), np.array(cb, np.uint16)) == want
    assert oracle.dot_zech_tplus1(p, g, np.array(ca, np.uint16), np.array(cb, np.uint16)) == want


@settings(max_examples=200, deadline=None)
@given(vectors(primes=[3, 101, 32749, 65521, 2147483647, 4294967291]))
def test_centered_equals_python_integers(v):
    p, a, b = v
    ca = np.array([bf.to_centered(p, x) for x in a], np.int64)
    cb = np.array([bf.to_centered(p, x) for x in b], np.int64)
    assert oracle.dot_centered(p, ca, cb) == bf.to_centered(p, bf.dot(p, a, b))


@settings(max_examples=150, deadline=None)
@given(vectors(max_n=30), st.integers(0, 2 ** 32), st.integers(0, 30))
def test_linearity_and_shard_additivity(v, c, cut):
    """dot(c a + b', b) = c dot(a, b) + dot(b', b) and dot over a split = sum of the shards' dots."""
    p, a, b = v
    cut = min(cut, len(a))
    dt = np.uint64
    lhs = oracle.dot_classical(p, np.array(a, dt), np.array(b, dt))
    parts = (oracle.dot_classical(p, np.array(a[:cut], dt), np.array(b[:cut], dt)) +
             oracle.dot_classical(p, np.array(a[cut:], dt), np.array(b[cut:], dt))) % p
    assert lhs == parts
    ca = [(c * x) % p for x in a]
    assert oracle.dot_classical(p, np.array(ca, dt), np.array(b, dt)) == (c % p) * lhs % p
    assert oracle.dot_classical(p, np.array(b, dt), np.array(a, dt)) == lhs

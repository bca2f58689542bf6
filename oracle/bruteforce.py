"""Pure-Python integer brute force for tiny inputs -- TEST INFRASTRUCTURE ONLY.

The same definition as oracle.c written with unbounded Python integers, used to pin the compiled
oracle (brute force on tiny inputs).  Exact by construction: no word size anywhere.
"""
from __future__ import annotations


def dot(p, a, b):
    """(sum a_i b_i) mod p with exact integers (sec. 3, the dot product being computed)."""
    if len(a) != len(b):
        raise ValueError("length mismatch")
    return sum(int(x) * int(y) for x, y in zip(a, b)) % p


def is_prime(n):
    return n >= 2 and all(n % d for d in range(2, int(n ** 0.5) + 1))


def primitive_root(p):
    """Smallest g whose powers enumerate all p-1 nonzero residues (set comparison)."""
    if p == 2:
        return 1
    full = set(range(1, p))
    for g in range(2, p):
        if {pow(g, k, p) for k in range(p - 1)} == full:
            return g
    raise ValueError("no primitive root")


def zech_decode(p, g, code):
    """0 -> 0, q-1 -> 1, i -> g^i (1 <= i < q-1)."""
    q = p
    if code == 0:
        return 0
    if code == q - 1:
        return 1
    return pow(g, code, p)


def zech_encode(p, g, x):
    q = p
    x %= p
    if x == 0:
        return 0
    if x == 1:
        return q - 1
    return next(i for i in range(1, q - 1) if pow(g, i, p) == x)


MONT_B = 1 << 32


def to_mont(p, a):
    return a * MONT_B % p


def from_mont(p, x):
    return x * pow(MONT_B, -1, p) % p


def to_centered(p, r):
    """sec. 3.2.2: residues above (p-1)/2 are stored as r - p."""
    r %= p
    return r - p if r > (p - 1) // 2 else r


def from_centered(p, c):
    return c % p

"""CPU oracle for the exact GF(p) dot product -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference legs) may import
this package.  It shares no code with paper_cs_0404008_b200 (the product) and never imports it.

`oracle.c` holds the compiled definition (one 128-bit remainder per term); `bruteforce.py` holds the
same definition in pure Python integers for tiny cases.  Both are pinned in tests/test_oracle_pins.py
against the paper's printed constants, closed forms, invariants and brute force.

Representation codes follow SURVEY.md 8(b): 0 classical, 1 Montgomery (B = 2^32), 2 fp64, 3 Zech.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CLASSICAL, MONTGOMERY, FP64, ZECH, CENTERED = 0, 1, 2, 3, 4
_DT = {np.dtype(np.uint16): 0, np.dtype(np.uint32): 1, np.dtype(np.uint64): 2}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", os.path.dirname(_HERE), "oracle"], check=True)
        lib = ctypes.CDLL(_LIB_PATH)
        u64, i64, vp, ci = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        sig = {
            "oracle_is_prime": (ci, [u64]),
            "oracle_pow": (u64, [u64, u64, u64]),
            "oracle_inv": (u64, [u64, u64]),
            "oracle_order": (u64, [u64, u64]),
            "oracle_primitive_root": (u64, [u64]),
            "oracle_dot_classical": (u64, [u64, vp, vp, ci, i64]),
            "oracle_dot_batch_classical": (None, [u64, vp, i64, vp, ci, i64, i64, vp]),
            "oracle_to_mont": (u64, [u64, u64]),
            "oracle_from_mont": (u64, [u64, u64]),
            "oracle_dot_montgomery": (u64, [u64, vp, vp, i64]),
            "oracle_f64_decode": (i64, [u64, vp, i64, vp]),
            "oracle_dot_fp64": (ctypes.c_double, [u64, vp, vp, i64, ctypes.POINTER(i64)]),
            "oracle_zech_powers": (None, [u64, u64, vp]),
            "oracle_zech_decode_one": (i64, [u64, u64, u64]),
            "oracle_zech_encode_one": (u64, [u64, u64, u64]),
            "oracle_dot_zech": (u64, [u64, u64, vp, vp, i64, vp, ctypes.POINTER(i64)]),
            "oracle_zech_tplus1": (None, [u64, u64, vp, vp]),
            "oracle_from_centered": (u64, [u64, i64]),
            "oracle_to_centered": (i64, [u64, u64]),
            "oracle_dot_centered": (i64, [u64, vp, vp, ci, i64, ctypes.POINTER(i64)]),
            "oracle_dot_centered_f64": (ctypes.c_double, [u64, vp, vp, i64, ctypes.POINTER(i64)]),
            "oracle_zech_mul": (u64, [u64, u64, u64]),
            "oracle_zech_add": (u64, [u64, vp, u64, u64]),
            "oracle_dot_zech_tplus1": (u64, [u64, u64, vp, vp, i64, vp, vp, ctypes.POINTER(i64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _c(arr: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(arr)


# ------------------------------------------------------------------ number theory
def is_prime(n: int) -> bool:
    return bool(_load().oracle_is_prime(n))


def pow_mod(a: int, e: int, m: int) -> int:
    return int(_load().oracle_pow(a, e, m))


def inv_mod(a: int, p: int) -> int:
    return int(_load().oracle_inv(a, p))


def order(g: int, p: int) -> int:
    return int(_load().oracle_order(g, p))


def primitive_root(p: int) -> int:
    """Smallest primitive element (sec. 2.4; reading G12)."""
    return int(_load().oracle_primitive_root(p))


# ------------------------------------------------------------------ representations
def to_mont(p: int, a: int) -> int:
    return int(_load().oracle_to_mont(p, a))


def from_mont(p: int, x: int) -> int:
    return int(_load().oracle_from_mont(p, x))


def zech_decode(p: int, g: int, code: int) -> int:
    v = int(_load().oracle_zech_decode_one(p, g, code))
    if v < 0:
        raise ValueError(f"invalid Zech code {code} for p={p}")
    return v


def zech_encode(p: int, g: int, x: int) -> int:
    return int(_load().oracle_zech_encode_one(p, g, x))


def zech_powers(p: int, g: int) -> np.ndarray:
    out = np.empty(p, dtype=np.uint64)
    _load().oracle_zech_powers(p, g, out.ctypes.data)
    return out


# ------------------------------------------------------------------ dot products
def dot_classical(p: int, a: np.ndarray, b: np.ndarray) -> int:
    a, b = _c(a), _c(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError("length or dtype mismatch")
    return int(_load().oracle_dot_classical(p, a.ctypes.data, b.ctypes.data, _DT[a.dtype], a.size))


def dot_montgomery(p: int, a: np.ndarray, b: np.ndarray) -> int:
    a, b = _c(a.astype(np.uint32, copy=False)), _c(b.astype(np.uint32, copy=False))
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    return int(_load().oracle_dot_montgomery(p, a.ctypes.data, b.ctypes.data, a.size))


def dot_fp64(p: int, a: np.ndarray, b: np.ndarray) -> float:
    a, b = _c(a.astype(np.float64, copy=False)), _c(b.astype(np.float64, copy=False))
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    bad = ctypes.c_int64(-1)
    r = float(_load().oracle_dot_fp64(p, a.ctypes.data, b.ctypes.data, a.size, ctypes.byref(bad)))
    if bad.value >= 0:
        raise ValueError(f"element {bad.value} is not an integer in [0, p)")
    return r


def dot_zech(p: int, g: int, a: np.ndarray, b: np.ndarray) -> int:
    a, b = _c(a.astype(np.uint16, copy=False)), _c(b.astype(np.uint16, copy=False))
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    pw = np.empty(p, dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    r = int(_load().oracle_dot_zech(p, g, a.ctypes.data, b.ctypes.data, a.size, pw.ctypes.data,
                                    ctypes.byref(bad)))
    if bad.value >= 0:
        raise ValueError(f"element {bad.value} is not a Zech code for p={p}")
    return r


def zech_tplus1(p: int, g: int) -> np.ndarray:
    """t_plus1[k], k = 0 .. q-1: the code of 1 + g^k (sec. 2.4; 0 when 1 + g^k = 0)."""
    t = np.empty(p, dtype=np.uint64)
    lg = np.empty(p, dtype=np.uint64)
    _load().oracle_zech_tplus1(p, g, t.ctypes.data, lg.ctypes.data)
    return t


def zech_mul(p: int, i: int, j: int) -> int:
    """Table 1 multiplication of Zech codes: i + j (- qbar)."""
    return int(_load().oracle_zech_mul(p, i, j))


def zech_add(p: int, t: np.ndarray, i: int, j: int) -> int:
    """Table 1 addition of Zech codes: k = j - i (+ qbar); i + t_plus1[k] (- qbar)."""
    return int(_load().oracle_zech_add(p, t.ctypes.data, i, j))


def dot_zech_tplus1(p: int, g: int, a: np.ndarray, b: np.ndarray) -> int:
    """Pure-Zech dot: Table 1 product and t_plus1 addition per term, result a code."""
    a, b = _c(a.astype(np.uint16, copy=False)), _c(b.astype(np.uint16, copy=False))
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    t = np.empty(p, dtype=np.uint64)
    lg = np.empty(p, dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    r = int(_load().oracle_dot_zech_tplus1(p, g, a.ctypes.data, b.ctypes.data, a.size, t.ctypes.data,
                                           lg.ctypes.data, ctypes.byref(bad)))
    if bad.value >= 0:
        raise ValueError(f"element {bad.value} is not a Zech code for p={p}")
    return r


def to_centered(p: int, r: int) -> int:
    """residue in [0, p) -> centered value in [-(p-1)/2, (p-1)/2] (sec. 3.2.2)."""
    return int(_load().oracle_to_centered(p, r))


def from_centered(p: int, c: int) -> int:
    return int(_load().oracle_from_centered(p, c))


_SDT = {np.dtype(np.int16): 0, np.dtype(np.int32): 1, np.dtype(np.int64): 2}


def dot_centered(p: int, a: np.ndarray, b: np.ndarray):
    """Dot of centered vectors (int16 / int32 / int64 / float64 storage); the result is centered, of
    the same kind (an int, or a float for binary64 storage)."""
    a, b = _c(a), _c(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError("length or dtype mismatch")
    bad = ctypes.c_int64(-1)
    if a.dtype == np.float64:
        r = float(_load().oracle_dot_centered_f64(p, a.ctypes.data, b.ctypes.data, a.size, ctypes.byref(bad)))
    else:
        r = int(_load().oracle_dot_centered(p, a.ctypes.data, b.ctypes.data, _SDT[a.dtype], a.size,
                                            ctypes.byref(bad)))
    if bad.value >= 0:
        raise ValueError(f"element {bad.value} is not a centered element for p={p}")
    return r


def dot(p: int, rep: int, a: np.ndarray, b: np.ndarray, g: int | None = None):
    """Dot product in representation `rep`; the result stays in that representation (reading G10)."""
    if rep == CLASSICAL:
        return dot_classical(p, a, b)
    if rep == MONTGOMERY:
        return dot_montgomery(p, a, b)
    if rep == FP64:
        return dot_fp64(p, a, b)
    if rep == ZECH:
        return dot_zech(p, primitive_root(p) if g is None else g, a, b)
    if rep == CENTERED:
        return dot_centered(p, a, b)
    raise ValueError(f"unknown representation {rep}")


def dot_batch_classical(p: int, A: np.ndarray, x: np.ndarray, lda: int | None = None,
                        rows: int | None = None, n: int | None = None) -> np.ndarray:
    """out[r] = (sum_j A[r*lda + j] x[j]) mod p over a flat buffer A (row-major, leading dim lda)."""
    A, x = _c(A), _c(x)
    if A.dtype != x.dtype:
        raise ValueError("dtype mismatch")
    if A.ndim == 2:
        rows_, n_ = A.shape
        lda = n_ if lda is None else lda
        rows = rows_ if rows is None else rows
        n = n_ if n is None else n
    out = np.empty(rows, dtype=np.uint64)
    _load().oracle_dot_batch_classical(p, A.ctypes.data, lda, x.ctypes.data, _DT[A.dtype], rows, n,
                                       out.ctypes.data)
    return out

"""Seeded synthetic inputs (counter-based SplitMix64), shared by tests, bench and oracle checks.

Holds none of the method's arithmetic: it only draws integers (see synth.c header).
Recipe per BASELINE.json config: DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

# seed = 0x0404008 + config index; streams: a=0, b=1, A=2, x=3
BASE_SEED = 0x0404008
STREAM_A, STREAM_B, STREAM_MAT, STREAM_X = 0, 1, 2, 3


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", os.path.dirname(_HERE), "synth"], check=True)
        lib = ctypes.CDLL(_LIB_PATH)
        u64, i64, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        lib.synth_raw.argtypes = [u64, u64, u64, i64, vp]
        for name in ("synth_uniform_u16", "synth_uniform_u32", "synth_uniform_u64", "synth_uniform_f64"):
            getattr(lib, name).argtypes = [u64, u64, u64, i64, u64, vp]
        lib.synth_zech_codes_u16.argtypes = [u64, u64, u64, i64, u64, u64, u64, vp]
        for name in ("synth_raw", "synth_uniform_u16", "synth_uniform_u32", "synth_uniform_u64",
                     "synth_uniform_f64", "synth_zech_codes_u16"):
            getattr(lib, name).restype = None
        _lib = lib
    return _lib


def _ptr(arr: np.ndarray) -> int:
    return arr.ctypes.data


def raw(seed: int, stream: int, start: int, n: int) -> np.ndarray:
    """The raw 64-bit SplitMix64 outputs h(seed, stream, start..start+n-1)."""
    out = np.empty(n, dtype=np.uint64)
    _load().synth_raw(seed, stream, start, n, _ptr(out))
    return out


def uniform(seed: int, stream: int, start: int, n: int, m: int, dtype) -> np.ndarray:
    """n integers uniform in [0, m) as `dtype` (uint16, uint32, uint64 or float64 exact integers)."""
    dtype = np.dtype(dtype)
    out = np.empty(n, dtype=dtype)
    fn = {np.dtype(np.uint16): "synth_uniform_u16", np.dtype(np.uint32): "synth_uniform_u32",
          np.dtype(np.uint64): "synth_uniform_u64", np.dtype(np.float64): "synth_uniform_f64"}[dtype]
    if dtype == np.uint16 and m > 1 << 16 or dtype == np.uint32 and m > 1 << 32 or \
            dtype == np.float64 and m > 1 << 53:
        raise ValueError("range does not fit dtype")
    getattr(_load(), fn)(seed, stream, start, n, m, _ptr(out))
    return out


def zech_codes(seed: int, stream: int, start: int, n: int, qbar: int,
               zero_num: int = 1, zero_den: int = 10) -> np.ndarray:
    """n uint16 codes: 0 w.p. zero_num/zero_den, else uniform in [1, qbar] (configs[3])."""
    if qbar >= 1 << 16:
        raise ValueError("qbar does not fit uint16 codes")
    out = np.empty(n, dtype=np.uint16)
    _load().synth_zech_codes_u16(seed, stream, start, n, qbar, zero_num, zero_den, _ptr(out))
    return out

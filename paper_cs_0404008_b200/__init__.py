"""Python binding of libgfp (include/gfp.h): the exact GF(p) dot product on B200.

Argument marshalling only: every step of the hot path runs in the CUDA kernels of libgfp.so.  The
library must be built in-tree (`make gfp`, or `python -c "import __graft_entry__ as g; g.build()"`);
importing fails loudly when it is missing -- there is no CPU fallback.

    import torch, paper_cs_0404008_b200 as gfp
    a = torch.randint(0, 65521, (10**6,), dtype=torch.int64).to(torch.uint32).cuda()
    r = gfp.dot(a, a, 65521, gfp.CLASSICAL)          # 1-element uint32 tensor on the device

Paper: arXiv cs/0404008; citations P:n are lines of its text.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "CLASSICAL", "MONTGOMERY", "FP64", "ZECH", "CENTERED", "AUTO", "DELAYED", "BLOCKED", "OVERFLOW", "HYBRID", "ZECH_ADD", "CARRY",
    "GfpError", "lib", "query", "plan", "dot", "dot_ex", "dot_batch", "dot_batch_ex",
    "dot_partial", "finalize", "to_rep", "from_rep", "dot_host", "dot_host_partial", "launch_count", "release_caches",
    "rep_dtype", "tune", "tune_entries", "tune_set", "tune_save", "tune_load", "tune_clear",
]

CLASSICAL, MONTGOMERY, FP64, ZECH, CENTERED = 0, 1, 2, 3, 4
U16, U32, F64 = 0, 1, 2
AUTO, DELAYED, BLOCKED, OVERFLOW, HYBRID = 0, 1, 2, 3, 4  # gfp_strategy (paper sec. 3)
ZECH_ADD = 5  # pure discrete-log accumulation through t_plus1 (sec. 2.4 Table 1), Zech only
CARRY = 6  # sec. 3.3 with the wrap corrections deferred: a carry word counts wraps (classical, Montgomery)
_STRAT_NAMES = {AUTO: "auto", DELAYED: "delayed", BLOCKED: "blocked", OVERFLOW: "overflow", HYBRID: "hybrid",
                ZECH_ADD: "zech_add", CARRY: "carry"}
_REP_NAMES = {CLASSICAL: "classical", MONTGOMERY: "montgomery", FP64: "fp64", ZECH: "zech", CENTERED: "centered"}

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("GFP_LIBRARY") or os.path.join(_HERE, "libgfp.so")  # override: A/B builds
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build it with `make gfp` (nvcc, sm_100a). "
                      "There is no CPU fallback.")


class GfpInfo(ctypes.Structure):
    _fields_ = [("p", ctypes.c_uint64), ("rep", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("bound", ctypes.c_uint64), ("acc_bits", ctypes.c_int32), ("mont_kr", ctypes.c_int32),
                ("k", ctypes.c_uint64), ("corr", ctypes.c_uint64), ("n_im", ctypes.c_uint32),
                ("pad0", ctypes.c_uint32), ("r2", ctypes.c_uint64), ("b_mod_p", ctypes.c_uint64),
                ("inv_p", ctypes.c_double), ("g", ctypes.c_uint64), ("qbar", ctypes.c_uint64),
                ("table_bytes", ctypes.c_uint64)]


class GfpOptions(ctypes.Structure):
    _fields_ = [("strategy", ctypes.c_int32), ("acc_bits", ctypes.c_int32), ("lanes_per_row", ctypes.c_int32)]


class GfpPlanInfo(ctypes.Structure):
    _fields_ = [("strategy", ctypes.c_int32), ("acc_bits", ctypes.c_int32), ("block", ctypes.c_uint64),
                ("grid", ctypes.c_int32), ("threads_per_block", ctypes.c_int32),
                ("terms_per_thread", ctypes.c_int64), ("reductions_per_thread", ctypes.c_int64),
                ("kernel", ctypes.c_char * 64)]


class GfpTuneCase(ctypes.Structure):
    _fields_ = [("rep", ctypes.c_int32), ("dtype", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("pad0", ctypes.c_int32), ("p", ctypes.c_uint64), ("n", ctypes.c_int64), ("rows", ctypes.c_int64)]


class GfpTuneEntry(ctypes.Structure):
    _fields_ = [("rep", ctypes.c_int32), ("dtype", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("acc_bits", ctypes.c_int32), ("pad0", ctypes.c_int32),
                ("p", ctypes.c_uint64), ("n", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("us_best", ctypes.c_double), ("us_builtin", ctypes.c_double)]


XCHG_MAX_WORLD = 16


class GfpXchg(ctypes.Structure):
    """gfp_xchg: this rank, the group size and every rank's exchange buffer as mapped in this process."""
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("peers", ctypes.c_void_p * XCHG_MAX_WORLD)]


lib = ctypes.CDLL(_LIB_PATH)
_u64, _i64, _int, _vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
_SIGS = {
    "gfp_query": [_u64, _int, _int, ctypes.POINTER(GfpInfo)],
    "gfp_dot": [_u64, _int, _int, _vp, _vp, _i64, _vp, _vp],
    "gfp_dot_batch": [_u64, _int, _int, _vp, _i64, _vp, _i64, _i64, _vp, _vp],
    "gfp_to_rep": [_u64, _int, _int, _vp, _int, _vp, _i64, _vp],
    "gfp_from_rep": [_u64, _int, _int, _vp, _int, _vp, _i64, _vp],
    "gfp_dot_partial": [_u64, _int, _int, _vp, _vp, _i64, _vp, _vp],
    "gfp_finalize": [_u64, _int, _int, _vp, _vp, _vp],
    "gfp_dot_host": [_u64, _int, _int, _vp, _vp, _i64, _vp, _vp],
    "gfp_dot_host_partial": [_u64, _int, _int, _vp, _vp, _i64, _vp, _vp],
    "gfp_dot_ex": [_u64, _int, _int, _vp, _vp, _i64, ctypes.POINTER(GfpOptions), _vp, _vp],
    "gfp_dot_batch_ex": [_u64, _int, _int, _vp, _i64, _vp, _i64, _i64, ctypes.POINTER(GfpOptions), _vp, _vp],
    "gfp_plan": [_u64, _int, _int, _i64, ctypes.POINTER(GfpOptions), ctypes.POINTER(GfpPlanInfo)],
    "gfp_tune": [ctypes.POINTER(GfpTuneCase), ctypes.c_int32, ctypes.c_double, _vp],
    "gfp_tune_entries": [ctypes.POINTER(GfpTuneEntry), ctypes.c_int32],
    "gfp_tune_set": [ctypes.POINTER(GfpTuneEntry), ctypes.c_int32],
    "gfp_tune_save": [ctypes.c_char_p],
    "gfp_tune_load": [ctypes.c_char_p],
    "gfp_xchg_create": [ctypes.POINTER(_vp), _vp],
    "gfp_xchg_open": [_vp, ctypes.POINTER(_vp)],
    "gfp_xchg_close": [_vp],
    "gfp_xchg_destroy": [_vp],
    "gfp_xchg_soft_timeout": [_vp, _u64],
    "gfp_xchg_timed_out": [_vp, ctypes.POINTER(ctypes.c_int32)],
    "gfp_dot_allreduce": [_u64, _int, _int, _vp, _vp, _i64, ctypes.POINTER(GfpXchg), _vp, _vp],
    "gfp_mc_create": [ctypes.c_int32, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_u64)],
    "gfp_mc_import": [ctypes.c_int32, _u64, ctypes.c_int32, ctypes.POINTER(_vp)],
    "gfp_mc_add_device": [_vp],
    "gfp_mc_bind": [_vp],
    "gfp_mc_destroy": [_vp],
    "gfp_dot_allreduce_mc": [_u64, _int, _int, _vp, _vp, _i64, _vp, _vp, _vp],
}
for _name, _args in _SIGS.items():
    getattr(lib, _name).argtypes = _args
    getattr(lib, _name).restype = _int
lib.gfp_xchg_bytes.argtypes = []
lib.gfp_xchg_bytes.restype = _u64
lib.gfp_tune_clear.argtypes = []
lib.gfp_tune_clear.restype = None
lib.gfp_launch_count.argtypes = [_int]
lib.gfp_launch_count.restype = _u64
lib.gfp_status_str.argtypes = [_int]
lib.gfp_status_str.restype = ctypes.c_char_p
lib.gfp_last_error.argtypes = []
lib.gfp_last_error.restype = ctypes.c_char_p
lib.gfp_release_caches.argtypes = []
lib.gfp_release_caches.restype = None
lib.gfp_version.argtypes = []
lib.gfp_version.restype = ctypes.c_char_p


class GfpError(RuntimeError):
    def __init__(self, status: int):
        self.status = status
        super().__init__(f"{lib.gfp_status_str(status).decode()}: {lib.gfp_last_error().decode()}")


def _check(status: int) -> None:
    if status != 0:
        raise GfpError(status)


# storage widths of gfp_dtype; the centered representation stores signed int16 / int32 in the same widths
_TORCH_DT = {torch.uint16: U16, torch.uint32: U32, torch.float64: F64, torch.int16: U16, torch.int32: U32}
_DT_TORCH = {U16: torch.uint16, U32: torch.uint32, F64: torch.float64}


def rep_dtype(rep: int, p: int) -> torch.dtype:
    """The natural storage dtype of a representation (gfp.h table)."""
    if rep == FP64:
        return torch.float64
    if rep == MONTGOMERY:
        return torch.uint32
    if rep == ZECH:
        return torch.uint16
    if rep == CENTERED:
        return torch.int16 if p <= 65521 else torch.int32
    return torch.uint16 if p <= 65521 else torch.uint32


def _dt(t: torch.Tensor, rep: int | None = None) -> int:
    """gfp_dtype of a tensor; with `rep`, the signedness must match the representation (signed int16 /
    int32 only for the centered representation, unsigned only for the others)."""
    try:
        d = _TORCH_DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}; use uint16, uint32, int16, int32 or float64") from None
    if rep is not None and t.dtype in (torch.int16, torch.int32, torch.uint16, torch.uint32):
        signed = t.dtype in (torch.int16, torch.int32)
        if signed != (rep == CENTERED):
            raise TypeError(f"{t.dtype} storage does not match representation {_REP_NAMES.get(rep, rep)}")
    return d


def _stream(t: torch.Tensor | None, stream) -> int:
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if t is not None and t.is_cuda:
        return torch.cuda.current_stream(t.device).cuda_stream
    return 0


def _flat_cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use dot_host for host buffers)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.reshape(-1)


def query(p: int, rep: int, dtype: torch.dtype | None = None) -> dict:
    """Host-side constants and bounds for (p, rep, dtype): k, CORR, n_im, R2, invP, g, ... (gfp_query)."""
    info = GfpInfo()
    dt = _TORCH_DT[dtype if dtype is not None else rep_dtype(rep, p)]
    _check(lib.gfp_query(p, rep, dt, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in GfpInfo._fields_ if f != "pad0"}


def dot(a: torch.Tensor, b: torch.Tensor, p: int, rep: int = CLASSICAL, out: torch.Tensor | None = None,
        stream=None) -> torch.Tensor:
    """a . b over GF(p) in representation `rep`; returns a 1-element device tensor in that representation."""
    a, b = _flat_cuda(a, "a"), _flat_cuda(b, "b")
    if a.numel() != b.numel() or a.dtype != b.dtype or a.device != b.device:
        raise ValueError("a and b must have the same length, dtype and device")
    if out is None:
        out = torch.empty(1, dtype=a.dtype, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib.gfp_dot(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(), _stream(a, stream)))
    return out


def _opts(strategy, acc_bits, lanes_per_row=0):
    return ctypes.byref(GfpOptions(strategy, acc_bits, lanes_per_row))


def plan(p: int, rep: int, n: int, dtype: torch.dtype | None = None, strategy: int = AUTO,
         acc_bits: int = 0) -> dict:
    """What gfp_dot_ex would run for n terms: kernel, grid, strategy, block length, per-thread bounds."""
    info = GfpPlanInfo()
    dt = _TORCH_DT[dtype if dtype is not None else rep_dtype(rep, p)]
    _check(lib.gfp_plan(p, rep, dt, n, _opts(strategy, acc_bits), ctypes.byref(info)))
    d = {f: getattr(info, f) for f, _ in GfpPlanInfo._fields_}
    d["kernel"] = info.kernel.decode()
    d["strategy_name"] = _STRAT_NAMES.get(info.strategy, "?")
    return d


def dot_ex(a: torch.Tensor, b: torch.Tensor, p: int, rep: int = CLASSICAL, strategy: int = AUTO, acc_bits: int = 0,
           out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """dot with an explicit accumulation strategy of the paper (sec. 3) and accumulator width m."""
    a, b = _flat_cuda(a, "a"), _flat_cuda(b, "b")
    if a.numel() != b.numel() or a.dtype != b.dtype or a.device != b.device:
        raise ValueError("a and b must have the same length, dtype and device")
    if out is None:
        out = torch.empty(1, dtype=a.dtype, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib.gfp_dot_ex(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), _opts(strategy, acc_bits),
                              out.data_ptr(), _stream(a, stream)))
    return out


def dot_partial(a: torch.Tensor, b: torch.Tensor, p: int, rep: int = CLASSICAL, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """This shard's partial residue (int64 device tensor of 1 element) for a later all-reduce + finalize."""
    a, b = _flat_cuda(a, "a"), _flat_cuda(b, "b")
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValueError("a and b must have the same length and dtype")
    if out is None:
        out = torch.empty(1, dtype=torch.int64, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib.gfp_dot_partial(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(),
                                   _stream(a, stream)))
    return out


def finalize(summed: torch.Tensor, p: int, rep: int, dtype: torch.dtype, out: torch.Tensor | None = None,
             stream=None) -> torch.Tensor:
    """mod p and encode a summed partial (int64 device tensor) into the representation's dtype."""
    if summed.dtype != torch.int64 or not summed.is_cuda:
        raise ValueError("summed must be an int64 CUDA tensor")
    if out is None:
        out = torch.empty(1, dtype=dtype, device=summed.device)
    with torch.cuda.device(summed.device):
        _check(lib.gfp_finalize(p, rep, _TORCH_DT[dtype], summed.data_ptr(), out.data_ptr(), _stream(summed, stream)))
    return out


def _batch_args(A: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None, rows, n, lda):
    """Validate a batch call against the tensors' storage (so that no kernel reads or writes out of bounds)
    and return (rows, n, lda, out)."""
    if not (A.is_cuda and x.is_cuda):
        raise ValueError("A and x must be CUDA tensors")
    if A.dtype != x.dtype or A.device != x.device:
        raise ValueError("A and x must have the same dtype and device")
    if A.dim() == 2:
        if A.shape[1] > 1 and A.stride(1) != 1:
            raise ValueError("A must be row-major with unit column stride")
        rows = A.shape[0] if rows is None else rows
        n = A.shape[1] if n is None else n
        lda = A.stride(0) if lda is None else lda
    elif A.dim() == 1:
        if rows is None or n is None:
            raise ValueError("flat A needs rows and n")
        if A.numel() > 1 and A.stride(0) != 1:
            raise ValueError("flat A must be contiguous")
        lda = n if lda is None else lda
    else:
        raise ValueError("A must be 1-D (flat, with rows and n) or 2-D")
    rows, n, lda = int(rows), int(n), int(lda)
    if rows < 0 or n < 0 or lda < n:
        raise ValueError("need rows >= 0, n >= 0 and lda >= n")
    # elements reachable from A's data pointer within its storage
    avail = A.untyped_storage().nbytes() // A.element_size() - A.storage_offset()
    if rows > 0 and n > 0 and (rows - 1) * lda + n > avail:
        raise ValueError(f"A holds {avail} elements from its data pointer; rows={rows}, n={n}, lda={lda} "
                         f"needs {(rows - 1) * lda + n}")
    if not x.is_contiguous() or x.numel() < n:
        raise ValueError("x must be contiguous with at least n elements")
    if out is None:
        out = torch.empty(rows, dtype=A.dtype, device=A.device)
    elif (not out.is_cuda or out.device != A.device or out.dtype != A.dtype or not out.is_contiguous()
          or out.numel() < rows):
        raise ValueError("out must be a contiguous CUDA tensor of A's dtype and device with >= rows elements")
    return rows, n, lda, out


def dot_batch(A: torch.Tensor, x: torch.Tensor, p: int, rep: int = CLASSICAL, out: torch.Tensor | None = None,
              rows: int | None = None, n: int | None = None, lda: int | None = None, stream=None) -> torch.Tensor:
    """out[r] = A[r, :n] . x over GF(p): many independent dots / a matrix-vector product."""
    rows, n, lda, out = _batch_args(A, x, out, rows, n, lda)
    with torch.cuda.device(A.device):
        _check(lib.gfp_dot_batch(p, rep, _dt(A, rep), A.data_ptr(), lda, x.data_ptr(), rows, n, out.data_ptr(),
                                 _stream(A, stream)))
    return out


def dot_batch_ex(A: torch.Tensor, x: torch.Tensor, p: int, rep: int = CLASSICAL, strategy: int = AUTO,
                 acc_bits: int = 0, out: torch.Tensor | None = None, rows: int | None = None, n: int | None = None,
                 lda: int | None = None, stream=None, lanes_per_row: int = 0) -> torch.Tensor:
    """dot_batch with an explicit accumulation strategy (sec. 3), accumulator width and lanes per row
    (1 = one accumulator walks the whole row, as in the paper's loop; gfp.h)."""
    rows, n, lda, out = _batch_args(A, x, out, rows, n, lda)
    with torch.cuda.device(A.device):
        _check(lib.gfp_dot_batch_ex(p, rep, _dt(A, rep), A.data_ptr(), lda, x.data_ptr(), rows, n,
                                    _opts(strategy, acc_bits, lanes_per_row), out.data_ptr(), _stream(A, stream)))
    return out


def to_rep(x: torch.Tensor, p: int, rep: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Canonical residues (uint16/uint32) -> representation `rep` (Montgomery aB mod p, Zech codes, fp64)."""
    x = _flat_cuda(x, "x")
    if out is None:
        out = torch.empty(x.numel(), dtype=rep_dtype(rep, p), device=x.device)
    with torch.cuda.device(x.device):
        _check(lib.gfp_to_rep(p, rep, _dt(x, CLASSICAL), x.data_ptr(), _dt(out, rep), out.data_ptr(), x.numel(),
                              _stream(x, stream)))
    return out


def from_rep(x: torch.Tensor, p: int, rep: int, out: torch.Tensor | None = None, dtype: torch.dtype | None = None,
             stream=None) -> torch.Tensor:
    """Representation `rep` -> canonical residues (uint32 unless `dtype`/`out` says otherwise)."""
    x = _flat_cuda(x, "x")
    if out is None:
        out = torch.empty(x.numel(), dtype=dtype or torch.uint32, device=x.device)
    with torch.cuda.device(x.device):
        _check(lib.gfp_from_rep(p, rep, _dt(x, rep), x.data_ptr(), _dt(out, CLASSICAL), out.data_ptr(), x.numel(),
                                _stream(x, stream)))
    return out


def dot_host(a: torch.Tensor, b: torch.Tensor, p: int, rep: int = CLASSICAL, stream=None):
    """End to end from HOST buffers (pinned for overlap): chunked H2D + kernels + D2H of the result.

    Returns the result as a Python number in the representation (int, or float for fp64)."""
    if a.is_cuda or b.is_cuda:
        raise ValueError("dot_host takes host tensors")
    a, b = a.contiguous().reshape(-1), b.contiguous().reshape(-1)
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValueError("a and b must have the same length and dtype")
    res = torch.empty(1, dtype=a.dtype)
    s = _stream(None, stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib.gfp_dot_host(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), res.data_ptr(), s))
    return res.item() if a.dtype == torch.float64 else int(res.to(torch.int64).item())


def dot_host_partial(a: torch.Tensor, b: torch.Tensor, p: int, rep: int = CLASSICAL, stream=None) -> int:
    """dot_host for one shard of a multi-GPU dot: the shard's partial residue in the representation's
    additive form (sum it over ranks, then `finalize`), as a Python int."""
    if a.is_cuda or b.is_cuda:
        raise ValueError("dot_host_partial takes host tensors")
    a, b = a.contiguous().reshape(-1), b.contiguous().reshape(-1)
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValueError("a and b must have the same length and dtype")
    res = ctypes.c_uint64(0)
    s = _stream(None, stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib.gfp_dot_host_partial(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), ctypes.byref(res), s))
    return int(res.value)


def launch_count(reset: bool = False) -> int:
    """Kernels libgfp launched on this host thread (since the last reset)."""
    return int(lib.gfp_launch_count(1 if reset else 0))


def release_caches() -> None:
    lib.gfp_release_caches()


def version() -> str:
    return lib.gfp_version().decode()


# ------------------------------------------------------------------------------ install-time tuning (F4)
_ENTRY_FIELDS = ("rep", "dtype", "kind", "strategy", "acc_bits", "p", "n", "rows", "us_best", "us_builtin")


def _entry_dict(e) -> dict:
    d = {f: getattr(e, f) for f in _ENTRY_FIELDS}
    d["strategy_name"] = _STRAT_NAMES.get(d["strategy"], "?")
    return d


def tune(cases, ms_per_candidate: float = 20.0, device=None, stream=None) -> list:
    """Time every admissible strategy for each case on the device and keep the fastest (gfp_tune).
    cases: iterable of dicts {rep, p, n, dtype (torch dtype, default the rep's), kind ("dot"/"batch"),
    rows}.  Returns the whole tuning table (list of dicts)."""
    cs = []
    for c in cases:
        rep = c["rep"]
        dt = _TORCH_DT[c.get("dtype") or rep_dtype(rep, c["p"])]
        kind = 1 if c.get("kind", "dot") in ("batch", 1) else 0
        cs.append(GfpTuneCase(rep, dt, kind, 0, c["p"], c["n"], c.get("rows", 0) if kind else 0))
    arr = (GfpTuneCase * max(len(cs), 1))(*cs)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        _check(lib.gfp_tune(arr, len(cs), ms_per_candidate, s.cuda_stream))
    return tune_entries()


def tune_entries() -> list:
    n = lib.gfp_tune_entries(None, 0)
    arr = (GfpTuneEntry * max(n, 1))()
    n = lib.gfp_tune_entries(arr, n)
    return [_entry_dict(arr[i]) for i in range(n)]


def tune_set(entries) -> None:
    es = [GfpTuneEntry(*(e.get(f, 0) if f != "pad0" else 0 for f, _ in GfpTuneEntry._fields_)) for e in entries]
    arr = (GfpTuneEntry * max(len(es), 1))(*es)
    _check(lib.gfp_tune_set(arr, len(es)))


def tune_save(path: str) -> None:
    _check(lib.gfp_tune_save(os.fsencode(path)))


def tune_load(path: str) -> None:
    _check(lib.gfp_tune_load(os.fsencode(path)))


def tune_clear() -> None:
    lib.gfp_tune_clear()


# ------------------------------------------------------------------------------ fused multi-GPU combine
def xchg_create() -> tuple[int, bytes]:
    """This rank's exchange buffer on the current device: (device pointer, 64-byte CUDA IPC handle)."""
    buf = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64)
    _check(lib.gfp_xchg_create(ctypes.byref(buf), handle))
    return int(buf.value), bytes(handle.raw)


def xchg_open(handle: bytes) -> int:
    ptr = ctypes.c_void_p()
    _check(lib.gfp_xchg_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)))
    return int(ptr.value)


def xchg_close(ptr: int) -> None:
    _check(lib.gfp_xchg_close(ptr))


def xchg_destroy(ptr: int) -> None:
    _check(lib.gfp_xchg_destroy(ptr))


def xchg_soft_timeout(ptr: int, ns: int) -> None:
    """Arm (ns > 0) or disarm (0) the soft timeout of this rank's exchange buffer (connectivity checks only)."""
    _check(lib.gfp_xchg_soft_timeout(ptr, ns))


def xchg_timed_out(ptr: int) -> bool:
    v = ctypes.c_int32(0)
    _check(lib.gfp_xchg_timed_out(ptr, ctypes.byref(v)))
    return bool(v.value)


def dot_allreduce(a: torch.Tensor, b: torch.Tensor, p: int, rep: int, xchg: GfpXchg,
                  out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Whole-group dot of the sharded vectors in ONE launch per rank (gfp_dot_allreduce): the kernel's
    last CTA exchanges the shard partial with every peer over NVLink peer memory and encodes the result."""
    a, b = _flat_cuda(a, "a"), _flat_cuda(b, "b")
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValueError("a and b must have the same length and dtype")
    if out is None:
        out = torch.empty(1, dtype=a.dtype, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib.gfp_dot_allreduce(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), ctypes.byref(xchg),
                                     out.data_ptr(), _stream(a, stream)))
    return out


# ------------------------------------------------------------------------------ NVLS multicast combine
def mc_create(world: int) -> tuple[int, int, int]:
    """Rank 0: a multicast object for `world` devices -> (handle, POSIX fd to pass to the other ranks, bytes)."""
    h, fd, nbytes = ctypes.c_void_p(), ctypes.c_int32(-1), ctypes.c_uint64(0)
    _check(lib.gfp_mc_create(world, ctypes.byref(h), ctypes.byref(fd), ctypes.byref(nbytes)))
    return int(h.value), int(fd.value), int(nbytes.value)


def mc_import(fd: int, nbytes: int, world: int) -> int:
    h = ctypes.c_void_p()
    _check(lib.gfp_mc_import(fd, nbytes, world, ctypes.byref(h)))
    return int(h.value)


def mc_add_device(h: int) -> None:
    _check(lib.gfp_mc_add_device(h))


def mc_bind(h: int) -> None:
    _check(lib.gfp_mc_bind(h))


def mc_destroy(h: int) -> None:
    _check(lib.gfp_mc_destroy(h))


def dot_allreduce_mc(a: torch.Tensor, b: torch.Tensor, p: int, rep: int, mc: int, out: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
    """gfp_dot_allreduce through an NVLS multicast buffer (gfp_dot_allreduce_mc): one launch per rank, the
    partials reduced in the NVSwitch."""
    a, b = _flat_cuda(a, "a"), _flat_cuda(b, "b")
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValueError("a and b must have the same length and dtype")
    if out is None:
        out = torch.empty(1, dtype=a.dtype, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib.gfp_dot_allreduce_mc(p, rep, _dt(a, rep), a.data_ptr(), b.data_ptr(), a.numel(), mc,
                                        out.data_ptr(), _stream(a, stream)))
    return out

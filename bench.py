#!/usr/bin/env python
"""Benchmark of the exact GF(p) dot product on B200 (arXiv cs/0404008 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 0..4] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one pass of the hot path over the workload:
the default workload is BASELINE.json configs[2] -- GF(2^31-1), Montgomery B = 2^32, n = 2^28 u32 per
operand, sharded over N GPUs (strong scaling: the total n is fixed), converted to Montgomery form on
device before timing (the paper excludes conversions from dot timings; the conversion is
timed separately and reported under "phases").  At N = 1 a step is one gfp_dot launch (delayed-modulus
streaming + last-CTA-done reduction and encoding); at N > 1 it is one gfp_dot_allreduce launch per rank
(the shard dot whose last CTA exchanges the partial with the peers over NVLink peer memory and encodes;
--combine nccl: gfp_dot_partial, one NCCL all_reduce of the int64 partial residue, and gfp_finalize).

`value` = total terms / max-over-ranks device time (CUDA events on the launching stream, barrier and
synchronize on both sides).  The inputs (1 GiB per operand at N = 1) exceed the 126 MB L2, so no flush
is needed for the headline; configs whose inputs are smaller rotate through enough device copies that
>= 3x the L2 is streamed between two uses of the same copy.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded input generator; holds no method arithmetic)

P31 = 2 ** 31 - 1
CONFIGS = {
    0: dict(name="C1", workload="configs[0]: GF(65521) classical u32 dot, n=100000", p=65521, rep=0,
            dtype=np.uint32, n=100_000, bpt=8, kind="dot"),
    1: dict(name="C2", workload="configs[1]: GF(67108859) fp64 dot, n=10^7", p=67108859, rep=2,
            dtype=np.float64, n=10 ** 7, bpt=16, kind="dot"),
    2: dict(name="C3", workload="configs[2]: GF(2^31-1) Montgomery B=2^32 u32 dot, n=2^28, sharded",
            p=P31, rep=1, dtype=np.uint32, n=1 << 28, bpt=8, kind="dot"),
    3: dict(name="C4", workload="configs[3]: GF(32749) Zech u16 dot, n=2^26, 10% zeros", p=32749, rep=3,
            dtype=np.uint16, n=1 << 26, bpt=4, kind="dot"),
    4: dict(name="C5", workload="configs[4]: GF(65521) classical u16 matrix-vector 65536x4096, rows sharded",
            p=65521, rep=0, dtype=np.uint16, rows=65536, n=4096, bpt=2, kind="batch"),
    # configs[3] again with the paper's own Zech accumulation: t_plus1 additions, no
    # integer accumulator (gfp_dot_ex, GFP_STRAT_ZECH_ADD = 5)
    5: dict(name="C4-zech_add", workload="configs[3] with pure-Zech t_plus1 accumulation (sec. 2.4 Table 1)",
            p=32749, rep=3, dtype=np.uint16, n=1 << 26, bpt=4, kind="dot", strategy=5, inputs_of=3),
    # configs[1] in the centered representation (sec. 3.2.2): binary64 in [-(p-1)/2, (p-1)/2],
    # blocks of k = 8 instead of 2; converted on device from the same residues (conversion timed apart)
    6: dict(name="C2-centered", workload="configs[1] in the centered representation (sec. 3.2.2), binary64, k=8",
            p=67108859, rep=4, dtype=np.float64, n=10 ** 7, bpt=16, kind="dot", inputs_of=1, host_dtype=np.uint32),
    # the fused multi-GPU dot (gfp_dot_allreduce, a9) run as a one-rank group: the shard dot, the exchange
    # protocol against the rank's own buffer (release/acquire flags, parity slots) and the finalize -- what the
    # fused combine costs over a plain dot on one GPU (the NVLink hop itself needs a second GPU)
    7: dict(name="C1-fused1", workload="configs[0] through gfp_dot_allreduce as a one-rank group", p=65521, rep=0,
            dtype=np.uint32, n=100_000, bpt=8, kind="dot", inputs_of=0, fused1=True),
    8: dict(name="C3-fused1", workload="configs[2] through gfp_dot_allreduce as a one-rank group", p=P31, rep=1,
            dtype=np.uint32, n=1 << 28, bpt=8, kind="dot", inputs_of=2, fused1=True),
    # configs[4]'s shape over Zech codes (sec. 2.4; 10% zero codes as in configs[3]): the Zech matrix-vector
    # product, bound by the shared-memory gather (one random table lookup per term) -- secondary lines only
    9: dict(name="C5-zech32749", workload="configs[4] shape, 65536x4096 Zech u16 codes over GF(32749)", p=32749,
            rep=3, dtype=np.uint16, rows=65536, n=4096, bpt=2, kind="batch"),
    10: dict(name="C5-zech65521", workload="configs[4] shape, 65536x4096 Zech u16 codes over GF(65521)", p=65521,
             rep=3, dtype=np.uint16, rows=65536, n=4096, bpt=2, kind="batch"),
    # configs[2]'s size at the largest word-size prime: (p-1)^2 ~ 2^64, so a thread's sum wraps on
    # nearly every product -- the sec. 3.3 carry word (the carry flag of each 64-bit add counted)
    11: dict(name="C3-p4294967291", workload="configs[2] size, GF(4294967291) classical u32 dot, n=2^28",
             p=4294967291, rep=0, dtype=np.uint32, n=1 << 28, bpt=8, kind="dot"),
}
REP_NAMES = {0: "classical", 1: "montgomery", 2: "fp64", 3: "zech", 4: "centered"}
DTYPE_NAMES = {np.dtype(np.uint16): "u16", np.dtype(np.uint32): "u32", np.dtype(np.float64): "f64"}
L2_BYTES = 126 * 10 ** 6


# ------------------------------------------------------------------------------ environment
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_plan(gpus, env, device_count):
    """How this invocation must run `--gpus N` (one process per GPU): ("run", None) in the current process,
    ("spawn", argv-prefix) to re-exec under torchrun with N ranks, or ("fail", reason).

    - WORLD_SIZE set (the driver's torchrun form): it must equal --gpus.
    - WORLD_SIZE unset and --gpus N > 1: self-launch N ranks (torch.distributed.run, 127.0.0.1).
    - N must not exceed the visible GPUs, except in the host-logic check mode GFP_BENCH_PG_BACKEND=gloo,
      where ranks may share devices (or run without one under --dry-run)."""
    if gpus < 1:
        return "fail", f"--gpus {gpus}: need at least 1"
    gloo = env.get("GFP_BENCH_PG_BACKEND", "nccl") == "gloo"
    ws = env.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus:
            return "fail", f"WORLD_SIZE={ws} but --gpus {gpus}: launch one rank per GPU (torchrun --nproc-per-node {gpus})"
        return "run", None
    if not gloo and gpus > device_count:
        return "fail", f"--gpus {gpus} but only {device_count} CUDA device(s) visible"
    if gpus == 1:
        return "run", None
    return "spawn", [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
                     "--master-addr", "127.0.0.1", f"--master-port={free_port()}"]


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def gather_peak():
    """Achievable L1TEX data-pipe wavefronts per SM per clock with the A stream (profiles/gather_peak.json,
    measured by scripts/gather_peak.cu), else the nominal 1."""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_peak.json")) as f:
            return float(json.load(f)["lookups_plus_stream"]), "measured (profiles/gather_peak.json, scripts/gather_peak.cu)"
    except Exception:
        return 1.0, "nominal (1 wavefront per clock per SM)"


def traffic_lookup(cfg_name, world):
    """dram bytes (read+write) per launch of the dominant kernel, from a committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(f"{cfg_name}/N{world}", t.get(cfg_name))
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML every ~5 ms while running."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4, "gpu_idle": 0x1,
               "applications_clocks_setting": 0x2, "sync_boost": 0x10}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        names = [k for k, bit in self.REASONS.items() if self.reasons & bit and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ inputs
def shard(n, rank, world):
    return n * rank // world, n * (rank + 1) // world


def host_inputs(cfg, rank, world, limit=None):
    """Host arrays of this rank's shard, in the representation's *input* form (classical residues for
    Montgomery, which is converted on device; Zech codes; fp64 integers; classical residues)."""
    idx = [k for k, v in CONFIGS.items() if v is cfg][0]
    seed = synth.BASE_SEED + cfg.get("inputs_of", idx)
    p = cfg["p"]
    if cfg["kind"] == "batch":
        r0, r1 = shard(cfg["rows"], rank, world)
        n = cfg["n"]
        if limit is not None:
            r1 = min(r1, r0 + max(1, limit // n))
        if cfg["rep"] == 3:
            A = synth.zech_codes(seed, synth.STREAM_MAT, r0 * n, (r1 - r0) * n, p - 1)
            x = synth.zech_codes(seed, synth.STREAM_X, 0, n, p - 1)
        else:
            A = synth.uniform(seed, synth.STREAM_MAT, r0 * n, (r1 - r0) * n, p, cfg["dtype"])
            x = synth.uniform(seed, synth.STREAM_X, 0, n, p, cfg["dtype"])
        return {"A": A.reshape(r1 - r0, n), "x": x, "rows": r1 - r0}
    s0, s1 = shard(cfg["n"], rank, world)
    if limit is not None:
        s1 = min(s1, s0 + limit)
    if cfg["rep"] == 3:
        a = synth.zech_codes(seed, synth.STREAM_A, s0, s1 - s0, p - 1)
        b = synth.zech_codes(seed, synth.STREAM_B, s0, s1 - s0, p - 1)
    else:
        hdt = cfg.get("host_dtype", cfg["dtype"])  # residues; converted on device when they differ
        a = synth.uniform(seed, synth.STREAM_A, s0, s1 - s0, p, hdt)
        b = synth.uniform(seed, synth.STREAM_B, s0, s1 - s0, p, hdt)
    return {"a": a, "b": b}


def graph_ms(fn, stream, per_graph=5, replays=4):
    """Milliseconds per call of fn() (device work on `stream`), timed as CUDA-graph replays of per_graph calls
    with CUDA events on the stream (no host launch gaps between the calls)."""
    with torch.cuda.stream(stream):
        fn()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(per_graph):
                fn()
        g.replay()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(replays):
            g.replay()
        e1.record(stream)
        stream.synchronize()
    return e0.elapsed_time(e1) / (per_graph * replays)


def to_device(gfp, cfg, h, dev, stream):
    """Device tensors in the representation; Montgomery conversion timed here (phase a2)."""
    p, rep = cfg["p"], cfg["rep"]
    phases = {}
    if cfg["kind"] == "batch":
        d = {"A": torch.from_numpy(h["A"]).to(dev), "x": torch.from_numpy(h["x"]).to(dev)}
        torch.cuda.synchronize()
        return d, phases
    a = torch.from_numpy(h["a"]).to(dev)
    b = torch.from_numpy(h["b"]).to(dev)
    torch.cuda.synchronize()  # copies ran on the default stream; the kernels run on `stream`
    if rep in (1, 4):  # Montgomery a -> aB mod p / centered r -> r or r - p, on device
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.uint32): torch.uint32,
               np.dtype(np.uint16): torch.uint16}[np.dtype(cfg["dtype"])] if rep == 1 else torch.float64
        am = torch.empty(a.numel(), dtype=tdt, device=a.device)
        bm = torch.empty(b.numel(), dtype=tdt, device=b.device)
        ms = graph_ms(lambda: (gfp.to_rep(a, p, rep, out=am, stream=stream),
                               gfp.to_rep(b, p, rep, out=bm, stream=stream)), stream)
        nbytes = 2 * a.numel() * (a.element_size() + am.element_size())  # read + write per element per operand
        if rep == 1:
            phases["to_montgomery"] = {"ms_per_pair": ms, "GB/s": nbytes / ms / 1e6,
                                       "note": "a -> aB mod p for both operands (P:83-84); excluded from the dot "
                                               "timing as in the paper (P:313-320)"}
        else:
            phases["to_centered"] = {"ms_per_pair": ms, "GB/s": nbytes / ms / 1e6,
                                     "note": "u32 residues -> centered binary64 for both operands (P:394-398); "
                                             "excluded from the dot timing (P:313-320)"}
        del a, b
        return {"a": am, "b": bm}, phases
    if rep == 3:  # Zech codes <-> residues with the tables staged in shared memory (a2), timed separately
        res = torch.empty_like(a)
        back = torch.empty_like(a)
        with torch.cuda.stream(stream):
            gfp.from_rep(a, p, rep, out=res, stream=stream)
            gfp.to_rep(res, p, rep, out=back, stream=stream)
            stream.synchronize()
            if not torch.equal(back, a):
                raise RuntimeError("Zech conversion round trip changed the codes")
        res_b = torch.empty_like(b)
        back_b = torch.empty_like(b)
        ms_from = graph_ms(lambda: (gfp.from_rep(a, p, rep, out=res, stream=stream),
                                    gfp.from_rep(b, p, rep, out=res_b, stream=stream)), stream)
        ms_to = graph_ms(lambda: (gfp.to_rep(res, p, rep, out=back, stream=stream),
                                  gfp.to_rep(res_b, p, rep, out=back_b, stream=stream)), stream)
        if not (torch.equal(back, a) and torch.equal(back_b, b)):
            raise RuntimeError("Zech conversion round trip changed the codes")
        nbytes = 2 * a.numel() * 2 * a.element_size()
        for name, ms, what in [("from_zech", ms_from, "code c -> g^c (antilog table)"),
                               ("to_zech", ms_to, "residue x -> log_g x (log table)")]:
            phases[name] = {"ms_per_pair": ms, "GB/s": nbytes / ms / 1e6,
                            "note": what + " for two operands of u16 (P:126-131), tables in shared memory; "
                                    "excluded from the dot timing (P:313-320); CUDA-graph replay"}
        del res, back, res_b, back_b
    return {"a": a, "b": b}, phases


# ------------------------------------------------------------------------------ one step
def replicas(d, nbytes):
    """Enough copies of the device inputs that cycling through them touches >= 3x the L2 between reuses
    (timing rule: inputs larger than L2); the headline configs need a single copy."""
    R = max(1, -(-3 * L2_BYTES // max(nbytes, 1)))
    return [d] + [{k: v.clone() for k, v in d.items()} for _ in range(R - 1)]


def make_step(gfp, cfg, reps, world, group, stream, xchg=None):
    """One step of the hot path.  N > 1 single dots: the fused combine (one kernel per rank: shard dot +
    peer-memory exchange + finalize, `xchg` a PeerExchange) or, with xchg None, gfp_dot_partial + one NCCL
    all_reduce of 8 bytes + gfp_finalize."""
    from paper_cs_0404008_b200 import dist as gfp_dist
    p, rep = cfg["p"], cfg["rep"]
    ev = []  # (start, end) events around the dominant kernel of each step
    it = [0]

    def nxt():
        d = reps[it[0] % len(reps)]
        it[0] += 1
        return d
    if cfg["kind"] == "batch":
        out = torch.empty(reps[0]["A"].shape[0], dtype=reps[0]["A"].dtype, device=reps[0]["A"].device)

        def step(record=True):
            d = nxt()
            if record:
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
            gfp.dot_batch(d["A"], d["x"], p, rep, out=out, stream=stream)
            if record:
                e.record(stream)
                ev.append((s, e))
        return step, ev, out
    a0 = reps[0]["a"]
    out = torch.empty(1, dtype=a0.dtype, device=a0.device)
    partial = torch.empty(1, dtype=torch.int64, device=a0.device)

    def step(record=True):
        d = nxt()
        a, b = d["a"], d["b"]
        if record:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
        if xchg is not None:
            gfp_dist.dot_fused(a, b, p, rep, xchg, out=out, stream=stream)
        elif world == 1 and cfg.get("strategy"):
            gfp.dot_ex(a, b, p, rep, strategy=cfg["strategy"], out=out, stream=stream)
        elif world == 1:
            gfp.dot(a, b, p, rep, out=out, stream=stream)
        else:
            gfp.dot_partial(a, b, p, rep, out=partial, stream=stream)
        if record:
            e.record(stream)
            ev.append((s, e))
        if world > 1 and xchg is None:
            gfp_dist.combine_partials(partial, group)  # one all_reduce(SUM) of 8 bytes over NCCL
            gfp.finalize(partial, p, rep, a.dtype, out=out, stream=stream)
    return step, ev, out


def time_steps(step, stream, K, W, world, record=True):
    """W untimed steps, then K steps between two CUDA events on the launching stream (barrier + synchronize
    on both sides).  record=False: no per-step events inside the region, so back-to-back launches keep their
    programmatic-dependent-launch overlap (an event between two kernels serialises them)."""
    for _ in range(W):
        step(record=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        step(record=record)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    return ms


def max_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def kernel_name(gfp, cfg, terms):
    """The kernel AUTO runs for this workload (gfp_plan: the plan a dot of `terms` elements gets)."""
    if cfg["kind"] == "batch":
        return "batch_cl16_kernel" if cfg["rep"] == 0 and np.dtype(cfg["dtype"]) == np.uint16 else "batch_kernel"
    try:
        tdt = {np.dtype(np.uint16): torch.uint16, np.dtype(np.uint32): torch.uint32,
               np.dtype(np.float64): torch.float64}[np.dtype(cfg["dtype"])]
        pl = gfp.plan(cfg["p"], cfg["rep"], int(terms), dtype=tdt, strategy=cfg.get("strategy", 0))
        return f"{pl['kernel']} (grid {pl['grid']})"
    except Exception:  # noqa: BLE001 -- the label is informative only
        return cfg["name"]


# ------------------------------------------------------------------------------ oracle legs
def host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_batch(p, rep, A, x):
    """The oracle's rows of A . x: classical residues, or Zech codes (one oracle Zech dot per row)."""
    import oracle
    if rep == 3:
        g = oracle.primitive_root(p)
        return np.array([oracle.dot_zech(p, g, A[r], x) for r in range(A.shape[0])], dtype=np.uint64)
    return oracle.dot_batch_classical(p, A, x)


def oracle_slice(cfg, h, lo, hi):
    """The oracle, as it stands, on elements (rows for the batch) [lo, hi) of the sample."""
    import oracle
    p, rep = cfg["p"], cfg["rep"]
    if cfg["kind"] == "batch":
        return oracle_batch(p, rep, h["A"][lo:hi], h["x"])
    a, b = h["a"][lo:hi], h["b"][lo:hi]
    if rep == 0:
        return oracle.dot_classical(p, a, b)
    if rep == 1:
        return oracle.dot_montgomery(p, a, b)
    if rep == 2:
        return oracle.dot_fp64(p, a, b)
    if rep == 4:
        return oracle.dot_centered(p, a, b)
    return oracle.dot_zech(p, 2, a, b)


def oracle_time_threads(cfg, h, m, threads, single=None):
    """The same oracle on the same m-element (m-row) sample, split into `threads` contiguous slices run
    concurrently (the ctypes calls release the GIL): terms/s over the whole sample.  When the single-thread
    result is given, the slices' results are combined and checked against it (additive representations;
    the batch's rows are concatenated)."""
    from concurrent.futures import ThreadPoolExecutor
    bounds = [(m * t // threads, m * (t + 1) // threads) for t in range(threads)]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda lh: oracle_slice(cfg, h, lh[0], min(lh[1], lh[0] + 1024)), bounds))  # warm
        t0 = time.perf_counter()
        parts = list(ex.map(lambda lh: oracle_slice(cfg, h, lh[0], lh[1]), bounds))
        dt = time.perf_counter() - t0
    terms = m * (cfg["n"] if cfg["kind"] == "batch" else 1)
    ok = None
    if single is not None:
        if cfg["kind"] == "batch":
            ok = bool(np.array_equal(np.concatenate(parts), single))
        elif cfg["rep"] in (0, 1, 2):  # classical / Montgomery form / fp64 integer: residues add
            ok = int(sum(int(v) for v in parts) % cfg["p"]) == int(single)
    return terms / dt, ok


def oracle_time(cfg, h, budget_s=10.0, full_ok=True):
    """Time the CPU oracle (as it stands, one thread) on a bounded prefix sample of the workload.
    Returns (terms/s, sample description, result-on-sample, sample_terms)."""
    import oracle
    p, rep = cfg["p"], cfg["rep"]
    if cfg["kind"] == "batch":
        A, x = h["A"], h["x"]

        def run(rows):
            return oracle_batch(p, rep, A[:rows], x)
        t0 = time.perf_counter()
        run(64)
        per_row = (time.perf_counter() - t0) / 64
        rows = int(min(A.shape[0], max(64, budget_s / max(per_row, 1e-9))))
        t0 = time.perf_counter()
        res = run(rows)
        dt = time.perf_counter() - t0
        terms = rows * A.shape[1]
        return terms / dt, f"first {rows} of {A.shape[0]} rows x {A.shape[1]} ({terms} terms)", res, rows

    a, b = h["a"], h["b"]

    def run(m):
        if rep == 0:
            return oracle.dot_classical(p, a[:m], b[:m])
        if rep == 1:
            return oracle.dot_montgomery(p, a[:m], b[:m])
        if rep == 2:
            return oracle.dot_fp64(p, a[:m], b[:m])
        if rep == 4:
            return oracle.dot_centered(p, a[:m], b[:m])
        return oracle.dot_zech(p, 2, a[:m], b[:m])
    m0 = min(len(a), 1 << 18)
    t0 = time.perf_counter()
    run(m0)
    per = (time.perf_counter() - t0) / max(m0, 1)
    m = int(min(len(a), max(m0, budget_s / max(per, 1e-12))))
    if not full_ok:
        m = min(m, len(a))
    t0 = time.perf_counter()
    res = run(m)
    dt = time.perf_counter() - t0
    return m / dt, f"first {m} of {len(a)} terms of this rank's shard", res, m


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true", help="skip the per-config kernel table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--combine", default="fused", choices=["fused", "nvls", "nccl"],
                    help="N > 1 single dots: one fused kernel per rank (peer stores over NVLink; nvls: multimem "
                         "reductions in the NVSwitch) or partial + NCCL all_reduce + finalize")
    ap.add_argument("--oracle-budget", type=float, default=12.0, help="seconds of oracle work per sample")
    ap.add_argument("--sweep", default=None, metavar="OUT.jsonl",
                    help="SURVEY 8(f) F1: paper-shaped prime sweep of DIM=512 batched dots per strategy, "
                         "written to OUT.jsonl (one GPU)")
    ap.add_argument("--sweep-rows", type=int, default=1 << 19,
                    help="rows per cell (2^19 x 512 u16 = 512 MiB streams from HBM; 2^15 = 32 MiB stays in L2, the "
                         "paper's cache-resident regime, where the kernels are bound by issue, not memory)")
    ap.add_argument("--sweep-graph", type=int, default=4, help="calls per captured CUDA graph")
    ap.add_argument("--sweep-reps", type=int, default=5, help="timed graph replays per cell (median reported)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check: set up the N ranks and their process group, print one JSON line with the "
                         "ranks that ran, no GPU work (CPU-testable with GFP_BENCH_PG_BACKEND=gloo)")
    args = ap.parse_args()
    if not args.sweep and args.impl == "ours":  # the reference arm is host-only (rank 0 works, others exit)
        ndev = torch.cuda.device_count()
        how, what = launch_plan(args.gpus, os.environ, ndev)
        if how == "fail":
            print(f"bench.py: {what}", file=sys.stderr, flush=True)
            raise SystemExit(2)
        if how == "spawn":  # one process per GPU: re-exec this command under torchrun
            os.execv(what[0], what + [os.path.abspath(__file__)] + sys.argv[1:])
    world, rank, local = dist_env()
    if args.dry_run:
        return dry_run(args, world, rank)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        return reference_arm(args, cfg, world, rank)
    if args.sweep:
        return prime_sweep(args)

    # GFP_BENCH_PG_BACKEND=gloo with --combine nccl: a host-logic check of the multi-rank bench on a box with
    # fewer GPUs than ranks (ranks share devices; no kernel ever waits on another rank's kernel).  Production
    # runs use NCCL, one GPU per rank.
    backend = os.environ.get("GFP_BENCH_PG_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if local >= ndev and not (backend == "gloo" and args.combine == "nccl"):
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {ndev} GPUs visible")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    import paper_cs_0404008_b200 as gfp

    stream = torch.cuda.Stream(device=dev)
    h = host_inputs(cfg, rank, world)
    d, phases = to_device(gfp, cfg, h, dev, stream)
    if cfg["kind"] == "batch":
        local_terms = d["A"].shape[0] * cfg["n"]
        local_bytes = d["A"].numel() * d["A"].element_size() + d["x"].numel() * d["x"].element_size() \
            + d["A"].shape[0] * d["A"].element_size()
    else:
        local_terms = d["a"].numel()
        local_bytes = local_terms * cfg["bpt"]
    total_terms = cfg["rows"] * cfg["n"] if cfg["kind"] == "batch" else cfg["n"]
    reps = replicas(d, local_bytes)
    xchg = None
    combine_note = None
    if cfg["kind"] == "dot" and ((world > 1 and args.combine in ("fused", "nvls")) or cfg.get("fused1")):
        from paper_cs_0404008_b200 import dist as gfp_dist
        # the exchange buffers need CUDA IPC between the ranks' processes and peer access between their GPUs
        # (nvls: a multicast team); if any rank cannot set them up, every rank falls back to the NCCL combine
        # (decided collectively)
        err = None
        try:
            if args.combine == "nvls" and world > 1:
                xchg = gfp_dist.MulticastExchange(group)
            else:
                xchg = gfp_dist.PeerExchange(group)
            if world > 1:  # one fused dot on a tiny input before the timed region: the group works end to end
                if isinstance(xchg, gfp_dist.PeerExchange):
                    if not xchg.check(dev):  # soft timeout: a broken exchange is reported, not trapped
                        raise RuntimeError("peer stores did not arrive within 10 s")
                else:
                    t = torch.ones(1024, dtype=reps[0]["a"].dtype, device=dev)
                    gfp_dist.dot_fused(t, t, cfg["p"], cfg["rep"], xchg, stream=stream)
                    torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 -- reported in the line, never silently
            err = f"{type(e).__name__}: {e}"
        if world > 1:
            flags = [None] * world
            dist.all_gather_object(flags, err)
            bad = [f for f in flags if f]
            if bad:
                if xchg is not None:
                    try:
                        xchg.close()
                    except Exception:  # noqa: BLE001
                        pass
                xchg = None
                combine_note = "fused combine unavailable, NCCL combine used: " + bad[0][:200]
                print(f"bench.py: {combine_note}", file=sys.stderr, flush=True)
        elif err:
            raise RuntimeError(err)
    step, ev, out = make_step(gfp, cfg, reps, world, group, stream, xchg)

    with torch.cuda.stream(stream):
        gfp.launch_count(reset=True)
        with ClockSampler(local) as clk:
            # one kernel per step (N = 1, or the fused combine): no per-step events; the NCCL path records
            # events around its partial kernel to separate it from the all_reduce + finalize
            per_step_events = world > 1 and xchg is None and cfg["kind"] == "dot"
            ms = time_steps(step, stream, args.steps, args.warmup, world, record=per_step_events)
        launches_total = gfp.launch_count()
    per_step = 1 if (world == 1 or cfg["kind"] == "batch" or xchg is not None) else 2
    launches_timed = launches_total - args.warmup * per_step
    if per_step_events:
        kern_avg = statistics.mean([s.elapsed_time(e) for s, e in ev[-args.steps:]])
    else:  # a step is exactly one launch of the dominant kernel: the region's events over K launches
        kern_avg = ms / args.steps
    # the distribution per launch (median and minimum), measured AFTER the timed region with a
    # pair of events around each of K more launches; the events serialise consecutive launches (no PDL
    # overlap), so these sit slightly above the back-to-back mean that `value` uses
    with torch.cuda.stream(stream):
        ev.clear()
        for _ in range(args.steps):
            step(record=True)
        torch.cuda.synchronize()
    per_launch = sorted(s_.elapsed_time(e_) for s_, e_ in ev[-args.steps:])
    launch_stats = {"median_ms": round(statistics.median(per_launch), 5), "min_ms": round(per_launch[0], 5),
                    "max_ms": round(per_launch[-1], 5), "back_to_back_mean_ms": round(kern_avg, 5), "n": len(per_launch),
                    "timing": "CUDA events around each of K further launches of the step's dominant kernel (serialised: "
                              "no PDL overlap between consecutive launches); back_to_back_mean_ms = the timed region / K"}
    ms_max = max_over_ranks(ms, world)
    value = total_terms * args.steps / (ms_max / 1e3)
    peak, peak_src = peak_hbm()
    achieved = local_bytes / (kern_avg / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic_lookup(cfg["name"], world),
            "kernel": kernel_name(gfp, cfg, local_terms),
            "algorithmic_bytes_per_launch": local_bytes, "avg_launch_ms": round(kern_avg, 4),
            "launch_timing": ("CUDA events around each partial-dot launch" if per_step_events else
                              "CUDA events around the K back-to-back launches of the timed region / K"),
            "peak_source": peak_src, "spec_8TBps_frac": round(achieved / 8000.0, 4)}

    # ---------------------------------------------------------------- correctness of the timed result
    combine_check = None
    if world > 1 and cfg["kind"] == "dot":  # the timed combine's result vs the NCCL path, every rank
        from paper_cs_0404008_b200 import dist as gfp_dist
        with torch.cuda.stream(stream):
            ref = gfp_dist.dot(reps[0]["a"], reps[0]["b"], cfg["p"], cfg["rep"], group=group, stream=stream)
            if xchg is not None:
                got = gfp_dist.dot_fused(reps[0]["a"], reps[0]["b"], cfg["p"], cfg["rep"], xchg, stream=stream)
        torch.cuda.synchronize()
        combine_check = bool(torch.equal(got.cpu(), ref.cpu())) if xchg is not None else None
    parity = None
    cpu = None
    parity_terms = None
    if rank == 0 and not args.no_cpu:
        hh = dict(h)
        if cfg["rep"] in (1, 4):  # the oracle reads the converted vectors the GPU dotted
            hh = {"a": d["a"].cpu().numpy(), "b": d["b"].cpu().numpy()}
        # cpu_baseline is reported at N = 1 only (the contract); at N > 1 rank 0 still checks parity of its
        # shard on a short oracle sample
        tps, sample, ores, m = oracle_time(cfg, hh, args.oracle_budget if world == 1 else 0.5)
        cpu = {"value": tps, "unit": "terms/s", "cores": 1, "kind": "oracle", "sample": sample,
               "threads_note": "oracle is single-threaded C (one 128-bit remainder per term)"}
        nthr = host_threads()
        if world == 1 and nthr > 1:  # the same oracle on every host core: slices of the same sample
            mt, mt_ok = oracle_time_threads(cfg, hh, m, nthr, single=ores)
            cpu = {"value": mt, "unit": "terms/s", "cores": nthr, "kind": "oracle", "sample": sample,
                   "threads_note": f"the single-threaded C oracle run on {nthr} contiguous slices of the sample, "
                                   f"one host thread each; slices combined and checked: {mt_ok}",
                   "single_thread_value": tps, "thread_scaling": mt / tps, "cpu_model": cpu_model()}
        # parity of the GPU path on the same sample (the whole shard when the sample covers it)
        if cfg["kind"] == "batch":
            got = gfp.dot_batch(d["A"][:m], d["x"], cfg["p"], cfg["rep"]).cpu().numpy().astype(np.uint64)
            parity = bool(np.array_equal(got, ores))
        else:
            if cfg.get("strategy"):
                r = gfp.dot_ex(d["a"][:m], d["b"][:m], cfg["p"], cfg["rep"], strategy=cfg["strategy"])
            else:
                r = gfp.dot(d["a"][:m], d["b"][:m], cfg["p"], cfg["rep"])
            got = r.cpu()[0].item() if r.dtype == torch.float64 else int(r.cpu().to(torch.int64)[0])
            parity = got == ores
        cpu["parity_checked_terms"] = int(m) if cfg["kind"] == "dot" else int(m) * cfg["n"]
        if world > 1:
            parity_terms, cpu = cpu["parity_checked_terms"], None

    # ---------------------------------------------------------------- end to end (host buffers)
    want = None  # the whole-group result of the device path, for the e2e leg's check
    if cfg["kind"] == "dot":
        r = ref if world > 1 else gfp.dot(reps[0]["a"], reps[0]["b"], cfg["p"], cfg["rep"])
        want = r.cpu()[0].item() if r.dtype == torch.float64 else int(r.cpu().to(torch.int64)[0])
    e2e = e2e_leg(gfp, cfg, d, world, args.e2e_steps, stream, dev, want)

    # ---------------------------------------------------------------- secondary configs (kernel only)
    secondary = None
    if not args.no_secondary and world == 1:
        secondary = secondary_table(gfp, args, dev, stream, exclude=args.config)

    if rank == 0:
        line = {
            "metric": "GF(p) dot-product terms/sec and HBM GB/s (% of peak) at 1/2/4/8 B200",
            "value": value, "unit": "terms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE_NAMES[np.dtype(cfg["dtype"])], "data": "synthetic",
            "config": {"workload": cfg["workload"], "p": cfg["p"], "representation": REP_NAMES[cfg["rep"]],
                       "n_total": total_terms, "terms_per_rank": local_terms,
                       "parallelism": f"shard x{world}" + (((" + fused NVLS multicast combine (1 launch)"
                                                              if args.combine == "nvls" else
                                                              " + fused peer-memory combine (1 launch)")
                                                             if xchg is not None else " + NCCL all_reduce(int64)")
                                                           if world > 1 and cfg["kind"] == "dot" else ""),
                       "l2": "inputs larger than L2: %.0f MiB per rank x %d rotating copies vs 126 MB L2"
                             % (local_bytes / 2 ** 20, len(reps)),
                       "seed": synth.BASE_SEED + cfg.get("inputs_of", args.config)},
            "roofline": roof, "launch_stats": launch_stats, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_timed,
            "clocks": clk.summary(), "parity_vs_oracle": parity, "phases": phases,
            "parity_checked_terms_rank0": parity_terms,
            "combine_equals_nccl_path": combine_check, "combine_note": combine_note,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if xchg is not None:
        torch.cuda.synchronize()
        xchg.close()
    if world > 1:
        dist.destroy_process_group()


def dry_run(args, world, rank):
    """--dry-run: the rank set-up of a real run (process group over the backend the bench would use) and one
    all_gather of (rank, LOCAL_RANK, pid); rank 0 prints what ran."""
    backend = os.environ.get("GFP_BENCH_PG_BACKEND", "nccl")
    _, _, local = dist_env()
    me = {"rank": rank, "local_rank": local, "pid": os.getpid()}
    seen = [me]
    if world > 1:
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        seen = [None] * world
        dist.all_gather_object(seen, me)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_arg": args.gpus, "backend": backend if world > 1 else None,
                          "ranks": seen}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_leg(gfp, cfg, d, world, steps, stream, dev, want=None):
    """Same metric through the public API from pinned HOST buffers: per step, the host->device copy of
    the inputs, the kernels, and the device->host read of the result are inside the timed region."""
    if steps <= 0:
        return None
    p, rep = cfg["p"], cfg["rep"]
    if cfg["kind"] == "batch":
        A = d["A"].cpu().pin_memory()
        x = d["x"].cpu().pin_memory()
        res = torch.empty(A.shape[0], dtype=A.dtype).pin_memory()
        h2d = A.numel() * A.element_size() + x.numel() * x.element_size()
        d2h = res.numel() * res.element_size()

        def one():
            with torch.cuda.stream(stream):
                Ad = A.to(dev, non_blocking=True)
                xd = x.to(dev, non_blocking=True)
                o = gfp.dot_batch(Ad, xd, p, rep, stream=stream)
                res.copy_(o, non_blocking=True)
            stream.synchronize()
        terms = A.shape[0] * cfg["n"]
    else:
        a = d["a"].cpu().pin_memory()
        b = d["b"].cpu().pin_memory()
        h2d = 2 * a.numel() * a.element_size() + (8 if world > 1 else 0)
        d2h = a.element_size() + (8 if world > 1 else 0)
        part_h = torch.empty(1, dtype=torch.int64).pin_memory()
        part = torch.empty(1, dtype=torch.int64, device=dev)
        fin = torch.empty(1, dtype=a.dtype, device=dev)
        fin_h = torch.empty(1, dtype=a.dtype).pin_memory()

        def one():
            if world == 1:
                return gfp.dot_host(a, b, p, rep, stream=stream)
            # N > 1: this rank's partial residue in the representation's ADDITIVE form from host buffers
            # (gfp_dot_host_partial: never a Zech code), summed over ranks, then mod p + encode on the device
            part_h[0] = gfp.dot_host_partial(a, b, p, rep, stream=stream)
            with torch.cuda.stream(stream):
                part.copy_(part_h, non_blocking=True)
                dist.all_reduce(part)
                gfp.finalize(part, p, rep, a.dtype, out=fin, stream=stream)
                fin_h.copy_(fin, non_blocking=True)
            stream.synchronize()
            return fin_h[0].item()
        terms = a.numel()
    first = one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, world)
    total = sum_over_ranks(terms, world)
    # the e2e roofline: this rank's host->device link, measured here with a plain pinned copy
    probe = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
    dprobe = torch.empty_like(probe, device=dev)
    dprobe.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        dprobe.copy_(probe, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    link = 4 * probe.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    del probe, dprobe
    achieved = h2d * steps / dt / 1e9
    equal = None
    if want is not None and first is not None:  # the end-to-end result vs the device path's (whole-group) result
        equal = bool(first == want)
    return {"value": total * steps / dt, "unit": "terms/s", "h2d_bytes_per_step": int(h2d),
            "result_equals_device_path": equal,
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "h2d_GBps": round(achieved, 2), "h2d_copy_peak_GBps": round(link, 2),
            "link_frac": round(achieved / link, 3),
            "api": "gfp_dot_host (chunked pinned H2D overlapped with the dot kernels)"
            if cfg["kind"] == "dot" else "torch H2D + gfp_dot_batch + D2H",
            "clock": "host wall clock around synchronous calls, max over ranks"}


def lookup_wavefronts(A, lanes=32, per_vec=8, sample_rows=64):
    """Shared-memory wavefronts per warp-wide lookup for the Zech matrix-vector kernel on these codes: lane l
    of a warp decodes code k of its 16-byte vector (codes 8 (v0 + l) + k of the row), i.e. 32 codes 8 apart;
    T[c] is the u16 at byte 2c, so bank (c >> 1) & 31, and a warp lookup takes as many wavefronts as the
    most distinct 32-bit words any one bank is asked for (distinct lanes reading the same word share it)."""
    A = np.asarray(A[:sample_rows], dtype=np.int64)
    n = A.shape[1] // (lanes * per_vec) * (lanes * per_vec)
    c = A[:, :n].reshape(-1, lanes, per_vec).transpose(0, 2, 1).reshape(-1, lanes)  # (warp lookups, lanes)
    words = c >> 1
    key = np.sort(((words & 31) << 20) | words, axis=1)
    new = np.ones_like(key, dtype=bool)
    new[:, 1:] = key[:, 1:] != key[:, :-1]
    counts = np.zeros((key.shape[0], 32), dtype=np.int64)
    np.add.at(counts, (np.repeat(np.arange(key.shape[0]), lanes)[new.reshape(-1)], (key >> 20)[new]), 1)
    return float(counts.max(axis=1).mean())


def split_lookup_wavefronts(A, p, lanes=32, per_vec=8, sample_rows=64):
    """Shared-memory wavefronts per warp-wide lookup of the split-exponent Zech matrix-vector kernel
    (batch_zsplit_kernel) on these codes, from its address map: e = c - 1 (16 bits), the L lookup reads byte
    address 0x10000 | (e & 255) << 8 | 4 lane, the H lookup 0x10000 | (e >> 8) << 8 | 128 + 4 lane (p > 65281: the
    zero code reads 0xFF80 + 4 lane instead); a warp lookup takes as many wavefronts as the most distinct 32-bit
    words any bank is asked for.  Returns the mean over the L and H lookups (1.0: every lane in its own bank)."""
    A = np.asarray(A[:sample_rows], dtype=np.int64)
    n = A.shape[1] // (lanes * per_vec) * (lanes * per_vec)
    c = A[:, :n].reshape(-1, lanes, per_vec).transpose(0, 2, 1).reshape(-1, lanes)  # (warp lookups, lanes)
    e = (c - 1) & 0xFFFF
    lane4 = 4 * np.arange(lanes, dtype=np.int64)[None, :]
    addr_l = 0x10000 | ((e & 255) << 8) | lane4
    addr_h = np.where((c == 0) & (p > 65281), 0xFF80 | lane4, 0x10000 | ((e >> 8) << 8) | (128 + lane4))
    out = []
    for addr in (addr_l, addr_h):
        words = addr >> 2
        key = np.sort(((words & 31) << 20) | words, axis=1)
        new = np.ones_like(key, dtype=bool)
        new[:, 1:] = key[:, 1:] != key[:, :-1]
        counts = np.zeros((key.shape[0], 32), dtype=np.int64)
        np.add.at(counts, (np.repeat(np.arange(key.shape[0]), lanes)[new.reshape(-1)], (key >> 20)[new]), 1)
        out.append(float(counts.max(axis=1).mean()))
    return (out[0] + out[1]) / 2


def secondary_table(gfp, args, dev, stream, exclude):
    """Kernel-only throughput of every other config (1 GPU), with roofline fraction."""
    peak, _ = peak_hbm()
    table = {}
    for idx, cfg in CONFIGS.items():
        if idx == exclude:
            continue
        h = host_inputs(cfg, 0, 1)
        d, phases = to_device(gfp, cfg, h, dev, stream)
        if cfg["kind"] == "batch":
            terms = cfg["rows"] * cfg["n"]
            nbytes = d["A"].numel() * 2 + d["x"].numel() * 2 + cfg["rows"] * 2
        else:
            terms = cfg["n"]
            nbytes = terms * cfg["bpt"]
        reps = replicas(d, nbytes)
        xchg = None
        if cfg.get("fused1"):
            from paper_cs_0404008_b200 import dist as gfp_dist
            xchg = gfp_dist.PeerExchange()  # one-rank group (no process group needed)
        step, ev, out = make_step(gfp, cfg, reps, 1, None, stream, xchg)
        # short kernels are launch-bound from Python: replay a CUDA graph of `per_graph` steps (one pass
        # over the rotating copies) and time the replays; per-step time includes the in-graph launch gaps
        per_graph = max(len(reps), 8)
        with torch.cuda.stream(stream):
            for _ in range(3):
                step(record=False)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(per_graph):
                    step(record=False)
            for _ in range(2):
                g.replay()
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            R_ = max(3, 200 // per_graph)
            e0.record(stream)
            for _ in range(R_):
                g.replay()
            e1.record(stream)
            stream.synchronize()
        avg = e0.elapsed_time(e1) / (R_ * per_graph)
        K, ms = R_ * per_graph, e0.elapsed_time(e1)
        table[cfg["name"]] = {"workload": cfg["workload"], "terms_per_s": terms / (avg / 1e3),
                              "us_per_step": avg * 1e3, "timing": "CUDA-graph replay of %d steps" % per_graph, "GB/s": nbytes / (avg / 1e3) / 1e9,
                              "frac_of_measured_hbm": nbytes / (avg / 1e3) / 1e9 / peak,
                              "step_terms_per_s": terms * K / (ms / 1e3),
                              "l2": f"{len(reps)} rotating input copies (>= 3x L2)"}
        if phases:
            table[cfg["name"]]["phases"] = phases
        if cfg["kind"] == "batch" and cfg["rep"] == 3:
            # the data-pipe roofline of batch_zsplit_kernel: each SM's L1TEX data pipe moves one 128-byte wavefront
            # per clock, shared by the table lookups (TWO per term, g^c = H[e >> 8] L[e & 255] with e = c - 1, each
            # a conflict-free warp lookup into the bank-replicated 256-entry tables: wavefronts per warp lookup
            # computed from the kernel's address map on these codes) and the stream of A through L1 (one wavefront
            # per 128 bytes).  HBM (2 bytes per term) is the other floor, about as low.
            wf = split_lookup_wavefronts(h["A"], cfg["p"])
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            clk = (ClockSampler(dev.index).max_mhz or 1965) * 1e6
            lookup_wf = 2 * terms / 32 * wf
            stream_wf = d["A"].numel() * d["A"].element_size() / 128
            peak_wf, peak_src = gather_peak()
            floor_us = (lookup_wf + stream_wf) / (sms * clk) * 1e6  # at the nominal 1 wavefront per clock
            roof_us = floor_us / peak_wf  # at the measured achievable rate
            table[cfg["name"]]["gather_roofline"] = {
                "bound": "l1tex_data_pipe", "kernel": "batch_zsplit_kernel", "lookups": 2 * terms,
                "wavefronts_per_warp_lookup": round(wf, 3),
                "lookup_wavefronts": int(lookup_wf), "stream_wavefronts": int(stream_wf),
                "sms": sms, "clock_mhz": clk / 1e6, "peak_wavefronts_per_clock": peak_wf, "peak_source": peak_src,
                "us": round(roof_us, 2), "frac": round(roof_us / (avg * 1e3), 4),
                "nominal_us": round(floor_us, 2), "frac_of_nominal": round(floor_us / (avg * 1e3), 4),
                "lookups_only_us": round(lookup_wf / (sms * clk) * 1e6, 2),
                "hbm_floor_us": round(nbytes / (peak * 1e9) * 1e6, 2),
                "note": "two conflict-free lookups per term (split exponent, bank-replicated 256-entry tables) plus A "
                        "streamed through L1, 1 data-pipe wavefront per clock per SM; the staged x reads (4 "
                        "wavefronts per warp and 2 rows of 256 terms) are implementation overhead, not in the floor; "
                        "the round-2 single-lookup kernel (3.37 wavefronts per lookup) had a 115.9 us floor"}
        if xchg is not None:  # the fused result must equal the plain dot's
            with torch.cuda.stream(stream):
                plain = gfp.dot(reps[0]["a"], reps[0]["b"], cfg["p"], cfg["rep"], stream=stream)
                fused = gfp_dist.dot_fused(reps[0]["a"], reps[0]["b"], cfg["p"], cfg["rep"], xchg, stream=stream)
            stream.synchronize()
            table[cfg["name"]]["equals_plain_dot"] = bool(torch.equal(plain.cpu(), fused.cpu()))
            xchg.close()
        del d, reps, step, ev, out, g
        torch.cuda.empty_cache()
    return table


def sweep_primes(gfp):
    """~48 log-spaced primes in [3, 65521] + the paper's landmarks, and word-size primes for u32 storage.
    Primality from the library's own gfp_query (GFP_E_NOT_PRIME)."""
    def prime(q):
        try:
            gfp.query(q, gfp.CLASSICAL, torch.uint32)
            return True
        except gfp.GfpError:
            return False

    def prev_prime(x):
        while x > 2 and not prime(x):
            x -= 1
        return x
    # landmarks: the paper's 2897 step (512 (p-1)^2 < 2^32, one accumulator per row) with its
    # neighbours 2887 / 2903, the same step for the default 8-lane kernel (64 terms per accumulator: 64 (p-1)^2
    # < 2^32 up to 8191, not at 8209), and the primes the paper names
    small = sorted({prev_prime(int(round(3 * (65521 / 3) ** (i / 47)))) for i in range(48)} |
                   {3, 2887, 2897, 2903, 8191, 8209, 32749, 40009, 40499, 46337, 65521})
    large = [65537, prev_prime(1 << 20), prev_prime(1 << 24), prev_prime(1 << 28), 2 ** 31 - 1, 3037000493,
             4294967291]
    return small, large


def prime_sweep(args):
    """F1: many independent length-512 dots (gfp_dot_batch_ex, classical) per prime and per strategy of the
    paper, with 32-bit accumulators where admissible (the m of Figs. 7-8) and 64-bit ones.  Each cell is
    timed by CUDA-graph replay over >= 3x L2 of rows and checked bit-for-bit against the library's
    default plan (itself oracle-checked in tests/)."""
    import paper_cs_0404008_b200 as gfp
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    small, large = sweep_primes(gfp)
    rows, n = args.sweep_rows, 512
    peak, _ = peak_hbm()
    # "auto": AUTO with the install-time table (F4); "builtin": AUTO with the table cleared (the analytic plan)
    # (column, strategy, m, lanes per row): lanes 0 = the library's choice (8 lanes for DIM = 512 rows, 64 terms
    # per accumulator); lanes 1 = ONE accumulator walks the whole row, the paper's own loop
    strategies = [("auto", gfp.AUTO, 0, 0), ("builtin", gfp.AUTO, 0, 0), ("blocked32", gfp.BLOCKED, 32, 0),
                  ("overflow32", gfp.OVERFLOW, 32, 0), ("hybrid32", gfp.HYBRID, 32, 0), ("carry32", gfp.CARRY, 32, 0),
                  ("blocked64", gfp.BLOCKED, 64, 0), ("overflow64", gfp.OVERFLOW, 64, 0), ("hybrid64", gfp.HYBRID, 64, 0),
                  ("carry64", gfp.CARRY, 64, 0),
                  ("blocked32_1lane", gfp.BLOCKED, 32, 1), ("hybrid32_1lane", gfp.HYBRID, 32, 1),
                  ("delayed64_1lane", gfp.DELAYED, 64, 1)]
    table = gfp.tune_entries()
    cells = []
    out = open(args.sweep, "w")
    for p in small + large:
        dt_np, dt_t = (np.uint16, torch.uint16) if p <= 65521 else (np.uint32, torch.uint32)
        A = torch.from_numpy(synth.uniform(synth.BASE_SEED + 5, synth.STREAM_MAT, 0, rows * n, p, dt_np)).to(dev)
        x = torch.from_numpy(synth.uniform(synth.BASE_SEED + 5, synth.STREAM_X, 0, n, p, dt_np)).to(dev)
        A = A.view(rows, n)
        torch.cuda.synchronize()
        ref = gfp.dot_batch(A, x, p, gfp.CLASSICAL)
        nbytes = A.numel() * A.element_size() + n * A.element_size() + rows * A.element_size()
        for name, strat, m, lanes in strategies:
            if name == "builtin":
                gfp.tune_clear()
            elif name == "blocked32":
                gfp.tune_set(table)
            try:
                pl = gfp.plan(p, gfp.CLASSICAL, n, dtype=dt_t, strategy=strat, acc_bits=m)
            except gfp.GfpError:
                continue
            o = torch.empty(rows, dtype=dt_t, device=dev)
            with torch.cuda.stream(stream):
                gfp.dot_batch_ex(A, x, p, gfp.CLASSICAL, strategy=strat, acc_bits=m, out=o, stream=stream,
                                 lanes_per_row=lanes)
                stream.synchronize()
                ok = bool(torch.equal(o, ref))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(args.sweep_graph):
                        gfp.dot_batch_ex(A, x, p, gfp.CLASSICAL, strategy=strat, acc_bits=m, out=o, stream=stream,
                                         lanes_per_row=lanes)
                g.replay()
                g.replay()
                stream.synchronize()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.sweep_reps + 1)]
                evs[0].record(stream)
                for r_ in range(args.sweep_reps):
                    g.replay()
                    evs[r_ + 1].record(stream)
                stream.synchronize()
            per_call = sorted(evs[r_].elapsed_time(evs[r_ + 1]) * 1e3 / args.sweep_graph for r_ in range(args.sweep_reps))
            us = statistics.median(per_call)
            blk = pl["block"] if pl["block"] else None
            # lanes the batch kernel gives a DIM = 512 row: the caller's choice, else 8 (n / W < 256 vectors)
            L = lanes if lanes else 8
            tpl = -(-n // L)  # terms one accumulator sums
            cell = {"p": p, "strategy": name, "acc_bits": pl["acc_bits"], "block_k": blk, "lanes_per_row": L,
                    "reductions_per_dim512_sequential": (None if not blk else -(-n // blk)) if name != "auto" else 1,
                    "terms_per_lane": tpl,
                    "reductions_per_lane": (None if not blk else -(-tpl // blk)),
                    "us": us, "us_min": per_call[0], "us_max": per_call[-1], "rows": rows,
                    "terms_per_s": rows * n / (us / 1e6), "GB/s": nbytes / (us / 1e6) / 1e9,
                    "frac_of_measured_hbm": nbytes / (us / 1e6) / 1e9 / peak, "equal_to_default": ok}
            cells.append(cell)
            out.write(json.dumps(cell) + "\n")
            out.flush()
        del A, x, ref
        torch.cuda.empty_cache()
    out.close()
    bad = [c for c in cells if not c["equal_to_default"]]
    summary = {"sweep": args.sweep, "cells": len(cells), "primes": len(small) + len(large), "dim": n, "rows": rows,
               "all_equal_to_default": not bad,
               "min_terms_per_s": min(c["terms_per_s"] for c in cells),
               "max_terms_per_s": max(c["terms_per_s"] for c in cells)}
    print(json.dumps(summary), flush=True)


def reference_arm(args, cfg, world, rank):
    """--impl reference: the CPU oracle as it stands (there is no reference code for this paper), timed on
    the host, each step a bounded sample of the same workload.  Rank 0 only; other ranks exit 0."""
    if rank != 0:
        return
    h = host_inputs(cfg, 0, 1, limit=1 << 24)
    if cfg["rep"] == 1:  # Montgomery form a*2^32 mod p of the sample, prepared on the host (p < 2^32)
        p = np.uint64(cfg["p"])
        h = {k: ((v.astype(np.uint64) << np.uint64(32)) % p).astype(np.uint32) for k, v in h.items()}
    budget = max(0.5, min(args.oracle_budget, 60.0 / max(args.steps + args.warmup, 1)))
    # the sample is sized on one thread (about `budget` seconds); each step then runs the same oracle on
    # that sample split over every host core (oracle_time_threads)
    nthr = host_threads()
    st, desc, ores, m = oracle_time(cfg, h, budget)
    vals = []
    checks = []
    for i in range(args.warmup + args.steps):
        tps, ok = oracle_time_threads(cfg, h, m, nthr, single=ores if i == 0 else None)
        if ok is not None:
            checks.append(ok)
        if i >= args.warmup:
            vals.append(tps)
    value = statistics.mean(vals)
    sample_terms = m if cfg["kind"] == "dot" else m * cfg["n"]
    line = {"impl": "reference", "metric": "GF(p) dot-product terms/sec and HBM GB/s (% of peak) at 1/2/4/8 B200",
            "value": value, "unit": "terms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sample_terms / value * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE_NAMES[np.dtype(cfg["dtype"])], "data": "synthetic",
            "config": {"workload": cfg["workload"], "p": cfg["p"], "representation": REP_NAMES[cfg["rep"]],
                       "n_total": cfg["n"] if cfg["kind"] == "dot" else cfg["rows"] * cfg["n"]},
            "cpu_baseline": {"value": value, "unit": "terms/s", "cores": nthr, "kind": "oracle", "sample": desc,
                             "single_thread_value": st, "cpu_model": cpu_model(),
                             "threads_note": "the single-threaded C oracle on "
                             f"{nthr} contiguous slices of the sample, one host thread each; combined result "
                             f"checked against one thread: {checks[0] if checks else None}"},
            "e2e": {"value": value, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "no reference implementation exists (paper only); the reference arm is the CPU oracle"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise an ncu --set full report (read here, no GPU needed) into a small text file for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep profiles/r01_c3_dot_full.txt [--traffic KEY]

--traffic KEY also records dram bytes (read + write) per launch into profiles/traffic.json under KEY,
which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_key = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary of {os.path.basename(rep)}", ""]
    traffic = []
    for v in vals:
        rec = dict(zip(hdr, v))
        lines.append(f"kernel: {rec.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k:85s} {v[i]:>18s} {units[i]}")
        try:
            r = float(rec["dram__bytes_read.sum"]) * scale(units[hdr.index("dram__bytes_read.sum")])
            w = float(rec["dram__bytes_write.sum"]) * scale(units[hdr.index("dram__bytes_write.sum")])
            traffic.append(r + w)
            lines.append(f"  dram bytes read+write per launch: {r + w:.0f}")
        except (KeyError, ValueError):
            pass
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_key and traffic:
        path = os.environ.get("TRAFFIC_JSON") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                              "profiles", "traffic.json")
        t = json.load(open(path)) if os.path.exists(path) else {}
        t[traffic_key] = int(sum(traffic) / len(traffic))
        json.dump(t, open(path, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


if __name__ == "__main__":
    main()

"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`, optionally gzipped) per kernel:
launches, total us, mean us, share of all profiled kernel time (cold-cache, serialised), plus the
headline kernel's per-launch statistics on the full 2^28 shard.

    python scripts/launch_summary.py gpurun_out/r01d_launches.csv.gz TAG > profiles/TAG_launches_summary.txt
"""
import csv
import gzip
import io
import sys
from collections import OrderedDict


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        text = f.read()
    start = text.index('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def main():
    path, tag = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "?"
    per = OrderedDict()
    head = []
    for r in rows(path):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"]
        per.setdefault(name, []).append(ns)
        if name.startswith("void gfp::dot_kernel<") and "Montgomery<2>" in name.split(",")[0] and ns > 150e3:
            head.append(ns)
    total = sum(sum(v) for v in per.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 4000, command: python bench.py (default), "
          f"evidence tag {tag}")
    print("# per kernel: launches, total us, mean us, share of all profiled kernel time (cold-cache, serialised)")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name[:90]:90s} {len(v):6d} {sum(v) / 1e3:12.1f} {sum(v) / len(v) / 1e3:10.2f} "
              f"{100 * sum(v) / total:6.2f}%")
    if head:
        mean = sum(head) / len(head)
        print(f"\n# headline step kernel dot_kernel<Montgomery<2>> on the full 2^28 shard: {len(head)} launches, "
              f"mean {mean / 1e3:.1f} us, min {min(head) / 1e3:.1f}, max {max(head) / 1e3:.1f} -> "
              f"{2 ** 31 / mean:.0f} GB/s; share of the N=1 step: 100% (a step is exactly one launch of this kernel)")


if __name__ == "__main__":
    main()

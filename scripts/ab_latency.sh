#!/bin/bash
# A/B of library builds on small-n per-call latency (scripts/small_n_latency.py), interleaved 2x.
for i in 1 2; do
  for v in "$@"; do
    echo "== $v"; GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python scripts/small_n_latency.py 2>/dev/null
  done
done

#!/bin/bash
# A/B of library builds on the headline (bench.py default timing: back-to-back launches), interleaved x3.
for i in 1 2 3; do
  for v in "$@"; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --no-secondary --no-cpu --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'C3 %.1f us per launch, %.0f GB/s' % (d['roofline']['avg_launch_ms']*1e3, d['roofline']['achieved']))"
  done
done

#!/bin/bash
# A/B of library builds on C5 alone (bench.py --config 4: CUDA-graph replay of rotating inputs) x3.
for i in 1 2 3; do
  for v in "$@"; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --config 4 --no-cpu --no-secondary --e2e-steps 0 --steps 50 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'C5 step %.2f us launch %.2f us %.0f GB/s' % (d['ms_per_step']*1e3, d['roofline']['avg_launch_ms']*1e3, d['roofline']['achieved']))"
  done
done

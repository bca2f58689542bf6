#!/bin/bash
# A/B of library builds on the short configs (CUDA-graph replay timings of bench.py's secondary table),
# interleaved 3x.  Usage: bash scripts/ab_secondary.sh libgfp.so libgfp_early.so
mkdir -p gpurun_out
for i in 1 2; do
  for v in "$@"; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --config 0 --no-cpu --e2e-steps 0 --steps 50 2>/dev/null \
      | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'C1 %.2f us' % d['ms_per_step'] if False else 'C1 %.2f us' % (d['roofline']['avg_launch_ms']*1e3),
      ' '.join('%s %.2f' % (k, v['us_per_step']) for k, v in d['secondary'].items()))"
  done
done

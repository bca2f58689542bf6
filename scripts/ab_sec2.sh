#!/bin/bash
# A/B of library builds on the secondary table of the default run (C1 included), interleaved x2.
for i in 1 2; do
  for v in "$@"; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --no-cpu --e2e-steps 0 --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'C3 %.1f' % (d['roofline']['avg_launch_ms']*1e3), ' '.join('%s %.2f' % (k, v['us_per_step']) for k, v in d['secondary'].items()))"
  done
done

#!/bin/bash
# A/B of library builds on the headline config: dot launch time and the to_montgomery conversion phase.
for i in 1 2 3; do
  for v in "$@"; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --no-secondary --no-cpu --e2e-steps 0 --steps 30 2>/dev/null \
      | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'C3 step %.1f us launch %.1f us' % (d['ms_per_step']*1e3, d['roofline']['avg_launch_ms']*1e3), 'to_mont pair %.1f us %.0f GB/s' % (d['phases']['to_montgomery']['ms_per_pair']*1e3, d['phases']['to_montgomery']['GB/s']))"
  done
done

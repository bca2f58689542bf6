#!/bin/bash
# A/B: AUTO with the shipped install-time table vs the built-in plan (GFP_TUNE_FILE=""), same box, x3.
for i in 1 2 3; do
  for t in shipped none; do
    if [ $t = none ]; then export GFP_TUNE_FILE=""; else unset GFP_TUNE_FILE; fi
    python bench.py --no-cpu --e2e-steps 0 --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$t', 'C3 launch %.1f us' % (d['roofline']['avg_launch_ms']*1e3), ' '.join('%s %.2f' % (k, v['us_per_step']) for k, v in d['secondary'].items()))"
  done
done

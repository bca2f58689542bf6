#!/bin/bash
# A/B of library builds on the conversions: Zech phases (C4) and to_montgomery (C3).
for i in 1 2; do
  for v in "$@"; do
    a=$(GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --config 3 --no-cpu --no-secondary --e2e-steps 0 --steps 20 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join('%s %.1f us %.0f GB/s' % (k, v['ms_per_pair']*1e3, v['GB/s']) for k, v in d['phases'].items()))")
    b=$(GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --config 2 --no-cpu --no-secondary --e2e-steps 0 --steps 5 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join('%s %.1f us %.0f GB/s' % (k, v['ms_per_pair']*1e3, v['GB/s']) for k, v in d['phases'].items()))")
    echo "$v $a $b"
  done
done

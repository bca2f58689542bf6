#!/bin/bash
# A/B: headline bench with the pipelined and unpipelined integer dot kernels, interleaved 3x.
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in libgfp.so libgfp_pipe.so; do
    GFP_LIBRARY=$PWD/paper_cs_0404008_b200/$v python bench.py --no-secondary --no-cpu --e2e-steps 0 --steps 200 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,1), 'Gterms/s', d['roofline']['achieved'], 'GB/s', d['roofline']['avg_launch_ms'])"
  done
done

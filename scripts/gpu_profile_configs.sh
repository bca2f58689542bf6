#!/bin/bash
# ncu --set full of the dominant kernel of each config (one launch each), after a clean plain run.
mkdir -p gpurun_out
TAG=${TAG:-r01}
for C in ${CONFIGS:-0 1 3 4}; do
  CMD="python bench.py --config $C --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 0"
  $CMD > gpurun_out/plain_c$C.log 2>&1 || { echo "plain run failed for config $C"; cat gpurun_out/plain_c$C.log; continue; }
  ncu --set full --clock-control none --import-source on -k regex:"dot_kernel|batch" -s 3 -c 1 \
      -o gpurun_out/${TAG}_prof_c$C $CMD > gpurun_out/ncu_c$C.log 2>&1
  echo "config $C ncu rc=$?"
done

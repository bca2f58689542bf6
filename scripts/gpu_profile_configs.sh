#!/bin/bash
# ncu --set full of the dominant kernel of each config (one launch each), after a clean plain run.
# The .ncu-rep files are summarised ON THE BOX (scripts/ncu_summary.py) and removed, so gpurun_out/ stays
# under gpurun's 64 MiB copy-back limit; KEEP_REP="2" keeps the reports of the listed configs.
mkdir -p gpurun_out
TAG=${TAG:-r02}
NAMES=(C1 C2 C3 C4 C5 C4-zech_add C2-centered C1-fused1 C3-fused1 C5-zech32749 C5-zech65521 C3-p4294967291)
export TRAFFIC_JSON=gpurun_out/${TAG}_traffic.json
for C in ${CONFIGS:-0 1 3 4}; do
  CMD="python bench.py --config $C --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 0"
  $CMD > gpurun_out/plain_c$C.log 2>&1 || { echo "plain run failed for config $C"; cat gpurun_out/plain_c$C.log; continue; }
  ncu --set full --clock-control none --import-source on -k regex:"dot_kernel|batch|zech_add" -s 3 -c 1 \
      -o gpurun_out/${TAG}_prof_c$C $CMD > gpurun_out/ncu_c$C.log 2>&1
  echo "config $C ncu rc=$?"
  python scripts/ncu_summary.py gpurun_out/${TAG}_prof_c$C.ncu-rep gpurun_out/${TAG}_c${C}_${NAMES[$C]}_ncu_full.txt \
      --traffic ${NAMES[$C]} > /dev/null 2>&1
  case " ${KEEP_REP} " in *" $C "*) ;; *) rm -f gpurun_out/${TAG}_prof_c$C.ncu-rep ;; esac
done

#!/bin/bash
# Pure-Zech dot (F3) on the GPU box: parity tests, a short bench of configs[3] with GFP_STRAT_ZECH_ADD,
# and one ncu --set full capture of the kernel.  TAG names the outputs.
mkdir -p gpurun_out
TAG=${TAG:-z}
python -m pytest tests/test_gpu_zech_add.py -q -x 2>&1 | tail -2
python bench.py --config 5 --steps 20 --warmup 3 --no-secondary --e2e-steps 0 --oracle-budget 3 \
    > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err
echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}.json'))
print('terms/s %.3e  GB/s %.1f  us %.1f  parity %s' % (d['value'], d['roofline']['achieved'], d['roofline']['avg_launch_ms']*1e3, d['parity_vs_oracle']))"
if [ -n "$NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:zech_add -s 3 -c 1 -o gpurun_out/${TAG} \
      python bench.py --config 5 --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 0 > /dev/null 2>&1
  echo "ncu rc=$?"
fi

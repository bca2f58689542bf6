#!/bin/bash
# compute-sanitizer memcheck (one tool per call) on a small parity subset.
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
compute-sanitizer --tool $TOOL --error-exitcode 3 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
  -k "sweep and (7 or 101) or misaligned or empty or shard or batch_shapes or conversions_exhaustive and 101" \
  > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"; tail -5 gpurun_out/sanitize_$TOOL.log

#!/bin/bash
# compute-sanitizer (TOOL = memcheck | racecheck | synccheck | initcheck) on a small parity subset that
# touches every kernel family: classical / Montgomery / fp64 / Zech dots and conversions, the generic and
# C5 batch kernels, the pure-Zech kernel (both paths), centered, the explicit strategies and the fused
# single-rank combine.
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
SEL=${SEL:-"sweep and (7 or 101) or misaligned or empty or shard or batch_shapes or conversions_exhaustive and 101 or fused or small_primes and (101 or 2897) or zech_add_random and (101 or 40009) or degenerate or centered_unaligned or centered_conversions"}
compute-sanitizer --tool $TOOL --error-exitcode 3 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zech_add.py \
  tests/test_gpu_centered.py tests/test_gpu_strategies.py -m gpu -q -x -k "$SEL" > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"; tail -4 gpurun_out/sanitize_$TOOL.log

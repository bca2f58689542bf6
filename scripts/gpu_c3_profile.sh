set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dot_kernel -s 3 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu2.log 2>&1
echo rc=$?

#!/bin/bash
# Round evidence: GPU tests, smoke, the default bench line, its ncu launch list (gzipped), and one
# ncu --set full capture of the dominant kernel of every config, summarised on the box.
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; cat gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
gzip -f gpurun_out/${TAG}_launches.csv
TAG=${TAG} CONFIGS="${CONFIGS:-0 1 2 3 4 5 6 9 10 11}" KEEP_REP="${KEEP_REP:-2}" bash scripts/gpu_profile_configs.sh
du -sh gpurun_out

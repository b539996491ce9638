#!/bin/bash
# One GPU pass (run under gpurun from the repo root): GPU test suite, the
# default bench line, its ncu launch list, and full ncu captures of the
# SpMM / SDDMM launches of the same command.  Usage: gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputests.log 2>&1
  echo "gpu tests rc=$?"; tail -3 gpurun_out/${TAG}_gputests.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "launches rc=$?"

#!/bin/bash
# A/B of the staircase dense-corner split (run under gpurun): parity tests,
# isolated SpMM timings and the cfg4 bench window at SVTB_HYBRID_BANDS=4 / 1.
set -u
TAG=${1:-bands}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -k "dense_corner or nccl_one_rank or config4 or no_device_allocation or sp_mult" \
  > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for B in 4 1; do
  SVTB_DEBUG_HYBRID=1 SVTB_HYBRID_BANDS=$B timeout 600 python scripts/sparse_bench.py 4 64,120,128 "" 10 > gpurun_out/${TAG}_sparse_b$B.jsonl 2>&1; echo "sparse b=$B rc=$?"
done
for B in 4 1; do
  SVTB_HYBRID_BANDS=$B timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_b$B.log 2>&1; echo "bench b=$B rc=$?"
  tail -1 gpurun_out/${TAG}_bench_b$B.log > gpurun_out/${TAG}_bench_b$B.json
done

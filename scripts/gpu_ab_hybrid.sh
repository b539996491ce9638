#!/bin/bash
# A/B of the dense-corner split (run under gpurun): parity tests, isolated
# SpMM timings and the cfg4 bench window with SVTB_HYBRID=1 / 0.
set -u
TAG=${1:-hyb}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -k "dense_corner or grouped_spmm or sddmm or config_matches_oracle_fixture or config4 or no_device_allocation or full_size_batched or sp_mult" \
  > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for H in 1 0; do
  SVTB_DEBUG_HYBRID=1 SVTB_HYBRID=$H timeout 600 python scripts/sparse_bench.py 4 32,64,120,128 "" 10 > gpurun_out/${TAG}_sparse_h$H.jsonl 2>&1; echo "sparse h=$H rc=$?"
done
for H in 1 0; do
  SVTB_HYBRID=$H timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_h$H.log 2>&1; echo "bench h=$H rc=$?"
  tail -1 gpurun_out/${TAG}_bench_h$H.log > gpurun_out/${TAG}_bench_h$H.json
done

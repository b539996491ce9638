#!/bin/bash
# Development pass (run under gpurun from the repo root): targeted GPU tests,
# isolated sparse-kernel timings, a device trace of two cfg4 iterations.
set -u
TAG=${1:-dev}
K=${2:-"sddmm or sp_mult or grouped_spmm or project_low_rank or held_out or svt_run_matches"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
timeout 600 python scripts/sparse_bench.py 4 ${SB_W:-10,64,120} ${SB_K:-3,10,20,50} 10 > gpurun_out/${TAG}_sparse_cfg4.jsonl 2>&1; echo "sparse4 rc=$?"
if [ -n "${SB5:-}" ]; then
  timeout 900 python scripts/sparse_bench.py 5 ${SB5_W:-120} ${SB5_K:-10,50} 5 > gpurun_out/${TAG}_sparse_cfg5.jsonl 2>&1; echo "sparse5 rc=$?"
fi
if [ -n "${TRACE:-}" ]; then
  timeout 600 python scripts/trace_step.py --config 4 --warm 8 --iters 2 --out gpurun_out/${TAG}_trace.json > gpurun_out/${TAG}_trace.txt 2>&1; echo "trace rc=$?"
  rm -f gpurun_out/${TAG}_trace.json
fi
if [ -n "${BENCH:-}" ]; then
  timeout 900 python bench.py ${BENCH} > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
fi

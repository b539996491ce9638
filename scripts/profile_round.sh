#!/bin/bash
# Round measurement of the committed state (run under gpurun from the repo root):
#  1. bench (no profiler), config 4, all legs (timed window, e2e, CPU matched iteration)
#  2. the reference arm (CPU oracle) on the same config
#  3. ncu launch list of the same command (durations only, cold / serialised)
#  4. ncu --set full on launches of the dominant kernel (split SpMM, cold gather) inside the bench
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/${TAG}_final_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_final_bench.log > gpurun_out/${TAG}_final_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${TAG}_final_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/${TAG}_final_ref.log > gpurun_out/${TAG}_final_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_final_launches.csv \
    python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu > gpurun_out/${TAG}_final_ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_grp --launch-skip 150 -c 2 \
    -o gpurun_out/${TAG}_final_full_spmm python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu \
    > gpurun_out/${TAG}_final_ncu_full.log 2>&1; echo "full spmm rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cutlass --launch-skip 100 -c 1 \
    -o gpurun_out/${TAG}_final_full_gemm python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu \
    > gpurun_out/${TAG}_final_ncu_full_gemm.log 2>&1; echo "full gemm rc=$?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_final_tests.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python scripts/trace_step.py --config 4 --warm 8 --iters 2 --out gpurun_out/${TAG}_trace.json > gpurun_out/${TAG}_final_trace.txt 2>&1; rm -f gpurun_out/${TAG}_trace.json

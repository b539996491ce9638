#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root):
#  1. bench (no profiler) -> gpurun_out/bench_cfg4.json
#  2. ncu launch list of the same command (durations only, cold/serialised)
#  3. ncu --set full on the top kernels (DMMA TN/NN, wide SpMM, SDDMM)
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg4.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_cfg4.log > gpurun_out/bench_cfg4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:dmma_cp_kernel<.int.128, .bool.1>" --launch-skip 120 -c 1 -o gpurun_out/full_dmma_tn_cfg4 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full1.log 2>&1; echo "full tn rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:dmma_cp_kernel<.int.128, .bool.0>" --launch-skip 120 -c 1 -o gpurun_out/full_dmma_nn_cfg4 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full2.log 2>&1; echo "full nn rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:spmm_wide_kernel<.int.4>" --launch-skip 60 -c 2 -o gpurun_out/full_spmm_cfg4 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full3.log 2>&1; echo "full spmm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sddmm_update --launch-skip 3 -c 1 \
    -o gpurun_out/full_sddmm_cfg4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full4.log 2>&1
echo "full sddmm rc=$?"
# cfg5 shapes of the CGS contraction in isolation (scripts/gemm_bench.py)
ncu --set full --clock-control none --import-source on -k regex:dmma --launch-skip 3 -c 1 \
    -o gpurun_out/full_dmma_tn_cfg5 python scripts/gemm_bench.py 4 > gpurun_out/ncu_full5.log 2>&1; echo "full tn5 rc=$?"
# tcgen05 INT8 (Ozaki) FP64 contraction on the cfg4 CGS shape
ncu --set full --clock-control none --import-source on -k regex:ozaki_tn -c 1 \
    -o gpurun_out/full_ozaki_tn python scripts/ozaki_bench.py 69878x1322x120 > gpurun_out/ncu_full6.log 2>&1; echo "full ozaki rc=$?"
# cfg5 bench line (no CPU leg: an oracle iteration takes hours) and the per-config table
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg5.log 2>&1; echo "bench cfg5 rc=$?"
tail -1 gpurun_out/bench_cfg5.log > gpurun_out/bench_cfg5.json
python scripts/config_table.py 1,2,3,4 > gpurun_out/config_table.log 2>&1; echo "table rc=$?"
cp profiles/r01_config_table.json gpurun_out/config_table.json

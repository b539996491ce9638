#!/bin/bash
# Round-end measurement of the committed state (run under gpurun from the repo root)
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg4.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_cfg4.log > gpurun_out/bench_cfg4.json
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_cfg4_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:spmm_wide --launch-skip 40 -c 1 \
    -o gpurun_out/full_spmm_cfg4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_spmm.log 2>&1; echo "full spmm rc=$?"
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg5.log 2>&1; echo "bench cfg5 rc=$?"
tail -1 gpurun_out/bench_cfg5.log > gpurun_out/bench_cfg5.json
python scripts/config_table.py 1,2,3,4 > gpurun_out/config_table.log 2>&1; echo "table rc=$?"
cp profiles/r01_config_table.json gpurun_out/config_table.json

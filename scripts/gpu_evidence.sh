#!/bin/bash
# Evidence pass (run under gpurun from the repo root): isolated sparse-kernel
# timings (cfg4, cfg5), the L2 gather ceiling microbenchmark, full ncu
# captures of the CSR / CSC SpMM and the fused SDDMM update, and
# compute-sanitizer memcheck / racecheck / synccheck over small GPU tests.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 300 ./scripts/gather_probe > gpurun_out/${TAG}_gather_probe.txt 2>&1; echo "probe rc=$?"
timeout 600 python scripts/sparse_bench.py 4 10,32,64,96,120,128 3,10,20,50 10 > gpurun_out/${TAG}_sparse_cfg4.jsonl 2>&1; echo "sparse4 rc=$?"
timeout 900 python scripts/sparse_bench.py 5 10,64,120 10,50 5 > gpurun_out/${TAG}_sparse_cfg5.jsonl 2>&1; echo "sparse5 rc=$?"
NCU="ncu --set full --clock-control none --import-source on"
# launches of sparse_bench with reps=1: Y X warm, Y X timed, Y^T X warm, Y^T X timed
timeout 900 $NCU -k regex:spmm_grp --launch-skip 1 -c 3 -o gpurun_out/${TAG}_full_spmm_cfg4_w120 \
    python scripts/sparse_bench.py 4 120 "" 1 > gpurun_out/${TAG}_ncu_spmm4.log 2>&1; echo "ncu spmm4 rc=$?"
timeout 900 $NCU -k regex:"sddmm_update|mirror_csc" --launch-skip 2 -c 4 -o gpurun_out/${TAG}_full_sddmm_cfg4 \
    python scripts/sparse_bench.py 4 "" 10 1 > gpurun_out/${TAG}_ncu_sddmm4.log 2>&1; echo "ncu sddmm4 rc=$?"
timeout 1200 $NCU -k regex:"spmm_grp|sddmm_update|mirror_csc" --launch-skip 1 -c 6 -o gpurun_out/${TAG}_full_sparse_cfg5 \
    python scripts/sparse_bench.py 5 120 50 1 > gpurun_out/${TAG}_ncu_sparse5.log 2>&1; echo "ncu sparse5 rc=$?"
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9"
K="r3svd_matches or r4svd_recycled or svt_run_matches_oracle_small or rank0 or sp_mult_and_t or qr_orthonormal or small_svd_matches or batched_rounds_equal"
timeout 1500 $SAN --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "$K" \
    > gpurun_out/${TAG}_san_memcheck.log 2>&1; echo "memcheck rc=$?"
K2="sym_eig or ozaki_tn or qr_orthonormal or tiled_spmm or small_svd_matches or grouped_spmm_bitwise"
timeout 1500 $SAN --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
    -k "($K2) and not config" > gpurun_out/${TAG}_san_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 1500 $SAN --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
    -k "($K2) and not config" > gpurun_out/${TAG}_san_synccheck.log 2>&1; echo "synccheck rc=$?"

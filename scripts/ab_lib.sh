# A/B of two builds of libsvt_b200 on the same box (bench cfg4, no CPU legs)
set -u
mkdir -p gpurun_out
HEAD=paper_1704_05528_b200/lib/libsvt_b200_head.so
for i in 1 2; do
  for L in $HEAD paper_1704_05528_b200/lib/libsvt_b200.so; do
    SVTB_LIB=$PWD/$L timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log >> gpurun_out/ab_lines.jsonl
    echo "$(basename $L) $(tail -1 gpurun_out/ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), d["host"], d["config"]["rounds"], d["gpu_launches"])')"
  done
done

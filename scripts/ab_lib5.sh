# cfg5 A/B of two library builds (bench, 3 timed iterations)
set -u
for L in paper_1704_05528_b200/lib/libsvt_b200_head.so paper_1704_05528_b200/lib/libsvt_b200.so; do
  SVTB_LIB=$PWD/$L timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab5.log 2>&1
  echo "$(basename $L) $(tail -1 gpurun_out/ab5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["kernel_ms_per_step"], d["config"]["rounds"])')"
done

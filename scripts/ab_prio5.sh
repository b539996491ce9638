set -u
for x in 0 1; do
  if [ $x = 1 ]; then export SVTB_FLAT_PRIORITY=1; else unset SVTB_FLAT_PRIORITY; fi
  timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/abp5.log 2>&1
  echo "flat=$x $(tail -1 gpurun_out/abp5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["kernel_ms_per_step"])')"
done

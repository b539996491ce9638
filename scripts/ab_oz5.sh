set -u
for x in 0 1; do
  SVTB_OZAKI=$x timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/abo5.log 2>&1
  echo "ozaki=$x $(tail -1 gpurun_out/abo5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["kernel_ms_per_step"], d["host"]["device_allocs_in_timed_region"])')"
done

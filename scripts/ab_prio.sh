set -u
for i in 1 2 3 4 5; do
  for x in 0 1; do
    if [ $x = 1 ]; then export SVTB_FLAT_PRIORITY=1; else unset SVTB_FLAT_PRIORITY; fi
    timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/abp.log 2>&1
    echo "flat=$x $(tail -1 gpurun_out/abp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3))')"
  done
done

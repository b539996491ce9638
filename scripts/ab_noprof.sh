set -u
for i in 1 2 3; do
  for x in 0 1; do
    if [ $x = 1 ]; then export SVTB_BENCH_NOPROF=1; else unset SVTB_BENCH_NOPROF; fi
    timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/abn.log 2>&1
    echo "noprof=$x $(tail -1 gpurun_out/abn.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), d["host"])')"
  done
done

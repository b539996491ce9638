# A/B of an environment switch on the cfg4 bench: bash scripts/ab_env.sh VAR [config]
set -u
V=$1; CFG=${2:-4}
for i in 1 2 3; do
  for x in 0 1; do
    env $V=$x timeout 600 python bench.py --config $CFG --no-cpu --no-e2e --steps ${STEPS:-5} --warmup 3 > gpurun_out/abe.log 2>&1
    echo "$V=$x $(tail -1 gpurun_out/abe.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["kernel_ms_per_step"], d["config"]["rounds"])')"
  done
done

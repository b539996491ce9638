#!/bin/bash
# A/B helpers for bench experiments on one GPU box (run under gpurun from the
# repo root).  Each run prints iterations/s, per-class kernel ms and the
# device allocations inside the timed region.
#   bash scripts/ab.sh lib [config] [steps]      lib/libsvt_b200_head.so vs lib/libsvt_b200.so (SVTB_LIB)
#   bash scripts/ab.sh env VAR [config] [steps]  VAR=0 vs VAR=1
#   bash scripts/ab.sh repeat N [config]         N runs of the current build (run-to-run spread)
set -u
mkdir -p gpurun_out
run() {  # label, config, steps, env...
  local label=$1 cfg=$2 steps=$3; shift 3
  env "$@" timeout 1200 python bench.py --config "$cfg" --steps "$steps" --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/ab_run.log 2>&1
  echo "$label $(tail -1 gpurun_out/ab_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); \
print(round(d["value"], 4), d["kernel_ms_per_step"], "allocs", d["host"]["device_allocs_in_timed_region"])')"
}
LIBDIR=$PWD/paper_1704_05528_b200/lib
case "${1:-}" in
  lib)  for i in 1 2; do
          run head "${2:-4}" "${3:-5}" SVTB_LIB=$LIBDIR/libsvt_b200_head.so
          run new  "${2:-4}" "${3:-5}" SVTB_LIB=$LIBDIR/libsvt_b200.so
        done ;;
  env)  for i in 1 2; do
          run "$2=0" "${3:-4}" "${4:-5}" "$2=0"
          run "$2=1" "${3:-4}" "${4:-5}" "$2=1"
        done ;;
  repeat) for i in $(seq 1 "${2:-5}"); do run "run$i" "${3:-4}" 5 X=0; done ;;
  *) echo "usage: ab.sh lib|env|repeat ..."; exit 2 ;;
esac

# other compute processes / GPU utilisation on the device during bench runs
( for i in $(seq 1 400); do nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv,noheader >> gpurun_out/apps.log 2>&1; echo "--" >> gpurun_out/apps.log; sleep 0.25; done ) &
SMI=$!
NRUNS=${NRUNS:-6} bash scripts/cpu_quota_probe.sh
kill $SMI 2>/dev/null
echo "distinct pids seen:"; grep -v "^--" gpurun_out/apps.log | awk -F, '{print $1, $2}' | sort | uniq -c
nvidia-smi -q | grep -i -A3 "compute mode\|MIG mode\|Accounting\|Virtualization" | head -20

# host CPU state around bench runs (load, steal, process CPU time, context switches):
# NRUNS=8 bash scripts/host_probe.sh — used to rule out host contention as the
# cause of the sporadic slow steps (they were device-wide syncs of cudaFree)
cat /proc/loadavg
python - <<'PY'
import json, resource, subprocess, time
def stat():
    f = open('/proc/stat').readline().split()[1:]
    return [int(x) for x in f]
for i in range(int(__import__("os").environ.get("NRUNS", "3"))):
    s0 = stat(); t0 = time.time(); r0 = resource.getrusage(resource.RUSAGE_CHILDREN)
    subprocess.run("timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/probe.log 2>&1", shell=True)
    s1 = stat(); t1 = time.time(); r1 = resource.getrusage(resource.RUSAGE_CHILDREN)
    d = [b - a for a, b in zip(s0, s1)]
    tot = sum(d)
    line = open('gpurun_out/probe.log').read().strip().splitlines()[-1]
    v = json.loads(line)
    print(f"value {v['value']:.2f} hs {v['host']} wall {t1-t0:.1f}s child user {r1.ru_utime-r0.ru_utime:.1f}s sys {r1.ru_stime-r0.ru_stime:.1f}s "
          f"host cpu: user {100*d[0]/tot:.1f}% sys {100*d[2]/tot:.1f}% idle {100*d[3]/tot:.1f}% steal {100*d[7]/tot:.2f}% "
          f"| vol/invol csw {r1.ru_nvcsw-r0.ru_nvcsw}/{r1.ru_nivcsw-r0.ru_nivcsw}", flush=True)
PY
cat /proc/loadavg

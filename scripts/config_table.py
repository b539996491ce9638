"""Per-config table of BASELINE.md §3 (GPU iters/s, SpMM / SDDMM GB/s, CPU
oracle iters/s) on one B200 — the numbers DESIGN.md §6 quotes.  Writes
profiles/r01_config_table.json.  Development tool (run under gpurun)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1704_05528_b200 import api as G  # noqa: E402
from paper_1704_05528_b200._abi import KCLASS  # noqa: E402

PLAN = {  # config: (GPU iterations, timed from, oracle iterations or 0)
    1: (10, 2, 2),
    2: (20, 2, 10),
    3: (12, 2, 4),
    4: (8, 4, 1),
    5: (4, 2, 0),
}


def main():
    ctx = G.default_context()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6554.9
    configs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4, 5]
    rows = {}
    for c in configs:
        iters, t_from, o_iters = PLAN[c]
        d = G.synth_config(c, 1)
        m, n = d["m"], d["n"]
        if c == 5:
            rp, co, va = d["csr"]
            test = None
        else:
            rp, co, va = G.build_csr(m, n, *d["train"])
            test = G.build_csr(m, n, *d["test"]) if d["test"] is not None else None
        A = G.SampledMatrix.from_csr(m, n, rp, co, va)
        cfg, stop = G.config_params(c, int(rp[-1]), m, n, float(np.sqrt(np.sum(va * va))))
        cfg.maxit = iters + 1
        S = G.Solver(A, cfg, stop)
        times = []
        for i in range(iters):
            if i + 1 == t_from:
                ctx.sync()
                ctx.reset_stats()
                ctx.set_profiling(True)
            t0 = time.perf_counter()
            S.step()
            ctx.join()
            ctx.sync()
            times.append(time.perf_counter() - t0)
        stats = {KCLASS[k]: ctx.kernel_stats(k) for k in range(8)}
        ctx.set_profiling(False)
        S.close()
        timed = times[t_from - 1:]
        row = {"m": m, "n": n, "nnz": int(rp[-1]), "gpu_iters_timed": f"{t_from}-{iters}",
               "gpu_iter_per_s": len(timed) / sum(timed)}
        for k in ("spmm", "spmm_t", "sddmm_update"):
            v = stats[k]
            if v["total_ms"] > 0:
                gbs = v["bytes"] / (v["total_ms"] * 1e-3) / 1e9
                row[f"{k}_gbs"] = gbs
                row[f"{k}_frac_hbm"] = gbs / peak
        if o_iters:
            Oa = O.Csr(m, n, rp, co, va)
            cfg.maxit = o_iters
            stamps = [time.perf_counter()]
            O.svt_run(Oa, cfg, stop, observer=lambda *a: stamps.append(time.perf_counter()) or True)
            dd = np.diff(stamps)
            row["cpu_iter_per_s"] = len(dd) / float(np.sum(dd))
            row["cpu_iters"] = len(dd)
        row["host_cores_used"] = 1
        rows[c] = row
        print(c, json.dumps(row), flush=True)
        A.close()
    out = os.path.join(ROOT, "profiles", "r01_config_table.json")
    json.dump({"nproc": os.cpu_count(), "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""SVT iterations/s (R4SVD) on B200 — the BASELINE.json headline metric.

One step = one SVT Bregman iteration (solver.hpp:239-325): the R4SVD partial
SVD of the sparse iterate Y (rank-revealing rounds + finalize) followed by the
fused SDDMM + update.  Iterations are taken consecutively from the kickstart;
W warm-up iterations run untimed, then exactly K are timed with CUDA events on
the library's stream (barrier + synchronize on both sides, max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Multi-GPU (torchrun): rows of Y / Q / U are sharded by nnz across ranks; the
NCCL communicator lives inside libsvt_b200.so (torch.distributed/gloo is only
used to pass the NCCL unique id and for the host barrier / max-reduction).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

# load every kernel of libsvt_b200 at context creation: with lazy module
# loading the first launch of a template variant (e.g. a wider DMMA tile once
# the basis grows) lands inside the timed region
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = 4
CONFIG_NAMES = {
    1: "cfg1: 1000x1000 rank-10 synthetic, 20% observed",
    2: "cfg2: 512x512 blob+cosine image, 50% observed",
    3: "cfg3: 6040x3706 power-law ratings (1,000,209; 10% held out)",
    4: "cfg4: 69878x10677 power-law half-star ratings (10,000,054; 10% held out)",
    5: "cfg5: 100000x100000 rank-50, 1% observed (1e8 nnz)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle CPU work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def load_problem(config, seed):
    """Host CSR (global) for train and test sets of a BASELINE config."""
    from paper_1704_05528_b200 import api as G
    d = G.synth_config(config, seed)
    m, n = d["m"], d["n"]
    if config == 5:
        train = d["csr"]
        test = None
    else:
        train = G.build_csr(m, n, *d["train"])
        test = G.build_csr(m, n, *d["test"]) if d["test"] is not None else None
    return m, n, train, test


def frob(val):
    return float(np.sqrt(np.dot(val, val)))


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in
    process through NVML (no nvidia-smi process spawns competing with the
    host thread); falls back to nvidia-smi when NVML is unavailable."""

    def __init__(self, index=0):
        self.samples, self.index, self.stop_ev = [], index, threading.Event()
        self.th = None
        self.max_mhz = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}

        def sample():
            sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            mask = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            return sm, sorted(k for k, b in bits.items() if mask & b)
        return sample

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def sample():
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            f = [x.strip() for x in out.split(",")]
            if f[1].replace(".", "").isdigit():
                self.max_mhz = float(f[1])
            return float(f[0]), sorted(names[i] for i in range(4) if f[2 + i] == "Active")
        return sample

    def start(self):
        try:
            sample = self._nvml()
        except Exception:
            sample = self._smi()

        def run():
            while not self.stop_ev.is_set():
                try:
                    self.samples.append(sample())
                except Exception:
                    pass
                self.stop_ev.wait(0.1)

        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def stop(self):
        self.stop_ev.set()
        if self.th:
            self.th.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_fp64_peak():
    """FP64 GEMM peak (TFLOP/s): cuBLAS DGEMM measured on this pool by
    scripts/measure_fp64_peak.py (profiles/fp64_peak.json); else B200's
    nominal 40 TFLOP/s FP64 tensor-core figure."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(p) as f:
            return float(json.load(f)["fp64_tflops"]), "measured (cuBLAS DGEMM, profiles/fp64_peak.json)"
    except Exception:
        return 40.0, "nominal B200 FP64 tensor spec (no measurement file)"


# ---------------------------------------------------------------------------
def cpu_oracle_rate(config, seed, m, n, train, test, budget, max_iters):
    """Times the CPU oracle (the reference's algorithm restated in C++,
    single-threaded like the reference) on the same workload; stops after the
    iteration that crosses `budget` seconds.  Returns (iters/s, sample text)."""
    from oracle import oracle as O
    from paper_1704_05528_b200 import api as G
    rp, co, va = train
    A = O.Csr(m, n, rp, co, va)
    T = O.Csr(m, n, *test) if test is not None else None
    cfg, stop = G.config_params(config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = max_iters
    stamps = []
    t0 = time.perf_counter()

    def obs(rec, U, s, V):
        stamps.append(time.perf_counter())
        return (time.perf_counter() - t0) < budget

    O.svt_run(A, cfg, stop, observer=obs, test=T)
    its = len(stamps)
    el = stamps[-1] - t0 if stamps else time.perf_counter() - t0
    return its / el, f"first {its} SVT iteration(s) from the kickstart on the full {CONFIG_NAMES[config]} ({el:.1f} s)", its, el


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm (CPU oracle port; the
    reference itself cannot be built here) on the same config/metric."""
    if rank != 0:
        return
    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable": "one cfg5 oracle iteration takes hours on one core "
                                                              "(SURVEY §8d); the reference arm runs on config 4"}),
              flush=True)
        return
    m, n, train, test = load_problem(args.config, args.seed)
    from oracle import oracle as O
    from paper_1704_05528_b200 import api as G
    rp, co, va = train
    A = O.Csr(m, n, rp, co, va)
    T = O.Csr(m, n, *test) if test is not None else None
    cfg, stop = G.config_params(args.config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = args.warmup + args.steps
    stamps = [time.perf_counter()]
    budget = max(90.0, args.cpu_budget * 4)

    def obs(rec, U, s, V):
        stamps.append(time.perf_counter())
        return (stamps[-1] - stamps[0]) < budget

    O.svt_run(A, cfg, stop, observer=obs, test=T)
    d = np.diff(stamps)
    timed = d[args.warmup:] if len(d) > args.warmup else d
    value = len(timed) / float(np.sum(timed))
    sample = (f"{len(d)} consecutive oracle SVT iterations (of W+K={args.warmup + args.steps}, {budget:.0f} s cap); "
              f"rate over the last {len(timed)}")
    print(json.dumps({
        "metric": "SVT iters/sec (R4SVD)", "value": value, "unit": "iter/s", "n_gpus": world, "steps": len(timed),
        "warmup": min(args.warmup, len(d)), "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": CONFIG_NAMES[args.config], "config": args.config, "m": m, "n": n,
                   "nnz": int(rp[-1]), "parallelism": "single CPU thread (reference has no threads)"},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
        return

    import torch
    from paper_1704_05528_b200 import api as G
    from paper_1704_05528_b200._abi import KCLASS

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_setup = time.perf_counter()
    m, n, train, test = load_problem(args.config, args.seed)
    rp, co, va = train
    bounds = G.partition_rows(rp, world)
    rb, re_ = int(bounds[rank]), int(bounds[rank + 1])
    if world > 1:
        obj = [G.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = G.Context(local, rank, world, obj[0])
    else:
        ctx = G.Context(local)
    torch.cuda.set_device(local)
    A = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx, row_block=(rb, re_))
    T = G.SampledMatrix.from_csr(m, n, *test, ctx=ctx, row_block=(rb, re_)) if test is not None else None
    cfg, stop = G.config_params(args.config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = max(cfg.maxit, args.warmup + args.steps + 1)
    solver = G.Solver(A, cfg, stop, test=T)
    setup_s = time.perf_counter() - t_setup

    for _ in range(args.warmup):
        solver.step()
    ctx.sync()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    ctx.reset_stats()
    ctx.set_profiling(not os.environ.get("SVTB_BENCH_NOPROF"))  # dev switch: A/B of the per-launch events
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    al0 = G.Context.alloc_stats()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs = []
    for _ in range(args.steps):
        recs.append(solver.step())
    ctx.join()  # the timed region also covers any speculative side-stream work still in flight
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    al1 = G.Context.alloc_stats()
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local)
    launches = ctx.launch_count()
    hstats = ctx.host_stats()
    stats = {KCLASS[k]: ctx.kernel_stats(k) for k in range(8)}
    ctx.set_profiling(False)
    value = args.steps * 1000.0 / ms  # whole-job iterations per second

    # roofline: the dominant kernel class of the step by device time.  The
    # sparse passes are held against HBM (algorithmic bytes); the dense FP64
    # contractions (CGS / CholQR / finalize GEMMs on the DMMA pipe) against
    # the FP64 GEMM peak when their arithmetic intensity exceeds the machine
    # balance, else against HBM.
    peak_bw, bw_kind = measured_peak()
    peak_f64, f64_kind = measured_fp64_peak()
    dom = max(stats, key=lambda k: stats[k]["total_ms"])
    s = stats[dom]
    secs = s["total_ms"] * 1e-3
    ai = s["flops"] / s["bytes"] if s["bytes"] > 0 else 0.0
    balance = peak_f64 * 1e12 / (peak_bw * 1e9)
    if dom in ("cgs_gemm", "qr", "finalize") and ai > balance:
        roof = {"bound": "tensor", "achieved": s["flops"] / secs / 1e12 if secs > 0 else 0.0, "peak": peak_f64,
                "unit": "TFLOP/s", "peak_kind": f64_kind, "dtype": "f64 (DMMA mma.sync.m8n8k4.f64)"}
    else:
        roof = {"bound": "hbm", "achieved": s["bytes"] / secs / 1e9 if secs > 0 else 0.0, "peak": peak_bw,
                "unit": "GB/s", "peak_kind": bw_kind}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof.update({"kernel": dom, "arith_intensity_flop_per_byte": ai, "machine_balance": balance,
                 "launches": s["launches"], "avg_launch_us": 1000.0 * s["total_ms"] / max(1, s["launches"]),
                 "share_of_step": s["total_ms"] / max(1e-9, sum(v["total_ms"] for v in stats.values()))})
    # the sparse passes, always reported against HBM (north star: SpMM/SDDMM
    # GB/s vs peak), plus the SpMMs' L2 gather rate: every stored entry reads
    # one 8w-byte panel row (= 4 x the 2 nnz w flops), which is what bounds
    # them (ncu: DRAM ~3 %, L2 hit ~96 %); ceiling = the LTS throughput cap
    # of the microarchitecture guide (~6300 B/clk at 1.965 GHz)
    l2_cap_tbs = 6300.0 * 1.965e9 / 1e12
    sparse = {}
    for k in ("spmm", "spmm_t", "sddmm_update"):
        v = stats[k]
        if v["total_ms"] > 0:
            sparse[k] = {"achieved_gbs": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9,
                         "frac": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9 / peak_bw}
            if k != "sddmm_update":
                g = 4.0 * v["flops"] / (v["total_ms"] * 1e-3) / 1e12
                sparse[k].update({"l2_gather_tbs": g, "l2_gather_ceiling_tbs": l2_cap_tbs,
                                  "l2_gather_frac": g / l2_cap_tbs})
    if dom in ("spmm", "spmm_t"):
        roof["note"] = ("L2-gather bound, not HBM: see sparse_roofline[%s].l2_gather_* (DRAM traffic per "
                        "launch ~ the algorithmic bytes)" % dom)
    step_ms_kernels = {k: v["total_ms"] / args.steps for k, v in stats.items()}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get(str(args.config), {}).get(dom)
        except Exception:
            traffic = None
    roof["traffic"] = traffic

    solver.close()  # release the timed run's basis before the e2e run allocates its own
    # e2e: the public C-ABI call with host buffers: upload + kickstart + K
    # iterations (each reads its record back) + factor download
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A2 = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx, row_block=(rb, re_))
        s2 = G.Solver(A2, cfg, stop)
        nsteps = args.warmup + args.steps
        for _ in range(nsteps):
            s2.step()
        res = s2.result()
        ctx.sync()
        el = max_over_ranks(time.perf_counter() - t0)
        nnz_l = int(rp[re_] - rp[rb])
        h2d = 8 * (re_ - rb + 1) + 16 * nnz_l
        d2h = 8 * 8 * nsteps + 8 * (res.U.size + res.V.size + res.sigma.size)
        e2e = {"value": nsteps / el, "unit": "iter/s", "h2d_bytes_per_step": int(h2d / nsteps),
               "d2h_bytes_per_step": int(d2h / nsteps),
               "note": "public C-ABI path from host buffers: CSR upload + kickstart + iterations 1..W+K "
                       "(each reads its record back) + factor download, wall clock; it includes the early, "
                       "cheaper iterations (smaller bases), while value times iterations W+1..W+K only"}
        s2.close()
        A2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == 5:
        cpu = {"value": None, "unit": "iter/s", "cores": 1, "kind": "port",
               "sample": "none: one cfg5 oracle iteration (t0 = 5000 sketch of a 1e8-entry matrix, ~2,000 "
                         "extension rounds to r ~ 20k) takes hours on one core (SURVEY §8d); the CPU baseline "
                         "is reported on the default workload (config 4)"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        v, sample, its, el = cpu_oracle_rate(args.config, args.seed, m, n, train, test, args.cpu_budget,
                                             args.warmup + args.steps)
        cpu = {"value": v, "unit": "iter/s", "cores": 1, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": "SVT iters/sec (R4SVD)", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "config": args.config, "m": m, "n": n,
                       "nnz": int(rp[-1]), "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU",
                       "iterations_timed": [r["iter"] for r in recs], "revealed_rank": [r["rank"] for r in recs],
                       "kept_rank": [r["kept"] for r in recs], "rounds": [r["extension_rounds"] for r in recs],
                       "l2": ("working set per pass below/near L2 for cfg1-4; no flush between steps" if args.config != 5
                              else "inputs larger than L2 (Y 1.2 GB, Q/B^T tens of GB): no flush needed"),
                       "setup_s": round(setup_s, 2)},
            "roofline": roof,
            "sparse_roofline": sparse,
            "kernel_ms_per_step": {k: round(v, 3) for k, v in step_ms_kernels.items()},
            "gpu_launches": launches,
            "host": {"syncs_per_step": hstats["syncs"] / args.steps,
                     "sync_wait_ms_per_step": hstats["sync_ms"] / args.steps,
                     "device_allocs_in_timed_region": al1["mallocs"] - al0["mallocs"],
                     "device_frees_in_timed_region": al1["frees"] - al0["frees"],
                     "alloc_ms_in_timed_region": al1["ms"] - al0["ms"],
                     "kernel_ms_per_step": sum(v["total_ms"] for v in stats.values()) / args.steps},
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

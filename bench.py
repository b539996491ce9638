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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle CPU work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="multi-rank collectives: NCCL (default) or host-staged over gloo (validates the multi-rank "
                         "path with several ranks on one GPU; never a measurement)")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="iterations of the separate per-launch-event pass (0: all K)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def load_problem(config, seed):
    """Host CSR (global) for train and test sets of a BASELINE config, from
    the shared generator (csrc/synth.cpp) compiled into liboracle.so: the
    CPU arms load no product library."""
    from oracle import oracle as O
    d = O.synth_config(config, seed)
    tr, te = d["train"], d["test"]
    return d["m"], d["n"], (tr.rowptr, tr.col, tr.val), ((te.rowptr, te.col, te.val) if te is not None else None)


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


def gather_ceiling():
    """Row-gather ceiling (TB/s): the best uniform-index rate of the gather
    microbenchmark (scripts/gather_probe.cu: random 1 KB panel rows, register
    accumulation — what one SpMM entry does), profiles/r02_gather_probe.txt."""
    p = os.path.join(ROOT, "profiles", "r02_gather_probe.txt")
    best = 0.0
    try:
        with open(p) as f:
            for line in f:
                if "uniform" in line and "ldg" in line and "TB/s" in line:
                    best = max(best, float(line.split("gather")[1].split("TB/s")[0]))
    except Exception:
        best = 0.0
    if best <= 0.0:
        return 20.9, "fallback constant (probe file missing)"
    return best, "profiles/r02_gather_probe.txt (uniform random 1 KB rows; L1 hits lift Zipf patterns above it)"


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
def oracle_threads():
    from oracle import oracle as O
    return O.num_threads()


def cpu_matched_iteration(config, m, n, train, test, ckpt, W):
    """The CPU oracle (the reference's algorithm restated, all host threads)
    on iteration W + 1 — the first iteration of the GPU's timed window —
    resumed from the device state after W iterations (svt_solver_checkpoint),
    so both arms time the same iteration of the same run.  Returns
    (seconds, record)."""
    from oracle import oracle as O
    rp, co, va = train
    A = O.Csr(m, n, rp, co, va)
    T = O.Csr(m, n, *test) if test is not None else None
    cfg, stop = O.config_params(config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = W + 1
    st = ckpt["state"]
    s = int(st.s)
    start = dict(iter=int(st.iter), y_vals=ckpt["y_vals"][: int(rp[-1])],
                 u_prev=np.asarray(ckpt["u_prev"][: m * s]).reshape(s, m).T if s else np.zeros((m, 0)),
                 eps_threshold=st.eps_threshold, eps_min=st.eps_min)
    t0 = time.perf_counter()
    r = O.svt_run(A, cfg, stop, test=T, start=start)
    return time.perf_counter() - t0, r.trace[0]


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the reference's algorithm on the host CPU (the
    oracle port: the reference itself cannot be built here),
    all host threads, on the same config / metric.  Bounded sample: SVT
    iterations from the kickstart (the first ones of the same run) until
    W + K iterations or a time cap.  Loads only liboracle.so."""
    if rank != 0:
        return
    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable": "one cfg5 oracle iteration takes hours on the host "
                                                              "(SURVEY §8d); the reference arm runs on config 4"}),
              flush=True)
        return
    m, n, train, test = load_problem(args.config, args.seed)
    from oracle import oracle as O
    rp, co, va = train
    A = O.Csr(m, n, rp, co, va)
    T = O.Csr(m, n, *test) if test is not None else None
    cfg, stop = O.config_params(args.config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = args.warmup + args.steps
    stamps = [time.perf_counter()]
    budget = max(120.0, args.cpu_budget * 6)

    def obs(rec, U, s, V):
        stamps.append(time.perf_counter())
        return (stamps[-1] - stamps[0]) < budget

    O.svt_run(A, cfg, stop, observer=obs, test=T)
    d = np.diff(stamps)
    value = len(d) / float(np.sum(d))
    cores = O.num_threads()
    sample = (f"SVT iterations 1-{len(d)} of the same run from the kickstart (GPU arm times {args.warmup + 1}-"
              f"{args.warmup + args.steps}; later iterations carry wider bases and cost more), {budget:.0f} s cap, "
              f"oracle port with {cores} OpenMP threads")
    print(json.dumps({
        "metric": "SVT iters/sec (R4SVD)", "value": value, "unit": "iter/s", "n_gpus": world, "steps": len(d),
        "warmup": 0, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": CONFIG_NAMES[args.config], "config": args.config, "m": m, "n": n,
                   "nnz": int(rp[-1]), "parallelism": f"host CPU, {cores} threads",
                   "iterations_timed": list(range(1, len(d) + 1))},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "port", "sample": sample},
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
    if world > 1 and args.comm == "host":
        def host_allreduce(x):
            dist.all_reduce(torch.from_numpy(x))  # sums the pinned staging buffer in place

        local = 0 if torch.cuda.device_count() == 1 else local
        ctx = G.Context.hostcomm(local, rank, world, host_allreduce)
    elif world > 1:
        obj = [G.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = G.Context(local, rank, world, obj[0])
    else:
        ctx = G.Context(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    A = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx, row_block=(rb, re_))
    T = G.SampledMatrix.from_csr(m, n, *test, ctx=ctx, row_block=(rb, re_)) if test is not None else None
    cfg, stop = G.config_params(args.config, int(rp[-1]), m, n, frob(va))
    cfg.maxit = max(cfg.maxit, args.warmup + args.steps + 1)
    solver = G.Solver(A, cfg, stop, test=T)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    # warm-up: iterations 1..W (iteration 1's device time feeds the matched
    # CPU comparison), then a host checkpoint of the state after W
    # iterations: the e2e leg and the profiled pass resume from it, and the
    # CPU leg times iteration W + 1 from the same state
    warm_ms = []
    for _ in range(args.warmup):
        a = ev()
        solver.step()
        ctx.join()
        b = ev()
        b.synchronize()
        warm_ms.append(a.elapsed_time(b))
    ctx.sync()
    ckpt = solver.checkpoint()

    # ---- timed window: iterations W+1..W+K, no instrumentation ----------
    ctx.reset_stats()
    ctx.set_profiling(False)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    al0 = G.Context.alloc_stats()
    e0 = ev()
    marks = []
    recs = []
    for _ in range(args.steps):
        recs.append(solver.step())
        marks.append(ev())
    ctx.join()  # the timed region also covers any speculative side-stream work still in flight
    e1 = ev()
    e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    al1 = G.Context.alloc_stats()
    ms = max_over_ranks(e0.elapsed_time(e1))
    step_ms = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i]) for i in range(1, len(marks))]
    launches = ctx.launch_count()
    hstats = ctx.host_stats()
    value = args.steps * 1000.0 / ms  # whole-job iterations per second
    solver.close()  # release the timed run's basis before the next legs allocate their own

    # ---- e2e: the public C-ABI path from pinned host buffers -------------
    # timed: upload of the sample sets (CSR) and of the iteration state
    # after W iterations, iterations W+1..W+K through svt_solver_step (each
    # reads its record back), download of the result factors
    e2e = None
    if not args.no_e2e:
        def pinned(x):
            t = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
            return t.numpy()
        lrp = rp[rb: re_ + 1]
        s0, s1 = int(lrp[0]), int(lrp[-1])
        host = {"rp": pinned(lrp - lrp[0]), "co": pinned(co[s0:s1]), "va": pinned(va[s0:s1])}
        if test is not None:
            trp = test[0][rb: re_ + 1]
            t0_, t1_ = int(trp[0]), int(trp[-1])
            host.update({"trp": pinned(trp - trp[0]), "tco": pinned(test[1][t0_:t1_]),
                         "tva": pinned(test[2][t0_:t1_])})
        ck_h = {k: (pinned(v) if isinstance(v, np.ndarray) else v) for k, v in ckpt.items()}
        h2d = sum(host[k].nbytes for k in host) + sum(ck_h[k].nbytes for k in
                                                      ("y_vals", "u_prev", "best_U", "best_sigma", "best_V"))
        # the timed solver's release of its basis reservation (tens of GB) can
        # complete lazily inside the next device allocation (seen as 0.7 s in
        # the first cudaMalloc of this leg on some runs): absorb it here, before
        # the clock starts, with one allocation / release cycle of our own
        ctx.sync()
        scratch = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        scratch.fill_(0)
        del scratch
        torch.cuda.empty_cache()
        tiny = G.SampledMatrix.from_csr(2, 2, np.array([0, 1, 2], np.int64), np.array([0, 1], np.int64),
                                        np.array([1.0, 1.0]), ctx=ctx)
        tiny.close()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A2 = G.SampledMatrix.from_csr(m, n, host["rp"], host["co"], host["va"], ctx=ctx, row_block=(0, re_ - rb)) \
            if world == 1 else G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx, row_block=(rb, re_))
        T2 = None
        if test is not None:
            T2 = G.SampledMatrix.from_csr(m, n, host["trp"], host["tco"], host["tva"], ctx=ctx,
                                          row_block=(0, re_ - rb)) \
                if world == 1 else G.SampledMatrix.from_csr(m, n, *test, ctx=ctx, row_block=(rb, re_))
        t_up = time.perf_counter()
        s2 = G.Solver.resume(A2, cfg, stop, ck_h, test=T2)
        t_res = time.perf_counter()
        recs2, t_it = [], []
        for _ in range(args.steps):
            recs2.append(s2.step())
            t_it.append(time.perf_counter())
        res = s2.result()
        ctx.sync()
        t_end = time.perf_counter()
        el = max_over_ranks(t_end - t0)
        e2e_breakdown = {"upload_and_build_ms": round(1e3 * (t_up - t0), 1), "resume_ms": round(1e3 * (t_res - t_up), 1),
                         "first_iteration_ms": round(1e3 * (t_it[0] - t_res), 1),
                         "other_iterations_ms": round(1e3 * (t_it[-1] - t_it[0]), 1),
                         "result_download_ms": round(1e3 * (t_end - t_it[-1]), 1)}
        d2h = 96 * args.steps + 8 * (res.U.size + res.V.size + res.sigma.size)
        same = all((a["rank"], a["extension_rounds"], a["kept"], a["residual"]) ==
                   (b["rank"], b["extension_rounds"], b["kept"], b["residual"]) for a, b in zip(recs, recs2))
        e2e = {"value": args.steps / el, "unit": "iter/s", "h2d_bytes_per_step": int(h2d / args.steps),
               "d2h_bytes_per_step": int(d2h / args.steps),
               "iterations": [r["iter"] for r in recs2], "same_records_as_timed_window": same,
               "breakdown_ms": e2e_breakdown,
               "note": "public C-ABI path, wall clock: CSR upload of the sample sets + resume from the host "
                       "checkpoint after W iterations (Y values, U_prev, best factors) from pinned memory, "
                       "iterations W+1..W+K (each reads its record back), factor download"}
        s2.close()
        A2.close()
        if T2 is not None:
            T2.close()

    # ---- profiled passes: the same iterations again, with per-launch events.
    # (1) serialised (speculative side-stream batches off: the same batches
    # and results, one stream at a time): per-kernel durations without the SM
    # sharing of two concurrent streams — the roofline and the kernel shares
    # (comparable to ncu's serialised launch list); (2) as timed, with the
    # overlap: the in-step per-class device times.
    psteps = args.profile_steps if 0 < args.profile_steps < args.steps else args.steps

    def profiled_pass(speculate):
        s3 = G.Solver.resume(A, cfg, stop, ckpt, test=T)
        ctx.set_speculation(speculate)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(psteps):
            s3.step()
        ctx.join()
        ctx.sync()
        st = {KCLASS[k]: ctx.kernel_stats(k) for k in range(8)}
        hs = ctx.host_stats()
        ctx.set_profiling(False)
        ctx.set_speculation(True)
        s3.close()
        return st, hs

    stats, hstats_prof = profiled_pass(False)
    stats_in_step, _ = profiled_pass(True)

    # roofline: the dominant kernel class by device time (per-launch CUDA
    # events of the profiled pass over the same iterations).  The sparse
    # passes are held against HBM (algorithmic bytes); the dense FP64
    # contractions (CGS / CholQR / finalize GEMMs on the DMMA pipe) against
    # the FP64 GEMM peak when their arithmetic intensity exceeds the machine
    # balance, else against HBM.
    peak_bw, bw_kind = measured_peak()
    peak_f64, f64_kind = measured_fp64_peak()
    # Y X and Y^T X are one kernel (the split gather SpMM) in two
    # directions: they count as one kernel for the dominance test and the
    # roofline (both directions' algorithmic bytes over both times)
    merged = dict(stats)
    sp, spt = stats["spmm"], stats["spmm_t"]
    merged["spmm"] = {k: sp[k] + spt[k] for k in ("launches", "total_ms", "bytes", "flops")}
    del merged["spmm_t"]
    dom = max(merged, key=lambda k: merged[k]["total_ms"])
    s = merged[dom]
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
                 "share_of_step": s["total_ms"] / max(1e-9, sum(v["total_ms"] for v in stats.values())),
                 "classes": ("spmm + spmm_t (the split gather SpMM, Y X and Y^T X)" if dom == "spmm" else dom),
                 "timing": "per-launch CUDA events in a separate serialised profiled pass over iterations "
                           "W+1..W+K (resumed from the same state, speculative side-stream batches off: same "
                           "batches and results, no SM sharing between streams); a split SpMM (cold gather || "
                           "dense corner || scatter-add) is one timed operation; the timed window runs without "
                           "events"})
    # the sparse passes, always reported against HBM (north star: SpMM/SDDMM
    # GB/s vs peak), plus the SpMMs' gather rate: every stored entry reads
    # one 8w-byte panel row (= 4 x the 2 nnz w flops)
    sparse = {}
    for k in ("spmm", "spmm_t", "sddmm_update"):
        v = stats[k]
        if v["total_ms"] > 0:
            sparse[k] = {"achieved_gbs": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9,
                         "frac": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9 / peak_bw,
                         "launches": v["launches"], "avg_launch_us": 1000.0 * v["total_ms"] / max(1, v["launches"])}
            if k != "sddmm_update":
                sparse[k]["gather_tbs"] = 4.0 * v["flops"] / (v["total_ms"] * 1e-3) / 1e12
                ceil_tbs, ceil_src = gather_ceiling()
                sparse[k]["gather_ceiling_tbs"] = ceil_tbs
                sparse[k]["gather_frac"] = sparse[k]["gather_tbs"] / ceil_tbs
                sparse[k]["gather_ceiling_source"] = ceil_src
    # the dense FP64 contractions against the measured DGEMM peak (north
    # star: FP64 tensor-pipe utilisation of the orthogonalisation GEMMs);
    # predicated products that the device skipped carry no flops
    dense = {}
    for k in ("cgs_gemm", "qr", "finalize"):
        v = stats[k]
        if v["total_ms"] > 0 and v["flops"] > 0:
            tf = v["flops"] / (v["total_ms"] * 1e-3) / 1e12
            dense[k] = {"achieved_tflops": tf, "peak_tflops": peak_f64, "frac": tf / peak_f64, "peak_kind": f64_kind,
                        "launches": v["launches"], "ms_per_step": v["total_ms"] / psteps,
                        "note": ("all launches of the class, incl. latency-bound single-CTA factorisations"
                                 if k != "cgs_gemm" else "block Gram-Schmidt products (DMMA)")}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            tc = tj.get(str(args.config), {})
            traffic = tc.get(dom)
            if dom == "spmm" and tc.get("spmm") and tc.get("spmm_t"):
                traffic = 0.5 * (tc["spmm"] + tc["spmm_t"])  # one launch of each direction, averaged
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    if dom == "spmm":
        g = 4.0 * s["flops"] / (s["total_ms"] * 1e-3) / 1e12 if s["total_ms"] > 0 else 0.0
        ceil_tbs, ceil_src = gather_ceiling()
        roof["gather"] = {"achieved_tbs": g, "ceiling_tbs": ceil_tbs, "frac": g / ceil_tbs, "source": ceil_src,
                          "note": "panel-row gather rate (nnz w 8 B per product): the bound of the gather form "
                                  "(DESIGN.md §7)"}

    cpu = None
    matched = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == 5:
        cpu = {"value": None, "unit": "iter/s", "cores": oracle_threads(), "kind": "port",
               "sample": "none: one cfg5 oracle iteration (~2,000 extension rounds to r ~ 20k on a 1e8-entry "
                         "matrix) takes hours on the host (SURVEY §8d); the CPU baseline is reported on config 4"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        cpu_s, crec = cpu_matched_iteration(args.config, m, n, train, test, ckpt, args.warmup)
        g = recs[0]
        cores = oracle_threads()
        par = {"rank_rounds_kept_equal": (g["rank"], g["extension_rounds"], g["kept"]) ==
               (crec["rank"], crec["extension_rounds"], crec["kept"]),
               "residual_rel_diff": abs(g["residual"] - crec["residual"]) / abs(crec["residual"])}
        cpu = {"value": 1.0 / cpu_s, "unit": "iter/s", "cores": cores, "kind": "port",
               "sample": f"SVT iteration {args.warmup + 1} (the first iteration of the timed window) resumed from "
                         f"the device state after {args.warmup} iterations; oracle port (the reference's "
                         f"algorithm restated), {cores} OpenMP threads; {cpu_s:.1f} s",
               "parity": par}
        matched = {"iteration": args.warmup + 1, "gpu_ms": step_ms[0], "cpu_ms": 1000.0 * cpu_s,
                   "gpu_over_cpu_speedup": 1000.0 * cpu_s / step_ms[0],
                   "iteration1_gpu_ms": warm_ms[0] if warm_ms else None}

    if rank == 0:
        line = {
            "metric": "SVT iters/sec (R4SVD)", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "config": args.config, "m": m, "n": n,
                       "nnz": int(rp[-1]), "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU",
                       "iterations_timed": [r["iter"] for r in recs], "revealed_rank": [r["rank"] for r in recs],
                       "kept_rank": [r["kept"] for r in recs], "rounds": [r["extension_rounds"] for r in recs],
                       "ms_per_iteration": [round(x, 2) for x in step_ms],
                       "l2": ("working set per pass below/near L2 for cfg1-4; no flush between steps" if args.config != 5
                              else "inputs larger than L2 (Y 1.2 GB, Q/B^T tens of GB): no flush needed"),
                       "setup_s": round(setup_s, 2)},
            "roofline": roof,
            "sparse_roofline": sparse,
            "dense_roofline": dense,
            "kernel_ms_per_step": {k: round(v["total_ms"] / psteps, 3) for k, v in stats.items()},
            "kernel_ms_per_step_in_step": {k: round(v["total_ms"] / psteps, 3) for k, v in stats_in_step.items()},
            "profiled_iterations": list(range(args.warmup + 1, args.warmup + psteps + 1)),
            "gpu_launches": launches,
            "host": {"syncs_per_step": hstats["syncs"] / args.steps,
                     "sync_wait_ms_per_step_profiled_pass": hstats_prof["sync_ms"] / psteps,
                     "device_allocs_in_timed_region": al1["mallocs"] - al0["mallocs"],
                     "device_frees_in_timed_region": al1["frees"] - al0["frees"],
                     "alloc_ms_in_timed_region": al1["ms"] - al0["ms"],
                     "kernel_ms_per_step_profiled_pass": sum(v["total_ms"] for v in stats.values()) / psteps},
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "matched_window": matched,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Isolated timings of the sparse kernels on a BASELINE config's sample set:
Y X (CSR), Y^T X (CSC) at panel widths w, and the fused SDDMM + Bregman
update (+ CSC mirror) at kept ranks k, each through the device-pointer C ABI
(svt_dev_sp_mult / svt_dev_sddmm_update) on the library stream, CUDA events,
after warm-up.  Checks each result against torch (fp64) once.  Development /
profiling tool: python scripts/sparse_bench.py [config] [widths] [ranks] [reps]
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402

HBM = 6558.7  # MEASURED_PEAKS.json hbm_gbs


def timed(fn, stream, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    widths = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10,32,64,120,128").split(",") if x]
    ranks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "3,10,50").split(",") if x]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    ctx = G.default_context()
    L = G.lib()
    st = torch.cuda.ExternalStream(ctx.stream)
    d = G.synth_config(cfg, 1)
    m, n = d["m"], d["n"]
    if cfg == 5:
        rp, co, va = d["csr"]
    else:
        rp, co, va = G.build_csr(m, n, *d["train"])
    A = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx)
    nnz = int(rp[-1])
    crow = torch.from_numpy(np.asarray(rp, np.int64)).cuda()
    cols = torch.from_numpy(np.asarray(co, np.int64)).cuda()
    vals = torch.from_numpy(np.asarray(va, np.float64)).cuda()
    rows = torch.repeat_interleave(torch.arange(m, device="cuda"), crow[1:] - crow[:-1])
    out = []
    for w in widths:
        X = torch.randn(n, w, dtype=torch.float64, device="cuda")
        Xt = torch.randn(m, w, dtype=torch.float64, device="cuda")
        o = torch.empty(m, w, dtype=torch.float64, device="cuda")
        ot = torch.empty(n, w, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        f = lambda: L.svt_dev_sp_mult(A.h, 0, C.c_int64(w), C.c_void_p(X.data_ptr()), C.c_int64(w),  # noqa: E731
                                      C.c_void_p(o.data_ptr()), C.c_int64(w))
        ft = lambda: L.svt_dev_sp_mult(A.h, 1, C.c_int64(w), C.c_void_p(Xt.data_ptr()), C.c_int64(w),  # noqa: E731
                                       C.c_void_p(ot.data_ptr()), C.c_int64(w))
        t, tt = timed(f, st, reps), timed(ft, st, reps)
        ctx.sync()
        ref = torch.zeros(m, w, dtype=torch.float64, device="cuda")
        reft = torch.zeros(n, w, dtype=torch.float64, device="cuda")
        ch = max(1, (1 << 31) // (8 * w))  # entries per chunk (<= 2 GB of gathered rows)
        for s0 in range(0, nnz, ch):
            sl = slice(s0, min(nnz, s0 + ch))
            ref.index_add_(0, rows[sl], vals[sl, None] * X[cols[sl]])
            reft.index_add_(0, cols[sl], vals[sl, None] * Xt[rows[sl]])
        e = ((o - ref).abs().max() / ref.abs().max()).item()
        et = ((ot - reft).abs().max() / reft.abs().max()).item()
        alg = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * w * (m + n)
        for name, tm, err in (("YX", t, e), ("YtX", tt, et)):
            r = {"kernel": "spmm" if name == "YX" else "spmm_t", "config": cfg, "w": w, "us": round(tm, 1),
                 "alg_GBs": round(alg / tm / 1e3, 1), "hbm_frac": round(alg / tm / 1e3 / HBM, 4),
                 "gather_TBs": round(nnz * w * 8.0 / tm / 1e6, 2), "max_rel_err": e}
            out.append(r)
            print(json.dumps(r), flush=True)
        del X, Xt, o, ot, ref, reft
    A_vals = vals
    for k in ranks:
        U = torch.randn(m, k, dtype=torch.float64, device="cuda")
        Vs = torch.randn(n, k, dtype=torch.float64, device="cuda") * 0.1
        Y0 = torch.randn(nnz, dtype=torch.float64, device="cuda")
        Y = Y0.clone()
        Yc = torch.empty_like(Y)
        delta = 1.2
        torch.cuda.synchronize()
        f = lambda: L.svt_dev_sddmm_update(A.h, C.c_int64(k), C.c_void_p(U.data_ptr()), C.c_int64(k),  # noqa: E731
                                           C.c_void_p(Vs.data_ptr()), C.c_int64(k), C.c_double(delta),
                                           C.c_void_p(Y.data_ptr()), C.c_void_p(Yc.data_ptr()), None)
        tm = timed(f, st, reps)
        ctx.sync()
        # parity of one application from Y0
        Y.copy_(Y0)
        torch.cuda.synchronize()
        sums = (C.c_double * 4)()
        L.svt_dev_sddmm_update(A.h, C.c_int64(k), C.c_void_p(U.data_ptr()), C.c_int64(k), C.c_void_p(Vs.data_ptr()),
                               C.c_int64(k), C.c_double(delta), C.c_void_p(Y.data_ptr()), C.c_void_p(Yc.data_ptr()),
                               sums)
        P = torch.cat([(U[rows[s0:s0 + (1 << 24)]] * Vs[cols[s0:s0 + (1 << 24)]]).sum(1)
                       for s0 in range(0, nnz, 1 << 24)])
        dd = A_vals - P
        Yr = Y0 + delta * dd
        e = ((Y - Yr).abs().max() / Yr.abs().max()).item()
        perm = torch.argsort(cols * m + rows)
        ec = (Yc - Yr[perm]).abs().max().item() / Yr.abs().max().item()
        del perm
        es = abs(sums[1] - float((dd * dd).sum())) / float((dd * dd).sum())
        alg = 48.0 * nnz + 8.0 * (m + 1) + 8.0 * k * (m + n)
        r = {"kernel": "sddmm_update+mirror", "config": cfg, "k": k, "us": round(tm, 1),
             "alg_GBs": round(alg / tm / 1e3, 1), "hbm_frac": round(alg / tm / 1e3 / HBM, 4),
             "factor_gather_TBs": round(nnz * k * 8.0 / tm / 1e6, 2), "max_rel_err": e, "csc_err": ec,
             "sum_d2_rel_err": es}
        out.append(r)
        print(json.dumps(r), flush=True)
        del U, Vs, Y, Y0, Yc, P, dd, Yr
    A.close()


if __name__ == "__main__":
    main()

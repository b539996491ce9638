"""SpMM roofline check: our segmented SpMM (svt_dev_sp_mult) against cuSPARSE
(torch.sparse.mm on a float64 CSR) on the BASELINE configs' sample sets, at
the panel widths of the sketch.  Reports the gather traffic (nnz x w x 8 B
from L2) and the algorithmic HBM bytes per pass.  Development tool."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402


def timed(fn, stream, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    configs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4").split(",")]
    widths = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10,120").split(",")]
    ctx = G.default_context()
    L = G.lib()
    ours_stream = torch.cuda.ExternalStream(ctx.stream)
    for cfg in configs:
        d = G.synth_config(cfg, 1)
        m, n = d["m"], d["n"]
        if cfg == 5:
            rp, co, va = d["csr"]
        else:
            rp, co, va = G.build_csr(m, n, *d["train"])
        A = G.SampledMatrix.from_csr(m, n, rp, co, va, ctx=ctx)
        nnz = int(rp[-1])
        crow = torch.from_numpy(np.asarray(rp, dtype=np.int64)).cuda()
        cols = torch.from_numpy(np.asarray(co, dtype=np.int64)).cuda()
        vals = torch.from_numpy(np.asarray(va, dtype=np.float64)).cuda()
        S = torch.sparse_csr_tensor(crow, cols, vals, size=(m, n))
        St = S.to_sparse_coo().t().coalesce().to_sparse_csr()
        for w in widths:
            X = torch.randn(n, w, dtype=torch.float64, device="cuda")
            Xt = torch.randn(m, w, dtype=torch.float64, device="cuda")
            out = torch.empty(m, w, dtype=torch.float64, device="cuda")
            outt = torch.empty(n, w, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()

            def ours():
                L.svt_dev_sp_mult(A.h, 0, C.c_int64(w), C.c_void_p(X.data_ptr()), C.c_int64(w),
                                  C.c_void_p(out.data_ptr()), C.c_int64(w))

            def ours_t():
                L.svt_dev_sp_mult(A.h, 1, C.c_int64(w), C.c_void_p(Xt.data_ptr()), C.c_int64(w),
                                  C.c_void_p(outt.data_ptr()), C.c_int64(w))

            t_o = timed(ours, ours_stream)
            t_ot = timed(ours_t, ours_stream)
            ref = torch.sparse.mm(S, X)
            reft = torch.sparse.mm(St, Xt)
            err = ((out - ref).abs().max() / ref.abs().max()).item()
            errt = ((outt - reft).abs().max() / reft.abs().max()).item()
            t_c = timed(lambda: torch.sparse.mm(S, X), torch.cuda.current_stream())
            t_ct = timed(lambda: torch.sparse.mm(St, Xt), torch.cuda.current_stream())
            gather = nnz * w * 8.0
            alg = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * w * (m + n)
            for name, t, tc, e in (("Y X  ", t_o, t_c, err), ("Y^T X", t_ot, t_ct, errt)):
                print(f"cfg{cfg} nnz={nnz} w={w:4d} {name}: ours {t*1e3:9.1f} us  gather {gather/t/1e9:7.2f} TB/s  "
                      f"alg-HBM {alg/t/1e6:7.1f} GB/s | cuSPARSE {tc*1e3:9.1f} us ({tc/t:5.2f}x ours)  "
                      f"max rel diff {e:.1e}", flush=True)
            del X, Xt, out, outt, ref, reft
        A.close()
        del S, St, crow, cols, vals
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

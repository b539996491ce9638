"""World-size-2 CPU tests (gloo) of the row-sharded decomposition the engine
uses for multi-GPU runs: rows of Y / Q / X / U are split by
the library's nnz-balanced partition; Y^T-products, Gram blocks and norms are
all-reduced; every rank then takes the same data-dependent branches.  Each
rank restates one extension round (sketch.hpp:114-154) and the fused SVT
update sums (solver.hpp:279-323) on its row block with gloo all-reduces and
checks them against the unsharded CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1704_05528_b200 import api as G
from tests.refutil import random_sampled

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        res = {}
        S = random_sampled(90, 70, 0.3, 11)
        bounds = G.partition_rows(S.rowptr, WORLD)
        rb, re_ = int(bounds[rank]), int(bounds[rank + 1])
        Dn = S.dense()
        Yl = Dn[rb:re_]  # this rank's row block of Y
        # --- one qb_extend round, sharded ---
        st = O.QB.init(S, 6, 1, 5)
        Q, _ = st.QB()
        Ql = Q[rb:re_]
        w = 4
        Om = O.gaussian_block(70, w, 77)
        X = Yl @ Om                                   # local rows
        T = allreduce(Yl.T @ X)                       # Y^T X (n x w)
        X = Yl @ T                                    # power pass
        C = allreduce(Ql.T @ X)                       # CGS
        X = X - Ql @ C
        C2 = allreduce(Ql.T @ X)
        nx = allreduce(np.array([np.sum(X * X)]))[0]
        if np.linalg.norm(C2) > 1e-8 * np.sqrt(nx):   # same branch on all ranks
            X = X - Ql @ C2
        Gm = allreduce(X.T @ X)                       # CholQR
        R = np.linalg.cholesky(Gm).T
        Qp = X @ np.linalg.inv(R)
        Gm2 = allreduce(Qp.T @ Qp)
        R2 = np.linalg.cholesky(Gm2).T
        Qp = Qp @ np.linalg.inv(R2)
        Bp = allreduce(Yl.T @ Qp)                     # coefficient block (replicated)
        res["energy"] = float(np.sum(Bp * Bp))
        st.extend(S, w, 1, 77)
        res["energy_ref"] = st.info()["norm_b_sq"] - O.QB.init(S, 6, 1, 5).info()["norm_b_sq"]
        # --- SVT fused update sums, sharded ---
        U = O.qr_orthonormal(O.gaussian_block(90, 3, 1))
        V = O.qr_orthonormal(O.gaussian_block(70, 3, 2))
        s = np.array([3.0, 2.0, 1.0])
        P = ((U * s) @ V.T)[rb:re_]
        mask = Yl != 0
        A = Yl
        Yv = 1.5 * Yl
        d = (A - P)[mask]
        loc = np.array([np.abs(d).sum(), (d * d).sum(), ((A - Yv)[mask] ** 2).sum()])
        res["sums"] = allreduce(loc)
        Pf = (U * s) @ V.T
        mfull = Dn != 0
        dfull = (Dn - Pf)[mfull]
        res["sums_ref"] = np.array([np.abs(dfull).sum(), (dfull * dfull).sum(),
                                    ((Dn - 1.5 * Dn)[mfull] ** 2).sum()])
        res["rows"] = (rb, re_)
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_sharded_round_and_update_match_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (a0, a1), (b0, b1) = results[0]["rows"], results[1]["rows"]
    assert a0 == 0 and a1 == b0 and b1 == 90
    for r in range(WORLD):
        res = results[r]
        assert abs(res["energy"] - res["energy_ref"]) <= 1e-10 * max(1.0, res["energy_ref"])
        np.testing.assert_allclose(res["sums"], res["sums_ref"], rtol=1e-12)
    assert results[0]["energy"] == results[1]["energy"]  # replicated, bit-identical

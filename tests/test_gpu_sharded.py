"""The row-sharded product path at world = 2.

Two processes share the one B200 of the test box; each owns an nnz-balanced
row block of Y (and of Q / X / U) and runs the library's own sharded engine:
every all-reduce of the path — the n x w partials of Y^T X
(sampled.hpp:130-144), the Gram-Schmidt / CholQR Gram blocks
(sketch.hpp:133-141), the norms and the fused-update sums
(solver.hpp:279-323) — goes through svt_ctx_create_hostcomm's host-staged
all-reduce (gloo).  The collective sequence is the one NCCL mode issues
(same call sites, counted by svt_ctx_comm_stats); only the transport
differs.  No kernel of one rank waits on the other rank (the host blocks in
gloo between launches), so the two processes may share the device.

Checked against the world = 1 device run and the oracle: revealed rank,
rounds and kept rank exact per iteration; residual / MAE / relative
residual / held-out metrics within 1e-8; the completed matrix X within 1e-8.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1704_05528_b200 import api as G
from paper_1704_05528_b200._abi import SketchParams, StopRule

WORLD = 2
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    """(name, m, n, train CSR, test CSR or None, cfg, iterations)."""
    out = []
    d = O.synth_config(3, 1)  # BASELINE config 3 at full size: power-law users, Zipf items
    A, T = d["train"], d["test"]
    cfg, _ = O.config_params(3, A.nnz, d["m"], d["n"], float(np.sqrt(np.sum(A.val * A.val))))
    out.append(("config3", d["m"], d["n"], A, T, cfg, 4))
    # skewed random problem: a few very dense rows next to near-empty ones,
    # so the nnz-balanced partition cuts far from m / 2
    rng = np.random.default_rng(5)
    m, n = 700, 300
    deg = np.minimum(n, (rng.pareto(0.7, m) * 3 + 1).astype(np.int64))
    rows = np.repeat(np.arange(m), deg)
    cols = np.concatenate([rng.choice(n, k, replace=False) for k in deg])
    L, R = rng.standard_normal((m, 5)), rng.standard_normal((n, 5))
    vals = np.einsum("ij,ij->i", L[rows], R[cols]) + 0.01 * rng.standard_normal(rows.size)
    S = O.sampled(m, n, rows, cols, vals)
    cfg = O.default_config(S)
    cfg.maxit = 12
    cfg.seed = 9
    out.append(("skewed", m, n, S, None, cfg, 12))
    return out


def _probe(U, s, V, m, n, seed=3):
    rng = np.random.default_rng(seed)
    r, c = rng.integers(0, m, 400), rng.integers(0, n, 400)
    return np.einsum("ij,j,ij->i", U[r], s, V[c]) if s.size else np.zeros(400)


def _worker(rank, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)

    def allreduce(x):
        t = torch.from_numpy(x)  # shares the pinned staging buffer: summed in place
        dist.all_reduce(t)

    try:
        ctx = G.Context.hostcomm(0, rank, WORLD, allreduce)
        res = {}
        for name, m, n, A, T, cfg, iters in _cases():
            # config 3 with the speculative side-stream batches (their Y^T X
            # all-reduces run on the side stream: the second-communicator
            # path of NCCL mode), the skewed case without
            os.environ["SVTB_SPEC_MULTI"] = "1" if name == "config3" else "0"
            b = G.partition_rows(A.rowptr, WORLD)
            rb, re_ = int(b[rank]), int(b[rank + 1])
            Ag = G.SampledMatrix.from_csr(m, n, A.rowptr, A.col, A.val, ctx=ctx, row_block=(rb, re_))
            Tg = (G.SampledMatrix.from_csr(m, n, T.rowptr, T.col, T.val, ctx=ctx, row_block=(rb, re_))
                  if T is not None else None)
            c0 = ctx.comm_stats()
            cfg.maxit = iters
            r = G.svt_run(Ag, cfg, StopRule.none(), test=Tg)
            c1 = ctx.comm_stats()
            res[name] = dict(trace=r.trace, U=r.U, sigma=r.sigma, V=r.V, rows=(rb, re_),
                             calls=c1["calls"] - c0["calls"], doubles=c1["doubles"] - c0["doubles"])
            Ag.close()
            if Tg is not None:
                Tg.close()
        # rank-deficient panels: a fully observed rank-3 matrix sketched past
        # its rank — the batched Cholesky QR loses its pivots, the rounds
        # rerun one by one and the sharded QR takes the gathered Householder
        # fallback (engine.cpp qr_panel) for the orthonormal fill
        M = O.make_low_rank(80, 60, 3, 17)
        S = O.to_sampled(M)
        b = G.partition_rows(S.rowptr, WORLD)
        rb, re_ = int(b[rank]), int(b[rank + 1])
        Sg = G.SampledMatrix.from_csr(80, 60, S.rowptr, S.col, S.val, ctx=ctx, row_block=(rb, re_))
        p = SketchParams(t=2, dt=4, np=1, eps_threshold=1e-12, seed=4)
        f = G.r3svd(Sg, p)
        res["deficient"] = dict(U=f.U, sigma=f.sigma, V=f.V, rank=f.rank, rounds=f.extension_rounds,
                                saturated=f.saturated, rows=(rb, re_))
        Sg.close()
        ctx.close()
        q.put((rank, res))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(WORLD):
        r, res = q.get(timeout=1500)
        out[r] = res
    for p in procs:
        p.join(timeout=120)
    for r in range(WORLD):
        assert "error" not in out[r], out[r].get("error")
    return out


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("name", ["config3", "skewed"])
def test_sharded_run_matches_world1_and_oracle(sharded, name):
    case = {c[0]: c for c in _cases()}[name]
    _, m, n, A, T, cfg, iters = case
    cfg.maxit = iters
    Ag = G.SampledMatrix.from_csr(m, n, A.rowptr, A.col, A.val)
    Tg = G.SampledMatrix.from_csr(m, n, T.rowptr, T.col, T.val) if T is not None else None
    one = G.svt_run(Ag, cfg, StopRule.none(), test=Tg)
    orc = O.svt_run(A, cfg, StopRule.none(), test=T)
    r0, r1 = sharded[0][name], sharded[1][name]
    # both ranks issued the same collective sequence, and it is non-trivial
    assert r0["calls"] == r1["calls"] > 0 and r0["doubles"] == r1["doubles"]
    assert r0["rows"][0] == 0 and r0["rows"][1] == r1["rows"][0] and r1["rows"][1] == m
    keys = ["residual", "train_mae", "rel_residual_x"] + (["test_mae", "test_rmse"] if T is not None else [])
    for it, (a, b, g, o) in enumerate(zip(r0["trace"], r1["trace"], one.trace, orc.trace)):
        assert {k: v for k, v in a.items() if not k.endswith("_ms")} == \
            {k: v for k, v in b.items() if not k.endswith("_ms")}, it  # the ranks agree on every record
        for ref in (g, o):
            assert (a["rank"], a["extension_rounds"], a["kept"]) == (ref["rank"], ref["extension_rounds"],
                                                                      ref["kept"]), (it, a, ref)
            assert a["eps_threshold"] == ref["eps_threshold"]
            for k in keys:
                assert _rel(a[k], ref[k]) <= 1e-8, (it, k, a[k], ref[k])
    assert len(r0["trace"]) == len(one.trace) == len(orc.trace)
    # factors: U row blocks stacked, V / sigma replicated
    U = np.vstack([r0["U"], r1["U"]])
    np.testing.assert_allclose(r0["sigma"], one.sigma, rtol=1e-8)
    np.testing.assert_array_equal(r0["sigma"], r1["sigma"])
    X2, X1, Xo = (_probe(U, r0["sigma"], r0["V"], m, n), _probe(one.U, one.sigma, one.V, m, n),
                  _probe(orc.U, orc.sigma, orc.V, m, n))
    assert np.linalg.norm(X2 - X1) <= 1e-8 * np.linalg.norm(X1)
    assert np.linalg.norm(X2 - Xo) <= 1e-8 * np.linalg.norm(Xo)
    Ag.close()
    if Tg is not None:
        Tg.close()


def test_sharded_rank_deficient_householder_fallback(sharded):
    """qr_orthonormal keeps all columns of a rank-deficient panel
    (dense.hpp:103-110): the sharded run reveals the same rank / rounds as
    world = 1 and the oracle, the factors reproduce the rank-3 target, and the
    stacked U is orthonormal (the fallback's orthonormal fill)."""
    M = O.make_low_rank(80, 60, 3, 17)
    S = O.to_sampled(M)
    p = SketchParams(t=2, dt=4, np=1, eps_threshold=1e-12, seed=4)
    g1 = G.r3svd(G.SampledMatrix.from_csr(80, 60, S.rowptr, S.col, S.val), p)
    o = O.r3svd(S, p)
    a, b = sharded[0]["deficient"], sharded[1]["deficient"]
    assert (a["rank"], a["rounds"], a["saturated"]) == (b["rank"], b["rounds"], b["saturated"]) == \
        (g1.rank, g1.extension_rounds, g1.saturated) == (o.rank, o.extension_rounds, o.saturated)
    U = np.vstack([a["U"], b["U"]])
    np.testing.assert_allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-10)
    np.testing.assert_allclose(a["sigma"][:3], o.sigma[:3], rtol=1e-8)
    np.testing.assert_allclose((U[:, :3] * a["sigma"][:3]) @ a["V"][:, :3].T, M, atol=1e-9 * np.abs(M).max())


def test_nccl_one_rank_communicator_runs_the_distributed_path():
    """NCCL mode itself on the one GPU of the test box: a one-rank NCCL
    communicator (svt_ctx_create_dist with world = 1 and an id) takes every
    distributed branch of the engine — the row-block all-reduces through
    ncclAllReduce on the main stream, the speculative batches' Y^T X
    all-reduces on the side communicator (ncclCommSplit), the sharded QR and
    its gathered Householder fallback — and must reproduce the plain
    single-GPU run.  (Two NCCL ranks cannot share one device; the two-rank
    collective sequence is covered by the host-staged tests above.)"""
    os.environ["SVTB_SPEC_MULTI"] = "1"
    try:
        ctx = G.Context(0, 0, 1, nccl_id=G.Context.nccl_unique_id())
        for name, m, n, A, T, cfg, iters in _cases():
            cfg.maxit = iters
            Ad = G.SampledMatrix.from_csr(m, n, A.rowptr, A.col, A.val, ctx=ctx, row_block=(0, m))
            c0 = ctx.comm_stats()
            r = G.svt_run(Ad, cfg, StopRule.none())
            calls = ctx.comm_stats()["calls"] - c0["calls"]
            Ad.close()
            Ap = G.SampledMatrix.from_csr(m, n, A.rowptr, A.col, A.val)
            one = G.svt_run(Ap, cfg, StopRule.none())
            Ap.close()
            assert calls > 0, name
            assert len(r.trace) == len(one.trace)
            for it, (a, b) in enumerate(zip(r.trace, one.trace)):
                assert (a["rank"], a["extension_rounds"], a["kept"]) == (b["rank"], b["extension_rounds"],
                                                                          b["kept"]), (name, it, a, b)
                for k in ("residual", "train_mae", "rel_residual_x"):
                    assert _rel(a[k], b[k]) <= 1e-8, (name, it, k, a[k], b[k])
            np.testing.assert_allclose(r.sigma, one.sigma, rtol=1e-8)
        M = O.make_low_rank(80, 60, 3, 17)
        S = O.to_sampled(M)
        p = SketchParams(t=2, dt=4, np=1, eps_threshold=1e-12, seed=4)
        Sd = G.SampledMatrix.from_csr(80, 60, S.rowptr, S.col, S.val, ctx=ctx, row_block=(0, 80))
        f = G.r3svd(Sd, p)
        o = O.r3svd(S, p)
        assert (f.rank, f.extension_rounds, f.saturated) == (o.rank, o.extension_rounds, o.saturated)
        np.testing.assert_allclose(f.U.T @ f.U, np.eye(f.U.shape[1]), atol=1e-10)
        Sd.close()
        ctx.close()
    finally:
        os.environ.pop("SVTB_SPEC_MULTI", None)

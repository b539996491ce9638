"""The `svt` command-line front end (paper_1704_05528_b200/tools/svt_main.cpp)
against the reference's own CLI tests, proj/tests/test_cli.cpp, restated case
by case (the binary is run as a subprocess with SVT_LOG=off, as there), plus
CPU-side checks of the synth.hpp generators behind its --synthetic / bench
modes against the oracle.

Input-error cases need no device (the CLI validates its inputs before it
creates a context); the run cases are `-m gpu`."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200 import InvalidArgument, StopRule
from paper_1704_05528_b200 import formats as F
from paper_1704_05528_b200.build import CLI

gpu = pytest.mark.gpu


def run_cli(*args, log="off"):
    env = dict(os.environ, SVT_LOG=log)
    return subprocess.run([CLI, *map(str, args)], env=env, capture_output=True, text=True, timeout=600)


def write_toy_matrix(tmp, m, n, rank, fill, seed):  # test_cli.cpp:62-69
    A = F.make_low_rank(m, n, rank, seed)
    _, _, r, c, v = F.sample_dense_triplets(A, fill, seed + 1)
    path = os.path.join(tmp, "toy.mtx")
    F.write_matrix_market_triplets(path, m, n, r, c, v)
    return path


def trace_length(csv_path):  # test_cli.cpp:71-81
    with open(csv_path) as f:
        return sum(1 for line in f if line.strip() and line[0] not in "#i")


def deterministic_rows(csv_path):  # trace rows without the two timing columns (test_cli.cpp:44-60)
    with open(csv_path) as f:
        return [line.rstrip("\n").rsplit(",", 2)[0] for line in f]


# ---- generators (CPU) -----------------------------------------------------------
def test_make_low_rank_and_sample_dense_match_the_oracle():
    for (m, n, rank, seed) in ((50, 50, 3, 80), (40, 35, 3, 83), (7, 12, 2, 5)):
        A = F.make_low_rank(m, n, rank, seed)
        assert np.array_equal(A, O.make_low_rank(m, n, rank, seed))
        _, _, r, c, v = F.sample_dense_triplets(A, 0.5, seed + 1)
        ns = int(np.floor(0.5 * m * n + 1e-9))
        pos = O.sample_positions(m * n, ns, seed + 1)
        assert np.array_equal(r * n + c, pos.astype(np.int64))
        assert np.array_equal(v, A[r, c])
    with pytest.raises(InvalidArgument):
        F.make_low_rank(4, 4, 5, 1)


def test_synthetic_image_follows_synth_hpp():
    """synth.hpp:89-114 restated in numpy from the oracle's Gaussian stream."""
    size, rank, seed = 48, 5, 8
    img = F.synthetic_image(size, rank, seed)
    g = O.gaussian_block(4 * rank, 1, O.derive_seed(seed, 2)).ravel()  # the stream, in draw order
    x = np.arange(size) / (size - 1)
    M = np.zeros((size, size))
    w, k = 1.0, 0
    for t in range(rank):
        prof = []
        for _ in range(2):
            freq = 0.5 + 0.35 * t + 0.25 * abs(g[k])
            phase = np.pi * g[k + 1]
            k += 2
            prof.append(np.sin(2.0 * np.pi * freq * x + phase))
        M += np.outer(w * prof[0], prof[1])
        w *= 0.8
    ref = np.clip(np.round(255.0 * (M - M.min()) / (M.max() - M.min())), 0, 255)
    assert img.pixels.shape == (size, size)
    assert np.abs(img.pixels.astype(int) - ref.astype(int)).max() <= 1  # libm sin vs numpy at rounding ties
    assert (img.pixels.astype(int) != ref.astype(int)).mean() < 1e-3
    assert img.pixels.min() == 0 and img.pixels.max() == 255


def test_synthetic_ratings_follows_synth_hpp():
    users, items, rank, fill, noise, seed = 120, 90, 3, 0.3, 0.25, 9
    ds = F.synthetic_ratings(users, items, rank, fill, noise, seed)
    ns = int(np.floor(fill * users * items + 1e-9))
    assert ds.vals.size == ns and ds.provenance == "synthetic"
    pos = O.sample_positions(users * items, ns, O.derive_seed(seed, 3)).astype(np.int64)
    assert np.array_equal(ds.rows * items + ds.cols, pos)
    U = O.gaussian_block(users, rank, O.derive_seed(seed, 0)) / np.sqrt(rank)
    V = O.gaussian_block(items, rank, O.derive_seed(seed, 1))
    z = O.gaussian_block(ns, 1, O.derive_seed(seed, 2)).ravel()
    raw = 3.0 + np.einsum("ij,ij->i", U[ds.rows], V[ds.cols]) + noise * z
    ref = np.clip(np.round(raw * 2.0) / 2.0, 1.0, 5.0)  # numpy rounds ties to even; count those out
    ties = np.abs(raw * 2.0 - np.floor(raw * 2.0) - 0.5) < 1e-9
    assert np.array_equal(ds.vals[~ties], ref[~ties])
    assert set(np.unique(ds.vals)) <= set(np.arange(1.0, 5.5, 0.5))


# ---- input errors (CPU; no artifacts, exit 2) ---------------------------------------
def test_missing_input_exits_2_without_partial_artifacts(tmp_path):  # test_cli.cpp:121-128
    prefix = str(tmp_path / "gone")
    assert run_cli("complete", tmp_path / "missing.mtx", "--out-prefix", prefix).returncode == 2
    for suffix in (".manifest.json", ".trace.csv", ".U.mtx"):
        assert not os.path.exists(prefix + suffix)


def test_conflicting_stop_flags_are_an_input_error(tmp_path):  # test_cli.cpp:223-228
    mtx = write_toy_matrix(str(tmp_path), 20, 20, 2, 0.5, 84)
    r = run_cli("complete", mtx, "--stop-mae", 0.1, "--stop-residual", 0.1, "--out-prefix", tmp_path / "x", log="error")
    assert r.returncode == 2 and "choose one of --stop-mae / --stop-residual" in r.stderr
    assert not os.path.exists(str(tmp_path / "x") + ".manifest.json")


def test_input_errors_are_reported_before_any_device_work(tmp_path):
    assert run_cli("image").returncode == 2                                   # svt_main.cpp:586-588
    assert run_cli("image", "--synthetic", tmp_path / "a.pgm").returncode == 2  # :589-591
    assert run_cli("ratings").returncode == 2                                 # :613-615
    assert run_cli().returncode == 2                                          # no subcommand: help, exit 2
    assert run_cli("--manifest", tmp_path / "none.json").returncode == 2
    assert run_cli("--help").returncode == 0
    assert run_cli("complete").returncode != 0                                # required positional
    assert run_cli("complete", "x.mtx", "--backend", "lanczos").returncode != 0  # IsMember check
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema": "svt-run v1", "command": "teleport"}')
    r = run_cli("--manifest", bad, log="error")
    assert r.returncode == 2 and "unknown command 'teleport'" in r.stderr


# ---- runs (GPU) -----------------------------------------------------------------------
@gpu
def test_complete_writes_factors_traces_and_a_manifest(tmp_path):  # test_cli.cpp:85-112
    mtx = write_toy_matrix(str(tmp_path), 50, 50, 3, 0.5, 80)
    prefix = str(tmp_path / "run")
    r = run_cli("complete", mtx, "--stop-mae", 0.05, "--maxit", 300, "--seed", 3, "--out-prefix", prefix, log="error")
    assert r.returncode == 0, r.stderr
    for suffix in (".U.mtx", ".sigma.mtx", ".V.mtx", ".trace.csv", ".trace.json", ".manifest.json", ".metrics.json"):
        assert os.path.exists(prefix + suffix), suffix
    with open(prefix + ".trace.csv") as f:
        assert f.readline().rstrip("\n") == "# svt-trace v1"
        assert f.readline().rstrip("\n") == "iter,rank,residual,eps_threshold,train_mae,sketch_ms,total_ms"
    U = F.read_matrix_market_array(prefix + ".U.mtx")
    sg = F.read_matrix_market_array(prefix + ".sigma.mtx")
    V = F.read_matrix_market_array(prefix + ".V.mtx")
    assert U.shape[0] == 50 and V.shape[0] == 50 and U.shape[1] == sg.shape[0] and sg.shape[1] == 1
    man = json.load(open(prefix + ".manifest.json"))
    assert list(man) == ["schema", "command", "backend", "fixed_rank", "threads", "outputs", "extras", "input",
                         "config", "stop"]
    assert man["schema"] == "svt-run v1" and man["stop"] == {"rule": "train_mae", "threshold": 0.05}
    assert list(man["config"]) == ["tau", "delta", "maxit", "dt", "np", "eps_stop", "eps_threshold0", "beta", "t0",
                                   "seed"]
    met = json.load(open(prefix + ".metrics.json"))
    assert met["converged"] is True and met["iterations"] == trace_length(prefix + ".trace.csv")

    # the run is the oracle's run: same manifest config through the CPU restatement
    m, n, rr, cc, vv = F.read_matrix_market_triplets(mtx)
    S = O.sampled(m, n, rr, cc, vv)
    cfg = O.default_config(S)
    for k, v in man["config"].items():
        setattr(cfg, k, v)
    ref = O.svt_run(S, cfg, StopRule.train_mae(0.05))
    rows = [line.split(",") for line in open(prefix + ".trace.csv") if line[0] not in "#i"]
    assert abs(len(rows) - len(ref.trace)) <= 1
    for row, rec in zip(rows, ref.trace):
        assert int(row[1]) == rec["rank"]
        assert abs(float(row[2]) - rec["residual"]) <= 1e-8 * abs(rec["residual"])
        assert abs(float(row[4]) - rec["train_mae"]) <= 1e-8 * abs(rec["train_mae"])
    np.testing.assert_allclose(sg.ravel(), ref.sigma, rtol=1e-8)


@gpu
def test_full_svd_and_sketching_backends_stop_within_one_iteration(tmp_path):  # test_cli.cpp:114-127
    mtx = write_toy_matrix(str(tmp_path), 50, 50, 3, 0.5, 81)
    pa, pb = str(tmp_path / "a"), str(tmp_path / "b")
    assert run_cli("complete", mtx, "--backend", "r4svd", "--stop-mae", 0.05, "--maxit", 300, "--seed", 4,
                   "--out-prefix", pa).returncode == 0
    assert run_cli("complete", mtx, "--backend", "full-oracle", "--stop-mae", 0.05, "--maxit", 300, "--seed", 4,
                   "--out-prefix", pb).returncode == 0
    assert abs(trace_length(pa + ".trace.csv") - trace_length(pb + ".trace.csv")) <= 1


@gpu
def test_unreachable_stop_rule_exits_3_and_writes_the_best_iterate(tmp_path):  # test_cli.cpp:130-138
    mtx = write_toy_matrix(str(tmp_path), 30, 30, 2, 0.5, 82)
    prefix = str(tmp_path / "stuck")
    assert run_cli("complete", mtx, "--stop-mae", 1e-14, "--maxit", 4, "--seed", 5, "--out-prefix", prefix).returncode == 3
    assert os.path.exists(prefix + ".U.mtx")
    assert trace_length(prefix + ".trace.csv") == 4


@gpu
def test_manifest_reexecution_reproduces_a_run_bit_for_bit(tmp_path):  # test_cli.cpp:140-160
    mtx = write_toy_matrix(str(tmp_path), 40, 35, 3, 0.5, 83)
    prefix = str(tmp_path / "det")
    assert run_cli("complete", mtx, "--stop-mae", 0.05, "--maxit", 200, "--seed", 6, "--threads", 1,
                   "--out-prefix", prefix).returncode == 0
    first = {s: open(prefix + s, "rb").read() for s in (".U.mtx", ".sigma.mtx", ".V.mtx", ".manifest.json")}
    rows1 = deterministic_rows(prefix + ".trace.csv")
    assert run_cli("--manifest", prefix + ".manifest.json").returncode == 0
    for s, blob in first.items():
        assert open(prefix + s, "rb").read() == blob, s
    assert deterministic_rows(prefix + ".trace.csv") == rows1


@gpu
def test_bench_emits_one_row_per_iteration_per_backend_with_stable_ranks(tmp_path):  # test_cli.cpp:162-187
    prefix, prefix2 = str(tmp_path / "bench"), str(tmp_path / "bench2")
    args = ("bench", "--sizes", 64, "--backends", "r4svd", "--fill", 0.3, "--instance-rank", 5, "--maxit", 5, "--seed", 7)
    assert run_cli(*args, "--out-prefix", prefix).returncode == 0
    csv = prefix + ".bench64.csv"
    assert trace_length(csv) == 5
    assert run_cli(*args, "--out-prefix", prefix2).returncode == 0

    def ranks(path):
        return [line.rstrip("\n").rsplit(",", 1)[1] for line in list(open(path))[1:]]

    assert ranks(csv) == ranks(prefix2 + ".bench64.csv")
    # two backends, two sizes: one file per size, rows per backend in order
    p3 = str(tmp_path / "bench3")
    assert run_cli("bench", "--sizes", "48,64", "--backends", "r4svd,full-oracle", "--fill", 0.3, "--instance-rank", 5,
                   "--maxit", 3, "--seed", 7, "--out-prefix", p3).returncode == 0
    for size in (48, 64):
        lines = list(open(f"{p3}.bench{size}.csv"))
        assert lines[0].strip() == "iter,backend,svd_ms,rank"
        assert [ln.split(",")[1] for ln in lines[1:]] == ["r4svd"] * 3 + ["full-oracle"] * 3
        assert all(int(ln.split(",")[3]) == size for ln in lines[4:])  # full SVD reports min(m, n)


@gpu
def test_image_with_full_sampling_reproduces_the_input_up_to_quantization(tmp_path):  # test_cli.cpp:189-208
    prefix = str(tmp_path / "full")
    assert run_cli("image", "--synthetic", "--size", 48, "--synthetic-rank", 5, "--fraction", 1.0, "--maxit", 400,
                   "--seed", 8, "--out-prefix", prefix).returncode == 0
    mae = json.load(open(prefix + ".metrics.json"))["full_image_mae"]
    assert mae <= 1.5  # train stop is MAE < 1.0; quantization adds at most 0.5
    rec, orig = F.read_pgm(prefix + ".recovered.pgm"), F.read_pgm(prefix + ".original.pgm")
    assert (rec.width, rec.height) == (orig.width, orig.height) == (48, 48)
    assert np.array_equal(orig.pixels, F.synthetic_image(48, 5, F.derive_seed(8, 901)).pixels)
    assert np.abs(rec.pixels.astype(float) - orig.pixels).mean() <= 1.5


@gpu
def test_ratings_early_stop_fires_on_the_test_mae_minimum(tmp_path):  # test_cli.cpp:210-221
    prefix = str(tmp_path / "early")
    assert run_cli("ratings", "--synthetic", "--users", 120, "--items", 90, "--synthetic-rank", 3, "--fill", 0.3,
                   "--noise", 0.25, "--train-fraction", 0.8, "--early-stop-patience", 8, "--stop-mae", 1e-6,
                   "--maxit", 60, "--seed", 9, "--out-prefix", prefix).returncode == 0
    assert os.path.exists(prefix + ".test_mae.csv")
    n_it = trace_length(prefix + ".trace.csv")
    assert n_it < 60  # patience stop: far fewer iterations than the cap
    rows = [ln.strip().split(",") for ln in list(open(prefix + ".test_mae.csv"))[1:]]
    test_mae = np.array([float(r[2]) for r in rows])
    met = json.load(open(prefix + ".metrics.json"))
    assert len(rows) == n_it and met["best_test_iter"] == int(np.argmin(test_mae)) + 1
    assert n_it - met["best_test_iter"] == 8 and met["best_test_mae"] == test_mae.min()

    # the held-out column is the oracle's train_mae(test, X) on the same split
    ds = F.synthetic_ratings(120, 90, 3, 0.3, 0.25, F.derive_seed(9, 903))
    (m, n, tr, tc, tv), (_, _, er, ec, ev) = F.split_ratings_triplets(ds, 0.8, F.derive_seed(9, 904))
    man = json.load(open(prefix + ".manifest.json"))
    S, T = O.sampled(m, n, tr, tc, tv), O.sampled(m, n, er, ec, ev)
    cfg = O.default_config(S)
    for k, v in man["config"].items():
        setattr(cfg, k, v)
    cfg.maxit = n_it
    ref = O.svt_run(S, cfg, StopRule.train_mae(1e-6), test=T)
    for r, rec in zip(rows, ref.trace):
        assert abs(float(r[1]) - rec["train_mae"]) <= 1e-8 * rec["train_mae"]
        assert abs(float(r[2]) - rec["test_mae"]) <= 1e-8 * rec["test_mae"]


@gpu
def test_image_and_ratings_from_files(tmp_path):
    """The file-input modes (svt_main.cpp:597-604, 626-636): a PGM image and
    a delimited ratings file; the manifests replay from the same files."""
    img = F.synthetic_image(40, 4, 11)
    pgm = str(tmp_path / "in.pgm")
    F.write_pgm(img, pgm)
    p1 = str(tmp_path / "img")
    assert run_cli("image", pgm, "--fraction", 0.7, "--maxit", 150, "--seed", 2, "--out-prefix", p1).returncode in (0, 3)
    assert os.path.exists(p1 + ".recovered.pgm") and not os.path.exists(p1 + ".original.pgm")
    man = json.load(open(p1 + ".manifest.json"))
    assert man["input"] == {"kind": "file", "path": pgm, "fraction": 0.7} and man["stop"]["threshold"] == 1.0
    rec = F.read_pgm(p1 + ".recovered.pgm")
    assert rec.pixels.shape == img.pixels.shape
    first = open(p1 + ".sigma.mtx", "rb").read()
    assert run_cli("--manifest", p1 + ".manifest.json").returncode in (0, 3)
    assert open(p1 + ".sigma.mtx", "rb").read() == first

    ds = F.synthetic_ratings(60, 45, 3, 0.4, 0.2, 5)
    path = str(tmp_path / "ratings.dat")
    with open(path, "w") as f:
        for u, i, r in zip(ds.rows, ds.cols, ds.vals):
            f.write(f"{1000 + u}::{77 + 2 * i}::{r:g}::0\n")
    p2 = str(tmp_path / "rat")
    rc = run_cli("ratings", path, "--train-fraction", 0.8, "--maxit", 30, "--stop-mae", 0.05, "--seed", 4,
                 "--out-prefix", p2).returncode
    assert rc in (0, 3)
    users = [ln.split("\t") for ln in open(p2 + ".users.tsv").read().splitlines()]
    items = [ln.split("\t") for ln in open(p2 + ".items.tsv").read().splitlines()]
    assert len(users) == len(set(ds.rows)) and len(items) == len(set(ds.cols))
    assert all(int(uid) >= 1000 for _, uid in users) and [int(k) for k, _ in users] == list(range(len(users)))
    rows = list(open(p2 + ".test_mae.csv"))[1:]
    assert len(rows) == trace_length(p2 + ".trace.csv") > 0
    met = json.load(open(p2 + ".metrics.json"))
    assert met["final_test_mae"] == float(rows[-1].split(",")[2])

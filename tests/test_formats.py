"""Formats module (csrc/io.cpp, formats.py) against the reference's own format
tests, restated (proj/tests/test_io.cpp; io.hpp).  The parsing / writing
tests run on the CPU (the library's host code); the ones that build a device
SampledMatrix are marked gpu."""
import numpy as np
import pytest

from paper_1704_05528_b200 import formats as F
from paper_1704_05528_b200._abi import InvalidArgument, SvtRuntimeError


def _write(tmp_path, name, body, binary=False):
    p = tmp_path / name
    if binary:
        p.write_bytes(body)
    else:
        p.write_text(body)
    return str(p)


# ---- MatrixMarket (test_io.cpp:42-118) ---------------------------------------------
def test_mm_reader_comments_case_insensitive(tmp_path):  # test_io.cpp:93-109
    p = _write(tmp_path, "c.mtx", "%%MatrixMarket MATRIX Coordinate Real General\n% a comment line\n% another\n"
                                  "2 3 2\n1 2 0.5\n2 3 -1.25\n")
    m, n, r, c, v = F.read_matrix_market_triplets(p)
    assert (m, n) == (2, 3) and list(r) == [0, 1] and list(c) == [1, 2] and list(v) == [0.5, -1.25]


@pytest.mark.parametrize("name,body,msg", [
    ("h.mtx", "garbage\n1 1 1\n", "MatrixMarket"),
    ("sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n", "general"),
    ("oob.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "outside"),
    ("short.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n", "ended"),
    ("size.mtx", "%%MatrixMarket matrix coordinate real general\n2 x 3\n", "malformed size line"),
    ("nan.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n", "non-finite"),
    ("trail.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.5x\n", "trailing"),
    ("word.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 one 1.5\n", "expected an integer"),
])
def test_mm_reader_rejects_malformed(tmp_path, name, body, msg):  # test_io.cpp:65-91
    with pytest.raises(SvtRuntimeError, match=msg):
        F.read_matrix_market_triplets(_write(tmp_path, name, body))


def test_mm_reader_missing_file(tmp_path):
    with pytest.raises(SvtRuntimeError, match="cannot open"):
        F.read_matrix_market_triplets(str(tmp_path / "missing.mtx"))


def test_dense_array_round_trip_is_exact(tmp_path):  # test_io.cpp:111-118
    X = np.random.default_rng(61).standard_normal((7, 4)) * 10.0 ** np.arange(-3, 4)[:, None][:7]
    p = str(tmp_path / "dense.mtx")
    F.write_matrix_market_array(X, p)
    text = open(p).read().splitlines()
    assert text[0] == "%%MatrixMarket matrix array real general" and text[1] == "7 4"
    assert float(text[2]) == X[0, 0] and float(text[3]) == X[1, 0]  # column-major
    assert np.array_equal(F.read_matrix_market_array(p), X)


def test_dense_array_rejects_coordinate(tmp_path):
    p = _write(tmp_path, "c.mtx", "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n")
    with pytest.raises(SvtRuntimeError, match="array real general"):
        F.read_matrix_market_array(p)


# ---- PGM (test_io.cpp:120-177) -----------------------------------------------------------
def test_pgm_single_white_pixel(tmp_path):  # test_io.cpp:120-130
    p = str(tmp_path / "white.pgm")
    F.write_pgm(F.GrayImage(np.array([[255]], np.uint8)), p)
    assert open(p, "rb").read() == b"P5\n1 1\n255\n\xff"


def test_pgm_round_trip_lossless(tmp_path):  # test_io.cpp:132-148
    px = np.random.default_rng(62).integers(0, 256, size=(64, 48), dtype=np.uint8)
    p = str(tmp_path / "rt.pgm")
    F.write_pgm(F.GrayImage(px), p)
    back = F.read_pgm(p)
    assert back.width == 48 and back.height == 64 and np.array_equal(back.pixels, px)


def test_pgm_ascii_p2_with_comment(tmp_path):  # test_io.cpp:150-160
    img = F.read_pgm(_write(tmp_path, "ascii.pgm", "P2\n# comment\n3 2\n255\n0 10 20\n30 40 255\n"))
    assert (img.width, img.height) == (3, 2) and img.pixels[0, 1] == 10 and img.pixels[1, 2] == 255


def test_pgm_rejects_color_deep_truncated(tmp_path):  # test_io.cpp:162-177
    with pytest.raises(SvtRuntimeError, match="grayscale"):
        F.read_pgm(_write(tmp_path, "color.ppm", b"P6\n1 1\n255\nabc", binary=True))
    with pytest.raises(SvtRuntimeError, match="255"):
        F.read_pgm(_write(tmp_path, "deep.pgm", b"P5\n1 1\n65535\nab", binary=True))
    with pytest.raises(SvtRuntimeError, match="truncated"):
        F.read_pgm(_write(tmp_path, "short.pgm", b"P5\n4 4\n255\nabc", binary=True))


def test_quantize_rounds_and_clamps():  # test_io.cpp:224-229
    assert list(F.quantize_image(np.array([[-3.0, 0.4, 121.6, 300.0]])).pixels.ravel()) == [0, 0, 122, 255]


# ---- sample_image (test_io.cpp:179-222) ---------------------------------------------------
def _image(size, seed):
    return F.GrayImage(np.random.default_rng(seed).integers(0, 256, size=(size, size), dtype=np.uint8))


def test_sample_image_fraction_one_keeps_every_pixel():
    img = _image(16, 63)
    m, n, r, c, v = F.sample_image_triplets(img, 1.0, 64)
    assert (m, n, r.size) == (16, 16, 256)
    assert np.array_equal(v, img.pixels[r, c].astype(float))
    assert len(set(zip(r.tolist(), c.tolist()))) == 256


def test_sample_image_floored_count_and_seed_dependence():
    img = _image(512, 65)
    assert F.sample_image_triplets(img, 0.2, 66)[2].size == 52428  # floor(0.2 * 512 * 512)
    small = _image(32, 67)
    a, b = F.sample_image_triplets(small, 0.3, 1), F.sample_image_triplets(small, 0.3, 2)
    assert a[2].size == b[2].size and set(zip(a[2], a[3])) != set(zip(b[2], b[3]))


def test_sample_image_inclusion_uniform():  # test_io.cpp:204-222
    img = _image(32, 68)
    hits = np.zeros((32, 32))
    for s in range(2000):
        _, _, r, c, _ = F.sample_image_triplets(img, 0.2, 5000 + s)
        hits[r, c] += 1
    ns = int(np.floor(0.2 * 1024 + 1e-9))
    assert np.max(np.abs(hits / 2000 - ns / 1024)) <= 0.05


def test_sample_image_rejects_fraction():
    with pytest.raises(InvalidArgument):
        F.sample_image_triplets(_image(4, 1), 0.0, 1)
    with pytest.raises(InvalidArgument):
        F.sample_image_triplets(_image(4, 1), 0.01, 1)  # selects no pixel


# ---- ratings (test_io.cpp:231-345) ----------------------------------------------------------
def test_read_ratings_single_line(tmp_path):  # :231-245
    ds = F.read_ratings(_write(tmp_path, "one.dat", "1::10::4.0::978300760\n"))
    assert (ds.users, ds.items) == (1, 1) and list(ds.rows) == [0] and list(ds.cols) == [0]
    assert list(ds.vals) == [4.0] and list(ds.user_ids) == [1] and list(ds.item_ids) == [10]
    assert ds.provenance.endswith("1 ratings, 1 users, 1 items, range [4, 4]")


def test_read_ratings_rejects_duplicates_and_junk(tmp_path):  # :247-264
    with pytest.raises(SvtRuntimeError, match="duplicate rating for user id 1, item id 10"):
        F.read_ratings(_write(tmp_path, "dup.dat", "1::10::4.0\n1::10::3.0\n"))
    with pytest.raises(SvtRuntimeError):
        F.read_ratings(_write(tmp_path, "junk.dat", "1::abc::4.0\n"))
    with pytest.raises(SvtRuntimeError, match="no ratings"):
        F.read_ratings(_write(tmp_path, "empty.dat", ""))
    with pytest.raises(SvtRuntimeError, match="fewer than 3 fields"):
        F.read_ratings(_write(tmp_path, "two.dat", "1::2\n"))


def test_read_ratings_dense_frame_and_first_appearance_order(tmp_path):  # :266-275
    ds = F.read_ratings(_write(tmp_path, "toy.dat", "7::100::3.5\r\n7::200::4.0\n\n8::100::2.0\n9::200::5.0\n"))
    assert (ds.users, ds.items, ds.rows.size) == (3, 2, 4)
    assert list(ds.user_ids) == [7, 8, 9] and list(ds.item_ids) == [100, 200]
    assert list(ds.rows) == [0, 0, 1, 2] and list(ds.cols) == [0, 1, 0, 1]


def test_read_ratings_custom_separator(tmp_path):  # :277-285
    ds = F.read_ratings(_write(tmp_path, "tab.dat", "1\t2\t3.0\n2\t2\t4.5\n"), "\t")
    assert (ds.users, ds.items) == (2, 1)


def test_split_ratings_divides_and_is_disjoint():  # :287-310
    k = np.arange(10)
    ds = F.ratings_dataset(5, 4, k % 5, k % 4, k + 1.0)
    (mt, nt, rt, ct, vt), (ms, ns_, rs, cs, vs) = F.split_ratings_triplets(ds, 0.8, 70)
    assert rt.size == 8 and rs.size == 2 and mt == ms == 5 and nt == ns_ == 4
    seen = set(zip(rt.tolist(), ct.tolist()))
    assert not (seen & set(zip(rs.tolist(), cs.tolist())))
    assert sorted(vt.tolist() + vs.tolist()) == list(range(1, 11))


def test_split_ratings_deterministic_and_exhaustive():  # :312-336
    rng = np.random.default_rng(71)
    flat = rng.choice(20 * 15, size=60, replace=False)
    ds = F.ratings_dataset(20, 15, flat // 15, flat % 15, rng.integers(1, 11, 60) / 2.0)
    a, b = F.split_ratings_triplets(ds, 0.8, 72), F.split_ratings_triplets(ds, 0.8, 72)
    assert all(np.array_equal(x, y) for x, y in zip(a[0][2:], b[0][2:]))
    got = set(zip(*a[0][2:])) | set(zip(*a[1][2:]))
    assert got == set(zip(ds.rows.tolist(), ds.cols.tolist(), ds.vals.tolist()))


def test_split_ratings_rejects_degenerate():  # :338-345
    ds = F.ratings_dataset(2, 2, [0, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(InvalidArgument):
        F.split_ratings_triplets(ds, 1.0, 1)
    with pytest.raises(InvalidArgument):
        F.split_ratings_triplets(ds, 0.1, 1)


# ---- device SampledMatrix construction from the formats ----------------------------------
@pytest.mark.gpu
def test_mm_round_trip_is_exact_on_device(tmp_path):  # test_io.cpp:42-63
    from paper_1704_05528_b200 import api as G
    S1 = G.SampledMatrix(2, 2, [0], [0], [5.0])
    p1 = str(tmp_path / "single.mtx")
    F.write_matrix_market(S1, p1)
    text = open(p1).read()
    assert text.startswith("%%MatrixMarket matrix coordinate real general") and "\n2 2 1\n" in text
    assert "\n1 1 5\n" in text
    rng = np.random.default_rng(60)
    flat = rng.choice(100 * 80, size=800, replace=False)
    S = G.SampledMatrix(100, 80, flat // 80, flat % 80, rng.standard_normal(800) * 1e-7)
    p = str(tmp_path / "rt.mtx")
    F.write_matrix_market(S, p)
    R = F.read_matrix_market(p)
    assert (R.m, R.n) == (100, 80) and np.array_equal(R.rowptr, S.rowptr) and np.array_equal(R.col, S.col)
    assert np.array_equal(R.values(), S.values())


@pytest.mark.gpu
def test_mm_duplicate_rejected_by_sampled_matrix(tmp_path):  # test_io.cpp:77-80
    p = _write(tmp_path, "dup.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n")
    with pytest.raises(InvalidArgument, match="duplicate"):
        F.read_matrix_market(p)


@pytest.mark.gpu
def test_split_ratings_and_sample_image_on_device(tmp_path):
    ds = F.read_ratings(_write(tmp_path, "toy.dat", "7::100::3.5\n7::200::4.0\n8::100::2.0\n9::200::5.0\n"
                                                    "9::100::1.0\n8::300::2.5\n"))
    train, test = F.split_ratings(ds, 0.5, 3)
    assert (train.m, train.n, train.nnz, test.nnz) == (3, 3, 3, 3)
    img = _image(16, 5)
    S = F.sample_image(img, 0.5, 9)
    assert (S.m, S.n, S.nnz) == (16, 16, 128)
    D = S.dense()
    mask = D != 0
    assert np.array_equal(D[mask], img.pixels[mask].astype(float))


# ---- trace export (solver.hpp:346-386) ------------------------------------------------
def _trace():
    return [dict(iter=1, rank=10, residual=0.1, eps_threshold=0.5, train_mae=1.0 / 3.0, sketch_ms=1.23456,
                 total_ms=2.0),
            dict(iter=2, rank=20, residual=2.5e-17, eps_threshold=0.475, train_mae=0.25, sketch_ms=0.0005,
                 total_ms=1e3)]


def test_trace_csv_schema(tmp_path):
    p = str(tmp_path / "t.csv")
    F.write_trace_csv(_trace(), p)
    assert open(p).read() == ("# svt-trace v1\niter,rank,residual,eps_threshold,train_mae,sketch_ms,total_ms\n"
                              "1,10,0.10000000000000001,0.5,0.33333333333333331,1.235,2.000\n"
                              "2,20,2.4999999999999999e-17,0.47499999999999998,0.25,0.001,1000.000\n")


def test_trace_json_schema(tmp_path):
    import json
    p = str(tmp_path / "t.json")
    F.write_trace_json(_trace(), p)
    text = open(p).read()
    assert text.startswith('{\n  "schema": "svt-trace v1",\n  "rows": [\n    {"iter": 1, "rank": 10, ')
    doc = json.loads(text)
    assert doc["rows"][1]["residual"] == 2.5e-17 and doc["rows"][0]["sketch_ms"] == 1.235
    F.write_trace_json([], p)
    assert json.loads(open(p).read()) == {"schema": "svt-trace v1", "rows": []}

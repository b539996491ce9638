"""Data formats either side of the SVT path (the reference's io.hpp), over the
C ABI of libsvt_b200.so: MatrixMarket coordinate / array, PGM images,
rating triples, and the image / ratings samplers that feed SampledMatrix.

Parsing and writing run in the library (csrc/io.cpp); SampledMatrix
construction from the parsed triplets runs on the device
(svt_matrix_from_triplets: sort, validation, duplicate detection in HBM).
Errors follow the reference: malformed files raise `SvtRuntimeError`
(std::runtime_error), bad arguments `InvalidArgument`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .api import P_I64, Context, SampledMatrix, _check, _ptr, default_context, lib

P_U8 = C.POINTER(C.c_uint8)


def _L():
    L = lib()
    if not getattr(L, "_formats_ready", False):
        L.svt_triplets_provenance.restype = C.c_char_p
        L.svt_triplets_provenance.argtypes = [C.c_void_p]
        L.svt_triplets_free.argtypes = [C.c_void_p]
        L._formats_ready = True
    return L


class _Triplets:
    """Owning handle of a host triplet set (svt_triplets)."""

    def __init__(self, h):
        self.h = h

    def info(self):
        m, n, k = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_L().svt_triplets_info(self.h, C.byref(m), C.byref(n), C.byref(k)))
        return m.value, n.value, k.value

    def arrays(self):
        m, n, k = self.info()
        r = np.zeros(max(k, 1), np.int64)
        c = np.zeros(max(k, 1), np.int64)
        v = np.zeros(max(k, 1))
        _check(_L().svt_triplets_copy(self.h, _ptr(r, P_I64), _ptr(c, P_I64), _ptr(v)))
        return m, n, r[:k], c[:k], v[:k]

    def to_matrix(self, ctx: Context | None = None, row_block=None) -> SampledMatrix:
        m, n, r, c, v = self.arrays()
        return SampledMatrix(m, n, r, c, v, ctx=ctx or default_context(), row_block=row_block)

    def close(self):
        if getattr(self, "h", None):
            _L().svt_triplets_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _new(fn, *args) -> _Triplets:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return _Triplets(h)


# ---- MatrixMarket ---------------------------------------------------------------
def read_matrix_market_triplets(path: str):
    """(m, n, rows, cols, vals) of a `coordinate real general` file, 0-based,
    in file order (io.hpp:118-173)."""
    return _new(_L().svt_read_matrix_market, str(path).encode()).arrays()


def read_matrix_market(path: str, ctx: Context | None = None, row_block=None) -> SampledMatrix:
    """read_matrix_market (io.hpp:118-173) -> device SampledMatrix."""
    return _new(_L().svt_read_matrix_market, str(path).encode()).to_matrix(ctx, row_block)


def write_matrix_market(S: SampledMatrix, path: str) -> None:
    """write_matrix_market (io.hpp:176-193): 1-based, %.17g values."""
    if S.row_begin != 0 or S.row_end != S.m:
        from ._abi import InvalidArgument
        raise InvalidArgument("write_matrix_market: needs the whole matrix (single row block)")
    vals = S.values()
    _check(_L().svt_write_matrix_market(str(path).encode(), C.c_int64(S.m), C.c_int64(S.n),
                                        _ptr(np.ascontiguousarray(S.rowptr, np.int64), P_I64),
                                        _ptr(np.ascontiguousarray(S.col if S.col.size else np.zeros(1, np.int64),
                                                                  np.int64), P_I64),
                                        _ptr(vals if vals.size else np.zeros(1))))


def read_matrix_market_array(path: str) -> np.ndarray:
    """read_matrix_market_array (io.hpp:196-231): dense, column-major file."""
    r, c = C.c_int64(), C.c_int64()
    _check(_L().svt_read_matrix_market_array(str(path).encode(), C.byref(r), C.byref(c), None))
    buf = np.zeros(max(r.value * c.value, 1))
    _check(_L().svt_read_matrix_market_array(str(path).encode(), C.byref(r), C.byref(c), _ptr(buf)))
    return buf[: r.value * c.value].reshape((c.value, r.value)).T.copy()


def write_matrix_market_array(X, path: str) -> None:
    """write_matrix_market_array (io.hpp:233-246)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    buf = np.ascontiguousarray(X.T).ravel()
    _check(_L().svt_write_matrix_market_array(str(path).encode(), C.c_int64(X.shape[0]), C.c_int64(X.shape[1]),
                                              _ptr(buf if buf.size else np.zeros(1))))


# ---- PGM images ------------------------------------------------------------------
@dataclass
class GrayImage:
    """8-bit grayscale image (io.hpp:31-40); pixels[r, c]."""
    pixels: np.ndarray

    @property
    def width(self) -> int:
        return int(self.pixels.shape[1])

    @property
    def height(self) -> int:
        return int(self.pixels.shape[0])


def read_pgm(path: str) -> GrayImage:
    """read_pgm (io.hpp:272-313): P5 or P2, maxval 255."""
    w, h = C.c_int64(), C.c_int64()
    _check(_L().svt_read_pgm(str(path).encode(), C.byref(w), C.byref(h), None))
    px = np.zeros(w.value * h.value, np.uint8)
    _check(_L().svt_read_pgm(str(path).encode(), C.byref(w), C.byref(h), px.ctypes.data_as(P_U8)))
    return GrayImage(px.reshape(h.value, w.value))


def write_pgm(img: GrayImage, path: str) -> None:
    """write_pgm (io.hpp:316-327): binary P5."""
    px = np.ascontiguousarray(img.pixels, dtype=np.uint8)
    _check(_L().svt_write_pgm(str(path).encode(), C.c_int64(px.shape[1] if px.ndim == 2 else 0),
                              C.c_int64(px.shape[0] if px.ndim == 2 else 0), px.ctypes.data_as(P_U8)))


def sample_image(img: GrayImage, fraction: float, seed: int, ctx: Context | None = None) -> SampledMatrix:
    """sample_image (io.hpp:329-350): floor(fraction * w * h) distinct pixels
    (seeded partial Fisher-Yates), a height x width SampledMatrix."""
    px = np.ascontiguousarray(img.pixels, dtype=np.uint8)
    t = _new(_L().svt_sample_image, C.c_int64(img.width), C.c_int64(img.height), px.ctypes.data_as(P_U8),
             C.c_double(fraction), C.c_uint64(seed))
    return t.to_matrix(ctx)


def quantize_image(X) -> GrayImage:
    """quantize_image (io.hpp:367-381): round and clamp to [0, 255]."""
    X = np.asarray(X, dtype=np.float64)
    buf = np.ascontiguousarray(X.T).ravel()
    px = np.zeros(X.shape[0] * X.shape[1], np.uint8)
    _check(_L().svt_quantize_image(C.c_int64(X.shape[0]), C.c_int64(X.shape[1]),
                                   _ptr(buf if buf.size else np.zeros(1)), px.ctypes.data_as(P_U8)))
    return GrayImage(px.reshape(X.shape[0], X.shape[1]))


# ---- ratings -----------------------------------------------------------------------
@dataclass
class RatingsDataset:
    """RatingsDataset (io.hpp:42-50): dense user / item indices in order of
    first appearance, the original ids, the provenance line."""
    users: int
    items: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    user_ids: np.ndarray
    item_ids: np.ndarray
    provenance: str
    _handle: _Triplets = field(default=None, repr=False)


def read_ratings(path: str, separator: str = "::") -> RatingsDataset:
    """read_ratings (io.hpp:383-470)."""
    t = _new(_L().svt_read_ratings, str(path).encode(), separator.encode())
    m, n, r, c, v = t.arrays()
    uid = np.zeros(max(m, 1), np.int64)
    iid = np.zeros(max(n, 1), np.int64)
    _check(_L().svt_triplets_ids(t.h, _ptr(uid, P_I64), _ptr(iid, P_I64)))
    prov = _L().svt_triplets_provenance(t.h).decode()
    return RatingsDataset(m, n, r, c, v, uid[:m], iid[:n], prov, t)


def ratings_dataset(users, items, rows, cols, vals) -> RatingsDataset:
    """A RatingsDataset from in-memory triples (ids = the dense indices)."""
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    v = np.ascontiguousarray(vals, np.float64)
    t = _new(_L().svt_triplets_create, C.c_int64(users), C.c_int64(items), C.c_int64(r.size),
             _ptr(r if r.size else np.zeros(1, np.int64), P_I64), _ptr(c if c.size else np.zeros(1, np.int64), P_I64),
             _ptr(v if v.size else np.zeros(1)))
    return RatingsDataset(int(users), int(items), r, c, v, np.arange(users), np.arange(items), "", t)


def split_ratings_triplets(ds: RatingsDataset, train_fraction: float, seed: int):
    """Host side of split_ratings: ((m, n, rows, cols, vals) train, ... test)."""
    a, b = C.c_void_p(), C.c_void_p()
    _check(_L().svt_split_ratings(ds._handle.h, C.c_double(train_fraction), C.c_uint64(seed), C.byref(a),
                                  C.byref(b)))
    return _Triplets(a).arrays(), _Triplets(b).arrays()


def sample_image_triplets(img: GrayImage, fraction: float, seed: int):
    """Host side of sample_image: (m, n, rows, cols, vals) in draw order."""
    px = np.ascontiguousarray(img.pixels, dtype=np.uint8)
    return _new(_L().svt_sample_image, C.c_int64(img.width), C.c_int64(img.height), px.ctypes.data_as(P_U8),
                C.c_double(fraction), C.c_uint64(seed)).arrays()


def split_ratings(ds: RatingsDataset, train_fraction: float, seed: int, ctx: Context | None = None):
    """split_ratings (io.hpp:474-497): disjoint uniform train / test split in
    the same users x items frame -> (train, test) SampledMatrix."""
    a, b = C.c_void_p(), C.c_void_p()
    _check(_L().svt_split_ratings(ds._handle.h, C.c_double(train_fraction), C.c_uint64(seed), C.byref(a),
                                  C.byref(b)))
    ta, tb = _Triplets(a), _Triplets(b)
    return ta.to_matrix(ctx), tb.to_matrix(ctx)


# ---- the reference's experiment generators (synth.hpp) -------------------------------
def derive_seed(seed: int, stream: int) -> int:
    """derive_seed (dense.hpp:44)."""
    L = _L()
    L.svt_derive_seed.restype = C.c_uint64
    return int(L.svt_derive_seed(C.c_uint64(seed), C.c_uint64(stream)))


def make_low_rank(m: int, n: int, rank: int, seed: int) -> np.ndarray:
    """make_low_rank (synth.hpp:21-28): G1 G2^T / sqrt(rank)."""
    buf = np.zeros(max(m * n, 1))
    _check(_L().svt_make_low_rank(C.c_int64(m), C.c_int64(n), C.c_int64(rank), C.c_uint64(seed), _ptr(buf)))
    return buf[: m * n].reshape(n, m).T.copy()


def sample_dense_triplets(A, fraction: float, seed: int):
    """sample_dense (synth.hpp:64-84), host side: (m, n, rows, cols, vals) in draw order."""
    A = np.asarray(A, dtype=np.float64)
    buf = np.ascontiguousarray(A.T).ravel()
    return _new(_L().svt_sample_dense, C.c_int64(A.shape[0]), C.c_int64(A.shape[1]),
                _ptr(buf if buf.size else np.zeros(1)), C.c_double(fraction), C.c_uint64(seed)).arrays()


def sample_dense(A, fraction: float, seed: int, ctx: Context | None = None) -> SampledMatrix:
    m, n, r, c, v = sample_dense_triplets(A, fraction, seed)
    return SampledMatrix(m, n, r, c, v, ctx=ctx or default_context())


def synthetic_image(size: int, rank: int, seed: int) -> GrayImage:
    """synthetic_image (synth.hpp:89-114)."""
    px = np.zeros(max(size * size, 1), np.uint8)
    _check(_L().svt_synthetic_image(C.c_int64(size), C.c_int64(rank), C.c_uint64(seed), px.ctypes.data_as(P_U8)))
    return GrayImage(px[: size * size].reshape(size, size))


def synthetic_ratings(users: int, items: int, rank: int, fill: float, noise: float, seed: int) -> RatingsDataset:
    """synthetic_ratings (synth.hpp:119-160)."""
    t = _new(_L().svt_synthetic_ratings, C.c_int64(users), C.c_int64(items), C.c_int64(rank), C.c_double(fill),
             C.c_double(noise), C.c_uint64(seed))
    m, n, r, c, v = t.arrays()
    return RatingsDataset(m, n, r, c, v, np.arange(m), np.arange(n), "synthetic", t)


def write_matrix_market_triplets(path: str, m: int, n: int, rows, cols, vals) -> None:
    """write_matrix_market (io.hpp:176-193) of host triplets (validated and
    ordered like the SampledMatrix constructor, sampled.hpp:27-62)."""
    from .api import build_csr
    rp, co, va = build_csr(m, n, rows, cols, vals)
    _check(_L().svt_write_matrix_market(str(path).encode(), C.c_int64(m), C.c_int64(n), _ptr(rp, P_I64),
                                        _ptr(co, P_I64), _ptr(va)))


# ---- trace export ------------------------------------------------------------------------
def _records(trace):
    from ._abi import IterationRecord
    arr = (IterationRecord * max(len(trace), 1))()
    for i, rec in enumerate(trace):
        for name, _ in IterationRecord._fields_:
            if name in rec:
                setattr(arr[i], name, rec[name])
    return arr


def write_trace_csv(trace, path: str) -> None:
    """write_trace_csv (solver.hpp:346-364), schema "svt-trace v1"; trace is
    SvtResult.trace (a list of IterationRecord dicts)."""
    _check(_L().svt_write_trace(_records(trace), C.c_int64(len(trace)), str(path).encode(), C.c_int(0)))


def write_trace_json(trace, path: str) -> None:
    """write_trace_json (solver.hpp:366-386)."""
    _check(_L().svt_write_trace(_records(trace), C.c_int64(len(trace)), str(path).encode(), C.c_int(1)))

"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/svt_b200.h declares, and its host-only entry points (SampledMatrix
construction, row partitioning, synthetic configs) behave like the
reference.  No compute call here touches a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1704_05528_b200 import InvalidArgument
from paper_1704_05528_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "svt_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|void\*|const char\*|int64_t|uint64_t) (svt_[a-z0-9_]+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = api.lib()
    names = declared_symbols()
    assert len(names) >= 40
    for n in names:
        assert hasattr(L, n), n


def test_build_csr_matches_reference_ctor():
    rng = np.random.default_rng(3)
    m, n = 37, 23
    cells = rng.choice(m * n, 200, replace=False)
    r, c = cells // n, cells % n
    v = rng.standard_normal(200)
    rp, co, va = api.build_csr(m, n, r, c, v)
    ref = O.sampled(m, n, r, c, v)
    assert np.array_equal(rp, ref.rowptr) and np.array_equal(co, ref.col) and np.array_equal(va, ref.val)


@pytest.mark.parametrize("case", [
    (2, 2, [], [], []), (2, 2, [0], [2], [1.0]), (2, 2, [-1], [0], [1.0]),
    (2, 2, [0, 0], [0, 0], [1.0, 2.0]), (2, 2, [0], [0], [np.nan]), (0, 2, [0], [0], [1.0])])
def test_build_csr_rejects_like_reference(case):  # test_sampled.cpp:10-17
    with pytest.raises(InvalidArgument):
        api.build_csr(*case)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_rows_balances_nnz(world):
    rng = np.random.default_rng(world)
    deg = np.maximum(1, (rng.pareto(1.6, 5000) * 20).astype(np.int64))
    rp = np.concatenate([[0], np.cumsum(deg)])
    b = api.partition_rows(rp, world)
    assert b[0] == 0 and b[-1] == 5000 and (np.diff(b) >= 0).all()
    loads = rp[b[1:]] - rp[b[:-1]]
    assert loads.sum() == rp[-1]
    assert loads.max() <= rp[-1] / world + deg.max()


def test_synth_config1_restates_reference_sampler():
    d = api.synth_config(1, seed=7)
    r, c, v = d["train"]
    assert d["m"] == d["n"] == 1000 and len(v) == 200000 and d["test"] is None
    pos = O.sample_positions(1000 * 1000, 200000, O.derive_seed(7, 3))
    assert np.array_equal(r * 1000 + c, pos.astype(np.int64))
    L = O.gaussian_block(1000, 10, O.derive_seed(7, 1))
    R = O.gaussian_block(1000, 10, O.derive_seed(7, 2))
    np.testing.assert_allclose(v[:500], np.einsum("ij,ij->i", L[r[:500]], R[c[:500]]), rtol=1e-12, atol=1e-12)


def test_synth_config2_image_range():
    d = api.synth_config(2, seed=3)
    r, c, v = d["train"]
    assert d["m"] == d["n"] == 512 and len(v) == 131072
    assert v.min() >= 0.0 and v.max() <= 255.0
    assert len(np.unique(r * 512 + c)) == len(v)


def test_synth_config3_shape_and_split():
    d = api.synth_config(3, seed=1)
    r, c, v = d["train"]
    tr, tc, tv = d["test"]
    assert d["m"] == 6040 and d["n"] == 3706
    assert len(v) == 900188 and len(tv) == 100021  # floor(0.9 * 1,000,209)
    assert set(np.unique(v)).issubset({1.0, 2.0, 3.0, 4.0, 5.0})
    deg = np.bincount(np.concatenate([r, tr]), minlength=6040)
    assert deg.min() >= 20 and deg.sum() == 1000209
    allc = np.concatenate([r * 3706 + c, tr * 3706 + tc])
    assert len(np.unique(allc)) == len(allc)


def test_synth_deterministic():
    a = api.synth_config(1, seed=11)["train"][2]
    api.synth_config(2, seed=1)  # evict the cache
    b = api.synth_config(1, seed=11)["train"][2]
    assert np.array_equal(a, b)

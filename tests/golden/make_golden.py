"""Regenerates tests/golden/*.npz from the CPU oracle.

Run after the oracle's RNG is pinned against the C++ standard's mt19937_64
known answer (tests/test_oracle_dense.py).  The fixtures freeze the
column-major Box-Muller fill (dense.hpp:56-98) so GPU-side RNG tests have a
committed reference that does not depend on rebuilding the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [(3, 2, 7), (1000, 1, 1), (5, 3, 42), (33, 10, 0x9E3779B97F4A7C15), (311, 1, 5), (313, 2, 6),
         (1, 1, 3), (157, 3, 8)]

if __name__ == "__main__":
    blocks = {f"g_{r}_{c}_{s}": O.gaussian_block(r, c, s) for r, c, s in CASES}
    np.savez_compressed(os.path.join(HERE, "gaussian_block.npz"), **blocks)
    print("wrote", len(blocks), "blocks")

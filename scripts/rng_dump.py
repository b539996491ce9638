import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from paper_1704_05528_b200 import api as G
out = {}
for (r, c, s) in [(1000, 10, 7), (100000, 10, 3), (10677, 10, 99), (5, 3, 1), (7, 1, 2)]:
    out[f"{r}_{c}_{s}"] = G.gaussian_block(r, c, s)
np.savez(sys.argv[1], **out)

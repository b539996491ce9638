"""One device eigensolve of a graded Gram (for ncu captures of the Jacobi kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402
from scripts.eig_bench import gram  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 512
decay = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
A = gram(r, max(r, 512), decay, r)
lam, W = G.dev_sym_eig(A)
torch.cuda.synchronize()
print("ok", lam[0].item())

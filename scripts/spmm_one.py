"""A few launches of the library's sparse product on config 4 (profiling
target): python scripts/spmm_one.py [w] [transpose] [config]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 120
tr = int(sys.argv[2]) if len(sys.argv) > 2 else 0
config = int(sys.argv[3]) if len(sys.argv) > 3 else 4
d = G.synth_config(config, 1)
m, n = d["m"], d["n"]
A = G.SampledMatrix(m, n, *d["train"])
ri, ro = (m, n) if tr else (n, m)
X = torch.randn(ri, w, dtype=torch.float64, device="cuda")
O = torch.zeros(ro, w, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    G.lib().svt_dev_sp_mult(A.h, tr, C.c_int64(w), C.c_void_p(X.data_ptr()), C.c_int64(w),
                            C.c_void_p(O.data_ptr()), C.c_int64(w))
A.ctx.sync()
print("ok", float(O.abs().sum()))

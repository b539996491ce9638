"""Does the panel row alignment matter for the wide gather SpMM?  Times
svt_dev_sp_mult on config 4 at panel widths w with ld = w and with ld
padded to a multiple of 16 doubles (128-byte aligned rows)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402

ctx = G.default_context()
L = G.lib()
st = torch.cuda.ExternalStream(ctx.stream)
d = G.synth_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4, 1)
m, n = d["m"], d["n"]
A = G.SampledMatrix(m, n, *d["train"])


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for w in (64, 80, 96, 112, 120, 128):
    for ld in sorted({w, (w + 15) // 16 * 16}):
        for tr in (0, 1):
            ri, ro = (m, n) if tr else (n, m)
            X = torch.randn(ri, ld, dtype=torch.float64, device="cuda")
            O = torch.zeros(ro, ld, dtype=torch.float64, device="cuda")
            t = timed(lambda: L.svt_dev_sp_mult(A.h, tr, C.c_int64(w), C.c_void_p(X.data_ptr()), C.c_int64(ld),
                                                C.c_void_p(O.data_ptr()), C.c_int64(ld)))
            print(f"w={w:4d} ld={ld:4d} {'Y^T X' if tr else 'Y X  '}: {t:8.1f} us  "
                  f"gather {A.nnz * w * 8 / t / 1e6:6.2f} TB/s", flush=True)

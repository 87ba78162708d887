"""Per-phase accumulated times of the column-tile kernel over one step launch (debug build with -DKFP_TRACE):

    nvcc ... -DKFP_TRACE -o tools/libkfp_trace.so paper_1306_4596_b200/csrc/kfp_api.cu
    KFP_LIB_PATH=tools/libkfp_trace.so python tools/trace_col.py c2
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import kfp  # noqa: E402

run = ki.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
pb = kfp.Problem(ki.make_problem(ki.scaled(run, nt=20, K=1, t_final=run.grid.t_final / run.grid.nt * 20)))
pb.setup(run.kind, run.p, run.overlap, run.n_sub, 4)
lib = kfp.load()
cap = 1 << 12
buf = np.zeros((cap, 64), dtype=np.uint64)
for rep in range(3):
    rc = lib.kfp_debug_trace_step(pb._h, ctypes.c_int(5), buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(cap))
t = buf[(buf[:, :9].sum(axis=1)) > 0].astype(np.float64)
print("rc", rc, "ctas", len(t), pb.plan())
names = ["tables+bar", "dataWait", "passA", "issueNext", "passB", "S1", "column", "S2", "passC+loop"]
tot = t[:, :9].sum(axis=1)
print("per-CTA accounted time us: median %.2f  max %.2f" % (np.median(tot) / 1e3, tot.max() / 1e3))
for i, nm in enumerate(names):
    print(f"{nm:>12s}: median {np.median(t[:, i]) / 1e3:8.2f} us ({100 * np.median(t[:, i] / tot):5.1f}%)  max {t[:, i].max() / 1e3:8.2f}")

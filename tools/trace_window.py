"""Per-phase accumulated times of the window kernel over one SWR iteration (debug build with -DKFP_TRACE):

    nvcc ... -DKFP_TRACE -o tools/libkfp_trace.so paper_1306_4596_b200/csrc/kfp_api.cu
    KFP_LIB_PATH=tools/libkfp_trace.so python tools/trace_window.py c2 [nt]
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import kfp  # noqa: E402

os.environ.setdefault("KFP_WINDOW", "1")
run = ki.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 100
pb = kfp.Problem(ki.make_problem(ki.scaled(run, nt=nt, K=1, t_final=run.grid.t_final / run.grid.nt * nt)))
pb.setup(run.kind, run.p, run.overlap, run.n_sub, 8)
lib = kfp.load()
cap = 1 << 12
buf = np.zeros((cap, 64), dtype=np.uint64)
for rep in range(2):
    t0 = time.perf_counter()
    rc = lib.kfp_debug_trace_window(pb._h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(cap))
    wall = time.perf_counter() - t0
t = buf[(buf[:, :9].sum(axis=1)) > 0].astype(np.float64)
print("rc", rc, "ctas", len(t), "wall ms %.2f" % (wall * 1e3), pb.plan(), "nt", nt)
names = ["Xwait", "L2+S2", "passC+ends", "S3", "dataWait", "passAB", "S1", "poll+L1+push", "drainWait"]
tot = t[:, :9].sum(axis=1)
print("per-CTA accounted time us: median %.1f" % (np.median(tot) / 1e3))
for i, nm in enumerate(names):
    print(f"{nm:>14s}: median {np.median(t[:, i]) / 1e3:9.1f} us  ({100 * np.median(t[:, i] / tot):5.1f}%)  max {t[:, i].max() / 1e3:9.1f}")
print("drains per CTA: median", np.median(t[:, 9]), "max", t[:, 9].max())

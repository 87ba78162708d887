"""Per-CTA, per-tile phase timeline of one fused step launch (debug build with -DKFP_TRACE):

    nvcc ... -DKFP_TRACE -o /tmp/libkfp_trace.so paper_1306_4596_b200/csrc/kfp_api.cu
    KFP_LIB_PATH=/tmp/libkfp_trace.so python tools/trace_step.py c2
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
t = buf[buf[:, 0] > 0].astype(np.int64)
t0 = t[:, 0].min()
print("rc", rc, "ctas", len(t), "span us", (t[:, 63].max() - t0) / 1e3, pb.plan())
us = lambda x: x / 1e3  # noqa: E731
print("start->t0issued median %.3f" % np.median(us(t[:, 1] - t[:, 0])))
names = ["ready", "passAB", "pushed", "Xrecv", "L2done", "tileEnd"]
for it in range(9):
    ev = t[:, 2 + 6 * it: 8 + 6 * it]
    ok = ev[:, 0] > 0
    if not ok.any():
        break
    ev = ev[ok]
    prev_end = t[ok, 1] if it == 0 else t[ok, 2 + 6 * (it - 1) + 5]
    cols = [ev[:, 0] - prev_end] + [ev[:, e] - ev[:, e - 1] for e in range(1, 6)]
    s = "  ".join(f"{nm}:{np.median(us(c)):6.2f}/{np.percentile(us(c), 90):6.2f}" for nm, c in zip(names, cols))
    print(f"tile {it} (n={ok.sum():4d}) abs ready {np.median(us(ev[:, 0] - t0)):7.2f}  {s}")
life = us(t[:, 63] - t[:, 0])
print("lifetime median %.2f p90 %.2f" % (np.median(life), np.percentile(life, 90)))
print("start quantiles us", np.round(np.percentile(us(t[:, 0] - t0), [10, 50, 90, 100]), 2))
print("end quantiles us", np.round(np.percentile(us(t[:, 63] - t0), [10, 50, 90, 100]), 2))

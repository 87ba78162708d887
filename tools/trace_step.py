"""Per-CTA phase timeline of one fused step launch (debug build with -DKFP_TRACE, KFP_LIB_PATH=...)."""
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
cap = 1 << 16
buf = np.zeros((cap, 8), dtype=np.uint64)
for rep in range(3):
    rc = lib.kfp_debug_trace_step(pb._h, ctypes.c_int(5), buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(cap))
t = buf[buf[:, 0] > 0].astype(np.int64)
t0 = t[:, 0].min()
t = t - t0
print("rc", rc, "ctas", len(t), "span us", (t[:, 7].max()) / 1e3, pb.plan())
names = ["start", "t0issued", "passAB(lastT)", "pushed", "Xrecv", "L2done", "tileEnd", "end"]
for i in range(7):
    a, b = t[:, i], t[:, i + 1]
    ok = (b > 0) | (i == 6)
    col = (b - a)[ok & (b >= a)] / 1e3
    if col.size:
        print(f"{names[i]:>8s}->{names[i+1]:<8s} median {np.median(col):8.3f} us  p90 {np.percentile(col, 90):8.3f}  max {col.max():8.3f}")
life = (t[:, 7] - t[:, 0]) / 1e3
print("lifetime median", np.median(life), "p90", np.percentile(life, 90))
st = np.sort(t[:, 0]) / 1e3
print("start quantiles us", np.percentile(st, [10, 25, 50, 75, 90, 100]))
en = np.sort(t[:, 7]) / 1e3
print("end quantiles us", np.percentile(en, [10, 25, 50, 75, 90, 100]))

"""c2 / c3 / c4w1 throughput at pipeline depths 1, 2, 5, 10 (the big windows; kfp_swr_set_pipeline)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import kfp_inputs as ki  # noqa: E402
from tools.pipeline_speed import timed  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    run = ki.config(name)
    g = run.grid
    ups = g.nx * g.nv * g.nt * run.K
    for d in (1, 2, 5, 10):
        if d > run.K or (d > 1 and run.K % d):
            continue
        t, e = timed(run, d)
        print(f"{name} depth {d}: {t:.1f} ms  {ups / t / 1e6:.1f} G upd/s  err_if[-1] {e:.6e}", flush=True)

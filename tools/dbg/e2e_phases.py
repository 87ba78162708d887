"""Host-timed phases of the bench's timed e2e solve (create / solve / history / destroy), repeated."""
import dataclasses
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

run = ki.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
prob = ki.make_problem(run)
g = run.grid


def pinned_copy(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t


pins = [pinned_copy(np.asarray(x, dtype=np.float64)) for x in (prob.ft, prob.fv, prob.fx, prob.u0v, prob.u0x)]
pp = dataclasses.replace(prob, **{k: t.numpy() for k, t in zip(("ft", "fv", "fx", "u0v", "u0x"), pins)})
uT = torch.empty((g.nv + 1, g.nx), dtype=torch.float64, pin_memory=True)
stream = torch.cuda.current_stream()
for rep in range(5):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    q = Problem(pp, device=0)
    q.set_stream(stream.cuda_stream)
    t.append(time.perf_counter())
    q.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    q.iterate(run.K)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    q.close() if hasattr(q, "close") else q.__exit__(None, None, None)
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with Problem(pp, device=0) as q2:
        q2.set_stream(stream.cuda_stream)
        q2.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, out=uT.numpy())
        q2.history()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d = np.diff(t) * 1e3
    print(f"rep {rep}: create {d[0]:.1f} setup {d[1]:.1f} iterate {d[2]:.1f} destroy {d[3]:.1f} | solve-leg {1e3*(t1-t0):.1f} ms",
          flush=True)

"""Differential check of the window kernel against the per-step fused kernel (same problem, same setup)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 20
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1
run = ki.config(wl)
run = ki.scaled(run, nt=nt, K=K, t_final=run.grid.t_final / run.grid.nt * nt)
prob = ki.make_problem(run)


def solve(env):
    env = dict(env, **({} if "KFP_NO_WINDOW" in env else {"KFP_WINDOW": "1"}))
    for k in ("KFP_NO_WINDOW", "KFP_WIN_G", "KFP_WINDOW"):
        os.environ.pop(k, None)
    os.environ.update(env)
    with Problem(prob) as pb:
        pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
        sl = [pb.subdomain_uT(s) for s in range(run.n_sub)]
        return pb.plan(), sl, pb.history()


ref_plan, ref, ref_h = solve({"KFP_NO_WINDOW": "1"})
print("reference", ref_plan, ref_h)
for env in ({}, {"KFP_WIN_G": "1"}, {"KFP_WIN_G": "2"}, {"KFP_WIN_G": "8"}):
    plan, sl, h = solve(env)
    errs = []
    for a, b in zip(sl, ref):
        d = np.abs(a - b)
        bad = np.argwhere(d > 1e-9 * np.abs(b).max())
        errs.append((d.max() / np.abs(b).max(), len(bad), bad[:3].tolist()))
    print(env, plan, "hist", h, "rel/nbad/first", errs, flush=True)

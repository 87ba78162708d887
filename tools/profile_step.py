"""Short run of one workload's SWR solve for ncu captures (a few windows of the real grid)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--nt", type=int, default=20)
ap.add_argument("--K", type=int, default=2)
a = ap.parse_args()
run = ki.config(a.workload)
g = run.grid
run = ki.scaled(run, nt=a.nt, K=a.K, t_final=g.t_final / g.nt * a.nt)
with Problem(ki.make_problem(run)) as pb:
    pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
    print(pb.plan(), pb.history())

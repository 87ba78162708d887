"""The monodomain reference of a tall column (the c4w8 grid: 2048 x 32768, 32767 unknown rows: three-phase path),
a few steps, for ncu captures of its kernels."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4w8")
ap.add_argument("--nt", type=int, default=6)
a = ap.parse_args()
run = ki.config(a.workload) if not a.workload.startswith("c4w") else ki.weak_scaling_config(int(a.workload[3:]))
g = run.grid
run = ki.scaled(run, nt=a.nt, t_final=g.t_final / g.nt * a.nt)
with Problem(ki.make_problem(run)) as pb:
    pb.monodomain(copy=False)
    print("monodomain", run.grid)

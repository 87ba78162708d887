"""Tiny solves for debugging on the GPU box: c0 monodomain and one SWR iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.scaled(ki.config(sys.argv[1] if len(sys.argv) > 1 else "c0"), K=1)
with Problem(ki.make_problem(run)) as pb:
    U = pb.monodomain()
    print("mono ok", abs(U).max())
    pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K)
    print("swr ok", pb.history())

"""Monodomain reference speed for the weak-scaling family (cluster kernel vs three-phase path; debugging aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
for g in (1, 2, 4, 8):
    run = ki.config(f"c4w{g}")
    gr = run.grid
    with Problem(ki.make_problem(run)) as pb:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        pb.monodomain(copy=False)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        ups = gr.nx * gr.nv * gr.nt
        print(f"c4w{g}: nv={gr.nv} monodomain {1e3*(t1-t0):8.1f} ms = {ups/(t1-t0)/1e9:6.1f} G upd/s  plan {pb.plan()}", flush=True)

"""Pipeline depth sweep on mid-size workloads (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
for run in [ki.config("paper_j4"), ki.config("c4w1"), ki.config("c3").with_(K=4)]:
    g = run.grid
    for D in (1, 2, 3, 4):
        with Problem(ki.make_problem(run)) as pb:
            pb.set_stream(stream.cuda_stream)
            pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
            if D > 1:
                pb.set_pipeline(D)
            ts = []
            for rep in range(2):
                pb.reset()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record(stream); pb.iterate(run.K); e1.record(stream); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ups = g.nx * g.nv * g.nt * run.K
            print(f"{run.name:10s} D={D}: {min(ts):9.1f} ms  {ups / min(ts) / 1e6:7.1f} G upd/s  plan {pb.plan()}", flush=True)

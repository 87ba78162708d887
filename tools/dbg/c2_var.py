"""Per-solve timing variance of c2 (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.config("c2")
stream = torch.cuda.current_stream()
pb = Problem(ki.make_problem(run)); pb.set_stream(stream.cuda_stream)
pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
for i in range(8):
    pb.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(stream); pb.iterate(run.K); e1.record(stream); torch.cuda.synchronize()
    it_ms, k_ms = pb.last_timing()
    print(f"solve {i}: {e0.elapsed_time(e1):8.2f} ms (library windows {k_ms:8.2f} ms)", flush=True)

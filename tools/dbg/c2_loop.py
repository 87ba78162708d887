"""bench.py's timed loop vs a bare iterate loop on c2 (debugging aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.config("c2")
stream = torch.cuda.current_stream()
pb = Problem(ki.make_problem(run)); pb.set_stream(stream.cuda_stream)
pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
def one():
    pb.reset(); pb.iterate(run.K)
for _ in range(2): one()
torch.cuda.synchronize()
for variant in ("bench loop (last_timing inside)", "no last_timing", "bench loop again"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record(stream)
    for _ in range(3):
        one()
        if "no last" not in variant:
            pb.last_timing()
    e1.record(stream); torch.cuda.synchronize()
    print(f"{variant}: {e0.elapsed_time(e1)/3:8.2f} ms/solve (wall {1e3*(time.perf_counter()-t0)/3:8.2f})", flush=True)
    t0 = time.perf_counter(); one(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"   host enqueue of one solve {1e3*(t1-t0):8.2f} ms, drain {1e3*(t2-t1):8.2f} ms", flush=True)

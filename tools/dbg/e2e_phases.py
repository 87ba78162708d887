"""Host-side phases of one end-to-end c2 solve through the public API (debugging aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.config("c2"); g = run.grid
prob = ki.make_problem(run)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
out = torch.empty((g.nv + 1, g.nx), dtype=torch.float64, pin_memory=True).numpy()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pb = Problem(prob); pb.set_stream(stream.cuda_stream); torch.cuda.synchronize(); t1 = time.perf_counter()
    pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K); torch.cuda.synchronize(); t2 = time.perf_counter()
    pb.reset(); pb.iterate(run.K); torch.cuda.synchronize(); t3 = time.perf_counter()
    import ctypes
    from paper_1306_4596_b200 import kfp
    pb.history(); t4 = time.perf_counter()
    pb.close(); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):7.1f} ms  setup(+monodomain) {1e3*(t2-t1):7.1f}  iterate {1e3*(t3-t2):7.1f}  "
          f"history {1e3*(t4-t3):6.1f}  destroy {1e3*(t5-t4):6.1f}", flush=True)

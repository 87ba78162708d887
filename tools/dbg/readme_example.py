"""The README usage example, verbatim (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.config("c2")
with Problem(ki.make_problem(run)) as pb:
    uT = pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K)      # q=... for OSWR(p, q)
    err_T, err_if = pb.history()

# the paper's own experiment: split-FEM scheme, SWR1-SWR4, random lambda^0, stop on |u1 - u2| < 1e-6
import numpy as np
g = ki.paper_grid(2)                                      # Delta t = h_x = h_v = 0.0025, T = 2
with Problem(ki.fem_problem(g)) as pb:                    # scheme "split_fem"
    pb.setup("robin", 11.0, 3, 2, 150, q=2.5)             # OSWR(p, q), overlap 3 h_v, K_max
    pb.set_schedule("gauss_seidel")
    pb.set_overlap_error(True)                            # err_ov = max |u_s - u_{s+1}| on the overlaps
    pb.set_pipeline(8)                                    # wavefront: 8 iterations per sweep, bitwise identical
    pb.reset()
    pb.set_initial_trace(0, 0, np.random.default_rng(0).uniform(-1, 1, (g.nt, g.nx)))
    k = pb.iterate_until(1e-6, 150, "overlap")            # the paper's Table 1 count for this level

print("c2 err_T[-1]", err_T[-1], "paper j2 iterations", k)

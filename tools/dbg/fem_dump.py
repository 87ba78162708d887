"""Dump GPU FEM monodomain results for offline comparison (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import kfp_inputs as ki
from paper_1306_4596_b200 import kfp

out = {}
for nv, nt in [(40, 2), (200, 2)]:
    g = ki.Grid(64, nv, nt, 1.0, 0.01 * nt)
    with kfp.Problem(ki.fem_problem(g, 1)) as pb:
        out[f"UT_{nv}_{nt}"] = pb.monodomain()
np.savez("gpurun_out/fem_dump.npz", **out)

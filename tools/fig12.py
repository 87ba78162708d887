"""The paper's Figs. 1-2 with the batched Robin-parameter sweep: on the Table 1 setup at j = 0
(Delta t = h_x = h_v = 0.01, T = 2, overlap 3 h_v, random lambda^0, SWR1-SWR4), the iteration count to reach
eps = 1e-6 and the interface error after 15 iterations, for OSWR(p) over a p grid (Fig. 1) and OSWR(p, q)
over a (p, q) grid (Fig. 2) -- every parameter value a replica of ONE batched solve.

    python tools/fig12.py > profiles/r1_fig12.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

EPS, K = 1e-6, 40


def sweep(ps, qs, ov=3):
    g = ki.Grid(100, 200, 200, 1.0, 2.0)
    rng = np.random.default_rng(1000)
    lam = [rng.uniform(-1.0, 1.0, size=(g.nt, g.nx)) for _ in range(2)]
    t0 = time.perf_counter()
    with Problem(ki.zero_problem(g)) as pb:
        pb.setup_batch("robin", ps, ov, 2, K, qs=qs)
        pb.set_schedule("gauss_seidel")
        pb.reset()
        pb.set_initial_trace(0, 0, lam[0])
        pb.set_initial_trace(0, 1, lam[1])
        pb.iterate(K)
        hist = [pb.batch_history(r)[1] for r in range(len(ps))]
    its = [int(np.argmax(h < EPS)) + 1 if (h < EPS).any() else None for h in hist]
    return its, [float(h[14]) for h in hist], time.perf_counter() - t0


ps1 = np.round(np.arange(1.0, 12.01, 0.1), 3)
its1, e15_1, t1 = sweep(ps1, None)
best1 = int(np.argmin(e15_1))
grid = np.round(np.geomspace(0.5, 40.0, 20), 3)
P2, Q2 = np.meshgrid(grid, grid, indexing="ij")
its2, e15_2, t2 = sweep(P2.ravel(), Q2.ravel())
best2 = int(np.argmin(e15_2))
out = {
    "setup": "Table 1 j=0 grid, overlap 3 h_v, random lambda^0 ~ U(-1,1), Gauss-Seidel, eps 1e-6",
    "fig1": {"p": ps1.tolist(), "iterations": its1, "err_if_after_15": e15_1, "seconds": t1,
             "p_star_min_error_15": float(ps1[best1]), "iterations_at_p_star": its1[best1]},
    "fig2": {"p": P2.ravel().tolist(), "q": Q2.ravel().tolist(), "iterations": its2, "err_if_after_15": e15_2,
             "seconds": t2, "pq_star_min_error_15": [float(P2.ravel()[best2]), float(Q2.ravel()[best2])],
             "iterations_at_pq_star": its2[best2]},
}
print(json.dumps(out))
print(f"fig1: {len(ps1)} replicas in {t1:.1f} s, p* = {ps1[best1]} (err15 {e15_1[best1]:.2e}, {its1[best1]} its); "
      f"fig2: {P2.size} replicas in {t2:.1f} s, (p,q)* = ({P2.ravel()[best2]}, {Q2.ravel()[best2]}) "
      f"(err15 {e15_2[best2]:.2e}, {its2[best2]} its)", file=sys.stderr)

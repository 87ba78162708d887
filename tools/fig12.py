"""The paper's Figs. 1-2 with the batched Robin-parameter sweep: on the Table 1 setup at j = 0
(Delta t = h_x = h_v = 0.01, T = 2, overlap 3 h_v, random lambda^0, SWR1-SWR4), the iteration count to reach
eps = 1e-6 and the interface error after 15 iterations, for OSWR(p) over a p grid (Fig. 1) and OSWR(p, q)
over a (p, q) grid (Fig. 2) -- every parameter value a replica of ONE batched solve.

    python tools/fig12.py > profiles/r1_fig12.json                    (IMEX FD, err_if)
    python tools/fig12.py --scheme fem > profiles/r1_fig12_fem.json   (the paper's split FEM and its
        stopping quantity max |u1 - u2| on the overlap; plus a fine p grid on [3.5, 5.5])
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

EPS, K = 1e-6, 40


ap = argparse.ArgumentParser()
ap.add_argument("--scheme", choices=["fd", "fem"], default="fd")
A = ap.parse_args()
FEM = A.scheme == "fem"


def sweep(ps, qs, ov=3):
    g = ki.Grid(100, 200, 200, 1.0, 2.0)
    rng = np.random.default_rng(1000)
    lam = [rng.uniform(-1.0, 1.0, size=(g.nt, g.nx)) for _ in range(2)]
    t0 = time.perf_counter()
    with Problem(ki.fem_problem(g) if FEM else ki.zero_problem(g)) as pb:
        pb.setup_batch("robin", ps, ov, 2, K, qs=qs)
        pb.set_schedule("gauss_seidel")
        if FEM:
            pb.set_overlap_error(True)
        pb.reset()
        pb.set_initial_trace(0, 0, lam[0])
        pb.set_initial_trace(0, 1, lam[1])
        pb.iterate(K)
        hist = [pb.overlap_history(r) if FEM else pb.batch_history(r)[1] for r in range(len(ps))]
    its = [int(np.argmax(h < EPS)) + 1 if (h < EPS).any() else None for h in hist]
    HIST[len(HIST)] = [list(map(float, h)) for h in hist]
    return its, [float(h[14]) for h in hist], time.perf_counter() - t0


HIST = {}  # full error histories of every sweep (replica-major)


def argmin_at(ps, hist, k):
    """p minimising the error after k iterations (k = 5..8 stay above round-off; at 15 every good p is at it)."""
    e = [h[k - 1] for h in hist]
    return float(np.asarray(ps)[int(np.argmin(e))]), float(min(e))


ps1 = np.round(np.arange(1.0, 12.01, 0.1), 3)
its1, e15_1, t1 = sweep(ps1, None)
best1 = int(np.argmin(e15_1))
grid = np.round(np.geomspace(0.5, 40.0, 20), 3)
P2, Q2 = np.meshgrid(grid, grid, indexing="ij")
its2, e15_2, t2 = sweep(P2.ravel(), Q2.ravel())
best2 = int(np.argmin(e15_2))
fine = None
if FEM:  # the paper samples (4, 5) with step 0.001; a 0.01 grid on [3.5, 5.5] here
    psf = np.round(np.arange(3.5, 5.5001, 0.01), 3)
    itsf, e15_f, tf = sweep(psf, None)
    bf = int(np.argmin(e15_f))
    hf = HIST[len(HIST) - 1]
    fine = {"p": psf.tolist(), "iterations": itsf, "err_after_15": e15_f, "seconds": tf,
            "p_star_min_error_15": float(psf[bf]), "iterations_at_p_star": itsf[bf],
            "p_star_min_error_k": {k: argmin_at(psf, hf, k) for k in (4, 5, 6, 7, 8)},
            "histories": hf}
    print("fine p* by the error after k iterations:", fine["p_star_min_error_k"], file=sys.stderr)
    print(f"fine: {len(psf)} replicas in {tf:.1f} s, p* = {psf[bf]} (err15 {e15_f[bf]:.2e}, {itsf[bf]} its)",
          file=sys.stderr)
out = {
    "scheme": "split_fem, err_ov (the paper's max |u1 - u2| on the overlap)" if FEM else "imex_fd, err_if",
    "fig1_fine": fine,
    "setup": "Table 1 j=0 grid, overlap 3 h_v, random lambda^0 ~ U(-1,1), Gauss-Seidel, eps 1e-6",
    "fig1": {"p": ps1.tolist(), "iterations": its1, "err_if_after_15": e15_1, "seconds": t1,
             "p_star_min_error_k": {k: argmin_at(ps1, HIST[0], k) for k in (4, 5, 6, 7, 8)},
             "p_star_min_error_15": float(ps1[best1]), "iterations_at_p_star": its1[best1]},
    "fig2": {"p": P2.ravel().tolist(), "q": Q2.ravel().tolist(), "iterations": its2, "err_if_after_15": e15_2,
             "seconds": t2, "pq_star_min_error_15": [float(P2.ravel()[best2]), float(Q2.ravel()[best2])],
             "pq_star_min_error_k": {k: [float(P2.ravel()[int(np.argmin([h[k - 1] for h in HIST[1]]))]),
                                         float(Q2.ravel()[int(np.argmin([h[k - 1] for h in HIST[1]]))])]
                                     for k in (4, 5, 6, 7, 8)},
             "iterations_at_pq_star": its2[best2]},
}
print(json.dumps(out))
print(f"fig1: {len(ps1)} replicas in {t1:.1f} s, p* = {ps1[best1]} (err15 {e15_1[best1]:.2e}, {its1[best1]} its); "
      f"fig2: {P2.size} replicas in {t2:.1f} s, (p,q)* = ({P2.ravel()[best2]}, {Q2.ravel()[best2]}) "
      f"(err15 {e15_2[best2]:.2e}, {its2[best2]} its)", file=sys.stderr)

"""The paper's Table 1 experiment re-run with this library's discretisation on one B200.

Error equation (f = 0, u0 = 0) on x in [0,1) periodic, v in [-1,1] (Dirichlet 0 ends; the paper uses Neumann and
notes the end condition does not matter), T = 2, Delta t = h_x = h_v = 0.01 / 2^j (j = 0..4), two
subdomains split at v = 0 with overlap 3 h_v or none, random initial traces lambda^0 ~ U(-1, 1), the
paper's serial schedule SWR1-SWR4 (Gauss-Seidel), stop when the interface error drops below
eps = 1e-6 (our err_if: max over interface nodes and time of |u_s^k| -- the exact solution is 0) or after 150
iterations.  Robin parameters as in the paper: OSWR(p) p = 4.23, OSWR(p, q) p = 11, q = 2.5.

    python tools/table1.py [jmax] > profiles/r1_table1.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

EPS, KMAX = 1e-6, 150
PAPER = {  # Table 1 of the paper (its own FEM discretisation), for context only
    ("CSWR", 3): [70, 105, 132, ">150", ">150"], ("OSWR(p)", 3): [9, 12, 15, 17, 18], ("OSWR(p,q)", 3): [9, 10, 10, 10, 13],
    ("CSWR", 0): ["-"] * 5, ("OSWR(p)", 0): [12, 17, 20, 23, 26], ("OSWR(p,q)", 0): [11, 12, 13, 14, 16],
}
METHODS = [("CSWR", "dirichlet", 0.0, None), ("OSWR(p)", "robin", 4.23, None), ("OSWR(p,q)", "robin", 11.0, 2.5)]


def run_level(j, ov, name, kind, p, q):
    g = ki.Grid(100 * 2 ** j, 200 * 2 ** j, 200 * 2 ** j, 1.0, 2.0)
    prob = ki.zero_problem(g)
    rng = np.random.default_rng(1000 + j)
    lam = [rng.uniform(-1.0, 1.0, size=(g.nt, g.nx)) for _ in range(2)]
    hist = []
    t0 = time.perf_counter()
    with Problem(prob) as pb:
        pb.setup(kind, p if kind == "robin" else 0.0, ov, 2, KMAX, q=q)
        pb.set_schedule("gauss_seidel")
        pb.reset()
        pb.set_initial_trace(0, 0, lam[0])  # lambda_1^0 (toward Omega_1's right end)
        pb.set_initial_trace(0, 1, lam[1])  # unused by SWR1-SWR4 (lambda_2^k comes from u_1^k)
        it = None
        for k in range(1, KMAX + 1):
            pb.iterate(1)
            e = float(pb.history()[1][-1])
            hist.append(e)
            if e < EPS:
                it = k
                break
            if not np.isfinite(e) or (k >= 30 and e > 0.999 * hist[k - 30]):
                break  # no progress (CSWR without overlap)
    return dict(grid=[g.nx, g.nv, g.nt], iterations=it if it is not None else (f">{KMAX}" if len(hist) == KMAX else "-"),
                err_if=hist, seconds=time.perf_counter() - t0)


def main():
    jmax = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    out = {"eps": EPS, "kmax": KMAX, "schedule": "gauss_seidel (SWR1-SWR4)", "results": {}}
    for ov in (3, 0):
        for name, kind, p, q in METHODS:
            row = []
            for j in range(jmax + 1):
                r = run_level(j, ov, name, kind, p, q)
                row.append(r)
                print(f"ov={ov} {name:10s} j={j} iterations={r['iterations']} ({r['seconds']:.1f} s)", file=sys.stderr,
                      flush=True)
            out["results"][f"{name} ov={ov}"] = {"ours": [r["iterations"] for r in row],
                                                 "paper": PAPER[(name, ov)], "levels": row}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

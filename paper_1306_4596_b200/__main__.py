"""Run one workload through the library and log every Jacobi iteration as a JSON line (SURVEY §5 metrics):

    python -m paper_1306_4596_b200 --workload c0 [--K 20] [--p 1.0] [--kind robin]

First line: the configuration (grid, decomposition, launch plan); then {"k", "err_T", "err_if", "ms"} per
iteration (ms: device time of the iteration, CUDA events on the library's stream); last line: the summary
(updates/s over the iterations).  The workloads are the BASELINE.json configs (kfp_inputs.config)."""
from __future__ import annotations

import argparse
import json
import os
import sys


def main(argv=None):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import kfp_inputs as ki

    from .kfp import Problem

    ap = argparse.ArgumentParser(prog="python -m paper_1306_4596_b200")
    ap.add_argument("--workload", default="c0")
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--kind", default=None, choices=["robin", "dirichlet"])
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--q", type=float, default=None)
    ap.add_argument("--overlap", type=int, default=None)
    ap.add_argument("--n-sub", type=int, default=None)
    a = ap.parse_args(argv)
    run = ki.config(a.workload)
    kw = {k: v for k, v in (("K", a.K), ("kind", a.kind), ("p", a.p), ("q", a.q), ("overlap", a.overlap),
                            ("n_sub", a.n_sub)) if v is not None}
    run = run.with_(**kw)
    g = run.grid
    with Problem(ki.make_problem(run)) as pb:
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
        print(json.dumps({"workload": run.name, "nx": g.nx, "nv": g.nv, "nt": g.nt, "kind": run.kind, "p": run.p,
                          "q": run.q, "overlap": run.overlap, "n_sub": run.n_sub, "K": run.K, "plan": pb.plan()}),
              flush=True)
        pb.reset()
        total = 0.0
        for k in range(1, run.K + 1):
            pb.iterate(1)
            ms, _ = pb.last_timing()
            total += ms
            eT, eI = pb.history()
            print(json.dumps({"k": k, "err_T": float(eT[-1]), "err_if": float(eI[-1]), "ms": ms}), flush=True)
        print(json.dumps({"summary": True, "updates_per_s": g.nx * g.nv * g.nt * run.K / (total / 1e3),
                          "ms": total}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""GPU vs C oracle on small-x versions of tall-column configs: per-subdomain max error and where."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki, oracle  # noqa
from paper_1306_4596_b200 import Problem  # noqa

cases = {
    "c3_rows": ki.scaled(ki.config("c3"), nx=64, nt=20, K=2),
    "c3_rows_K1": ki.scaled(ki.config("c3"), nx=64, nt=20, K=1),
    "c3_rows_nt1": ki.scaled(ki.config("c3"), nx=64, nt=1, K=1),
    "c2_rows": ki.scaled(ki.config("c2"), nx=64, nt=20, K=2),
    "c4_rows": ki.scaled(ki.config("c4"), nx=64, nt=20, K=2),
}
for name in (sys.argv[1:] or cases):
    run = cases[name]
    prob = ki.make_problem(run)
    with Problem(prob) as pb:
        pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
        g = [pb.subdomain_uT(s) for s in range(run.n_sub)]
        eT, eI = pb.history()
        plan = pb.plan()
    r = oracle.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K)
    print(name, plan, "hist", np.abs(eT - r["err_T"]).max() / r["err_T"].max(), np.abs(eI - r["err_if"]).max() / r["err_if"].max())
    for s in range(run.n_sub):
        d = np.abs(g[s] - r["uT_sub"][s])
        rel = d.max() / np.abs(r["uT_sub"][s]).max()
        if rel > 1e-9:
            rows = np.where(d.max(axis=1) > 1e-9 * np.abs(r["uT_sub"][s]).max())[0]
            print(f"  sub {s}: rel {rel:.2e} bad rows {rows.min()}..{rows.max()} ({len(rows)}) of {g[s].shape[0]}")
    sys.stdout.flush()

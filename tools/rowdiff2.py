import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki, oracle  # noqa
from paper_1306_4596_b200 import Problem  # noqa
run = ki.scaled(ki.config("c3"), nx=64, nt=20, K=1)
if len(sys.argv) > 1 and sys.argv[1] == "s2":
    run = ki.scaled(ki.config("c3"), nx=64, nv=8192, nt=20, K=1).with_(n_sub=4)
prob = ki.make_problem(run)
with Problem(prob) as pb:
    pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
    g = [pb.subdomain_uT(s) for s in range(run.n_sub)]
    plan = pb.plan()
    UTg = pb.monodomain_uT()
r = oracle.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K)
print(plan, "monodomain rel", np.abs(UTg - r["UT"]).max() / np.abs(r["UT"]).max())
for s in (0, 1):
    d = np.abs(g[s] - r["uT_sub"][s]).max(axis=1)
    sc = np.abs(r["uT_sub"][s]).max()
    idx = np.argsort(d)[::-1][:8]
    print("sub", s, "top rows", sorted(idx.tolist()), "rel", (d[idx] / sc).round(6).tolist())
    print("  profile every 132 rows:", [f"{d[i]/sc:.1e}" for i in range(0, len(d), 132)])

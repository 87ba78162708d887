import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki, oracle  # noqa
from paper_1306_4596_b200 import Problem  # noqa
c3 = ki.config("c3")
base = ki.scaled(c3, nx=64, nt=20, K=1)
V = {
    "c3_K1": base,
    "c3_p4": base.with_(p=4.0),
    "c3_dir_ov4": base.with_(kind="dirichlet", p=0.0, overlap=4),
    "c3_smalla": ki.scaled(c3, nx=64, nt=20, K=1, t_final=0.02 * 20 / 1000 / 6.4),   # a ~ 13
    "c2_biga": ki.scaled(ki.config("c2"), nx=64, nt=20, K=1, t_final=20 * 84 * (8 / 4096) ** 2),  # a = 84, n = 2048
    "S2_n2049": ki.scaled(c3, nx=64, nv=4096, nt=20, K=1).with_(n_sub=2),
    "S4_n2049": ki.scaled(c3, nx=64, nv=8192, nt=20, K=1).with_(n_sub=4),
    "S8_nv4096": ki.scaled(c3, nx=64, nv=4096, nt=20, K=1),   # n = 513
}
for name in (sys.argv[1:] or V):
    run = V[name]
    prob = ki.make_problem(run)
    g = run.grid
    a = (g.t_final / g.nt) / (2 * g.vmax / g.nv) ** 2
    with Problem(prob) as pb:
        pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
        sl = [pb.subdomain_uT(s) for s in range(run.n_sub)]
        plan = pb.plan()
    r = oracle.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K)
    rel = max(np.abs(x - y).max() / np.abs(y).max() for x, y in zip(sl, r["uT_sub"]))
    print(f"{name:12s} a={a:7.2f} n_sub={run.n_sub} kind={run.kind} p={run.p} rel={rel:.2e}  {plan}", flush=True)

import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kfp_inputs as ki, oracle  # noqa
from paper_1306_4596_b200 import Problem  # noqa
for nv, nsub, kind, ov in [(520, 2, "robin", 0), (520, 2, "dirichlet", 4), (512, 2, "robin", 0), (1040, 4, "robin", 0)]:
    for nt in (1, 2):
        run = ki.scaled(ki.config("c0"), nx=32, nv=nv, nt=nt, K=1, t_final=0.0025 * nt).with_(
            n_sub=nsub, kind=kind, overlap=ov, p=1.0 if kind == "robin" else 0.0)
        prob = ki.make_problem(run)
        with Problem(prob) as pb:
            pb.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, copy=False)
            sl = [pb.subdomain_uT(s) for s in range(run.n_sub)]
            plan = pb.plan()
        r = oracle.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K)
        out = []
        for s in range(nsub):
            d = np.abs(sl[s] - r["uT_sub"][s])
            sc = np.abs(r["uT_sub"][s]).max()
            bad = np.where(d.max(axis=1) > 1e-12 * sc)[0]
            out.append(f"s{s}: {d.max()/sc:.1e} rows {bad[:6].tolist()}..{bad[-3:].tolist() if len(bad) else []}")
        print(nv, nsub, kind, "nt", nt, plan, "|", " ; ".join(out), flush=True)

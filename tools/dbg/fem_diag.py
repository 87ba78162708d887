"""FEM monodomain GPU vs oracle diagnostics (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import kfp_inputs as ki
import oracle
from paper_1306_4596_b200 import kfp

for nx, nv, nt, seed, u0x_const in [(64, 200, 1, 1, False), (64, 200, 2, 1, False), (64, 200, 3, 1, False),
                                    (64, 200, 2, 1, True), (64, 40, 1, 1, False), (64, 40, 2, 1, True)]:
    g = ki.Grid(nx, nv, nt, 1.0, 0.01 * nt)
    prob = ki.fem_problem(g, seed)
    if u0x_const:
        prob.u0x = np.ones_like(prob.u0x)
    UT, _ = oracle.monodomain(prob)
    with kfp.Problem(prob) as pb:
        G = pb.monodomain()
        plan = pb.plan() if hasattr(pb, 'plan') else ''
    d = np.abs(G - UT)
    j, m = np.unravel_index(d.argmax(), d.shape)
    rowerr = d.max(axis=1)
    print(f"nx={nx} nv={nv} nt={nt} xconst={u0x_const}: rel={d.max()/np.abs(UT).max():.3e} at (j={j}, m={m}); "
          f"rows with err>1e-12: {np.nonzero(rowerr > 1e-12 * np.abs(UT).max())[0][:12]} ; "
          f"cols: {np.nonzero(d.max(axis=0) > 1e-12 * np.abs(UT).max())[0][:12]}", flush=True)

python - <<'P'
import time, torch, kfp_inputs as ki
from paper_1306_4596_b200 import Problem
for w in ["c3", "c4", "c4w2", "c4w8"]:
    run = ki.config(w) if not w.startswith("c4w") else ki.weak_scaling_config(int(w[3:]))
    g = run.grid
    with Problem(ki.make_problem(run)) as pb:
        torch.cuda.synchronize(); t = time.perf_counter()
        pb.monodomain(copy=False)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(w, g.nx, g.nv, g.nt, f"{dt*1e3:.1f} ms", f"{g.nx*g.nv*g.nt/dt/1e9:.1f} G upd/s", flush=True)
P

"""Pipelined vs unpipelined Jacobi SWR throughput on one B200 (kfp_swr_set_pipeline).

    python tools/pipeline_speed.py > profiles/r1_pipeline_speed.json

For each workload: one warm-up solve, then the K iterations timed with CUDA events on the library's stream
(the monodomain reference is built at setup and not timed), depth 1 (one launch per step and iteration)
against depth D (one sweep of nt + D - 1 launches per D iterations)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kfp_inputs as ki  # noqa: E402
from paper_1306_4596_b200 import Problem  # noqa: E402

RUNS = [
    ki.config("c0"), ki.config("c1"),
    ki.Run("paper_j0_jacobi", ki.paper_grid(0), "random_u0", "robin", 11.0, 3, 2, 20, q=2.5, scheme="split_fem"),
    ki.Run("paper_j2_jacobi", ki.paper_grid(2), "random_u0", "robin", 11.0, 3, 2, 20, q=2.5, scheme="split_fem"),
    ki.config("c2").with_(K=10),
]


def timed(run, depth):
    stream = torch.cuda.Stream()  # a real stream shared with the library (not the legacy default)
    torch.cuda.set_stream(stream)
    with Problem(ki.make_problem(run)) as pb:
        pb.set_stream(stream.cuda_stream)
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
        if depth > 1:
            pb.set_pipeline(depth)
        best = None
        for rep in range(3):
            pb.reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            pb.iterate(run.K)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if rep > 0:
                best = ms if best is None else min(best, ms)
        hist = pb.history()[1]
    return best, float(hist[-1])


def main():
    out = []
    for run in RUNS:
        g = run.grid
        t1, e1 = timed(run, 1)
        D = run.K
        tD, eD = timed(run, D)
        ups = g.nx * g.nv * g.nt * run.K
        row = dict(workload=run.name, grid=[g.nx, g.nv, g.nt], K=run.K, scheme=run.scheme, depth=D,
                   ms_unpipelined=t1, ms_pipelined=tD, speedup=t1 / tD, gups_unpipelined=ups / t1 / 1e6,
                   gups_pipelined=ups / tD / 1e6, same_err_if=e1 == eD)
        out.append(row)
        print(f"{run.name:16s} depth {D:3d}: {t1:9.2f} ms -> {tD:9.2f} ms  ({t1 / tD:5.2f}x; "
              f"{ups / t1 / 1e6:7.1f} -> {ups / tD / 1e6:7.1f} G upd/s)", file=sys.stderr, flush=True)
    print(json.dumps({"runs": out}))


if __name__ == "__main__":
    main()

"""One process per GPU: the Jacobi SWR iteration over contiguous blocks of v-subdomains.

Rank r of a world of g solves subdomains [r*S/g, (r+1)*S/g).
Within an iteration the subdomains are independent (the parallel schedule of
the Remark at PAPER.md:594-597); the only data-path exchange is the
whole-window interface traces of the two block edges, sent to the neighbour
ranks after every iteration with NCCL point-to-point send/recv
(torch.distributed, NVLink/NVSwitch on one box), and the per-iteration error
history reduced with one all_reduce(MAX) at the end.

The local solver is pluggable so that this host logic is testable on CPU:
``CudaBlock`` wraps the C-ABI (``kfp_swr_bind_edge_buffers`` points the
library's edge traces at torch tensors that NCCL sends/receives in place);
tests/test_dist_gloo.py drives the same ``run_swr`` with an oracle-backed
block over the gloo backend.
"""
from __future__ import annotations

import os
import time
from typing import Optional

import torch
import torch.distributed as dist


def block_of(rank: int, world: int, n_sub: int):
    """Contiguous subdomain block [s_begin, s_end) of `rank` (n_sub % world == 0)."""
    if n_sub % world != 0:
        raise ValueError(f"n_sub={n_sub} must be a multiple of the world size {world}")
    per = n_sub // world
    return rank * per, (rank + 1) * per


class CudaBlock:
    """The local block on this rank's GPU, through the C-ABI (libkfp.so)."""

    def __init__(self, prob, kind: str, p: float, overlap: int, n_sub: int, K: int, rank: int, world: int,
                 device: int, q=None):
        from .kfp import Problem

        self.s_begin, self.s_end = block_of(rank, world, n_sub)
        self.n_sub = n_sub
        g = prob.grid
        torch.cuda.set_device(device)
        self.stream = torch.cuda.current_stream()
        self.pb = Problem(prob, device=device)
        self.pb.set_stream(self.stream.cuda_stream)
        self.pb.setup(kind, p, overlap, n_sub, K, self.s_begin, self.s_end, q=q)
        shape = (g.nt, g.nx)
        mk = lambda: torch.zeros(shape, dtype=torch.float64, device=f"cuda:{device}")
        self.has_left, self.has_right = self.s_begin > 0, self.s_end < n_sub
        self.send_left = [mk() for _ in range(2)] if self.has_left else None
        self.recv_left = [mk() for _ in range(2)] if self.has_left else None
        self.send_right = [mk() for _ in range(2)] if self.has_right else None
        self.recv_right = [mk() for _ in range(2)] if self.has_right else None
        for par in (0, 1):
            ptr = lambda lst: lst[par].data_ptr() if lst is not None else None
            self.pb.bind_edge_buffers(par, ptr(self.send_left), ptr(self.recv_left), ptr(self.send_right),
                                      ptr(self.recv_right))

    def reset(self):
        self.pb.reset()

    def iterate(self):
        self.pb.iterate(1)

    def history(self):
        eT, eI = self.pb.history()
        return torch.tensor(eT, dtype=torch.float64), torch.tensor(eI, dtype=torch.float64)

    def subdomain_uT(self, s: int):
        return self.pb.subdomain_uT(s)

    def close(self):
        self.pb.close()


def exchange(block, rank: int, world: int, parity: int):
    """Send this block's outgoing edge traces of `parity` to the neighbour ranks and receive theirs."""
    ops = []
    if block.has_left:
        ops.append(dist.P2POp(dist.isend, block.send_left[parity], rank - 1))
        ops.append(dist.P2POp(dist.irecv, block.recv_left[parity], rank - 1))
    if block.has_right:
        ops.append(dist.P2POp(dist.isend, block.send_right[parity], rank + 1))
        ops.append(dist.P2POp(dist.irecv, block.recv_right[parity], rank + 1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def run_swr(block, K: int, rank: int, world: int):
    """K Jacobi iterations with the edge exchange after each; returns the global (err_T, err_if)."""
    for k in range(1, K + 1):
        block.iterate()  # reads recv_*[(k-1)&1], writes send_*[k&1]
        exchange(block, rank, world, k & 1)
    eT, eI = block.history()
    hist = torch.stack([eT, eI])
    if world > 1:
        dev = block.send_left[0].device if block.has_left else (block.send_right[0].device if block.has_right else "cpu")
        h = hist.to(dev)
        dist.all_reduce(h, op=dist.ReduceOp.MAX)  # errors are maxima over subdomains
        hist = h.cpu()
    return hist[0].numpy(), hist[1].numpy()


def bench_main(args, default_workload):
    """bench.py --gpus N under torchrun: the weak-scaling c4 family, one block of S/N subdomains per rank."""
    import json

    import numpy as np

    import kfp_inputs as ki

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    run = ki.config(args.workload or default_workload(world))
    g = run.grid
    prob = ki.make_problem(run)
    blk = CudaBlock(prob, run.kind, run.p, run.overlap, run.n_sub, run.K * (args.steps + args.warmup) + 1, rank,
                    world, local)
    stream = torch.cuda.current_stream()

    def one():
        blk.reset()
        run_swr(blk, run.K, rank, world)

    for _ in range(args.warmup):
        one()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = blk.pb.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # slowest rank
    launches = torch.tensor([blk.pb.launch_count() - l0], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    ms = float(ms.item())
    if rank == 0:
        value = run.updates * args.steps / (ms / 1e3)
        line = {
            "metric": "grid-point updates/s (N_x*N_v*N_t*K / wall)", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": run.name, "nx": g.nx, "nv": g.nv, "nt": g.nt, "K": run.K, "n_sub": run.n_sub,
                       "kind": run.kind, "overlap": run.overlap, "parallelism": f"v-subdomain blocks x{world}, NCCL P2P",
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches.item()),
        }
        print(json.dumps(line), flush=True)
    blk.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0

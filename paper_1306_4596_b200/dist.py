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
                 device: int, q=None, stream=None):
        from .kfp import Problem

        self.s_begin, self.s_end = block_of(rank, world, n_sub)
        self.n_sub = n_sub
        g = prob.grid
        torch.cuda.set_device(device)
        # a real stream made current: the library's launches, torch's NCCL exchange (which orders itself
        # after the current stream) and the timing events all sit on it (the legacy default stream, handle 0,
        # would leave the library on its own non-blocking stream, unordered with the exchange)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        torch.cuda.set_stream(self.stream)
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


def run_swr(block, K: int, rank: int, world: int, on_iterate=None):
    """K Jacobi iterations with the edge exchange after each; returns the global (err_T, err_if).
    on_iterate(block) runs after each iteration's launches (e.g. to read the library's window timing)."""
    for k in range(1, K + 1):
        block.iterate()  # reads recv_*[(k-1)&1], writes send_*[k&1]
        if on_iterate:
            on_iterate(block)
        exchange(block, rank, world, k & 1)
    eT, eI = block.history()
    hist = torch.stack([eT, eI])
    if world > 1:
        dev = block.send_left[0].device if block.has_left else (block.send_right[0].device if block.has_right else "cpu")
        h = hist.to(dev)
        dist.all_reduce(h, op=dist.ReduceOp.MAX)  # errors are maxima over subdomains
        hist = h.cpu()
    return hist[0].numpy(), hist[1].numpy()


def bench_main(args, default_workload, clock_sampler=None, peaks=None):
    """bench.py --gpus N under torchrun: the weak-scaling c4 family, one block of S/N subdomains per rank.
    Prints (rank 0) the bench JSON line: device-timed value (max over ranks), the roofline of the step kernel
    (algorithmic bytes per launch / average launch time, max over ranks), clocks sampled during the timed
    region, and the end-to-end number through the public API (create from host tables, setup incl. the
    monodomain reference, K iterations with the NCCL exchange, u(T) of the local subdomains back to the host)."""
    import json

    import numpy as np

    import kfp_inputs as ki

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # rank 0's stdout carries exactly one JSON line (bench.py points file descriptor 1 at stderr for native
    # output such as NCCL's banner and prints the line through a duplicate of the original stdout)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    run = ki.config(args.workload or default_workload(world))
    g = run.grid
    prob = ki.make_problem(run)
    blk = CudaBlock(prob, run.kind, run.p, run.overlap, run.n_sub, run.K, rank, world, local)
    stream = blk.stream  # current (CudaBlock made it so)

    kernel_ms = [0.0]

    def tally(b):  # the step launches of the iteration just run (library events on the same stream)
        kernel_ms[0] += b.pb.last_timing()[1]

    def one(b, timed=False):
        b.reset()
        return run_swr(b, run.K, rank, world, tally if timed else None)

    # W untimed warm-up solves, then more until >= 5 s of warm-up (as bench.py); every rank runs the same
    # count (the ranks exchange traces), agreed by a MAX all-reduce
    t_w = time.perf_counter()
    for _ in range(args.warmup):
        one(blk)
    torch.cuda.synchronize()
    per = (time.perf_counter() - t_w) / max(1, args.warmup)
    extra = torch.tensor([min(200, max(0, int((5.0 - (time.perf_counter() - t_w)) / max(per, 1e-3)) + 1))],
                         device=dev, dtype=torch.int64)
    dist.all_reduce(extra, op=dist.ReduceOp.MAX)
    for _ in range(int(extra.item())):
        one(blk)
    warm = args.warmup + int(extra.item())
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_sampler(local) if clock_sampler else None
    if clocks:
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = blk.pb.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        one(blk, timed=True)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # slowest rank
    n_launch = blk.pb.launch_count() - l0
    launches = torch.tensor([n_launch], device=dev, dtype=torch.float64)
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    # roofline of the step kernel on this rank: algorithmic bytes (16 B per unknown-row update) per launch
    rows = sum(blk.pb.subdomain_range(s)[1] - blk.pb.subdomain_range(s)[0] + 1 for s in range(blk.s_begin, blk.s_end))
    ends = 2 * (blk.s_end - blk.s_begin)  # end nodes that are not unknowns (Dirichlet / physical); Robin: upper bound
    bytes_per_launch = 16.0 * g.nx * (rows - ends)
    step_launches = g.nt * run.K * args.steps
    per_launch = torch.tensor([kernel_ms[0] / 1e3 / step_launches], device=dev)
    dist.all_reduce(per_launch, op=dist.ReduceOp.MAX)
    plan = blk.pb.plan()
    ranges = [blk.pb.subdomain_range(s) for s in range(blk.s_begin, blk.s_end)]  # for the e2e output buffers
    blk.close()

    # end to end through the public API (host tables in, u(T) out), max over ranks
    dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # input tables and results in pinned host memory (allocated outside the timed region), same stream
    import dataclasses

    pins = {k: torch.empty(np.shape(getattr(prob, k)), dtype=torch.float64, pin_memory=True)
            for k in ("ft", "fv", "fx", "u0v", "u0x")}
    for k, t in pins.items():
        t.numpy()[...] = getattr(prob, k)
    prob_pinned = dataclasses.replace(prob, **{k: t.numpy() for k, t in pins.items()})
    outs = [torch.empty((hi - lo + 1, g.nx), dtype=torch.float64, pin_memory=True) for lo, hi in ranges]
    f0.record(stream)
    b2 = CudaBlock(prob_pinned, run.kind, run.p, run.overlap, run.n_sub, run.K, rank, world, local, stream=stream)
    hist = one(b2)
    uT = [b2.pb.subdomain_uT(s, out=o.numpy()) for s, o in zip(range(b2.s_begin, b2.s_end), outs)]
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    d2h = sum(a.nbytes for a in uT) + hist[0].nbytes + hist[1].nbytes
    h2d = prob.table_bytes()
    b2.close()
    ms = float(ms.item())
    if rank == 0:
        value = run.updates * args.steps / (ms / 1e3)
        achieved = bytes_per_launch / float(per_launch.item()) / 1e9
        peak, peak_kind = peaks() if peaks else (None, None)
        line = {
            "metric": "grid-point updates/s (N_x*N_v*N_t*K / wall)", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": warm, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": run.name, "nx": g.nx, "nv": g.nv, "nt": g.nt, "K": run.K, "n_sub": run.n_sub,
                       "kind": run.kind, "overlap": run.overlap, "plan": plan,
                       "parallelism": f"v-subdomain blocks x{world}, NCCL P2P",
                       "l2": "inputs larger than L2", "updates_per_step": run.updates},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "kfp::step_fused_tma (rank 0 geometry, slowest rank's launch time)",
                         "bytes_per_launch": bytes_per_launch, "avg_launch_us": float(per_launch.item()) * 1e6},
            "e2e": {"value": run.updates / (float(e2e_ms.item()) / 1e3), "unit": "updates/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches.item()),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0

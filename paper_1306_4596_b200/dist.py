"""One process per GPU: the Jacobi SWR iteration over contiguous blocks of v-subdomains.

Rank r of a world of g solves subdomains [r*S/g, (r+1)*S/g).
Within an iteration the subdomains are independent (the parallel schedule of
the Remark at PAPER.md:594-597); the only data-path exchange is the
interface traces of the two block edges, sent to the neighbour ranks with NCCL
point-to-point send/recv (torch.distributed, NVLink/NVSwitch on one box), and
the per-iteration error history reduced with one all_reduce(MAX) at the end.

Overlap (``chunks > 1``): step n of iteration k+1 needs only trace row n of
iteration k, so the window is cut into time chunks; chunk c's edge
rows go out on a communication stream as soon as the library has written them
(kfp_swr_chunk_send_wait), and chunk c of the next iteration waits only for
chunk c's incoming rows (kfp_swr_chunk_recv_done).  The exchange of the last
chunk overlaps the next iteration's first chunks; the host never waits.

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


def decompose(nv: int, n_sub: int, overlap: int):
    """Subdomain node ranges [lo_s, hi_s] (R9: split nodes s nv / S, the overlap placed with
    floor(ov/2) nodes below and ceil(ov/2) above each split) -- the same ranges kfp_swr_setup uses."""
    c = [s * (nv // n_sub) for s in range(n_sub + 1)]
    lo = [0 if s == 0 else c[s] - overlap // 2 for s in range(n_sub)]
    hi = [nv if s == n_sub - 1 else c[s + 1] + (overlap + 1) // 2 for s in range(n_sub)]
    return lo, hi


def column_range(rank: int, world: int, nx: int):
    """This rank's x-columns of the sharded monodomain reference: a contiguous run of whole 32-column tiles."""
    ntiles = (nx + 31) // 32
    t0, t1 = rank * ntiles // world, (rank + 1) * ntiles // world
    return t0 * 32, min(nx, t1 * 32)


def sharded_monodomain(pb, grid, n_sub: int, overlap: int, rank: int, world: int, device):
    """The monodomain reference computed ONCE by the whole job: rank r solves the columns
    column_range(r) with a one-column halo exchanged with its x-neighbours after every step (NCCL P2P), then
    every rank receives, from every other, the columns it lacks of the U(T) rows of its own subdomains and of
    its interface lines (one all-to-all of point-to-point pairs).  Afterwards kfp_swr_setup finds the reference in place."""
    nx, nv, nt = grid.nx, grid.nv, grid.nt
    lo, hi = decompose(nv, n_sub, overlap)
    lines = sorted({lo[s] for s in range(1, n_sub)} | {hi[s] for s in range(n_sub - 1)})
    x0, x1 = column_range(rank, world, nx)
    rows = nv + 1
    halo = [torch.empty(rows, dtype=torch.float64, device=device) for _ in range(4)]
    pb.mono_shard_begin(x0, x1, lines, halo)
    left, right = (rank - 1) % world, (rank + 1) % world
    for _ in range(nt):
        pb.mono_shard_step()
        # column x1-1 to the right neighbour, column x0 to the left one; their edge columns back.  Sends
        # and receives in this order so that with two ranks (left == right) each receive pairs with the
        # matching send of the peer.
        ops = [dist.P2POp(dist.isend, halo[1], right), dist.P2POp(dist.isend, halo[0], left),
               dist.P2POp(dist.irecv, halo[2], left), dist.P2POp(dist.irecv, halo[3], right)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    pb.mono_shard_end()
    # what each rank needs: the U(T) node rows of its subdomains, the U-line rows of its interface lines
    need = []
    for r in range(world):
        sb, se = block_of(r, world, n_sub)
        ranges = [(0, lo[sb], hi[se - 1] + 1)]
        for s in range(sb, se):
            for node in ([lo[s]] if s > 0 else []) + ([hi[s]] if s < n_sub - 1 else []):
                li = lines.index(node)
                ranges.append((1, li * nt, (li + 1) * nt))
        need.append(ranges)
    cols = [column_range(r, world, nx) for r in range(world)]
    nrows = lambda rg: sum(b - a for _, a, b in rg)
    send = [torch.empty((nrows(need[r]), x1 - x0), dtype=torch.float64, device=device) for r in range(world)]
    for r in range(world):
        if r == rank:
            continue
        off = 0
        for what, a, b in need[r]:
            pb.mono_shard_copy(what, 0, a, b, x0, x1, send[r][off:off + b - a])
            off += b - a
    recv = [torch.empty((nrows(need[rank]), cols[r][1] - cols[r][0]), dtype=torch.float64, device=device)
            for r in range(world)]
    ops = []  # the all-to-all as point-to-point pairs (NCCL and gloo alike)
    for r in range(world):
        if r != rank:
            ops.append(dist.P2POp(dist.isend, send[r], r))
            ops.append(dist.P2POp(dist.irecv, recv[r], r))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r in range(world):
        if r == rank:
            continue
        off = 0
        for what, a, b in need[rank]:
            pb.mono_shard_copy(what, 1, a, b, cols[r][0], cols[r][1], recv[r][off:off + b - a])
            off += b - a
    return lines


class CudaBlock:
    """The local block on this rank's GPU, through the C-ABI (libkfp.so)."""

    def __init__(self, prob, kind: str, p: float, overlap: int, n_sub: int, K: int, rank: int, world: int,
                 device: int, q=None, stream=None, shard_reference: bool = True):
        from .kfp import Problem

        self.s_begin, self.s_end = block_of(rank, world, n_sub)
        self.n_sub = n_sub
        g = prob.grid
        torch.cuda.set_device(device)
        # a real stream made current: the library's launches, torch's NCCL exchange (which orders itself
        # after the current stream) and the timing events all sit on it (the legacy default stream, handle 0,
        # would leave the library on its own non-blocking stream, unordered with the exchange)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        self.comm = torch.cuda.Stream(device=device)  # the chunked exchange (NCCL orders itself after it)
        torch.cuda.set_stream(self.stream)
        self.pb = Problem(prob, device=device)
        self.pb.set_stream(self.stream.cuda_stream)
        if shard_reference and world > 1 and getattr(prob, "scheme", "imex_fd") == "imex_fd":
            sharded_monodomain(self.pb, g, n_sub, overlap, rank, world, f"cuda:{device}")
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

    def iterate_chunk(self, c: int, nchunks: int):
        self.pb.iterate_chunk(c, nchunks)

    def comm_begin(self, c: int):
        """Enter the communication stream once chunk c's outgoing rows are written (returns a context)."""
        ctx = torch.cuda.stream(self.comm)
        ctx.__enter__()
        self.pb.chunk_send_wait(self.comm.cuda_stream, c)
        return ctx

    def comm_end(self, c: int, ctx):
        self.pb.chunk_recv_done(self.comm.cuda_stream, c)
        ctx.__exit__(None, None, None)

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


def exchange_chunk(block, rank: int, world: int, parity: int, c: int, nchunks: int, nt: int):
    """Send rows [c nt / C, (c+1) nt / C) of this block's outgoing edge traces of `parity` to the neighbour
    ranks and receive theirs (on the block's communication stream when it has one; the requests make that
    stream, not the host, wait)."""
    n0, n1 = c * nt // nchunks, (c + 1) * nt // nchunks
    ctx = block.comm_begin(c) if hasattr(block, "comm_begin") else None
    ops = []
    if block.has_left:
        ops.append(dist.P2POp(dist.isend, block.send_left[parity][n0:n1], rank - 1))
        ops.append(dist.P2POp(dist.irecv, block.recv_left[parity][n0:n1], rank - 1))
    if block.has_right:
        ops.append(dist.P2POp(dist.isend, block.send_right[parity][n0:n1], rank + 1))
        ops.append(dist.P2POp(dist.irecv, block.recv_right[parity][n0:n1], rank + 1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if ctx is not None:
        block.comm_end(c, ctx)


def run_swr(block, K: int, rank: int, world: int, chunks: int = 1, nt: int = 0):
    """K Jacobi iterations; returns the global (err_T, err_if).  chunks == 1: whole-window exchange after each
    iteration.  chunks > 1: the time-chunked protocol (module docstring); nt = steps per window."""
    for k in range(1, K + 1):
        if chunks <= 1:
            block.iterate()  # reads recv_*[(k-1)&1], writes send_*[k&1]
            exchange(block, rank, world, k & 1)
        else:
            for c in range(chunks):
                block.iterate_chunk(c, chunks)  # waits (on the device) for chunk c of recv_*[(k-1)&1]
                exchange_chunk(block, rank, world, k & 1, c, chunks, nt)
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

    chunks = max(1, min(int(getattr(args, "chunks", 4) or 1), g.nt))

    def one(b):
        b.reset()
        return run_swr(b, run.K, rank, world, chunks=chunks, nt=g.nt)

    # exactly W untimed warm-up solves
    for _ in range(args.warmup):
        one(blk)
    warm = args.warmup
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_sampler(local) if clock_sampler else None
    if clocks:
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = blk.pb.launch_count()
    e0.record(stream)
    step_ev = []
    for _ in range(args.steps):  # no host synchronisation inside the timed region
        one(blk)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        step_ev.append(ev)
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
    # average step-launch time: the timed region over its step launches (an upper bound: the region also
    # holds the exchange waits and the error reductions; conservative for the roofline fraction)
    per_launch = torch.tensor([float(ms.item()) / 1e3 / step_launches], device=dev)
    dist.all_reduce(per_launch, op=dist.ReduceOp.MAX)
    sms = []
    prev = e0
    for ev in step_ev:
        sms.append(prev.elapsed_time(ev))
        prev = ev
    med = torch.tensor([float(np.median(sms))], device=dev)
    dist.all_reduce(med, op=dist.ReduceOp.MAX)
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
            "ms_per_step_median": float(med.item()),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": run.name, "nx": g.nx, "nv": g.nv, "nt": g.nt, "K": run.K, "n_sub": run.n_sub,
                       "kind": run.kind, "overlap": run.overlap, "plan": plan,
                       "parallelism": f"v-subdomain blocks x{world}, NCCL P2P in {chunks} time chunks "
                                      "overlapped with compute",
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

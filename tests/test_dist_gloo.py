"""-m "not gpu": the multi-rank host logic (paper_1306_4596_b200/dist.py) on CPU with gloo, world_size 2.

The distributed driver (block partition, edge-trace exchange by point-to-point
send/recv after every Jacobi iteration, MAX all-reduce of the error history)
is run with an oracle-backed local block: each rank owns half of the
subdomains.  Because the exchange only moves bytes, the result must be
bitwise identical to the single-process oracle SWR.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import kfp_inputs as ki

RUNS = {
    "robin4": ki.scaled(ki.config("c3"), nx=16, nv=64, nt=30, K=5).with_(n_sub=4),
    "dirichlet4": ki.scaled(ki.config("c4"), nx=16, nv=64, nt=30, K=5).with_(n_sub=4, overlap=4),
    # two-sided OSWR(p, q): the traces that cross the rank boundary carry q one way and p the other
    "robin_pq4": ki.scaled(ki.config("c3"), nx=16, nv=64, nt=30, K=5).with_(n_sub=4, p=3.0, q=0.8),
    # the paper's split-FEM scheme: the driver moves the same trace bytes
    "fem_robin_pq4": ki.Run("fem_pq4", ki.Grid(16, 64, 30, 1.0, 0.3), "random_u0", "robin", 4.23, 2, 4, 5, q=2.5,
                            scheme="split_fem"),
}


class OracleBlock:
    """The dist.py local-block interface backed by the CPU oracle (tests only)."""

    def __init__(self, prob, run, rank, world):
        import oracle
        from paper_1306_4596_b200.dist import block_of

        self.orc = oracle
        self.prob, self.run = prob, run
        g = run.grid
        self.s_begin, self.s_end = block_of(rank, world, run.n_sub)
        self.lo, self.hi = oracle.subdomains(g.nv, run.n_sub, run.overlap)
        S = run.n_sub
        lines = sorted({int(self.lo[s]) for s in range(1, S)} | {int(self.hi[s]) for s in range(S - 1)})
        self.UT, rec = oracle.monodomain(prob, lines)
        self.Uline = {j: rec[i] for i, j in enumerate(lines)}
        shape = (g.nt, g.nx)
        self.has_left, self.has_right = self.s_begin > 0, self.s_end < S
        z = lambda: [torch.zeros(shape, dtype=torch.float64) for _ in range(2)]
        self.send_left, self.recv_left = (z(), z()) if self.has_left else (None, None)
        self.send_right, self.recv_right = (z(), z()) if self.has_right else (None, None)
        # local interfaces: toL[i] (sent by i+1 to i), toR[i] (sent by i to i+1), by parity
        self.toL = {i: z() for i in range(self.s_begin, self.s_end - 1)}
        self.toR = {i: z() for i in range(self.s_begin, self.s_end - 1)}
        self.k = 0
        self.eT, self.eI = [], []
        self.uT = {}

    def reset(self):
        pass

    def iterate(self):
        o, run = self.orc, self.run
        self.k += 1
        pin, pout = (self.k - 1) & 1, self.k & 1
        S = run.n_sub
        et = o.END_ROBIN if run.kind == "robin" else o.END_DIRICHLET
        eT = eI = 0.0
        for s in range(self.s_begin, self.s_end):
            lo, hi = int(self.lo[s]), int(self.hi[s])
            if s == 0:
                gL = None
            elif s == self.s_begin:
                gL = self.recv_left[pin].numpy()
            else:
                gL = self.toR[s - 1][pin].numpy()
            if s == S - 1:
                gR = None
            elif s == self.s_end - 1:
                gR = self.recv_right[pin].numpy()
            else:
                gR = self.toL[s][pin].numpy()
            rec = [n for n in ((lo,) if s > 0 else ()) + ((hi,) if s < S - 1 else ())]
            uT, sL, sR, r = o.window(self.prob, lo, hi, o.END_PHYS if s == 0 else et, o.END_PHYS if s == S - 1 else et,
                                     run.p, gL, gR, run.kind, int(self.hi[s - 1]) if s > 0 else -1,
                                     int(self.lo[s + 1]) if s < S - 1 else -1, rec_nodes=rec, q=run.q)
            if s > 0:
                dst = self.send_left[pout] if s == self.s_begin else self.toL[s - 1][pout]
                dst.copy_(torch.from_numpy(sL))
            if s < S - 1:
                dst = self.send_right[pout] if s == self.s_end - 1 else self.toR[s][pout]
                dst.copy_(torch.from_numpy(sR))
            for i, node in enumerate(rec):
                eI = max(eI, float(np.abs(r[i] - self.Uline[node]).max()))
            eT = max(eT, float(np.abs(uT - self.UT[lo:hi + 1]).max()))
            self.uT[s] = uT
        self.eT.append(eT)
        self.eI.append(eI)

    def iterate_chunk(self, c, nchunks):
        """The time-chunked protocol (dist.exchange_chunk): the oracle solves the whole window with the first
        chunk (every incoming row of the previous iteration has arrived by then); the exchange still moves
        one chunk of rows at a time."""
        if c == 0:
            self.iterate()

    def history(self):
        return torch.tensor(self.eT, dtype=torch.float64), torch.tensor(self.eI, dtype=torch.float64)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out, chunks=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1306_4596_b200.dist import run_swr

    run = RUNS[name]
    blk = OracleBlock(ki.make_problem(run), run, rank, world)
    eT, eI = run_swr(blk, run.K, rank, world, chunks=chunks, nt=run.grid.nt)
    out[rank] = (eT, eI, {s: blk.uT[s] for s in blk.uT})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", list(RUNS))
def test_two_rank_gloo_matches_single_process(orc, name):
    run = RUNS[name]
    ref = orc.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    for rank in (0, 1):
        eT, eI, slabs = out[rank]
        assert np.array_equal(eT, ref["err_T"]) and np.array_equal(eI, ref["err_if"])  # MAX all-reduce is exact
        for s, a in slabs.items():
            assert np.array_equal(a, ref["uT_sub"][s]), (rank, s)
    # both ranks together hold every subdomain
    assert sorted(list(out[0][2]) + list(out[1][2])) == list(range(run.n_sub))


@pytest.mark.parametrize("name,world,chunks", [("robin4", 2, 4), ("dirichlet4", 2, 4), ("fem_robin_pq4", 2, 3),
                                               ("robin_pq4", 4, 1), ("dirichlet4", 4, 3)])
def test_chunked_exchange_matches_single_process(orc, name, world, chunks):
    """The overlapped, time-chunked exchange protocol (dist.exchange_chunk; chunks of 30 // C rows, a ragged
    last chunk for C = 4) and world size 4 (one subdomain per rank: both edges cross ranks): bitwise the
    single-process oracle, like the whole-window exchange."""
    run = RUNS[name]
    ref = orc.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, out, chunks), nprocs=world, join=True)
    held = []
    for rank in range(world):
        eT, eI, slabs = out[rank]
        assert np.array_equal(eT, ref["err_T"]) and np.array_equal(eI, ref["err_if"])
        for s, a in slabs.items():
            assert np.array_equal(a, ref["uT_sub"][s]), (rank, s)
        held += list(slabs)
    assert sorted(held) == list(range(run.n_sub))


def test_block_partition():
    from paper_1306_4596_b200.dist import block_of

    assert [block_of(r, 8, 32) for r in range(8)] == [(4 * r, 4 * r + 4) for r in range(8)]
    with pytest.raises(ValueError):
        block_of(0, 3, 32)


class FakeShardProblem:
    """The library side of dist.sharded_monodomain on CPU (tests only): U(T) and the U-lines come from the
    oracle's monodomain, with every column outside this rank's range poisoned (NaN) until the all_to_all
    fills it; each step writes (rank, step, side) markers into the send halo and checks that the receive
    halo holds the right neighbour's marker -- the exchange pattern of the x-halo, including two ranks where
    the left and the right neighbour are the same process."""

    def __init__(self, prob, rank, world):
        self.prob, self.rank, self.world = prob, rank, world

    def mono_shard_begin(self, x0, x1, lines, halo):
        import oracle

        self.x0, self.x1, self.halo, self.n = x0, x1, halo, 0
        UT, rec = oracle.monodomain(self.prob, lines)
        self.UT = UT.copy()
        self.UL = rec.reshape(len(lines) * self.prob.grid.nt, self.prob.grid.nx).copy()
        self.ref = (UT, rec.reshape(self.UL.shape).copy())
        for a in (self.UT, self.UL):
            a[:, :x0] = np.nan
            a[:, x1:] = np.nan

    def mono_shard_step(self):
        if self.n > 0:  # recv_lo: the left neighbour's send_hi (side 1); recv_hi: the right one's send_lo (side 0)
            left, right = (self.rank - 1) % self.world, (self.rank + 1) % self.world
            assert self.halo[2][0].item() == 1000 * left + 10 * (self.n - 1) + 1, (self.rank, self.halo[2][0])
            assert self.halo[3][0].item() == 1000 * right + 10 * (self.n - 1) + 0, (self.rank, self.halo[3][0])
        self.halo[0].fill_(1000 * self.rank + 10 * self.n + 0)
        self.halo[1].fill_(1000 * self.rank + 10 * self.n + 1)
        self.n += 1

    def mono_shard_end(self):
        pass

    def mono_shard_copy(self, what, direction, a, b, xa, xb, buf):
        arr = self.UT if what == 0 else self.UL
        if direction == 0:
            buf.copy_(torch.from_numpy(np.ascontiguousarray(arr[a:b, xa:xb])))
        else:
            arr[a:b, xa:xb] = buf.numpy()


def _shard_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1306_4596_b200.dist import block_of, decompose, sharded_monodomain

    run = ki.scaled(ki.config("c4"), nx=128, nv=64, nt=6, K=2).with_(n_sub=4)
    prob = ki.make_problem(run)
    pb = FakeShardProblem(prob, rank, world)
    lines = sharded_monodomain(pb, run.grid, run.n_sub, run.overlap, rank, world, "cpu")
    lo, hi = decompose(run.grid.nv, run.n_sub, run.overlap)
    sb, se = block_of(rank, world, run.n_sub)
    UT, UL = pb.ref
    ok = np.array_equal(pb.UT[lo[sb]:hi[se - 1] + 1], UT[lo[sb]:hi[se - 1] + 1])
    nt = run.grid.nt
    for s in range(sb, se):
        for node in ([lo[s]] if s > 0 else []) + ([hi[s]] if s < run.n_sub - 1 else []):
            li = lines.index(node)
            ok &= np.array_equal(pb.UL[li * nt:(li + 1) * nt], UL[li * nt:(li + 1) * nt])
    out[rank] = bool(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_monodomain_exchange(world):
    """dist.sharded_monodomain's host logic (x-halo P2P every step, the all_to_all redistribution) with gloo:
    every rank ends with the complete U(T) rows of its subdomains and its interface lines."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))

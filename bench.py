#!/usr/bin/env python
"""Benchmark of the SWR hot path (BASELINE.json metric: grid-point updates/s, N_x N_v N_t K / wall).

One bench "step" = one complete Jacobi SWR solve of the workload (K iterations:
every subdomain's window of N_t fused step launches, trace exchange, error
accumulation), inputs resident in HBM (the monodomain reference is computed
once before timing, as SURVEY.md §8(d) prescribes).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c3|c4|c4wG|...]

N = 1: workload c2 (BASELINE.json configs[2], "single-GPU large Robin SWR").
N > 1 (torchrun, one process per GPU, NCCL): the weak-scaling c4 family
(N_v = 4096 N, S = 4 N); configs[4] itself at N = 8.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import kfp_inputs as ki  # noqa: E402

BYTES_PER_UPDATE = 16  # read u^n + write u^{n+1}, fp64
NOMINAL_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth (report both bases)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"  # /opt/skills/guides/B200_PROFILING.md fallback


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def committed_traffic(plan: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture of the same plan, or None."""
    import glob

    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json"))):
        try:
            d = json.load(open(f))
            if d.get("bench", {}).get("config", {}).get("plan") == plan:
                best = float(d["dram_traffic_bytes_per_launch"])
        except Exception:
            pass
    return best


L2_BYTES = 126 * 1024 * 1024


def default_workload(n_gpus: int) -> str:
    return "c2" if n_gpus == 1 else f"c4w{n_gpus}"


def oracle_sample(run: ki.Run, budget_updates: float = 2.5e9):
    """A bounded sample of the workload for the CPU oracle: the same grid (same a, CFL, dt), the
    window cut to n_t' steps (t_final scaled so dt is unchanged) and K' = 1 iteration."""
    g = run.grid
    per_step = g.nx * g.nv * 2  # monodomain + one SWR iteration per step
    nt = int(max(1, min(g.nt, budget_updates // per_step)))
    dt = g.t_final / g.nt
    return ki.scaled(run, nt=nt, K=1, t_final=dt * nt, name=run.name + "_sample")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def run_cpu_oracle(run: ki.Run, steps: int = 1):
    """Time the oracle as it stands on the host cores; returns (updates/s, cores, sample text, s per step)."""
    import oracle

    sample = oracle_sample(run)
    prob = ki.make_problem(sample)
    g = sample.grid
    updates = g.nx * g.nv * g.nt * (1 + sample.K)  # monodomain window + K iterations of windows
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.swr(prob, sample.kind, sample.p, sample.overlap, sample.n_sub, sample.K, q=sample.q)
    dt = time.perf_counter() - t0
    text = (f"{run.name} grid {g.nx}x{g.nv}, same dt/CFL, window cut to n_t={g.nt} steps, K=1, "
            f"plus the monodomain window; {updates:.3g} updates per step; host: {cpu_model()}, "
            f"nproc={os.cpu_count()}, OpenMP threads={oracle.num_threads()}")
    return updates * steps / dt, oracle.num_threads(), text, dt / steps


def bench_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    run = ki.config(args.workload or default_workload(args.gpus))
    for _ in range(max(0, min(args.warmup, 1))):
        run_cpu_oracle(run, 1)
    value, cores, text, per_step = run_cpu_oracle(run, args.steps)
    line = {
        "impl": "reference", "metric": "grid-point updates/s (N_x*N_v*N_t*K / wall)", "value": value,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {"workload": run.name, "oracle_sample": text},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": "oracle", "sample": text,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_single(args):
    import torch

    from paper_1306_4596_b200 import KfpError, Problem

    run = ki.config(args.workload or default_workload(1))
    g = run.grid
    prob = ki.make_problem(run)
    dev = 0
    torch.cuda.set_device(dev)
    # a real stream (not the legacy default, handle 0, which kfp_set_stream reads as "the library's own
    # stream"): the library launches on it and the timing events are recorded on it
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    pb = Problem(prob, device=dev)
    pb.set_stream(stream.cuda_stream)
    pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)  # monodomain reference here (untimed)
    try:
        pb.set_pipeline(0)  # the library's automatic schedule, as kfp_swr_solve (pipelines only latency-bound windows)
    except KfpError as exc:  # (kfp_swr_solve ignores this too: one iteration per sweep)
        print(f"bench: automatic pipelining not applied: {exc}", file=sys.stderr)
    torch.cuda.synchronize()

    def one():
        pb.reset()
        pb.iterate(run.K)

    # exactly W untimed warm-up solves
    warm = 0
    while warm < args.warmup:
        one()
        torch.cuda.synchronize()
        warm += 1
    launches0 = pb.launch_count()
    # the slabs (two buffers per subdomain) against the 126 MB L2: a working set that fits is flushed
    # between the timed steps (a 256 MB write, outside the per-step events)
    slab_bytes = 2 * 8 * g.nx * sum(pb.subdomain_range(s)[1] - pb.subdomain_range(s)[0] + 1 for s in range(run.n_sub))
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev) if slab_bytes < 2 * L2_BYTES else None
    clocks = ClockSampler(dev)
    clocks.start()
    step_kernel_ms = 0.0
    ms = 0.0
    step_ms = []
    torch.cuda.synchronize()
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        one()
        ev1.record(stream)
        # window times of this solve (events recorded by the library on the same stream)
        _, kms = pb.last_timing()
        step_kernel_ms += kms
        torch.cuda.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        ms += step_ms[-1]
    clk = clocks.stop()
    launches = pb.launch_count() - launches0
    updates = run.updates
    value = updates * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (the fused step): algorithmic bytes per launch / avg duration
    rows = sum(pb.subdomain_range(s)[1] - pb.subdomain_range(s)[0] + 1 for s in range(run.n_sub))
    # Dirichlet interface ends and (IMEX FD) the physical ends are not solved; the split-FEM scheme's
    # physical ends are Neumann (unknown)
    unknown_rows = rows - 2 * (run.n_sub - 1) * (0 if run.kind == "robin" else 1) - (0 if run.scheme == "split_fem" else 2)
    # per launch of the step kernel: the launches actually made (a pipelined sweep advances several iterations
    # per launch; otherwise nt * K per solve) and the algorithmic bytes they moved
    nominal = g.nt * run.K * args.steps
    step_launches = launches if 0 < launches < nominal else nominal
    per_launch_s = step_kernel_ms / 1e3 / step_launches
    bytes_per_launch = BYTES_PER_UPDATE * g.nx * unknown_rows * nominal / step_launches
    achieved = bytes_per_launch / per_launch_s / 1e9
    peak, peak_kind = measured_peaks()
    traffic = committed_traffic(plan := pb.plan())
    eT, eI = pb.history()

    # end to end through the public API with host buffers (create -> solve -> read back): the input tables and
    # the result live in pinned host memory (allocated outside the timed region)
    e2e_steps = 0 if args.no_e2e else max(1, min(args.steps, 5))

    def pinned_copy(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t

    pins = [pinned_copy(np.asarray(x, dtype=np.float64)) for x in (prob.ft, prob.fv, prob.fx, prob.u0v, prob.u0x)]
    prob_pinned = dataclasses.replace(prob, **{k: t.numpy() for k, t in zip(("ft", "fv", "fx", "u0v", "u0x"), pins)})
    uT_pinned = torch.empty((g.nv + 1, g.nx), dtype=torch.float64, pin_memory=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d2h = 0

    def e2e_solve():
        with Problem(prob_pinned, device=dev) as q:
            q.set_stream(stream.cuda_stream)
            uT = q.solve(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q, out=uT_pinned.numpy())
            h = q.history()
        return uT.nbytes + h[0].nbytes + h[1].nbytes

    if e2e_steps:
        e2e_solve()  # one untimed warm-up solve through the same calls
    torch.cuda.synchronize()
    e2e_host_ms = []
    e0.record(stream)
    for _ in range(e2e_steps):
        th = time.perf_counter()
        d2h = e2e_solve()
        e2e_host_ms.append(round((time.perf_counter() - th) * 1e3, 3))
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / max(1, e2e_steps)
    e2e_value = updates / (e2e_ms / 1e3) if e2e_steps else None

    # where an end-to-end solve spends its time (separate, untimed for the headline: a host synchronisation
    # after each public call): create (table H2D), setup (allocations, the monodomain reference with its
    # recorded interface lines, constant tables), the K iterations, the D2H of u(T) and the history, destroy
    phases = None
    mono = None
    if e2e_steps:
        ph = {}
        outs_pinned = []
        for s_ in range(run.n_sub):
            lo_, hi_ = pb.subdomain_range(s_)
            outs_pinned.append(torch.empty((hi_ - lo_ + 1, g.nx), dtype=torch.float64, pin_memory=True))
        torch.cuda.synchronize()
        t = time.perf_counter()
        q = Problem(prob_pinned, device=dev)
        q.set_stream(stream.cuda_stream)
        torch.cuda.synchronize()
        ph["create"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
        q.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
        torch.cuda.synchronize()
        ph["setup_incl_monodomain"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
        q.iterate(run.K)
        torch.cuda.synchronize()
        ph["iterate"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
        for s_ in range(run.n_sub):  # into pinned host buffers, as the timed leg's assembled u(T)
            q.subdomain_uT(s_, out=outs_pinned[s_].numpy())
        q.history()
        ph["d2h"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
        q.close()
        torch.cuda.synchronize()
        ph["destroy"] = (time.perf_counter() - t) * 1e3
        phases = {k: round(v, 3) for k, v in ph.items()}
        # the monodomain reference alone (reported separately, N_x N_v N_t updates / s)
        with Problem(prob, device=dev) as q:
            q.set_stream(stream.cuda_stream)
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            m0.record(stream)
            q.monodomain(copy=False)
            m1.record(stream)
            torch.cuda.synchronize()
            mms = m0.elapsed_time(m1)
            mono = {"value": g.nx * g.nv * g.nt / (mms / 1e3), "unit": "updates/s", "ms": mms}

    cpu = None
    if not args.no_cpu:
        v, cores, text, _ = run_cpu_oracle(run, 1)
        cpu = {"value": v, "unit": "updates/s", "cores": cores, "kind": "oracle", "sample": text,
               "cpu_model": cpu_model(), "nproc": os.cpu_count()}

    line = {
        "metric": "grid-point updates/s (N_x*N_v*N_t*K / wall)", "value": value, "unit": "updates/s",
        "n_gpus": 1, "steps": args.steps, "warmup": warm, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": run.name, "nx": g.nx, "nv": g.nv, "nt": g.nt, "K": run.K, "n_sub": run.n_sub,
                   "kind": run.kind, "p": run.p, "q": run.q, "overlap": run.overlap, "scheme": run.scheme, "plan": plan,
                   "l2": ("inputs larger than L2 (slab buffers %.0f MB vs 126 MB L2)" % (slab_bytes / 1e6))
                         if flush is None else
                         ("slab buffers %.0f MB, under twice the 126 MB L2 (part stays L2-resident from step to "
                          "step within a solve); L2 flushed between timed solves (256 MB write, outside the "
                          "per-solve events)" % (slab_bytes / 1e6)),
                   "parallelism": "v-subdomains on 1 GPU", "updates_per_step": updates},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "traffic": traffic, "peak_kind": peak_kind, "kernel": "kfp::step_fused_tma",
                     "traffic_source": "profiles/*_ncu_summary.json (ncu --set full, same plan)" if traffic else None,
                     "bytes_per_launch": bytes_per_launch, "avg_launch_us": per_launch_s * 1e6},
        "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": pb.h2d_bytes,
                "d2h_bytes_per_step": int(d2h), "ms": e2e_ms, "host_ms_per_solve": e2e_host_ms, "phases_ms": phases},
        "monodomain": mono,
        "ms_per_step_median": float(np.median(step_ms)), "ms_per_step_all": [round(x, 3) for x in step_ms],
        "gpu_launches": int(launches),
        "clocks": clk,
        "cpu_baseline": cpu,
        "err_T_last": float(eT[-1]), "err_if_last": float(eI[-1]),
    }
    pb.close()
    print(json.dumps(line), flush=True)
    return 0


def _json_stdout():
    """Keep stdout for the one JSON line: native code (NCCL's banner and messages, any printf) writes to file
    descriptor 1, so fd 1 is pointed at stderr and the JSON line goes to a duplicate of the original stdout."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = out
    return out


def spawn_ranks(args):
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU, NCCL) through torch.distributed.run
    on 127.0.0.1 and pass rank 0's JSON line through (the driver's own launch is the same command)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            print(line, flush=True)
    return r.returncode


def main():
    _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg (kernel experiments)")
    ap.add_argument("--chunks", type=int, default=4, help="N > 1: time chunks of the overlapped trace exchange")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1306_4596_b200 import dist

        return dist.bench_main(args, default_workload, ClockSampler, measured_peaks)
    return bench_single(args)


if __name__ == "__main__":
    sys.exit(main())

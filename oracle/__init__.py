"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SWR solve (arXiv 1306.4596).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1306_4596_b200``) never imports it and shares no code
with it; it takes its inputs from ``kfp_inputs`` like the CUDA path does.

Contents
--------
* ``kfp_oracle.c`` (built into ``liborc.so``): the plain fp64 step-by-step
  monodomain + Jacobi / Gauss-Seidel SWR solver (see its header for the paper
  passages), for both discretisations: the IMEX finite-difference scheme of
  BASELINE.json's north_star and the paper's own split finite-element scheme
  (``prob.scheme == "split_fem"``).
* ``modal.py``: the mode-reduced oracle for the manufactured-solution configs
  (a special case that reduces the 2-D scheme to one complex 1-D recurrence
  per step, solved with LAPACK's banded solver).
* ``dense.py``: brute-force dense space-time assemblies for tiny grids.

Parity status per function: every function here is pinned by
``tests/test_oracle_pins.py``; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kfp_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None

KIND = {"dirichlet": 0, "robin": 1}
END_PHYS, END_DIRICHLET, END_ROBIN = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2, OpenMP over x-columns)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", _LIB_PATH, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB_PATH


class _Problem(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int32), ("nv", ctypes.c_int32), ("nt", ctypes.c_int32),
        ("vmax", ctypes.c_double), ("t_final", ctypes.c_double),
        ("f_rank", ctypes.c_int32),
        ("ft", ctypes.c_void_p), ("fv", ctypes.c_void_p), ("fx", ctypes.c_void_p),
        ("u0_rank", ctypes.c_int32),
        ("u0v", ctypes.c_void_p), ("u0x", ctypes.c_void_p),
        ("scheme", ctypes.c_int32),
    ]


SCHEME = {"imex_fd": 0, "split_fem": 1}


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.POINTER(_Problem)
            dp = ctypes.c_void_p
            lib.orc_num_threads.restype = ctypes.c_int
            lib.orc_subdomains.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp]
            lib.orc_monodomain.argtypes = [P, ctypes.c_int, dp, dp, dp]
            lib.orc_window.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       dp, dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, dp,
                                       ctypes.c_int, dp, dp, dp]
            lib.orc_swr.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    dp, dp, dp, dp, dp, dp]
            lib.orc_swr_pq.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, dp, dp, dp, dp, dp, dp]
            lib.orc_swr_gs.argtypes = lib.orc_swr_pq.argtypes
            lib.orc_swr_ex.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp, dp, dp]
            lib.orc_window_pq.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_double, dp, dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, dp,
                                          ctypes.c_int, dp, dp, dp]
            _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class _Bound:
    """Keeps the numpy tables alive while the C struct points at them."""

    def __init__(self, prob):
        g = prob.grid
        self.arrays = [np.ascontiguousarray(x, dtype=np.float64) for x in (prob.ft, prob.fv, prob.fx, prob.u0v, prob.u0x)]
        ft, fv, fx, u0v, u0x = self.arrays
        self.s = _Problem(g.nx, g.nv, g.nt, g.vmax, g.t_final, prob.f_rank,
                          _ptr(ft), _ptr(fv), _ptr(fx), prob.u0_rank, _ptr(u0v), _ptr(u0x),
                          SCHEME[getattr(prob, "scheme", "imex_fd")])

    def ref(self):
        return ctypes.byref(self.s)


def num_threads() -> int:
    return int(_load().orc_num_threads())


def subdomains(nv: int, n_sub: int, overlap: int):
    lo = np.zeros(n_sub, np.int32)
    hi = np.zeros(n_sub, np.int32)
    if _load().orc_subdomains(nv, n_sub, overlap, _ptr(lo), _ptr(hi)) != 0:
        raise ValueError("invalid decomposition")
    return lo, hi


def monodomain(prob, rec_nodes=()):
    """U(T) [(nv+1), nx] and U at rec_nodes for n=1..nt ([len, nt, nx])."""
    g = prob.grid
    b = _Bound(prob)
    nodes = np.ascontiguousarray(rec_nodes, dtype=np.int32)
    rec = np.zeros((max(len(nodes), 1), g.nt, g.nx))
    UT = np.zeros((g.nv + 1, g.nx))
    _load().orc_monodomain(b.ref(), len(nodes), _ptr(nodes), _ptr(rec), _ptr(UT))
    return UT, rec[: len(nodes)]


def window(prob, lo, hi, ltype, rtype, p, gL, gR, send_kind, sendL_node=-1, sendR_node=-1, rec_nodes=(), q=None):
    """One subdomain window solve; returns (uT, sendL, sendR, rec).  Robin ends: p on the right (hi) end and
    on the trace sent left, q (default p) on the left (lo) end and on the trace sent right (OSWR(p,q))."""
    g = prob.grid
    b = _Bound(prob)
    gL = None if gL is None else np.ascontiguousarray(gL, dtype=np.float64)
    gR = None if gR is None else np.ascontiguousarray(gR, dtype=np.float64)
    sendL = np.zeros((g.nt, g.nx)) if sendL_node >= 0 else None
    sendR = np.zeros((g.nt, g.nx)) if sendR_node >= 0 else None
    nodes = np.ascontiguousarray(rec_nodes, dtype=np.int32)
    rec = np.zeros((max(len(nodes), 1), g.nt, g.nx))
    uT = np.zeros((hi - lo + 1, g.nx))
    _load().orc_window_pq(b.ref(), lo, hi, ltype, rtype, p if q is None else q, p, _ptr(gL), _ptr(gR),
                          KIND[send_kind] if isinstance(send_kind, str) else send_kind,
                          sendL_node, _ptr(sendL), sendR_node, _ptr(sendR), len(nodes), _ptr(nodes), _ptr(rec), _ptr(uT))
    return uT, sendL, sendR, rec[: len(nodes)]


def swr(prob, kind: str, p: float, overlap: int, n_sub: int, K: int, want_traces: bool = False, q=None,
        schedule: str = "jacobi", init_traces=None):
    """Jacobi SWR; returns dict(uT, uT_sub (list of slabs), UT, err_T, err_if, err_ov, traces, lo, hi); err_ov is
    the paper's convergence quantity (eq. 'error'): max over the closed overlaps of |u_s - u_{s+1}|.
    Robin: OSWR(p, q) with p on every right end and q (default p: one-sided OSWR(p)) on every left end.
    schedule: "jacobi" (parallel) or "gauss_seidel" (the paper's SWR1-SWR4).
    init_traces: None (zero lambda^0) or (toL, toR), each [n_sub-1, nt, nx]: the initial traces toward the left
    subdomain's right end and toward the right subdomain's left end of every interface."""
    g = prob.grid
    b = _Bound(prob)
    lo, hi = subdomains(g.nv, n_sub, overlap)
    tot = int(sum((h - l + 1) for l, h in zip(lo, hi))) * g.nx
    uT_sub = np.zeros(tot)
    uT = np.zeros((g.nv + 1, g.nx))
    UT = np.zeros((g.nv + 1, g.nx))
    err_T = np.zeros(K)
    err_if = np.zeros(K)
    err_ov = np.zeros(K)
    traces = np.zeros((max(2 * (n_sub - 1), 1), g.nt, g.nx)) if want_traces else None
    gs = {"jacobi": 0, "gauss_seidel": 1}[schedule]
    iL = iR = None
    if init_traces is not None:
        iL, iR = (np.ascontiguousarray(a, dtype=np.float64).reshape(n_sub - 1, g.nt, g.nx) for a in init_traces)
    rc = _load().orc_swr_ex(b.ref(), KIND[kind], p, p if q is None else q, overlap, n_sub, K, gs, _ptr(iL), _ptr(iR),
                            _ptr(uT_sub), _ptr(uT), _ptr(UT), _ptr(err_T), _ptr(err_if), _ptr(traces), _ptr(err_ov))
    if rc != 0:
        raise ValueError("orc_swr rejected the arguments")
    slabs, off = [], 0
    for l, h in zip(lo, hi):
        n = (h - l + 1) * g.nx
        slabs.append(uT_sub[off:off + n].reshape(h - l + 1, g.nx))
        off += n
    return dict(uT=uT, uT_sub=slabs, UT=UT, err_T=err_T, err_if=err_if, err_ov=err_ov,
                traces=None if traces is None else traces[: 2 * (n_sub - 1)], lo=lo, hi=hi)

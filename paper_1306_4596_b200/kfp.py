"""Thin ctypes binding of the C-ABI in ``include/kfp.h`` (argument marshalling only).

Every numerical step runs in ``libkfp.so`` (sm_100a CUDA kernels).  There is no
CPU fallback: if the library cannot be loaded, or no B200 is present, the
calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KFP_LIB_PATH") or os.path.join(_HERE, "libkfp.so")  # override: debugging builds only

KFP_OK, KFP_E_INVAL, KFP_E_CFL, KFP_E_NOMEM, KFP_E_CUDA, KFP_E_STATE, KFP_E_NONFINITE = 0, -1, -2, -3, -4, -6, -7
KIND = {"dirichlet": 0, "robin": 1}
SCHEME = {"imex_fd": 0, "split_fem": 1}
METRIC = {"err_T": 0, "err_if": 1, "overlap": 2}  # kfp_metric  # kfp_scheme (include/kfp.h)

# Every symbol include/kfp.h declares (checked by tests/test_abi.py).
SYMBOLS = (
    "kfp_problem_create", "kfp_problem_create_ex", "kfp_problem_destroy", "kfp_set_stream", "kfp_monodomain_solve", "kfp_swr_setup", "kfp_swr_setup_pq", "kfp_swr_solve_pq", "kfp_swr_set_schedule", "kfp_swr_setup_batch",
    "kfp_swr_batch_history", "kfp_swr_batch_subdomain_uT", "kfp_swr_set_initial_trace",
    "kfp_swr_reset", "kfp_swr_iterate", "kfp_swr_edge_buffers", "kfp_swr_bind_edge_buffers", "kfp_swr_solve", "kfp_error_history",
    "kfp_swr_subdomain_uT", "kfp_swr_subdomain_range", "kfp_swr_trace", "kfp_monodomain_uT", "kfp_launch_count",
    "kfp_plan", "kfp_last_timing", "kfp_last_error", "kfp_release_cached_memory",
    "kfp_swr_set_overlap_error", "kfp_swr_overlap_history", "kfp_swr_iterate_until", "kfp_swr_set_pipeline",
    "kfp_swr_iterate_chunk", "kfp_swr_chunk_send_wait", "kfp_swr_chunk_recv_done",
    "kfp_monodomain_shard_begin", "kfp_monodomain_shard_step", "kfp_monodomain_shard_end", "kfp_monodomain_shard_copy",
)


class KfpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kfp status {status}: {msg}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int32), ("nv", ctypes.c_int32), ("nt", ctypes.c_int32),
        ("vmax", ctypes.c_double), ("t_final", ctypes.c_double),
        ("f_rank", ctypes.c_int32),
        ("ft", ctypes.c_void_p), ("fv", ctypes.c_void_p), ("fx", ctypes.c_void_p),
        ("u0_rank", ctypes.c_int32),
        ("u0v", ctypes.c_void_p), ("u0x", ctypes.c_void_p),
        ("device", ctypes.c_int32),
    ]


_lib = None


def load(path: str = LIB_PATH):
    """Load libkfp.so and declare the prototypes (raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA library is required; there is no CPU path)")
    lib = ctypes.CDLL(path)
    vp, i32, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
    pd = ctypes.POINTER(ctypes.c_double)
    ppd = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "kfp_problem_create": (i32, [ctypes.POINTER(_Desc), ctypes.POINTER(vp)]),
        "kfp_problem_create_ex": (i32, [ctypes.POINTER(_Desc), i32, ctypes.POINTER(vp)]),
        "kfp_problem_destroy": (None, [vp]),
        "kfp_set_stream": (i32, [vp, vp]),
        "kfp_monodomain_solve": (i32, [vp, vp]),
        "kfp_swr_setup": (i32, [vp, i32, dbl, i32, i32, i32, i32, i32]),
        "kfp_swr_setup_pq": (i32, [vp, i32, dbl, dbl, i32, i32, i32, i32, i32]),
        "kfp_swr_set_schedule": (i32, [vp, i32]),
        "kfp_swr_setup_batch": (i32, [vp, i32, vp, vp, i32, i32, i32, i32]),
        "kfp_swr_batch_history": (i32, [vp, i32, i32, vp, vp, vp]),
        "kfp_swr_batch_subdomain_uT": (i32, [vp, i32, i32, vp]),
        "kfp_swr_set_initial_trace": (i32, [vp, i32, i32, vp]),
        "kfp_swr_solve_pq": (i32, [vp, i32, dbl, dbl, i32, i32, i32, vp]),
        "kfp_swr_reset": (i32, [vp]),
        "kfp_swr_iterate": (i32, [vp, i32]),
        "kfp_swr_edge_buffers": (i32, [vp, i32, ppd, ppd, ppd, ppd]),
        "kfp_swr_bind_edge_buffers": (i32, [vp, i32, vp, vp, vp, vp]),
        "kfp_swr_solve": (i32, [vp, i32, dbl, i32, i32, i32, vp]),
        "kfp_error_history": (i32, [vp, i32, ctypes.POINTER(i32), vp, vp]),
        "kfp_swr_subdomain_uT": (i32, [vp, i32, vp]),
        "kfp_swr_subdomain_range": (i32, [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "kfp_swr_trace": (i32, [vp, i32, i32, vp]),
        "kfp_monodomain_uT": (i32, [vp, vp]),
        "kfp_launch_count": (ctypes.c_int64, [vp]),
        "kfp_plan": (ctypes.c_char_p, [vp]),
        "kfp_last_timing": (i32, [vp, pd, pd]),
        "kfp_last_error": (ctypes.c_char_p, []),
        "kfp_release_cached_memory": (None, []),
        "kfp_swr_set_overlap_error": (i32, [vp, i32]),
        "kfp_swr_set_pipeline": (i32, [vp, i32]),
        "kfp_swr_overlap_history": (i32, [vp, i32, i32, ctypes.POINTER(i32), vp]),
        "kfp_swr_iterate_until": (i32, [vp, i32, dbl, i32, ctypes.POINTER(i32)]),
        "kfp_swr_iterate_chunk": (i32, [vp, i32, i32]),
        "kfp_monodomain_shard_begin": (i32, [vp, i32, i32, vp, i32, vp, vp, vp, vp]),
        "kfp_monodomain_shard_step": (i32, [vp]),
        "kfp_monodomain_shard_end": (i32, [vp]),
        "kfp_monodomain_shard_copy": (i32, [vp, i32, i32, i32, i32, i32, i32, vp]),
        "kfp_swr_chunk_send_wait": (i32, [vp, vp, i32]),
        "kfp_swr_chunk_recv_done": (i32, [vp, vp, i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st: int):
    if st != KFP_OK:
        raise KfpError(st, load().kfp_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Problem:
    """One problem on one device (``kfp_problem``).  ``prob`` is a ``kfp_inputs.Problem``-like object
    (``grid`` with nx, nv, nt, vmax, t_final and tables ft, fv, fx, u0v, u0x).  The discretisation is
    ``scheme`` if given, else ``prob.scheme`` (default "imex_fd"; "split_fem" is the paper's own)."""

    def __init__(self, prob, device: int = 0, scheme: Optional[str] = None):
        lib = load()
        g = prob.grid
        self.grid = g
        tabs = [np.ascontiguousarray(x, dtype=np.float64) for x in (prob.ft, prob.fv, prob.fx, prob.u0v, prob.u0x)]
        ft, fv, fx, u0v, u0x = tabs
        d = _Desc(g.nx, g.nv, g.nt, g.vmax, g.t_final, ft.shape[0], _ptr(ft), _ptr(fv), _ptr(fx),
                  u0v.shape[0], _ptr(u0v), _ptr(u0x), device)
        h = ctypes.c_void_p()
        self.scheme = scheme or getattr(prob, "scheme", "imex_fd")
        _check(lib.kfp_problem_create_ex(ctypes.byref(d), SCHEME[self.scheme], ctypes.byref(h)))
        self._h = h
        self.h2d_bytes = int(sum(t.nbytes for t in tabs))
        self.n_sub = None
        self.s_begin = self.s_end = None

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().kfp_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- calls
    def set_stream(self, stream_handle: int):
        _check(load().kfp_set_stream(self._h, ctypes.c_void_p(stream_handle or None)))

    def monodomain(self, copy: bool = True):
        g = self.grid
        out = np.empty((g.nv + 1, g.nx)) if copy else None
        _check(load().kfp_monodomain_solve(self._h, _ptr(out)))
        return out

    def monodomain_uT(self):
        g = self.grid
        out = np.empty((g.nv + 1, g.nx))
        _check(load().kfp_monodomain_uT(self._h, _ptr(out)))
        return out

    def setup(self, kind: str, p: float, overlap: int, n_sub: int, K_max: int, s_begin: int = 0,
              s_end: Optional[int] = None, q: Optional[float] = None):
        """q: Robin parameter of the left ends (two-sided OSWR(p, q)); None = one-sided OSWR(p)."""
        s_end = n_sub if s_end is None else s_end
        if q is None:
            _check(load().kfp_swr_setup(self._h, KIND[kind], float(p), int(overlap), int(n_sub), int(s_begin),
                                        int(s_end), int(K_max)))
        else:
            _check(load().kfp_swr_setup_pq(self._h, KIND[kind], float(p), float(q), int(overlap), int(n_sub),
                                           int(s_begin), int(s_end), int(K_max)))
        self.n_sub, self.s_begin, self.s_end = n_sub, s_begin, s_end

    def setup_batch(self, kind: str, ps, overlap: int, n_sub: int, K_max: int, qs=None):
        """Batched parameter sweep: replica r runs OSWR(ps[r], qs[r]) (qs None: one-sided)."""
        ps = np.ascontiguousarray(ps, dtype=np.float64)
        qs = None if qs is None else np.ascontiguousarray(qs, dtype=np.float64)
        _check(load().kfp_swr_setup_batch(self._h, KIND[kind], _ptr(ps), _ptr(qs), int(len(ps)), int(overlap),
                                          int(n_sub), int(K_max)))
        self.n_sub, self.s_begin, self.s_end, self.n_rep = n_sub, 0, n_sub, len(ps)

    def batch_history(self, rep: int):
        cap = 1 << 16
        kk = ctypes.c_int32()
        eT = np.zeros(cap)
        eI = np.zeros(cap)
        _check(load().kfp_swr_batch_history(self._h, int(rep), cap, ctypes.byref(kk), _ptr(eT), _ptr(eI)))
        return eT[: kk.value].copy(), eI[: kk.value].copy()

    def batch_subdomain_uT(self, rep: int, s: int):
        lo, hi = self.subdomain_range(s)
        out = np.empty((hi - lo + 1, self.grid.nx))
        _check(load().kfp_swr_batch_subdomain_uT(self._h, int(rep), int(s), _ptr(out)))
        return out

    def set_initial_trace(self, i: int, direction: int, values):
        """lambda^0 of local interface i toward the left subdomain's right end (0) / right subdomain's left end (1)."""
        v = np.ascontiguousarray(values, dtype=np.float64)
        assert v.shape == (self.grid.nt, self.grid.nx)
        _check(load().kfp_swr_set_initial_trace(self._h, int(i), int(direction), _ptr(v)))

    def set_schedule(self, schedule: str):
        """'jacobi' (default after setup) or 'gauss_seidel' (the paper's SWR1-SWR4, single process)."""
        _check(load().kfp_swr_set_schedule(self._h, {"jacobi": 0, "gauss_seidel": 1}[schedule]))

    def reset(self):
        _check(load().kfp_swr_reset(self._h))

    def iterate(self, n: int = 1):
        _check(load().kfp_swr_iterate(self._h, int(n)))

    def iterate_chunk(self, chunk: int, nchunks: int):
        """Launch chunk `chunk` of the current iteration (time-chunked exchange, include/kfp.h)."""
        _check(load().kfp_swr_iterate_chunk(self._h, int(chunk), int(nchunks)))

    def chunk_send_wait(self, stream_handle: int, chunk: int):
        _check(load().kfp_swr_chunk_send_wait(self._h, ctypes.c_void_p(stream_handle), int(chunk)))

    def chunk_recv_done(self, stream_handle: int, chunk: int):
        _check(load().kfp_swr_chunk_recv_done(self._h, ctypes.c_void_p(stream_handle), int(chunk)))

    def mono_shard_begin(self, x0: int, x1: int, lines, halo=(None, None, None, None)):
        """x-sharded monodomain reference: columns [x0, x1); halo = (send_lo, send_hi, recv_lo, recv_hi), device
        tensors or pointers of nv+1 doubles each (include/kfp.h)."""
        arr = np.ascontiguousarray(lines, dtype=np.int32)
        c = lambda p: None if p is None else ctypes.c_void_p(p if isinstance(p, int) else p.data_ptr())
        _check(load().kfp_monodomain_shard_begin(self._h, int(x0), int(x1), _ptr(arr) if arr.size else None,
                                                 int(arr.size), *[c(p) for p in halo]))

    def mono_shard_step(self):
        _check(load().kfp_monodomain_shard_step(self._h))

    def mono_shard_end(self):
        _check(load().kfp_monodomain_shard_end(self._h))

    def mono_shard_copy(self, what: int, direction: int, r0: int, r1: int, xa: int, xb: int, buf):
        """U(T) (what 0) / U-lines (what 1) rows [r0, r1) x columns [xa, xb) <-> a contiguous device buffer
        (tensor or pointer) of (r1 - r0) x (xb - xa) doubles."""
        ptr = buf if isinstance(buf, int) else buf.data_ptr()
        _check(load().kfp_monodomain_shard_copy(self._h, int(what), int(direction), int(r0), int(r1), int(xa), int(xb),
                                                ctypes.c_void_p(ptr)))

    def edge_buffers(self, parity: int):
        """(send_left, recv_left, send_right, recv_right) device pointers (int or None)."""
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        _check(load().kfp_swr_edge_buffers(self._h, int(parity), *[ctypes.byref(p) for p in ptrs]))
        return tuple(p.value for p in ptrs)

    def bind_edge_buffers(self, parity: int, send_left=None, recv_left=None, send_right=None, recv_right=None):
        """Point the cross-block exchange of `parity` at caller-owned device buffers (int pointers)."""
        c = lambda p: ctypes.c_void_p(p) if p else None
        _check(load().kfp_swr_bind_edge_buffers(self._h, int(parity), c(send_left), c(recv_left), c(send_right),
                                                c(recv_right)))

    def solve(self, kind: str, p: float, overlap: int, n_sub: int, K: int, copy: bool = True,
              q: Optional[float] = None, out: Optional[np.ndarray] = None):
        """Setup + K iterations; returns the assembled u^K(T) (into `out`, e.g. a pinned buffer, if given)."""
        g = self.grid
        if out is None:
            out = np.empty((g.nv + 1, g.nx)) if copy else None
        elif not (out.dtype == np.float64 and out.flags.c_contiguous and out.size == (g.nv + 1) * g.nx):
            raise ValueError("solve: out must be a C-contiguous float64 array of (nv+1)*nx elements")
        if q is None:
            _check(load().kfp_swr_solve(self._h, KIND[kind], float(p), int(overlap), int(n_sub), int(K), _ptr(out)))
        else:
            _check(load().kfp_swr_solve_pq(self._h, KIND[kind], float(p), float(q), int(overlap), int(n_sub), int(K),
                                           _ptr(out)))
        self.n_sub, self.s_begin, self.s_end = n_sub, 0, n_sub
        return out

    def history(self):
        cap = 1 << 16
        kk = ctypes.c_int32()
        eT = np.zeros(cap)
        eI = np.zeros(cap)
        _check(load().kfp_error_history(self._h, cap, ctypes.byref(kk), _ptr(eT), _ptr(eI)))
        return eT[: kk.value].copy(), eI[: kk.value].copy()

    def subdomain_range(self, s: int):
        lo, hi = ctypes.c_int32(), ctypes.c_int32()
        _check(load().kfp_swr_subdomain_range(self._h, int(s), ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def subdomain_uT(self, s: int, out: Optional[np.ndarray] = None):
        lo, hi = self.subdomain_range(s)
        if out is None:
            out = np.empty((hi - lo + 1, self.grid.nx))
        if not (out.dtype == np.float64 and out.flags.c_contiguous and out.size == (hi - lo + 1) * self.grid.nx):
            raise ValueError("subdomain_uT: out must be a C-contiguous float64 array of the slab's size")
        _check(load().kfp_swr_subdomain_uT(self._h, int(s), _ptr(out)))
        return out

    def trace(self, i: int, direction: int):
        g = self.grid
        out = np.empty((g.nt, g.nx))
        _check(load().kfp_swr_trace(self._h, int(i), int(direction), _ptr(out)))
        return out

    def set_overlap_error(self, on: bool = True):
        """Record the paper's convergence quantity max |u_s - u_{s+1}| over the overlaps."""
        _check(load().kfp_swr_set_overlap_error(self._h, 1 if on else 0))

    def set_pipeline(self, depth: int):
        """Pipelined Jacobi: advance `depth` consecutive iterations per sweep of nt + depth - 1 launches."""
        _check(load().kfp_swr_set_pipeline(self._h, int(depth)))

    def overlap_history(self, rep: int = 0):
        k = ctypes.c_int32(0)
        cap = 1 << 16
        out = np.zeros(cap)
        _check(load().kfp_swr_overlap_history(self._h, rep, cap, ctypes.byref(k), _ptr(out)))
        return out[: k.value].copy()

    def iterate_until(self, eps: float, k_max: int, metric: str = "overlap") -> int:
        """Iterate until the chosen error of the last iteration is below eps (or k_max more iterations);
        returns the iterations done since the last reset."""
        k = ctypes.c_int32(0)
        _check(load().kfp_swr_iterate_until(self._h, METRIC[metric], float(eps), int(k_max), ctypes.byref(k)))
        return int(k.value)

    def launch_count(self) -> int:
        return int(load().kfp_launch_count(self._h))

    def plan(self) -> str:
        return load().kfp_plan(self._h).decode()

    def last_timing(self):
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(load().kfp_last_timing(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


def last_error() -> str:
    return load().kfp_last_error().decode()


def release_cached_memory() -> None:
    """Return the device buffers of destroyed problems (kept for reuse, include/kfp.h) to the CUDA driver."""
    load().kfp_release_cached_memory()

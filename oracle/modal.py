"""TEST INFRASTRUCTURE ONLY -- mode-reduced oracle for the manufactured-solution configs.

Why it is exact (the Fourier-in-x idea of PAPER.md:118-130,
eq. Kolmogorov0): every operator of the discrete scheme (upwind transport in x
with periodic wrap; the per-column v-tridiagonal; the
Dirichlet / Robin transmission rows and traces) commutes with the
x-translation m -> m+1.  The manufactured data of BASELINE.json configs[0..3]
live in the single Fourier mode e^{i theta m}, theta = 2 pi / N_x:

    u0(x_m, v_j)   = Im( W_j e^{i theta m} ),
    f(t, x_m, v_j) = Im( e^{-t} [(2 - W_j) + i 2 pi v_j W_j] e^{i theta m} ),

so every iterate is exactly u^n_{j,m} = Im(c^n_j e^{i theta m}) with complex
amplitudes c^n_j that obey the same scheme with the transport replaced by its
symbol:  v_j > 0: 1 - nu_j (1 - e^{-i theta}),  v_j < 0: 1 - nu_j (e^{i theta} - 1),
v_j = 0: 1  (nu_j = v_j dt / h_x, reading R7).

This implementation is independent of ``kfp_oracle.c``: it does not read the
input tables (it evaluates the manufactured formulas itself), and it solves
the v-systems with LAPACK's banded solver (``scipy.linalg.solve_banded``), a
library primitive.  Cost O(N_v N_t K) instead of O(N_x N_v N_t K), so it gives
reference outputs at the full sizes of c2 and c3.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.linalg import solve_banded

__all__ = ["modal_swr", "modal_monodomain", "realize", "max_abs_real"]


def _grid(g):
    hx = 1.0 / g.nx
    hv = 2.0 * g.vmax / g.nv
    dt = g.t_final / g.nt
    v = -g.vmax + np.arange(g.nv + 1) * hv
    return hx, hv, dt, v


def _symbol(g):
    hx, hv, dt, v = _grid(g)
    th = 2.0 * math.pi / g.nx
    nu = v * dt / hx
    sym = np.ones(g.nv + 1, dtype=np.complex128)
    pos, neg = v > 0, v < 0
    sym[pos] = 1.0 - nu[pos] * (1.0 - np.exp(-1j * th))
    sym[neg] = 1.0 - nu[neg] * (np.exp(1j * th) - 1.0)
    W = g.vmax ** 2 - v * v
    F = (2.0 - W) + 1j * 2.0 * math.pi * v * W
    return sym, F, W


def max_abs_real(d: np.ndarray, nx: int, chunk: int = 1 << 22) -> float:
    """max over entries of d and m = 0..nx-1 of |Im(d e^{i theta m})| (exact on the grid)."""
    d = np.asarray(d).ravel()
    E = np.exp(1j * 2.0 * math.pi * np.arange(nx) / nx)
    best = 0.0
    step = max(1, chunk // nx)
    for i in range(0, d.size, step):
        blk = np.abs((d[i:i + step, None] * E[None, :]).imag)
        if blk.size:
            best = max(best, float(blk.max()))
    return best


def realize(c: np.ndarray, nx: int) -> np.ndarray:
    """u[j, m] = Im(c_j e^{i theta m})."""
    E = np.exp(1j * 2.0 * math.pi * np.arange(nx) / nx)
    return (np.asarray(c)[:, None] * E[None, :]).imag


class _Sub:
    """One subdomain [lo, hi] with end kinds ('phys' | 'dirichlet' | 'robin')."""

    def __init__(self, g, lo, hi, lkind, rkind, p):
        hx, hv, dt, v = _grid(g)
        self.lo, self.hi, self.lk, self.rk, self.p = lo, hi, lkind, rkind, p
        self.a = dt / (hv * hv)
        self.hv, self.dt = hv, dt
        self.first = lo if lkind == "robin" else lo + 1
        self.last = hi if rkind == "robin" else hi - 1
        nu = self.last - self.first + 1
        a = self.a
        ab = np.zeros((3, nu))
        ab[0, 1:] = -a  # super-diagonal
        ab[1, :] = 1.0 + 2.0 * a
        ab[2, :-1] = -a  # sub-diagonal
        if lkind == "robin":
            ab[1, 0] = 1.0 + 2.0 * a + 2.0 * a * p * hv
            if nu > 1:
                ab[0, 1] = -2.0 * a
        if rkind == "robin":
            ab[1, -1] = 1.0 + 2.0 * a + 2.0 * a * p * hv
            if nu > 1:
                ab[2, -2] = -2.0 * a
        self.ab = ab

    def step(self, c, sym, Fn1, gL, gR):
        """c: complex amplitudes on nodes lo..hi at t_n -> (c at t_{n+1}, r on lo..hi)."""
        lo, hi, a = self.lo, self.hi, self.a
        r = sym[lo:hi + 1] * c + self.dt * Fn1[lo:hi + 1]
        rhs = r[self.first - lo:self.last - lo + 1].copy()
        if self.lk == "robin":
            rhs[0] += 2.0 * a * self.hv * gL
        else:
            rhs[0] += a * (gL if self.lk == "dirichlet" else 0.0)
        if self.rk == "robin":
            rhs[-1] += 2.0 * a * self.hv * gR
        else:
            rhs[-1] += a * (gR if self.rk == "dirichlet" else 0.0)
        x = solve_banded((1, 1), self.ab, rhs, check_finite=False)
        out = np.empty(hi - lo + 1, dtype=np.complex128)
        out[self.first - lo:self.last - lo + 1] = x
        if self.first > lo:
            out[0] = gL if self.lk == "dirichlet" else 0.0
        if self.last < hi:
            out[-1] = gR if self.rk == "dirichlet" else 0.0
        return out, r


def _subdomains(nv, S, ov):
    lo, hi = [], []
    for s in range(S):
        cs, cs1 = s * (nv // S), (s + 1) * (nv // S)
        lo.append(0 if s == 0 else cs - ov // 2)
        hi.append(nv if s == S - 1 else cs1 + (ov + 1) // 2)
    return lo, hi


def modal_monodomain(g, rec_nodes=()):
    """Complex U(T) on nodes 0..nv and U at rec_nodes for n=1..nt ([len, nt])."""
    _, _, dt, _ = _grid(g)
    sym, F, W = _symbol(g)
    sub = _Sub(g, 0, g.nv, "phys", "phys", 0.0)
    c = W.astype(np.complex128)
    rec = np.zeros((len(rec_nodes), g.nt), dtype=np.complex128)
    for n in range(g.nt):
        c, _ = sub.step(c, sym, math.exp(-(n + 1) * dt) * F, 0.0, 0.0)
        for i, j in enumerate(rec_nodes):
            rec[i, n] = c[j]
    return c, rec


def modal_swr(g, kind: str, p: float, overlap: int, S: int, K: int):
    """Jacobi SWR on the mode amplitudes; returns dict(err_T, err_if, c_sub, C, traces, lo, hi)."""
    hx, hv, dt, v = _grid(g)
    sym, F, W = _symbol(g)
    lo, hi = _subdomains(g.nv, S, overlap)
    lines = sorted({lo[s] for s in range(1, S)} | {hi[s] for s in range(S - 1)})
    C, Ul = modal_monodomain(g, lines)
    Uline = {j: Ul[i] for i, j in enumerate(lines)}
    ek = "robin" if kind == "robin" else "dirichlet"
    subs = [_Sub(g, lo[s], hi[s], "phys" if s == 0 else ek, "phys" if s == S - 1 else ek, p) for s in range(S)]
    zeros = np.zeros(g.nt, dtype=np.complex128)
    toL_in = [zeros.copy() for _ in range(S - 1)]  # used at hi_i by subdomain i (sent by i+1)
    toR_in = [zeros.copy() for _ in range(S - 1)]  # used at lo_{i+1} by subdomain i+1 (sent by i)
    err_T, err_if = np.zeros(K), np.zeros(K)
    c_final = [None] * S
    for k in range(K):
        toL_out = [np.zeros(g.nt, dtype=np.complex128) for _ in range(S - 1)]
        toR_out = [np.zeros(g.nt, dtype=np.complex128) for _ in range(S - 1)]
        eT = eI = 0.0
        for s in range(S):
            sd = subs[s]
            c = W[lo[s]:hi[s] + 1].astype(np.complex128)
            recL = np.zeros(g.nt, dtype=np.complex128)
            recR = np.zeros(g.nt, dtype=np.complex128)
            for n in range(g.nt):
                gL = toR_in[s - 1][n] if s > 0 else 0.0
                gR = toL_in[s][n] if s < S - 1 else 0.0
                c, r = sd.step(c, sym, math.exp(-(n + 1) * dt) * F, gL, gR)
                if s > 0:  # trace for the left neighbour at node hi_{s-1}
                    jc = hi[s - 1] - lo[s]
                    if kind == "robin":
                        toL_out[s - 1][n] = p * c[jc] - ((c[jc] - c[jc + 1]) / hv + 0.5 * hv * (c[jc] - r[jc]) / dt)
                    else:
                        toL_out[s - 1][n] = c[jc]
                if s < S - 1:  # trace for the right neighbour at node lo_{s+1}
                    jc = lo[s + 1] - lo[s]
                    if kind == "robin":
                        toR_out[s][n] = p * c[jc] - ((c[jc] - c[jc - 1]) / hv + 0.5 * hv * (c[jc] - r[jc]) / dt)
                    else:
                        toR_out[s][n] = c[jc]
                recL[n] = c[0]
                recR[n] = c[-1]
            if s > 0:
                eI = max(eI, max_abs_real(recL - Uline[lo[s]], g.nx))
            if s < S - 1:
                eI = max(eI, max_abs_real(recR - Uline[hi[s]], g.nx))
            eT = max(eT, max_abs_real(c - C[lo[s]:hi[s] + 1], g.nx))
            c_final[s] = c
        err_T[k], err_if[k] = eT, eI
        toL_in, toR_in = toL_out, toR_out
    return dict(err_T=err_T, err_if=err_if, c_sub=c_final, C=C, lo=lo, hi=hi,
                toL=toL_in, toR=toR_in)

"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no transport, no diffusion, no
tridiagonal solve, no transmission condition, no error metric).  It only
samples the problem DATA of BASELINE.json's configs on the grid nodes:

* the manufactured solution's forcing ``f`` and initial value ``u0`` for
  configs c0-c3 (BASELINE.json configs[0..3]):
  ``u = e^{-t} sin(2 pi x) W(v)``, ``W(v) = Vmax^2 - v^2``,
  ``f = e^{-t}[(2 - W) sin 2 pi x + 2 pi v W cos 2 pi x]``;
* the random non-negative forcing of c4 (configs[4]):
  ``f = W(v) |sum_{k=1..16} a_k sin(2 pi k x + phi_k)|``,
  ``a_k ~ N(0, 1/k^2)``, ``phi_k ~ U[0, 2 pi)`` from ``numpy.random.default_rng(0)``
  (draw order: all ``a`` first, then all ``phi``; reading R15), ``u0 = 0``.

Every data field is handed to both sides as separable tables
(``f(t_n, x_m, v_j) = sum_r ft[r, n] fv[r, j] fx[r, m]``,
``u0(x_m, v_j) = sum_r u0v[r, j] u0x[r, m]``) -- the layout the C-ABI
(`include/kfp.h`, ``kfp_problem_desc``) takes.  The oracle and the CUDA path
both receive exactly these arrays; neither imports the other.

Grid node convention (readings R5/R6): ``x_m = m / N_x``
(m = 0..N_x-1, periodic), ``v_j = -Vmax + j * 2 Vmax / N_v`` (j = 0..N_v),
``t_n = n T / N_t`` (n = 0..N_t).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "Grid",
    "Problem",
    "Run",
    "CONFIGS",
    "config",
    "mms_problem",
    "random_forcing_problem",
    "make_problem",
    "weak_scaling_config",
    "fem_problem",
    "paper_grid",
    "SCHEMES",
]

# The two discretisations the library implements; a problem names its own.
SCHEMES = ("imex_fd", "split_fem")


@dataclasses.dataclass(frozen=True)
class Grid:
    nx: int
    nv: int
    nt: int
    vmax: float
    t_final: float

    def x_nodes(self) -> np.ndarray:
        return np.arange(self.nx, dtype=np.float64) / self.nx

    def v_nodes(self) -> np.ndarray:
        hv = 2.0 * self.vmax / self.nv
        return -self.vmax + np.arange(self.nv + 1, dtype=np.float64) * hv

    def t_nodes(self) -> np.ndarray:
        dt = self.t_final / self.nt
        return np.arange(self.nt + 1, dtype=np.float64) * dt


@dataclasses.dataclass
class Problem:
    """Grid + separable data tables (all float64, C-contiguous)."""

    grid: Grid
    ft: np.ndarray  # [f_rank, nt+1]
    fv: np.ndarray  # [f_rank, nv+1]
    fx: np.ndarray  # [f_rank, nx]
    u0v: np.ndarray  # [u0_rank, nv+1]  (u0_rank may be 0)
    u0x: np.ndarray  # [u0_rank, nx]
    data: str = "mms"
    scheme: str = "imex_fd"  # "imex_fd" (BASELINE.json north_star) | "split_fem" (the paper's, §3b)

    @property
    def f_rank(self) -> int:
        return int(self.ft.shape[0])

    @property
    def u0_rank(self) -> int:
        return int(self.u0v.shape[0])

    def f_dense(self, n: int) -> np.ndarray:
        """f(t_n, x_m, v_j) as a v-major [nv+1, nx] array (test helper)."""
        return np.einsum("r,rj,rm->jm", self.ft[:, n], self.fv, self.fx)

    def u0_dense(self) -> np.ndarray:
        if self.u0_rank == 0:
            return np.zeros((self.grid.nv + 1, self.grid.nx))
        return np.einsum("rj,rm->jm", self.u0v, self.u0x)

    def table_bytes(self) -> int:
        return int(self.ft.nbytes + self.fv.nbytes + self.fx.nbytes + self.u0v.nbytes + self.u0x.nbytes)


@dataclasses.dataclass(frozen=True)
class Run:
    """A named BASELINE.json config: grid + data kind + SWR parameters."""

    name: str
    grid: Grid
    data: str  # "mms" | "random"
    kind: str  # "dirichlet" | "robin"
    p: float
    overlap: int
    n_sub: int
    K: int
    q: Optional[float] = None  # two-sided OSWR(p, q): Robin parameter of the left ends (None: q = p)
    scheme: str = "imex_fd"    # discretisation (SCHEMES)

    @property
    def updates(self) -> int:
        """N_x * N_v * N_t * K -- the metric's unit count (BASELINE.json metric)."""
        g = self.grid
        return g.nx * g.nv * g.nt * self.K

    def with_(self, **kw) -> "Run":
        return dataclasses.replace(self, **kw)


def mms_problem(grid: Grid) -> Problem:
    """Manufactured solution of BASELINE.json configs[0] (rank-2 forcing, rank-1 u0)."""
    v = grid.v_nodes()
    x = grid.x_nodes()
    t = grid.t_nodes()
    W = grid.vmax ** 2 - v * v
    ft = np.stack([np.exp(-t), np.exp(-t)])
    fv = np.stack([2.0 - W, 2.0 * math.pi * v * W])
    fx = np.stack([np.sin(2.0 * math.pi * x), np.cos(2.0 * math.pi * x)])
    u0v = W[None, :].copy()
    u0x = np.sin(2.0 * math.pi * x)[None, :].copy()
    return Problem(grid, *(np.ascontiguousarray(a) for a in (ft, fv, fx, u0v, u0x)), data="mms")


def random_coefficients(seed: int = 0, n_modes: int = 16):
    """a_k ~ N(0, 1/k^2) (std 1/k) then phi_k ~ U[0, 2 pi) from default_rng(seed) (reading R15)."""
    rng = np.random.default_rng(seed)
    k = np.arange(1, n_modes + 1, dtype=np.float64)
    a = rng.normal(0.0, 1.0 / k)
    phi = rng.uniform(0.0, 2.0 * math.pi, n_modes)
    return a, phi


def random_forcing_problem(grid: Grid, seed: int = 0) -> Problem:
    """BASELINE.json configs[4] data: f = W(v) |sum_k a_k sin(2 pi k x + phi_k)|, time independent, u0 = 0."""
    a, phi = random_coefficients(seed)
    v = grid.v_nodes()
    x = grid.x_nodes()
    k = np.arange(1, a.size + 1, dtype=np.float64)
    s = np.abs((a[:, None] * np.sin(2.0 * math.pi * k[:, None] * x[None, :] + phi[:, None])).sum(axis=0))
    W = grid.vmax ** 2 - v * v
    ft = np.ones((1, grid.nt + 1))
    fv = W[None, :].copy()
    fx = s[None, :].copy()
    u0v = np.zeros((0, grid.nv + 1))
    u0x = np.zeros((0, grid.nx))
    return Problem(grid, *(np.ascontiguousarray(a) for a in (ft, fv, fx, u0v, u0x)), data="random")


def zero_problem(grid: Grid) -> Problem:
    """The error equation of the paper's experiments: f = 0, u0 = 0 (exact solution 0); the iterates
    are then the SWR errors themselves, driven by the initial traces (Table 1: random lambda^0)."""
    ft = np.zeros((1, grid.nt + 1))
    fv = np.zeros((1, grid.nv + 1))
    fx = np.zeros((1, grid.nx))
    u0v = np.zeros((0, grid.nv + 1))
    u0x = np.zeros((0, grid.nx))
    return Problem(grid, ft, fv, fx, u0v, u0x, data="zero")


def fem_problem(grid: Grid, u0_seed: Optional[int] = None) -> Problem:
    """Data of the paper's own experiments for the split-FEM scheme: the error
    equation f = 0 (rank-0 forcing tables) and u0 = 0 -- the iterates are then driven by the initial traces
    (random lambda^0) -- or, for parity cases, a rank-2 random u0 drawn from default_rng(u0_seed)
    (u0v ~ N(0, 1), u0x ~ N(0, 1), in that order)."""
    ft = np.zeros((0, grid.nt + 1))
    fv = np.zeros((0, grid.nv + 1))
    fx = np.zeros((0, grid.nx))
    if u0_seed is None:
        u0v = np.zeros((0, grid.nv + 1))
        u0x = np.zeros((0, grid.nx))
    else:
        rng = np.random.default_rng(u0_seed)
        u0v = rng.normal(size=(2, grid.nv + 1))
        u0x = rng.normal(size=(2, grid.nx))
    return Problem(grid, ft, fv, fx, u0v, u0x, data="zero" if u0_seed is None else "random_u0", scheme="split_fem")


def paper_grid(j: int) -> Grid:
    """The paper's Table 1 mesh at refinement level j: Delta t = h_x = h_v = 0.01 / 2^j on
    x in [0,1), v in [-1,1], T = 2 -- N_x = 100 2^j, N_v = 200 2^j cells, N_t = 200 2^j steps."""
    return Grid(100 * 2 ** j, 200 * 2 ** j, 200 * 2 ** j, 1.0, 2.0)


def make_problem(run: Run) -> Problem:
    if run.scheme == "split_fem":
        return fem_problem(run.grid, u0_seed=0 if run.data == "random_u0" else None)
    if run.data == "mms":
        return mms_problem(run.grid)
    if run.data == "random":
        return random_forcing_problem(run.grid)
    if run.data == "zero":
        return zero_problem(run.grid)
    raise ValueError(f"unknown data kind {run.data!r}")


# BASELINE.json configs[0..4].
CONFIGS = {
    "c0": Run("c0", Grid(64, 64, 100, 4.0, 0.25), "mms", "robin", 1.0, 0, 2, 20),
    "c1": Run("c1", Grid(256, 256, 1000, 4.0, 0.1), "mms", "dirichlet", 0.0, 8, 2, 40),
    "c2": Run("c2", Grid(4096, 4096, 1000, 4.0, 0.05), "mms", "robin", 4.0, 0, 2, 10),
    "c3": Run("c3", Grid(8192, 16384, 1000, 4.0, 0.02), "mms", "robin", 8.0, 0, 8, 15),
    "c4": Run("c4", Grid(2048, 32768, 500, 4.0, 0.01), "random", "dirichlet", 0.0, 4, 32, 30),
    # not a BASELINE.json config: the paper's finest Table 1 mesh with its own split-FEM scheme,
    # OSWR(11, 2.5) with overlap 3 h_v, Jacobi, random rank-2 u0 (a bench workload for that kernel)
    "paper_j4": Run("paper_j4", Grid(1600, 3200, 3200, 1.0, 2.0), "random_u0", "robin", 11.0, 3, 2, 10, q=2.5,
                    scheme="split_fem"),
}


def config(name: str) -> Run:
    if name.startswith("c4w"):
        return weak_scaling_config(int(name[3:] or 1))
    return CONFIGS[name]


def weak_scaling_config(g: int) -> Run:
    """SURVEY.md §8(d) weak-scaling family: N_v = 4096 g, S = 4 g, everything else as c4."""
    base = CONFIGS["c4"]
    return base.with_(name=f"c4w{g}", grid=dataclasses.replace(base.grid, nv=4096 * g), n_sub=4 * g)


def scaled(run: Run, *, nx: Optional[int] = None, nv: Optional[int] = None, nt: Optional[int] = None,
           K: Optional[int] = None, t_final: Optional[float] = None, name: Optional[str] = None) -> Run:
    """A reduced-size copy of a config with the same structure (used for oracle-sized parity cases)."""
    g = run.grid
    g2 = Grid(nx or g.nx, nv or g.nv, nt or g.nt, g.vmax, t_final if t_final is not None else g.t_final)
    return run.with_(name=name or (run.name + "_small"), grid=g2, K=K or run.K)

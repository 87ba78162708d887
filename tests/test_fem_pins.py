"""Pins of the oracle's second discretisation -- the paper's own split finite-element scheme
 -- against what the paper and the mathematics fix (-m "not gpu").

* a brute-force reference (oracle/dense.py): M and S from the Cavalieri-Simpson rule on the hat
  functions, dense LAPACK solves, Step 2 as interpolation at the characteristic foot;
* the closed-form decay of x-constant cosine modes (eigenvectors of the Neumann M and S);
* conservation of the discrete mass sum_j (M 1)_j sum_m u_jm (Neumann ends, periodic x);
* the discrete maximum principle;
* the algebraic fixed point of the SWR iteration = the monodomain solution (trace consistency);
* the iteration counts the paper prints in Table 1 (tests/golden/paper_table1.json).
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import kfp_inputs as ki
from oracle import END_DIRICHLET, END_PHYS, END_ROBIN
from oracle.dense import dense_fem_window, fem_matrices
from test_oracle_pins import _probe_fixed_point

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_simpson_matrices_are_the_p1_element_matrices():
    """Cavalieri-Simpson integrates the P1 products exactly -- the assembled M, S equal the
    exact integrals (M = h/6 [.. 1 4 1 ..], ends h/3; S = 1/h [.. -1 2 -1 ..], ends 1/h) and S 1 = 0."""
    v = np.linspace(-1.0, 1.0, 9)
    h = v[1] - v[0]
    M, S = fem_matrices(v)
    Mx = (np.diag(np.r_[1.0, 2.0 * np.ones(7), 1.0]) * 2 + np.eye(9, k=1) + np.eye(9, k=-1)) * h / 6
    Sx = (np.diag(np.r_[1.0, 2.0 * np.ones(7), 1.0]) - np.eye(9, k=1) - np.eye(9, k=-1)) / h
    assert np.abs(M - Mx).max() < 1e-15 and np.abs(S - Sx).max() < 1e-13
    assert np.abs(S @ np.ones(9)).max() < 1e-13
    # exactness: int phi_i phi_j against a fine midpoint rule
    xs = np.linspace(-1, 1, 200001)
    phi = np.maximum(0.0, 1.0 - np.abs(xs[None, :] - v[:, None]) / h)
    Mq = (phi[:, None, :] * phi[None, :, :]).sum(-1) * (xs[1] - xs[0])
    assert np.abs(M - Mq).max() < 1e-5


@pytest.mark.parametrize("seed", [3, 4])
def test_fem_monodomain_matches_quadrature_brute_force(orc, seed):
    """Steps 1-2 with Neumann ends: oracle == dense Simpson-assembled solve + interpolation at the
    characteristic foot, at every recorded w^{n+1/2} line and at u(T)."""
    g = ki.Grid(6, 10, 5, 1.0, 0.2)
    prob = ki.fem_problem(g, u0_seed=seed)
    us, ws = dense_fem_window(prob, 0, g.nv)
    UT, rec = orc.monodomain(prob, [0, 3, 10])
    scale = np.abs(us).max()
    assert np.abs(UT - us[-1]).max() < 1e-12 * scale
    for i, j in enumerate([0, 3, 10]):
        assert np.abs(rec[i] - ws[:, j]).max() < 1e-12 * scale


@pytest.mark.parametrize("lk,rk,q", [("robin", "robin", None), ("dirichlet", "robin", None), ("robin", "phys", None),
                                     ("dirichlet", "dirichlet", None), ("phys", "dirichlet", None),
                                     ("robin", "robin", 0.45)])
def test_fem_subdomain_window_matches_brute_force(orc, lk, rk, q):
    """SWR1/SWR3 with the paper's scheme: weak Robin ends ((q - d_v) left, (p + d_v) right,
    P:550), strong Dirichlet ends, Neumann physical ends, arbitrary traces == brute force."""
    g = ki.Grid(6, 16, 5, 1.0, 0.2)
    prob = ki.fem_problem(g, u0_seed=5)
    rng = np.random.default_rng(6)
    gL = rng.normal(size=(g.nt, g.nx))
    gR = rng.normal(size=(g.nt, g.nx))
    lo, hi, p = 3, 12, 1.7
    kind = {"phys": END_PHYS, "dirichlet": END_DIRICHLET, "robin": END_ROBIN}
    uT, _, _, rec = orc.window(prob, lo, hi, kind[lk], kind[rk], p, gL, gR, "robin", rec_nodes=(lo, lo + 1, hi), q=q)
    us, ws = dense_fem_window(prob, lo, hi, lk, rk, p, gL, gR, q=q)
    scale = np.abs(us).max()
    assert np.abs(uT - us[-1]).max() < 1e-12 * scale
    for i, j in enumerate((lo, lo + 1, hi)):
        assert np.abs(rec[i] - ws[:, j - lo]).max() < 1e-12 * scale


@pytest.mark.parametrize("k", [1, 3, 8])
def test_fem_cosine_mode_closed_form(orc, k):
    """x-constant data in the k-th Neumann cosine mode v_j -> cos(k pi j / N_v) is an eigenvector of both the
    P1 mass and stiffness matrices (eigenvalues h (4 + 2c)/6 and 2 (1 - c)/h times diag(1/2, 1, .., 1, 1/2),
    c = cos(k pi / N_v)); Step 2 leaves it unchanged, so u^n = mu^n u^0 with
    mu = (h (4 + 2c) / (6 tau)) / (h (4 + 2c) / (6 tau) + 2 (1 - c) / h), tau = dt / 2."""
    g = ki.Grid(8, 16, 7, 1.0, 0.3)
    prob = ki.fem_problem(g)
    j = np.arange(g.nv + 1)
    prob.u0v = np.cos(k * math.pi * j / g.nv)[None, :].copy()
    prob.u0x = np.ones((1, g.nx))
    prob.data = "cosine"
    UT, _ = orc.monodomain(prob)
    h, tau = 2.0 / g.nv, 0.5 * g.t_final / g.nt
    c = math.cos(k * math.pi / g.nv)
    lm, ls = h * (4 + 2 * c) / 6, 2 * (1 - c) / h
    mu = (lm / tau) / (lm / tau + ls)
    expect = mu ** g.nt * prob.u0_dense()
    assert np.abs(UT - expect).max() < 1e-13


def test_fem_mass_is_conserved(orc):
    """Neumann ends (S 1 = 0, S symmetric) and periodic x: Step 1 keeps 1^T M u, Step 2 keeps every row sum,
    so sum_j (M 1)_j sum_m u_jm (trapezoid weights h/2, h, .., h, h/2) is invariant."""
    g = ki.Grid(12, 20, 9, 1.0, 0.3)
    prob = ki.fem_problem(g, u0_seed=8)
    UT, _ = orc.monodomain(prob)
    wts = np.full(g.nv + 1, 2.0 / g.nv)
    wts[[0, -1]] *= 0.5
    m0 = wts @ prob.u0_dense().sum(axis=1)
    assert abs(wts @ UT.sum(axis=1) - m0) < 1e-13 * np.abs(prob.u0_dense()).sum()


def test_fem_maximum_principle(orc):
    """tau / h_v^2 >= 1/3: (M/tau + S) is an M-matrix and (M/tau + S)^{-1} M/tau has non-negative entries and
    unit row sums; Step 2 is a convex combination (CFL <= 1): max |u^n| never grows (an upwind/downwind
    mix-up or a wrong weight breaks it)."""
    g = ki.Grid(16, 20, 40, 1.0, 0.8)
    prob = ki.fem_problem(g, u0_seed=9)
    u0 = prob.u0_dense()
    UT, rec = orc.monodomain(prob, list(range(0, g.nv + 1, 4)))
    assert np.abs(UT).max() <= np.abs(u0).max() * (1 + 1e-14)
    assert np.abs(rec).max() <= np.abs(u0).max() * (1 + 1e-14)
    assert np.abs(UT).max() < 0.9 * np.abs(u0).max()  # and it really diffuses


@pytest.mark.parametrize("kind,p,ov,S,q", [("robin", 1.3, 0, 2, None), ("robin", 2.0, 0, 3, None),
                                           ("robin", 0.7, 3, 2, None), ("dirichlet", 0.0, 2, 2, None),
                                           ("dirichlet", 0.0, 3, 3, None), ("robin", 1.3, 0, 2, 0.35),
                                           ("robin", 0.6, 1, 3, 2.4)])
def test_fem_swr_fixed_point_is_monodomain(orc, kind, p, ov, S, q):
    """the fixed point of the SWR trace map is the monodomain solution -- holds for the paper's scheme
    only with the flux-consistent FEM trace (reading F4): the sender's half-row residual."""
    g = ki.Grid(4, 12, 3, 1.0, 0.1)
    prob = ki.fem_problem(g, u0_seed=10)
    gstar, gnext, slabs, lo, hi, _ = _probe_fixed_point(orc, prob, kind, p, ov, S, q=q)
    assert np.abs(gnext - gstar).max() < 1e-10 * np.abs(gstar).max()
    UT, _ = orc.monodomain(prob)
    for s in range(S):
        assert np.abs(slabs[s] - UT[lo[s]:hi[s] + 1]).max() < 1e-11 * np.abs(UT).max()


def test_fem_jacobi_converges_to_monodomain(orc):
    """Theorems ConvergenceClassical / ConvergenceRobin for the paper's scheme: the Jacobi
    iterates reach the monodomain solution to round-off."""
    g = ki.Grid(16, 40, 20, 1.0, 0.2)
    prob = ki.fem_problem(g, u0_seed=12)
    r = orc.swr(prob, "robin", 6.0, 0, 4, 60)
    assert r["err_T"][-1] < 1e-12 * np.abs(r["UT"]).max()
    assert r["err_if"][-1] < 1e-11 * np.abs(r["UT"]).max()
    assert np.abs(r["uT"] - r["UT"]).max() < 1e-12 * np.abs(r["UT"]).max()


def _paper_table1(orc, j, ov, kind, p, q, kmax, eps=1e-6, seed=1000):
    """The paper's experiment with its own stopping rule (eq. 'error'):
    SWR1-SWR4 (serial) on two subdomains of [-1, 1], f = u0 = 0, random lambda_1^0 ~ U(-1, 1),
    stop when max over t, x and the closed overlap [alpha, beta] of |u1 - u2| < eps."""
    g = ki.paper_grid(j)
    prob = ki.fem_problem(g)
    lo, hi = orc.subdomains(g.nv, 2, ov)
    lam1 = np.random.default_rng(seed + j).uniform(-1.0, 1.0, size=(g.nt, g.nx))
    et = END_ROBIN if kind == "robin" else END_DIRICHLET
    alpha, beta = int(lo[1]), int(hi[0])
    nodes = list(range(alpha, beta + 1))
    hist, size = [], []  # ||u1 - u2|| on the overlap; max |u_s| there (the exact solution is 0)
    for k in range(1, kmax + 1):
        _, _, lam2, r1 = orc.window(prob, 0, beta, END_PHYS, et, p, None, lam1, kind, -1, alpha, nodes, q=q)
        _, lam1, _, r2 = orc.window(prob, alpha, g.nv, et, END_PHYS, p, lam2, None, kind, beta, -1, nodes, q=q)
        hist.append(float(np.abs(r1 - r2).max()))
        size.append(float(max(np.abs(r1).max(), np.abs(r2).max())))
        if hist[-1] < eps:
            return k, hist, size
    return None, hist, size


def test_fem_reproduces_paper_table1_level0(orc):
    """Table 1, j = 0: with the paper's discretisation and stopping rule the optimized methods
    converge in the paper's iteration counts to within +-2 (random lambda^0 differs; the paper's counts
    are OSWR(p) 9 / 12 and OSWR(p,q) 9 / 11 with / without overlap), CSWR needs far more with overlap
    (paper: 70; ours 86) and stalls without."""
    with open(os.path.join(GOLDEN, "paper_table1.json")) as fh:
        gold = json.load(fh)
    for name, (p, q) in gold["params"].items():
        for ov, key in ((3, "overlapping_L3"), (0, "non_overlapping")):
            it, hist, _ = _paper_table1(orc, 0, ov, "robin", p, q, kmax=30, eps=gold["eps"])
            assert it is not None and abs(it - gold[key][name][0]) <= 2, (name, ov, it, hist)
    it, hist, _ = _paper_table1(orc, 0, 3, "dirichlet", 0.0, None, kmax=150, eps=gold["eps"])
    assert it is not None and 50 <= it <= 110, it  # paper: 70
    # without overlap the overlap is the single interface node where both Dirichlet values are the same
    # trace, so u1 - u2 vanishes identically; the iterates themselves do not approach the solution 0
    _, _, size = _paper_table1(orc, 0, 0, "dirichlet", 0.0, None, kmax=25, eps=0.0)
    assert size[-1] > 0.5 * size[9] > 1e-3


@pytest.mark.parametrize("kind,p,q,ov", [("robin", 11.0, 2.5, 3), ("robin", 4.23, None, 0), ("dirichlet", 0.0, None, 3)])
def test_overlap_error_matches_direct_loop(orc, kind, p, q, ov):
    """err_ov of the oracle's SWR driver (Gauss-Seidel, random lambda_1^0) == the paper's quantity computed
    directly from SWR1-SWR4 window by window (eq. 'error')."""
    g = ki.Grid(50, 100, 40, 1.0, 0.4)
    seed = 77
    lam1 = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(g.nt, g.nx))
    prob = ki.fem_problem(g)
    r = orc.swr(prob, kind, p, ov, 2, 5, q=q, schedule="gauss_seidel",
                init_traces=(lam1[None], np.zeros((1, g.nt, g.nx))))
    lo, hi = orc.subdomains(g.nv, 2, ov)
    et = END_ROBIN if kind == "robin" else END_DIRICHLET
    alpha, beta = int(lo[1]), int(hi[0])
    nodes = list(range(alpha, beta + 1))
    lam = lam1
    for k in range(5):
        _, _, lam2, r1 = orc.window(prob, 0, beta, END_PHYS, et, p, None, lam, kind, -1, alpha, nodes, q=q)
        _, lam, _, r2 = orc.window(prob, alpha, g.nv, et, END_PHYS, p, lam2, None, kind, beta, -1, nodes, q=q)
        assert abs(r["err_ov"][k] - np.abs(r1 - r2).max()) <= 1e-14 * max(1.0, r["err_ov"][0]), k

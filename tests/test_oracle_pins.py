"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage / property it pins.  None of them re-types the
oracle's formulas: they compare against closed forms (the manufactured
solution), global dense assemblies solved by LAPACK, an independent mode-
reduced implementation, conservation laws, the discrete maximum principle, the
algebraic fixed point of the iteration, and the paper's qualitative claims.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import kfp_inputs as ki
from oracle import END_DIRICHLET, END_PHYS, END_ROBIN
from oracle.dense import dense_monodomain, dense_window
from oracle.modal import modal_swr, realize

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _exact_mms(g, t):
    x, v = g.x_nodes(), g.v_nodes()
    return math.exp(-t) * np.sin(2 * np.pi * x)[None, :] * (g.vmax ** 2 - v ** 2)[:, None]


# --------------------------------------------------------------------------
# O1: one window of the monodomain scheme


@pytest.mark.parametrize("data", ["mms", "random"])
def test_monodomain_matches_dense_space_time_solve(orc, data):
    """O1: step-by-step Thomas marching == global dense space-time LU."""
    g = ki.Grid(5, 10, 4, 4.0, 0.02)
    prob = ki.mms_problem(g) if data == "mms" else ki.random_forcing_problem(g)
    if data == "random":  # give the random case a non-zero initial value too
        rng = np.random.default_rng(7)
        prob.u0v = rng.normal(size=(1, g.nv + 1))
        prob.u0x = rng.normal(size=(1, g.nx))
    U = dense_monodomain(prob)
    UT, rec = orc.monodomain(prob, [1, 4, 9])
    assert np.abs(UT - U[-1]).max() < 1e-12 * max(1.0, np.abs(U).max())
    for i, j in enumerate([1, 4, 9]):
        assert np.abs(rec[i] - U[1:, j]).max() < 1e-12 * max(1.0, np.abs(U).max())


@pytest.mark.parametrize("lk,rk,q", [("robin", "robin", None), ("dirichlet", "robin", None), ("robin", "phys", None),
                                     ("dirichlet", "dirichlet", None), ("phys", "dirichlet", None),
                                     ("robin", "robin", 0.45)])
def test_subdomain_window_matches_dense(orc, lk, rk, q):
    """O2: Dirichlet / Robin end rows with arbitrary traces == dense LU;
    q != p: the two-sided rows of OSWR(p,q) (left end q, right end p)."""
    g = ki.Grid(6, 16, 5, 4.0, 0.03)
    prob = ki.mms_problem(g)
    rng = np.random.default_rng(3)
    gL = rng.normal(size=(g.nt, g.nx))
    gR = rng.normal(size=(g.nt, g.nx))
    lo, hi, p = 3, 12, 1.7
    code = {"phys": END_PHYS, "dirichlet": END_DIRICHLET, "robin": END_ROBIN}
    uT, _, _, rec = orc.window(prob, lo, hi, code[lk], code[rk], p, gL, gR, "dirichlet", rec_nodes=[lo, hi, 7], q=q)
    D = dense_window(prob, lo, hi, lk, rk, p, gL, gR, q=q)
    scale = np.abs(D).max()
    assert np.abs(uT - D[-1]).max() < 1e-12 * scale
    for i, j in enumerate([lo, hi, 7]):
        assert np.abs(rec[i] - D[1:, j - lo]).max() < 1e-12 * scale


def test_mms_first_order_in_joint_refinement(orc):
    """Closed form (BJ north_star: manufactured solution, first-order convergence).

    Joint refinement of (N_x, N_t) at fixed CFL halves ||U - u||_inf; the v
    discretisation is exact for the quadratic-in-v solution."""
    errs = []
    for lvl in range(4):
        g = ki.Grid(16 * 2 ** lvl, 16, 25 * 2 ** lvl, 4.0, 0.25)
        UT, _ = orc.monodomain(ki.mms_problem(g))
        errs.append(np.abs(UT - _exact_mms(g, g.t_final)).max())
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(1.8 < r < 2.1 for r in ratios), (errs, ratios)
    assert ratios[-1] > ratios[0]  # approaching 2 from below


def test_mms_error_independent_of_nv(orc):
    """Centred 3-point v-diffusion is exact on quadratics (W(v) = Vmax^2 - v^2): refining N_v alone
    leaves the error unchanged up to O(h_x + dt) cross terms."""
    errs = []
    for nv in (16, 32, 64, 128):
        g = ki.Grid(64, nv, 100, 4.0, 0.25)
        UT, _ = orc.monodomain(ki.mms_problem(g))
        errs.append(np.abs(UT - _exact_mms(g, g.t_final)).max())
    assert max(errs) / min(errs) < 1.01, errs


def test_x_mean_obeys_pure_v_heat_equation(orc):
    """Conservation: periodic upwind transport preserves sum_m u, so the
    x-mean of the scheme must follow the 1-D backward-Euler heat equation in v alone."""
    g = ki.Grid(8, 12, 6, 2.0, 0.05)
    prob = ki.random_forcing_problem(g)
    rng = np.random.default_rng(11)
    prob.u0v = np.abs(rng.normal(size=(1, g.nv + 1)))
    prob.u0x = np.abs(rng.normal(size=(1, g.nx)))
    UT, _ = orc.monodomain(prob)
    hv, dt = 2 * g.vmax / g.nv, g.t_final / g.nt
    a = dt / hv ** 2
    n = g.nv - 1
    A = (1 + 2 * a) * np.eye(n) - a * np.eye(n, k=1) - a * np.eye(n, k=-1)
    w = prob.u0_dense().mean(axis=1)[1:-1]
    for k in range(1, g.nt + 1):
        w = np.linalg.solve(A, w + dt * prob.f_dense(k).mean(axis=1)[1:-1])
    assert np.abs(UT.mean(axis=1)[1:-1] - w).max() < 1e-13 * np.abs(w).max()


# --------------------------------------------------------------------------
# O2-O4: the iteration


def _probe_fixed_point(orc, prob, kind, p, ov, S, q=None):
    """Dense probing of the affine one-iteration trace map g -> A g + b."""
    g = prob.grid
    lo, hi = orc.subdomains(g.nv, S, ov)
    et = END_ROBIN if kind == "robin" else END_DIRICHLET
    TR = g.nt * g.nx

    def iterate(vec):
        toL = vec[: (S - 1) * TR].reshape(S - 1, g.nt, g.nx)
        toR = vec[(S - 1) * TR:].reshape(S - 1, g.nt, g.nx)
        oL, oR = np.zeros_like(toL), np.zeros_like(toR)
        slabs = []
        for s in range(S):
            uT, sL, sR, _ = orc.window(prob, int(lo[s]), int(hi[s]), END_PHYS if s == 0 else et,
                                       END_PHYS if s == S - 1 else et, p,
                                       toR[s - 1] if s > 0 else None, toL[s] if s < S - 1 else None, kind,
                                       int(hi[s - 1]) if s > 0 else -1, int(lo[s + 1]) if s < S - 1 else -1, q=q)
            if s > 0:
                oL[s - 1] = sL
            if s < S - 1:
                oR[s] = sR
            slabs.append(uT)
        return np.concatenate([oL.ravel(), oR.ravel()]), slabs

    dim = 2 * (S - 1) * TR
    b, _ = iterate(np.zeros(dim))
    A = np.zeros((dim, dim))
    for i in range(dim):
        e = np.zeros(dim)
        e[i] = 1.0
        A[:, i] = iterate(e)[0] - b
    gstar = np.linalg.solve(np.eye(dim) - A, b)
    gnext, slabs = iterate(gstar)
    return gstar, gnext, slabs, lo, hi, A


@pytest.mark.parametrize("kind,p,ov,S,q", [("robin", 1.3, 0, 2, None), ("robin", 2.0, 0, 3, None),
                                           ("robin", 0.7, 2, 2, None), ("dirichlet", 0.0, 2, 2, None),
                                           ("dirichlet", 0.0, 3, 3, None),
                                           ("robin", 1.3, 0, 2, 0.35), ("robin", 0.6, 1, 3, 2.4)])
def test_swr_fixed_point_is_monodomain(orc, kind, p, ov, S, q):
    """P:57 / BJ north_star: the SWR fixed point is the monodomain discrete solution.

    The fixed point of the exact affine trace map is found by a dense solve (no
    iteration), then one pass with it must reproduce U on every subdomain.  A
    transmission row or trace formula that is not flux-consistent fails here
    (SURVEY.md §7 hard part 1: a 2-point trace plateaus at 0.12)."""
    g = ki.Grid(4, 12, 3, 4.0, 0.02)
    prob = ki.mms_problem(g)
    gstar, gnext, slabs, lo, hi, _ = _probe_fixed_point(orc, prob, kind, p, ov, S, q=q)
    assert np.abs(gnext - gstar).max() < 1e-10 * np.abs(gstar).max()
    UT, _ = orc.monodomain(prob)
    for s in range(S):
        assert np.abs(slabs[s] - UT[lo[s]:hi[s] + 1]).max() < 1e-11 * np.abs(UT).max()


def test_swr_iterates_converge_to_monodomain(orc):
    """P:57, Theorems ConvergenceClassical / ConvergenceRobin: iterates converge to u (here: to the
    discrete monodomain solution, BJ north_star 'to 1e-12')."""
    run = ki.scaled(ki.config("c1"), nx=32, nv=64, nt=100, K=40)
    prob = ki.make_problem(run)
    r = orc.swr(prob, "dirichlet", 0.0, 8, 2, 40)
    assert r["err_T"][-1] < 1e-12 * np.abs(r["UT"]).max()
    assert r["err_if"][-1] < 1e-12 * np.abs(r["UT"]).max()
    assert np.abs(r["uT"] - r["UT"]).max() < 1e-12 * np.abs(r["UT"]).max()
    run = ki.scaled(ki.config("c0"), nt=40, K=160)
    r = orc.swr(ki.make_problem(run), "robin", 1.0, 0, 2, 160)
    assert r["err_T"][-1] < 1e-11 * np.abs(r["UT"]).max()


def test_dirichlet_error_monotone_and_equals_global_max(orc):
    """Step 1 of Theorem ConvergenceClassical (max principle): for CSWR the interface error
    bounds the subdomain error, so err_if is non-increasing and >= err_T."""
    run = ki.scaled(ki.config("c1"), nx=32, nv=64, nt=200, K=12)
    r = orc.swr(ki.make_problem(run), "dirichlet", 0.0, 4, 4, 12)
    e = r["err_if"]
    assert np.all(np.diff(e) <= 1e-14 * e[0]), e
    assert np.all(r["err_T"] <= e + 1e-13 * e[0])  # up to round-off at the floor


def test_maximum_principle_and_monotone_iterates(orc):
    """Discrete maximum principle on BASELINE configs[4]-shaped data: f >= 0, u0 = 0,
    zero initial traces => 0 <= u^{k-1} <= u^k <= U pointwise."""
    run = ki.scaled(ki.config("c4"), nx=32, nv=128, nt=60, K=6, t_final=0.01)
    run = run.with_(n_sub=8)
    prob = ki.make_problem(run)
    assert (prob.fx >= 0).all() and (prob.fv >= 0).all()
    prev = None
    for K in range(1, 6):
        r = orc.swr(prob, "dirichlet", 0.0, 4, 8, K)
        cur = np.concatenate([s.ravel() for s in r["uT_sub"]])
        assert cur.min() >= 0.0
        U = np.concatenate([r["UT"][l:h + 1].ravel() for l, h in zip(r["lo"], r["hi"])])
        assert (cur <= U + 1e-14).all()
        if prev is not None:
            assert (prev <= cur + 1e-14).all()
        prev = cur


def test_optimized_converges_without_overlap_classical_does_not(orc):
    """P:75 and P:535-537, Table 1: OSWR converges with no overlap, CSWR does not."""
    run = ki.scaled(ki.config("c0"), nt=40, K=30)
    prob = ki.make_problem(run)
    rob = orc.swr(prob, "robin", 1.0, 0, 2, 30)
    dir0 = orc.swr(prob, "dirichlet", 0.0, 0, 2, 30)
    assert rob["err_T"][-1] < 1e-3 * rob["err_T"][0]
    assert dir0["err_T"][-1] > 0.5 * dir0["err_T"][0]


def test_optimized_needs_fewer_iterations_than_classical(orc):
    """P:75, P:655-657 (Table 1): with the same overlap, OSWR(p) reaches a tolerance in fewer iterations."""
    run = ki.scaled(ki.config("c1"), nx=32, nv=64, nt=200, K=40, t_final=0.5)
    prob = ki.make_problem(run)
    d = orc.swr(prob, "dirichlet", 0.0, 2, 2, 40)
    r = orc.swr(prob, "robin", 4.0, 2, 2, 40)
    tol = 1e-6 * d["err_T"][0]
    it = lambda e: int(np.argmax(e < tol)) if (e < tol).any() else 10 ** 9
    assert it(r["err_if"]) < it(d["err_if"])


def test_linearity(orc):
    """The scheme is linear: solution(f1 + 2 f2) = solution(f1) + 2 solution(f2)."""
    g = ki.Grid(16, 32, 20, 4.0, 0.05)
    p1 = ki.mms_problem(g)
    p2 = ki.random_forcing_problem(g)
    both = ki.Problem(g, np.concatenate([p1.ft, p2.ft]), np.concatenate([p1.fv, 2 * p2.fv]),
                      np.concatenate([p1.fx, p2.fx]), p1.u0v, p1.u0x)
    r1 = orc.swr(p1, "robin", 2.0, 0, 4, 3)
    r2 = orc.swr(p2, "robin", 2.0, 0, 4, 3)
    rb = orc.swr(both, "robin", 2.0, 0, 4, 3)
    assert np.abs(rb["uT"] - (r1["uT"] + 2 * r2["uT"])).max() < 1e-12 * np.abs(rb["uT"]).max()


def test_mms_point_antisymmetry(orc):
    """(x, v) -> (-x, -v) maps the MMS data to minus themselves and the scheme (upwind by sign(v),
    symmetric split at v=0, p = q) onto itself, so the discrete monodomain solution is odd and the
    two subdomain iterates are reflections of each other.  The tolerance
    covers the rounding of sin(2 pi m/N_x) vs -sin(2 pi (N_x-m)/N_x) in the input tables."""
    run = ki.scaled(ki.config("c0"), nt=50, K=5)
    r = orc.swr(ki.make_problem(run), "robin", 1.0, 0, 2, 5)
    nx = run.grid.nx
    refl = lambda a: a[::-1, (-np.arange(nx)) % nx]
    scale = np.abs(r["UT"]).max()
    assert np.abs(r["UT"] + refl(r["UT"])).max() < 1e-11 * scale
    assert np.abs(r["uT_sub"][0] + refl(r["uT_sub"][1])).max() < 1e-11 * scale


# --------------------------------------------------------------------------
# the mode-reduced oracle and the survey's scratch histories


@pytest.mark.parametrize("name", ["c0", "c1", "c3"])
def test_mode_reduced_oracle_agrees_with_direct(orc, name):
    """Fourier-in-x reduction: the complex 1-D recurrence reproduces the 2-D oracle."""
    run = ki.config(name)
    if name == "c1":
        run = ki.scaled(run, nt=250, K=20)
    if name == "c3":  # same structure (S = 8 Robin, p = 8, no overlap), reduced grid
        run = ki.scaled(run, nx=32, nv=128, nt=50, K=6)
    r = orc.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K)
    m = modal_swr(run.grid, run.kind, run.p, run.overlap, run.n_sub, run.K)
    for e in ("err_T", "err_if"):
        assert np.abs(m[e] - r[e]).max() < 1e-12 * r[e].max()
    for s in range(run.n_sub):
        assert np.abs(realize(m["c_sub"][s], run.grid.nx) - r["uT_sub"][s]).max() < 1e-12 * np.abs(r["UT"]).max()


def test_survey_scratch_histories_c0(orc):
    """Cross-check of the readings against the survey's independent scratch model (tests/golden/
    survey_scratch_c0.json, values copied from SURVEY.md §8(c) 'Survey-time scratch histories')."""
    with open(os.path.join(GOLDEN, "survey_scratch_c0.json")) as fh:
        gold = json.load(fh)
    run = ki.config("c0")
    r = orc.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K)
    assert abs(np.abs(r["UT"]).max() - gold["max_abs_UT"]) < 1e-4 * gold["max_abs_UT"]
    for k, (eT, eI) in gold["history"].items():
        k = int(k)
        assert abs(r["err_T"][k - 1] - eT) <= 1.5e-4 * eT
        assert abs(r["err_if"][k - 1] - eI) <= 1.5e-4 * eI


def test_two_sided_beats_one_sided(orc):
    """Table 1 ordering: optimized two-sided OSWR(p, q) converges faster than the best
    one-sided OSWR(p).  On the c0 problem cut to 50 steps, the best (p, q) of a 9 x 9 grid
    (p, q in 2 .. 32, ratio sqrt 2) reaches a clearly smaller interface error after K = 12 iterations
    than the best p of the same grid (measured 1.7e-3 at (11.3, 8) vs 3.5e-3 at p = 8), and p = q
    reproduces one-sided OSWR(p) exactly."""
    run = ki.scaled(ki.config("c0"), nt=50, K=12)
    prob = ki.make_problem(run)
    ps = list(np.geomspace(2.0, 32.0, 9))
    one = {p: orc.swr(prob, "robin", p, 0, 2, run.K)["err_if"][-1] for p in ps}
    two = {(p, q): orc.swr(prob, "robin", p, 0, 2, run.K, q=q)["err_if"][-1] for p in ps for q in ps}
    assert all(two[(p, p)] == one[p] for p in ps)
    assert min(two.values()) < 0.7 * min(one.values()), (min(one.values()), min(two.values()))


@pytest.mark.parametrize("kind,p,ov", [("robin", 2.0, 0), ("dirichlet", 0.0, 4)])
def test_gauss_seidel_is_interleaved_jacobi(orc, kind, p, ov):
    """The paper's serial SWR1-SWR4 against its parallel Remark: for two
    subdomains from zero traces, Gauss-Seidel iterate k of subdomain 0 is Jacobi iterate 2k-1 and
    of subdomain 1 Jacobi iterate 2k -- the Jacobi sequence interleaves two Gauss-Seidel sequences.
    Same arithmetic on both sides, so the identity is bitwise."""
    run = ki.scaled(ki.config("c0"), nt=30, K=5)
    prob = ki.make_problem(run)
    K = 5
    gs = orc.swr(prob, kind, p, ov, 2, K, schedule="gauss_seidel")
    assert np.array_equal(gs["uT_sub"][0], orc.swr(prob, kind, p, ov, 2, 2 * K - 1)["uT_sub"][0])
    assert np.array_equal(gs["uT_sub"][1], orc.swr(prob, kind, p, ov, 2, 2 * K)["uT_sub"][1])


def test_gauss_seidel_converges_to_monodomain(orc):
    """Gauss-Seidel has the same fixed point (the monodomain solution) and, per iteration,
    converges at least as fast as Jacobi on a 4-subdomain Robin problem (err_if at every k >= 5)."""
    run = ki.scaled(ki.config("c1"), nx=32, nv=64, nt=100, K=30)
    prob = ki.make_problem(run)
    gs = orc.swr(prob, "robin", 4.0, 0, 4, 30, schedule="gauss_seidel")
    ja = orc.swr(prob, "robin", 4.0, 0, 4, 30)
    assert np.all(gs["err_if"][4:] <= ja["err_if"][4:] * (1 + 1e-12))
    gs = orc.swr(prob, "robin", 4.0, 0, 4, 160, schedule="gauss_seidel")
    assert gs["err_T"][-1] < 1e-11 * np.abs(gs["UT"]).max(), gs["err_T"][-1]


def _check_scratch(gold, UT_max, err_exact, err_T, err_if):
    assert abs(UT_max - gold["max_abs_UT"]) <= 1.5e-4 * gold["max_abs_UT"]
    assert abs(err_exact - gold["err_exact_T"]) <= 1.5e-3 * gold["err_exact_T"]
    for k, (eT, eI) in gold["history"].items():
        k = int(k)
        assert abs(err_T[k - 1] - eT) <= 1.5e-4 * eT, (k, err_T[k - 1], eT)
        assert abs(err_if[k - 1] - eI) <= 1.5e-4 * eI, (k, err_if[k - 1], eI)


def _gold(name):
    with open(os.path.join(GOLDEN, f"survey_scratch_{name}.json")) as fh:
        return json.load(fh)


def test_subdomain_ranges_match_survey(orc):
    """Overlap placement (R9; O2 of SURVEY.md §8(c)) against the survey's explicit node ranges:
    c1 [0,132] / [124,256]; c3 [2048 s, 2048 (s+1)]; c4 [1024 s - 2, 1024 (s+1) + 2] clipped to
    [0, 32768] -- and, for an odd overlap (where floor and ceil differ), R9's text: the left
    subdomain extends to c + ceil(ov/2), the right one starts at c - floor(ov/2).  The mode-reduced
    oracle's own decomposition must agree."""
    from oracle.modal import _subdomains

    gold = _gold("c1")["node_ranges"]
    cases = [((256, 2, 8), (gold["lo"], gold["hi"])),
             ((16384, 8, 0), ([2048 * s for s in range(8)], [2048 * (s + 1) for s in range(8)])),
             ((32768, 32, 4), ([max(0, 1024 * s - 2) for s in range(32)],
                               [min(32768, 1024 * (s + 1) + 2) for s in range(32)])),
             ((64, 2, 3), ([0, 31], [34, 64])),
             ((60, 3, 5), ([0, 18, 38], [23, 43, 60]))]
    for (nv, S, ov), (lo, hi) in cases:
        olo, ohi = orc.subdomains(nv, S, ov)
        assert list(olo) == list(lo) and list(ohi) == list(hi), (nv, S, ov, olo, ohi)
        mlo, mhi = _subdomains(nv, S, ov)
        assert mlo == list(lo) and mhi == list(hi)


def test_survey_scratch_histories_c1(orc):
    """c1 (Dirichlet, overlap 8: exercises R9's placement and err_if at Dirichlet interface ends) on the
    C oracle at full size, against the survey's independent scratch model
    (tests/golden/survey_scratch_c1.json)."""
    run = ki.config("c1")
    r = orc.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, 10)
    lo, hi = r["lo"], r["hi"]
    assert list(lo) == [0, 124] and list(hi) == [132, 256]
    g = run.grid
    x = np.arange(g.nx) / g.nx
    v = -g.vmax + np.arange(g.nv + 1) * (2 * g.vmax / g.nv)
    u_ex = math.exp(-g.t_final) * np.outer(g.vmax ** 2 - v ** 2, np.sin(2 * np.pi * x))
    _check_scratch(_gold("c1"), np.abs(r["UT"]).max(), np.abs(r["UT"] - u_ex).max(), r["err_T"], r["err_if"])


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_survey_scratch_histories_modal(name):
    """c2 (S = 2 Robin p = 4) and c3 (S = 8 Robin p = 8, K = 15) at full size on the mode-reduced oracle
    (exact for the manufactured data, pinned to the 2-D oracle by test_mode_reduced_oracle_agrees_with_direct),
    against the survey's independent scratch histories (tests/golden/survey_scratch_{c2,c3}.json)."""
    from oracle.modal import max_abs_real

    run = ki.config(name)
    g = run.grid
    m = modal_swr(g, run.kind, run.p, run.overlap, run.n_sub, run.K)
    v = -g.vmax + np.arange(g.nv + 1) * (2 * g.vmax / g.nv)
    c_ex = math.exp(-g.t_final) * (g.vmax ** 2 - v ** 2)
    _check_scratch(_gold(name), max_abs_real(m["C"], g.nx), max_abs_real(m["C"] - c_ex, g.nx), m["err_T"], m["err_if"])


def test_x_translation_equivariance(orc):
    """Every operator of the scheme commutes with x-translation (periodic x, upwind by a column, the v-solve per
    column): rolling the x-tables of f and u0 by k columns rolls the monodomain solution, every
    subdomain iterate and the traces by k columns.  Per-column arithmetic is identical, so the identity is
    bitwise; a transposed or mis-shifted transport stencil breaks it."""
    import dataclasses

    run = ki.scaled(ki.config("c4"), nx=24, nv=48, nt=12, K=3).with_(n_sub=3, overlap=2)
    prob = ki.make_problem(run)
    k = 5
    rolled = dataclasses.replace(prob, fx=np.roll(prob.fx, k, axis=1), u0x=np.roll(prob.u0x, k, axis=1))
    a = orc.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K, want_traces=True)
    b = orc.swr(rolled, run.kind, run.p, run.overlap, run.n_sub, run.K, want_traces=True)
    assert np.array_equal(np.roll(a["UT"], k, axis=1), b["UT"])
    assert np.array_equal(np.roll(a["uT"], k, axis=1), b["uT"])
    assert np.array_equal(np.roll(a["traces"], k, axis=2), b["traces"])
    assert np.array_equal(a["err_T"], b["err_T"]) and np.array_equal(a["err_if"], b["err_if"])
    assert not np.array_equal(a["UT"], b["UT"])  # control: the roll does change the solution

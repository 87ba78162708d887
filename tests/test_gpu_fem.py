"""-m gpu: the split-FEM instantiation of the cluster kernel (the paper's own scheme, P:443-525,
DESIGN.md §3b) through the C-ABI against the oracle's window_fem(), element by element.

Bar: max-abs relative error <= 1e-9 (fp64) per u(T) slab, per trace array and per error-history vector,
as for the IMEX FD scheme (tests/test_gpu_parity.py).  Geometries: ragged x-tiles, one to four
subdomains, Dirichlet / one-sided and two-sided Robin, overlaps 0-3, 33-row chunks and multi-block
columns, the P = 16 path (3201-row monodomain), random initial traces with both schedules, and the
paper's Table 1 meshes at levels 0 and 1.
"""
from __future__ import annotations

import collections
import functools

import numpy as np
import pytest

import kfp_inputs as ki

pytestmark = pytest.mark.gpu
TOL = 1e-9

Case = collections.namedtuple("Case", "grid seed kind p q ov S K schedule lam")

CASES = {
    "robin_S2": Case(ki.Grid(64, 200, 40, 1.0, 0.4), 1, "robin", 4.23, None, 0, 2, 6, "jacobi", False),
    "robin_pq_S3_ragged_ov1": Case(ki.Grid(70, 198, 40, 1.0, 0.4), 2, "robin", 11.0, 2.5, 1, 3, 6, "jacobi", False),
    "dirichlet_ov3": Case(ki.Grid(64, 200, 40, 1.0, 0.4), 3, "dirichlet", 0.0, None, 3, 2, 6, "jacobi", False),
    "dirichlet_ov2_S4": Case(ki.Grid(96, 400, 30, 1.0, 0.3), 4, "dirichlet", 0.0, None, 2, 4, 5, "jacobi", False),
    "dirichlet_ov0": Case(ki.Grid(64, 200, 20, 1.0, 0.2), 4, "dirichlet", 0.0, None, 0, 2, 4, "jacobi", False),
    "robin_ov3_S4": Case(ki.Grid(64, 400, 30, 1.0, 0.3), 5, "robin", 4.23, None, 3, 4, 5, "jacobi", False),
    "chunk33_blocks": Case(ki.Grid(64, 1040, 8, 1.0, 0.08), 6, "robin", 4.0, None, 0, 2, 3, "jacobi", False),
    "chunk33_dirichlet": Case(ki.Grid(96, 1040, 8, 1.0, 0.08), 6, "dirichlet", 0.0, None, 4, 2, 3, "jacobi", False),
    "gs_robin_pq": Case(ki.Grid(64, 300, 30, 1.0, 0.3), 8, "robin", 11.0, 2.5, 3, 3, 5, "gauss_seidel", False),
    "lam_jacobi": Case(ki.Grid(64, 200, 20, 1.0, 0.2), None, "robin", 4.23, None, 3, 2, 5, "jacobi", True),
    "lam_dirichlet_gs": Case(ki.Grid(64, 200, 20, 1.0, 0.2), None, "dirichlet", 0.0, None, 3, 2, 5, "gauss_seidel",
                             True),
    # the paper's Table 1 meshes, its experiment: f = u0 = 0, random lambda^0, SWR1-SWR4
    "paper_j0": Case(ki.paper_grid(0), None, "robin", 11.0, 2.5, 3, 2, 4, "gauss_seidel", True),
    "paper_j1": Case(ki.paper_grid(1), None, "robin", 4.23, None, 0, 2, 3, "gauss_seidel", True),
}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def kfp():
    from paper_1306_4596_b200 import build, kfp as k

    build.build()
    k.load()
    return k


def _lam(c):
    g = c.grid
    rng = np.random.default_rng(2024)
    return (rng.uniform(-1, 1, size=(c.S - 1, g.nt, g.nx)), rng.uniform(-1, 1, size=(c.S - 1, g.nt, g.nx)))


@functools.lru_cache(maxsize=None)
def _oracle(name):
    import oracle

    c = CASES[name]
    prob = ki.fem_problem(c.grid, c.seed)
    return oracle.swr(prob, c.kind, c.p, c.ov, c.S, c.K, want_traces=True, q=c.q, schedule=c.schedule,
                      init_traces=_lam(c) if c.lam else None)


def _gpu(kfp, name):
    c = CASES[name]
    prob = ki.fem_problem(c.grid, c.seed)
    with kfp.Problem(prob) as pb:
        pb.setup(c.kind, c.p, c.ov, c.S, c.K, q=c.q)
        pb.set_schedule(c.schedule)
        pb.reset()
        if c.lam:
            toL, toR = _lam(c)
            for i in range(c.S - 1):
                pb.set_initial_trace(i, 0, toL[i])
                pb.set_initial_trace(i, 1, toR[i])
        pb.iterate(c.K)
        eT, eI = pb.history()
        out = dict(err_T=eT, err_if=eI, uT_sub=[pb.subdomain_uT(s) for s in range(c.S)], UT=pb.monodomain_uT(),
                   traces=sum(([pb.trace(i, 0), pb.trace(i, 1)] for i in range(c.S - 1)), []), plan=pb.plan(),
                   launches=pb.launch_count())
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_fem_parity_vs_oracle(kfp, name):
    g, r = _gpu(kfp, name), _oracle(name)
    assert "fused-tma-cluster-fem" in g["plan"], g["plan"]
    assert rel(g["UT"], r["UT"]) <= TOL, name
    for s, (a, b) in enumerate(zip(g["uT_sub"], r["uT_sub"])):
        assert rel(a, b) <= TOL, (name, s, rel(a, b))
    for i, (a, b) in enumerate(zip(g["traces"], r["traces"])):
        assert rel(a, b) <= TOL, (name, "trace", i, rel(a, b))
    assert rel(g["err_T"], r["err_T"]) <= TOL, (name, g["err_T"], r["err_T"])
    assert rel(g["err_if"], r["err_if"]) <= TOL, (name, g["err_if"], r["err_if"])


@pytest.mark.parametrize("nv,nx", [(3200, 64), (1200, 70)])
def test_fem_monodomain_tall_columns(kfp, nv, nx):
    """Neumann monodomain columns of 3201 rows (P = 16 warps, 7-CTA clusters) and 1201 rows (P = 8), ragged x:
    U(T) against the oracle; one subdomain equals the monodomain bitwise."""
    import oracle

    g = ki.Grid(nx, nv, 6, 1.0, 0.06)
    prob = ki.fem_problem(g, 7)
    UT_ref, _ = oracle.monodomain(prob)
    with kfp.Problem(prob) as pb:
        uT = pb.solve("robin", 1.0, 0, 1, 1)
        UT = pb.monodomain_uT()
        plan = pb.plan()
    assert "fem" in plan, plan
    assert rel(UT, UT_ref) <= TOL
    assert np.array_equal(uT, UT)


def test_fem_batched_sweep_equals_individual(kfp):
    """The batched Robin-parameter sweep (Fig. 1's experiment) with the paper's scheme: every
    replica bitwise equals its individual solve."""
    c = CASES["lam_jacobi"]
    prob = ki.fem_problem(c.grid, 11)
    ps = [1.0, 4.23, 9.0]
    with kfp.Problem(prob) as pb:
        pb.setup_batch("robin", ps, c.ov, c.S, c.K)
        pb.reset()
        pb.iterate(c.K)
        batch = [(pb.batch_history(r), [pb.batch_subdomain_uT(r, s) for s in range(c.S)]) for r in range(len(ps))]
    for r, p in enumerate(ps):
        with kfp.Problem(prob) as pb:
            pb.solve("robin", p, c.ov, c.S, c.K, copy=False)
            hist = pb.history()
            slabs = [pb.subdomain_uT(s) for s in range(c.S)]
        (eT, eI), bs = batch[r]
        assert np.array_equal(eT, hist[0]) and np.array_equal(eI, hist[1]), r
        for a, b in zip(bs, slabs):
            assert np.array_equal(a, b), r


@pytest.mark.parametrize("name", ["robin_S2", "robin_pq_S3_ragged_ov1", "dirichlet_ov3", "robin_ov3_S4",
                                  "gs_robin_pq", "lam_dirichlet_gs", "paper_j0"])
def test_overlap_error_vs_oracle(kfp, name):
    """The paper's convergence quantity max |u_s - u_{s+1}| over the closed overlaps (eq. 'error'),
    recorded by the cluster kernel and reduced on the device, against the oracle's."""
    c = CASES[name]
    prob = ki.fem_problem(c.grid, c.seed)
    with kfp.Problem(prob) as pb:
        pb.setup(c.kind, c.p, c.ov, c.S, c.K, q=c.q)
        pb.set_schedule(c.schedule)
        pb.set_overlap_error(True)
        pb.reset()
        if c.lam:
            toL, toR = _lam(c)
            for i in range(c.S - 1):
                pb.set_initial_trace(i, 0, toL[i])
                pb.set_initial_trace(i, 1, toR[i])
        pb.iterate(c.K)
        eo = pb.overlap_history()
        eT, eI = pb.history()
    r = _oracle(name)
    assert rel(eo, r["err_ov"]) <= TOL, (name, eo, r["err_ov"])
    assert rel(eT, r["err_T"]) <= TOL and rel(eI, r["err_if"]) <= TOL  # the recording changes nothing else


def test_overlap_error_imex_fd(kfp):
    """The same quantity for the IMEX FD scheme (Dirichlet end nodes of CSWR included)."""
    import oracle

    run = ki.scaled(ki.config("c1"), nx=40, nt=100, K=5, name="ov_fd").with_(n_sub=4, overlap=6)
    prob = ki.make_problem(run)
    with kfp.Problem(prob) as pb:
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
        pb.set_overlap_error(True)
        pb.reset()
        pb.iterate(run.K)
        eo = pb.overlap_history()
    r = oracle.swr(prob, run.kind, run.p, run.overlap, run.n_sub, run.K)
    assert rel(eo, r["err_ov"]) <= TOL, (eo, r["err_ov"])


def test_iterate_until_tolerance(kfp):
    """Tolerance stopping: kfp_swr_iterate_until stops at the first iteration whose overlap error is
    below eps -- the same k the oracle's history gives."""
    import oracle

    c = CASES["paper_j0"]
    prob = ki.fem_problem(c.grid, c.seed)
    toL, toR = _lam(c)
    r = oracle.swr(prob, c.kind, c.p, c.ov, c.S, 20, q=c.q, schedule=c.schedule, init_traces=(toL, toR))
    eps = 1e-6
    k_ref = int(np.nonzero(r["err_ov"] < eps)[0][0]) + 1
    with kfp.Problem(prob) as pb:
        pb.setup(c.kind, c.p, c.ov, c.S, 20, q=c.q)
        pb.set_schedule(c.schedule)
        pb.set_overlap_error(True)
        pb.reset()
        for i in range(c.S - 1):
            pb.set_initial_trace(i, 0, toL[i])
            pb.set_initial_trace(i, 1, toR[i])
        k = pb.iterate_until(eps, 20)
        eo = pb.overlap_history()
    assert k == k_ref, (k, k_ref, r["err_ov"])
    assert rel(eo, r["err_ov"][:k]) <= TOL


def test_fem_paper_j4_full_size_properties(kfp):
    """The paper's finest Table 1 mesh (j = 4: 1600 x 3200 cells, 3200 steps) on the GPU, checked by
    properties that hold at any size: the monodomain conserves sum_j (M 1)_j sum_m u_jm exactly (Neumann ends,
    periodic x; pinned on CPU in test_fem_mass_is_conserved) and obeys the maximum principle; the SWR iterates
    (Jacobi, OSWR(11, 2.5), overlap 3) approach it, and the paper's overlap quantity decreases."""
    g = ki.paper_grid(4)
    prob = ki.fem_problem(g, 3)
    u0 = prob.u0_dense()
    with kfp.Problem(prob) as pb:
        UT = pb.monodomain()
        pb.setup("robin", 11.0, 3, 2, 6, q=2.5)
        pb.set_overlap_error(True)
        pb.reset()
        pb.iterate(6)
        eT, eI = pb.history()
        eo = pb.overlap_history()
    wts = np.full(g.nv + 1, 2.0 / g.nv)
    wts[[0, -1]] *= 0.5
    m0, m1 = wts @ u0.sum(axis=1), wts @ UT.sum(axis=1)
    assert abs(m1 - m0) <= 1e-12 * (wts @ np.abs(u0).sum(axis=1)), (m0, m1)
    assert np.abs(UT).max() <= np.abs(u0).max() * (1 + 1e-13)
    assert np.all(np.diff(eo) < 0) and eo[-1] < 0.3 * eo[0], eo  # Jacobi: ~0.7x per iteration here
    assert eI[-1] < 0.3 * eI[0], (eT, eI)

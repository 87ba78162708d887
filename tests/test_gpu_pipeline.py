"""-m gpu: pipelined Jacobi iterations (kfp_swr_set_pipeline) are bitwise the
unpipelined ones -- the same per-tile arithmetic, only the launch schedule changes: slot d of a sweep runs
iteration k0 + d at step L - d, reading trace row L - d of iteration k0 + d - 1 from a ring of buffers --
and the first case is also checked against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import kfp_inputs as ki

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kfp():
    from paper_1306_4596_b200 import build, kfp as k

    build.build()
    k.load()
    return k


RUNS = {
    "c0": ki.config("c0"),
    "c1_K12": ki.config("c1").with_(K=12),
    "ragged_dirichlet_ov": ki.scaled(ki.config("c1"), nx=38, nv=96, nt=200, K=8, name="rd").with_(n_sub=4, overlap=6),
    "oswr_pq_S3": ki.config("c0").with_(name="pq3", p=2.5, q=0.4, K=7, n_sub=4),
    "c4_small": ki.scaled(ki.config("c4"), nx=64, nv=32 * 32, nt=60, K=6, name="c4_small"),
    "fem_paper_j0": ki.Run("fem_j0", ki.paper_grid(0), "random_u0", "robin", 11.0, 3, 2, 7, q=2.5, scheme="split_fem"),
    "fem_dirichlet": ki.Run("fem_d", ki.Grid(64, 200, 40, 1.0, 0.4), "random_u0", "dirichlet", 0.0, 2, 4, 6,
                            scheme="split_fem"),
}


def _solve(kfp, run, depth, lam=None, schedule="jacobi"):
    with kfp.Problem(ki.make_problem(run)) as pb:
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
        pb.set_schedule(schedule)
        if depth != 1:
            pb.set_pipeline(depth)  # 0: the library's automatic depth
        pb.reset()
        if lam is not None:
            for i in range(run.n_sub - 1):
                pb.set_initial_trace(i, 0, lam[0][i])
                pb.set_initial_trace(i, 1, lam[1][i])
        pb.iterate(run.K)
        eT, eI = pb.history()
        return dict(eT=eT, eI=eI, slabs=[pb.subdomain_uT(s) for s in range(run.n_sub)],
                    traces=[pb.trace(i, d) for i in range(run.n_sub - 1) for d in (0, 1)], launches=pb.launch_count())


@pytest.mark.parametrize("schedule", ["jacobi", "gauss_seidel"])
@pytest.mark.parametrize("name", list(RUNS))
@pytest.mark.parametrize("depth", [2, 3, 64])
def test_pipelined_equals_unpipelined(kfp, name, depth, schedule):
    """Jacobi: slots lag by the iteration offset; Gauss-Seidel (SWR1-SWR4): a wavefront, subdomain s of slot d
    lagging 2 d + s steps."""
    run = RUNS[name]
    a, b = _solve(kfp, run, 1, schedule=schedule), _solve(kfp, run, min(depth, run.K), schedule=schedule)
    assert np.array_equal(a["eT"], b["eT"]) and np.array_equal(a["eI"], b["eI"]), (name, a["eI"], b["eI"])
    for x, y in zip(a["slabs"], b["slabs"]):
        assert np.array_equal(x, y), name
    for x, y in zip(a["traces"], b["traces"]):
        assert np.array_equal(x, y), name


def test_pipelined_random_initial_traces_vs_oracle(kfp):
    """Random lambda^0 through the pipelined path (the ring's slot 0) against the oracle."""
    import oracle

    run = ki.Run("fem_lam", ki.Grid(64, 198, 30, 1.0, 0.3), "zero", "robin", 4.23, 3, 3, 6, scheme="split_fem")
    g = run.grid
    rng = np.random.default_rng(9)
    lam = (rng.uniform(-1, 1, size=(run.n_sub - 1, g.nt, g.nx)), rng.uniform(-1, 1, size=(run.n_sub - 1, g.nt, g.nx)))
    b = _solve(kfp, run, 4, lam)
    r = oracle.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K, init_traces=lam)

    def rel(x, y):
        return float(np.abs(np.asarray(x) - y).max() / np.abs(y).max())

    assert rel(b["eT"], r["err_T"]) <= 1e-9 and rel(b["eI"], r["err_if"]) <= 1e-9
    for x, y in zip(b["slabs"], r["uT_sub"]):
        assert rel(x, y) <= 1e-9


def test_pipeline_launch_count(kfp):
    """One sweep of nt + depth - 1 step launches per group of depth iterations (+ nothing else for IMEX FD)."""
    run = RUNS["c0"]
    a, b = _solve(kfp, run, 1), _solve(kfp, run, run.K)
    g = run.grid
    mono = g.nt  # the monodomain reference at setup
    assert a["launches"] - mono == g.nt * run.K
    assert b["launches"] - mono == g.nt + run.K - 1


def test_pipeline_rejected_combinations(kfp):
    run = RUNS["c0"]
    with kfp.Problem(ki.make_problem(run)) as pb:
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
        pb.set_pipeline(4)
        with pytest.raises(kfp.KfpError):
            pb.set_overlap_error(True)
        with pytest.raises(kfp.KfpError):
            pb.set_pipeline(1)
    with kfp.Problem(ki.make_problem(run)) as pb:
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
        pb.reset()
        pb.iterate(1)
        with pytest.raises(kfp.KfpError):  # only right after setup / reset
            pb.set_pipeline(4)


def test_pipelined_gauss_seidel_random_traces_vs_oracle(kfp):
    """The paper's own experiment shape (SWR1-SWR4, random lambda^0, the split-FEM scheme) through the
    wavefront: against the oracle's Gauss-Seidel."""
    import oracle

    run = ki.Run("fem_gs", ki.Grid(64, 200, 30, 1.0, 0.3), "zero", "robin", 11.0, 3, 2, 6, q=2.5, scheme="split_fem")
    g = run.grid
    rng = np.random.default_rng(13)
    lam = (rng.uniform(-1, 1, size=(1, g.nt, g.nx)), rng.uniform(-1, 1, size=(1, g.nt, g.nx)))
    b = _solve(kfp, run, 6, lam, schedule="gauss_seidel")
    r = oracle.swr(ki.make_problem(run), run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q,
                   schedule="gauss_seidel", init_traces=lam)

    def rel(x, y):
        return float(np.abs(np.asarray(x) - y).max() / np.abs(y).max())

    assert rel(b["eT"], r["err_T"]) <= 1e-9 and rel(b["eI"], r["err_if"]) <= 1e-9
    for x, y in zip(b["slabs"], r["uT_sub"]):
        assert rel(x, y) <= 1e-9


@pytest.mark.parametrize("schedule", ["jacobi", "gauss_seidel"])
def test_pipelined_overlap_error_and_tolerance_stopping(kfp, schedule):
    """The paper's overlap quantity recorded per slot under pipelining is bitwise the unpipelined
    one, and tolerance stopping finds the same first iteration (group-wise: it may run further)."""
    run = ki.Run("fem_j0", ki.paper_grid(0), "zero", "robin", 11.0, 3, 2, 24, q=2.5, scheme="split_fem")
    g = run.grid
    lam = np.random.default_rng(21).uniform(-1, 1, size=(g.nt, g.nx))
    out = {}
    for depth in (1, 5):
        with kfp.Problem(ki.make_problem(run)) as pb:
            pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K, q=run.q)
            pb.set_schedule(schedule)
            pb.set_overlap_error(True)
            if depth > 1:
                pb.set_pipeline(depth)
            pb.reset()
            pb.set_initial_trace(0, 0, lam)
            k = pb.iterate_until(1e-6, run.K)
            out[depth] = (k, pb.overlap_history(), pb.history())
    (k1, eo1, h1), (k5, eo5, h5) = out[1], out[5]
    assert k1 == k5, (k1, k5)
    n = len(eo1)
    assert np.array_equal(eo1, eo5[:n]) and np.array_equal(h1[1], h5[1][:n])


@pytest.mark.parametrize("schedule", ["jacobi", "gauss_seidel"])
def test_pipelined_batched_sweep_equals_unpipelined(kfp, schedule):
    """A batched Robin-parameter sweep (replicas with their own (p, q)) through the pipeline, with overlap
    recording: every replica's err_T, err_if, err_ov and slabs bitwise the unpipelined batch's."""
    run = ki.Run("fem_b", ki.Grid(64, 200, 24, 1.0, 0.24), "zero", "robin", 4.0, 3, 2, 7, scheme="split_fem")
    g = run.grid
    lam = np.random.default_rng(31).uniform(-1, 1, size=(g.nt, g.nx))
    ps, qs = [1.0, 4.23, 11.0], [1.0, 4.23, 2.5]
    res = {}
    for depth in (1, 4):
        with kfp.Problem(ki.make_problem(run)) as pb:
            pb.setup_batch("robin", ps, run.overlap, run.n_sub, run.K, qs=qs)
            pb.set_schedule(schedule)
            pb.set_overlap_error(True)
            if depth > 1:
                pb.set_pipeline(depth)
            pb.reset()
            pb.set_initial_trace(0, 0, lam)
            pb.iterate(run.K)
            res[depth] = [(pb.batch_history(r), pb.overlap_history(r), [pb.batch_subdomain_uT(r, s) for s in range(2)])
                          for r in range(len(ps))]
    for r in range(len(ps)):
        (h1, o1, u1), (h4, o4, u4) = res[1][r], res[4][r]
        assert np.array_equal(h1[0], h4[0]) and np.array_equal(h1[1], h4[1]) and np.array_equal(o1, o4), r
        for a, b in zip(u1, u4):
            assert np.array_equal(a, b), r


def test_api_error_paths(kfp):
    """The documented error codes of the newer calls (include/kfp.h): wrong call order -> KFP_E_STATE, bad
    arguments -> KFP_E_INVAL; the handle stays usable afterwards."""
    run = RUNS["c0"].with_(K=4)
    with kfp.Problem(ki.make_problem(run)) as pb:
        with pytest.raises(kfp.KfpError) as e:  # before any setup
            pb.set_overlap_error(True)
        assert e.value.status == kfp.KFP_E_STATE
        with pytest.raises(kfp.KfpError) as e:
            pb.set_pipeline(2)
        assert e.value.status == kfp.KFP_E_STATE
        pb.setup(run.kind, run.p, run.overlap, run.n_sub, run.K)
        with pytest.raises(kfp.KfpError) as e:  # overlap history with the recording off
            pb.reset()
            pb.iterate(1)
            pb.overlap_history()
        assert e.value.status == kfp.KFP_E_STATE
        with pytest.raises(kfp.KfpError) as e:  # KFP_ERR_OVERLAP without recording
            pb.iterate_until(1e-6, 2, "overlap")
        assert e.value.status == kfp.KFP_E_STATE
        with pytest.raises(kfp.KfpError) as e:  # beyond K_max
            pb.iterate_until(1e-6, run.K, "err_if")
        assert e.value.status == kfp.KFP_E_STATE
        with pytest.raises(kfp.KfpError) as e:
            pb.set_pipeline(-1)  # (0 = the automatic depth)
        assert e.value.status == kfp.KFP_E_INVAL
        pb.reset()  # still usable
        k = pb.iterate_until(0.0, run.K, "err_T")  # eps = 0: never met, runs K_max
        assert k == run.K and len(pb.history()[0]) == run.K


def test_automatic_depth(kfp):
    """set_pipeline(0): a latency-bound window (configs[0]) is pipelined -- bitwise the unpipelined results in
    fewer launches -- and a window that fills the GPU (configs[2]) is left at one iteration per sweep."""
    run = RUNS["c0"]
    a, b = _solve(kfp, run, 1), _solve(kfp, run, 0)
    assert np.array_equal(a["eT"], b["eT"]) and np.array_equal(a["eI"], b["eI"])
    for x, y in zip(a["slabs"] + a["traces"], b["slabs"] + b["traces"]):
        assert np.array_equal(x, y)
    assert b["launches"] < a["launches"] // 2
    big = ki.config("c2")
    with kfp.Problem(ki.make_problem(big)) as pb:
        pb.setup(big.kind, big.p, big.overlap, big.n_sub, big.K)
        pb.set_pipeline(0)
        pb.reset()
        l0 = pb.launch_count()
        pb.iterate(1)
        assert pb.launch_count() - l0 == big.grid.nt

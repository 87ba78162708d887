"""TEST INFRASTRUCTURE ONLY -- brute-force dense solves on tiny grids.

Instead of marching step by step with a Thomas solve, these functions assemble
the WHOLE space-time linear system of one window -- every unknown u(t_n, x_m,
v_j), n = 1..N_t, of a subdomain at once -- from the stencil definitions of
DESIGN.md §3 (transport P:496-516, backward-Euler centred diffusion P:480-485,
transmission rows P:539-551 / reading R11) and solve it with a dense LU
(``numpy.linalg.solve``).  Nothing is shared with ``kfp_oracle.c``: the
assembly is global (one matrix for all time levels), the data come straight
from the ``kfp_inputs`` tables, and the solve is a library routine.

Only usable on tiny grids (the matrix has (N_t * N_unknown_v * N_x)^2 entries).
"""
from __future__ import annotations

import numpy as np

__all__ = ["dense_window", "dense_monodomain", "fem_matrices", "dense_fem_window"]


def dense_window(prob, lo, hi, lkind="phys", rkind="phys", p=0.0, gL=None, gR=None, q=None):
    """Solve the space-time system of subdomain [lo, hi]; returns u [(nt+1), (hi-lo+1), nx].

    lkind/rkind: 'phys' (Dirichlet 0), 'dirichlet' (value = trace), 'robin'
    ((q - d_v) u = trace at the left end, (p + d_v) u = trace at the right end, half-cell rows;
    q defaults to p).  gL/gR: [nt, nx] traces (row n-1 = t_n)."""
    pl = p if q is None else q
    g = prob.grid
    nx, nt = g.nx, g.nt
    hx, hv, dt = 1.0 / nx, 2.0 * g.vmax / g.nv, g.t_final / nt
    a = dt / hv ** 2
    v = -g.vmax + np.arange(g.nv + 1) * hv
    first = lo if lkind == "robin" else lo + 1
    last = hi if rkind == "robin" else hi - 1
    nu = last - first + 1
    N = nt * nu * nx

    def idx(n, j, m):  # n = 1..nt, j = first..last
        return ((n - 1) * nu + (j - first)) * nx + (m % nx)

    u0 = prob.u0_dense()
    A = np.zeros((N, N))
    b = np.zeros(N)
    known = {}  # (n, j) -> row vector over m of known end values

    def end_value(n, j):
        if j < first:
            return np.zeros(nx) if lkind == "phys" else np.asarray(gL[n - 1])
        return np.zeros(nx) if rkind == "phys" else np.asarray(gR[n - 1])

    for n in range(1, nt + 1):
        f = prob.f_dense(n)
        for j in range(first, last + 1):
            nuj = v[j] * dt / hx
            for m in range(nx):
                row = idx(n, j, m)
                # implicit diffusion part
                diag = 1.0 + 2.0 * a
                cl, cr = -a, -a
                rhs = dt * f[j, m]
                if j == lo and lkind == "robin":
                    diag += 2.0 * a * pl * hv
                    cr = -2.0 * a
                    cl = 0.0
                    rhs += 2.0 * a * hv * gL[n - 1, m]
                if j == hi and rkind == "robin":
                    diag += 2.0 * a * p * hv
                    cl = -2.0 * a
                    cr = 0.0
                    rhs += 2.0 * a * hv * gR[n - 1, m]
                A[row, row] += diag
                for jn, coef in ((j - 1, cl), (j + 1, cr)):
                    if coef == 0.0:
                        continue
                    if first <= jn <= last:
                        A[row, idx(n, jn, m)] += coef
                    else:
                        rhs -= coef * end_value(n, jn)[m]
                # explicit transport of level n-1 (minus sign: moved to the left side)
                if v[j] > 0:
                    terms = ((m, 1.0 - nuj), (m - 1, nuj))
                elif v[j] < 0:
                    terms = ((m, 1.0 + nuj), (m + 1, -nuj))
                else:
                    terms = ((m, 1.0),)
                for mm, coef in terms:
                    if n == 1:
                        rhs += coef * u0[j, mm % nx]
                    else:
                        A[row, idx(n - 1, j, mm)] -= coef
                b[row] = rhs
    x = np.linalg.solve(A, b)
    out = np.zeros((nt + 1, hi - lo + 1, nx))
    out[0] = u0[lo:hi + 1]
    for n in range(1, nt + 1):
        for j in range(lo, hi + 1):
            if first <= j <= last:
                out[n, j - lo] = x[idx(n, j, 0):idx(n, j, 0) + nx]
            else:
                out[n, j - lo] = end_value(n, j)
    return out


def dense_monodomain(prob):
    """All time levels of the monodomain solution, [(nt+1), (nv+1), nx]."""
    return dense_window(prob, 0, prob.grid.nv)


# ---------------------------------------------------------------------------
# The paper's split finite-element scheme, brute force.
#
# Independent of kfp_oracle.c's window_fem(): the mass and stiffness matrices are
# assembled by evaluating the hat functions (and their derivatives) at the three
# Cavalieri-Simpson points of every cell (P:519-521 literally), the columns are
# solved together by a dense LAPACK solve, and Step 2 evaluates the periodic
# piecewise-linear interpolant of w at the foot of the characteristic x_m - tau v_j
# with numpy.interp instead of using the upwind weights.


def _hat(v_nodes, i, v):
    """P1 nodal basis function phi_i of the node set v_nodes evaluated at v (scalar)."""
    h = v_nodes[1] - v_nodes[0]
    return max(0.0, 1.0 - abs(v - v_nodes[i]) / h)


def _dhat(v_nodes, i, v_left, v_right):
    """d phi_i / dv on the open cell (v_left, v_right)."""
    h = v_right - v_left
    if abs(v_nodes[i] - v_left) < 1e-12 * h:
        return -1.0 / h
    if abs(v_nodes[i] - v_right) < 1e-12 * h:
        return 1.0 / h
    return 0.0


def fem_matrices(v_nodes):
    """M_ij = int phi_j phi_i dv and S_ij = int phi_j' phi_i' dv (eq. MMvS) over the span of
    v_nodes, every cell integrated with the Cavalieri-Simpson rule."""
    n = len(v_nodes)
    M = np.zeros((n, n))
    S = np.zeros((n, n))
    for e in range(n - 1):
        a, b = v_nodes[e], v_nodes[e + 1]
        pts, wts = (a, 0.5 * (a + b), b), ((b - a) / 6.0, 4.0 * (b - a) / 6.0, (b - a) / 6.0)
        for i in (e, e + 1):
            for j in (e, e + 1):
                M[i, j] += sum(w * _hat(v_nodes, i, x) * _hat(v_nodes, j, x) for x, w in zip(pts, wts))
                S[i, j] += sum(w * _dhat(v_nodes, i, a, b) * _dhat(v_nodes, j, a, b) for x, w in zip(pts, wts))
    return M, S


def dense_fem_window(prob, lo, hi, lkind="phys", rkind="phys", p=0.0, gL=None, gR=None, q=None):
    """Split-FEM window of subdomain [lo, hi]; returns (u [(nt+1), nn, nx], w [nt, nn, nx]) -- u^n after
    every full step and w^{n+1/2}, the Step-1 results.  lkind/rkind: 'phys' (homogeneous Neumann,
    P:435-436), 'dirichlet' (w = trace at the node), 'robin' ((q - d_v) w = trace at the left end,
    (p + d_v) w = trace at the right end, through the boundary term of the weak form)."""
    pl = p if q is None else q
    g = prob.grid
    nx, nt = g.nx, g.nt
    dt = g.t_final / nt
    tau = 0.5 * dt
    v = g.v_nodes()[lo:hi + 1]
    x = g.x_nodes()
    nn = hi - lo + 1
    M, S = fem_matrices(v)
    A = M / tau + S
    if lkind == "robin":
        A[0, 0] += pl
    if rkind == "robin":
        A[-1, -1] += p
    unknown = np.ones(nn, bool)
    if lkind == "dirichlet":
        unknown[0] = False
    if rkind == "dirichlet":
        unknown[-1] = False
    Au = A[np.ix_(unknown, unknown)]
    u = prob.u0_dense()[lo:hi + 1].copy()
    us, ws = [u.copy()], []
    for n in range(nt):
        rhs = (M / tau) @ u
        wv = np.zeros((nn, nx))
        if lkind == "robin":
            rhs[0] += gL[n]
        if rkind == "robin":
            rhs[-1] += gR[n]
        if lkind == "dirichlet":
            wv[0] = gL[n]
        if rkind == "dirichlet":
            wv[-1] = gR[n]
        rhs = rhs - A[:, ~unknown] @ wv[~unknown]
        wv[unknown] = np.linalg.solve(Au, rhs[unknown])
        ws.append(wv.copy())
        u = np.stack([np.interp(x - tau * v[j], x, wv[j], period=1.0) for j in range(nn)])
        us.append(u.copy())
    return np.array(us), np.array(ws)

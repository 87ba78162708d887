/*
 * oracle/kfp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct fp64 CPU oracle for the Schwarz waveform
 * relaxation (SWR) solve of the Kolmogorov equation
 *        u_t + v u_x - u_vv = f          (eq. Intro1)
 * on x in [0,1) periodic, v in [-Vmax, Vmax] with homogeneous Dirichlet ends,
 * split along v into S contiguous subdomains, iterated with the
 * parallel (Jacobi) schedule of the Remark at P:594-597.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  The product path (the CUDA
 * library under paper_1306_4596_b200/) never calls it, and this file shares
 * no code, header, table or constant with the CUDA path.
 *
 * Everything follows DESIGN.md §3 ("readings") in the paper's order:
 *   O1  one time step = explicit first-order upwind transport in x
 *       (eqs. step2_a/step2_b, weight |v_j| dt/h_x, reading R7)
 *       followed by one backward-Euler centred diffusion solve in v per
 *       x-column (eq. step1; centred FD = lumped-mass FEM, R1),
 *       both over the full dt (R2), forcing at t_{n+1} (R3).  The tridiagonal
 *       system is solved by the textbook Thomas algorithm.
 *   O2  subdomain [lo, hi] with end nodes of three kinds: physical Dirichlet 0
 *       (R4), Dirichlet interface (CSWR, value moved to the RHS, R10),
 *       Robin interface (OSWR: (p + d_v) on the right end,
 *       (p - d_v) on the left end, one-sided p = q, R13/R16) imposed with the
 *       half-cell flux row (R11).
 *   O3  outgoing traces lambda (eq. lambda12 / SWR2 / SWR4) at every
 *       step: Dirichlet value, or the same half-cell flux combination (R11).
 *   O4  Jacobi iteration from zero traces (R17), K fixed; error of
 *       every iterate against the monodomain discrete solution (BASELINE.json
 *       north_star (c); a stopping diagnostic in the spirit of eq. (error),
 *       P:588-592).
 * A second discretisation, the paper's own (operator splitting with
 * consistent-mass linear finite elements in v, tau = dt/2, semi-Lagrangian
 * transport, Neumann physical ends), is selected by orc_problem.scheme and
 * implemented by window_fem() below; the SWR driver is shared.
 *
 * Layout of every 2-D array: v-major, element (node j, x-node m) at [j*nx + m].
 * Trace arrays [nt][nx]: row n-1 holds the value at t_n (n = 1..nt); the value
 * at t_0 is never used (reading R12).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t nx, nv, nt;
    double vmax, t_final;
    int32_t f_rank;
    const double *ft, *fv, *fx;   /* ft[r*(nt+1)+n], fv[r*(nv+1)+j], fx[r*nx+m] */
    int32_t u0_rank;
    const double *u0v, *u0x;      /* u0v[r*(nv+1)+j], u0x[r*nx+m] */
    int32_t scheme;               /* SCHEME_IMEX_FD or SCHEME_SPLIT_FEM (§3b) */
} orc_problem;

enum { END_PHYS = 0, END_DIRICHLET = 1, END_ROBIN = 2 };
enum { KIND_DIRICHLET = 0, KIND_ROBIN = 1 };
enum { SCHEME_IMEX_FD = 0, SCHEME_SPLIT_FEM = 1 };

/* Grid spacings (readings R5/R6). */
static double hx_of(const orc_problem *P) { return 1.0 / P->nx; }
static double hv_of(const orc_problem *P) { return 2.0 * P->vmax / P->nv; }
static double dt_of(const orc_problem *P) { return P->t_final / P->nt; }
static double v_of(const orc_problem *P, int j) { return -P->vmax + j * hv_of(P); }

/* f(t_n, x_m, v_j) from the separable input tables. */
static double forcing(const orc_problem *P, int n, int j, int m) {
    double s = 0.0;
    for (int r = 0; r < P->f_rank; ++r)
        s += P->ft[(size_t)r * (P->nt + 1) + n] * P->fv[(size_t)r * (P->nv + 1) + j] * P->fx[(size_t)r * P->nx + m];
    return s;
}

/* u0(x_m, v_j). */
static double initial(const orc_problem *P, int j, int m) {
    double s = 0.0;
    for (int r = 0; r < P->u0_rank; ++r)
        s += P->u0v[(size_t)r * (P->nv + 1) + j] * P->u0x[(size_t)r * P->nx + m];
    return s;
}

/* Textbook Thomas algorithm (no pivoting) for
 *   sub[i] x[i-1] + diag[i] x[i] + sup[i] x[i+1] = rhs[i],  i = 0..n-1.
 * The systems solved here are strictly diagonally dominant, so no pivoting is
 * needed.  cp, dp: scratch of length n. */
static void thomas(int n, const double *sub, const double *diag, const double *sup,
                   const double *rhs, double *cp, double *dp, double *x) {
    cp[0] = sup[0] / diag[0];
    dp[0] = rhs[0] / diag[0];
    for (int i = 1; i < n; ++i) {
        double den = diag[i] - sub[i] * cp[i - 1];
        cp[i] = sup[i] / den;
        dp[i] = (rhs[i] - sub[i] * dp[i - 1]) / den;
    }
    x[n - 1] = dp[n - 1];
    for (int i = n - 2; i >= 0; --i) x[i] = dp[i] - cp[i] * x[i + 1];
}

/* Window solve of one subdomain with the paper's own discretisation (DESIGN.md §3b,
 * readings F1-F6).  Operator splitting, per step n -> n+1:
 *   Step 1 (eq. step1): for every x-column m solve
 *              (1/tau) M w + S w = (1/tau) M u^n
 *          with M, S the P1 finite-element mass and stiffness matrices of eq. MMvS
 *          on the subdomain's nodes, assembled element by element; the P1 element integrals are
 *          integrated exactly by the Cavalieri-Simpson rule:
 *              Me = h/6 [2 1; 1 2],   Se = 1/h [1 -1; -1 1].
 *   Step 2 (eqs. step2_a / step2_b): u^{n+1}(x_m, v_j) = w(x_m - tau v_j, v_j) by linear
 *          interpolation between the two x-nodes around the foot of the characteristic:
 *              (1 - |v_j| tau/h_x) w_m + (|v_j| tau/h_x) w_{m-1}  (v_j > 0; m+1 for v_j < 0),
 *          the weight of P:501 with the /h_x the formula drops (reading F3 = R7).
 *   tau = dt/2 in both steps, dt = T/nt, as printed (reading F2).
 * End nodes: END_PHYS = homogeneous Neumann: natural, nothing added to the weak form;
 * END_ROBIN = the Robin condition imposed weakly through the boundary term of the weak form:
 * left end (pl - d_v) w = g adds pl to the lo row's diagonal and g to its right-hand side, right
 * end (pr + d_v) w = g likewise at hi; END_DIRICHLET = w = g at the node (its
 * equation dropped, the known value moved to the neighbour's right-hand side).
 * Outgoing traces (reading F4): Dirichlet: w_c.  Robin: p w_c - (the residual of the sender's
 * half-row at c on the element toward the receiver's exterior), i.e. the flux the receiver's
 * weak form needs, so that the monodomain solution is the fixed point (pinned).
 * rec: w (the Step-1 result, where the transmission conditions act) at rec_nodes for every step;
 * uT: u^{nt}, after the last Step 2.  Arguments as in window(). */
static void window_fem(const orc_problem *P, int lo, int hi, int ltype, int rtype, double pl, double pr,
                       const double *gL, const double *gR, int send_kind,
                       int sendL_node, double *sendL, int sendR_node, double *sendR,
                       int nrec, const int *rec_nodes, double *rec, double *uT) {
    const int nx = P->nx, nt = P->nt, nn = hi - lo + 1;
    const double hx = hx_of(P), hv = hv_of(P), dt = dt_of(P), tau = 0.5 * dt;
    /* P1 element matrices on a cell of length hv (exact integrals) */
    const double Me_d = hv / 3.0, Me_o = hv / 6.0, Se_d = 1.0 / hv, Se_o = -1.0 / hv;
    /* global tridiagonal M and S on nodes lo..hi: *_d[i] diagonal of node lo+i, *_o[i] coupling (i, i+1) */
    double *Md = (double *)calloc(nn, sizeof(double)), *Sd = (double *)calloc(nn, sizeof(double));
    double *Mo = (double *)calloc(nn, sizeof(double)), *So = (double *)calloc(nn, sizeof(double));
    for (int e = 0; e + 1 < nn; ++e) { /* element [lo+e, lo+e+1] */
        Md[e] += Me_d; Md[e + 1] += Me_d; Mo[e] += Me_o;
        Sd[e] += Se_d; Sd[e + 1] += Se_d; So[e] += Se_o;
    }
    double *u = (double *)malloc(sizeof(double) * (size_t)nn * nx);   /* u^n on all nodes */
    double *w = (double *)malloc(sizeof(double) * (size_t)nn * nx);   /* Step-1 result */
    for (int j = lo; j <= hi; ++j)
        for (int m = 0; m < nx; ++m) u[(size_t)(j - lo) * nx + m] = initial(P, j, m);
    const int first = (ltype == END_DIRICHLET) ? lo + 1 : lo;
    const int last = (rtype == END_DIRICHLET) ? hi - 1 : hi;
    const int nu = last - first + 1;

    for (int n = 0; n < nt; ++n) {
#pragma omp parallel
        {
            double *sub = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *diag = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *sup = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *rhs = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *cp = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *dp = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *x = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
#pragma omp for schedule(static)
            for (int m = 0; m < nx; ++m) {
#define U_(j) u[(size_t)((j) - lo) * nx + m]
#define W_(j) w[(size_t)((j) - lo) * nx + m]
                const double left_val = (ltype == END_DIRICHLET) ? gL[(size_t)n * nx + m] : 0.0;
                const double right_val = (rtype == END_DIRICHLET) ? gR[(size_t)n * nx + m] : 0.0;
                for (int j = first; j <= last; ++j) {
                    const int i = j - lo, r = j - first;
                    /* row i of (1/tau) M w + S w = (1/tau) M u^n */
                    double b = Md[i] * U_(j);
                    if (i > 0) b += Mo[i - 1] * U_(j - 1);
                    if (i < nn - 1) b += Mo[i] * U_(j + 1);
                    rhs[r] = b / tau;
                    diag[r] = Md[i] / tau + Sd[i];
                    sub[r] = (i > 0) ? Mo[i - 1] / tau + So[i - 1] : 0.0;
                    sup[r] = (i < nn - 1) ? Mo[i] / tau + So[i] : 0.0;
                    if (j == lo && ltype == END_ROBIN) { /* (pl - d_v) w = g: boundary term of the weak form */
                        diag[r] += pl;
                        rhs[r] += gL[(size_t)n * nx + m];
                    }
                    if (j == hi && rtype == END_ROBIN) { /* (pr + d_v) w = g */
                        diag[r] += pr;
                        rhs[r] += gR[(size_t)n * nx + m];
                    }
                    if (j == lo + 1 && ltype == END_DIRICHLET) { rhs[r] -= sub[r] * left_val; sub[r] = 0.0; }
                    if (j == hi - 1 && rtype == END_DIRICHLET) { rhs[r] -= sup[r] * right_val; sup[r] = 0.0; }
                }
                if (nu > 0) thomas(nu, sub, diag, sup, rhs, cp, dp, x);
                for (int j = lo; j <= hi; ++j)
                    W_(j) = (j < first) ? left_val : (j > last) ? right_val : x[j - first];
                /* outgoing traces at step n+1 (reading F4) */
                if (sendL_node >= 0) { /* to the left neighbour's right end: (pr + d_v) w, half-row on [c, c+1] */
                    const int c = sendL_node;
                    double g = W_(c);
                    if (send_kind == KIND_ROBIN) {
                        const double half = (Me_d * (W_(c) - U_(c)) + Me_o * (W_(c + 1) - U_(c + 1))) / tau +
                                            Se_d * W_(c) + Se_o * W_(c + 1);
                        g = pr * W_(c) - half;
                    }
                    sendL[(size_t)n * nx + m] = g;
                }
                if (sendR_node >= 0) { /* to the right neighbour's left end: (pl - d_v) w, half-row on [c-1, c] */
                    const int c = sendR_node;
                    double g = W_(c);
                    if (send_kind == KIND_ROBIN) {
                        const double half = (Me_d * (W_(c) - U_(c)) + Me_o * (W_(c - 1) - U_(c - 1))) / tau +
                                            Se_d * W_(c) + Se_o * W_(c - 1);
                        g = pl * W_(c) - half;
                    }
                    sendR[(size_t)n * nx + m] = g;
                }
#undef U_
#undef W_
            }
            free(sub); free(diag); free(sup); free(rhs); free(cp); free(dp); free(x);
        }
        for (int i = 0; i < nrec; ++i)
            memcpy(rec + ((size_t)i * nt + n) * nx, w + (size_t)(rec_nodes[i] - lo) * nx, sizeof(double) * nx);
        /* Step 2: u^{n+1}(x_m, v_j) = w(x_m - tau v_j, v_j), linear interpolation in x */
#pragma omp parallel for schedule(static)
        for (int j = lo; j <= hi; ++j) {
            const double v = v_of(P, j), c = fabs(v) * tau / hx;
            const double *wr = w + (size_t)(j - lo) * nx;
            double *ur = u + (size_t)(j - lo) * nx;
            for (int m = 0; m < nx; ++m) {
                const int nb = (v > 0.0) ? (m + nx - 1) % nx : (m + 1) % nx;  /* node on the foot's side */
                ur[m] = (v == 0.0) ? wr[m] : (1.0 - c) * wr[m] + c * wr[nb];
            }
        }
    }
    if (uT) memcpy(uT, u, sizeof(double) * (size_t)nn * nx);
    free(Md); free(Sd); free(Mo); free(So); free(u); free(w);
}

/* Window solve of one subdomain, nodes [lo, hi], from u0 over all nt steps
 * (one solve of SWR1 / SWR3, with the Jacobi data of P:594-597).
 *
 *  ltype/rtype : END_PHYS | END_DIRICHLET | END_ROBIN for the end nodes lo/hi.
 *  pl, pr      : Robin parameters of the lo (left) and hi (right) ends:
 *                the left end imposes (pl - d_v) u = g, the right end (pr + d_v) u = g.
 *                Two-sided OSWR(p,q): every right end uses p and every
 *                left end q, so pr = p, pl = q for all subdomains; one-sided OSWR(p):
 *                pl = pr = p.  The trace sent to the left neighbour lands on its
 *                right end and uses pr; the one sent right uses pl.
 *  gL, gR      : incoming traces [nt][nx] for the lo / hi end (NULL if physical).
 *  send_kind   : KIND_DIRICHLET or KIND_ROBIN, the kind of the outgoing traces.
 *  sendL_node  : node whose trace is sent to the left neighbour (its hi end),
 *                -1 if none; sendL [nt][nx] receives it.
 *  sendR_node  : node whose trace is sent to the right neighbour (its lo end),
 *                -1 if none; sendR [nt][nx] receives it.
 *  nrec, rec_nodes, rec : record u at nodes rec_nodes[i] for n = 1..nt into
 *                rec[i][n-1][m] (used for the interface error and U-lines).
 *  uT          : [(hi-lo+1)][nx] solution at t = T (may be NULL).
 */
static void window(const orc_problem *P, int lo, int hi, int ltype, int rtype, double pl, double pr,
                   const double *gL, const double *gR, int send_kind,
                   int sendL_node, double *sendL, int sendR_node, double *sendR,
                   int nrec, const int *rec_nodes, double *rec, double *uT) {
    if (P->scheme == SCHEME_SPLIT_FEM) {
        window_fem(P, lo, hi, ltype, rtype, pl, pr, gL, gR, send_kind, sendL_node, sendL, sendR_node, sendR,
                   nrec, rec_nodes, rec, uT);
        return;
    }
    const int nx = P->nx, nt = P->nt, nn = hi - lo + 1;
    const double hx = hx_of(P), hv = hv_of(P), dt = dt_of(P);
    const double a = dt / (hv * hv);
    double *uo = (double *)malloc(sizeof(double) * (size_t)nn * nx);
    double *un = (double *)malloc(sizeof(double) * (size_t)nn * nx);
    double *rL = (double *)malloc(sizeof(double) * nx);
    double *rR = (double *)malloc(sizeof(double) * nx);

    /* u(0) = u0 on the subdomain. */
    for (int j = lo; j <= hi; ++j)
        for (int m = 0; m < nx; ++m) uo[(size_t)(j - lo) * nx + m] = initial(P, j, m);

    /* unknown node range */
    const int first = (ltype == END_ROBIN) ? lo : lo + 1;
    const int last = (rtype == END_ROBIN) ? hi : hi - 1;
    const int nu = last - first + 1;

    for (int n = 0; n < nt; ++n) { /* step t_n -> t_{n+1} */
#pragma omp parallel
        {
            double *r = (double *)malloc(sizeof(double) * nn);
            double *sub = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *diag = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *sup = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *rhs = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *cp = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *dp = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
            double *x = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
#pragma omp for schedule(static)
            for (int m = 0; m < nx; ++m) {
                const int mm = (m + nx - 1) % nx, mp = (m + 1) % nx;
                /* Step a: explicit upwind transport in x (R7/R8) plus
                 * dt * f(t_{n+1}) (R3).  v > 0 takes the m-1 neighbour, v < 0 the
                 * m+1 neighbour, v = 0 is not transported. */
                for (int j = lo; j <= hi; ++j) {
                    const double *row = uo + (size_t)(j - lo) * nx;
                    const double v = v_of(P, j), nuj = v * dt / hx;
                    double rj;
                    if (v > 0.0) rj = row[m] - nuj * (row[m] - row[mm]);
                    else if (v < 0.0) rj = row[m] - nuj * (row[mp] - row[m]);
                    else rj = row[m];
                    r[j - lo] = rj + dt * forcing(P, n + 1, j, m);
                }
                /* Step b: backward Euler in v, centred 3-point FD (R1):
                 *   -a u_{j-1} + (1+2a) u_j - a u_{j+1} = r_j. */
                const double left_val = (ltype == END_DIRICHLET) ? gL[(size_t)n * nx + m] : 0.0;
                const double right_val = (rtype == END_DIRICHLET) ? gR[(size_t)n * nx + m] : 0.0;
                for (int j = first; j <= last; ++j) {
                    int i = j - first;
                    sub[i] = -a;
                    diag[i] = 1.0 + 2.0 * a;
                    sup[i] = -a;
                    rhs[i] = r[j - lo];
                    if (j == lo) { /* Robin left end: (pl - d_v) u = g, half-cell row (R11, R13) */
                        diag[i] = 1.0 + 2.0 * a + 2.0 * a * pl * hv;
                        sup[i] = -2.0 * a;
                        rhs[i] += 2.0 * a * hv * gL[(size_t)n * nx + m];
                    } else if (j == lo + 1) { /* known node lo moved to the RHS (R10) */
                        rhs[i] += a * left_val;
                    }
                    if (j == hi) { /* Robin right end: (pr + d_v) u = g */
                        diag[i] = 1.0 + 2.0 * a + 2.0 * a * pr * hv;
                        sub[i] = -2.0 * a;
                        rhs[i] += 2.0 * a * hv * gR[(size_t)n * nx + m];
                    } else if (j == hi - 1) {
                        rhs[i] += a * right_val;
                    }
                }
                if (nu > 0) thomas(nu, sub, diag, sup, rhs, cp, dp, x);
                for (int j = lo; j <= hi; ++j) {
                    double val;
                    if (j < first) val = left_val;
                    else if (j > last) val = right_val;
                    else val = x[j - first];
                    un[(size_t)(j - lo) * nx + m] = val;
                }
                if (sendL_node >= 0) rL[m] = r[sendL_node - lo];
                if (sendR_node >= 0) rR[m] = r[sendR_node - lo];
            }
            free(r); free(sub); free(diag); free(sup); free(rhs); free(cp); free(dp); free(x);
        }
        /* Outgoing traces at t_{n+1} (O3 / reading R11). */
        if (sendL_node >= 0) {
            const double *uc = un + (size_t)(sendL_node - lo) * nx;
            for (int m = 0; m < nx; ++m) {
                double g;
                if (send_kind == KIND_DIRICHLET) g = uc[m];
                else { /* (pr + d_v) u at node c, d_v u = half-cell flux on [c, c + h/2] */
                    const double ucp = uc[m + nx]; /* node c+1 */
                    g = pr * uc[m] - ((uc[m] - ucp) / hv + 0.5 * hv * (uc[m] - rL[m]) / dt);
                }
                sendL[(size_t)n * nx + m] = g;
            }
        }
        if (sendR_node >= 0) {
            const double *uc = un + (size_t)(sendR_node - lo) * nx;
            for (int m = 0; m < nx; ++m) {
                double g;
                if (send_kind == KIND_DIRICHLET) g = uc[m];
                else { /* (pl - d_v) u at node c, d_v u = half-cell flux on [c - h/2, c] */
                    const double ucm = uc[m - nx]; /* node c-1 */
                    g = pl * uc[m] - ((uc[m] - ucm) / hv + 0.5 * hv * (uc[m] - rR[m]) / dt);
                }
                sendR[(size_t)n * nx + m] = g;
            }
        }
        for (int i = 0; i < nrec; ++i) {
            const double *src = un + (size_t)(rec_nodes[i] - lo) * nx;
            memcpy(rec + ((size_t)i * nt + n) * nx, src, sizeof(double) * nx);
        }
        double *t = uo; uo = un; un = t;
    }
    if (uT) memcpy(uT, uo, sizeof(double) * (size_t)nn * nx);
    free(uo); free(un); free(rL); free(rR);
}

/* ---------------------------------------------------------------------- */
/* Public (ctypes) entry points.                                           */

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Subdomain node ranges (reading R9):
 * c_s = s*nv/S, lo_0 = 0, lo_s = c_s - floor(ov/2), hi_s = c_{s+1} + ceil(ov/2),
 * hi_{S-1} = nv.  Returns 0 on success. */
int orc_subdomains(int nv, int n_sub, int overlap, int32_t *lo, int32_t *hi) {
    if (n_sub < 1 || nv % n_sub != 0 || overlap < 0) return -1;
    for (int s = 0; s < n_sub; ++s) {
        int cs = s * (nv / n_sub), cs1 = (s + 1) * (nv / n_sub);
        lo[s] = (s == 0) ? 0 : cs - overlap / 2;
        hi[s] = (s == n_sub - 1) ? nv : cs1 + (overlap + 1) / 2;
    }
    return 0;
}

/* Monodomain solve on nodes [0, nv] with physical ends (Dirichlet 0 for the IMEX FD scheme, Neumann for
 * the split FEM scheme) (BJ north_star
 * (c): the reference every SWR iterate is compared with).  Records U at
 * rec_nodes for n = 1..nt and returns U(T). */
int orc_monodomain(const orc_problem *P, int nrec, const int32_t *rec_nodes, double *rec, double *UT) {
    int *nodes = (int *)malloc(sizeof(int) * (nrec > 0 ? nrec : 1));
    for (int i = 0; i < nrec; ++i) nodes[i] = rec_nodes[i];
    window(P, 0, P->nv, END_PHYS, END_PHYS, 0.0, 0.0, NULL, NULL, KIND_DIRICHLET, -1, NULL, -1, NULL,
           nrec, nodes, rec, UT);
    free(nodes);
    return 0;
}

/* One subdomain window with explicit ends and traces (used by the tests'
 * distributed-driver backend).  Arguments as in window(); orc_window is the
 * one-sided form pl = pr = p. */
int orc_window_pq(const orc_problem *P, int lo, int hi, int ltype, int rtype, double pl, double pr,
                  const double *gL, const double *gR, int send_kind,
                  int sendL_node, double *sendL, int sendR_node, double *sendR,
                  int nrec, const int32_t *rec_nodes, double *rec, double *uT) {
    int *nodes = (int *)malloc(sizeof(int) * (nrec > 0 ? nrec : 1));
    for (int i = 0; i < nrec; ++i) nodes[i] = rec_nodes[i];
    window(P, lo, hi, ltype, rtype, pl, pr, gL, gR, send_kind, sendL_node, sendL, sendR_node, sendR,
           nrec, nodes, rec, uT);
    free(nodes);
    return 0;
}
int orc_window(const orc_problem *P, int lo, int hi, int ltype, int rtype, double p,
               const double *gL, const double *gR, int send_kind,
               int sendL_node, double *sendL, int sendR_node, double *sendR,
               int nrec, const int32_t *rec_nodes, double *rec, double *uT) {
    return orc_window_pq(P, lo, hi, ltype, rtype, p, p, gL, gR, send_kind, sendL_node, sendL, sendR_node, sendR,
                         nrec, rec_nodes, rec, uT);
}

/* Jacobi SWR (P:554-597 with the Remark at P:594-597), K iterations from zero
 * traces, errors against the monodomain solution.
 *
 *  kind        : KIND_DIRICHLET (CSWR, Q = identity) or KIND_ROBIN: OSWR(p, q) with p on
 *                every right (hi) end and q on every left (lo) end;
 *                orc_swr is the one-sided OSWR(p), q = p.
 *  uT_sub      : concatenated per-subdomain slabs u_s^K(T), s = 0..S-1 (may be NULL).
 *  uT          : [(nv+1)][nx] assembled by nominal ownership (node j belongs to
 *                the s with c_s <= j < c_{s+1}; node nv to S-1) (may be NULL).
 *  UT          : [(nv+1)][nx] monodomain U(T) (may be NULL).
 *  err_T[k-1]  : max_{s, m, j in [lo_s,hi_s]} |u_s^k(T) - U(T)|.
 *  err_if[k-1] : max_{s, interface end nodes of s, n>=1, m} |u_s^k(t_n) - U(t_n)|.
 *  traces      : final-iteration outgoing traces, [2*(S-1)][nt][nx]: for interface i
 *                (between s=i and s=i+1) first toLeft[i] (sent by i+1, used at hi_i)
 *                then toRight[i] (sent by i, used at lo_{i+1}); may be NULL.
 */
static int swr_impl(const orc_problem *P, int kind, double p, double q, int overlap, int n_sub, int K, int gauss_seidel,
                    const double *init_toL, const double *init_toR,
                    double *uT_sub, double *uT, double *UT, double *err_T, double *err_if, double *traces,
                    double *err_ov) {
    const int nx = P->nx, nt = P->nt, nv = P->nv, S = n_sub;
    if (S < 1 || nv % S != 0 || K < 1) return -1;
    int32_t *lo = (int32_t *)malloc(sizeof(int32_t) * S), *hi = (int32_t *)malloc(sizeof(int32_t) * S);
    if (orc_subdomains(nv, S, overlap, lo, hi)) { free(lo); free(hi); return -1; }
    const size_t TR = (size_t)nt * nx;

    /* interface lines for err_if: lo_s (s>0) and hi_s (s<S-1) */
    int nl = 0;
    int32_t *lines = (int32_t *)malloc(sizeof(int32_t) * (2 * S + 1));
    for (int s = 0; s < S; ++s) {
        if (s > 0) lines[nl++] = lo[s];
        if (s < S - 1) lines[nl++] = hi[s];
    }
    double *Ulines = (double *)malloc(sizeof(double) * (nl > 0 ? nl : 1) * TR);
    double *Ut = (double *)malloc(sizeof(double) * (size_t)(nv + 1) * nx);
    orc_monodomain(P, nl, lines, Ulines, Ut);
    if (UT) memcpy(UT, Ut, sizeof(double) * (size_t)(nv + 1) * nx);

    int ni = S - 1;
    double *toL_in = (double *)calloc((ni > 0 ? ni : 1) * TR, sizeof(double));
    double *toR_in = (double *)calloc((ni > 0 ? ni : 1) * TR, sizeof(double));
    double *toL_out = (double *)calloc((ni > 0 ? ni : 1) * TR, sizeof(double));
    /* initial traces lambda^0: zero unless given (Table 1 uses random ones) */
    if (init_toL && ni > 0) memcpy(toL_in, init_toL, sizeof(double) * ni * TR);
    if (init_toR && ni > 0) memcpy(toR_in, init_toR, sizeof(double) * ni * TR);
    double *toR_out = (double *)calloc((ni > 0 ? ni : 1) * TR, sizeof(double));
    size_t tot = 0;
    for (int s = 0; s < S; ++s) tot += (size_t)(hi[s] - lo[s] + 1) * nx;
    double *slabs = (double *)malloc(sizeof(double) * tot);
    /* overlap records for the paper's stopping quantity (eq. 'error'): interface i's closed
     * overlap [lo_{i+1}, hi_i] as seen by subdomain i (ovA) and by i+1 (ovB) */
    int ovmax = 1;
    for (int i = 0; i + 1 < S; ++i) if (hi[i] - lo[i + 1] + 1 > ovmax) ovmax = hi[i] - lo[i + 1] + 1;
    double *rec = (double *)malloc(sizeof(double) * (2 + 2 * (size_t)ovmax) * TR);
    double *ovA = err_ov ? (double *)malloc(sizeof(double) * (ni > 0 ? ni : 1) * ovmax * TR) : NULL;
    double *ovB = err_ov ? (double *)malloc(sizeof(double) * (ni > 0 ? ni : 1) * ovmax * TR) : NULL;

    const int etype = (kind == KIND_ROBIN) ? END_ROBIN : END_DIRICHLET;
    for (int k = 1; k <= K; ++k) {
        double eT = 0.0, eI = 0.0;
        size_t off = 0;
        for (int s = 0; s < S; ++s) {
            int lt = (s == 0) ? END_PHYS : etype, rt = (s == S - 1) ? END_PHYS : etype;
            /* Jacobi: both incoming traces from iteration k-1.  Gauss-Seidel (SWR1-SWR4,
             * P:554-585, in subdomain order): the left trace is the one s-1 sent in this iteration. */
            const double *gL = (s > 0) ? (gauss_seidel ? toR_out : toR_in) + (size_t)(s - 1) * TR : NULL;
            const double *gR = (s < S - 1) ? toL_in + (size_t)s * TR : NULL;
            int sendL = (s > 0) ? hi[s - 1] : -1, sendR = (s < S - 1) ? lo[s + 1] : -1;
            int nrec = 0;
            int *rn = (int *)malloc(sizeof(int) * (2 + 2 * (size_t)ovmax));
            int32_t lidx[2];
            if (s > 0) { rn[nrec] = lo[s]; lidx[nrec++] = lo[s]; }
            if (s < S - 1) { rn[nrec] = hi[s]; lidx[nrec++] = hi[s]; }
            const int nif = nrec, cntL = (err_ov && s > 0) ? hi[s - 1] - lo[s] + 1 : 0,
                      cntR = (err_ov && s < S - 1) ? hi[s] - lo[s + 1] + 1 : 0;
            for (int r = 0; r < cntL; ++r) rn[nrec++] = lo[s] + r;      /* shared with s-1 */
            for (int r = 0; r < cntR; ++r) rn[nrec++] = lo[s + 1] + r;  /* shared with s+1 */
            double *us = slabs + off;
            window(P, lo[s], hi[s], lt, rt, q, p, gL, gR, kind,
                   sendL, (s > 0) ? toL_out + (size_t)(s - 1) * TR : NULL,
                   sendR, (s < S - 1) ? toR_out + (size_t)s * TR : NULL, nrec, rn, rec, us);
            free(rn);
            if (cntL) memcpy(ovB + (size_t)(s - 1) * ovmax * TR, rec + (size_t)nif * TR, sizeof(double) * cntL * TR);
            if (cntR) memcpy(ovA + (size_t)s * ovmax * TR, rec + (size_t)(nif + cntL) * TR, sizeof(double) * cntR * TR);
            /* interface error (all steps n = 1..nt) */
            for (int i = 0; i < nif; ++i) {
                int li = -1;
                for (int q = 0; q < nl; ++q) if (lines[q] == lidx[i]) { li = q; break; }
                const double *Ul = Ulines + (size_t)li * TR, *ul = rec + (size_t)i * TR;
                for (size_t t = 0; t < TR; ++t) { double d = fabs(ul[t] - Ul[t]); if (d > eI) eI = d; }
            }
            /* error at T on every node of the subdomain */
            for (int j = lo[s]; j <= hi[s]; ++j)
                for (int m = 0; m < nx; ++m) {
                    double d = fabs(us[(size_t)(j - lo[s]) * nx + m] - Ut[(size_t)j * nx + m]);
                    if (d > eT) eT = d;
                }
            off += (size_t)(hi[s] - lo[s] + 1) * nx;
        }
        err_T[k - 1] = eT;
        err_if[k - 1] = eI;
        if (err_ov) { /* max over the closed overlaps, steps and x-nodes of |u_s - u_{s+1}| */
            double eo = 0.0;
            for (int i = 0; i < ni; ++i) {
                const size_t cnt = (size_t)(hi[i] - lo[i + 1] + 1) * TR;
                const double *a = ovA + (size_t)i * ovmax * TR, *b = ovB + (size_t)i * ovmax * TR;
                for (size_t t = 0; t < cnt; ++t) { double d = fabs(a[t] - b[t]); if (d > eo) eo = d; }
            }
            err_ov[k - 1] = eo;
        }
        /* Jacobi exchange: iteration k's outgoing traces feed iteration k+1. */
        double *t;
        t = toL_in; toL_in = toL_out; toL_out = t;
        t = toR_in; toR_in = toR_out; toR_out = t;
    }
    if (uT_sub) memcpy(uT_sub, slabs, sizeof(double) * tot);
    if (uT) {
        size_t off = 0;
        for (int s = 0; s < S; ++s) {
            int c0 = s * (nv / S), c1 = (s == S - 1) ? nv : (s + 1) * (nv / S) - 1;
            for (int j = c0; j <= c1; ++j)
                memcpy(uT + (size_t)j * nx, slabs + off + (size_t)(j - lo[s]) * nx, sizeof(double) * nx);
            off += (size_t)(hi[s] - lo[s] + 1) * nx;
        }
    }
    if (traces && ni > 0) {
        for (int i = 0; i < ni; ++i) {
            memcpy(traces + (size_t)(2 * i) * TR, toL_in + (size_t)i * TR, sizeof(double) * TR);
            memcpy(traces + (size_t)(2 * i + 1) * TR, toR_in + (size_t)i * TR, sizeof(double) * TR);
        }
    }
    free(lo); free(hi); free(lines); free(Ulines); free(Ut);
    free(toL_in); free(toR_in); free(toL_out); free(toR_out); free(slabs); free(rec); free(ovA); free(ovB);
    return 0;
}
int orc_swr_pq(const orc_problem *P, int kind, double p, double q, int overlap, int n_sub, int K,
               double *uT_sub, double *uT, double *UT, double *err_T, double *err_if, double *traces) {
    return swr_impl(P, kind, p, q, overlap, n_sub, K, 0, NULL, NULL, uT_sub, uT, UT, err_T, err_if, traces, NULL);
}
/* Gauss-Seidel schedule (the paper's serial SWR1-SWR4, subdomains in increasing v). */
int orc_swr_gs(const orc_problem *P, int kind, double p, double q, int overlap, int n_sub, int K,
               double *uT_sub, double *uT, double *UT, double *err_T, double *err_if, double *traces) {
    return swr_impl(P, kind, p, q, overlap, n_sub, K, 1, NULL, NULL, uT_sub, uT, UT, err_T, err_if, traces, NULL);
}
/* General form: schedule (0 Jacobi, 1 Gauss-Seidel) and initial traces init_toL / init_toR
 * ([n_sub-1][nt][nx]: toward the left subdomain's right end / the right subdomain's left end; NULL = 0);
 * err_ov[k-1] (may be NULL): the paper's convergence quantity (eq. 'error'), max over every
 * closed overlap [lo_{s+1}, hi_s], step and x-node of |u_s^k - u_{s+1}^k| (split FEM: of the Step-1
 * values w, where the transmission conditions act). */
int orc_swr_ex(const orc_problem *P, int kind, double p, double q, int overlap, int n_sub, int K, int gauss_seidel,
               const double *init_toL, const double *init_toR,
               double *uT_sub, double *uT, double *UT, double *err_T, double *err_if, double *traces, double *err_ov) {
    return swr_impl(P, kind, p, q, overlap, n_sub, K, gauss_seidel, init_toL, init_toR, uT_sub, uT, UT, err_T, err_if,
                    traces, err_ov);
}
int orc_swr(const orc_problem *P, int kind, double p, int overlap, int n_sub, int K,
            double *uT_sub, double *uT, double *UT, double *err_T, double *err_if, double *traces) {
    return orc_swr_pq(P, kind, p, p, overlap, n_sub, K, uT_sub, uT, UT, err_T, err_if, traces);
}

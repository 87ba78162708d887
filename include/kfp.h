/*
 * kfp.h -- C-ABI of the B200 (sm_100a) Schwarz-waveform-relaxation solver for
 * the Kolmogorov equation  u_t + v u_x - u_vv = f  (arXiv 1306.4596,
 * PAPER.md:22-25 eq. Intro1 and P:33-38 eq. Kolmogorovmain).
 *
 * The solver computes, on x in [0,1) periodic (N_x nodes) and v in
 * [-Vmax, Vmax] (N_v cells, N_v+1 nodes, homogeneous Dirichlet ends), with
 * N_t steps of dt = T/N_t:
 *   - one step = explicit first-order upwind transport in x (P:496-516,
 *     weight |v_j| dt/h_x) then a backward-Euler centred diffusion solve in v,
 *     one tridiagonal system per x-column; full dt, forcing at
 *     t_{n+1} (readings R1-R8);
 *   - the v-axis split into n_sub contiguous subdomains iterated
 *     by Jacobi SWR (the Remark at P:594-597) with Dirichlet
 *     (classical) or Robin (optimised; one-sided p = q,
 *     P:613) transmission of whole-window traces (eq. lambda12);
 *   - per-iteration errors of the iterates against the monodomain discrete
 *     solution (BASELINE.json north_star (c)).
 *
 * Conventions (all entry points):
 *   - every floating-point array is fp64;
 *   - 2-D arrays are v-major: element (v-node j, x-node m) at [j*nx + m];
 *   - pointers marked "host" are host memory owned by the caller; the library
 *     copies inputs during the call and never keeps a host pointer;
 *   - pointers marked "device" are CUDA device memory on the problem's device,
 *     owned by the caller, and must stay valid while the library uses them;
 *   - every call returns a kfp_status; on error the state of the problem is
 *     unchanged unless stated otherwise, and kfp_last_error() returns a
 *     thread-local human-readable message;
 *   - a handle is used by one host thread at a time;
 *   - work is queued on the problem's CUDA stream (kfp_set_stream); calls that
 *     return host data synchronise that stream.
 * There is no CPU fallback: every numerical step runs in this library's CUDA
 * kernels; creating a problem without a usable sm_100 device returns
 * KFP_E_CUDA.
 */
#ifndef KFP_H
#define KFP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kfp_problem_s *kfp_problem; /* opaque; owns all device memory it allocates */

typedef enum {
    KFP_OK = 0,
    KFP_E_INVAL = -1,  /* invalid argument (sizes, decomposition, p, K, ...) */
    KFP_E_CFL = -2,    /* Vmax * dt / h_x > 1: the upwind step would not be a convex combination */
    KFP_E_NOMEM = -3,  /* device allocation failed */
    KFP_E_CUDA = -4,   /* CUDA runtime error or no usable device */
    KFP_E_STATE = -6,  /* call order (e.g. history before any solve) */
    KFP_E_NONFINITE = -7 /* an iteration's error is NaN or infinite (the solve blew up; failure detection) */
} kfp_status;

typedef enum {
    KFP_DIRICHLET = 0, /* classical SWR (CSWR): Q1 = Q2 = identity */
    KFP_ROBIN = 1      /* optimised SWR OSWR(p): Q1 = p + d_v, Q2 = p - d_v (p = q) */
} kfp_kind;

typedef enum {
    KFP_JACOBI = 0,      /* parallel schedule (Remark P:594-597) */
    KFP_GAUSS_SEIDEL = 1 /* the paper's serial SWR1-SWR4 */
} kfp_schedule;

/* Discretisation of a problem (fixed at creation; every later call follows it).
 * KFP_SCHEME_IMEX_FD: BASELINE.json north_star's scheme: per step dt = T/nt, upwind
 *   x-transport then one backward-Euler centred-FD v-solve (lumped-mass P1), forcing at t_{n+1},
 *   Dirichlet 0 physical ends.
 * KFP_SCHEME_SPLIT_FEM: the paper's own scheme: per step, Step 1 solves
 *   (1/tau) M w + S w = (1/tau) M u^n with the consistent P1 mass and stiffness matrices (eq. MMvS),
 *   Step 2 sets u^{n+1}(x, v) = w(x - tau v, v) by linear interpolation, tau = (t_final/nt)/2 in both
 *   (P:452); homogeneous Neumann physical ends; Robin transmission imposed weakly; no
 *   forcing (f_rank must be 0: the paper's error equation); requires tau/h_v^2 > 1/6 and
 *   vmax*tau/h_x <= 1.  Interface errors (err_if) compare the Step-1 results w at the interface nodes;
 *   u(T) and err_T are after the last Step 2. */
typedef enum {
    KFP_SCHEME_IMEX_FD = 0,
    KFP_SCHEME_SPLIT_FEM = 1
} kfp_scheme;

/* Problem description (PAPER.md:33-38 data f, u0, T; grid per DESIGN.md R5/R6).
 * f(t_n, x_m, v_j) = sum_{r<f_rank} ft[r*(nt+1)+n] * fv[r*(nv+1)+j] * fx[r*nx+m]
 * u0(x_m, v_j)     = sum_{r<u0_rank} u0v[r*(nv+1)+j] * u0x[r*nx+m]   (u0_rank = 0: u0 = 0)
 * with x_m = m/nx, v_j = -vmax + j*2*vmax/nv, t_n = n*t_final/nt.
 * Requirements: nx >= 2 and even, nv >= 2 and even, nt >= 1, vmax > 0,
 * t_final > 0, 0 <= f_rank <= 4, 0 <= u0_rank <= 4; tables are host memory. */
typedef struct {
    int32_t nx, nv, nt;
    double vmax, t_final;
    int32_t f_rank;
    const double *ft, *fv, *fx; /* host */
    int32_t u0_rank;
    const double *u0v, *u0x;    /* host */
    int32_t device;             /* CUDA device ordinal */
} kfp_problem_desc;

/* Validate the description, select the device, copy the tables to device
 * memory and create the problem's stream.  KFP_E_INVAL for bad sizes/ranks,
 * KFP_E_CFL if vmax*(t_final/nt)*nx > 1, KFP_E_CUDA if the device is unusable.
 * *out is set only on success. */
kfp_status kfp_problem_create(const kfp_problem_desc *desc, kfp_problem *out);

/* As kfp_problem_create with an explicit discretisation (kfp_problem_create = KFP_SCHEME_IMEX_FD).
 * KFP_SCHEME_SPLIT_FEM additionally returns KFP_E_INVAL for f_rank != 0 or tau/h_v^2 <= 1/6, and
 * KFP_E_CFL for vmax*tau*nx > 1.  Its columns must fit the cluster kernel (<= 4224 unknown rows per
 * subdomain and in the monodomain), else the setup / monodomain call returns KFP_E_INVAL. */
kfp_status kfp_problem_create_ex(const kfp_problem_desc *desc, kfp_scheme scheme, kfp_problem *out);

/* Release the handle and its device buffers (NULL is a no-op).  The buffers go to a process-wide cache
 * keyed by (device, size) after a device synchronisation, and the next problem of the same shape reuses
 * them instead of calling cudaMalloc (cudaFree of a large problem costs milliseconds to ~0.1 s).  An
 * allocation that fails for lack of memory first returns that device's cached buffers to the driver. */
void kfp_problem_destroy(kfp_problem pb);

/* Return every cached device buffer (see kfp_problem_destroy) to the CUDA driver, e.g. before another
 * library needs the memory.  Safe to call at any time; problems that are alive are not affected. */
void kfp_release_cached_memory(void);

/* Run all subsequent work on `stream` (a cudaStream_t on the problem's
 * device, e.g. torch.cuda.current_stream().cuda_stream); NULL restores the
 * problem's own stream. */
kfp_status kfp_set_stream(kfp_problem pb, void *stream);

/* Monodomain solve (the SWR reference, BJ north_star (c)): the same scheme on
 * nodes [0, nv] with the scheme's physical ends (Dirichlet 0; split FEM: Neumann).
 * uT: host [(nv+1)*nx] receiving U(T), or NULL to keep it on the device only. */
kfp_status kfp_monodomain_solve(kfp_problem pb, double *uT);

/* Configure a Jacobi SWR solve and allocate its buffers.
 *  kind     : KFP_DIRICHLET or KFP_ROBIN;  p > 0 required for KFP_ROBIN.
 *  overlap  : overlap in v-cells; subdomain s covers nodes [lo_s, hi_s] with
 *             c_s = s*nv/n_sub, lo_0 = 0, lo_s = c_s - floor(overlap/2),
 *             hi_s = c_{s+1} + ceil(overlap/2), hi_{n_sub-1} = nv (R9).
 *  n_sub    : number of subdomains, nv % n_sub == 0, 0 <= overlap < nv/n_sub - 2.
 *  s_begin, s_end : the contiguous block [s_begin, s_end) of subdomains this
 *             process solves (0, n_sub for a single process); traces across the
 *             block's edges are exchanged by the caller (kfp_swr_edge_buffers).
 *  K_max    : capacity of the error history (K_max >= 1).
 * Runs the monodomain reference if it has not been run for the interface
 * lines this decomposition needs.  Dirichlet with overlap 0 is accepted (it
 * does not converge) and sets a warning in kfp_last_error(). */
kfp_status kfp_swr_setup(kfp_problem pb, kfp_kind kind, double p, int32_t overlap, int32_t n_sub,
                         int32_t s_begin, int32_t s_end, int32_t K_max);

/* Two-sided optimized SWR, OSWR(p, q) (Table 1): every right (hi) end
 * imposes (p + d_v) u = g and every left (lo) end (q - d_v) u = g, with the half-cell rows and
 * traces of DESIGN.md R11; the trace a subdomain sends to its left neighbour uses p, the one it
 * sends right uses q.  p, q > 0 for KFP_ROBIN (ignored for KFP_DIRICHLET); q = p is
 * kfp_swr_setup.  Other arguments, ownership and errors as kfp_swr_setup. */
kfp_status kfp_swr_setup_pq(kfp_problem pb, kfp_kind kind, double p, double q, int32_t overlap, int32_t n_sub,
                            int32_t s_begin, int32_t s_end, int32_t K_max);

/* Iteration schedule of the configured solve (default after every setup: KFP_JACOBI).
 *  KFP_JACOBI       : every subdomain reads the traces of iteration k-1 (the parallel form, Remark P:594-597).
 *  KFP_GAUSS_SEIDEL : the paper's SWR1-SWR4: the subdomains in increasing v, each reading the
 *                     trace its left neighbour wrote in the same iteration and the right neighbour's of k-1.
 *                     Needs all subdomains on this process (s_begin = 0, s_end = n_sub) and a per-step plan;
 *                     KFP_E_INVAL otherwise.  For two subdomains from zero traces, iterate k of subdomain 0
 *                     (1) equals Jacobi iterate 2k-1 (2k). */
kfp_status kfp_swr_set_schedule(kfp_problem pb, kfp_schedule schedule);

/* Reset to iteration 0: zero incoming traces (the initial guess) and
 * clear the error history. */
kfp_status kfp_swr_reset(kfp_problem pb);

/* Initial trace lambda^0 (SWR1 at k = 1; Table 1 uses a random one) of local interface i
 * (between subdomains i and i+1, both on this process) in direction dir: 0 = toward subdomain i's right end,
 * 1 = toward subdomain i+1's left end.  host: [nt][nx] fp64 (row n-1 = t_n), copied.  Must follow
 * kfp_swr_reset (which zeroes them) and precede the first iteration; applies to every replica of a batch. */
kfp_status kfp_swr_set_initial_trace(kfp_problem pb, int32_t i, int32_t dir, const double *host);

/* Run n_iter Jacobi iterations on the local block (each: every local
 * subdomain solves the whole window [0,T] from u0 with the previous
 * iteration's traces, writes its outgoing traces and accumulates its errors;
 * local interfaces are exchanged on the device).  Asynchronous on the
 * problem's stream.  KFP_E_STATE if more than K_max iterations in total, or while a chunked iteration
 * (kfp_swr_iterate_chunk) is in progress. */
kfp_status kfp_swr_iterate(kfp_problem pb, int32_t n_iter);

/* Time-chunked Jacobi iteration for overlapping the cross-GPU trace exchange with compute (step n
 * of iteration k+1 needs only trace row n of iteration k; SURVEY §8(e) "Overlap").  The window's nt steps
 * are split into nchunks chunks, chunk c = steps [c*nt/nchunks, (c+1)*nt/nchunks) = trace rows of the same
 * indices.  kfp_swr_iterate_chunk launches chunk `chunk` of the current iteration on the problem's stream
 * (chunks in order 0..nchunks-1; the last one completes the iteration, like kfp_swr_iterate(pb, 1)); before
 * its first step the stream waits for the event most recently recorded by kfp_swr_chunk_recv_done(chunk)
 * (the previous iteration's incoming edge rows of the chunk), after its last step the library records that
 * the chunk's outgoing edge rows are written.  kfp_swr_chunk_send_wait makes `stream` (a cudaStream_t, e.g.
 * the communication stream) wait for that; kfp_swr_chunk_recv_done records on `stream` that the incoming
 * rows of the chunk have arrived.  Unpipelined Jacobi only (else KFP_E_STATE); KFP_E_INVAL for a bad chunk;
 * KFP_E_STATE for chunks out of order or a changed nchunks inside an iteration.  kfp_swr_reset waits for the
 * last recorded arrivals before it zeroes the incoming traces. */
kfp_status kfp_swr_iterate_chunk(kfp_problem pb, int32_t chunk, int32_t nchunks);
kfp_status kfp_swr_chunk_send_wait(kfp_problem pb, void *stream, int32_t chunk);
kfp_status kfp_swr_chunk_recv_done(kfp_problem pb, void *stream, int32_t chunk);

/* Device pointers of the cross-block exchange buffers, each [nt][nx] fp64
 * (row n-1 = value at t_n), for the parity iteration `k & 1` that the NEXT
 * kfp_swr_iterate call reads: after iteration k the caller must copy the left
 * neighbour block's send_right into recv_left and the right neighbour's
 * send_left into recv_right (NCCL send/recv).  Pointers are NULL where the
 * block touches a physical end.  Parity: buffers written by iteration k are
 * send_*[k & 1]; buffers read by iteration k+1 are recv_*[k & 1]. */
kfp_status kfp_swr_edge_buffers(kfp_problem pb, int32_t parity, double **send_left, double **recv_left,
                                double **send_right, double **recv_right);

/* Replace the library's cross-block exchange buffers of iteration parity
 * `parity` with caller-owned device buffers (e.g. torch tensors that NCCL
 * send/recv use directly), each [nt][nx] fp64; NULL keeps the current buffer.
 * Buffers for a side the block does not have must be NULL.  recv buffers of
 * parity 0 are zeroed by kfp_swr_reset (the zero initial guess). */
kfp_status kfp_swr_bind_edge_buffers(kfp_problem pb, int32_t parity, double *send_left, double *recv_left,
                                     double *send_right, double *recv_right);

/* Convenience: setup(s_begin=0, s_end=n_sub, K_max=K) + reset + iterate(K) on
 * one process.  A latency-bound problem (e.g. BASELINE configs[0] and [1]) iterates pipelined
 * (kfp_swr_set_pipeline(pb, 0), automatic depth): the results are bitwise those of the unpipelined schedule.  uT: host [(nv+1)*nx] receiving u^K(T) assembled by nominal
 * ownership (node j from the subdomain s with c_s <= j < c_{s+1}, node nv from
 * n_sub-1), or NULL. */
kfp_status kfp_swr_solve(kfp_problem pb, kfp_kind kind, double p, int32_t overlap, int32_t n_sub, int32_t K,
                         double *uT);

/* Batched Robin-parameter sweep (the Fig. 1 experiment): n_rep
 * independent replicas of the decomposition, replica r solved with OSWR(ps[r], qs[r]) (qs = NULL: one-sided
 * qs = ps; ignored for KFP_DIRICHLET), all in the same launches.  Single process; the other arguments as
 * kfp_swr_setup.  Then kfp_swr_reset / kfp_swr_iterate / kfp_swr_set_schedule as usual;
 * kfp_error_history and kfp_swr_subdomain_uT report replica 0, the _batch_ calls any replica.
 * ps, qs: host arrays of n_rep doubles, copied. */
kfp_status kfp_swr_setup_batch(kfp_problem pb, kfp_kind kind, const double *ps, const double *qs, int32_t n_rep,
                               int32_t overlap, int32_t n_sub, int32_t K_max);

/* Error history (as kfp_error_history) of replica rep of a batch. */
kfp_status kfp_swr_batch_history(kfp_problem pb, int32_t rep, int32_t cap, int32_t *K_out, double *err_T,
                                 double *err_if);

/* u^k(T) of subdomain s (0 <= s < n_sub) of replica rep, host [(hi_s - lo_s + 1) * nx].  KFP_E_INVAL for a
 * bad rep / s or a setup that does not hold every subdomain (s_begin > 0 or s_end < n_sub); KFP_E_STATE
 * before the first iteration after a setup / reset. */
kfp_status kfp_swr_batch_subdomain_uT(kfp_problem pb, int32_t rep, int32_t s, double *out);

/* kfp_swr_solve with OSWR(p, q) (see kfp_swr_setup_pq). */
kfp_status kfp_swr_solve_pq(kfp_problem pb, kfp_kind kind, double p, double q, int32_t overlap, int32_t n_sub,
                            int32_t K, double *uT);

/* Error history of the iterations run since the last reset, from the local
 * block: err_T[k-1] = max_{s,m, j in [lo_s,hi_s]} |u_s^k(T) - U(T)|,
 * err_if[k-1] = max over s, its interface end nodes (lo_s for s>0, hi_s for
 * s<n_sub-1), n = 1..nt and m of |u_s^k(t_n) - U(t_n)|.  Host arrays of
 * length cap; *K_out = number of iterations run.  KFP_E_STATE before any
 * iteration. */
kfp_status kfp_error_history(kfp_problem pb, int32_t cap, int32_t *K_out, double *err_T, double *err_if);

/* Error quantities an iteration records (per replica, per iteration k = 1..K):
 *  KFP_ERR_T       err_T[k]  = max over every node of every subdomain of |u_s^k(T) - U(T)|;
 *  KFP_ERR_IF      err_if[k] = max over each subdomain's interface end nodes and all steps of |u_s^k - U|;
 *  KFP_ERR_OVERLAP err_ov[k] = max over every closed overlap [lo_{s+1}, hi_s], all steps and x-nodes of
 *                  |u_s^k - u_{s+1}^k| -- the paper's convergence test (eq. 'error'); only with
 *                  kfp_swr_set_overlap_error(pb, 1), only interfaces whose two subdomains are local.
 * (Split FEM: err_if and err_ov use the Step-1 values w, where the transmission conditions act.) */
typedef enum { KFP_ERR_T = 0, KFP_ERR_IF = 1, KFP_ERR_OVERLAP = 2 } kfp_metric;

/* Turn the overlap recording of KFP_ERR_OVERLAP on (1) or off (0) for the current setup.  On first use it
 * allocates, per local interface and side, (hi_s - lo_{s+1} + 1) * nt * nx doubles of device memory; every
 * step then also stores the subdomains' overlap rows (Dirichlet end nodes from the incoming trace), and
 * every iteration ends with one reduction launch.  KFP_E_STATE before a setup; KFP_E_INVAL unless the plan
 * is the per-step cluster kernel (not the three-phase path of columns above 4224 rows). */
kfp_status kfp_swr_set_overlap_error(kfp_problem pb, int32_t on);

/* err_ov history of replica `rep` (0 for an ordinary setup): as kfp_error_history.  KFP_E_STATE if the
 * recording is off or no iteration ran. */
kfp_status kfp_swr_overlap_history(kfp_problem pb, int32_t rep, int32_t cap, int32_t *K_out, double *err_ov);

/* Pipelined Jacobi iterations (the Remark P:594-597): iteration k+1's step n needs
 * only trace row n of iteration k, so one sweep of nt + depth - 1 launches advances `depth` consecutive
 * iterations, slot d running iteration k0 + d at step L - d in launch L.  Results are identical to the
 * unpipelined schedule (bitwise: same per-tile arithmetic); latency-bound small problems gain up to
 * depth x parallelism per launch.  With the Gauss-Seidel schedule (SWR1-SWR4) the same sweep is a
 * wavefront: subdomain s of slot d runs step L - (2 d + s) (its left trace, same iteration, was written
 * one launch earlier by s - 1; its right trace by s + 1 of the previous iteration), so the serial
 * schedule runs its subdomains concurrently; results are again bitwise the unpipelined schedule's.
 * Allocates (depth - 1) extra slabs per subdomain and depth + 1 trace buffers per interface and
 * direction.  depth >= 2 needs a fresh setup (call right after setup / reset), every subdomain on this
 * process, the per-step cluster kernel and no overlap recording -> else KFP_E_INVAL / KFP_E_STATE.
 * kfp_swr_iterate then runs in groups of <= depth iterations (one host synchronisation per group);
 * kfp_last_timing reports per-group windows.  depth 0 = automatic: a latency-bound problem (one step launch
 * fills at most half of the GPU's co-resident cluster slots) gets depth min(K_max, 16, slots / clusters per
 * step), any other problem stays unpipelined; returns KFP_OK without a change where pipelining does not
 * apply (kfp_swr_solve uses this). */
kfp_status kfp_swr_set_pipeline(kfp_problem pb, int32_t depth);

/* Tolerance stopping: run iterations until `metric` of one of them (replica 0) is below eps,
 * or k_max more iterations have run; *k_out = the first iteration (counted since the last reset) that met
 * the tolerance, else the iterations done.  A NaN / infinite error (every error reduction propagates NaN)
 * stops at once and returns KFP_E_NONFINITE with *k_out = that iteration.  Unpipelined: one iteration at a time,
 * one stream synchronisation each (8 bytes read).  Pipelined (kfp_swr_set_pipeline): whole groups of
 * up to depth iterations, so up to depth - 1 iterations beyond *k_out may have run (kfp_error_history
 * and the solution reflect all that ran).  KFP_E_STATE if k_done + k_max > K_max or KFP_ERR_OVERLAP
 * without recording. */
kfp_status kfp_swr_iterate_until(kfp_problem pb, kfp_metric metric, double eps, int32_t k_max, int32_t *k_out);

/* Copy the local subdomain s's current u_s(T) slab [(hi_s-lo_s+1)*nx] to host
 * memory (s is the global subdomain index, s_begin <= s < s_end).  KFP_E_STATE before the first
 * iteration after a setup / reset (the slab would be stale). */
kfp_status kfp_swr_subdomain_uT(kfp_problem pb, int32_t s, double *out);

/* Node range of global subdomain s under the current setup. */
kfp_status kfp_swr_subdomain_range(kfp_problem pb, int32_t s, int32_t *lo, int32_t *hi);

/* Copy the most recent outgoing trace of interface i (between subdomains i and
 * i+1; both must be local) to host memory [nt*nx]: dir 0 = sent leftwards by
 * i+1 (used at hi_i), dir 1 = sent rightwards by i (used at lo_{i+1}). */
kfp_status kfp_swr_trace(kfp_problem pb, int32_t i, int32_t dir, double *out);

/* x-sharded monodomain reference (multi-GPU; BJ.ns (c)).  A job of g processes computes the
 * reference once instead of g times: this process solves only the columns [x0, x1) (whole 32-column tiles:
 * x0 % 32 == 0, x1 % 32 == 0 or x1 == nx), recording U at the node lines[0..nlines) on those columns.  The
 * upwind transport couples a column to its x-neighbours only, so after every kfp_monodomain_shard_step the
 * caller moves send_lo (column x0 of u^{n+1}, all nv+1 nodes) to the process owning column x0 - 1 and
 * send_hi (column x1 - 1) to the one owning x1 (periodic in x), into their recv_hi / recv_lo, on the
 * problem's stream, before the next step; all four are caller-owned device buffers of nv+1 doubles (NULL
 * allowed for the full range [0, nx), which needs no exchange).  shard_end completes the reference: U(T) and
 * the U-lines are then valid on [x0, x1) only; the caller fills the other columns of the rows it needs
 * with kfp_monodomain_shard_copy (dir 0: rows [r0, r1) x columns [xa, xb) of U(T) (what 0, node rows) or
 * of the U-lines (what 1, row = line * nt + step) -> the contiguous device buffer buf [(r1-r0)][(xb-xa)];
 * dir 1: buf -> the reference), after which kfp_swr_setup uses it like its own reference (its lines must
 * be among `lines`).  Bitwise the unsharded reference on every column.  Errors: KFP_E_INVAL for a bad range,
 * missing halo buffers, the split-FEM scheme with a partial range or bad copy bounds; KFP_E_STATE for steps
 * outside [0, nt), shard_end before nt steps, a copy without a reference. */
kfp_status kfp_monodomain_shard_begin(kfp_problem pb, int32_t x0, int32_t x1, const int32_t *lines, int32_t nlines,
                                      double *send_lo, double *send_hi, double *recv_lo, double *recv_hi);
kfp_status kfp_monodomain_shard_step(kfp_problem pb);
kfp_status kfp_monodomain_shard_end(kfp_problem pb);
kfp_status kfp_monodomain_shard_copy(kfp_problem pb, int32_t what, int32_t dir, int32_t r0, int32_t r1, int32_t xa,
                                     int32_t xb, double *buf);

/* Copy the monodomain U(T) [(nv+1)*nx] to host memory. */
kfp_status kfp_monodomain_uT(kfp_problem pb, double *out);

/* Number of this library's kernels launched since creation (for the bench's
 * gpu_launches claim) and a short description of the selected launch plan. */
int64_t kfp_launch_count(kfp_problem pb);
const char *kfp_plan(kfp_problem pb);

/* Device time in milliseconds of the most recent kfp_swr_iterate call and of
 * the step kernels inside it, measured with CUDA events on the problem's
 * stream (synchronises).  *kernel_ms may be NULL. */
kfp_status kfp_last_timing(kfp_problem pb, double *iterate_ms, double *kernel_ms);

const char *kfp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* KFP_H */

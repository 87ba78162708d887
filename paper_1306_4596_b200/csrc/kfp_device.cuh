// kfp_device.cuh -- sm_100a device code of the SWR solver (arXiv 1306.4596).
//
// One launch of a "step" kernel advances every local subdomain by one time
// step t_n -> t_{n+1} of the scheme of PAPER.md:449-516 as fixed by DESIGN.md
// (transport first, full dt, readings R1-R8):
//
//   r_j   = (1-|nu_j|) u^n_j + |nu_j| u^n_{j, m-+1} + dt f(t_{n+1}, x_m, v_j)
//   A u^{n+1} = r   with A = tridiag(-a, 1+2a, -a) plus Dirichlet/Robin end rows
//
// The per-column tridiagonal solve is NOT the textbook Thomas recurrence (whose
// per-row factors form one long serial chain per column).  It uses the
// constant-coefficient factorisation of the Toeplitz part:
//
//   T_n = B + a q e_0 e_0^T,  B = (a/q) (I - q E_down)(I - q E_up),
//   q = ((1+2a) - sqrt(1+4a)) / (2a)  (the root of a q^2 - (1+2a) q + a = 0),
//   A   = B + e_0 d_t^T + e_{n-1} d_b^T                     (rank-2 boundary part),
//
// so that x = B^{-1}(r - c0 e_0 - c1 e_{n-1}) with the 2-vector c from a 2x2
// Woodbury system.  B^{-1} is a forward then a backward first-order linear
// recurrence with the single constant q, which parallelises along v by
// chunks: every warp owns a chunk of rows of 32 x-columns (lane = column),
// scans it locally from zero, and the chunk carries are resolved afterwards
// (a chain over chunks in the CTA and over CTAs in the column) with powers of
// q.  The two boundary values c0, c1 enter as the carries entering the top
// (y_{-1} = -c0/a) and the bottom (x_n = -c1/a) of the column.
//
// Per update the kernel moves 16 B of HBM (read u^n, write u^{n+1}); every
// other quantity (forcing, u0, transport and Thomas coefficients) comes from
// O(N_x + N_v) tables.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace kfp {
namespace cg = cooperative_groups;

constexpr int kWarp = 32;
constexpr int kMaxRank = 4;
constexpr int kMaxWarps = 16;
constexpr int kMaxCluster = 16;
// END_NEU: homogeneous Neumann physical end of the split-FEM scheme -- an unknown end row
// like END_ROBIN with p = 0 and no incoming trace
enum : int { END_PHYS = 0, END_DIRI = 1, END_ROBIN = 2, END_NEU = 3 };

// One subdomain as the kernels see it (global index s, nodes [lo, hi]).
struct SubDev {
    int lo, hi;        // node range
    int first, n;      // first unknown node, number of unknown rows
    int ltype, rtype;  // END_* of the lo / hi end
    int iL_tr, iR_tr;  // unknown-row index of the node sent left (hi_{s-1}) / right (lo_{s+1}); -2 none,
                       // -1 / n: the Dirichlet end node itself (no overlap)
    int ifL, ifR;      // U-line index of the lo / hi interface end node for err_if; -1 none
    int nblk;          // row blocks in use (<= C)
    int grp;           // replica (batched parameter sweep): error slots errT/errIF + grp * err_stride
    double injL, injR;           // RHS weight of the incoming trace: a (Dirichlet) or 2 a h_v (Robin)
    double wt0, wt1, wb0, wb1;   // d_t (rows 0,1) and d_b (rows n-2, n-1)
    double Mi00, Mi01, Mi10, Mi11;  // (I_2 + D^T B^{-1} E)^{-1}
    double *slab[2];             // [(hi-lo+1)][nx], ping-pong by step parity
    const double *gL[2], *gR[2]; // incoming traces [nt][nx] by iteration parity
    double *sendL[2], *sendR[2]; // outgoing traces [nt][nx] by iteration parity
    double tpL, tpR;             // Robin parameter of the trace sent left (p: it lands on a right end) and right (q)
    // overlap recording (the paper's stopping rule, eq. 'error' P:588-592; opt-in): side 0 = the nodes
    // [lo_s, hi_{s-1}] shared with s-1, side 1 = [lo_{s+1}, hi_s] shared with s+1; ovn = 0: not recorded
    int ovr0[2], ovn[2];         // first node, node count
    double *ovb[2];              // [ovn][nt][nx] this subdomain's values there (u; split FEM: w)
    // pipelined Jacobi iterations: this descriptor runs step P.n - lag of its
    // iteration; outside [0, nt) the CTA exits (pipeline fill / drain).  0 otherwise.
    int lag;
    // rows [wlo, whi) of the column are stored (whi == 0: every row).  A tall monodomain column is solved as
    // overlapping segments (kfp_api.cu mono_segments): each writes only its interior rows.
    int wlo, whi, pad_;
};
static_assert(sizeof(SubDev) % 16 == 0, "SubDev arrays are copied with cp.async.bulk (16-B granules)");

struct StepParams {
    const SubDev *subs;
    int nx, nv, nt;
    int n;                 // this launch computes level n+1
    int par_in, par_out;   // iteration parities of the traces read / written
    int err_stride;        // error slots per replica (K_max)
    int par_in_lo;         // parity of the incoming LEFT trace: par_in (Jacobi) or par_out
                           // (Gauss-Seidel SWR1-SWR4: the left neighbour already ran this iteration)
    int from_u0;           // n == 0: u^0 from the u0 tables (no slab read)
    int last;              // n+1 == nt (the cluster kernel: "errors at T wanted" -- it tests step == nt-1 itself)
    int send_robin;        // outgoing trace kind: 0 Dirichlet value, 1 Robin combination
    int f_rank, u0_rank;
    int P, b, R, C;        // warps per CTA, rows per chunk, rows per block, blocks per column
    int qtab_len;
    int tile0, xend;       // x-columns [32 tile0, xend) of this launch (a sharded monodomain); 0, nx otherwise
    int record;            // monodomain: record rows listed in line_of_node
    int ovrec;             // record the overlap rows into SubDev::ovb (cluster kernel only)
    double q, a, qa, hv, dt, p;   // split FEM: a = tau/h_v^2 - 1/6, dt = tau
    double dnu, nu0;       // split FEM transport weight of node j: |j dnu + nu0| = |v_j| tau / h_x (0 at n = 0)
    double cf[kMaxRank];   // dt * ft[r][n+1] of this launch's step (the cluster kernel's forcing weights)
    const double *cfn;     // [nt][kMaxRank] dt * ft[r][n+1] per step (cluster kernel: steps differ per slot)
    const double2 *rowc;   // per node: (1-|nu_j|, |nu_j|)
    const double *fv;      // [f_rank][nv+1]
    const double *fx;      // [f_rank][nx]
    const double *u0v;     // [u0_rank][nv+1]
    const double *u0x;     // [u0_rank][nx]
    const double *qp;      // q^k, k < qtab_len
    const double *s2;      // sum_{t<k} q^{2t}, k < qtab_len
    unsigned long long *errT, *errIF;  // this iteration's error slots (bit patterns of doubles >= 0)
    const double *UT;                  // monodomain U(T)
    const double *Ulines;              // [nlines][nt][nx]
    const int *line_of_node;           // [nv+1], -1 none
    double *rec;                       // [nlines][nt][nx] (monodomain recording)
    // general (non-cluster) path scratch
    double *blkagg;   // [sub][blk][6][nx]   F, G, a0..a3
    double *chkagg;   // [sub][blk][P][2][nx] he, ks
    double *carry;    // [sub][blk][2][nx]   Y_in, X_in of the block
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// The waiting thread may be suspended (up to the hint, 1 ms) instead of spinning, so that a
// co-resident CTA gets the issue slots; it resumes when the phase completes.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// Bulk asynchronous copy global -> shared (TMA engine, no tensor map);
// bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// st.global through a generic pointer known to address global memory (the slabs)
__device__ __forceinline__ void st_global_f64(double *p, double v) {
    asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ void st_cs(double *p, double v) {  // streaming store (evict-first)
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void atomic_max_pos(unsigned long long *addr, double v) {
    // v >= 0 or NaN: the IEEE bit pattern orders like an unsigned integer, and every NaN pattern
    // (|v| of a NaN: 0x7ff8...) is above +inf, so a NaN error survives the reduction.
    atomicMax(addr, static_cast<unsigned long long>(__double_as_longlong(v)));
}
// max that propagates NaN from either side (fmax drops it: a solve that blew up must not report
// a finite error)
__device__ __forceinline__ double nmax(double a, double b) { return (a > b || a != a) ? a : b; }
// an error worth an atomic: positive, or NaN
__device__ __forceinline__ bool err_pos(double v) { return !(v <= 0.0); }
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------------ sharded monodomain halo columns
// Column m of every node row of a node-major slab [(nv+1)][nx] <-> a contiguous [(nv+1)] buffer (the x-halo of
// an x-sharded monodomain reference, exchanged between processes every step).  grid ceil((nv+1)/256).
__global__ void __launch_bounds__(256) halo_pack(const double *slab, int nx, int rows, int m, double *out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < rows) out[j] = slab[static_cast<size_t>(j) * nx + m];
}
__global__ void __launch_bounds__(256) halo_unpack(double *slab, int nx, int rows, int m, const double *in) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < rows) slab[static_cast<size_t>(j) * nx + m] = in[j];
}

// ------------------------------------------------------------------ geometry of one CTA
struct Tile {
    const SubDev *sd;
    int sub;        // local subdomain index (blockIdx.z)
    int m0, w;      // first column, columns in this tile (<= 32)
    int blk;        // row block index within the column
    int rb0, Rb;    // first unknown row of the block, rows in block
    int warp, lane;
    int r0, L;      // first row of this warp's chunk within the block, chunk length (may be 0)
    int m;          // this lane's column (valid if lane < w)
};

__device__ __forceinline__ Tile make_tile(const StepParams &P, int blk) {
    Tile t;
    t.sub = blockIdx.z;
    t.sd = P.subs + t.sub;
    t.m0 = (P.tile0 + blockIdx.y) * kWarp;
    t.w = min(kWarp, P.xend - t.m0);
    t.blk = blk;
    t.rb0 = blk * P.R;
    t.Rb = max(0, min(P.R, t.sd->n - t.rb0));
    t.warp = threadIdx.x >> 5;
    t.lane = threadIdx.x & 31;
    t.r0 = t.warp * P.b;
    t.L = max(0, min(P.b, t.Rb - t.r0));
    t.m = t.m0 + min(t.lane, t.w - 1);
    return t;
}

// kap(l, L) = sum_{t=l}^{L-1} q^{t-l} q^{t+1} = q^{l+1} * s2[L-l]:
// response of the local backward scan at local row l to a forward carry entering the chunk.
__device__ __forceinline__ double kapf(const double *qp, const double *s2, int l, int L) {
    return qp[l + 1] * s2[L - l];
}

// Issue the bulk copies of this warp's chunk rows [t.r0, t.r0+t.L) of `src`
// (slab rows relative to the node `first`) into the tile buffer.
__device__ __forceinline__ void load_chunk(const StepParams &P, const Tile &t, const double *src_rows,
                                           double *tile, uint64_t *bar) {
    if (t.L == 0) return;
    const uint32_t rowbytes = static_cast<uint32_t>(t.w) * 8u;
    if (t.lane == 0) mbar_expect_tx(bar, rowbytes * t.L);
    __syncwarp();
    for (int l = t.lane; l < t.L; l += kWarp) {
        const int i = t.rb0 + t.r0 + l;  // unknown row
        bulk_g2s(tile + (t.r0 + l) * kWarp, src_rows + static_cast<size_t>(i) * P.nx + t.m0, rowbytes, bar);
    }
}

// Pass A: transport + forcing + boundary injection, forward local scan
// h_i = q h_{i-1} + (q/a) r_i (zero carry), in place over the tile.
// Also: Dirichlet-end interface error, raw r at the outgoing trace rows,
// end-node rows of the slab at the last step.
__device__ __forceinline__ void pass_a(const StepParams &P, const Tile &t, double *tile, const double *uold_rows,
                                       double *unew_slab, double *rtr, double &err_if, double &err_t,
                                       double &h_end) {
    const SubDev &S = *t.sd;
    const int lane = t.lane;
    const bool active = lane < t.w;
    double fx[kMaxRank], u0x[kMaxRank], u0xl[kMaxRank], u0xr[kMaxRank];
    const int mL = (t.m0 + P.nx - 1) % P.nx;        // left halo column (lane 0)
    const int mR = (t.m0 + t.w) % P.nx;             // right halo column (lane w-1)
#pragma unroll
    for (int r = 0; r < kMaxRank; ++r) {
        fx[r] = (r < P.f_rank) ? __ldg(P.fx + r * P.nx + t.m) : 0.0;
        if (P.from_u0) {
            u0x[r] = (r < P.u0_rank) ? __ldg(P.u0x + r * P.nx + t.m) : 0.0;
            u0xl[r] = (r < P.u0_rank) ? __ldg(P.u0x + r * P.nx + mL) : 0.0;
            u0xr[r] = (r < P.u0_rank) ? __ldg(P.u0x + r * P.nx + mR) : 0.0;
        }
    }
    // Halo prefetch: lane l holds the halo of chunk row l and l+32 (for the
    // side its row's sign of v needs); broadcast by shuffle inside the loop.
    double halo0 = 0.0, halo1 = 0.0;
    if (!P.from_u0) {
        for (int hpass = 0; hpass < 2; ++hpass) {
            const int l = lane + hpass * kWarp;
            if (l < t.L) {
                const int j = S.first + t.rb0 + t.r0 + l;
                const double2 rc = __ldg(P.rowc + j);
                double hv = 0.0;
                if (rc.y != 0.0) {
                    const int jv2 = 2 * j - P.nv;  // sign of v_j
                    const int mm = (jv2 > 0) ? mL : mR;
                    hv = __ldg(uold_rows + static_cast<size_t>(j - S.first) * P.nx + mm);
                }
                if (hpass == 0) halo0 = hv; else halo1 = hv;
            }
        }
    }
    double h = 0.0;
    const int i0 = t.rb0 + t.r0;
    for (int l = 0; l < t.L; ++l) {
        const int i = i0 + l;
        const int j = S.first + i;
        const double2 rc = __ldg(P.rowc + j);
        double u, nb;
        const int jv2 = 2 * j - P.nv;
        if (P.from_u0) {
            double s = 0.0, sl = 0.0, sr = 0.0;
#pragma unroll
            for (int r = 0; r < kMaxRank; ++r)
                if (r < P.u0_rank) {
                    const double vv = __ldg(P.u0v + r * (P.nv + 1) + j);
                    s = fma(vv, u0x[r], s);
                    sl = fma(vv, u0xl[r], sl);
                    sr = fma(vv, u0xr[r], sr);
                }
            u = s;
            const double up = __shfl_up_sync(0xffffffffu, u, 1);
            const double dn = __shfl_down_sync(0xffffffffu, u, 1);
            nb = (jv2 > 0) ? (lane == 0 ? sl : up) : (lane == t.w - 1 ? sr : dn);
        } else {
            u = tile[(t.r0 + l) * kWarp + lane];
            const double up = __shfl_up_sync(0xffffffffu, u, 1);
            const double dn = __shfl_down_sync(0xffffffffu, u, 1);
            const double hb = __shfl_sync(0xffffffffu, (l < kWarp) ? halo0 : halo1, l & 31);
            nb = (jv2 > 0) ? (lane == 0 ? hb : up) : (lane == t.w - 1 ? hb : dn);
        }
        // forcing dt*f(t_{n+1}, x_m, v_j)
        double f = 0.0;
#pragma unroll
        for (int r = 0; r < kMaxRank; ++r)
            if (r < P.f_rank) f = fma(P.cf[r] * __ldg(P.fv + r * (P.nv + 1) + j), fx[r], f);
        double rr = fma(rc.x, u, fma(rc.y, nb, f));
        // r_c of the outgoing Robin trace is the O1 right-hand side without the incoming trace term
        if (i == S.iL_tr) rtr[lane] = rr;
        if (i == S.iR_tr) rtr[kWarp + lane] = rr;
        if (i == 0 && S.ltype != END_PHYS) {
            const double g = S.gL[P.par_in_lo][static_cast<size_t>(P.n) * P.nx + t.m];
            rr = fma(S.injL, g, rr);
            if (S.ltype == END_DIRI && S.iL_tr == -1 && active)  // Dirichlet, no overlap: the end node is the trace node
                S.sendL[P.par_out][static_cast<size_t>(P.n) * P.nx + t.m] = g;
            if (S.ltype == END_DIRI && active) {
                if (S.ifL >= 0)
                    err_if = nmax(err_if, fabs(g - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + P.n) * P.nx + t.m]));
                if (P.last) {
                    err_t = nmax(err_t, fabs(g - P.UT[static_cast<size_t>(S.lo) * P.nx + t.m]));
                    unew_slab[t.m] = g;
                }
            }
        }
        if (i == S.n - 1 && S.rtype != END_PHYS) {
            const double g = S.gR[P.par_in][static_cast<size_t>(P.n) * P.nx + t.m];
            rr = fma(S.injR, g, rr);
            if (S.rtype == END_DIRI && S.iR_tr == S.n && active)
                S.sendR[P.par_out][static_cast<size_t>(P.n) * P.nx + t.m] = g;
            if (S.rtype == END_DIRI && active) {
                if (S.ifR >= 0)
                    err_if = nmax(err_if, fabs(g - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + P.n) * P.nx + t.m]));
                if (P.last) {
                    err_t = nmax(err_t, fabs(g - P.UT[static_cast<size_t>(S.hi) * P.nx + t.m]));
                    unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + t.m] = g;
                }
            }
        }
        if (P.last) {  // physical ends hold 0 at T
            if (i == 0 && S.ltype == END_PHYS && active) unew_slab[t.m] = 0.0;
            if (i == S.n - 1 && S.rtype == END_PHYS && active) unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + t.m] = 0.0;
        }
        h = fma(P.q, h, P.qa * rr);
        tile[(t.r0 + l) * kWarp + lane] = h;
    }
    h_end = h;
}

// Pass B: backward local scan k_i = q k_{i+1} + h_i (zero carry), in place.
__device__ __forceinline__ double pass_b(const StepParams &P, const Tile &t, double *tile) {
    double k = 0.0;
    for (int l = t.L - 1; l >= 0; --l) {
        double *p = tile + (t.r0 + l) * kWarp + t.lane;
        k = fma(P.q, k, *p);
        *p = k;
    }
    return k;
}

// Level 1 with zero block carries: chain over the P chunks of the block.
// Inputs he[w], ks[w] (smem, per lane); writes Y0[w], X0[w]; returns the
// block aggregates F (y at the block's last row) and G (x at its first row)
// and the zero-carry values of the boundary rows 0,1,n-2,n-1 held by the block.
struct BlockAgg {
    double F, G, ab[4];
};

__device__ __forceinline__ BlockAgg level1_zero(const StepParams &P, const Tile &t, const double *tile,
                                                const double *he, const double *ks, double *Y0, double *X0) {
    const int lane = t.lane;
    BlockAgg g;
    double Y = 0.0;
    int nw = 0;
    for (int w = 0; w < P.P; ++w) {
        const int L = max(0, min(P.b, t.Rb - w * P.b));
        if (L == 0) break;
        Y0[w * kWarp + lane] = Y;
        Y = fma(P.qp[L], Y, he[w * kWarp + lane]);
        nw = w + 1;
    }
    g.F = Y;
    double X = 0.0;
    for (int w = nw - 1; w >= 0; --w) {
        const int L = min(P.b, t.Rb - w * P.b);
        X0[w * kWarp + lane] = X;
        X = fma(P.qp[L], X, fma(kapf(P.qp, P.s2, 0, L), Y0[w * kWarp + lane], ks[w * kWarp + lane]));
    }
    g.G = X;
    const int n = t.sd->n;
    const int brow[4] = {0, 1, n - 2, n - 1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int li = brow[q] - t.rb0;  // row within block
        g.ab[q] = 0.0;
        if (brow[q] >= 0 && li >= 0 && li < t.Rb) {
            const int w = li / P.b, l = li - w * P.b;
            const int L = min(P.b, t.Rb - w * P.b);
            g.ab[q] = tile[li * kWarp + lane] + kapf(P.qp, P.s2, l, L) * Y0[w * kWarp + lane] +
                      P.qp[L - l] * X0[w * kWarp + lane];
        }
    }
    return g;
}

// Level 2: given every block's (F, G) and the boundary-row partial values,
// resolve the Woodbury boundary terms and return this block's carries
// (Y_in: forward carry entering its first row; X_in: x just below its last row).
// Fn(c), Gn(c), Ab(q) are accessors (DSMEM or global).
template <class FF, class GG, class AA>
__device__ __forceinline__ void level2(const StepParams &P, const SubDev &S, int nblk, int me, FF Fn, GG Gn, AA Ab,
                                       double &Yme, double &Xme) {
    const int n = S.n;
    auto Rc = [&](int c) { return min(P.R, n - c * P.R); };
    const int brow[4] = {0, 1, n - 2, n - 1};
    double Fv[kMaxCluster], Gv[kMaxCluster], Yarr[kMaxCluster];
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
        if (c < nblk) {
            Fv[c] = Fn(c);
            Gv[c] = Gn(c);
        }
    // zero-boundary chain (Y_top = X_bot = 0)
    double yb[4] = {0, 0, 0, 0}, xb[4] = {0, 0, 0, 0};
    double Y = 0.0;
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
        if (c < nblk) {
            Yarr[c] = Y;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (brow[q] / P.R == c) yb[q] = Y;
            Y = fma(P.qp[Rc(c)], Y, Fv[c]);
        }
    double X = 0.0;
#pragma unroll
    for (int c = kMaxCluster - 1; c >= 0; --c)
        if (c < nblk) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (brow[q] / P.R == c) xb[q] = X;
            X = fma(P.qp[Rc(c)], X, fma(kapf(P.qp, P.s2, 0, Rc(c)), Yarr[c], Gv[c]));
        }
    // x~ (zero top/bottom carries) at rows 0, 1, n-2, n-1
    double xt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int c = brow[q] / P.R, l = brow[q] - c * P.R, R = Rc(c);
        xt[q] = Ab(q) + kapf(P.qp, P.s2, l, R) * yb[q] + P.qp[R - l] * xb[q];
    }
    // Woodbury: c = M^{-1} D^T x~, then y_{-1} = -c0/a, x_n = -c1/a
    const double s0 = S.wt0 * xt[0] + S.wt1 * xt[1];
    const double s1 = S.wb0 * xt[2] + S.wb1 * xt[3];
    const double c0 = S.Mi00 * s0 + S.Mi01 * s1;
    const double c1 = S.Mi10 * s0 + S.Mi11 * s1;
    Y = -c0 / P.a;
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
        if (c < nblk) {
            Yarr[c] = Y;
            Y = fma(P.qp[Rc(c)], Y, Fv[c]);
        }
    X = -c1 / P.a;
#pragma unroll
    for (int c = kMaxCluster - 1; c >= 0; --c)
        if (c < nblk && c > me) X = fma(P.qp[Rc(c)], X, fma(kapf(P.qp, P.s2, 0, Rc(c)), Yarr[c], Gv[c]));
    Yme = 0.0;
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
        if (c == me) Yme = Yarr[c];
    Xme = X;
}

// Level 1 with the block's real carries: per-chunk carries into Yc[w], Xc[w].
__device__ __forceinline__ void level1_carry(const StepParams &P, const Tile &t, const double *he, const double *ks,
                                             double Yin, double Xin, double *Yc, double *Xc) {
    const int lane = t.lane;
    int nw = 0;
    double Y = Yin;
    for (int w = 0; w < P.P; ++w) {
        const int L = max(0, min(P.b, t.Rb - w * P.b));
        if (L == 0) break;
        Yc[w * kWarp + lane] = Y;
        Y = fma(P.qp[L], Y, he[w * kWarp + lane]);
        nw = w + 1;
    }
    double X = Xin;
    for (int w = nw - 1; w >= 0; --w) {
        const int L = min(P.b, t.Rb - w * P.b);
        Xc[w * kWarp + lane] = X;
        X = fma(P.qp[L], X, fma(kapf(P.qp, P.s2, 0, L), Yc[w * kWarp + lane], ks[w * kWarp + lane]));
    }
}

// Pass C: x_i = k_i + kap_l Y + q^{L-l} X; store u^{n+1}; errors; trace rows; line recording.
__device__ __forceinline__ void pass_c(const StepParams &P, const Tile &t, const double *tile, double Y, double X,
                                       double *unew_rows, double *xtr, double &err_if, double &err_t) {
    const SubDev &S = *t.sd;
    const bool active = t.lane < t.w;
    const int i0 = t.rb0 + t.r0;
    for (int l = t.L - 1; l >= 0; --l) {
        const int i = i0 + l;
        const int j = S.first + i;
        const double x = tile[(t.r0 + l) * kWarp + t.lane] + kapf(P.qp, P.s2, l, t.L) * Y + P.qp[t.L - l] * X;
        if (active) st_cs(unew_rows + static_cast<size_t>(i) * P.nx + t.m, x);
        if (P.last && active) err_t = nmax(err_t, fabs(x - P.UT[static_cast<size_t>(j) * P.nx + t.m]));
        if (active && i == 0 && S.ltype == END_ROBIN && S.ifL >= 0)
            err_if = nmax(err_if, fabs(x - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + P.n) * P.nx + t.m]));
        if (active && i == S.n - 1 && S.rtype == END_ROBIN && S.ifR >= 0)
            err_if = nmax(err_if, fabs(x - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + P.n) * P.nx + t.m]));
        if (S.iL_tr >= 0) {
            if (i == S.iL_tr) xtr[0 * kWarp + t.lane] = x;
            if (i == S.iL_tr + 1) xtr[1 * kWarp + t.lane] = x;
        }
        if (S.iR_tr >= 0) {
            if (i == S.iR_tr) xtr[2 * kWarp + t.lane] = x;
            if (i == S.iR_tr - 1) xtr[3 * kWarp + t.lane] = x;
        }
        if (P.record) {
            const int li = __ldg(P.line_of_node + j);
            if (li >= 0 && active) P.rec[(static_cast<size_t>(li) * P.nt + P.n) * P.nx + t.m] = x;
        }
    }
}

// Outgoing traces at t_{n+1} (R11): warp 0 of the block
// holding the trace rows.
__device__ __forceinline__ void write_traces(const StepParams &P, const Tile &t, const double *rtr, const double *xtr) {
    const SubDev &S = *t.sd;
    if (t.lane >= t.w) return;
    const size_t off = static_cast<size_t>(P.n) * P.nx + t.m;
    const double inv_h = 1.0 / P.hv, half_h_dt = 0.5 * P.hv / P.dt;
    if (S.iL_tr >= 0 && S.iL_tr >= t.rb0 && S.iL_tr < t.rb0 + t.Rb) {
        const double uc = xtr[t.lane];
        double g = uc;
        if (P.send_robin) {  // (p + d_v) u with the half-cell flux on [c, c+h/2]
            const double up = xtr[kWarp + t.lane];
            g = t.sd->tpL * uc - ((uc - up) * inv_h + half_h_dt * (uc - rtr[t.lane]));
        }
        S.sendL[P.par_out][off] = g;
    }
    if (S.iR_tr >= 0 && S.iR_tr >= t.rb0 && S.iR_tr < t.rb0 + t.Rb) {
        const double uc = xtr[2 * kWarp + t.lane];
        double g = uc;
        if (P.send_robin) {  // (q - d_v) u with the half-cell flux on [c-h/2, c]
            const double um = xtr[3 * kWarp + t.lane];
            g = t.sd->tpR * uc - ((uc - um) * inv_h + half_h_dt * (uc - rtr[kWarp + t.lane]));
        }
        S.sendR[P.par_out][off] = g;
    }
}

// Shared-memory layout of one CTA (dynamic smem).
struct Smem {
    double *tile;   // [R][32]
    double *he, *ks, *Y0, *X0;  // [P][32]
    double *pub;    // [6][32]: F, G, a0..a3 (read by the cluster)
    double *rtr;    // [2][32]
    double *xtr;    // [4][32]
    double *red;    // [2][kMaxWarps]
    uint64_t *bar;  // [P]
};
__host__ __device__ inline size_t smem_bytes(int R, int Pw) {
    return sizeof(double) * (static_cast<size_t>(R) * kWarp + 4 * Pw * kWarp + 6 * kWarp + 2 * kWarp + 4 * kWarp +
                             2 * kMaxWarps) +
           sizeof(uint64_t) * kMaxWarps + 16;
}
__device__ __forceinline__ Smem carve(char *base, int R, int Pw) {
    Smem s;
    double *d = reinterpret_cast<double *>(base);
    s.tile = d; d += R * kWarp;
    s.he = d; d += Pw * kWarp;
    s.ks = d; d += Pw * kWarp;
    s.Y0 = d; d += Pw * kWarp;
    s.X0 = d; d += Pw * kWarp;
    s.pub = d; d += 6 * kWarp;
    s.rtr = d; d += 2 * kWarp;
    s.xtr = d; d += 4 * kWarp;
    s.red = d; d += 2 * kMaxWarps;
    s.bar = reinterpret_cast<uint64_t *>(d);
    return s;
}

__device__ __forceinline__ void block_err_flush(const StepParams &P, const Tile &t, Smem &sm, double eif, double et) {
    eif = warp_max(eif);
    et = warp_max(et);
    if (t.lane == 0) {
        sm.red[t.warp] = eif;
        sm.red[kMaxWarps + t.warp] = et;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < P.P; ++w) {
            a = nmax(a, sm.red[w]);
            b = nmax(b, sm.red[kMaxWarps + w]);
        }
        const size_t go = static_cast<size_t>(t.sd->grp) * P.err_stride;
        if (err_pos(a) && P.errIF) atomic_max_pos(P.errIF + go, a);
        if (err_pos(b) && P.errT) atomic_max_pos(P.errT + go, b);
    }
}

// ------------------------------------------------------------------ kernels

// General path, phase 1: passes A and B on one row block; the scanned values
// k go to the new slab (in place), block and chunk aggregates to global.
__global__ void __launch_bounds__(kMaxWarps * kWarp) step_phase1(const StepParams P) {
    extern __shared__ __align__(128) char smraw[];
    Tile t = make_tile(P, blockIdx.x);
    const SubDev &S = *t.sd;
    if (t.Rb == 0) return;
    Smem sm = carve(smraw, P.R, P.P);
    const double *uold = S.slab[P.n & 1] + static_cast<size_t>(S.first - S.lo) * P.nx;
    double *unew_slab = S.slab[(P.n + 1) & 1];
    double *unew = unew_slab + static_cast<size_t>(S.first - S.lo) * P.nx;
    if (t.lane == 0 && t.warp < P.P) mbar_init(&sm.bar[t.warp], 1);
    fence_mbar_init();
    __syncwarp();
    if (!P.from_u0 && t.warp < P.P) load_chunk(P, t, uold, sm.tile, &sm.bar[t.warp]);
    double eif = 0.0, et = 0.0, hend = 0.0, kst = 0.0;
    if (t.warp < P.P && t.L > 0) {
        if (!P.from_u0) mbar_wait(&sm.bar[t.warp], 0);
        pass_a(P, t, sm.tile, uold, unew_slab, sm.rtr, eif, et, hend);
        kst = pass_b(P, t, sm.tile);
        // k to the new slab (re-read in phase 3)
        if (t.lane < t.w)
            for (int l = 0; l < t.L; ++l)
                unew[static_cast<size_t>(t.rb0 + t.r0 + l) * P.nx + t.m] = sm.tile[(t.r0 + l) * kWarp + t.lane];
    }
    if (t.warp < P.P) {
        sm.he[t.warp * kWarp + t.lane] = hend;
        sm.ks[t.warp * kWarp + t.lane] = kst;
        const size_t base = ((static_cast<size_t>(t.sub) * P.C + t.blk) * P.P + t.warp) * 2 * P.nx;
        if (t.lane < t.w) {
            P.chkagg[base + t.m] = hend;
            P.chkagg[base + P.nx + t.m] = kst;
        }
    }
    // raw r at the trace rows to global (phase 3 needs it): stash in blkagg slots 6,7
    __syncthreads();
    if (t.warp == 0) {
        BlockAgg g = level1_zero(P, t, sm.tile, sm.he, sm.ks, sm.Y0, sm.X0);
        const size_t base = (static_cast<size_t>(t.sub) * P.C + t.blk) * 8 * P.nx;
        if (t.lane < t.w) {
            P.blkagg[base + 0 * P.nx + t.m] = g.F;
            P.blkagg[base + 1 * P.nx + t.m] = g.G;
#pragma unroll
            for (int q = 0; q < 4; ++q) P.blkagg[base + (2 + q) * P.nx + t.m] = g.ab[q];
            if (S.iL_tr >= t.rb0 && S.iL_tr < t.rb0 + t.Rb) P.blkagg[base + 6 * P.nx + t.m] = sm.rtr[t.lane];
            if (S.iR_tr >= t.rb0 && S.iR_tr < t.rb0 + t.Rb) P.blkagg[base + 7 * P.nx + t.m] = sm.rtr[kWarp + t.lane];
        }
    }
    block_err_flush(P, t, sm, eif, et);
}

// General path, phase 2, warp per column: the same algebra as step_phase2, with the block recurrences
//   Y_{c+1} = q^{R_c} Y_c + F_c            (forward, Y_0 given)
//   X_c     = q^{R_c} X_{c+1} + kap(0, R_c) Y_c + G_c   (backward, X_nblk given)
// evaluated as affine scans over the blocks: lane i owns a segment of ceil(nblk / 32) consecutive blocks,
// composes its segment's affine map, a Kogge-Stone shuffle scan gives every segment its incoming value,
// and the lane replays its segment.  Two sweeps: zero carries (for the Woodbury end terms), then the
// final carries.  For tall columns (many blocks) this replaces a serial per-thread chain.
__device__ __forceinline__ void p2w_sweep(const StepParams &P, int sub, int m, int lane, int nblk, int n, double yinit,
                                          double xinit, bool final_pass, double (&yb)[4], double (&xb)[4]) {
    const int per = (nblk + kWarp - 1) / kWarp, c0 = min(nblk, lane * per), c1 = min(nblk, c0 + per);
    const int brow[4] = {0, 1, n - 2, n - 1};
    auto Bv = [&](int c, int slot) { return P.blkagg[((static_cast<size_t>(sub) * P.C + c) * 8 + slot) * P.nx + m]; };
    auto Rc = [&](int c) { return min(P.R, n - c * P.R); };
    double *car = P.carry + static_cast<size_t>(sub) * P.C * 2 * P.nx + m;  // [c][2][nx]
    // forward: segment map, inclusive scan (lower lanes first), exclusive incoming value
    double a = 1.0, b = 0.0;
    for (int c = c0; c < c1; ++c) {
        const double qr = P.qp[Rc(c)];
        a *= qr;
        b = fma(qr, b, Bv(c, 0));
    }
    for (int d = 1; d < kWarp; d <<= 1) {
        const double au = __shfl_up_sync(0xffffffffu, a, d), bu = __shfl_up_sync(0xffffffffu, b, d);
        if (lane >= d) {
            b = fma(a, bu, b);
            a *= au;
        }
    }
    double ain = __shfl_up_sync(0xffffffffu, a, 1), bin = __shfl_up_sync(0xffffffffu, b, 1);
    if (lane == 0) {
        ain = 1.0;
        bin = 0.0;
    }
    double Y = fma(ain, yinit, bin);
    for (int c = c0; c < c1; ++c) {
        for (int q = 0; q < 4; ++q)
            if (brow[q] / P.R == c) yb[q] = Y;
        car[(static_cast<size_t>(c) * 2 + 0) * P.nx] = Y;
        Y = fma(P.qp[Rc(c)], Y, Bv(c, 0));
    }
    // backward: segment map over (c1-1 .. c0), scan from the high lanes, incoming value from lane + 1
    a = 1.0;
    b = 0.0;
    for (int c = c1 - 1; c >= c0; --c) {
        const double qr = P.qp[Rc(c)];
        const double Yc = car[(static_cast<size_t>(c) * 2 + 0) * P.nx];
        a *= qr;
        b = fma(qr, b, fma(kapf(P.qp, P.s2, 0, Rc(c)), Yc, Bv(c, 1)));
    }
    for (int d = 1; d < kWarp; d <<= 1) {
        const double ad = __shfl_down_sync(0xffffffffu, a, d), bd = __shfl_down_sync(0xffffffffu, b, d);
        if (lane + d < kWarp) {
            b = fma(a, bd, b);
            a *= ad;
        }
    }
    double aout = __shfl_down_sync(0xffffffffu, a, 1), bout = __shfl_down_sync(0xffffffffu, b, 1);
    if (lane == kWarp - 1) {
        aout = 1.0;
        bout = 0.0;
    }
    double X = fma(aout, xinit, bout);
    for (int c = c1 - 1; c >= c0; --c) {
        for (int q = 0; q < 4; ++q)
            if (brow[q] / P.R == c) xb[q] = X;
        if (final_pass) car[(static_cast<size_t>(c) * 2 + 1) * P.nx] = X;
        const double Yc = car[(static_cast<size_t>(c) * 2 + 0) * P.nx];
        X = fma(P.qp[Rc(c)], X, fma(kapf(P.qp, P.s2, 0, Rc(c)), Yc, Bv(c, 1)));
    }
    // the block-boundary captures live on the lane owning that block: broadcast them
    for (int q = 0; q < 4; ++q) {
        const int owner = per > 0 ? min(kWarp - 1, (brow[q] / P.R) / per) : 0;
        yb[q] = __shfl_sync(0xffffffffu, yb[q], owner);
        xb[q] = __shfl_sync(0xffffffffu, xb[q], owner);
    }
}

__global__ void __launch_bounds__(128) step_phase2_warp(const StepParams P) {
    const int lane = threadIdx.x & 31, m = P.tile0 * kWarp + blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
    const int sub = blockIdx.z;
    if (m >= P.xend) return;  // a whole warp per column
    const SubDev &S = P.subs[sub];
    const int nblk = S.nblk, n = S.n;
    const int brow[4] = {0, 1, n - 2, n - 1};
    auto Bv = [&](int c, int slot) { return P.blkagg[((static_cast<size_t>(sub) * P.C + c) * 8 + slot) * P.nx + m]; };
    auto Rc = [&](int c) { return min(P.R, n - c * P.R); };
    double yb[4] = {0, 0, 0, 0}, xb[4] = {0, 0, 0, 0}, xt[4];
    p2w_sweep(P, sub, m, lane, nblk, n, 0.0, 0.0, false, yb, xb);  // zero block carries
    for (int q = 0; q < 4; ++q) {
        const int c = brow[q] / P.R, l = brow[q] - c * P.R, R = Rc(c);
        xt[q] = Bv(c, 2 + q) + kapf(P.qp, P.s2, l, R) * yb[q] + P.qp[R - l] * xb[q];
    }
    const double s0 = S.wt0 * xt[0] + S.wt1 * xt[1];
    const double s1 = S.wb0 * xt[2] + S.wb1 * xt[3];
    const double c0 = S.Mi00 * s0 + S.Mi01 * s1;
    const double c1 = S.Mi10 * s0 + S.Mi11 * s1;
    p2w_sweep(P, sub, m, lane, nblk, n, -c0 / P.a, -c1 / P.a, true, yb, xb);  // the final carries
}

// General path, phase 3: reload k, level 1 with the block carries, pass C.
__global__ void __launch_bounds__(kMaxWarps * kWarp) step_phase3(const StepParams P) {
    extern __shared__ __align__(128) char smraw[];
    Tile t = make_tile(P, blockIdx.x);
    const SubDev &S = *t.sd;
    if (t.Rb == 0) return;
    Smem sm = carve(smraw, P.R, P.P);
    double *unew = S.slab[(P.n + 1) & 1] + static_cast<size_t>(S.first - S.lo) * P.nx;
    if (t.lane == 0 && t.warp < P.P) mbar_init(&sm.bar[t.warp], 1);
    fence_mbar_init();
    __syncwarp();
    if (t.warp < P.P) load_chunk(P, t, unew, sm.tile, &sm.bar[t.warp]);
    if (t.warp < P.P) {
        const size_t base = ((static_cast<size_t>(t.sub) * P.C + t.blk) * P.P + t.warp) * 2 * P.nx;
        sm.he[t.warp * kWarp + t.lane] = P.chkagg[base + t.m];
        sm.ks[t.warp * kWarp + t.lane] = P.chkagg[base + P.nx + t.m];
    }
    {
        const size_t bb = (static_cast<size_t>(t.sub) * P.C + t.blk) * 8 * P.nx;
        if (threadIdx.x < kWarp) {
            if (S.iL_tr >= t.rb0 && S.iL_tr < t.rb0 + t.Rb) sm.rtr[t.lane] = P.blkagg[bb + 6 * P.nx + t.m];
            if (S.iR_tr >= t.rb0 && S.iR_tr < t.rb0 + t.Rb) sm.rtr[kWarp + t.lane] = P.blkagg[bb + 7 * P.nx + t.m];
        }
    }
    __syncthreads();
    if (t.warp == 0) {
        const double Yin = P.carry[((static_cast<size_t>(t.sub) * P.C + t.blk) * 2 + 0) * P.nx + t.m];
        const double Xin = P.carry[((static_cast<size_t>(t.sub) * P.C + t.blk) * 2 + 1) * P.nx + t.m];
        level1_carry(P, t, sm.he, sm.ks, Yin, Xin, sm.Y0, sm.X0);
    }
    __syncthreads();
    double eif = 0.0, et = 0.0;
    if (t.warp < P.P && t.L > 0) {
        mbar_wait(&sm.bar[t.warp], 0);
        pass_c(P, t, sm.tile, sm.Y0[t.warp * kWarp + t.lane], sm.X0[t.warp * kWarp + t.lane], unew, sm.xtr, eif, et);
    }
    __syncthreads();
    if (t.warp == 0) write_traces(P, t, sm.rtr, sm.xtr);
    block_err_flush(P, t, sm, eif, et);
}

}  // namespace kfp

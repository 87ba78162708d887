// kfp_fused.cuh -- the hot kernel: one fused time step of every local subdomain
// (transport + forcing + v-tridiagonal solve + transmission traces + errors),
// sm_100a: TMA tile loads, register-resident chunks, thread-block clusters with
// distributed-shared-memory pushes, persistent over x-tiles.
//
// Geometry.  A cluster of C CTAs owns a 32-column x-tile of one
// subdomain's column stack at a time and walks over the subdomain's x-tiles
// (persistent, next tile prefetched by TMA while the current one is finished).
// CTA `blk` owns the unknown rows [blk*R, blk*R+R), R = 16 L; warp w owns the
// chunk of L <= B rows starting at blk*R + w*L; lane = x-column.  Per tile:
//   A  r' = (q/a)[(1-|nu|) u + |nu| u_nb + dt f], forward scan h_l = q h_{l-1} + r'_l
//   B  backward scan k_l = q k_{l+1} + h_l                        (zero carries)
//   L1 transposed layout (warp w: columns 2w, 2w+1; lane = chunk): affine
//      Kogge-Stone scans over the 16 chunks give every chunk's carries with zero
//      carries at the block ends, the block aggregates F, G and the boundary rows;
//   X  every CTA pushes (F, G) and its boundary rows into every CTA of the
//      cluster (st.async + mbarrier);
//   L2 the block carries = a 22-term linear map of the received values (host-
//      precomputed: block chain + Woodbury boundary terms + incoming traces),
//      summed across the 16 lanes of a column;
//   C  x_l = k_l + kap(l, L) Y + q^{L-l} X, stored with coalesced st.global.
// The forward/backward scans are B^{-1} of T_n = B + a q e_0 e_0^T (see
// kfp_device.cuh); the boundary terms make it the exact solve of the column system.
#pragma once
#include <cuda.h>

#include "kfp_device.cuh"

namespace kfp {

// halo columns per side in the smem tile: 2, so that the TMA box starts on a
// 16-B aligned global column (a box starting at an odd column faults)
constexpr int kHalo = 2;
constexpr int kTW = kWarp + 2 * kHalo;       // 36 doubles (288 B) per smem tile row
constexpr int kFusedWarpsMax = 16;           // largest P (warps per CTA) instantiated
constexpr int kNRmax = 4;                    // forcing ranks supported by the coefficient table
constexpr int kMaxFusedCluster = 8;          // portable cluster size
constexpr int kL2N = 22;                     // inputs of the level-2 map: F_0..7, G_0..7, x~ at 4 rows, g_lo, g_hi
constexpr int kL2M = 48;                     // per (subdomain, block): cY[24] | cX[24]
constexpr int kCS = kWarp + 1;               // row stride of the [chunk|block|row][column] smem arrays (no bank conflicts
                                             // when the 16 lanes of a column walk the chunks)

struct FusedParams {
    StepParams S;                 // common step parameters (kfp_device.cuh)
    const CUtensorMap *tmaps;     // [nsub][2] load maps (box 36 x L) of the slabs' unknown rows, by step parity
    int L;                        // chunk length (rows per warp), R = P*L rows per CTA
    int Gc;                       // clusters per subdomain (each walks the x-tiles t = y, y+Gc, ...)
    int ntiles;                   // 32-column x-tiles per subdomain
    int nrec;                     // monodomain line recording: number of recorded rows
    const int *rec_rows;          // [nrec] node index of each recorded line (in line order)
    const double *l2m;            // [nsub][C][kL2M] level-2 linear maps (host-computed, kfp_api.cu)
    const double *coefT;          // [nv+1][2+NR] per-node (q/a)(1-|nu|), (q/a)|nu|, (q/a) fv_r(j)
    const double *tabs;           // qp[kQ] | s2[kQ] | kr[2B] for this plan (host-computed)
};

// --------------------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa_u32(const void *local_addr, int rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(rank));
    return remote;
}
// push into CTA `rank`'s shared memory (same offset as the local dst), completing
// the bytes on that CTA's mbarrier at the offset of the local bar
__device__ __forceinline__ void st_async_v2(const void *dst, int rank, double a, double b, const uint64_t *bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                     mapa_u32(dst, rank)),
                 "d"(a), "d"(b), "r"(mapa_u32(bar, rank))
                 : "memory");
}
__device__ __forceinline__ void st_async_f64(const void *dst, int rank, double a, const uint64_t *bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(mapa_u32(dst, rank)),
                 "d"(a), "r"(mapa_u32(bar, rank))
                 : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}

// --------------------------------------------------------------------------- smem
// per-warp tile slot: B rows of kTW doubles, padded to a multiple of 128 B (TMA destination alignment)
template <int B>
constexpr int slot_doubles() {
    return ((B * kTW * 8 + 127) / 128) * 128 / 8;
}
// q^k and s2(k) tables for k <= R + 1 (R <= P B), rounded to an even count (16-B bulk copies)
template <int B, int P>
__host__ __device__ constexpr int fused_kq() {
    return ((P * B + 2) + 1) / 2 * 2;
}

// FEM (the paper's split scheme): the tile holds the chunk's rows plus the row above and
// the row below (the 3-point mass average), and no per-row coefficient table (weights computed).
template <int B, int NR, int P, bool FEM = false>
struct FusedSmem {
    static constexpr int kTileRows = B + (FEM ? 2 : 0);
    static constexpr int kSlot = slot_doubles<kTileRows>();
    static constexpr int kRows = P * B;
    static constexpr int kCoef = 2 + (NR < 2 ? 2 : NR);  // c0', c1', g_0' .. g_{NR-1}' (rows padded to 4)
    static constexpr int kQ = fused_kq<B, P>();
    static constexpr int kTab = 2 * kQ + 2 * B + 4;  // + (1/q, 1/(1-q^2), q^{L+1}, q^L) for pass C
    alignas(128) double tile[P * kSlot];  // per warp: u^n rows [L][36] (FEM: [L+2][36], rows cr0-1 .. cr0+L)
    alignas(16) double coef[FEM ? 2 : kRows * kCoef];  // per warp: its chunk's rows of coefT
    alignas(16) double tab[kTab];                   // qp[kQ] | s2[kQ] | kr[2B] | ex[4]  (copy of FusedParams::tabs)
    alignas(16) double l2m[kL2M];                   // level-2 map of this (subdomain, block)
    double he[P * kCS];          // y at the chunk's last row (zero carry); then final Y carries
    double ks[P * kCS];          // k at the chunk's first row (zero carry); then final X carries
    double kb[4 * kCS];                    // k at the column's rows 0,1,n-2,n-1 (chunk-local zero carries)
    double2 rFG[2][kMaxFusedCluster * kCS];  // received (F, G) per block, double-buffered by tile parity
    double rA[2][4 * kCS];                 // received x~ at rows 0,1,n-2,n-1 (zero column carries)
    double gin[2 * kWarp];                 // incoming traces at t_{n+1} (lo end, hi end)
    double rtr[2][2 * kWarp];              // raw r at the outgoing-trace rows (by tile parity)
    double xsp[6 * kWarp];                 // x at the special rows: trace rows (c, c+1 | c, c-1), rows 0, n-1
    SubDev sd;                             // this subdomain's descriptor
    double red[2 * P];
    uint64_t bar[P];             // per warp: u^n tile (+ coefficient rows on the first tile)
    uint64_t tbar;                         // tables
    uint64_t xbar[2];                      // cluster exchange, by tile parity
};

template <int B, int NR, int P, bool FEM = false>
__host__ __device__ constexpr size_t fused_smem_bytes() {
    return sizeof(FusedSmem<B, NR, P, FEM>);
}

// --------------------------------------------------------------------------- passes
// DIR = -1: every row of the chunk has v >= 0 (upwind neighbour m-1); +1: v < 0
// (neighbour m+1); 0: generic (per-row side, ragged length).
// ONFLY (the cluster kernel's full chunks, DIR != 0): the transport weights come from the row index
// instead of the table, c1 = (q/a)|nu_l| = |l dq + vbq|, c0 u + c1 nb = (q/a) u + c1 (nb - u) -- one
// shared-memory load per row fewer (+3 % on c2); the forcing coefficients stay in the table.
template <int B, int NR, int DIR, bool ONFLY = false>
__device__ __forceinline__ void pass_a_reg(const double *tile_w, const double *coef_w, int lane, double q,
                                           const double (&fx)[NR], double (&h)[B], int Lw, int jv2_0, double &hend,
                                           double qa = 0.0, double vbq = 0.0, double dq = 0.0, int uoff = 0) {
    constexpr int kC = 2 + (NR < 2 ? 2 : NR);  // the table's row stride (NR = 1 rows padded to 4 doubles)
    double hp = 0.0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
        const double *row = tile_w + l * kTW + kHalo + lane;
        const double *c = coef_w + l * kC;
        const double u = row[0];
        double nb;
        if (DIR == 0) {
            const int off = (jv2_0 + 2 * l >= 0) ? -1 : 1;  // 2j - nv >= 0: v >= 0 -> left neighbour
            nb = row[off];
        } else if (DIR == 2) {
            nb = row[uoff];  // the whole chunk on one side of v = 0: a warp-uniform offset
        } else {
            nb = row[DIR];
        }
        double f = 0.0;
#pragma unroll
        for (int r = 0; r < NR; ++r) f = fma(c[2 + r], fx[r], f);
        double rp;
        if (DIR == 0 || !ONFLY) {
            rp = fma(c[1], nb, fma(c[0], u, f));
        } else {
            const double c1 = fabs(fma(static_cast<double>(l), dq, vbq));
            rp = fma(c1, nb - u, fma(qa, u, f));
        }
        if (DIR == 0) {
            h[l] = (l < Lw) ? fma(q, hp, rp) : 0.0;
            hend = (l == Lw - 1) ? h[l] : hend;
        } else {
            h[l] = fma(q, hp, rp);
        }
        hp = h[l];
    }
    if (DIR != 0) hend = h[B - 1];
}

// Split-FEM pass A (P:480-516 reordered): the slab holds w^{n-1/2}; tile row i (node
// jb + i, i = 0 .. B+1) is transported on the fly, u_i = w_i + nu_i (w_nb - w_i) with
// nu_i = |vb + i dnu| = |v_j| tau / h_x (Step 2 of the previous step), and the right-hand side of
// row l is the consistent-mass average (q/a)(u_{l-1} + 4 u_l + u_{l+1}) / 6 (Step 1, scaled by tau/h);
// c1 = (q/a)/6, c4 = 4 c1.  Forward scan as in pass_a_reg.
// Neumann / Robin end rows (unknown end node c): the doubled row's right-hand side (2 u_c + u_{c-+1}) / 3
// is the interior average with the reflected ghost u_{c+-1} := u_{c-+1} -- the TRANSPORTED neighbour
// (its own transport weight, not the ghost node's): gtop reflects at the chunk's first row, gl >= 0
// at row gl (the column's last row; only ragged chunks, DIR = 0, hold it).
template <int B, int DIR>
__device__ __forceinline__ void pass_a_fem(const double *tile_w, int lane, double q, double c1, double c4, double vb,
                                           double dnu, int jv2_0, double (&h)[B], int Lw, double &hend, bool gtop,
                                           int gl) {
    auto tr = [&](int i) -> double {
        const double *row = tile_w + i * kTW + kHalo + lane;
        const double w = row[0];
        double nb;
        if (DIR == 0) {
            nb = row[(jv2_0 + 2 * i >= 0) ? -1 : 1];  // v_j >= 0: foot of the characteristic toward m-1
        } else {
            nb = row[DIR];
        }
        const double nu = fabs(fma(static_cast<double>(i), dnu, vb));
        return fma(nu, nb - w, w);
    };
    double tm = tr(0), tc = tr(1), hp = 0.0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
        double tn = tr(l + 2);
        if (DIR == 0 && l == gl) tn = tm;  // bottom ghost
        if (l == 0 && gtop) tm = tn;       // top ghost
        const double rp = fma(c4, tc, c1 * (tm + tn));
        if (DIR == 0) {
            h[l] = (l < Lw) ? fma(q, hp, rp) : 0.0;
            hend = (l == Lw - 1) ? h[l] : hend;
        } else {
            h[l] = fma(q, hp, rp);
        }
        hp = h[l];
        tm = tc;
        tc = tn;
    }
    if (DIR != 0) hend = h[B - 1];
}

template <int B>
__device__ __forceinline__ double pass_b_full(double (&h)[B], double q) {
    double kn = 0.0;
#pragma unroll
    for (int l = B - 1; l >= 0; --l) {
        kn = fma(q, kn, h[l]);
        h[l] = kn;
    }
    return kn;
}
// Ragged chunk: rows l >= Lw are not part of the column; also captures k at
// the chunk's last two rows.
template <int B>
__device__ __forceinline__ double pass_b_ragged(double (&h)[B], double q, int Lw, double &k_last, double &k_last2) {
    double kn = 0.0;
#pragma unroll
    for (int l = B - 1; l >= 0; --l) {
        kn = (l < Lw) ? fma(q, kn, h[l]) : 0.0;
        h[l] = kn;
        k_last = (l == Lw - 1) ? kn : k_last;
        k_last2 = (l == Lw - 2) ? kn : k_last2;
    }
    return kn;
}
// response at row r (local) of the x-recurrence to a unit carry entering above row 0
// of a segment of `len` rows: kap(r, len) = q^{r+1} s2(len - r)
__device__ __forceinline__ double kap_s(const double *qp, const double *s2, int r, int len) {
    return qp[r + 1] * s2[len - r];
}

#ifdef KFP_TRACE
// debug builds only: phase timestamps (ns, %globaltimer) of thread 0 of every CTA: [cta][8]
__device__ unsigned long long *g_kfp_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define KFP_T(k)                                                                                            \
    if (g_kfp_trace && threadIdx.x == 0) {                                                                  \
        const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
        g_kfp_trace[cta * 64 + (k)] = gtime();                                                              \
    }
// per-tile event e (0..5) of tile iteration `it` (first 9 tiles)
#define KFP_TT(e)                                                                                           \
    if (g_kfp_trace && threadIdx.x == 0 && it < 9) {                                                        \
        const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
        g_kfp_trace[cta * 64 + 2 + 6 * it + (e)] = gtime();                                                 \
    }
#else
#define KFP_T(k)
#define KFP_TT(e)
#endif

#ifdef KFP_TRACE
// debug builds only: accumulated phase times (ns) of thread 0 of every CTA, [cta][64]
#define KFP_WT_DECL unsigned long long wt_acc[10] = {0}, wt_last = 0;
#define KFP_WT(k)                                              \
    if (g_kfp_trace && threadIdx.x == 0) {                     \
        const unsigned long long now_ = gtime();               \
        if ((k) >= 0 && wt_last) wt_acc[(k)] += now_ - wt_last; \
        wt_last = now_;                                        \
    }
#define KFP_WT_FLUSH                                                                                        \
    if (g_kfp_trace && threadIdx.x == 0) {                                                                  \
        const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
        for (int i_ = 0; i_ < 10; ++i_) g_kfp_trace[cta * 64 + i_] = wt_acc[i_];                            \
    }
#else
#define KFP_WT_DECL
#define KFP_WT(k)
#define KFP_WT_FLUSH
#endif

// --------------------------------------------------------------------------- the kernel
// PIPE: pipelined iterations -- every descriptor carries its own step (P.n - S.lag); otherwise the step
// and its flags come from the launch parameters (constant bank, no registers held).
template <int B, int NR, int P_, bool FEM = false, bool PIPE = false>
__global__ void __launch_bounds__(P_ * kWarp, 16 / P_) step_fused_tma(const FusedParams FP) {
    constexpr int NW = P_;            // warps (= chunks) per CTA
    constexpr int kCPW = kWarp / NW;  // columns per warp in the transposed phase
    constexpr int kX = FEM ? 1 : 0;   // FEM: extra tile rows above and below the chunk
    using Sm = FusedSmem<B, NR, NW, FEM>;
    extern __shared__ __align__(128) char smraw[];
    Sm &sm = *reinterpret_cast<Sm *>(smraw);
    const StepParams &P = FP.S;
    const int blk = static_cast<int>(cg::this_cluster().block_rank());
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = blockIdx.z;
    {  // this subdomain's descriptor -> shared memory (read many times below)
        constexpr int kWords = sizeof(SubDev) / sizeof(uint64_t);
        static_assert(sizeof(SubDev) % sizeof(uint64_t) == 0, "SubDev size");
        if (threadIdx.x < kWords)
            reinterpret_cast<uint64_t *>(&sm.sd)[threadIdx.x] = reinterpret_cast<const uint64_t *>(P.subs + sub)[threadIdx.x];
        __syncthreads();
    }
    const SubDev &S = sm.sd;
    // the step this descriptor computes (pipelined iterations: each slot lags by S.lag steps); recomputed
    // where used (constant bank + shared memory) rather than held in registers across the tile loop
#define step (PIPE ? P.n - S.lag : P.n)
#define from_u0 (PIPE ? step == 0 : P.from_u0 != 0)
#define last (PIPE ? (P.last && step == P.nt - 1) : P.last != 0)  // pipelined: P.last = errors at T wanted
    const int n = S.n, L = FP.L, R = NW * L;
    const int rb0 = blk * R;                                    // first unknown row of this block
    const int Rb = max(0, min(R, n - rb0));                     // rows of this block
    const int s_w = warp * L;                                   // chunk start (block-local)
    const int Lw = max(0, min(L, Rb - s_w));                    // rows of this warp's chunk
    const int cr0 = rb0 + s_w;                                  // first column row of the chunk
    const int nblk = S.nblk;
    // the block holds rows of the column, and the slot's step exists (pipeline fill / drain: whole cluster)
    const bool live = blk < nblk && (!PIPE || (step >= 0 && step < P.nt));
    const double q = P.q;
    const CUtensorMap *tmap = FP.tmaps + 2 * sub + (step & 1);
    double *unew_slab = S.slab[(step + 1) & 1];
    double *unew = unew_slab + static_cast<size_t>(S.first - S.lo) * P.nx;
    double *tile_w = sm.tile + warp * Sm::kSlot;
    double *coef_w = sm.coef + warp * B * Sm::kCoef;
    const double *qp = sm.tab, *s2 = sm.tab + Sm::kQ, *kr = sm.tab + 2 * Sm::kQ;
    auto inblk = [&](int i) { return i >= rb0 && i < rb0 + Rb; };
    auto inchunk = [&](int i) { return i >= cr0 && i < cr0 + Lw; };
    // does this block compute an outgoing trace?
    const bool tr_L = S.iL_tr >= 0 && (inblk(S.iL_tr) || inblk(S.iL_tr + 1));
    const bool tr_R = S.iR_tr >= 0 && S.iR_tr < n && (inblk(S.iR_tr) || inblk(S.iR_tr - 1));
    const bool trace_cta = tr_L || tr_R;
    // rows whose x is needed after pass C: trace stencils and the Robin-end interface rows
    const int sp_row[6] = {tr_L ? S.iL_tr : -1, tr_L ? S.iL_tr + 1 : -1, tr_R ? S.iR_tr : -1, tr_R ? S.iR_tr - 1 : -1,
                           (S.ltype == END_ROBIN && S.ifL >= 0) ? 0 : -1, (S.rtype == END_ROBIN && S.ifR >= 0) ? n - 1 : -1};
    bool chunk_special = false;
#pragma unroll
    for (int qq = 0; qq < 6; ++qq) chunk_special |= sp_row[qq] >= cr0 && sp_row[qq] < cr0 + Lw;
    bool cta_special = trace_cta || P.record || P.ovrec;
#ifdef KFP_ABLATE_SPECIAL  // experiments only (results invalid): no special-rows block
    cta_special = false;
#endif
#pragma unroll
    for (int qq = 4; qq < 6; ++qq) cta_special |= inblk(sp_row[qq]);
    const int t_first = P.tile0 + blockIdx.y;  // (a sharded monodomain starts at tile0; ntiles = its end)
    // x-tile of walk index tt: odd steps walk the tiles in reverse, so that a step first reads the tiles the
    // previous step wrote last (still in L2)
    auto phys = [&](int tt) { return (step & 1) ? P.tile0 + FP.ntiles - 1 - tt : tt; };
    const uint32_t tile_bytes = static_cast<uint32_t>(kTW * (L + 2 * kX) * sizeof(double));
    // tensor-map row of the tile's first row: FD maps start at the first unknown row, FEM maps at the
    // slab's first node (the row above the chunk may be a Dirichlet end node)
    const int ty0 = FEM ? cr0 + (S.first - S.lo) - 1 : cr0;
    // node of tile row 0 (re-read from shared memory where used: not kept live across the tile loop)
#define KFP_JB (S.first + cr0 - kX)
    KFP_T(0)

    // ---- prologue: barriers, constant tables (overlaps the previous step under PDL)
    if (threadIdx.x == 0) {
        mbar_init(&sm.xbar[0], 1);
        mbar_init(&sm.xbar[1], 1);
        mbar_init(&sm.tbar, 1);
        prefetch_tmap(tmap);
    }
    if (lane == 0) mbar_init(&sm.bar[warp], 1);
    fence_mbar_init();
    cluster_arrive_relaxed();  // every CTA's xbar is initialised before anybody pushes (wait below)
    if (!live) {               // a row block beyond this subdomain's column (shorter edge subdomain)
        cluster_wait();
        return;
    }
    if (lane == 0 && Lw > 0) { // this chunk's per-row coefficients (+ its first u^n tile below)
        if (FEM) {
            mbar_expect_tx(&sm.bar[warp], from_u0 ? 0u : tile_bytes);  // 0: completes phase 0 at once
        } else {
            const uint32_t coef_bytes = static_cast<uint32_t>(Lw * Sm::kCoef * sizeof(double));
            mbar_expect_tx(&sm.bar[warp], coef_bytes + (from_u0 ? 0u : tile_bytes));
            bulk_g2s(coef_w, FP.coefT + static_cast<size_t>(S.first + cr0) * Sm::kCoef, coef_bytes, &sm.bar[warp]);
        }
    }
    if (threadIdx.x == 0) {    // q-power tables, pass-C coefficients, this block's level-2 map
        mbar_expect_tx(&sm.tbar, static_cast<uint32_t>((Sm::kTab + kL2M) * sizeof(double)));
        bulk_g2s(sm.tab, FP.tabs, Sm::kTab * sizeof(double), &sm.tbar);
        bulk_g2s(sm.l2m, FP.l2m + (static_cast<size_t>(sub) * P.C + blk) * kL2M, kL2M * sizeof(double), &sm.tbar);
    }
    grid_dep_wait();  // the previous step's u^n is complete
    if (Lw > 0 && !from_u0 && lane == 0 && t_first < FP.ntiles)
        tma_load_2d(tile_w, tmap, phys(t_first) * kWarp - kHalo, ty0, &sm.bar[warp]);
    cluster_wait();  // matches the prologue arrive
    KFP_T(1)

    double eif = 0.0, et = 0.0;
    int it = 0;
    for (int t = t_first; t < FP.ntiles; t += FP.Gc, ++it) {
        const int par = it & 1;
        const int m0 = phys(t) * kWarp, w = min(kWarp, P.nx - m0);
        const int m = m0 + min(lane, w - 1);
        const bool active = lane < w;
        const size_t goff = static_cast<size_t>(step) * P.nx + m;  // row t_{n+1} of [nt][nx] arrays
        double fx[NR];  // this lane's forcing profile times dt ft_r(t_{n+1})
#pragma unroll
        for (int r = 0; r < NR; ++r)
            fx[r] = (r < P.f_rank) ? (PIPE ? __ldg(P.cfn + step * kMaxRank + r) : P.cf[r]) * __ldg(P.fx + r * P.nx + m) : 0.0;
        if (warp == 0) {  // incoming traces of this step (written by the previous iteration)
            sm.gin[lane] = (S.ltype == END_DIRI || S.ltype == END_ROBIN) ? S.gL[P.par_in_lo][goff] : 0.0;
            sm.gin[kWarp + lane] = (S.rtype == END_DIRI || S.rtype == END_ROBIN) ? S.gR[P.par_in][goff] : 0.0;
        }

        // ---- passes A and B (registers)
        double h[B];
        double hend = 0.0, kst = 0.0;
        if (Lw > 0) {
            if (!from_u0 || it == 0) mbar_wait(&sm.bar[warp], par);
            KFP_TT(0)
            if (from_u0) {  // u^0 from the separable u0 tables (0 B of HBM), incl. the halo columns
                for (int l = 0; l < Lw + 2 * kX; ++l) {
                    const int j = KFP_JB + l;
                    if (FEM && (j < S.lo || j > S.hi)) continue;  // ghost row outside the subdomain (set below)
                    for (int c = lane; c < kTW; c += kWarp) {
                        const int mm = ((m0 - kHalo + c) % P.nx + P.nx) % P.nx;
                        double s = 0.0;
                        for (int r = 0; r < P.u0_rank; ++r)
                            s = fma(__ldg(P.u0v + r * (P.nv + 1) + j), __ldg(P.u0x + r * P.nx + mm), s);
                        tile_w[l * kTW + c] = s;
                    }
                }
                __syncwarp();
            } else if (m0 == 0 || m0 + w == P.nx) {
                // periodic wrap of the halo at the ends of the x range (TMA zero-fills out-of-range columns)
                const int jb = KFP_JB;
                const double *src = S.slab[step & 1] + static_cast<ptrdiff_t>(jb - S.lo) * P.nx;
                // one row per lane, strided: a chunk may hold more rows (L <= 33) than a warp has lanes
                for (int l = lane; l < Lw + 2 * kX; l += kWarp) {
                    if (FEM && (jb + l < S.lo || jb + l > S.hi)) continue;
                    if (m0 == 0) tile_w[l * kTW + kHalo - 1] = src[static_cast<ptrdiff_t>(l) * P.nx + P.nx - 1];
                    if (m0 + w == P.nx) tile_w[l * kTW + kHalo + w] = src[static_cast<ptrdiff_t>(l) * P.nx];
                }
                __syncwarp();
            }
            const int jb = KFP_JB;
            const int jv2_0 = 2 * jb - P.nv;                   // 2 j - nv of the tile's first row
            const int jv2_1 = jv2_0 + 2 * (Lw - 1 + 2 * kX);   // ... of its last row
            // full chunks take the unpredicated paths; the chunk holding the column's
            // last two rows takes the ragged one (it captures their k values)
            const bool full = (Lw == B) && (cr0 + Lw <= n - 2);
            if (FEM) {
                const double dnu = from_u0 ? 0.0 : P.dnu, nu0 = from_u0 ? 0.0 : P.nu0;  // step 0: u0, no Step 2
                const double c1 = P.qa * (1.0 / 6.0), c4 = 4.0 * c1, vb = fma(static_cast<double>(jb), dnu, nu0);
                // unknown end nodes (Neumann / Robin ends) in this chunk: reflected ghosts
                const bool gtop = cr0 == 0 && S.first == S.lo;
                const int gl = (cr0 + Lw == n && S.first + n - 1 == S.hi) ? Lw - 1 : -1;
                if (full && jv2_0 >= 0) pass_a_fem<B, -1>(tile_w, lane, q, c1, c4, vb, dnu, jv2_0, h, Lw, hend, gtop, gl);
                else if (full && jv2_1 < 0) pass_a_fem<B, 1>(tile_w, lane, q, c1, c4, vb, dnu, jv2_0, h, Lw, hend, gtop, gl);
                else pass_a_fem<B, 0>(tile_w, lane, q, c1, c4, vb, dnu, jv2_0, h, Lw, hend, gtop, gl);
            } else {
                // (q/a) v_j dt / h_x at the chunk's first row and its increment per row
                const double dq = P.qa * P.hv * P.dt * P.nx, vbq = fma(static_cast<double>(jb), dq, -P.qa * (0.5 * P.nv) * P.hv * P.dt * P.nx);
                // full chunks on one side of v = 0 share one body with a warp-uniform neighbour offset (the
                // two sign-specialised copies doubled the hot code; the kernel is instruction-cache sensitive)
                if (full && (jv2_0 >= 0 || jv2_1 < 0))
                    pass_a_reg<B, NR, 2, true>(tile_w, coef_w, lane, q, fx, h, Lw, jv2_0, hend, P.qa, vbq, dq,
                                                jv2_0 >= 0 ? -1 : 1);
                else pass_a_reg<B, NR, 0>(tile_w, coef_w, lane, q, fx, h, Lw, jv2_0, hend);
            }
            if (trace_cta) {  // raw r (no incoming-trace term) at the outgoing-trace rows, for the Robin trace (R11)
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const int itr = side ? S.iR_tr : S.iL_tr;
                    if (FEM && itr >= 0 && inchunk(itr)) {
                        // one-sided mass average (2 u_c + u_nb) / 3 of the transported rows at the trace node
                        // c and its neighbour toward the sender's interior (reading F4)
                        const int i = itr - cr0 + 1, inb = side ? i - 1 : i + 1, jb = KFP_JB;
                        const double dnu = from_u0 ? 0.0 : P.dnu, vb = from_u0 ? 0.0 : fma(static_cast<double>(jb), P.dnu, P.nu0);
                        auto trr = [&](int ii) {
                            const double *row = tile_w + ii * kTW + kHalo + lane;
                            const double nu = fabs(fma(static_cast<double>(ii), dnu, vb));
                            return fma(nu, row[(2 * (jb + ii) - P.nv >= 0) ? -1 : 1] - row[0], row[0]);
                        };
                        sm.rtr[par][side * kWarp + lane] = (2.0 * trr(i) + trr(inb)) * (1.0 / 3.0);
                    } else if (!FEM && itr >= 0 && inchunk(itr)) {
                        const int l = itr - cr0, j = S.first + itr;
                        const double2 rc = __ldg(P.rowc + j);
                        const double u = tile_w[l * kTW + kHalo + lane];
                        const double nb = tile_w[l * kTW + kHalo + lane + ((2 * j - P.nv >= 0) ? -1 : 1)];
                        double f = 0.0;
                        for (int r = 0; r < P.f_rank; ++r) f = fma(__ldg(P.fv + r * (P.nv + 1) + j), fx[r], f);
                        sm.rtr[par][side * kWarp + lane] = fma(rc.x, u, fma(rc.y, nb, f));
                    }
                }
            }
            // the slot is consumed: prefetch this warp's chunk of the next tile
            __syncwarp();
            if (lane == 0 && !from_u0 && t + FP.Gc < FP.ntiles) {
                fence_proxy_async_smem();
                mbar_expect_tx(&sm.bar[warp], tile_bytes);
                tma_load_2d(tile_w, tmap, phys(t + FP.Gc) * kWarp - kHalo, ty0, &sm.bar[warp]);
            }
            if (full) {
                kst = pass_b_full<B>(h, q);
            } else {
                double kl = 0.0, kl2 = 0.0;
                kst = pass_b_ragged<B>(h, q, Lw, kl, kl2);
                if (cr0 + Lw == n) {
                    sm.kb[3 * kCS + lane] = kl;
                    if (Lw >= 2) sm.kb[2 * kCS + lane] = kl2;
                } else if (cr0 + Lw == n - 1) {
                    sm.kb[2 * kCS + lane] = kl;
                }
            }
            if (cr0 == 0) {
                sm.kb[0 * kCS + lane] = h[0];
                if (Lw >= 2) sm.kb[1 * kCS + lane] = h[1];
            } else if (cr0 == 1) {
                sm.kb[1 * kCS + lane] = h[0];
            }
        }
        sm.he[warp * kCS + lane] = hend;
        sm.ks[warp * kCS + lane] = kst;
        if (it == 0) mbar_wait(&sm.tbar, 0);  // tables (long since arrived)
        KFP_TT(1)
        __syncthreads();

        // ---- levels 1 and 2 in the transposed layout: warp w owns the kCPW columns
        //      col = kCPW w + lane / NW; lane k = lane % NW stands for chunk k of the block.
        {
            const int col = kCPW * warp + lane / NW, k = lane % NW;
            const int sk = k * L, Lk = max(0, min(L, Rb - sk)), ek = sk + Lk;
            const double Qk = qp[Lk];
            // level 1: affine Kogge-Stone scans over the chunks (zero block carries)
            //   y_out(k) = q^{L_k} y_out(k-1) + he_k,   x_start(k) = q^{L_k} x_start(k+1) + Z0_k
            double A = Qk, Bv = sm.he[k * kCS + col];
            const double ksk = sm.ks[k * kCS + col];
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const double Au = __shfl_up_sync(0xffffffffu, A, d, NW), Bu = __shfl_up_sync(0xffffffffu, Bv, d, NW);
                if (k >= d) {
                    Bv = fma(A, Bu, Bv);
                    A *= Au;
                }
            }
            const double F = __shfl_sync(0xffffffffu, Bv, NW - 1, NW);  // y at the block's last row
            double y0 = __shfl_up_sync(0xffffffffu, Bv, 1, NW);
            if (k == 0) y0 = 0.0;
            const double z0 = (Lk > 0) ? fma(kap_s(qp, s2, 0, Lk), y0, ksk) : 0.0;
            A = Qk;
            Bv = z0;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const double Ad = __shfl_down_sync(0xffffffffu, A, d, NW), Bd = __shfl_down_sync(0xffffffffu, Bv, d, NW);
                if (k + d < NW) {
                    Bv = fma(A, Bd, Bv);
                    A *= Ad;
                }
            }
            const double G = __shfl_sync(0xffffffffu, Bv, 0, NW);   // x at the block's first row
            double x0 = __shfl_down_sync(0xffffffffu, Bv, 1, NW);
            if (k == NW - 1) x0 = 0.0;
            // push this block's aggregates of column col into every block of the cluster
            if (k == 0)
                for (int c = 0; c < nblk; ++c) st_async_v2(&sm.rFG[par][blk * kCS + col], c, F, G, &sm.xbar[par]);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {  // column boundary rows held by chunk k: x~ with zero block carries
                const int row = (qq < 2) ? qq : n - 4 + qq;
                const int l = row - rb0 - sk;
                if (row >= 0 && l >= 0 && l < Lk) {
                    const double a = sm.kb[qq * kCS + col] + kap_s(qp, s2, l, Lk) * y0 + qp[Lk - l] * x0;
                    for (int c = 0; c < nblk; ++c) st_async_f64(&sm.rA[par][qq * kCS + col], c, a, &sm.xbar[par]);
                }
            }
            if (threadIdx.x == 0)
                mbar_expect_tx(&sm.xbar[par],
                               static_cast<uint32_t>(nblk * kWarp * sizeof(double2) + 4 * kWarp * sizeof(double)));
            KFP_TT(2)
            mbar_wait(&sm.xbar[par], (it >> 1) & 1);
            KFP_TT(3)
            // level 2: block carries = the precomputed linear map of (F_c, G_c, x~_q, g_lo, g_hi);
            // terms j = k, k + P, ... on lane k, summed over the NW lanes of the column
            double yv = 0.0, xv = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < kL2N; j0 += NW) {
                const int j = j0 + k;
                if (j < kL2N) {
                    double v = 0.0;
                    if (j < 16) {
                        const int c = j & 7;
                        if (c < nblk) v = (j < 8) ? sm.rFG[par][c * kCS + col].x : sm.rFG[par][c * kCS + col].y;
                    } else if (j < 20) {
                        v = sm.rA[par][(j - 16) * kCS + col];
                    } else {
                        v = sm.gin[(j - 20) * kWarp + col];
                    }
                    yv = fma(sm.l2m[j], v, yv);
                    xv = fma(sm.l2m[24 + j], v, xv);
                }
            }
#pragma unroll
            for (int o = NW / 2; o > 0; o >>= 1) {
                yv += __shfl_xor_sync(0xffffffffu, yv, o, NW);
                xv += __shfl_xor_sync(0xffffffffu, xv, o, NW);
            }
            // final carries of chunk k: y just above it, x just below it
            sm.he[k * kCS + col] = fma(qp[sk], yv, y0);
            sm.ks[k * kCS + col] = fma(qp[Rb - ek], xv, fma(kap_s(qp, s2, ek, Rb), yv, x0));
        }
        KFP_TT(4)
        __syncthreads();

        // ---- pass C: x = k + kap Y + rho X; coalesced stores of u^{n+1}
        if (Lw > 0) {
            const double Y = sm.he[warp * kCS + lane], X = sm.ks[warp * kCS + lane];
            double *dst = unew + static_cast<size_t>(cr0) * P.nx + m;
            const size_t pitch = P.nx;
            if (Lw == B && L == B) {
                // kap(l, L) Y + q^{L-l} X = (c Y) q^{l+1} + (X - c q^{L+1} Y) q^{L-l}, c = 1/(1 - q^2):
                // two running products instead of a table load per row
                const double *ex = kr + 2 * B;  // 1/q, 1/(1-q^2), q^{L+1}, q^L
                double A = ex[1] * Y * q, Rr = fma(-ex[1] * ex[2], Y, X) * ex[3];
#pragma unroll
                for (int l = 0; l < B; ++l) {
                    h[l] += A + Rr;
                    A *= q;
                    Rr *= ex[0];
                }
            } else {
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) h[l] = fma(kap_s(qp, s2, l, Lw), Y, fma(qp[Lw - l], X, h[l]));
            }
            const int wlo = S.wlo, whi = S.whi > 0 ? S.whi : n;  // rows this descriptor stores
            if (active) {
                if (Lw == B && cr0 >= wlo && cr0 + B <= whi) {  // full chunk: unpredicated stores, one pointer step per row
                    double *p = dst;
#pragma unroll
                    for (int l = 0; l < B; ++l) {
                        st_global_f64(p, h[l]);
                        p += pitch;
                    }
                } else {
#pragma unroll
                    for (int l = 0; l < B; ++l)
                        if (l < Lw && cr0 + l >= wlo && cr0 + l < whi) dst[l * pitch] = h[l];
                }
            }
            if (!FEM && last && active) {  // error at T on every unknown row (a 1/N_t fraction of the steps)
                const double *ut = P.UT + static_cast<size_t>(S.first + cr0) * P.nx + m;
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) et = nmax(et, fabs(h[l] - ut[l * pitch]));
            }
            // rows needed after the barrier (trace stencils, Robin-end interface rows)
            if (chunk_special) {
#pragma unroll
                for (int l = 0; l < B; ++l)
#pragma unroll
                    for (int qq = 0; qq < 6; ++qq)
                        if (l < Lw && cr0 + l == sp_row[qq]) sm.xsp[qq * kWarp + lane] = h[l];
            }
        }
        // ---- Dirichlet ends: the end node value is the incoming trace
        if (warp == 0 && active) {
            if (blk == 0 && S.ltype == END_DIRI) {
                const double g = sm.gin[lane];
                if (S.iL_tr == -1) S.sendL[P.par_out][goff] = g;  // no overlap: the end node is the trace node
                if (S.ifL >= 0) eif = nmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + step) * P.nx + m]));
                if (FEM) {  // the node's value enters the next step's transport and mass average
                    unew_slab[m] = g;
                } else if (last) {
                    et = nmax(et, fabs(g - P.UT[static_cast<size_t>(S.lo) * P.nx + m]));
                    unew_slab[m] = g;
                }
            } else if (blk == 0 && S.ltype == END_PHYS && last) {
                unew_slab[m] = 0.0;
            }
            if (blk == nblk - 1 && S.rtype == END_DIRI) {
                const double g = sm.gin[kWarp + lane];
                if (S.iR_tr == n) S.sendR[P.par_out][goff] = g;
                if (S.ifR >= 0) eif = nmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + step) * P.nx + m]));
                if (FEM) {
                    unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + m] = g;
                } else if (last) {
                    et = nmax(et, fabs(g - P.UT[static_cast<size_t>(S.hi) * P.nx + m]));
                    unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + m] = g;
                }
            } else if (blk == nblk - 1 && S.rtype == END_PHYS && last) {
                unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + m] = 0.0;
            }
        }
        // ---- outgoing traces at t_{n+1} (R11), Robin-end interface errors,
        //      monodomain line recording
        if (cta_special) {
            __syncthreads();
            if (warp == 0 && active) {
                const double inv_h = 1.0 / P.hv, half_h_dt = 0.5 * P.hv / P.dt;
                if (tr_L && inblk(S.iL_tr)) {  // (p + d_v) u at hi_{s-1}, half-cell flux on [c, c+h/2]
                    const double uc = sm.xsp[lane];
                    double g = uc;
                    if (P.send_robin) {
                        const double xn = sm.xsp[kWarp + lane], xb = FEM ? (2.0 * uc + xn) * (1.0 / 3.0) : uc;
                        g = S.tpL * uc - ((uc - xn) * inv_h + half_h_dt * (xb - sm.rtr[par][lane]));
                    }
                    S.sendL[P.par_out][goff] = g;
                }
                if (tr_R && inblk(S.iR_tr)) {  // (q - d_v) u at lo_{s+1}, flux on [c-h/2, c]
                    const double uc = sm.xsp[2 * kWarp + lane];
                    double g = uc;
                    if (P.send_robin) {
                        const double xn = sm.xsp[3 * kWarp + lane], xb = FEM ? (2.0 * uc + xn) * (1.0 / 3.0) : uc;
                        g = S.tpR * uc - ((uc - xn) * inv_h + half_h_dt * (xb - sm.rtr[par][kWarp + lane]));
                    }
                    S.sendR[P.par_out][goff] = g;
                }
                if (inblk(sp_row[4]))
                    eif = nmax(eif, fabs(sm.xsp[4 * kWarp + lane] - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + step) * P.nx + m]));
                if (inblk(sp_row[5]))
                    eif = nmax(eif, fabs(sm.xsp[5 * kWarp + lane] - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + step) * P.nx + m]));
                if (P.record)  // read back this block's recorded rows of u^{n+1} (stored above by this CTA)
                    for (int i = 0; i < FP.nrec; ++i) {
                        const int row = FP.rec_rows[i] - S.first;  // (rec_rows: node indices)
                        if (inblk(row) && row >= S.wlo && row < (S.whi > 0 ? S.whi : n))
                            P.rec[(static_cast<size_t>(i) * P.nt + step) * P.nx + m] = unew[static_cast<size_t>(row) * P.nx + m];
                    }
                if (P.ovrec)  // this subdomain's overlap rows (unknown rows of this block; Dirichlet end nodes)
                    for (int side = 0; side < 2; ++side)
                        for (int r = 0; r < S.ovn[side]; ++r) {
                            const int node = S.ovr0[side] + r, row = node - S.first;
                            double val = 0.0;
                            bool have = true;
                            if (row >= 0 && row < n && inblk(row)) val = unew[static_cast<size_t>(row) * P.nx + m];
                            else if (node == S.lo && S.ltype == END_DIRI && blk == 0) val = sm.gin[lane];
                            else if (node == S.hi && S.rtype == END_DIRI && blk == nblk - 1) val = sm.gin[kWarp + lane];
                            else have = false;
                            if (have) S.ovb[side][(static_cast<size_t>(r) * P.nt + step) * P.nx + m] = val;
                        }
            }
        }
        KFP_TT(5)
    }
    grid_dep_launch();  // the next step may start its prologue

    // ---- errors: block max, one atomic per CTA
    if (P.errIF) {
        eif = warp_max(eif);
        et = warp_max(et);
        if (lane == 0) {
            sm.red[warp] = eif;
            sm.red[NW + warp] = et;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int c = 0; c < NW; ++c) {
                a = nmax(a, sm.red[c]);
                b = nmax(b, sm.red[NW + c]);
            }
            const size_t go = static_cast<size_t>(S.grp) * P.err_stride;  // replica of this CTA's subdomain
            if (err_pos(a)) atomic_max_pos(P.errIF + go, a);
            if (err_pos(b) && P.errT) atomic_max_pos(P.errT + go, b);
        }
    }
    KFP_T(63)
}
#undef KFP_JB
#undef step
#undef from_u0
#undef last

// Split FEM: the slab after the window's last step holds w^{nt-1/2}; the scheme's
// u(T) is its last Step 2, u_j(x_m) = w_j + nu_j (w_j(x_nb) - w_j(x_m)).  One pass over
// every node of every listed subdomain: writes u(T) into the other slab buffer and, when UT is given,
// max |u(T) - U(T)| into err_T (one atomic per CTA).  grid (ceil(nx / 128), row groups, nsub).
__global__ void __launch_bounds__(128) fem_finish(const StepParams P) {
    const SubDev &S = P.subs[blockIdx.z];
    const int rows = S.hi - S.lo + 1, m = blockIdx.x * blockDim.x + threadIdx.x;
    const double *src = S.slab[P.nt & 1];
    double *dst = S.slab[(P.nt + 1) & 1];
    double e = 0.0;
    if (m < P.nx) {
        const int ml = (m == 0) ? P.nx - 1 : m - 1, mr = (m == P.nx - 1) ? 0 : m + 1;
        for (int r = blockIdx.y; r < rows; r += gridDim.y) {
            const int j = S.lo + r;
            const double *row = src + static_cast<size_t>(r) * P.nx;
            const double w = row[m], wn = row[(2 * j - P.nv >= 0) ? ml : mr];
            const double u = fma(fabs(fma(static_cast<double>(j), P.dnu, P.nu0)), wn - w, w);
            dst[static_cast<size_t>(r) * P.nx + m] = u;
            if (P.UT) e = nmax(e, fabs(u - P.UT[static_cast<size_t>(j) * P.nx + m]));
        }
    }
    if (P.errT) {
        __shared__ double red[4];
        e = warp_max(e);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
        __syncthreads();
        if (threadIdx.x == 0) {
            e = nmax(nmax(red[0], red[1]), nmax(red[2], red[3]));
            if (err_pos(e)) atomic_max_pos(P.errT + static_cast<size_t>(S.grp) * P.err_stride, e);
        }
    }
}

// The paper's stopping quantity (eq. 'error'): max over the closed overlap of interface z
// (nodes [lo_{s+1}, hi_s]), every step and x-node of |u_s - u_{s+1}|, from the two subdomains' overlap
// records; one atomic max per CTA into errOV + grp * err_stride.  grid (blocks, 1, interfaces).
__global__ void __launch_bounds__(256) overlap_diff(const SubDev *subs, const int2 *pairs, int nt, int nx,
                                                    unsigned long long *errOV, int err_stride) {
    const int2 pr = pairs[blockIdx.z];
    const SubDev &L = subs[pr.x], &R = subs[pr.y];
    const size_t N = static_cast<size_t>(L.ovn[1]) * nt * nx;
    const double *a = L.ovb[1], *b = R.ovb[0];
    double e = 0.0;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        e = nmax(e, fabs(a[i] - b[i]));
    __shared__ double red[8];
    e = warp_max(e);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) e = nmax(e, red[w]);
        if (err_pos(e)) atomic_max_pos(errOV + static_cast<size_t>(L.grp) * err_stride, e);
    }
}

}  // namespace kfp

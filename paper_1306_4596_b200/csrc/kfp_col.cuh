// kfp_col.cuh -- the fused time step without thread-block clusters: one CTA owns an
// 8-column x-tile over the WHOLE column height of a subdomain (n <= 4 P L rows), so the
// v-tridiagonal solve, its Woodbury boundary terms and the transmission traces are resolved
// inside one CTA -- no distributed shared memory, no cross-SM rendezvous per tile, and every
// SM of the device can take tiles (clusters of 8 only pack onto ~132 of 148 SMs).
//
// Geometry.  Warp w, lane = c + 8 s (c = column of the tile, s = sub-chunk): the thread owns
// column m = 8 t + c and the chunk k = 4 w + s of L rows [k L, k L + L) of the subdomain's
// unknown rows (NC = 4 P chunks per column).  Per tile:
//   load  one TMA box of 8 x 4L doubles per warp (64-B rows, aligned) + the upwind neighbour
//         column of each row (the x-halo: column 8t-1 where v >= 0, 8t+8 where v < 0) with
//         8-B cp.async, both completing on the warp's mbarrier; the next tile's load is
//         issued as soon as pass A has consumed the slot;
//   A     r' = (q/a)[(1-|nu|) u + |nu| u_nb + dt f], forward scan h = q h + r'   (registers)
//   B     backward scan k = q k + h                                            (registers)
//   scan  (S1) warp c < 8 takes column c, lane i the chunks NC/32 i ...: affine scans of the
//         forward (y) and backward (x) chunk carries over all NC chunks, with the incoming
//         traces as the end carries, then the Woodbury correction of the Dirichlet/Robin end
//         rows and the final carries of every chunk; the same warp forms the
//         outgoing traces (R11) and the interface errors from the carried values;
//   C     (S2) x = k + kap(l, L_k) Y_k + q^{L_k - l} X_k, coalesced 64-B row stores.
// The chunk constants (q^{L_k}, kap(0, L_k), q^{s_k}, kap(e_k, n), q^{n - e_k}) are host-
// computed per subdomain; the transport weights are formed from j (nu_j = nu0 + j dnu).
#pragma once
#include "kfp_fused.cuh"

namespace kfp {

constexpr int kColW = 8;                   // columns per tile
constexpr int kColSub = kWarp / kColW;     // sub-chunks (chunks) per warp
constexpr int kCT = 5;                     // chunk-table entries per chunk
constexpr int kColMaxSub = 32;             // subdomain descriptors resident in shared memory

struct ColParams {
    StepParams S;               // common step parameters (kfp_device.cuh)
    const CUtensorMap *tmaps;   // [nsub][2] load maps (box 8 x 4L) of the slabs' unknown rows, by step parity
    const double *fvq;          // [nv+1][NR]: (q/a) fv_r(j)
    const double *ctab;         // [nsub][NC][kCT]
    const double *tabs;         // qp[kQ] | s2[kQ] | kr[2B]
    const int *rec_rows;        // [nrec] unknown-row index of each recorded monodomain line
    int nrec;
    int L, ntiles;              // chunk rows; 8-column tiles per subdomain
    int nsub;                   // subdomains of the launch
    double qdn;                 // (q/a) dnu: (q/a) |nu_j| = qdn |j - nv/2|  (nu_j = v_j dt / h_x, exact 0 at v = 0)
};

template <int B, int NR, int P>
struct ColSmem {
    static constexpr int NC = kColSub * P;          // chunks per column
    static constexpr int kRows = NC * B;
    static constexpr int kQ = ((B + 2) + 1) / 2 * 2;
    static constexpr int kTab = 2 * kQ + 2 * B;
    static constexpr int kHS = NC + 4;              // row stride of the [column][chunk] arrays (bank spread)
    alignas(128) double tile[P][kColSub * B * kColW];  // per warp: its 4L rows x 8 columns (TMA box)
    alignas(16) double halo[kRows];                    // per unknown row: the upwind neighbour column value
    alignas(16) double fv[kRows * NR];                 // (q/a) fv_r of the current subdomain's rows
    alignas(16) double ctab[NC * kCT];
    alignas(16) double tab[kTab];
    double he[kColW * kHS];     // y at chunk ends -> final Y carries  ([column][chunk])
    double ks[kColW * kHS];     // k at chunk starts -> final X carries
    double kb[4 * kColW];       // k (zero carries) at rows 0, 1, n-2, n-1
    double ktr[4 * kColW];      // k (zero carries) at the trace stencil rows iL, iL+1, iR, iR-1
    double rtr[2 * kColW];      // raw r at the outgoing-trace rows (lo side, hi side)
    SubDev sd[kColMaxSub];      // descriptors of the launch's subdomains
    double gio[4 * kColW];      // per column of the tile: incoming traces g_lo, g_hi; U lines at the lo / hi interface
    double red[2 * P];
    uint64_t bar[P];            // per warp: its u^n box (tx bytes) and halo (cp.async arrivals) landed
    uint64_t tbar;              // per-subdomain tables
};

template <int B, int NR, int P>
__host__ __device__ constexpr size_t col_smem_bytes() {
    return sizeof(ColSmem<B, NR, P>);
}

__device__ __forceinline__ void cp_async_8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t *bar) {  // tracked by the barrier (count +1, then arrive)
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// pass A over one chunk.  DIR = -1: every row has v >= 0 (neighbour m-1), +1: v < 0 (m+1), 0: generic.
// tile_t: this thread's column in row 0 of its chunk (row stride 8); the neighbour of row l is
// nbp[l * nbs] (the next column in the tile, or halo_t[l] for the tile's edge column); jh0 = j - nv/2
// of the chunk's first row.
template <int B, int NR, int DIR>
__device__ __forceinline__ void col_pass_a(const double *tile_t, const double *halo_t, const double *fv_t, int c,
                                           double qa, double q, double qdn, double jh0, const double (&fx)[NR],
                                           double (&h)[B], int Lw, double &hend) {
    const double *nbp = nullptr;
    int nbs = 0;
    if (DIR == -1) {
        nbp = (c == 0) ? halo_t : tile_t - 1;
        nbs = (c == 0) ? 1 : kColW;
    } else if (DIR == 1) {
        nbp = (c == kColW - 1) ? halo_t : tile_t + 1;
        nbs = (c == kColW - 1) ? 1 : kColW;
    }
    double hp = 0.0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
        if (DIR == 0 && l >= Lw) break;  // ragged chunk: rows past its end are never read
        const double u = tile_t[l * kColW];
        double nb;
        if (DIR != 0) {
            nb = nbp[l * nbs];
        } else {  // v_j >= 0 <=> j >= nv/2 (exact)
            nb = (jh0 + l >= 0.0) ? ((c == 0) ? halo_t[l] : tile_t[l * kColW - 1])
                                  : ((c == kColW - 1) ? halo_t[l] : tile_t[l * kColW + 1]);
        }
        const double c1 = qdn * fabs(jh0 + l);  // (q/a) |nu_j|
        double f = 0.0;
#pragma unroll
        for (int r = 0; r < NR; ++r) f = fma(fv_t[l * NR + r], fx[r], f);
        const double rp = fma(c1, nb - u, fma(qa, u, f));  // (q/a)[(1-|nu|) u + |nu| nb] + (q/a) dt f
        if (DIR == 0) {
            h[l] = fma(q, hp, rp);
            hend = h[l];
        } else {
            h[l] = fma(q, hp, rp);
        }
        hp = h[l];
    }
    if (DIR != 0) hend = h[B - 1];
}

// --------------------------------------------------------------------------- the kernel
template <int B, int NR, int P_>
__global__ void __launch_bounds__(P_ * kWarp, (P_ >= 16) ? 1 : 16 / P_) step_col(const ColParams CP) {
    constexpr int NW = P_;
    using Sm = ColSmem<B, NR, NW>;
    constexpr int NC = Sm::NC, HS = Sm::kHS;
    constexpr int CPL = (NC + kWarp - 1) / kWarp;  // chunks per lane in the column phase (1 or 2)
    extern __shared__ __align__(128) char smraw[];
    Sm &sm = *reinterpret_cast<Sm *>(smraw);
    const StepParams &P = CP.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lane & (kColW - 1), s = lane >> 3;
    const int k = kColSub * warp + s;  // this thread's chunk
    const int L = CP.L;
    const int cr0 = k * L;             // its first unknown row
    const double q = P.q, qa = P.qa;
    const double *qp = sm.tab, *s2 = sm.tab + Sm::kQ, *kr = sm.tab + 2 * Sm::kQ;
    const int total = CP.nsub * CP.ntiles;
    const uint32_t box_bytes = static_cast<uint32_t>(kColW * kColSub * L * sizeof(double));

    // ---- prologue
    if (threadIdx.x == 0) mbar_init(&sm.tbar, 1);
    if (lane == 0) mbar_init(&sm.bar[warp], 1);
    fence_mbar_init();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&sm.tbar, static_cast<uint32_t>(Sm::kTab * sizeof(double) + CP.nsub * sizeof(SubDev)));
        bulk_g2s(sm.tab, CP.tabs, Sm::kTab * sizeof(double), &sm.tbar);
        bulk_g2s(sm.sd, P.subs, static_cast<uint32_t>(CP.nsub * sizeof(SubDev)), &sm.tbar);
    }
    __syncthreads();
    mbar_wait(&sm.tbar, 0);
    uint32_t tph = 1;  // tables barrier: next phase parity
    uint32_t bph = 0;  // this warp's slot barrier: next phase parity

    // issue this warp's load of tile g (u^n box + halo column); no-op for steps from u0
    auto issue = [&](int g) {
        const int sub = g / CP.ntiles, t = g - sub * CP.ntiles;
        const SubDev &S = sm.sd[sub];
        const int n = S.n, first = S.first, lo = S.lo;
        const int rows = max(0, min(kColSub * L, n - kColSub * L * warp));  // rows of this warp's box
        if (rows == 0) return;
        const double *src = S.slab[P.n & 1];
        const int r0 = kColSub * L * warp;
        const int mL = (kColW * t - 1 + P.nx) % P.nx, mR = (kColW * t + kColW) % P.nx;
        for (int i = lane; i < rows; i += kWarp) {
            const int row = r0 + i, j = first + row;
            const int mm = (2 * j - P.nv >= 0) ? mL : mR;
            cp_async_8(&sm.halo[row], src + static_cast<size_t>(first - lo + row) * P.nx + mm);
        }
        cp_async_arrive(&sm.bar[warp]);
        __syncwarp();
        if (lane == 0) {  // two boxes of 8 x 2L (smaller boxes stream faster; both 128-B aligned in smem)
            fence_proxy_async_smem();
            mbar_expect_tx(&sm.bar[warp], box_bytes);
            const CUtensorMap *map = CP.tmaps + 2 * sub + (P.n & 1);
            tma_load_2d(sm.tile[warp], map, kColW * t, r0, &sm.bar[warp]);
            tma_load_2d(sm.tile[warp] + 2 * L * kColW, map, kColW * t, r0 + 2 * L, &sm.bar[warp]);
        }
    };

    int cur_sub = -1;
    double eif = 0.0, et = 0.0;
    KFP_WT_DECL
    // contiguous tile range of this CTA (at most one change of subdomain per step for ranges <= ntiles)
    const int per = (total + gridDim.x - 1) / gridDim.x;
    const int g_begin = blockIdx.x * per, g_end = min(total, g_begin + per);
    grid_dep_wait();  // the previous step's u^n is complete
    if (g_begin < g_end && !P.from_u0) issue(g_begin);
    for (int g = g_begin; g < g_end; ++g) {
        const int sub = g / CP.ntiles, t = g - sub * CP.ntiles;
        if (sub != cur_sub) {
            __syncthreads();  // nobody still reads the previous subdomain's fv / chunk table
            if (threadIdx.x == 0) {
                const int n = sm.sd[sub].n, first = sm.sd[sub].first;
                const uint32_t fvb = static_cast<uint32_t>(((n * NR * 8) + 15) / 16 * 16);
                const uint32_t ctb = static_cast<uint32_t>(NC * kCT * sizeof(double));
                mbar_expect_tx(&sm.tbar, fvb + ctb);
                bulk_g2s(sm.fv, CP.fvq + static_cast<size_t>(first) * NR, fvb, &sm.tbar);
                bulk_g2s(sm.ctab, CP.ctab + static_cast<size_t>(sub) * NC * kCT, ctb, &sm.tbar);
            }
            mbar_wait(&sm.tbar, tph & 1);
            tph ^= 1;
            cur_sub = sub;
        }
        KFP_WT(8)  // 8: pass C of the previous tile + tables
        const SubDev &S = sm.sd[sub];
        const int n = S.n;
        const int Lw = max(0, min(L, n - cr0));     // rows of this thread's chunk
        const int m0 = kColW * t, m = m0 + c;
        if (warp == NW - 1 && lane < 4 * kColW) {  // incoming traces and U lines of this step, for the column phase
            const int qq = lane >> 3, mc = m0 + (lane & (kColW - 1));
            const size_t go = static_cast<size_t>(P.n) * P.nx + mc;
            double v = 0.0;
            if (qq == 0 && S.ltype != END_PHYS) v = __ldg(S.gL[P.par_in_lo] + go);
            if (qq == 1 && S.rtype != END_PHYS) v = __ldg(S.gR[P.par_in] + go);
            if (qq == 2 && S.ifL >= 0 && P.Ulines) v = __ldg(P.Ulines + (static_cast<size_t>(S.ifL) * P.nt + P.n) * P.nx + mc);
            if (qq == 3 && S.ifR >= 0 && P.Ulines) v = __ldg(P.Ulines + (static_cast<size_t>(S.ifR) * P.nt + P.n) * P.nx + mc);
            sm.gio[lane] = v;
        }
        double fx[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) fx[r] = (r < P.f_rank) ? P.cf[r] * __ldg(P.fx + r * P.nx + m) : 0.0;

        // ---- passes A and B (registers)
        double h[B];
        double hend = 0.0, kst = 0.0;
        const int wrows = max(0, min(kColSub * L, n - kColSub * L * warp));
        double *tile_w = sm.tile[warp];
        if (wrows > 0) {
            if (!P.from_u0) {
                mbar_wait(&sm.bar[warp], bph);
                bph ^= 1;
                KFP_WT(1)  // 1: data wait
            } else {  // u^0 from the separable u0 tables (0 B of HBM), incl. the halo column
                const int r0 = kColSub * L * warp;
                const int mL = (m0 - 1 + P.nx) % P.nx, mR = (m0 + kColW) % P.nx;
                for (int i = lane; i < wrows * kColW; i += kWarp) {
                    const int row = i / kColW, cc = i - row * kColW, jn = S.first + r0 + row;
                    double sacc = 0.0;
                    for (int r = 0; r < P.u0_rank; ++r)
                        sacc = fma(__ldg(P.u0v + r * (P.nv + 1) + jn), __ldg(P.u0x + r * P.nx + m0 + cc), sacc);
                    tile_w[row * kColW + cc] = sacc;
                }
                for (int i = lane; i < wrows; i += kWarp) {
                    const int row = r0 + i, jn = S.first + row;
                    const int mm = (2 * jn - P.nv >= 0) ? mL : mR;
                    double sacc = 0.0;
                    for (int r = 0; r < P.u0_rank; ++r)
                        sacc = fma(__ldg(P.u0v + r * (P.nv + 1) + jn), __ldg(P.u0x + r * P.nx + mm), sacc);
                    sm.halo[row] = sacc;
                }
                __syncwarp();
            }
        }
        if (Lw > 0) {
            const double *tile_t = tile_w + s * L * kColW + c;
            const double *halo_t = sm.halo + cr0;
            const double *fv_t = sm.fv + cr0 * NR;
            const int jv2_0 = 2 * (S.first + cr0) - P.nv, jv2_1 = jv2_0 + 2 * (Lw - 1);
            const double jh0 = static_cast<double>(S.first + cr0 - P.nv / 2);
            const bool full = (Lw == B) && (cr0 + Lw <= n - 2);
            if (full && jv2_0 >= 0)
                col_pass_a<B, NR, -1>(tile_t, halo_t, fv_t, c, qa, q, CP.qdn, jh0, fx, h, Lw, hend);
            else if (full && jv2_1 < 0)
                col_pass_a<B, NR, 1>(tile_t, halo_t, fv_t, c, qa, q, CP.qdn, jh0, fx, h, Lw, hend);
            else
                col_pass_a<B, NR, 0>(tile_t, halo_t, fv_t, c, qa, q, CP.qdn, jh0, fx, h, Lw, hend);
            // raw r (no incoming-trace term) at the outgoing-trace rows, for the Robin trace (R11)
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const int itr = side ? S.iR_tr : S.iL_tr;
                const bool on = itr >= 0 && itr < n && itr >= cr0 && itr < cr0 + Lw;
                if (on) {  // r = r'/(q/a) with r' formed exactly as in pass A
                    const int l = itr - cr0, jn = S.first + itr;
                    const double u = tile_t[l * kColW];
                    const double nb = (2 * jn - P.nv >= 0) ? ((c == 0) ? halo_t[l] : tile_t[l * kColW - 1])
                                                            : ((c == kColW - 1) ? halo_t[l] : tile_t[l * kColW + 1]);
                    double f = 0.0;
#pragma unroll
                    for (int r = 0; r < NR; ++r) f = fma(fv_t[l * NR + r], fx[r], f);
                    const double c1 = CP.qdn * fabs(static_cast<double>(jn - P.nv / 2));
                    sm.rtr[side * kColW + c] = fma(c1, nb - u, fma(qa, u, f)) / qa;
                }
            }
        }
        // the slot (and halo) are consumed: prefetch this warp's share of the next tile
        __syncwarp();
        KFP_WT(2)  // 2: pass A
        if (g + 1 < g_end && !P.from_u0) issue(g + 1);
        KFP_WT(3)  // 3: issue next
        if (Lw > 0) {
            double kl = 0.0, kl2 = 0.0;
            const bool full = (Lw == B) && (cr0 + Lw <= n - 2);
            if (full) {
                kst = pass_b_full<B>(h, q);
            } else {
                kst = pass_b_ragged<B>(h, q, Lw, kl, kl2);
                if (cr0 + Lw == n) {
                    sm.kb[3 * kColW + c] = kl;
                    if (Lw >= 2) sm.kb[2 * kColW + c] = kl2;
                } else if (cr0 + Lw == n - 1) {
                    sm.kb[2 * kColW + c] = kl;
                }
            }
            if (cr0 == 0) {
                sm.kb[0 * kColW + c] = h[0];
                if (Lw >= 2) sm.kb[1 * kColW + c] = h[1];
            } else if (cr0 == 1) {
                sm.kb[1 * kColW + c] = h[0];
            }
            // k (zero carries) at the trace stencil rows
            const int trow[4] = {S.iL_tr, S.iL_tr + 1, S.iR_tr, S.iR_tr - 1};
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int rr = trow[qq];
                if (rr >= cr0 && rr < cr0 + Lw && (qq < 2 ? S.iL_tr >= 0 : (S.iR_tr >= 0 && S.iR_tr < n))) {
#pragma unroll
                    for (int l = 0; l < B; ++l)
                        if (cr0 + l == rr) sm.ktr[qq * kColW + c] = h[l];
                }
            }
        }
        sm.he[c * HS + k] = hend;
        sm.ks[c * HS + k] = kst;
        KFP_WT(4)  // 4: pass B
        __syncthreads();  // S1
        KFP_WT(5)  // 5: S1

        // ---- column phase: warp c handles column c, lane i the chunks CPL i .. CPL i + CPL - 1
        if (warp < kColW) {
            const int cc = warp, mc = m0 + cc;
            const size_t go = static_cast<size_t>(P.n) * P.nx + mc;
            const double *ct = sm.ctab;
            const double gl = sm.gio[0 * kColW + cc], gh = sm.gio[1 * kColW + cc];
            const double Yt0 = S.injL * gl / P.a, Xb0 = S.injR * gh / P.a;
            double Qv[CPL], he_[CPL], ks_[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int kk = CPL * lane + e;
                const bool ok = kk < NC;
                Qv[e] = ok ? ct[kk * kCT + 0] : 1.0;
                he_[e] = ok ? sm.he[cc * HS + kk] : 0.0;
                ks_[e] = ok ? sm.ks[cc * HS + kk] : 0.0;
            }
            // forward: y_out(k) = Q_k y_out(k-1) + he_k ; lane map (A, Bv): y -> A y + Bv
            double A = 1.0, Bv = 0.0;
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                Bv = fma(Qv[e], Bv, he_[e]);
                A *= Qv[e];
            }
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const double Au = __shfl_up_sync(0xffffffffu, A, d), Bu = __shfl_up_sync(0xffffffffu, Bv, d);
                if (lane >= d) {
                    Bv = fma(A, Bu, Bv);
                    A *= Au;
                }
            }
            const double yinc = fma(A, Yt0, Bv);                        // y after this lane's chunks
            double ybef = __shfl_up_sync(0xffffffffu, yinc, 1);
            if (lane == 0) ybef = Yt0;
            double yin[CPL], z0[CPL];
            {
                double y = ybef;
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    const int kk = CPL * lane + e;
                    yin[e] = y;
                    z0[e] = (kk < NC) ? fma(ct[kk * kCT + 1], y, ks_[e]) : 0.0;
                    y = fma(Qv[e], y, he_[e]);
                }
            }
            // backward: x_start(k) = Q_k x_in(k) + z0_k, x_in(k) = x_start(k+1), x_in(NC-1) = Xb0
            A = 1.0;
            Bv = 0.0;
#pragma unroll
            for (int e = CPL - 1; e >= 0; --e) {
                Bv = fma(Qv[e], Bv, z0[e]);
                A *= Qv[e];
            }
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const double Ad = __shfl_down_sync(0xffffffffu, A, d), Bd = __shfl_down_sync(0xffffffffu, Bv, d);
                if (lane + d < kWarp) {
                    Bv = fma(A, Bd, Bv);
                    A *= Ad;
                }
            }
            const double xinc = fma(A, Xb0, Bv);                        // x at the first row of this lane's chunks
            double xaft = __shfl_down_sync(0xffffffffu, xinc, 1);
            if (lane == kWarp - 1) xaft = Xb0;
            double xin[CPL];
            {
                double x = xaft;
#pragma unroll
                for (int e = CPL - 1; e >= 0; --e) {
                    xin[e] = x;
                    x = fma(Qv[e], x, z0[e]);
                }
            }
            // x~ at the column's rows 0, 1, n-2, n-1 with these carries (the lane owning each row)
            auto x_at = [&](int row, const double *kz, const double *Yc, const double *Xc) -> double {
                double val = 0.0;
                const int kk = row / L, l = row - kk * L;
                const int owner = kk / CPL, e = kk - owner * CPL;
                if (lane == owner) {
                    const int Lk = max(0, min(L, n - kk * L));
#pragma unroll
                    for (int ee = 0; ee < CPL; ++ee)
                        if (ee == e) val = *kz + kap_s(qp, s2, l, Lk) * Yc[ee] + qp[Lk - l] * Xc[ee];
                }
                return __shfl_sync(0xffffffffu, val, owner);
            };
            const double x0 = x_at(0, &sm.kb[0 * kColW + cc], yin, xin);
            const double x1 = x_at(1, &sm.kb[1 * kColW + cc], yin, xin);
            const double xn2 = x_at(n - 2, &sm.kb[2 * kColW + cc], yin, xin);
            const double xn1 = x_at(n - 1, &sm.kb[3 * kColW + cc], yin, xin);
            const double s0 = fma(S.wt0, x0, S.wt1 * x1), s1 = fma(S.wb0, xn2, S.wb1 * xn1);
            const double dY = -fma(S.Mi00, s0, S.Mi01 * s1) / P.a, dX = -fma(S.Mi10, s0, S.Mi11 * s1) / P.a;
            double Yf[CPL], Xf[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int kk = CPL * lane + e;
                if (kk < NC) {
                    Yf[e] = fma(ct[kk * kCT + 2], dY, yin[e]);
                    Xf[e] = fma(ct[kk * kCT + 4], dX, fma(ct[kk * kCT + 3], dY, xin[e]));
                    sm.he[cc * HS + kk] = Yf[e];
                    sm.ks[cc * HS + kk] = Xf[e];
                } else {
                    Yf[e] = Xf[e] = 0.0;
                }
            }
            // outgoing traces at t_{n+1} (R11) and interface errors; every x_at
            // (a shuffle) is evaluated unconditionally on clamped rows, the results are used below
            const bool rob = P.send_robin;
            const double inv_h = 1.0 / P.hv, half_h_dt = 0.5 * P.hv / P.dt;
            auto clampr = [&](int r) { return min(max(r, 0), n - 1); };
            const double xL = x_at(clampr(S.iL_tr), &sm.ktr[0 * kColW + cc], Yf, Xf);
            const double xL1 = x_at(clampr(S.iL_tr + 1), &sm.ktr[1 * kColW + cc], Yf, Xf);
            const double xR = x_at(clampr(S.iR_tr), &sm.ktr[2 * kColW + cc], Yf, Xf);
            const double xR1 = x_at(clampr(S.iR_tr - 1), &sm.ktr[3 * kColW + cc], Yf, Xf);
            const double xe0 = x_at(0, &sm.kb[0 * kColW + cc], Yf, Xf);
            const double xe1 = x_at(n - 1, &sm.kb[3 * kColW + cc], Yf, Xf);
            if (lane == 0) {
                if (S.iL_tr >= 0)  // (p + d_v) u at hi_{s-1}, half-cell flux on [c, c+h/2]
                    S.sendL[P.par_out][go] = rob ? S.tpL * xL - ((xL - xL1) * inv_h + half_h_dt * (xL - sm.rtr[0 * kColW + cc])) : xL;
                else if (S.iL_tr == -1)
                    S.sendL[P.par_out][go] = gl;  // Dirichlet without overlap: the end node is the trace node
                if (S.iR_tr >= 0 && S.iR_tr < n)  // (q - d_v) u at lo_{s+1}, flux on [c-h/2, c]
                    S.sendR[P.par_out][go] = rob ? S.tpR * xR - ((xR - xR1) * inv_h + half_h_dt * (xR - sm.rtr[1 * kColW + cc])) : xR;
                else if (S.iR_tr == n)
                    S.sendR[P.par_out][go] = gh;
                if (P.errIF) {
                    if (S.ifL >= 0) eif = fmax(eif, fabs(((S.ltype == END_DIRI) ? gl : xe0) - sm.gio[2 * kColW + cc]));
                    if (S.ifR >= 0) eif = fmax(eif, fabs(((S.rtype == END_DIRI) ? gh : xe1) - sm.gio[3 * kColW + cc]));
                }
            }
            if (P.last && lane == 0) {  // end nodes of the slab at T: Dirichlet value or 0 (physical)
                double *un = S.slab[(P.n + 1) & 1];
                if (S.ltype == END_DIRI) {
                    un[mc] = gl;
                    if (P.errT) et = fmax(et, fabs(gl - P.UT[static_cast<size_t>(S.lo) * P.nx + mc]));
                } else if (S.ltype == END_PHYS) {
                    un[mc] = 0.0;
                }
                if (S.rtype == END_DIRI) {
                    un[static_cast<size_t>(S.hi - S.lo) * P.nx + mc] = gh;
                    if (P.errT) et = fmax(et, fabs(gh - P.UT[static_cast<size_t>(S.hi) * P.nx + mc]));
                } else if (S.rtype == END_PHYS) {
                    un[static_cast<size_t>(S.hi - S.lo) * P.nx + mc] = 0.0;
                }
            }
        }
        KFP_WT(6)  // 6: column phase
        __syncthreads();  // S2: final carries visible
        KFP_WT(7)  // 7: S2

        // ---- pass C: x = k + kap Y + rho X; coalesced stores of u^{n+1}
        if (Lw > 0) {
            const double Y = sm.he[c * HS + k], X = sm.ks[c * HS + k];
            if (Lw == B && L == B) {
#pragma unroll
                for (int l = 0; l < B; ++l) h[l] = fma(kr[2 * l], Y, fma(kr[2 * l + 1], X, h[l]));
            } else {
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) h[l] = fma(kap_s(qp, s2, l, Lw), Y, fma(qp[Lw - l], X, h[l]));
            }
            double *dst = S.slab[(P.n + 1) & 1] + static_cast<size_t>(S.first - S.lo + cr0) * P.nx + m;
            const size_t pitch = P.nx;
            if (Lw == B) {
#pragma unroll
                for (int l = 0; l < B; ++l) st_global_f64(dst + l * pitch, h[l]);
            } else {
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) dst[l * pitch] = h[l];
            }
            if (P.last && P.errT) {  // error at T on every unknown row
                const double *ut = P.UT + static_cast<size_t>(S.first + cr0) * P.nx + m;
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) et = fmax(et, fabs(h[l] - ut[l * pitch]));
            }
            if (P.record)  // monodomain: U at the recorded lines
                for (int i = 0; i < CP.nrec; ++i) {
                    const int row = __ldg(CP.rec_rows + i);
                    if (row >= cr0 && row < cr0 + Lw) {
#pragma unroll
                        for (int l = 0; l < B; ++l)
                            if (cr0 + l == row) P.rec[(static_cast<size_t>(i) * P.nt + P.n) * P.nx + m] = h[l];
                    }
                }
        }
    }
    KFP_WT(8)  // 8: pass C (+ loop)
    KFP_WT_FLUSH
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
            for (int w = 0; w < NW; ++w) {
                a = fmax(a, sm.red[w]);
                b = fmax(b, sm.red[NW + w]);
            }
            if (a > 0.0) atomic_max_pos(P.errIF, a);
            if (b > 0.0 && P.errT) atomic_max_pos(P.errT, b);
        }
    }
}

}  // namespace kfp

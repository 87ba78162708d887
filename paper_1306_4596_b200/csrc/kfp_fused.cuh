// kfp_fused.cuh -- the hot kernel: one fused time step of every local subdomain
// (transport + forcing + v-tridiagonal solve + transmission traces + errors),
// sm_100a, TMA tile loads, register-resident chunks, cluster (DSMEM) carries.
//
// Geometry.  A cluster of C CTAs owns one 32-column x-tile of one
// subdomain's column stack; CTA `blk` owns the unknown rows [blk*R, blk*R+R),
// R = P*L; warp w owns the chunk of L <= B rows starting at blk*R + w*L, lane =
// x-column.  The chunk lives in registers through the three passes:
//   A  r' = (q/a)[(1-|nu|) u + |nu| u_nb + dt f]  and the forward scan
//      h_l = q h_{l-1} + r'_l (zero carry)                       (P:496-516 + B^{-1} part 1)
//   B  backward scan k_l = q k_{l+1} + h_l (zero carry)          (B^{-1} part 2)
//   C  x_l = k_l + kap(l, L) Y + q^{L-l} X with the chunk carries Y (y just above
//      the chunk) and X (x just below it).
// The carries of a linear constant-coefficient recurrence are closed-form sums
// of powers of q over the preceding / following chunks, so every warp computes
// its own from the other chunks' end values (no serial chain); the same holds
// across the CTAs of the cluster (distributed shared memory) and for the two
// Woodbury boundary terms of the column system (kfp_device.cuh header).
// u^n arrives by one cp.async.bulk.tensor (TMA) per warp: a box of (2+32+2) x L
// fp64 (the tile plus a 2-column halo on each side) into shared memory; the
// upwind neighbour is then a shared-memory load at lane +- 1.
#pragma once
#include <cuda.h>

#include "kfp_device.cuh"

namespace kfp {

// halo columns per side in the smem tile: 2, so that the TMA box starts on a
// 16-B aligned global column (a box starting at an odd column faults)
constexpr int kHalo = 2;
constexpr int kTW = kWarp + 2 * kHalo;       // 36 doubles (288 B) per smem tile row
constexpr int kFusedWarps = 16;              // P
constexpr int kNRmax = 4;                    // forcing ranks supported by the coefficient table
constexpr int kMaxFusedCluster = 8;          // portable cluster size

struct FusedParams {
    StepParams S;                 // common step parameters (kfp_device.cuh)
    const CUtensorMap *tmaps;     // [nsub][2] tensor maps of the slabs' unknown rows (by step parity)
    int L;                        // chunk length (rows per warp), R = P*L rows per CTA
    int nrec;                     // monodomain line recording: number of recorded rows
    const int *rec_rows;          // [nrec] unknown-row index of each recorded line (in line order)
    const double *l2c;            // [nsub][kL2C] level-2 constants per subdomain (host-computed, see kfp_api.cu)
    const CUtensorMap *smaps;     // [nsub][2] store maps (box 32 x L) of the slabs' unknown rows
    const double *coefT;          // [nv+1][2+NR] per-node (q/a)(1-|nu|), (q/a)|nu|, (q/a) fv_r(j)
    const double *tabs;           // qp[kQ] | s2[kQ] | kr[2B] for this plan (host-computed)
};
// level-2 constants of one subdomain (doubles): for block c < 8: q^{R_c}, kap(0,R_c), q^{b_c},
// kap_col(e_c), q^{n-e_c} (b_c = c R, e_c = b_c + R_c, kap_col(r) = q^{r+1} s2(n-r)); for the
// boundary rows 0,1,n-2,n-1: kap(l, R_c), q^{R_c - l} of their block.
constexpr int kL2C = 5 * 8 + 8;
enum : int { L2_QR = 0, L2_K0 = 8, L2_QB = 16, L2_KB = 24, L2_QE = 32, L2_KQ = 40, L2_RQ = 44 };

// --------------------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int x, int y, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ double ld_dsmem(const double *local_addr, int rank) {
    // read a double of CTA `rank`'s shared memory at the same offset as local_addr
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t mapa_u32(const void *local_addr, int rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(rank));
    return remote;
}
// push two doubles into CTA `rank`'s shared memory (same offset as local dst), completing
// 16 bytes of transaction count on that CTA's mbarrier at the offset of local bar
__device__ __forceinline__ void st_async_v2(const void *dst, int rank, double a, double b, const uint64_t *bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                     mapa_u32(dst, rank)),
                 "d"(a), "d"(b), "r"(mapa_u32(bar, rank))
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
template <int B>
__host__ __device__ constexpr int fused_kq() {
    return ((kFusedWarps * B + 2) + 1) / 2 * 2;
}

template <int B, int NR>
struct FusedSmem {
    static constexpr int kSlot = slot_doubles<B>();
    static constexpr int kRows = kFusedWarps * B;
    static constexpr int kCoef = 2 + NR;   // c0', c1', g_0' .. g_{NR-1}'
    static constexpr int kQ = fused_kq<B>();
    static constexpr int kTab = 2 * kQ + 2 * B;
    alignas(128) double tile[kFusedWarps * kSlot];  // per warp: u^n rows [L][36], then x rows [L][32] (dense)
    alignas(16) double coef[kRows * kCoef];         // per warp: its chunk's rows of coefT
    alignas(16) double tab[kTab];                   // qp[kQ] | s2[kQ] | kr[2B]  (copy of FusedParams::tabs)
    alignas(16) double l2c[kL2C];                   // level-2 constants of this subdomain
    double he[kFusedWarps * kWarp];        // y at the chunk's last row (zero carry); reused as Yb[8][32]
    double ks[kFusedWarps * kWarp];        // k at the chunk's first row (zero carry); reused as Xb[8][32]
    double Y0[kFusedWarps * kWarp];        // chunk carries with zero block carries
    double X0[kFusedWarps * kWarp];
    double kb[4 * kWarp];                  // k at the column's rows 0,1,n-2,n-1 (chunk-local zero carries)
    double pub[6 * kWarp];                 // this block's F, G and boundary values (pushed to the cluster)
    double2 rFG[kMaxFusedCluster * kWarp]; // received (F, G) of every block of the cluster
    double2 rA[2 * kWarp];                 // received boundary values: (x~_0, x~_1), (x~_{n-2}, x~_{n-1})
    double cb[2 * kWarp];                  // this block's carries Y_blk, X_blk
    double gin[2 * kWarp];                 // incoming traces at t_{n+1} (lo end, hi end)
    double rtr[2 * kWarp];                 // raw r at the outgoing-trace rows
    double red[2 * kFusedWarps];
    uint64_t bar[kFusedWarps];             // tile (TMA) + coefficient rows, per warp
    uint64_t tbar;                         // tables
    uint64_t xbar;                         // cluster exchange completion
};

template <int B, int NR>
__host__ __device__ constexpr size_t fused_smem_bytes() {
    return sizeof(FusedSmem<B, NR>);
}

// --------------------------------------------------------------------------- passes
// DIR = -1: every row of the chunk has v >= 0 (upwind neighbour m-1); +1: v < 0
// (neighbour m+1); 0: generic (per-row side, ragged length).
template <int B, int NR, int DIR>
__device__ __forceinline__ void pass_a_reg(const double *tile_w, const double *coef_w, int lane, double q,
                                           const double (&fx)[NR], double (&h)[B], int Lw, int jv2_0, double &hend) {
    constexpr int kC = 2 + NR;
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
        } else {
            nb = row[DIR];
        }
        double f = 0.0;
#pragma unroll
        for (int r = 0; r < NR; ++r) f = fma(c[2 + r], fx[r], f);
        const double rp = fma(c[1], nb, fma(c[0], u, f));
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

// --------------------------------------------------------------------------- the kernel
template <int B, int NR>
__global__ void __launch_bounds__(kFusedWarps * kWarp, 2) step_fused_tma(const FusedParams FP) {
    using Sm = FusedSmem<B, NR>;
    extern __shared__ __align__(128) char smraw[];
    Sm &sm = *reinterpret_cast<Sm *>(smraw);
    const StepParams &P = FP.S;
    const int blk = static_cast<int>(cg::this_cluster().block_rank());
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = blockIdx.z;
    const SubDev &S = P.subs[sub];
    const int n = S.n, L = FP.L, R = kFusedWarps * L;
    const int m0 = blockIdx.y * kWarp, w = min(kWarp, P.nx - m0);
    const int m = m0 + min(lane, w - 1);
    const bool active = lane < w;
    const int rb0 = blk * R;                                    // first unknown row of this block
    const int Rb = max(0, min(R, n - rb0));                     // rows of this block
    const int s_w = warp * L;                                   // chunk start (block-local)
    const int Lw = max(0, min(L, Rb - s_w));                    // rows of this warp's chunk
    const int e_w = s_w + Lw;                                   // chunk end (block-local, exclusive)
    const int cr0 = rb0 + s_w;                                  // first column row of the chunk
    const int nblk = S.nblk;
    const bool live = blk < nblk;                               // the block holds rows of the column
    const double q = P.q;
    const CUtensorMap *tmap = FP.tmaps + 2 * sub + (P.n & 1);
    double *unew_slab = S.slab[(P.n + 1) & 1];
    double *unew = unew_slab + static_cast<size_t>(S.first - S.lo) * P.nx;
    double *tile_w = sm.tile + warp * Sm::kSlot;
    const size_t goff = static_cast<size_t>(P.n) * P.nx + m;   // row t_{n+1} of [nt][nx] arrays
    auto inblk = [&](int i) { return i >= rb0 && i < rb0 + Rb; };
    // rows that need a look after pass C (outgoing traces, Robin-end interface errors, recorded lines)
    bool special = false;
    if (S.iL_tr >= 0) special |= inblk(S.iL_tr) || inblk(S.iL_tr + 1);
    if (S.iR_tr >= 0 && S.iR_tr < n) special |= inblk(S.iR_tr) || inblk(S.iR_tr - 1);
    if (S.ltype == END_ROBIN && S.ifL >= 0) special |= inblk(0);
    if (S.rtype == END_ROBIN && S.ifR >= 0) special |= inblk(n - 1);
    if (P.record) special = special || live;
    const bool errs = (P.errIF != nullptr) && (special || P.last || blk == 0 || blk == nblk - 1);

    const double *qp = sm.tab, *s2 = sm.tab + Sm::kQ, *kr = sm.tab + 2 * Sm::kQ;
    double *coef_w = sm.coef + warp * B * Sm::kCoef;
    const uint32_t coef_bytes = static_cast<uint32_t>(Lw * Sm::kCoef * sizeof(double));

    // ---- prologue (constant data only: overlaps the previous step under PDL)
    if (threadIdx.x == 0) {
        mbar_init(&sm.xbar, 1);
        mbar_init(&sm.tbar, 1);
        prefetch_tmap(tmap);
    }
    if (lane == 0) mbar_init(&sm.bar[warp], 1);
    fence_mbar_init();
    cluster_arrive_relaxed();  // every CTA's xbar is initialised before anybody pushes (wait below)
    if (threadIdx.x == 0) {    // q-power tables, pass-C coefficients, level-2 constants
        mbar_expect_tx(&sm.tbar, static_cast<uint32_t>((Sm::kTab + kL2C) * sizeof(double)));
        bulk_g2s(sm.tab, FP.tabs, Sm::kTab * sizeof(double), &sm.tbar);
        bulk_g2s(sm.l2c, FP.l2c + sub * kL2C, kL2C * sizeof(double), &sm.tbar);
    }
    if (lane == 0 && Lw > 0) { // this chunk's per-row coefficients (+ its tile below)
        const uint32_t tile_bytes = P.from_u0 ? 0u : static_cast<uint32_t>(kTW * L * sizeof(double));
        mbar_expect_tx(&sm.bar[warp], coef_bytes + tile_bytes);
        bulk_g2s(coef_w, FP.coefT + static_cast<size_t>(S.first + cr0) * Sm::kCoef, coef_bytes, &sm.bar[warp]);
    }
    double fx[NR];  // this lane's forcing profile times dt ft_r(t_{n+1})
#pragma unroll
    for (int r = 0; r < NR; ++r) fx[r] = (r < P.f_rank) ? P.cf[r] * __ldg(P.fx + r * P.nx + m) : 0.0;
    // incoming traces of this step (written by the previous iteration, complete before this launch chain)
    if (warp == 0) {
        sm.gin[lane] = (S.ltype != END_PHYS) ? S.gL[P.par_in][goff] : 0.0;
        sm.gin[kWarp + lane] = (S.rtype != END_PHYS) ? S.gR[P.par_in][goff] : 0.0;
    }

    // ---- wait for the previous step, then load this warp's chunk of u^n with one TMA
    grid_dep_wait();
    if (Lw > 0 && !P.from_u0 && lane == 0) tma_load_2d(tile_w, tmap, m0 - kHalo, cr0, &sm.bar[warp]);

    double h[B];
    double hend = 0.0, kst = 0.0, eif = 0.0, et = 0.0;
    if (Lw > 0) {
        mbar_wait(&sm.bar[warp], 0);  // coefficient rows (and the tile unless from u0)
        if (P.from_u0) {  // u^0 from the separable u0 tables (0 B of HBM), incl. the halo columns
            for (int l = 0; l < Lw; ++l) {
                const int j = S.first + cr0 + l;
                for (int c = lane; c < kTW; c += kWarp) {
                    const int mm = ((m0 - kHalo + c) % P.nx + P.nx) % P.nx;
                    double s = 0.0;
                    for (int r = 0; r < P.u0_rank; ++r)
                        s = fma(__ldg(P.u0v + r * (P.nv + 1) + j), __ldg(P.u0x + r * P.nx + mm), s);
                    tile_w[l * kTW + c] = s;
                }
            }
            __syncwarp();
        } else {
            // periodic wrap of the halo at the ends of the x range (TMA zero-fills out-of-range columns)
            if (m0 == 0 || m0 + w == P.nx) {
                const double *src = S.slab[P.n & 1] + static_cast<size_t>(S.first - S.lo + cr0) * P.nx;
                if (m0 == 0 && lane < Lw) tile_w[lane * kTW + kHalo - 1] = src[static_cast<size_t>(lane) * P.nx + P.nx - 1];
                if (m0 + w == P.nx && lane < Lw) tile_w[lane * kTW + kHalo + w] = src[static_cast<size_t>(lane) * P.nx];
                __syncwarp();
            }
        }
        const int jv2_0 = 2 * (S.first + cr0) - P.nv;          // 2 j - nv of the chunk's first row
        const int jv2_1 = jv2_0 + 2 * (Lw - 1);
        // full chunks take the unpredicated paths; the chunk holding the column's
        // last two rows takes the ragged one (it captures their k values)
        const bool full = (Lw == B) && (cr0 + Lw <= n - 2);
        if (full && jv2_0 >= 0) pass_a_reg<B, NR, -1>(tile_w, coef_w, lane, q, fx, h, Lw, jv2_0, hend);
        else if (full && jv2_1 < 0) pass_a_reg<B, NR, 1>(tile_w, coef_w, lane, q, fx, h, Lw, jv2_0, hend);
        else pass_a_reg<B, NR, 0>(tile_w, coef_w, lane, q, fx, h, Lw, jv2_0, hend);
        // raw r (no incoming-trace term) at the outgoing-trace rows, for the Robin trace (R11)
        if (special) {
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const int itr = side ? S.iR_tr : S.iL_tr;
                if (itr >= cr0 && itr < cr0 + Lw) {
                    const int l = itr - cr0, j = S.first + itr;
                    const double2 rc = __ldg(P.rowc + j);
                    const double u = tile_w[l * kTW + kHalo + lane];
                    const double nb = tile_w[l * kTW + kHalo + lane + ((2 * j - P.nv >= 0) ? -1 : 1)];
                    double f = 0.0;
                    for (int r = 0; r < P.f_rank; ++r) f = fma(__ldg(P.fv + r * (P.nv + 1) + j), fx[r], f);  // fx has dt f_t
                    sm.rtr[side * kWarp + lane] = fma(rc.x, u, fma(rc.y, nb, f));
                }
            }
        }
        if (full) {
            kst = pass_b_full<B>(h, q);
        } else {
            double kl = 0.0, kl2 = 0.0;
            kst = pass_b_ragged<B>(h, q, Lw, kl, kl2);
            if (cr0 + Lw == n) {
                sm.kb[3 * kWarp + lane] = kl;
                if (Lw >= 2) sm.kb[2 * kWarp + lane] = kl2;
            } else if (cr0 + Lw == n - 1) {
                sm.kb[2 * kWarp + lane] = kl;
            }
        }
        if (cr0 == 0) {
            sm.kb[0 * kWarp + lane] = h[0];
            if (Lw >= 2) sm.kb[1 * kWarp + lane] = h[1];
        } else if (cr0 == 1) {
            sm.kb[1 * kWarp + lane] = h[0];
        }
    }
    sm.he[warp * kWarp + lane] = hend;
    sm.ks[warp * kWarp + lane] = kst;
    mbar_wait(&sm.tbar, 0);  // q-power tables (long since arrived)
    __syncthreads();

    // ---- level 1, transposed: warp w scans the 16 chunks of columns 2w, 2w+1 (half-warp each,
    //      lane = chunk) with affine Kogge-Stone scans:  y_out(k) = q^{L_k} y_out(k-1) + he_k,
    //      x_start(k) = q^{L_k} x_start(k+1) + Z0_k,  Z0_k = ks_k + kap(0, L_k) Y0_k.
    {
        const int col = 2 * warp + (lane >> 4), k = lane & 15;
        const int Lk = max(0, min(L, Rb - k * L));
        const double Qk = qp[Lk];
        double A = Qk, Bv = sm.he[k * kWarp + col];
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
            const double Au = __shfl_up_sync(0xffffffffu, A, d, 16), Bu = __shfl_up_sync(0xffffffffu, Bv, d, 16);
            if (k >= d) {
                Bv = fma(A, Bu, Bv);
                A *= Au;
            }
        }
        const double F = __shfl_sync(0xffffffffu, Bv, 15, 16);   // y at the block's last row
        double y0 = __shfl_up_sync(0xffffffffu, Bv, 1, 16);
        if (k == 0) y0 = 0.0;
        const double z0 = (Lk > 0) ? fma(kap_s(qp, s2, 0, Lk), y0, sm.ks[k * kWarp + col]) : 0.0;
        A = Qk;
        Bv = z0;
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
            const double Ad = __shfl_down_sync(0xffffffffu, A, d, 16), Bd = __shfl_down_sync(0xffffffffu, Bv, d, 16);
            if (k + d < 16) {
                Bv = fma(A, Bd, Bv);
                A *= Ad;
            }
        }
        const double G = __shfl_sync(0xffffffffu, Bv, 0, 16);    // x at the block's first row
        double x0 = __shfl_down_sync(0xffffffffu, Bv, 1, 16);
        if (k == 15) x0 = 0.0;
        sm.Y0[k * kWarp + col] = y0;
        sm.X0[k * kWarp + col] = x0;
        if (k == 0) {
            sm.pub[0 * kWarp + col] = F;
            sm.pub[1 * kWarp + col] = G;
        }
        // column boundary rows held by chunk k of this block: x with zero block carries
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const int row = (qq < 2) ? qq : n - 4 + qq;
            const int l = row - rb0 - k * L;
            if (row >= 0 && l >= 0 && l < Lk)
                sm.pub[(2 + qq) * kWarp + col] = sm.kb[qq * kWarp + col] + kap_s(qp, s2, l, Lk) * y0 + qp[Lk - l] * x0;
        }
    }
    __syncthreads();

    // ---- level 2 (warp 0): push this block's aggregates into every block of the cluster,
    //      receive everybody's, and resolve the block carries (Woodbury boundary terms and
    //      incoming-trace injections included).
    cluster_wait();  // (matches the arrive in the prologue: every xbar is initialised)
    if (warp == 0 && live) {
        const int nA = (rb0 <= 1 ? ((rb0 + Rb > 1) ? 1 : 0) : 0) + (inblk(n - 1) || inblk(n - 2) ? 1 : 0);
        (void)nA;
        if (lane == 0) mbar_expect_tx(&sm.xbar, static_cast<uint32_t>(nblk * kWarp * 16 + 2 * kWarp * 16));
        __syncwarp();
        const double F = sm.pub[lane], G = sm.pub[kWarp + lane];
        const bool has01 = inblk(0) || inblk(1), hasN = inblk(n - 2) || inblk(n - 1);
        // rows 0,1 (and n-2,n-1) always sit in the first (last) block: both values come from one block
        for (int c = 0; c < nblk; ++c) {
            st_async_v2(&sm.rFG[blk * kWarp + lane], c, F, G, &sm.xbar);
            if (has01) st_async_v2(&sm.rA[0 * kWarp + lane], c, sm.pub[2 * kWarp + lane], sm.pub[3 * kWarp + lane], &sm.xbar);
            if (hasN) st_async_v2(&sm.rA[1 * kWarp + lane], c, sm.pub[4 * kWarp + lane], sm.pub[5 * kWarp + lane], &sm.xbar);
        }
        mbar_wait(&sm.xbar, 0);
        const double *l2 = sm.l2c;
        double *Yb = sm.he, *Xb = sm.ks;  // [c][lane] scratch (he/ks are dead)
        const double Yt0 = S.injL * sm.gin[lane] / P.a, Xb0 = S.injR * sm.gin[kWarp + lane] / P.a;
        double Y = Yt0;
        for (int c = 0; c < nblk; ++c) {
            Yb[c * kWarp + lane] = Y;
            Y = fma(l2[L2_QR + c], Y, sm.rFG[c * kWarp + lane].x);
        }
        double X = Xb0;
        for (int c = nblk - 1; c >= 0; --c) {
            Xb[c * kWarp + lane] = X;
            X = fma(l2[L2_QR + c], X, fma(l2[L2_K0 + c], Yb[c * kWarp + lane], sm.rFG[c * kWarp + lane].y));
        }
        const double2 a01 = sm.rA[lane], aN = sm.rA[kWarp + lane];
        const int c0 = 0, cN = (n - 1) / R;
        const double xt0 = a01.x + l2[L2_KQ + 0] * Yb[c0 * kWarp + lane] + l2[L2_RQ + 0] * Xb[c0 * kWarp + lane];
        const double xt1 = a01.y + l2[L2_KQ + 1] * Yb[c0 * kWarp + lane] + l2[L2_RQ + 1] * Xb[c0 * kWarp + lane];
        const double xt2 = aN.x + l2[L2_KQ + 2] * Yb[cN * kWarp + lane] + l2[L2_RQ + 2] * Xb[cN * kWarp + lane];
        const double xt3 = aN.y + l2[L2_KQ + 3] * Yb[cN * kWarp + lane] + l2[L2_RQ + 3] * Xb[cN * kWarp + lane];
        const double s0 = S.wt0 * xt0 + S.wt1 * xt1;
        const double s1 = S.wb0 * xt2 + S.wb1 * xt3;
        const double dY = -(S.Mi00 * s0 + S.Mi01 * s1) / P.a;  // correction of the top carry
        const double dX = -(S.Mi10 * s0 + S.Mi11 * s1) / P.a;  // correction of the bottom carry
        sm.cb[lane] = fma(l2[L2_QB + blk], dY, Yb[blk * kWarp + lane]);
        sm.cb[kWarp + lane] = fma(l2[L2_QE + blk], dX, fma(l2[L2_KB + blk], dY, Xb[blk * kWarp + lane]));
        // Dirichlet ends: the end node value is the incoming trace
        if (blk == 0 && active && S.ltype == END_DIRI) {
            const double g = sm.gin[lane];
            if (S.iL_tr == -1) S.sendL[P.par_out][goff] = g;  // no overlap: the end node is the trace node
            if (S.ifL >= 0) eif = fmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + P.n) * P.nx + m]));
            if (P.last) {
                et = fmax(et, fabs(g - P.UT[static_cast<size_t>(S.lo) * P.nx + m]));
                unew_slab[m] = g;
            }
        } else if (blk == 0 && active && S.ltype == END_PHYS && P.last) {
            unew_slab[m] = 0.0;
        }
        if (blk == nblk - 1 && active && S.rtype == END_DIRI) {
            const double g = sm.gin[kWarp + lane];
            if (S.iR_tr == n) S.sendR[P.par_out][goff] = g;
            if (S.ifR >= 0) eif = fmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + P.n) * P.nx + m]));
            if (P.last) {
                et = fmax(et, fabs(g - P.UT[static_cast<size_t>(S.hi) * P.nx + m]));
                unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + m] = g;
            }
        } else if (blk == nblk - 1 && active && S.rtype == END_PHYS && P.last) {
            unew_slab[static_cast<size_t>(S.hi - S.lo) * P.nx + m] = 0.0;
        }
    }
    __syncthreads();

    // ---- pass C: x = k + kap Y + rho X with this chunk's carries; x -> dense slot -> TMA store of u^{n+1}
    double *xs = tile_w;  // [L][32] over the (consumed) u^n rows
    if (Lw > 0) {
        const double Yb = sm.cb[lane], Xb = sm.cb[kWarp + lane];
        const double Y = fma(qp[s_w], Yb, sm.Y0[warp * kWarp + lane]);
        const double X = fma(qp[Rb - e_w], Xb, fma(kap_s(qp, s2, e_w, Rb), Yb, sm.X0[warp * kWarp + lane]));
        __syncwarp();
        if (Lw == B && L == B) {
#pragma unroll
            for (int l = 0; l < B; ++l) {
                const double x = fma(kr[2 * l], Y, fma(kr[2 * l + 1], X, h[l]));
                h[l] = x;
                xs[l * kWarp + lane] = x;
            }
        } else {
#pragma unroll
            for (int l = 0; l < B; ++l) {
                if (l < Lw) {
                    const double x = fma(kap_s(qp, s2, l, Lw), Y, fma(qp[Lw - l], X, h[l]));
                    h[l] = x;
                    xs[l * kWarp + lane] = x;
                }
            }
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the TMA store
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(FP.smaps + 2 * sub + ((P.n + 1) & 1), m0, cr0, xs);
            bulk_commit();
        }
        if (P.last && active) {  // error at T on every unknown row (a 1/N_t fraction of the steps)
            const double *ut = P.UT + static_cast<size_t>(S.first + cr0) * P.nx + m;
            const size_t pitch = P.nx;
#pragma unroll
            for (int l = 0; l < B; ++l)
                if (l < Lw) et = fmax(et, fabs(h[l] - ut[l * pitch]));
        }
    }
    grid_dep_launch();  // the next step may start its prologue

    // ---- special rows of this block, read back from the tile
    if (special) {
        __syncthreads();
        if (warp == 0) {
            auto xrow = [&](int i) {
                const int li = i - rb0;
                return sm.tile[(li / L) * Sm::kSlot + (li % L) * kWarp + lane];
            };
            const double inv_h = 1.0 / P.hv, half_h_dt = 0.5 * P.hv / P.dt;
            if (active && S.iL_tr >= 0 && inblk(S.iL_tr)) {  // (p + d_v) u at hi_{s-1}, half-cell flux on [c, c+h/2]
                const double uc = xrow(S.iL_tr);
                double g = uc;
                if (P.send_robin) g = P.p * uc - ((uc - xrow(S.iL_tr + 1)) * inv_h + half_h_dt * (uc - sm.rtr[lane]));
                S.sendL[P.par_out][goff] = g;
            }
            if (active && S.iR_tr >= 0 && S.iR_tr < n && inblk(S.iR_tr)) {  // (p - d_v) u at lo_{s+1}, flux on [c-h/2, c]
                const double uc = xrow(S.iR_tr);
                double g = uc;
                if (P.send_robin) g = P.p * uc - ((uc - xrow(S.iR_tr - 1)) * inv_h + half_h_dt * (uc - sm.rtr[kWarp + lane]));
                S.sendR[P.par_out][goff] = g;
            }
            if (active && S.ltype == END_ROBIN && S.ifL >= 0 && inblk(0))
                eif = fmax(eif, fabs(xrow(0) - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + P.n) * P.nx + m]));
            if (active && S.rtype == END_ROBIN && S.ifR >= 0 && inblk(n - 1))
                eif = fmax(eif, fabs(xrow(n - 1) - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + P.n) * P.nx + m]));
            if (P.record && active)
                for (int i = 0; i < FP.nrec; ++i) {
                    const int row = FP.rec_rows[i];
                    if (inblk(row)) P.rec[(static_cast<size_t>(i) * P.nt + P.n) * P.nx + m] = xrow(row);
                }
        }
    }
    // ---- errors: block max, one atomic per CTA (only where errors can be non-zero)
    if (errs) {
        eif = warp_max(eif);
        et = warp_max(et);
        if (lane == 0) {
            sm.red[warp] = eif;
            sm.red[kFusedWarps + warp] = et;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int c = 0; c < kFusedWarps; ++c) {
                a = fmax(a, sm.red[c]);
                b = fmax(b, sm.red[kFusedWarps + c]);
            }
            if (a > 0.0) atomic_max_pos(P.errIF, a);
            if (b > 0.0 && P.errT) atomic_max_pos(P.errT, b);
        }
    }
    if (lane == 0 && Lw > 0) bulk_wait_read0();  // the slot must outlive the TMA store's read
}

}  // namespace kfp

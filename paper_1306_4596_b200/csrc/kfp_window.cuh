// kfp_window.cuh -- the hot kernel of the SWR iterations: ONE persistent launch per
// Schwarz iteration (the whole window t_0 -> t_{N_t}, every local subdomain), with
// the per-tile work of kfp_fused.cuh (transport + forcing + v-tridiagonal solve +
// transmission traces + errors) software-pipelined across tiles and steps.
//
// Why (profiles/r1_v8_*): the per-step kernel spends most of each
// tile waiting -- on its cluster partners (the row blocks of one column live on
// C SMs and must exchange carries before anybody can finish the tile), on the
// tile's TMA load, and on the launch/ramp of every one of the N_t steps.  Here
//   * tile j's "start" (wait data, passes A/B, level 1, push aggregates) runs
//     BEFORE tile j-1's "finish" (wait exchange, level 2, pass C, traces), so the
//     exchange latency of j-1 is hidden behind the work of j;
//   * u^n tiles are double-buffered per warp and loaded two tiles ahead;
//   * steps follow each other inside the launch: the cluster walks its x-tiles
//     of step n, then of step n+1, ...  Step n+1 of tile t needs step n of tiles
//     t-1, t, t+1 (the x-halo is one column, first-order upwind) -- and nothing
//     else, since every column's v-solve is local to its tile.  That dependency
//     (and the write-after-read hazard on the ping-pong slabs, which it implies)
//     is carried by per-(subdomain, tile, row block) step flags in global memory:
//     release after the block's stores, acquire before the block's next load.
//
// Geometry as kfp_fused.cuh: a cluster of C CTAs owns a 32-column x-tile at a
// time, CTA `blk` the rows [blk R, blk R + R), warp w the chunk of L rows at
// blk R + w L, lane = column.  The G clusters of the grid walk the global tile
// list g = sub * ntiles + t in rounds: cluster y takes g = y, y + G, ... at every
// step.  All clusters must be co-resident (grid <= cudaOccupancyMaxActiveClusters,
// checked on the host); a flag wait that exceeds a few seconds traps instead of
// hanging the device.
//
// Deadlock freedom: a CTA that cannot issue the load of its next tile first
// finishes and publishes every tile it holds ("drain"), so a blocked CTA never
// holds an unpublished tile; flag waits point strictly backwards in steps.
#pragma once
#include "kfp_fused.cuh"

namespace kfp {

struct WinParams {
    StepParams S;              // common parameters; n / last / from_u0 / cf are derived per tile here
    const CUtensorMap *tmaps;  // [nsub][2] load maps (box 36 x L) of the slabs' unknown rows, by step parity
    const double *l2m;         // [nsub][C][kL2M] level-2 linear maps (host-computed)
    const double *coefT;       // [nv+1][2+NR] per-node (q/a)(1-|nu|), (q/a)|nu|, (q/a) fv_r(j)
    const double *tabs;        // qp[kQ] | s2[kQ] | kr[2B]
    const double *cfn;         // [nt][kMaxRank]: dt ft_r(t_{n+1})
    unsigned int *flags;       // [nsub][ntiles][C]: epoch + n + 1 once step n of (sub, tile, blk) is stored
    unsigned int *fault;       // watchdog word (set before a trap)
    int L, G, ntiles, nsub, n0, n1;
    unsigned int epoch;
    int dbg;  // experiments only (KFP_WIN_DBG, results invalid when set): 1 no fences, 2 no u stores
};

template <int B, int NR, int P>
struct WinSmem {
    static constexpr int kSlot = slot_doubles<B>();
    static constexpr int kQ = fused_kq<B, P>();
    static constexpr int kTab = 2 * kQ + 2 * B;
    alignas(128) double tile[2][P * kSlot];  // per warp: u^n rows [L][36], double-buffered by tile parity
    alignas(16) double coef[2][P * B * (2 + NR)];  // per slot and warp: its chunk's rows of coefT (with the tile)
    alignas(16) double tab[kTab];            // qp | s2 | kr
    double he[3][P * kCS];                   // per tile (j % 3): y at chunk ends -> y0 -> final Y carries
    double ks[3][P * kCS];                   // per tile (j % 3): k at chunk starts -> x0 -> final X carries
    double kb[4 * kCS];                      // k at the column's rows 0, 1, n-2, n-1 (chunk-local zero carries)
    double2 rFG[4][kMaxFusedCluster * kCS];  // received (F, G) per block, by tile (j & 3)
    double rA[4][4 * kCS];                   // received x~ at rows 0, 1, n-2, n-1, by tile (j & 3)
    double gin[2][2 * kWarp];                // incoming traces at t_{n+1} (lo end, hi end), by tile parity
    double rtr[2][2 * kWarp];                // raw r at the outgoing-trace rows, by tile parity
    double xsp[6 * kWarp];                   // x at the special rows of the tile being finished
    SubDev sd[4];                            // subdomain descriptor of tile j (j & 3), loaded two tiles ahead
    alignas(16) double l2m[4][kL2M];         // level-2 map of tile j's (subdomain, block), same ring
    int4 tinfo[4];                           // (n, sub, t, -) of tile j, same ring
    double red[2 * P];
    uint64_t bar[2][P];                      // per slot and warp: its coefficient rows (+ u^n chunk) landed
    uint64_t tbar;                           // tables
    uint64_t xbar[4];                        // cluster exchange, by tile (j & 3)
    int ready_upto;                          // tiles <= ready_upto may be loaded (their flags were seen)
};

template <int B, int NR, int P>
__host__ __device__ constexpr size_t window_smem_bytes() {
    return sizeof(WinSmem<B, NR, P>);
}

// --------------------------------------------------------------------------- PTX
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}


// --------------------------------------------------------------------------- pass A (coefficients from global/L1)
// DIR = -1: every row of the chunk has v >= 0 (upwind neighbour m-1); +1: v < 0; 0: generic / ragged.
template <int B, int NR, int DIR>
__device__ __forceinline__ void win_pass_a(const double *tile_w, const double *coef_g, int lane, double q,
                                           const double (&fx)[NR], double (&h)[B], int Lw, int jv2_0, double &hend) {
    constexpr int kC = 2 + NR;
    double hp = 0.0;
#pragma unroll
    for (int l = 0; l < B; ++l) {
        const double *row = tile_w + l * kTW + kHalo + lane;
        const double2 c01 = __ldg(reinterpret_cast<const double2 *>(coef_g + l * kC));
        double f = 0.0;
#pragma unroll
        for (int r = 0; r < NR; r += 2) {
            const double2 g = __ldg(reinterpret_cast<const double2 *>(coef_g + l * kC + 2 + r));
            f = fma(g.x, fx[r], f);
            f = fma(g.y, fx[r + 1], f);
        }
        const double u = row[0];
        double nb;
        if (DIR == 0) {
            const int off = (jv2_0 + 2 * l >= 0) ? -1 : 1;  // 2j - nv >= 0: v >= 0 -> left neighbour
            nb = row[off];
        } else {
            nb = row[DIR];
        }
        const double rp = fma(c01.y, nb, fma(c01.x, u, f));
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

// --------------------------------------------------------------------------- the kernel
template <int B, int NR, int P_>
__global__ void __launch_bounds__(P_ * kWarp, 1) step_window(const WinParams W) {
    static_assert(NR % 2 == 0, "forcing ranks are read in pairs");
    constexpr int NW = P_;            // warps (= chunks) per CTA
    constexpr int kCPW = kWarp / NW;  // columns per warp in the transposed phases
    constexpr int kC = 2 + NR;
    using Sm = WinSmem<B, NR, NW>;
    extern __shared__ __align__(128) char smraw[];
    Sm &sm = *reinterpret_cast<Sm *>(smraw);
    const StepParams &P = W.S;
    const int blk = static_cast<int>(cg::this_cluster().block_rank());
    const int C = P.C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int y = blockIdx.y;
    const int L = W.L, R = NW * L;
    const int rb0 = blk * R, s_w = warp * L, cr0 = rb0 + s_w;
    const int total = W.nsub * W.ntiles;
    const int per_step = (total - y + W.G - 1) / W.G;  // tiles of this cluster per step (G <= total)
    const int J = per_step * (W.n1 - W.n0);             // tiles of this cluster in the launch
    const double q = P.q;
    const double *qp = sm.tab, *s2 = sm.tab + Sm::kQ, *kr = sm.tab + 2 * Sm::kQ;
    const uint32_t tile_bytes = static_cast<uint32_t>(kTW * L * sizeof(double));

    auto decode = [&](int j, int &n, int &sub, int &t) {
        n = W.n0 + j / per_step;
        const int g = y + (j - (j / per_step) * per_step) * W.G;
        sub = g / W.ntiles;
        t = g - sub * W.ntiles;
    };
    // May step n of (sub, t) be loaded by this CTA: step n-1 of tiles t-1, t, t+1 stored?  The poller
    // warp (the last one) reads the flags of tiles r+1 and r+2 (r = ready_upto) with acquire loads on
    // lanes 0-5 just before it waits for a cluster exchange (finish), where it would idle anyway; the
    // other warps issue the loads after the next barrier.  (Relaxed loads + barrier are NOT enough: with
    // them the TMA reads occasionally saw stale rows -- measured, tools/win_diff.py.)
    constexpr int kPollWarp = NW - 1;
    auto flag_need = [&](int j, unsigned int *&addr, int d) -> unsigned int {  // 0 = no flag needed
        int n, sub, t;
        decode(j, n, sub, t);
        if (n == W.n0 || n == 0) return 0u;
        const int tt = (t + d + W.ntiles) % W.ntiles;
        addr = W.flags + (static_cast<size_t>(sub) * W.ntiles + tt) * C + blk;
        return W.epoch + static_cast<unsigned int>(n);
    };
    unsigned int poll_v = 0, poll_need = 0;
    int poll_r = -1;
    auto poll_issue = [&]() {  // poller warp: relaxed loads of the flags of tiles r+1, r+2
        poll_r = sm.ready_upto;
        poll_need = 0;
        const int jj = poll_r + 1 + lane / 3;
        if (lane < 6 && jj < J) {
            unsigned int *a = nullptr;
            poll_need = flag_need(jj, a, lane % 3 - 1);
            if (poll_need) poll_v = ld_acquire_u32(a);
        }
    };
    auto poll_eval = [&]() {  // poller warp, after a barrier: advance ready_upto
        const bool ok = (poll_need == 0) || static_cast<int>(poll_v - poll_need) >= 0;
        const unsigned int bad = __ballot_sync(0xffffffffu, !ok && lane < 6);
        int r = poll_r;
        if (r + 1 < J && (bad & 0x7u) == 0) {
            ++r;
            if (r + 1 < J && (bad & 0x38u) == 0) ++r;
        }
        if (lane == 0 && r > sm.ready_upto) sm.ready_upto = r;
    };
    auto tile_ready_blocking = [&](int j) -> bool {  // one thread: all three flags of tile j (relaxed)
        for (int d = -1; d <= 1; ++d) {
            unsigned int *a = nullptr;
            const unsigned int need = flag_need(j, a, d);
            if (need && static_cast<int>(ld_acquire_u32(a) - need) < 0) return false;
        }
        return true;
    };
    auto load_sd = [&](int j) {  // warp 0: descriptor, level-2 map and (n, sub, t) of tile j -> ring slot j & 3
        if (j >= J) return;
        int n, sub, t;
        decode(j, n, sub, t);
        constexpr int kWords = sizeof(SubDev) / sizeof(uint64_t);
        static_assert(sizeof(SubDev) % sizeof(uint64_t) == 0, "SubDev size");
        for (int i = lane; i < kWords; i += kWarp)
            reinterpret_cast<uint64_t *>(&sm.sd[j & 3])[i] = reinterpret_cast<const uint64_t *>(P.subs + sub)[i];
        const double *l2 = W.l2m + (static_cast<size_t>(sub) * C + blk) * kL2M;
        for (int i = lane; i < kL2M; i += kWarp) sm.l2m[j & 3][i] = __ldg(l2 + i);
        if (lane == 0) sm.tinfo[j & 3] = make_int4(n, sub, t, 0);
    };
    auto info = [&](int j, int &n, int &sub, int &t) {  // (n, sub, t) of a tile in the ring
        const int4 v = sm.tinfo[j & 3];
        n = v.x;
        sub = v.y;
        t = v.z;
    };
    // this warp's TMA loads of every ready tile in (issued, limit]; slot jj & 1 must be consumed by A(jj - 2)
    int issued = -1;
    uint32_t tph = 0;  // expected phase of bar[s][warp] (bit s)
    auto issue_loads = [&](int limit) {
        const int lim = min(limit, sm.ready_upto);
        for (int jj = issued + 1; jj <= lim; ++jj) {
            int n, sub, t;
            info(jj, n, sub, t);
            const SubDev &S = sm.sd[jj & 3];
            const int Rb = max(0, min(R, S.n - rb0)), Lw = max(0, min(L, Rb - s_w));
            if (Lw > 0 && lane == 0) {
                const int slot = jj & 1;
                const uint32_t coef_bytes = static_cast<uint32_t>(Lw * kC * sizeof(double));
                fence_proxy_async_global();  // the flags were observed (poller + barrier): order the async-proxy reads
                fence_proxy_async_smem();    // the slot was read through the generic proxy
                mbar_expect_tx(&sm.bar[slot][warp], coef_bytes + (n != 0 ? tile_bytes : 0u));
                bulk_g2s(sm.coef[slot] + warp * B * kC, W.coefT + static_cast<size_t>(S.first + cr0) * kC, coef_bytes,
                         &sm.bar[slot][warp]);
                if (n != 0)
                    tma_load_2d(sm.tile[slot] + warp * Sm::kSlot, W.tmaps + 2 * sub + (n & 1), t * kWarp - kHalo, cr0,
                                &sm.bar[slot][warp]);
            }
            issued = jj;
        }
    };

    // Step flags.  A barrier plus one thread's fence before the release is NOT enough to make the other
    // warps' stores visible to a TMA reader on another SM (measured: stale rows, tools/win_diff.py), so
    // every thread fences its own stores -- one iteration later, when they have long completed and the
    // fence is cheap -- and the flags of finished tiles are released after the following barrier.
    int fin_upto = -1, pub_upto = -1;  // last finished / last published tile (uniform)
    auto fence_all = [&]() {
        if (W.dbg & 1) return;
        __threadfence();
        fence_proxy_async_global();
    };
    auto publish = [&]() {  // after fence_all + a barrier
        if (threadIdx.x == 0)
            for (int x = pub_upto + 1; x <= fin_upto; ++x) {
                int n, sub, t;
                decode(x, n, sub, t);
                st_release_u32(W.flags + (static_cast<size_t>(sub) * W.ntiles + t) * C + blk,
                               W.epoch + static_cast<unsigned int>(n) + 1u);
            }
        pub_upto = fin_upto;
    };

    // ---- prologue
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&sm.xbar[i], 1);
        mbar_init(&sm.tbar, 1);
        sm.ready_upto = -1;
    }
    if (lane == 0) {
        mbar_init(&sm.bar[0][warp], 1);
        mbar_init(&sm.bar[1][warp], 1);
    }
    fence_mbar_init();
    cluster_arrive_relaxed();  // every CTA's barriers are initialised before anybody pushes (wait below)
    if (warp == 0) {
        load_sd(0);
        load_sd(1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&sm.tbar, static_cast<uint32_t>(Sm::kTab * sizeof(double)));
        bulk_g2s(sm.tab, W.tabs, Sm::kTab * sizeof(double), &sm.tbar);
    }
    if (warp == kPollWarp) {
        poll_issue();
        poll_eval();
    }
    __syncthreads();
    issue_loads(1);
    cluster_wait();
    mbar_wait(&sm.tbar, 0);

    double eif = 0.0, et = 0.0;
    KFP_WT_DECL
    double cur[B], prev[B];
#pragma unroll
    for (int l = 0; l < B; ++l) cur[l] = prev[l] = 0.0;

    // ================================================================ finish(x): level 2, pass C, traces
    auto finish = [&](int x, int limit) {
        int n, sub, t;
        info(x, n, sub, t);
        const SubDev &S = sm.sd[x & 3];
        const int sn = S.n;
        const int Rb = max(0, min(R, sn - rb0)), Lw = max(0, min(L, Rb - s_w));
        const int m0 = t * kWarp, w = min(kWarp, P.nx - m0);
        const int m = m0 + min(lane, w - 1);
        const bool active = lane < w;
        const size_t goff = static_cast<size_t>(n) * P.nx + m;
        const bool last = (n + 1 == P.nt);
        const int hb = x % 3;
        double *he = sm.he[hb], *ks = sm.ks[hb];
        auto inblk = [&](int i) { return i >= rb0 && i < rb0 + Rb; };
        const bool tr_L = S.iL_tr >= 0 && (inblk(S.iL_tr) || inblk(S.iL_tr + 1));
        const bool tr_R = S.iR_tr >= 0 && S.iR_tr < sn && (inblk(S.iR_tr) || inblk(S.iR_tr - 1));
        const int sp_row[6] = {tr_L ? S.iL_tr : -1, tr_L ? S.iL_tr + 1 : -1, tr_R ? S.iR_tr : -1, tr_R ? S.iR_tr - 1 : -1,
                               (S.ltype == END_ROBIN && S.ifL >= 0) ? 0 : -1, (S.rtype == END_ROBIN && S.ifR >= 0) ? sn - 1 : -1};

        KFP_WT(-1)
        if (warp == kPollWarp) {  // acquire-poll the flags of the next tiles while the exchange completes
            poll_issue();
            poll_eval();
        }
        mbar_wait(&sm.xbar[x & 3], (x >> 2) & 1);
        KFP_WT(0)  // 0: exchange wait
        // level 2: block carries = the precomputed linear map of (F_c, G_c, x~_q, g_lo, g_hi)
        {
            const int col = kCPW * warp + lane / NW, k = lane % NW;
            const int sk = k * L, Lk = max(0, min(L, Rb - sk)), ek = sk + Lk;
            const double *l2m = sm.l2m[x & 3];
            const double2 *rFG = sm.rFG[x & 3];
            const double *rA = sm.rA[x & 3], *gin = sm.gin[x & 1];
            double yv = 0.0, xv = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < kL2N; j0 += NW) {
                const int jj = j0 + k;
                if (jj < kL2N) {
                    double v;
                    if (jj < 16) {
                        const int c = jj & 7;
                        v = (c < C) ? ((jj < 8) ? rFG[c * kCS + col].x : rFG[c * kCS + col].y) : 0.0;
                    } else if (jj < 20) {
                        v = rA[(jj - 16) * kCS + col];
                    } else {
                        v = gin[(jj - 20) * kWarp + col];
                    }
                    yv = fma(l2m[jj], v, yv);
                    xv = fma(l2m[24 + jj], v, xv);
                }
            }
#pragma unroll
            for (int o = NW / 2; o > 0; o >>= 1) {
                yv += __shfl_xor_sync(0xffffffffu, yv, o, NW);
                xv += __shfl_xor_sync(0xffffffffu, xv, o, NW);
            }
            const double y0 = he[k * kCS + col], x0 = ks[k * kCS + col];
            he[k * kCS + col] = fma(qp[sk], yv, y0);
            ks[k * kCS + col] = fma(qp[Rb - ek], xv, fma(kap_s(qp, s2, ek, Rb), yv, x0));
        }
        __syncthreads();  // S2: final carries visible; every warp has consumed its slot of the tile started last
        KFP_WT(1)  // 1: level 2 + S2
        issue_loads(limit);

        // pass C: x = k + kap Y + rho X; coalesced stores of u^{n+1}
        if (Lw > 0) {
            double *unew = S.slab[(n + 1) & 1] + static_cast<size_t>(S.first - S.lo + cr0) * P.nx + m;
            const size_t pitch = P.nx;
            const double Y = he[warp * kCS + lane], X = ks[warp * kCS + lane];
            if (Lw == B && L == B) {
#pragma unroll
                for (int l = 0; l < B; ++l) prev[l] = fma(kr[2 * l], Y, fma(kr[2 * l + 1], X, prev[l]));
            } else {
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) prev[l] = fma(kap_s(qp, s2, l, Lw), Y, fma(qp[Lw - l], X, prev[l]));
            }
            if (active && !(W.dbg & 2)) {
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) unew[l * pitch] = prev[l];
            }
            if (last && active) {  // error at T on every unknown row
                const double *ut = P.UT + static_cast<size_t>(S.first + cr0) * P.nx + m;
#pragma unroll
                for (int l = 0; l < B; ++l)
                    if (l < Lw) et = fmax(et, fabs(prev[l] - ut[l * pitch]));
            }
            bool chunk_special = false;
#pragma unroll
            for (int qq = 0; qq < 6; ++qq) chunk_special |= sp_row[qq] >= cr0 && sp_row[qq] < cr0 + Lw;
            if (chunk_special) {
#pragma unroll
                for (int l = 0; l < B; ++l)
#pragma unroll
                    for (int qq = 0; qq < 6; ++qq)
                        if (l < Lw && cr0 + l == sp_row[qq]) sm.xsp[qq * kWarp + lane] = prev[l];
            }
        }
        // Dirichlet ends: the end node value is the incoming trace
        if (warp == 0 && active) {
            const double *gin = sm.gin[x & 1];
            const int nblk = S.nblk;
            if (blk == 0 && S.ltype == END_DIRI) {
                const double g = gin[lane];
                if (S.iL_tr == -1) S.sendL[P.par_out][goff] = g;  // no overlap: the end node is the trace node
                if (S.ifL >= 0) eif = fmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + n) * P.nx + m]));
                if (last) {
                    et = fmax(et, fabs(g - P.UT[static_cast<size_t>(S.lo) * P.nx + m]));
                    S.slab[(n + 1) & 1][m] = g;
                }
            } else if (blk == 0 && S.ltype == END_PHYS && last) {
                S.slab[(n + 1) & 1][m] = 0.0;
            }
            if (blk == nblk - 1 && S.rtype == END_DIRI) {
                const double g = gin[kWarp + lane];
                if (S.iR_tr == sn) S.sendR[P.par_out][goff] = g;
                if (S.ifR >= 0) eif = fmax(eif, fabs(g - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + n) * P.nx + m]));
                if (last) {
                    et = fmax(et, fabs(g - P.UT[static_cast<size_t>(S.hi) * P.nx + m]));
                    S.slab[(n + 1) & 1][static_cast<size_t>(S.hi - S.lo) * P.nx + m] = g;
                }
            } else if (blk == nblk - 1 && S.rtype == END_PHYS && last) {
                S.slab[(n + 1) & 1][static_cast<size_t>(S.hi - S.lo) * P.nx + m] = 0.0;
            }
        }
        KFP_WT(2)  // 2: pass C + ends
        __syncthreads();  // S3: x at the special rows visible
        KFP_WT(3)  // 3: S3
        fin_upto = x;  // published after the next fence_all + barrier (publish)
        // outgoing traces at t_{n+1} (R11), Robin-end interface errors
        if (warp == 0 && active) {
            const double inv_h = 1.0 / P.hv, half_h_dt = 0.5 * P.hv / P.dt;
            const double *rtr = sm.rtr[x & 1];
            if (tr_L && inblk(S.iL_tr)) {  // (p + d_v) u at hi_{s-1}, half-cell flux on [c, c+h/2]
                const double uc = sm.xsp[lane];
                double g = uc;
                if (P.send_robin) g = S.tpL * uc - ((uc - sm.xsp[kWarp + lane]) * inv_h + half_h_dt * (uc - rtr[lane]));
                S.sendL[P.par_out][goff] = g;
            }
            if (tr_R && inblk(S.iR_tr)) {  // (q - d_v) u at lo_{s+1}, flux on [c-h/2, c]
                const double uc = sm.xsp[2 * kWarp + lane];
                double g = uc;
                if (P.send_robin)
                    g = S.tpR * uc - ((uc - sm.xsp[3 * kWarp + lane]) * inv_h + half_h_dt * (uc - rtr[kWarp + lane]));
                S.sendR[P.par_out][goff] = g;
            }
            if (inblk(sp_row[4]))
                eif = fmax(eif, fabs(sm.xsp[4 * kWarp + lane] - P.Ulines[(static_cast<size_t>(S.ifL) * P.nt + n) * P.nx + m]));
            if (inblk(sp_row[5]))
                eif = fmax(eif, fabs(sm.xsp[5 * kWarp + lane] - P.Ulines[(static_cast<size_t>(S.ifR) * P.nt + n) * P.nx + m]));
        }
    };

    // ================================================================ start(j): passes A/B, level 1, push
    auto start = [&](int j) {
        int n, sub, t;
        info(j, n, sub, t);
        const SubDev &S = sm.sd[j & 3];
        const int sn = S.n;
        const int Rb = max(0, min(R, sn - rb0)), Lw = max(0, min(L, Rb - s_w));
        const int m0 = t * kWarp, w = min(kWarp, P.nx - m0);
        const int m = m0 + min(lane, w - 1);
        const bool from_u0 = (n == 0);
        const size_t goff = static_cast<size_t>(n) * P.nx + m;
        const int hb = j % 3;
        double *he = sm.he[hb], *ks = sm.ks[hb];
        auto inblk = [&](int i) { return i >= rb0 && i < rb0 + Rb; };
        double fx[NR];  // this lane's forcing profile times dt ft_r(t_{n+1})
#pragma unroll
        for (int r = 0; r < NR; ++r)
            fx[r] = (r < P.f_rank) ? __ldg(W.cfn + static_cast<size_t>(n) * kMaxRank + r) * __ldg(P.fx + r * P.nx + m) : 0.0;
        if (warp == 0) {  // incoming traces of this step (written by the previous iteration)
            sm.gin[j & 1][lane] = (S.ltype != END_PHYS) ? __ldg(S.gL[P.par_in_lo] + goff) : 0.0;
            sm.gin[j & 1][kWarp + lane] = (S.rtype != END_PHYS) ? __ldg(S.gR[P.par_in] + goff) : 0.0;
        }
        double hend = 0.0, kst = 0.0;
        KFP_WT(-1)
        if (Lw > 0) {
            const int slot = j & 1;
            double *tile_w = sm.tile[slot] + warp * Sm::kSlot;
            mbar_wait(&sm.bar[slot][warp], (tph >> slot) & 1u);
            tph ^= 1u << slot;
            if (!from_u0) {
                KFP_WT(4)  // 4: data wait
                if (m0 == 0 || m0 + w == P.nx) {
                    // periodic wrap of the halo at the ends of the x range (TMA zero-fills out-of-range columns);
                    // L2 loads (.cg): this SM may hold a stale L1 line of the ping-pong slab
                    const double *src = S.slab[n & 1] + static_cast<size_t>(S.first - S.lo + cr0) * P.nx;
                    for (int l = lane; l < Lw; l += kWarp) {  // strided: a chunk may hold 33 rows
                        if (m0 == 0) tile_w[l * kTW + kHalo - 1] = __ldcg(src + static_cast<size_t>(l) * P.nx + P.nx - 1);
                        if (m0 + w == P.nx) tile_w[l * kTW + kHalo + w] = __ldcg(src + static_cast<size_t>(l) * P.nx);
                    }
                    __syncwarp();
                }
            } else {  // u^0 from the separable u0 tables (0 B of HBM), incl. the halo columns
                for (int l = 0; l < Lw; ++l) {
                    const int jn = S.first + cr0 + l;
                    for (int c = lane; c < kTW; c += kWarp) {
                        const int mm = ((m0 - kHalo + c) % P.nx + P.nx) % P.nx;
                        double s = 0.0;
                        for (int r = 0; r < P.u0_rank; ++r)
                            s = fma(__ldg(P.u0v + r * (P.nv + 1) + jn), __ldg(P.u0x + r * P.nx + mm), s);
                        tile_w[l * kTW + c] = s;
                    }
                }
                __syncwarp();
            }
            const double *coef_w = sm.coef[slot] + warp * B * kC;
            const int jv2_0 = 2 * (S.first + cr0) - P.nv;  // 2 j - nv of the chunk's first row
            const int jv2_1 = jv2_0 + 2 * (Lw - 1);
            const bool full = (Lw == B) && (cr0 + Lw <= sn - 2);
            if (full && jv2_0 >= 0) pass_a_reg<B, NR, -1>(tile_w, coef_w, lane, q, fx, cur, Lw, jv2_0, hend);
            else if (full && jv2_1 < 0) pass_a_reg<B, NR, 1>(tile_w, coef_w, lane, q, fx, cur, Lw, jv2_0, hend);
            else pass_a_reg<B, NR, 0>(tile_w, coef_w, lane, q, fx, cur, Lw, jv2_0, hend);
            // raw r (no incoming-trace term) at the outgoing-trace rows, for the Robin trace (R11)
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const int itr = side ? S.iR_tr : S.iL_tr;
                const bool on = side ? (itr >= 0 && itr < sn) : (itr >= 0);
                if (on && itr >= cr0 && itr < cr0 + Lw) {
                    const int l = itr - cr0, jn = S.first + itr;
                    const double2 rc = __ldg(P.rowc + jn);
                    const double u = tile_w[l * kTW + kHalo + lane];
                    const double nb = tile_w[l * kTW + kHalo + lane + ((2 * jn - P.nv >= 0) ? -1 : 1)];
                    double f = 0.0;
                    for (int r = 0; r < P.f_rank; ++r) f = fma(__ldg(P.fv + r * (P.nv + 1) + jn), fx[r], f);
                    sm.rtr[j & 1][side * kWarp + lane] = fma(rc.x, u, fma(rc.y, nb, f));
                }
            }
            if (full) {
                kst = pass_b_full<B>(cur, q);
            } else {
                double kl = 0.0, kl2 = 0.0;
                kst = pass_b_ragged<B>(cur, q, Lw, kl, kl2);
                if (cr0 + Lw == sn) {
                    sm.kb[3 * kCS + lane] = kl;
                    if (Lw >= 2) sm.kb[2 * kCS + lane] = kl2;
                } else if (cr0 + Lw == sn - 1) {
                    sm.kb[2 * kCS + lane] = kl;
                }
            }
            if (cr0 == 0) {
                sm.kb[0 * kCS + lane] = cur[0];
                if (Lw >= 2) sm.kb[1 * kCS + lane] = cur[1];
            } else if (cr0 == 1) {
                sm.kb[1 * kCS + lane] = cur[0];
            }
        }
        he[warp * kCS + lane] = hend;
        ks[warp * kCS + lane] = kst;
        KFP_WT(5)  // 5: passes A/B
        fence_all();      // the stores of the tile finished in the previous iteration (long completed)
        __syncthreads();  // S1
        publish();
        KFP_WT(6)  // 6: S1
        if (warp == 0) load_sd(j + 2);

        // level 1 in the transposed layout: warp w owns the kCPW columns col = kCPW w + lane / NW;
        // lane k = lane % NW stands for chunk k of the block
        {
            const int col = kCPW * warp + lane / NW, k = lane % NW;
            const int sk = k * L, Lk = max(0, min(L, Rb - sk));
            const double Qk = qp[Lk];
            double A = Qk, Bv = he[k * kCS + col];
            const double ksk = ks[k * kCS + col];
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
            const double G = __shfl_sync(0xffffffffu, Bv, 0, NW);  // x at the block's first row
            double x0 = __shfl_down_sync(0xffffffffu, Bv, 1, NW);
            if (k == NW - 1) x0 = 0.0;
            // lane k < C pushes this block's aggregates of column col into CTA k of the cluster
            if (k < C) st_async_v2(&sm.rFG[j & 3][blk * kCS + col], k, F, G, &sm.xbar[j & 3]);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {  // column boundary rows: x~ with zero block carries, to every CTA
                const int row = (qq < 2) ? qq : sn - 4 + qq;
                if (row >= 0 && inblk(row)) {
                    const int kq = (row - rb0) / L, l = row - rb0 - kq * L;
                    const int Lq = max(0, min(L, Rb - kq * L));
                    const double a = sm.kb[qq * kCS + col] + kap_s(qp, s2, l, Lq) * y0 + qp[Lq - l] * x0;
                    const double av = __shfl_sync(0xffffffffu, a, kq, NW);
                    if (k < C) st_async_f64(&sm.rA[j & 3][qq * kCS + col], k, av, &sm.xbar[j & 3]);
                }
            }
            he[k * kCS + col] = y0;  // chunk carries with zero block carries, completed by level 2
            ks[k * kCS + col] = x0;
        }
        if (threadIdx.x == 0)
            mbar_expect_tx(&sm.xbar[j & 3], static_cast<uint32_t>(C * kWarp * sizeof(double2) + 4 * kWarp * sizeof(double)));
        KFP_WT(7)  // 7: poll + level 1 + push
    };

    // ================================================================ the pipelined walk
    for (int j = 0; j <= J; ++j) {
        bool prev_done = (j == 0);
        if (j < J && issued < j) {
            // drain: the next load is not ready -- finish and publish everything held, then wait for it
            fence_all();
            __syncthreads();
            publish();
            if (!prev_done) {
                finish(j - 1, j + 1);
                prev_done = true;
                fence_all();
                __syncthreads();
                publish();
            }
            KFP_WT(-1)
            if (warp == kPollWarp && lane == 0) {
                const unsigned long long t0 = global_ns();
                while (!tile_ready_blocking(j)) {
                    if (global_ns() - t0 > 4000000000ull) {  // 4 s: a non-resident cluster -- trap, never hang
                        atomicExch(W.fault, 1u);
                        __trap();
                    }
                    __nanosleep(64);
                }
                sm.ready_upto = max(sm.ready_upto, j);
            }
            __syncthreads();
            issue_loads(j + 1);
            KFP_WT(8)  // 8: drain waits
#ifdef KFP_TRACE
            if (threadIdx.x == 0) wt_acc[9] += 1;  // 9: drain count
#endif
        }
        if (j < J) start(j);
        if (!prev_done) finish(j - 1, j + 2);
        else __syncthreads();  // every iteration ends with a barrier (single-buffered kb / xsp, rings)
#pragma unroll
        for (int l = 0; l < B; ++l) prev[l] = cur[l];
    }

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
                a = fmax(a, sm.red[c]);
                b = fmax(b, sm.red[NW + c]);
            }
            if (a > 0.0) atomic_max_pos(P.errIF, a);
            if (b > 0.0 && P.errT) atomic_max_pos(P.errT, b);
        }
    }
    KFP_WT_FLUSH
    // no CTA leaves while a partner may still push into its shared memory
    cluster_arrive();
    cluster_wait();
}

}  // namespace kfp

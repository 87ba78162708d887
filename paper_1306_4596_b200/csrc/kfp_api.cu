// kfp_api.cu -- host side of the C-ABI declared in include/kfp.h.
//
// Owns the device memory of one problem, validates arguments, precomputes the
// O(N_v + N_x) constant tables (transport weights, powers of q, Woodbury 2x2
// inverses per subdomain), plans the launch geometry and drives the Jacobi
// SWR iteration as a sequence of step launches on one
// CUDA stream.  Every numerical step of the path runs in kfp_device.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/kfp.h"
#include "kfp_device.cuh"
#include "kfp_fused.cuh"

using kfp::SubDev;
using kfp::StepParams;

namespace {
thread_local std::string g_err;

// Process-wide cache of device buffers keyed by (device, bytes).  A destroyed problem's buffers serve the next
// problem of the same shape: cudaFree of the ~0.7 GB of a c2 problem cost 4-130 ms per destroy (it synchronises
// the device and unmaps), which made the end-to-end solve time vary by 25 %.  "Freeing" synchronises the device
// (as cudaFree did) and parks the buffer; an allocation that finds no parked buffer of its size calls cudaMalloc,
// and on out-of-memory releases the parked buffers of the device and retries.  kfp_release_cached_memory()
// returns everything to the driver.
struct DevCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void *> parked;
    std::unordered_map<void *, std::pair<int, size_t>> live;
    size_t parked_bytes = 0;
};
DevCache &dcache() {
    static DevCache *c = new DevCache();  // never destroyed: buffers may be freed from static destructors
    return *c;
}
constexpr size_t kCacheCapBytes = size_t(32) << 30;

void release_parked(int dev_only) {  // dev_only < 0: every device (caller holds no lock)
    std::vector<std::pair<int, void *>> drop;
    {
        DevCache &c = dcache();
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.parked.begin(); it != c.parked.end();) {
            if (dev_only < 0 || it->first.first == dev_only) {
                drop.emplace_back(it->first.first, it->second);
                c.parked_bytes -= it->first.second;
                it = c.parked.erase(it);
            } else {
                ++it;
            }
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &d : drop) {
        cudaSetDevice(d.first);
        cudaFree(d.second);
    }
    cudaSetDevice(cur);
}

cudaError_t dev_malloc_raw(void **p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    bytes = (std::max<size_t>(bytes, 1) + 255) / 256 * 256;
    const auto key = std::make_pair(dev, bytes);
    DevCache &c = dcache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.parked.find(key);
        if (it != c.parked.end()) {
            *p = it->second;
            c.parked.erase(it);
            c.parked_bytes -= bytes;
            c.live[*p] = key;
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        release_parked(dev);
        e = cudaMalloc(p, bytes);
    }
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(c.mu);
        c.live[*p] = key;
    }
    return e;
}
template <class T>
cudaError_t dev_malloc(T **p, size_t bytes) {
    void *v = nullptr;
    const cudaError_t e = dev_malloc_raw(&v, bytes);
    *p = static_cast<T *>(v);
    return e;
}
cudaError_t dev_free(void *p) {
    if (!p) return cudaSuccess;
    DevCache &c = dcache();
    std::pair<int, size_t> key;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.live.find(p);
        if (it == c.live.end()) return cudaFree(p);
        key = it->second;
        c.live.erase(it);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != key.first) cudaSetDevice(key.first);
    cudaDeviceSynchronize();  // no kernel or copy of the old owner still uses it (cudaFree's own semantics)
    cudaError_t e = cudaSuccess;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.parked_bytes + key.second <= kCacheCapBytes) {
            c.parked.emplace(key, p);
            c.parked_bytes += key.second;
            p = nullptr;
        }
    }
    if (p) e = cudaFree(p);
    if (cur != key.first) cudaSetDevice(cur);
    return e;
}

void set_err(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

#define KFP_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            set_err("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__,    \
                    cudaGetErrorString(e_));                                                   \
            return e_ == cudaErrorMemoryAllocation ? KFP_E_NOMEM : KFP_E_CUDA;                 \
        }                                                                                      \
    } while (0)

struct Plan {
    bool fused = false;  // fused TMA/cluster kernel; else the three-phase path
    bool fem = false;    // the split-FEM instantiation of the fused kernel
    int P = 8, b = 32, R = 256, C = 1;
    int L = 0, B = 0, NR = 2;  // fused: chunk rows, register-array size (template), forcing ranks (template)
    int Gc_total = 1;          // fused: co-resident clusters (persistent grid size over all subdomains)
                               // col: co-resident CTAs
    size_t smem = 0;
    std::string text;
};

struct FusedData {
    CUtensorMap *maps = nullptr;  // [2][nsub][2]: load maps then store maps
    double *l2c = nullptr, *coefT = nullptr, *tabs = nullptr;
};

using FusedKernel = void (*)(const kfp::FusedParams);
template <int B, int NR, int P, bool FEM = false, bool PIPE = false>
void fused_entry(FusedKernel *k, size_t *smem) {
    *k = kfp::step_fused_tma<B, NR, P, FEM, PIPE>;
    *smem = kfp::fused_smem_bytes<B, NR, P, FEM>();
}
// instantiated (B, NR, P) combinations of the fused kernel; the split-FEM scheme (no forcing) uses NR = 2;
// pipelined-iteration variants (pipe) exist for NR = 2
bool fused_kernel(int B, int NR, int P, FusedKernel *k, size_t *smem, bool fem = false, bool pipe = false) {
#define KFP_ENTRY(BB, NN, PP)                                    \
    if (!fem && B == BB && NR == NN && P == PP) {                \
        if (!pipe) fused_entry<BB, NN, PP>(k, smem);             \
        else if (NN == 2) fused_entry<BB, 2, PP, false, true>(k, smem); \
        else return false;                                       \
        return true;                                             \
    }
#define KFP_FENTRY(BB, PP)                                       \
    if (fem && B == BB && NR == 2 && P == PP) {                  \
        if (!pipe) fused_entry<BB, 2, PP, true>(k, smem);        \
        else fused_entry<BB, 2, PP, true, true>(k, smem);        \
        return true;                                             \
    }
    KFP_ENTRY(8, 2, 8) KFP_ENTRY(16, 2, 8) KFP_ENTRY(17, 2, 8) KFP_ENTRY(32, 2, 8) KFP_ENTRY(33, 2, 8)
    KFP_ENTRY(8, 4, 8) KFP_ENTRY(16, 4, 8) KFP_ENTRY(17, 4, 8) KFP_ENTRY(32, 4, 8) KFP_ENTRY(33, 4, 8)
    KFP_ENTRY(32, 2, 16) KFP_ENTRY(33, 2, 16)
    // rank-1 forcing (the c4 family): one 8-B coefficient load per row instead of a 16-B pair
    if (!fem && !pipe && NR == 1) {
        if (B == 32 && P == 8) { fused_entry<32, 1, 8>(k, smem); return true; }
        if (B == 33 && P == 8) { fused_entry<33, 1, 8>(k, smem); return true; }
        if (B == 32 && P == 16) { fused_entry<32, 1, 16>(k, smem); return true; }
        if (B == 33 && P == 16) { fused_entry<33, 1, 16>(k, smem); return true; }
    }
    KFP_FENTRY(8, 8) KFP_FENTRY(16, 8) KFP_FENTRY(17, 8) KFP_FENTRY(32, 8) KFP_FENTRY(33, 8)
    KFP_FENTRY(32, 16) KFP_FENTRY(33, 16)
#undef KFP_ENTRY
#undef KFP_FENTRY
    return false;
}
constexpr int kBs[] = {8, 16, 17, 32, 33};

// Launch geometry for columns of at most n_max unknown rows.
// Fused path: P = 16 warps per CTA, chunks of L rows (target 17), row blocks of
// R = 16 L rows, C = ceil(n_max / R) <= 8 CTAs per cluster.  Otherwise the
// three-phase path (P = 8, b = 32, block aggregates through global memory).
Plan make_plan(const std::vector<int> &ns, int f_rank, bool allow_fused, bool fem = false) {
    Plan pl;
    const int n_max = *std::max_element(ns.begin(), ns.end());
    const int NR = (f_rank <= 2) ? 2 : 4;
    // P = 8 warps (2 CTAs per SM) first, then P = 16 (1 CTA per SM): the smallest cluster whose
    // warps hold at most 33 rows; the column's first/last row blocks must hold >= 2 rows.
    for (int P : {8, 16}) {
        int C = 1;
        while (C < 8 && (n_max + P * C - 1) / (P * C) > 33) ++C;
        int L = (n_max + P * C - 1) / (P * C);
        for (bool ok = false; !ok && L <= 33;) {
            ok = true;
            for (int n : ns)
                if (n % (P * L) == 1) ok = false;
            if (!ok) ++L;
        }
        int B = 0;
        for (int bb : kBs)
            if (bb >= L) {
                B = bb;
                break;
            }
        FusedKernel k;
        size_t smem = 0;
        // rank <= 1 forcing takes the NR = 1 instantiation where one exists (the tables keep 4-double rows)
        const int NRc = (f_rank <= 1 && !fem && B > 0 && fused_kernel(B, 1, P, &k, &smem)) ? 1 : NR;
        if (allow_fused && B > 0 && L <= 33 && f_rank <= kfp::kNRmax && fused_kernel(B, NRc, P, &k, &smem, fem)) {
            pl.fused = true;
            pl.fem = fem;
            pl.P = P;
            pl.C = C;
            pl.L = L;
            pl.B = B;
            pl.NR = NRc;
            pl.b = L;
            pl.R = P * L;
            pl.smem = smem;
            break;
        }
    }
    if (!pl.fused) {
        pl.P = 8;
        pl.b = 32;
        pl.C = (n_max + pl.P * pl.b - 1) / (pl.P * pl.b);
        pl.R = pl.P * pl.b;
        pl.smem = kfp::smem_bytes(pl.R, pl.P);
    }
    char buf[200];
    if (pl.fused)
        snprintf(buf, sizeof buf, "fused-tma-cluster%s P=%d L=%d (B=%d) R=%d C=%d NR=%d smem=%zu", pl.fem ? "-fem" : "",
                 pl.P, pl.L, pl.B, pl.R, pl.C, pl.NR, pl.smem);
    else
        snprintf(buf, sizeof buf, "three-phase P=%d b=%d R=%d C=%d smem=%zu", pl.P, pl.b, pl.R, pl.C, pl.smem);
    pl.text = buf;
    return pl;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Tensor map of a slab's unknown rows: 2-D fp64 [n rows][nx], box (32 + 2*halo) x L.
bool make_tmap(CUtensorMap *map, double *rows_base, int nx, int nrows, int L, int box_w = kfp::kTW) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)nrows};
    cuuint64_t strides[1] = {(cuuint64_t)nx * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)L};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, rows_base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace

struct MonoRun {  // an in-progress monodomain reference (run_monodomain, kfp_monodomain_shard_*)
    bool active = false, sharded = false;
    int x0 = 0, x1 = 0, n = 0;
    Plan pl;
    std::vector<SubDev> segs;  // the column, or its overlapping segments
    SubDev *d_sd = nullptr;
    StepParams P;
    FusedData fd;
    std::vector<double *> tmp;
    std::vector<void *> tmp2;
    int *d_rec = nullptr;
    std::vector<int> rec_rows, lines;
    double *halo[4] = {nullptr, nullptr, nullptr, nullptr};  // caller's send_lo, send_hi, recv_lo, recv_hi
};

struct kfp_problem_s {
    int device = 0;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    int nx = 0, nv = 0, nt = 0;
    double vmax = 0, T = 0, hx = 0, hv = 0, dt = 0, a = 0, q = 0;
    // scheme: KFP_SCHEME_IMEX_FD, or KFP_SCHEME_SPLIT_FEM: then dt = tau = T/(2 nt),
    // a = tau/h_v^2 - 1/6 (the scaled off-diagonal of M/tau + S), ar = tau/h_v^2 (Robin / trace weight)
    int scheme = KFP_SCHEME_IMEX_FD;
    double ar = 0, dnu = 0, nu0 = 0;  // FD: ar = a.  FEM transport weight |j dnu + nu0| = |v_j| tau / h_x
    int f_rank = 0, u0_rank = 0;
    std::vector<double> ft;  // host [f_rank][nt+1]
    std::vector<double> fv_host;  // host [f_rank][nv+1]
    double *d_fv = nullptr, *d_fx = nullptr, *d_u0v = nullptr, *d_u0x = nullptr;
    double2 *d_rowc = nullptr;
    double *d_cfn = nullptr;  // [nt][kMaxRank] dt * ft[r][n+1] (the cluster kernel's per-step forcing weights)
    double *d_qp = nullptr, *d_s2 = nullptr;
    int qtab_len = 0;
    std::vector<void *> allocs;  // everything else (freed at destroy)

    // monodomain
    bool mono_done = false;
    std::vector<int> mono_lines;  // node list recorded in d_Ulines
    double *d_mono[2] = {nullptr, nullptr};
    double *d_UT = nullptr;
    double *d_Ulines = nullptr;
    int *d_line_of_node = nullptr;

    // SWR
    bool setup = false;
    int kind = 0;
    double p = 0, q_rob = 0;  // Robin parameters: p on right (hi) ends, q_rob on left (lo) ends
    bool gauss_seidel = false;  // schedule: Jacobi (false) or Gauss-Seidel SWR1-SWR4 (true)
    int n_rep = 1;              // independent replicas of the decomposition (batched Robin-parameter sweep)
    int ov = 0, S = 0, s_begin = 0, s_end = 0, K_max = 0, k_done = 0;
    std::vector<int> lo, hi;
    std::vector<SubDev> subs;  // local block
    SubDev *d_subs = nullptr;
    unsigned long long *d_errT = nullptr, *d_errIF = nullptr;
    unsigned long long *d_errOV = nullptr;  // [n_rep][K_max] overlap differences (the paper's eq. 'error')
    bool ovrec = false;                     // overlap recording on (kfp_swr_set_overlap_error)
    bool ov_alloc = false;                  // its buffers / pairs exist (they stay until the next setup)
    int2 *d_pairs = nullptr;                // local interfaces (left, right subdomain index) of every replica
    int npairs = 0;
    // pipelined Jacobi iterations (kfp_swr_set_pipeline): depth D, D slots of every descriptor (slot d
    // runs iteration k0 + d, lagging d steps), trace rings of D + 1 buffers per interface and direction
    int pipe = 1;
    std::vector<SubDev> psubs;             // [D][ntot], slot-major
    SubDev *d_psubs = nullptr;
    FusedData pfd;                         // tensor maps / level-2 maps of psubs (tables shared with fd)
    std::vector<std::vector<double *>> ringL, ringR;  // [rep * (nloc-1) + i][D+1]: sent left / right
    std::vector<const double *> final_slab;           // [ntot] u(T) of the last iteration (pipelined)
    int2 *d_ppairs = nullptr;                         // [D][npairs] overlap pairs of the slot descriptors
    Plan plan;
    double *d_blkagg = nullptr, *d_chkagg = nullptr, *d_carry = nullptr;
    FusedData fd;                    // fused-kernel tensor maps and tables of the SWR setup
    std::vector<double *> swr_allocs;
    double *edge_sendL[2] = {nullptr, nullptr}, *edge_recvL[2] = {nullptr, nullptr};
    double *edge_sendR[2] = {nullptr, nullptr}, *edge_recvR[2] = {nullptr, nullptr};
    std::vector<double *> zero_on_reset;  // parity-0 incoming buffers

    int64_t launches = 0;
    MonoRun mr;
    // time-chunked iterations (kfp_swr_iterate_chunk): per chunk, "outgoing rows written" and "incoming rows
    // arrived" events; the next chunk expected
    int nchunks = 0, chunk_next = 0;
    std::vector<cudaEvent_t> chunk_sent, chunk_recv;
    std::vector<char> chunk_recv_set;
    std::vector<cudaEvent_t> ev;  // 2 per iteration of the last iterate call + 2 around it
    int ev_used = 0;
    std::string plan_text;
};

namespace {

template <class T>
kfp_status dalloc(kfp_problem pb, T **p, size_t count, std::vector<void *> *list = nullptr) {
    void *q = nullptr;
    KFP_CUDA(dev_malloc(&q, std::max<size_t>(count, 1) * sizeof(T)));
    *p = static_cast<T *>(q);
    (list ? *list : pb->allocs).push_back(q);
    return KFP_OK;
}

void free_swr(kfp_problem pb) {
    for (double *p : pb->swr_allocs) dev_free(p);
    pb->swr_allocs.clear();
    pb->subs.clear();
    pb->zero_on_reset.clear();
    if (pb->d_subs) dev_free(pb->d_subs);
    pb->d_subs = nullptr;
    if (pb->d_errT) dev_free(pb->d_errT);
    if (pb->d_errIF) dev_free(pb->d_errIF);
    pb->d_errT = pb->d_errIF = nullptr;
    pb->d_errOV = nullptr;  // (in swr_allocs)
    pb->d_pairs = nullptr;
    pb->npairs = 0;
    pb->ovrec = false;
    pb->ov_alloc = false;
    pb->pipe = 1;
    pb->psubs.clear();
    pb->d_psubs = nullptr;  // (in swr_allocs)
    pb->pfd = FusedData();
    pb->ringL.clear();
    pb->ringR.clear();
    pb->final_slab.clear();
    pb->d_ppairs = nullptr;
    pb->d_blkagg = pb->d_chkagg = pb->d_carry = nullptr;
    pb->fd = FusedData();
    for (int q = 0; q < 2; ++q) pb->edge_sendL[q] = pb->edge_recvL[q] = pb->edge_sendR[q] = pb->edge_recvR[q] = nullptr;
    pb->setup = false;
}

kfp_status swr_alloc(kfp_problem pb, double **p, size_t count) {
    void *q = nullptr;
    KFP_CUDA(dev_malloc(&q, std::max<size_t>(count, 1) * sizeof(double)));
    *p = static_cast<double *>(q);
    pb->swr_allocs.push_back(*p);
    return KFP_OK;
}

// Subdomain node ranges (R9).
void decompose(int nv, int S, int ov, std::vector<int> &lo, std::vector<int> &hi) {
    lo.assign(S, 0);
    hi.assign(S, 0);
    for (int s = 0; s < S; ++s) {
        const int cs = s * (nv / S), cs1 = (s + 1) * (nv / S);
        lo[s] = (s == 0) ? 0 : cs - ov / 2;
        hi[s] = (s == S - 1) ? nv : cs1 + (ov + 1) / 2;
    }
}

// Woodbury constants of one column system.
// pl, pr: Robin parameters of the lo (left) and hi (right) end rows (OSWR(p, q): pl = q, pr = p).
void woodbury(const kfp_problem pb, SubDev &sd, double pl, double pr) {
    const long double a = pb->a, q = pb->q, h = pb->hv, ar = pb->ar;
    const int n = sd.n;
    // d_t on rows (0,1), d_b on rows (n-2, n-1).  Unknown end rows (Robin, or the split-FEM scheme's
    // Neumann ends = Robin with p = 0) are the doubled rows (1 + 2a + 2 ar p h) u_c - 2a u_{c-+1}.
    if (sd.ltype == kfp::END_NEU) pl = 0.0;
    if (sd.rtype == kfp::END_NEU) pr = 0.0;
    const bool lrow = sd.ltype == kfp::END_ROBIN || sd.ltype == kfp::END_NEU;
    const bool rrow = sd.rtype == kfp::END_ROBIN || sd.rtype == kfp::END_NEU;
    long double wt0, wt1, wb0, wb1;
    if (lrow) {
        wt0 = a * q + 2.0L * ar * pl * h;
        wt1 = -a;
    } else {
        wt0 = a * q;
        wt1 = 0.0L;
    }
    if (rrow) {
        wb0 = -a;
        wb1 = 2.0L * ar * pr * h;
    } else {
        wb0 = 0.0L;
        wb1 = 0.0L;
    }
    // z0 = B^{-1} e_0, z1 = B^{-1} e_{n-1}: forward y_i = q y_{i-1} + (q/a) e_i, backward x_i = q x_{i+1} + y_i.
    auto solveB = [&](int unit, long double out[4]) {
        std::vector<long double> y(n), x(n + 1, 0.0L);
        long double prev = 0.0L;
        for (int i = 0; i < n; ++i) {
            prev = q * prev + ((i == unit) ? q / a : 0.0L);
            y[i] = prev;
        }
        for (int i = n - 1; i >= 0; --i) x[i] = q * x[i + 1] + y[i];
        const int rows[4] = {0, 1, n - 2, n - 1};
        for (int k = 0; k < 4; ++k) out[k] = (rows[k] >= 0 && rows[k] < n) ? x[rows[k]] : 0.0L;
    };
    long double z0[4], z1[4];
    solveB(0, z0);
    solveB(n - 1, z1);
    const long double M00 = 1.0L + wt0 * z0[0] + wt1 * z0[1];
    const long double M01 = wt0 * z1[0] + wt1 * z1[1];
    const long double M10 = wb0 * z0[2] + wb1 * z0[3];
    const long double M11 = 1.0L + wb0 * z1[2] + wb1 * z1[3];
    const long double det = M00 * M11 - M01 * M10;
    sd.wt0 = (double)wt0;
    sd.wt1 = (double)wt1;
    sd.wb0 = (double)wb0;
    sd.wb1 = (double)wb1;
    sd.Mi00 = (double)(M11 / det);
    sd.Mi01 = (double)(-M01 / det);
    sd.Mi10 = (double)(-M10 / det);
    sd.Mi11 = (double)(M00 / det);
}

kfp_status ensure_qtab(kfp_problem pb, int len) {
    if (len <= pb->qtab_len) return KFP_OK;
    std::vector<double> qp(len), s2(len);
    long double qq = 1.0L, ss = 0.0L;
    const long double q = pb->q;
    for (int k = 0; k < len; ++k) {
        qp[k] = (double)qq;
        s2[k] = (double)ss;  // sum_{t<k} q^{2t}
        ss += qq * qq;
        qq *= q;
    }
    double *dq = nullptr, *ds = nullptr;
    if (kfp_status st = dalloc(pb, &dq, len)) return st;
    if (kfp_status st = dalloc(pb, &ds, len)) return st;
    KFP_CUDA(cudaMemcpy(dq, qp.data(), len * sizeof(double), cudaMemcpyHostToDevice));
    KFP_CUDA(cudaMemcpy(ds, s2.data(), len * sizeof(double), cudaMemcpyHostToDevice));
    pb->d_qp = dq;
    pb->d_s2 = ds;
    pb->qtab_len = len;
    return KFP_OK;
}

StepParams base_params(kfp_problem pb) {
    StepParams P;
    std::memset(&P, 0, sizeof P);
    P.nx = pb->nx;
    P.nv = pb->nv;
    P.nt = pb->nt;
    P.f_rank = pb->f_rank;
    P.u0_rank = pb->u0_rank;
    P.q = pb->q;
    P.a = pb->a;
    P.qa = pb->q / pb->a;
#ifdef KFP_MUTATE  // test-only mutant build (libkfp_mut.so): one step-kernel coefficient off by 1e-3
    P.qa *= 1.0 + 1e-3;
#endif
    P.hv = pb->hv;
    P.dt = pb->dt;
    P.dnu = pb->dnu;
    P.nu0 = pb->nu0;
    P.rowc = pb->d_rowc;
    P.cfn = pb->d_cfn;
    P.fv = pb->d_fv;
    P.fx = pb->d_fx;
    P.u0v = pb->d_u0v;
    P.u0x = pb->d_u0x;
    P.qp = pb->d_qp;
    P.s2 = pb->d_s2;
    P.qtab_len = pb->qtab_len;
    return P;
}

// One time step of every subdomain in P.subs (nsub entries); pipe: the pipelined-iteration variant
// (each descriptor at step n - lag).
kfp_status launch_step(kfp_problem pb, const Plan &pl, StepParams &P, int nsub, int n, const FusedData &fd,
                       int nrec = 0, const int *rec_rows = nullptr, bool pipe = false) {
    P.n = n;
    P.from_u0 = (n == 0);
    // split FEM: step n transports w^{n-1/2} (the previous step's Step 2) before its Step 1; the kernel
    // drops the transport at step 0 (it starts from u0)
    P.dnu = pb->dnu;
    P.nu0 = pb->nu0;
    for (int r = 0; r < kfp::kMaxRank; ++r) P.cf[r] = (r < pb->f_rank) ? pb->dt * pb->ft[(size_t)r * (pb->nt + 1) + n + 1] : 0.0;
    P.P = pl.P;
    P.b = pl.b;
    P.R = pl.R;
    P.C = pl.C;
    // x-tiles [tile0, tile_end) of this launch: every tile, or a sharded monodomain's column range
    if (P.xend <= 0) P.xend = pb->nx;
    const int tile_end = (P.xend + kfp::kWarp - 1) / kfp::kWarp, ntiles = tile_end - P.tile0;
    const dim3 block(pl.P * kfp::kWarp);
    if (pl.fused) {
        kfp::FusedParams FP;
        FP.S = P;
        FP.tmaps = fd.maps;
        FP.L = pl.L;
        FP.ntiles = tile_end;  // (absolute: clusters walk t = tile0 + y, + Gc, ... < tile_end)
        FP.Gc = std::max(1, std::min(ntiles, pl.Gc_total / std::max(1, nsub)));
        FP.nrec = nrec;
        FP.rec_rows = rec_rows;
        FP.l2m = fd.l2c;
        FP.coefT = fd.coefT;
        FP.tabs = fd.tabs;
        FusedKernel k;
        size_t smem;
        if (!fused_kernel(pl.B, pl.NR, pl.P, &k, &smem, pl.fem, pipe)) {
            set_err("launch_step: no fused kernel for B=%d NR=%d P=%d%s", pl.B, pl.NR, pl.P, pipe ? " (pipelined)" : "");
            return KFP_E_INVAL;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(pl.C, FP.Gc, nsub);
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = pb->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = pl.C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        KFP_CUDA(cudaLaunchKernelEx(&cfg, k, FP));
        pb->launches += 1;
    } else {
        kfp::step_phase1<<<dim3(pl.C, ntiles, nsub), block, pl.smem, pb->stream>>>(P);
        // phase 2: a warp per column (block recurrences as shuffle scans; step_phase2 is the serial reference form)
        kfp::step_phase2_warp<<<dim3((P.xend - P.tile0 * kfp::kWarp + 3) / 4, 1, nsub), 128, 0, pb->stream>>>(P);
        kfp::step_phase3<<<dim3(pl.C, ntiles, nsub), block, pl.smem, pb->stream>>>(P);
        pb->launches += 3;
    }
    KFP_CUDA(cudaGetLastError());
    return KFP_OK;
}

// Level-2 linear maps (kfp_fused.cuh, kL2M layout): for every subdomain and row block
// `me`, the block carries (Y_blk(me), X_blk(me)) as linear functions of the 22 inputs
// v = (F_0..7, G_0..7, x~ at rows 0,1,n-2,n-1, g_lo, g_hi), obtained by running the
// block chain + Woodbury solve on the unit vectors, in long double.
kfp_status build_l2m(kfp_problem pb, const Plan &pl, const std::vector<SubDev> &subs, double **out,
                     std::vector<void *> *owner) {
    *out = nullptr;
    if (!pl.fused) return KFP_OK;
    const long double q = pb->q, a = pb->a;
    auto qp = [&](long double e) { return powl(q, e); };
    auto s2 = [&](int k) {  // sum_{t<k} q^{2t}
        long double s = 0, t = 1;
        for (int i = 0; i < k; ++i) {
            s += t;
            t *= q * q;
        }
        return s;
    };
    auto kap = [&](int r, int len) { return qp(r + 1) * s2(len - r); };
    const int C = pl.C, R = pl.R;
    std::vector<double> h(subs.size() * C * kfp::kL2M, 0.0);
    for (size_t i = 0; i < subs.size(); ++i) {
        const SubDev &sd = subs[i];
        const int n = sd.n, nb = sd.nblk;
        std::vector<long double> QR(nb), K0(nb), QB(nb), KB(nb), QE(nb);
        for (int b = 0; b < nb; ++b) {
            const int Rc = std::min(R, n - b * R), bc = b * R, ec = bc + Rc;
            QR[b] = qp(Rc);
            K0[b] = kap(0, Rc);
            QB[b] = qp(bc);
            KB[b] = (ec >= n) ? 0.0L : kap(ec, n);
            QE[b] = qp(n - ec);
        }
        const int rows[4] = {0, 1, n - 2, n - 1};
        for (int j = 0; j < kfp::kL2N; ++j) {
            long double v[kfp::kL2N] = {0};
            v[j] = 1.0L;
            const long double Yt0 = sd.injL * v[20] / a, Xb0 = sd.injR * v[21] / a;
            std::vector<long double> Yb(nb), Xb(nb);
            long double Y = Yt0;
            for (int b = 0; b < nb; ++b) {
                Yb[b] = Y;
                Y = QR[b] * Y + (b < 8 ? v[b] : 0.0L);
            }
            long double X = Xb0;
            for (int b = nb - 1; b >= 0; --b) {
                Xb[b] = X;
                X = QR[b] * X + K0[b] * Yb[b] + (b < 8 ? v[8 + b] : 0.0L);
            }
            long double xt[4];
            for (int qq = 0; qq < 4; ++qq) {
                const int r = std::max(rows[qq], 0), b = r / R, l = r - b * R, Rc = std::min(R, n - b * R);
                xt[qq] = v[16 + qq] + kap(l, Rc) * Yb[b] + qp(Rc - l) * Xb[b];
            }
            const long double s0 = sd.wt0 * xt[0] + (long double)sd.wt1 * xt[1];
            const long double s1 = sd.wb0 * xt[2] + (long double)sd.wb1 * xt[3];
            const long double dY = -(sd.Mi00 * s0 + (long double)sd.Mi01 * s1) / a;
            const long double dX = -(sd.Mi10 * s0 + (long double)sd.Mi11 * s1) / a;
            for (int me = 0; me < nb; ++me) {
                double *c = h.data() + (i * C + me) * kfp::kL2M;
                c[j] = (double)(Yb[me] + QB[me] * dY);
                c[24 + j] = (double)(Xb[me] + KB[me] * dY + QE[me] * dX);
            }
        }
    }
    void *d = nullptr;
    KFP_CUDA(dev_malloc(&d, sizeof(double) * h.size()));
    KFP_CUDA(cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    *out = static_cast<double *>(d);
    if (owner) owner->push_back(d);
    return KFP_OK;
}

// Per-node coefficient rows (q/a)(1-|nu_j|), (q/a)|nu_j|, (q/a) fv_r(j) (NR columns) and the
// per-plan table qp[kQ] | s2[kQ] | kr[2B] of the fused kernel.
kfp_status build_fused_tables(kfp_problem pb, const Plan &pl, std::vector<double> *fv_host, double **coefT,
                              double **tabs, std::vector<void *> *owner) {
    *coefT = *tabs = nullptr;
    if (!pl.fused) return KFP_OK;
    const int kc = 2 + std::max(2, pl.NR), nn = pb->nv + 1;  // NR = 1 rows padded (kfp_fused.cuh kCoef)
    const long double qa = (long double)pb->q / pb->a;
    std::vector<double> c((size_t)nn * kc, 0.0);
    for (int j = 0; j < nn; ++j) {
        const double v = -pb->vmax + (double)j * pb->hv;
        const double nu = std::fabs(v * pb->dt / pb->hx);
        c[(size_t)j * kc + 0] = (double)(qa * (1.0 - nu));
        c[(size_t)j * kc + 1] = (double)(qa * nu);
        for (int r = 0; r < pb->f_rank; ++r) c[(size_t)j * kc + 2 + r] = (double)(qa * (*fv_host)[(size_t)r * nn + j]);
    }
    const int kQ = ((pl.P * pl.B + 2) + 1) / 2 * 2;
    std::vector<double> t(2 * kQ + 2 * pl.B + 4, 0.0);
    const long double q = pb->q;
    long double qq = 1.0L, ss = 0.0L;
    for (int k = 0; k < kQ; ++k) {
        t[k] = (double)qq;
        t[kQ + k] = (double)ss;
        ss += qq * qq;
        qq *= q;
    }
    for (int l = 0; l < pl.L; ++l) {
        long double kap = 0.0L;  // kap(l, L) = sum_{i=l}^{L-1} q^{i-l} q^{i+1}
        for (int i = l; i < pl.L; ++i) kap += powl(q, i - l) * powl(q, i + 1);
        t[2 * kQ + 2 * l] = (double)kap;
        t[2 * kQ + 2 * l + 1] = (double)powl(q, pl.L - l);
    }
    // pass C of full chunks (kfp_fused.cuh): 1/q, 1/(1-q^2), q^{L+1}, q^L
    t[2 * kQ + 2 * pl.B + 0] = (double)(1.0L / q);
    t[2 * kQ + 2 * pl.B + 1] = (double)(1.0L / (1.0L - q * q));
    t[2 * kQ + 2 * pl.B + 2] = (double)powl(q, pl.L + 1);
    t[2 * kQ + 2 * pl.B + 3] = (double)powl(q, pl.L);
    void *d1 = nullptr, *d2 = nullptr;
    KFP_CUDA(dev_malloc(&d1, sizeof(double) * c.size()));
    KFP_CUDA(cudaMemcpy(d1, c.data(), sizeof(double) * c.size(), cudaMemcpyHostToDevice));
    KFP_CUDA(dev_malloc(&d2, sizeof(double) * t.size()));
    KFP_CUDA(cudaMemcpy(d2, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice));
    *coefT = static_cast<double *>(d1);
    *tabs = static_cast<double *>(d2);
    owner->push_back(d1);
    owner->push_back(d2);
    return KFP_OK;
}

// Tensor maps of the slabs of nsub subdomains (host copy -> device array).
// Load maps (box 36 x L, incl. halo) then store maps (box 32 x L): [2][nsub][2].
kfp_status build_tmaps(kfp_problem pb, const Plan &pl, const std::vector<SubDev> &subs, CUtensorMap **out,
                       std::vector<void *> *owner) {
    *out = nullptr;
    if (!pl.fused) return KFP_OK;
    const size_t ns = subs.size();
    std::vector<CUtensorMap> maps(4 * ns);
    for (size_t i = 0; i < ns; ++i)
        for (int q = 0; q < 2; ++q) {
            // FD: rows = the unknown rows, box L rows.  FEM: rows = every node of the slab, box L + 2 rows
            // (the chunk and the rows above and below it; the kernel starts the box one row above)
            const int off = pl.fem ? 0 : subs[i].first - subs[i].lo;
            const int nrows = pl.fem ? subs[i].hi - subs[i].lo + 1 : subs[i].n, box = pl.fem ? pl.L + 2 : pl.L;
            double *base = subs[i].slab[q] + (size_t)off * pb->nx;
            if (!make_tmap(&maps[2 * i + q], base, pb->nx, nrows, box) ||
                !make_tmap(&maps[2 * ns + 2 * i + q], base, pb->nx, nrows, box, kfp::kWarp)) {
                set_err("cuTensorMapEncodeTiled failed (nx=%d rows=%d L=%d)", pb->nx, subs[i].n, pl.L);
                return KFP_E_CUDA;
            }
        }
    void *d = nullptr;
    KFP_CUDA(dev_malloc(&d, sizeof(CUtensorMap) * maps.size()));
    KFP_CUDA(cudaMemcpy(d, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
    *out = static_cast<CUtensorMap *>(d);
    if (owner) owner->push_back(d);
    return KFP_OK;
}

kfp_status configure_kernels(Plan &pl) {
    if (pl.fused) {
        FusedKernel k;
        size_t smem;
        fused_kernel(pl.B, pl.NR, pl.P, &k, &smem, pl.fem);
        KFP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(pl.C, 1024, 1);
        cfg.blockDim = dim3(pl.P * kfp::kWarp);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = pl.C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int ncl = 0;
        KFP_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
        pl.Gc_total = std::max(1, ncl);
    } else {
        KFP_CUDA(cudaFuncSetAttribute(kfp::step_phase1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        KFP_CUDA(cudaFuncSetAttribute(kfp::step_phase3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    }
    return KFP_OK;
}

kfp_status alloc_general_scratch(kfp_problem pb, const Plan &pl, int nsub, double **blkagg, double **chkagg,
                                 double **carry, std::vector<double *> &owner) {
    const size_t nx = pb->nx;
    auto al = [&](double **p, size_t c) -> kfp_status {
        void *q = nullptr;
        KFP_CUDA(dev_malloc(&q, std::max<size_t>(c, 1) * sizeof(double)));
        *p = static_cast<double *>(q);
        owner.push_back(*p);
        return KFP_OK;
    };
    if (pl.fused) {
        *blkagg = *chkagg = *carry = nullptr;
        return KFP_OK;
    }
    if (kfp_status st = al(blkagg, (size_t)nsub * pl.C * 8 * nx)) return st;
    if (kfp_status st = al(chkagg, (size_t)nsub * pl.C * pl.P * 2 * nx)) return st;
    if (kfp_status st = al(carry, (size_t)nsub * pl.C * 2 * nx)) return st;
    KFP_CUDA(cudaMemset(*blkagg, 0, (size_t)nsub * pl.C * 8 * nx * sizeof(double)));
    return KFP_OK;
}

// Split FEM: the window's last Step 2 for every subdomain in P.subs (nsub entries) -> the other slab
// buffer, plus err_T against P.UT when set (kfp_fused.cuh fem_finish).
kfp_status launch_fem_finish(kfp_problem pb, StepParams P, int nsub, int max_rows) {
    P.dnu = pb->dnu;
    P.nu0 = pb->nu0;
    const int gy = std::max(1, std::min(max_rows, std::max(1, 4096 / std::max(1, nsub))));
    kfp::fem_finish<<<dim3((pb->nx + 127) / 128, gy, nsub), 128, 0, pb->stream>>>(P);
    pb->launches += 1;
    KFP_CUDA(cudaGetLastError());
    return KFP_OK;
}

// slab buffer that holds u(T) after a window: the last step's output (FD), or the fem_finish output
int final_parity(const kfp_problem pb) { return (pb->nt + (pb->scheme == KFP_SCHEME_SPLIT_FEM ? 1 : 0)) & 1; }
// u(T) slab of local descriptor ii after the last iteration
const double *final_slab(const kfp_problem pb, size_t ii) {
    if (pb->pipe > 1 && ii < pb->final_slab.size() && pb->final_slab[ii]) return pb->final_slab[ii];
    return pb->subs[ii].slab[final_parity(pb)];
}

// Monodomain solve recording U at `lines` (BJ north_star (c)).
// Monodomain reference in three pieces (mono_begin / mono_step / mono_end) so that a multi-GPU job can shard
// it along x: each process computes the columns [x0, x1) and exchanges the halo columns x0 - 1 and x1 (the
// upwind transport's only coupling between columns) after every step (kfp_monodomain_shard_*).
kfp_status mono_begin(kfp_problem pb, const std::vector<int> &lines, int x0, int x1, double *const halo[4]) {
    MonoRun &mr = pb->mr;
    const size_t nx = pb->nx, nn = (size_t)pb->nv + 1;
    if (!pb->d_mono[0]) {
        for (int q = 0; q < 2; ++q)
            if (kfp_status st = dalloc(pb, &pb->d_mono[q], nn * nx)) return st;
        if (kfp_status st = dalloc(pb, &pb->d_line_of_node, nn)) return st;
    }
    for (int q = 0; q < 2; ++q) KFP_CUDA(cudaMemsetAsync(pb->d_mono[q], 0, nn * nx * sizeof(double), pb->stream));
    std::vector<int> lon(nn, -1);
    for (size_t i = 0; i < lines.size(); ++i) lon[lines[i]] = (int)i;
    KFP_CUDA(cudaMemcpyAsync(pb->d_line_of_node, lon.data(), nn * sizeof(int), cudaMemcpyHostToDevice, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));  // (lon is a host temporary)
    if (pb->d_Ulines) {
        dev_free(pb->d_Ulines);
        pb->allocs.erase(std::find(pb->allocs.begin(), pb->allocs.end(), (void *)pb->d_Ulines));
        pb->d_Ulines = nullptr;
    }
    if (!lines.empty())
        if (kfp_status st = dalloc(pb, &pb->d_Ulines, lines.size() * (size_t)pb->nt * nx)) return st;
    pb->mono_done = false;

    // The column [first, first + n) -- or, when it is taller than the cluster kernel's 8 x 16 x 33 rows (the
    // c3 / c4 monodomain), overlapping segments of it.  A segment is solved as a column of its own with zero
    // Dirichlet data just outside it and stores only its interior rows [wlo, whi); the artificial ends
    // perturb the solution by ~ q^d / (1 - q^2) of its size at distance d (the discrete Green's function of
    // tridiag(-a, 1 + 2a, -a) decays like q^d), so interiors H rows away with q^H / (1 - q^2) < 2^-60 are
    // the column's solution to round-off.  (The FD scheme; the split-FEM reference stays one column.)
    const bool fem = pb->scheme == KFP_SCHEME_SPLIT_FEM;
    const int first = fem ? 0 : 1, ncol = fem ? pb->nv + 1 : pb->nv - 1;
    auto column_sd = [&](int r0, int r1, int w0, int w1) {  // rows [r0, r1) of the column, stores [w0, w1)
        SubDev sd;
        std::memset(&sd, 0, sizeof sd);
        sd.first = first + r0;
        sd.n = r1 - r0;
        sd.lo = sd.first - (fem ? 0 : 1);
        sd.hi = sd.first + sd.n - (fem ? 1 : 0);
        sd.ltype = sd.rtype = fem ? kfp::END_NEU : kfp::END_PHYS;
        sd.iL_tr = sd.iR_tr = -2;
        sd.ifL = sd.ifR = -1;
        sd.slab[0] = pb->d_mono[0] + (size_t)sd.lo * nx;
        sd.slab[1] = pb->d_mono[1] + (size_t)sd.lo * nx;
        sd.wlo = w0 - r0;
        sd.whi = w1 - r0;
        woodbury(pb, sd, 0.0, 0.0);
        return sd;
    };
    mr.segs.clear();
    constexpr int kMaxCol = 8 * 16 * 33;  // the cluster kernel's tallest column
    if (!fem && ncol > kMaxCol) {
        const long double q = pb->q;
        const int H = (int)std::ceil(std::log(std::ldexp(1.0L, -60) * (1.0L - q * q)) / std::log(q));
        const int I = kMaxCol - 2 * H;  // interior rows per segment
        if (I >= kMaxCol / 4)
            for (int w0 = 0; w0 < ncol; w0 += I) {
                const int w1 = std::min(ncol, w0 + I);
                mr.segs.push_back(column_sd(std::max(0, w0 - H), std::min(ncol, w1 + H), w0, w1));
            }
    }
    if (mr.segs.empty()) mr.segs.push_back(column_sd(0, ncol, 0, ncol));
    std::vector<int> ns;
    for (const SubDev &sd : mr.segs) ns.push_back(sd.n);
    mr.pl = make_plan(ns, pb->f_rank, true, fem);
    Plan &pl = mr.pl;
    if (fem && !pl.fused) {
        set_err("monodomain: the split-FEM scheme needs the cluster kernel (column of %d rows > %d)", ncol, kMaxCol);
        return KFP_E_INVAL;
    }
    int nmax = 0;
    for (SubDev &sd : mr.segs) {
        sd.nblk = (sd.n + pl.R - 1) / pl.R;
        nmax = std::max(nmax, sd.n);
    }
    if (kfp_status st = ensure_qtab(pb, std::max(pl.R, nmax) + 2)) return st;
    if (kfp_status st = configure_kernels(pl)) return st;
    KFP_CUDA(dev_malloc(&mr.d_sd, sizeof(SubDev) * mr.segs.size()));
    KFP_CUDA(cudaMemcpyAsync(mr.d_sd, mr.segs.data(), sizeof(SubDev) * mr.segs.size(), cudaMemcpyHostToDevice, pb->stream));
    StepParams &P = mr.P;
    P = base_params(pb);
    P.subs = mr.d_sd;
    P.record = lines.empty() ? 0 : 1;
    P.line_of_node = pb->d_line_of_node;
    P.rec = pb->d_Ulines;
    P.last = 0;  // no error accumulation on the reference itself; end rows stay 0 (memset)
    P.tile0 = x0 / kfp::kWarp;
    P.xend = x1;
    mr.rec_rows = lines;  // node indices (the cluster kernel converts per descriptor)
    kfp_status st = alloc_general_scratch(pb, pl, (int)mr.segs.size(), &P.blkagg, &P.chkagg, &P.carry, mr.tmp);
    if (!st) st = build_tmaps(pb, pl, mr.segs, &mr.fd.maps, &mr.tmp2);
    if (!st) st = build_l2m(pb, pl, mr.segs, &mr.fd.l2c, &mr.tmp2);
    if (!st) st = build_fused_tables(pb, pl, &pb->fv_host, &mr.fd.coefT, &mr.fd.tabs, &mr.tmp2);
    if (!st && !mr.rec_rows.empty()) {
        if (dev_malloc(&mr.d_rec, sizeof(int) * mr.rec_rows.size()) != cudaSuccess ||
            cudaMemcpy(mr.d_rec, mr.rec_rows.data(), sizeof(int) * mr.rec_rows.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            st = KFP_E_CUDA;
    }
    mr.x0 = x0;
    mr.x1 = x1;
    mr.n = 0;
    mr.lines = lines;
    mr.sharded = !(x0 == 0 && x1 == pb->nx);
    for (int k = 0; k < 4; ++k) mr.halo[k] = halo ? halo[k] : nullptr;
    mr.active = true;
    return st;
}

void mono_free(kfp_problem pb) {
    MonoRun &mr = pb->mr;
    if (mr.d_sd) dev_free(mr.d_sd);
    if (mr.d_rec) dev_free(mr.d_rec);
    for (double *q : mr.tmp) dev_free(q);
    for (void *q : mr.tmp2) dev_free(q);
    mr = MonoRun();
}

kfp_status mono_step(kfp_problem pb) {
    MonoRun &mr = pb->mr;
    const int n = mr.n, nx = pb->nx, rows = pb->nv + 1;
    const unsigned gb = (unsigned)((rows + 255) / 256);
    if (mr.sharded && n > 0) {  // the halo columns of u^n from the neighbouring shards
        kfp::halo_unpack<<<gb, 256, 0, pb->stream>>>(pb->d_mono[n & 1], nx, rows, (mr.x0 - 1 + nx) % nx, mr.halo[2]);
        kfp::halo_unpack<<<gb, 256, 0, pb->stream>>>(pb->d_mono[n & 1], nx, rows, mr.x1 % nx, mr.halo[3]);
        pb->launches += 2;
    }
    if (kfp_status st = launch_step(pb, mr.pl, mr.P, (int)mr.segs.size(), n, mr.fd, (int)mr.rec_rows.size(), mr.d_rec))
        return st;
    if (mr.sharded) {  // this shard's edge columns of u^{n+1} for the neighbours
        kfp::halo_pack<<<gb, 256, 0, pb->stream>>>(pb->d_mono[(n + 1) & 1], nx, rows, mr.x0, mr.halo[0]);
        kfp::halo_pack<<<gb, 256, 0, pb->stream>>>(pb->d_mono[(n + 1) & 1], nx, rows, mr.x1 - 1, mr.halo[1]);
        pb->launches += 2;
        KFP_CUDA(cudaGetLastError());
    }
    mr.n = n + 1;
    return KFP_OK;
}

kfp_status mono_end(kfp_problem pb) {
    MonoRun &mr = pb->mr;
    kfp_status st = KFP_OK;
    if (pb->scheme == KFP_SCHEME_SPLIT_FEM) {  // U(T): the last Step 2 (no error slot)
        StepParams P = mr.P;
        P.UT = nullptr;
        P.errT = nullptr;
        st = launch_fem_finish(pb, P, 1, pb->nv + 1);
    }
    cudaError_t e = cudaStreamSynchronize(pb->stream);
    const std::vector<int> lines = mr.lines;
    mono_free(pb);
    if (st != KFP_OK) return st;
    KFP_CUDA(e);
    pb->d_UT = pb->d_mono[final_parity(pb)];
    pb->mono_lines = lines;
    pb->mono_done = true;
    return KFP_OK;
}

kfp_status run_monodomain(kfp_problem pb, const std::vector<int> &lines) {
    if (pb->mr.active) mono_free(pb);
    kfp_status st = mono_begin(pb, lines, 0, pb->nx, nullptr);
    for (int n = 0; st == KFP_OK && n < pb->nt; ++n) st = mono_step(pb);
    if (st != KFP_OK) {
        cudaStreamSynchronize(pb->stream);
        mono_free(pb);
        return st;
    }
    return mono_end(pb);
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

const char *kfp_last_error(void) { return g_err.c_str(); }

void kfp_release_cached_memory(void) { release_parked(-1); }

kfp_status kfp_problem_create(const kfp_problem_desc *d, kfp_problem *out) {
    return kfp_problem_create_ex(d, KFP_SCHEME_IMEX_FD, out);
}

kfp_status kfp_problem_create_ex(const kfp_problem_desc *d, kfp_scheme scheme, kfp_problem *out) {
    if (!d || !out) {
        set_err("kfp_problem_create: NULL argument");
        return KFP_E_INVAL;
    }
    if (scheme != KFP_SCHEME_IMEX_FD && scheme != KFP_SCHEME_SPLIT_FEM) {
        set_err("kfp_problem_create: unknown scheme %d", (int)scheme);
        return KFP_E_INVAL;
    }
    const bool fem = scheme == KFP_SCHEME_SPLIT_FEM;
    if (d->nx < 2 || d->nx % 2 || d->nv < 2 || d->nv % 2 || d->nt < 1 || !(d->vmax > 0) || !(d->t_final > 0) ||
        d->f_rank < 0 || d->f_rank > kfp::kMaxRank || d->u0_rank < 0 || d->u0_rank > kfp::kMaxRank) {
        set_err("kfp_problem_create: invalid sizes (nx=%d nv=%d nt=%d vmax=%g T=%g f_rank=%d u0_rank=%d); "
                "need nx,nv >= 2 even, nt >= 1, vmax,T > 0, ranks in [0,%d]",
                d->nx, d->nv, d->nt, d->vmax, d->t_final, d->f_rank, d->u0_rank, kfp::kMaxRank);
        return KFP_E_INVAL;
    }
    if ((d->f_rank > 0 && (!d->ft || !d->fv || !d->fx)) || (d->u0_rank > 0 && (!d->u0v || !d->u0x))) {
        set_err("kfp_problem_create: missing table pointer");
        return KFP_E_INVAL;
    }
    // split FEM: both sub-steps over tau = dt/2, no forcing (the paper's error
    // equation), and tau/h_v^2 > 1/6 so that M/tau + S has negative off-diagonals (the
    // kernel's constant-coefficient recurrence needs a = tau/h_v^2 - 1/6 > 0)
    const double hx = 1.0 / d->nx, dt = d->t_final / d->nt * (fem ? 0.5 : 1.0);
    const double cfl = d->vmax * dt / hx;
    if (cfl > 1.0) {
        set_err("kfp_problem_create: CFL Vmax*%s/h_x = %.6g > 1 (upwind step not a convex combination)",
                fem ? "tau" : "dt", cfl);
        return KFP_E_CFL;
    }
    if (fem) {
        const double hv = 2.0 * d->vmax / d->nv, r = dt / (hv * hv);
        if (d->f_rank != 0) {
            set_err("kfp_problem_create: the split-FEM scheme has no forcing term (P:602-605); f_rank must be 0");
            return KFP_E_INVAL;
        }
        if (!(r > 1.0 / 6.0 + 1e-12)) {
            set_err("kfp_problem_create: split FEM needs tau/h_v^2 > 1/6 (got %.6g)", r);
            return KFP_E_INVAL;
        }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_err("kfp_problem_create: no CUDA device available (this library has no CPU path)");
        return KFP_E_CUDA;
    }
    if (d->device < 0 || d->device >= ndev) {
        set_err("kfp_problem_create: device %d out of range (%d devices)", d->device, ndev);
        return KFP_E_INVAL;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d->device) != cudaSuccess || prop.major < 10) {
        set_err("kfp_problem_create: device %d is not sm_100 (compute capability %d.%d)", d->device, prop.major,
                prop.minor);
        return KFP_E_CUDA;
    }
    kfp_problem pb = new kfp_problem_s();
    pb->device = d->device;
    if (cudaSetDevice(d->device) != cudaSuccess || cudaStreamCreateWithFlags(&pb->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        set_err("kfp_problem_create: cannot set device / create stream");
        delete pb;
        return KFP_E_CUDA;
    }
    pb->stream = pb->own_stream;
    pb->nx = d->nx;
    pb->nv = d->nv;
    pb->nt = d->nt;
    pb->vmax = d->vmax;
    pb->T = d->t_final;
    pb->hx = hx;
    pb->hv = 2.0 * d->vmax / d->nv;
    pb->dt = dt;
    pb->scheme = scheme;
    pb->ar = dt / (pb->hv * pb->hv);
    pb->a = fem ? pb->ar - 1.0 / 6.0 : pb->ar;  // FEM: (M/tau + S) tau/h = tridiag(-a, 1 + 2a, -a)
    pb->q = ((1.0 + 2.0 * pb->a) - std::sqrt(1.0 + 4.0 * pb->a)) / (2.0 * pb->a);
    pb->dnu = pb->hv * dt / hx;
    pb->nu0 = -d->vmax * dt / hx;
    pb->f_rank = d->f_rank;
    pb->u0_rank = d->u0_rank;
    pb->ft.assign(d->ft, d->ft + (size_t)d->f_rank * (d->nt + 1));
    pb->fv_host.assign(d->fv, d->fv + (size_t)d->f_rank * (d->nv + 1));
    const size_t nn = (size_t)d->nv + 1;
    std::vector<double2> rowc(nn);
    for (size_t j = 0; j < nn; ++j) {
        const double v = -d->vmax + (double)j * pb->hv;
        const double nu = std::fabs(v * dt / hx);
        rowc[j] = make_double2(1.0 - nu, nu);
    }
    kfp_status st = KFP_OK;
    auto up = [&](double **dst, const double *src, size_t cnt) -> kfp_status {
        if (kfp_status s2 = dalloc(pb, dst, cnt)) return s2;
        if (cnt) KFP_CUDA(cudaMemcpy(*dst, src, cnt * sizeof(double), cudaMemcpyHostToDevice));
        return KFP_OK;
    };
    if (!st) st = up(&pb->d_fv, d->fv, (size_t)d->f_rank * nn);
    if (!st) st = up(&pb->d_fx, d->fx, (size_t)d->f_rank * d->nx);
    if (!st) st = up(&pb->d_u0v, d->u0v, (size_t)d->u0_rank * nn);
    if (!st) st = up(&pb->d_u0x, d->u0x, (size_t)d->u0_rank * d->nx);
    if (!st) st = up(reinterpret_cast<double **>(&pb->d_rowc), reinterpret_cast<const double *>(rowc.data()), 2 * nn);
    {
        std::vector<double> cfn((size_t)d->nt * kfp::kMaxRank, 0.0);
        for (int n = 0; n < d->nt; ++n)
            for (int r = 0; r < d->f_rank; ++r)  // the same product launch_step forms for P.cf
                cfn[(size_t)n * kfp::kMaxRank + r] = pb->dt * pb->ft[(size_t)r * (d->nt + 1) + n + 1];
        if (!st) st = up(&pb->d_cfn, cfn.data(), cfn.size());
    }
    if (st) {
        kfp_problem_destroy(pb);
        return st;
    }
    *out = pb;
    return KFP_OK;
}

void kfp_problem_destroy(kfp_problem pb) {
    if (!pb) return;
    cudaSetDevice(pb->device);
    if (pb->stream) cudaStreamSynchronize(pb->stream);
    if (pb->mr.active) mono_free(pb);
    free_swr(pb);
    for (void *p : pb->allocs) dev_free(p);
    for (cudaEvent_t e : pb->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : pb->chunk_sent) cudaEventDestroy(e);
    for (cudaEvent_t e : pb->chunk_recv) cudaEventDestroy(e);
    if (pb->own_stream) cudaStreamDestroy(pb->own_stream);
    delete pb;
}

kfp_status kfp_set_stream(kfp_problem pb, void *stream) {
    if (!pb) {
        set_err("kfp_set_stream: NULL problem");
        return KFP_E_INVAL;
    }
    pb->stream = stream ? static_cast<cudaStream_t>(stream) : pb->own_stream;
    return KFP_OK;
}

kfp_status kfp_monodomain_solve(kfp_problem pb, double *uT) {
    if (!pb) {
        set_err("kfp_monodomain_solve: NULL problem");
        return KFP_E_INVAL;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    if (!pb->mono_done)
        if (kfp_status st = run_monodomain(pb, pb->mono_lines)) return st;
    if (uT) {
        KFP_CUDA(cudaMemcpyAsync(uT, pb->d_UT, sizeof(double) * ((size_t)pb->nv + 1) * pb->nx, cudaMemcpyDeviceToHost,
                                 pb->stream));
        KFP_CUDA(cudaStreamSynchronize(pb->stream));
    }
    return KFP_OK;
}

kfp_status kfp_monodomain_shard_begin(kfp_problem pb, int32_t x0, int32_t x1, const int32_t *lines, int32_t nlines,
                                      double *send_lo, double *send_hi, double *recv_lo, double *recv_hi) {
    if (!pb || nlines < 0 || (nlines > 0 && !lines)) {
        set_err("kfp_monodomain_shard_begin: NULL problem or lines");
        return KFP_E_INVAL;
    }
    const bool full = (x0 == 0 && x1 == pb->nx);
    if (x0 < 0 || x1 > pb->nx || x0 >= x1 || x0 % kfp::kWarp || (x1 % kfp::kWarp && x1 != pb->nx)) {
        set_err("kfp_monodomain_shard_begin: columns [%d, %d) must be a range of 32-column tiles of [0, %d)", x0, x1, pb->nx);
        return KFP_E_INVAL;
    }
    if (!full && (!send_lo || !send_hi || !recv_lo || !recv_hi)) {
        set_err("kfp_monodomain_shard_begin: a partial column range needs the four halo buffers");
        return KFP_E_INVAL;
    }
    if (!full && pb->scheme == KFP_SCHEME_SPLIT_FEM) {
        set_err("kfp_monodomain_shard_begin: the split-FEM reference is not sharded");
        return KFP_E_INVAL;
    }
    std::vector<int> ls(lines, lines + nlines);
    for (int l : ls)
        if (l < 0 || l > pb->nv) {
            set_err("kfp_monodomain_shard_begin: line node %d outside [0, %d]", l, pb->nv);
            return KFP_E_INVAL;
        }
    KFP_CUDA(cudaSetDevice(pb->device));
    if (pb->mr.active) mono_free(pb);
    double *halo[4] = {send_lo, send_hi, recv_lo, recv_hi};
    if (kfp_status st = mono_begin(pb, ls, x0, x1, halo)) {
        cudaStreamSynchronize(pb->stream);
        mono_free(pb);
        return st;
    }
    return KFP_OK;
}

kfp_status kfp_monodomain_shard_step(kfp_problem pb) {
    if (!pb || !pb->mr.active || pb->mr.n >= pb->nt) {
        set_err("kfp_monodomain_shard_step: no sharded reference in progress (or all %d steps done)", pb ? pb->nt : 0);
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    return mono_step(pb);
}

kfp_status kfp_monodomain_shard_end(kfp_problem pb) {
    if (!pb || !pb->mr.active || pb->mr.n != pb->nt) {
        set_err("kfp_monodomain_shard_end: the reference has not run its %d steps", pb ? pb->nt : 0);
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    return mono_end(pb);
}

kfp_status kfp_monodomain_shard_copy(kfp_problem pb, int32_t what, int32_t dir, int32_t r0, int32_t r1, int32_t xa,
                                     int32_t xb, double *buf) {
    if (!pb || !buf || (what != 0 && what != 1) || (dir != 0 && dir != 1)) {
        set_err("kfp_monodomain_shard_copy: bad arguments");
        return KFP_E_INVAL;
    }
    if (!pb->mono_done || (what == 1 && !pb->d_Ulines)) {
        set_err("kfp_monodomain_shard_copy: no reference (or no recorded lines)");
        return KFP_E_STATE;
    }
    const int rows = what == 0 ? pb->nv + 1 : (int)pb->mono_lines.size() * pb->nt;
    if (r0 < 0 || r1 > rows || r0 > r1 || xa < 0 || xb > pb->nx || xa > xb) {
        set_err("kfp_monodomain_shard_copy: rows [%d, %d) of %d / columns [%d, %d) of %d", r0, r1, rows, xa, xb, pb->nx);
        return KFP_E_INVAL;
    }
    if (r0 == r1 || xa == xb) return KFP_OK;
    KFP_CUDA(cudaSetDevice(pb->device));
    double *base = (what == 0 ? pb->d_UT : pb->d_Ulines) + (size_t)r0 * pb->nx + xa;
    const size_t w = (size_t)(xb - xa) * sizeof(double), pitch = (size_t)pb->nx * sizeof(double);
    if (dir == 0)
        KFP_CUDA(cudaMemcpy2DAsync(buf, w, base, pitch, w, r1 - r0, cudaMemcpyDefault, pb->stream));
    else
        KFP_CUDA(cudaMemcpy2DAsync(base, pitch, buf, w, w, r1 - r0, cudaMemcpyDefault, pb->stream));
    return KFP_OK;
}

kfp_status kfp_monodomain_uT(kfp_problem pb, double *out) {
    if (!pb || !out) {
        set_err("kfp_monodomain_uT: NULL argument");
        return KFP_E_INVAL;
    }
    if (!pb->mono_done) {
        set_err("kfp_monodomain_uT: no monodomain solve yet");
        return KFP_E_STATE;
    }
    return kfp_monodomain_solve(pb, out);
}

kfp_status kfp_swr_setup(kfp_problem pb, kfp_kind kind, double p, int32_t overlap, int32_t n_sub, int32_t s_begin,
                         int32_t s_end, int32_t K_max) {
    return kfp_swr_setup_pq(pb, kind, p, p, overlap, n_sub, s_begin, s_end, K_max);
}

}  // extern "C"

namespace {
// Setup of n_rep independent replicas of the decomposition (replica r: OSWR(ps[r], qs[r])); n_rep = 1 is
// the ordinary solve (kfp_swr_setup_pq), n_rep > 1 the batched parameter sweep (kfp_swr_setup_batch).
kfp_status swr_setup_impl(kfp_problem pb, kfp_kind kind, const double *ps, const double *qs, int n_rep,
                          int32_t overlap, int32_t n_sub, int32_t s_begin, int32_t s_end, int32_t K_max) {
    const double p = ps[0], q = qs[0];
    if (!pb) {
        set_err("kfp_swr_setup: NULL problem");
        return KFP_E_INVAL;
    }
    if (kind != KFP_DIRICHLET && kind != KFP_ROBIN) {
        set_err("kfp_swr_setup: unknown kind %d", (int)kind);
        return KFP_E_INVAL;
    }
    for (int r = 0; r < n_rep; ++r)
        if (kind == KFP_ROBIN && !(ps[r] > 0 && qs[r] > 0)) {
            set_err("kfp_swr_setup: Robin parameters p, q must be > 0 (P:58), got %g, %g", ps[r], qs[r]);
            return KFP_E_INVAL;
        }
    (void)p;
    (void)q;
    if (n_sub < 1 || pb->nv % n_sub != 0) {
        set_err("kfp_swr_setup: n_sub=%d must divide nv=%d", n_sub, pb->nv);
        return KFP_E_INVAL;
    }
    const int cells = pb->nv / n_sub;
    if (overlap < 0 || (n_sub > 1 && overlap >= cells - 2)) {
        set_err("kfp_swr_setup: overlap=%d must satisfy 0 <= overlap < nv/n_sub - 2 = %d", overlap, cells - 2);
        return KFP_E_INVAL;
    }
    if (s_begin < 0 || s_end > n_sub || s_begin >= s_end) {
        set_err("kfp_swr_setup: bad local block [%d,%d) of %d subdomains", s_begin, s_end, n_sub);
        return KFP_E_INVAL;
    }
    if (K_max < 1) {
        set_err("kfp_swr_setup: K_max must be >= 1 (SPEC S:214)");
        return KFP_E_INVAL;
    }
    if (n_rep < 1 || (n_rep > 1 && (s_begin != 0 || s_end != n_sub))) {
        set_err("kfp_swr_setup: a batch of %d replicas needs every subdomain on this process", n_rep);
        return KFP_E_INVAL;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    free_swr(pb);
    std::string warn;
    if (kind == KFP_DIRICHLET && overlap == 0 && n_sub > 1)
        warn = "warning: Dirichlet transmission without overlap does not converge (P:661)";

    pb->kind = kind;
    pb->gauss_seidel = false;
    pb->ovrec = false;
    pb->d_pairs = nullptr;
    pb->npairs = 0;
    pb->n_rep = n_rep;
    pb->p = ps[0];
    pb->q_rob = (kind == KFP_ROBIN) ? qs[0] : ps[0];
    pb->ov = overlap;
    pb->S = n_sub;
    pb->s_begin = s_begin;
    pb->s_end = s_end;
    pb->K_max = K_max;
    pb->k_done = 0;
    decompose(pb->nv, n_sub, overlap, pb->lo, pb->hi);

    // interface lines needed by the local block
    std::vector<int> lines;
    for (int s = s_begin; s < s_end; ++s) {
        if (s > 0) lines.push_back(pb->lo[s]);
        if (s < n_sub - 1) lines.push_back(pb->hi[s]);
    }
    std::sort(lines.begin(), lines.end());
    lines.erase(std::unique(lines.begin(), lines.end()), lines.end());
    bool have = pb->mono_done;
    for (int l : lines)
        if (std::find(pb->mono_lines.begin(), pb->mono_lines.end(), l) == pb->mono_lines.end()) have = false;
    if (!have) {
        std::vector<int> all = pb->mono_lines;
        all.insert(all.end(), lines.begin(), lines.end());
        std::sort(all.begin(), all.end());
        all.erase(std::unique(all.begin(), all.end()), all.end());
        if (kfp_status st = run_monodomain(pb, all)) return st;
    }
    auto line_index = [&](int node) {
        auto it = std::find(pb->mono_lines.begin(), pb->mono_lines.end(), node);
        return (int)(it - pb->mono_lines.begin());
    };

    const int et = (kind == KFP_ROBIN) ? kfp::END_ROBIN : kfp::END_DIRI;
    const int nloc = s_end - s_begin;
    const size_t nx = pb->nx, TR = (size_t)pb->nt * nx;
    int n_max = 0;
    const int ntot = n_rep * nloc;  // all subdomains of all replicas (replica-major)
    pb->subs.resize(ntot);
    for (int ii = 0; ii < ntot; ++ii) {
        const int rr = ii / nloc, i = ii - rr * nloc, s = s_begin + i;
        SubDev &sd = pb->subs[ii];
        std::memset(&sd, 0, sizeof sd);
        sd.lo = pb->lo[s];
        sd.hi = pb->hi[s];
        const int phys = (pb->scheme == KFP_SCHEME_SPLIT_FEM) ? kfp::END_NEU : kfp::END_PHYS;
        sd.ltype = (s == 0) ? phys : et;
        sd.rtype = (s == n_sub - 1) ? phys : et;
        sd.first = (sd.ltype == kfp::END_ROBIN || sd.ltype == kfp::END_NEU) ? sd.lo : sd.lo + 1;
        const int last = (sd.rtype == kfp::END_ROBIN || sd.rtype == kfp::END_NEU) ? sd.hi : sd.hi - 1;
        sd.n = last - sd.first + 1;
        // unknown-row index of the node whose trace is sent left / right; -2 = none.
        // Dirichlet without overlap sends its own end node (index -1 / n): the received value.
        sd.iL_tr = (s > 0) ? pb->hi[s - 1] - sd.first : -2;
        sd.iR_tr = (s < n_sub - 1) ? pb->lo[s + 1] - sd.first : -2;
        sd.ifL = (s > 0) ? line_index(sd.lo) : -1;
        sd.ifR = (s < n_sub - 1) ? line_index(sd.hi) : -1;
        sd.injL = (sd.ltype == kfp::END_ROBIN) ? 2.0 * pb->ar * pb->hv : (sd.ltype == kfp::END_DIRI) ? pb->a : 0.0;
        sd.injR = (sd.rtype == kfp::END_ROBIN) ? 2.0 * pb->ar * pb->hv : (sd.rtype == kfp::END_DIRI) ? pb->a : 0.0;
        if (sd.n < 2) {
            set_err("kfp_swr_setup: subdomain %d has %d unknown rows (need >= 2)", s, sd.n);
            return KFP_E_INVAL;
        }
        sd.grp = rr;
        sd.tpL = ps[rr];                                   // sent left: lands on a right end (p)
        sd.tpR = (kind == KFP_ROBIN) ? qs[rr] : ps[rr];    // sent right: lands on a left end (q)
        woodbury(pb, sd, (kind == KFP_ROBIN) ? qs[rr] : ps[rr], ps[rr]);
        n_max = std::max(n_max, sd.n);
    }
    std::vector<int> ns;
    for (const SubDev &sd : pb->subs) ns.push_back(sd.n);
    const bool fem = pb->scheme == KFP_SCHEME_SPLIT_FEM;
    pb->plan = make_plan(ns, pb->f_rank, true, fem);
    Plan &pl = pb->plan;
    if (fem && !pl.fused) {
        set_err("kfp_swr_setup: the split-FEM scheme needs the cluster kernel (column of %d rows > %d)", n_max,
                8 * 16 * 33);
        return KFP_E_INVAL;
    }
    // the rows of each outgoing trace stencil must sit in one row block
    for (int ii = 0; ii < ntot; ++ii) {
        const int i = ii % nloc;
        SubDev &sd = pb->subs[ii];
        sd.nblk = (sd.n + pl.R - 1) / pl.R;
        auto same = [&](int r1, int r2) { return r1 / pl.R == r2 / pl.R; };
        const bool rob = (kind == KFP_ROBIN);
        bool bad = false;
        if (sd.iL_tr != -2) bad |= rob ? (sd.iL_tr < 0 || sd.iL_tr + 1 >= sd.n || !same(sd.iL_tr, sd.iL_tr + 1))
                                       : (sd.iL_tr < -1 || sd.iL_tr >= sd.n);
        if (sd.iR_tr != -2) bad |= rob ? (sd.iR_tr - 1 < 0 || sd.iR_tr >= sd.n || !same(sd.iR_tr, sd.iR_tr - 1))
                                       : (sd.iR_tr < 0 || sd.iR_tr > sd.n);
        if (bad) {
            set_err("kfp_swr_setup: trace stencil of subdomain %d straddles a row block (overlap too large for R=%d)",
                    s_begin + i, pl.R);
            return KFP_E_INVAL;
        }
    }
    if (kfp_status st = ensure_qtab(pb, std::max(pl.R, n_max) + 2)) return st;
    if (kfp_status st = configure_kernels(pl)) return st;

    // slabs and traces (each replica its own chain of interfaces)
    for (int ii = 0; ii < ntot; ++ii) {
        SubDev &sd = pb->subs[ii];
        const size_t rows = (size_t)(sd.hi - sd.lo + 1);
        for (int q = 0; q < 2; ++q)
            if (kfp_status st = swr_alloc(pb, &sd.slab[q], rows * nx)) return st;
    }
    for (int rr = 0; rr < n_rep; ++rr) {
        std::vector<double *> toL(2 * std::max(0, nloc - 1)), toR(2 * std::max(0, nloc - 1));
        for (int i = 0; i + 1 < nloc; ++i)
            for (int q = 0; q < 2; ++q) {
                if (kfp_status st = swr_alloc(pb, &toL[2 * i + q], TR)) return st;
                if (kfp_status st = swr_alloc(pb, &toR[2 * i + q], TR)) return st;
                if (q == 0) {
                    pb->zero_on_reset.push_back(toL[2 * i]);
                    pb->zero_on_reset.push_back(toR[2 * i]);
                }
            }
        for (int i = 0; i < nloc; ++i) {
            SubDev &sd = pb->subs[rr * nloc + i];
            for (int q = 0; q < 2; ++q) {
                if (i + 1 < nloc) {
                    sd.gR[q] = toL[2 * i + q];
                    sd.sendR[q] = toR[2 * i + q];
                }
                if (i > 0) {
                    sd.gL[q] = toR[2 * (i - 1) + q];
                    sd.sendL[q] = toL[2 * (i - 1) + q];
                }
            }
        }
    }
    // cross-block edges
    if (s_begin > 0)
        for (int q = 0; q < 2; ++q) {
            if (kfp_status st = swr_alloc(pb, &pb->edge_sendL[q], TR)) return st;
            if (kfp_status st = swr_alloc(pb, &pb->edge_recvL[q], TR)) return st;
            pb->subs[0].gL[q] = pb->edge_recvL[q];
            pb->subs[0].sendL[q] = pb->edge_sendL[q];
        }
    if (s_end < n_sub)
        for (int q = 0; q < 2; ++q) {
            if (kfp_status st = swr_alloc(pb, &pb->edge_sendR[q], TR)) return st;
            if (kfp_status st = swr_alloc(pb, &pb->edge_recvR[q], TR)) return st;
            pb->subs[nloc - 1].gR[q] = pb->edge_recvR[q];
            pb->subs[nloc - 1].sendR[q] = pb->edge_sendR[q];
        }
    {
        void *q = nullptr;
        KFP_CUDA(dev_malloc(&q, sizeof(SubDev) * ntot));
        pb->d_subs = static_cast<SubDev *>(q);
        KFP_CUDA(dev_malloc(&q, sizeof(unsigned long long) * K_max * n_rep));
        pb->d_errT = static_cast<unsigned long long *>(q);
        KFP_CUDA(dev_malloc(&q, sizeof(unsigned long long) * K_max * n_rep));
        pb->d_errIF = static_cast<unsigned long long *>(q);
        KFP_CUDA(dev_malloc(&q, sizeof(unsigned long long) * K_max * n_rep));
        pb->d_errOV = static_cast<unsigned long long *>(q);
        pb->swr_allocs.push_back(reinterpret_cast<double *>(pb->d_errOV));
    }
    KFP_CUDA(cudaMemcpy(pb->d_subs, pb->subs.data(), sizeof(SubDev) * ntot, cudaMemcpyHostToDevice));
    {
        std::vector<void *> own;
        kfp_status st = build_tmaps(pb, pl, pb->subs, &pb->fd.maps, &own);
        if (!st) st = build_l2m(pb, pl, pb->subs, &pb->fd.l2c, &own);
        if (!st) st = build_fused_tables(pb, pl, &pb->fv_host, &pb->fd.coefT, &pb->fd.tabs, &own);
        for (void *q : own) pb->swr_allocs.push_back(static_cast<double *>(q));
        if (st) return st;
    }
    if (kfp_status st = alloc_general_scratch(pb, pl, ntot, &pb->d_blkagg, &pb->d_chkagg, &pb->d_carry, pb->swr_allocs))
        return st;
    pb->setup = true;
    if (kfp_status st = kfp_swr_reset(pb)) return st;
    g_err = warn;
    return KFP_OK;
}
}  // namespace

extern "C" {

kfp_status kfp_swr_setup_pq(kfp_problem pb, kfp_kind kind, double p, double q, int32_t overlap, int32_t n_sub,
                            int32_t s_begin, int32_t s_end, int32_t K_max) {
    return swr_setup_impl(pb, kind, &p, &q, 1, overlap, n_sub, s_begin, s_end, K_max);
}

kfp_status kfp_swr_setup_batch(kfp_problem pb, kfp_kind kind, const double *ps, const double *qs, int32_t n_rep,
                               int32_t overlap, int32_t n_sub, int32_t K_max) {
    if (!ps || n_rep < 1) {
        set_err("kfp_swr_setup_batch: need n_rep >= 1 parameters");
        return KFP_E_INVAL;
    }
    return swr_setup_impl(pb, kind, ps, qs ? qs : ps, n_rep, overlap, n_sub, 0, n_sub, K_max);
}

kfp_status kfp_swr_batch_history(kfp_problem pb, int32_t rep, int32_t cap, int32_t *K_out, double *err_T,
                                 double *err_if) {
    if (!pb || !pb->setup || rep < 0 || rep >= pb->n_rep || pb->k_done == 0 || cap < pb->k_done) {
        set_err("kfp_swr_batch_history: bad replica, no iteration or cap < K");
        return pb && pb->setup && pb->k_done == 0 ? KFP_E_STATE : KFP_E_INVAL;
    }
    std::vector<unsigned long long> a(pb->k_done), b(pb->k_done);
    const size_t off = (size_t)rep * pb->K_max;
    KFP_CUDA(cudaMemcpyAsync(a.data(), pb->d_errT + off, sizeof(unsigned long long) * pb->k_done, cudaMemcpyDeviceToHost,
                             pb->stream));
    KFP_CUDA(cudaMemcpyAsync(b.data(), pb->d_errIF + off, sizeof(unsigned long long) * pb->k_done,
                             cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    for (int k = 0; k < pb->k_done; ++k) {
        std::memcpy(&err_T[k], &a[k], 8);
        std::memcpy(&err_if[k], &b[k], 8);
    }
    *K_out = pb->k_done;
    return KFP_OK;
}

kfp_status kfp_swr_batch_subdomain_uT(kfp_problem pb, int32_t rep, int32_t s, double *out) {
    if (!pb || !pb->setup || rep < 0 || rep >= pb->n_rep || s < 0 || s >= pb->S || !out) {
        set_err("kfp_swr_batch_subdomain_uT: bad replica/subdomain");
        return KFP_E_INVAL;
    }
    if (pb->s_begin != 0 || pb->s_end != pb->S) {  // replicas exist only for setups that hold every subdomain
        set_err("kfp_swr_batch_subdomain_uT: the setup holds subdomains [%d, %d) of %d, not a batch", pb->s_begin,
                pb->s_end, pb->S);
        return KFP_E_INVAL;
    }
    if (pb->k_done == 0) {
        set_err("kfp_swr_batch_subdomain_uT: no iteration since the setup / reset");
        return KFP_E_STATE;
    }
    const SubDev &sd = pb->subs[(size_t)rep * pb->S + s];
    KFP_CUDA(cudaMemcpyAsync(out, final_slab(pb, (size_t)rep * pb->S + s), sizeof(double) * (size_t)(sd.hi - sd.lo + 1) * pb->nx,
                             cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    return KFP_OK;
}

kfp_status kfp_swr_reset(kfp_problem pb) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_reset: no setup");
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    // chunked exchange of an earlier solve: the traces it received must have landed before they are zeroed
    for (int c = 0; c < pb->nchunks; ++c)
        if (pb->chunk_recv_set[c]) KFP_CUDA(cudaStreamWaitEvent(pb->stream, pb->chunk_recv[c], 0));
    std::fill(pb->chunk_recv_set.begin(), pb->chunk_recv_set.end(), 0);
    pb->chunk_next = 0;
    const size_t TR = (size_t)pb->nt * pb->nx;
    for (double *p : pb->zero_on_reset) KFP_CUDA(cudaMemsetAsync(p, 0, TR * sizeof(double), pb->stream));
    if (pb->edge_recvL[0]) KFP_CUDA(cudaMemsetAsync(pb->edge_recvL[0], 0, TR * sizeof(double), pb->stream));
    if (pb->edge_recvR[0]) KFP_CUDA(cudaMemsetAsync(pb->edge_recvR[0], 0, TR * sizeof(double), pb->stream));
    KFP_CUDA(cudaMemsetAsync(pb->d_errT, 0, sizeof(unsigned long long) * pb->K_max * pb->n_rep, pb->stream));
    KFP_CUDA(cudaMemsetAsync(pb->d_errIF, 0, sizeof(unsigned long long) * pb->K_max * pb->n_rep, pb->stream));
    KFP_CUDA(cudaMemsetAsync(pb->d_errOV, 0, sizeof(unsigned long long) * pb->K_max * pb->n_rep, pb->stream));
    pb->k_done = 0;
    return KFP_OK;
}

kfp_status kfp_swr_set_initial_trace(kfp_problem pb, int32_t i, int32_t dir, const double *host) {
    if (!pb || !pb->setup || i < pb->s_begin || i + 1 >= pb->s_end || dir < 0 || dir > 1 || !host || pb->k_done != 0) {
        set_err("kfp_swr_set_initial_trace: interface %d not local, bad dir, or not right after a reset", i);
        return KFP_E_INVAL;
    }
    const int nloc = pb->s_end - pb->s_begin;
    const size_t bytes = sizeof(double) * (size_t)pb->nt * pb->nx;
    for (int r = 0; r < pb->n_rep; ++r) {  // every replica of a batch starts from the same lambda^0
        const SubDev &left = pb->subs[(size_t)r * nloc + (i - pb->s_begin)];
        const SubDev &right = pb->subs[(size_t)r * nloc + (i + 1 - pb->s_begin)];
        double *dst = const_cast<double *>(dir == 0 ? left.gR[0] : right.gL[0]);
        KFP_CUDA(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, pb->stream));
    }
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    return KFP_OK;
}

kfp_status kfp_swr_set_schedule(kfp_problem pb, kfp_schedule schedule) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_set_schedule: no setup");
        return KFP_E_STATE;
    }
    if (schedule != KFP_JACOBI && schedule != KFP_GAUSS_SEIDEL) {
        set_err("kfp_swr_set_schedule: unknown schedule %d", (int)schedule);
        return KFP_E_INVAL;
    }
    if (schedule == KFP_GAUSS_SEIDEL && (pb->s_begin != 0 || pb->s_end != pb->S)) {
        set_err("kfp_swr_set_schedule: Gauss-Seidel needs every subdomain on this process and a per-step plan");
        return KFP_E_INVAL;
    }
    pb->gauss_seidel = (schedule == KFP_GAUSS_SEIDEL);
    return KFP_OK;
}

kfp_status kfp_swr_iterate(kfp_problem pb, int32_t n_iter) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_iterate: no setup");
        return KFP_E_STATE;
    }
    if (n_iter < 0 || pb->k_done + n_iter > pb->K_max) {
        set_err("kfp_swr_iterate: %d + %d iterations exceed K_max=%d", pb->k_done, n_iter, pb->K_max);
        return KFP_E_STATE;
    }
    if (pb->chunk_next != 0) {
        set_err("kfp_swr_iterate: a chunked iteration is in progress (next chunk %d of %d)", pb->chunk_next, pb->nchunks);
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    const int need = 2 + 2 * n_iter;
    while ((int)pb->ev.size() < need) {
        cudaEvent_t e;
        KFP_CUDA(cudaEventCreate(&e));
        pb->ev.push_back(e);
    }
    pb->ev_used = need;
    const int nloc = (int)pb->subs.size();
    StepParams P = base_params(pb);
    P.subs = pb->d_subs;
    P.send_robin = (pb->kind == KFP_ROBIN);
    P.p = pb->p;
    P.UT = pb->d_UT;
    P.Ulines = pb->d_Ulines;
    P.blkagg = pb->d_blkagg;
    P.chkagg = pb->d_chkagg;
    P.carry = pb->d_carry;
    P.ovrec = pb->ovrec ? 1 : 0;
    KFP_CUDA(cudaEventRecord(pb->ev[0], pb->stream));
    if (pb->pipe > 1) {
        // pipelined iterations: groups of up to D iterations in one sweep of launches.
        // Jacobi: slot d runs iteration k0 + d at step L - d, reading trace row L - d of iteration
        // k0 + d - 1 (written by slot d - 1 one launch earlier) from the ring.  Gauss-Seidel (SWR1-SWR4):
        // subdomain s of slot d lags 2 d + s steps -- its left trace (same iteration) was written by s - 1 one
        // launch earlier, its right trace (previous iteration) by s + 1 of slot d - 1 one launch earlier.
        const int D = pb->pipe, R = D + 1, ntot = nloc, nl = pb->s_end - pb->s_begin;
        const bool gs = pb->gauss_seidel;
        int it = 0, g = 0;
        while (it < n_iter) {
            const int G = std::min(D, n_iter - it), k0 = pb->k_done + 1;
            for (int d = 0; d < G; ++d) {
                const int k = k0 + d;
                for (int ii = 0; ii < ntot; ++ii) {
                    SubDev &sd = pb->psubs[(size_t)d * ntot + ii];
                    const int r = ii / nl, i = ii % nl;
                    sd.lag = gs ? 2 * d + i : d;
                    if (i > 0) {
                        sd.gL[0] = pb->ringR[(size_t)r * (nl - 1) + i - 1][(gs ? k : k - 1) % R];
                        sd.sendL[0] = pb->ringL[(size_t)r * (nl - 1) + i - 1][k % R];
                    }
                    if (i < nl - 1) {
                        sd.gR[0] = pb->ringL[(size_t)r * (nl - 1) + i][(k - 1) % R];
                        sd.sendR[0] = pb->ringR[(size_t)r * (nl - 1) + i][k % R];
                    }
                    sd.grp = r * pb->K_max + (k - 1);  // error slot (err_stride 1)
                }
            }
            KFP_CUDA(cudaMemcpyAsync(pb->d_psubs, pb->psubs.data(), sizeof(SubDev) * (size_t)G * ntot,
                                     cudaMemcpyHostToDevice, pb->stream));
            StepParams Pp = P;
            Pp.subs = pb->d_psubs;
            Pp.par_in = Pp.par_out = Pp.par_in_lo = 0;
            Pp.errT = pb->d_errT;
            Pp.errIF = pb->d_errIF;
            Pp.err_stride = 1;
            Pp.last = 1;  // errors at T on each slot's own last step
            KFP_CUDA(cudaEventRecord(pb->ev[2 + 2 * g], pb->stream));
            const int max_lag = gs ? 2 * (G - 1) + (nl - 1) : G - 1;
            for (int L = 0; L < pb->nt + max_lag; ++L)
                if (kfp_status st = launch_step(pb, pb->plan, Pp, G * ntot, L, pb->pfd, 0, nullptr, true)) return st;
            if (pb->scheme == KFP_SCHEME_SPLIT_FEM) {
                int rows = 0;
                for (const SubDev &sd : pb->subs) rows = std::max(rows, sd.hi - sd.lo + 1);
                if (kfp_status st = launch_fem_finish(pb, Pp, G * ntot, rows)) return st;
            }
            if (pb->ovrec && pb->npairs > 0) {  // err_ov of every iteration of the group (slot grp = its slot)
                kfp::overlap_diff<<<dim3(64, 1, G * pb->npairs), 256, 0, pb->stream>>>(pb->d_psubs, pb->d_ppairs, pb->nt,
                                                                                   pb->nx, pb->d_errOV, 1);
                pb->launches += 1;
                KFP_CUDA(cudaGetLastError());
            }
            KFP_CUDA(cudaEventRecord(pb->ev[3 + 2 * g], pb->stream));
            pb->final_slab.assign(ntot, nullptr);
            for (int ii = 0; ii < ntot; ++ii) pb->final_slab[ii] = pb->psubs[(size_t)(G - 1) * ntot + ii].slab[final_parity(pb)];
            KFP_CUDA(cudaStreamSynchronize(pb->stream));  // psubs is rewritten for the next group
            pb->k_done += G;
            it += G;
            ++g;
        }
        pb->ev_used = 2 + 2 * g;
        KFP_CUDA(cudaEventRecord(pb->ev[1], pb->stream));
        return KFP_OK;
    }
    for (int it = 0; it < n_iter; ++it) {
        const int k = pb->k_done + 1;  // 1-based iteration number
        P.par_in = (k - 1) & 1;
        P.par_out = k & 1;
        P.par_in_lo = pb->gauss_seidel ? P.par_out : P.par_in;
        P.errT = pb->d_errT + (k - 1);
        P.errIF = pb->d_errIF + (k - 1);
        P.err_stride = pb->K_max;  // replica r's slots: + r * K_max
        KFP_CUDA(cudaEventRecord(pb->ev[2 + 2 * it], pb->stream));
        if (pb->gauss_seidel) {
            // SWR1-SWR4: the subdomains in increasing v, each over the whole window, each
            // reading the trace its left neighbour wrote in this iteration (stream order)
            const Plan &pl = pb->plan;
            for (int s = 0; s < nloc; ++s) {
                StepParams Ps = P;
                Ps.subs = pb->d_subs + s;
                FusedData fs = pb->fd;  // the tables of subdomain s
                if (fs.maps) fs.maps += 2 * s;
                if (fs.l2c) fs.l2c += (size_t)s * pl.C * kfp::kL2M;
                for (int n = 0; n < pb->nt; ++n) {
                    Ps.last = (n + 1 == pb->nt);  // (the cluster kernel tests its own step; see StepParams)
                    if (kfp_status st = launch_step(pb, pl, Ps, 1, n, fs)) return st;
                }
            }
        } else {
            for (int n = 0; n < pb->nt; ++n) {
                P.last = (n + 1 == pb->nt);
                if (kfp_status st = launch_step(pb, pb->plan, P, nloc, n, pb->fd)) return st;
            }
        }
        if (pb->scheme == KFP_SCHEME_SPLIT_FEM) {  // u(T) = the last Step 2, and err_T
            int rows = 0;
            for (const SubDev &sd : pb->subs) rows = std::max(rows, sd.hi - sd.lo + 1);
            if (kfp_status st = launch_fem_finish(pb, P, nloc, rows)) return st;
        }
        if (pb->ovrec && pb->npairs > 0) {  // max |u_s - u_{s+1}| over every local overlap (eq. 'error')
            kfp::overlap_diff<<<dim3(64, 1, pb->npairs), 256, 0, pb->stream>>>(pb->d_subs, pb->d_pairs, pb->nt, pb->nx,
                                                                             pb->d_errOV + (k - 1), pb->K_max);
            pb->launches += 1;
            KFP_CUDA(cudaGetLastError());
        }
        KFP_CUDA(cudaEventRecord(pb->ev[3 + 2 * it], pb->stream));
        pb->k_done = k;
    }
    KFP_CUDA(cudaEventRecord(pb->ev[1], pb->stream));
    return KFP_OK;
}

kfp_status kfp_swr_iterate_chunk(kfp_problem pb, int32_t chunk, int32_t nchunks) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_iterate_chunk: no setup");
        return KFP_E_STATE;
    }
    if (nchunks < 1 || nchunks > pb->nt || chunk < 0 || chunk >= nchunks) {
        set_err("kfp_swr_iterate_chunk: chunk %d of %d (need 0 <= chunk < nchunks <= nt=%d)", chunk, nchunks, pb->nt);
        return KFP_E_INVAL;
    }
    if (pb->pipe > 1 || pb->gauss_seidel) {
        set_err("kfp_swr_iterate_chunk: needs the unpipelined Jacobi schedule");
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    if (nchunks != pb->nchunks) {  // (re)create the chunk events
        if (pb->chunk_next != 0) {
            set_err("kfp_swr_iterate_chunk: the iteration in progress has %d chunks", pb->nchunks);
            return KFP_E_STATE;
        }
        for (cudaEvent_t e : pb->chunk_sent) cudaEventDestroy(e);
        for (cudaEvent_t e : pb->chunk_recv) cudaEventDestroy(e);
        pb->chunk_sent.assign(nchunks, nullptr);
        pb->chunk_recv.assign(nchunks, nullptr);
        pb->chunk_recv_set.assign(nchunks, 0);
        for (int c = 0; c < nchunks; ++c) {
            KFP_CUDA(cudaEventCreateWithFlags(&pb->chunk_sent[c], cudaEventDisableTiming));
            KFP_CUDA(cudaEventCreateWithFlags(&pb->chunk_recv[c], cudaEventDisableTiming));
        }
        pb->nchunks = nchunks;
    }
    if (chunk != pb->chunk_next) {
        set_err("kfp_swr_iterate_chunk: expected chunk %d, got %d", pb->chunk_next, chunk);
        return KFP_E_STATE;
    }
    if (chunk == 0 && pb->k_done + 1 > pb->K_max) {
        set_err("kfp_swr_iterate_chunk: %d iterations exceed K_max=%d", pb->k_done + 1, pb->K_max);
        return KFP_E_STATE;
    }
    const int k = pb->k_done + 1;
    StepParams P = base_params(pb);
    P.subs = pb->d_subs;
    P.send_robin = (pb->kind == KFP_ROBIN);
    P.p = pb->p;
    P.UT = pb->d_UT;
    P.Ulines = pb->d_Ulines;
    P.blkagg = pb->d_blkagg;
    P.chkagg = pb->d_chkagg;
    P.carry = pb->d_carry;
    P.ovrec = pb->ovrec ? 1 : 0;
    P.par_in = P.par_in_lo = (k - 1) & 1;
    P.par_out = k & 1;
    P.errT = pb->d_errT + (k - 1);
    P.errIF = pb->d_errIF + (k - 1);
    P.err_stride = pb->K_max;
    // the incoming edge rows of this chunk (the previous iteration's) must have arrived
    if (pb->chunk_recv_set[chunk]) KFP_CUDA(cudaStreamWaitEvent(pb->stream, pb->chunk_recv[chunk], 0));
    const int nloc = (int)pb->subs.size();
    const int n0 = (int)((int64_t)chunk * pb->nt / nchunks), n1 = (int)((int64_t)(chunk + 1) * pb->nt / nchunks);
    for (int n = n0; n < n1; ++n) {
        P.last = (n + 1 == pb->nt);
        if (kfp_status st = launch_step(pb, pb->plan, P, nloc, n, pb->fd)) return st;
    }
    KFP_CUDA(cudaEventRecord(pb->chunk_sent[chunk], pb->stream));  // outgoing rows [n0, n1) written
    if (chunk + 1 == nchunks) {
        if (pb->scheme == KFP_SCHEME_SPLIT_FEM) {
            int rows = 0;
            for (const SubDev &sd : pb->subs) rows = std::max(rows, sd.hi - sd.lo + 1);
            if (kfp_status st = launch_fem_finish(pb, P, nloc, rows)) return st;
        }
        if (pb->ovrec && pb->npairs > 0) {
            kfp::overlap_diff<<<dim3(64, 1, pb->npairs), 256, 0, pb->stream>>>(pb->d_subs, pb->d_pairs, pb->nt, pb->nx,
                                                                             pb->d_errOV + (k - 1), pb->K_max);
            pb->launches += 1;
            KFP_CUDA(cudaGetLastError());
        }
        pb->k_done = k;
        pb->chunk_next = 0;
    } else {
        pb->chunk_next = chunk + 1;
    }
    return KFP_OK;
}

kfp_status kfp_swr_chunk_send_wait(kfp_problem pb, void *stream, int32_t chunk) {
    if (!pb || !pb->setup || chunk < 0 || chunk >= pb->nchunks) {
        set_err("kfp_swr_chunk_send_wait: no chunked iteration or bad chunk %d", chunk);
        return KFP_E_INVAL;
    }
    KFP_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), pb->chunk_sent[chunk], 0));
    return KFP_OK;
}

kfp_status kfp_swr_chunk_recv_done(kfp_problem pb, void *stream, int32_t chunk) {
    if (!pb || !pb->setup || chunk < 0 || chunk >= pb->nchunks) {
        set_err("kfp_swr_chunk_recv_done: no chunked iteration or bad chunk %d", chunk);
        return KFP_E_INVAL;
    }
    KFP_CUDA(cudaEventRecord(pb->chunk_recv[chunk], static_cast<cudaStream_t>(stream)));
    pb->chunk_recv_set[chunk] = 1;
    return KFP_OK;
}

// Automatic depth (kfp_swr_set_pipeline(pb, 0)): latency-bound problems -- one step launch occupies at most
// half of the co-resident cluster slots, e.g. the small windows of BASELINE configs[0] and [1] -- get up to
// min(K_max, 16) iterations per sweep; a problem that fills the GPU keeps 1.
static int auto_pipeline_depth(kfp_problem pb) {
    const Plan &pl = pb->plan;
    if (!pl.fused || pb->ovrec) return 1;
    const int nsub = std::max(1, (int)pb->subs.size());
    const int ntiles = (pb->nx + kfp::kWarp - 1) / kfp::kWarp;
    const int per_launch = std::max(1, std::min(ntiles, pl.Gc_total / nsub)) * nsub;  // clusters of one step
    return std::max(1, std::min({pb->K_max, 16, pl.Gc_total / per_launch}));
}

kfp_status kfp_swr_set_pipeline(kfp_problem pb, int32_t depth) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_set_pipeline: no setup");
        return KFP_E_STATE;
    }
    if (depth == 0) {
        if (pb->k_done != 0 || pb->pipe != 1) return KFP_OK;  // automatic: only on a fresh unpipelined setup
        depth = auto_pipeline_depth(pb);
        if (depth < 2) return KFP_OK;
    }
    if (depth < 1 || depth > 64) {
        set_err("kfp_swr_set_pipeline: depth %d outside [1, 64]", depth);
        return KFP_E_INVAL;
    }
    if (pb->k_done != 0) {
        set_err("kfp_swr_set_pipeline: call right after setup / reset");
        return KFP_E_STATE;
    }
    if (depth == pb->pipe) return KFP_OK;
    const Plan &pl = pb->plan;
    if (depth > 1 && (pb->s_begin != 0 || pb->s_end != pb->S || !pl.fused || pb->pipe != 1)) {
        set_err("kfp_swr_set_pipeline: needs every subdomain on this process, the per-step cluster kernel and a "
                "fresh setup (plan: %s)", pl.text.c_str());
        return KFP_E_INVAL;
    }
    if (depth == 1) {
        set_err("kfp_swr_set_pipeline: a pipelined setup cannot go back to depth 1; set it up again");
        return KFP_E_INVAL;
    }
    // everything below is built on copies and committed only at the end: a failed call leaves the
    // problem as it was (include/kfp.h: state unchanged on error)
    Plan npl = pb->plan;
    if (npl.NR == 1) npl.NR = 2;  // no pipelined NR = 1 variants: same table rows, zero 2nd coefficient
    {
        FusedKernel k;
        size_t smem = 0;
        if (!fused_kernel(npl.B, npl.NR, npl.P, &k, &smem, npl.fem, true)) {
            set_err("kfp_swr_set_pipeline: no pipelined kernel variant for this plan (%s)", npl.text.c_str());
            return KFP_E_INVAL;
        }
        KFP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    const int D = depth, R = D + 1, ntot = (int)pb->subs.size(), nl = pb->s_end - pb->s_begin;
    const size_t nx = pb->nx, TR = (size_t)pb->nt * nx;
    std::vector<double *> fresh;  // this call's allocations (freed if it fails)
    auto al = [&](double **p, size_t count) -> kfp_status {
        void *q = nullptr;
        if (dev_malloc(&q, std::max<size_t>(count, 1) * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            set_err("kfp_swr_set_pipeline: device allocation of %zu doubles failed", count);
            return KFP_E_NOMEM;
        }
        fresh.push_back(static_cast<double *>(q));
        *p = static_cast<double *>(q);
        return KFP_OK;
    };
    auto fail = [&](kfp_status st) {
        for (double *p : fresh) dev_free(p);
        return st;
    };
    // trace rings: slots 0 and 1 are the setup's parity buffers (slot 0 is what reset / set_initial_trace write)
    std::vector<std::vector<double *>> ringL((size_t)pb->n_rep * (nl - 1), std::vector<double *>(R, nullptr));
    std::vector<std::vector<double *>> ringR = ringL;
    for (int r = 0; r < pb->n_rep; ++r)
        for (int i = 0; i + 1 < nl; ++i) {
            const SubDev &left = pb->subs[(size_t)r * nl + i];
            auto &rl = ringL[(size_t)r * (nl - 1) + i], &rr = ringR[(size_t)r * (nl - 1) + i];
            for (int q = 0; q < 2; ++q) {
                rl[q] = const_cast<double *>(left.gR[q]);
                rr[q] = left.sendR[q];
            }
            for (int q = 2; q < R; ++q) {
                if (kfp_status st = al(&rl[q], TR)) return fail(st);
                if (kfp_status st = al(&rr[q], TR)) return fail(st);
            }
        }
    // slot descriptors: slot 0 = the setup's subdomains; slots d > 0 get their own slabs
    std::vector<SubDev> psubs((size_t)D * ntot, SubDev());
    for (int d = 0; d < D; ++d)
        for (int ii = 0; ii < ntot; ++ii) {
            SubDev sd = pb->subs[ii];
            sd.lag = d;
            if (d > 0) {
                for (int q = 0; q < 2; ++q)
                    if (kfp_status st = al(&sd.slab[q], (size_t)(sd.hi - sd.lo + 1) * nx)) return fail(st);
                for (int side = 0; side < 2; ++side)  // overlap records of this slot (recording on)
                    if (sd.ovn[side] > 0)
                        if (kfp_status st = al(&sd.ovb[side], (size_t)sd.ovn[side] * TR)) return fail(st);
            }
            psubs[(size_t)d * ntot + ii] = sd;
        }
    int2 *d_ppairs = nullptr;
    if (pb->ovrec && pb->npairs > 0) {  // the overlap pairs of every slot, slot-major
        std::vector<int2> pp;
        for (int d = 0; d < D; ++d)
            for (int r = 0; r < pb->n_rep; ++r)
                for (int i = 0; i + 1 < nl; ++i)
                    pp.push_back(make_int2(d * ntot + r * nl + i, d * ntot + r * nl + i + 1));
        double *q = nullptr;
        if (kfp_status st = al(&q, (sizeof(int2) * pp.size() + 7) / 8)) return fail(st);
        d_ppairs = reinterpret_cast<int2 *>(q);
        if (cudaMemcpy(d_ppairs, pp.data(), sizeof(int2) * pp.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return fail(KFP_E_CUDA);
    }
    FusedData pfd;
    double *d_psubs_raw = nullptr;
    if (kfp_status st = al(&d_psubs_raw, (sizeof(SubDev) * psubs.size() + 7) / 8)) return fail(st);
    {
        std::vector<void *> own;
        kfp_status st = build_tmaps(pb, npl, psubs, &pfd.maps, &own);
        if (!st) st = build_l2m(pb, npl, psubs, &pfd.l2c, &own);
        for (void *o : own) fresh.push_back(static_cast<double *>(o));
        if (st) return fail(st);
        pfd.coefT = pb->fd.coefT;
        pfd.tabs = pb->fd.tabs;
    }
    // commit
    pb->plan.NR = npl.NR;
    pb->ringL = std::move(ringL);
    pb->ringR = std::move(ringR);
    pb->psubs = std::move(psubs);
    pb->d_psubs = reinterpret_cast<SubDev *>(d_psubs_raw);
    if (d_ppairs) pb->d_ppairs = d_ppairs;
    pb->pfd = pfd;
    pb->swr_allocs.insert(pb->swr_allocs.end(), fresh.begin(), fresh.end());
    pb->pipe = D;
    return KFP_OK;
}

kfp_status kfp_swr_set_overlap_error(kfp_problem pb, int32_t on) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_set_overlap_error: no setup");
        return KFP_E_STATE;
    }
    const Plan &pl = pb->plan;
    if (on && pb->pipe > 1 && !pb->ovrec) {
        set_err("kfp_swr_set_overlap_error: turn the recording on before kfp_swr_set_pipeline");
        return KFP_E_STATE;
    }
    if (on && (!pl.fused)) {
        set_err("kfp_swr_set_overlap_error: needs the per-step cluster kernel (plan: %s)", pl.text.c_str());
        return KFP_E_INVAL;
    }
    if (!on || pb->ov_alloc) {  // off, or back on with the buffers of an earlier call
        pb->ovrec = on != 0;
        return KFP_OK;
    }
    KFP_CUDA(cudaSetDevice(pb->device));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    const int nloc = pb->s_end - pb->s_begin;
    const size_t TR = (size_t)pb->nt * pb->nx;
    std::vector<int2> pairs;
    for (int r = 0; r < pb->n_rep; ++r)
        for (int i = 0; i + 1 < nloc; ++i) {  // interface between local subdomains i and i+1 of replica r
            SubDev &L = pb->subs[(size_t)r * nloc + i], &R = pb->subs[(size_t)r * nloc + i + 1];
            const int a = R.lo, b = L.hi, cnt = b - a + 1;  // the closed overlap [lo_{s+1}, hi_s]
            L.ovr0[1] = R.ovr0[0] = a;
            L.ovn[1] = R.ovn[0] = cnt;
            if (kfp_status st = swr_alloc(pb, &L.ovb[1], (size_t)cnt * TR)) return st;
            if (kfp_status st = swr_alloc(pb, &R.ovb[0], (size_t)cnt * TR)) return st;
            pairs.push_back(make_int2(r * nloc + i, r * nloc + i + 1));
        }
    if (!pairs.empty()) {
        void *q = nullptr;
        KFP_CUDA(dev_malloc(&q, sizeof(int2) * pairs.size()));
        pb->d_pairs = static_cast<int2 *>(q);
        pb->swr_allocs.push_back(static_cast<double *>(q));
        KFP_CUDA(cudaMemcpy(pb->d_pairs, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice));
    }
    pb->npairs = (int)pairs.size();
    KFP_CUDA(cudaMemcpy(pb->d_subs, pb->subs.data(), sizeof(SubDev) * pb->subs.size(), cudaMemcpyHostToDevice));
    pb->ovrec = true;
    pb->ov_alloc = true;
    return KFP_OK;
}

kfp_status kfp_swr_overlap_history(kfp_problem pb, int32_t rep, int32_t cap, int32_t *K_out, double *err_ov) {
    if (!pb || !pb->setup || rep < 0 || rep >= pb->n_rep) {
        set_err("kfp_swr_overlap_history: no setup or bad replica");
        return KFP_E_INVAL;
    }
    if (!pb->ovrec || pb->k_done == 0) {
        set_err("kfp_swr_overlap_history: overlap recording off or no iteration");
        return KFP_E_STATE;
    }
    std::vector<unsigned long long> a(pb->k_done);
    KFP_CUDA(cudaMemcpyAsync(a.data(), pb->d_errOV + (size_t)rep * pb->K_max, sizeof(unsigned long long) * pb->k_done,
                             cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    if (K_out) *K_out = pb->k_done;
    for (int k = 0; k < std::min<int>(cap, pb->k_done); ++k) std::memcpy(&err_ov[k], &a[k], 8);
    return KFP_OK;
}

kfp_status kfp_swr_iterate_until(kfp_problem pb, kfp_metric metric, double eps, int32_t k_max, int32_t *k_out) {
    if (!pb || !pb->setup) {
        set_err("kfp_swr_iterate_until: no setup");
        return KFP_E_STATE;
    }
    if (metric != KFP_ERR_T && metric != KFP_ERR_IF && metric != KFP_ERR_OVERLAP) {
        set_err("kfp_swr_iterate_until: unknown metric %d", (int)metric);
        return KFP_E_INVAL;
    }
    if (metric == KFP_ERR_OVERLAP && !pb->ovrec) {
        set_err("kfp_swr_iterate_until: KFP_ERR_OVERLAP needs kfp_swr_set_overlap_error(pb, 1)");
        return KFP_E_STATE;
    }
    if (k_max < 0 || pb->k_done + k_max > pb->K_max) {
        set_err("kfp_swr_iterate_until: %d + %d iterations exceed K_max=%d", pb->k_done, k_max, pb->K_max);
        return KFP_E_STATE;
    }
    const unsigned long long *hist = metric == KFP_ERR_T ? pb->d_errT : metric == KFP_ERR_IF ? pb->d_errIF : pb->d_errOV;
    // pipelined: whole groups of up to `pipe` iterations, then the first of them that met the tolerance
    const int step_iters = std::max(1, pb->pipe);
    int done = 0, hit = -1;
    bool bad = false;
    while (done < k_max && hit < 0) {
        const int n = std::min(step_iters, k_max - done), k0 = pb->k_done;
        if (kfp_status st = kfp_swr_iterate(pb, n)) return st;
        std::vector<unsigned long long> bits(n);  // replica 0 (the batch's first replica)
        KFP_CUDA(cudaMemcpyAsync(bits.data(), hist + k0, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost,
                                 pb->stream));
        KFP_CUDA(cudaStreamSynchronize(pb->stream));
        for (int i = 0; i < n && hit < 0; ++i) {
            double e;
            std::memcpy(&e, &bits[i], 8);
            if (!std::isfinite(e)) {  // the solve blew up (failure detection)
                hit = k0 + i + 1;
                bad = true;
            } else if (e < eps) {
                hit = k0 + i + 1;
            }
        }
        done += n;
    }
    if (k_out) *k_out = hit > 0 ? hit : pb->k_done;
    if (bad) {
        set_err("kfp_swr_iterate_until: iteration %d has a non-finite error", hit);
        return KFP_E_NONFINITE;
    }
    return KFP_OK;
}

kfp_status kfp_last_timing(kfp_problem pb, double *iterate_ms, double *kernel_ms) {
    if (!pb || pb->ev_used < 2) {
        set_err("kfp_last_timing: nothing timed yet");
        return KFP_E_STATE;
    }
    KFP_CUDA(cudaEventSynchronize(pb->ev[1]));
    float ms = 0;
    KFP_CUDA(cudaEventElapsedTime(&ms, pb->ev[0], pb->ev[1]));
    if (iterate_ms) *iterate_ms = ms;
    if (kernel_ms) {
        double tot = 0;
        for (int i = 2; i + 1 < pb->ev_used; i += 2) {
            KFP_CUDA(cudaEventElapsedTime(&ms, pb->ev[i], pb->ev[i + 1]));
            tot += ms;
        }
        *kernel_ms = tot;
    }
    return KFP_OK;
}

kfp_status kfp_swr_edge_buffers(kfp_problem pb, int32_t parity, double **send_left, double **recv_left,
                                double **send_right, double **recv_right) {
    if (!pb || !pb->setup || parity < 0 || parity > 1) {
        set_err("kfp_swr_edge_buffers: no setup or bad parity");
        return KFP_E_STATE;
    }
    if (send_left) *send_left = pb->edge_sendL[parity];
    if (recv_left) *recv_left = pb->edge_recvL[parity];
    if (send_right) *send_right = pb->edge_sendR[parity];
    if (recv_right) *recv_right = pb->edge_recvR[parity];
    return KFP_OK;
}

kfp_status kfp_swr_bind_edge_buffers(kfp_problem pb, int32_t parity, double *send_left, double *recv_left,
                                     double *send_right, double *recv_right) {
    if (!pb || !pb->setup || parity < 0 || parity > 1) {
        set_err("kfp_swr_bind_edge_buffers: no setup or bad parity");
        return KFP_E_STATE;
    }
    const bool hasL = pb->s_begin > 0, hasR = pb->s_end < pb->S;
    if ((!hasL && (send_left || recv_left)) || (!hasR && (send_right || recv_right))) {
        set_err("kfp_swr_bind_edge_buffers: buffer given for a side without a neighbour block");
        return KFP_E_INVAL;
    }
    const int nloc = (int)pb->subs.size();
    if (send_left) pb->edge_sendL[parity] = pb->subs[0].sendL[parity] = send_left;
    if (recv_left) pb->edge_recvL[parity] = recv_left, pb->subs[0].gL[parity] = recv_left;
    if (send_right) pb->edge_sendR[parity] = pb->subs[nloc - 1].sendR[parity] = send_right;
    if (recv_right) pb->edge_recvR[parity] = recv_right, pb->subs[nloc - 1].gR[parity] = recv_right;
    KFP_CUDA(cudaMemcpyAsync(pb->d_subs, pb->subs.data(), sizeof(SubDev) * nloc, cudaMemcpyHostToDevice, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    if (parity == 0) return kfp_swr_reset(pb);
    return KFP_OK;
}

kfp_status kfp_swr_solve(kfp_problem pb, kfp_kind kind, double p, int32_t overlap, int32_t n_sub, int32_t K,
                         double *uT) {
    return kfp_swr_solve_pq(pb, kind, p, p, overlap, n_sub, K, uT);
}

kfp_status kfp_swr_solve_pq(kfp_problem pb, kfp_kind kind, double p, double q, int32_t overlap, int32_t n_sub,
                            int32_t K, double *uT) {
    if (kfp_status st = kfp_swr_setup_pq(pb, kind, p, q, overlap, n_sub, 0, n_sub, K)) return st;
    std::string warn = g_err;
    kfp_swr_set_pipeline(pb, 0);  // latency-bound problems: pipelined iterations (on failure: unchanged)
    if (kfp_status st = kfp_swr_iterate(pb, K)) return st;
    if (uT) {
        const size_t nx = pb->nx;
        for (int s = 0; s < n_sub; ++s) {
            const SubDev &sd = pb->subs[s];
            const int c0 = s * (pb->nv / n_sub);
            const int c1 = (s == n_sub - 1) ? pb->nv : (s + 1) * (pb->nv / n_sub) - 1;
            KFP_CUDA(cudaMemcpyAsync(uT + (size_t)c0 * nx, final_slab(pb, s) + (size_t)(c0 - sd.lo) * nx,
                                     sizeof(double) * (size_t)(c1 - c0 + 1) * nx, cudaMemcpyDeviceToHost, pb->stream));
        }
    }
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    g_err = warn;
    return KFP_OK;
}

kfp_status kfp_error_history(kfp_problem pb, int32_t cap, int32_t *K_out, double *err_T, double *err_if) {
    if (!pb || !pb->setup || pb->k_done == 0) {
        set_err("kfp_error_history: no iteration has run");
        return KFP_E_STATE;
    }
    std::vector<unsigned long long> a(pb->k_done), b(pb->k_done);
    KFP_CUDA(cudaMemcpyAsync(a.data(), pb->d_errT, sizeof(unsigned long long) * pb->k_done, cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaMemcpyAsync(b.data(), pb->d_errIF, sizeof(unsigned long long) * pb->k_done, cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    if (K_out) *K_out = pb->k_done;
    for (int k = 0; k < std::min<int>(cap, pb->k_done); ++k) {
        double x, y;
        std::memcpy(&x, &a[k], 8);
        std::memcpy(&y, &b[k], 8);
        if (err_T) err_T[k] = x;
        if (err_if) err_if[k] = y;
    }
    return KFP_OK;
}

kfp_status kfp_swr_subdomain_range(kfp_problem pb, int32_t s, int32_t *lo, int32_t *hi) {
    if (!pb || !pb->setup || s < 0 || s >= pb->S) {
        set_err("kfp_swr_subdomain_range: bad subdomain");
        return KFP_E_INVAL;
    }
    if (lo) *lo = pb->lo[s];
    if (hi) *hi = pb->hi[s];
    return KFP_OK;
}

kfp_status kfp_swr_subdomain_uT(kfp_problem pb, int32_t s, double *out) {
    if (!pb || !pb->setup || s < pb->s_begin || s >= pb->s_end || !out) {
        set_err("kfp_swr_subdomain_uT: subdomain %d not local", s);
        return KFP_E_INVAL;
    }
    if (pb->k_done == 0) {
        set_err("kfp_swr_subdomain_uT: no iteration since the setup / reset");
        return KFP_E_STATE;
    }
    const SubDev &sd = pb->subs[s - pb->s_begin];
    KFP_CUDA(cudaMemcpyAsync(out, final_slab(pb, s - pb->s_begin), sizeof(double) * (size_t)(sd.hi - sd.lo + 1) * pb->nx,
                             cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    return KFP_OK;
}

kfp_status kfp_swr_trace(kfp_problem pb, int32_t i, int32_t dir, double *out) {
    if (!pb || !pb->setup || i < pb->s_begin || i + 1 >= pb->s_end || dir < 0 || dir > 1 || !out || pb->k_done == 0) {
        set_err("kfp_swr_trace: interface %d not local or no iteration", i);
        return KFP_E_INVAL;
    }
    const int par = pb->k_done & 1;
    const SubDev &sd = pb->subs[i - pb->s_begin];
    const double *src = (dir == 0) ? sd.gR[par] : sd.sendR[par];
    if (pb->pipe > 1) {  // the ring slot of the last iteration
        const int R = pb->pipe + 1;
        src = (dir == 0 ? pb->ringL : pb->ringR)[i - pb->s_begin][pb->k_done % R];
    }
    KFP_CUDA(cudaMemcpyAsync(out, src, sizeof(double) * (size_t)pb->nt * pb->nx, cudaMemcpyDeviceToHost, pb->stream));
    KFP_CUDA(cudaStreamSynchronize(pb->stream));
    return KFP_OK;
}

int64_t kfp_launch_count(kfp_problem pb) { return pb ? pb->launches : -1; }

#ifdef KFP_TRACE
// debug builds only (not part of include/kfp.h): one traced step launch of the current setup
extern "C" int kfp_debug_trace_step(kfp_problem pb, int n, unsigned long long *host, int cap) {
    unsigned long long *d = nullptr;
    dev_malloc(&d, sizeof(unsigned long long) * cap * 64);
    cudaMemset(d, 0, sizeof(unsigned long long) * cap * 64);
    cudaMemcpyToSymbol(kfp::g_kfp_trace, &d, sizeof(d));
    StepParams P = base_params(pb);
    P.subs = pb->d_subs;
    P.send_robin = (pb->kind == KFP_ROBIN);
    P.p = pb->p;
    P.UT = pb->d_UT;
    P.Ulines = pb->d_Ulines;
    P.errT = pb->d_errT;
    P.errIF = pb->d_errIF;
    P.err_stride = pb->K_max;
    P.par_in = 0;
    P.par_out = 1;
    P.par_in_lo = 0;
    P.last = 0;
    launch_step(pb, pb->plan, P, (int)pb->subs.size(), n, pb->fd);
    cudaDeviceSynchronize();
    unsigned long long *z = nullptr;
    cudaMemcpyToSymbol(kfp::g_kfp_trace, &z, sizeof(z));
    cudaMemcpy(host, d, sizeof(unsigned long long) * cap * 64, cudaMemcpyDeviceToHost);
    dev_free(d);
    return (int)cudaGetLastError();
}
#endif

const char *kfp_plan(kfp_problem pb) {
    if (!pb) return "";
    pb->plan_text = pb->plan.text;
    return pb->plan_text.c_str();
}

}  // extern "C"

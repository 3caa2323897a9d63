#include <chrono>
// bminres.cu -- host driver and C ABI (include/bminres.h) of the B200 block-MINRES hot path.
//
// One block step k (p banded iterations) is a main branch and a side branch:
//   main  K1 SpMM+epilogue -> K2 orthogonalisation, Grams, Cholesky (C_k) -> K4a U_{k+1}
//   side  K3b small banded QR (z_j, residuals, stop) -> K4b directions M_k and X
// In steady state one CUDA graph per block runs {main of block s+1} || {side of block s} and
// joins before K4a (two graphs, one per panel-slot parity), so the serial small QR hides
// behind the next SpMM.  The host never waits per step: kernels publish flags into mapped
// pinned memory and the host polls the flags of the graph launched LAG graphs earlier.  Rare
// events (a breakdown, a Cholesky cancellation, live retained vectors; P:562-577,
// P:791-801) stop the main branch after K2 and the host runs the column-by-column path (the
// paper's per-iteration order) with small GPU kernels, then resumes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bminres.h"
#include "aux_kernels.cuh"
#include "common.cuh"
#include "step_kernels.cuh"
#include "dmma_kernels.cuh"
#include "row_kernels.cuh"
#include "comm.cuh"
#include "prec_kernels.cuh"

using namespace bmr;

namespace {

enum Phase { PH_SPMM = 0, PH_ORTH, PH_SMALLQR, PH_UPDATE, PH_SLOW, PH_START, PH_RESID, PH_OTHER, PH_REDUCE,
             PH_SPMM_FUSED, PH_SPMM_AV, PH_EPI, PH_EPI_FUSED, PH_UPD_MAIN, PH_PREC };

struct Retained {
    double* v;
    long long expiry;
};

struct Kfn {  // per-p kernel table
    void (*k1)(K1Args);
    void (*k1plain)(K1Args);
    void (*k1a)(K1Args);     // split mode: the SpMM alone (null: no split kernels for this p)
    void (*k1a_long)(K1Args) = nullptr;   // its long-row variant (index prefetch; chosen per matrix in bminres_solve)
    void (*k1pre)(K1Args);   // split mode: K1 streaming A V_k
    size_t smem1pre;
    void (*k1u)(K1Args);     // split mode, p >= 16: the M/X update of block k-2 as its own kernel
    size_t smem1u;
    int nt1u = 256;          // k1u_update threads per CTA
    void (*k1ws)(K1Args);    // large panels, p >= 16: the warp-specialised K1 (SpMM + epilogue, one kernel)
    size_t smem1ws;
    int nt1ws;
    // start block / exit residual: Gram, V R^{-1}, plain SpMM (DMMA / K1a versions for p = 8, 16, 32)
    void (*red2f)(DevState*, int, int);   // reduce2 + factorisation for the DMMA K1 (null: k_reduce)
    void (*fac2)(DevState*, int);         // row partition: the factorisation after the allreduce
    void (*gram)(const double*, long long, int, double*, int, double*, unsigned*);
    void (*mat)(const double*, const double*, double*, long long, int);
    size_t smem_gram, smem_mat;
    void (*k2)(K2Args);
    void (*k3b)(DevState*);
    void (*k4b)(K4bArgs);
    size_t smem1, smem2, smem3, smem4b;
    int nt1, nt2, nt4b, nt1pre;
    bool fused;   // K1 applies the M/X update of block k-2 in graph mode (DMMA K1)
    // f3 (prec_kernels.cuh): Z = L^-T V (backward), AV = L^-1 (A Z) (SpMM + forward), Y = L^-1 X
    void (*tbwd)(TriArgs);
    void (*tfwd)(TriArgs);
    void (*tfwdp)(TriArgs);
};

template <int P>
Kfn make_kfn(int q) {
    Kfn f;
    f.fused = false;
    f.k1a = nullptr;
    f.k1pre = nullptr;
    f.smem1pre = 0;
    f.k1u = nullptr;
    f.smem1u = 0;
    f.k1ws = nullptr;
    f.smem1ws = 0;
    f.nt1ws = 0;
    f.red2f = nullptr;
    f.fac2 = nullptr;
    f.gram = k_gram;
    f.mat = k_materialize;
    f.smem_gram = f.smem_mat = 0;
    f.k1 = k1_spmm<P, true>;
    f.nt1 = NT;
    f.nt1pre = NT;
    f.smem1 = K1Smem<P>::bytes;
    f.k1plain = k1_spmm<P, false>;
    f.k2 = k2_orth<P>;
    f.nt2 = NT;
    f.smem2 = K2Smem<P>::bytes;
    f.k3b = k3b_smallqr<P>;
    f.tbwd = k_trsv<P, true, false>;
    f.tfwd = k_trsv<P, false, true>;
    f.tfwdp = k_trsv<P, false, false>;
    if constexpr (P % 8 == 0) {
        if (!getenv("BMINRES_NO_DMMA")) {
            f.k1 = k1_dmma<P>;
            f.fused = getenv("BMINRES_NO_FUSE") == nullptr;
            f.smem1 = K1DSmem<P>::bytes;
            f.nt1 = K1DSmem<P>::WARPS * 32;
            f.k1a = k1a_spmm<P>;
            f.k1a_long = k1a_spmm<P, true>;
            f.k1pre = k1_dmma<P, true>;
            // p <= 16 (the register Cholesky keeps reduce2's serial tail short: config 3 98k -> 106k
            // it/s; with the serial general Cholesky it was a loss)
            // (p = 8: the one-cluster variant, 136k vs 134k it/s; p = 16: the ticketed one, 106k vs 103k)
            if constexpr (P <= 8) f.red2f = k_red2f<P, DM<P>::FR, DM<P>::NC>;
            else if constexpr (P <= 16) f.red2f = k_red2f_t<P, DM<P>::FR, DM<P>::NC>;
            if constexpr (P <= 16) f.fac2 = k_fac2<P, DM<P>::FR, DM<P>::NC>;
            f.smem1pre = K1DSmem<P, true>::bytes;
            f.nt1pre = K1DSmem<P, true>::WARPS * 32;
            if constexpr (P >= 16) {
                f.k1u = k1u_update<P>;
                f.smem1u = UpdB<P>::bytes;
                f.nt1u = UpdB<P>::WARPS * 32;
                f.k1ws = k1_ws<P>;
                f.smem1ws = K1WS<P>::bytes;
                f.nt1ws = K1WS<P>::THREADS;
            }
            f.k2 = k2_dmma<P>;
            f.smem2 = K2DSmem<P>::bytes;
            f.nt2 = K2DSmem<P>::WARPS * 32;
        }
        f.k4b = k4b_dmma<P>;
        f.smem4b = K4bDSmem<P>::bytes;
        f.k1a = k1a_spmm<P>;   // (also the plain SpMM of the start / exit residual)
        f.gram = k_gram_dmma<P>;
        f.smem_gram = GramDSmem<P>::bytes;
        f.mat = k_materialize_dmma<P>;
        f.smem_mat = mat_dmma_smem<P>();
        f.nt4b = 128;
    } else {
        f.k4b = k4b_update<P>;
        f.smem4b = K4bSmem<P>::bytes;
        f.nt4b = NT;
    }
    if constexpr (P <= 8) {   // thread-per-row TMA kernels (row_kernels.cuh)
        if (q <= K2R_QMAX && !getenv("BMINRES_NO_ROWK")) {
            f.k2 = k2_row<P>;
            f.smem2 = K2RSmem<P>::bytes;
            f.nt2 = RT;
        }
    }
    f.smem3 = K3Smem<P>::bytes;
    return f;
}

bool kfn_for(int p, Kfn* out, int q = 0) {
    switch (p) {
        case 1: *out = make_kfn<1>(q); return true;
        case 2: *out = make_kfn<2>(q); return true;
        case 3: *out = make_kfn<3>(q); return true;
        case 4: *out = make_kfn<4>(q); return true;
        case 5: *out = make_kfn<5>(q); return true;
        case 6: *out = make_kfn<6>(q); return true;
        case 7: *out = make_kfn<7>(q); return true;
        case 8: *out = make_kfn<8>(q); return true;
        case 16: *out = make_kfn<16>(q); return true;
        case 32: *out = make_kfn<32>(q); return true;
        default: return false;
    }
}

struct Err {
    int code;
};

}  // namespace

constexpr int GB_MAX = 25;   // block steps per graph, at most

struct bminres_ctx {
    bminres_options opt{};
    int device = 0;
    int n_sm = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;   // side branch during graph capture
    cudaStream_t cstream = nullptr;   // host-A staging copies, overlapped with the start block
    cudaStream_t ustream = nullptr;   // split mode: the M/X update (k1u_update) beside K1a
    cudaEvent_t ev_u0 = nullptr, ev_u1 = nullptr;
    cudaEvent_t ev_a = nullptr;       // host A staged (recorded on cstream)
    double* startbuf = nullptr;       // k_start_cgs: S, ||F0(:,i)||, events
    bool coop_ok = false;             // cooperative launches supported
    DevState* hstate = nullptr;       // pinned host copy of the state (initial value, exit read)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool own_stream = false;
    std::string err;
    // workspace
    long long n_ws = -1;
    int p_ws = -1, q_ws = -1;
    double* V[3] = {nullptr, nullptr, nullptr};   // V_k in slot k mod 3 (U_k = V_k Tr_k)
    double* M[2] = {nullptr, nullptr};            // M_k in slot k mod 2
    double* scr[2] = {nullptr, nullptr};          // column path: materialised U_{k-1}, U_k (lazy)
    double* pool = nullptr;
    double* part = nullptr;
    size_t part_elems = 0;
    double* part1 = nullptr;
    double* part2[2] = {nullptr, nullptr};
    double* dsc = nullptr;        // scratch for dot results (MAXREF+8)
    double* gdev = nullptr;       // start block: Gram columns, then a p x p inverse (2 MAXP^2)
    unsigned* dcnt = nullptr;     // tickets of the generic kernels
    DevState* st = nullptr;
    HostFlags* hf = nullptr;      // host pointer (mapped)
    HostFlags* hf_dev = nullptr;  // device alias
    double* hist = nullptr;
    size_t hist_elems = 0;   // capacity of hist in doubles (rows x p of any earlier solve)
    // staged inputs (host-pointer calls)
    int* a_rowptr = nullptr;
    int* a_col = nullptr;
    double* a_val = nullptr;
    size_t a_rows_cap = 0, a_nnz_cap = 0;
    double* bx = nullptr;         // staged B
    double* xx = nullptr;         // staged X
    size_t bx_cap = 0, xx_cap = 0;
    // graphs
    cudaGraphExec_t gexec[6] = {};
    long long graph_launches = 0;   // kernels captured in one graph
    const void* gkey[9] = {};
    // per-solve
    std::vector<Retained> retained;
    std::vector<bminres_event> events;
    std::vector<double> hist_host;
    bminres_stats_t stats{};
    long long launches = 0;
    // timing
    std::vector<cudaEvent_t> evpool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> ev_marks;   // (phase, index of start event)
    int nb1 = 0, nb2 = 0, nb4 = 0, tpw = 4, csz = 2;
    // split mode: K1a (SpMM alone, full occupancy) -> AV, then K1<P, true>
    bool split = false;
    bool upd_sep = false;    // split mode: the M/X update of block k-2 runs as k1u_update before K1a(k)
    bool ws = false;         // split mode, single rank: K1 = k1_ws (no K1a, no A V_k panel)
    bool red2_fac = false;   // reduce2 factors the new block once (k_red2f)
    bool xdefer = false;   // fused updates defer X in pairs
    int nb1a = 0;
    bool k1a_long = false, k1a_long_ws = false;
    int k1a_ku = 0;   // K1a chunk length in row groups per warp (0: the kernel's default)
    double* AV = nullptr;
    bool pdl = true;   // programmatic dependent launch of the block-step kernels
    int gblocks = 3;   // block steps per captured graph (per solve: choose_gblocks)
    bool gblocks_env = false;
    int prio_hi = 0;   // greatest stream priority (side branch)
    long long side_blocks = 0, slow_blocks = 0;
    Kfn kf{};
    unsigned long long* trace = nullptr;   // timeline tracing buffers (tooling)
    unsigned* trace_tick = nullptr;
    // row partition (world > 1; comm.cuh)
    Transport* tp = nullptr;
    HaloPlan plan;
    const void* plan_key[5] = {};
    long long n_ext = -1;                  // n_loc + n_halo rows of the V slots
    long long next_ws = -1;                // n_ext the workspace was sized for
    int* d_lcol = nullptr;                 // CSR column indices remapped into the extended panel
    long long* d_send_rows = nullptr;      // local rows the peers read, grouped by peer
    double* d_sendbuf = nullptr;
    size_t lcol_cap = 0, send_cap = 0, sendbuf_cap = 0;
    std::vector<long long> sc_d, rc_d;     // halo counts in doubles (rows x p) per peer
    // halo overlap (split mode): rows [int_lo, int_hi) reference no halo row, so K1a runs them while
    // the exchange of V_{k+1} is in flight on hstream
    long long int_lo = 0, int_hi = 0;
    bool overlap = false, halo_pending = false;
    cudaStream_t hstream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    int world() const { return opt.world; }
    // f3: IC(0) split preconditioning (bminres_set_preconditioner; prec_kernels.cuh)
    struct Sched {
        int* order = nullptr;   // device: rows by level
        int* tstart = nullptr;  // device: task offsets
        long long ntask = 0;
        int rpw = 0;            // rows per task (0: not built)
    };
    struct Prec {
        bool on = false;
        bool active = false;
        bool ws = false;        // the workspace was sized for a preconditioned core (split, AV)    // inside the core solve of a preconditioned bminres_solve
        unsigned gen = 0;       // generation (graph key)
        long long n = 0, nnzl = 0;
        int levels_f = 0, levels_b = 0;
        int *Lp = nullptr, *Li = nullptr, *Up = nullptr, *Ui = nullptr, *Uperm = nullptr;
        double *Lx = nullptr, *Ux = nullptr;
        std::vector<int> lev_f, lev_b;     // host: level of each row (forward / backward DAG)
        Sched fs, bs, fac;                 // forward / backward task lists (per rpw), factor (rows)
        unsigned* flags = nullptr;
        TriCtl* ctl = nullptr;
        double *Bh = nullptr, *Yh = nullptr, *Z = nullptr;
        size_t panel_cap = 0;
        std::vector<std::pair<const void*, int>> occ;   // resident CTAs per SM of each triangular kernel
    } prec;
};

namespace {

thread_local std::string g_create_err;

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            h->err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
            throw Err{e_ == cudaErrorMemoryAllocation ? BMINRES_ENOMEM : BMINRES_ECUDA}; \
        }                                                                              \
    } while (0)

void fail(bminres_ctx* h, int code, const std::string& msg) {
    h->err = msg;
    throw Err{code};
}

// sum over ranks (world > 1) of count doubles at dev, in place, stream-ordered on s
void allred(bminres_ctx* h, double* dev, long long count, cudaStream_t s) {
    if (!h->tp) return;
    std::string err;
    if (!h->tp->allreduce(dev, count, s, err)) fail(h, BMINRES_ENCCL, err);
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <typename T>
void dalloc(bminres_ctx* h, T** p, size_t elems) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (elems == 0) return;
    CK(cudaMalloc((void**)p, elems * sizeof(T)));
    static const char* poison = getenv("BMINRES_POISON");   // debugging: NaN-fill new buffers
    if (poison && (poison[0] == '*' || strstr(poison, "dalloc"))) CK(cudaMemsetAsync(*p, 0xFF, elems * sizeof(T), h->stream));
}

cudaEvent_t next_event(bminres_ctx* h) {
    if (h->ev_used == h->evpool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        h->evpool.push_back(e);
    }
    return h->evpool[h->ev_used++];
}

// record a timing mark around a launch (timing mode only)
struct TimeMark {
    bminres_ctx* h;
    int phase;
    size_t idx;
    bool on;
    TimeMark(bminres_ctx* h_, int ph) : h(h_), phase(ph), idx(0), on(h_->opt.timing != 0) {
        if (on) {
            idx = h->ev_used;
            cudaEvent_t e = next_event(h);
            CK(cudaEventRecord(e, h->stream));
        }
    }
    ~TimeMark() noexcept(false) {
        if (on) {
            cudaEvent_t e = next_event(h);
            CK(cudaEventRecord(e, h->stream));
            h->ev_marks.push_back({phase, idx});
        }
    }
};

void check_launch(bminres_ctx* h, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    h->launches++;
}

int grid_for(bminres_ctx* h, long long items, int per_block, int cap) {
    long long g = (items + per_block - 1) / per_block;
    g = std::max<long long>(1, std::min<long long>(g, cap));
    return (int)g;
}

// ------------------------------------------------------------------ workspace

int cluster_grid(bminres_ctx* h, const void* fn, size_t smem, long long n, long long rows_per_cta) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL * 64);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl <= 0) {
        cudaGetLastError();
        ncl = std::max(1, h->n_sm / CL);
    }
    long long need = (n + rows_per_cta - 1) / std::max<long long>(1, rows_per_cta);
    long long cl_need = std::max<long long>(1, (need + CL - 1) / CL);
    ncl = (int)std::min<long long>(ncl, cl_need);
    ncl = std::min(ncl, NB_MAX / CL);
    return ncl * CL;
}

// Block-step kernels are launched with programmatic stream serialization (PDL): a kernel may
// start while its predecessor drains and runs its pre-wait work (prefetch of panels written two
// launches back) before griddepcontrol.wait (common.cuh pdl_wait).
template <typename K, typename A>
void launch_cluster(bminres_ctx* h, K kern, int grid, int nt, size_t smem, A args, const char* what) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = h->csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
    if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    h->launches++;
}

void ensure_workspace(bminres_ctx* h, long long n, int p, int q) {
    if (h->n_ws == n && h->p_ws == p && h->q_ws == q && h->next_ws == h->n_ext && h->prec.ws == h->prec.active &&
        h->k1a_long_ws == h->k1a_long)
        return;
    h->k1a_long_ws = h->k1a_long;   // (the graphs hold the kernel, the grid its occupancy)
    h->next_ws = h->n_ext;
    h->prec.ws = h->prec.active;
    for (int s = 0; s < 6; ++s) {
        if (h->gexec[s]) cudaGraphExecDestroy(h->gexec[s]);
        h->gexec[s] = nullptr;
    }
    // panels carry 32 doubles of slack past row n-1 (the 16-byte round-up of TMA bulk copies);
    // the V slots also hold the halo rows of a row partition (n_ext >= n)
    size_t panel = (size_t)n * p + 32;
    const size_t vpanel = (size_t)std::max(n, h->n_ext) * p + 32;
    for (int s = 0; s < 3; ++s) {
        dalloc(h, &h->V[s], vpanel);
        CK(cudaMemsetAsync(h->V[s], 0, vpanel * sizeof(double), h->stream));   // (defined contents, incl. the slack)
    }
    dalloc(h, &h->M[0], panel);
    dalloc(h, &h->M[1], panel);
    // split mode for large panels (the gathers of a big SpMM need more warps per SM than the fused
    // K1 has; below ~128 MB the extra AV write + read costs more than it saves)
    {
        const char* se = getenv("BMINRES_SPLIT");
        const bool can = h->kf.k1pre != nullptr;
        const int mode = se ? (atoi(se) != 0 ? 1 : 2) : h->opt.split_spmm;
        // (a preconditioned solve always splits: its operator L^-1 A L^-T runs as its own kernels
        // into AV -- prec_kernels.cuh -- and K1 streams AV)
        h->split = can && (h->prec.active || mode == 1 || (mode == 0 && (double)n * p * 8.0 >= 128e6));
        // the update as its own kernel (k1u_update) in split mode where it is compiled
        h->upd_sep = h->split && h->kf.k1u != nullptr && getenv("BMINRES_FUSED_UPD") == nullptr;
        if (h->split || h->prec.active) {   // (generic p, preconditioned: the generic K1 reads AV)
            dalloc(h, &h->AV, panel);
        } else if (h->AV) {
            cudaFree(h->AV);
            h->AV = nullptr;
        }
    }
    for (int s = 0; s < 2; ++s) {
        if (h->scr[s]) cudaFree(h->scr[s]);
        h->scr[s] = nullptr;
    }
    dalloc(h, &h->pool, (size_t)n * std::max(q, 1) + 32);
    CK(cudaMemsetAsync(h->pool, 0, ((size_t)n * std::max(q, 1) + 32) * sizeof(double), h->stream));
    // generic-kernel partials, then K1 partials (ncl1 x (p*p+p)) and K2 partials x 2 parities
    h->part_elems = (size_t)NB_MAX * (MAXP * MAXP + MAXQ * MAXP + MAXREF + 8);
    const size_t e1 = (size_t)NB_MAX * (MAXP * MAXP + MAXP), e2 = (size_t)NB_MAX * (MAXP * MAXP + MAXQ * MAXP);
    if (!h->part) CK(cudaMalloc((void**)&h->part, (h->part_elems + e1 + 2 * e2) * sizeof(double)));
    h->part1 = h->part + h->part_elems;
    h->part2[0] = h->part1 + e1;
    h->part2[1] = h->part2[0] + e2;
    if (!h->dsc) CK(cudaMalloc((void**)&h->dsc, (MAXREF + 64) * sizeof(double)));
    if (!h->gdev) CK(cudaMalloc((void**)&h->gdev, 2 * MAXP * MAXP * sizeof(double)));
    if (!h->dcnt) {
        CK(cudaMalloc((void**)&h->dcnt, 16 * sizeof(unsigned)));
        CK(cudaMemsetAsync(h->dcnt, 0, 16 * sizeof(unsigned), h->stream));
    }
    if (!h->st) CK(cudaMalloc((void**)&h->st, sizeof(DevState)));
    if (!h->hf) {
        CK(cudaHostAlloc((void**)&h->hf, sizeof(HostFlags), cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void**)&h->hf_dev, h->hf, 0));
    }
    h->n_ws = n;
    h->p_ws = p;
    h->q_ws = q;
    // persistent one-wave grids, balanced: every SM gets the same number of CTAs; the reducing
    // kernels use clusters of h->csz CTAs (BMINRES_CLUSTER overrides, for experiments)
    auto occ_of = [&](const void* fn, int nt, size_t smem) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, nt, smem);
        return std::max(1, o);
    };
    h->pdl = getenv("BMINRES_NO_PDL") == nullptr;
    h->xdefer = h->kf.fused && getenv("BMINRES_NO_XDEFER") == nullptr;
    if (const char* gb = getenv("BMINRES_GRAPH_BLOCKS")) {
        h->gblocks = std::max(1, std::min(GB_MAX, atoi(gb)));
        h->gblocks_env = true;
    }
    const char* ce = getenv("BMINRES_CLUSTER");
    h->csz = ce ? std::max(1, std::min(8, atoi(ce))) : 2;
    const char* oe = getenv("BMINRES_CTAS_PER_SM");
    const int cap = oe ? std::max(1, atoi(oe)) : 8;
    const int o1 = std::min(cap, occ_of((const void*)h->kf.k1, h->kf.nt1, h->kf.smem1));
    const int o2 = std::min(cap, occ_of((const void*)h->kf.k2, h->kf.nt2, h->kf.smem2));
    int o4 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, (const void*)h->kf.k4b, h->kf.nt4b, h->kf.smem4b);
    o4 = std::min(cap, std::max(1, o4));
    // the main-branch grids leave one CTA slot free on csz SMs, so the side branch (K3b, one
    // CTA) is never starved of a register file while K1 / K2 run
    h->nb1 = (std::min(NB_MAX, h->n_sm * o1) - (o1 > 1 ? h->csz : 0)) / h->csz * h->csz;
    h->nb2 = (std::min(NB_MAX, h->n_sm * o2) - (o2 > 1 ? h->csz : 0)) / h->csz * h->csz;
    h->nb4 = h->n_sm * o4;
    if (h->split) {
        int oa = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, (const void*)h->kf.k1a, NT, 0);
        // (BMINRES_K1A_CPS, experiment: fewer K1a CTAs per SM, so the update branch's CTA fits beside them)
        if (const char* ce = getenv("BMINRES_K1A_CPS")) oa = std::min(oa, std::max(1, atoi(ce)));
        h->nb1a = h->n_sm * std::max(1, oa) - 1;   // one CTA slot left for K3b (side stream)
        if (const char* ke = getenv("BMINRES_K1A_KU")) h->k1a_ku = std::max(0, atoi(ke));
        const int o1p = std::min(cap, occ_of((const void*)h->kf.k1pre, h->kf.nt1pre, h->kf.smem1pre));
        h->nb1 = (std::min(NB_MAX, h->n_sm * o1p) - (o1p > 1 ? h->csz : 0)) / h->csz * h->csz;
    }
    // BMINRES_WS (experiment): the warp-specialised K1 in place of K1a + K1 on a single rank (a row
    // partition keeps the split pair: its K1a overlaps the halo exchange with the interior rows).
    // Measured (one B200): config 4 6.58 ms vs the pair's 2.88 + 3.54 ms, config 5 2.48 ms vs
    // 1.36 + 0.34 ms -- eight producer warps per SM keep fewer gathers in flight than K1a's forty
    // (twelve: the consumers spill at 128 registers), so the pair stays the default
    h->ws = h->split && h->kf.k1ws && !h->tp && !h->prec.active && getenv("BMINRES_WS") != nullptr;
    if (h->ws) h->nb1 = h->n_sm / h->csz * h->csz;
    (void)cluster_grid;

}

// ------------------------------------------------------------------ generic column ops

struct Col {
    const double* p;
    long long s;
};

void launch_dots(bminres_ctx* h, long long n, const std::vector<Col>& v, Col t, double* out) {
    DotArgs a{};
    if ((int)v.size() > MAXREF) fail(h, BMINRES_EINVAL, "too many vectors in one dot launch");
    for (size_t k = 0; k < v.size(); ++k) a.v[k] = {v[k].p, v[k].s};
    a.K = (int)v.size();
    a.t = t.p;
    a.ts = t.s;
    a.n = n;
    a.nb = grid_for(h, n, 8 * 64, std::min(NB_MAX, 2 * h->n_sm));
    a.part = h->part;
    a.out = out;
    a.cnt = h->dcnt;
    k_dots<<<a.nb, 256, 0, h->stream>>>(a);
    check_launch(h, "k_dots");
    allred(h, out, a.K, h->stream);
}

// debugging (BMINRES_DEBUG_TIMES): host wall time of the solve's segments, synchronising
struct SegTimer {
    bminres_ctx* h;
    bool on;
    std::chrono::steady_clock::time_point t0;
    explicit SegTimer(bminres_ctx* hh) : h(hh), on(getenv("BMINRES_DEBUG_TIMES") != nullptr) {
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        CK(cudaStreamSynchronize(h->stream));
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "  [seg] %-12s %9.1f us\n", what, std::chrono::duration<double, std::micro>(t - t0).count());
        t0 = t;
    }
};

// k_colstep (aux_kernels.cuh) for the compiled p; out gets Kd dots (+ the norm), allreduced
void launch_colstep(bminres_ctx* h, double* F, long long n, int p, int col, int Kc, const double* cin, int Kd,
                    bool want_norm, int ncol, const double* nsrc, double* out, double* text = nullptr,
                    long long ts = 1) {
    ColStepArgs a{F, n, text ? 0 : col, Kc, Kd, ncol, want_norm ? 1 : 0, cin, nsrc, h->part, 0, out, h->dcnt + 3,
                  text, ts};
    static const int cps = getenv("BMINRES_COLSTEP_CPS") ? std::max(1, atoi(getenv("BMINRES_COLSTEP_CPS"))) : 4;
    a.nb = grid_for(h, n, 256, std::min(NB_MAX, cps * h->n_sm));   // one wave (4 CTAs per SM)
    switch (p) {
#define CS(P)                                                                           \
    case P:                                                                             \
        if (text) k_colstep<P, true><<<a.nb, 256, 0, h->stream>>>(a);                  \
        else k_colstep<P, false><<<a.nb, 256, 0, h->stream>>>(a);                      \
        break;
        CS(1) CS(2) CS(3) CS(4) CS(5) CS(6) CS(7) CS(8) CS(16) CS(32)
#undef CS
        default: fail(h, BMINRES_EINVAL, "k_colstep: p not compiled");
    }
    check_launch(h, "k_colstep");
    const int nv = Kd + (want_norm ? 1 : 0);
    if (nv > 0) allred(h, out, nv, h->stream);
}

// k_start_cgs (aux_kernels.cuh): cooperative launch, one wave of co-resident CTAs
void launch_start_cgs(bminres_ctx* h, double* F, long long n, int p, const double* f0n, double tau,
                      unsigned long long seed, long long row_begin, double* S, double* ev) {
    StartArgs sa{F, n, f0n, tau, seed, row_begin, h->part, S, ev, h->opt.policy == 1 ? 1 : 0};
    void* args[] = {&sa};
    const void* fn = nullptr;
    switch (p) {
#define SC(P) case P: fn = (const void*)k_start_cgs<P>; break;
        SC(1) SC(2) SC(3) SC(4) SC(5) SC(6) SC(7) SC(8) SC(16) SC(32)
#undef SC
        default: fail(h, BMINRES_EINVAL, "k_start_cgs: p not compiled");
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0));
    const int nb = std::max(1, std::min(NB_MAX, std::max(1, occ) * h->n_sm));
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(256), args, 0, h->stream);
    if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k_start_cgs: ") + cudaGetErrorString(e));
    h->launches++;
}

// host-visible dot products (synchronising)
std::vector<double> dots_host(bminres_ctx* h, long long n, const std::vector<Col>& v, Col t) {
    launch_dots(h, n, v, t, h->dsc);
    std::vector<double> r(v.size());
    CK(cudaMemcpyAsync(r.data(), h->dsc, v.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return r;
}

// t = scale*(t - sum_k c_k v_k)
void launch_axpy(bminres_ctx* h, long long n, const std::vector<Col>& v, const double* cval, const double* cdev,
                 double csign, Col t, double scale, const double* scale_dev = nullptr) {
    AxpyArgs a{};
    if ((int)v.size() > MAXREF) fail(h, BMINRES_EINVAL, "too many vectors in one axpy launch");
    for (size_t k = 0; k < v.size(); ++k) {
        a.v[k] = {v[k].p, v[k].s};
        a.cval[k] = cval ? cval[k] : 0.0;
    }
    a.K = (int)v.size();
    a.cdev = cdev;
    a.csign = csign;
    a.t = const_cast<double*>(t.p);
    a.ts = t.s;
    a.n = n;
    a.scale = scale;
    a.scale_dev = scale_dev;
    int g = grid_for(h, n, 256, 8 * h->n_sm);
    k_axpy<<<g, 256, 0, h->stream>>>(a);
    check_launch(h, "k_axpy");
}

void launch_rand(bminres_ctx* h, double* out, long long stride, long long n, long long row_begin, uint64_t seed,
                 uint64_t stream, uint64_t event) {
    int g = grid_for(h, n, 256, 8 * h->n_sm);
    k_rand<<<g, 256, 0, h->stream>>>(out, stride, n, row_begin, seed, stream, event);
    check_launch(h, "k_rand");
}

// out[c] = ||X(:,c) - Y(:,c)||^2  (device result)
void launch_colsq(bminres_ctx* h, const double* X, const double* Y, long long n, int p, double* out) {
    int R = 256 / p;
    int nb = grid_for(h, n, R * 16, std::min(NB_MAX, 2 * h->n_sm));
    k_colsq<<<nb, 256, 0, h->stream>>>(X, Y, n, p, h->part, nb, out, h->dcnt + 1);
    check_launch(h, "k_colsq");
    allred(h, out, p, h->stream);
}

// ------------------------------------------------------------------ block-step launches

struct StepPtrs {
    const int* rowptr;
    const int* col;
    const double* val;
    double* X;
};

// main branch of block k: gathers V_k (slot k%3), reads V_{k-1} (slot (k-1)%3), writes W and
// then W' into slot (k+1)%3 (= V_{k+1}); parity k%2 selects the double-buffered small state
void launch_reduce(bminres_ctx* h, cudaStream_t s, int which, long long k) {
    TimeMark tm(h, PH_REDUCE);
    const int P = h->p_ws;
    const int Emax = P * P + (which == 1 ? P : MAXQ * P);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
    cfg.gridDim = dim3((Emax + 7) / 8);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // row partition: the totals are summed by k_reduce, allreduced, then factored by k_fac2
    const bool fac_after = which == 2 && h->red2_fac && h->tp;
    if (which == 2 && h->red2_fac && !h->tp && P <= 8) {   // k_red2f: one cluster of RF_CL CTAs
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = RF_CL;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(RF_CL);
        cfg.blockDim = dim3(rf_warps<8>() * 32);
        cfg.numAttrs = 2;
    }
    // reduce2 triggers its dependent (K1(k+1) / K1a) right after its own wait: K1's fused update
    // overlaps the reduction (+1.8% at config 2)
    // (not in split mode: its dependent K1a has no pre-wait work, and its early-resident CTAs would
    // take the SM slots K3b needs)
    static const int early2 = getenv("BMINRES_NO_EARLY_RED2") ? 0 : 1;
    // reduce1 too: K2 launches during it and issues its first TMA stages (W, V_k: written by
    // K1, which completed before reduce1's wait returned) -- config 2 145.8k -> 146.8k it/s
    static const int early1 = getenv("BMINRES_NO_EARLY_RED1") ? 0 : 1;
    const int early = h->split ? 0 : (which == 2 ? early2 : early1);
    cudaError_t e = (which == 2 && h->red2_fac && !fac_after)
                        ? cudaLaunchKernelEx(&cfg, h->kf.red2f, h->st, (int)(k & 1), early)
                        : cudaLaunchKernelEx(&cfg, k_reduce, h->st, which, (int)(k & 1), P, fac_after ? 0 : early);
    if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k_reduce: ") + cudaGetErrorString(e));
    h->launches++;
    if (h->tp) {   // the totals over all ranks (K3b then runs replicated)
        double* tot = which == 1 ? h->st->red1 : h->st->red2[k & 1];
        allred(h, tot, which == 1 ? P * P + P : P * P + MAXQ * P, s);
    }
    if (fac_after) {   // every rank factors the bitwise-identical totals once (K1's prologue loads them)
        cudaLaunchConfig_t fc{};
        fc.gridDim = dim3(1);
        fc.blockDim = dim3(256);
        fc.stream = s;
        fc.attrs = at;
        fc.numAttrs = 1;   // (PDL after the allreduce)
        cudaError_t e2 = cudaLaunchKernelEx(&fc, h->kf.fac2, h->st, (int)(k & 1));
        if (e2 != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k_fac2: ") + cudaGetErrorString(e2));
        h->launches++;
    }
}

// Halo exchange of a V slot (world > 1): pack the rows the peers read, land the peers' rows in
// this slot's halo region [n_loc, n_loc + n_halo).  Every rank calls it at the same points.
void halo_exchange(bminres_ctx* h, double* V, int p, cudaStream_t s) {
    if (!h->tp) return;
    TimeMark tm(h, PH_OTHER);
    const long long ns = (long long)h->plan.send_rows.size();
    if (ns > 0) {
        k_pack_rows<<<grid_for(h, ns * p, 256, 4 * h->n_sm), 256, 0, s>>>(V, h->d_send_rows, ns, p, h->d_sendbuf);
        check_launch(h, "k_pack_rows");
    }
    std::string err;
    if (!h->tp->exchange(h->d_sendbuf, h->sc_d.data(), V + h->plan.n_loc * p, h->rc_d.data(), s, err))
        fail(h, BMINRES_ENCCL, err);
}
// The exchange of V_{k+1} after K2(k), overlapped (split mode with an interior): the rows are
// packed on s, the transport runs on hstream; K1a(k+1) processes the interior rows meanwhile and
// waits for ev_halo before the boundary rows (launch_k1).  halo_join makes s wait for a pending
// exchange (every other consumer of the halo, graph ends, the end of the block loop).
void halo_exchange_async(bminres_ctx* h, double* V, int p, cudaStream_t s) {
    if (!h->tp) return;
    if (!h->overlap) {
        halo_exchange(h, V, p, s);
        return;
    }
    TimeMark tm(h, PH_OTHER);
    const long long ns = (long long)h->plan.send_rows.size();
    if (ns > 0) {
        k_pack_rows<<<grid_for(h, ns * p, 256, 4 * h->n_sm), 256, 0, s>>>(V, h->d_send_rows, ns, p, h->d_sendbuf);
        check_launch(h, "k_pack_rows");
    }
    CK(cudaEventRecord(h->ev_pack, s));
    CK(cudaStreamWaitEvent(h->hstream, h->ev_pack, 0));
    std::string err;
    if (!h->tp->exchange(h->d_sendbuf, h->sc_d.data(), V + h->plan.n_loc * p, h->rc_d.data(), h->hstream, err))
        fail(h, BMINRES_ENCCL, err);
    CK(cudaEventRecord(h->ev_halo, h->hstream));
    h->halo_pending = true;
}
void halo_join(bminres_ctx* h, cudaStream_t s) {
    if (!h->halo_pending) return;
    CK(cudaStreamWaitEvent(s, h->ev_halo, 0));
    h->halo_pending = false;
}

// Y = A X alone (start block with X0, exit residual, bminres_spmm): the full-occupancy K1a kernel
// for p in {8, 16, 32}, else the plain variant of the generic K1.  Both sum each row in CSR order
// with fma from 0 (bitwise the same A X as the block steps' SpMM).
void spmm_plain(bminres_ctx* h, const Kfn& f, const int* rowptr, const int* col, const double* val, const double* X,
                double* Y, long long n, cudaStream_t s, int tpw) {
    K1Args a{rowptr, col, val, X, nullptr, Y, n, nullptr, nullptr, 0, 0, tpw};
    if (f.k1a) {
        int oa = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, (const void*)f.k1a, NT, 0);
        const long long groups = (n + 3) / 4;   // >= one row group per warp
        const long long g = std::min<long long>((long long)h->n_sm * std::max(1, oa), std::max(1ll, (groups + 7) / 8));
        f.k1a<<<(unsigned)g, NT, 0, s>>>(a);
        check_launch(h, "k1a_spmm(plain)");
    } else {
        f.k1plain<<<(unsigned)(h->nb4 > 0 ? h->nb4 : 4 * h->n_sm), NT, 0, s>>>(a);   // grid-stride
        check_launch(h, "k1_spmm(plain)");
    }
}

// ------------------------------------------------------------------ f3: the preconditioned operator
// One triangular kernel over a task list (prec_kernels.cuh), persistent: the grid never exceeds
// the resident capacity (the flag waits are deadlock-free only among resident warps), less one
// CTA slot for the side branch.
void launch_trsv(bminres_ctx* h, cudaStream_t s, void (*kern)(TriArgs), const bminres_ctx::Sched& sc, bool upper,
                 const StepPtrs* sp, const double* X, double* Y, long long n) {
    auto& pr = h->prec;
    TriArgs a{};
    if (sp) {
        a.rowptr = sp->rowptr;
        a.col = sp->col;
        a.val = sp->val;
    }
    a.Tp = upper ? pr.Up : pr.Lp;
    a.Ti = upper ? pr.Ui : pr.Li;
    a.Tx = upper ? pr.Ux : pr.Lx;
    a.X = X;
    a.Y = Y;
    a.flags = pr.flags;
    a.ctl = pr.ctl;
    a.s = TriSched{sc.order, sc.tstart, sc.ntask};
    a.n = n;
    int occ = 0;
    for (auto& c : pr.occ)
        if (c.first == (const void*)kern) occ = c.second;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)kern, NT, 0);
        occ = std::max(1, occ);
        pr.occ.push_back({(const void*)kern, occ});
    }
    const long long cap = std::max(1ll, (long long)h->n_sm * occ - 1);
    const long long need = (sc.ntask + NT / 32 - 1) / (NT / 32);
    const int grid = (int)std::max(1ll, std::min(cap, need));
    kern<<<grid, NT, 0, s>>>(a);
    check_launch(h, "k_trsv");
}

// out = L^-1 A L^-T V (reading R8): Z = L^-T V, then out = L^-1 (A Z)
void launch_prec_op(bminres_ctx* h, cudaStream_t s, const StepPtrs& sp, const double* V, double* out, long long n) {
    cudaStream_t keep = h->stream;
    h->stream = s;   // (TimeMark records on h->stream)
    {
        TimeMark tm(h, PH_PREC);
        launch_trsv(h, s, h->kf.tbwd, h->prec.bs, true, nullptr, V, h->prec.Z, n);
        launch_trsv(h, s, h->kf.tfwd, h->prec.fs, false, &sp, h->prec.Z, out, n);
    }
    h->stream = keep;
}

void launch_k1(bminres_ctx* h, cudaStream_t s, const StepPtrs& sp, long long n, long long k, int fuse = 0) {
    const int sk = (int)(k % 3), par = (int)(k & 1);
    K1Args a{sp.rowptr, sp.col, sp.val, h->V[sk], h->V[(sk + 2) % 3], h->V[(sk + 1) % 3], n, h->st, h->part,
             par, sk, h->tpw, fuse, h->M[par], h->M[par ^ 1], sp.X, nullptr, h->xdefer ? 1 : 0};
    // the M/X update of block k-2 (row a5): its V_{k-2} rows are overwritten by K1(k)'s W, so it runs
    // on this stream before K1a(k) (PDL).  BMINRES_UPD_BRANCH (experiment): on its own high-priority
    // branch beside K1a(k) (independent data), joined before K1(k) -- measured no faster at config 4
    // (2.10k vs 2.10k it/s; the pair is bound by HBM and the power cap together)
    bool upd_branch = false;
    if (h->split && h->upd_sep && fuse) {
        static const bool branch = getenv("BMINRES_UPD_BRANCH") != nullptr;
        upd_branch = !h->opt.timing && branch;
        cudaStream_t us = s;
        if (upd_branch) {
            CK(cudaEventRecord(h->ev_u0, s));
            CK(cudaStreamWaitEvent(h->ustream, h->ev_u0, 0));
            us = h->ustream;
        }
        cudaStream_t keep = h->stream;
        h->stream = us;
        {
            TimeMark tm(h, PH_UPD_MAIN);
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = (h->pdl && !upd_branch) ? 1 : 0;
            cfg.gridDim = dim3(h->n_sm - 1);   // (one SM left for K3b: the two do not fit one SM together)
            cfg.blockDim = dim3(h->kf.nt1u);
            cfg.dynamicSmemBytes = h->kf.smem1u;
            cfg.stream = us;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, h->kf.k1u, a);
            if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k1u_update: ") + cudaGetErrorString(e));
            h->launches++;
        }
        h->stream = keep;
        if (upd_branch) CK(cudaEventRecord(h->ev_u1, us));
        a.fuse = 0;
        fuse = 0;
    }
    if (h->ws) {
        // one kernel: gathers (producer warps) + DMMA epilogue (consumer warps)
        if (upd_branch) CK(cudaStreamWaitEvent(s, h->ev_u1, 0));   // the update read V_{k-2}
        {
            TimeMark tm(h, PH_SPMM);
            cudaStream_t keep = h->stream;
            h->stream = s;
            launch_cluster(h, h->kf.k1ws, h->nb1, h->kf.nt1ws, h->kf.smem1ws, a, "k1_ws");
            h->stream = keep;
        }
        launch_reduce(h, s, 1, k);
        return;
    }
    if (h->split) {
        // K1a: AV = A V_k (PDL after reduce2 / K2), then K1 streams AV
        K1Args aa = a;
        aa.Vprev = nullptr;
        aa.Y = h->AV;
        aa.fuse = 0;
        // (BMINRES_K1A_DYN, experiment: chunks in order from st->k1a_ctr -- for K1a beside the update
        // branch; alone it measured slower, 3.09 vs 2.63 ms at config 4)
        aa.dyn = getenv("BMINRES_K1A_DYN") ? 1 : 0;
        aa.ku = h->k1a_ku;
        cudaStream_t keep = h->stream;
        h->stream = s;
        auto k1a_launch = [&](const K1Args& args) {
            TimeMark tm(h, PH_SPMM_AV);
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
            cfg.gridDim = dim3(h->nb1a);
            cfg.blockDim = dim3(NT);
            cfg.dynamicSmemBytes = 0;
            cfg.stream = s;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, h->kf.k1a, args);
            if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k1a_spmm: ") + cudaGetErrorString(e));
            h->launches++;
        };
        if (h->prec.active) {
            launch_prec_op(h, s, sp, h->V[sk], h->AV, n);   // (f3: in place of K1a)
        } else if (h->halo_pending) {
            // row partition: the interior rows while V_k's halo is in flight, then the boundary
            // rows [0, int_lo) and [int_hi, n) once it has landed
            K1Args ai = aa;
            ai.r0 = h->int_lo;
            ai.nrows = h->int_hi - h->int_lo;
            k1a_launch(ai);
            halo_join(h, s);
            K1Args ab = aa;
            ab.r0 = 0;
            ab.nrows = h->int_lo + (n - h->int_hi);
            ab.gap_at = h->int_lo;
            ab.gap = h->int_hi - h->int_lo;
            if (ab.dyn) ab.dyn = 2;
            if (ab.nrows > 0) k1a_launch(ab);
        } else {
            k1a_launch(aa);
        }
        a.AV = h->AV;
        if (upd_branch) CK(cudaStreamWaitEvent(s, h->ev_u1, 0));   // the update read V_{k-2}
        {
            TimeMark tm(h, fuse ? PH_EPI_FUSED : PH_EPI);
            launch_cluster(h, h->kf.k1pre, h->nb1, h->kf.nt1pre, h->kf.smem1pre, a, "k1_dmma(split)");
        }
        h->stream = keep;
        launch_reduce(h, s, 1, k);
        return;
    }
    halo_join(h, s);
    if (h->prec.active) {   // (f3, generic p: the generic K1 reads A V_k from AV)
        launch_prec_op(h, s, sp, h->V[sk], h->AV, n);
        a.AV = h->AV;
    }
    {
        TimeMark tm(h, fuse ? PH_SPMM_FUSED : PH_SPMM);
        cudaStream_t keep = h->stream;
        h->stream = s;
        launch_cluster(h, h->kf.k1, h->nb1, h->kf.nt1, h->kf.smem1, a, "k1_spmm");
        h->stream = keep;
    }
    launch_reduce(h, s, 1, k);
}
void launch_k2(bminres_ctx* h, cudaStream_t s, long long n, long long k, bool with_reduce = true) {
    const int sk = (int)(k % 3), par = (int)(k & 1);
    K2Args a{h->V[(sk + 1) % 3], h->V[sk], h->pool, n, h->st, h->part + (size_t)NB_MAX * (MAXP * MAXP + MAXP),
             par, sk, h->tpw};
    {
        TimeMark tm(h, PH_ORTH);
        cudaStream_t keep = h->stream;
        h->stream = s;
        launch_cluster(h, h->kf.k2, h->nb2, h->kf.nt2, h->kf.smem2, a, "k2_orth");
        h->stream = keep;
    }
    halo_exchange_async(h, h->V[(sk + 1) % 3], h->p_ws, s);   // V_{k+1} rows the peers' SpMM reads
    if (with_reduce) launch_reduce(h, s, 2, k);
}
// side branch of block k: M_k -> M[k%2] (over M_{k-2}), M_{k-1} = M[(k+1)%2]
void launch_k3b(bminres_ctx* h, cudaStream_t s) {
    TimeMark tm(h, PH_SMALLQR);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;   // (also recorded into graph kernel nodes)
    at[0].val.priority = h->prio_hi;
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(K3T);
    cfg.dynamicSmemBytes = h->kf.smem3;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, h->kf.k3b, h->st);
    if (e != cudaSuccess) fail(h, BMINRES_ECUDA, std::string("k3b_smallqr: ") + cudaGetErrorString(e));
    h->launches++;
}
// (blk = 0: the block is not recorded in upd_last -- graph captures, whose k is a residue)
void launch_k4b(bminres_ctx* h, cudaStream_t s, const StepPtrs& sp, long long n, long long k, int force = 0,
                bool record = true) {
    TimeMark tm(h, PH_UPDATE);
    const int sk = (int)(k % 3), par = (int)(k & 1);
    K4bArgs a{h->V[sk], h->M[par], h->M[par ^ 1], sp.X, n, h->st, sk, h->tpw, par, force, record ? k : 0};
    h->kf.k4b<<<h->nb4, h->kf.nt4b, h->kf.smem4b, s>>>(a);
    check_launch(h, "k4b_update");
}

// Block steps per graph for a solve of nblocks block steps.  A graph boundary costs a stall:
// each graph joins its last K3b, and the PDL overlap of K1's fused update with reduce2 is lost
// across the boundary (~6 us at config 2; 3 -> 5 blocks per graph: 141.6k -> 143.7k it/s).
// Blocks launched past the last one are wasted main-branch work (~9 boundaries' worth each),
// so among 3..GB_MAX pick the count with the least boundaries + 9 x overshoot.
int choose_gblocks(long long nblocks) {
    int best = 3;
    double bc = 1e300;
    for (int g = 3; g <= GB_MAX; ++g) {
        const long long graphs = (nblocks + g - 1) / g;
        const double cost = (double)graphs + 9.0 * (double)(graphs * g - nblocks);
        if (cost < bc) {
            bc = cost;
            best = g;
        }
    }
    return best;
}

// Graph for side block s (s mod 6): main {reduce2 of block s, K1 + reduce1 + K2 of block s+1}
// || side {K3b (, K4b) of block s}, forked after reduce2(s), whose totals K3b factors.  Inside a
// graph every main-branch edge is programmatic (PDL).  Fused mode: K1(s+1) applies the M/X
// update of block s-1 and the side branch is K3b alone.
void build_graphs(bminres_ctx* h, const StepPtrs& sp, long long n) {
    const void* key[9] = {sp.rowptr, sp.col, sp.val, sp.X, h->V[0], h->M[0], (const void*)(intptr_t)n,
                          (const void*)(intptr_t)((h->p_ws * 16 + h->gblocks) * 2 + (h->red2_fac ? 1 : 0)),
                          (const void*)(intptr_t)(h->prec.active ? (long long)h->prec.gen + 1 : 0)};
    bool same = h->gexec[0] && std::equal(key, key + 9, h->gkey);
    if (same) return;
    for (int q = 0; q < 6; ++q) {
        if (h->gexec[q]) cudaGraphExecDestroy(h->gexec[q]);
        h->gexec[q] = nullptr;
        cudaGraph_t g;
        long long saved = h->launches;
        const long long sblk = 6 + q;   // any block with this residue mod 6
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        for (int j = 0; j < h->gblocks; ++j) {   // block steps t = s .. s+gblocks-1 of one graph
            const long long t = sblk + j;
            launch_reduce(h, h->stream, 2, t);
            CK(cudaEventRecord(h->ev_fork, h->stream));
            CK(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
            // K1(t+1) applies the update of block t-1 (fused) and overwrites V_{t-1}: it waits for
            // the side work of block t-1 (inside this graph from the second step on)
            if (j > 0) CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
            launch_k1(h, h->stream, sp, n, t + 1, h->kf.fused ? 1 : 0);
            launch_k2(h, h->stream, n, t + 1, false);
            launch_k3b(h, h->side);
            if (!h->kf.fused) launch_k4b(h, h->side, sp, n, t, 0, false);
            CK(cudaEventRecord(h->ev_join, h->side));
        }
        CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
        halo_join(h, h->stream);   // (a graph ends with no exchange in flight)
        CK(cudaStreamEndCapture(h->stream, &g));
        h->graph_launches = h->launches - saved;   // kernels per graph (the same for every residue)
        h->launches = saved;
        CK(cudaGraphInstantiate(&h->gexec[q], g, 0));
        cudaGraphDestroy(g);
    }
    std::copy(key, key + 9, h->gkey);
}

// write a few DevState fields from the host (after draining the stream)
// Host -> device copy ordered on the solver's stream.  (A plain cudaMemcpy runs on the legacy
// stream, which does not order against the non-blocking h->stream, and from pageable memory it
// may return before the DMA lands: a kernel launched next on h->stream could read the old value.)
void h2d(bminres_ctx* h, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
}

template <typename T>
void set_state(bminres_ctx* h, size_t offset, T value) {
    h2d(h, (char*)h->st + offset, &value, sizeof(T));
}
#define SET_STATE(h, field, val) set_state(h, offsetof(DevState, field), (decltype(DevState::field))(val))

template <typename T>
T get_state(bminres_ctx* h, size_t offset) {
    T v;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(&v, (char*)h->st + offset, sizeof(T), cudaMemcpyDeviceToHost));
    return v;
}
#define GET_STATE(h, field) get_state<decltype(DevState::field)>(h, offsetof(DevState, field))

// ------------------------------------------------------------------ column-by-column path

// The paper's per-iteration orthogonalisation for the p columns of block b (Alg. 1 P:286-293,
// breakdown P:562-577, replacement P:690-729, retention P:797-805).  On entry the V slot of
// block b+1 holds W' (the candidates already orthogonalised against U_{b-1} and U_b by
// K1/K2) and om2[par] the raw candidate norms.  On exit it holds U_{b+1} (normalised) with
// Tr_{b+1} = I, DevState.Ck[par] = C_b and the pool coefficients of block b are zero (the
// pool was updated here, column by column).
void slow_block(bminres_ctx* h, long long n, int p, long long b, double tau, long long maxit) {
    halo_join(h, h->stream);   // (the exchange of the candidates' halo, replaced below)
    TimeMark tm(h, PH_SLOW);
    const int par = (int)(b & 1);
    const long long j0 = GET_STATE(h, j_done) + 1;
    std::vector<double> om2(MAXP);
    CK(cudaMemcpy(om2.data(), (char*)h->st + offsetof(DevState, om2) + par * MAXP * sizeof(double),
                  MAXP * sizeof(double), cudaMemcpyDeviceToHost));
    int q_first = GET_STATE(h, q_first), q_live = GET_STATE(h, q_live);
    const int qc = h->q_ws;
    std::vector<double> Ck(MAXP * MAXP, 0.0);
    int stop_after = 0;
    const int sk = (int)(b % 3);
    double* Wp = h->V[(sk + 1) % 3];
    auto Wc = [&](int m) { return Col{Wp + m, p}; };
    // U_{b-1}, U_b are materialised (V Tr) only if a replacement needs them as a window
    bool have_window = false;
    auto materialise = [&]() {
        if (have_window) return;
        for (int s2 = 0; s2 < 2; ++s2)
            if (!h->scr[s2]) {
                CK(cudaMalloc((void**)&h->scr[s2], ((size_t)n * p + 32) * sizeof(double)));
                CK(cudaMemsetAsync(h->scr[s2], 0, ((size_t)n * p + 32) * sizeof(double), h->stream));
            }
        const int slots[2] = {(sk + 2) % 3, sk};
        for (int s2 = 0; s2 < 2; ++s2) {
            const double* Tr = (const double*)((char*)h->st + offsetof(DevState, Tr)) + (size_t)slots[s2] * MAXP * MAXP;
            h->kf.mat<<<grid_for(h, n * p, 256, 8 * h->n_sm), 256, h->kf.smem_mat, h->stream>>>(
                h->V[slots[s2]], Tr, h->scr[s2], n, p);
            check_launch(h, "k_materialize");
        }
        have_window = true;
    };
    const double* Uprev = nullptr;
    const double* Ucur = nullptr;
    // shrink policy: the lanes already removed in block b+1, and the ones removed here
    const bool shrink = h->opt.policy == 1;
    std::vector<long long> absent_from(MAXP, KINF);
    if (shrink)
        CK(cudaMemcpy(absent_from.data(), (char*)h->st + offsetof(DevState, absent_from), MAXP * sizeof(long long),
                      cudaMemcpyDeviceToHost));
    bool absent_changed = false;
    for (int m = 0; m < p; ++m) {
        const long long j = j0 + m;
        if (j > maxit) break;
        if (shrink && absent_from[m] <= b + 1) {
            // u_{j+p} was removed with an earlier u of this lane (A 0 = 0): the candidate is
            // zero, h_{j+p,j} = 0, no event
            Ck[m * MAXP + m] = 0.0;
            continue;
        }
        // MGS against the new vectors of this block (u_{bp+1} .. u_{bp+m})
        for (int mp = 0; mp < m; ++mp) {
            double c = dots_host(h, n, {Wc(mp)}, Wc(m))[0];
            launch_axpy(h, n, {Wc(mp)}, &c, nullptr, 1.0, Wc(m), 1.0);
            Ck[mp * MAXP + m] = c;
        }
        // retained near-dependent vectors
        for (auto& r : h->retained) {
            if (r.expiry < j) continue;
            double c = dots_host(h, n, {Col{r.v, 1}}, Wc(m))[0];
            launch_axpy(h, n, {Col{r.v, 1}}, &c, nullptr, 1.0, Wc(m), 1.0);
        }
        const double hh = std::sqrt(dots_host(h, n, {Wc(m)}, Wc(m))[0]);
        const double omega = std::sqrt(om2[m]);
        if (hh <= tau * omega) {
            bminres_event ev{};
            ev.j = j;
            ev.col = m + 1;
            ev.kind = hh <= 1e-12 * omega ? 0 : 1;
            ev.action = 1;
            ev.ratio = omega > 0 ? hh / omega : 0.0;
            if (ev.kind == 1) {
                Retained r{nullptr, j + 2 * p};
                CK(cudaMalloc((void**)&r.v, n * sizeof(double)));
                CK(cudaMemsetAsync(r.v, 0, n * sizeof(double), h->stream));
                double mone = -1.0;
                // v = w / h  (t = (0 - (-1) w) / h)
                launch_axpy(h, n, {Wc(m)}, &mone, nullptr, 1.0, Col{r.v, 1}, 1.0 / hh);
                h->retained.push_back(r);
                ev.action = 2;
            }
            if (shrink) {
                // block-size reduction: u_{j+p} = 0 is not added; lane m is removed from
                // block b+1 on
                launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Wc(m), 0.0);
                ev.action = ev.kind == 1 ? 5 : 4;
                absent_from[m] = b + 1;
                absent_changed = true;
            } else if (q_live > 0) {
                // replacement: pool vector (already orthogonal to u_1..u_{j+p-1}),
                // orthogonalised twice more against retained + window, normalised
                std::vector<Col> src = {Col{h->pool + q_first, qc}};
                launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Wc(m), 0.0);
                double mone = -1.0;
                launch_axpy(h, n, src, &mone, nullptr, 1.0, Wc(m), 1.0);
                q_first++;
                q_live--;
                materialise();
                Uprev = h->scr[0];
                Ucur = h->scr[1];
                std::vector<Col> win;
                for (auto& r : h->retained)
                    if (r.expiry >= j) win.push_back(Col{r.v, 1});
                if (b > 1)
                    for (int mp = m; mp < p; ++mp) win.push_back(Col{Uprev + mp, p});
                for (int mp = 0; mp < p; ++mp) win.push_back(Col{Ucur + mp, p});
                for (int mp = 0; mp < m; ++mp) win.push_back(Wc(mp));
                for (int pass = 0; pass < 2; ++pass)
                    for (auto& v : win) {
                        double c = dots_host(h, n, {v}, Wc(m))[0];
                        launch_axpy(h, n, {v}, &c, nullptr, 1.0, Wc(m), 1.0);
                    }
                const double rn = std::sqrt(dots_host(h, n, {Wc(m)}, Wc(m))[0]);
                launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Wc(m), 1.0 / rn);
            } else {
                launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Wc(m), 0.0);
                ev.action = 3;
                stop_after = m + 1;
            }
            h->events.push_back(ev);
            Ck[m * MAXP + m] = 0.0;   // h_{j+p,j} := 0
        } else {
            launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Wc(m), 1.0 / hh);
            Ck[m * MAXP + m] = hh;
        }
        // pool vectors orthogonalised against the new Lanczos vector
        for (int q = q_first; q < q_first + q_live; ++q) {
            Col r{h->pool + q, qc};
            double c = dots_host(h, n, {Wc(m)}, r)[0];
            launch_axpy(h, n, {Wc(m)}, &c, nullptr, 1.0, r, 1.0);
        }
        if (stop_after) break;
    }
    CK(cudaStreamSynchronize(h->stream));
    if (absent_changed)
        h2d(h, (char*)h->st + offsetof(DevState, absent_from), absent_from.data(), MAXP * sizeof(long long));
    h2d(h, (char*)h->st + offsetof(DevState, Ck) + par * MAXP * MAXP * sizeof(double), Ck.data(),
        MAXP * MAXP * sizeof(double));
    SET_STATE(h, q_first, q_first);
    SET_STATE(h, q_live, q_live);
    SET_STATE(h, stop_after, stop_after);
    SET_STATE(h, need_slow, 0);
    SET_STATE(h, given_blk, b);
    SET_STATE(h, bd_at, KINF);
    SET_STATE(h, run_main, 1);
    SET_STATE(h, k_main, b + 1);
    // Tr_{b+1} = I (V_{b+1} is the normalised basis block); pool coefficients of block b = 0
    std::vector<double> I(MAXP * MAXP, 0.0), Z0(MAXP * MAXQ, 0.0);
    for (int c = 0; c < MAXP; ++c) I[c * MAXP + c] = 1.0;
    h2d(h, (char*)h->st + offsetof(DevState, Tr) + (size_t)((sk + 1) % 3) * MAXP * MAXP * sizeof(double), I.data(),
        MAXP * MAXP * sizeof(double));
    h2d(h, (char*)h->st + offsetof(DevState, coef) + (size_t)par * MAXP * MAXQ * sizeof(double), Z0.data(),
        MAXP * MAXQ * sizeof(double));
    h->hf->need_slow = 0;
    h->slow_blocks++;
    halo_exchange(h, Wp, p, h->stream);   // the new U_{b+1} rows the peers read
}

// Finish block b after the column path: its side branch (K3b, K4b).
void debug_state(bminres_ctx* h, const char* tag);
void finish_given_block(bminres_ctx* h, const StepPtrs& sp, long long n, long long b) {
    if (getenv("BMINRES_DEBUG_STATE")) debug_state(h, "before given K3b");
    launch_k3b(h, h->stream);
    if (getenv("BMINRES_DEBUG_STATE")) debug_state(h, "after given K3b");
    launch_k4b(h, h->stream, sp, n, b);
    CK(cudaStreamSynchronize(h->stream));
}

// Fused mode: apply the M/X updates of blocks whose K3b has run but whose K1 (two blocks
// later, which applies them) did not (end of a graph run).  Drains the stream.
void flush_updates(bminres_ctx* h, const StepPtrs& sp, long long n) {
    if (!h->kf.fused) return;
    const long long last = GET_STATE(h, upd_last), ks = GET_STATE(h, k_side);
    const long long b0 = GET_STATE(h, k_upd_min);
    if (h->xdefer && last >= b0 && ((last - b0) & 1) == 0) {
        // the last fused update deferred its X: X += M_last Z_last (M[last % 2] holds M_last)
        K4bArgs a{nullptr, h->M[last & 1], nullptr, sp.X, n, h->st, 0, h->tpw, (int)(last & 1), 1, 0, 3, last};
        h->kf.k4b<<<h->nb4, h->kf.nt4b, h->kf.smem4b, h->stream>>>(a);
        check_launch(h, "k4b(x only)");
    }
    for (long long b = last + 1; b < ks; ++b) launch_k4b(h, h->stream, sp, n, b, 1);
    CK(cudaStreamSynchronize(h->stream));
}

// Gram G = F^T F of a row-major n x p panel (one k_gram launch), copied to the host (synchronising).
std::vector<double> panel_gram(bminres_ctx* h, const double* F, long long n, int p) {
    const int nb = grid_for(h, n, 64, std::min(NB_MAX, 2 * h->n_sm));
    h->kf.gram<<<nb, 256, h->kf.smem_gram, h->stream>>>(F, n, p, h->part, nb, h->gdev, h->dcnt + 2);
    check_launch(h, "k_gram");
    allred(h, h->gdev, (long long)p * p, h->stream);
    std::vector<double> G((size_t)p * p);
    CK(cudaMemcpyAsync(G.data(), h->gdev, G.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return G;
}

// Upper Cholesky G = R^T R (p x p, row-major, ld p).  Fails when a pivot keeps less than
// `keep` of its column's squared norm (cancellation) or is not positive.
bool host_chol(const std::vector<double>& G, int p, double keep, std::vector<double>& R) {
    R.assign((size_t)p * p, 0.0);
    std::vector<double> A = G;
    for (int m = 0; m < p; ++m) {
        const double d = A[m * p + m];
        if (!(d > 0.0) || !(d > keep * G[m * p + m])) return false;
        const double r = std::sqrt(d);
        for (int c = m; c < p; ++c) R[m * p + c] = (c == m) ? r : A[m * p + c] / r;
        for (int i = m + 1; i < p; ++i)
            for (int j = i; j < p; ++j) A[i * p + j] -= R[m * p + i] * R[m * p + j];
    }
    return true;
}

// Start block fast path (row a0): thin QR F0 = U_p S by CholQR2 -- two Gram passes, the p x p
// factors on the host, U = F R^{-1} on the device.  It is taken only when no column of F0 can be
// (near-)dependent: every first-pass pivot must keep >= 1e-4 of its column's squared norm, far
// above the deflation threshold tau^2 (C13); otherwise the caller runs the column-by-column MGS2
// path, which decides step-0 deflation exactly as the oracle does.  In exact arithmetic S and U
// are those of the Gram-Schmidt QR (R with positive diagonal is unique).
bool fast_start(bminres_ctx* h, double* F, long long n, int p, double tau, std::vector<double>& S) {
    if (getenv("BMINRES_NO_FAST_START")) return false;
    std::vector<double> R1, R2;
    // pivot m = ||f_m - proj||^2, G_mm = ||f_m||^2 = ||F0(:,m)||^2: a pivot <= tau^2 G_mm is exactly the
    // oracle's step-0 test ||f_m|| <= tau ||F0(:,m)|| (C13), so such a block takes the column path
    if (!host_chol(panel_gram(h, F, n, p), p, std::max(1e-4, tau * tau), R1)) return false;
    auto upload_inverse = [&](const std::vector<double>& R) {   // R^{-1} (upper), ld MAXP
        std::vector<double> Ri((size_t)MAXP * MAXP, 0.0);
        for (int l = 0; l < p; ++l)
            for (int r = l; r >= 0; --r) {
                double s = (r == l) ? 1.0 : 0.0;
                for (int c = r + 1; c <= l; ++c) s -= R[r * p + c] * Ri[c * MAXP + l];
                Ri[r * MAXP + l] = s / R[r * p + r];
            }
        CK(cudaMemcpyAsync(h->gdev + MAXP * MAXP, Ri.data(), Ri.size() * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream));
    };
    double* U = h->V[0];   // free until block 3
    const int g = grid_for(h, n * p, 256, 8 * h->n_sm);
    upload_inverse(R1);
    h->kf.mat<<<g, 256, h->kf.smem_mat, h->stream>>>(F, h->gdev + MAXP * MAXP, U, n, p);
    check_launch(h, "k_materialize");
    if (!host_chol(panel_gram(h, U, n, p), p, 0.5, R2)) {
        CK(cudaMemsetAsync(U, 0, (size_t)n * p * sizeof(double), h->stream));   // U_0 = 0 again
        return false;
    }
    upload_inverse(R2);
    h->kf.mat<<<g, 256, h->kf.smem_mat, h->stream>>>(U, h->gdev + MAXP * MAXP, F, n, p);
    check_launch(h, "k_materialize");
    CK(cudaMemsetAsync(U, 0, (size_t)n * p * sizeof(double), h->stream));
    std::fill(S.begin(), S.end(), 0.0);
    for (int r = 0; r < p; ++r)   // S = R2 R1
        for (int c = r; c < p; ++c) {
            double s = 0.0;
            for (int t = r; t <= c; ++t) s += R2[r * p + t] * R1[t * p + c];
            S[r * MAXP + c] = s;
        }
    return true;
}

bool retained_live(bminres_ctx* h, long long jfirst) {
    for (auto& r : h->retained)
        if (r.expiry >= jfirst) return true;
    return false;
}

// ------------------------------------------------------------------ row partition setup

// Build (or reuse) the halo plan of this rank's CSR rows: offsets of all ranks, remote columns by
// owner, the lists the peers read from this rank (exchanged), the remapped column indices.
void setup_partition(bminres_ctx* h, const bminres_csr* A, const int* rowptr_dev, const int* col_dev, int p) {
    const int world = h->opt.world, rank = h->opt.rank;
    const void* key[5] = {A->col_idx, (const void*)(intptr_t)A->nnz, (const void*)(intptr_t)A->row_begin,
                          (const void*)(intptr_t)A->n_loc, (const void*)(intptr_t)A->n};
    std::string err;
    // the plan is rebuilt on every solve unless the caller opted into reuse (header: plan_reuse)
    if (!(h->opt.plan_reuse && h->d_lcol && std::equal(key, key + 5, h->plan_key))) {
        // offsets of every rank: all-to-all of (row_begin, n_loc)
        std::vector<long long> snd(2 * world), rcv(2 * world), one(world, 2);
        for (int q = 0; q < world; ++q) {
            snd[2 * q] = A->row_begin;
            snd[2 * q + 1] = A->n_loc;
        }
        if (!h->tp->alltoallv(snd.data(), one.data(), rcv.data(), one.data(), h->stream, err))
            fail(h, BMINRES_ENCCL, err);
        std::vector<long long> off(world + 1, 0);
        for (int q = 0; q < world; ++q) {
            if (rcv[2 * q] != off[q]) fail(h, BMINRES_EINVAL, "ranks must own contiguous row blocks in rank order");
            off[q + 1] = off[q] + rcv[2 * q + 1];
        }
        if (off[world] != A->n) fail(h, BMINRES_EINVAL, "the ranks' rows do not cover 0..n-1");
        std::vector<int> col(std::max<long long>(A->nnz, 1)), rp(A->n_loc + 1);
        // (stream-ordered: a host CSR is staged on h->stream just before)
        CK(cudaMemcpyAsync(col.data(), col_dev, A->nnz * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(rp.data(), rowptr_dev, (A->n_loc + 1) * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        HaloPlan& pl = h->plan;
        if (!build_halo_plan(world, rank, off.data(), A->nnz, col.data(), pl))
            fail(h, BMINRES_EINVAL, "column index outside [0, n)");
        // tell every owner which of its rows this rank reads
        std::vector<long long> rq(world, 1), cnt_in(world);
        if (!h->tp->alltoallv(pl.recv_count.data(), rq.data(), cnt_in.data(), rq.data(), h->stream, err))
            fail(h, BMINRES_ENCCL, err);
        pl.send_count = cnt_in;
        long long ns = 0;
        for (long long c : cnt_in) ns += c;
        std::vector<long long> req(std::max<long long>(ns, 1));
        if (!h->tp->alltoallv(pl.halo_rows.data(), pl.recv_count.data(), req.data(), pl.send_count.data(), h->stream,
                              err))
            fail(h, BMINRES_ENCCL, err);
        pl.send_rows.assign(req.begin(), req.begin() + ns);
        for (auto& r : pl.send_rows) {
            r -= A->row_begin;
            if (r < 0 || r >= A->n_loc) fail(h, BMINRES_EINVAL, "halo request outside this rank's rows");
        }
        if (h->lcol_cap < (size_t)std::max<long long>(A->nnz, 1)) {
            dalloc(h, &h->d_lcol, std::max<long long>(A->nnz, 1));
            h->lcol_cap = std::max<long long>(A->nnz, 1);
        }
        h2d(h, h->d_lcol, pl.local_col.data(), A->nnz * sizeof(int));
        if (h->send_cap < (size_t)std::max<long long>(ns, 1)) {
            dalloc(h, &h->d_send_rows, std::max<long long>(ns, 1));
            h->send_cap = std::max<long long>(ns, 1);
        }
        h2d(h, h->d_send_rows, pl.send_rows.data(), ns * sizeof(long long));
        long long lo = 0, hi = 0;
        interior_rows(A->n_loc, rp.data(), pl.local_col.data(), &lo, &hi);
        h->int_lo = lo;
        h->int_hi = hi;
        std::copy(key, key + 5, h->plan_key);
    }
    const long long ns = (long long)h->plan.send_rows.size();
    if (h->sendbuf_cap < (size_t)std::max<long long>(ns * p, 1)) {
        dalloc(h, &h->d_sendbuf, std::max<long long>(ns * p, 1));
        h->sendbuf_cap = std::max<long long>(ns * p, 1);
    }
    h->sc_d.assign(world, 0);
    h->rc_d.assign(world, 0);
    for (int q = 0; q < world; ++q) {
        h->sc_d[q] = h->plan.send_count[q] * p;
        h->rc_d[q] = h->plan.recv_count[q] * p;
    }
    h->n_ext = A->n_loc + h->plan.n_halo;
}

// Y = A X for the local rows with X extended by its halo (world > 1): X's local rows are copied
// into the scratch slot Vs, the halo exchanged, and the SpMM gathers from Vs.
const double* extended_input(bminres_ctx* h, const double* X, long long n, int p, double* Vs) {
    if (!h->tp) return X;
    halo_join(h, h->stream);
    CK(cudaMemcpyAsync(Vs, X, (size_t)n * p * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    halo_exchange(h, Vs, p, h->stream);
    return Vs;
}

// ------------------------------------------------------------------ the solve

// debugging (BMINRES_DEBUG_STATE): the side branch's state, printed to stderr
void debug_state(bminres_ctx* h, const char* tag) {
    CK(cudaStreamSynchronize(h->stream));
    static DevState d;
    CK(cudaMemcpy(&d, h->st, sizeof(DevState), cudaMemcpyDeviceToHost));
    const int p = h->p_ws;
    auto pm = [&](const char* nm, const double* M, int rows, int ld, int cols) {
        fprintf(stderr, "%s\n", nm);
        for (int r = 0; r < rows; ++r) {
            for (int c = 0; c < cols; ++c) fprintf(stderr, " % .6e", M[r * ld + c]);
            fprintf(stderr, "\n");
        }
    };
    fprintf(stderr, "[%s] k_side %lld k_main %lld j_done %lld given %lld side_go %d stop_after %d\n", tag, d.k_side,
            d.k_main, d.j_done, d.given_blk, d.side_go, d.stop_after);
    pm("G1", d.G[1], p, MAXP, p); pm("Ck0", d.Ck[0], p, MAXP, p); pm("Ck1", d.Ck[1], p, MAXP, p); pm("CprevS", d.CprevS, p, MAXP, p);
    pm("T", d.T, p, MAXP, p); pm("res", d.res, 1, p, p);
    pm("Qacc[0]", d.Qacc[0], 2 * p, 2 * MAXP, 2 * p); pm("Qacc[1]", d.Qacc[1], 2 * p, 2 * MAXP, 2 * p);
}

int do_solve(bminres_ctx* h, const bminres_csr* A, const double* Bin, double* Xin, int p, double tol, long long maxit,
             double tau) {
    const bminres_options& o = h->opt;
    if (!A || !Bin || !Xin) fail(h, BMINRES_EINVAL, "null argument");
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world) fail(h, BMINRES_EINVAL, "rank / world out of range");
    if (o.world > 1 && !h->tp) fail(h, BMINRES_EINVAL, "world > 1 needs a transport (bminres_init_nccl / callbacks)");
    const long long n = A->n_loc;
    if (o.world == 1 && (A->n != A->n_loc || A->row_begin != 0))
        fail(h, BMINRES_EINVAL, "world = 1 needs n_loc = n, row_begin = 0");
    if (p < 1 || p > BMINRES_MAX_P || !kfn_for(p, &h->kf, o.pool_size)) fail(h, BMINRES_EINVAL, "unsupported block size p");
    if (n < p) fail(h, BMINRES_EINVAL, "n < p");
    // K1a's long-row variant for matrices with >= 12 entries per row on average (dmma_kernels.cuh)
    h->k1a_long = h->kf.k1a_long != nullptr && A->nnz >= 12 * n && getenv("BMINRES_K1A_PLAIN") == nullptr;
    if (h->k1a_long) h->kf.k1a = h->kf.k1a_long;
    if (!std::isfinite(tol) || tol < 0 || maxit < 0 || !std::isfinite(tau) || tau < 0)
        fail(h, BMINRES_EINVAL, "tol / maxit / deflation_tol out of range");
    if (A->nnz < 0 || A->nnz >= (1ll << 31)) fail(h, BMINRES_EINVAL, "nnz must be < 2^31");
    if (o.pool_size > MAXQ || o.pool_size < 0) fail(h, BMINRES_EINVAL, "pool_size must be in 0..8");
    const int q = o.pool_size;

    CK(cudaSetDevice(h->device));
    cudaEvent_t e_solve0, e_solve1, e_loop0, e_loop1;
    CK(cudaEventCreate(&e_solve0));
    CK(cudaEventCreate(&e_solve1));
    CK(cudaEventCreate(&e_loop0));
    CK(cudaEventCreate(&e_loop1));
    h->events.clear();
    for (auto& r : h->retained) cudaFree(r.v);
    h->retained.clear();
    h->launches = 0;
    h->ev_used = 0;
    h->ev_marks.clear();
    h->stats = bminres_stats_t{};
    h->slow_blocks = 0;
    CK(cudaEventRecord(e_solve0, h->stream));
    SegTimer seg(h);

    // ---- inputs: device pointers are used in place; host pointers are staged
    StepPtrs sp{};
    const size_t panel = (size_t)n * p;
    bool x_host = false;
    bool a_stage = false, a_async = false;
    {
        TimeMark tm(h, PH_OTHER);
        const bool a_dev = is_device_ptr(A->row_ptr) && is_device_ptr(A->col_idx) && is_device_ptr(A->values);
        if (a_dev) {
            sp.rowptr = A->row_ptr;
            sp.col = A->col_idx;
            sp.val = A->values;
        } else {
            if (h->a_rows_cap < (size_t)n + 1) {
                dalloc(h, &h->a_rowptr, n + 1);
                h->a_rows_cap = n + 1;
            }
            if (h->a_nnz_cap < (size_t)std::max<long long>(A->nnz, 1)) {
                dalloc(h, &h->a_col, std::max<long long>(A->nnz, 1));
                dalloc(h, &h->a_val, std::max<long long>(A->nnz, 1));
                h->a_nnz_cap = std::max<long long>(A->nnz, 1);
            }
            a_stage = true;
            sp.rowptr = h->a_rowptr;
            sp.col = h->a_col;
            sp.val = h->a_val;
        }
        if (!is_device_ptr(Bin)) {
            if (h->bx_cap < panel) {
                dalloc(h, &h->bx, panel);
                h->bx_cap = panel;
            }
            CK(cudaMemcpyAsync(h->bx, Bin, panel * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            Bin = h->bx;
        }
        if (!is_device_ptr(Xin)) {
            x_host = true;
            if (h->xx_cap < panel) {
                dalloc(h, &h->xx, panel);
                h->xx_cap = panel;
            }
            if (o.use_x0) CK(cudaMemcpyAsync(h->xx, Xin, panel * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            sp.X = h->xx;
        } else {
            sp.X = Xin;
        }
        if ((((uintptr_t)Bin) | ((uintptr_t)sp.X)) & 15) fail(h, BMINRES_EINVAL, "B and X must be 16-byte aligned");
        if (a_stage) {
            // A host CSR is staged after B: with X0 = 0 the start block needs only B, so (single
            // rank) A's copies run on their own stream beside it and the block loop waits for them
            a_async = !o.use_x0 && !h->tp;
            cudaStream_t cs = h->stream;
            if (a_async) {
                if (!h->cstream) CK(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
                if (!h->ev_a) CK(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
                CK(cudaEventRecord(h->ev_a, h->stream));   // (after the buffers' (re)allocation)
                CK(cudaStreamWaitEvent(h->cstream, h->ev_a, 0));
                cs = h->cstream;
            }
            CK(cudaMemcpyAsync(h->a_rowptr, A->row_ptr, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, cs));
            CK(cudaMemcpyAsync(h->a_col, A->col_idx, A->nnz * sizeof(int), cudaMemcpyHostToDevice, cs));
            CK(cudaMemcpyAsync(h->a_val, A->values, A->nnz * sizeof(double), cudaMemcpyHostToDevice, cs));
            if (a_async) CK(cudaEventRecord(h->ev_a, cs));
        }
    }
    if (h->tp) {   // (a transport at world = 1 runs the same path with an empty halo)
        setup_partition(h, A, sp.rowptr, sp.col, p);   // halo plan; the SpMM reads the remapped columns
        sp.col = h->d_lcol;
    } else {
        h->n_ext = n;
    }
    ensure_workspace(h, n, p, q);
    // row partition, split mode: overlap the exchange with K1a's interior rows when they are at least
    // a quarter of the rows (z-slabs of config 4: all but the first and last planes; config 5's
    // long-range entries leave no interior at G > 1)
    h->overlap = h->tp && h->split && (h->int_hi - h->int_lo) * 4 >= n && getenv("BMINRES_NO_HALO_OVERLAP") == nullptr;
    h->halo_pending = false;
    const double* B = Bin;

    // ---- history buffer
    long long hist_cap = o.record_history ? std::min<long long>(maxit + 1, std::max<long long>(1, (8ll << 20) / p)) : 0;
    if ((size_t)hist_cap * p > h->hist_elems) {   // (capacity in doubles: p may change between solves)
        dalloc(h, &h->hist, (size_t)hist_cap * p);
        h->hist_elems = (size_t)hist_cap * p;
    }

    // ---- state init
    // the state's initial value, built in pinned host memory (one fast copy; also the exit copy)
    if (!h->hstate) CK(cudaMallocHost((void**)&h->hstate, sizeof(DevState)));
    DevState& init = *h->hstate;
    std::memset(&init, 0, sizeof(init));
    init.run_main = 1;
    init.k_main = 1;
    init.bd_at = KINF;
    init.q_first = 0;
    init.q_live = q;
    init.pool_cap = std::max(q, 1);
    init.status = 1;
    init.k_side = 1;
    init.stop_side_at = KINF;
    init.j_done = 0;
    init.maxit = maxit;
    init.hist_cap = hist_cap;
    init.tol = tol;
    init.tau = tau;
    init.hist = hist_cap ? h->hist : nullptr;
    init.hflags = h->hf_dev;
    init.part1 = h->part1;
    init.part2[0] = h->part2[0];
    init.part2[1] = h->part2[1];
    init.ncl1 = h->nb1 / h->csz;
    init.ncl2 = h->nb2 / h->csz;
    // reduce2 factors the new block once (a row partition: k_fac2 after the allreduce of the totals)
    h->red2_fac = h->kf.red2f && !getenv("BMINRES_NO_RED2F");
    init.red2_fac = h->red2_fac ? 1 : 0;
    init.fac_blk = -1;
    init.fac_bad = 0;
    init.given_blk = -1;
    init.policy = o.policy;
    for (int c = 0; c < MAXP; ++c) init.absent_from[c] = KINF;
    init.k_upd_min = KINF;
    init.upd_last = 0;
    // timeline tracing (tooling): BMINRES_TRACE=<launch number> records that launch of every
    // block-step kernel (globaltimer per CTA and phase point), dumped to BMINRES_TRACE_FILE
    const char* trace_env = getenv("BMINRES_TRACE");
    const size_t trace_elems = (size_t)TR_NKIND * TRACE_CTAS * TRACE_PTS;
    if (trace_env) {
        if (!h->trace) {
            CK(cudaMalloc((void**)&h->trace, trace_elems * sizeof(unsigned long long)));
            CK(cudaMalloc((void**)&h->trace_tick, TR_NKIND * sizeof(unsigned)));
        }
        CK(cudaMemsetAsync(h->trace, 0, trace_elems * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->trace_tick, 0, TR_NKIND * sizeof(unsigned), h->stream));
        init.trace = h->trace;
        init.trace_tick = h->trace_tick;
        init.trace_launch = atoll(trace_env);
    }
    for (int t = 0; t < 3; ++t)
        for (int c = 0; c < MAXP; ++c) init.Tr[t][c * MAXP + c] = 1.0;
    std::vector<double> S(MAXP * MAXP, 0.0), beta(p, 0.0), f0n(p, 0.0);

    {
        TimeMark tm(h, PH_START);
        CK(cudaMemsetAsync(h->M[0], 0, panel * sizeof(double), h->stream));
        CK(cudaMemsetAsync(h->M[1], 0, panel * sizeof(double), h->stream));
        CK(cudaMemsetAsync(h->V[0], 0, panel * sizeof(double), h->stream));
        if (!o.use_x0) CK(cudaMemsetAsync(sp.X, 0, panel * sizeof(double), h->stream));
        // beta_i = ||b_i||
        launch_colsq(h, B, nullptr, n, p, h->dsc);
        std::vector<double> b2(p);
        CK(cudaMemcpyAsync(b2.data(), h->dsc, p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        // F0 = B - A X0 (C6) into the V slot of block 1 (U_1 = V_1, Tr_1 = I)
        double* F = h->V[1];
        if (o.use_x0) {
            const double* Xe = extended_input(h, sp.X, n, p, h->V[0]);
            spmm_plain(h, h->kf, sp.rowptr, sp.col, sp.val, Xe, F, n, h->stream, h->tpw);
            k_sub_from<<<grid_for(h, panel, 256, 8 * h->n_sm), 256, 0, h->stream>>>(B, F, (long long)panel);
            check_launch(h, "k_sub_from");
        } else {
            CK(cudaMemcpyAsync(F, B, panel * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        }
        std::vector<double> f2(p);
        if (o.use_x0) {
            launch_colsq(h, F, nullptr, n, p, h->dsc);
            CK(cudaMemcpyAsync(f2.data(), h->dsc, p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        }
        CK(cudaStreamSynchronize(h->stream));
        if (!o.use_x0) f2 = b2;   // F0 = B (bitwise)
        for (int c = 0; c < p; ++c) {
            beta[c] = std::sqrt(b2[c]);
            f0n[c] = std::sqrt(f2[c]);
        }
        // thin QR F0 = U_p S with one re-orthogonalisation (classical GS, two passes) and
        // step-0 deflation (eqn.init-QR; reading C13); CholQR2 fast path when no
        // column can deflate
        long long nrep0 = 0;
        seg.mark("stage+norms");
        const bool fast = fast_start(h, F, n, p, tau, S);
        seg.mark(fast ? "fast_start" : "fast_fail");
        // Column path: per column one pass per CGS step over the panel (k_colstep: 1 -- normalise
        // the previous column, dots; 2 -- subtract, dots; 3 -- subtract, norm) and one host read
        double* d1 = h->dsc + 8;
        double* d2 = h->dsc + 8 + MAXP;
        double* dn[2] = {h->dsc + 8 + 2 * MAXP, h->dsc + 8 + 2 * MAXP + 1};   // ||f_i||^2 by parity
        int pend = -1;   // column whose normalisation (by 1/sqrt(*dn[pend & 1])) is pending
        const bool coop = !fast && !h->tp && h->coop_ok && !getenv("BMINRES_NO_COOP_START");
        if (coop) {   // single rank: the whole column path in one cooperative launch
            if (!h->startbuf) CK(cudaMalloc((void**)&h->startbuf, (MAXP * MAXP + 3 * MAXP) * sizeof(double)));
            double* dS = h->startbuf;
            double* dF0 = dS + MAXP * MAXP;
            double* dEv = dF0 + MAXP;
            h2d(h, dF0, f0n.data(), p * sizeof(double));
            CK(cudaMemsetAsync(dS, 0, MAXP * MAXP * sizeof(double), h->stream));
            launch_start_cgs(h, F, n, p, dF0, tau, o.seed, A->row_begin, dS, dEv);
            std::vector<double> ev(2 * p);
            CK(cudaMemcpyAsync(S.data(), dS, MAXP * MAXP * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaMemcpyAsync(ev.data(), dEv, 2 * p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            for (int i = 0; i < p; ++i)
                if (ev[2 * i + 1] >= 0.0) {
                    bminres_event e{};
                    e.j = 0;
                    e.col = i + 1;
                    e.kind = (int)ev[2 * i + 1];
                    e.action = o.policy == 1 ? 4 : 1;   // removed (shrink) / replaced
                    e.ratio = ev[2 * i];
                    h->events.push_back(e);
                    if (o.policy == 1) init.absent_from[i] = 1;
                }
        }
        for (int i = 0; i < ((fast || coop) ? 0 : p); ++i) {
            const double* nsrc = pend >= 0 ? dn[pend & 1] : nullptr;
            if (i == 0) {
                launch_colstep(h, F, n, p, 0, 0, nullptr, 0, true, -1, nullptr, dn[0]);
            } else {
                launch_colstep(h, F, n, p, i, 0, nullptr, i, false, pend, nsrc, d1);
                launch_colstep(h, F, n, p, i, i, d1, i, false, -1, nullptr, d2);
                launch_colstep(h, F, n, p, i, i, d2, 0, true, -1, nullptr, dn[i & 1]);
            }
            pend = -1;
            std::vector<double> c2(2 * MAXP + 2, 0.0);
            CK(cudaMemcpyAsync(c2.data(), h->dsc + 8, (2 * MAXP + 2) * sizeof(double), cudaMemcpyDeviceToHost,
                               h->stream));
            CK(cudaStreamSynchronize(h->stream));
            const double hh = std::sqrt(c2[2 * MAXP + (i & 1)]);
            for (int l = 0; l < i; ++l) S[l * MAXP + i] = c2[l] + c2[MAXP + l];
            if (hh <= tau * f0n[i] && o.policy == 1) {
                // shrink: the dependent start column is removed -- u_i = 0
                bminres_event ev{};
                ev.j = 0;
                ev.col = i + 1;
                ev.kind = hh <= 1e-12 * f0n[i] ? 0 : 1;
                ev.action = 4;
                ev.ratio = f0n[i] > 0 ? hh / f0n[i] : 0.0;
                h->events.push_back(ev);
                S[i * MAXP + i] = 0.0;
                init.absent_from[i] = 1;
                launch_axpy(h, n, {}, nullptr, nullptr, 1.0, Col{F + i, p}, 0.0);
                pend = -1;
            } else if (hh <= tau * f0n[i]) {
                bminres_event ev{};
                ev.j = 0;
                ev.col = i + 1;
                ev.kind = hh <= 1e-12 * f0n[i] ? 0 : 1;
                ev.action = 1;
                ev.ratio = f0n[i] > 0 ? hh / f0n[i] : 0.0;
                h->events.push_back(ev);
                S[i * MAXP + i] = 0.0;
                // replaced by a random vector (C17), orthogonalised twice against f_1..f_{i-1} and
                // normalised (deferred, as a kept column; no host read)
                launch_rand(h, F + i, p, n, A->row_begin, o.seed, 0, (uint64_t)nrep0++);
                if (i > 0) {
                    launch_colstep(h, F, n, p, i, 0, nullptr, i, false, -1, nullptr, d1);
                    launch_colstep(h, F, n, p, i, i, d1, i, false, -1, nullptr, d2);
                    launch_colstep(h, F, n, p, i, i, d2, 0, true, -1, nullptr, dn[i & 1]);
                } else {
                    launch_colstep(h, F, n, p, 0, 0, nullptr, 0, true, -1, nullptr, dn[0]);
                }
                pend = i;
            } else {
                S[i * MAXP + i] = hh;
                pend = i;   // f_i / hh, applied by the next column's first pass (or below)
            }
        }
        if (pend >= 0) launch_colstep(h, F, n, p, 0, 0, nullptr, 0, false, pend, dn[pend & 1], nullptr);
        seg.mark("column path");
        // replacement pool (reading C18): drawn now, orthogonalised twice against U_p
        for (int qq = 0; qq < q; ++qq) {
            double* r = h->pool + qq;
            const long long rs = std::max(q, 1);
            launch_rand(h, r, rs, n, A->row_begin, o.seed, 1, (uint64_t)qq);
            // two classical Gram-Schmidt passes against U_p, one pass over the panel each
            launch_colstep(h, F, n, p, 0, 0, nullptr, p, false, -1, nullptr, h->dsc + 8, r, rs);
            launch_colstep(h, F, n, p, 0, p, h->dsc + 8, p, false, -1, nullptr, h->dsc + 8 + MAXP, r, rs);
            launch_colstep(h, F, n, p, 0, p, h->dsc + 8 + MAXP, 0, false, -1, nullptr, nullptr, r, rs);
        }
    }
    // T = S, history[0], while-test (Alg. 2, reading C7)
    double mx0 = 0.0;
    std::vector<double> h0(p);
    for (int c = 0; c < p; ++c) {
        double s = 0.0;
        for (int r = 0; r < p; ++r) s += S[r * MAXP + c] * S[r * MAXP + c];
        h0[c] = beta[c] > 0 ? std::sqrt(s) / beta[c] : 0.0;
        mx0 = std::max(mx0, h0[c]);
    }
    for (int r = 0; r < p; ++r)
        for (int c = 0; c < p; ++c) init.T[r * MAXP + c] = S[r * MAXP + c];
    for (int c = 0; c < p; ++c) {
        init.beta[c] = beta[c];
        init.res[c] = h0[c];
    }
    bool finished = false;
    if (mx0 < tol) {
        init.status = 0;
        finished = true;
    } else if (maxit == 0) {
        init.status = 1;
        finished = true;
    }
    seg.mark("pool+S");
    CK(cudaMemcpyAsync(h->st, &init, sizeof(DevState), cudaMemcpyHostToDevice, h->stream));
    halo_exchange(h, h->V[1], p, h->stream);   // U_1 rows the peers' first SpMM reads
    if (hist_cap) CK(cudaMemcpyAsync(h->hist, h0.data(), p * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    h->hf->side_done = finished ? 1 : 0;
    h->hf->stop_blk = KINF;
    h->hf->status = init.status;
    h->hf->need_slow = 0;
    h->hf->bd_at = KINF;
    h->hf->j_done = 0;
    h->hf->k_side = 1;
    h->hf->k_main = 1;
    CK(cudaStreamSynchronize(h->stream));

    // ---- block loop
    const bool graphs = o.use_graphs && !o.timing && (!h->tp || h->tp->capturable());
    // timing mode of a fused kernel set: the graph's launches issued explicitly, in the graph's
    // order, with an event pair around each (the kernels the product runs, timed one by one)
    const bool fused_expl = o.timing && h->kf.fused;
    if (a_async) CK(cudaStreamWaitEvent(h->stream, h->ev_a, 0));   // A staged before its first use
    seg.mark("init state");
    const long long nblocks = (maxit + p - 1) / p;
    if (!h->gblocks_env) h->gblocks = choose_gblocks(nblocks);
    if (graphs && !finished) build_graphs(h, sp, n);
    seg.mark("graphs");
    CK(cudaEventRecord(e_loop0, h->stream));
    const int GB = h->gblocks;               // block steps per graph
    const int LAG = std::max(2, 6 / GB);     // graphs in flight before the host polls
    std::vector<cudaEvent_t> lag_ev(LAG);
    for (auto& e : lag_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    long long b = 1;          // next block of the side branch
    bool main_ahead = false;  // K1, K2 of block b already done (V_{b+1} ready)
    while (!h->hf->side_done) {
        const bool ret = retained_live(h, (b - 1) * p + 1);
        const bool expl = (!graphs && !fused_expl) || ret;
        if (!main_ahead) {   // (reduce2 of block b is left pending: the graph / explicit path runs it)
            launch_k1(h, h->stream, sp, n, b);
            launch_k2(h, h->stream, n, b, false);
            main_ahead = true;
        }
        if (ret) {   // candidates of block b meet a live retained vector: column path
            CK(cudaStreamSynchronize(h->stream));
            slow_block(h, n, p, b, tau, maxit);
            finish_given_block(h, sp, n, b);
            b++;
            main_ahead = false;
            continue;
        }
        if (expl) {
            launch_reduce(h, h->stream, 2, b);
            launch_k3b(h, h->stream);
            launch_k4b(h, h->stream, sp, n, b);
            CK(cudaStreamSynchronize(h->stream));
            if (h->hf->need_slow) {   // K3b found a breakdown in block b
                slow_block(h, n, p, b, tau, maxit);
                finish_given_block(h, sp, n, b);
            }
            b++;
            main_ahead = false;
            continue;
        }
        // pipelined graphs: side block s with main block s+1 (fused: K1(s+1) applies the
        // update of block s-1; updates of blocks < b were applied explicitly)
        halo_join(h, h->stream);   // (the graphs' first K1 does not wait for an exchange launched before them)
        if (h->kf.fused) SET_STATE(h, k_upd_min, b);
        long long launched = 0;
        // The host stops launching on a stop / breakdown seen in a graph it has synchronised
        // with, i.e. of a block <= the last side block of graph `launched - LAG`: the decision
        // depends only on completed graphs, so every rank of a partitioned solve launches the
        // same graphs (their collectives match).
        for (long long s = b; s <= nblocks && graphs; s += GB) {
            CK(cudaGraphLaunch(h->gexec[s % 6], h->stream));
            h->launches += h->graph_launches;
            CK(cudaEventRecord(lag_ev[launched % LAG], h->stream));
            launched++;
            if (launched >= LAG) {
                CK(cudaEventSynchronize(lag_ev[launched % LAG]));
                const long long done_last = b + (launched - LAG + 1) * GB - 1;   // last side block synced
                if ((h->hf->side_done && h->hf->stop_blk <= done_last) ||
                    (h->hf->need_slow && h->hf->bd_at <= done_last))
                    break;
            }
        }
        for (long long s = b; s <= nblocks && !graphs; ++s) {   // fused_expl (timing mode)
            launch_reduce(h, h->stream, 2, s);
            launch_k3b(h, h->stream);
            launch_k1(h, h->stream, sp, n, s + 1, 1);
            launch_k2(h, h->stream, n, s + 1, false);
            CK(cudaStreamSynchronize(h->stream));
            if (h->hf->side_done || h->hf->need_slow) break;
        }
        CK(cudaStreamSynchronize(h->stream));
        flush_updates(h, sp, n);
        if (h->kf.fused) SET_STATE(h, k_upd_min, KINF);
        if (h->hf->side_done) break;
        b = GET_STATE(h, k_side);
        if (h->hf->need_slow) {
            // breakdown of block bd_at == b (found by K1(b+1) and K3b(b)); the side finished b-1
            slow_block(h, n, p, b, tau, maxit);
            finish_given_block(h, sp, n, b);
            b++;
            main_ahead = false;
            continue;
        }
        main_ahead = true;
    }
    halo_join(h, h->stream);
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaEventRecord(e_loop1, h->stream));
    for (auto& e : lag_ev) cudaEventDestroy(e);

    // ---- exit: status, true residuals (K7), history, copy-back
    DevState* fin = &init;   // reuse the pinned buffer
    CK(cudaMemcpyAsync(fin, h->st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (getenv("BMINRES_DEBUG_STATE")) debug_state(h, "exit");
    {
        seg.mark("loop");
        TimeMark tm(h, PH_RESID);
        if (h->prec.active) {   // f3: the transformed system's residual Rhat_0 - Ahat Yhat
            launch_prec_op(h, h->stream, sp, sp.X, h->M[0], n);
        } else {
            const double* Xe = extended_input(h, sp.X, n, p, h->V[0]);   // (V slots are free now)
            spmm_plain(h, h->kf, sp.rowptr, sp.col, sp.val, Xe, h->M[0], n, h->stream, h->tpw);
        }
        launch_colsq(h, B, h->M[0], n, p, h->dsc);
    }
    std::vector<double> r2(p);
    CK(cudaMemcpyAsync(r2.data(), h->dsc, p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    if (x_host) CK(cudaMemcpyAsync(Xin, sp.X, panel * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaEventRecord(e_solve1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    bminres_stats_t& s = h->stats;
    s.status = fin->status;
    s.p = p;
    s.n = n;
    s.iterations = fin->j_done;
    s.block_steps = fin->k_side - 1;
    s.slow_blocks = h->slow_blocks;
    s.n_events = (int64_t)h->events.size();
    for (int c = 0; c < p; ++c) {
        s.comp_res[c] = fin->res[c];
        s.true_res[c] = beta[c] > 0 ? std::sqrt(r2[c]) / beta[c] : 0.0;
    }
    s.history_len = std::min<long long>(fin->j_done + 1, hist_cap);
    h->hist_host.assign((size_t)s.history_len * p, 0.0);
    if (s.history_len)
        CK(cudaMemcpy(h->hist_host.data(), h->hist, h->hist_host.size() * sizeof(double), cudaMemcpyDeviceToHost));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e_solve0, e_solve1));
    s.solve_ms = ms;
    CK(cudaEventElapsedTime(&ms, e_loop0, e_loop1));
    s.loop_ms = ms;
    for (auto& mk : h->ev_marks) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, h->evpool[mk.second], h->evpool[mk.second + 1]));
        s.phase_ms[mk.first] += t;
        s.phase_launches[mk.first] += 1;
    }
    s.gpu_launches = h->launches;
    if (trace_env && getenv("BMINRES_TRACE_FILE")) {
        std::vector<unsigned long long> tb(trace_elems);
        CK(cudaMemcpy(tb.data(), h->trace, trace_elems * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(getenv("BMINRES_TRACE_FILE"), "wb")) {
            fwrite(tb.data(), sizeof(unsigned long long), tb.size(), f);
            fclose(f);
        }
    }
    const double abytes = 12.0 * A->nnz + 4.0 * (n + 1);
    s.bytes_per_block_step = abytes + 10.0 * 8.0 * (double)panel;   // SURVEY §8(d) algorithmic model
    s.spmm_bytes_per_launch = abytes + 3.0 * 8.0 * (double)panel;
    cudaEventDestroy(e_solve0);
    cudaEventDestroy(e_solve1);
    cudaEventDestroy(e_loop0);
    cudaEventDestroy(e_loop1);
    for (auto& r : h->retained) cudaFree(r.v);
    h->retained.clear();
    return fin->status;
}


// ------------------------------------------------------------------ f3: IC(0) split preconditioning
// (reading R8 and "Preconditioning")

void free_sched(bminres_ctx::Sched& sc) {
    if (sc.order) cudaFree(sc.order);
    if (sc.tstart) cudaFree(sc.tstart);
    sc = bminres_ctx::Sched{};
}

void prec_free(bminres_ctx* h) {
    auto& pr = h->prec;
    for (int* q : {pr.Lp, pr.Li, pr.Up, pr.Ui, pr.Uperm})
        if (q) cudaFree(q);
    for (double* q : {pr.Lx, pr.Ux, pr.Bh, pr.Yh, pr.Z})
        if (q) cudaFree(q);
    if (pr.flags) cudaFree(pr.flags);
    if (pr.ctl) cudaFree(pr.ctl);
    free_sched(pr.fs);
    free_sched(pr.bs);
    free_sched(pr.fac);
    const unsigned gen = pr.gen;
    pr = bminres_ctx::Prec{};
    pr.gen = gen + 1;
}

// Rows sorted by level (ascending row within a level) and tasks of at most rpw rows that never
// cross a level (the rows of one task are independent); host analysis, setup only.
void build_sched(bminres_ctx* h, bminres_ctx::Sched& sc, const std::vector<int>& lev, int nlev, int rpw) {
    free_sched(sc);
    const long long n = (long long)lev.size();
    std::vector<long long> cnt((size_t)nlev + 1, 0);
    for (int l : lev) cnt[(size_t)l + 1]++;
    for (int l = 0; l < nlev; ++l) cnt[(size_t)l + 1] += cnt[(size_t)l];
    std::vector<int> order((size_t)n);
    {
        std::vector<long long> pos(cnt.begin(), cnt.end() - 1);
        for (long long i = 0; i < n; ++i) order[(size_t)pos[(size_t)lev[(size_t)i]]++] = (int)i;
    }
    std::vector<int> ts;
    ts.reserve((size_t)(n / rpw + nlev + 1));
    for (int l = 0; l < nlev; ++l)
        for (long long r = cnt[(size_t)l]; r < cnt[(size_t)l + 1]; r += rpw) ts.push_back((int)r);
    ts.push_back((int)n);
    CK(cudaMalloc((void**)&sc.order, std::max<size_t>(1, (size_t)n) * sizeof(int)));
    CK(cudaMalloc((void**)&sc.tstart, ts.size() * sizeof(int)));
    CK(cudaMemcpy(sc.order, order.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(sc.tstart, ts.data(), ts.size() * sizeof(int), cudaMemcpyHostToDevice));
    sc.ntask = (long long)ts.size() - 1;
    sc.rpw = rpw;
}

// IC(0) of M: host analysis (pattern of M's lower triangle, the forward and backward level DAGs,
// the pattern of U = L^T), then the numeric factorisation on the device (k_ic0) and U's values.
void prec_setup(bminres_ctx* h, const bminres_csr* M) {
    if (h->opt.world != 1) fail(h, BMINRES_EINVAL, "preconditioning is single-rank only");
    const long long n = M->n;
    if (n < 1 || M->n_loc != n || M->row_begin != 0) fail(h, BMINRES_EINVAL, "M: n_loc = n >= 1, row_begin = 0");
    if (M->nnz < n || M->nnz >= (1ll << 31) || n >= (1ll << 31))
        fail(h, BMINRES_EINVAL, "M: nnz must be in [n, 2^31)");
    if (!M->row_ptr || !M->col_idx || !M->values) fail(h, BMINRES_EINVAL, "M: null array");
    CK(cudaSetDevice(h->device));
    std::vector<int> rp((size_t)n + 1), ci((size_t)M->nnz);
    std::vector<double> va((size_t)M->nnz);
    CK(cudaMemcpy(rp.data(), M->row_ptr, rp.size() * sizeof(int), cudaMemcpyDefault));
    CK(cudaMemcpy(ci.data(), M->col_idx, ci.size() * sizeof(int), cudaMemcpyDefault));
    CK(cudaMemcpy(va.data(), M->values, va.size() * sizeof(double), cudaMemcpyDefault));
    if (rp[0] != 0 || rp[(size_t)n] != M->nnz) fail(h, BMINRES_EINVAL, "M: row_ptr[0] = 0, row_ptr[n] = nnz");
    std::vector<int> Lp((size_t)n + 1, 0), Li;
    std::vector<double> Lx;
    Li.reserve((size_t)(M->nnz / 2 + n));
    Lx.reserve((size_t)(M->nnz / 2 + n));
    for (long long i = 0; i < n; ++i) {
        if (rp[(size_t)i + 1] < rp[(size_t)i]) fail(h, BMINRES_EINVAL, "M: row_ptr not monotone");
        int prev = -1;
        for (int k = rp[(size_t)i]; k < rp[(size_t)i + 1]; ++k) {
            const int c = ci[(size_t)k];
            if (c <= prev || c >= n) fail(h, BMINRES_EINVAL, "M: columns must be strictly increasing and < n");
            prev = c;
            if (c <= i) {
                Li.push_back(c);
                Lx.push_back(va[(size_t)k]);
            }
        }
        Lp[(size_t)i + 1] = (int)Li.size();
        if (Lp[(size_t)i + 1] == Lp[(size_t)i] || Li.back() != i)
            fail(h, BMINRES_EINVAL, "M: no diagonal entry in row " + std::to_string(i));
    }
    const long long nzl = (long long)Li.size();
    // levels: forward (row i after the rows j < i of its L row), backward (after j > i of its U row)
    std::vector<int> lf((size_t)n, 0), lb((size_t)n, 0);
    int nlf = 0, nlb = 0;
    for (long long i = 0; i < n; ++i) {
        int l = 0;
        for (int e = Lp[(size_t)i]; e < Lp[(size_t)i + 1] - 1; ++e) l = std::max(l, lf[(size_t)Li[(size_t)e]] + 1);
        lf[(size_t)i] = l;
        nlf = std::max(nlf, l + 1);
    }
    std::vector<int> Up((size_t)n + 1, 0), Ui((size_t)nzl), Uperm((size_t)nzl);
    for (long long e = 0; e < nzl; ++e) Up[(size_t)Li[(size_t)e] + 1]++;
    for (long long i = 0; i < n; ++i) Up[(size_t)i + 1] += Up[(size_t)i];
    {
        std::vector<int> fill((size_t)n, 0);
        for (long long i = 0; i < n; ++i)   // rows of L ascending: each U row ascending, diagonal first
            for (int e = Lp[(size_t)i]; e < Lp[(size_t)i + 1]; ++e) {
                const int c = Li[(size_t)e];
                const int d = Up[(size_t)c] + fill[(size_t)c]++;
                Ui[(size_t)d] = (int)i;
                Uperm[(size_t)d] = e;
            }
    }
    for (long long i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int e = Up[(size_t)i] + 1; e < Up[(size_t)i + 1]; ++e) l = std::max(l, lb[(size_t)Ui[(size_t)e]] + 1);
        lb[(size_t)i] = l;
        nlb = std::max(nlb, l + 1);
    }
    prec_free(h);
    auto& pr = h->prec;
    try {
        CK(cudaMalloc((void**)&pr.Lp, Lp.size() * sizeof(int)));
        CK(cudaMalloc((void**)&pr.Li, (size_t)nzl * sizeof(int)));
        CK(cudaMalloc((void**)&pr.Lx, (size_t)nzl * sizeof(double)));
        CK(cudaMalloc((void**)&pr.Up, Up.size() * sizeof(int)));
        CK(cudaMalloc((void**)&pr.Ui, (size_t)nzl * sizeof(int)));
        CK(cudaMalloc((void**)&pr.Uperm, (size_t)nzl * sizeof(int)));
        CK(cudaMalloc((void**)&pr.Ux, (size_t)nzl * sizeof(double)));
        CK(cudaMalloc((void**)&pr.flags, (size_t)n * sizeof(unsigned)));
        CK(cudaMalloc((void**)&pr.ctl, sizeof(TriCtl)));
        CK(cudaMemcpy(pr.Lp, Lp.data(), Lp.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pr.Li, Li.data(), (size_t)nzl * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pr.Lx, Lx.data(), (size_t)nzl * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pr.Up, Up.data(), Up.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pr.Ui, Ui.data(), (size_t)nzl * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pr.Uperm, Uperm.data(), (size_t)nzl * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemset(pr.flags, 0, (size_t)n * sizeof(unsigned)));
        TriCtl c0{0u, 0u, 0x7fffffff, 0};
        CK(cudaMemcpy(pr.ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice));
        pr.n = n;
        pr.nnzl = nzl;
        pr.levels_f = nlf;
        pr.levels_b = nlb;
        pr.lev_f = std::move(lf);
        pr.lev_b = std::move(lb);
        build_sched(h, pr.fac, pr.lev_f, nlf, 1);
        // numeric IC(0): one thread per row, a persistent grid within the resident capacity
        TriArgs a{};
        a.Tp = pr.Lp;
        a.Ti = pr.Li;
        a.Tx = pr.Lx;
        a.flags = pr.flags;
        a.ctl = pr.ctl;
        a.s = TriSched{pr.fac.order, pr.fac.tstart, pr.fac.ntask};
        a.n = n;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k_ic0, NT, 0);
        const long long cap = std::max(1ll, (long long)h->n_sm * std::max(1, occ) - 1);
        const int grid = (int)std::max(1ll, std::min(cap, (n + NT - 1) / NT));
        k_ic0<<<grid, NT, 0, h->stream>>>(a);
        check_launch(h, "k_ic0");
        k_gather_vals<<<grid_for(h, nzl, 256, 8 * h->n_sm), 256, 0, h->stream>>>(pr.Lx, pr.Uperm, pr.Ux, nzl);
        check_launch(h, "k_gather_vals");
        TriCtl c1{};
        CK(cudaMemcpyAsync(&c1, pr.ctl, sizeof(c1), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (c1.bad_row != 0x7fffffff)
            fail(h, BMINRES_EPIVOT, "IC(0) pivot <= 0 at row " + std::to_string(c1.bad_row));
        pr.on = true;
    } catch (Err&) {
        prec_free(h);
        throw;
    }
}

// panels and this p's task lists
void prec_ensure(bminres_ctx* h, int p) {
    auto& pr = h->prec;
    const size_t panel = (size_t)pr.n * p + 32;
    if (pr.panel_cap < panel) {
        dalloc(h, &pr.Bh, panel);
        dalloc(h, &pr.Yh, panel);
        dalloc(h, &pr.Z, panel);
        CK(cudaMemsetAsync(pr.Z, 0, panel * sizeof(double), h->stream));
        pr.panel_cap = panel;
    }
    const int vec = (p % 2 == 0) ? 2 : 1, lanes = p / vec;
    int lp = 1;
    while (lp < lanes) lp <<= 1;
    const int rpw = 32 / lp;   // PC<P>::RPW
    if (pr.fs.rpw != rpw) {
        build_sched(h, pr.fs, pr.lev_f, pr.levels_f, rpw);
        build_sched(h, pr.bs, pr.lev_b, pr.levels_b, rpw);
    }
}

// Preconditioned solve (reading R8): Rhat_0 = L^-1 (B - A X_0); the core solve (do_solve) on
// (L^-1 A L^-T, Rhat_0) from Yhat_0 = 0; X = X_0 + L^-T Yhat.
int do_solve_prec(bminres_ctx* h, const bminres_csr* A, const double* Bin, double* Xin, int p, double tol,
                  long long maxit, double tau) {
    auto& pr = h->prec;
    const bminres_options o = h->opt;
    if (!A || !Bin || !Xin) fail(h, BMINRES_EINVAL, "null argument");
    if (o.world != 1) fail(h, BMINRES_EINVAL, "preconditioning is single-rank only");
    if (A->n != pr.n || A->n_loc != pr.n || A->row_begin != 0)
        fail(h, BMINRES_EINVAL, "A and the preconditioner M differ in size");
    Kfn f;
    if (p < 1 || p > BMINRES_MAX_P || !kfn_for(p, &f, o.pool_size)) fail(h, BMINRES_EINVAL, "unsupported block size p");
    const long long n = pr.n;
    if (n < p) fail(h, BMINRES_EINVAL, "n < p");
    if (A->nnz < 0 || A->nnz >= (1ll << 31)) fail(h, BMINRES_EINVAL, "nnz must be < 2^31");
    CK(cudaSetDevice(h->device));
    const size_t panel = (size_t)n * p;
    h->launches = 0;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h->stream));
    // host inputs are staged here, so the core sees device pointers
    bminres_csr Ad = *A;
    if (!(is_device_ptr(A->row_ptr) && is_device_ptr(A->col_idx) && is_device_ptr(A->values))) {
        if (h->a_rows_cap < (size_t)n + 1) {
            dalloc(h, &h->a_rowptr, n + 1);
            h->a_rows_cap = n + 1;
        }
        if (h->a_nnz_cap < (size_t)std::max<long long>(A->nnz, 1)) {
            dalloc(h, &h->a_col, std::max<long long>(A->nnz, 1));
            dalloc(h, &h->a_val, std::max<long long>(A->nnz, 1));
            h->a_nnz_cap = std::max<long long>(A->nnz, 1);
        }
        CK(cudaMemcpyAsync(h->a_rowptr, A->row_ptr, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(h->a_col, A->col_idx, A->nnz * sizeof(int), cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(h->a_val, A->values, A->nnz * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        Ad.row_ptr = h->a_rowptr;
        Ad.col_idx = h->a_col;
        Ad.values = h->a_val;
    }
    const double* B = Bin;
    if (!is_device_ptr(Bin)) {
        if (h->bx_cap < panel) {
            dalloc(h, &h->bx, panel);
            h->bx_cap = panel;
        }
        CK(cudaMemcpyAsync(h->bx, Bin, panel * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        B = h->bx;
    }
    double* X = Xin;
    const bool x_host = !is_device_ptr(Xin);
    if (x_host) {
        if (h->xx_cap < panel) {
            dalloc(h, &h->xx, panel);
            h->xx_cap = panel;
        }
        if (o.use_x0) CK(cudaMemcpyAsync(h->xx, Xin, panel * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        X = h->xx;
    }
    if ((((uintptr_t)B) | ((uintptr_t)X)) & 15) fail(h, BMINRES_EINVAL, "B and X must be 16-byte aligned");
    prec_ensure(h, p);
    StepPtrs sp{};
    sp.rowptr = Ad.row_ptr;
    sp.col = Ad.col_idx;
    sp.val = Ad.values;
    // Rhat_0 = L^-1 (B - A X_0)
    const double* R0 = B;
    if (o.use_x0) {
        spmm_plain(h, f, sp.rowptr, sp.col, sp.val, X, pr.Z, n, h->stream, h->tpw);
        k_sub_from<<<grid_for(h, panel, 256, 8 * h->n_sm), 256, 0, h->stream>>>(B, pr.Z, (long long)panel);
        check_launch(h, "k_sub_from");
        R0 = pr.Z;
    }
    launch_trsv(h, h->stream, f.tfwdp, pr.fs, false, nullptr, R0, pr.Bh, n);
    const long long pre_launches = h->launches;
    // the core solve on the transformed system
    h->opt.use_x0 = 0;
    pr.active = true;
    int r;
    try {
        r = do_solve(h, &Ad, pr.Bh, pr.Yh, p, tol, maxit, tau);
    } catch (Err&) {
        h->opt.use_x0 = o.use_x0;
        pr.active = false;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    h->opt.use_x0 = o.use_x0;
    pr.active = false;
    const long long core_launches = h->launches;
    // X = X_0 + L^-T Yhat; the unpreconditioned true residual ||b_i - A x_i|| / ||b_i||
    launch_trsv(h, h->stream, f.tbwd, pr.bs, true, nullptr, pr.Yh, pr.Z, n);
    k_add_panel<<<grid_for(h, panel, 256, 8 * h->n_sm), 256, 0, h->stream>>>(X, pr.Z, (long long)panel, o.use_x0);
    check_launch(h, "k_add_panel");
    spmm_plain(h, f, sp.rowptr, sp.col, sp.val, X, pr.Z, n, h->stream, h->tpw);
    std::vector<double> r2(p), b2(p);
    launch_colsq(h, B, pr.Z, n, p, h->dsc);
    CK(cudaMemcpyAsync(r2.data(), h->dsc, p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    launch_colsq(h, B, nullptr, n, p, h->dsc);
    CK(cudaMemcpyAsync(b2.data(), h->dsc, p * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    if (x_host) CK(cudaMemcpyAsync(Xin, X, panel * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaEventRecord(e1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    bminres_stats_t& s = h->stats;
    for (int c = 0; c < p; ++c) {
        s.prec_true_res[c] = s.true_res[c];
        s.true_res[c] = b2[c] > 0 ? std::sqrt(r2[c]) / std::sqrt(b2[c]) : 0.0;
    }
    s.preconditioned = 1;
    s.prec_levels = pr.levels_f;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    s.solve_ms = ms;
    s.gpu_launches += pre_launches + (h->launches - core_launches);   // (the core counted its own)
    // the triangular factors (fp64 + int32 entries, int32 row offsets) are read twice per block step,
    // and Z = L^-T V_k is written once and gathered once
    s.bytes_per_block_step += 2.0 * (12.0 * (double)pr.nnzl + 4.0 * (double)(n + 1)) + 2.0 * 8.0 * (double)panel;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return r;
}
}  // namespace

// ================================================================== C ABI

extern "C" {

void bminres_default_options(bminres_options* opt) {
    if (!opt) return;
    std::memset(opt, 0, sizeof(*opt));
    opt->device = 0;
    opt->rank = 0;
    opt->world = 1;
    opt->stream = nullptr;
    opt->seed = 0;
    opt->pool_size = 1;
    opt->use_x0 = 0;
    opt->record_history = 1;
    opt->use_graphs = 1;
    opt->timing = 0;
}

int bminres_create(const bminres_options* opt, bminres_handle* out) {
    if (!out) return BMINRES_EINVAL;
    *out = nullptr;
    bminres_options o;
    if (opt)
        o = *opt;
    else
        bminres_default_options(&o);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        g_create_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return BMINRES_ECUDA;
    }
    if (o.device < 0 || o.device >= ndev) {
        g_create_err = "bad device ordinal";
        return BMINRES_EINVAL;
    }
    if (o.split_spmm < 0 || o.split_spmm > 2) {
        g_create_err = "split_spmm must be 0 (auto), 1 (always) or 2 (never)";
        return BMINRES_EINVAL;
    }
    if (o.policy != 0 && o.policy != 1) {
        g_create_err = "policy must be 0 (replacement, P:690-729) or 1 (block-size reduction, P:582-688)";
        return BMINRES_EINVAL;
    }
    if (o.coeff_mode != 0) {
        g_create_err = "coeff_mode: only 0 (symmetric reuse, P:270-272) is built";
        return BMINRES_EINVAL;
    }
    auto* h = new bminres_ctx();
    h->opt = o;
    h->device = o.device;
    try {
        CK(cudaSetDevice(o.device));
        CK(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, o.device));
        int coop = 0;
        CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, o.device));
        h->coop_ok = coop != 0;
        if (o.stream) {
            h->stream = (cudaStream_t)o.stream;
        } else {
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        // the side branch (K3b: one CTA, serial) gets the highest stream priority so its CTA is
        // dispatched ahead of the main-branch grids
        int prio_lo = 0, prio_hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        h->prio_hi = prio_hi;
        CK(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, prio_hi));
        CK(cudaStreamCreateWithPriority(&h->ustream, cudaStreamNonBlocking, prio_hi));
        CK(cudaStreamCreateWithPriority(&h->hstream, cudaStreamNonBlocking, prio_hi));
        CK(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_u0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_u1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        // large dynamic shared memory for the p = 32 kernels
        for (int p : {1, 2, 3, 4, 5, 6, 7, 8, 16, 32})
            for (int qv : {0, MAXQ}) {   // (the K2 variant depends on the pool size)
            Kfn f;
            kfn_for(p, &f, qv);
            CK(cudaFuncSetAttribute((const void*)f.k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem1));
            if (f.k1pre)
                CK(cudaFuncSetAttribute((const void*)f.k1pre, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)f.smem1pre));
            if (f.k1u)
                CK(cudaFuncSetAttribute((const void*)f.k1u, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)f.smem1u));
            if (f.k1ws)
                CK(cudaFuncSetAttribute((const void*)f.k1ws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)f.smem1ws));
            CK(cudaFuncSetAttribute((const void*)f.k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem2));
            CK(cudaFuncSetAttribute((const void*)f.k3b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem3));
            CK(cudaFuncSetAttribute((const void*)f.k4b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem4b));
        }
    } catch (Err& x) {
        g_create_err = h->err;
        delete h;
        return x.code;
    }
    *out = h;
    return BMINRES_OK;
}

int bminres_solve(bminres_handle h, const bminres_csr* A, const double* B, double* X, int32_t p, double tol,
                  int64_t maxit, double deflation_tol) {
    if (!h) return BMINRES_EINVAL;
    try {
        int r = h->prec.on ? do_solve_prec(h, A, B, X, p, tol, maxit, deflation_tol)
                           : do_solve(h, A, B, X, p, tol, maxit, deflation_tol);
        h->stats.status = r;
        return r;
    } catch (Err& x) {
        h->stats.status = x.code;
        return x.code;
    }
}

int bminres_stats(bminres_handle h, bminres_stats_t* out) {
    if (!h || !out) return BMINRES_EINVAL;
    *out = h->stats;
    return BMINRES_OK;
}

int64_t bminres_get_history(bminres_handle h, double* buf, int64_t cap) {
    if (!h || !buf || cap <= 0) return 0;
    int64_t rows = std::min<int64_t>(cap, h->stats.history_len);
    std::memcpy(buf, h->hist_host.data(), (size_t)rows * h->stats.p * sizeof(double));
    return rows;
}

int64_t bminres_get_events(bminres_handle h, bminres_event* buf, int64_t cap) {
    if (!h || !buf || cap <= 0) return 0;
    int64_t c = std::min<int64_t>(cap, (int64_t)h->events.size());
    std::memcpy(buf, h->events.data(), (size_t)c * sizeof(bminres_event));
    return c;
}

int bminres_spmm(bminres_handle h, const bminres_csr* A, const double* X, double* Y, int32_t p) {
    if (!h || !A || !X || !Y) return BMINRES_EINVAL;
    try {
        Kfn f;
        if (!kfn_for(p, &f)) fail(h, BMINRES_EINVAL, "unsupported block size p");
        if (!is_device_ptr(A->row_ptr) || !is_device_ptr(A->col_idx) || !is_device_ptr(A->values) ||
            !is_device_ptr(X) || !is_device_ptr(Y))
            fail(h, BMINRES_EINVAL, "bminres_spmm takes device pointers");
        if ((((uintptr_t)X) | ((uintptr_t)Y)) & 15) fail(h, BMINRES_EINVAL, "X and Y must be 16-byte aligned");
        CK(cudaSetDevice(h->device));
        const long long n = A->n_loc;
        const int vec = (p % 2 == 0) ? 2 : 1, lanes = p / vec;
        int lp = 1;
        while (lp < lanes) lp <<= 1;
        const long long rpw = 32 / lp, ntiles = (n + rpw - 1) / rpw, warps = NT / 32;
        const int tpw = (int)std::max<long long>(4, (ntiles + warps * 65536 - 1) / (warps * 65536));
        spmm_plain(h, f, A->row_ptr, A->col_idx, A->values, X, Y, n, h->stream, tpw);
        CK(cudaStreamSynchronize(h->stream));
        return BMINRES_OK;
    } catch (Err& x) {
        return x.code;
    }
}

int bminres_random_vector(bminres_handle h, uint64_t seed, uint64_t stream, uint64_t event, int64_t row_begin,
                          int64_t n_loc, double* out, int64_t stride) {
    if (!h || !out) return BMINRES_EINVAL;
    try {
        if (!is_device_ptr(out)) fail(h, BMINRES_EINVAL, "bminres_random_vector takes a device pointer");
        CK(cudaSetDevice(h->device));
        launch_rand(h, out, stride, n_loc, row_begin, seed, stream, event);
        CK(cudaStreamSynchronize(h->stream));
        return BMINRES_OK;
    } catch (Err& x) {
        return x.code;
    }
}

size_t bminres_workspace_bytes(int64_t n_loc, int32_t p, int32_t pool_size) {
    // the allocations of ensure_workspace / do_solve (single rank; a row partition adds n_halo rows
    // to each V slot), as an upper bound: V[3], M[2] and the pool (each with 32 doubles of slack),
    // the split-mode AV panel (same rule as ensure_workspace), the partial-sum buffers, the history
    // at its cap (8 Mi doubles), the two column-path scratch panels (allocated on the first
    // breakdown only), the small buffers and the state
    const size_t panel = (size_t)n_loc * p + 32;
    Kfn f;
    const bool split = kfn_for(p, &f, pool_size) && f.k1pre != nullptr && (double)n_loc * p * 8.0 >= 128e6;
    const size_t part = (size_t)NB_MAX * (MAXP * MAXP + MAXQ * MAXP + MAXREF + 8) +
                        (size_t)NB_MAX * (MAXP * MAXP + MAXP) + 2 * (size_t)NB_MAX * (MAXP * MAXP + MAXQ * MAXP);
    const size_t hist = std::min<size_t>((size_t)8 << 20, (size_t)std::max(p, 1) * ((8ull << 20) / std::max(p, 1)));
    size_t d = 5 * panel + (split ? panel : 0) + (size_t)n_loc * std::max(pool_size, 1) + 32 + part + hist +
               2 * panel + (MAXREF + 64) + 2 * MAXP * MAXP + (MAXP * MAXP + 3 * MAXP);
    return sizeof(double) * d + 16 * sizeof(unsigned) + sizeof(DevState);
}

int bminres_get_unique_id(uint8_t out[128]) {
    if (!out) return BMINRES_EINVAL;
    std::string err;
    NcclApi& a = nccl_api();
    if (!a.load(err)) {
        g_create_err = err;
        return BMINRES_ENCCL;
    }
    const int r = a.getUniqueId(out);
    if (r != 0) {
        g_create_err = "ncclGetUniqueId failed";
        return BMINRES_ENCCL;
    }
    return BMINRES_OK;
}

int bminres_init_nccl(bminres_handle h, const uint8_t id[128]) {
    if (!h || !id) return BMINRES_EINVAL;
    if (h->opt.world < 1 || h->opt.rank < 0 || h->opt.rank >= h->opt.world) return BMINRES_EINVAL;
    cudaSetDevice(h->device);
    auto* t = new NcclTransport();
    std::string err;
    if (!t->init(id, h->opt.rank, h->opt.world, err)) {
        delete t;
        h->err = err;
        return BMINRES_ENCCL;
    }
    delete h->tp;
    h->tp = t;
    return BMINRES_OK;
}

int bminres_set_comm_callbacks(bminres_handle h, const bminres_comm_callbacks* cb) {
    if (!h || !cb || !cb->allreduce || !cb->alltoallv || !cb->exchange) return BMINRES_EINVAL;
    auto* t = new CallbackTransport();
    t->cb = *cb;
    t->rank = h->opt.rank;
    t->world = h->opt.world;
    delete h->tp;
    h->tp = t;
    return BMINRES_OK;
}

int bminres_halo_plan(int32_t world, int32_t rank, const int64_t* offsets, int64_t nnz, const int32_t* col_idx,
                      int32_t* local_col, int64_t* halo_rows, int64_t* n_halo, int64_t* halo_count) {
    if (world < 1 || rank < 0 || rank >= world || !offsets || nnz < 0 || (nnz > 0 && !col_idx) || !n_halo)
        return BMINRES_EINVAL;
    for (int q = 0; q < world; ++q)
        if (offsets[q + 1] < offsets[q]) return BMINRES_EINVAL;
    HaloPlan pl;
    if (!build_halo_plan(world, rank, reinterpret_cast<const long long*>(offsets), nnz, col_idx, pl))
        return BMINRES_EINVAL;
    *n_halo = pl.n_halo;
    if (local_col) std::copy(pl.local_col.begin(), pl.local_col.end(), local_col);
    if (halo_rows) std::copy(pl.halo_rows.begin(), pl.halo_rows.end(), halo_rows);
    if (halo_count) std::copy(pl.recv_count.begin(), pl.recv_count.end(), halo_count);
    return BMINRES_OK;
}

int bminres_interior_rows(int64_t n_loc, const int32_t* row_ptr, const int32_t* local_col, int64_t* lo, int64_t* hi) {
    if (n_loc < 0 || !row_ptr || (n_loc > 0 && row_ptr[n_loc] > 0 && !local_col) || !lo || !hi) return BMINRES_EINVAL;
    long long l = 0, u = 0;
    interior_rows(n_loc, row_ptr, local_col, &l, &u);
    *lo = l;
    *hi = u;
    return BMINRES_OK;
}

int bminres_set_preconditioner(bminres_handle h, const bminres_csr* M) {
    if (!h) return BMINRES_EINVAL;
    try {
        if (!M) {
            prec_free(h);
            return BMINRES_OK;
        }
        prec_setup(h, M);
        return BMINRES_OK;
    } catch (Err& x) {
        return x.code;
    }
}

int64_t bminres_get_preconditioner(bminres_handle h, double* l_values, int64_t cap) {
    if (!h || !h->prec.on) return 0;
    if (!l_values || cap <= 0) return h->prec.nnzl;
    const int64_t c = std::min<int64_t>(cap, h->prec.nnzl);
    if (cudaMemcpy(l_values, h->prec.Lx, (size_t)c * sizeof(double), cudaMemcpyDefault) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return h->prec.nnzl;
}

int bminres_precond_apply(bminres_handle h, const bminres_csr* A, const double* X, double* Y, int32_t p,
                          int32_t mode) {
    if (!h || !X || !Y) return BMINRES_EINVAL;
    try {
        if (!h->prec.on) fail(h, BMINRES_EINVAL, "no preconditioner set");
        Kfn f;
        if (!kfn_for(p, &f)) fail(h, BMINRES_EINVAL, "unsupported block size p");
        if (mode < 0 || mode > 2) fail(h, BMINRES_EINVAL, "mode must be 0, 1 or 2");
        if (!is_device_ptr(X) || !is_device_ptr(Y)) fail(h, BMINRES_EINVAL, "bminres_precond_apply takes device pointers");
        if ((((uintptr_t)X) | ((uintptr_t)Y)) & 15) fail(h, BMINRES_EINVAL, "X and Y must be 16-byte aligned");
        if (mode == 2 && (!A || A->n != h->prec.n || A->n_loc != h->prec.n || !is_device_ptr(A->row_ptr) ||
                          !is_device_ptr(A->col_idx) || !is_device_ptr(A->values)))
            fail(h, BMINRES_EINVAL, "mode 2 needs the n x n operator A in device memory");
        CK(cudaSetDevice(h->device));
        prec_ensure(h, p);
        const long long n = h->prec.n;
        if (mode == 0) {
            launch_trsv(h, h->stream, f.tfwdp, h->prec.fs, false, nullptr, X, Y, n);
        } else if (mode == 1) {
            launch_trsv(h, h->stream, f.tbwd, h->prec.bs, true, nullptr, X, Y, n);
        } else {
            StepPtrs sp{};
            sp.rowptr = A->row_ptr;
            sp.col = A->col_idx;
            sp.val = A->values;
            const Kfn keep = h->kf;
            h->kf = f;
            launch_prec_op(h, h->stream, sp, X, Y, n);
            h->kf = keep;
        }
        CK(cudaStreamSynchronize(h->stream));
        return BMINRES_OK;
    } catch (Err& x) {
        return x.code;
    }
}

const char* bminres_last_error(bminres_handle h) {
    if (!h) return g_create_err.c_str();
    return h->err.c_str();
}

void bminres_destroy(bminres_handle h) {
    if (!h) return;
    cudaSetDevice(h->device);
    prec_free(h);
    for (int s = 0; s < 6; ++s)
        if (h->gexec[s]) cudaGraphExecDestroy(h->gexec[s]);
    for (double* p : {h->V[0], h->V[1], h->V[2], h->M[0], h->M[1], h->AV, h->scr[0], h->scr[1], h->pool, h->part, h->dsc,
                      h->gdev, h->a_val, h->bx, h->xx, h->hist})
        if (p) cudaFree(p);
    if (h->trace) cudaFree(h->trace);
    if (h->trace_tick) cudaFree(h->trace_tick);
    if (h->d_lcol) cudaFree(h->d_lcol);
    if (h->d_send_rows) cudaFree(h->d_send_rows);
    if (h->d_sendbuf) cudaFree(h->d_sendbuf);
    delete h->tp;
    if (h->a_rowptr) cudaFree(h->a_rowptr);
    if (h->a_col) cudaFree(h->a_col);
    if (h->dcnt) cudaFree(h->dcnt);
    if (h->st) cudaFree(h->st);
    if (h->hf) cudaFreeHost(h->hf);
    for (auto& r : h->retained) cudaFree(r.v);
    for (auto& e : h->evpool) cudaEventDestroy(e);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ustream) cudaStreamDestroy(h->ustream);
    if (h->hstream) cudaStreamDestroy(h->hstream);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_halo) cudaEventDestroy(h->ev_halo);
    if (h->ev_u0) cudaEventDestroy(h->ev_u0);
    if (h->ev_u1) cudaEventDestroy(h->ev_u1);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->startbuf) cudaFree(h->startbuf);
    if (h->hstate) cudaFreeHost(h->hstate);
    if (h->ev_a) cudaEventDestroy(h->ev_a);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
}

}  // extern "C"

// comm.cuh -- row-partitioned solves (world > 1).
//
// Rank r owns the contiguous rows [row_begin, row_begin + n_loc) of A, B, X and of every
// panel; ranks are in row order.  Everything in a block step is row-local except
//   (1) the SpMM's halo: K1 gathers V_k rows by column index, some of them owned by other
//       ranks.  The halo plan (built once per operator) lists, per peer, the remote rows this
//       rank reads; the V slots are extended to [n_loc own rows | n_halo halo rows] and the CSR
//       column indices are remapped into that extended panel, so K1 runs unchanged.  After K2
//       writes V_{k+1} (= W', the unnormalised candidates, SURVEY design D2) each rank packs the
//       rows its peers read and the exchange lands them directly in the peers' halo regions;
//   (2) the reductions: the totals of k_reduce (V_k^T W, ||A u_j||^2; W'^T W', r_q^T W') and
//       the start block's / column path's dot products are sum-allreduced.  K3b then runs
//       replicated on bitwise identical inputs.
// Transports: NCCL (dlopen'd libnccl.so.2; capturable in CUDA graphs) for production, and host
// callbacks (e.g. a torch.distributed process group) for testing; callbacks move data through
// host memory and force plain launches.
#pragma once
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bminres.h"
#include "common.cuh"

namespace bmr {

// ------------------------------------------------------------------ halo plan (host)

struct HaloPlan {
    int world = 1, rank = 0;
    long long n_loc = 0, n_halo = 0;
    std::vector<long long> offsets;      // world+1 global row offsets
    std::vector<int> local_col;          // remapped column indices (nnz)
    std::vector<long long> halo_rows;    // global rows of the halo, by owner rank, ascending
    std::vector<long long> recv_count;   // halo rows from each rank
    std::vector<long long> send_rows;    // local rows each peer reads, grouped by peer
    std::vector<long long> send_count;   // rows sent to each rank
};

// Remap GLOBAL column indices into the extended panel [own rows | halo rows].  Returns false on
// a column outside [0, offsets[world]).
inline bool build_halo_plan(int world, int rank, const long long* offsets, long long nnz, const int* col,
                            HaloPlan& pl) {
    pl.world = world;
    pl.rank = rank;
    pl.offsets.assign(offsets, offsets + world + 1);
    const long long rb = offsets[rank], re = offsets[rank + 1], n = offsets[world];
    pl.n_loc = re - rb;
    std::vector<long long> remote;
    for (long long e = 0; e < nnz; ++e) {
        const long long c = col[e];
        if (c < 0 || c >= n) return false;
        if (c < rb || c >= re) remote.push_back(c);
    }
    std::sort(remote.begin(), remote.end());
    remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
    pl.halo_rows = remote;   // ascending global index = grouped by owner (ranks in row order)
    pl.n_halo = (long long)remote.size();
    pl.recv_count.assign(world, 0);
    for (long long c : remote) {
        const int owner = (int)(std::upper_bound(offsets, offsets + world + 1, c) - offsets) - 1;
        pl.recv_count[owner]++;
    }
    pl.local_col.resize(nnz);
    for (long long e = 0; e < nnz; ++e) {
        const long long c = col[e];
        if (c >= rb && c < re) {
            pl.local_col[e] = (int)(c - rb);
        } else {
            const long long pos = std::lower_bound(remote.begin(), remote.end(), c) - remote.begin();
            pl.local_col[e] = (int)(pl.n_loc + pos);
        }
    }
    return true;
}

// The longest run of rows [lo, hi) whose columns are all local (remapped index < n_loc): the
// interior, whose SpMM rows need no halo row.  (lo = hi = 0 when there is none.)
inline void interior_rows(long long n_loc, const int* row_ptr, const int* local_col, long long* lo, long long* hi) {
    long long best_lo = 0, best = 0, cur = 0;
    for (long long i = 0; i < n_loc; ++i) {
        bool in = true;
        for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
            if (local_col[e] >= n_loc) {
                in = false;
                break;
            }
        cur = in ? cur + 1 : 0;
        if (cur > best) {
            best = cur;
            best_lo = i - cur + 1;
        }
    }
    *lo = best_lo;
    *hi = best_lo + best;
}

// ------------------------------------------------------------------ transports

struct Transport {
    virtual ~Transport() {}
    // in-place sum over ranks of count doubles at dev (device memory, stream-ordered on s)
    virtual bool allreduce(double* dev, long long count, cudaStream_t s, std::string& err) = 0;
    // host all-to-all of int64: send (grouped by destination, scount each) -> recv (rcount each)
    virtual bool alltoallv(const long long* send, const long long* scount, long long* recv, const long long* rcount,
                           cudaStream_t s, std::string& err) = 0;
    // device halo exchange: segment of sendbuf for each peer -> segment of recvbuf from each peer
    // (counts in doubles, segments contiguous in rank order)
    virtual bool exchange(const double* sendbuf, const long long* scount, double* recvbuf, const long long* rcount,
                          cudaStream_t s, std::string& err) = 0;
    virtual bool capturable() const = 0;
    int world = 1, rank = 0;
};

// ---- NCCL, resolved at run time (no link-time dependency; the library loads without NCCL)
struct NcclApi {
    void* so = nullptr;
    int (*getUniqueId)(void* id) = nullptr;
    int (*commInitRank)(void** comm, int nranks, char id[128], int rank) = nullptr;   // see call site
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*commSplit)(void* comm, int color, int key, void** newcomm, void* config) = nullptr;   // optional (NCCL >= 2.18)
    const char* (*errStr)(int) = nullptr;
    bool load(std::string& err) {
        if (so) return true;
        const char* env = getenv("BMINRES_NCCL_LIB");
        for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
            if (!name) continue;
            so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (so) break;
        }
        if (!so) {
            err = "libnccl.so.2 not found (set BMINRES_NCCL_LIB)";
            return false;
        }
        getUniqueId = (int (*)(void*))dlsym(so, "ncclGetUniqueId");
        commInitRank = (int (*)(void**, int, char*, int))dlsym(so, "ncclCommInitRank");
        allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(so, "ncclAllReduce");
        send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(so, "ncclSend");
        recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(so, "ncclRecv");
        groupStart = (int (*)())dlsym(so, "ncclGroupStart");
        groupEnd = (int (*)())dlsym(so, "ncclGroupEnd");
        commDestroy = (int (*)(void*))dlsym(so, "ncclCommDestroy");
        commSplit = (int (*)(void*, int, int, void**, void*))dlsym(so, "ncclCommSplit");
        errStr = (const char* (*)(int))dlsym(so, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !allReduce || !send || !recv || !groupStart || !groupEnd ||
            !commDestroy) {
            err = "libnccl.so.2 lacks a required symbol";
            return false;
        }
        return true;
    }
};
inline NcclApi& nccl_api() {
    static NcclApi api;
    return api;
}
constexpr int NCCL_INT64 = 4, NCCL_FLOAT64 = 8, NCCL_SUM = 0;   // nccl.h ncclDataType_t / ncclRedOp_t

// ncclCommInitRank takes the 128-byte ncclUniqueId by value; on x86-64 SysV a 128-byte struct
// argument is passed in memory, so a wrapper type with the same layout is used.
struct NcclId {
    char internal[128];
};

struct NcclTransport : Transport {
    void* comm = nullptr;    // the allreduces (and the plan's all-to-all)
    // The halo exchange gets a communicator of its own (ncclCommSplit of comm, same ranks): NCCL
    // serialises the operations of ONE communicator in issue order even across streams, so with a
    // shared communicator reduce2's allreduce, issued on the main stream right after the exchange
    // went to hstream, would wait for the whole exchange and the overlap with the update and the
    // interior SpMM would start only after it.  Both communicators see their operations in the
    // same order on every rank (the host code is deterministic and K3b's decisions are replicated),
    // and no kernel of the solver spins on another kernel, so the two NCCL kernels can never wait
    // on each other.  Without ncclCommSplit (or with BMINRES_NCCL_ONE_COMM=1) the exchange shares
    // comm (correct, serialised).
    void* hcomm = nullptr;
    long long* dbuf = nullptr;   // device staging of the plan lists
    size_t dcap = 0;
    bool init(const unsigned char id[128], int rank_, int world_, std::string& err) {
        // The allreduces' summation order must be fixed (bitwise reproducible runs,
        // and every rank's replicated small QR depends on it): pin the ring algorithm and the LL
        // protocol (the allreduced buffers are <= 9 KB, where LL is also the fastest) unless the
        // caller set them.  (NCCL_PROTO applies to collectives only; the halo send/recv keep
        // NCCL's own point-to-point protocol choice.)
        setenv("NCCL_ALGO", "Ring", 0);
        setenv("NCCL_PROTO", "LL", 0);
        NcclApi& a = nccl_api();
        if (!a.load(err)) return false;
        rank = rank_;
        world = world_;
        NcclId nid;
        std::memcpy(nid.internal, id, 128);
        auto fn = reinterpret_cast<int (*)(void**, int, NcclId, int)>(a.commInitRank);
        const int r = fn(&comm, world, nid, rank);
        if (r != 0) {
            err = std::string("ncclCommInitRank: ") + (a.errStr ? a.errStr(r) : std::to_string(r));
            return false;
        }
        const char* one = getenv("BMINRES_NCCL_ONE_COMM");
        if (a.commSplit && !(one && one[0] == '1')) {
            // (collective; a failure is an error rather than a silent fallback, which could leave
            // the ranks with different communicators for the same exchange)
            const int r2 = a.commSplit(comm, 0, rank, &hcomm, nullptr);
            if (r2 != 0) {
                hcomm = nullptr;
                err = std::string("ncclCommSplit (halo communicator; BMINRES_NCCL_ONE_COMM=1 shares one): ") +
                      (a.errStr ? a.errStr(r2) : std::to_string(r2));
                return false;
            }
        }
        return true;
    }
    bool two_comms() const { return hcomm != nullptr; }
    ~NcclTransport() override {
        if (hcomm) nccl_api().commDestroy(hcomm);
        if (comm) nccl_api().commDestroy(comm);
        if (dbuf) cudaFree(dbuf);
    }
    bool check(int r, const char* what, std::string& err) {
        if (r == 0) return true;
        err = std::string(what) + ": " + (nccl_api().errStr ? nccl_api().errStr(r) : std::to_string(r));
        return false;
    }
    bool allreduce(double* dev, long long count, cudaStream_t s, std::string& err) override {
        return check(nccl_api().allReduce(dev, dev, (size_t)count, NCCL_FLOAT64, NCCL_SUM, comm, s), "ncclAllReduce",
                     err);
    }
    bool exchange(const double* sendbuf, const long long* scount, double* recvbuf, const long long* rcount,
                  cudaStream_t s, std::string& err) override {
        NcclApi& a = nccl_api();
        void* xc = hcomm ? hcomm : comm;
        if (!check(a.groupStart(), "ncclGroupStart", err)) return false;
        long long so = 0, ro = 0;
        for (int q = 0; q < world; ++q) {
            if (q != rank && scount[q] > 0 &&
                !check(a.send(sendbuf + so, (size_t)scount[q], NCCL_FLOAT64, q, xc, s), "ncclSend", err))
                return false;
            if (q != rank && rcount[q] > 0 &&
                !check(a.recv(recvbuf + ro, (size_t)rcount[q], NCCL_FLOAT64, q, xc, s), "ncclRecv", err))
                return false;
            so += scount[q];
            ro += rcount[q];
        }
        return check(a.groupEnd(), "ncclGroupEnd", err);
    }
    bool alltoallv(const long long* send, const long long* scount, long long* recv, const long long* rcount,
                   cudaStream_t s, std::string& err) override {
        long long ns = 0, nr = 0;
        for (int q = 0; q < world; ++q) {
            ns += scount[q];
            nr += rcount[q];
        }
        const size_t need = (size_t)std::max<long long>(1, ns + nr);
        if (need > dcap) {
            if (dbuf) cudaFree(dbuf);
            if (cudaMalloc((void**)&dbuf, need * sizeof(long long)) != cudaSuccess) {
                err = "alltoallv staging allocation failed";
                return false;
            }
            dcap = need;
        }
        cudaMemcpyAsync(dbuf, send, ns * sizeof(long long), cudaMemcpyHostToDevice, s);
        NcclApi& a = nccl_api();
        if (!check(a.groupStart(), "ncclGroupStart", err)) return false;
        long long so = 0, ro = 0;
        for (int q = 0; q < world; ++q) {
            if (scount[q] > 0 && !check(a.send(dbuf + so, (size_t)scount[q], NCCL_INT64, q, comm, s), "ncclSend", err))
                return false;
            if (rcount[q] > 0 &&
                !check(a.recv(dbuf + ns + ro, (size_t)rcount[q], NCCL_INT64, q, comm, s), "ncclRecv", err))
                return false;
            so += scount[q];
            ro += rcount[q];
        }
        if (!check(a.groupEnd(), "ncclGroupEnd", err)) return false;
        cudaMemcpyAsync(recv, dbuf + ns, nr * sizeof(long long), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) {
            err = "alltoallv: stream error";
            return false;
        }
        return true;
    }
    bool capturable() const override { return true; }
};

// ---- host callbacks (testing transport: e.g. a torch.distributed gloo group)
struct CallbackTransport : Transport {
    bminres_comm_callbacks cb{};
    std::vector<double> hs, hr;
    bool allreduce(double* dev, long long count, cudaStream_t s, std::string& err) override {
        hs.resize(count);
        cudaMemcpyAsync(hs.data(), dev, count * sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (cb.allreduce(cb.ctx, hs.data(), count) != 0) {
            err = "allreduce callback failed";
            return false;
        }
        cudaMemcpyAsync(dev, hs.data(), count * sizeof(double), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        return true;
    }
    bool exchange(const double* sendbuf, const long long* scount, double* recvbuf, const long long* rcount,
                  cudaStream_t s, std::string& err) override {
        long long ns = 0, nr = 0;
        for (int q = 0; q < world; ++q) {
            ns += scount[q];
            nr += rcount[q];
        }
        hs.resize(std::max<long long>(ns, 1));
        hr.resize(std::max<long long>(nr, 1));
        cudaMemcpyAsync(hs.data(), sendbuf, ns * sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (cb.exchange(cb.ctx, hs.data(), (const int64_t*)scount, hr.data(), (const int64_t*)rcount) != 0) {
            err = "exchange callback failed";
            return false;
        }
        cudaMemcpyAsync(recvbuf, hr.data(), nr * sizeof(double), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        return true;
    }
    bool alltoallv(const long long* send, const long long* scount, long long* recv, const long long* rcount,
                   cudaStream_t, std::string& err) override {
        if (cb.alltoallv(cb.ctx, (const int64_t*)send, (const int64_t*)scount, (int64_t*)recv,
                         (const int64_t*)rcount) != 0) {
            err = "alltoallv callback failed";
            return false;
        }
        return true;
    }
    bool capturable() const override { return false; }
};

// ------------------------------------------------------------------ pack kernel

// sendbuf(j, :) = V(rows[j], :)  (the rows of V_{k+1} the peers read), row-major p doubles
__global__ void k_pack_rows(const double* V, const long long* rows, long long nrows, int P, double* out) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nrows * P;
         e += (long long)gridDim.x * blockDim.x) {
        const long long j = e / P;
        out[e] = V[rows[j] * P + (e - j * P)];
    }
}

}  // namespace bmr

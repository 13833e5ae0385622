// dist_reorder.cpp -- multi-GPU Schur-form reordering (SURVEY.md 8e, config
// C4): S distributed over the ranks in COLUMN SLABS, Q in ROW SLABS, every
// window's Q_w broadcast by its owner (NCCL) per wavefront, point-to-point
// transfers only for windows that straddle a slab boundary.
//
// Why this layout (reference: the per-window L/R/Q tasks of
// window_tasks.cpp:12-102, scheduled by reorder.cpp:330-364):
//   * the LEFT update S[a:b, b:n] <- Q_w^T S[a:b, b:n] acts column by column,
//     so with column slabs every rank updates its own columns of every
//     window's row panel -- no data exchange, only Q_w;
//   * the RIGHT update S[0:a, a:b] <- S[0:a, a:b] Q_w and the window kernel
//     need whole columns [a, b): they run on the rank owning column a; when
//     the window straddles into the next slab, the neighbour ships the missing
//     columns into a 128-column halo of the owner's slab and takes them back
//     afterwards ("gather/scatter windows that straddle blocks via
//     ncclSend/ncclRecv");
//   * the Q update Q[:, a:b] <- Q[:, a:b] Q_w acts row by row: Q in row slabs
//     spreads that half of all flops evenly over the ranks.
// Slab boundaries are chosen from the plan's per-column work profile so
// every rank gets the same S-update flops (teig_dist_balance).
//
// Per wavefront level (windows pairwise disjoint), on every rank:
//   P1 halo-in  (window rows)   neighbour -> owner, for straddling windows
//   P2 window kernels of the windows this rank owns
//   P3 every rank broadcasts its segment of the level's Q_w slots (the
//      accumulators of the windows it owns + its deviation flag): one NCCL
//      group of `world` broadcasts -- each rank receives each accumulator
//      once (an all-reduce of zero-padded slots moved twice the bytes)
//   P4 left updates of all windows, this rank's columns
//   P5 halo-in  (rows above the window, after P4 -- the neighbour's left
//      updates of the level touched them)
//   P6 right updates of the owned windows (slab + halo)
//   P7 halo-out (rows 0..b of the halo columns) owner -> neighbour
//   P8 Q updates of all windows, this rank's Q rows
// Every matrix element receives exactly the single-GPU sequence of updates
// (same kernels, same per-element k order): the distributed result is
// bitwise identical to teig_reorder_schur_device.
//
// Communication is behind `Comm`: NCCL with one rank per process (torchrun),
// NCCL with every rank in this process on its own GPU (ncclCommInitAll:
// teig_dist_reorder_schur_multi), or a loopback that runs all ranks inside
// one process on one device (device-local copies) -- used to test the
// distributed algorithm on a single GPU.  Each rank works on its own device
// and stream pair (RankBufs::dev / st / st2).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "device_types.h"
#include "launch.h"
#include "plan.h"

namespace teig {

int set_error(int code, const std::string& msg);
int64_t default_tile_size(int64_t n);

namespace {

#define TEIG_CUDA(expr)                                                                          \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                 \
    } while (0)

constexpr int64_t kHalo = 128;  // halo columns right of every S slab

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (no link-time dependency of the library)

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one torch already loaded, if any
    if (!h) {
        const char* env = getenv("TEIG_NCCL_LIB");
        h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return api;
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
             api.CommInitAll && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
    return api;
}

#define TEIG_NCCL(expr)                                                                              \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != ncclSuccess)                                                                       \
            throw std::runtime_error(std::string("NCCL error ") + nccl().GetErrorString(_r) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                     \
    } while (0)

// ---------------------------------------------------------------------------
// per-rank state

struct RankBufs {
    int rank = 0;
    double* S = nullptr;  // virtual base: absolute (i, j) at S[i + j*lds]
    double* Q = nullptr;  // virtual base: absolute (i, j) at Q[i + j*ldq]
    double* T = nullptr;  // generalized pencil (C5): T column slab, like S
    double* Z = nullptr;  // generalized pencil: Z row slab, like Q
    int64_t ldq = 0;
    double* mat(int m) const { return m ? T : S; }
    double* qw = nullptr;       // Q_w slots of the pass (all windows)
    WinDesc* descs = nullptr;   // per-level descriptor arrays of this rank
    uint8_t *sizes = nullptr, *sel = nullptr, *order = nullptr, *stuck = nullptr;
    int32_t* status = nullptr;
    int32_t* dev_level = nullptr;  // deviation level of the pass (window_reorder.cu)
    double* stage = nullptr;    // contiguous staging for NCCL transfers
    size_t stage_cap = 0;
    int dev = -1;                   // the rank's device (-1: current)
    cudaStream_t st = nullptr;      // critical path: window kernels, panel updates, collectives
    cudaStream_t st2 = nullptr;     // factor (Q / Z) updates
    cudaEvent_t ev = nullptr;       // st -> st2 ordering
};

// makes `dev` current for the scope (no-op for -1 or the current device)
struct DevScope {
    int prev = -1;
    explicit DevScope(int dev) {
        if (dev < 0) return;
        int cur = 0;
        TEIG_CUDA(cudaGetDevice(&cur));
        if (cur != dev) {
            TEIG_CUDA(cudaSetDevice(dev));
            prev = cur;
        }
    }
    ~DevScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// a submatrix move between two ranks' slabs (absolute coordinates)
struct Xfer {
    int src, dst;
    int64_t r0, r1, c0, c1;
    int mat = 0;  // 0: S, 1: T
};

class Comm {
   public:
    virtual ~Comm() = default;
    virtual bool local(int r) const = 0;
    // element-wise sum of `count` elements of every rank's buffer bufs[r],
    // written back to all of them (each local rank on its own stream)
    virtual void allreduce(std::vector<RankBufs>& R, const std::vector<void*>& bufs, size_t count,
                           ncclDataType_t t) = 0;
    // segment r of every rank's buffer := rank r's segment r (float64; one
    // broadcast per owner, grouped): what each window owner publishes
    virtual void bcast_segments(std::vector<RankBufs>& R, const std::vector<double*>& bufs,
                                const std::vector<int64_t>& off, const std::vector<int64_t>& len) = 0;
    virtual void transfer(std::vector<RankBufs>& R, const std::vector<Xfer>& xs, int64_t lds) = 0;
};

size_t dtype_size(ncclDataType_t t) {
    switch (t) {
        case ncclFloat64: return 8;
        case ncclInt32: return 4;
        default: return 1;
    }
}

// all ranks in this process, one device, one stream pair: collectives are
// device-local copies (tests the distributed algorithm on a single GPU)
class LoopbackComm : public Comm {
   public:
    explicit LoopbackComm(int world) : world_(world) {}
    bool local(int) const override { return true; }
    void allreduce(std::vector<RankBufs>& R, const std::vector<void*>& bufs, size_t count,
                   ncclDataType_t t) override {
        TEIG_CUDA(launch_sum_buffers(bufs.data(), (int)bufs.size(), count, (int)dtype_size(t), R[0].st));
    }
    void bcast_segments(std::vector<RankBufs>& R, const std::vector<double*>& bufs, const std::vector<int64_t>& off,
                        const std::vector<int64_t>& len) override {
        for (int r = 0; r < world_; ++r)
            for (int k = 0; k < world_; ++k)
                if (k != r && len[r] > 0)
                    TEIG_CUDA(cudaMemcpyAsync(bufs[k] + off[r], bufs[r] + off[r], (size_t)len[r] * 8,
                                              cudaMemcpyDeviceToDevice, R[0].st));
    }
    void transfer(std::vector<RankBufs>& R, const std::vector<Xfer>& xs, int64_t lds) override {
        for (const auto& x : xs) {
            const int64_t rows = x.r1 - x.r0, cols = x.c1 - x.c0;
            if (rows <= 0 || cols <= 0) continue;
            TEIG_CUDA(cudaMemcpy2DAsync(R[x.dst].mat(x.mat) + x.r0 + x.c0 * lds, lds * 8,
                                        R[x.src].mat(x.mat) + x.r0 + x.c0 * lds, lds * 8, rows * 8, cols,
                                        cudaMemcpyDeviceToDevice, R[0].st));
        }
    }

   private:
    int world_;
};

// NCCL, one communicator per LOCAL rank: either one rank per process
// (comms[rank] only, the torchrun layout) or every rank of the job in this
// process, one device each (comms from ncclCommInitAll).  Every collective
// is one NCCL group over the local ranks, each on its own device / stream.
class NcclComm : public Comm {
   public:
    explicit NcclComm(std::vector<ncclComm_t> comms) : c_(std::move(comms)) {}
    bool local(int r) const override { return c_[r] != nullptr; }
    void allreduce(std::vector<RankBufs>& R, const std::vector<void*>& bufs, size_t count,
                   ncclDataType_t t) override {
        TEIG_NCCL(nccl().GroupStart());
        for (int r = 0; r < (int)c_.size(); ++r)
            if (local(r)) TEIG_NCCL(nccl().AllReduce(bufs[r], bufs[r], count, t, ncclSum, c_[r], R[r].st));
        TEIG_NCCL(nccl().GroupEnd());
    }
    void bcast_segments(std::vector<RankBufs>& R, const std::vector<double*>& bufs, const std::vector<int64_t>& off,
                        const std::vector<int64_t>& len) override {
        TEIG_NCCL(nccl().GroupStart());
        for (int k = 0; k < (int)c_.size(); ++k) {
            if (!local(k)) continue;
            for (int r = 0; r < (int)off.size(); ++r)
                if (len[r] > 0)
                    TEIG_NCCL(nccl().Broadcast(bufs[k] + off[r], bufs[k] + off[r], (size_t)len[r], ncclFloat64, r,
                                               c_[k], R[k].st));
        }
        TEIG_NCCL(nccl().GroupEnd());
    }
    void transfer(std::vector<RankBufs>& R, const std::vector<Xfer>& xs, int64_t lds) override {
        // per local rank: pack its outgoing pieces, exchange in one group, unpack
        const int world = (int)c_.size();
        std::vector<std::vector<size_t>> offs(world, std::vector<size_t>(xs.size(), 0));
        for (int me = 0; me < world; ++me) {
            if (!local(me)) continue;
            RankBufs& B = R[me];
            DevScope dsc(B.dev);
            size_t need = 0;
            for (const auto& x : xs)
                if (x.src == me || x.dst == me)
                    need += (size_t)std::max<int64_t>(0, x.r1 - x.r0) * std::max<int64_t>(0, x.c1 - x.c0);
            if (need == 0) continue;
            if (need > B.stage_cap) {
                if (B.stage) TEIG_CUDA(cudaFreeAsync(B.stage, B.st));
                B.stage_cap = std::max(need, B.stage_cap * 2);
                TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.stage), B.stage_cap * 8, B.st));
            }
            size_t off = 0;
            for (size_t i = 0; i < xs.size(); ++i) {
                const auto& x = xs[i];
                offs[me][i] = off;
                if (x.src != me && x.dst != me) continue;
                const int64_t rows = x.r1 - x.r0, cols = x.c1 - x.c0;
                if (rows <= 0 || cols <= 0) continue;
                if (x.src == me)
                    TEIG_CUDA(cudaMemcpy2DAsync(B.stage + off, rows * 8, B.mat(x.mat) + x.r0 + x.c0 * lds, lds * 8,
                                                rows * 8, cols, cudaMemcpyDeviceToDevice, B.st));
                off += (size_t)rows * cols;
            }
        }
        TEIG_NCCL(nccl().GroupStart());
        for (int me = 0; me < world; ++me) {
            if (!local(me)) continue;
            for (size_t i = 0; i < xs.size(); ++i) {
                const auto& x = xs[i];
                const int64_t rows = x.r1 - x.r0, cols = x.c1 - x.c0;
                if (rows <= 0 || cols <= 0) continue;
                if (x.src == me)
                    TEIG_NCCL(nccl().Send(R[me].stage + offs[me][i], (size_t)rows * cols, ncclFloat64, x.dst, c_[me],
                                          R[me].st));
                else if (x.dst == me)
                    TEIG_NCCL(nccl().Recv(R[me].stage + offs[me][i], (size_t)rows * cols, ncclFloat64, x.src, c_[me],
                                          R[me].st));
            }
        }
        TEIG_NCCL(nccl().GroupEnd());
        for (int me = 0; me < world; ++me) {
            if (!local(me)) continue;
            DevScope dsc(R[me].dev);
            for (size_t i = 0; i < xs.size(); ++i) {
                const auto& x = xs[i];
                const int64_t rows = x.r1 - x.r0, cols = x.c1 - x.c0;
                if (rows <= 0 || cols <= 0 || x.dst != me) continue;
                TEIG_CUDA(cudaMemcpy2DAsync(R[me].mat(x.mat) + x.r0 + x.c0 * lds, lds * 8, R[me].stage + offs[me][i],
                                            rows * 8, rows * 8, cols, cudaMemcpyDeviceToDevice, R[me].st));
            }
        }
    }

   private:
    std::vector<ncclComm_t> c_;
};

// ---------------------------------------------------------------------------

struct LevelPlan {
    // per rank: offsets (into that rank's desc array) and counts
    struct Part {
        int64_t w_off = 0, w_cnt = 0;                  // window kernels (owned)
        int64_t l_off = 0, l_cnt = 0, l_tiles = 0;     // left updates
        int64_t r_off = 0, r_cnt = 0, r_tiles = 0;     // right updates (owned)
        int64_t q_off = 0, q_cnt = 0, q_tiles = 0;     // Q updates
        int64_t z_off = 0, z_cnt = 0, z_tiles = 0;     // Z updates (generalized)
    };
    std::vector<Part> part;          // [rank]
    int64_t qw_off = 0, qw_len = 0;  // the level's Q_w slots
    std::vector<int64_t> seg_off, seg_len;  // per owner rank: its windows' slots + its deviation flag (last)
    std::vector<Xfer> halo_win, halo_panel, halo_back;
    int dmax = 64;
};

int owner_of(const std::vector<int64_t>& C, int64_t col) {
    return (int)(std::upper_bound(C.begin(), C.end(), col) - C.begin()) - 1;
}

struct PassOut {
    int64_t windows = 0, levels = 0, launches = 0;
    bool deviated = false;
    double fl = 0, fr = 0, fq = 0;  // executed update flops of the LOCAL ranks (left, right, factors)
};

PassOut run_dist_pass(ReorderPlan& plan, int64_t n, int world, std::vector<RankBufs>& R, Comm& comm, int64_t lds,
                      const std::vector<int64_t>& C, const std::vector<int64_t>& Rw, bool with_q, bool gen,
                      std::vector<BlockState>& blocks, std::vector<int64_t>& rejected, std::vector<int64_t>& plan_log,
                      bool strict, std::vector<FactorSupport>* qsupp, std::vector<FactorSupport>* zsupp) {
    PassOut po;
    const int64_t nw = (int64_t)plan.windows.size();
    schedule_levels(plan, n);
    const int nl = plan.n_levels;
    std::vector<int64_t> idx(nw);
    for (int64_t i = 0; i < nw; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int64_t x, int64_t y) { return plan.windows[x].level < plan.windows[y].level; });
    // Q_w slots level by level; inside a level, owner by owner: rank r's
    // segment = the accumulators of the windows it owns, then its deviation
    // flag -- one broadcast per owner publishes the segment to every rank
    std::vector<int64_t> qw_off(nw);
    int64_t qw_total = 0;
    // per-rank descriptor arrays, level by level
    std::vector<std::vector<WinDesc>> D(world);
    std::vector<std::vector<int64_t>> Dp(world);  // plan index of every descriptor
    std::vector<LevelPlan> L(nl);
    int64_t k = 0;
    for (int lv = 0; lv < nl; ++lv) {
        LevelPlan& lp = L[lv];
        lp.part.resize(world);
        const int64_t k0 = k;
        while (k < nw && plan.windows[idx[k]].level == lv) ++k;
        lp.qw_off = qw_total;
        lp.seg_off.assign(world, 0);
        lp.seg_len.assign(world, 0);
        for (int r = 0; r < world; ++r) {
            lp.seg_off[r] = qw_total;
            for (int64_t t = k0; t < k; ++t) {
                const auto& w = plan.windows[idx[t]];
                if (owner_of(C, w.wtop) != r) continue;
                qw_off[idx[t]] = qw_total;
                qw_total += (gen ? 2 : 1) * (w.wbot - w.wtop) * (w.wbot - w.wtop);
            }
            qw_total += 1;  // rank r's deviation flag
            lp.seg_len[r] = qw_total - lp.seg_off[r];
        }
        lp.qw_len = qw_total - lp.qw_off;
        for (int64_t t = k0; t < k; ++t) {
            const auto& w = plan.windows[idx[t]];
            lp.dmax = std::max<int>(lp.dmax, (int)(w.wbot - w.wtop));
        }
        lp.dmax = lp.dmax <= 64 ? 64 : 128;
        for (int r = 0; r < world; ++r) {
            auto& P = lp.part[r];
            auto base = [&](int64_t t) {
                const auto& w = plan.windows[idx[t]];
                WinDesc d{};
                d.a = (int32_t)w.wtop;
                d.d = (int32_t)(w.wbot - w.wtop);
                d.nb = (int32_t)w.count;
                d.level = lv;
                d.qw_off = qw_off[idx[t]];
                d.blk_off = w.blk_off;
                return d;
            };
            // window kernels of the owned windows
            P.w_off = (int64_t)D[r].size();
            for (int64_t t = k0; t < k; ++t)
                if (owner_of(C, plan.windows[idx[t]].wtop) == r) D[r].push_back(base(t)), Dp[r].push_back(idx[t]), ++P.w_cnt;
            // left updates: this rank's columns of every row panel
            P.l_off = (int64_t)D[r].size();
            for (int64_t t = k0; t < k; ++t) {
                const auto& w = plan.windows[idx[t]];
                const int64_t c0 = std::max<int64_t>(w.wbot, C[r]), c1 = C[r + 1];
                if (c1 <= c0) continue;
                WinDesc d = base(t);
                d.lc0 = (int32_t)c0;
                if (comm.local(r)) po.fl += (gen ? 2.0 : 1.0) * 2.0 * double(d.d) * d.d * double(c1 - c0);
                d.lc1 = (int32_t)c1;
                d.tl_pref = (int32_t)P.l_tiles;
                P.l_tiles += (c1 - c0 + kLeftBN - 1) / kLeftBN;
                D[r].push_back(d);
                Dp[r].push_back(-1);
                ++P.l_cnt;
            }
            // right updates of the owned windows
            P.r_off = (int64_t)D[r].size();
            for (int64_t t = k0; t < k; ++t) {
                const auto& w = plan.windows[idx[t]];
                if (owner_of(C, w.wtop) != r || w.wtop == 0) continue;
                WinDesc d = base(t);
                if (gen) d.qw_off += (int64_t)d.d * d.d;  // the pencil's right side uses Z_w
                d.rr0 = 0;
                d.rr1 = (int32_t)w.wtop;
                if (comm.local(r)) po.fr += (gen ? 2.0 : 1.0) * 2.0 * double(d.d) * d.d * double(w.wtop);
                d.tr_pref = (int32_t)P.r_tiles;
                P.r_tiles += (w.wtop + kRightBM - 1) / kRightBM;
                D[r].push_back(d);
                Dp[r].push_back(-1);
                ++P.r_cnt;
            }
            // Q updates: this rank's Q rows -- within them, only the tracked
            // support of the window's columns (plan.h FactorSupport; per rank:
            // a row of the result depends only on the same row of the input)
            auto factor_rows = [&](FactorSupport* fs, int64_t t, int64_t* q0, int64_t* q1) {
                const auto& w = plan.windows[idx[t]];
                *q0 = Rw[r];
                *q1 = Rw[r + 1];
                if (fs && fs->on) fs->window(w.wtop, w.wbot, q0, q1);
            };
            P.q_off = (int64_t)D[r].size();
            if (with_q && Rw[r + 1] > Rw[r])
                for (int64_t t = k0; t < k; ++t) {
                    WinDesc d = base(t);
                    int64_t q0, q1;
                    factor_rows(qsupp ? &(*qsupp)[r] : nullptr, t, &q0, &q1);
                    d.qr0 = (int32_t)q0;
                    d.qr1 = (int32_t)q1;
                    if (comm.local(r)) po.fq += 2.0 * double(d.d) * d.d * double(q1 - q0);
                    d.tq_pref = (int32_t)P.q_tiles;
                    P.q_tiles += (q1 - q0 + kRightBM - 1) / kRightBM;
                    D[r].push_back(d);
                    Dp[r].push_back(-1);
                    ++P.q_cnt;
                }
            P.z_off = (int64_t)D[r].size();
            if (gen && with_q && Rw[r + 1] > Rw[r])
                for (int64_t t = k0; t < k; ++t) {
                    WinDesc d = D[r][P.q_off + (t - k0)];
                    d.qw_off += (int64_t)d.d * d.d;
                    int64_t z0, z1;
                    factor_rows(zsupp ? &(*zsupp)[r] : nullptr, t, &z0, &z1);
                    d.qr0 = (int32_t)z0;
                    d.qr1 = (int32_t)z1;
                    if (comm.local(r)) po.fq += 2.0 * double(d.d) * d.d * double(z1 - z0);
                    d.tq_pref = (int32_t)P.z_tiles;
                    P.z_tiles += (z1 - z0 + kRightBM - 1) / kRightBM;
                    D[r].push_back(d);
                    Dp[r].push_back(-1);
                    ++P.z_cnt;
                }
        }
        // straddling windows: halo transfers
        for (int64_t t = k0; t < k; ++t) {
            const auto& w = plan.windows[idx[t]];
            const int o = owner_of(C, w.wtop);
            if (w.wbot <= C[o + 1]) continue;
            const int nbr = o + 1;
            if (nbr >= world || w.wbot > C[nbr + 1] || w.wbot - C[nbr] > kHalo)
                throw std::runtime_error("distributed reorder: a window spans more than two slabs");
            for (int m = 0; m < (gen ? 2 : 1); ++m) {
                lp.halo_win.push_back(Xfer{nbr, o, w.wtop, w.wbot, C[nbr], w.wbot, m});
                if (w.wtop > 0) lp.halo_panel.push_back(Xfer{nbr, o, 0, w.wtop, C[nbr], w.wbot, m});
                lp.halo_back.push_back(Xfer{o, nbr, 0, w.wbot, C[nbr], w.wbot, m});
            }
        }
    }
    // device buffers of the pass, per local rank (on the rank's device and
    // stream: one device in loopback, one device per rank otherwise)
    const size_t ne = plan.sizes.size();
    std::vector<void*> ord_bufs(world, nullptr), stk_bufs(world, nullptr);
    for (int r = 0; r < world; ++r) {
        if (!comm.local(r)) continue;
        RankBufs& B = R[r];
        DevScope dsc(B.dev);
        cudaStream_t st = B.st;
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.qw), sizeof(double) * std::max<int64_t>(qw_total, 1), st));
        TEIG_CUDA(cudaMemsetAsync(B.qw, 0, sizeof(double) * std::max<int64_t>(qw_total, 1), st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.descs), sizeof(WinDesc) * std::max<size_t>(D[r].size(), 1), st));
        if (!D[r].empty())
            TEIG_CUDA(cudaMemcpyAsync(B.descs, D[r].data(), sizeof(WinDesc) * D[r].size(), cudaMemcpyHostToDevice, st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.sizes), ne + 1, st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.sel), ne + 1, st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.order), ne + 1, st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.stuck), ne + 1, st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.status), sizeof(int32_t) * std::max<size_t>(D[r].size(), 1), st));
        TEIG_CUDA(cudaMemsetAsync(B.order, 0, ne + 1, st));
        TEIG_CUDA(cudaMemsetAsync(B.stuck, 0, ne + 1, st));
        TEIG_CUDA(cudaMemsetAsync(B.status, 0, sizeof(int32_t) * std::max<size_t>(D[r].size(), 1), st));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&B.dev_level), sizeof(int32_t), st));
        TEIG_CUDA(cudaMemsetAsync(B.dev_level, 0x7f, sizeof(int32_t), st));
        TEIG_CUDA(cudaMemcpyAsync(B.sizes, plan.sizes.data(), ne, cudaMemcpyHostToDevice, st));
        TEIG_CUDA(cudaMemcpyAsync(B.sel, plan.sel.data(), ne, cudaMemcpyHostToDevice, st));
        ord_bufs[r] = B.order;
        stk_bufs[r] = B.stuck;
    }
    int64_t launches = 0;
    // runs f(r, B) for every local rank on its device
    auto each = [&](auto&& f) {
        for (int r = 0; r < world; ++r) {
            if (!comm.local(r)) continue;
            DevScope dsc(R[r].dev);
            f(r, R[r]);
        }
    };
    for (int lv = 0; lv < nl; ++lv) {
        LevelPlan& lp = L[lv];
        if (!lp.halo_win.empty()) comm.transfer(R, lp.halo_win, lds);  // P1
        each([&](int r, RankBufs& B) {  // P2
            const auto& P = lp.part[r];
            if (!P.w_cnt) return;
            if (gen)
                TEIG_CUDA(launch_gwindow_reorder(B.descs + P.w_off, (int)P.w_cnt, lp.dmax, B.S, lds, B.T, lds, B.qw,
                                                 B.sizes, B.sel, B.order, B.stuck, B.status + P.w_off, B.st,
                                                 B.dev_level));
            else
                TEIG_CUDA(launch_window_reorder(B.descs + P.w_off, (int)P.w_cnt, lp.dmax, B.S, lds, B.qw, B.sizes,
                                                B.sel, B.order, B.stuck, B.status + P.w_off, B.st, nullptr,
                                                B.dev_level));
            ++launches;
        });
        {  // P3: every owner broadcasts its segment (accumulators + deviation flag)
            std::vector<double*> b(world, nullptr);
            std::vector<int64_t> flags(world);
            for (int r = 0; r < world; ++r) flags[r] = lp.seg_off[r] + lp.seg_len[r] - 1;
            each([&](int r, RankBufs& B) {
                b[r] = B.qw;
                TEIG_CUDA(launch_dist_flag(B.dev_level, B.qw, &flags[r], 1, lv, 0, B.st));
            });
            comm.bcast_segments(R, b, lp.seg_off, lp.seg_len);
            each([&](int, RankBufs& B) {
                TEIG_CUDA(launch_dist_flag(B.dev_level, B.qw, flags.data(), world, lv, 1, B.st));
            });
        }
        each([&](int r, RankBufs& B) {  // P4
            const auto& P = lp.part[r];
            if (!P.l_tiles) return;
            TEIG_CUDA(launch_update_left(B.descs + P.l_off, (int)P.l_cnt, (int)P.l_tiles, lp.dmax, B.qw, B.S, lds,
                                         (int)n, B.st, n, C[r + 1] + kHalo));
            if (gen)
                TEIG_CUDA(launch_update_left(B.descs + P.l_off, (int)P.l_cnt, (int)P.l_tiles, lp.dmax, B.qw, B.T, lds,
                                             (int)n, B.st, n, C[r + 1] + kHalo));
            ++launches;
        });
        if (!lp.halo_panel.empty()) comm.transfer(R, lp.halo_panel, lds);  // P5
        each([&](int r, RankBufs& B) {  // P6
            const auto& P = lp.part[r];
            if (!P.r_tiles) return;
            TEIG_CUDA(launch_update_right(B.descs + P.r_off, (int)P.r_cnt, (int)P.r_tiles, lp.dmax, B.qw, B.S, lds,
                                          (int)n, false, B.st, n, C[r + 1] + kHalo));
            if (gen)
                TEIG_CUDA(launch_update_right(B.descs + P.r_off, (int)P.r_cnt, (int)P.r_tiles, lp.dmax, B.qw, B.T,
                                              lds, (int)n, false, B.st, n, C[r + 1] + kHalo));
            ++launches;
        });
        if (!lp.halo_back.empty()) comm.transfer(R, lp.halo_back, lds);  // P7
        // P8 on each rank's second stream: the Q (and Z) updates only need
        // the level's broadcast Q_w; they overlap the next levels' window
        // kernels and panel updates (the single-GPU driver's schedule)
        each([&](int r, RankBufs& B) {
            const auto& P = lp.part[r];
            if (!P.q_tiles && !P.z_tiles) return;
            TEIG_CUDA(cudaEventRecord(B.ev, B.st));
            TEIG_CUDA(cudaStreamWaitEvent(B.st2, B.ev, 0));
            TEIG_CUDA(launch_update_right(B.descs + P.q_off, (int)P.q_cnt, (int)P.q_tiles, lp.dmax, B.qw, B.Q, B.ldq,
                                          (int)n, true, B.st2, Rw[r + 1], n));
            if (gen && P.z_cnt && B.Z)
                TEIG_CUDA(launch_update_right(B.descs + P.z_off, (int)P.z_cnt, (int)P.z_tiles, lp.dmax, B.qw, B.Z,
                                              B.ldq, (int)n, true, B.st2, Rw[r + 1], n));
            ++launches;
        });
    }
    each([&](int, RankBufs& B) {
        TEIG_CUDA(cudaEventRecord(B.ev, B.st2));
        TEIG_CUDA(cudaStreamWaitEvent(B.st, B.ev, 0));
    });
    // share the window outcomes (each written by its owner only), fold
    comm.allreduce(R, ord_bufs, ne + 1, ncclUint8);
    comm.allreduce(R, stk_bufs, ne + 1, ncclUint8);
    int me = 0;
    while (!comm.local(me)) ++me;
    std::vector<int32_t> status(std::max<int64_t>(nw, 1), 0);
    std::vector<uint8_t> order(ne + 1), stuck(ne + 1);
    {
        DevScope dsc(R[me].dev);
        TEIG_CUDA(cudaMemcpyAsync(order.data(), R[me].order, ne + 1, cudaMemcpyDeviceToHost, R[me].st));
        TEIG_CUDA(cudaMemcpyAsync(stuck.data(), R[me].stuck, ne + 1, cudaMemcpyDeviceToHost, R[me].st));
        TEIG_CUDA(cudaStreamSynchronize(R[me].st));
    }
    each([&](int r, RankBufs& B) {
        if (D[r].empty()) return;
        std::vector<int32_t> st(D[r].size());
        TEIG_CUDA(cudaMemcpyAsync(st.data(), B.status, sizeof(int32_t) * st.size(), cudaMemcpyDeviceToHost, B.st));
        TEIG_CUDA(cudaStreamSynchronize(B.st));
        for (size_t i = 0; i < st.size(); ++i)
            if (Dp[r][i] >= 0) status[Dp[r][i]] |= st[i];
    });
    if (!comm.local((me + 1) % world) && world > 1) {  // one rank per process: combine the ranks' statuses
        DevScope dsc(R[me].dev);
        int32_t* dst = nullptr;
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dst), sizeof(int32_t) * status.size(), R[me].st));
        TEIG_CUDA(cudaMemcpyAsync(dst, status.data(), sizeof(int32_t) * status.size(), cudaMemcpyHostToDevice, R[me].st));
        std::vector<void*> b(world, nullptr);
        b[me] = dst;
        comm.allreduce(R, b, status.size(), ncclInt32);
        TEIG_CUDA(cudaMemcpyAsync(status.data(), dst, sizeof(int32_t) * status.size(), cudaMemcpyDeviceToHost, R[me].st));
        TEIG_CUDA(cudaFreeAsync(dst, R[me].st));
        TEIG_CUDA(cudaStreamSynchronize(R[me].st));
    }
    each([&](int, RankBufs& B) {
        cudaFreeAsync(B.qw, B.st);
        cudaFreeAsync(B.descs, B.st);
        cudaFreeAsync(B.sizes, B.st);
        cudaFreeAsync(B.sel, B.st);
        cudaFreeAsync(B.order, B.st);
        cudaFreeAsync(B.stuck, B.st);
        cudaFreeAsync(B.status, B.st);
        cudaFreeAsync(B.dev_level, B.st);
        B.qw = nullptr;
        TEIG_CUDA(cudaStreamSynchronize(B.st));
    });
    status.resize(nw);
    po.deviated = fold_outcomes(plan, blocks, status, order, stuck, rejected, plan_log, strict);
    po.windows = 0;
    for (int64_t k = 0; k < nw; ++k) po.windows += (status[k] & kWinSkipped) ? 0 : 1;
    po.levels = nl;
    po.launches = launches;
    return po;
}

}  // namespace

// balanced column slabs: equal left+right update flops per rank (from the
// first-pass plan), widths >= 2*kHalo; Q row slabs: equal rows.
int dist_balance(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags, int64_t window_size, int world,
                 int64_t* col_bounds, int64_t* row_bounds) {
    if (world < 1) return set_error(-6, "world must be >= 1");
    if (n < 2 * kHalo * world) return set_error(-1, "n too small for this many slabs (>= 256 columns per rank)");
    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-3, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-3, "selection does not match n");
    const int64_t ws = std::min<int64_t>(std::max<int64_t>(window_size ? window_size : default_tile_size(n), 8), 128);
    ReorderPlan plan = plan_reorder(blocks, ws);
    std::vector<double> dens(n + 1, 0.0);
    for (const auto& w : plan.windows) {
        const double d = double(w.wbot - w.wtop);
        dens[w.wbot] += 2.0 * d * d;  // left: 2d^2 per column >= b
    }
    for (int64_t j = 1; j <= n; ++j) dens[j] += dens[j - 1];
    std::vector<double> right(n + 1, 0.0);
    for (const auto& w : plan.windows) {
        const double d = double(w.wbot - w.wtop);
        right[w.wtop] += 2.0 * d * double(w.wtop);  // right: 2d^2 a spread over [a, b)
        right[w.wbot] -= 2.0 * d * double(w.wtop);
    }
    std::vector<double> cum(n + 1, 0.0);
    double run = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        run += right[j];
        cum[j + 1] = cum[j] + dens[j] + run;
    }
    const double tot = cum[n];
    col_bounds[0] = 0;
    for (int g = 1; g < world; ++g) {
        const double target = tot * g / world;
        int64_t c = (int64_t)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        c = std::max<int64_t>(c, col_bounds[g - 1] + 2 * kHalo);
        c = std::min<int64_t>(c, n - (int64_t)(world - g) * 2 * kHalo);
        col_bounds[g] = c;
    }
    col_bounds[world] = n;
    for (int g = 0; g <= world; ++g) row_bounds[g] = n * g / world;
    return 0;
}

}  // namespace teig

using namespace teig;

extern "C" {

int teig_dist_balance(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags, int64_t window_size,
                      int32_t world, int64_t* col_bounds, int64_t* row_bounds) {
    try {
        return dist_balance(n, nb, sizes, flags, window_size, world, col_bounds, row_bounds);
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_INTERNAL, e.what());
    }
}

int64_t teig_dist_schedule(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags, int64_t window_size,
                           int32_t world, const int64_t* col_bounds, int64_t* out, int64_t cap) {
    if (n < 1 || world < 1 || !col_bounds) return set_error(-1, "bad arguments");
    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-3, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-3, "selection does not match n");
    try {
        const int64_t ws = std::min<int64_t>(std::max<int64_t>(window_size ? window_size : default_tile_size(n), 8), 128);
        ReorderPlan plan = plan_reorder(blocks, ws);
        schedule_levels(plan, n);
        std::vector<int64_t> C(col_bounds, col_bounds + world + 1);
        std::vector<int64_t> idx(plan.windows.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int64_t)i;
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int64_t x, int64_t y) { return plan.windows[x].level < plan.windows[y].level; });
        int64_t k = 0;
        auto put = [&](int64_t lv, int64_t ph, const Xfer& x) {
            if (out && k < cap) {
                int64_t* o = out + 8 * k;
                o[0] = lv; o[1] = ph; o[2] = x.src; o[3] = x.dst; o[4] = x.r0; o[5] = x.r1; o[6] = x.c0; o[7] = x.c1;
            }
            ++k;
        };
        for (int64_t t : idx) {
            const auto& w = plan.windows[t];
            const int o = owner_of(C, w.wtop);
            if (w.wbot <= C[o + 1]) continue;
            const int nbr = o + 1;
            if (nbr >= world || w.wbot > C[nbr + 1] || w.wbot - C[nbr] > kHalo)
                return set_error(-7, "a window spans more than two slabs");
            put(w.level, 0, Xfer{nbr, o, w.wtop, w.wbot, C[nbr], w.wbot});
            if (w.wtop > 0) put(w.level, 1, Xfer{nbr, o, 0, w.wtop, C[nbr], w.wbot});
            put(w.level, 2, Xfer{o, nbr, 0, w.wbot, C[nbr], w.wbot});
        }
        return k;
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_INTERNAL, e.what());
    }
}

int teig_nccl_available(void) { return nccl().ok ? 1 : 0; }

int teig_nccl_unique_id(uint8_t* id128) {
    if (!nccl().ok) return set_error(TEIG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    const ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return set_error(TEIG_ERR_INTERNAL, nccl().GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, 128);
    return 0;
}

int teig_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id128, void** comm) {
    if (!nccl().ok) return set_error(TEIG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t c;
    const ncclResult_t r = nccl().CommInitRank(&c, world, id, rank);
    if (r != ncclSuccess) return set_error(TEIG_ERR_INTERNAL, nccl().GetErrorString(r));
    *comm = c;
    return 0;
}

int teig_nccl_comm_destroy(void* comm) {
    if (!comm || !nccl().ok) return 0;
    nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    return 0;
}

// NCCL communicators of the single-process multi-GPU entry points, one
// clique per device list (ncclCommInitAll), kept for the process lifetime.
std::mutex g_clique_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_cliques;

std::vector<ncclComm_t> clique(const std::vector<int>& devs) {
    std::lock_guard<std::mutex> lk(g_clique_mu);
    auto it = g_cliques.find(devs);
    if (it != g_cliques.end()) return it->second;
    std::vector<ncclComm_t> comms(devs.size(), nullptr);
    TEIG_NCCL(nccl().CommInitAll(comms.data(), (int)devs.size(), devs.data()));
    g_cliques[devs] = comms;
    return comms;
}

// Three execution modes share one driver:
//   loopback      nccl_comm == NULL, devices == NULL: all ranks in this
//                 process on the current device, device-local collectives
//   one rank per  nccl_comm != NULL: this process is rank `rank` (torchrun)
//   process
//   multi-GPU     devices != NULL: all ranks in this process, rank r on
//                 devices[r], NCCL clique from ncclCommInitAll
static int dist_impl(int64_t n, int32_t world, int32_t rank, void* nccl_comm, const int32_t* devices,
                     double* const* dS_slabs, double* const* dT_slabs, int64_t lds, double* const* dQ_slabs,
                     double* const* dZ_slabs, const int64_t* col_bounds, const int64_t* row_bounds, int64_t nb,
                     const uint8_t* sizes, const uint8_t* flags, const teig_reorder_opts* opts, int64_t* perm,
                     int64_t* rejected_out, teig_reorder_info* info, void* stream_v, bool gen,
                     int64_t* plan_out = nullptr, int64_t plan_cap = 0) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (world < 1 || world > 16) return set_error(-2, "world must be in [1, 16]");
    const bool multi = devices != nullptr;
    const bool loop = !multi && nccl_comm == nullptr;
    if (!loop && (rank < 0 || rank >= world)) return set_error(-3, "rank out of range");
    if (!dS_slabs || !col_bounds || !row_bounds) return set_error(-5, "null slabs/bounds");
    if (lds < n) return set_error(-6, "lds < n");
    if (col_bounds[0] != 0 || col_bounds[world] != n || row_bounds[0] != 0 || row_bounds[world] != n)
        return set_error(-9, "bounds must start at 0 and end at n");
    for (int g = 0; g < world; ++g) {
        if (col_bounds[g + 1] - col_bounds[g] < kHalo) return set_error(-9, "column slabs must be >= 128 wide");
        if (row_bounds[g + 1] < row_bounds[g]) return set_error(-9, "row bounds must be nondecreasing");
    }
    teig_reorder_opts o;
    teig_reorder_opts_default(&o);
    if (opts) o = *opts;
    // windows beyond one CTA's shared memory run at the limit (as the single-GPU drivers)
    const int64_t ws = std::min<int64_t>(std::max<int64_t>(o.window_size ? o.window_size : (gen ? 64 : default_tile_size(n)), 8), gen ? 64 : 128);
    if (gen && !dT_slabs) return set_error(-5, "null T slabs");
    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-12, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-12, "reorder_schur: selection does not match s");
    cudaStream_t s = (cudaStream_t)stream_v;
    std::vector<int64_t> C(col_bounds, col_bounds + world + 1), Rw(row_bounds, row_bounds + world + 1);
    teig_reorder_info inf{};
    std::vector<int64_t> rejected, plan_log;
    // per-rank streams: loopback / one rank per process run on the caller's
    // stream plus one side stream; multi-GPU creates a stream pair per device
    struct Streams {
        std::vector<RankBufs>* R = nullptr;
        std::vector<cudaStream_t> own_s;
        std::vector<cudaEvent_t> own_e;
        std::vector<int> dev_s, dev_e;
        ~Streams() {
            for (size_t i = 0; i < own_s.size(); ++i) {
                DevScope d(dev_s[i]);
                cudaStreamSynchronize(own_s[i]);
                cudaStreamDestroy(own_s[i]);
            }
            for (size_t i = 0; i < own_e.size(); ++i) {
                DevScope d(dev_e[i]);
                cudaEventDestroy(own_e[i]);
            }
        }
        cudaStream_t stream(int dev) {
            DevScope d(dev);
            cudaStream_t x = nullptr;
            TEIG_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            own_s.push_back(x);
            dev_s.push_back(dev);
            return x;
        }
        cudaEvent_t event(int dev) {
            DevScope d(dev);
            cudaEvent_t x = nullptr;
            TEIG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
            own_e.push_back(x);
            dev_e.push_back(dev);
            return x;
        }
    };
    try {
        if (!loop && !nccl().ok) return set_error(TEIG_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
        std::vector<RankBufs> R(world);
        Streams streams;
        cudaStream_t side = nullptr;
        cudaEvent_t side_ev = nullptr;
        if (!multi) {
            side = streams.stream(-1);
            side_ev = streams.event(-1);
        }
        for (int r = 0; r < world; ++r) {
            R[r].rank = r;
            const int li = (loop || multi) ? r : (r == rank ? 0 : -1);
            if (li < 0) continue;
            if (multi) {
                R[r].dev = devices[r];
                R[r].st = streams.stream(devices[r]);
                R[r].st2 = streams.stream(devices[r]);
                R[r].ev = streams.event(devices[r]);
            } else {
                R[r].st = s;
                R[r].st2 = side;
                R[r].ev = side_ev;
            }
            R[r].S = dS_slabs[li] - C[r] * lds;
            R[r].ldq = std::max<int64_t>(Rw[r + 1] - Rw[r], 1);
            R[r].Q = (dQ_slabs && dQ_slabs[li]) ? dQ_slabs[li] - Rw[r] : nullptr;
            if (gen) {
                R[r].T = dT_slabs[li] - C[r] * lds;
                R[r].Z = (dZ_slabs && dZ_slabs[li]) ? dZ_slabs[li] - Rw[r] : nullptr;
            }
        }
        const bool with_q = dQ_slabs != nullptr;
        LoopbackComm lb(world);
        std::vector<ncclComm_t> comms(world, nullptr);
        if (multi) comms = clique(std::vector<int>(devices, devices + world));
        else if (!loop) comms[rank] = static_cast<ncclComm_t>(nccl_comm);
        NcclComm nc(comms);
        Comm& comm = loop ? static_cast<Comm&>(lb) : static_cast<Comm&>(nc);
        // per-rank row supports of the local Q (Z) slabs: one device scan each
        std::vector<FactorSupport> qsupp(world), zsupp(world);
        static const bool no_supp = getenv("TEIG_NO_Q_SUPPORT") && atoi(getenv("TEIG_NO_Q_SUPPORT"));
        auto scan = [&](int r, double* M, FactorSupport& fs) {
            const int64_t rows = Rw[r + 1] - Rw[r];
            fs.lo.assign(n, (int32_t)Rw[r]);
            fs.hi.assign(n, (int32_t)Rw[r] - 1);
            fs.on = true;
            if (rows <= 0) return;
            DevScope dsc(R[r].dev);
            int32_t *dlo = nullptr, *dhi = nullptr;
            TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dlo), sizeof(int32_t) * n, R[r].st));
            TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dhi), sizeof(int32_t) * n, R[r].st));
            // M is the virtual base (absolute row i at M[i]): the slab starts at row Rw[r]
            TEIG_CUDA(launch_column_support(M + Rw[r], R[r].ldq, rows, n, dlo, dhi, R[r].st));
            TEIG_CUDA(cudaMemcpyAsync(fs.lo.data(), dlo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, R[r].st));
            TEIG_CUDA(cudaMemcpyAsync(fs.hi.data(), dhi, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, R[r].st));
            TEIG_CUDA(cudaFreeAsync(dlo, R[r].st));
            TEIG_CUDA(cudaFreeAsync(dhi, R[r].st));
            TEIG_CUDA(cudaStreamSynchronize(R[r].st));
            for (int64_t c = 0; c < n; ++c) {  // slab-relative -> absolute rows
                if (fs.lo[c] <= fs.hi[c]) {
                    fs.lo[c] += (int32_t)Rw[r];
                    fs.hi[c] += (int32_t)Rw[r];
                } else {
                    fs.lo[c] = (int32_t)Rw[r];
                    fs.hi[c] = (int32_t)Rw[r] - 1;
                }
            }
        };
        for (int r = 0; r < world && with_q && !no_supp && !o.full_factor; ++r) {
            if (!comm.local(r)) continue;
            scan(r, R[r].Q, qsupp[r]);
            if (gen && R[r].Z) scan(r, R[r].Z, zsupp[r]);
        }
        for (int pass = 0; pass < 64; ++pass) {
            ReorderPlan plan = plan_reorder(blocks, ws);
            if (plan.windows.empty()) break;
            if (pass == 0) inf.n_groups = plan.n_groups;
            inf.update_flops += (gen ? 2.0 : 1.0) * plan_update_flops(plan, n, with_q);
            inf.update_bytes += (gen ? 2.0 : 1.0) * plan_update_bytes(plan, n, with_q);
            PassOut po = run_dist_pass(plan, n, world, R, comm, lds, C, Rw, with_q, gen, blocks, rejected, plan_log,
                                       o.strict != 0, with_q ? &qsupp : nullptr, (gen && with_q) ? &zsupp : nullptr);
            inf.n_windows += po.windows;
            inf.n_levels += po.levels;
            inf.n_launches += po.launches;
            inf.n_passes += 1;
            // per-class flops: executed by this process's ranks (the slabs it owns)
            inf.flops_left += po.fl;
            inf.flops_right += po.fr;
            inf.flops_factor_exec += po.fq;
            if (!po.deviated) break;
        }
        for (auto& B : R)
            if (B.st) {
                DevScope d(B.dev);
                if (B.stage) cudaFreeAsync(B.stage, B.st);
                TEIG_CUDA(cudaStreamSynchronize(B.st));
            }
    } catch (const std::domain_error& e) {
        return set_error(TEIG_ERR_STRICT, e.what());
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    bool leading = true, seen_unsel = false;
    for (const auto& b : blocks) {
        if (!b.selected) seen_unsel = true;
        else if (seen_unsel) leading = false;
    }
    // ascending original index: the reference's order of discovery (it runs
    // the groups top-down and a window's stuck blocks in slice order, so its
    // rejected_blocks come out sorted; pipelined groups here fold out of it)
    std::sort(rejected.begin(), rejected.end());
    inf.n_rejected = (int64_t)rejected.size();
    inf.clean = (rejected.empty() && leading) ? 1 : 0;
    if (perm)
        for (int64_t i = 0; i < nb; ++i) perm[blocks[i].orig] = i;
    if (rejected_out)
        for (size_t i = 0; i < rejected.size(); ++i) rejected_out[i] = rejected[i];
    if (plan_out)
        for (int64_t i = 0; i < (int64_t)plan_log.size() / 3 && i < plan_cap; ++i)
            for (int k = 0; k < 3; ++k) plan_out[3 * i + k] = plan_log[3 * i + k];
    if (info) *info = inf;
    return 0;
}

int teig_dist_reorder_schur(int64_t n, int32_t world, int32_t rank, void* nccl_comm, double* const* dS_slabs,
                            int64_t lds, double* const* dQ_slabs, const int64_t* col_bounds,
                            const int64_t* row_bounds, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                            const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected, teig_reorder_info* info,
                            void* stream) {
    return dist_impl(n, world, rank, nccl_comm, nullptr, dS_slabs, nullptr, lds, dQ_slabs, nullptr, col_bounds,
                     row_bounds, nb, sizes, flags, opts, perm, rejected, info, stream, false);
}

int teig_dist_greorder_schur(int64_t n, int32_t world, int32_t rank, void* nccl_comm, double* const* dS_slabs,
                             double* const* dT_slabs, int64_t lds, double* const* dQ_slabs, double* const* dZ_slabs,
                             const int64_t* col_bounds, const int64_t* row_bounds, int64_t nb, const uint8_t* sizes,
                             const uint8_t* flags, const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                             teig_reorder_info* info, void* stream) {
    return dist_impl(n, world, rank, nccl_comm, nullptr, dS_slabs, dT_slabs, lds, dQ_slabs, dZ_slabs, col_bounds,
                     row_bounds, nb, sizes, flags, opts, perm, rejected, info, stream, true);
}

int teig_dist_reorder_schur_multi(int64_t n, int32_t world, const int32_t* devices, double* const* dS_slabs,
                                  int64_t lds, double* const* dQ_slabs, const int64_t* col_bounds,
                                  const int64_t* row_bounds, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                                  const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                                  int64_t* plan, int64_t plan_cap, teig_reorder_info* info) {
    if (!devices) return set_error(-3, "devices is null");
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < r; ++k)
            if (devices[k] == devices[r]) return set_error(-3, "devices must be distinct (one rank per GPU)");
    return dist_impl(n, world, 0, nullptr, devices, dS_slabs, nullptr, lds, dQ_slabs, nullptr, col_bounds, row_bounds,
                     nb, sizes, flags, opts, perm, rejected, info, nullptr, false, plan, plan_cap);
}

int teig_gen_schur_input_cols_device(int64_t n, double* dS, int64_t lds, int64_t c0, int64_t c1, uint64_t fill_seed,
                                     void* stream) {
    DeviceGuard device_guard(dS);
    if (n < 1 || lds < n || c0 < 0 || c1 > n || c1 < c0) return set_error(-1, "bad shape");
    cudaError_t e = launch_gen_schur_cols(dS, lds, n, fill_seed, c0, c1, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

int teig_set_identity_rows_device(int64_t n, double* dQ, int64_t ldq, int64_t r0, int64_t r1, void* stream) {
    DeviceGuard device_guard(dQ);
    if (n < 1 || r0 < 0 || r1 > n || r1 < r0 || ldq < r1 - r0) return set_error(-1, "bad shape");
    cudaError_t e = launch_identity_rows(dQ, ldq, n, r0, r1, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"

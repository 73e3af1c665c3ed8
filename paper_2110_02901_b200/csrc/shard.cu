// shard.cu — multi-GPU mini-batch solves.
//
// Rows of P (and c) are sharded by contiguous state ownership; every rank
// keeps a full replica of V.  The partition pi_k is global (every rank draws
// the same permutation), so batch t is the same set of states everywhere.
// Per batch:
//   1. compact:   this rank's states of the batch (perm ∩ [row_begin,row_end));
//   2. compute:   their backups against the replica V (the dense persistent
//                 kernel in MODE_SHARD_*: one launch, one batch) -> send list
//                 (value, state, argmin) of capacity cap = min(b, max rows);
//   3. exchange:  all-gather of the fixed-size send lists (NCCL over NVLink,
//                 or device copies between the logical ranks of one GPU);
//   4. commit:    every rank scatters all ranks' updates into its replica
//                 (identical on every rank), max |new - old| -> sweep residual.
// Eq. 12 holds exactly: the batch's reads all happen in step 2, against the
// replica as it was after the previous batch's commit.
// Each state's arithmetic is the single-GPU kernel's (the chunk plan depends on
// (n, A, b) only), so V, pi and the residual trace are bitwise identical for
// any number of ranks (tested with logical ranks on one GPU).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "nccl_min.h"
#include "partition.cuh"

namespace rmb {

// ---------------------------------------------------------------- NCCL API
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// dlopen'ed (not linked) so that the process uses the one NCCL it already has
// loaded (torch's); falls back to the system library.
static NcclApi& nccl()
{
    static NcclApi api = [] {
        NcclApi x;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            x.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return x;
        }
#define RMB_SYM(name, field)                                                      \
    x.field = reinterpret_cast<decltype(x.field)>(dlsym(h, name));               \
    if (!x.field) {                                                               \
        x.why = std::string("libnccl lacks ") + name;                             \
        return x;                                                                 \
    }
        RMB_SYM("ncclGetUniqueId", GetUniqueId);
        RMB_SYM("ncclCommInitRank", CommInitRank);
        RMB_SYM("ncclCommDestroy", CommDestroy);
        RMB_SYM("ncclCommCount", CommCount);
        RMB_SYM("ncclCommUserRank", CommUserRank);
        RMB_SYM("ncclAllGather", AllGather);
        RMB_SYM("ncclCommGetAsyncError", CommGetAsyncError);
        RMB_SYM("ncclCommAbort", CommAbort);
        RMB_SYM("ncclGetErrorString", GetErrorString);
#undef RMB_SYM
        x.ok = true;
        return x;
    }();
    return api;
}

static rmb_status nccl_fail(ncclResult_t r, const char* where)
{
    set_error(std::string(where) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
    return RMB_ERR_NCCL;
}

// Wait for the stream while watching the communicator (failure
// detection): a peer that died or an NCCL failure surfaces as an async error
// -> the communicator is aborted (its kernels exit) and RMB_ERR_NCCL returned
// instead of hanging in the exchange forever.  Also bounded in time.
static rmb_status wait_stream(cudaStream_t st, ncclComm_t comm, const char* where)
{
    constexpr double kTimeoutS = 900.0;
    if (!comm) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) return RMB_OK;
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    }
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev, st);
    const auto t0 = std::chrono::steady_clock::now();
    unsigned spins = 0;
    while (e == cudaSuccess) {
        e = cudaEventQuery(ev);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) break;
        e = cudaSuccess;
        ncclResult_t ar = ncclSuccess;
        ncclResult_t r = nccl().CommGetAsyncError(comm, &ar);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (r != ncclSuccess || ar != ncclSuccess || el > kTimeoutS) {
            nccl().CommAbort(comm);
            cudaEventDestroy(ev);
            set_error(std::string(where) + ": " +
                      (el > kTimeoutS ? std::string("exchange timed out; communicator aborted")
                                      : std::string("NCCL async error (") +
                                            nccl().GetErrorString(r != ncclSuccess ? r : ar) +
                                            "); communicator aborted"));
            return RMB_ERR_NCCL;
        }
        if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    cudaEventDestroy(ev);
    if (e == cudaSuccess) return RMB_OK;
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return RMB_ERR_CUDA;
}

// ---------------------------------------------------------------- kernels
// this rank's states of batch positions [lo, lo+cnt): order-free compaction
// (the list order does not affect any state's result)
__global__ void compact_owned_kernel(const uint32_t* perm, int64_t lo, int64_t cnt, int64_t row0, int64_t row1,
                                     uint32_t* olist, int* ocount)
{
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < cnt; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        int64_t s = -1;
        if (i < cnt) s = perm ? (int64_t)perm[lo + i] : lo + i;
        const bool own = i < cnt && s >= row0 && s < row1;
        const unsigned m = __ballot_sync(0xffffffffu, own);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(ocount, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (own) olist[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)s;
    }
}

// Exchange record layout (per rank, `chunk` bytes): int count | pad to 16 |
// double val[cap] | uint32 idx[cap] | int32 arg[cap]
struct Rec {
    int64_t cap;
    size_t chunk;
    __host__ __device__ size_t off_val() const { return 16; }
    __host__ __device__ size_t off_idx() const { return 16 + 8 * (size_t)cap; }
    __host__ __device__ size_t off_arg() const { return 16 + 12 * (size_t)cap; }
};

__global__ void copy_count_kernel(const int* ocount, char* send) { *reinterpret_cast<int*>(send) = *ocount; }

// apply all ranks' updates to this rank's replica; residual / nonfinite
// (max reduced per thread, then per warp: one atomic per warp, not per entry)
__global__ void commit_kernel(double* V, int32_t* pi, int64_t row0, int64_t row1, const char* recv, int G, Rec rec,
                              unsigned long long* resid_bits, int* bad)
{
    const int64_t total = (int64_t)G * rec.cap;
    double rmax = 0.0;
    int nonfin = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(j / rec.cap);
        const int64_t q = j - (int64_t)r * rec.cap;
        const char* base = recv + (size_t)r * rec.chunk;
        if (q >= *reinterpret_cast<const int*>(base)) continue;
        const double v = reinterpret_cast<const double*>(base + rec.off_val())[q];
        const int64_t s = reinterpret_cast<const uint32_t*>(base + rec.off_idx())[q];
        const int arg = reinterpret_cast<const int32_t*>(base + rec.off_arg())[q];
        const double d = fabs(v - V[s]);
        // NaN-propagating max (a NaN update also raises the nonfinite flag)
        rmax = (d > rmax || d != d) ? d : rmax;
        nonfin |= !isfinite(v);
        V[s] = v;
        if (pi && s >= row0 && s < row1) pi[s] = arg;
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(rmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = ob > bits ? ob : bits;  // non-negative doubles (and NaN) order as their bits
        nonfin |= __shfl_xor_sync(0xffffffffu, nonfin, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bits) atomicMax(resid_bits, bits);
        if (nonfin) atomicOr(bad, 1);
    }
}

// ------------------------------------------------------------------ driver
struct RankWs {
    Problem* pr;
    DevBuf buf;  // perm (n) | olist (cap) | ocount | send (chunk) | recv (G*chunk) | resid | bad | imp
    uint32_t* perm;
    uint32_t* olist;
    int* ocount;
    char* send;
    char* recv;
    unsigned long long* resid;
    int* bad;
    char* imp_send;  // improvement record: double resid | int64 changed | int64 status | pad (32 B);
    char* imp_recv;  //   also the layout-consensus record at the start of a solve
};

static int blocks_for(int64_t work) { return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8)); }

rmb_status sharded_solve(Problem** ranks, int G_local, bool use_nccl, const SolveRequest& rq0, double* trace_host,
                         int64_t trace_len, int64_t* chg_host, int64_t chg_len, SolveResult* res)
{
    Problem& p0 = *ranks[0];
    if (rq0.fused) {
        if (!p0.dense) {
            set_error("RMB_FUSED: dense shard handles only (sparse shards use the per-batch all-gather)");
            return RMB_ERR_UNSUPPORTED;
        }
        return dense_fused_solve(ranks, G_local, use_nccl, rq0, trace_host, trace_len, chg_host, chg_len, res);
    }
    const int64_t n = p0.n;
    cudaStream_t st = p0.stream;
    int G = G_local;
    ncclComm_t comm = nullptr;
    if (use_nccl) {
        if (!nccl().ok) {
            set_error("NCCL unavailable: " + nccl().why);
            return RMB_ERR_NCCL;
        }
        comm = static_cast<ncclComm_t>(p0.nccl_comm);
        ncclResult_t r = nccl().CommCount(comm, &G);
        if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
    }
    for (int r = 0; r < G_local; ++r)
        if (ranks[r]->dense != p0.dense) {
            set_error("sharded solve: every rank's handle must have the same storage (dense or CSR)");
            return RMB_ERR_INVALID_ARG;
        }
    // the per-rank step: dense (TMA/warp kernels in MODE_SHARD_*) or sparse
    auto shard_step = p0.dense ? dense_shard_step : sparse_shard_step;
    // capacity: the largest owned range (identical on every rank: ranges from
    // rmb_shard_range, i.e. ceil(n / G))
    const int64_t max_rows = (n + G - 1) / G;
    int64_t local_max = 0;
    for (int r = 0; r < G_local; ++r) local_max = std::max(local_max, ranks[r]->row_end - ranks[r]->row_begin);
    if (local_max > max_rows) {
        set_error("owned row ranges must come from rmb_shard_range (at most ceil(n/G) rows per rank)");
        return RMB_ERR_INVALID_ARG;
    }
    Rec rec;
    rec.cap = std::min<int64_t>(rq0.b, max_rows);
    rec.chunk = ((16 + 16 * (size_t)rec.cap) + 255) / 256 * 256;

    std::vector<RankWs> ws(G_local);
    for (int r = 0; r < G_local; ++r) {
        RankWs& w = ws[r];
        w.pr = ranks[r];
        const size_t need = (size_t)n * 4 + (size_t)rec.cap * 4 + 256 + rec.chunk + (size_t)G * rec.chunk + 256 +
                            256 + 32 * (size_t)G + 256;
        if (w.pr->aux.ensure(need + 1024) != cudaSuccess) {
            set_error("sharded solve: workspace allocation failed");
            return RMB_ERR_OOM;
        }
        char* b = static_cast<char*>(w.pr->aux.p);
        auto take = [&](size_t bytes) {
            char* q = b;
            b += (bytes + 255) / 256 * 256;
            return q;
        };
        w.perm = reinterpret_cast<uint32_t*>(take((size_t)n * 4));
        w.olist = reinterpret_cast<uint32_t*>(take((size_t)rec.cap * 4));
        w.ocount = reinterpret_cast<int*>(take(16));
        w.send = take(rec.chunk);
        w.recv = take((size_t)G * rec.chunk);
        w.resid = reinterpret_cast<unsigned long long*>(take(16));
        w.bad = reinterpret_cast<int*>(take(16));
        w.imp_send = take(32);
        w.imp_recv = take(32 * (size_t)G);
    }

    // Layout consensus (every rank must pick the layout -- hence the summation
    // order -- a single handle over ALL rows would pick): gather each rank's
    // (nnz, rows, ELL width, 16-byte aligned) and combine.
    {
        std::vector<long long> all(4 * (size_t)G);
        auto local_rec = [](const Problem& p, long long* r) {
            r[0] = p.dense ? 0 : p.nnz;
            r[1] = (p.row_end - p.row_begin) * (long long)p.A;
            r[2] = p.dense ? 0 : p.ell_K;
            r[3] = p.dense ? ((reinterpret_cast<uintptr_t>(p.P) & 15u) == 0)
                           : ((uintptr_t)p.col % 16 == 0 && (uintptr_t)p.val % 16 == 0);
        };
        if (use_nccl) {
            long long mine[4];
            local_rec(p0, mine);
            cudaError_t e = cudaMemcpyAsync(ws[0].imp_send, mine, 32, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) { set_error(std::string("layout consensus: ") + cudaGetErrorString(e)); return RMB_ERR_CUDA; }
            ncclResult_t nr = nccl().AllGather(ws[0].imp_send, ws[0].imp_recv, 32, ncclUint8, comm, st);
            if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather(layout)");
            e = cudaMemcpyAsync(all.data(), ws[0].imp_recv, 32 * (size_t)G, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) { set_error(std::string("layout consensus: ") + cudaGetErrorString(e)); return RMB_ERR_CUDA; }
            if (rmb_status s = wait_stream(st, comm, "layout consensus"); s != RMB_OK) return s;
        } else {
            for (int r = 0; r < G_local; ++r) local_rec(*ranks[r], all.data() + 4 * r);
        }
        long long nnz = 0, rows = 0, K = -1;
        bool aligned = true;
        for (int r = 0; r < G; ++r) {
            nnz += all[4 * r];
            rows += all[4 * r + 1];
            aligned = aligned && all[4 * r + 3] != 0;
            if (all[4 * r + 1] == 0) continue;  // a rank owning no rows does not constrain the ELL width
            if (K < 0) K = all[4 * r + 2];
            else if (all[4 * r + 2] != K) K = 0;  // widths differ: not ELL as a whole
        }
        K = std::max(K, 0LL);
        for (int r = 0; r < G_local; ++r) {
            ranks[r]->g_set = true;
            ranks[r]->g_nnz = nnz;
            ranks[r]->g_rows = rows;
            ranks[r]->g_ell_K = (int)K;
            ranks[r]->g_aligned = aligned;
        }
    }

    auto check = [&](cudaError_t e, const char* where) -> rmb_status {
        if (e == cudaSuccess) return RMB_OK;
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    int64_t launches = 0;

    // the batch sequence of one operator application (B_b if !eval, else
    // B_{pi,b}) against the partition already drawn into every rank's perm
    auto enqueue_batches = [&](bool eval, cudaStream_t qs) -> rmb_status {
        for (int r = 0; r < G_local; ++r) {
            RankWs& w = ws[r];
            cudaError_t e = cudaMemsetAsync(w.resid, 0, 8, qs);
            if (e == cudaSuccess) e = cudaMemsetAsync(w.bad, 0, sizeof(int), qs);
            if (rmb_status s = check(e, "shard residual reset"); s != RMB_OK) return s;
        }
        for (int64_t lo = 0; lo < n; lo += rq0.b) {
            const int64_t cnt = std::min<int64_t>(rq0.b, n - lo);
            for (int r = 0; r < G_local; ++r) {
                RankWs& w = ws[r];
                Problem& pr = *w.pr;
                cudaError_t e = cudaMemsetAsync(w.ocount, 0, sizeof(int), qs);
                if (e != cudaSuccess) return check(e, "shard compact");
                compact_owned_kernel<<<blocks_for(cnt), 256, 0, qs>>>(w.perm, lo, cnt, pr.row_begin, pr.row_end, w.olist,
                                                                       w.ocount);
                if (rmb_status s = check(cudaGetLastError(), "shard compact"); s != RMB_OK) return s;
                SolveRequest rq = rq0;
                rq.mode = eval ? MODE_SHARD_EVAL : MODE_SHARD_MIN;
                rq.V = ranks[r]->stage_V;
                rq.pi = ranks[r]->stage_pi;
                rmb_status s = shard_step(pr, rq, w.olist, w.ocount,
                                          reinterpret_cast<double*>(w.send + rec.off_val()),
                                          reinterpret_cast<uint32_t*>(w.send + rec.off_idx()),
                                          reinterpret_cast<int32_t*>(w.send + rec.off_arg()), qs, nullptr);
                if (s != RMB_OK) return s;
                copy_count_kernel<<<1, 1, 0, qs>>>(w.ocount, w.send);
                launches += 3;
            }
            if (use_nccl) {
                ncclResult_t nr = nccl().AllGather(ws[0].send, ws[0].recv, rec.chunk, ncclUint8, comm, qs);
                if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather");
            } else {
                for (int r = 0; r < G_local; ++r)
                    for (int q = 0; q < G_local; ++q) {
                        cudaError_t e = cudaMemcpyAsync(ws[r].recv + (size_t)q * rec.chunk, ws[q].send, rec.chunk,
                                                        cudaMemcpyDeviceToDevice, qs);
                        if (e != cudaSuccess) return check(e, "logical exchange");
                    }
            }
            for (int r = 0; r < G_local; ++r) {
                RankWs& w = ws[r];
                Problem& pr = *w.pr;
                commit_kernel<<<blocks_for((int64_t)G * rec.cap), 256, 0, qs>>>(
                    pr.stage_V, eval ? nullptr : pr.stage_pi, pr.row_begin, pr.row_end, w.recv, G, rec, w.resid, w.bad);
                if (rmb_status s = check(cudaGetLastError(), "shard commit"); s != RMB_OK) return s;
                ++launches;
            }
        }
        return RMB_OK;
    };

    // CUDA graphs: the batch sequence of a sweep is the same stream work every
    // sweep (only the perm contents change, drawn by the partition kernel
    // launched before it), so after one eager sweep per kind (which also sizes
    // every workspace: no allocation may happen under capture) it is captured
    // once and replayed -- one host launch per sweep instead of ~5 per batch
    // per rank.  The decision is the same on every rank (it depends on the
    // create flag RMB_SHARD_NO_GRAPH and on nothing rank-local).  A capture
    // failure in a logical group (one process, no NCCL) falls back to the eager
    // sequence (the same kernels); under NCCL it is an error: the failed
    // capture may already hold recorded collectives, and one rank replaying
    // while another runs eagerly would desynchronise the communicator.
    const int64_t nbatches = (n + rq0.b - 1) / rq0.b;
    bool graph_on = true;
    for (int r = 0; r < G_local; ++r) graph_on = graph_on && !ranks[r]->shard_no_graph;
    int64_t graph_launches = 0;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int64_t gkern[2] = {0, 0};
    int warm[2] = {0, 0};
    bool gfail[2] = {false, false};
    struct GraphGuard {
        cudaGraphExec_t* g;
        ~GraphGuard()
        {
            for (int i = 0; i < 2; ++i)
                if (g[i]) cudaGraphExecDestroy(g[i]);
        }
    } gguard{gexec};
    // capture needs a stream other than the legacy default stream (which is
    // what torch's current stream usually is): a private non-blocking stream
    cudaStream_t gst = nullptr;
    struct StreamGuard {
        cudaStream_t* s;
        ~StreamGuard()
        {
            if (*s) cudaStreamDestroy(*s);
        }
    } sguard{&gst};

    auto run_batches = [&](bool eval) -> rmb_status {
        const int kind = eval ? 1 : 0;
        if (graph_on && !gfail[kind] && warm[kind] >= 1) {
            if (!gexec[kind]) {
                const int64_t l0 = launches;
                cudaGraph_t g = nullptr;
                cudaError_t e = gst ? cudaSuccess : cudaStreamCreateWithFlags(&gst, cudaStreamNonBlocking);
                if (e == cudaSuccess) e = cudaStreamBeginCapture(gst, cudaStreamCaptureModeThreadLocal);
                rmb_status s = e == cudaSuccess ? enqueue_batches(eval, gst) : RMB_ERR_CUDA;
                cudaError_t e2 = e == cudaSuccess ? cudaStreamEndCapture(gst, &g) : e;
                if (s == RMB_OK && e2 == cudaSuccess && g) e2 = cudaGraphInstantiate(&gexec[kind], g, 0);
                if (g) cudaGraphDestroy(g);
                gkern[kind] = launches - l0;
                launches = l0;
                if (s != RMB_OK || e2 != cudaSuccess || !gexec[kind]) {
                    gfail[kind] = true;
                    gexec[kind] = nullptr;
                    cudaGetLastError();  // clear the capture error
                    if (use_nccl) {
                        set_error(std::string("sharded solve: CUDA graph capture of the sweep failed (") +
                                  cudaGetErrorString(e2) + "); create the handles with RMB_SHARD_NO_GRAPH");
                        return RMB_ERR_CUDA;
                    }
                }
            }
            if (gexec[kind]) {
                if (rmb_status s = check(cudaGraphLaunch(gexec[kind], st), "shard graph launch"); s != RMB_OK) return s;
                launches += gkern[kind];
                ++graph_launches;
                return RMB_OK;
            }
        }
        ++warm[kind];
        return enqueue_batches(eval, st);
    };

    // one operator application (B_b if !eval, else B_{pi,b}) with sweep index k
    auto sweep = [&](int64_t k, bool eval, double* r_out, bool* bad_out) -> rmb_status {
        for (int r = 0; r < G_local; ++r) {
            cudaError_t e = launch_partition(n, rq0.seed, k, rq0.identity, ws[r].perm, st);
            if (rmb_status s = check(e, "shard partition"); s != RMB_OK) return s;
            ++launches;
        }
        if (rmb_status s = run_batches(eval); s != RMB_OK) return s;
        res->batches += nbatches;
        unsigned long long rb = 0;
        int bb = 0;
        cudaError_t e = cudaMemcpyAsync(&rb, ws[0].resid, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&bb, ws[0].bad, 4, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return check(e, "shard residual");
        if (rmb_status s = wait_stream(st, comm, "shard sweep"); s != RMB_OK) return s;
        memcpy(r_out, &rb, 8);
        *bad_out = bb != 0;
        return RMB_OK;
    };

    // improvement over every rank's own states; (max residual, sum changed, any bad)
    auto improve = [&](double* r_out, long long* changed_out, bool* bad_out) -> rmb_status {
        std::vector<long long*> outs(G_local);
        for (int r = 0; r < G_local; ++r) {
            SolveRequest rq = rq0;
            rq.mode = MODE_SHARD_IMPROVE;
            rq.V = ranks[r]->stage_V;
            rq.pi = ranks[r]->stage_pi;
            rmb_status s = shard_step(*ranks[r], rq, nullptr, nullptr, nullptr, nullptr, nullptr, st, &outs[r]);
            if (s != RMB_OK) return s;
            ++launches;
            // record: residual bits, changed, status
            cudaError_t e = cudaMemcpyAsync(ws[r].imp_send, outs[r] + OUT_RESID_BITS, 8, cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(ws[r].imp_send + 8, outs[r] + OUT_CHANGED, 8, cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(ws[r].imp_send + 16, outs[r] + OUT_STATUS, 8, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return check(e, "shard improve record");
        }
        std::vector<long long> all(4 * (size_t)G);  // 32-byte records
        if (use_nccl) {
            ncclResult_t nr = nccl().AllGather(ws[0].imp_send, ws[0].imp_recv, 32, ncclUint8, comm, st);
            if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather(improve)");
            cudaError_t e = cudaMemcpyAsync(all.data(), ws[0].imp_recv, 32 * (size_t)G, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return check(e, "improve gather");
        } else {
            for (int r = 0; r < G_local; ++r) {
                cudaError_t e = cudaMemcpyAsync(all.data() + 4 * r, ws[r].imp_send, 24, cudaMemcpyDeviceToHost, st);
                if (e != cudaSuccess) return check(e, "improve gather");
            }
        }
        if (rmb_status s = wait_stream(st, comm, "shard improve"); s != RMB_OK) return s;
        double rmax = 0.0;
        long long ch = 0;
        bool bad = false;
        for (int r = 0; r < G; ++r) {
            double d;
            memcpy(&d, &all[4 * r], 8);
            if (!std::isfinite(d) || all[4 * r + 2] == RMB_ERR_NONFINITE) bad = true;
            rmax = std::max(rmax, d);
            ch += all[4 * r + 1];
        }
        *r_out = rmax;
        *changed_out = ch;
        *bad_out = bad;
        return RMB_OK;
    };

    rmb_status status = RMB_ERR_NOT_CONVERGED;
    int64_t k = rq0.k0, it = 0, outer = 0;
    double last = 0.0;
    long long changed = 0;
    if (rq0.mode == MODE_VI) {
        while (it < rq0.max_iter) {
            double r;
            bool bad;
            if (rmb_status s = sweep(k, false, &r, &bad); s != RMB_OK) return s;
            if (trace_host && it < trace_len) trace_host[it] = r;
            ++it;
            ++k;
            last = r;
            if (bad) { status = RMB_ERR_NONFINITE; break; }
            if (r <= rq0.eps) { status = RMB_OK; break; }
        }
    } else if (rq0.mode == MODE_MPI) {
        bool bad = false;
        if (!rq0.pi_given) {
            double r;
            long long ch;
            if (rmb_status s = improve(&r, &ch, &bad); s != RMB_OK) return s;
        }
        while (!bad && outer < rq0.max_iter) {
            const int64_t row = outer * (rq0.msweeps + 1);
            for (int e = 0; e < rq0.msweeps && !bad; ++e) {
                double r;
                if (rmb_status s = sweep(k, true, &r, &bad); s != RMB_OK) return s;
                if (trace_host && row + e < trace_len) trace_host[row + e] = r;
                ++k;
                ++it;
            }
            if (bad) { ++outer; break; }
            double r;
            long long ch;
            if (rmb_status s = improve(&r, &ch, &bad); s != RMB_OK) return s;
            if (trace_host && row + rq0.msweeps < trace_len) trace_host[row + rq0.msweeps] = r;
            if (chg_host && outer < chg_len) chg_host[outer] = ch;
            ++outer;
            last = r;
            changed = ch;
            if (bad) break;
            if (ch == 0 && r <= rq0.eps) { status = RMB_OK; break; }
        }
        if (bad) status = RMB_ERR_NONFINITE;
    } else {
        set_error("sharded solve: unsupported mode");
        return RMB_ERR_UNSUPPORTED;
    }
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    res->sweeps = it;
    res->outer = outer;
    res->status = status;
    res->final_resid = last;
    res->changed = changed;
    res->ms = ms;
    res->launches = (int)launches;
    for (int r = 0; r < G_local; ++r) {
        ranks[r]->last_launches = launches;
        ranks[r]->last_graph_launches = graph_launches;
    }
    return RMB_OK;
}

// Map every rank's fused-exchange buffer into this process:
// CUDA IPC handles all-gathered over the handle's NCCL communicator, opened
// once and kept for the handle's lifetime (NVLink / NVSwitch peer memory).
rmb_status fused_peers(Problem& pr, int* G, int* rank)
{
    if (!nccl().ok) {
        set_error("NCCL unavailable: " + nccl().why);
        return RMB_ERR_NCCL;
    }
    ncclComm_t comm = static_cast<ncclComm_t>(pr.nccl_comm);
    ncclResult_t r = nccl().CommCount(comm, G);
    if (r == ncclSuccess) r = nccl().CommUserRank(comm, rank);
    if (r != ncclSuccess) return nccl_fail(r, "fused peers");
    if (*G > 8) {
        set_error("fused solve: at most 8 ranks");
        return RMB_ERR_UNSUPPORTED;
    }
    if (pr.xpeer_G == *G) return RMB_OK;
    // Every step below is collective: a rank that fails locally still takes
    // part in both all-gathers, so all ranks reach the same verdict and either
    // all launch the fused kernel or none does (no rank left waiting in it).
    std::string why;
    int ok = 1;
    if (fused_buffer(pr) != RMB_OK) ok = 0, why = rmb_last_error();
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof mine);
    if (ok) {
        cudaError_t e = cudaIpcGetMemHandle(&mine, pr.xbuf.p);
        if (e != cudaSuccess) ok = 0, why = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
    }
    const size_t H = sizeof(cudaIpcMemHandle_t);
    DevBuf tmp;
    if (tmp.ensure(H * (size_t)(*G + 1) + 8 * (size_t)(*G + 1)) != cudaSuccess) {
        set_error("fused peers: allocation failed");
        return RMB_ERR_OOM;
    }
    char* d = static_cast<char*>(tmp.p);
    int* flags = reinterpret_cast<int*>(d + H * (size_t)(*G + 1));
    std::vector<cudaIpcMemHandle_t> all((size_t)*G);
    cudaError_t e = cudaMemcpyAsync(d, &mine, H, cudaMemcpyHostToDevice, pr.stream);
    if (e == cudaSuccess) {
        r = nccl().AllGather(d, d + H, H, ncclUint8, comm, pr.stream);
        if (r != ncclSuccess) {
            tmp.release();
            return nccl_fail(r, "fused peers: ncclAllGather");
        }
        e = cudaMemcpyAsync(all.data(), d + H, H * (size_t)*G, cudaMemcpyDeviceToHost, pr.stream);
    }
    if (e == cudaSuccess) {
        rmb_status s = wait_stream(pr.stream, comm, "fused peers");
        if (s != RMB_OK) {
            tmp.release();
            return s;
        }
    }
    void* opened[8] = {nullptr};
    for (int q = 0; q < *G && ok && e == cudaSuccess; ++q) {
        if (q == *rank) continue;
        cudaError_t eo = cudaIpcOpenMemHandle(&opened[q], all[q], cudaIpcMemLazyEnablePeerAccess);
        if (eo != cudaSuccess) {
            ok = 0;
            why = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(eo);
            opened[q] = nullptr;
            cudaGetLastError();
        }
    }
    // the verdict: every rank's ok flag
    std::vector<int> oks((size_t)*G, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, &ok, 4, cudaMemcpyHostToDevice, pr.stream);
    if (e == cudaSuccess) {
        r = nccl().AllGather(flags, flags + 1, 4, ncclUint8, comm, pr.stream);
        if (r != ncclSuccess) {
            tmp.release();
            return nccl_fail(r, "fused peers: ncclAllGather(verdict)");
        }
        e = cudaMemcpyAsync(oks.data(), flags + 1, 4 * (size_t)*G, cudaMemcpyDeviceToHost, pr.stream);
    }
    if (e == cudaSuccess) {
        rmb_status s = wait_stream(pr.stream, comm, "fused peers");
        if (s != RMB_OK) {
            tmp.release();
            return s;
        }
    }
    tmp.release();
    bool all_ok = e == cudaSuccess;
    for (int q = 0; q < *G; ++q) all_ok = all_ok && oks[q] == 1;
    if (!all_ok) {
        for (int q = 0; q < *G; ++q)
            if (opened[q]) cudaIpcCloseMemHandle(opened[q]);
        set_error("fused solve: peer memory unavailable on some rank" + (why.empty() ? std::string() : " (" + why + ")"));
        return RMB_ERR_UNSUPPORTED;
    }
    for (int q = 0; q < *G; ++q) {
        pr.xpeer[q] = q == *rank ? pr.xbuf.p : opened[q];
        pr.xpeer_open[q] = q != *rank;
    }
    pr.xpeer_G = *G;
    return RMB_OK;
}

}  // namespace rmb

// ------------------------------------------------------------ C entry points
using namespace rmb;

extern "C" rmb_status rmb_nccl_unique_id(void* id128)
{
    if (!id128) {
        set_error("id buffer is NULL");
        return RMB_ERR_INVALID_ARG;
    }
    if (!nccl().ok) {
        set_error("NCCL unavailable: " + nccl().why);
        return RMB_ERR_NCCL;
    }
    ncclUniqueId id;
    ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id128, &id, sizeof(id));
    return RMB_OK;
}

extern "C" rmb_status rmb_nccl_comm_init(int32_t nranks, int32_t rank, const void* id128, void** comm)
{
    if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("rmb_nccl_comm_init: invalid argument");
        return RMB_ERR_INVALID_ARG;
    }
    if (!nccl().ok) {
        set_error("NCCL unavailable: " + nccl().why);
        return RMB_ERR_NCCL;
    }
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    ncclResult_t r = nccl().CommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return RMB_OK;
}

extern "C" rmb_status rmb_nccl_comm_destroy(void* comm)
{
    if (!comm) {
        set_error("comm is NULL");
        return RMB_ERR_INVALID_ARG;
    }
    if (!nccl().ok) return RMB_ERR_NCCL;
    ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return RMB_OK;
}

extern "C" rmb_status rmb_shard_range(int64_t n, int32_t G, int32_t g, int64_t* begin, int64_t* end)
{
    if (n < 1 || G < 1 || g < 0 || g >= G || !begin || !end) {
        set_error("rmb_shard_range: invalid argument");
        return RMB_ERR_INVALID_ARG;
    }
    // contiguous blocks of ceil(n/G) rows; trailing ranks may own fewer (or none)
    const int64_t q = (n + G - 1) / G;
    *begin = std::min<int64_t>(n, (int64_t)g * q);
    *end = std::min<int64_t>(n, (int64_t)(g + 1) * q);
    return RMB_OK;
}

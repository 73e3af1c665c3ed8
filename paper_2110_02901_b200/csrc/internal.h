// internal.h — library-internal types shared by the ABI layer and kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rmb.h"

namespace rmb {

enum Mode : int {
    MODE_VI = 0,       // MB-VI: sweeps of B_b to r_k <= eps
    MODE_MPI = 1,      // MB-MPI: Algorithm 1 with B_{pi,b} evaluation
    MODE_APPLY = 2,    // one application of B_b
    MODE_APPLY_PI = 3, // one application of B_{pi,b}
    MODE_IMPROVE = 4,  // one policy improvement (greedy, ||TV-V||, changed)
    // multi-GPU shard steps (one launch each, host-driven exchange between them)
    MODE_SHARD_MIN = 5,     // B_b backups of this rank's states of one batch -> send list
    MODE_SHARD_EVAL = 6,    // B_{pi,b} backups of this rank's states of one batch -> send list
    MODE_SHARD_IMPROVE = 7, // improvement of this rank's states (pi owned entries, resid, changed)
    MODE_POLICY_VALUE = 8,  // B_{pi,b} applied until ||V_k - V_{k-1}|| <= eps (policy evaluation)
};

// Device-side result block written by the solver kernels (long long[8]).
enum OutSlot : int {
    OUT_SWEEPS = 0,
    OUT_OUTER = 1,
    OUT_STATUS = 2,
    OUT_RESID_BITS = 3,
    OUT_BATCHES = 4,
    OUT_CHANGED = 5,
    OUT_XEPOCHS = 6,  // fused multi-rank solves: cross-rank barrier epochs of the launch
    OUT_N = 8
};

struct SolveRequest {
    int mode = MODE_VI;
    int64_t b = 1;
    uint64_t seed = 0;
    int64_t k0 = 1;          // first sweep index
    bool identity = false;   // RMB_ORDER_IDENTITY
    bool chunked = false;    // RMB_CHUNKED_T: VI* (T in chunks of b against the sweep-start values)
    bool fused = false;      // RMB_FUSED: multi-rank solve with the in-kernel peer-memory exchange
    int select = 0;          // 0: partition (R2); 1 / 2: draws with replacement, uniform / weighted (R28-R29)
    bool async = false;      // RMB_ASYNC: no batch barrier, reads of V as found in memory (R31)
    // RMB_TRACE_ERROR_VS_REF: etrace[i] = ||V_i - vref||_inf after operator
    // application i of the launch (device, zeroed by the caller); null = off
    const double* vref = nullptr;
    double* etrace = nullptr;
    int64_t etrace_len = 0;
    double eps = -1.0;       // < 0: no convergence test
    int64_t max_iter = 1;    // VI: sweeps; MPI: outer iterations
    int msweeps = 1;         // MPI evaluation sweeps per outer iteration
    bool pi_given = false;
    double* V = nullptr;     // device [n]
    int32_t* pi = nullptr;   // device [n] (may be null for APPLY)
};

struct SolveResult {
    int64_t sweeps = 0, outer = 0, batches = 0, changed = 0;
    int status = RMB_OK;
    double final_resid = 0.0;
    float ms = 0.f;
    int launches = 0;
};

// Grow-only device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need)
    {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, need);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct Problem {
    int64_t n = 0;
    int A = 0;
    double gamma = 0.0;
    rmb_dtype pdt = RMB_F32;
    bool dense = true;
    // device views (borrowed or owned)
    const void* P = nullptr;
    const void* c = nullptr;
    const int64_t* row_ptr = nullptr;
    const int32_t* col = nullptr;
    const void* val = nullptr;
    int64_t nnz = 0;
    // multi-GPU: owned states [row_begin, row_end) and the exchange backend
    int64_t row_begin = 0, row_end = 0;
    void* nccl_comm = nullptr;
    double* stage_V = nullptr;    // sharded solves: this rank's replica of V (device)
    int32_t* stage_pi = nullptr;  //                 this rank's pi (owned entries meaningful)
    int ell_K = 0;  // > 0: fixed-stride rows (ELL)
    // multi-GPU layout consensus (shard.cu): the shape of the WHOLE problem, so
    // that every shard picks the layout (and hence the arithmetic) a single
    // handle over all rows would pick; g_set == false: use this handle's own
    bool g_set = false;
    int64_t g_nnz = 0, g_rows = 0;
    int g_ell_K = 0;
    bool g_aligned = true;
    // A/B and test switches from the create flags (never needed for correctness)
    bool sparse_full_grid = false;  // RMB_SPARSE_FULL_GRID
    bool shard_no_graph = false;    // RMB_SHARD_NO_GRAPH
    int64_t last_graph_launches = 0;
    // fused multi-rank solves (K8f): exchange buffer (xval | xarg | xbar | ximp |
    // xlist | xcnt, sized for b <= n), its peers' mappings, epochs done so far
    DevBuf xbuf;
    void* xpeer[8] = {nullptr};    // per rank: the mapped exchange buffer (own: xbuf.p)
    bool xpeer_open[8] = {false};  // opened through CUDA IPC (closed at destroy)
    int xpeer_G = 0;
    int64_t xepochs = 0;
    bool no_tma = false;  // dense: RMB_DENSE_NO_TMA (register-streaming warp path)
    bool vglobal = false; // dense: RMB_DENSE_VGLOBAL (V and pi in global memory)
    bool no_cluster = false;  // dense: RMB_DENSE_NO_CLUSTER (tiny batches on the grid solver too)
    // weighted selection (rmb_set_selection_weights): inclusive prefix sums of
    // the integer weights (device [n]) and their total; null = none set
    DevBuf sel_buf;
    const uint64_t* sel_cum = nullptr;
    uint64_t sel_W = 0;
    // reference V* for RMB_TRACE_ERROR_VS_REF (rmb_set_reference) and the
    // last solve's error trace (rmb_error_trace)
    DevBuf ref_buf, etrace;
    bool has_ref = false;
    int64_t etrace_count = 0;
    cudaStream_t stream = nullptr;
    int device = 0;
    int num_sms = 0;
    size_t smem_optin = 0;
    std::vector<void*> owned;  // host-staged inputs
    // workspace
    DevBuf perm, part, ctrl, trace, chg, vstage, pistage, aux, rowrec;
    int64_t last_launches = 0;
    long long prof[4] = {0, 0, 0, 0};  // last solve: compute / barrier / combine ns (CTA 0), barriers
};

// dense.cu
rmb_status dense_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                       long long* chg_dev, int64_t chg_len, SolveResult* res);
// async.cu: asynchronous dense MB-VI / MB-MPI (RMB_ASYNC, reading R31)
rmb_status dense_async_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                             long long* chg_dev, int64_t chg_len, SolveResult* res);
// cluster.cu: tiny dense batches on one thread-block cluster (DSMEM combine,
// hardware cluster barrier); eligible = inside that path's envelope
bool dense_cluster_eligible(const Problem& pr, const SolveRequest& rq);
rmb_status dense_cluster_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                               SolveResult* res);
// fused multi-rank dense solve (K8f): G logical ranks in one launch on one
// device (nccl == false) or this process's rank of an NCCL group (peer memory
// through CUDA IPC)
rmb_status dense_fused_solve(Problem** ranks, int G, bool nccl, const SolveRequest& rq, double* trace_host,
                             int64_t trace_len, int64_t* chg_host, int64_t chg_len, SolveResult* res);
rmb_status dense_shard_step(Problem& pr, const SolveRequest& rq, const uint32_t* olist, const int* ocount,
                            double* send_val, uint32_t* send_idx, int32_t* send_arg, cudaStream_t st,
                            long long** out_dev);
// shard.cu: multi-GPU (NCCL) and logical-group (one GPU) sharded solves;
// fused_peers maps every rank's exchange buffer (CUDA IPC handles all-gathered
// over the handle's NCCL communicator) into this process: pr.xpeer[0..G)
rmb_status fused_peers(Problem& pr, int* G, int* rank);
rmb_status fused_buffer(Problem& pr);  // dense.cu: allocate + zero the exchange buffer (once)
rmb_status sharded_solve(Problem** ranks, int G, bool nccl, const SolveRequest& rq, double* trace_host,
                         int64_t trace_len, int64_t* chg_host, int64_t chg_len, SolveResult* res);
// sparse.cu
rmb_status sparse_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                        long long* chg_dev, int64_t chg_len, SolveResult* res);
rmb_status sparse_shard_step(Problem& pr, const SolveRequest& rq, const uint32_t* olist, const int* ocount,
                             double* send_val, uint32_t* send_idx, int32_t* send_arg, cudaStream_t st,
                             long long** out_dev);
// gen_kernels.cu
cudaError_t launch_partition(int64_t n, uint64_t seed, int64_t sweep, bool identity, uint32_t* perm,
                             cudaStream_t st);
cudaError_t launch_select(int64_t n, uint64_t seed, int64_t sweep, int sel, const uint64_t* cum, uint64_t W,
                          uint32_t* out, cudaStream_t st);
cudaError_t launch_validate(const Problem& pr, int* bad_dev, cudaStream_t st);
cudaError_t launch_check_policy(const int32_t* pi, int64_t lo, int64_t hi, int A, int* bad, cudaStream_t st);

// abi.cu
void set_error(const std::string& msg);

}  // namespace rmb

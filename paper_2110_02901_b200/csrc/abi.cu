// abi.cu — the extern "C" boundary (include/rmb.h): argument checks, host
// buffer staging, workspace, dispatch to the dense / sparse solvers.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "internal.h"
#include "partition.cuh"

namespace rmb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static rmb_status fail(rmb_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

static rmb_status cuda_fail(cudaError_t e, const char* where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return RMB_ERR_OOM;
    return RMB_ERR_CUDA;
}

// true for device (or managed) memory; false for pageable / pinned host memory
static bool is_device_ptr(const void* p)
{
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Returns a device view of `p` (size bytes): p itself, or an owned copy.
static rmb_status device_view(Problem& pr, const void* p, size_t bytes, const void** out, const char* what)
{
    if (is_device_ptr(p)) {
        *out = p;
        return RMB_OK;
    }
    // stream-ordered allocation from the device's pool, which keeps freed
    // memory reserved: a handle created right after another one's destroy
    // (a new host problem per solve -- the e2e path) reuses it without a
    // fresh cudaMalloc / cudaFree of gigabytes
    static bool pool_set = false;
    if (!pool_set) {
        cudaMemPool_t mp;
        if (cudaDeviceGetDefaultMemPool(&mp, pr.device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool_set = true;
    }
    void* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, bytes, pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, what);
    pr.owned.push_back(d);
    e = cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, what);
    *out = d;
    return RMB_OK;
}

static rmb_status check_desc(const rmb_desc* d)
{
    if (!d) return fail(RMB_ERR_INVALID_ARG, "desc is NULL");
    if (d->n_states < 1 || d->n_states > 0x7fffffffLL) return fail(RMB_ERR_INVALID_ARG, "n_states out of [1, 2^31)");
    if (d->n_actions < 1) return fail(RMB_ERR_INVALID_ARG, "n_actions < 1");
    if (!(d->gamma > 0.0 && d->gamma < 1.0)) return fail(RMB_ERR_INVALID_ARG, "gamma not in (0,1)");
    if (d->p_dtype != RMB_F32 && d->p_dtype != RMB_F64) return fail(RMB_ERR_INVALID_ARG, "bad p_dtype");
    if (d->v_dtype != RMB_F64) return fail(RMB_ERR_INVALID_ARG, "v_dtype must be RMB_F64 in this build");
    if (!(0 <= d->row_begin && d->row_begin <= d->row_end && d->row_end <= d->n_states))
        return fail(RMB_ERR_INVALID_ARG, "need 0 <= row_begin <= row_end <= n_states");
    return RMB_OK;
}

static rmb_status init_problem(Problem& pr, const rmb_desc* d)
{
    pr.n = d->n_states;
    pr.A = d->n_actions;
    pr.gamma = d->gamma;
    pr.pdt = d->p_dtype;
    pr.stream = (cudaStream_t)d->stream;
    pr.row_begin = d->row_begin;
    pr.row_end = d->row_end;
    pr.nccl_comm = d->nccl_comm;
    cudaError_t e = cudaGetDevice(&pr.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int v = 0;
    e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, pr.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    pr.num_sms = v;
    e = cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    pr.smem_optin = (size_t)v;
    return RMB_OK;
}

static void free_problem(Problem* pr)
{
    if (!pr) return;
    for (void* p : pr->owned) cudaFreeAsync(p, pr->stream);
    if (!pr->owned.empty()) cudaStreamSynchronize(pr->stream);
    pr->perm.release();
    pr->part.release();
    pr->ctrl.release();
    pr->trace.release();
    pr->chg.release();
    pr->vstage.release();
    pr->pistage.release();
    pr->aux.release();
    pr->rowrec.release();
    pr->sel_buf.release();
    pr->ref_buf.release();
    pr->etrace.release();
    for (int q = 0; q < 8; ++q)
        if (pr->xpeer_open[q]) cudaIpcCloseMemHandle(pr->xpeer[q]);
    pr->xbuf.release();
    delete pr;
}

static rmb_status validate_mdp(Problem& pr)
{
    if (pr.aux.ensure(256) != cudaSuccess) return fail(RMB_ERR_OOM, "validate: allocation failed");
    int* bad = static_cast<int*>(pr.aux.p);
    cudaError_t e = launch_validate(pr, bad, pr.stream);
    int h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "validate");
    if (h) {
        std::string m = "invalid MDP:";
        if (h & 1) m += " a row of P does not sum to 1;";
        if (h & 2) m += " a successor index is out of range;";
        if (h & 4) m += " a probability or cost is not finite / not in [0,1];";
        return fail(RMB_ERR_INVALID_MDP, m);
    }
    return RMB_OK;
}

// pi (device) must hold actions in [0, A) on [lo, hi): an out-of-range entry
// would index a row past the end of P (checked on the device, on the stream)
static rmb_status check_policy(Problem& pr, const int32_t* pi_dev, int64_t lo, int64_t hi)
{
    if (pr.aux.ensure(256) != cudaSuccess) return fail(RMB_ERR_OOM, "policy check: allocation failed");
    int* bad = static_cast<int*>(pr.aux.p);
    cudaError_t e = launch_check_policy(pi_dev, lo, hi, pr.A, bad, pr.stream);
    int h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "policy check");
    if (h) return fail(RMB_ERR_INVALID_ARG, "pi holds an action outside [0, A)");
    return RMB_OK;
}

static void apply_create_flags(Problem& pr, uint32_t flags)
{
    pr.sparse_full_grid = (flags & RMB_SPARSE_FULL_GRID) != 0;
    pr.shard_no_graph = (flags & RMB_SHARD_NO_GRAPH) != 0;
}

static bool is_shard(const Problem& pr) { return pr.nccl_comm || pr.row_begin != 0 || pr.row_end != pr.n; }

// RMB_TRACE_ERROR_VS_REF (the paper's plotted metric P:L496,
// L575): etrace[i] = ||V_i - V*||_inf after application i, V* from
// rmb_set_reference; `apps` = applications the solve may run
static rmb_status error_trace_of(Problem& pr, uint32_t flags, int64_t apps, SolveRequest& rq)
{
    pr.etrace_count = 0;
    if (!(flags & RMB_TRACE_ERROR_VS_REF)) return RMB_OK;
    if (!pr.has_ref) return fail(RMB_ERR_INVALID_ARG, "RMB_TRACE_ERROR_VS_REF: no reference set (rmb_set_reference)");
    if (is_shard(pr) || (flags & RMB_FUSED))
        return fail(RMB_ERR_UNSUPPORTED, "RMB_TRACE_ERROR_VS_REF is single-GPU (not for row-range handles)");
    if (pr.etrace.ensure((size_t)std::max<int64_t>(1, apps) * 8) != cudaSuccess)
        return fail(RMB_ERR_OOM, "error trace allocation failed");
    cudaError_t e = cudaMemsetAsync(pr.etrace.p, 0, (size_t)std::max<int64_t>(1, apps) * 8, pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "error trace init");
    rq.vref = static_cast<const double*>(pr.ref_buf.p);
    rq.etrace = static_cast<double*>(pr.etrace.p);
    rq.etrace_len = apps;
    return RMB_OK;
}

// RMB_ASYNC (reading R31): single-GPU, partition order only
static rmb_status async_of(const Problem& pr, uint32_t flags, bool* as)
{
    *as = (flags & RMB_ASYNC) != 0;
    if (!*as) return RMB_OK;
    if (flags & (RMB_CHUNKED_T | RMB_SELECT_REPLACE | RMB_SELECT_WEIGHTED))
        return fail(RMB_ERR_INVALID_ARG, "RMB_ASYNC excludes RMB_CHUNKED_T and the RMB_SELECT_* draws");
    if (is_shard(pr) || (flags & RMB_FUSED))
        return fail(RMB_ERR_UNSUPPORTED, "RMB_ASYNC is single-GPU (not for row-range handles)");
    return RMB_OK;
}

// RMB_SELECT_REPLACE / RMB_SELECT_WEIGHTED (readings
// R28-R29): *sel = 0 (the partition), 1 (uniform draws) or 2 (weighted draws)
static rmb_status selection_of(const Problem& pr, uint32_t flags, int* sel)
{
    *sel = (flags & RMB_SELECT_WEIGHTED) ? 2 : ((flags & RMB_SELECT_REPLACE) ? 1 : 0);
    if (!*sel) return RMB_OK;
    if (*sel == 2 && !pr.sel_cum)
        return fail(RMB_ERR_INVALID_ARG, "RMB_SELECT_WEIGHTED: no weights set (rmb_set_selection_weights)");
    if (flags & (RMB_ORDER_IDENTITY | RMB_CHUNKED_T))
        return fail(RMB_ERR_INVALID_ARG, "draws with replacement exclude RMB_ORDER_IDENTITY and RMB_CHUNKED_T");
    if (is_shard(pr) || (flags & RMB_FUSED))
        return fail(RMB_ERR_UNSUPPORTED, "draws with replacement are single-GPU (not for row-range handles)");
    return RMB_OK;
}

static rmb_status solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t tl, long long* chg_dev,
                        int64_t cl, SolveResult* res)
{
    if (is_shard(pr))
        return fail(RMB_ERR_INVALID_ARG, "this handle owns a row range: use rmb_vi / rmb_mpi with an NCCL "
                                         "communicator, or rmb_vi_group / rmb_mpi_group");
    if (rq.async && pr.dense) return dense_async_solve(pr, rq, trace_dev, tl, chg_dev, cl, res);
    return pr.dense ? dense_solve(pr, rq, trace_dev, tl, chg_dev, cl, res)
                    : sparse_solve(pr, rq, trace_dev, tl, chg_dev, cl, res);
}

// Stage V (and optionally pi) to device.  Returns device pointers.
struct Staged {
    double* V = nullptr;
    int32_t* pi = nullptr;
    bool v_host = false, pi_host = false;
};

static rmb_status stage_in(Problem& pr, void* V, int32_t* pi, bool v_zero, bool copy_pi_in, Staged& s)
{
    const size_t vb = (size_t)pr.n * 8, pb = (size_t)pr.n * 4;
    cudaError_t e = cudaSuccess;
    if (is_device_ptr(V)) {
        s.V = static_cast<double*>(V);
    } else {
        if (pr.vstage.ensure(vb) != cudaSuccess) return fail(RMB_ERR_OOM, "V staging allocation failed");
        s.V = static_cast<double*>(pr.vstage.p);
        s.v_host = true;
        if (!v_zero) e = cudaMemcpyAsync(s.V, V, vb, cudaMemcpyHostToDevice, pr.stream);
    }
    if (e == cudaSuccess && v_zero) e = cudaMemsetAsync(s.V, 0, vb, pr.stream);
    if (pi) {
        if (is_device_ptr(pi)) {
            s.pi = pi;
        } else {
            if (pr.pistage.ensure(pb) != cudaSuccess) return fail(RMB_ERR_OOM, "pi staging allocation failed");
            s.pi = static_cast<int32_t*>(pr.pistage.p);
            s.pi_host = true;
            if (e == cudaSuccess && copy_pi_in) e = cudaMemcpyAsync(s.pi, pi, pb, cudaMemcpyHostToDevice, pr.stream);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "stage in");
    return RMB_OK;
}

static rmb_status stage_out(Problem& pr, void* V, int32_t* pi, const Staged& s)
{
    cudaError_t e = cudaSuccess;
    if (s.v_host) e = cudaMemcpyAsync(V, s.V, (size_t)pr.n * 8, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess && s.pi_host && pi)
        e = cudaMemcpyAsync(pi, s.pi, (size_t)pr.n * 4, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "stage out");
    return RMB_OK;
}

static rmb_status copy_trace(Problem& pr, double* host, const double* dev, int64_t cnt)
{
    if (!host || cnt <= 0) return RMB_OK;
    cudaError_t e = cudaMemcpyAsync(host, dev, (size_t)cnt * 8, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "trace copy");
    return RMB_OK;
}

static void fill_stats(rmb_stats* st, const SolveResult& r, rmb_status s)
{
    if (!st) return;
    st->sweeps = r.sweeps;
    st->batches = r.batches;
    st->outer_iters = r.outer;
    st->final_residual = r.final_resid;
    st->seconds = r.ms * 1e-3;
    st->converged = r.status == RMB_OK;
    st->status = s;
}

// MB-VI with draws with replacement (reading R30): the sweep residual r_k
// covers only the drawn states, so r_k <= eps only triggers a confirmation:
// ||TV - V||_inf over all states (the improvement pass, pi <- greedy(V));
// the solve stops iff that is <= eps, else it resumes with the next sweep.
// pi starts at 0 (states never drawn keep it until a confirmation pass).
static rmb_status vi_with_replacement(Problem& pr, const SolveRequest& rq0, SolveResult* res)
{
    cudaError_t e = cudaMemsetAsync(rq0.pi, 0, (size_t)pr.n * 4, pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "pi init");
    double* trace = static_cast<double*>(pr.trace.p);
    SolveResult tot;
    tot.status = RMB_ERR_NOT_CONVERGED;
    int64_t done = 0, launches = 0;
    while (done < rq0.max_iter) {
        SolveRequest rq = rq0;
        rq.k0 = rq0.k0 + done;
        rq.max_iter = rq0.max_iter - done;
        if (rq0.etrace) {
            rq.etrace = rq0.etrace + done;
            rq.etrace_len = rq0.etrace_len - done;
        }
        SolveResult r;
        rmb_status s = solve(pr, rq, trace + done, rq.max_iter, nullptr, 0, &r);
        if (s != RMB_OK) return s;
        done += r.sweeps;
        tot.sweeps += r.sweeps;
        tot.batches += r.batches;
        tot.ms += r.ms;
        tot.final_resid = r.final_resid;
        launches += r.launches;
        if (r.status != RMB_OK) {  // max_sweeps reached, or a non-finite value
            tot.status = r.status;
            break;
        }
        SolveRequest iq;
        iq.mode = MODE_IMPROVE;
        iq.b = pr.n;
        iq.identity = true;
        iq.V = rq0.V;
        iq.pi = rq0.pi;
        SolveResult ri;
        s = solve(pr, iq, nullptr, 0, nullptr, 0, &ri);
        if (s != RMB_OK) return s;
        tot.ms += ri.ms;
        launches += ri.launches;
        tot.final_resid = ri.final_resid;
        if (ri.status != RMB_OK) {
            tot.status = ri.status;
            break;
        }
        if (ri.final_resid <= rq0.eps) {
            tot.status = RMB_OK;
            break;
        }
    }
    tot.launches = (int)launches;
    pr.last_launches = launches;
    *res = tot;
    return RMB_OK;
}

}  // namespace rmb

using namespace rmb;

// ===================================================================== ABI
extern "C" {
rmb_status rmb_shard_range(int64_t n, int32_t G, int32_t g, int64_t* begin, int64_t* end);

const char* rmb_version(void) { return "rmb 0.1 (sm_100a)"; }

const char* rmb_last_error(void) { return g_err.c_str(); }

const char* rmb_status_string(rmb_status s)
{
    switch (s) {
    case RMB_OK: return "RMB_OK";
    case RMB_ERR_INVALID_ARG: return "RMB_ERR_INVALID_ARG";
    case RMB_ERR_INVALID_MDP: return "RMB_ERR_INVALID_MDP";
    case RMB_ERR_NOT_CONVERGED: return "RMB_ERR_NOT_CONVERGED";
    case RMB_ERR_NONFINITE: return "RMB_ERR_NONFINITE";
    case RMB_ERR_CUDA: return "RMB_ERR_CUDA";
    case RMB_ERR_NCCL: return "RMB_ERR_NCCL";
    case RMB_ERR_OOM: return "RMB_ERR_OOM";
    case RMB_ERR_UNSUPPORTED: return "RMB_ERR_UNSUPPORTED";
    }
    return "RMB_ERR_UNKNOWN";
}

rmb_status rmb_create_dense(const rmb_desc* desc, const void* P, const void* c, uint32_t flags, rmb_problem* out)
{
    g_err.clear();
    if (!out) return fail(RMB_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    rmb_status s = check_desc(desc);
    if (s != RMB_OK) return s;
    if (!P || !c) return fail(RMB_ERR_INVALID_ARG, "P or c is NULL");
    Problem* pr = new Problem();
    s = init_problem(*pr, desc);
    const size_t psz = desc->p_dtype == RMB_F32 ? 4 : 8;
    const size_t rows = (size_t)(desc->row_end - desc->row_begin);  // owned states (all of them on one GPU)
    const size_t pbytes = std::max<size_t>(1, rows * pr->A * pr->n * psz);
    if (s == RMB_OK) s = device_view(*pr, P, pbytes, &pr->P, "copy P to device");
    if (s == RMB_OK) s = device_view(*pr, c, std::max<size_t>(1, rows * pr->A * psz), &pr->c, "copy c to device");
    pr->dense = true;
    pr->no_tma = (flags & RMB_DENSE_NO_TMA) != 0;
    pr->vglobal = (flags & RMB_DENSE_VGLOBAL) != 0;
    pr->no_cluster = (flags & RMB_DENSE_NO_CLUSTER) != 0;
    apply_create_flags(*pr, flags);
    if (s == RMB_OK && (flags & RMB_VALIDATE)) s = validate_mdp(*pr);
    if (s != RMB_OK) {
        free_problem(pr);
        return s;
    }
    *out = reinterpret_cast<rmb_problem>(pr);
    return RMB_OK;
}

rmb_status rmb_create_csr(const rmb_desc* desc, const int64_t* row_ptr, const int32_t* col, const void* val,
                          const void* c, uint32_t flags, rmb_problem* out)
{
    g_err.clear();
    if (!out) return fail(RMB_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    rmb_status s = check_desc(desc);
    if (s != RMB_OK) return s;
    if (!row_ptr || !col || !val || !c) return fail(RMB_ERR_INVALID_ARG, "row_ptr, col, val or c is NULL");
    Problem* pr = new Problem();
    s = init_problem(*pr, desc);
    pr->dense = false;
    apply_create_flags(*pr, flags);
    const int64_t rows = (desc->row_end - desc->row_begin) * (int64_t)desc->n_actions;  // owned rows
    const size_t psz = desc->p_dtype == RMB_F32 ? 4 : 8;
    // row_ptr is inspected on the host (nnz, fixed stride -> ELL)
    std::vector<int64_t> rp;
    if (s == RMB_OK) {
        rp.resize((size_t)rows + 1);
        cudaError_t e = cudaMemcpy(rp.data(), row_ptr, (rows + 1) * sizeof(int64_t), cudaMemcpyDefault);
        if (e != cudaSuccess) s = cuda_fail(e, "read row_ptr");
    }
    if (s == RMB_OK) {
        if (rp[0] != 0) s = fail(RMB_ERR_INVALID_ARG, "row_ptr[0] != 0");
        for (int64_t r = 0; s == RMB_OK && r < rows; ++r)
            if (rp[r + 1] < rp[r]) s = fail(RMB_ERR_INVALID_ARG, "row_ptr is not nondecreasing");
    }
    if (s == RMB_OK) {
        pr->nnz = rp[rows];
        const int64_t K = rows > 0 ? rp[1] - rp[0] : 0;
        bool ell = K > 0;
        for (int64_t r = 0; ell && r <= rows; ++r) ell = rp[r] == r * K;
        pr->ell_K = ell ? (int)K : 0;
    }
    if (s == RMB_OK) s = device_view(*pr, row_ptr, (rows + 1) * sizeof(int64_t), (const void**)&pr->row_ptr, "copy row_ptr");
    if (s == RMB_OK) s = device_view(*pr, col, (size_t)pr->nnz * 4, (const void**)&pr->col, "copy col");
    if (s == RMB_OK) s = device_view(*pr, val, (size_t)pr->nnz * psz, &pr->val, "copy val");
    if (s == RMB_OK) s = device_view(*pr, c, (size_t)rows * psz, &pr->c, "copy c");
    if (s == RMB_OK && (flags & RMB_VALIDATE)) s = validate_mdp(*pr);
    if (s != RMB_OK) {
        free_problem(pr);
        return s;
    }
    *out = reinterpret_cast<rmb_problem>(pr);
    return RMB_OK;
}

rmb_status rmb_destroy(rmb_problem h)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem* pr = reinterpret_cast<Problem*>(h);
    cudaStreamSynchronize(pr->stream);
    free_problem(pr);
    return RMB_OK;
}

int64_t rmb_last_launch_count(rmb_problem h)
{
    return h ? reinterpret_cast<Problem*>(h)->last_launches : 0;
}

int64_t rmb_last_graph_launches(rmb_problem h)
{
    return h ? reinterpret_cast<Problem*>(h)->last_graph_launches : 0;
}

rmb_status rmb_last_phase_times(rmb_problem h, int64_t* ns4)
{
    if (!h || !ns4) return fail(RMB_ERR_INVALID_ARG, "handle or ns4 is NULL");
    const Problem* pr = reinterpret_cast<const Problem*>(h);
    for (int i = 0; i < 4; ++i) ns4[i] = pr->prof[i];
    return RMB_OK;
}

rmb_status rmb_vi(rmb_problem h, int64_t b, uint64_t seed, double eps, int64_t max_sweeps, uint32_t flags, void* V,
                  int32_t* pi, double* trace, rmb_stats* stats)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (b < 1 || b > pr.n) return fail(RMB_ERR_INVALID_ARG, "b not in [1, n]");
    if (!(eps > 0.0) || !std::isfinite(eps)) return fail(RMB_ERR_INVALID_ARG, "eps must be finite and > 0");
    if (max_sweeps < 1) return fail(RMB_ERR_INVALID_ARG, "max_sweeps < 1");
    if (!V || !pi) return fail(RMB_ERR_INVALID_ARG, "V or pi is NULL");
    int sel = 0;
    bool as = false;
    rmb_status s = selection_of(pr, flags, &sel);
    if (s == RMB_OK) s = async_of(pr, flags, &as);
    if (s != RMB_OK) return s;
    Staged sg;
    s = stage_in(pr, V, pi, flags & RMB_V0_ZERO, false, sg);
    if (s != RMB_OK) return s;
    if (pr.trace.ensure((size_t)max_sweeps * 8) != cudaSuccess) return fail(RMB_ERR_OOM, "trace allocation failed");
    SolveRequest rq;
    rq.select = sel;
    rq.async = as;
    s = error_trace_of(pr, flags, max_sweeps, rq);
    if (s != RMB_OK) return s;
    rq.mode = MODE_VI;
    rq.b = b;
    rq.seed = seed;
    rq.k0 = 1;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.fused = flags & RMB_FUSED;
    rq.chunked = flags & RMB_CHUNKED_T;
    rq.eps = eps;
    rq.max_iter = max_sweeps;
    rq.V = sg.V;
    rq.pi = sg.pi;
    SolveResult r;
    if (is_shard(pr) && rq.chunked) return fail(RMB_ERR_UNSUPPORTED, "RMB_CHUNKED_T on a row-range (sharded) handle");
    if (is_shard(pr)) {  // multi-GPU: this rank's rows, NCCL exchange per batch
        if (!pr.nccl_comm) return fail(RMB_ERR_INVALID_ARG, "a row-range handle needs nccl_comm (or rmb_vi_group)");
        pr.stage_V = sg.V;
        pr.stage_pi = sg.pi;
        std::vector<double> tr((size_t)max_sweeps);
        Problem* one = &pr;
        s = sharded_solve(&one, 1, true, rq, tr.data(), max_sweeps, nullptr, 0, &r);
        if (s != RMB_OK) return s;
        s = stage_out(pr, V, pi, sg);
        if (s == RMB_OK && trace) memcpy(trace, tr.data(), (size_t)r.sweeps * 8);
        if (s != RMB_OK) return s;
        rmb_status ret = (rmb_status)r.status;
        fill_stats(stats, r, ret);
        return ret;
    }
    s = sel ? vi_with_replacement(pr, rq, &r) : solve(pr, rq, static_cast<double*>(pr.trace.p), max_sweeps, nullptr, 0, &r);
    if (s != RMB_OK) return s;
    if (rq.etrace) pr.etrace_count = std::min<int64_t>(r.sweeps, max_sweeps);
    s = stage_out(pr, V, pi, sg);
    if (s == RMB_OK) s = copy_trace(pr, trace, static_cast<double*>(pr.trace.p), r.sweeps);
    if (s != RMB_OK) return s;
    rmb_status ret = (rmb_status)r.status;
    if (ret == RMB_ERR_NOT_CONVERGED) g_err = sel ? "max_sweeps reached before ||TV - V|| <= eps" : "max_sweeps reached before r_k <= eps";
    if (ret == RMB_ERR_NONFINITE) g_err = "a backup produced a non-finite value";
    fill_stats(stats, r, ret);
    return ret;
}

rmb_status rmb_mpi(rmb_problem h, int64_t b, int32_t m, uint64_t seed, double eps, int64_t max_outer, uint32_t flags,
                   void* V, int32_t* pi, double* trace, int64_t* changed, rmb_stats* stats)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (b < 1 || b > pr.n) return fail(RMB_ERR_INVALID_ARG, "b not in [1, n]");
    if (m < 1) return fail(RMB_ERR_INVALID_ARG, "m < 1");
    if (!(eps > 0.0) || !std::isfinite(eps)) return fail(RMB_ERR_INVALID_ARG, "eps must be finite and > 0");
    if (max_outer < 1) return fail(RMB_ERR_INVALID_ARG, "max_outer < 1");
    if (!V || !pi) return fail(RMB_ERR_INVALID_ARG, "V or pi is NULL");
    const bool pi_given = flags & RMB_PI_GIVEN;
    int sel = 0;
    bool as = false;
    rmb_status s = selection_of(pr, flags, &sel);
    if (s == RMB_OK) s = async_of(pr, flags, &as);
    if (s != RMB_OK) return s;
    Staged sg;
    s = stage_in(pr, V, pi, flags & RMB_V0_ZERO, pi_given, sg);
    if (s != RMB_OK) return s;
    if (pi_given) {  // the given policy's owned entries must be actions in [0, A)
        s = check_policy(pr, sg.pi, pr.row_begin, pr.row_end);
        if (s != RMB_OK) return s;
    }
    const int64_t tl = max_outer * (int64_t)(m + 1);
    if (pr.trace.ensure((size_t)tl * 8) != cudaSuccess || pr.chg.ensure((size_t)max_outer * 8) != cudaSuccess)
        return fail(RMB_ERR_OOM, "trace allocation failed");
    SolveRequest rq;
    rq.mode = MODE_MPI;
    rq.select = sel;
    rq.async = as;
    s = error_trace_of(pr, flags, max_outer * (int64_t)m, rq);
    if (s != RMB_OK) return s;
    rq.b = b;
    rq.msweeps = m;
    rq.seed = seed;
    rq.k0 = 1;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.fused = flags & RMB_FUSED;
    rq.eps = eps;
    rq.max_iter = max_outer;
    rq.pi_given = pi_given;
    rq.V = sg.V;
    rq.pi = sg.pi;
    SolveResult r;
    if (is_shard(pr)) {
        if (!pr.nccl_comm) return fail(RMB_ERR_INVALID_ARG, "a row-range handle needs nccl_comm (or rmb_mpi_group)");
        pr.stage_V = sg.V;
        pr.stage_pi = sg.pi;
        std::vector<double> tr((size_t)tl);
        std::vector<int64_t> ch((size_t)max_outer);
        Problem* one = &pr;
        s = sharded_solve(&one, 1, true, rq, tr.data(), tl, ch.data(), max_outer, &r);
        if (s != RMB_OK) return s;
        s = stage_out(pr, V, pi, sg);
        if (s != RMB_OK) return s;
        if (trace) memcpy(trace, tr.data(), (size_t)(r.outer * (m + 1)) * 8);
        if (changed) memcpy(changed, ch.data(), (size_t)r.outer * 8);
        rmb_status ret = (rmb_status)r.status;
        fill_stats(stats, r, ret);
        return ret;
    }
    s = solve(pr, rq, static_cast<double*>(pr.trace.p), tl, static_cast<long long*>(pr.chg.p), max_outer, &r);
    if (s != RMB_OK) return s;
    if (rq.etrace) pr.etrace_count = std::min<int64_t>(r.sweeps, max_outer * (int64_t)m);
    s = stage_out(pr, V, pi, sg);
    if (s == RMB_OK) s = copy_trace(pr, trace, static_cast<double*>(pr.trace.p), r.outer * (int64_t)(m + 1));
    if (s == RMB_OK && changed && r.outer > 0) {
        cudaError_t e = cudaMemcpyAsync(changed, pr.chg.p, (size_t)r.outer * 8, cudaMemcpyDeviceToHost, pr.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
        if (e != cudaSuccess) s = cuda_fail(e, "changed copy");
    }
    if (s != RMB_OK) return s;
    rmb_status ret = (rmb_status)r.status;
    if (ret == RMB_ERR_NOT_CONVERGED) g_err = "max_outer reached before the policy was stable with ||TV-V|| <= eps";
    if (ret == RMB_ERR_NONFINITE) g_err = "a backup produced a non-finite value";
    fill_stats(stats, r, ret);
    return ret;
}

// G logical ranks on ONE device (handles created with rmb_shard_range row
// ranges): the sharded protocol with device-copy exchange.  Each rank keeps its
// own replica of V; outputs are rank 0's V and pi assembled from the owners.
static rmb_status group_solve(rmb_problem* hs, int32_t G, SolveRequest rq, uint32_t flags, void* V, int32_t* pi,
                              double* trace, int64_t tl, int64_t* changed, int64_t cl, rmb_stats* stats)
{
    if (!hs || G < 1) return fail(RMB_ERR_INVALID_ARG, "handles NULL or G < 1");
    if (flags & (RMB_SELECT_REPLACE | RMB_SELECT_WEIGHTED | RMB_ASYNC | RMB_TRACE_ERROR_VS_REF))
        return fail(RMB_ERR_UNSUPPORTED, "draws with replacement, RMB_ASYNC and RMB_TRACE_ERROR_VS_REF are single-GPU (not for rmb_*_group)");
    if (!V || !pi) return fail(RMB_ERR_INVALID_ARG, "V or pi is NULL");
    std::vector<Problem*> rk((size_t)G);
    for (int g = 0; g < G; ++g) {
        if (!hs[g]) return fail(RMB_ERR_INVALID_ARG, "a handle is NULL");
        rk[g] = reinterpret_cast<Problem*>(hs[g]);
        const Problem& p = *rk[g];
        const Problem& p0 = *rk[0];
        int64_t b0, b1;
        rmb_shard_range(p0.n, G, g, &b0, &b1);
        if (p.n != p0.n || p.A != p0.A || p.gamma != p0.gamma || p.pdt != p0.pdt || p.dense != p0.dense || p.nccl_comm ||
            p.row_begin != b0 || p.row_end != b1 || p.stream != p0.stream)
            return fail(RMB_ERR_INVALID_ARG, "group handles must share n, A, gamma, dtype, stream and own the "
                                             "rmb_shard_range(n, G, g) rows in rank order");
    }
    Problem& p0 = *rk[0];
    const int64_t n = p0.n;
    if (rq.b < 1 || rq.b > n) return fail(RMB_ERR_INVALID_ARG, "b not in [1, n]");
    const size_t vb = (size_t)n * 8, pb = (size_t)n * 4;
    const bool v_zero = flags & RMB_V0_ZERO;
    cudaStream_t st = p0.stream;
    for (int g = 0; g < G; ++g) {
        Problem& p = *rk[g];
        if (p.vstage.ensure(vb) != cudaSuccess || p.pistage.ensure(pb) != cudaSuccess)
            return fail(RMB_ERR_OOM, "replica allocation failed");
        p.stage_V = static_cast<double*>(p.vstage.p);
        p.stage_pi = static_cast<int32_t*>(p.pistage.p);
        cudaError_t e = v_zero ? cudaMemsetAsync(p.stage_V, 0, vb, st)
                               : cudaMemcpyAsync(p.stage_V, V, vb, cudaMemcpyDefault, st);
        if (e == cudaSuccess) e = rq.pi_given ? cudaMemcpyAsync(p.stage_pi, pi, pb, cudaMemcpyDefault, st)
                                              : cudaMemsetAsync(p.stage_pi, 0, pb, st);
        if (e != cudaSuccess) return cuda_fail(e, "group staging");
        if (rq.pi_given) {
            rmb_status cs = check_policy(p, p.stage_pi, p.row_begin, p.row_end);
            if (cs != RMB_OK) return cs;
        }
    }
    SolveResult r;
    rmb_status s = sharded_solve(rk.data(), G, false, rq, trace, tl, changed, cl, &r);
    if (s != RMB_OK) return s;
    cudaError_t e = cudaMemcpyAsync(V, p0.stage_V, vb, cudaMemcpyDefault, st);
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        const Problem& p = *rk[g];
        if (p.row_end > p.row_begin)
            e = cudaMemcpyAsync(pi + p.row_begin, p.stage_pi + p.row_begin, (size_t)(p.row_end - p.row_begin) * 4,
                                cudaMemcpyDefault, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "group outputs");
    rmb_status ret = (rmb_status)r.status;
    if (ret == RMB_ERR_NOT_CONVERGED) g_err = "iteration limit reached before the stopping test passed";
    fill_stats(stats, r, ret);
    return ret;
}

rmb_status rmb_vi_group(rmb_problem* hs, int32_t G, int64_t b, uint64_t seed, double eps, int64_t max_sweeps,
                        uint32_t flags, void* V, int32_t* pi, double* trace, rmb_stats* stats)
{
    g_err.clear();
    if (!(eps > 0.0) || !std::isfinite(eps) || max_sweeps < 1) return fail(RMB_ERR_INVALID_ARG, "eps or max_sweeps");
    SolveRequest rq;
    rq.mode = MODE_VI;
    rq.b = b;
    rq.seed = seed;
    rq.k0 = 1;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.fused = flags & RMB_FUSED;
    rq.eps = eps;
    rq.max_iter = max_sweeps;
    return group_solve(hs, G, rq, flags, V, pi, trace, trace ? max_sweeps : 0, nullptr, 0, stats);
}

rmb_status rmb_mpi_group(rmb_problem* hs, int32_t G, int64_t b, int32_t m, uint64_t seed, double eps,
                         int64_t max_outer, uint32_t flags, void* V, int32_t* pi, double* trace, int64_t* changed,
                         rmb_stats* stats)
{
    g_err.clear();
    if (m < 1 || !(eps > 0.0) || !std::isfinite(eps) || max_outer < 1)
        return fail(RMB_ERR_INVALID_ARG, "m, eps or max_outer");
    SolveRequest rq;
    rq.mode = MODE_MPI;
    rq.b = b;
    rq.msweeps = m;
    rq.seed = seed;
    rq.k0 = 1;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.fused = flags & RMB_FUSED;
    rq.eps = eps;
    rq.max_iter = max_outer;
    rq.pi_given = flags & RMB_PI_GIVEN;
    return group_solve(hs, G, rq, flags, V, pi, trace, trace ? max_outer * (int64_t)(m + 1) : 0, changed,
                       changed ? max_outer : 0, stats);
}

rmb_status rmb_apply(rmb_problem h, int64_t b, uint64_t seed, int64_t sweep, uint32_t flags, const int32_t* pi_or_null,
                     const void* V_in, void* V_out, int32_t* argmin_out, double* resid_out)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (b < 1 || b > pr.n) return fail(RMB_ERR_INVALID_ARG, "b not in [1, n]");
    if (sweep < 1) return fail(RMB_ERR_INVALID_ARG, "sweep < 1");
    if (!V_in || !V_out) return fail(RMB_ERR_INVALID_ARG, "V_in or V_out is NULL");
    int sel = 0;
    bool as = false;
    {
        rmb_status ss = selection_of(pr, flags, &sel);
        if (ss == RMB_OK) ss = async_of(pr, flags, &as);
        if (ss != RMB_OK) return ss;
    }
    const size_t vb = (size_t)pr.n * 8, pb = (size_t)pr.n * 4;
    cudaError_t e = cudaSuccess;
    // working V on device: V_out if device, else staging
    const bool out_dev = is_device_ptr(V_out);
    double* Vw;
    if (out_dev) {
        Vw = static_cast<double*>(V_out);
    } else {
        if (pr.vstage.ensure(vb) != cudaSuccess) return fail(RMB_ERR_OOM, "V staging allocation failed");
        Vw = static_cast<double*>(pr.vstage.p);
    }
    if (V_in != (const void*)Vw) e = cudaMemcpyAsync(Vw, V_in, vb, cudaMemcpyDefault, pr.stream);
    // policy / argmin buffer on device
    if (pr.pistage.ensure(pb) != cudaSuccess) return fail(RMB_ERR_OOM, "pi staging allocation failed");
    int32_t* pw = nullptr;
    if (pi_or_null) {
        if (is_device_ptr(pi_or_null)) {
            pw = const_cast<int32_t*>(pi_or_null);
        } else {
            pw = static_cast<int32_t*>(pr.pistage.p);
            if (e == cudaSuccess) e = cudaMemcpyAsync(pw, pi_or_null, pb, cudaMemcpyHostToDevice, pr.stream);
        }
    } else if (argmin_out) {
        pw = is_device_ptr(argmin_out) ? argmin_out : static_cast<int32_t*>(pr.pistage.p);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rmb_apply staging");
    if (pi_or_null) {
        rmb_status cs = check_policy(pr, pw, 0, pr.n);
        if (cs != RMB_OK) return cs;
    }
    if (pr.trace.ensure(64) != cudaSuccess) return fail(RMB_ERR_OOM, "trace allocation failed");
    SolveRequest rq;
    rq.mode = pi_or_null ? MODE_APPLY_PI : MODE_APPLY;
    rq.select = sel;
    rq.async = as;
    rq.b = b;
    rq.seed = seed;
    rq.k0 = sweep;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.chunked = flags & RMB_CHUNKED_T;
    rq.eps = -1.0;
    rq.max_iter = 1;
    rq.V = Vw;
    rq.pi = pw;
    SolveResult r;
    rmb_status s = solve(pr, rq, static_cast<double*>(pr.trace.p), 1, nullptr, 0, &r);
    if (s != RMB_OK) return s;
    if (!out_dev) e = cudaMemcpyAsync(V_out, Vw, vb, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess && argmin_out && argmin_out != pw)
        e = cudaMemcpyAsync(argmin_out, pw, pb, cudaMemcpyDefault, pr.stream);
    double rr = 0.0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&rr, pr.trace.p, 8, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "rmb_apply copy out");
    if (resid_out) *resid_out = rr;
    if (r.status == RMB_ERR_NONFINITE) g_err = "a backup produced a non-finite value";
    return (rmb_status)r.status;
}

rmb_status rmb_improve(rmb_problem h, const void* V, int32_t* pi, double* bellman_resid, int64_t* changed)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (!V || !pi) return fail(RMB_ERR_INVALID_ARG, "V or pi is NULL");
    Staged sg;
    rmb_status s = stage_in(pr, const_cast<void*>(V), pi, false, true, sg);
    if (s != RMB_OK) return s;
    if (pr.trace.ensure(64) != cudaSuccess) return fail(RMB_ERR_OOM, "trace allocation failed");
    SolveRequest rq;
    rq.mode = MODE_IMPROVE;
    rq.b = pr.n;
    rq.identity = true;
    rq.V = sg.V;
    rq.pi = sg.pi;
    SolveResult r;
    s = solve(pr, rq, static_cast<double*>(pr.trace.p), 1, nullptr, 0, &r);
    if (s != RMB_OK) return s;
    cudaError_t e = cudaSuccess;
    if (sg.pi_host) e = cudaMemcpyAsync(pi, sg.pi, (size_t)pr.n * 4, cudaMemcpyDeviceToHost, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "rmb_improve copy out");
    if (bellman_resid) *bellman_resid = r.final_resid;
    if (changed) *changed = r.changed;
    return (rmb_status)r.status;
}

rmb_status rmb_policy_value(rmb_problem h, const int32_t* pi, int64_t b, uint64_t seed, double eps, int64_t max_sweeps,
                            uint32_t flags, void* V, double* trace, rmb_stats* stats)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (b < 1 || b > pr.n) return fail(RMB_ERR_INVALID_ARG, "b not in [1, n]");
    if (!(eps > 0.0) || !std::isfinite(eps)) return fail(RMB_ERR_INVALID_ARG, "eps must be finite and > 0");
    if (max_sweeps < 1) return fail(RMB_ERR_INVALID_ARG, "max_sweeps < 1");
    if (!V || !pi) return fail(RMB_ERR_INVALID_ARG, "V or pi is NULL");
    if (flags & (RMB_SELECT_REPLACE | RMB_SELECT_WEIGHTED))
        return fail(RMB_ERR_UNSUPPORTED, "rmb_policy_value: draws with replacement are not offered (its stop test is the sweep residual)");
    bool as = false;
    rmb_status s = async_of(pr, flags, &as);
    if (s != RMB_OK) return s;
    Staged sg;
    s = stage_in(pr, V, const_cast<int32_t*>(pi), flags & RMB_V0_ZERO, true, sg);
    if (s != RMB_OK) return s;
    s = check_policy(pr, sg.pi, 0, pr.n);
    if (s != RMB_OK) return s;
    if (pr.trace.ensure((size_t)max_sweeps * 8) != cudaSuccess) return fail(RMB_ERR_OOM, "trace allocation failed");
    SolveRequest rq;
    rq.mode = MODE_POLICY_VALUE;
    rq.async = as;
    s = error_trace_of(pr, flags, max_sweeps, rq);
    if (s != RMB_OK) return s;
    rq.b = b;
    rq.seed = seed;
    rq.k0 = 1;
    rq.identity = flags & RMB_ORDER_IDENTITY;
    rq.eps = eps;
    rq.max_iter = max_sweeps;
    rq.V = sg.V;
    rq.pi = sg.pi;
    SolveResult r;
    s = solve(pr, rq, static_cast<double*>(pr.trace.p), max_sweeps, nullptr, 0, &r);
    if (s != RMB_OK) return s;
    if (rq.etrace) pr.etrace_count = std::min<int64_t>(r.sweeps, max_sweeps);
    Staged vo = sg;
    vo.pi_host = false;  // pi is an input here
    s = stage_out(pr, V, nullptr, vo);
    if (s == RMB_OK) s = copy_trace(pr, trace, static_cast<double*>(pr.trace.p), r.sweeps);
    if (s != RMB_OK) return s;
    rmb_status ret = (rmb_status)r.status;
    if (ret == RMB_ERR_NOT_CONVERGED) g_err = "max_sweeps reached before r_k <= eps";
    fill_stats(stats, r, ret);
    return ret;
}

rmb_status rmb_partition(int64_t n, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* perm)
{
    g_err.clear();
    if (n < 1 || n > 0xffffffffLL || !perm) return fail(RMB_ERR_INVALID_ARG, "n out of range or perm NULL");
    if (flags & RMB_ORDER_IDENTITY) {
        for (int64_t p = 0; p < n; ++p) perm[p] = (uint32_t)p;
        return RMB_OK;
    }
    Permutation pm;
    pm.init(n, seed, sweep);
    for (int64_t p = 0; p < n; ++p) perm[p] = (uint32_t)pm((uint64_t)p);
    return RMB_OK;
}

rmb_status rmb_set_reference(rmb_problem h, const void* Vref)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (!Vref) {
        pr.has_ref = false;
        return RMB_OK;
    }
    if (pr.ref_buf.ensure((size_t)pr.n * 8) != cudaSuccess) return fail(RMB_ERR_OOM, "reference allocation failed");
    cudaError_t e = cudaMemcpyAsync(pr.ref_buf.p, Vref, (size_t)pr.n * 8, cudaMemcpyDefault, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "copy reference");
    pr.has_ref = true;
    return RMB_OK;
}

rmb_status rmb_error_trace(rmb_problem h, double* out, int64_t len, int64_t* count)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (count) *count = pr.etrace_count;
    const int64_t m = std::min<int64_t>(len, pr.etrace_count);
    if (!out || m <= 0) return RMB_OK;
    cudaError_t e = cudaMemcpyAsync(out, pr.etrace.p, (size_t)m * 8, cudaMemcpyDefault, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "error trace copy");
    return RMB_OK;
}

rmb_status rmb_set_selection_weights(rmb_problem h, const uint32_t* w)
{
    g_err.clear();
    if (!h) return fail(RMB_ERR_INVALID_ARG, "handle is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    if (!w) {
        pr.sel_cum = nullptr;
        pr.sel_W = 0;
        return RMB_OK;
    }
    const int64_t n = pr.n;
    if (n > 0x7fffffffLL) return fail(RMB_ERR_UNSUPPORTED, "weighted selection needs n < 2^31");
    std::vector<uint32_t> hw((size_t)n);
    cudaError_t e = cudaMemcpy(hw.data(), w, (size_t)n * 4, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(e, "read weights");
    std::vector<uint64_t> cum((size_t)n);
    uint64_t W = 0;
    for (int64_t s = 0; s < n; ++s) {
        if (hw[(size_t)s] == 0) return fail(RMB_ERR_INVALID_ARG, "a selection weight is 0 (every state needs w >= 1)");
        W += hw[(size_t)s];
        cum[(size_t)s] = W;
    }
    if (pr.sel_buf.ensure((size_t)n * 8) != cudaSuccess) return fail(RMB_ERR_OOM, "weights allocation failed");
    e = cudaMemcpyAsync(pr.sel_buf.p, cum.data(), (size_t)n * 8, cudaMemcpyHostToDevice, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "upload weights");
    pr.sel_cum = static_cast<const uint64_t*>(pr.sel_buf.p);
    pr.sel_W = W;
    return RMB_OK;
}

rmb_status rmb_select(int64_t n, uint64_t seed, int64_t sweep, const uint32_t* w, uint32_t* sel)
{
    g_err.clear();
    if (n < 1 || n > 0x7fffffffLL || !sel) return fail(RMB_ERR_INVALID_ARG, "n out of range or sel NULL");
    std::vector<uint64_t> cum;
    uint64_t W = 0;
    if (w) {
        cum.resize((size_t)n);
        for (int64_t s = 0; s < n; ++s) {
            if (w[s] == 0) return fail(RMB_ERR_INVALID_ARG, "a selection weight is 0");
            W += w[s];
            cum[(size_t)s] = W;
        }
    }
    fill_order(n, seed, sweep, OrderSpec{w ? 2 : 1, w ? cum.data() : nullptr, W}, sel, 0, 1);
    return RMB_OK;
}

rmb_status rmb_select_device(rmb_problem h, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* sel)
{
    g_err.clear();
    if (!h || !sel) return fail(RMB_ERR_INVALID_ARG, "handle or sel is NULL");
    Problem& pr = *reinterpret_cast<Problem*>(h);
    int s = 0;
    rmb_status st = selection_of(pr, flags & (RMB_SELECT_REPLACE | RMB_SELECT_WEIGHTED), &s);
    if (st != RMB_OK) return st;
    if (!s) return fail(RMB_ERR_INVALID_ARG, "flags must hold RMB_SELECT_REPLACE or RMB_SELECT_WEIGHTED");
    cudaError_t e = launch_select(pr.n, seed, sweep, s, pr.sel_cum, pr.sel_W, sel, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) return cuda_fail(e, "rmb_select_device");
    return RMB_OK;
}

rmb_status rmb_partition_device(int64_t n, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* perm, void* stream)
{
    g_err.clear();
    if (n < 1 || n > 0xffffffffLL || !perm) return fail(RMB_ERR_INVALID_ARG, "n out of range or perm NULL");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = launch_partition(n, seed, sweep, flags & RMB_ORDER_IDENTITY, perm, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "rmb_partition_device");
    return RMB_OK;
}

}  // extern "C"

/*
 * rmb.h — C ABI of the B200-native randomized mini-batch DP library.
 *
 * Method: the randomized mini-batch operator of arXiv 2110.02901
 * (Gargiani, Martinelli, Ruts Martinez, Lygeros), Sec. III:
 *   B_b J(i)      = min_u [ g(i,u) + a sum_{j in S\M(i)} p_ij(u) J(j)
 *                                  + a sum_{j in M(i)}   p_ij(u) B_b J(j) ]   (Eq. 12)
 *   B_{mu,b} J(i) = the same with u = mu(i)                                  (Eq. 13)
 * where M(i) is the set of states in earlier batches of size b (Eq. M(i),
 * P:L163-166) after a random re-indexing drawn before every operator
 * application.  b = |S| gives the Bellman operator T, b = 1
 * the Gauss-Seidel operator F.  MB-VI and MB-MPI (Alg. 1
 * P:L103-131) apply it until the sup-norm residual falls below eps.
 *
 * Notation: b = batch size (the paper's m), m = MPI
 * evaluation sweeps per outer iteration (the paper's K), gamma = alpha,
 * c(s,a) = g(i,u), V = J, pi = mu.
 *
 * Conventions for every entry point:
 *   - all sizes are int64_t; states are 0-based;
 *   - P, c, row_ptr/col/val, V and pi may be DEVICE pointers or HOST
 *     pointers (pageable or pinned); the library inspects each pointer
 *     (cudaPointerGetAttributes) and stages host buffers through device
 *     memory it owns, copying results back before returning;
 *   - every call returns only after its results are complete and, for host
 *     outputs, copied back (the stream given at create is synchronised);
 *   - no call aborts the process: errors are returned as rmb_status and a
 *     human-readable message is available from rmb_last_error() (per thread).
 *   - one handle is used by one host thread at a time.
 */
#ifndef RMB_H
#define RMB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rmb_problem_s* rmb_problem; /* opaque */

typedef enum {
    RMB_OK = 0,
    RMB_ERR_INVALID_ARG = 1,   /* argument check failed; no device work was done          */
    RMB_ERR_INVALID_MDP = 2,   /* RMB_VALIDATE: a row does not sum to 1, a column is out
                                  of range, or a cost is not finite */
    RMB_ERR_NOT_CONVERGED = 3, /* max sweeps / outer iterations reached; V, pi, trace valid */
    RMB_ERR_NONFINITE = 4,     /* a backup produced inf/nan; the solve stopped there        */
    RMB_ERR_CUDA = 5,          /* a CUDA runtime error (message in rmb_last_error)          */
    RMB_ERR_NCCL = 6,          /* reserved: multi-GPU exchange error                        */
    RMB_ERR_OOM = 7,           /* device or host allocation failed                          */
    RMB_ERR_UNSUPPORTED = 8    /* a valid request outside this build's supported envelope   */
} rmb_status;

typedef enum { RMB_F32 = 0, RMB_F64 = 1 } rmb_dtype;

/* Problem description: the tuple (S, U, P, g, alpha) of P:L37 with a uniform
 * action count (state-dependent U(i) is encoded by duplicating an admissible
 * action's row; the lowest-index tie-break makes that exact). */
typedef struct {
    int64_t n_states;   /* |S| >= 1                                                  */
    int32_t n_actions;  /* |A| >= 1                                                  */
    double gamma;       /* discount alpha in (0,1)                                   */
    rmb_dtype p_dtype;  /* storage type of P (or CSR val) and c                      */
    rmb_dtype v_dtype;  /* storage type of V: RMB_F64 only in this build             */
    int64_t row_begin;  /* owned states [row_begin,row_end); 0 and n_states on 1 GPU  */
    int64_t row_end;    /*   (sharded handles: see the multi-GPU section below)      */
    void* nccl_comm;    /* ncclComm_t from rmb_nccl_comm_init for sharded solves, or NULL */
    void* stream;       /* cudaStream_t used for all work of this handle (NULL = legacy default) */
} rmb_desc;

/* flags */
#define RMB_ORDER_IDENTITY 0x1u /* no shuffle: ascending order (the paper's Sec. III analysis) */
#define RMB_V0_ZERO 0x2u        /* ignore V's content on entry and start from V0 = 0        */
#define RMB_PI_GIVEN 0x4u       /* rmb_mpi: pi holds the initial policy (else pi_0 = greedy(V0))     */
#define RMB_VALIDATE 0x8u       /* rmb_create_*: check the MDP on device (RMB_ERR_INVALID_MDP)       */
#define RMB_DENSE_VGLOBAL 0x20u /* rmb_create_dense: keep V and pi in global memory (L2) even when a
                                   shared-memory copy fits (automatic for n > ~20k: the TMA path's
                                   global-V mode); for tests of that mode on small instances    */
#define RMB_DENSE_NO_TMA 0x10u  /* rmb_create_dense: stream P rows with per-warp register loads instead
                                   of the default TMA (cp.async.bulk) shared-memory ring; results agree
                                   to fp64 rounding (A/B measurement and cross-path tests)            */
#define RMB_CHUNKED_T 0x40u     /* rmb_vi / rmb_apply: "VI*" of P:L570, L577 (Sec. IV-B) -- every sweep is
                                   the Bellman operator T computed in chunks of b states (the batches of
                                   the sweep's partition), each chunk "using the old values": all chunks
                                   read the sweep-start V, the new values land at the end of the sweep.
                                   One barrier per chunk, like B_b; the result is T V for any b, order
                                   and chunking (DESIGN reading R21).  Not for sharded handles.        */
#define RMB_DENSE_NO_CLUSTER 0x1000u /* rmb_create_dense: never use the one-cluster solver for tiny batches
                                      (<= 2 MB of P and <= 256 rows per batch: 16 CTAs, DSMEM combine,
                                      hardware cluster barrier; b = 1 with <= 16 rows: a look-ahead
                                      kernel exchanging partials by st.async); results agree to fp64
                                      rounding                                                          */
#define RMB_SELECT_REPLACE 0x2000u  /* rmb_vi / rmb_mpi / rmb_apply: SURVEY 8(f) row 4, P:L605 ("sampling the
                                       states with replacement and/or according to a non-uniform
                                       distribution") -- every operator application draws n states
                                       i.i.d. uniformly WITH replacement (DESIGN R28: counter-based,
                                       s_i = floor(mix64(skey_k + i) * n / 2^64)); batches are
                                       consecutive blocks of b draws; a state drawn twice in a batch is
                                       backed up once; undrawn states keep their values.  rmb_vi's stop
                                       test then confirms r_k <= eps with ||TV - V||_inf <= eps over all
                                       states (R30; pi = greedy(V) on OK).  Single-GPU handles only;
                                       excludes RMB_ORDER_IDENTITY and RMB_CHUNKED_T.                   */
#define RMB_SELECT_WEIGHTED 0x4000u /* as RMB_SELECT_REPLACE, drawing state s with probability w_s / W for
                                       the handle's integer weights (rmb_set_selection_weights; DESIGN
                                       R29: inverse CDF on integer prefix sums).  Importance-sampling and
                                       epsilon-greedy laws are choices of w.                             */
#define RMB_ASYNC 0x8000u /* rmb_vi / rmb_mpi / rmb_apply / rmb_policy_value: ASYNCHRONOUS applications
                             ("asynchronous variants of MB-VI and MB-MPI ...
                             avoiding synchronization"; DESIGN R31): every application walks the
                             states in the order of its partition with no batch barrier -- each
                             state is backed up against V as found in memory (every value read is
                             one its state held since the application began) and written at once;
                             one grid barrier per application (residual, stop test).  b is not used
                             (pass any value in [1, n]).  Results are NOT deterministic: for V0 with
                             T V0 <= V0 every iterate lies between J* and the Bellman iterate T^k V0.
                             MB-MPI: asynchronous evaluation sweeps, synchronous improvement.
                             Single-GPU; excludes RMB_CHUNKED_T and RMB_SELECT_*.                */
#define RMB_TRACE_ERROR_VS_REF 0x10000u /* rmb_vi / rmb_mpi / rmb_policy_value: also record the paper's plotted
                                          metric -- err[i] = ||V_i - V*||_inf
                                          after operator application i (VI sweeps, MPI evaluation sweeps),
                                          V* from rmb_set_reference; read with rmb_error_trace.  Computed
                                          on the device after each application (asynchronous applications
                                          add one grid barrier for it).  Single-GPU handles only.         */
/* A/B and test switches of rmb_create_* (performance choices only: results are bitwise the same) */
#define RMB_SPARSE_FULL_GRID 0x80u  /* sparse: 148-CTA grid even for tiny batches (default: 1 CTA)  */
#define RMB_SHARD_NO_GRAPH 0x400u   /* shard handles: launch each sweep's batch sequence eagerly
                                       instead of replaying it from a captured CUDA graph          */
#define RMB_FUSED 0x800u  /* rmb_vi / rmb_mpi (+ _group) on DENSE shard handles: the fused multi-GPU
                             path -- one persistent kernel per rank for the whole solve; each rank
                             stores its batch results straight into every rank's exchange arrays
                             (NVLink peer memory, CUDA IPC handles exchanged over the handle's NCCL
                             communicator) and the ranks meet at an in-kernel cross-rank barrier:
                             no host round trip or NCCL launch per batch.  Needs the TMA path
                             (16-byte aligned rows), <= 8 ranks; results bitwise those of the
                             single-GPU grid solver.
                             With rmb_*_group the G logical ranks share one launch on one device. */

/* Create a handle over a DENSE MDP.
 *   P: [n][A][n] row-major, P[(s*A + a)*n + j] = p(j | s, a), dtype desc->p_dtype.
 *   c: [n][A], c[s*A + a] = stage cost, same dtype.
 * Device pointers are BORROWED (must outlive the handle; never copied).
 * Host pointers are copied once into owned device memory, allocated
 * stream-ordered from the device's default memory pool; rmb_destroy returns
 * it to that pool, which keeps it reserved for the next handle (release
 * threshold raised on first use; cudaMemPoolTrimTo gives it back).
 * The library allocates its workspace here and in the first solve.
 * Errors: INVALID_ARG (sizes, gamma, dtype, NULL pointers), INVALID_MDP
 * (with RMB_VALIDATE), OOM, CUDA. */
rmb_status rmb_create_dense(const rmb_desc* desc, const void* P, const void* c, uint32_t flags,
                            rmb_problem* out);

/* Create a handle over a SPARSE MDP in CSR form over rows r = s*A + a.
 *   row_ptr: int64 [n*A + 1], row_ptr[0] = 0, nondecreasing;
 *   col:     int32 [nnz] successor state ids in [0, n);
 *   val:     [nnz] probabilities (p_dtype);  c: [n][A] costs (p_dtype).
 * A fixed-stride row_ptr (row_ptr[r] = r*K) is detected and served by the
 * ELL kernel.  Ownership and errors as rmb_create_dense. */
rmb_status rmb_create_csr(const rmb_desc* desc, const int64_t* row_ptr, const int32_t* col,
                          const void* val, const void* c, uint32_t flags, rmb_problem* out);

typedef struct {
    int64_t sweeps;        /* operator applications done (VI sweeps or MPI evaluation sweeps) */
    int64_t batches;       /* batches processed                                              */
    int64_t outer_iters;   /* MPI outer iterations (0 for VI)                                */
    double final_residual; /* VI: last r_k; MPI: last ||TV - V||_inf                         */
    double seconds;        /* device time of the solve (CUDA events)                         */
    int32_t converged;     /* 1 if the stopping test passed                                  */
    int32_t status;        /* the rmb_status returned                                        */
} rmb_stats;

/* MB-VI: V <- V0 (V's content, or 0 with RMB_V0_ZERO); for sweeps
 * k = 1, 2, ...: draw the partition of sweep k (seed, k), apply B_b, record
 * r_k = ||V_k - V_{k-1}||_inf; stop at the first r_k <= eps.
 *   flags: RMB_ORDER_IDENTITY, RMB_V0_ZERO, RMB_CHUNKED_T (VI*: T in chunks).
 *   b in [1, n]; eps > 0; max_sweeps >= 1.
 *   V: [n] float64 in/out.  pi: [n] int32 out (the argmin of each state's
 *   final-sweep backup).  trace: HOST [max_sweeps] or NULL (r_k, k = 1..).
 *   stats: HOST or NULL.
 * Returns OK, NOT_CONVERGED (outputs valid), NONFINITE, or an error. */
rmb_status rmb_vi(rmb_problem h, int64_t b, uint64_t seed, double eps, int64_t max_sweeps,
                  uint32_t flags, void* V, int32_t* pi, double* trace, rmb_stats* stats);

/* MB-MPI: Algorithm 1 with B_{pi,b} evaluation sweeps and warm
 * start.  pi_0 = greedy(V0) unless RMB_PI_GIVEN.  Each outer
 * iteration: m evaluation sweeps (each draws its own partition, sweep
 * counter k continues across outer iterations), then the improvement
 * pi' = argmin_a Q(s,a) over all states (no V write) with
 * changed = #{pi' != pi} and r_T = ||TV - V||_inf; stop when changed == 0
 * and r_T <= eps.
 *   trace: HOST [max_outer*(m+1)] or NULL: trace[o*(m+1)+e] = residual of
 *          evaluation sweep e of outer o, trace[o*(m+1)+m] = r_T.
 *   changed: HOST [max_outer] or NULL.
 * Returns as rmb_vi. */
rmb_status rmb_mpi(rmb_problem h, int64_t b, int32_t m, uint64_t seed, double eps, int64_t max_outer,
                   uint32_t flags, void* V, int32_t* pi, double* trace, int64_t* changed,
                   rmb_stats* stats);

/* One application of B_b (pi_or_null == NULL) or B_{pi,b} with the
 * partition of sweep number `sweep` (>= 1): V_out = B V_in.  V_in and V_out
 * may alias.  argmin_out ([n] int32, may be NULL) receives the argmin (or
 * pi).  resid_out (HOST, may be NULL) receives ||V_out - V_in||_inf.
 * pi_or_null entries outside [0, A) return RMB_ERR_INVALID_ARG (checked on
 * the device before the sweep).  flags: RMB_ORDER_IDENTITY, RMB_CHUNKED_T. */
rmb_status rmb_apply(rmb_problem h, int64_t b, uint64_t seed, int64_t sweep, uint32_t flags,
                     const int32_t* pi_or_null, const void* V_in, void* V_out, int32_t* argmin_out,
                     double* resid_out);

/* Policy evaluation: V <- B_{pi,b} V applied until ||V_k - V_{k-1}||_inf <= eps
 * (MPI's evaluation operator, Eq. 13, run to convergence; its fixed
 * point is J_pi, Eq. 4, Lemma 4; on return ||V - J_pi||_inf <=
 * gamma * r_K / (1 - gamma)).  pi: [n] int32 in.  V: [n] float64 in (V0, or 0
 * with RMB_V0_ZERO) / out.  trace: HOST [max_sweeps] or NULL.
 * Returns OK, NOT_CONVERGED (V valid), NONFINITE or an error. */
rmb_status rmb_policy_value(rmb_problem h, const int32_t* pi, int64_t b, uint64_t seed, double eps, int64_t max_sweeps,
                            uint32_t flags, void* V, double* trace, rmb_stats* stats);

/* Policy improvement of Algorithm 1 alone: pi <- greedy(V)
 * (lowest index on ties), *changed = #{states whose action changed},
 * *bellman_resid = ||TV - V||_inf.  pi: [n] int32 in/out.  Outputs HOST or NULL. */
rmb_status rmb_improve(rmb_problem h, const void* V, int32_t* pi, double* bellman_resid, int64_t* changed);

/* ------------------------------------------------------------------------
 * Multi-GPU: rows of P sharded by contiguous state ownership,
 * V replicated, one exchange of the batch's updated (state, value, argmin)
 * entries per batch (an all-gather).  The partition of every sweep is global,
 * so each batch is the same set of states on every rank, and every state's
 * backup is computed with the single-GPU grid solver's arithmetic: V, pi and
 * the residual trace are bitwise identical for any number of ranks (and to a
 * single handle created with RMB_DENSE_NO_CLUSTER; tiny batches on one GPU
 * otherwise run on the one-cluster path, equal to fp64 rounding).
 * A shard handle is created with desc.row_begin/row_end from rmb_shard_range
 * and P / c pointing at the owned rows only ([row_end-row_begin][A][n] and
 * [row_end-row_begin][A]) -- for rmb_create_csr: row_ptr [(row_end-row_begin)*A+1]
 * starting at 0, col holding GLOBAL successor ids, val/c the owned rows; V and
 * pi are full-length on every rank (pi entries outside the owned range are
 * unspecified on return).  Dense and sparse (CSR/ELL) MDPs; all ranks of one
 * solve use the same storage.
 * ------------------------------------------------------------------------ */

/* Owned rows of rank g of G: [begin, end) = [g*ceil(n/G), (g+1)*ceil(n/G)) ∩ [0,n). */
rmb_status rmb_shard_range(int64_t n, int32_t G, int32_t g, int64_t* begin, int64_t* end);

/* NCCL bootstrap: rank 0 draws a 128-byte unique id (HOST buffer), the
 * caller broadcasts it (e.g. over torch.distributed), every rank creates its
 * communicator (returned as an opaque ncclComm_t, stored in desc.nccl_comm).
 * NCCL is loaded at run time (the process's libnccl.so.2). */
rmb_status rmb_nccl_unique_id(void* id128);
rmb_status rmb_nccl_comm_init(int32_t nranks, int32_t rank, const void* id128, void** comm);
rmb_status rmb_nccl_comm_destroy(void* comm);

/* With desc.nccl_comm set, rmb_vi / rmb_mpi above run the sharded protocol;
 * they are collective: every rank calls with identical b, m, seed, eps,
 * limits and flags, and identical V0 (and pi0 with RMB_PI_GIVEN).
 *
 * Logical group on ONE device: G shard handles (rank order, rmb_shard_range
 * rows, same stream) run the same protocol with device-copy exchange; V and
 * pi (full, host or device) are shared in/out.  Used to test the sharded path
 * on one GPU; results equal the single-handle solve bit for bit. */
rmb_status rmb_vi_group(rmb_problem* handles, int32_t G, int64_t b, uint64_t seed, double eps, int64_t max_sweeps,
                        uint32_t flags, void* V, int32_t* pi, double* trace, rmb_stats* stats);
rmb_status rmb_mpi_group(rmb_problem* handles, int32_t G, int64_t b, int32_t m, uint64_t seed, double eps,
                         int64_t max_outer, uint32_t flags, void* V, int32_t* pi, double* trace, int64_t* changed,
                         rmb_stats* stats);

/* Host-side partition generator: perm[p] = pi_sweep(p),
 * the state processed at position p of operator application `sweep`;
 * batch t = positions [t*b, min(n,(t+1)*b)).  perm: HOST [n] uint32.
 * flags: RMB_ORDER_IDENTITY gives the identity. */
rmb_status rmb_partition(int64_t n, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* perm);

/* State selection with replacement (DESIGN R28-R29).
 * rmb_set_selection_weights: w = [n] uint32 weights >= 1 (HOST or DEVICE,
 * copied; NULL clears) for RMB_SELECT_WEIGHTED; a zero weight returns
 * INVALID_ARG (every state needs a positive probability for convergence).
 * rmb_select: HOST generator of application `sweep`'s n draws, sel [n] HOST
 * uint32 (w HOST or NULL = uniform).  rmb_select_device: the same draws from
 * the device kernel the solvers use (flags RMB_SELECT_REPLACE or
 * RMB_SELECT_WEIGHTED with the handle's weights), sel: DEVICE [n]. */
rmb_status rmb_set_selection_weights(rmb_problem h, const uint32_t* w);

/* Error-vs-reference tracing (RMB_TRACE_ERROR_VS_REF).  rmb_set_reference:
 * Vref = [n] float64 (HOST or DEVICE, copied; NULL clears) -- typically V*
 * from a tight solve or exact policy iteration.  rmb_error_trace: copies the
 * last solve's errors (HOST or DEVICE out, up to len) and sets *count (HOST,
 * may be NULL) to the number recorded (0 when the last solve did not trace). */
rmb_status rmb_set_reference(rmb_problem h, const void* Vref);
rmb_status rmb_error_trace(rmb_problem h, double* out, int64_t len, int64_t* count);
rmb_status rmb_select(int64_t n, uint64_t seed, int64_t sweep, const uint32_t* w, uint32_t* sel);
rmb_status rmb_select_device(rmb_problem h, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* sel);

/* The same permutation evaluated by the device kernel the solver uses
 * (perm: DEVICE [n] uint32) — exposed for parity tests. */
rmb_status rmb_partition_device(int64_t n, uint64_t seed, int64_t sweep, uint32_t flags, uint32_t* perm,
                                void* stream);

/* Synthetic instance generators (gen/rmb_gen.h), evaluated on device.
 * All output pointers are DEVICE pointers of the documented sizes.
 *   kind 0 = dense random, 1 = dense dyadic: P [n][A][n], c [n][A];
 *   rows [s0, s1) only (pass 0, n for the whole instance; P/c then hold
 *   (s1-s0) states).                                                      */
rmb_status rmb_generate_dense(int32_t kind, uint64_t seed, int64_t n, int32_t A, int64_t s0, int64_t s1,
                              rmb_dtype dtype, void* P, void* c, void* stream);
/* sparse random, K successors per (s,a): row_ptr [(s1-s0)*A+1], col/val [(s1-s0)*A*K], c [(s1-s0)*A] */
rmb_status rmb_generate_sparse(uint64_t seed, int64_t n, int32_t A, int32_t K, int64_t s0, int64_t s1,
                               rmb_dtype dtype, int64_t* row_ptr, int32_t* col, void* val, void* c,
                               void* stream);
/* N x N slip gridworld, A = 4, ELL width 5: row_ptr [(s1-s0)*4+1], col/val [(s1-s0)*20], c [(s1-s0)*4] */
rmb_status rmb_generate_grid(int64_t N, int64_t s0, int64_t s1, rmb_dtype dtype, int64_t* row_ptr,
                             int32_t* col, void* val, void* c, void* stream);

/* Kernel launches issued by the last solve/apply/improve call on this handle
 * (evidence for bench.py's gpu_launches). */
int64_t rmb_last_launch_count(rmb_problem h);

/* Sharded solves: sweeps of the last solve replayed from a captured CUDA graph
 * (0 when every sweep was launched eagerly). */
int64_t rmb_last_graph_launches(rmb_problem h);

/* Phase breakdown of the last solve as seen by CTA 0 of the persistent
 * kernel (globaltimer): ns4[0] compute (streaming P), ns4[1] waiting in grid
 * barriers, ns4[2] combine/patch, ns4[3] number of grid barriers.
 * ns4: HOST [4] int64. */
rmb_status rmb_last_phase_times(rmb_problem h, int64_t* ns4);

/* Destroy the handle and free its workspace (borrowed buffers untouched). */
rmb_status rmb_destroy(rmb_problem h);

const char* rmb_status_string(rmb_status s);
const char* rmb_last_error(void);   /* thread-local, "" if none */
const char* rmb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RMB_H */

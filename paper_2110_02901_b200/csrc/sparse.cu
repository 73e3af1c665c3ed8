// sparse.cu — persistent sm_100a solver for SPARSE MDPs (CSR over rows
// r = s*A + a; fixed-stride rows are served as ELL).
//
// One cooperative launch runs a whole MB-VI / MB-MPI solve (Alg. 1).
// V does not fit in shared memory (config 3: 8 MB, config 4: 33.5 MB), so the
// interim vector lives in L2-resident global memory, ping-ponged by batch:
//
//   invariant: at the start of (global) batch g, X[g & 1] is the interim V.
//   batch g reads successors from X_cur = X[g & 1] (one 8-byte gather per
//   nonzero, no select), writes its states' new values into X_next, and also
//   re-copies the previous batch's states X_cur -> X_next, so that X_next is
//   the interim V of batch g+1 after the single grid barrier.
//
// This realises Eq. 12 exactly: every read of batch g sees the
// values of earlier batches (they are in X_cur) and the previous sweep's
// values of every other state, including same-batch states.
//
// Per state, a lane group does the backup:
//   row mode (ELL width K <= 8, A <= 32): lane a sums row (s, a) sequentially,
//     then an argmin butterfly over the group (ties -> lower action);
//   strided mode (wide or ragged rows): the group's lanes stride over each
//     row's nonzeros, butterfly sum, actions in order (strict < keeps the
//     lowest index).
// The residual and nonfinite flag are reduced per CTA and combined with one
// atomicMax / atomicOr per CTA before the sweep's last barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "partition.cuh"

namespace rmb {

constexpr int64_t kSparseSmallBatchNnz = 2048;  // nonzeros per batch up to which a solve runs on one CTA


// CTA size per layout: row mode (a lane per action row, short rows, many
// dependent gathers) wants the warps; vec / strided fit 512 threads without spills
constexpr int kSWarpsMax = 32;
template <int MODE>
struct SThreads {
    static constexpr int v = 512;  // 1024 for row mode: config-4 VI 1.5x faster, config-4 MPI 1.7x slower
};
// Two register budgets per layout: MINB = 1 (one 512-thread CTA per SM, no
// spills) and MINB = 2 (64 registers, two CTAs per SM: twice the gathers in
// flight, a few spills off the hot loop, a grid barrier over 2x the CTAs).
// Measured on B200 (tools/sparse_perf.py): MINB = 2 wins for B_b sweeps with
// large batches (config 3 b = n/8: 1.53 -> 1.41 ms per sweep; config 4 VI
// b = n: 0.60 -> 0.38 ms) and loses for small batches (barrier cost) and
// MPI (config 4: 8.9 -> 12.7 s), so it is chosen per solve (sparse_solve).
constexpr int64_t kSparseWideNnz = int64_t(1) << 24;  // nonzeros per batch from which MINB = 2 pays

struct SparseArgs {
    const int64_t* row_ptr;
    const int32_t* col;
    const void* val;
    const void* c;
    int64_t n;
    int A;
    int K;  // > 0: ELL width
    int GS; // lanes per state in min modes (power of two <= 32)
    int GSE;  // lanes per state in B_{pi,b} sweeps
    double gamma;
    double* V;
    int32_t* pi;
    double* X0;
    double* X1;
    int32_t* pw0;  // MPI policy ping-pong
    int32_t* pw1;
    int64_t b;
    uint64_t seed;
    int64_t k0;
    int identity;
    int mode;
    int pi_given;
    double eps;
    int64_t max_iter;
    int msweeps;
    int chunked;     // RMB_CHUNKED_T (VI*): every batch reads the sweep-start values
    uint32_t* perm;  // 3 * n
    unsigned long long* bar;
    int* err;
    unsigned long long* red;  // [4] residual bits ring, [4..8) nonfinite ring, [8..12) changed ring
    double* trace;
    int64_t trace_len;
    long long* chg;
    int64_t chg_len;
    long long* out;
    long long* prof;
};

template <typename PT>
__device__ __forceinline__ double ldv(const void* p, int64_t e)
{
    return (double)__ldg(static_cast<const PT*>(p) + e);
}

// Layout modes of the sparse backup (chosen on the host from the CSR shape).
enum SMode : int {
    SM_STRIDED = 0,  // general CSR: group lanes stride over each row, actions in turn
    SM_ROW = 1,      // ELL, K <= 8: a lane per action row (bit-exact with the oracle)
    SM_VEC = 2,      // ELL, K % 8 == 0, A*K/8 a power of two <= 32: 8 consecutive nonzeros per lane
};

__device__ __forceinline__ int4 ld_nc_int4(const int32_t* p)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <typename PT>
__device__ __forceinline__ void ld8(const void* val, int64_t e, double (&v)[8])
{
    if constexpr (sizeof(PT) == 4) {
        const float4 a = ld_stream(reinterpret_cast<const float4*>(static_cast<const float*>(val) + e));
        const float4 b = ld_stream(reinterpret_cast<const float4*>(static_cast<const float*>(val) + e + 4));
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
    } else {
        const double* d = static_cast<const double*>(val) + e;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 x = ld_stream(reinterpret_cast<const double2*>(d + 2 * q));
            v[2 * q] = x.x, v[2 * q + 1] = x.y;
        }
    }
}

// (lower value, then lower action) butterfly over lane offsets [o_lo, GS)
__device__ __forceinline__ void argmin_butterfly(double& Q, int& arg, int o_lo, int GS)
{
    for (int o = GS >> 1; o >= o_lo && o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, Q, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        // lane order == action order, so (lower value, then lower index)
        // reproduces "first strict minimum"; a NaN in the lowest action stays
        // (as in the oracle, where a NaN Q_0 is never replaced)
        if (ov < Q || (ov == Q && oa < arg) || (arg == 0x7fffffff && oa != 0x7fffffff)) {
            Q = ov;
            arg = oa;
        }
    }
}

// Backup of state s against X by a group of GS lanes (g = lane in group).
// act_fixed >= 0: B_{pi,b} row only.  Result valid in lane g == 0 (all modes)
// and in every lane for SM_ROW / SM_VEC min.
template <typename PT, int MODE>
__device__ __forceinline__ void backup_state(const SparseArgs& a, const double* X, int64_t s, int act_fixed, int g,
                                             int GS, bool valid, double& best, int& barg)
{
    if (MODE == SM_ROW) {
        double Q = INFINITY;
        int arg = 0x7fffffff;
        const int act = !valid ? -1 : act_fixed >= 0 ? (g == 0 ? act_fixed : -1) : (g < a.A ? g : -1);
        if (act >= 0) {
            const int64_t row = s * a.A + act;
            const int64_t e0 = a.K > 0 ? row * a.K : __ldg(a.row_ptr + row);
            const int64_t e1 = a.K > 0 ? e0 + a.K : __ldg(a.row_ptr + row + 1);
            // one lane, storage order, separately rounded products and sums
            // (no FMA contraction): the same arithmetic as the oracle's row
            // sum, so row mode is bit-exact and exact Q ties (symmetric grids)
            // break identically on both sides
            double acc = 0.0;
            for (int64_t e = e0; e < e1; ++e)
                acc = __dadd_rn(acc, __dmul_rn(ldv<PT>(a.val, e), __ldcg(X + __ldg(a.col + e))));
            Q = __dadd_rn(ldv<PT>(a.c, row), __dmul_rn(a.gamma, acc));
            arg = act;
        }
        argmin_butterfly(Q, arg, 1, GS);
        best = Q;
        barg = arg;
        return;
    }
    if (MODE == SM_VEC) {
        // lane g owns nonzeros [8g, 8g+8) of the state's block (min) or of the
        // row pi(s) (eval): 2x128-bit col + 2x128-bit val loads, 8 gathers in
        // flight, a sequential 8-term sum, then a butterfly over the K/8 lanes
        // of the action and an argmin butterfly over the actions
        const int L = a.K >> 3;  // lanes per action row
        double Q = INFINITY;
        int arg = 0x7fffffff;
        if (valid) {
            const int act = act_fixed >= 0 ? act_fixed : (8 * g) / a.K;
            const int64_t e = act_fixed >= 0 ? (s * a.A + act_fixed) * a.K + 8 * g : s * a.A * a.K + 8 * g;
            const int4 c0 = ld_nc_int4(a.col + e);
            const int4 c1 = ld_nc_int4(a.col + e + 4);
            double v[8];
            ld8<PT>(a.val, e, v);
            const double x0 = __ldcg(X + c0.x), x1 = __ldcg(X + c0.y), x2 = __ldcg(X + c0.z), x3 = __ldcg(X + c0.w);
            const double x4 = __ldcg(X + c1.x), x5 = __ldcg(X + c1.y), x6 = __ldcg(X + c1.z), x7 = __ldcg(X + c1.w);
            double acc = v[0] * x0;
            acc = fma(v[1], x1, acc);
            acc = fma(v[2], x2, acc);
            acc = fma(v[3], x3, acc);
            acc = fma(v[4], x4, acc);
            acc = fma(v[5], x5, acc);
            acc = fma(v[6], x6, acc);
            acc = fma(v[7], x7, acc);
            Q = acc;
            arg = act;
        }
        for (int o = 1; o < L; o <<= 1) Q += __shfl_xor_sync(0xffffffffu, Q, o);
        if (valid) Q = ldv<PT>(a.c, s * a.A + arg) + a.gamma * Q;
        if (act_fixed < 0) argmin_butterfly(Q, arg, L, GS);
        best = Q;
        barg = arg;
        return;
    }
    const int a_lo = act_fixed >= 0 ? act_fixed : 0;
    const int a_hi = act_fixed >= 0 ? act_fixed + 1 : a.A;
    best = 0.0;
    barg = a_lo;
    for (int act = a_lo; act < a_hi; ++act) {
        const int64_t row = s * a.A + act;
        const int64_t e0 = !valid ? 0 : a.K > 0 ? row * a.K : __ldg(a.row_ptr + row);
        const int64_t e1 = !valid ? 0 : a.K > 0 ? e0 + a.K : __ldg(a.row_ptr + row + 1);
        double acc = 0.0;
        for (int64_t e = e0 + g; e < e1; e += GS) acc = fma(ldv<PT>(a.val, e), __ldcg(X + __ldg(a.col + e)), acc);
        for (int o = GS >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double Q = valid ? ldv<PT>(a.c, row) + a.gamma * acc : 0.0;
        if (act == a_lo || Q < best) best = Q, barg = act;
    }
}

struct SCtx {
    GridBarrier g;
    int64_t gb;  // global batch counter (X parity)
    int64_t batches;
    // previous batch (for the X_cur -> X_next re-copy)
    const uint32_t* prev_perm;
    int64_t prev_lo, prev_cnt;
    bool prev_valid;
    unsigned long long t_mark;
    long long t_comp, t_bar, n_bar;
};

__device__ __forceinline__ void s_prof(SCtx& x, long long* slot)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long t = globaltimer_ns();
        *slot += (long long)(t - x.t_mark);
        x.t_mark = t;
    }
}

// CTA reduction (max, or, sum) then one global atomic per CTA.
__device__ void cta_publish(const SparseArgs& a, int slot, double rmax, int bad, long long changed)
{
    __shared__ double sd[kSWarpsMax];
    __shared__ int si[kSWarpsMax];
    __shared__ long long sl[kSWarpsMax];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        changed += __shfl_xor_sync(0xffffffffu, changed, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sd[w] = rmax, si[w] = bad, sl[w] = changed;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        int bb = 0;
        long long cc = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, sd[k]), bb |= si[k], cc += sl[k];
        atomicMax(a.red + slot, (unsigned long long)__double_as_longlong(r));
        if (bb) atomicOr(reinterpret_cast<unsigned int*>(a.red + 4 + slot), 1u);
        if (cc) atomicAdd(a.red + 8 + slot, (unsigned long long)cc);
    }
}

struct SweepResult {
    double r;
    int bad;
    long long changed;
};

__device__ __forceinline__ SweepResult read_slot(const SparseArgs& a, int slot)
{
    SweepResult s;
    s.r = __longlong_as_double((long long)ld_acquire_gpu(a.red + slot));
    s.bad = ld_acquire_gpu(a.red + 4 + slot) != 0;
    s.changed = (long long)ld_acquire_gpu(a.red + 8 + slot);
    return s;
}

// One application of B_b (EVAL false) or B_{pi,b} (EVAL true), sweep k.
template <typename PT, int MODE, bool EVAL>
__device__ SweepResult run_sweep(const SparseArgs& a, SCtx& x, int64_t k, const int32_t* pol)
{
    const uint32_t* perm = a.identity ? nullptr : a.perm + (k % 3) * a.n;
    const int GS = EVAL ? a.GSE : a.GS;
    const int g = threadIdx.x & (GS - 1);
    // warp-uniform trip counts: all 32 lanes stay in the loop for the shuffles
    const int64_t ngroups = (int64_t)gridDim.x * ((int)blockDim.x / GS);
    const int64_t gid = (int64_t)blockIdx.x * ((int)blockDim.x / GS) + threadIdx.x / GS;
    const int64_t wfirst = gid - (threadIdx.x & 31) / GS;  // first group of this warp
    const int slot = (int)(k & 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // rearm the ring slot used two sweeps ahead
        const int z = (int)((k + 2) & 3);
        atomicExch(a.red + z, 0ull);
        atomicExch(a.red + 4 + z, 0ull);
        atomicExch(a.red + 8 + z, 0ull);
    }
    const bool single = a.b >= a.n;  // one batch per sweep: every state rewritten each batch
    // chunked T (VI*): every chunk reads X_cur = the sweep-start
    // values and writes X_next; no re-copies, X flips once per sweep
    const bool chunked = !EVAL && a.chunked && !single;
    double rmax = 0.0;
    int bad = 0;
    for (int64_t lo = 0; lo < a.n; lo += a.b) {
        const int64_t cnt = min(a.b, a.n - lo);
        const double* Xc = (x.gb & 1) ? a.X1 : a.X0;
        double* Xn = (x.gb & 1) ? a.X0 : a.X1;
        // states in processing order; a single batch is order-free, so walk it
        // in state order (coalesced rows)
        const uint32_t* bperm = single ? nullptr : perm;
        for (int64_t w0 = wfirst; w0 < cnt; w0 += ngroups) {
            const int64_t i = w0 + (gid - wfirst);
            const bool valid = i < cnt;
            const int64_t s = !valid ? 0 : bperm ? (int64_t)__ldg(bperm + lo + i) : lo + i;
            double v;
            int arg;
            backup_state<PT, MODE>(a, Xc, s, EVAL && valid ? pol[s] : (EVAL ? 0 : -1), g, GS, valid, v, arg);
            if (valid && g == 0) {
                const double old = __ldcg(Xc + s);
                rmax = fmax(rmax, fabs(v - old));
                bad |= !isfinite(v);
                Xn[s] = v;
                if (!EVAL && a.pi) a.pi[s] = arg;
            }
        }
        // carry the previous batch's new values into X_next.  In the first
        // batch of a sweep the previous batch belongs to the previous sweep and
        // may share states with this batch: those get this batch's new value,
        // so their copy is skipped (membership through the inverse permutation).
        if (x.prev_valid && !single) {
            Permutation pk;
            if (lo == 0 && !a.identity) pk.init(a.n, a.seed, k);
            const int64_t stride = (int64_t)gridDim.x * blockDim.x;
            for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < x.prev_cnt; i += stride) {
                const int64_t s = x.prev_perm ? (int64_t)x.prev_perm[x.prev_lo + i] : x.prev_lo + i;
                if (lo == 0) {
                    const int64_t pos = a.identity ? s : (int64_t)pk.position((uint64_t)s);
                    if (pos < cnt) continue;
                }
                Xn[s] = __ldcg(Xc + s);
            }
        }
        if (lo == 0 && !a.identity) {  // next sweep's order, off the critical path
            Permutation pm;
            pm.init(a.n, a.seed, k + 1);
            uint32_t* dst = a.perm + ((k + 1) % 3) * a.n;
            const int64_t stride = (int64_t)gridDim.x * blockDim.x;
            for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.n; p += stride)
                dst[p] = (uint32_t)pm((uint64_t)p);
        }
        const bool last = lo + a.b >= a.n;
        if (last) cta_publish(a, slot, rmax, bad, 0);
        s_prof(x, &x.t_comp);
        grid_sync(x.g);
        s_prof(x, &x.t_bar);
        x.n_bar++;
        x.prev_perm = single ? nullptr : perm;
        x.prev_lo = lo;
        x.prev_cnt = cnt;
        x.prev_valid = !single && !chunked;
        if (!chunked) ++x.gb;
        ++x.batches;
    }
    if (chunked) ++x.gb;
    return read_slot(a, slot);
}

// Policy improvement over all states against X_cur (no X write):
// pw_next = greedy, changed vs pw_cur, ||TV - V||_inf.
template <typename PT, int MODE>
__device__ SweepResult run_improve(const SparseArgs& a, SCtx& x, int64_t imp_idx, const int32_t* pcur, int32_t* pnext,
                                   bool count_changed)
{
    const int GS = a.GS;
    const int g = threadIdx.x & (GS - 1);
    const int64_t ngroups = (int64_t)gridDim.x * ((int)blockDim.x / GS);
    const int64_t gid = (int64_t)blockIdx.x * ((int)blockDim.x / GS) + threadIdx.x / GS;
    const int64_t wfirst = gid - (threadIdx.x & 31) / GS;
    // improvement steps use their own ring (slots 2,3 parity of imp_idx) via the
    // same red[] words offset by 16
    const SparseArgs* ap = &a;
    const double* Xc = (x.gb & 1) ? a.X1 : a.X0;
    double rmax = 0.0;
    int bad = 0;
    long long changed = 0;
    for (int64_t w0 = wfirst; w0 < a.n; w0 += ngroups) {
        const int64_t s = w0 + (gid - wfirst);
        const bool valid = s < a.n;
        double v;
        int arg;
        backup_state<PT, MODE>(a, Xc, valid ? s : 0, -1, g, GS, valid, v, arg);
        if (valid && g == 0) {
            rmax = fmax(rmax, fabs(v - __ldcg(Xc + s)));
            bad |= !isfinite(v);
            if (count_changed) changed += (arg != pcur[s]);
            pnext[s] = arg;
        }
    }
    // improvement ring: red[16 + 4*q .. ] with q = imp_idx & 1 (rearmed for q^1)
    unsigned long long* base = a.red + 16 + 4 * (imp_idx & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long* other = a.red + 16 + 4 * ((imp_idx + 1) & 1);
        atomicExch(other, 0ull);
        atomicExch(other + 1, 0ull);
        atomicExch(other + 2, 0ull);
    }
    {
        __shared__ double sd[kSWarpsMax];
        __shared__ int si[kSWarpsMax];
        __shared__ long long sl[kSWarpsMax];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
            changed += __shfl_xor_sync(0xffffffffu, changed, o);
        }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) sd[w] = rmax, si[w] = bad, sl[w] = changed;
        __syncthreads();
        if (threadIdx.x == 0) {
            double r = 0.0;
            int bb = 0;
            long long cc = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, sd[k]), bb |= si[k], cc += sl[k];
            atomicMax(base, (unsigned long long)__double_as_longlong(r));
            if (bb) atomicOr(base + 1, 1ull);
            if (cc) atomicAdd(base + 2, (unsigned long long)cc);
        }
    }
    (void)ap;
    s_prof(x, &x.t_comp);
    grid_sync(x.g);
    s_prof(x, &x.t_bar);
    x.n_bar++;
    SweepResult r;
    r.r = __longlong_as_double((long long)ld_acquire_gpu(base));
    r.bad = ld_acquire_gpu(base + 1) != 0;
    r.changed = (long long)ld_acquire_gpu(base + 2);
    return r;
}

template <typename PT, int MODE, int MINB>
__global__ void __launch_bounds__(SThreads<MODE>::v, MINB) sparse_solver_kernel(const SparseArgs a)
{
    SCtx x{};
    x.g = GridBarrier{a.bar, a.bar + 32, 0ull, (unsigned long long)gridDim.x, a.err};
    if (blockIdx.x == 0 && threadIdx.x == 0) x.t_mark = globaltimer_ns();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t s = tid; s < a.n; s += stride) {
        const double v = a.V[s];
        a.X0[s] = v;
        a.X1[s] = v;
        if (a.mode == MODE_MPI || a.mode == MODE_APPLY_PI || a.mode == MODE_IMPROVE || a.mode == MODE_POLICY_VALUE)
            a.pw0[s] = a.pi[s];
    }
    if (!a.identity && a.mode != MODE_IMPROVE) {
        Permutation pm;
        pm.init(a.n, a.seed, a.k0);
        uint32_t* dst = a.perm + (a.k0 % 3) * a.n;
        for (int64_t p = tid; p < a.n; p += stride) dst[p] = (uint32_t)pm((uint64_t)p);
    }
    grid_sync(x.g);

    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    long long status = RMB_ERR_NOT_CONVERGED;
    int64_t k = a.k0, it = 0, outer = 0, imp = 0;
    long long changed = 0;
    double last = 0.0;
    int pcur = 0;  // which pw buffer holds the current policy
    if (a.mode == MODE_VI || a.mode == MODE_APPLY || a.mode == MODE_APPLY_PI ||
               a.mode == MODE_POLICY_VALUE) {
        const bool eval = a.mode == MODE_APPLY_PI || a.mode == MODE_POLICY_VALUE;
        const int64_t iters = (a.mode == MODE_VI || a.mode == MODE_POLICY_VALUE) ? a.max_iter : 1;
        while (it < iters) {
            SweepResult r = eval ? run_sweep<PT, MODE, true>(a, x, k, a.pw0)
                                                    : run_sweep<PT, MODE, false>(a, x, k, nullptr);
            if (lead && it < a.trace_len) a.trace[it] = r.r;
            ++it;
            ++k;
            last = r.r;
            if (r.bad) { status = RMB_ERR_NONFINITE; break; }
            if (a.eps >= 0.0 && r.r <= a.eps) { status = RMB_OK; break; }
        }
        if ((a.mode == MODE_APPLY || a.mode == MODE_APPLY_PI) && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
    } else if (a.mode == MODE_IMPROVE) {
        SweepResult r = run_improve<PT, MODE>(a, x, imp++, a.pw0, a.pw1, true);
        pcur = 1;
        last = r.r;
        changed = r.changed;
        status = r.bad ? RMB_ERR_NONFINITE : RMB_OK;
    } else {  // MODE_MPI
        bool bad = false;
        if (!a.pi_given) {
            SweepResult r = run_improve<PT, MODE>(a, x, imp++, a.pw0, a.pw1, false);
            pcur = 1;
            bad = r.bad;
        }
        while (!bad && outer < a.max_iter) {
            const int64_t row = outer * (a.msweeps + 1);
            const int32_t* pol = pcur ? a.pw1 : a.pw0;
            for (int e = 0; e < a.msweeps && !bad; ++e) {
                SweepResult r = run_sweep<PT, MODE, true>(a, x, k, pol);
                if (lead && row + e < a.trace_len) a.trace[row + e] = r.r;
                ++k;
                ++it;
                bad = r.bad;
            }
            if (bad) { ++outer; break; }
            SweepResult r = run_improve<PT, MODE>(a, x, imp++, pol, pcur ? a.pw0 : a.pw1, true);
            pcur ^= 1;
            if (lead && row + a.msweeps < a.trace_len) a.trace[row + a.msweeps] = r.r;
            if (lead && outer < a.chg_len) a.chg[outer] = r.changed;
            ++outer;
            last = r.r;
            changed = r.changed;
            if (r.bad) { bad = true; break; }
            if (r.changed == 0 && r.r <= a.eps) { status = RMB_OK; break; }
        }
        if (bad) status = RMB_ERR_NONFINITE;
    }
    // outputs: the interim vector after the last batch, and the policy
    const double* Xf = (x.gb & 1) ? a.X1 : a.X0;
    const int32_t* pf = pcur ? a.pw1 : a.pw0;
    const bool write_pi_buf = a.mode == MODE_MPI || a.mode == MODE_IMPROVE;
    for (int64_t s = tid; s < a.n; s += stride) {
        if (a.mode != MODE_IMPROVE) a.V[s] = Xf[s];
        if (write_pi_buf) a.pi[s] = pf[s];
    }
    if (lead) {
        a.out[OUT_SWEEPS] = it;
        a.out[OUT_OUTER] = outer;
        a.out[OUT_STATUS] = status;
        a.out[OUT_RESID_BITS] = __double_as_longlong(last);
        a.out[OUT_BATCHES] = x.batches;
        a.out[OUT_CHANGED] = changed;
        a.prof[0] = x.t_comp;
        a.prof[1] = x.t_bar;
        a.prof[2] = 0;
        a.prof[3] = x.n_bar;
    }
}

template <typename PT, int MODE, int MINB>
static cudaError_t launch_sparse_minb(const SparseArgs& a, int grid, cudaStream_t st)
{
    auto kern = sparse_solver_kernel<PT, MODE, MINB>;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SThreads<MODE>::v, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
    if (grid > 1) grid *= std::min(per_sm, MINB);
    void* args[] = {const_cast<SparseArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(SThreads<MODE>::v), args, 0, st);
}

template <typename PT, int MODE>
static cudaError_t launch_sparse(const SparseArgs& a, int grid, bool wide, cudaStream_t st)
{
    return wide ? launch_sparse_minb<PT, MODE, 2>(a, grid, st) : launch_sparse_minb<PT, MODE, 1>(a, grid, st);
}

// Layout of the sparse backup (mode, lanes per state) chosen from the CSR
// shape; shared by the persistent solver and the shard step so that a state's
// arithmetic is the same on one GPU and on G.
static void sparse_layout(const Problem& pr, int& mode, int& GS, int& GSE)
{
    // shape of the whole problem: this handle's own rows on one GPU, the
    // agreed global shape on a shard (shard.cu layout consensus)
    const int64_t rows = pr.g_set ? pr.g_rows : (pr.row_end - pr.row_begin) * (int64_t)pr.A;
    const int64_t nnz = pr.g_set ? pr.g_nnz : pr.nnz;
    const int ellK = pr.g_set ? pr.g_ell_K : pr.ell_K;
    const double avg = rows > 0 ? (double)nnz / (double)rows : 1.0;
    const int64_t AK = (int64_t)pr.A * ellK;
    const bool aligned = ((uintptr_t)pr.col % 16 == 0) && ((uintptr_t)pr.val % 16 == 0) && (!pr.g_set || pr.g_aligned);
    mode = SM_STRIDED;
    GS = 1, GSE = 1;
    if (ellK > 0 && ellK % 8 == 0 && aligned && AK / 8 <= 32 && ((AK / 8) & (AK / 8 - 1)) == 0 &&
        ((ellK / 8) & (ellK / 8 - 1)) == 0) {
        mode = SM_VEC;
        GS = (int)(AK / 8);
        GSE = ellK / 8;
    } else if (ellK > 0 && ellK <= 8 && pr.A <= 32) {
        mode = SM_ROW;
        while (GS < pr.A) GS <<= 1;
        GSE = 1;  // B_{pi,b}: one row per state -> a lane per state
    } else {
        while (GS < 32 && GS < avg) GS <<= 1;
        GSE = GS;
    }
}

rmb_status sparse_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                        long long* chg_dev, int64_t chg_len, SolveResult* res)
{
    const int64_t n = pr.n;
    SparseArgs a{};
    a.row_ptr = pr.row_ptr;
    a.col = pr.col;
    a.val = pr.val;
    a.c = pr.c;
    a.n = n;
    a.A = pr.A;
    a.K = pr.ell_K;
    a.gamma = pr.gamma;
    a.V = rq.V;
    a.pi = rq.pi;
    a.b = rq.b;
    a.seed = rq.seed;
    a.k0 = rq.k0;
    a.identity = rq.identity ? 1 : 0;
    a.mode = rq.mode;
    a.pi_given = rq.pi_given ? 1 : 0;
    a.eps = rq.eps;
    a.max_iter = rq.max_iter;
    a.msweeps = rq.msweeps;
    a.chunked = rq.chunked ? 1 : 0;
    int mode, GS, GSE;
    sparse_layout(pr, mode, GS, GSE);
    a.GS = GS;
    a.GSE = GSE;

    cudaStream_t st = pr.stream;
    if (pr.perm.ensure((size_t)3 * n * 4) != cudaSuccess || pr.part.ensure((size_t)2 * n * 8 + (size_t)2 * n * 4 + 256) != cudaSuccess ||
        pr.ctrl.ensure(4096) != cudaSuccess) {
        set_error("sparse solver: workspace allocation failed");
        return RMB_ERR_OOM;
    }
    a.perm = static_cast<uint32_t*>(pr.perm.p);
    a.X0 = static_cast<double*>(pr.part.p);
    a.X1 = a.X0 + n;
    a.pw0 = reinterpret_cast<int32_t*>(a.X1 + n);
    a.pw1 = a.pw0 + n;
    unsigned long long* ctrl = static_cast<unsigned long long*>(pr.ctrl.p);
    a.bar = ctrl;
    a.err = reinterpret_cast<int*>(ctrl + 64);
    a.out = reinterpret_cast<long long*>(ctrl + 128);
    a.prof = reinterpret_cast<long long*>(ctrl + 192);
    a.red = ctrl + 256;  // [256 .. 280)
    a.trace = trace_dev;
    a.trace_len = trace_len;
    a.chg = chg_dev;
    a.chg_len = chg_len;

    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaMemsetAsync(ctrl, 0, 4096, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(e0, st);
    // tiny batches (<= 2048 nonzeros, e.g. GS-VI on the paper's environments)
    // are latency-bound: one CTA with CTA barriers beats a 148-CTA grid
    // barrier per batch (measured: FrozenLake b=1 96 vs 125 ms, maze80 b=1
    // 5.96 vs 7.35 s; from ~10^4 nonzeros per batch the full grid wins)
    const int64_t nnz_batch = (int64_t)((double)std::min<int64_t>(rq.b, n) * (double)pr.nnz / (double)std::max<int64_t>(1, n));
    int grid = nnz_batch <= kSparseSmallBatchNnz && !pr.sparse_full_grid ? 1 : pr.num_sms;
    // two CTAs per SM for B_b sweeps over large batches (see kSparseWideNnz)
    bool wide = grid > 1 && (rq.mode == MODE_VI || rq.mode == MODE_APPLY) && nnz_batch >= kSparseWideNnz;
    if (pr.sparse_wide >= 0) wide = grid > 1 && pr.sparse_wide == 1;
    if (ce == cudaSuccess) {
        if (pr.pdt == RMB_F32)
            ce = mode == SM_VEC   ? launch_sparse<float, SM_VEC>(a, grid, wide, st)
                 : mode == SM_ROW ? launch_sparse<float, SM_ROW>(a, grid, wide, st)
                                  : launch_sparse<float, SM_STRIDED>(a, grid, wide, st);
        else
            ce = mode == SM_VEC   ? launch_sparse<double, SM_VEC>(a, grid, wide, st)
                 : mode == SM_ROW ? launch_sparse<double, SM_ROW>(a, grid, wide, st)
                                  : launch_sparse<double, SM_STRIDED>(a, grid, wide, st);
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(e1, st);
    long long out[OUT_N + 4] = {0};
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, a.out, sizeof(long long) * OUT_N, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out + OUT_N, a.prof, sizeof(long long) * 4, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    float ms = 0.f;
    if (ce == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) {
        set_error(std::string("sparse solver: ") + cudaGetErrorString(ce));
        return RMB_ERR_CUDA;
    }
    res->sweeps = out[OUT_SWEEPS];
    res->outer = out[OUT_OUTER];
    res->status = (int)out[OUT_STATUS];
    double d;
    memcpy(&d, &out[OUT_RESID_BITS], 8);
    res->final_resid = d;
    res->batches = out[OUT_BATCHES];
    res->changed = out[OUT_CHANGED];
    res->ms = ms;
    res->launches = 1;
    for (int i = 0; i < 4; ++i) pr.prof[i] = out[OUT_N + i];
    pr.last_launches = 1;
    return RMB_OK;
}

// ------------------------------------------------------------ shard step
// One launch of the multi-GPU protocol (shard.cu) on a sparse
// shard handle: CSR/ELL rows of the owned states [row0, row0+nloc) with
// global successor ids, backed up against this rank's replica Vr of the
// interim V (Eq. 12: the replica holds every earlier batch's
// committed values).  MIN / EVAL: the states of olist[0..*ocount) -> send
// record (value, state, argmin).  IMPROVE: greedy over the owned states,
// ||TV - V|| and #changed into out[] (pi updated in place, owned entries).
// Per-state arithmetic is backup_state<PT, MODE>, the single-GPU one.
template <typename PT, int MODE, int SMODE>
__global__ void __launch_bounds__(256) sparse_shard_kernel(SparseArgs a, int64_t row0, int64_t nloc, const double* Vr,
                                                           int32_t* pir, const uint32_t* olist, const int* ocount,
                                                           double* send_val, uint32_t* send_idx, int32_t* send_arg,
                                                           long long* out)
{
    constexpr bool EVAL = SMODE == MODE_SHARD_EVAL;
    const int GS = EVAL ? a.GSE : a.GS;
    const int g = threadIdx.x & (GS - 1);
    const int64_t ngroups = (int64_t)gridDim.x * ((int)blockDim.x / GS);
    const int64_t gid = (int64_t)blockIdx.x * ((int)blockDim.x / GS) + threadIdx.x / GS;
    const int64_t wfirst = gid - (threadIdx.x & 31) / GS;
    const int64_t cnt = SMODE == MODE_SHARD_IMPROVE ? nloc : (int64_t)*ocount;
    double rmax = 0.0;
    int bad = 0;
    long long changed = 0;
    for (int64_t w0 = wfirst; w0 < cnt; w0 += ngroups) {
        const int64_t i = w0 + (gid - wfirst);
        const bool valid = i < cnt;
        const int64_t s = !valid ? row0 : SMODE == MODE_SHARD_IMPROVE ? row0 + i : (int64_t)olist[i];
        double v;
        int arg;
        backup_state<PT, MODE>(a, Vr, s - row0, EVAL && valid ? pir[s] : (EVAL ? 0 : -1), g, GS, valid, v, arg);
        if (valid && g == 0) {
            if (SMODE == MODE_SHARD_IMPROVE) {
                rmax = fmax(rmax, fabs(v - Vr[s]));
                bad |= !isfinite(v);
                changed += (arg != pir[s]);
                pir[s] = arg;
            } else {
                send_val[i] = v;
                send_idx[i] = (uint32_t)s;
                send_arg[i] = EVAL ? pir[s] : arg;
            }
        }
    }
    if (SMODE != MODE_SHARD_IMPROVE) return;
    __shared__ double sd[8];
    __shared__ int si[8];
    __shared__ long long sl[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        changed += __shfl_xor_sync(0xffffffffu, changed, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sd[w] = rmax, si[w] = bad, sl[w] = changed;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        int bb = 0;
        long long cc = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, sd[k]), bb |= si[k], cc += sl[k];
        atomicMax(reinterpret_cast<unsigned long long*>(out + OUT_RESID_BITS), (unsigned long long)__double_as_longlong(r));
        if (cc) atomicAdd(reinterpret_cast<unsigned long long*>(out + OUT_CHANGED), (unsigned long long)cc);
        if (bb) atomicExch(reinterpret_cast<unsigned long long*>(out + OUT_STATUS), (unsigned long long)RMB_ERR_NONFINITE);
    }
}

template <typename PT, int MODE>
static cudaError_t launch_sparse_shard(const SparseArgs& a, int smode, int64_t row0, int64_t nloc, const double* Vr,
                                       int32_t* pir, const uint32_t* olist, const int* ocount, double* sv,
                                       uint32_t* si, int32_t* sa, long long* out, int grid, cudaStream_t st)
{
    if (smode == MODE_SHARD_MIN)
        sparse_shard_kernel<PT, MODE, MODE_SHARD_MIN><<<grid, 256, 0, st>>>(a, row0, nloc, Vr, pir, olist, ocount, sv, si, sa, out);
    else if (smode == MODE_SHARD_EVAL)
        sparse_shard_kernel<PT, MODE, MODE_SHARD_EVAL><<<grid, 256, 0, st>>>(a, row0, nloc, Vr, pir, olist, ocount, sv, si, sa, out);
    else
        sparse_shard_kernel<PT, MODE, MODE_SHARD_IMPROVE><<<grid, 256, 0, st>>>(a, row0, nloc, Vr, pir, olist, ocount, sv, si, sa, out);
    return cudaGetLastError();
}

rmb_status sparse_shard_step(Problem& pr, const SolveRequest& rq, const uint32_t* olist, const int* ocount,
                             double* send_val, uint32_t* send_idx, int32_t* send_arg, cudaStream_t st,
                             long long** out_dev)
{
    SparseArgs a{};
    a.row_ptr = pr.row_ptr;
    a.col = pr.col;
    a.val = pr.val;
    a.c = pr.c;
    a.n = pr.n;
    a.A = pr.A;
    a.K = pr.ell_K;
    a.gamma = pr.gamma;
    int mode;
    sparse_layout(pr, mode, a.GS, a.GSE);
    if (pr.ctrl.ensure(4096) != cudaSuccess) {
        set_error("sparse shard step: workspace allocation failed");
        return RMB_ERR_OOM;
    }
    long long* out = static_cast<long long*>(pr.ctrl.p);
    const int64_t nloc = pr.row_end - pr.row_begin;
    // work items: the batch's owned states (<= min(b, nloc)) or all owned states
    const int64_t items = rq.mode == MODE_SHARD_IMPROVE ? nloc : std::min<int64_t>(rq.b, nloc);
    const int GS = rq.mode == MODE_SHARD_EVAL ? a.GSE : a.GS;
    const int64_t groups_per_cta = 256 / GS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((items + groups_per_cta - 1) / groups_per_cta,
                                                                 (int64_t)pr.num_sms * 8));
    cudaError_t ce = cudaSuccess;
    if (rq.mode == MODE_SHARD_IMPROVE) ce = cudaMemsetAsync(out, 0, sizeof(long long) * OUT_N, st);
    if (ce == cudaSuccess) {
        const int sm = rq.mode;
        if (pr.pdt == RMB_F32)
            ce = mode == SM_VEC   ? launch_sparse_shard<float, SM_VEC>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st)
                 : mode == SM_ROW ? launch_sparse_shard<float, SM_ROW>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st)
                                  : launch_sparse_shard<float, SM_STRIDED>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st);
        else
            ce = mode == SM_VEC   ? launch_sparse_shard<double, SM_VEC>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st)
                 : mode == SM_ROW ? launch_sparse_shard<double, SM_ROW>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st)
                                  : launch_sparse_shard<double, SM_STRIDED>(a, sm, pr.row_begin, nloc, rq.V, rq.pi, olist, ocount, send_val, send_idx, send_arg, out, grid, st);
    }
    if (ce != cudaSuccess) {
        set_error(std::string("sparse shard step: ") + cudaGetErrorString(ce));
        return RMB_ERR_CUDA;
    }
    if (out_dev) *out_dev = out;
    return RMB_OK;
}

}  // namespace rmb

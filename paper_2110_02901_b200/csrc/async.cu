// async.cu — asynchronous MB-VI / MB-MPI on DENSE MDPs (SURVEY 8(f) row 4,
// "asynchronous variants of MB-VI and MB-MPI, which hold the
// promise of further speedup by avoiding synchronization", citing Tsitsiklis
// & Bertsekas' asynchronous DP).  DESIGN reading R31:
//
//   each operator application k walks the states in the order of its
//   partition (R2) with NO batch barrier: a CTA takes the next position from
//   a counter, backs its state up against V as it is in memory at that moment
//   (values written earlier in this application by any CTA may or may not be
//   seen -- every value read is one the state held since the application
//   started) and writes V(s) at once.  One grid barrier per application
//   (residual, stopping test, the next order).  The result is not
//   deterministic; it is pinned by properties that hold for every
//   interleaving (tests/test_gpu_async.py, test_oracle_async.py).
//
// One state per CTA (4 CTAs of 128 threads per SM): its A rows (all n columns) stream through registers
// (16-byte loads, L1 bypassed, L2 evict_first), each V vector is loaded once
// from L2 (.cg: the coherence point, never a stale L1 line) and used for AG
// rows; the CTA reduces the partial sums in a fixed order (thread columns ->
// warp butterfly -> warps in order) and takes the min over actions (lowest
// index on ties, R8).  MPI: evaluation sweeps are asynchronous B_{pi} sweeps,
// the improvement is an ordinary synchronous pass (no V write).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "partition.cuh"

namespace rmb {

namespace {

// threads per CTA: 4 CTAs of 128 per SM (tools/ab_async.py on config 2: 512 x 1
// 1.43 ms per application, 256 x 2 1.17, 128 x 4 1.12, 64 x 8 1.08 but more
// states in flight -> more applications to eps; a software-pipelined column
// loop measured 1.10, not kept; A/B builds only override these)
#ifndef RMB_ASYNC_NT
#define RMB_ASYNC_NT 128
#endif
#ifndef RMB_ASYNC_AGMAX
#define RMB_ASYNC_AGMAX 16
#endif
constexpr int kAThreads = RMB_ASYNC_NT;
constexpr int kAWarps = kAThreads / 32;
constexpr int kACtasPerSm = 512 / kAThreads;

struct AsyncArgs {
    const void* P;
    const void* c;
    int64_t n;
    int A;
    double gamma;
    double* V;
    int32_t* pi;
    uint64_t seed;
    int64_t k0;
    int identity;
    int mode;
    int pi_given;
    double eps;
    int64_t max_iter;
    int msweeps;
    uint32_t* perm;           // 3 * n
    unsigned long long* bar;  // grid barrier words
    int* err;
    unsigned int* ctr;        // [4] position counters (application parity, improvement)
    unsigned long long* red;  // [4 slots x 4]: residual bits, bad, changed
    const double* vref;       // RMB_TRACE_ERROR_VS_REF (null = off)
    double* etrace;
    int64_t etrace_len;
    double* trace;
    int64_t trace_len;
    long long* chg;
    int64_t chg_len;
    long long* out;
};

template <typename PT>
__device__ __forceinline__ double cost_at(const AsyncArgs& a, int64_t r)
{
    return (double)__ldg(static_cast<const PT*>(a.c) + r);
}

// V(j .. j+VE) from L2 (values written by other CTAs during the application)
template <int VE>
__device__ __forceinline__ void ld_v(const double* V, int64_t j, double (&v)[VE])
{
    if constexpr (VE == 4) {
        const double2 x = __ldcg(reinterpret_cast<const double2*>(V + j));
        const double2 y = __ldcg(reinterpret_cast<const double2*>(V + j + 2));
        v[0] = x.x, v[1] = x.y, v[2] = y.x, v[3] = y.y;
    } else if constexpr (VE == 2) {
        const double2 x = __ldcg(reinterpret_cast<const double2*>(V + j));
        v[0] = x.x, v[1] = x.y;
    } else {
        v[0] = __ldcg(V + j);
    }
}

// raw P vectors (converted to double inside the FMA loop: fewer registers)
template <typename PT, int VE>
struct PVec {
    PT x[VE];
};
template <typename PT, int VE>
__device__ __forceinline__ PVec<PT, VE> ld_p(const PT* p, uint64_t pol)
{
    PVec<PT, VE> r;
    if constexpr (VE == 4) {
        const float4 q = ld_first(reinterpret_cast<const float4*>(p), pol);
        r.x[0] = q.x, r.x[1] = q.y, r.x[2] = q.z, r.x[3] = q.w;
    } else if constexpr (VE == 2) {
        const double2 q = ld_first(reinterpret_cast<const double2*>(p), pol);
        r.x[0] = q.x, r.x[1] = q.y;
    } else {
        r.x[0] = ld_first(p, pol);
    }
    return r;
}

// Q(s, a) for the rows rows[0 .. na) of state s (all n columns) into Qs[slot[r]].
// Every thread of the CTA calls it; ends with the CTA synchronised.
template <typename PT, int VE, int AG>
__device__ __forceinline__ void state_rows(const AsyncArgs& a, int64_t s, const int* rows, int na, double* red,
                                           double* Qs, uint64_t pol)
{
    const PT* P = static_cast<const PT*>(a.P);
    const int64_t n = a.n;
    double acc[AG];
#pragma unroll
    for (int r = 0; r < AG; ++r) acc[r] = 0.0;
    // the rows of one call are consecutive actions (min) or the single row pi(s)
    const PT* base = P + ((int64_t)s * a.A + rows[0]) * n;
    for (int64_t j = (int64_t)threadIdx.x * VE; j < n; j += (int64_t)kAThreads * VE) {
        PVec<PT, VE> x[AG];
#pragma unroll
        for (int r = 0; r < AG; ++r)
            if (r < na) x[r] = ld_p<PT, VE>(base + (int64_t)r * n + j, pol);
        double v[VE];
        ld_v<VE>(a.V, j, v);
#pragma unroll
        for (int r = 0; r < AG; ++r)
            if (r < na) {
#pragma unroll
                for (int e = 0; e < VE; ++e) acc[r] = fma((double)x[r].x[e], v[e], acc[r]);
            }
    }

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < AG; ++r) {
        if (r < na) {
            double t = acc[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) red[warp * AG + r] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < na) {
        const int r = threadIdx.x;
        double t = 0.0;
        for (int w = 0; w < kAWarps; ++w) t += red[w * AG + r];
        Qs[r] = cost_at<PT>(a, (int64_t)s * a.A + rows[r]) + a.gamma * t;
    }
    __syncthreads();
}

struct AAcc {
    double rmax;
    int bad;
    long long changed;
};

// publish a CTA's accumulator into reduction slot q (thread 0 only)
__device__ __forceinline__ void publish(const AsyncArgs& a, int q, const AAcc& acc)
{
    unsigned long long* slot = a.red + 4 * (q & 3);
    atomicMax(slot, (unsigned long long)__double_as_longlong(acc.rmax));
    if (acc.bad) atomicOr(slot + 1, 1ull);
    if (acc.changed) atomicAdd(slot + 2, (unsigned long long)acc.changed);
}

// One pass over the states: KIND 0 = asynchronous B (min), 1 = asynchronous
// B_pi, 2 = improvement (greedy vs V, pi written, no V write; identity order).
// Positions are dealt dynamically, one state per CTA at a time.
template <typename PT, int VE, int AG, int KIND>
__device__ AAcc run_pass(const AsyncArgs& a, const uint32_t* perm, unsigned int* ctr, double* red, double* Qs,
                         int* rows, int64_t* sp)
{
    const uint64_t pol = l2_evict_first();
    AAcc acc{0.0, 0, 0};
    const int64_t n = a.n;
    if (threadIdx.x == 0) sp[0] = (int64_t)atomicAdd(ctr, 1u);
    __syncthreads();
    int64_t pos = sp[0];
    while (pos < n) {
        const int64_t s = perm ? (int64_t)__ldcg(perm + pos) : pos;
        __syncthreads();  // every thread has read sp[0]
        if (threadIdx.x == 0) sp[0] = (int64_t)atomicAdd(ctr, 1u);  // the next position, in flight
        double best = 0.0;
        int barg = 0;
        if (KIND == 1) {
            if (threadIdx.x == 0) rows[0] = __ldcg(a.pi + s);
            __syncthreads();
            state_rows<PT, VE, AG>(a, s, rows, 1, red, Qs, pol);
            best = Qs[0];
            barg = rows[0];
        } else {
            for (int a0 = 0; a0 < a.A; a0 += AG) {
                const int na = min(AG, a.A - a0);
                if (threadIdx.x < AG) rows[threadIdx.x] = a0 + threadIdx.x;
                __syncthreads();
                state_rows<PT, VE, AG>(a, s, rows, na, red, Qs + a0, pol);
            }
            if (threadIdx.x == 0) {
                best = Qs[0];
                for (int act = 1; act < a.A; ++act)
                    if (Qs[act] < best) best = Qs[act], barg = act;
            }
        }
        if (threadIdx.x == 0) {
            const double old = __ldcg(a.V + s);
            acc.bad |= !isfinite(best);
            acc.rmax = fmax(acc.rmax, fabs(best - old));
            if (KIND == 2) {
                acc.changed += (barg != __ldcg(a.pi + s));
                __stcg(a.pi + s, barg);
            } else {
                __stcg(a.V + s, best);  // visible to every later read of the application
                if (KIND == 0 && a.pi) __stcg(a.pi + s, barg);
            }
        }
        __syncthreads();
        pos = sp[0];
    }
    return acc;
}

template <typename PT, int VE, int AG>
__global__ void __launch_bounds__(kAThreads, kACtasPerSm) dense_async_kernel(const AsyncArgs a)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* red = reinterpret_cast<double*>(smem_raw);        // kAWarps * AG
    double* Qs = red + kAWarps * AG;                           // A (rounded up to AG)
    __shared__ int rows[AG];
    __shared__ int64_t sp[1];
    GridBarrier g{a.bar, a.bar + 32, 0ull, (unsigned long long)gridDim.x, a.err};
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    const int64_t n = a.n;
    const int64_t tid = (int64_t)blockIdx.x * kAThreads + threadIdx.x, stride = (int64_t)gridDim.x * kAThreads;
    auto fill = [&](int64_t k) {
        if (!a.identity) fill_order(n, a.seed, k, OrderSpec{0, nullptr, 0}, a.perm + (k % 3) * n, tid, stride);
    };
    fill(a.k0);
    grid_sync(g);
    int q = 0;  // reduction slot sequence
    // every pass uses counter q & 3 and slot q & 3; the ones two passes ahead
    // are re-armed by CTA 0 (their last users finished before the previous barrier)
    auto pass = [&](int kind, int64_t k) -> AAcc {
        if (lead) {
            a.ctr[(q + 2) & 3] = 0u;
            unsigned long long* z = a.red + 4 * ((q + 2) & 3);
            z[0] = z[1] = z[2] = 0ull;
        }
        const uint32_t* perm = (kind == 2 || a.identity) ? nullptr : a.perm + (k % 3) * n;
        AAcc acc = kind == 0   ? run_pass<PT, VE, AG, 0>(a, perm, a.ctr + (q & 3), red, Qs, rows, sp)
                   : kind == 1 ? run_pass<PT, VE, AG, 1>(a, perm, a.ctr + (q & 3), red, Qs, rows, sp)
                               : run_pass<PT, VE, AG, 2>(a, nullptr, a.ctr + (q & 3), red, Qs, rows, sp);
        if (threadIdx.x == 0) publish(a, q, acc);
        if (kind != 2) fill(k + 1);  // the next application's order (read after the barrier)
        grid_sync(g);
        unsigned long long* slot = a.red + 4 * (q & 3);
        AAcc r;
        r.rmax = __longlong_as_double((long long)ld_acquire_gpu(slot));
        r.bad = ld_acquire_gpu(slot + 1) != 0;
        r.changed = (long long)ld_acquire_gpu(slot + 2);
        ++q;
        return r;
    };
    // error trace after application it (V is global and written at once by
    // the next application: a barrier closes the pass)
    auto etrace_pass = [&](int64_t it_) {
        trace_error([&](int64_t j) { return __ldcg(a.V + j); }, a.vref, n, tid, stride, a.etrace + it_);
        grid_sync(g);
    };
    long long status = RMB_ERR_NOT_CONVERGED, changed = 0;
    int64_t k = a.k0, it = 0, outer = 0;
    double last = 0.0;
    if (a.mode == MODE_MPI) {
        bool bad = false;
        if (!a.pi_given) bad = pass(2, 0).bad;
        while (!bad && outer < a.max_iter) {
            const int64_t row = outer * (a.msweeps + 1);
            for (int e = 0; e < a.msweeps && !bad; ++e) {
                AAcc r = pass(1, k);
                if (lead && row + e < a.trace_len) a.trace[row + e] = r.rmax;
                if (a.etrace && it < a.etrace_len) etrace_pass(it);
                ++k, ++it;
                bad = r.bad;
            }
            if (bad) { ++outer; break; }
            AAcc r = pass(2, 0);
            if (lead && row + a.msweeps < a.trace_len) a.trace[row + a.msweeps] = r.rmax;
            if (lead && outer < a.chg_len) a.chg[outer] = r.changed;
            ++outer;
            last = r.rmax;
            changed = r.changed;
            if (r.bad) { bad = true; break; }
            if (r.changed == 0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if (bad) status = RMB_ERR_NONFINITE;
    } else {
        const int kind = (a.mode == MODE_APPLY_PI || a.mode == MODE_POLICY_VALUE) ? 1 : 0;
        const int64_t iters = (a.mode == MODE_VI || a.mode == MODE_POLICY_VALUE) ? a.max_iter : 1;
        while (it < iters) {
            AAcc r = pass(kind, k);
            if (lead && it < a.trace_len) a.trace[it] = r.rmax;
            if (a.etrace && it < a.etrace_len) etrace_pass(it);
            ++it, ++k;
            last = r.rmax;
            if (r.bad) { status = RMB_ERR_NONFINITE; break; }
            if (a.eps >= 0.0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if (a.eps < 0.0 && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
    }
    if (lead) {
        a.out[OUT_SWEEPS] = it;
        a.out[OUT_OUTER] = outer;
        a.out[OUT_STATUS] = status;
        a.out[OUT_RESID_BITS] = __double_as_longlong(last);
        a.out[OUT_BATCHES] = it;  // one "batch" (barrier) per application
        a.out[OUT_CHANGED] = changed;
    }
}

template <typename PT, int VE, int AG>
cudaError_t launch_async(const AsyncArgs& a, size_t smem, int grid, cudaStream_t st)
{
    auto kern = dense_async_kernel<PT, VE, AG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kAThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < kACtasPerSm) return cudaErrorCooperativeLaunchTooLarge;
    void* args[] = {const_cast<AsyncArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid * kACtasPerSm), dim3(kAThreads), args, smem, st);
}

template <typename PT, int VE>
cudaError_t launch_async_ag(const AsyncArgs& a, size_t smem_base, int grid, cudaStream_t st, int& AG)
{
    // rows streamed together per V vector: up to 16 (registers: 16 accumulators
    // + 16 x VE loads in flight per thread)
    // + 16 x VE loads in flight per thread); fp64 16-byte rows: up to 8 (spills at 16)
    constexpr int kAGMax = (sizeof(PT) == 8 && VE == 2) ? 8 : RMB_ASYNC_AGMAX;
    AG = a.A <= 4 ? 4 : (a.A <= 8 || kAGMax == 8 ? 8 : 16);
    const size_t smem = smem_base + (size_t)kAWarps * AG * 8 + (size_t)((a.A + AG - 1) / AG * AG) * 8;
    if (AG == 4) return launch_async<PT, VE, 4>(a, smem, grid, st);
    if constexpr (kAGMax == 8) return launch_async<PT, VE, 8>(a, smem, grid, st);
    else {
        if (AG == 8) return launch_async<PT, VE, 8>(a, smem, grid, st);
        return launch_async<PT, VE, 16>(a, smem, grid, st);
    }
}


// ===================================================================== TMA
// The same asynchronous applications (R31) with the rows streamed by TMA
// (cp.async.bulk) instead of per-thread loads: register streaming reaches
// ~0.83-0.88 of the copy peak, the bulk-copy ring ~0.95 (dense_tma_kernel).
//
// Warps 0..15 consume, warp 16 (kTCons) finishes states, warp 17 produces.
//  * producer (one lane): claims the next position of the application from
//    the global counter, and streams the state's UNITS (up to 16 consecutive
//    action rows -- or the row pi(s) -- of all n columns) as stages: a window
//    of V (from L2, a snapshot taken now: every value is one its state held
//    since the application began) plus the unit's rows over the same columns;
//  * consumers: warp w owns row w % R and column sub-slice w / R of every
//    stage, accumulates its lanes' partial dot products over the unit's
//    windows, and at the unit's last window posts the warp sum to a 4-slot
//    unit queue;
//  * finisher: adds the warps' partials in a fixed order, Q = c + gamma*sum,
//    takes min / argmin over the state's actions (lowest index on ties, R8)
//    and writes V(s) (and pi) at once -- off the consumers' path, so the ring
//    never waits for a state to be finished.
// One grid barrier per pass (consumers + finisher; the producer waits for the
// next pass's go signal, so no V window of pass q+1 is read before it starts).
#ifndef RMB_TA_CONS
#define RMB_TA_CONS 16
#endif
constexpr int kTCons = RMB_TA_CONS;              // consumer warps
constexpr int kTProd = kTCons + 1;               // producer warp index
constexpr int kTBar = (kTCons + 1) * 32;         // threads in the pass barrier (consumers + finisher)
constexpr int kTThreads = (kTCons + 2) * 32;     // 576
constexpr int kTUnitQ = 4;                       // unit queue depth
#ifndef RMB_TA_RMAX
#define RMB_TA_RMAX 16
#endif
constexpr int kTRMax = RMB_TA_RMAX;              // rows per unit (accumulators per lane)
constexpr int kTMaxStages = 12;

enum : int { TF_FIRST = 1, TF_LAST = 2, TF_STATE_LAST = 4, TF_END = 8 };

struct TMeta {
    long long s;
    int a0;     // first row's action (min kinds) or pi(s) (evaluation)
    int rows;   // rows in this unit
    int c0, len;
    int flags;
    int pad;
};

struct TUnit {
    long long s;
    int a0, rows, flags, pad;
};

struct TLayout {
    int nst;           // ring stages
    int slot;          // bytes per stage
    int w[3];          // columns per stage by kind (0 min, 1 eval, 2 improvement)
    int R[3];          // rows per unit by kind
};

struct TSmem {
    unsigned char* ring;
    unsigned long long *full, *empty, *ufull, *uempty;
    TMeta* meta;
    TUnit* unit;
    double* red;  // [kTUnitQ][kTRMax][kTCons]
    double* Qs;   // [A]
    long long* ctl;  // [0] go pass (-1 stop), [1] kind, [2] application k
};

__device__ __forceinline__ TSmem tsmem(unsigned char* raw, const TLayout& L, int A)
{
    TSmem m;
    size_t off = 0;
    m.ring = raw;
    off += (size_t)L.nst * L.slot;
    m.full = reinterpret_cast<unsigned long long*>(raw + off);
    m.empty = m.full + L.nst;
    m.ufull = m.empty + L.nst;
    m.uempty = m.ufull + kTUnitQ;
    off += (size_t)(2 * L.nst + 2 * kTUnitQ) * 8;
    m.meta = reinterpret_cast<TMeta*>(raw + off);
    off += (size_t)L.nst * sizeof(TMeta);
    m.unit = reinterpret_cast<TUnit*>(raw + off);
    off += (size_t)kTUnitQ * sizeof(TUnit);
    m.red = reinterpret_cast<double*>(raw + off);
    off += (size_t)kTUnitQ * kTRMax * kTCons * 8;
    m.Qs = reinterpret_cast<double*>(raw + off);
    off += (size_t)((A + 1) & ~1) * 8;
    m.ctl = reinterpret_cast<long long*>(raw + off);
    return m;
}

inline size_t tsmem_bytes(const TLayout& L, int A)
{
    return (size_t)L.nst * L.slot + (size_t)(2 * L.nst + 2 * kTUnitQ) * 8 + (size_t)L.nst * sizeof(TMeta) +
           (size_t)kTUnitQ * sizeof(TUnit) + (size_t)kTUnitQ * kTRMax * kTCons * 8 + (size_t)((A + 1) & ~1) * 8 + 64;
}

struct TmaAsyncArgs {
    AsyncArgs a;
    TLayout L;
};

template <typename PT>
__device__ void tma_async_producer(const AsyncArgs& a, const TLayout& L, const TSmem& m)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const PT* P = static_cast<const PT*>(a.P);
    const int64_t n = a.n;
    int st = 0;
    unsigned ph = 0;
    auto acquire = [&]() {
        SpinGuard sg;
        while (!mbar_try(m.empty + st, ph ^ 1u)) sg.tick();
    };
    auto advance = [&]() {
        if (++st == L.nst) st = 0, ph ^= 1u;
    };
    for (long long q = 0;; ++q) {
        long long go;
        {
            SpinGuard sg;
            while ((go = ld_acquire_cta(m.ctl)) != q && go != -1) {
                sg.tick();
                __nanosleep(128);
            }
        }
        if (go == -1) return;
        const int kind = (int)m.ctl[1];
        const long long k = m.ctl[2];
        // V windows of this pass are read after every write of the previous
        // pass (ordered by the grid barrier): make them visible to the async proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint32_t* perm = (kind == 2 || a.identity) ? nullptr : a.perm + (k % 3) * n;
        unsigned int* ctr = a.ctr + (q & 3);
        const int R = L.R[kind], w = L.w[kind];
        const int vbytes = ((w * 8) + 127) & ~127;
        const int rslot = ((w * (int)sizeof(PT)) + 127) & ~127;
        long long pos = atomicAdd(ctr, 1u);
        while (pos < n) {
            const long long s = perm ? (long long)__ldcg(perm + pos) : pos;
            const long long pos_next = atomicAdd(ctr, 1u);  // in flight while this state streams
            const int act = kind == 1 ? __ldcg(a.pi + s) : 0;
            const int ngroups = kind == 1 ? 1 : (a.A + R - 1) / R;
            for (int g = 0; g < ngroups; ++g) {
                const int a0 = kind == 1 ? act : g * R;
                const int rows = kind == 1 ? 1 : min(R, a.A - a0);
                for (int c0 = 0; c0 < n; c0 += w) {
                    const int len = (int)min((int64_t)w, n - c0);
                    acquire();
                    TMeta& md = m.meta[st];
                    md.s = s;
                    md.a0 = a0;
                    md.rows = rows;
                    md.c0 = c0;
                    md.len = len;
                    md.flags = (c0 == 0 ? TF_FIRST : 0) | (c0 + w >= n ? TF_LAST : 0) |
                               (c0 + w >= n && g == ngroups - 1 ? TF_STATE_LAST : 0);
                    unsigned char* stage = m.ring + (size_t)st * L.slot;
                    mbar_arrive_tx(m.full + st, (unsigned)(len * 8 + rows * len * (int)sizeof(PT)));
                    bulk_g2s(stage, a.V + c0, (unsigned)(len * 8), m.full + st, pol);
                    for (int r = 0; r < rows; ++r)
                        bulk_g2s(stage + vbytes + r * rslot, P + ((int64_t)s * a.A + a0 + r) * n + c0,
                                 (unsigned)(len * (int)sizeof(PT)), m.full + st, pol);
                    advance();
                }
            }
            pos = pos_next;
        }
        acquire();  // end of the pass
        m.meta[st].flags = TF_END;
        mbar_arrive(m.full + st);
        advance();
    }
}

// Warps split a stage into NRG = ceil(rows / kTRW) row groups x NCS =
// kTCons / NRG column slices: warp w takes rows [rg kTRW, rg kTRW + kTRW) of
// column slice cs (rg = w % NRG, cs = w / NRG) -- each V vector it reads from
// shared memory serves kTRW rows.
#ifndef RMB_TA_RW
#define RMB_TA_RW 4
#endif
constexpr int kTRW = RMB_TA_RW;

__device__ __forceinline__ void tma_split(int rows, int& nrg, int& ncs)
{
    nrg = (rows + kTRW - 1) / kTRW;
    ncs = kTCons / nrg;
}

template <typename PT>
__device__ __forceinline__ void tma_dot(const unsigned char* stage, const TMeta& md, int vbytes, int rslot, int warp,
                                        int lane, double (&acc)[kTRW])
{
    constexpr int VE = 16 / (int)sizeof(PT);
    int nrg, ncs;
    tma_split(md.rows, nrg, ncs);
    const int rg = warp % nrg, cs = warp / nrg;
    if (cs >= ncs) return;
    const int nv = md.len / VE;  // 16-byte vectors in the window
    const int v0 = (int)((int64_t)nv * cs / ncs), v1 = (int)((int64_t)nv * (cs + 1) / ncs);
    const double* Vw = reinterpret_cast<const double*>(stage);
    const unsigned char* rows = stage + vbytes + (size_t)rg * kTRW * rslot;
    const int nr = min(kTRW, md.rows - rg * kTRW);
    for (int v = v0 + lane; v < v1; v += 32) {
        if constexpr (VE == 4) {
            const double2 x = reinterpret_cast<const double2*>(Vw)[2 * v];
            const double2 y = reinterpret_cast<const double2*>(Vw)[2 * v + 1];
#pragma unroll
            for (int r = 0; r < kTRW; ++r)
                if (r < nr) {
                    const float4 p = reinterpret_cast<const float4*>(rows + r * rslot)[v];
                    acc[r] = fma((double)p.x, x.x, acc[r]);
                    acc[r] = fma((double)p.y, x.y, acc[r]);
                    acc[r] = fma((double)p.z, y.x, acc[r]);
                    acc[r] = fma((double)p.w, y.y, acc[r]);
                }
        } else {
            const double2 x = reinterpret_cast<const double2*>(Vw)[v];
#pragma unroll
            for (int r = 0; r < kTRW; ++r)
                if (r < nr) {
                    const double2 p = reinterpret_cast<const double2*>(rows + r * rslot)[v];
                    acc[r] = fma(p.x, x.x, acc[r]);
                    acc[r] = fma(p.y, x.y, acc[r]);
                }
        }
    }
}

template <typename PT>
__global__ void __launch_bounds__(kTThreads, 1) dense_async_tma_kernel(const TmaAsyncArgs ta)
{
    const AsyncArgs& a = ta.a;
    const TLayout& L = ta.L;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TSmem m = tsmem(smem_raw, L, a.A);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = a.n;
    if (threadIdx.x == 0) {
        for (int q = 0; q < L.nst; ++q) {
            mbar_init(m.full + q, 1);
            mbar_init(m.empty + q, kTCons);
        }
        for (int q = 0; q < kTUnitQ; ++q) {
            mbar_init(m.ufull + q, kTCons);
            mbar_init(m.uempty + q, 1);
        }
        m.ctl[0] = -2;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the first application's order (every thread of the grid), then the barrier
    const int64_t tid = (int64_t)blockIdx.x * kTThreads + threadIdx.x, stride = (int64_t)gridDim.x * kTThreads;
    if (!a.identity) fill_order(n, a.seed, a.k0, OrderSpec{0, nullptr, 0}, a.perm + (a.k0 % 3) * n, tid, stride);
    __syncthreads();  // the only full-CTA barrier: the producer warp leaves here
    if (warp == kTProd) {
        if (lane == 0) tma_async_producer<PT>(a, L, m);
        return;
    }
    GridBarrier g{a.bar, a.bar + 32, 0ull, (unsigned long long)gridDim.x, a.err};
    grid_sync<kTBar>(g);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    int st = 0;
    unsigned ph = 0;
    long long units = 0;  // unit queue sequence (consumers and finisher count alike)
    int q = 0;
    // one pass: the consumers stream stages until END, the finisher drains the
    // unit queue and publishes the CTA's (rmax, bad, changed) into slot q & 3
    auto pass = [&](int kind, int64_t k) -> AAcc {
        if (lead) {
            a.ctr[(q + 2) & 3] = 0u;
            unsigned long long* z = a.red + 4 * ((q + 2) & 3);
            z[0] = z[1] = z[2] = 0ull;
        }
        if (kind != 2 && !a.identity)  // the next application's order (read after this pass's barrier)
            fill_order(n, a.seed, k + 1, OrderSpec{0, nullptr, 0}, a.perm + ((k + 1) % 3) * n,
                       (int64_t)blockIdx.x * kTBar + threadIdx.x, (int64_t)gridDim.x * kTBar);
        if (threadIdx.x == 0) {
            m.ctl[1] = kind;
            m.ctl[2] = k;
            st_release_cta(m.ctl, q);
        }
        const int w = L.w[kind];
        const int vbytes = ((w * 8) + 127) & ~127;
        const int rslot = ((w * (int)sizeof(PT)) + 127) & ~127;
        if (warp < kTCons) {
            double acc[kTRW];
#pragma unroll
            for (int r = 0; r < kTRW; ++r) acc[r] = 0.0;
            while (true) {
                {
                    SpinGuard sg;
                    while (!mbar_try(m.full + st, ph)) sg.tick();
                }
                const TMeta md = m.meta[st];
                if (md.flags & TF_END) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(m.empty + st);
                    if (++st == L.nst) st = 0, ph ^= 1u;
                    // the END unit
                    const int us = (int)(units & (kTUnitQ - 1));
                    {
                        SpinGuard sg;
                        while (!mbar_try(m.uempty + us, (unsigned)((units / kTUnitQ) & 1) ^ 1u)) sg.tick();
                    }
                    if (warp == 0 && lane == 0) m.unit[us].flags = TF_END;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(m.ufull + us);
                    ++units;
                    break;
                }
                if (md.flags & TF_FIRST) {
#pragma unroll
                    for (int r = 0; r < kTRW; ++r) acc[r] = 0.0;
                }
                tma_dot<PT>(m.ring + (size_t)st * L.slot, md, vbytes, rslot, warp, lane, acc);
                __syncwarp();
                if (lane == 0) mbar_arrive(m.empty + st);
                if (++st == L.nst) st = 0, ph ^= 1u;
                if (md.flags & TF_LAST) {  // the unit's partials of this warp -> the unit queue
                    const int us = (int)(units & (kTUnitQ - 1));
                    {
                        SpinGuard sg;
                        while (!mbar_try(m.uempty + us, (unsigned)((units / kTUnitQ) & 1) ^ 1u)) sg.tick();
                    }
                    int nrg, ncs;
                    tma_split(md.rows, nrg, ncs);
                    const int rg = warp % nrg, cs = warp / nrg;
                    if (cs < ncs) {
#pragma unroll
                        for (int r = 0; r < kTRW; ++r)
                            if (rg * kTRW + r < md.rows) {
                                const double t = warp_sum(acc[r]);
                                if (lane == 0) m.red[(us * kTRMax + rg * kTRW + r) * kTCons + cs] = t;
                            }
                    }
                    if (warp == 0 && lane == 0) {
                        m.unit[us].s = md.s;
                        m.unit[us].a0 = md.a0;
                        m.unit[us].rows = md.rows;
                        m.unit[us].flags = md.flags;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(m.ufull + us);
                    ++units;
                }
            }
        } else {  // finisher warp
            AAcc acc{0.0, 0, 0};
            while (true) {
                const int us = (int)(units & (kTUnitQ - 1));
                {
                    SpinGuard sg;
                    while (!mbar_try(m.ufull + us, (unsigned)((units / kTUnitQ) & 1))) sg.tick();
                }
                const TUnit u = m.unit[us];
                if (u.flags & TF_END) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(m.uempty + us);
                    ++units;
                    break;
                }
                if (lane < u.rows) {
                    double t = 0.0;
                    int nrg, ncs;
                    tma_split(u.rows, nrg, ncs);
                    for (int cs = 0; cs < ncs; ++cs) t += m.red[(us * kTRMax + lane) * kTCons + cs];
                    const int act = u.a0 + (kind == 1 ? 0 : lane);
                    m.Qs[kind == 1 ? 0 : act] = cost_at<PT>(a, u.s * a.A + act) + a.gamma * t;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(m.uempty + us);
                ++units;
                if ((u.flags & TF_STATE_LAST) && lane == 0) {
                    double best = m.Qs[0];
                    int barg = kind == 1 ? u.a0 : 0;
                    if (kind != 1)
                        for (int act = 1; act < a.A; ++act)
                            if (m.Qs[act] < best) best = m.Qs[act], barg = act;
                    const double old = __ldcg(a.V + u.s);
                    acc.bad |= !isfinite(best);
                    acc.rmax = fmax(acc.rmax, fabs(best - old));
                    if (kind == 2) {
                        acc.changed += (barg != __ldcg(a.pi + u.s));
                        __stcg(a.pi + u.s, barg);
                    } else {
                        __stcg(a.V + u.s, best);
                        if (kind == 0 && a.pi) __stcg(a.pi + u.s, barg);
                    }
                }
                __syncwarp();
            }
            if (lane == 0) publish(a, q, acc);
        }
        grid_sync<kTBar>(g);
        unsigned long long* slot = a.red + 4 * (q & 3);
        AAcc r;
        r.rmax = __longlong_as_double((long long)ld_acquire_gpu(slot));
        r.bad = ld_acquire_gpu(slot + 1) != 0;
        r.changed = (long long)ld_acquire_gpu(slot + 2);
        ++q;
        return r;
    };
    auto etrace_pass = [&](int64_t it_) {
        trace_error([&](int64_t j) { return __ldcg(a.V + j); }, a.vref, n, (int64_t)blockIdx.x * kTBar + threadIdx.x,
                    (int64_t)gridDim.x * kTBar, a.etrace + it_);
        grid_sync<kTBar>(g);
    };
    long long status = RMB_ERR_NOT_CONVERGED, changed = 0;
    int64_t k = a.k0, it = 0, outer = 0;
    double last = 0.0;
    if (a.mode == MODE_MPI) {
        bool bad = false;
        if (!a.pi_given) bad = pass(2, 0).bad;
        while (!bad && outer < a.max_iter) {
            const int64_t row = outer * (a.msweeps + 1);
            for (int e = 0; e < a.msweeps && !bad; ++e) {
                AAcc r = pass(1, k);
                if (lead && row + e < a.trace_len) a.trace[row + e] = r.rmax;
                if (a.etrace && it < a.etrace_len) etrace_pass(it);
                ++k, ++it;
                bad = r.bad;
            }
            if (bad) { ++outer; break; }
            AAcc r = pass(2, 0);
            if (lead && row + a.msweeps < a.trace_len) a.trace[row + a.msweeps] = r.rmax;
            if (lead && outer < a.chg_len) a.chg[outer] = r.changed;
            ++outer;
            last = r.rmax;
            changed = r.changed;
            if (r.bad) { bad = true; break; }
            if (r.changed == 0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if (bad) status = RMB_ERR_NONFINITE;
    } else {
        const int kind = (a.mode == MODE_APPLY_PI || a.mode == MODE_POLICY_VALUE) ? 1 : 0;
        const int64_t iters = (a.mode == MODE_VI || a.mode == MODE_POLICY_VALUE) ? a.max_iter : 1;
        while (it < iters) {
            AAcc r = pass(kind, k);
            if (lead && it < a.trace_len) a.trace[it] = r.rmax;
            if (a.etrace && it < a.etrace_len) etrace_pass(it);
            ++it, ++k;
            last = r.rmax;
            if (r.bad) { status = RMB_ERR_NONFINITE; break; }
            if (a.eps >= 0.0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if (a.eps < 0.0 && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
    }
    if (threadIdx.x == 0) st_release_cta(m.ctl, -1);  // the producer exits
    if (lead) {
        a.out[OUT_SWEEPS] = it;
        a.out[OUT_OUTER] = outer;
        a.out[OUT_STATUS] = status;
        a.out[OUT_RESID_BITS] = __double_as_longlong(last);
        a.out[OUT_BATCHES] = it;
        a.out[OUT_CHANGED] = changed;
    }
}

// Stage geometry (tools/ab_async_tma.py on config 2): 72 KB slots, 3 stages
// -- a V window + up to 16 rows of ~4 KB (fp32, 1000-1024 columns); each
// kind's windows are equal multiples of 32 columns that fit (40 KB slots:
// 1.45-3.1 ms per application, 56 KB 1.31, 72 KB 0.98, 104 KB 1.12).
#ifndef RMB_TA_SLOT_KB
#define RMB_TA_SLOT_KB 72
#endif
inline bool tma_layout(int64_t n, int A, int psz, size_t smem_optin, TLayout& L)
{
    // every row of a unit needs a warp: ceil(R / kTRW) row groups <= kTCons
    const int R0 = std::min(std::min(A, kTRMax), kTCons * kTRW);
    L.R[0] = L.R[2] = R0;
    L.R[1] = 1;
    const int slot = RMB_TA_SLOT_KB * 1024;
    L.slot = slot;
    for (int kd = 0; kd < 3; ++kd) {
        const int R = L.R[kd];
        auto fits = [&](int64_t w) { return ((w * 8 + 127) & ~127) + R * ((w * psz + 127) & ~127) <= slot; };
        int64_t wmax = 32;
        while (fits(wmax + 32)) wmax += 32;
        // equal windows (multiples of 32 columns) -- no nearly empty last stage
        int64_t win = (n + wmax - 1) / wmax, w = wmax;
        while (true) {
            w = ((n + win - 1) / win + 31) / 32 * 32;
            if (w <= wmax) break;
            ++win;
        }
        L.w[kd] = (int)w;
    }
    L.nst = kTMaxStages;
    while (L.nst >= 3 && tsmem_bytes(L, A) + 1024 > smem_optin) --L.nst;
    return L.nst >= 3;
}

}  // namespace

rmb_status dense_async_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                             long long* chg_dev, int64_t chg_len, SolveResult* res)
{
    const int64_t n = pr.n;
    const int psz = pr.pdt == RMB_F32 ? 4 : 8;
    int VE = 16 / psz;
    if ((n % VE) != 0 || (reinterpret_cast<uintptr_t>(pr.P) & 15u) != 0) VE = 1;
    AsyncArgs a{};
    a.P = pr.P;
    a.c = pr.c;
    a.n = n;
    a.A = pr.A;
    a.gamma = pr.gamma;
    a.V = rq.V;
    a.pi = rq.pi;
    a.seed = rq.seed;
    a.k0 = rq.k0;
    a.identity = rq.identity ? 1 : 0;
    a.mode = rq.mode;
    a.pi_given = rq.pi_given ? 1 : 0;
    a.eps = rq.eps;
    a.max_iter = rq.max_iter;
    a.msweeps = rq.msweeps;
    a.vref = rq.vref;
    a.etrace = rq.etrace;
    a.etrace_len = rq.etrace_len;
    if (pr.perm.ensure((size_t)3 * n * 4) != cudaSuccess || pr.ctrl.ensure(4096) != cudaSuccess) {
        set_error("async solver: workspace allocation failed");
        return RMB_ERR_OOM;
    }
    a.perm = static_cast<uint32_t*>(pr.perm.p);
    unsigned long long* ctrl = static_cast<unsigned long long*>(pr.ctrl.p);
    a.bar = ctrl;                                          // [0], [32]
    a.err = reinterpret_cast<int*>(ctrl + 64);             // [64]
    a.out = reinterpret_cast<long long*>(ctrl + 128);      // [128..136)
    a.ctr = reinterpret_cast<unsigned int*>(ctrl + 256);   // [256..258)
    a.red = ctrl + 320;                                    // [320..336)
    a.trace = trace_dev;
    a.trace_len = trace_len;
    a.chg = chg_dev;
    a.chg_len = chg_len;
    cudaStream_t st = pr.stream;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaMemsetAsync(ctrl, 0, 4096, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(e0, st);
    int AG = 0;
    // 16-byte rows: the TMA ring kernel; else per-thread register streaming
    TmaAsyncArgs ta{a, TLayout{}};
    const bool tma = VE * psz == 16 && !pr.no_tma && tma_layout(n, pr.A, psz, pr.smem_optin, ta.L);
    if (ce == cudaSuccess) {
        const int grid = pr.num_sms;
        if (tma) {
            const size_t smem = tsmem_bytes(ta.L, pr.A);
            auto kern = pr.pdt == RMB_F32 ? dense_async_tma_kernel<float> : dense_async_tma_kernel<double>;
            ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int per_sm = 0;
            if (ce == cudaSuccess) ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTThreads, smem);
            if (ce == cudaSuccess && per_sm < 1) ce = cudaErrorCooperativeLaunchTooLarge;
            void* args[] = {&ta};
            if (ce == cudaSuccess)
                ce = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kTThreads), args, smem, st);
        } else if (pr.pdt == RMB_F32) {
            ce = VE == 4 ? launch_async_ag<float, 4>(a, 0, grid, st, AG) : launch_async_ag<float, 1>(a, 0, grid, st, AG);
        } else {
            ce = VE == 2 ? launch_async_ag<double, 2>(a, 0, grid, st, AG) : launch_async_ag<double, 1>(a, 0, grid, st, AG);
        }
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(e1, st);
    long long out[OUT_N] = {0};
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, a.out, sizeof(long long) * OUT_N, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    float ms = 0.f;
    if (ce == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) {
        set_error(std::string("async solver: ") + cudaGetErrorString(ce));
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
    pr.last_launches = 1;
    for (int i = 0; i < 4; ++i) pr.prof[i] = 0;
    return RMB_OK;
}

}  // namespace rmb

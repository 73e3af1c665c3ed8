// dense.cu — persistent sm_100a solver for DENSE MDPs (P [n][A][n]).
//
// One cooperative launch runs a whole MB-VI or MB-MPI solve (PAPER.md P:L186,
// Alg. 1): every batch, every sweep and the stopping test, with no
// host round trip.  Design:
//
//  * Each CTA (one per SM, 512 threads) keeps the interim value function V
//    (fp64) resident in shared memory for the whole solve, plus pi for MPI.
//  * Batch t of sweep k = positions [t*b, min(n,(t+1)*b)) of the permutation
//    pi_k (partition.cuh; perm of sweep k+1 is generated during sweep k).
//  * COMPUTE: the batch's rows are cut into items (state, 4 actions, column
//    chunk); items are dealt to CTAs round-robin (per-SM balance within one
//    item) and to warps through a shared-memory counter.  A warp streams its
//    4 P-row chunks with 128-bit L1::no_allocate loads (each P byte read once
//    per sweep) and dots them with the smem V in fp64.
//      - C == 1 (rows not split): the warp finishes the backup itself:
//        Q = c + gamma * dot per action, and writes the group's (min Q, argmin).
//      - C > 1 (small b, rows split to fill 148 SMs): fp64 partial sums per
//        (state, action, chunk).
//  * BARRIER: one grid barrier per batch ("the batch is written back before
//    the next batch starts").
//  * COMBINE: per state, sum partials in chunk order / take the min over the
//    action groups in order (lowest index on exact ties), residual |Q - V_old|
//    and the smem patch of V.  Small partial volumes: every CTA reduces all
//    states itself (redundant, no second barrier).  Large: CTA x reduces the
//    states i = x mod grid into a list, a second barrier, every CTA patches.
//    Every CTA ends each batch with an identical V, residual and stop decision.
//  * Reads within a batch see only pre-batch values (Eq. 12: S \ M(i) with J,
//    M(i) with B J): smem V is patched only after the batch's barrier.
//  * Reduction order is a function of (n, b, mode) only: bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "partition.cuh"

namespace rmb {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / kWarp;
constexpr int kAG = 4;                     // actions per compute item (min modes)
constexpr int kPathWarp = 0, kPathTma = 3;  // compute path of a kernel instantiation
// TMA path with V (and pi) in GLOBAL memory (L2-resident) instead of shared
// memory: dense n too large for a shared-memory copy of V (n > ~27k)
constexpr int kPathTmaG = 4;
// kernel instantiations of the fused multi-rank path (K8f): the same two TMA
// variants with the exchange compiled in (the single-GPU kernels carry none of it)
constexpr int kPathTmaF = 5, kPathTmaGF = 6;
__host__ __device__ constexpr bool is_tma(int c) { return c >= kPathTma && c <= kPathTmaGF; }
__host__ __device__ constexpr bool is_vgl(int c) { return c == kPathTmaG || c == kPathTmaGF; }
__host__ __device__ constexpr bool is_fused(int c) { return c == kPathTmaF || c == kPathTmaGF; }
constexpr int64_t kRedundantMax = 8192;    // doubles of batch partials reduced by every CTA
constexpr int kMaxRanks = 8;               // ranks of a fused multi-GPU group (one NVSwitch box)

// CTA barrier of the 512 compute threads (named barrier 1).  Identical to
// __syncthreads() for the 512-thread paths; the TMA path adds a producer warp
// (threads 512..543) that never joins it.
__device__ __forceinline__ void csync() { bar_sync_n<kThreads>(); }

struct Plan {
    int Lc;         // chunk length (elements)
    int C;          // chunks per row
    int redundant;  // 1: every CTA reduces every state (single barrier)
    int ng;         // action rows per warp item in min modes (4, or 1 for short-tail batches)
    int raw;        // 1 (TMA path): items store raw row dot products part[(i*Ae + a)*C + ch]; costs,
                    //   chunk sums and min/argmin are all done by the combine (S-mode, even at C == 1)
};

struct DenseArgs {
    const void* P;
    const void* c;
    int64_t n;
    int A;
    double gamma;
    double* V;
    int32_t* pi;
    int64_t b;
    uint64_t seed;
    int64_t k0;
    int identity;
    int mode;
    int pi_given;
    double eps;
    int64_t max_iter;
    int msweeps;
    Plan plan[3];        // 0 = B_b sweep, 1 = B_{pi,b} sweep, 2 = improvement
    int64_t imp_sub;     // improvement sub-batch (states)
    double* vnext;       // chunked T (VI*): new values of the sweep, applied at its end; null = B_b
    uint32_t* perm;      // 3 * n (triple-buffered by sweep index)
    OrderSpec order;     // permutation, or draws with replacement (R28-R29)
    const double* vref;  // RMB_TRACE_ERROR_VS_REF: reference V*, etrace[i] = ||V_i - V*|| (null = off)
    double* etrace;
    int64_t etrace_len;
    double* part;        // 2 * part_stride
    int64_t part_stride;
    double* lval;        // distributed-combine list: value per batch position
    int32_t* larg;       //                           argmin per batch position
    unsigned int* scnt;  // per batch position: items completed (last-arriver)
    unsigned long long* bar;
    int* err;
    double* trace;
    int64_t trace_len;
    long long* chg;
    int64_t chg_len;
    long long* out;
    unsigned int* wctr;  // [2] work-stealing counters (phase parity)
    int path;            // compute path (kPathWarp / kPathTma / kPathTmaG)
    int64_t vs_half;     // smem V: offset of the hi plane (VE == 4), 0 = linear
    // multi-GPU shard steps
    int64_t row0, row1;        // owned states (P and c are offset so that global state ids index them)
    const uint32_t* olist;     // this rank's states of the batch (compacted)
    const int* ocount;         // their number (device)
    double* send_val;          // per owned batch state: new value
    uint32_t* send_idx;        //                        state id
    int32_t* send_arg;         //                        argmin (or pi(s))
    int64_t qs_cap;      // doubles of smem scratch for S-mode reductions
    int64_t qs_off;      // byte offset of that scratch in dynamic smem
    long long* prof;     // [0] compute ns, [1] barrier ns, [2] combine ns, [3] barriers (CTA 0)
    int64_t tma_off;     // TMA path: byte offset of the stage ring in dynamic smem
    int tma_nst;         //           ring stages
    unsigned long long* gred;  // global-V path: 4 reduction slots x 4 words (rmax bits, bad, changed)
    int tma_piece;       //           columns per stage and row slot
    int tma_static;      //           batches with <= tma_static * grid items are dealt statically
    int tma_slot;        //           bytes per ring slot (piece bytes rounded up to 128)
    // this rank's CTAs: [cta0, cta0 + nctas) of the launch (several ranks share
    // one launch when a multi-GPU group is emulated on one device)
    int cta0, nctas;
    // fused multi-rank exchange (K8f; xG == 0: off).  Rank xrank of xG owns
    // states [row0, row1); per batch it backs up its states of the batch and
    // stores (value, argmin) at the batch position into EVERY rank's xval/xarg
    // (peer memory), then a cross-rank barrier; every rank then patches its
    // replica of V from its own xval/xarg.
    int xG, xrank;
    double* xval[kMaxRanks];              // per rank: [2][lcap] by batch position (batch parity)
    int32_t* xarg[kMaxRanks];             // per rank: [2][lcap]
    unsigned long long* xbar[kMaxRanks];  // per rank: cross-rank arrival counter (monotonic)
    unsigned long long* ximp[kMaxRanks];  // per rank: [2][kMaxRanks][4] improvement records
    unsigned long long xbase;             // cross-rank epochs completed before this launch
    double* xval_own;                     // this rank's entries of the arrays above (no dynamic
    int32_t* xarg_own;                    //   indexing of parameter arrays in the kernel)
    unsigned long long* xbar_own;
    unsigned long long* ximp_own;
    uint32_t* xlist;                      // this rank: [3][2 xlcap] (position, state) of its batch states
    unsigned int* xcnt;                   // this rank: [3] list lengths
    int64_t xlcap;                        // batch positions per xval / xarg parity
    unsigned long long* xloc;             // this rank: local arrival counter of the cross-rank barrier
    unsigned long long* xrel;             // this rank: release epoch of the cross-rank barrier
};

// this CTA's index among its rank's CTAs
__device__ __forceinline__ int cta_rank(const DenseArgs& a) { return (int)blockIdx.x - a.cta0; }

// ---------------------------------------------------------------- loads
template <typename PT, int VE>
struct Vec;
template <>
struct Vec<float, 4> {
    using T = float4;
    __device__ static __forceinline__ void get(const T& x, double (&d)[4])
    {
        d[0] = x.x, d[1] = x.y, d[2] = x.z, d[3] = x.w;
    }
};
template <>
struct Vec<double, 2> {
    using T = double2;
    __device__ static __forceinline__ void get(const T& x, double (&d)[2]) { d[0] = x.x, d[1] = x.y; }
};
template <>
struct Vec<float, 1> {
    using T = float;
    __device__ static __forceinline__ void get(const T& x, double (&d)[1]) { d[0] = x; }
};
template <>
struct Vec<double, 1> {
    using T = double;
    __device__ static __forceinline__ void get(const T& x, double (&d)[1]) { d[0] = x; }
};

// Shared-memory layout of V.  With float4 P vectors (VE == 4) a lane needs
// V[j..j+3] (32 B); stored linearly, 8 lanes of a quarter warp would hit the
// same banks twice.  So V is split into two planes: lo holds (V[4q], V[4q+1])
// at [2q, 2q+1], hi holds (V[4q+2], V[4q+3]) at half + [2q, 2q+1]; each
// 128-bit read is then at a 16-byte lane stride (conflict-free).  Other VE: linear.
__device__ __forceinline__ int64_t vs_index(int64_t j, int64_t half)
{
    return half ? ((j & 2) ? half : 0) + ((j >> 2) << 1) + (j & 1) : j;
}

template <int VE>
__device__ __forceinline__ void load_v(const double* Vs, int64_t j, double (&v)[VE], int64_t half = 0)
{
    if constexpr (VE == 4) {
        const double2 a = *reinterpret_cast<const double2*>(Vs + (j >> 1));
        const double2 b = *reinterpret_cast<const double2*>(Vs + half + (j >> 1));
        v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
    } else if constexpr (VE == 2) {
        const double2 a = *reinterpret_cast<const double2*>(Vs + j);
        v[0] = a.x, v[1] = a.y;
    } else {
        v[0] = Vs[j];
    }
}

// acc[g] += sum_{j in [j0,j1)} P_row_g[j] * Vs[j], lane-strided over VE-vectors,
// in increasing j order per lane (fixed order -> reproducible).
template <typename PT, int VE, int NG, int U>
__device__ __forceinline__ void dot_rows(const PT* __restrict__ row0, int64_t n, int na, int64_t j0,
                                         int64_t j1, const double* Vs, int lane, double (&acc)[NG], int64_t half)
{
    using VT = typename Vec<PT, VE>::T;
    // single-row streams keep VE independent partial sums (one per vector
    // component) so the fp64 FMA chain per iteration is U long, not U*VE;
    // multi-row streams already interleave NG chains
    constexpr int NA = 1;  // (VE partial sums for single rows measured slower: register pressure)
    double part[NG][NA];
#pragma unroll
    for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int e = 0; e < NA; ++e) part[g][e] = 0.0;
    const int64_t nvec = (j1 - j0) / VE;  // j0, j1 multiples of VE
    const VT* rows[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) rows[g] = reinterpret_cast<const VT*>(row0 + (int64_t)g * n + j0);
    for (int64_t v = lane; v < nvec; v += kWarp * U) {
        VT x[U][NG];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vv = v + (int64_t)kWarp * u;
#pragma unroll
            for (int g = 0; g < NG; ++g)
                if (g < na && vv < nvec) x[u][g] = ld_stream(rows[g] + vv);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vv = v + (int64_t)kWarp * u;
            if (vv < nvec) {
                double vs[VE];
                load_v<VE>(Vs, j0 + vv * VE, vs, half);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (g < na) {
                        double p[VE];
                        Vec<PT, VE>::get(x[u][g], p);
#pragma unroll
                        for (int e = 0; e < VE; ++e) part[g][e % NA] = fma(p[e], vs[e], part[g][e % NA]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        double t = part[g][0];
        if constexpr (NA == 4) t = (part[g][0] + part[g][1]) + (part[g][2] + part[g][3]);
        if constexpr (NA == 2) t = part[g][0] + part[g][1];
        acc[g] += t;
    }
}

// pi may live in shared memory (copy) or in global memory (global-V path,
// written by other SMs between phases: read through L2, never a stale L1 line)
__device__ __forceinline__ int ld_pi(const int32_t* pis, int64_t s)
{
    return __isGlobal(pis) ? __ldcg(pis + s) : pis[s];
}

template <typename PT>
__device__ __forceinline__ double load_cost(const DenseArgs& a, int64_t idx)
{
    return (double)__ldg(static_cast<const PT*>(a.c) + idx);
}

// The last-arriving warp of state i reduces its partials (L2) into
// (lval[i], larg[i]).  F-mode: the (min, argmin) of the action groups in group
// order; S-mode: lane a sums action a's chunk partials in chunk order, then an
// argmin butterfly (lower value, then lower action).
template <typename PT, bool EVAL>
__device__ __forceinline__ void finish_state_warp(const DenseArgs& a, const double* part, int C, int64_t i, int64_t s,
                                                  int act_eval, int ng = kAG)
{
    const int lane = threadIdx.x & 31;
    if (C == 1) {  // F-mode, NAG > 1 groups
        if (lane == 0) {
            const int NAG = (a.A + ng - 1) / ng;
            const double2* pp = reinterpret_cast<const double2*>(part) + i * NAG;
            double best = 0.0;
            int barg = 0;
            for (int ag = 0; ag < NAG; ++ag) {
                const double2 q = __ldcg(pp + ag);
                if (ag == 0 || q.x < best) best = q.x, barg = (int)q.y;
            }
            a.lval[i] = best;
            a.larg[i] = barg;
        }
        return;
    }
    if (EVAL) {
        double sum = 0.0;
        for (int ch = lane; ch < C; ch += kWarp) sum += __ldcg(part + i * C + ch);
        sum = warp_sum(sum);
        if (lane == 0) {
            a.lval[i] = load_cost<PT>(a, s * a.A + act_eval) + a.gamma * sum;
            a.larg[i] = act_eval;
        }
        return;
    }
    double best = INFINITY;
    int barg = 0x7fffffff;
    for (int act = lane; act < a.A; act += kWarp) {
        const double* pp = part + (i * a.A + act) * C;
        double sum = 0.0;
        for (int c0 = 0; c0 < C; c0 += 8) {  // issue up to 8 loads, then add in chunk order
            double t[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) t[q] = c0 + q < C ? __ldcg(pp + c0 + q) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (c0 + q < C) sum += t[q];
        }
        const double Q = load_cost<PT>(a, s * a.A + act) + a.gamma * sum;
        if (barg == 0x7fffffff || Q < best) best = Q, barg = act;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, barg, o);
        if (ov < best || (ov == best && oa < barg) || (barg == 0x7fffffff && oa != 0x7fffffff)) {
            best = ov;
            barg = oa;
        }
    }
    if (lane == 0) {
        a.lval[i] = best;
        a.larg[i] = barg;
    }
}

// ------------------------------------------------------------ compute phase
// EVAL: rows (s, pi(s)); else rows (s, a) for all a in groups of kAG.
// states: perm[lo + i] (perm != null) or lo + i; i < cnt.
// Output layout (per batch position i):
//   C == 1, EVAL: part[i] = Q                  (per_state = 1)
//   C == 1, min : part[2(i*NAG+ag)+{0,1}] = (min Q over the group, argmin)   (2*NAG)
//   C >  1, EVAL: part[i*C + ch]               (C)
//   C >  1, min : part[(i*A + a)*C + ch]       (A*C)
// Item epilogue (warp-wide, acc[] identical in all lanes): write the item's
// result into the partial buffer and, in last-arriver mode, finish the state
// once all its items are in (shared by the warp and TMA compute paths).
template <typename PT, bool EVAL, int NG>
__device__ __forceinline__ void item_epilogue(const DenseArgs& a, const Plan& pl, double* part, int64_t i, int64_t s,
                                              int a0, int na, int ch, const double (&acc)[NG])
{
    const int lane = threadIdx.x & 31;
    const int C = pl.C;
    const int NAG = EVAL ? 1 : (a.A + NG - 1) / NG;
    const int64_t per_state = (int64_t)NAG * C;
    const int ag = a0 / NG;
    if (C == 1) {
        if (lane == 0) {
            if (EVAL) {
                part[i] = load_cost<PT>(a, s * a.A + a0) + a.gamma * acc[0];
            } else {
                double best = 0.0;
                int barg = a0;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (g < na) {
                        const double Q = load_cost<PT>(a, s * a.A + a0 + g) + a.gamma * acc[g];
                        if (g == 0 || Q < best) best = Q, barg = a0 + g;
                    }
                }
                part[2 * (i * NAG + ag)] = best;
                part[2 * (i * NAG + ag) + 1] = (double)barg;
            }
        }
    } else if (EVAL) {
        if (lane == 0) part[i * C + ch] = acc[0];
    } else {
#pragma unroll
        for (int g = 0; g < NG; ++g)
            if (lane == g && g < na) part[(i * a.A + a0 + g) * C + ch] = acc[g];
    }
    if (!pl.redundant) {
        // last arriver of state i finishes its backup into the list
        if (per_state == 1) {
            if (lane == 0) {
                if (EVAL) {
                    a.lval[i] = part[i];
                    a.larg[i] = a0;
                } else {
                    a.lval[i] = part[2 * i];
                    a.larg[i] = (int)part[2 * i + 1];
                }
            }
        } else {
            __syncwarp();
            unsigned int prev = 0;
            if (lane == 0) {
                __threadfence();
                prev = atomicAdd(a.scnt + i, 1u);
            }
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev == (unsigned int)(per_state - 1)) {
                __threadfence();
                finish_state_warp<PT, EVAL>(a, part, C, i, s, a0, NG);
                if (lane == 0) a.scnt[i] = 0u;  // rearmed for the next batch (ordered by its barrier)
            }
        }
    }
}


template <typename PT, int VE, bool EVAL, int NGT>
__device__ void compute_phase(const DenseArgs& a, const double* Vs, const int32_t* pis, const uint32_t* perm,
                              int64_t lo, int64_t cnt, const Plan& pl, double* part, unsigned int* ctr)
{
    const int lane = threadIdx.x & 31;
    const int C = pl.C;
    const int64_t Lc = pl.Lc;
    constexpr int NG = EVAL ? 1 : NGT;
    const int NAG = EVAL ? 1 : (a.A + NG - 1) / NG;
    const int64_t per_state = (int64_t)NAG * C;
    const int64_t items = cnt * per_state;
    const PT* P = static_cast<const PT*>(a.P);
    constexpr int U = NG == 1 ? 8 : 2;
    // dynamic work stealing over the whole grid (balances SMs whose HBM share
    // differs); the next item index is fetched while the current one streams
    // batches with at most one item per warp: a static deal (CTA-major, so
    // the items spread over all SMs) — 2368 warps grabbing from ONE counter at
    // the same instant serialise on that L2 address for several microseconds
    const int64_t W = (int64_t)a.nctas * kWarps;
    const bool stat = items <= W;
    int64_t static_it = (int64_t)(threadIdx.x >> 5) * a.nctas + cta_rank(a);
    auto grab = [&]() -> int64_t {
        if (stat) {
            const int64_t r = static_it;
            static_it = items;  // one item per warp
            return r;
        }
        unsigned int r = 0;
        if (lane == 0) r = atomicAdd(ctr, 1u);
        return (int64_t)__shfl_sync(0xffffffffu, r, 0);
    };
    // the next item is requested while this one streams (1 deep: a deeper
    // reservation turns the end of the batch into a static deal), and its
    // state id (a dependent L2 load) is looked up right after this item's
    // rows have streamed, overlapping the epilogue
    auto state_of = [&](int64_t t) -> int64_t {
        if (t >= items) return 0;
        const int64_t i = t / per_state;
        return perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
    };
    int64_t it = grab();
    int64_t s_cur = state_of(it);
    while (it < items) {
        const int64_t it_next = grab();
        const int64_t i = it / per_state;
        const int rr = (int)(it - i * per_state);
        const int ag = rr / C;
        const int ch = rr - ag * C;
        const int64_t s = s_cur;
        const int a0 = EVAL ? pis[s] : ag * NG;
        const int na = EVAL ? 1 : min(NG, a.A - a0);
        const int64_t j0 = (int64_t)ch * Lc;
        const int64_t j1 = min(a.n, j0 + Lc);
        double acc[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) acc[g] = 0.0;
        dot_rows<PT, VE, NG, U>(P + ((int64_t)s * a.A + a0) * a.n, a.n, na, j0, j1, Vs, lane, acc, a.vs_half);
        const int64_t s_next = state_of(it_next);
#pragma unroll
        for (int g = 0; g < NG; ++g) acc[g] = warp_sum(acc[g]);
        item_epilogue<PT, EVAL, NG>(a, pl, part, i, s, a0, na, ch, acc);
        it = it_next;
        s_cur = s_next;
    }
}

// ------------------------------------------------- TMA ring path (default)
// The compute phase as a bulk-copy pipeline.  Per SM, a PRODUCER warp (threads
// 512..543, one elected lane) takes items (state, action group, column chunk)
// from the batch's global work counter and streams each item's P rows into a
// shared-memory ring of 16 KB stages with cp.async.bulk (TMA engine, L2
// evict-first policy: P is read once per sweep), completion signalled on the
// stage's `full` mbarrier.  The 16 compute warps read a stage from shared
// memory (thread t: 16-byte vectors t and t + 512 of the stage), accumulate
// fp64 dot products against the shared-memory V across the item's stages and
// release the stage on its `empty` mbarrier.  At an item's last stage each
// warp reduces its sums into a per-stage slot; the last arriving warp adds the
// 32 slots in a fixed (half, warp) order — reproducible — and runs the item
// epilogue (the same as the warp path's).
//
// Why: the bytes in flight per SM are set by the ring (~100 KB), not by
// registers, and P does not depend on V — so the producer RUNS AHEAD into the
// next batch while the compute warps are still in this batch's tail, grid
// barrier and combine ("the batch is written back before the next batch
// starts" constrains the V reads, not the P loads).  The ring is full when
// the compute warps start the next batch.  Run-ahead is bounded to one batch,
// and fenced where a batch's rows depend on the previous batch's outcome (an
// evaluation sweep right after a policy improvement reads rows pi(s)).
// Work counters: a producer leaves a batch with exactly one failing grab; the
// one that draws items + grid - 1 (the last) re-arms the counter, before its
// end-of-batch marker, hence before that batch's grid barrier (2 counters).
constexpr int kTmaStage = 32768;           // bytes per ring stage
constexpr int kTmaMaxStages = 24;
constexpr int kTmaVecs = kTmaStage / 16;   // 16-byte vectors per stage
constexpr int kTmaThreads = kThreads + kWarp;
constexpr int kTmaCW = 16;                 // compute warps that consume the ring

struct TmaMeta {         // one per stage, written by the producer before its arrive
    long long i;         // batch position (END marker: batch sequence number)
    int e;               // first column of this stage's window
    int nvec;            // 16-byte vectors per row in this stage
    int a0;              // rows in the item (na)
    int na;              // action group index ag
    int ch;              // chunk of the group range
    int flags;           // 1: last stage of the item, 2: end of batch
};
constexpr int kTmaPerStageX = (int)sizeof(TmaMeta) + 16 + kWarps * kAG * 8 + 4;  // + the slot itself

struct TmaSmem {
    unsigned char* ring;
    TmaMeta* meta;
    unsigned long long* full;
    unsigned long long* empty;
    double* red;         // [stage][warp][2]
    int* redcnt;         // [stage]
    long long* ctl;      // [0] consumers' batch sequence number (-1 before the first), [1] stop flag
    int nst;
};

__device__ __forceinline__ TmaSmem tma_smem(unsigned char* base, const DenseArgs& a)
{
    TmaSmem m;
    m.nst = a.tma_nst;
    m.ring = base + a.tma_off;
    m.meta = reinterpret_cast<TmaMeta*>(m.ring + (size_t)m.nst * a.tma_slot);
    m.full = reinterpret_cast<unsigned long long*>(m.meta + m.nst);
    m.empty = m.full + m.nst;
    m.red = reinterpret_cast<double*>(m.empty + m.nst);
    m.redcnt = reinterpret_cast<int*>(m.red + (size_t)m.nst * kWarps * kAG);
    m.ctl = reinterpret_cast<long long*>(m.redcnt + ((m.nst + 1) & ~1));
    return m;
}

// The batch sequence of a launch, as the compute threads will run it (one
// entry per run_batch call), assuming no early stop.  Kinds as run_batch KIND.
struct TmaBatch {
    int kind;
    const uint32_t* perm;
    int64_t lo, cnt;
    const uint32_t* list;  // fused multi-rank sweep batches: this rank's (position, state) pairs
    const unsigned* lcnt;  //   and their number (final once the compute threads enter the batch)
};

__device__ __forceinline__ bool tma_segment(const DenseArgs& a, int64_t sg, int& kind, int64_t& k)
{
    k = a.k0;
    switch (a.mode) {
    case MODE_VI: kind = 0; k = a.k0 + sg; return sg < a.max_iter;
    case MODE_POLICY_VALUE: kind = 1; k = a.k0 + sg; return sg < a.max_iter;
    case MODE_APPLY: kind = 0; return sg < 1;
    case MODE_APPLY_PI: kind = 1; return sg < 1;
    case MODE_IMPROVE: case MODE_SHARD_IMPROVE: kind = 2; return sg < 1;
    case MODE_SHARD_MIN: kind = 3; return sg < 1;
    case MODE_SHARD_EVAL: kind = 4; return sg < 1;
    default: {  // MODE_MPI
        int64_t q = sg;
        if (!a.pi_given) {
            if (q == 0) { kind = 2; return true; }
            q -= 1;
        }
        const int64_t per = (int64_t)a.msweeps + 1;
        const int64_t outer = q / per, r = q - outer * per;
        if (outer >= a.max_iter) return false;
        if (r < a.msweeps) {
            kind = 1;
            k = a.k0 + outer * a.msweeps + r;
        } else {
            kind = 2;
        }
        return true;
    }
    }
}

struct TmaSched {
    int64_t sg = 0, lo = -1, k = 0;
    int64_t sb = 0;  // sweep batches so far (list slot sb % 3)
    int kind = -1;
    __device__ bool next(const DenseArgs& a, TmaBatch& bt)
    {
        while (true) {
            if (lo >= 0) {
                const int64_t end = kind == 2 ? a.row1 : (kind >= 3 ? 1 : a.n);
                if (lo < end) break;
                ++sg;
            }
            if (!tma_segment(a, sg, kind, k)) return false;
            lo = kind == 2 ? a.row0 : 0;
        }
        bt.kind = kind;
        bt.list = nullptr;
        bt.lcnt = nullptr;
        if (kind >= 3) {
            bt.perm = a.olist;
            bt.lo = 0;
            bt.cnt = *(volatile const int*)a.ocount;
            lo = 1;
        } else if (kind == 2) {
            bt.perm = nullptr;
            bt.lo = lo;
            bt.cnt = min(a.imp_sub, a.row1 - lo);
            lo += a.imp_sub;
        } else {
            bt.perm = a.identity ? nullptr : a.perm + (k % 3) * a.n;
            bt.lo = lo;
            bt.cnt = min(a.b, a.n - lo);
            lo += a.b;
            if (a.xG > 0) {
                bt.list = a.xlist + (sb % 3) * 2 * a.xlcap;
                bt.lcnt = a.xcnt + (sb % 3);
            }
            ++sb;
        }
        return true;
    }
};

// Producer: one lane.  q = batch sequence number (== the compute threads' x.phase).
// An ITEM is (state s, action group ag = rows a0 .. a0+na-1, column chunk ch)
// — or (s, row pi(s), ch) in B_{pi,b} batches.  It streams as stages of the
// same column window [col, col + w) of its na rows: na bulk copies per stage
// into na row slots of the ring slot, so a compute thread reads each V vector
// once for all the rows of the group.
template <typename PT>
__device__ void tma_producer(const DenseArgs& a, const int32_t* pis, const TmaSmem& m)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const PT* P = static_cast<const PT*>(a.P);
    constexpr int VB = 16 / (int)sizeof(PT);  // elements per 16-byte vector
    const int n = (int)a.n;
    int st = 0;
    unsigned ph = 0;
    long long issued = 0;
    bool stop = false;
    auto stopped = [&]() -> bool { return ld_acquire_cta(m.ctl + 1) != 0; };
    auto acquire = [&]() -> bool {
        SpinGuard sg;
        while (!mbar_try(m.empty + st, ph ^ 1u)) {
            if (stopped()) return false;
            sg.tick();
        }
        return true;
    };
    auto advance = [&]() {
        ++issued;
        if (++st == m.nst) st = 0, ph ^= 1u;
    };
    TmaSched sc;
    TmaBatch bt;
    int prev_kind = -1;
    const unsigned G = (unsigned)a.nctas;
    for (long long q = 0; !stop && sc.next(a, bt); ++q) {
        // run-ahead bound: one batch past the compute threads; fenced batches
        // (the first, and B_{pi,b} batches right after an improvement) wait
        // until the compute threads are in them
        const bool fence = q == 0 || ((bt.kind == 1 || bt.kind == 4) && prev_kind == 2) ||
                           (bt.perm != nullptr && bt.kind <= 1 && bt.lo == 0 && a.b >= a.n) ||
                           bt.list != nullptr;  // fused: the batch's list is built during the previous batch
        {
            SpinGuard sg;
            while (true) {
                const long long cq = ld_acquire_cta(m.ctl);
                if (q <= cq + (fence ? 0 : 1)) break;
                if (stopped()) { stop = true; break; }
                sg.tick();
                __nanosleep(64);
            }
        }
        if (stop) break;
        prev_kind = bt.kind;
        if (bt.list) bt.cnt = (int64_t)__ldcg(bt.lcnt);
        const bool eval = bt.kind == 1 || bt.kind == 4;
        const Plan& pl = a.plan[eval ? 1 : (bt.kind == 2 ? 2 : 0)];
        const int NG = eval ? 1 : pl.ng;
        const int rslot = kTmaStage / NG;                     // bytes per row slot
        const int w = rslot / (int)sizeof(PT);                // columns per stage
        const unsigned NAG = eval ? 1u : (unsigned)((a.A + NG - 1) / NG);
        const unsigned C = (unsigned)pl.C;
        const unsigned per_state = NAG * C;
        const unsigned items = (unsigned)bt.cnt * per_state;
        // small batches: a static deal (CTA x: items x, x + grid, ...), no
        // counter; else grabs of g items (>= ~4 stages) from the batch counter
        const bool stat = items <= (unsigned)a.tma_static * G;
        const unsigned spi = max(1u, (unsigned)(n / C / w));  // ~stages per item
        unsigned g = 1;
        if (!stat) g = max(1u, min((4u + spi - 1) / spi, max(1u, items / (4u * G))));
        unsigned int* ctr = a.wctr + (q & 1);
        // failing grabs return multiples of g from fail0 on; each producer does
        // exactly one, and the last of them re-arms the counter
        const unsigned fail0 = (items + g - 1) / g * g;
        unsigned r = stat ? (unsigned)cta_rank(a) : atomicAdd(ctr, g);
        unsigned r_end = stat ? r + 1 : r + g;
        const unsigned nvecs = (unsigned)(n / VB);
        while (true) {
            if (r >= items) {
                if (!stat && r == fail0 + (G - 1) * g) atomicExch(ctr, 0u);
                break;
            }
            // next grab, in flight while this one streams
            const bool local = !stat && r + 1 < r_end && r + 1 < items;
            const unsigned rn = stat ? r + G : (local ? r + 1 : atomicAdd(ctr, g));
            const unsigned j = r / per_state;
            const unsigned rr = r - j * per_state;
            const unsigned ag = rr / C;
            const unsigned ch = rr - ag * C;
            // batch position i and state s of list entry j
            unsigned i = j;
            int64_t s;
            if (bt.list) {
                i = __ldcg(bt.list + 2 * j);
                s = (int64_t)__ldcg(bt.list + 2 * j + 1);
            } else {
                s = bt.perm ? (int64_t)__ldcg(bt.perm + bt.lo + j) : bt.lo + j;
            }
            const int a0 = eval ? ld_pi(pis, s) : (int)ag * NG;
            const int na = eval ? 1 : min(NG, a.A - a0);
            // columns [c0, c1) (vector aligned) of the group's rows
            const int c1 = (int)((uint64_t)nvecs * (ch + 1) / C) * VB;
            const PT* rowp = P + ((int64_t)s * a.A + a0) * n;
            const int c0 = (int)((uint64_t)nvecs * ch / C) * VB;
            for (int col = c0; col < c1 && !stop; col += w) {
                const int len = min(w, c1 - col);
                if (!acquire()) { stop = true; break; }
                TmaMeta& md = m.meta[st];
                md.i = i;
                md.e = col;
                md.nvec = len / VB;
                md.a0 = na;
                md.na = (int)ag;
                md.ch = (int)ch;
                md.flags = col + len >= c1 ? 1 : 0;
                const unsigned bytes = (unsigned)(len * (int)sizeof(PT));
                mbar_arrive_tx(m.full + st, bytes * (unsigned)na);
                unsigned char* dst = m.ring + (size_t)st * kTmaStage;
                const PT* src = rowp + col;
                for (int gg = 0; gg < na; ++gg) {
                    bulk_g2s(dst, src, bytes, m.full + st, pol);
                    dst += rslot;
                    src += n;
                }
                advance();
            }
            if (stop) break;
            if (!stat && !local) r_end = rn + g;
            r = rn;
        }
        if (stop) break;
        if (!acquire()) break;
        m.meta[st].i = q;
        m.meta[st].flags = 2;
        mbar_arrive(m.full + st);
        advance();
    }
    // drain: every issued bulk copy must land before the CTA may exit
    const long long last = issued < m.nst ? issued : m.nst;
    int s2 = st;
    unsigned p2 = ph;
    for (long long d = 0; d < last; ++d) {
        if (s2 == 0) s2 = m.nst, p2 ^= 1u;
        --s2;
        SpinGuard sg;
        while (!mbar_try(m.full + s2, p2)) sg.tick();
    }
}

// Compute threads: consume this batch's stages up to its end marker.  A stage
// holds the column window [col, col + 4*nvec) of the item's na rows (row g at
// slot offset g * kTmaStage/NG); thread t takes column vectors t, t + 512, ...
// and, per vector, reads V once and dots it with every row.  Raw partials:
//   part[((i*NAG + ag)*C + ch)*NG + g] = sum over the item of P(row a0+g) . V
template <int VE>
__device__ __forceinline__ void load_v_global(const double* V, int64_t j, double (&v)[VE])
{
#pragma unroll
    for (int q = 0; q < VE; q += 2) {
        const double2 x = __ldcg(reinterpret_cast<const double2*>(V + j + q));
        v[q] = x.x, v[q + 1] = x.y;
    }
}

template <typename PT, bool EVAL, bool VGL = false>
__device__ void compute_phase_tma(const DenseArgs& a, const double* Vs, const Plan& pl, double* part,
                                  const TmaSmem& m, int& st, unsigned& ph)
{
    constexpr int E = 16 / (int)sizeof(PT);
    constexpr int NG = EVAL ? 1 : kAG;
    constexpr int RV = kTmaStage / NG / 16;  // vectors per row slot
    using VT = typename Vec<PT, E>::T;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (warp >= kTmaCW) return;  // fewer, fuller consumer warps: less issue overhead per byte
    const int NAG = EVAL ? 1 : (a.A + NG - 1) / NG;
    const int C = pl.C;
    const int64_t half = a.vs_half;
    double acc[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) acc[g] = 0.0;
    while (true) {
        {
            SpinGuard sg;
            while (!mbar_try(m.full + st, ph)) sg.tick();
        }
        const TmaMeta md = m.meta[st];
        if (md.flags & 2) {
            __syncwarp();
            if (lane == 0) mbar_arrive(m.empty + st);
            if (++st == m.nst) st = 0, ph ^= 1u;
            break;
        }
        const VT* stg = reinterpret_cast<const VT*>(m.ring + (size_t)st * kTmaStage);
        {
#pragma unroll
            for (int f0 = 0; f0 < RV; f0 += kTmaCW * kWarp) {
                const int f = f0 + t;
                if (f < md.nvec) {
                    double vs[E];
                    if constexpr (VGL) load_v_global<E>(Vs, md.e + f * E, vs);
                    else load_v<E>(Vs, md.e + f * E, vs, half);
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        if (g < md.a0) {
                            const VT x = stg[g * RV + f];
                            double p[E];
                            Vec<PT, E>::get(x, p);
#pragma unroll
                            for (int k = 0; k < E; ++k) acc[g] = fma(p[k], vs[k], acc[g]);
                        }
                    }
                }
            }
        }
        if (md.flags & 1) {
            double* red = m.red + (size_t)st * kTmaCW * kAG;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const double w = warp_sum(acc[g]);
                acc[g] = 0.0;
                if (lane == 0) red[warp * kAG + g] = w;
            }
            // arrival count with acq_rel semantics at CTA scope
            int prev = 0;
            if (lane == 0) {
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(prev)
                             : "r"(smem_addr(m.redcnt + st))
                             : "memory");
            }
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev == kTmaCW - 1) {
                // lane g < NG sums row g over the warps in order; plain stores,
                // no global round trip on the streaming warps (costs, chunk
                // sums and the min are the combine's); rows >= na store 0
                if (lane < NG) {
                    double dsum = 0.0;
                    for (int w = 0; w < kTmaCW; ++w) dsum += red[w * kAG + lane];
                    part[(((int64_t)md.i * NAG + md.na) * C + md.ch) * NG + lane] = dsum;
                }
                if (lane == 0) m.redcnt[st] = 0;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(m.empty + st);
        if (++st == m.nst) st = 0, ph ^= 1u;
    }
}

struct PhaseAcc {
    double rmax;
    int bad;
    long long changed;
};

// ------------------------------------------------- per-state reductions
// F-mode (C == 1): one thread per state.
template <bool EVAL>
__device__ __forceinline__ void reduce_state_F(const DenseArgs& a, const double* part, int64_t i, double& best,
                                               int& barg, int ng)
{
    if (EVAL) {
        best = __ldcg(part + i);
        barg = -1;
        return;
    }
    const int NAG = (a.A + ng - 1) / ng;
    const double2* pp = reinterpret_cast<const double2*>(part) + i * NAG;
    best = 0.0;
    barg = 0;
    for (int ag = 0; ag < NAG; ++ag) {
        const double2 q = __ldcg(pp + ag);
        if (ag == 0 || q.x < best) best = q.x, barg = (int)q.y;
    }
}

// S-mode (C > 1): the CTA reduces the states i = first + k*step (k < m):
// warp per (state, action) sums its C partials (lane-strided, then a fixed
// butterfly), Q = c + gamma*sum goes to smem Qs, then a thread per state takes
// the argmin over actions in index order (lowest index on ties).  sink(i, s,
// v, arg) is called by exactly one thread per state.
// olist != null (fused multi-rank batches): the entries are this rank's
// states of the batch, olist[2j] = batch position, olist[2j+1] = state, and
// cnt is their number.
template <typename PT, bool EVAL, typename Sink>
__device__ __forceinline__ void reduce_states_S(const DenseArgs& a, const double* part, int C, const uint32_t* perm,
                                                int64_t lo, int64_t cnt, int64_t first, int64_t step,
                                                const int32_t* pis, double* Qs, Sink&& sink, bool raw = false,
                                                const uint32_t* olist = nullptr)
{
    auto pos_state = [&](int64_t j, int64_t& i, int64_t& s) {
        if (olist) {
            i = (int64_t)__ldcg(olist + 2 * j);
            s = (int64_t)__ldcg(olist + 2 * j + 1);
        } else {
            i = j;
            s = perm ? (int64_t)__ldcg(perm + lo + j) : lo + j;
        }
    };
    // partial layout: (i, a, ch) -> (i*A + a)*C + ch, stride 1 over ch; raw
    // (TMA path, min modes): ((i*NAG + a/kAG)*C + ch)*kAG + a%kAG, stride kAG
    const int NAGr = (a.A + kAG - 1) / kAG;
    auto pbase = [&](int64_t i, int act) -> int64_t {
        if (EVAL) return i * C;
        return raw ? ((i * NAGr + act / kAG) * C) * kAG + act % kAG : (i * a.A + act) * C;
    };
    const int pstr = (raw && !EVAL) ? kAG : 1;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int Ae = EVAL ? 1 : a.A;
    if (first >= cnt) return;
    const int64_t m_all = (cnt - first + step - 1) / step;
    const int64_t per_round = max((int64_t)1, a.qs_cap / Ae);
    for (int64_t k0 = 0; k0 < m_all; k0 += per_round) {
        const int64_t m = min(per_round, m_all - k0);
        if (C <= 8) {  // many short sums: a thread per (state, action), chunk order
            for (int64_t q = threadIdx.x; q < m * Ae; q += kThreads) {
                const int64_t kk = q / Ae;
                const int ai = (int)(q - kk * Ae);
                int64_t i, s;
                pos_state(first + (k0 + kk) * step, i, s);
                const int act = EVAL ? ld_pi(pis, s) : ai;
                const double* pp = part + pbase(i, act);
                double sum = 0.0;
                for (int ch = 0; ch < C; ++ch) sum += __ldcg(pp + (int64_t)ch * pstr);
                Qs[q] = load_cost<PT>(a, s * a.A + act) + a.gamma * sum;
            }
        } else {       // few long sums: a warp per (state, action)
            for (int64_t q = warp; q < m * Ae; q += kWarps) {
                const int64_t kk = q / Ae;
                const int ai = (int)(q - kk * Ae);
                int64_t i, s;
                pos_state(first + (k0 + kk) * step, i, s);
                const int act = EVAL ? ld_pi(pis, s) : ai;
                const double* pp = part + pbase(i, act);
                double sum = 0.0;
                for (int ch = lane; ch < C; ch += kWarp) sum += __ldcg(pp + (int64_t)ch * pstr);
                sum = warp_sum(sum);
                if (lane == 0) Qs[q] = load_cost<PT>(a, s * a.A + act) + a.gamma * sum;
            }
        }
        csync();
        for (int64_t kk = threadIdx.x; kk < m; kk += kThreads) {
            int64_t i, s;
            pos_state(first + (k0 + kk) * step, i, s);
            double best = Qs[kk * Ae];
            int barg = EVAL ? ld_pi(pis, s) : 0;
            if (!EVAL)
                for (int act = 1; act < a.A; ++act) {
                    const double Q = Qs[kk * Ae + act];
                    if (Q < best) best = Q, barg = act;
                }
            sink(i, s, best, barg);
        }
        csync();
    }
}

// Apply a state's new value to this CTA's smem copy (KIND 0: B_b, 1: B_pi,b,
// 2: improvement).  CTA 0 also writes the global outputs.
// KIND 3 / 4 (shard B_b / B_pi,b): the new value goes to this rank's send list
// (position i) instead of the local V; the exchange + commit apply it.
template <int KIND, bool VGL = false>
__device__ __forceinline__ void patch_state(const DenseArgs& a, double* Vs, int32_t* pis, int64_t i, int64_t s, double v,
                                            int arg, PhaseAcc& acc)
{
    if (VGL) {
        // global V / pi: every state is patched by exactly one CTA (distributed
        // combine) and the residual / changed counts are reduced over the grid
        acc.bad |= !isfinite(v);
        if (KIND == 0 && a.vnext) {  // chunked T: V stays at the sweep-start values
            acc.rmax = fmax(acc.rmax, fabs(v - __ldcg(a.V + s)));
            a.vnext[s] = v;
            if (a.pi) a.pi[s] = arg;
        } else if (KIND >= 3) {
            a.send_val[i] = v;
            a.send_idx[i] = (uint32_t)s;
            a.send_arg[i] = arg;
        } else if (KIND == 2) {
            const double old = __ldcg(a.V + s);
            acc.rmax = fmax(acc.rmax, fabs(v - old));
            acc.changed += (arg != __ldcg(a.pi + s));
            a.pi[s] = arg;
        } else {
            const double old = __ldcg(a.V + s);
            acc.rmax = fmax(acc.rmax, fabs(v - old));
            a.V[s] = v;
            if (KIND == 0 && a.pi) a.pi[s] = arg;
        }
        return;
    }
    if (KIND >= 3) {
        acc.bad |= !isfinite(v);
        if (cta_rank(a) == 0) {
            a.send_val[i] = v;
            a.send_idx[i] = (uint32_t)s;
            a.send_arg[i] = arg;
        }
        return;
    }
    const int64_t vi = vs_index(s, a.vs_half);
    const double old = Vs[vi];
    acc.rmax = fmax(acc.rmax, fabs(v - old));
    acc.bad |= !isfinite(v);
    const bool writer = cta_rank(a) == 0;
    if (KIND == 0 && a.vnext) {  // chunked T (VI*): the smem V keeps the sweep-start values
        if (writer) {
            a.vnext[s] = v;
            if (a.pi) a.pi[s] = arg;
        }
    } else if (KIND == 2) {
        acc.changed += (arg != pis[s]);
        pis[s] = arg;
        if (writer) a.pi[s] = arg;
    } else {
        Vs[vi] = v;
        if (writer) {
            a.V[s] = v;
            if (KIND == 0 && a.pi) a.pi[s] = arg;
        }
    }
}

struct Ctx {
    GridBarrier g;
    long long phase;  // running compute/combine phase counter (partial buffer parity)
    int64_t batches;
    unsigned long long t_mark;
    long long t_comp, t_bar, t_comb, n_bar;
    TmaSmem tm;       // TMA path: ring and the compute threads' position in it
    int tst;
    unsigned tph;
    long long gred_seq;  // global-V path: grid reductions so far (ring slot)
    unsigned long long xepoch;  // fused multi-rank: cross-rank barriers so far in this launch
    long long nimp;             //                   improvements so far (record parity)
    bool cta0;                  // this is CTA 0 of its rank (phase profile)
};

__device__ __forceinline__ void prof_mark(Ctx& x, long long* slot)
{
    if (x.cta0 && threadIdx.x == 0) {
        const unsigned long long t = globaltimer_ns();
        *slot += (long long)(t - x.t_mark);
        x.t_mark = t;
    }
}

__device__ __forceinline__ void timed_sync(Ctx& x)
{
    prof_mark(x, &x.t_comp);
    grid_sync<kThreads>(x.g);
    prof_mark(x, &x.t_bar);
    x.n_bar++;
}

// ------------------------------------------- fused multi-rank exchange (K8f)
__device__ __forceinline__ void red_release_add_sys(unsigned long long* p, unsigned long long v)
{
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <typename F>
__device__ __forceinline__ void spin_until(F&& done, const DenseArgs& a)
{
    unsigned spins = 0;
    unsigned long long t0 = 0;
    while (!done()) {
        if (++spins == 4096u) {
            spins = 0;
            const unsigned long long t = globaltimer_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 30ull * 1000000000ull) {  // a rank is gone: fail loudly, do not wedge the GPU
                atomicExch(a.err, 2);
                __trap();
            }
        }
    }
}

// Cross-rank barrier: every CTA of every rank.  The CTAs of a rank arrive on a
// local counter (after a system-scope fence: their peer stores are visible to
// every rank first); the rank's leader (CTA 0) signals every rank's arrival
// counter, waits for all G signals of this epoch on its own, and releases its
// CTAs.  Counters are monotonic across launches (a.xbase), so no rank ever
// needs to reset a counter another rank may already be signalling.
__device__ void xrank_sync(const DenseArgs& a, Ctx& x)
{
    prof_mark(x, &x.t_comp);
    csync();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned long long e = ++x.xepoch;
        red_release_add(a.xloc, 1ull);
        if (cta_rank(a) == 0) {
            const unsigned long long local = e * (unsigned long long)a.nctas;
            spin_until([&] { return ld_acquire_gpu(a.xloc) >= local; }, a);
            __threadfence_system();
#pragma unroll
            for (int r = 0; r < kMaxRanks; ++r)
                if (r < a.xG) red_release_add_sys(a.xbar[r], 1ull);
            const unsigned long long all = (a.xbase + e) * (unsigned long long)a.xG;
            spin_until([&] { return ld_acquire_sys(a.xbar_own) >= all; }, a);
            st_release_gpu(a.xrel, e);
        } else {
            spin_until([&] { return ld_acquire_gpu(a.xrel) >= e; }, a);
        }
    }
    csync();
    prof_mark(x, &x.t_bar);
    x.n_bar++;
}

// This rank's states of the sweep batch with sequence number sb (positions
// [lo, lo + cnt) of perm, or lo + i for the identity order) into list slot
// sb % 3 as (position, state) pairs.  Order-free (no state's arithmetic
// depends on the list order).  Run by all compute threads of the rank.
__device__ void build_own_list(const DenseArgs& a, const uint32_t* perm, int64_t lo, int64_t cnt, int64_t sb)
{
    uint32_t* list = a.xlist + (sb % 3) * 2 * a.xlcap;
    unsigned int* count = a.xcnt + (sb % 3);
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)a.nctas * kThreads;
    for (int64_t i0 = (int64_t)cta_rank(a) * kThreads; i0 < cnt; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        int64_t s = -1;
        if (i < cnt) s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
        const bool own = i < cnt && s >= a.row0 && s < a.row1;
        const unsigned m = __ballot_sync(0xffffffffu, own);
        unsigned base = 0;
        if (lane == 0 && m) base = atomicAdd(count, (unsigned)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (own) {
            const unsigned k = base + __popc(m & ((1u << lane) - 1u));
            list[2 * k] = (uint32_t)i;
            list[2 * k + 1] = (uint32_t)s;
        }
    }
}

// Fused improvement: this rank's (residual, changed, bad) to every rank, then
// every rank reduces all G records (the improvement covers owned states only).
__device__ PhaseAcc xrank_reduce(const DenseArgs& a, Ctx& x, PhaseAcc r)
{
    const int par = (int)(x.nimp++ & 1);
    if (cta_rank(a) == 0 && threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < kMaxRanks; ++q) {
            if (q < a.xG) {
                unsigned long long* rec = a.ximp[q] + ((size_t)par * kMaxRanks + a.xrank) * 4;
                rec[0] = (unsigned long long)__double_as_longlong(r.rmax);
                rec[1] = (unsigned long long)r.changed;
                rec[2] = (unsigned long long)r.bad;
            }
        }
    }
    xrank_sync(a, x);
    PhaseAcc g{0.0, 0, 0};
    const unsigned long long* mine = a.ximp_own + (size_t)par * kMaxRanks * 4;
    for (int q = 0; q < a.xG; ++q) {
        g.rmax = fmax(g.rmax, __longlong_as_double((long long)__ldcg(mine + 4 * q)));
        g.changed += (long long)__ldcg(mine + 4 * q + 1);
        g.bad |= (int)__ldcg(mine + 4 * q + 2);
    }
    return g;
}


// Fast redundant combine (TMA path, small batches): L = pow2 >= Ae lanes per
// state, thread t serves action t % L of the states t / L + k * (512 / L).  The
// state ids and costs (independent of V) are loaded BEFORE the grid barrier;
// after it, the chunk partials are summed and the argmin (lower value, then
// lower action) is a shuffle butterfly inside the L lanes: no smem scratch,
// no CTA barrier, one L2 round trip after the grid barrier.
constexpr int kFastK = 2;  // rounds per thread (states per batch <= kFastK * 512 / L)
struct FastPre {
    int s[kFastK];  // state id (< 2^31), -1 = idle lane
    int act[kFastK];
    double cost[kFastK];
};
__device__ __forceinline__ int fast_lanes(int Ae) { return Ae <= 1 ? 1 : 1 << (32 - __clz(Ae - 1)); }

template <typename PT, bool EVAL>
__device__ __forceinline__ void fast_pre(const DenseArgs& a, const uint32_t* perm, int64_t lo, int64_t cnt,
                                         const int32_t* pis, int L, FastPre& fp)
{
    const int Ae = EVAL ? 1 : a.A;
    const int t = threadIdx.x;
    const int per_round = kThreads / L;
#pragma unroll
    for (int k = 0; k < kFastK; ++k) {
        const int64_t kk = (int64_t)k * per_round + t / L;
        const int act = t % L;
        fp.s[k] = -1;
        fp.act[k] = act;
        fp.cost[k] = 0.0;
        if (kk < cnt && act < Ae) {
            const int64_t s = perm ? (int64_t)__ldcg(perm + lo + kk) : lo + kk;
            fp.s[k] = (int)s;
            const int ac = EVAL ? ld_pi(pis, s) : act;
            fp.act[k] = ac;
            fp.cost[k] = load_cost<PT>(a, s * a.A + ac);
        }
    }
}

template <int L>
__device__ __forceinline__ void fast_argmin(double& v, int& arg)
{
    if constexpr (L > 1) group_argmin<L>(v, arg);
}

template <typename PT, int KIND>
__device__ __forceinline__ void fast_finish(const DenseArgs& a, double* Vs, int32_t* pis, const double* part,
                                            int C, int64_t cnt, int L, const FastPre& fp, PhaseAcc& acc)
{
    constexpr bool EVAL = KIND == 1 || KIND == 4;
    const int t = threadIdx.x;
    const int per_round = kThreads / L;
    const int NAGr = (a.A + kAG - 1) / kAG;
#pragma unroll
    for (int k = 0; k < kFastK; ++k) {
        const int64_t kk = (int64_t)k * per_round + t / L;
        if (k * per_round >= cnt) break;  // uniform
        double v = INFINITY;
        int arg = 0x7fffffff;
        if (fp.s[k] >= 0) {
            const int act = fp.act[k];
            const double* pp = part + (EVAL ? kk * C : ((kk * NAGr + act / kAG) * C) * kAG + act % kAG);
            const int pstr = EVAL ? 1 : kAG;
            double sum = 0.0;
            for (int c0 = 0; c0 < C; c0 += 4) {  // 4 loads in flight, added in chunk order
                double tv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) tv[q] = c0 + q < C ? __ldcg(pp + (int64_t)(c0 + q) * pstr) : 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (c0 + q < C) sum += tv[q];
            }
            v = fp.cost[k] + a.gamma * sum;
            arg = act;
        }
        switch (L) {
        case 2: fast_argmin<2>(v, arg); break;
        case 4: fast_argmin<4>(v, arg); break;
        case 8: fast_argmin<8>(v, arg); break;
        case 16: fast_argmin<16>(v, arg); break;
        case 32: fast_argmin<32>(v, arg); break;
        default: break;
        }
        if (t % L == 0 && fp.s[k] >= 0) patch_state<KIND>(a, Vs, pis, kk, (int64_t)fp.s[k], v, arg, acc);
    }
}

// One batch (or improvement sub-batch): compute -> barrier -> combine/patch.
// Fused multi-rank sweeps (a.xG > 0): (perm_next, lo_next, cnt_next) is the
// next sweep batch, whose list of this rank's states is built now.
template <typename PT, int VE, int KIND, int CTA>
__device__ void run_batch(const DenseArgs& a, Ctx& x, double* Vs, int32_t* pis, const uint32_t* perm, int64_t lo,
                          int64_t cnt, const Plan& pl, PhaseAcc& acc, double* Qs, int64_t fill_next_k,
                          const uint32_t* perm_next = nullptr, int64_t lo_next = 0, int64_t cnt_next = 0)
{
    constexpr bool EVAL = KIND == 1 || KIND == 4;
    double* part = a.part + (x.phase & 1) * a.part_stride;
    if constexpr (is_tma(CTA)) {
        // the producer may now run one batch ahead of this one (counters are
        // re-armed by the producers themselves)
        if (threadIdx.x == 0) st_release_cta(x.tm.ctl, x.phase);
    } else if (cta_rank(a) == 0 && threadIdx.x == 0) {
        // the other parity's work counter was last used before the previous
        // barrier: CTA 0 rearms it for the next phase (ordered by this phase's barrier)
        atomicExch(a.wctr + ((x.phase + 1) & 1), 0u);
    }
    // one compute path per kernel instantiation (register allocation is per
    // kernel: mixing paths made every path spill)
    if constexpr (is_tma(CTA))
        compute_phase_tma<PT, EVAL, is_vgl(CTA)>(a, Vs, pl, part, x.tm, x.tst, x.tph);
    else
        compute_phase<PT, VE, EVAL, kAG>(a, Vs, pis, perm, lo, cnt, pl, part, a.wctr + (x.phase & 1));
    if (fill_next_k > 0)  // next sweep's order, off the critical path
        fill_order(a.n, a.seed, fill_next_k, a.order, a.perm + (fill_next_k % 3) * a.n,
                   (int64_t)cta_rank(a) * kThreads + threadIdx.x, (int64_t)a.nctas * kThreads);
    constexpr bool fused = is_fused(CTA) && KIND <= 1;
    if constexpr (fused) {
        if (cta_rank(a) == 0 && threadIdx.x == 0) a.xcnt[(x.batches + 2) % 3] = 0u;  // slot of batch sb - 1
        if (cnt_next > 0) build_own_list(a, perm_next, lo_next, cnt_next, x.batches + 1);
    }
    constexpr int AeK = EVAL ? 1 : 0;
    const int Ae = AeK ? 1 : a.A;
    const int L = fast_lanes(Ae);
    // decided from the plan's batch size, not cnt (a shard step's cnt is its
    // share): the same states take the same summation order for any G
    const int64_t plan_cnt = KIND == 2 ? a.imp_sub : a.b;
    const bool fast = CTA == kPathTma && pl.raw && pl.redundant && pl.C <= 4 && L <= 32 &&
                      plan_cnt * L <= (int64_t)kFastK * kThreads && !fused;
    FastPre fp;
    if (fast) fast_pre<PT, EVAL>(a, perm, lo, cnt, pis, L, fp);
    timed_sync(x);
    const bool F = pl.C == 1 && !pl.raw;
    auto patch = [&](int64_t i, int64_t s, double v, int arg) { patch_state<KIND>(a, Vs, pis, i, s, v, arg, acc); };
    if constexpr (fused) {
        // CTA x finishes this rank's states x, x + grid, ... of the batch and
        // stores (value, argmin) at their batch positions into every rank's
        // exchange arrays; after the cross-rank barrier every rank patches all
        // of the batch from its own arrays (Eq. 12: no state of the batch is
        // patched before every read of the batch is done, on every rank)
        const int64_t sb = x.batches;
        const uint32_t* ol = a.xlist + (sb % 3) * 2 * a.xlcap;
        const int64_t own = (int64_t)__ldcg(a.xcnt + (sb % 3));
        const size_t par = (size_t)(sb & 1) * (size_t)a.xlcap;
        reduce_states_S<PT, EVAL>(
            a, part, pl.C, nullptr, 0, own, cta_rank(a), a.nctas, pis, Qs,
            [&](int64_t i, int64_t s, double v, int arg) {
                (void)s;
#pragma unroll
                for (int r = 0; r < kMaxRanks; ++r) {
                    if (r < a.xG) {
                        a.xval[r][par + i] = v;
                        a.xarg[r][par + i] = arg;
                    }
                }
            },
            true, ol);
        xrank_sync(a, x);
        const double* xv = a.xval_own + par;
        const int32_t* xa = a.xarg_own + par;
        if constexpr (is_vgl(CTA)) {
            const int64_t stride = (int64_t)a.nctas * kThreads;
            for (int64_t i = (int64_t)cta_rank(a) * kThreads + threadIdx.x; i < cnt; i += stride) {
                const int64_t s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
                patch_state<KIND, true>(a, Vs, pis, i, s, __ldcg(xv + i), __ldcg(xa + i), acc);
            }
            timed_sync(x);
        } else {
            for (int64_t i = threadIdx.x; i < cnt; i += kThreads) {
                const int64_t s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
                patch_state<KIND>(a, Vs, pis, i, s, __ldcg(xv + i), __ldcg(xa + i), acc);
            }
        }
    } else if constexpr (is_vgl(CTA)) {
        // global V: CTA x finishes and writes the states x, x + grid, ...; a
        // second barrier makes the batch visible before the next batch reads
        reduce_states_S<PT, EVAL>(
            a, part, pl.C, perm, lo, cnt, cta_rank(a), a.nctas, pis, Qs,
            [&](int64_t i, int64_t s, double v, int arg) { patch_state<KIND, true>(a, Vs, pis, i, s, v, arg, acc); },
            true);
        timed_sync(x);
    } else if (fast) {
        fast_finish<PT, KIND>(a, Vs, pis, part, pl.C, cnt, L, fp, acc);
    } else if (pl.raw && !pl.redundant) {
        // distributed combine: CTA x finishes the states x, x + grid, ... into
        // the list, a second grid barrier, then every CTA patches from it
        reduce_states_S<PT, EVAL>(a, part, pl.C, perm, lo, cnt, cta_rank(a), a.nctas, pis, Qs,
                                  [&](int64_t i, int64_t s, double v, int arg) {
                                      (void)s;
                                      a.lval[i] = v;
                                      a.larg[i] = arg;
                                  },
                                  true);
        timed_sync(x);
        for (int64_t i = threadIdx.x; i < cnt; i += kThreads) {
            const int64_t s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
            patch_state<KIND>(a, Vs, pis, i, s, __ldcg(a.lval + i), __ldcg(a.larg + i), acc);
        }
    } else if (pl.redundant) {
        if (F) {
            for (int64_t i = threadIdx.x; i < cnt; i += kThreads) {
                const int64_t s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
                double v;
                int arg;
                reduce_state_F<EVAL>(a, part, i, v, arg, pl.ng);
                patch_state<KIND>(a, Vs, pis, i, s, v, arg, acc);
            }
        } else {
            reduce_states_S<PT, EVAL>(a, part, pl.C, perm, lo, cnt, 0, 1, pis, Qs, patch, pl.raw != 0);
        }
    } else {
        // last-arriver mode: the list was completed during the compute phase
        for (int64_t i = threadIdx.x; i < cnt; i += kThreads) {
            const int64_t s = perm ? (int64_t)__ldcg(perm + lo + i) : lo + i;
            patch_state<KIND>(a, Vs, pis, i, s, __ldcg(a.lval + i), __ldcg(a.larg + i), acc);
        }
    }
    csync();
    prof_mark(x, &x.t_comb);
    ++x.phase;
}

// block-wide reduction of a PhaseAcc; every thread receives the result
__device__ PhaseAcc block_reduce(PhaseAcc v)
{
    __shared__ double sd[kWarps];
    __shared__ int si[kWarps];
    __shared__ long long sl[kWarps];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.rmax = fmax(v.rmax, __shfl_xor_sync(0xffffffffu, v.rmax, o));
        v.bad |= __shfl_xor_sync(0xffffffffu, v.bad, o);
        v.changed += __shfl_xor_sync(0xffffffffu, v.changed, o);
    }
    const int w = threadIdx.x >> 5;
    csync();
    if ((threadIdx.x & 31) == 0) sd[w] = v.rmax, si[w] = v.bad, sl[w] = v.changed;
    csync();
    PhaseAcc r{0.0, 0, 0};
    for (int k = 0; k < kWarps; ++k) r.rmax = fmax(r.rmax, sd[k]), r.bad |= si[k], r.changed += sl[k];
    csync();
    return r;
}

// Grid-wide reduction of a PhaseAcc (global-V path, where each CTA saw only
// its share of the states): CTA partials -> atomics on a ring slot -> barrier.
__device__ PhaseAcc grid_reduce(const DenseArgs& a, Ctx& x, PhaseAcc v)
{
    PhaseAcc r = block_reduce(v);
    unsigned long long* slot = a.gred + 4 * (x.gred_seq & 3);
    if (cta_rank(a) == 0 && threadIdx.x == 0) {  // re-arm the slot used two reductions ahead
        unsigned long long* z = a.gred + 4 * ((x.gred_seq + 2) & 3);
        atomicExch(z, 0ull);
        atomicExch(z + 1, 0ull);
        atomicExch(z + 2, 0ull);
    }
    if (threadIdx.x == 0) {
        atomicMax(slot, (unsigned long long)__double_as_longlong(r.rmax));  // rmax >= 0: bits order = value order
        if (r.bad) atomicOr(slot + 1, 1ull);
        if (r.changed) atomicAdd(slot + 2, (unsigned long long)r.changed);
    }
    timed_sync(x);
    PhaseAcc g;
    g.rmax = __longlong_as_double((long long)ld_acquire_gpu(slot));
    g.bad = ld_acquire_gpu(slot + 1) != 0;
    g.changed = (long long)ld_acquire_gpu(slot + 2);
    ++x.gred_seq;
    return g;
}

template <int CTA>
__device__ __forceinline__ PhaseAcc phase_reduce(const DenseArgs& a, Ctx& x, PhaseAcc v)
{
    if constexpr (is_vgl(CTA)) return grid_reduce(a, x, v);
    else return block_reduce(v);
}

// One application of B_b (EVAL = false) or B_{pi,b} (EVAL = true), sweep k.
template <typename PT, int VE, bool EVAL, int CTA>
__device__ PhaseAcc run_sweep(const DenseArgs& a, Ctx& x, double* Vs, int32_t* pis, int64_t k, double* Qs)
{
    const uint32_t* perm = a.identity ? nullptr : a.perm + (k % 3) * a.n;
    const Plan& pl = a.plan[EVAL ? 1 : 0];
    PhaseAcc acc{0.0, 0, 0};
    for (int64_t lo = 0; lo < a.n; lo += a.b) {
        const int64_t cnt = min(a.b, a.n - lo);
        // the next sweep batch: later in this sweep, or the first of the next
        // sweep (its order is drawn in this sweep's batch 0)
        const bool more = lo + a.b < a.n;
        const uint32_t* pn = more ? perm : (a.identity ? nullptr : a.perm + ((k + 1) % 3) * a.n);
        run_batch<PT, VE, EVAL ? 1 : 0, CTA>(a, x, Vs, pis, perm, lo, cnt, pl, acc, Qs,
                                         (lo == 0 && !a.identity) ? k + 1 : 0, pn, more ? lo + a.b : 0,
                                         more ? min(a.b, a.n - lo - a.b) : min(a.b, a.n));
        ++x.batches;
    }
    if (!EVAL && a.vnext) {
        // chunked T (VI*): every chunk read the sweep-start values; the
        // new values were parked in vnext and land now, for the next sweep
        timed_sync(x);
        if constexpr (is_vgl(CTA)) {
            const int64_t stride = (int64_t)a.nctas * kThreads;
            for (int64_t j = (int64_t)cta_rank(a) * kThreads + threadIdx.x; j < a.n; j += stride)
                a.V[j] = __ldcg(a.vnext + j);
            timed_sync(x);
        } else {
            for (int64_t j = threadIdx.x; j < a.n; j += kThreads) {
                const double v = __ldcg(a.vnext + j);
                Vs[vs_index(j, a.vs_half)] = v;
                if (cta_rank(a) == 0) a.V[j] = v;
            }
            csync();
        }
    }
    return phase_reduce<CTA>(a, x, acc);
}

template <typename PT, int VE, int CTA>
__device__ PhaseAcc run_improve(const DenseArgs& a, Ctx& x, double* Vs, int32_t* pis, double* Qs)
{
    PhaseAcc acc{0.0, 0, 0};
    for (int64_t lo = a.row0; lo < a.row1; lo += a.imp_sub) {
        const int64_t cnt = min(a.imp_sub, a.row1 - lo);
        run_batch<PT, VE, 2, CTA>(a, x, Vs, pis, nullptr, lo, cnt, a.plan[2], acc, Qs, 0);
    }
    PhaseAcc r = phase_reduce<CTA>(a, x, acc);
    if constexpr (is_fused(CTA)) r = xrank_reduce(a, x, r);  // each rank improved its own states
    return r;
}

// error trace after application `it`: each CTA folds its share of the states
// (its shared-memory copy of V is complete after the application's last
// patch; global V after the grid reduction).  A non-inlined call with scalar
// arguments: the solver loop keeps the register allocation of the untraced
// kernel (inlined, or passing DenseArgs by reference, made it spill).
__device__ __noinline__ void trace_error_dense(const double* V, int smem, int64_t vs_half, const double* vref,
                                               int64_t n, int64_t j0, int64_t stride, double* slot)
{
    if (smem)
        trace_error([&](int64_t j) { return V[vs_index(j, vs_half)]; }, vref, n, j0, stride, slot);
    else
        trace_error([&](int64_t j) { return __ldcg(V + j); }, vref, n, j0, stride, slot);
}

#ifndef RMB_AB_NO_ETRACE
#define RMB_ETRACE_DENSE()                                                                                       \
    do {                                                                                                          \
        if (a.etrace && it < a.etrace_len)                                                                        \
            trace_error_dense(is_vgl(CTA) ? a.V : Vs, !is_vgl(CTA), a.vs_half, a.vref, a.n,                       \
                              (int64_t)cta_rank(a) * kThreads + threadIdx.x, (int64_t)a.nctas * kThreads,          \
                              a.etrace + it);                                                                     \
    } while (0)
#else  // A/B builds: the solver without the trace call
#define RMB_ETRACE_DENSE() \
    do {                   \
    } while (0)
#endif

template <typename PT, int VE, int CTA>
__device__ __forceinline__ void dense_solver_body(const DenseArgs& a)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* Vs = reinterpret_cast<double*>(smem_raw);
    const int64_t n_pad = (a.n + 3) & ~int64_t(3);
    int32_t* pis = reinterpret_cast<int32_t*>(Vs + n_pad);
    double* Qs = reinterpret_cast<double*>(smem_raw + a.qs_off);
    const bool need_pi = a.mode == MODE_MPI || a.mode == MODE_APPLY_PI || a.mode == MODE_IMPROVE || a.mode == MODE_POLICY_VALUE ||
                         a.mode == MODE_SHARD_EVAL || a.mode == MODE_SHARD_IMPROVE;
    const bool shard = a.mode == MODE_SHARD_MIN || a.mode == MODE_SHARD_EVAL || a.mode == MODE_SHARD_IMPROVE;

    Ctx x{{a.bar, a.bar + 32, 0ull, (unsigned long long)a.nctas, a.err}, 0, 0, 0, 0, 0, 0, 0};
    x.cta0 = cta_rank(a) == 0;
    x.gred_seq = 0;
    if constexpr (is_vgl(CTA)) {  // V and pi stay in global memory (L2)
        Vs = a.V;
        pis = a.pi;
    }
    if constexpr (is_tma(CTA)) {
        x.tm = tma_smem(smem_raw, a);
        x.tst = 0;
        x.tph = 0;
        if (threadIdx.x == 0) {
            for (int q = 0; q < x.tm.nst; ++q) {
                mbar_init(x.tm.full + q, 1);
                mbar_init(x.tm.empty + q, kTmaCW);
                x.tm.redcnt[q] = 0;
            }
            x.tm.ctl[0] = -1;
            x.tm.ctl[1] = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();  // the only CTA-wide barrier: the producer warp leaves here
        if (threadIdx.x >= kThreads) {
            if (threadIdx.x == kThreads) tma_producer<PT>(a, pis, x.tm);
            return;
        }
    }
    if constexpr (!is_vgl(CTA)) {
        for (int64_t j = threadIdx.x; j < a.n; j += kThreads) {
            Vs[vs_index(j, a.vs_half)] = a.V[j];
            if (need_pi) pis[j] = a.pi[j];
        }
    }
    if (cta_rank(a) == 0 && threadIdx.x == 0) x.t_mark = globaltimer_ns();
    if (!a.identity && a.mode != MODE_IMPROVE && !shard)
        fill_order(a.n, a.seed, a.k0, a.order, a.perm + (a.k0 % 3) * a.n,
                   (int64_t)cta_rank(a) * kThreads + threadIdx.x, (int64_t)a.nctas * kThreads);
    timed_sync(x);  // perm of the first sweep visible; also orders the smem loads
    if (is_fused(CTA) && a.mode != MODE_IMPROVE) {  // fused: this rank's states of the first sweep batch
        build_own_list(a, a.identity ? nullptr : a.perm + (a.k0 % 3) * a.n, 0, min(a.b, a.n), 0);
        timed_sync(x);
    }

    const bool lead = cta_rank(a) == 0 && threadIdx.x == 0;
    long long status = RMB_ERR_NOT_CONVERGED;
    int64_t k = a.k0, it = 0, outer = 0;
    long long changed = 0;
    double last = 0.0;

    if (a.mode == MODE_SHARD_MIN || a.mode == MODE_SHARD_EVAL) {
        // one batch of this rank's states, against the replica V, into the send list
        PhaseAcc acc{0.0, 0, 0};
        const int64_t cnt = *a.ocount;
        if (a.mode == MODE_SHARD_MIN)
            run_batch<PT, VE, 3, CTA>(a, x, Vs, pis, a.olist, 0, cnt, a.plan[0], acc, Qs, 0);
        else
            run_batch<PT, VE, 4, CTA>(a, x, Vs, pis, a.olist, 0, cnt, a.plan[1], acc, Qs, 0);
        PhaseAcc r = phase_reduce<CTA>(a, x, acc);
        status = r.bad ? RMB_ERR_NONFINITE : RMB_OK;
        x.batches = 1;
    } else if (a.mode == MODE_SHARD_IMPROVE) {
        PhaseAcc r = run_improve<PT, VE, CTA>(a, x, Vs, pis, Qs);
        last = r.rmax;
        changed = r.changed;
        status = r.bad ? RMB_ERR_NONFINITE : RMB_OK;
    } else if (a.mode == MODE_VI || a.mode == MODE_APPLY || a.mode == MODE_APPLY_PI ||
               a.mode == MODE_POLICY_VALUE) {
        const bool eval = a.mode == MODE_APPLY_PI || a.mode == MODE_POLICY_VALUE;
        const int64_t iters = (a.mode == MODE_VI || a.mode == MODE_POLICY_VALUE) ? a.max_iter : 1;
        while (it < iters) {
            PhaseAcc r = eval ? run_sweep<PT, VE, true, CTA>(a, x, Vs, pis, k, Qs)
                                                 : run_sweep<PT, VE, false, CTA>(a, x, Vs, pis, k, Qs);
            if (lead && it < a.trace_len) a.trace[it] = r.rmax;
            RMB_ETRACE_DENSE();
            ++it;
            ++k;
            last = r.rmax;
            if (r.bad) { status = RMB_ERR_NONFINITE; break; }
            if (a.eps >= 0.0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if ((a.mode == MODE_APPLY || a.mode == MODE_APPLY_PI) && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
    } else if (a.mode == MODE_IMPROVE) {
        PhaseAcc r = run_improve<PT, VE, CTA>(a, x, Vs, pis, Qs);
        last = r.rmax;
        changed = r.changed;
        status = r.bad ? RMB_ERR_NONFINITE : RMB_OK;
    } else {  // MODE_MPI
        bool bad = false;
        if (!a.pi_given) {
            PhaseAcc r = run_improve<PT, VE, CTA>(a, x, Vs, pis, Qs);
            bad = r.bad;
        }
        while (!bad && outer < a.max_iter) {
            const int64_t row = outer * (a.msweeps + 1);
            for (int e = 0; e < a.msweeps && !bad; ++e) {
                PhaseAcc r = run_sweep<PT, VE, true, CTA>(a, x, Vs, pis, k, Qs);
                if (lead && row + e < a.trace_len) a.trace[row + e] = r.rmax;
                RMB_ETRACE_DENSE();
                ++k;
                ++it;
                bad = r.bad;
            }
            if (bad) { ++outer; break; }
            PhaseAcc r = run_improve<PT, VE, CTA>(a, x, Vs, pis, Qs);
            if (lead && row + a.msweeps < a.trace_len) a.trace[row + a.msweeps] = r.rmax;
            if (lead && outer < a.chg_len) a.chg[outer] = r.changed;
            ++outer;
            last = r.rmax;
            changed = r.changed;
            if (r.bad) { bad = true; break; }
            if (r.changed == 0 && r.rmax <= a.eps) { status = RMB_OK; break; }
        }
        if (bad) status = RMB_ERR_NONFINITE;
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
        a.prof[2] = x.t_comb;
        a.prof[3] = x.n_bar;
        a.out[OUT_XEPOCHS] = (long long)x.xepoch;
    }
    if constexpr (is_tma(CTA)) {
        csync();  // every compute thread is done with the ring
        if (threadIdx.x == 0) st_release_cta(x.tm.ctl + 1, 1);  // the producer drains and exits
    }
}

// register-streaming paths: 512 threads, 128 registers
template <typename PT, int VE, int CTA>
__global__ void __launch_bounds__(kThreads, 1) dense_solver_kernel(const DenseArgs a)
{
    dense_solver_body<PT, VE, CTA>(a);
}

// TMA ring path: 512 compute threads + the producer warp (17 warps: one SM
// sub-partition holds 5 of them, so 96 registers per thread).  VGL: V and pi
// in global memory (dense n too large for a shared-memory copy of V).
template <typename PT, int VE, bool VGL>
__global__ void __launch_bounds__(kTmaThreads, 1) dense_tma_kernel(const DenseArgs a)
{
    dense_solver_body<PT, VE, VGL ? kPathTmaG : kPathTma>(a);
}

// one rank of a fused multi-GPU group (K8f), one launch per device
template <typename PT, int VE, bool VGL>
__global__ void __launch_bounds__(kTmaThreads, 1) dense_tma_fused_kernel(const DenseArgs a)
{
    dense_solver_body<PT, VE, VGL ? kPathTmaGF : kPathTmaF>(a);
}

// ------------------------------------------------------------------ host
// rows = (states per batch) x (items per state before chunking).  Items are
// NG rows x Lc columns of P: at most ~16 KB so that the dynamically scheduled
// tail (one warp finishing one item) stays a few microseconds, and at least
// ~32 items per SM when the batch is small (b = 1 must still fill 148 SMs).
static Plan plan_chunks(int64_t n, int64_t cnt, int64_t groups_per_state, int A_eff, int VE, int num_sms,
                        bool allow_split, int ng, int psz)
{
    const int64_t rows = cnt * groups_per_state;
    const int64_t unit = (int64_t)kWarp * VE;
    const int64_t maxC = std::max<int64_t>(1, (n + unit - 1) / unit);
    const int64_t lc_target = std::max<int64_t>(unit, (int64_t(16) << 10) / ((int64_t)ng * psz));
    int64_t c = 1;
    (void)lc_target;
    if (allow_split && rows < 16LL * num_sms) {
        // at most one item per warp (the dynamic deal then has no second round)
        c = std::max<int64_t>(1, (16LL * num_sms) / rows);
        // bound the partial-sum scratch (A_eff * C doubles per state) to 64 MB
        c = std::min<int64_t>(c, std::max<int64_t>(1, (int64_t(1) << 23) / std::max<int64_t>(1, cnt * A_eff)));
        c = std::min(std::max<int64_t>(c, 1), maxC);
    }
    int64_t L = (n + c - 1) / c;
    L = (L + unit - 1) / unit * unit;
    Plan p{};
    p.Lc = (int)L;
    p.C = (int)((n + L - 1) / L);
    const int64_t per_state = p.C == 1 ? (A_eff == 1 ? 1 : 2 * groups_per_state) : (int64_t)A_eff * p.C;
    p.redundant = cnt * per_state <= kRedundantMax ? 1 : 0;
    return p;
}

static int64_t plan_doubles(const Plan& p, int64_t cnt, int64_t groups_per_state, int A_eff)
{
    if (p.raw) return A_eff == 1 ? cnt * p.C : cnt * groups_per_state * kAG * p.C;
    return p.C == 1 ? cnt * (A_eff == 1 ? 1 : 2 * groups_per_state) : cnt * A_eff * p.C;
}

template <typename PT, int VE>
static cudaError_t launch_typed(const DenseArgs& a, size_t smem, int grid, cudaStream_t st)
{
    auto kern = dense_solver_kernel<PT, VE, kPathWarp>;
    int threads = kThreads;
    if constexpr (VE * sizeof(PT) == 16) {
        if (a.path == kPathTma) {
            kern = dense_tma_kernel<PT, VE, false>;
            threads = kTmaThreads;
        } else if (a.path == kPathTmaG) {
            kern = dense_tma_kernel<PT, VE, true>;
            threads = kTmaThreads;
        }
    }
    // under stream capture (the sharded protocol's graph of a sweep) the
    // attribute and occupancy were set / checked by the eager warm-up sweep
    // with the same plan; these calls are not permitted while capturing
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(st, &cs);
    if (e != cudaSuccess) return e;
    if (cs == cudaStreamCaptureStatusNone) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
    }
    void* args[] = {const_cast<DenseArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, smem, st);
}

struct DenseLaunch {
    DenseArgs a;
    size_t smem;
    int VE;
    int64_t lcap;
};

// Plans (chunking, combine mode) and workspace for one launch.  The plan
// depends on (n, A, b, mode) only — never on how many states a shard owns —
// so every state's reduction order is identical for any number of GPUs.
static rmb_status dense_prepare(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                                long long* chg_dev, int64_t chg_len, DenseLaunch& L)
{
    const int64_t n = pr.n;
    const int psz = pr.pdt == RMB_F32 ? 4 : 8;
    int VE = 16 / psz;
    // 16-byte vectors need aligned rows; a shard uses the whole problem's
    // choice (g_aligned: every rank aligned), so its arithmetic is the same
    const bool aligned = (reinterpret_cast<uintptr_t>(pr.P) & 15u) == 0 && (!pr.g_set || pr.g_aligned);
    if ((n % VE) != 0 || !aligned) VE = 1;
    const bool need_pi = rq.mode == MODE_MPI || rq.mode == MODE_APPLY_PI || rq.mode == MODE_IMPROVE || rq.mode == MODE_POLICY_VALUE ||
                         rq.mode == MODE_SHARD_EVAL || rq.mode == MODE_SHARD_IMPROVE;
    const int64_t n_pad = (n + 3) & ~int64_t(3);
    size_t smem_v = (size_t)n_pad * 8 + (need_pi ? ((size_t)n * 4 + 15) / 16 * 16 : 0);
    // a shared-memory copy of V (and pi) plus a 2-stage ring must fit; else V
    // and pi stay in global memory (L2-resident) on the TMA path
    const bool vglob = pr.vglobal || smem_v + 12288 + 2 * 33000 > pr.smem_optin;
    if (vglob) {
        if (!(!pr.no_tma && VE * psz == 16)) {
            set_error("dense solver: n = " + std::to_string(n) + " needs " + std::to_string(smem_v) +
                      " B of shared memory for V (limit " + std::to_string(pr.smem_optin) +
                      "); larger n needs the TMA path (16-byte aligned rows: n % " + std::to_string(16 / psz) +
                      " == 0, RMB_DENSE_NO_TMA unset)");
            return RMB_ERR_UNSUPPORTED;
        }
        smem_v = 0;
    }
    DenseArgs& a = L.a;
    a = DenseArgs{};
    // P and c hold the rows of the owned states [row0, row1); offset the base
    // pointers so that global state ids index them directly
    const int64_t row0 = pr.row_begin, row1 = pr.row_end;
    a.P = static_cast<const char*>(pr.P) - (size_t)row0 * pr.A * n * psz;
    a.c = static_cast<const char*>(pr.c) - (size_t)row0 * pr.A * psz;
    a.row0 = row0;
    a.row1 = row1;
    a.vs_half = (VE == 4 && !vglob) ? n_pad / 2 : 0;
    a.n = n;
    a.A = pr.A;
    a.gamma = pr.gamma;
    a.V = rq.V;
    a.pi = rq.pi;
    a.b = rq.b;
    a.seed = rq.seed;
    a.k0 = rq.k0;
    // b >= n: one batch per sweep, whose result does not depend on the order
    // of its states -> no permutation needed (draws with replacement are not
    // a permutation: they always need the order array)
    a.identity = rq.select ? 0 : ((rq.identity || rq.b >= n) ? 1 : 0);
    a.order = OrderSpec{rq.select, pr.sel_cum, pr.sel_W};
    a.vref = rq.vref;
    a.etrace = rq.etrace;
    a.etrace_len = rq.etrace_len;
    a.mode = rq.mode;
    a.pi_given = rq.pi_given ? 1 : 0;
    a.eps = rq.eps;
    a.max_iter = rq.max_iter;
    a.msweeps = rq.msweeps;
    const int sms = pr.num_sms;
    // min-mode items are groups of kAG action rows (single-row items were
    // measured slower at b = 1000: 4x the smem V traffic and per-item atomics)
    const int ng_b = kAG;
    const int64_t NAG = (pr.A + ng_b - 1) / ng_b;
    // smem scratch for split-row (S-mode) reductions: up to 32 KB after V / pi
    a.qs_off = (int64_t)smem_v;
    a.qs_cap = std::min<int64_t>(4096, ((int64_t)pr.smem_optin - (int64_t)smem_v - 12288) / 8);
    L.smem = smem_v + (size_t)std::max<int64_t>(a.qs_cap, 0) * 8;
    const bool split_ok = a.qs_cap >= pr.A;  // else every row stays whole (C = 1)
    a.plan[0] = plan_chunks(n, rq.b, NAG, pr.A, VE, sms, split_ok, ng_b, psz);
    a.plan[0].ng = ng_b;
    a.plan[1] = plan_chunks(n, rq.b, 1, 1, VE, sms, split_ok, 1, psz);
    a.plan[1].ng = 1;
    // improvement (no V write): as few sub-batches as a bounded scratch allows
    const int64_t NAG4 = (pr.A + kAG - 1) / kAG;
    a.imp_sub = n * NAG4 * 2 <= (int64_t(1) << 22) ? n : std::max<int64_t>(1, (int64_t(1) << 22) / (2 * NAG4));
    a.plan[2] = plan_chunks(n, a.imp_sub, NAG4, pr.A, VE, sms, split_ok, kAG, psz);
    a.plan[2].ng = kAG;
    a.path = kPathWarp;
    // TMA ring path (default): 16-byte rows (VE full) and >= 2 ring stages next
    // to V / pi / the reduction scratch.  Chosen from (n, A, dtype, need_pi),
    // never from the shard, so every state's arithmetic is the same for any G.
    {
        const int64_t qs_tma = std::min<int64_t>(a.qs_cap, std::max<int64_t>(512, pr.A));  // >= A for the S-mode combine
        const size_t ring_off = (smem_v + (size_t)std::max<int64_t>(qs_tma, 0) * 8 + 127) / 128 * 128;
        const int64_t room = (int64_t)pr.smem_optin - (int64_t)ring_off - 16 - 2048;  // static smem
        // ring slots of kTmaStage bytes: NG row slots of one column window
        const int64_t piece = kTmaStage / psz, slot = kTmaStage;
        int nst = (int)std::min<int64_t>(kTmaMaxStages, std::max<int64_t>(0, room / (slot + kTmaPerStageX)));
        if (!pr.no_tma && a.path == kPathWarp && VE * psz == 16 && nst >= 2 && qs_tma >= pr.A) {
            a.path = vglob ? kPathTmaG : kPathTma;
            a.qs_cap = qs_tma;
            a.tma_off = (int64_t)ring_off;
            a.tma_nst = nst;
            a.tma_piece = (int)piece;
            a.tma_slot = (int)slot;
            L.smem = ring_off + (size_t)nst * (slot + kTmaPerStageX) + 16;
            // raw partials (A doubles per state and chunk), S-mode combines
            a.imp_sub = n * pr.A <= (int64_t(1) << 22) ? n : std::max<int64_t>(1, (int64_t(1) << 22) / pr.A);
            a.plan[2] = plan_chunks(n, a.imp_sub, NAG4, pr.A, VE, sms, split_ok, kAG, psz);
            a.plan[2].ng = kAG;
            // partial volumes up to red_max doubles are combined redundantly by
            // every CTA (one barrier); items = contiguous chunks of a state's
            // action-group range (or of its row pi(s)): >= ipsm items per SM
            const int64_t red_max = 2048, ipsm = 1;
            a.tma_static = 16;
            const int64_t cnts[3] = {rq.b, rq.b, a.imp_sub};
            const int64_t grp[3] = {NAG, 1, NAG4};
            const int na_min = (pr.A % kAG) ? pr.A % kAG : kAG;
            for (int q = 0; q < 3; ++q) {
                Plan& p = a.plan[q];
                const int64_t groups = cnts[q] * grp[q];
                const int64_t vg_min = (q == 1 ? 1 : std::min(na_min, pr.A)) * n / VE;
                const int64_t per = q == 1 ? 1 : kAG;  // doubles per item
                int64_t C = groups >= ipsm * sms ? 1 : (ipsm * sms + groups - 1) / groups;
                C = std::min<int64_t>(C, std::max<int64_t>(1, vg_min));
                C = std::min<int64_t>(C, std::max<int64_t>(1, (int64_t(1) << 23) / std::max<int64_t>(1, groups * per)));
                p.C = (int)C;
                p.Lc = 0;
                p.raw = 1;
                p.ng = q == 1 ? 1 : kAG;
                p.redundant = groups * per * C <= red_max ? 1 : 0;
            }
        }
    }
    if (vglob && a.path != kPathTmaG) {
        set_error("dense solver: n = " + std::to_string(n) + " needs the global-V TMA path (disable RMB_DENSE_ROWS/CTA)");
        return RMB_ERR_UNSUPPORTED;
    }
    const int64_t stride = std::max<int64_t>({plan_doubles(a.plan[0], rq.b, NAG, pr.A),
                                              plan_doubles(a.plan[1], rq.b, 1, 1),
                                              plan_doubles(a.plan[2], a.imp_sub, NAG4, pr.A), 2 * rq.b,
                                              2 * a.imp_sub});
    a.part_stride = (stride + 31) / 32 * 32;
    L.lcap = std::max<int64_t>(rq.b, a.imp_sub);
    L.VE = VE;

    const bool chunked = rq.chunked && (rq.mode == MODE_VI || rq.mode == MODE_APPLY) && rq.b < n;
    const size_t part_bytes = (size_t)2 * a.part_stride * 8 + (size_t)L.lcap * 16 + 64;
    if (pr.perm.ensure((size_t)3 * n * 4) != cudaSuccess ||
        pr.part.ensure(part_bytes + (chunked ? (size_t)n * 8 : 0)) != cudaSuccess ||
        pr.ctrl.ensure(4096) != cudaSuccess) {
        set_error("dense solver: workspace allocation failed");
        return RMB_ERR_OOM;
    }
    a.perm = static_cast<uint32_t*>(pr.perm.p);
    a.part = static_cast<double*>(pr.part.p);
    a.lval = a.part + 2 * a.part_stride;
    a.larg = reinterpret_cast<int32_t*>(a.lval + L.lcap);
    a.scnt = reinterpret_cast<unsigned int*>(a.larg + L.lcap);
    a.vnext = chunked ? reinterpret_cast<double*>(static_cast<char*>(pr.part.p) + part_bytes) : nullptr;
    unsigned long long* ctrl = static_cast<unsigned long long*>(pr.ctrl.p);
    a.bar = ctrl;                                          // [0], [32]
    a.err = reinterpret_cast<int*>(ctrl + 64);             // [64]
    a.out = reinterpret_cast<long long*>(ctrl + 128);      // [128..136)
    a.prof = reinterpret_cast<long long*>(ctrl + 192);     // [192..196)
    a.wctr = reinterpret_cast<unsigned int*>(ctrl + 256);  // [256]
    a.gred = ctrl + 320;                                   // [320..336): global-V grid reductions
    a.trace = trace_dev;
    a.trace_len = trace_len;
    a.chg = chg_dev;
    a.chg_len = chg_len;
    return RMB_OK;
}

static cudaError_t dense_launch(Problem& pr, DenseLaunch& L, cudaStream_t st)
{
    L.a.cta0 = 0;
    L.a.nctas = pr.num_sms;
    cudaError_t ce = cudaMemsetAsync(L.a.bar, 0, 4096, st);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(L.a.scnt, 0, (size_t)L.lcap * 4, st);
    if (ce != cudaSuccess) return ce;
    const int sms = pr.num_sms;
    if (pr.pdt == RMB_F32)
        return L.VE == 4 ? launch_typed<float, 4>(L.a, L.smem, sms, st) : launch_typed<float, 1>(L.a, L.smem, sms, st);
    return L.VE == 2 ? launch_typed<double, 2>(L.a, L.smem, sms, st) : launch_typed<double, 1>(L.a, L.smem, sms, st);
}

// One shard step (MODE_SHARD_*) launched asynchronously on `st`: the result
// block (status, residual, changed) lands in the returned device pointer.
rmb_status dense_shard_step(Problem& pr, const SolveRequest& rq, const uint32_t* olist, const int* ocount,
                            double* send_val, uint32_t* send_idx, int32_t* send_arg, cudaStream_t st,
                            long long** out_dev)
{
    DenseLaunch L;
    rmb_status s = dense_prepare(pr, rq, nullptr, 0, nullptr, 0, L);
    if (s != RMB_OK) return s;
    L.a.olist = olist;
    L.a.ocount = ocount;
    L.a.send_val = send_val;
    L.a.send_idx = send_idx;
    L.a.send_arg = send_arg;
    cudaError_t ce = dense_launch(pr, L, st);
    if (ce != cudaSuccess) {
        set_error(std::string("dense shard step: ") + cudaGetErrorString(ce));
        return RMB_ERR_CUDA;
    }
    if (out_dev) *out_dev = L.a.out;
    return RMB_OK;
}

rmb_status dense_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                       long long* chg_dev, int64_t chg_len, SolveResult* res)
{
    // tiny batches (<= 2 MB of P, <= 256 rows): one thread-block cluster
    if (!pr.no_cluster && dense_cluster_eligible(pr, rq)) {
        rmb_status s = dense_cluster_solve(pr, rq, trace_dev, trace_len, res);
        if (s != RMB_ERR_UNSUPPORTED) return s;
    }
    DenseLaunch L;
    rmb_status s = dense_prepare(pr, rq, trace_dev, trace_len, chg_dev, chg_len, L);
    if (s != RMB_OK) return s;
    cudaStream_t st = pr.stream;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaEventRecord(e0, st);
    if (ce == cudaSuccess) ce = dense_launch(pr, L, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(e1, st);
    long long out[OUT_N + 8] = {0};
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, L.a.out, sizeof(long long) * OUT_N, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out + OUT_N, L.a.prof, sizeof(long long) * 4, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    float ms = 0.f;
    if (ce == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) {
        set_error(std::string("dense solver: ") + cudaGetErrorString(ce));
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

}  // namespace rmb

namespace rmb {

// ------------------------------------------------------------------ K8f
// Multi-GPU solve with the exchange fused into the persistent kernel (SURVEY
// 8(e) "B200-native fused path"): no host round trip, no NCCL launch per
// batch -- each rank stores its batch results straight into every rank's
// exchange arrays over NVLink (peer memory) and the ranks meet at an in-kernel
// cross-rank barrier.  Each state's arithmetic is the single-GPU kernel's
// (plan from (n, A, b) and the device's SM count), so V, pi and the trace are
// bitwise those of one GPU.

// Every rank of a group launches with one DenseArgs; with G logical ranks on
// one device the launch holds all of them (CTA groups of `per` CTAs).
template <typename PT, int VE, bool VGL>
__global__ void __launch_bounds__(kTmaThreads, 1) dense_tma_group_kernel(const DenseArgs* __restrict__ set, int per)
{
    dense_solver_body<PT, VE, VGL ? kPathTmaGF : kPathTmaF>(set[blockIdx.x / per]);
}

// exchange buffer layout for batches of up to `cap` positions
struct XLayout {
    size_t val, arg, bar, imp, list, cnt, bytes;
    explicit XLayout(int64_t cap)
    {
        auto up = [](size_t x) { return (x + 255) / 256 * 256; };
        val = 0;
        arg = up(val + (size_t)2 * cap * 8);
        bar = up(arg + (size_t)2 * cap * 4);
        imp = up(bar + 8);
        list = up(imp + (size_t)2 * kMaxRanks * 4 * 8);
        cnt = up(list + (size_t)3 * 2 * cap * 4);
        bytes = up(cnt + 3 * 4);
    }
};

rmb_status fused_buffer(Problem& pr)
{
    const XLayout X(pr.n);
    if (pr.xbuf.p && pr.xbuf.bytes >= X.bytes) return RMB_OK;
    if (pr.xpeer_G > 0) {
        set_error("fused solve: exchange buffer already shared with peers");
        return RMB_ERR_INVALID_ARG;
    }
    if (pr.xbuf.ensure(X.bytes) != cudaSuccess) {
        set_error("fused solve: exchange buffer allocation failed");
        return RMB_ERR_OOM;
    }
    cudaError_t e = cudaMemsetAsync(pr.xbuf.p, 0, X.bytes, pr.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr.stream);
    if (e != cudaSuccess) {
        set_error(std::string("fused solve: ") + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    }
    pr.xepochs = 0;
    return RMB_OK;
}

rmb_status dense_fused_solve(Problem** ranks, int G, bool nccl, const SolveRequest& rq0, double* trace_host,
                             int64_t trace_len, int64_t* chg_host, int64_t chg_len, SolveResult* res)
{
    Problem& p0 = *ranks[0];
    const int L = nccl ? 1 : G;  // ranks in this launch
    int world = G, me = 0;
    if (nccl) {
        rmb_status s = fused_peers(p0, &world, &me);  // shard.cu: IPC handles over NCCL
        if (s != RMB_OK) return s;
    }
    if (world > kMaxRanks) {
        set_error("fused solve: at most 8 ranks");
        return RMB_ERR_UNSUPPORTED;
    }
    const XLayout X(p0.n);
    std::vector<DenseLaunch> Ls((size_t)L);
    if (!nccl)  // every rank's exchange buffer exists before any rank's arguments point at it
        for (int r = 0; r < L; ++r)
            if (rmb_status s = fused_buffer(*ranks[r]); s != RMB_OK) return s;
    for (int r = 0; r < L; ++r) {
        Problem& pr = *ranks[r];
        SolveRequest rq = rq0;
        rq.V = pr.stage_V;
        rq.pi = pr.stage_pi;
        if (pr.trace.ensure((size_t)std::max<int64_t>(1, trace_len) * 8) != cudaSuccess ||
            pr.chg.ensure((size_t)std::max<int64_t>(1, chg_len) * 8) != cudaSuccess) {
            set_error("fused solve: trace allocation failed");
            return RMB_ERR_OOM;
        }
        rmb_status s = dense_prepare(pr, rq, static_cast<double*>(pr.trace.p), trace_len,
                                     static_cast<long long*>(pr.chg.p), chg_len, Ls[r]);
        if (s != RMB_OK) return s;
        DenseArgs& a = Ls[r].a;
        if (!is_tma(a.path)) {
            set_error("fused solve: needs the TMA path (16-byte aligned rows, RMB_DENSE_NO_TMA unset)");
            return RMB_ERR_UNSUPPORTED;
        }
        if (Ls[r].smem != Ls[0].smem || Ls[r].lcap > p0.n) {
            set_error("fused solve: ranks disagree on the launch shape");
            return RMB_ERR_INVALID_ARG;
        }
        a.xG = world;
        a.xrank = nccl ? me : r;
        for (int q = 0; q < world; ++q) {
            char* base = static_cast<char*>(nccl ? p0.xpeer[q] : ranks[q]->xbuf.p);
            a.xval[q] = reinterpret_cast<double*>(base + X.val);
            a.xarg[q] = reinterpret_cast<int32_t*>(base + X.arg);
            a.xbar[q] = reinterpret_cast<unsigned long long*>(base + X.bar);
            a.ximp[q] = reinterpret_cast<unsigned long long*>(base + X.imp);
        }
        a.xval_own = a.xval[a.xrank];
        a.xarg_own = a.xarg[a.xrank];
        a.xbar_own = a.xbar[a.xrank];
        a.ximp_own = a.ximp[a.xrank];
        char* own = static_cast<char*>(pr.xbuf.p);
        a.xlist = reinterpret_cast<uint32_t*>(own + X.list);
        a.xcnt = reinterpret_cast<unsigned int*>(own + X.cnt);
        a.xlcap = p0.n;
        a.xbase = (unsigned long long)pr.xepochs;
        unsigned long long* ctrl = static_cast<unsigned long long*>(pr.ctrl.p);
        a.xloc = ctrl + 352;
        a.xrel = ctrl + 384;
    }
    const int per = nccl ? p0.num_sms : p0.num_sms / L;
    if (per < 1) {
        set_error("fused solve: more logical ranks than SMs");
        return RMB_ERR_UNSUPPORTED;
    }
    cudaStream_t st = p0.stream;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaEventRecord(e0, st);
    for (int r = 0; r < L && ce == cudaSuccess; ++r) {
        DenseLaunch& D = Ls[r];
        D.a.cta0 = r * per;
        D.a.nctas = per;
        ce = cudaMemsetAsync(D.a.bar, 0, 4096, st);
        if (ce == cudaSuccess) ce = cudaMemsetAsync(D.a.scnt, 0, (size_t)D.lcap * 4, st);
        if (ce == cudaSuccess) ce = cudaMemsetAsync(D.a.xcnt, 0, 3 * 4, st);
    }
    const DenseLaunch& D0 = Ls[0];
    const bool f32 = ranks[0]->pdt == RMB_F32;
    const bool vgl = D0.a.path == kPathTmaG;
    if (ce == cudaSuccess) {
        // same launch shape for every instantiation: 544 threads, D0.smem bytes
        const void* kern = f32 ? (vgl ? (const void*)dense_tma_group_kernel<float, 4, true>
                                      : (const void*)dense_tma_group_kernel<float, 4, false>)
                               : (vgl ? (const void*)dense_tma_group_kernel<double, 2, true>
                                      : (const void*)dense_tma_group_kernel<double, 2, false>);
        ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D0.smem);
        // the argument sets live in device memory (rank 0's aux buffer)
        if (ce == cudaSuccess && p0.aux.ensure(sizeof(DenseArgs) * (size_t)L + 256) != cudaSuccess)
            ce = cudaErrorMemoryAllocation;
        std::vector<DenseArgs> host((size_t)L);
        for (int r = 0; r < L; ++r) host[r] = Ls[r].a;
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(p0.aux.p, host.data(), sizeof(DenseArgs) * (size_t)L, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess && L == 1) {
            // one rank per device: the regular entry (arguments in parameter space)
            const void* k1 = f32 ? (vgl ? (const void*)dense_tma_fused_kernel<float, 4, true>
                                        : (const void*)dense_tma_fused_kernel<float, 4, false>)
                                 : (vgl ? (const void*)dense_tma_fused_kernel<double, 2, true>
                                        : (const void*)dense_tma_fused_kernel<double, 2, false>);
            ce = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D0.smem);
            void* args[] = {&host[0]};
            if (ce == cudaSuccess)
                ce = cudaLaunchCooperativeKernel(k1, dim3(per), dim3(kTmaThreads), args, D0.smem, st);
        } else if (ce == cudaSuccess) {
            const DenseArgs* set = static_cast<const DenseArgs*>(p0.aux.p);
            int per_arg = per;
            void* args[] = {&set, &per_arg};
            ce = cudaLaunchCooperativeKernel(kern, dim3(per * L), dim3(kTmaThreads), args, D0.smem, st);
        }
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);  // the host copy of the args stays alive until here
    }
    if (ce == cudaSuccess) ce = cudaEventRecord(e1, st);
    long long out[OUT_N + 4] = {0};
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out, D0.a.out, sizeof(long long) * OUT_N, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(out + OUT_N, D0.a.prof, sizeof(long long) * 4, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && trace_host && trace_len > 0)
        ce = cudaMemcpyAsync(trace_host, D0.a.trace, (size_t)trace_len * 8, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && chg_host && chg_len > 0)
        ce = cudaMemcpyAsync(chg_host, D0.a.chg, (size_t)chg_len * 8, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    float ms = 0.f;
    if (ce == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) {
        set_error(std::string("fused solve: ") + cudaGetErrorString(ce));
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
    for (int r = 0; r < L; ++r) {
        ranks[r]->xepochs += out[OUT_XEPOCHS];  // every rank ran the same epochs
        ranks[r]->last_launches = 1;
        ranks[r]->last_graph_launches = 0;
        for (int i = 0; i < 4; ++i) ranks[r]->prof[i] = out[OUT_N + i];
    }
    return RMB_OK;
}

}  // namespace rmb

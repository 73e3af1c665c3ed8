// cluster.cu — dense MB-VI / B_{pi,b} sweeps for TINY batches on one
// thread-block cluster (sm_100a: up to 16 CTAs, distributed shared memory,
// hardware cluster barrier).
//
// Small b is latency-bound by construction (SURVEY 7 hard part #1): b = 1 is
// the Gauss-Seidel operator F, 10^4 batches per sweep on
// config 2, each only b*|A|*n*4 bytes of P (640 KB at b = 1).  On the 148-CTA
// grid a batch costs a grid barrier (~2 us through L2 atomics) plus a combine
// that reads every CTA's partial sums back from L2 -- ~5 us against 0.1 us of
// HBM time.  Here one cluster of CS CTAs does the whole solve:
//   * CTA q owns the column slab [q*slab, (q+1)*slab) of every row; a batch's
//     rows (state s, action a) are streamed slab by slab with cp.async.bulk
//     into a shared-memory ring, up to RING stages ahead (P does not depend on
//     V: the loads of the next batches are in flight across the barrier);
//   * each warp dots its rows' slab with the shared-memory copy of V (fp64),
//     the row partials stay in the CTA's shared memory;
//   * one hardware cluster barrier per batch (barrier.cluster release/acquire);
//   * every CTA then reads all CS partials of every row through DSMEM
//     (ld.shared::cluster), adds them in CTA order (fixed: reproducible), takes
//     min / argmin (lowest action on exact ties) and patches its own V copy --
//     Eq. 12: V changes only after the barrier that ends every read of the batch.
// The per-state arithmetic is fixed by (n, CS): bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "partition.cuh"

namespace rmb {

constexpr int kCThreads = 288;  // 8 compute warps + the issuing warp (all take part in the combine)
constexpr int kCWarps = kCThreads / kWarp;
constexpr int kCDot = 8;        // warps that dot the stages; warp kCDot issues the bulk copies
constexpr int kCRowsMax = 16;   // rows per ring stage
constexpr int kCBatchRows = 256;  // rows (states x actions) per batch this path serves

struct ClusterArgs {
    const void* P;
    const void* c;
    int n, A;
    double gamma;
    double* V;
    int32_t* pi;
    int b;
    uint64_t seed;
    int64_t k0;
    int identity;
    int eval;       // 1: B_{pi,b} sweeps (row pi(s)), 0: B_b
    double eps;     // < 0: no stopping test (single application)
    int64_t max_iter;
    uint32_t* perm; // 3 * n
    OrderSpec order;  // permutation, or draws with replacement (R28-R29)
    const double* vref;  // RMB_TRACE_ERROR_VS_REF (null = off)
    double* etrace;
    int64_t etrace_len;
    double* trace;
    int64_t trace_len;
    long long* out;
    long long* prof;
    int slab;       // columns per CTA (multiple of 16 bytes)
    int row_bytes;  // bytes per row slot of a stage
    int rows;       // rows per stage
    int ring;       // stages
    int64_t v_off, pi_off, ring_off, part_off, bar_off;  // dynamic smem layout (bytes)
};

__device__ __forceinline__ unsigned cluster_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// generic address of the same shared-memory variable in CTA `rank` of the cluster
__device__ __forceinline__ const double* dsmem(const double* p, unsigned rank)
{
    uint64_t r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return reinterpret_cast<const double*>(r);
}

// One row job of the solve: the rows [r0, r0 + nr) of batch `bt` (rows are
// (position, action) pairs, position-major).
struct CJob {
    int64_t k;   // sweep
    int lo, cnt; // batch positions
    int r0, nr;  // rows of the batch in this stage
};

template <typename PT>
__global__ void __launch_bounds__(kCThreads, 1) dense_cluster_kernel(const ClusterArgs a)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double* Vs = reinterpret_cast<double*>(sm + a.v_off);
    int32_t* pis = reinterpret_cast<int32_t*>(sm + a.pi_off);
    unsigned char* ring = sm + a.ring_off;
    double* part = reinterpret_cast<double*>(sm + a.part_off);  // [2][kCBatchRows]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + a.bar_off);
    const unsigned q = cluster_rank();
    const unsigned CS = gridDim.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = a.n;
    const int Ae = a.eval ? 1 : a.A;
    // this CTA's columns (possibly none when n is small)
    const int c0 = min(n, (int)q * a.slab), c1 = min(n, c0 + a.slab);
    constexpr int E = 16 / (int)sizeof(PT);
    using VT = typename std::conditional<sizeof(PT) == 4, float4, double2>::type;

    // V in shared memory; fp32 P: split planes (lo: V[4q], V[4q+1]; hi:
    // V[4q+2], V[4q+3]) so that a lane's two 16-byte reads are conflict-free
    const int vhalf = sizeof(PT) == 4 ? ((n + 3) & ~3) / 2 : 0;
    auto vidx = [&](int j) { return vhalf ? ((j & 2) ? vhalf : 0) + ((j >> 2) << 1) + (j & 1) : j; };
    for (int j = t; j < n; j += kCThreads) {
        Vs[vidx(j)] = a.V[j];
        if (a.eval) pis[j] = a.pi[j];
    }
    if (t == 0)
        for (int s = 0; s < a.ring; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the first sweep's order: every CTA draws its share of the positions
    if (!a.identity)
        fill_order(n, a.seed, a.k0, a.order, a.perm + (a.k0 % 3) * n, (int64_t)q * kCThreads + t,
                   (int64_t)CS * kCThreads);
    cluster_sync();

    // ---- the row-job stream (identical on every CTA; each loads its own slab)
    const int nbatch = (n + a.b - 1) / a.b;
    auto job_at = [&](int64_t sweep, int bi, int st, CJob& J) {
        J.k = sweep;
        J.lo = bi * a.b;
        J.cnt = min(a.b, n - J.lo);
        J.r0 = st * a.rows;
        J.nr = min(a.rows, J.cnt * Ae - J.r0);
    };
    // producer state (thread 0): the next job to issue
    int64_t pk = a.k0;
    int pb = 0, ps = 0;
    int64_t issued = 0;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const PT* P = static_cast<const PT*>(a.P);
    const int64_t last_sweep = a.k0 + a.max_iter - 1;
    // a job may be issued only once the perm of its sweep is visible: the next
    // sweep's order is drawn in batch 0 of the current one (so >= 2 batches per
    // sweep lets the stream run across sweeps; this path serves tiny batches)
    int64_t ck = a.k0;  // consumer position
    auto may_issue = [&](int64_t cons_k, int cons_b) {
        return pk <= last_sweep && (pk == cons_k || (pk == cons_k + 1 && cons_b >= 1));
    };
    // lane r's state id of job J, a raw L2 load: nothing consumes it until
    // the job is issued (no scoreboard stall here)
    auto state_of = [&](const CJob& J) -> int {
        if (lane >= J.nr) return 0;
        const uint32_t* pm = a.identity ? nullptr : a.perm + (J.k % 3) * n;
        const int i = (J.r0 + lane) / Ae;
        return pm ? (int)__ldcg(pm + J.lo + i) : J.lo + i;
    };
    auto source = [&](const CJob& J, int s) -> const PT* {
        if (lane >= J.nr) return nullptr;
        const int row = J.r0 + lane;
        const int act = a.eval ? __ldcg(a.pi + s) : row - (row / Ae) * Ae;
        return P + ((int64_t)s * a.A + act) * n + c0;
    };
    // warp 0: the next job into ring slot issued % ring (lane r: row r); the
    // state ids of the job after it are looked up right away, so that their
    // round trip overlaps everything until the next call
    int pre_s = 0;
    bool pre_ok = false;
    auto issue_one = [&](int64_t cons_k, int cons_b) {
        if (pk > last_sweep) return;
        CJob J;
        job_at(pk, pb, ps, J);
        const PT* src = source(J, pre_ok ? pre_s : state_of(J));
        const int slot = (int)(issued % a.ring);
        unsigned char* dst = ring + (size_t)slot * a.rows * a.row_bytes;
        const unsigned bytes = (unsigned)((c1 - c0) * (int)sizeof(PT));
        if (lane == 0) mbar_arrive_tx(full + slot, bytes * (unsigned)J.nr);
        __syncwarp();
        if (lane < J.nr && bytes > 0) bulk_g2s(dst + (size_t)lane * a.row_bytes, src, bytes, full + slot, pol);
        ++issued;
        if (++ps * a.rows >= J.cnt * Ae) {  // next batch
            ps = 0;
            if (++pb == nbatch) pb = 0, ++pk;
        }
        pre_ok = may_issue(cons_k, cons_b);
        if (pre_ok) {
            CJob J2;
            job_at(pk, pb, ps, J2);
            pre_s = state_of(J2);
        }
    };
    if (warp == kCDot)
        for (int s = 0; s < a.ring && may_issue(ck, 0); ++s) issue_one(ck, 0);

    // phase profile of CTA 0 (rmb_last_phase_times): stream + dot, cluster barrier, combine
    const bool lead = q == 0 && t == 0;
    unsigned long long tmark = lead ? globaltimer_ns() : 0, t_comp = 0, t_bar = 0, t_comb = 0, t_wait = 0;
    auto mark = [&](unsigned long long& acc) {
        if (lead) {
            const unsigned long long now = globaltimer_ns();
            acc += now - tmark;
            tmark = now;
        }
    };
    int L = 1;  // lanes per state in the combine (pow2 >= Ae)
    while (L < Ae) L <<= 1;
    int cs_s[2] = {0, 0};
    double cs_c[2] = {0.0, 0.0};
    bool pre_comb = false;
    int64_t consumed = 0;
    long long status = RMB_ERR_NOT_CONVERGED;
    int64_t it = 0, batches = 0;
    double last = 0.0;
    double rmax = 0.0;
    int bad = 0;
    while (it < a.max_iter) {
        const int64_t k = ck;
        const uint32_t* pm = a.identity ? nullptr : a.perm + (k % 3) * n;
        rmax = 0.0;
        bad = 0;
        for (int bi = 0; bi < nbatch; ++bi) {
            const int lo = bi * a.b, cnt = min(a.b, n - lo);
            const int nrows = cnt * Ae;
            double* pr = part + (size_t)(batches & 1) * kCBatchRows;
            // the combine's states and costs: looked up one batch ahead (the
            // state ids at the start of the previous batch, the costs after its
            // combine), here only when nothing was prefetched
            if (!pre_comb) {
#pragma unroll
                for (int rd = 0; rd < 2; ++rd) {
                    const int id = rd * kCThreads + t;
                    const int i = id / L, g = id - i * L;
                    cs_s[rd] = i < cnt ? (pm ? (int)__ldcg(pm + lo + i) : lo + i) : 0;
                    cs_c[rd] = i < cnt && g < Ae
                                   ? (double)__ldg(static_cast<const PT*>(a.c) + (int64_t)cs_s[rd] * a.A +
                                                   (a.eval ? pis[cs_s[rd]] : g))
                                   : 0.0;
                }
            }
            // the next batch's state ids (later in this sweep, or the first of
            // the next sweep once its order is visible, i.e. from batch 1 on)
            const bool nx_same = bi + 1 < nbatch;
            const bool nx_ok = nx_same || (it + 1 < a.max_iter && nbatch >= 2);
            const int nx_lo = nx_same ? lo + a.b : 0;
            const int nx_cnt = min(a.b, n - nx_lo);
            const uint32_t* nx_pm = a.identity ? nullptr : a.perm + ((nx_same ? k : k + 1) % 3) * n;
            int nx_s[2] = {0, 0};
            if (nx_ok && (nx_same || bi >= 1)) {
#pragma unroll
                for (int rd = 0; rd < 2; ++rd) {
                    const int i = (rd * kCThreads + t) / L;
                    nx_s[rd] = i < nx_cnt ? (nx_pm ? (int)__ldcg(nx_pm + nx_lo + i) : nx_lo + i) : 0;
                }
            }
            for (int st = 0; st * a.rows < nrows; ++st) {
                const int slot = (int)(consumed % a.ring);
                const unsigned ph = (unsigned)((consumed / a.ring) & 1);
                CJob J;
                job_at(k, bi, st, J);
                if (warp == kCDot) {  // refill the ring (the slot of the previous job is free) while the others dot
                    ck = k;
                    while (issued < consumed + a.ring && may_issue(k, bi)) issue_one(k, bi);
                }
                {
                    mark(t_comp);
                    SpinGuard sg;
                    while (!mbar_try(full + slot, ph)) sg.tick();
                    mark(t_wait);
                }
                const unsigned char* stg = ring + (size_t)slot * a.rows * a.row_bytes;
                const int nv = (c1 - c0) / E;  // 16-byte vectors of the slab (slab and n are multiples of E)
                // warp w dots rows w and w + 8 of the stage; each V vector is
                // read once (conflict-free split planes) for both rows
                if (warp < kCDot && warp < J.nr) {
                    const bool two = warp + kCDot < J.nr;
                    const VT* row0 = reinterpret_cast<const VT*>(stg + (size_t)warp * a.row_bytes);
                    const VT* row1 = reinterpret_cast<const VT*>(stg + (size_t)(warp + kCDot) * a.row_bytes);
                    double acc0 = 0.0, acc1 = 0.0;
                    for (int v = lane; v < nv; v += kWarp) {
                        const int j = c0 + v * E;
                        double vs[E];
                        if constexpr (sizeof(PT) == 4) {
                            const double2 lo = *reinterpret_cast<const double2*>(Vs + (j >> 1));
                            const double2 hi = *reinterpret_cast<const double2*>(Vs + vhalf + (j >> 1));
                            vs[0] = lo.x, vs[1] = lo.y, vs[2] = hi.x, vs[3] = hi.y;
                        } else {
                            const double2 x = *reinterpret_cast<const double2*>(Vs + j);
                            vs[0] = x.x, vs[1] = x.y;
                        }
                        const VT x0 = row0[v];
                        const double p0[4] = {(double)x0.x, (double)x0.y, sizeof(PT) == 4 ? (double)((const float*)&x0)[2] : 0.0,
                                              sizeof(PT) == 4 ? (double)((const float*)&x0)[3] : 0.0};
#pragma unroll
                        for (int e = 0; e < E; ++e) acc0 = fma(p0[e], vs[e], acc0);
                        if (two) {
                            const VT x1 = row1[v];
                            const double p1[4] = {(double)x1.x, (double)x1.y,
                                                  sizeof(PT) == 4 ? (double)((const float*)&x1)[2] : 0.0,
                                                  sizeof(PT) == 4 ? (double)((const float*)&x1)[3] : 0.0};
#pragma unroll
                            for (int e = 0; e < E; ++e) acc1 = fma(p1[e], vs[e], acc1);
                        }
                    }
                    acc0 = warp_sum(acc0);
                    acc1 = warp_sum(acc1);
                    if (lane == 0) {
                        pr[J.r0 + warp] = acc0;
                        if (two) pr[J.r0 + warp + kCDot] = acc1;
                    }
                }
                __syncthreads();  // every warp is done with the slot
                ++consumed;
            }
            // next sweep's order, off the critical path (batch 0)
            if (bi == 0 && !a.identity)
                fill_order(n, a.seed, k + 1, a.order, a.perm + ((k + 1) % 3) * n, (int64_t)q * kCThreads + t,
                           (int64_t)CS * kCThreads);
            mark(t_comp);
            cluster_sync();  // the batch's partials of every CTA are complete (and its reads of V done)
            mark(t_bar);
            // combine: L = pow2 >= Ae lanes per state; lane g takes action g;
            // partials of the CS CTAs added in CTA order (cnt * L <= 2 * 256 < 2 * kCThreads)
            for (int rd = 0; rd * kCThreads < cnt * L; ++rd) {
                const int id = rd * kCThreads + t;
                const int i = id / L, g = id - i * L;
                const bool valid = i < cnt && g < Ae;
                double Q = INFINITY;
                int arg = 0x7fffffff;
                const int s = rd ? cs_s[1] : cs_s[0];
                if (valid) {
                    // all CS remote loads in flight at once, then added in CTA order
                    double pv[16];
#pragma unroll
                    for (unsigned cq = 0; cq < 16; ++cq) pv[cq] = cq < CS ? *dsmem(pr + i * Ae + g, cq) : 0.0;
                    double sum = 0.0;
#pragma unroll
                    for (unsigned cq = 0; cq < 16; ++cq)
                        if (cq < CS) sum += pv[cq];
                    const int act = a.eval ? pis[s] : g;
                    Q = (rd ? cs_c[1] : cs_c[0]) + a.gamma * sum;
                    arg = act;
                }
                // argmin over the L lanes of the state (lower value, then lower action)
                for (int o = 1; o < L; o <<= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, Q, o);
                    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
                    if (ov < Q || (ov == Q && oa < arg)) Q = ov, arg = oa;
                }
                if (valid && g == 0) {
                    rmax = fmax(rmax, fabs(Q - Vs[vidx(s)]));
                    bad |= !isfinite(Q);
                    Vs[vidx(s)] = Q;
                    if (q == 0) {
                        a.V[s] = Q;
                        if (!a.eval && a.pi) a.pi[s] = arg;
                    }
                }
            }
            __syncthreads();  // the patched V is visible to the CTA's next batch
            pre_comb = nx_ok && (nx_same || bi >= 1);
            if (pre_comb) {  // the next batch's costs (its state ids arrived during this batch)
#pragma unroll
                for (int rd = 0; rd < 2; ++rd) {
                    const int id = rd * kCThreads + t;
                    const int i = id / L, g = id - i * L;
                    cs_s[rd] = nx_s[rd];
                    cs_c[rd] = i < nx_cnt && g < Ae
                                   ? (double)__ldg(static_cast<const PT*>(a.c) + (int64_t)nx_s[rd] * a.A +
                                                   (a.eval ? pis[nx_s[rd]] : g))
                                   : 0.0;
                }
            }
            mark(t_comb);
            ++batches;
        }
        // sweep residual: every CTA patched every state, so the CTA-local max
        // is the sweep's; reduce it over the CTA
        __shared__ double red[kCWarps];
        __shared__ int redb[kCWarps];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
        if (lane == 0) red[warp] = rmax, redb[warp] = bad;
        __syncthreads();
        double r = 0.0;
        int bb = 0;
        for (int w = 0; w < kCWarps; ++w) r = fmax(r, red[w]), bb |= redb[w];
        __syncthreads();
        if (q == 0 && t == 0 && it < a.trace_len) a.trace[it] = r;
        if (a.etrace && it < a.etrace_len)  // every CTA holds all of V: CTA q folds its share
            trace_error([&](int64_t j) { return Vs[vidx((int)j)]; }, a.vref, n, (int64_t)q * kCThreads + t,
                        (int64_t)CS * kCThreads, a.etrace + it);
        ++it;
        ++ck;
        last = r;
        if (bb) { status = RMB_ERR_NONFINITE; break; }
        if (a.eps >= 0.0 && r <= a.eps) { status = RMB_OK; break; }
        if (warp == kCDot)  // the next sweep's first batch may now stream (its order is visible)
            while (issued < consumed + a.ring && may_issue(ck, 0)) issue_one(ck, 0);
    }
    if (a.eps < 0.0 && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
    // drain: bulk copies in flight must land before the CTA exits (the
    // issuing warp's lane 0 holds the issue count)
    if (warp == kCDot && lane == 0) {
        for (int64_t d = consumed; d < issued; ++d) {
            const int slot = (int)(d % a.ring);
            const unsigned ph = (unsigned)((d / a.ring) & 1);
            SpinGuard sg;
            while (!mbar_try(full + slot, ph)) sg.tick();
        }
    }
    cluster_sync();  // no CTA exits while another may still read its shared memory
    if (q == 0 && t == 0) {
        a.out[OUT_SWEEPS] = it;
        a.out[OUT_OUTER] = 0;
        a.out[OUT_STATUS] = status;
        a.out[OUT_RESID_BITS] = __double_as_longlong(last);
        a.out[OUT_BATCHES] = batches;
        a.out[OUT_CHANGED] = 0;
        a.prof[0] = (long long)t_comp;
        a.prof[1] = (long long)t_bar;
        a.prof[2] = (long long)t_comb;
        a.prof[3] = batches + 2;  // cluster barriers (one per batch, one at each end)
        a.out[7] = (long long)t_wait;  // of prof[0]: waiting for the ring
    }
}


// ------------------------------------------------------------------ b = 1
// Gauss-Seidel batches (b = 1, <= 16 rows per state) with the dot of the
// next batch taken OFF the per-batch chain.  Batch u's rows are dotted
// against V with batch u-1's column left out (its value is not final yet),
// the owner CTA keeps P(row, s_{u-1}); once batch u-1 is combined, a combine
// warp adds P(row, s_{u-1}) V(s_{u-1}) to its partial -- the same sum in a
// different (fixed) order, R26.  Warps 0-7 dot, warp 8 issues the ring, warp
// 9 corrects, signals every CTA (remote mbarrier arrive, release.cluster),
// waits for the cluster's partials of the batch, combines them through DSMEM
// and patches V; the dot warps meanwhile dot batch u+1 (they wait only for
// batch u-1's patch).  Per batch the chain is correction + cluster signal +
// combine, not stream + dot + barrier + combine.
constexpr int kLThreads = 320;  // 8 dot warps + the issuing warp + the combine warp
constexpr int kLGroup = 288;    // dot + issuing warps (named barrier 1)
constexpr int kLComb = 9;       // the combine warp

__device__ __forceinline__ void mbar_arrive_remote(unsigned long long* bar, unsigned rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
// 8-byte store into CTA `rank`'s shared memory, completing 8 bytes of its
// mbarrier `bar` (same offsets in every CTA of the cluster)
__device__ __forceinline__ void st_async_remote(double* dst, double v, unsigned long long* bar, unsigned rank)
{
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_addr(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                 "l"(__double_as_longlong(v)), "r"(rb)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_cluster(unsigned long long* b, unsigned parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, "
        "0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

template <typename PT>
__global__ void __launch_bounds__(kLThreads, 1) dense_cluster_la_kernel(const ClusterArgs a)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double* Vs = reinterpret_cast<double*>(sm + a.v_off);
    int32_t* pis = reinterpret_cast<int32_t*>(sm + a.pi_off);
    unsigned char* ring = sm + a.ring_off;
    // batch u's slot u % 4 (received from every CTA by st.async): [16 CTAs][16 rows]
    // row partials, then [16] coefficients P(row, s_{u-1}) from the column's owner
    double* xb = reinterpret_cast<double*>(sm + a.part_off);
    constexpr int kXSlot = 16 * 16 + 16;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + a.bar_off);  // [ring]
    unsigned long long* xbar = full + a.ring;  // [4] batch u's data has arrived (slot u % 4)
    long long* flg = reinterpret_cast<long long*>(xbar + 4);  // [1] patched, [2] stop
    const unsigned q = cluster_rank();
    const unsigned CS = gridDim.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = a.n;
    const int Ae = a.eval ? 1 : a.A;  // <= 16
    const int c0 = min(n, (int)q * a.slab), c1 = min(n, c0 + a.slab);
    constexpr int E = 16 / (int)sizeof(PT);
    using VT = typename std::conditional<sizeof(PT) == 4, float4, double2>::type;
    const int vhalf = sizeof(PT) == 4 ? ((n + 3) & ~3) / 2 : 0;
    auto vidx = [&](int j) { return vhalf ? ((j & 2) ? vhalf : 0) + ((j >> 2) << 1) + (j & 1) : j; };
    for (int j = t; j < n; j += kLThreads) {
        Vs[vidx(j)] = a.V[j];
        if (a.eval) pis[j] = a.pi[j];
    }
    const int64_t total = a.max_iter * (int64_t)n;  // batches of the launch
    // bytes batch u brings into every CTA: CS x Ae partials, plus Ae coefficients
    // from the owner of column s_{u-1} (none for the launch's first batch)
    auto xbytes = [&](int64_t u) { return (unsigned)((CS * Ae + (u > 0 ? Ae : 0)) * 8); };
    if (t == 0) {
        for (int s = 0; s < a.ring; ++s) mbar_init(full + s, 1);
        for (int s = 0; s < 4; ++s) mbar_init(xbar + s, 1);
        flg[1] = -1;
        flg[2] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (t == 0)  // slots armed for batches 0..3 (re-armed after each batch's combine)
        for (int s = 0; s < 4 && s < total; ++s) mbar_arrive_tx(xbar + s, xbytes(s));
    if (!a.identity)
        fill_order(n, a.seed, a.k0, a.order, a.perm + (a.k0 % 3) * n, (int64_t)q * kLThreads + t,
                   (int64_t)CS * kLThreads);
    cluster_sync();

    auto state_at = [&](int64_t u) -> int {
        const int64_t k = a.k0 + u / n;
        const int bi = (int)(u % n);
        return a.identity ? bi : (int)__ldcg(a.perm + (k % 3) * n + bi);
    };
    const PT* P = static_cast<const PT*>(a.P);
    long long status = RMB_ERR_NOT_CONVERGED;
    int64_t it = 0, batches = 0;
    double last = 0.0;
    int64_t consumed = 0, issued = 0;

    if (warp < kLComb) {
        // ---------------------------------------------- dot + issuing warps
        const int64_t last_sweep = a.k0 + a.max_iter - 1;
        int64_t pk = a.k0;
        int pb = 0;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        // the next sweep's order is filled in its predecessor's batch 0, visible
        // here once batch 0's patch is (acquired with patched >= batch 0 in the
        // sweep's batch 2; the refill at the top of batch 3 comes after it)
        auto may_issue = [&](int64_t cons_k, int cons_b) {
            return pk <= last_sweep && (pk == cons_k || (pk == cons_k + 1 && cons_b >= 3));
        };
        int pre_s = 0;
        bool pre_ok = false;
        auto issue_one = [&](int64_t cons_k, int cons_b) {
            if (pk > last_sweep) return;
            const int s = pre_ok ? pre_s : (lane < Ae ? state_at((pk - a.k0) * n + pb) : 0);
            const int act = lane < Ae ? (a.eval ? __ldcg(a.pi + s) : lane) : 0;
            const int slot = (int)(issued % a.ring);
            unsigned char* dst = ring + (size_t)slot * a.rows * a.row_bytes;
            const unsigned bytes = (unsigned)((c1 - c0) * (int)sizeof(PT));
            if (lane == 0) mbar_arrive_tx(full + slot, bytes * (unsigned)Ae);
            __syncwarp();
            if (lane < Ae && bytes > 0)
                bulk_g2s(dst + (size_t)lane * a.row_bytes, P + ((int64_t)s * a.A + act) * n + c0, bytes, full + slot, pol);
            ++issued;
            if (++pb == n) pb = 0, ++pk;
            pre_ok = may_issue(cons_k, cons_b) && pk <= last_sweep;
            if (pre_ok) pre_s = lane < Ae ? state_at((pk - a.k0) * n + pb) : 0;
        };
        if (warp == kCDot)
            for (int s = 0; s < a.ring && may_issue(a.k0, 0); ++s) issue_one(a.k0, 0);
        int s_prev = -1;
        int s_this = state_at(0);
        for (int64_t u = 0; u < total; ++u) {
            const int64_t k = a.k0 + u / n;
            const int bi = (int)(u % n);
            // refill the ring first (the slot of batch u-1 is free): the copies
            // must not wait for the patch below
            if (warp == kCDot)
                while (issued < consumed + a.ring && may_issue(k, bi)) issue_one(k, bi);
            if (bi == 0 && u > 0) {
                // a new sweep: the combine warp's verdict on the previous one first
                // (published with the patch of its last batch).  One thread reads
                // it and the group follows: per-warp reads could split the group
                // across the named barrier at the end of the batch
                if (t == 0) {
                    SpinGuard sg;
                    while (ld_acquire_cta(flg + 1) < u - 1) sg.tick();
                    flg[3] = ld_acquire_cta(flg + 2);
                }
                bar_sync_n<kLGroup>();
                if (flg[3] != 0) break;
            } else if (lane == 0) {  // V must hold batch u-2's value (batch u-1's column is left out)
                SpinGuard sg;
                while (ld_acquire_cta(flg + 1) < u - 2) sg.tick();
            }
            __syncwarp();
            const int s_next = u + 1 < total ? state_at(u + 1) : 0;  // in flight during this batch
            const int slot = (int)(consumed % a.ring);
            const unsigned ph = (unsigned)((consumed / a.ring) & 1);
            {
                SpinGuard sg;
                while (!mbar_try(full + slot, ph)) sg.tick();
            }
            const unsigned char* stg = ring + (size_t)slot * a.rows * a.row_bytes;
            const int nv = (c1 - c0) / E;
            const int jx = (s_prev >= c0 && s_prev < c1) ? s_prev - c0 : -1;  // column left out (this CTA's)
            double* xs = xb + (u % 4) * kXSlot;
            unsigned long long* xu = xbar + (u % 4);
            if (warp < kCDot && warp < Ae) {
                const bool two = warp + kCDot < Ae;
                const VT* row0 = reinterpret_cast<const VT*>(stg + (size_t)warp * a.row_bytes);
                const VT* row1 = reinterpret_cast<const VT*>(stg + (size_t)(warp + kCDot) * a.row_bytes);
                double acc0 = 0.0, acc1 = 0.0;
                for (int v = lane; v < nv; v += kWarp) {
                    const int j = c0 + v * E;
                    double vs[E];
                    if constexpr (sizeof(PT) == 4) {
                        const double2 lo = *reinterpret_cast<const double2*>(Vs + (j >> 1));
                        const double2 hi = *reinterpret_cast<const double2*>(Vs + vhalf + (j >> 1));
                        vs[0] = lo.x, vs[1] = lo.y, vs[2] = hi.x, vs[3] = hi.y;
                    } else {
                        const double2 x = *reinterpret_cast<const double2*>(Vs + j);
                        vs[0] = x.x, vs[1] = x.y;
                    }
                    // the left-out column: a select per element (a dynamic index
                    // would put vs[] in local memory)
#pragma unroll
                    for (int e = 0; e < E; ++e) vs[e] = (jx == v * E + e) ? 0.0 : vs[e];
                    const VT x0 = row0[v];
                    const double p0[4] = {(double)x0.x, (double)x0.y, sizeof(PT) == 4 ? (double)((const float*)&x0)[2] : 0.0,
                                          sizeof(PT) == 4 ? (double)((const float*)&x0)[3] : 0.0};
#pragma unroll
                    for (int e = 0; e < E; ++e) acc0 = fma(p0[e], vs[e], acc0);
                    if (two) {
                        const VT x1 = row1[v];
                        const double p1[4] = {(double)x1.x, (double)x1.y,
                                              sizeof(PT) == 4 ? (double)((const float*)&x1)[2] : 0.0,
                                              sizeof(PT) == 4 ? (double)((const float*)&x1)[3] : 0.0};
#pragma unroll
                        for (int e = 0; e < E; ++e) acc1 = fma(p1[e], vs[e], acc1);
                    }
                }
                acc0 = warp_sum(acc0);
                acc1 = warp_sum(acc1);
                // to every CTA: lane l < CS row `warp`, lane 16 + l row `warp + 8`
                const unsigned dst = lane & 15;
                if (dst < CS && (lane < 16 || two))
                    st_async_remote(xs + q * 16 + warp + (lane < 16 ? 0 : kCDot), lane < 16 ? acc0 : acc1, xu, dst);
            }
            if (jx >= 0 && t < 16 * 16) {  // the left-out column's P (owner): thread r + 16 d -> row r, CTA d
                const int r = t & 15, d = t >> 4;
                if (r < Ae && (unsigned)d < CS)
                    st_async_remote(xs + 16 * 16 + r,
                                    (double)reinterpret_cast<const PT*>(stg + (size_t)r * a.row_bytes)[jx], xu,
                                    (unsigned)d);
            }
            if (bi == 0 && !a.identity)  // the next sweep's order (covered by this batch's signal)
                fill_order(n, a.seed, k + 1, a.order, a.perm + ((k + 1) % 3) * n, (int64_t)q * kLGroup + t,
                           (int64_t)CS * kLGroup);
            bar_sync_n<kLGroup>();  // every warp is done with the ring slot
            ++consumed;
            s_prev = s_this;
            s_this = s_next;
        }
    } else {
        // ---------------------------------------------------- combine warp
        int L = 1;  // lanes per state in the argmin (pow2 >= Ae)
        while (L < Ae) L <<= 1;
        int s_cur = state_at(0), s_prev = -1;
        int s_nx = total > 1 ? state_at(1) : 0;
        auto cost = [&](int s) -> double {
            return lane < Ae ? (double)__ldg(static_cast<const PT*>(a.c) + (int64_t)s * a.A + (a.eval ? pis[s] : lane))
                             : 0.0;
        };
        double cc = cost(s_cur);
        double rmax = 0.0;
        int bad = 0;
        bool stop = false;
        // phase profile of CTA 0's combine warp: waiting for the dot warps,
        // correction + cluster exchange, combine + patch
        const bool prof = q == 0 && lane == 0;
        unsigned long long tm = prof ? globaltimer_ns() : 0, t_x = 0, t_cb = 0;
        auto mark = [&](unsigned long long& acc) {
            if (prof) {
                const unsigned long long now = globaltimer_ns();
                acc += now - tm;
                tm = now;
            }
        };
        for (int64_t u = 0; u < total && !stop; ++u) {
            const int bi = (int)(u % n);
            const double* xs = xb + (u % 4) * kXSlot;
            {
                SpinGuard sg;
                // st.async data is visible to the CTA once the mbarrier phase completes
                while (!mbar_try(xbar + (u % 4), (unsigned)((u / 4) & 1))) sg.tick();
            }
            mark(t_x);
            double Q = INFINITY;
            int arg = 0x7fffffff;
            if (lane < Ae) {
                double sum = 0.0;
                for (unsigned cq = 0; cq < CS; ++cq) sum += xs[cq * 16 + lane];  // CTA order
                if (u > 0) sum = fma(xs[16 * 16 + lane], Vs[vidx(s_prev)], sum);  // the left-out column
                Q = cc + a.gamma * sum;
                arg = a.eval ? pis[s_cur] : lane;
            }
            for (int o = 1; o < L; o <<= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, Q, o);
                const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
                if (ov < Q || (ov == Q && oa < arg)) Q = ov, arg = oa;
            }
            if (lane == 0) {
                rmax = fmax(rmax, fabs(Q - Vs[vidx(s_cur)]));
                bad |= !isfinite(Q);
                Vs[vidx(s_cur)] = Q;
                if (q == 0) {
                    a.V[s_cur] = Q;
                    if (!a.eval && a.pi) a.pi[s_cur] = arg;
                }
            }
            __syncwarp();
            if (bi == n - 1) {  // end of a sweep: every CTA holds the same residual
                const double r = __shfl_sync(0xffffffffu, rmax, 0);
                const int bb = __shfl_sync(0xffffffffu, bad, 0);
                if (q == 0 && lane == 0 && it < a.trace_len) a.trace[it] = r;
                if (a.etrace && it < a.etrace_len)
                    trace_error([&](int64_t j) { return Vs[vidx((int)j)]; }, a.vref, n, (int64_t)q * kWarp + lane,
                                (int64_t)CS * kWarp, a.etrace + it);
                ++it;
                last = r;
                rmax = 0.0;
                bad = 0;
                if (bb) status = RMB_ERR_NONFINITE, stop = true;
                else if (a.eps >= 0.0 && r <= a.eps) status = RMB_OK, stop = true;
                if (stop && lane == 0) flg[2] = 1;  // published by the release of this batch's patch
            }
            if (lane == 0) {
                if (u + 4 < total) mbar_arrive_tx(xbar + (u % 4), xbytes(u + 4));  // the slot, for batch u + 4
                st_release_cta(flg + 1, u);
            }
            mark(t_cb);
            ++batches;
            s_prev = s_cur;
            s_cur = s_nx;
            s_nx = u + 2 < total ? state_at(u + 2) : 0;
            cc = u + 1 < total ? cost(s_cur) : 0.0;
        }
        if (a.eps < 0.0 && status == RMB_ERR_NOT_CONVERGED) status = RMB_OK;
        if (lane == 0) st_release_cta(flg + 2, 1);  // the dot warps stop
        if (prof) {
            a.prof[0] = 0;
            a.prof[1] = (long long)t_x;    // waiting for the batch's partials from every CTA
            a.prof[2] = (long long)t_cb;   // combine + patch
        }
    }
    __syncthreads();
    // drain: bulk copies in flight must land before the CTA exits (the
    // issuing warp's lane 0 holds the issue count)
    if (warp == kCDot && lane == 0) {
        for (int64_t d = consumed; d < issued; ++d) {
            const int slot = (int)(d % a.ring);
            const unsigned ph = (unsigned)((d / a.ring) & 1);
            SpinGuard sg;
            while (!mbar_try(full + slot, ph)) sg.tick();
        }
    }
    cluster_sync();  // no CTA exits while another may still read its shared memory
    if (q == 0 && warp == kLComb && lane == 0) {
        a.out[OUT_SWEEPS] = it;
        a.out[OUT_OUTER] = 0;
        a.out[OUT_STATUS] = status;
        a.out[OUT_RESID_BITS] = __double_as_longlong(last);
        a.out[OUT_BATCHES] = batches;
        a.out[OUT_CHANGED] = 0;
        a.prof[3] = batches + 2;  // one cluster-wide exchange per batch + the barriers at both ends
        a.out[7] = 0;
    }
}

// The cluster path serves dense B_b / B_{pi,b} solves whose batches hold at
// most kCBatchRows rows and kClusterBatchBytes of P; returns false when the
// request is outside that envelope (the grid solver takes it).
constexpr int64_t kClusterBatchBytes = int64_t(2) << 20;

bool dense_cluster_eligible(const Problem& pr, const SolveRequest& rq)
{
    if (!pr.dense || pr.no_tma || pr.vglobal || rq.chunked || rq.fused) return false;
    if (pr.row_begin != 0 || pr.row_end != pr.n || pr.nccl_comm) return false;
    const bool eval = rq.mode == MODE_APPLY_PI || rq.mode == MODE_POLICY_VALUE;
    if (!(rq.mode == MODE_VI || rq.mode == MODE_APPLY || eval)) return false;
    const int psz = pr.pdt == RMB_F32 ? 4 : 8;
    const int64_t n = pr.n;
    if (n % (16 / psz) != 0 || (reinterpret_cast<uintptr_t>(pr.P) & 15u) != 0) return false;
    const int Ae = eval ? 1 : pr.A;
    if (rq.b >= n || rq.b * Ae > kCBatchRows) return false;
    if (rq.b * Ae * n * psz > kClusterBatchBytes) return false;
    return true;
}

template <typename PT>
static cudaError_t launch_cluster(const ClusterArgs& a, int CS, size_t smem, cudaStream_t st, bool la)
{
    auto kern = la ? dense_cluster_la_kernel<PT> : dense_cluster_kernel<PT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(la ? kLThreads : kCThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// largest cluster (16, else 8, ...) that can be scheduled with this shared memory
template <typename PT>
static int cluster_size(size_t smem)
{
    auto kern = dense_cluster_kernel<PT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs = 16; cs >= 1; cs >>= 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kCThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc >= 1) return cs;
        cudaGetLastError();
    }
    return 0;
}

rmb_status dense_cluster_solve(Problem& pr, const SolveRequest& rq, double* trace_dev, int64_t trace_len,
                               SolveResult* res)
{
    const int psz = pr.pdt == RMB_F32 ? 4 : 8;
    const int n = (int)pr.n;
    const bool eval = rq.mode == MODE_APPLY_PI || rq.mode == MODE_POLICY_VALUE;
    ClusterArgs a{};
    a.P = pr.P;
    a.c = pr.c;
    a.n = n;
    a.A = pr.A;
    a.gamma = pr.gamma;
    a.V = rq.V;
    a.pi = rq.pi;
    a.b = (int)rq.b;
    a.seed = rq.seed;
    a.k0 = rq.k0;
    a.identity = rq.identity && !rq.select ? 1 : 0;
    a.order = OrderSpec{rq.select, pr.sel_cum, pr.sel_W};
    a.vref = rq.vref;
    a.etrace = rq.etrace;
    a.etrace_len = rq.etrace_len;
    a.eval = eval ? 1 : 0;
    a.eps = rq.eps;
    a.max_iter = rq.max_iter;
    a.trace = trace_dev;
    a.trace_len = trace_len;
    const int E = 16 / psz;
    auto layout = [&](int CS, size_t& smem) {
        a.slab = ((n + CS - 1) / CS + E - 1) / E * E;
        a.row_bytes = (a.slab * psz + 127) / 128 * 128;
        size_t off = 0;
        auto take = [&](size_t bytes) {
            const size_t o = off;
            off = (off + bytes + 127) / 128 * 128;
            return (int64_t)o;
        };
        a.v_off = take((size_t)n * 8);
        a.pi_off = take(eval ? (size_t)n * 4 : 16);
        a.part_off = take(std::max<size_t>((size_t)2 * kCBatchRows * 8, (size_t)4 * (16 * 16 + 16) * 8));
        a.bar_off = take(32 * 8);  // ring mbarriers (<= 8), the b = 1 kernel's cluster mbarrier and flags
        const int64_t room = (int64_t)pr.smem_optin - (int64_t)off - 1024;
        const int Ae = eval ? 1 : pr.A;
        a.rows = (int)std::min<int64_t>(kCRowsMax, std::min<int64_t>(rq.b * Ae, room / (2 * a.row_bytes)));
        a.ring = (int)std::min<int64_t>(8, room / std::max<int64_t>(1, (int64_t)a.rows * a.row_bytes));
        a.ring_off = take((size_t)std::max(0, a.ring) * std::max(0, a.rows) * a.row_bytes);
        smem = off;
        return a.rows >= 1 && a.ring >= 2;
    };
    size_t smem = 0;
    int CS = 16;
    if (!layout(CS, smem)) return RMB_ERR_UNSUPPORTED;
    CS = pr.pdt == RMB_F32 ? cluster_size<float>(smem) : cluster_size<double>(smem);
    // at least ~256 columns per CTA: fewer CTAs for small n (less to synchronise)
    while (CS > 1 && (int64_t)CS * 256 > n) CS >>= 1;
    if (CS < 1) return RMB_ERR_UNSUPPORTED;
    if (!layout(CS, smem)) return RMB_ERR_UNSUPPORTED;
    if (pr.perm.ensure((size_t)3 * n * 4) != cudaSuccess || pr.ctrl.ensure(4096) != cudaSuccess) {
        set_error("cluster solver: workspace allocation failed");
        return RMB_ERR_OOM;
    }
    a.perm = static_cast<uint32_t*>(pr.perm.p);
    unsigned long long* ctrl = static_cast<unsigned long long*>(pr.ctrl.p);
    a.out = reinterpret_cast<long long*>(ctrl + 128);
    a.prof = reinterpret_cast<long long*>(ctrl + 192);
    cudaStream_t st = pr.stream;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaError_t ce = cudaMemsetAsync(ctrl, 0, 4096, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(e0, st);
    // Gauss-Seidel batches (b = 1, <= 16 rows): the look-ahead kernel
#ifndef RMB_AB_NO_CLUSTER_LA
    const bool la = rq.b == 1 && (eval ? 1 : pr.A) <= 16 && n >= 5;
#else
    const bool la = false;
#endif
    if (ce == cudaSuccess)
        ce = pr.pdt == RMB_F32 ? launch_cluster<float>(a, CS, smem, st, la) : launch_cluster<double>(a, CS, smem, st, la);
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
        set_error(std::string("cluster solver: ") + cudaGetErrorString(ce));
        return RMB_ERR_CUDA;
    }
    res->sweeps = out[OUT_SWEEPS];
    res->outer = 0;
    res->status = (int)out[OUT_STATUS];
    double d;
    memcpy(&d, &out[OUT_RESID_BITS], 8);
    res->final_resid = d;
    res->batches = out[OUT_BATCHES];
    res->changed = 0;
    res->ms = ms;
    res->launches = 1;
    for (int i = 0; i < 4; ++i) pr.prof[i] = out[OUT_N + i];
    pr.prof[0] += out[7];  // stream + dot = ring wait + the rest of the compute phase
    pr.last_launches = 1;
    if (getenv("RMB_CLUSTER_DEBUG")) fprintf(stderr, "cluster CS=%d ring=%d rows=%d slab=%d ring_wait_ns=%lld\n", CS, a.ring, a.rows, a.slab, out[7]);
    return RMB_OK;
}

}  // namespace rmb

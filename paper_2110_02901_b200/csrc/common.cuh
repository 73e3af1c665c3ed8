// common.cuh — device helpers shared by the rmb kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rmb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- loads
// P rows are streamed exactly once per sweep: bypass L1 allocation.
__device__ __forceinline__ float4 ld_stream(const float4* p)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_stream(const float* p)
{
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_stream(const double* p)
{
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// ------------------------------------------------------ L2 cache hints
// Sparse solves stream their CSR/ELL rows (hundreds of MB, random rows) past
// an interim V that must stay in L2 (8-34 MB per copy): rows are loaded with
// an evict_first policy, V gathers and writes with evict_last.
#ifndef RMB_AB_L2_FIRST  // A/B builds only (tools/): the policies actually used
#define RMB_AB_L2_FIRST "evict_first"
#endif
#ifndef RMB_AB_L2_LAST
#define RMB_AB_L2_LAST "evict_last"
#endif
__device__ __forceinline__ uint64_t l2_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::" RMB_AB_L2_FIRST ".b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::" RMB_AB_L2_LAST ".b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only streams (never written during the kernel): non-coherent path, no L1 allocation
__device__ __forceinline__ int ld_first(const int* p, uint64_t pol)
{
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float ld_first(const float* p, uint64_t pol)
{
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_first(const double* p, uint64_t pol)
{
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int4 ld_first(const int4* p, uint64_t pol)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float4 ld_first(const float4* p, uint64_t pol)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double2 ld_first(const double2* p, uint64_t pol)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
// short scattered rows (a few consecutive words each): L1-allocating, so the
// words of one row after the first hit the line its first word brought in
__device__ __forceinline__ int ld_rows(const int* p, uint64_t pol)
{
    int r;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float ld_rows(const float* p, uint64_t pol)
{
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_rows(const double* p, uint64_t pol)
{
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
// 32 bytes (one sector) per thread in one instruction (sm_100: 256-bit LDG)
__device__ __forceinline__ void ld_v8(const uint32_t* p, uint32_t (&w)[8])
{
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
// data written during the kernel by other CTAs (interim V, policies, permutations): L2 only (.cg)
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol)
{
    double r;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_keep(const int* p, uint64_t pol)
{
    int r;
    asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// ------------------------------------------------------------ grid barrier
// Sense-free monotonic barrier for a co-resident (cooperative) grid.
// bar[0] = arrival counter, bar[32] = released epoch (separate 256-B lines).
// Both zeroed by the host before the launch; each CTA keeps its own epoch.
struct GridBarrier {
    unsigned long long* arrive;
    unsigned long long* release;
    unsigned long long epoch;
    unsigned long long nblocks;
    int* error_flag;
};

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Hang guard: a barrier that waits more than 30 s means a broken grid
// (not all CTAs resident); trap instead of wedging the GPU.
#ifndef RMB_BARRIER_VARIANT
#define RMB_BARRIER_VARIANT 1
#endif
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v)
{
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// CTA-level barrier of the first NT threads (named barrier 1).  With NT ==
// blockDim.x it is __syncthreads(); kernels with a producer warp outside the
// first NT threads (dense TMA path) keep that warp out of every CTA barrier.
template <int NT>
__device__ __forceinline__ void bar_sync_n()
{
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

template <int NT = 0>
__device__ __forceinline__ void grid_sync(GridBarrier& g)
{
    auto csync = [] {
        if constexpr (NT == 0) __syncthreads();
        else bar_sync_n<NT>();
    };
    if (g.nblocks == 1) {  // single-CTA launch (small problems): a CTA barrier is the grid barrier
        csync();
        return;
    }
#if RMB_BARRIER_VARIANT == 1
    // arrive with a fire-and-forget release reduction, then poll the arrival
    // counter itself (no separate release flag round trip)
    csync();
    if (threadIdx.x == 0) {
        g.epoch += 1;
        const unsigned long long target = g.epoch * g.nblocks;
        red_release_add(g.arrive, 1ULL);
        unsigned long long t0 = 0;
        unsigned spins = 0;
        while (ld_acquire_gpu(g.arrive) < target) {
            if (++spins == 4096u) {
                spins = 0;
                unsigned long long t = globaltimer_ns();
                if (t0 == 0) t0 = t;
                else if (t - t0 > 30ull * 1000000000ull) {
                    atomicExch(g.error_flag, 1);
                    __trap();
                }
            }
        }
    }
    csync();
    return;
#endif
    csync();
    if (threadIdx.x == 0) {
        g.epoch += 1;
        const unsigned long long target = g.epoch * g.nblocks;
        __threadfence();
        unsigned long long v = atomicAdd(g.arrive, 1ULL) + 1ULL;
        if (v == target) {
            st_release_gpu(g.release, g.epoch);
        } else {
            unsigned long long t0 = 0;
            unsigned spins = 0;
            while (ld_acquire_gpu(g.release) < g.epoch) {
                if (++spins == 4096u) {
                    spins = 0;
                    unsigned long long t = globaltimer_ns();
                    if (t0 == 0) t0 = t;
                    else if (t - t0 > 30ull * 1000000000ull) {
                        atomicExch(g.error_flag, 1);
                        __trap();
                    }
                }
            }
        }
    }
    csync();
}

// ------------------------------------------- mbarrier / bulk-copy (TMA) helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned tx)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Hang guard for ring waits (a broken pipeline traps instead of wedging the GPU).
struct SpinGuard {
    unsigned spins = 0;
    unsigned long long t0 = 0;
    __device__ __forceinline__ void tick()
    {
        if (++spins == 8192u) {
            spins = 0;
            const unsigned long long t = globaltimer_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 20ull * 1000000000ull) __trap();
        }
    }
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ long long ld_acquire_cta(const long long* p)
{
    long long v;
    asm volatile("ld.acquire.cta.shared.b64 %0, [%1];" : "=l"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(long long* p, long long v)
{
    asm volatile("st.release.cta.shared.b64 [%0], %1;" ::"r"(smem_addr(p)), "l"(v) : "memory");
}


// ------------------------------------------------------------- error trace
// RMB_TRACE_ERROR_VS_REF: ||V - Vref||_inf over the entries j0, j0 + stride,
// ... < n (V read through get(j)), folded into *slot (>= 0 doubles order like
// their bits).  Every lane of every calling warp must call it (warp max).
template <typename Get>
__device__ __forceinline__ void trace_error(Get get, const double* vref, int64_t n, int64_t j0, int64_t stride,
                                            double* slot)
{
    double e = 0.0;
    for (int64_t j = j0; j < n; j += stride) e = fmax(e, fabs(get(j) - __ldg(vref + j)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if ((threadIdx.x & 31) == 0 && e > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(slot), (unsigned long long)__double_as_longlong(e));
}

// ------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (value, index) argmin within aligned groups of G lanes; ties -> lower index.
template <int G>
__device__ __forceinline__ void group_argmin(double& v, int& a)
{
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oa = __shfl_xor_sync(0xffffffffu, a, o);
        if (ov < v || (ov == v && oa < a)) {
            v = ov;
            a = oa;
        }
    }
}

}  // namespace rmb

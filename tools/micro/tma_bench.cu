// Microbenchmark: HBM streaming through a per-SM shared-memory ring filled by
// cp.async.bulk (one producer lane) and consumed by 16 warps, vs plain
// 128-bit LDG streaming.  Used to choose the dense TMA-path configuration.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, unsigned tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ bool mb_try(uint64_t* b, unsigned p) {
    uint32_t ok;
    asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(ok) : "r"(sa(b)), "r"(p) : "memory");
    return ok;
}
__device__ __forceinline__ bool mb_test(uint64_t* b, unsigned p) {
    uint32_t ok;
    asm volatile("{.reg .pred q; mbarrier.test_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(ok) : "r"(sa(b)), "r"(p) : "memory");
    return ok;
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

// mode: 0 = consumers wait with try_wait (all lanes), 1 = lane 0 test_wait spin + syncwarp, 2 = lane 0 try_wait + syncwarp
template <int MODE>
__global__ void __launch_bounds__(544, 1) ring_kernel(const float4* __restrict__ src, size_t nvec_total, int stage_bytes,
                                                      int nst, int copies, double* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nst * stage_bytes);
    uint64_t* empty = full + nst;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mb_init(full + i, 1); mb_init(empty + i, 16); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this CTA's contiguous slice, in stage-sized tiles
    const size_t per_cta = nvec_total / gridDim.x;
    const float4* base = src + per_cta * blockIdx.x;
    const int vec_stage = stage_bytes / 16;
    const size_t tiles = per_cta / vec_stage;
    if (threadIdx.x >= 512) {
        if (threadIdx.x != 512) return;
        int st = 0; unsigned ph = 0;
        const int cb = stage_bytes / copies;
        for (size_t t = 0; t < tiles; ++t) {
            while (!mb_try(empty + st, ph ^ 1u)) {}
            mb_arrive_tx(full + st, stage_bytes);
            const char* g = reinterpret_cast<const char*>(base + t * vec_stage);
            for (int c = 0; c < copies; ++c) bulk(sm + (size_t)st * stage_bytes + c * cb, g + (size_t)c * cb, cb, full + st);
            if (++st == nst) st = 0, ph ^= 1u;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    int st = 0; unsigned ph = 0;
    double acc = 0.0;
    for (size_t t = 0; t < tiles; ++t) {
        if (MODE == 0 || MODE == 3) { while (!mb_try(full + st, ph)) {} }
        else {
            if (lane == 0) { if (MODE == 1) while (!mb_test(full + st, ph)) {} else while (!mb_try(full + st, ph)) {} }
            __syncwarp();
            if (MODE == 1 || MODE == 2) { while (!mb_test(full + st, ph)) {} }  // acquire for all lanes (cheap, complete)
        }
        const float4* s4 = reinterpret_cast<const float4*>(sm + (size_t)st * stage_bytes);
        if (MODE == 3) {
            const double* Vs = reinterpret_cast<const double*>(sm + (size_t)nst * stage_bytes + 16 * nst);
            for (int v = threadIdx.x; v < vec_stage; v += 512) {
                float4 x = s4[v];
                const int j = (int)((t * vec_stage + v) % 2500) * 4;
                const double2 lo = *reinterpret_cast<const double2*>(Vs + (j >> 1));
                const double2 hi = *reinterpret_cast<const double2*>(Vs + 5000 + (j >> 1));
                acc = fma((double)x.x, lo.x, acc); acc = fma((double)x.y, lo.y, acc);
                acc = fma((double)x.z, hi.x, acc); acc = fma((double)x.w, hi.y, acc);
            }
        } else
        for (int v = threadIdx.x; v < vec_stage; v += 512) { float4 x = s4[v]; acc += (double)x.x + x.y + x.z + x.w; }
        __syncwarp();
        if (lane == 0) mb_arrive(empty + st);
        if (++st == nst) st = 0, ph ^= 1u;
    }
    if (acc == 1234.5) out[0] = acc;
}

// item pattern: items (s, group g) -> 4 rows of n floats, streamed as stages of 4 x (1024 floats)
template <int DYN>
__global__ void __launch_bounds__(544, 1) item_kernel(const float* __restrict__ P, int n, int nitems, int nst,
                                                      unsigned* ctr, double* out)
{
    constexpr int S = 16384;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nst * S);
    uint64_t* empty = full + nst;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mb_init(full + i, 1); mb_init(empty + i, 16); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int* nstage = reinterpret_cast<int*>(empty + nst);  // per stage: vectors per row (0 = end)
    if (threadIdx.x >= 512) {
        if (threadIdx.x != 512) return;
        int st = 0; unsigned ph = 0;
        int r = DYN ? (int)atomicAdd(ctr, 1u) : blockIdx.x;
        while (r < nitems) {
            const int rn = DYN ? (int)atomicAdd(ctr, 1u) : r + gridDim.x;
            const int s = r / 4, g = r % 4;
            const float* rows = P + ((size_t)s * 16 + g * 4) * n;
            for (int jt = 0; jt < n; jt += 1024) {
                const int cols = min(1024, n - jt);
                while (!mb_try(empty + st, ph ^ 1u)) {}
                nstage[st] = cols / 4;
                mb_arrive_tx(full + st, cols * 16);
                for (int q = 0; q < 4; ++q) bulk(sm + (size_t)st * S + q * 4096, rows + (size_t)q * n + jt, cols * 4, full + st);
                if (++st == nst) st = 0, ph ^= 1u;
            }
            r = rn;
        }
        while (!mb_try(empty + st, ph ^ 1u)) {}
        nstage[st] = 0;
        mb_arrive(full + st);
        return;
    }
    const int lane = threadIdx.x & 31;
    int st = 0; unsigned ph = 0;
    double acc = 0.0;
    while (true) {
        while (!mb_try(full + st, ph)) {}
        const int nv = nstage[st];
        if (nv == 0) break;
        const float4* s4 = reinterpret_cast<const float4*>(sm + (size_t)st * S);
        for (int h = 0; h < 2; ++h) {
            const int f = threadIdx.x + 512 * h, row = f / 256, v = f % 256;
            if (v < nv) { float4 x = s4[row * 256 + v]; acc += (double)x.x + x.y + x.z + x.w; }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(empty + st);
        if (++st == nst) st = 0, ph ^= 1u;
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(512, 1) ldg_kernel(const float4* __restrict__ src, size_t nvec_total, double* out)
{
    const size_t per_cta = nvec_total / gridDim.x;
    const float4* base = src + per_cta * blockIdx.x;
    double acc = 0.0;
    for (size_t v = threadIdx.x; v < per_cta; v += 512 * U) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (v + u * 512 < per_cta) ? __ldcs(base + v + u * 512) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (double)x[u].x + x[u].y + x[u].z + x[u].w;
    }
    if (acc == 1234.5) out[0] = acc;
}

int main(int argc, char** argv)
{
    const size_t bytes = (size_t)6 << 30;
    const size_t nvec = bytes / 16;
    float4* src; double* out;
    cudaMalloc(&src, bytes); cudaMalloc(&out, 8);
    cudaMemset(src, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("%-48s %8.3f ms  %7.0f GB/s %s\n", name, best, bytes / best / 1e6, err ? cudaGetErrorString(err) : "");
    };
    timeit([&] { ldg_kernel<8><<<sms, 512>>>(src, nvec, out); }, "ldg U=8 (8 x 16B per thread in flight)");
    timeit([&] { ldg_kernel<4><<<sms, 512>>>(src, nvec, out); }, "ldg U=4");
    {
        for (int S : {16384, 32768}) for (int D : {4, 6}) {
            if ((size_t)S * D > 140 * 1024) continue;
            size_t smem = (size_t)S * D + 16 * D + 80000;
            char name[128];
            snprintf(name, sizeof name, "ring S=%dK D=%d +V80KB, F2F+DFMA work", S / 1024, D);
            cudaFuncSetAttribute(ring_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            timeit([&] { ring_kernel<3><<<sms, 544, smem>>>(src, nvec, S, D, 4, out); }, name);
        }
    }
    {
        const int n = 10000;
        unsigned* ctr; cudaMalloc(&ctr, 4);
        for (int D : {4, 6}) {
            size_t smem = (size_t)16384 * D + 16 * D + 64;
            cudaFuncSetAttribute(item_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(item_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            char name[128];
            snprintf(name, sizeof name, "items 4 rows x 4KB, static, D=%d (6.4 GB)", D);
            timeit([&] { item_kernel<0><<<sms, 544, smem>>>((const float*)src, n, n * 4, D, ctr, out); }, name);
            snprintf(name, sizeof name, "items 4 rows x 4KB, dynamic, D=%d (6.4 GB)", D);
            timeit([&] { cudaMemsetAsync(ctr, 0, 4); item_kernel<1><<<sms, 544, smem>>>((const float*)src, n, n * 4, D, ctr, out); }, name);
        }
    }
    int stages[] = {16384};
    for (int S : stages) {
        for (int D : {2, 4, 6, 12}) {
            if ((size_t)S * D > 200 * 1024) continue;
            for (int copies : {1, 4}) {
                size_t smem = (size_t)S * D + 16 * D;
                char name[128];
                snprintf(name, sizeof name, "ring S=%dK D=%d copies=%d try", S / 1024, D, copies);
                cudaFuncSetAttribute(ring_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                timeit([&] { ring_kernel<0><<<sms, 544, smem>>>(src, nvec, S, D, copies, out); }, name);
                if (copies == 4 && S == 16384) {
                    cudaFuncSetAttribute(ring_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    snprintf(name, sizeof name, "ring S=%dK D=%d copies=%d lane0 test", S / 1024, D, copies);
                    timeit([&] { ring_kernel<1><<<sms, 544, smem>>>(src, nvec, S, D, copies, out); }, name);
                    cudaFuncSetAttribute(ring_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    snprintf(name, sizeof name, "ring S=%dK D=%d copies=%d lane0 try", S / 1024, D, copies);
                    timeit([&] { ring_kernel<2><<<sms, 544, smem>>>(src, nvec, S, D, copies, out); }, name);
                }
            }
        }
    }
    return 0;
}

// gen_kernels.cu — device-side instance generation (gen/rmb_gen.h), the
// device partition kernel, and the RMB_VALIDATE check kernel.
#include <cuda_runtime.h>

#include "../../gen/rmb_gen.h"
#include "internal.h"
#include "partition.cuh"

namespace rmb {

// ------------------------------------------------------------- partition
__global__ void partition_kernel(int64_t n, uint64_t seed, int64_t sweep, int identity, uint32_t* perm)
{
    Permutation pm;
    pm.init(n, seed, sweep);
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        perm[p] = identity ? (uint32_t)p : (uint32_t)pm((uint64_t)p);
}

cudaError_t launch_partition(int64_t n, uint64_t seed, int64_t sweep, bool identity, uint32_t* perm,
                             cudaStream_t st)
{
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    partition_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, seed, sweep, identity ? 1 : 0, perm);
    return cudaGetLastError();
}

// ------------------------------------------------------------- selection
__global__ void select_kernel(int64_t n, uint64_t seed, int64_t sweep, OrderSpec os, uint32_t* sel)
{
    fill_order(n, seed, sweep, os, sel, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

cudaError_t launch_select(int64_t n, uint64_t seed, int64_t sweep, int sel, const uint64_t* cum, uint64_t W,
                          uint32_t* out, cudaStream_t st)
{
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    select_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, seed, sweep, OrderSpec{sel, cum, W}, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------- dense gen
// one warp per (s, a) row: exact integer row sum, then the normalised row
template <typename T>
__global__ void gen_dense_kernel(int kind, uint64_t seed, int64_t n, int A, int64_t s0, int64_t s1, T* P, T* c)
{
    const int lane = threadIdx.x & 31;
    const int64_t rows = (s1 - s0) * A;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < rows; r += nw) {
        const int64_t s = s0 + r / A;
        const int a = (int)(r % A);
        T* row = P + r * n;
        if (kind == RMBGEN_DENSE_RANDOM) {
            unsigned long long W = 0;
            for (int64_t j = lane; j < n; j += 32) W += rmbgen_dense_w(seed, s, a, j);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
            for (int64_t j = lane; j < n; j += 32) row[j] = (T)rmbgen_dense_p(seed, s, a, j, W);
            if (lane == 0) c[r] = (T)rmbgen_cost_u01(seed, s, a);
        } else {
            for (int64_t j = lane; j < n; j += 32) row[j] = (T)rmbgen_dyadic_p(seed, n, s, a, j);
            if (lane == 0) c[r] = (T)rmbgen_dyadic_cost(seed, s, a);
        }
    }
}

// ------------------------------------------------------------ sparse gen
template <typename T>
__global__ void gen_sparse_kernel(uint64_t seed, int64_t n, int A, int K, int64_t s0, int64_t s1,
                                  int64_t* row_ptr, int32_t* col, T* val, T* c)
{
    const int64_t rows = (s1 - s0) * A;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = s0 + r / A;
        const int a = (int)(r % A);
        unsigned long long W = 0;
        for (int q = 0; q < K; ++q) W += rmbgen_sparse_w(seed, s, a, q);
        for (int q = 0; q < K; ++q) {
            const int64_t e = r * K + q;
            col[e] = (int32_t)rmbgen_sparse_col(seed, n, K, s, a, q);
            val[e] = (T)((double)rmbgen_sparse_w(seed, s, a, q) / (double)W);
        }
        c[r] = (T)rmbgen_cost_u01(seed, s, a);
        row_ptr[r] = r * K;
        if (r == rows - 1) row_ptr[rows] = rows * K;
    }
}

template <typename T>
__global__ void gen_grid_kernel(int64_t N, int64_t s0, int64_t s1, int64_t* row_ptr, int32_t* col, T* val, T* c)
{
    const int64_t rows = (s1 - s0) * 4;
    const int K = RMBGEN_GRID_W;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = s0 + r / 4;
        const int a = (int)(r % 4);
        for (int q = 0; q < K; ++q) {
            col[r * K + q] = (int32_t)rmbgen_grid_slot_col(N, s, q);
            val[r * K + q] = (T)rmbgen_grid_p(N, s, a, q);
        }
        c[r] = (T)rmbgen_grid_cost(s);
        row_ptr[r] = r * K;
        if (r == rows - 1) row_ptr[rows] = rows * K;
    }
}

static unsigned grid_for(int64_t work, int per_block)
{
    int64_t b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

// ------------------------------------------------------------- validation
// bad |= 1: row sum off by more than tol; 2: column out of range; 4: nonfinite cost/prob
template <typename T>
__global__ void validate_dense_kernel(const T* P, const T* c, int64_t n, int64_t rows, double tol, int* bad)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < rows; r += nw) {
        double s = 0.0;
        int f = 0;
        for (int64_t j = lane; j < n; j += 32) {
            const double p = (double)P[r * n + j];
            s += p;
            f |= !(p >= 0.0 && p <= 1.0 + tol);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            f |= __shfl_xor_sync(0xffffffffu, f, o);
        }
        if (lane == 0) {
            int e = 0;
            if (fabs(s - 1.0) > tol) e |= 1;
            if (f) e |= 4;
            if (!isfinite((double)c[r])) e |= 4;
            if (e) atomicOr(bad, e);
        }
    }
}

template <typename T>
__global__ void validate_csr_kernel(const int64_t* row_ptr, const int32_t* col, const T* val, const T* c,
                                    int64_t n, int64_t rows, double tol, int* bad)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        int e = 0;
        const int64_t b0 = row_ptr[r], b1 = row_ptr[r + 1];
        if (b1 < b0) e |= 2;
        for (int64_t k = b0; k < b1; ++k) {
            const double p = (double)val[k];
            s += p;
            if (!(p >= 0.0 && p <= 1.0 + tol)) e |= 4;
            if (col[k] < 0 || col[k] >= n) e |= 2;
        }
        if (fabs(s - 1.0) > tol) e |= 1;
        if (!isfinite((double)c[r])) e |= 4;
        if (e) atomicOr(bad, e);
    }
}

cudaError_t launch_validate(const Problem& pr, int* bad, cudaStream_t st)
{
    const int64_t rows = (pr.row_end - pr.row_begin) * pr.A;  // owned rows
    const double tol = pr.pdt == RMB_F64 ? 1e-9 : 1e-5;
    if (rows == 0) return cudaMemsetAsync(bad, 0, sizeof(int), st);
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (pr.dense) {
        if (pr.pdt == RMB_F32)
            validate_dense_kernel<float><<<grid_for(rows * 32, 256), 256, 0, st>>>(
                (const float*)pr.P, (const float*)pr.c, pr.n, rows, tol, bad);
        else
            validate_dense_kernel<double><<<grid_for(rows * 32, 256), 256, 0, st>>>(
                (const double*)pr.P, (const double*)pr.c, pr.n, rows, tol, bad);
    } else {
        if (pr.pdt == RMB_F32)
            validate_csr_kernel<float><<<grid_for(rows, 256), 256, 0, st>>>(
                pr.row_ptr, pr.col, (const float*)pr.val, (const float*)pr.c, pr.n, rows, tol, bad);
        else
            validate_csr_kernel<double><<<grid_for(rows, 256), 256, 0, st>>>(
                pr.row_ptr, pr.col, (const double*)pr.val, (const double*)pr.c, pr.n, rows, tol, bad);
    }
    return cudaGetLastError();
}

}  // namespace rmb

// ------------------------------------------------------------ C entry points
using namespace rmb;

extern "C" rmb_status rmb_generate_dense(int32_t kind, uint64_t seed, int64_t n, int32_t A, int64_t s0, int64_t s1,
                                         rmb_dtype dtype, void* P, void* c, void* stream)
{
    if (n < 1 || A < 1 || s0 < 0 || s1 > n || s0 >= s1 || !P || !c || (kind != 0 && kind != 1) ||
        (dtype != RMB_F32 && dtype != RMB_F64)) {
        set_error("rmb_generate_dense: invalid argument");
        return RMB_ERR_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = (s1 - s0) * A;
    if (dtype == RMB_F32)
        gen_dense_kernel<float><<<grid_for(rows * 32, 256), 256, 0, st>>>(kind, seed, n, A, s0, s1, (float*)P, (float*)c);
    else
        gen_dense_kernel<double><<<grid_for(rows * 32, 256), 256, 0, st>>>(kind, seed, n, A, s0, s1, (double*)P, (double*)c);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_error(std::string("rmb_generate_dense: ") + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    }
    return RMB_OK;
}

extern "C" rmb_status rmb_generate_sparse(uint64_t seed, int64_t n, int32_t A, int32_t K, int64_t s0, int64_t s1,
                                          rmb_dtype dtype, int64_t* row_ptr, int32_t* col, void* val, void* c,
                                          void* stream)
{
    if (n < 1 || A < 1 || K < 1 || K > n || s0 < 0 || s1 > n || s0 >= s1 || !row_ptr || !col || !val || !c ||
        (dtype != RMB_F32 && dtype != RMB_F64)) {
        set_error("rmb_generate_sparse: invalid argument");
        return RMB_ERR_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = (s1 - s0) * A;
    if (dtype == RMB_F32)
        gen_sparse_kernel<float><<<grid_for(rows, 256), 256, 0, st>>>(seed, n, A, K, s0, s1, row_ptr, col, (float*)val, (float*)c);
    else
        gen_sparse_kernel<double><<<grid_for(rows, 256), 256, 0, st>>>(seed, n, A, K, s0, s1, row_ptr, col, (double*)val, (double*)c);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_error(std::string("rmb_generate_sparse: ") + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    }
    return RMB_OK;
}

extern "C" rmb_status rmb_generate_grid(int64_t N, int64_t s0, int64_t s1, rmb_dtype dtype, int64_t* row_ptr,
                                        int32_t* col, void* val, void* c, void* stream)
{
    if (N < 2 || s0 < 0 || s1 > N * N || s0 >= s1 || !row_ptr || !col || !val || !c ||
        (dtype != RMB_F32 && dtype != RMB_F64)) {
        set_error("rmb_generate_grid: invalid argument");
        return RMB_ERR_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = (s1 - s0) * 4;
    if (dtype == RMB_F32)
        gen_grid_kernel<float><<<grid_for(rows, 256), 256, 0, st>>>(N, s0, s1, row_ptr, col, (float*)val, (float*)c);
    else
        gen_grid_kernel<double><<<grid_for(rows, 256), 256, 0, st>>>(N, s0, s1, row_ptr, col, (double*)val, (double*)c);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_error(std::string("rmb_generate_grid: ") + cudaGetErrorString(e));
        return RMB_ERR_CUDA;
    }
    return RMB_OK;
}

namespace rmb {
// Policy range check: *bad = 1 if some pi[s], s in [lo, hi), is outside [0, A)
// (an out-of-range action would index a row beyond P).
__global__ void check_policy_kernel(const int32_t* pi, int64_t lo, int64_t hi, int A, int* bad)
{
    for (int64_t s = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < hi; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = pi[s];
        if (a < 0 || a >= A) atomicExch(bad, 1);
    }
}

cudaError_t launch_check_policy(const int32_t* pi, int64_t lo, int64_t hi, int A, int* bad, cudaStream_t st)
{
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (e != cudaSuccess || hi <= lo) return e;
    check_policy_kernel<<<grid_for(hi - lo, 256), 256, 0, st>>>(pi, lo, hi, A, bad);
    return cudaGetLastError();
}
}  // namespace rmb

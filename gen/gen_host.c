/*
 * gen/gen_host.c — host (CPU) instance generators built from gen/rmb_gen.h.
 * Used by tests/, the oracle-side of parity checks and bench.py's CPU legs.
 * Holds none of the method's arithmetic (see rmb_gen.h header).
 */
#include <stdint.h>
#include <stddef.h>
#include "rmb_gen.h"

/* Dense [rows s0..s1)[A][n] block of P plus c[s0..s1)[A].
 * kind: RMBGEN_DENSE_RANDOM or RMBGEN_DENSE_DYADIC. f32 != 0 -> float storage. */
int gen_dense_rows(int kind, uint64_t seed, int64_t n, int32_t A, int64_t s0, int64_t s1,
                   int f32, void* P, void* c)
{
    if (n <= 0 || A <= 0 || s0 < 0 || s1 > n || s0 > s1) return 1;
    if (kind != RMBGEN_DENSE_RANDOM && kind != RMBGEN_DENSE_DYADIC) return 1;
    /* rows are independent: threads over states (each row's content is a
       function of (seed, s, a, j) only) */
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = s0; s < s1; ++s) {
        for (int32_t a = 0; a < A; ++a) {
            size_t row = (size_t)((s - s0) * A + a);
            double cost;
            if (kind == RMBGEN_DENSE_RANDOM) {
                uint64_t W = 0;
                for (int64_t j = 0; j < n; ++j) W += rmbgen_dense_w(seed, s, a, j);
                for (int64_t j = 0; j < n; ++j) {
                    double p = rmbgen_dense_p(seed, s, a, j, W);
                    if (f32) ((float*)P)[row * (size_t)n + (size_t)j] = (float)p;
                    else ((double*)P)[row * (size_t)n + (size_t)j] = p;
                }
                cost = rmbgen_cost_u01(seed, s, a);
            } else if (kind == RMBGEN_DENSE_DYADIC) {
                for (int64_t j = 0; j < n; ++j) {
                    double p = rmbgen_dyadic_p(seed, n, s, a, j);
                    if (f32) ((float*)P)[row * (size_t)n + (size_t)j] = (float)p;
                    else ((double*)P)[row * (size_t)n + (size_t)j] = p;
                }
                cost = rmbgen_dyadic_cost(seed, s, a);
            }
            if (f32) ((float*)c)[row] = (float)cost;
            else ((double*)c)[row] = cost;
        }
    }
    return 0;
}

/* Sparse random rows s0..s1 in fixed-width CSR (= ELL): K successors per (s,a).
 * row_ptr has (s1-s0)*A+1 entries (relative to the block), col int32, val f32/f64. */
int gen_sparse_rows(uint64_t seed, int64_t n, int32_t A, int32_t K, int64_t s0, int64_t s1,
                    int f32, int64_t* row_ptr, int32_t* col, void* val, void* c)
{
    if (n <= 0 || A <= 0 || K <= 0 || K > n || s0 < 0 || s1 > n || s0 > s1) return 1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t s = s0; s < s1; ++s) {
        for (int32_t a = 0; a < A; ++a) {
            size_t row = (size_t)((s - s0) * A + a);
            uint64_t W = 0;
            for (int32_t q = 0; q < K; ++q) W += rmbgen_sparse_w(seed, s, a, q);
            for (int32_t q = 0; q < K; ++q) {
                size_t e = row * (size_t)K + (size_t)q;
                col[e] = (int32_t)rmbgen_sparse_col(seed, n, K, s, a, q);
                double p = (double)rmbgen_sparse_w(seed, s, a, q) / (double)W;
                if (f32) ((float*)val)[e] = (float)p;
                else ((double*)val)[e] = p;
            }
            double cost = rmbgen_cost_u01(seed, s, a);
            if (f32) ((float*)c)[row] = (float)cost;
            else ((double*)c)[row] = cost;
        }
    }
    if (row_ptr)
        for (int64_t r = 0; r <= (s1 - s0) * A; ++r) row_ptr[r] = r * K;
    return 0;
}

/* Gridworld N x N, 4 actions, ELL width 5, rows s0..s1. */
int gen_grid_rows(int64_t N, int64_t s0, int64_t s1, int f32, int64_t* row_ptr, int32_t* col,
                  void* val, void* c)
{
    const int32_t A = 4, K = RMBGEN_GRID_W;
    int64_t n = N * N;
    if (N <= 1 || s0 < 0 || s1 > n || s0 > s1) return 1;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t s = s0; s < s1; ++s) {
        for (int32_t a = 0; a < A; ++a) {
            size_t row = (size_t)((s - s0) * A + a);
            for (int32_t q = 0; q < K; ++q) {
                size_t e = row * (size_t)K + (size_t)q;
                col[e] = (int32_t)rmbgen_grid_slot_col(N, s, q);
                double p = rmbgen_grid_p(N, s, a, q);
                if (f32) ((float*)val)[e] = (float)p;
                else ((double*)val)[e] = p;
            }
            double cost = rmbgen_grid_cost(s);
            if (f32) ((float*)c)[row] = (float)cost;
            else ((double*)c)[row] = cost;
        }
    }
    if (row_ptr)
        for (int64_t r = 0; r <= (s1 - s0) * A; ++r) row_ptr[r] = r * K;
    return 0;
}

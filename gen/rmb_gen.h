/*
 * gen/rmb_gen.h — seeded synthetic MDP instance generators.
 *
 * This module is the ONE piece of code shared by the CUDA product path
 * (paper_2110_02901_b200/csrc/gen_kernels.cu, device-side generation of
 * multi-GB instances) and the CPU oracle side (gen/gen_host.c, used by tests
 * and bench.py's cpu_baseline).  It holds none of the method's arithmetic:
 * no Bellman backup, no partition, no residual.  It only defines WHAT instance
 * a (seed, shape) pair denotes, so that both sides see bit-identical inputs.
 *
 * The shapes follow BASELINE.json's configs and the paper's workloads
 * (Sec. IV-A): random dense MDPs, sparse random MDPs with a
 * fixed number of successors, and a 2-D gridworld "maze" with slip.
 *
 * All hashing is a SplitMix64-style finaliser over (seed, indices); all
 * floating point is a single correctly rounded IEEE division or an exact
 * scaling, so host (gcc, no fast-math) and device (nvcc default, prec-div)
 * produce identical bits.
 *
 * Portable C99 header: compiles under gcc and nvcc.
 */
#ifndef RMB_GEN_H
#define RMB_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define RMBGEN_HD __host__ __device__ __forceinline__
#else
#define RMBGEN_HD static inline
#endif

/* Domain tags keep the streams for weights, successors and costs apart. */
#define RMBGEN_TAG_W    0x5741454947485453ULL /* weights          */
#define RMBGEN_TAG_COL  0x434f4c554d4e5353ULL /* successor choice */
#define RMBGEN_TAG_COST 0x434f535453535353ULL /* stage costs      */

/* Instance kinds (argument `kind` of the generators). */
#define RMBGEN_DENSE_RANDOM 0 /* w ~ U{1..2^24}, P = w / sum(w), c ~ U[0,1)           */
#define RMBGEN_DENSE_DYADIC 1 /* P = multiples of 1/4 on <=4 columns, c in {0..3}      */

RMBGEN_HD uint64_t rmbgen_fmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

RMBGEN_HD uint64_t rmbgen_h3(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t h = rmbgen_fmix(seed ^ tag);
    h = rmbgen_fmix(h ^ a);
    h = rmbgen_fmix(h ^ b);
    return rmbgen_fmix(h ^ c);
}

/* ---------------- dense random (configs 1, 2, 5) ----------------------- */

/* Integer weight of P(j | s, a) before normalisation: in [1, 2^24]. */
RMBGEN_HD uint64_t rmbgen_dense_w(uint64_t seed, int64_t s, int32_t a, int64_t j)
{
    return (rmbgen_h3(seed, RMBGEN_TAG_W, (uint64_t)s, (uint64_t)a, (uint64_t)j) >> 40) + 1ULL;
}

/* Stage cost c(s,a) ~ U[0,1) with 53 random bits (exact). */
RMBGEN_HD double rmbgen_cost_u01(uint64_t seed, int64_t s, int32_t a)
{
    uint64_t h = rmbgen_h3(seed, RMBGEN_TAG_COST, (uint64_t)s, (uint64_t)a, 0);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

/* P(j|s,a) in fp64 given the exact integer row sum W(s,a) = sum_j w. */
RMBGEN_HD double rmbgen_dense_p(uint64_t seed, int64_t s, int32_t a, int64_t j, uint64_t W)
{
    return (double)rmbgen_dense_w(seed, s, a, j) / (double)W;
}

/* Dyadic dense instance: four quarter-units of mass dropped on columns
 * h(q) mod n, q = 0..3 (repeats accumulate), integer cost in {0,1,2,3}.
 * With gamma = 1/2 every Bellman product and partial sum is exact in fp64
 * for many sweeps, so any summation order yields identical bits. */
RMBGEN_HD double rmbgen_dyadic_p(uint64_t seed, int64_t n, int64_t s, int32_t a, int64_t j)
{
    double p = 0.0;
    for (int q = 0; q < 4; ++q) {
        uint64_t h = rmbgen_h3(seed, RMBGEN_TAG_COL, (uint64_t)s, (uint64_t)a, (uint64_t)q);
        if ((int64_t)(h % (uint64_t)n) == j) p += 0.25;
    }
    return p;
}

RMBGEN_HD double rmbgen_dyadic_cost(uint64_t seed, int64_t s, int32_t a)
{
    return (double)(rmbgen_h3(seed, RMBGEN_TAG_COST, (uint64_t)s, (uint64_t)a, 7) & 3ULL);
}

/* ---------------- sparse random, fixed K successors (config 3) ---------- */

/* Stratified successor choice: slot q of row (s,a) lies in stratum
 * [floor(q*n/K), floor((q+1)*n/K)), so the K successors are distinct and
 * sorted ascending.  Requires K <= n. */
RMBGEN_HD int64_t rmbgen_sparse_col(uint64_t seed, int64_t n, int32_t K, int64_t s, int32_t a, int32_t q)
{
    int64_t lo = ((int64_t)q * n) / K;       /* n*K < 2^63 for every config */
    int64_t hi = ((int64_t)(q + 1) * n) / K;
    uint64_t h = rmbgen_h3(seed, RMBGEN_TAG_COL, (uint64_t)s, (uint64_t)a, (uint64_t)q);
    return lo + (int64_t)(h % (uint64_t)(hi - lo));
}

RMBGEN_HD uint64_t rmbgen_sparse_w(uint64_t seed, int64_t s, int32_t a, int32_t q)
{
    return (rmbgen_h3(seed, RMBGEN_TAG_W, (uint64_t)s, (uint64_t)a, (uint64_t)q) >> 40) + 1ULL;
}

/* ---------------- 2-D gridworld with slip (config 4) -------------------- */
/* N x N open grid, state s = r*N + col, actions 0:N(r-1) 1:S(r+1) 2:W(col-1)
 * 3:E(col+1).  Goal = state 0 (a corner): cost 0, absorbing.  Elsewhere cost
 * 1; the intended neighbour gets 0.7 (stay if it is off-grid); the remaining
 * 0.3 is spread uniformly over {stay} U {the other in-grid neighbours}.
 * (PAPER.md L492 leaves the law unstated; reading R-grid.)
 * ELL layout, width 5, fixed slot order {stay, N, S, W, E}; off-grid slots
 * carry probability 0 and point at s itself. */
#define RMBGEN_GRID_W 5

RMBGEN_HD int64_t rmbgen_grid_slot_col(int64_t N, int64_t s, int32_t slot)
{
    int64_t r = s / N, q = s % N;
    switch (slot) {
    case 1: return r > 0 ? s - N : s;
    case 2: return r < N - 1 ? s + N : s;
    case 3: return q > 0 ? s - 1 : s;
    case 4: return q < N - 1 ? s + 1 : s;
    default: return s;
    }
}

RMBGEN_HD int rmbgen_grid_slot_valid(int64_t N, int64_t s, int32_t slot)
{
    int64_t r = s / N, q = s % N;
    switch (slot) {
    case 1: return r > 0;
    case 2: return r < N - 1;
    case 3: return q > 0;
    case 4: return q < N - 1;
    default: return 1;
    }
}

/* probability stored in ELL slot `slot` of row (s, a) */
RMBGEN_HD double rmbgen_grid_p(int64_t N, int64_t s, int32_t a, int32_t slot)
{
    if (s == 0) return slot == 0 ? 1.0 : 0.0; /* goal: absorbing */
    int intended = a + 1;                      /* slot of the intended move */
    int cnt = 1;                               /* stay */
    for (int q = 1; q <= 4; ++q)
        if (q != intended && rmbgen_grid_slot_valid(N, s, q)) ++cnt;
    double p_other = 0.3 / (double)cnt;
    int intended_valid = rmbgen_grid_slot_valid(N, s, intended);
    if (slot == 0) return intended_valid ? p_other : 0.7 + p_other;
    if (!rmbgen_grid_slot_valid(N, s, slot)) return 0.0;
    if (slot == intended) return 0.7;
    return p_other;
}

RMBGEN_HD double rmbgen_grid_cost(int64_t s)
{
    return s == 0 ? 0.0 : 1.0;
}

#endif /* RMB_GEN_H */

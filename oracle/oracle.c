/*
 * oracle/oracle.c — plain CPU oracle for the randomized mini-batch operator
 * of arXiv 2110.02901 (Gargiani, Martinelli, Ruts Martinez, Lygeros).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.
 * The product path (paper_2110_02901_b200/, include/rmb.h) never links,
 * includes or calls anything here, and this file includes nothing from it.
 *
 * Plain, slow, obviously correct:
 *   - fp64 arithmetic throughout; P/c may be *stored* as float (converted
 *     exactly to double on load);
 *   - every row sum is accumulated sequentially in storage order (dense: j
 *     ascending; CSR: row order), Q = c + gamma * sum;
 *   - no blocking, fusion or reordering.  Optional worker threads
 *     (orc_set_threads, OpenMP) split the states of ONE batch (or of the
 *     improvement) among workers; each state's backup is still one
 *     sequential row sum written to its own slot, and every reduction
 *     (residual max, changed count) stays a sequential loop afterwards,
 *     so results are bitwise independent of the thread count.
 *
 * References are PAPER.md line numbers ("P:Lxxx") with the equation /
 * algorithm they fall in, and the DESIGN.md readings R1..R21 (= SURVEY
 * 8(c) A1..A21) where the paper is silent.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py
 * against values that do not come from this file (closed forms, brute force,
 * worked examples, textbook special cases, invariants).
 * "Oracle pins".
 */
#include <math.h>
#include <omp.h>
/* the shared instance definition (no method arithmetic): rows of the dense
   random instance are regenerated on the fly by orc_bellman_residual_dense_gen */
#include "../gen/rmb_gen.h"
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes — the same numbers as the product ABI documents, restated */
#define ORC_OK 0
#define ORC_INVALID_ARG 1
#define ORC_NOT_CONVERGED 3
#define ORC_NONFINITE 4
#define ORC_OOM 7

/* Worker threads for the within-batch loops (1 = plain sequential). */
static int orc_nthreads = 1;
void orc_set_threads(int w) { orc_nthreads = w < 1 ? 1 : w; }
int orc_get_threads(void) { return orc_nthreads; }

/* ------------------------------------------------------------------ */
/* MDP description (Sec. II-A: the tuple (S, U, P, g, alpha)).  */
/* Uniform |A| actions per state (reading R19: inadmissible controls   */
/* are encoded by duplicating an admissible row).                      */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n;        /* |S|                                             */
    int32_t A;        /* |U(i)| (uniform)                                */
    int32_t kind;     /* 0 = dense P[n][A][n], 1 = CSR rows r = s*A + a  */
    double gamma;     /* alpha in (0,1)                                  */
    int32_t p_f32;    /* P / val stored as float (1) or double (0)       */
    int32_t c_f32;    /* c stored as float (1) or double (0)             */
    const void* P;    /* dense transition probabilities                  */
    const int64_t* row_ptr; /* CSR [n*A+1]                               */
    const int32_t* col;     /* CSR [nnz]                                 */
    const void* val;        /* CSR [nnz]                                 */
    const void* c;    /* stage cost g(i,u), [n][A]                        */
} orc_mdp;

static double ld(const void* p, int f32, size_t i)
{
    return f32 ? (double)((const float*)p)[i] : ((const double*)p)[i];
}

/* ------------------------------------------------------------------ */
/* Partition (reading R2): the paper shuffles the states */
/* "before every evaluation of the operators" and processes    */
/* them in ascending order of their random index.  We fix the  */
/* shuffle as a counter-based permutation pi_k(p) of [0,n): SplitMix64  */
/* round keys, 6 balanced Feistel rounds on w = max(2,bitlen(n-1))      */
/* (rounded up to even) bits, cycle walking into [0,n).                 */
/* ------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t rk[6];
    int h;
    uint64_t mask;
} orc_feistel;

static void feistel_init(orc_feistel* f, int64_t n, uint64_t seed, int64_t k)
{
    int w = 0;
    uint64_t x = (uint64_t)(n - 1);
    while (x) { ++w; x >>= 1; }   /* bitlen(n-1) */
    if (w < 2) w = 2;
    if (w & 1) ++w;
    f->h = w / 2;
    f->mask = (f->h >= 64) ? ~0ULL : ((1ULL << f->h) - 1ULL);
    uint64_t key = orc_mix64(orc_mix64(seed) ^ (uint64_t)k);
    for (int r = 0; r < 6; ++r) f->rk[r] = orc_mix64(key ^ (uint64_t)r);
}

static uint64_t feistel_enc(const orc_feistel* f, uint64_t x)
{
    uint64_t L = x >> f->h, R = x & f->mask;
    for (int r = 0; r < 6; ++r) {
        uint64_t nl = R;
        uint64_t nr = L ^ (orc_mix64(f->rk[r] ^ R) >> (64 - f->h));
        L = nl;
        R = nr;
    }
    return (L << f->h) | R;
}

static uint64_t feistel_dec(const orc_feistel* f, uint64_t x)
{
    uint64_t L = x >> f->h, R = x & f->mask;
    for (int r = 5; r >= 0; --r) {
        /* forward: (L', R') = (R, L ^ F(R))  =>  R = L', L = R' ^ F(L') */
        uint64_t pr = L;
        uint64_t pl = R ^ (orc_mix64(f->rk[r] ^ L) >> (64 - f->h));
        L = pl;
        R = pr;
    }
    return (L << f->h) | R;
}

/* perm[p] = pi_k(p): the state processed at position p of sweep k.
 * identity != 0 gives the paper's ascending order. */
int orc_partition(int64_t n, uint64_t seed, int64_t k, int identity, uint32_t* perm)
{
    if (n < 1 || n > 0xFFFFFFFFLL || !perm) return ORC_INVALID_ARG;
    if (identity) {
        for (int64_t p = 0; p < n; ++p) perm[p] = (uint32_t)p;
        return ORC_OK;
    }
    orc_feistel f;
    feistel_init(&f, n, seed, k);
    for (int64_t p = 0; p < n; ++p) {
        uint64_t x = feistel_enc(&f, (uint64_t)p);
        while (x >= (uint64_t)n) x = feistel_enc(&f, x);
        perm[p] = (uint32_t)x;
    }
    return ORC_OK;
}

/* inv[s] = pi_k^{-1}(s), via the decryption rounds with the same walk. */
int orc_partition_inverse(int64_t n, uint64_t seed, int64_t k, int identity, uint32_t* inv)
{
    if (n < 1 || n > 0xFFFFFFFFLL || !inv) return ORC_INVALID_ARG;
    if (identity) {
        for (int64_t p = 0; p < n; ++p) inv[p] = (uint32_t)p;
        return ORC_OK;
    }
    orc_feistel f;
    feistel_init(&f, n, seed, k);
    for (int64_t s = 0; s < n; ++s) {
        uint64_t x = feistel_dec(&f, (uint64_t)s);
        while (x >= (uint64_t)n) x = feistel_dec(&f, x);
        inv[s] = (uint32_t)x;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* State selection WITH replacement ("there  */
/* could be advantages in sampling the states with replacement and/or   */
/* according to a non-uniform distribution ... importance-sampling ...  */
/* epsilon-greedy").  The paper defines no law; DESIGN readings R28-R29: */
/*   key_k  = mix64(mix64(seed) ^ k)           (as the partition, R2)    */
/*   skey_k = mix64(key_k ^ 0x5E1EC7105E1EC710)                          */
/*   u_i    = mix64(skey_k + i),  i = 0 .. n-1  (n draws per sweep)      */
/*   uniform:  s_i = floor(u_i * n / 2^64)                               */
/*   weighted (integer w_s >= 1, W = sum w_s < 2^63):                    */
/*             t_i = floor(u_i * W / 2^64),                              */
/*             s_i = min { s : w_0 + ... + w_s > t_i }                   */
/* i.e. P(s_i = s) = w_s / W up to 2^-64.  Batch t = draws [t*b, ...)   */
/* as R4; a state drawn twice in one batch is backed up once (both      */
/* copies read the same interim V, Eq. 12 is a statement about the set  */
/* of the batch's states).                                              */
/* ------------------------------------------------------------------ */
#define ORC_SEL_C 0x5E1EC7105E1EC710ULL

static uint64_t mulhi64(uint64_t a, uint64_t b)
{
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

int orc_select(int64_t n, uint64_t seed, int64_t k, const uint32_t* w, uint32_t* sel)
{
    if (n < 1 || n > 0x7FFFFFFFLL || !sel) return ORC_INVALID_ARG;
    uint64_t* cum = NULL;
    uint64_t W = 0;
    if (w) {
        /* inclusive prefix sums C_s = w_0 + ... + w_s, sequential */
        cum = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
        if (!cum) return ORC_OOM;
        for (int64_t s = 0; s < n; ++s) {
            if (w[s] == 0) { free(cum); return ORC_INVALID_ARG; }
            W += w[s];
            cum[s] = W;
        }
    }
    const uint64_t key = orc_mix64(orc_mix64(seed) ^ (uint64_t)k);
    const uint64_t skey = orc_mix64(key ^ ORC_SEL_C);
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t u = orc_mix64(skey + (uint64_t)i);
        if (!w) {
            sel[i] = (uint32_t)mulhi64(u, (uint64_t)n);
        } else {
            const uint64_t t = mulhi64(u, W);
            /* smallest s with cum[s] > t (plain binary search) */
            int64_t lo = 0, hi = n - 1;
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (cum[mid] > t) hi = mid;
                else lo = mid + 1;
            }
            sel[i] = (uint32_t)lo;
        }
    }
    free(cum);
    return ORC_OK;
}

/* the order of operator application k: the partition (R2) or, with
   select != 0, the n draws with replacement (R28-R29) */
static int draw_order(int64_t n, uint64_t seed, int64_t k, int identity, int select, const uint32_t* w,
                      uint32_t* perm)
{
    return select ? orc_select(n, seed, k, w, perm) : orc_partition(n, seed, k, identity, perm);
}

/* ------------------------------------------------------------------ */
/* Q-value: g(i,u) + alpha * sum_j p_ij(u) J(j)   (Eq. 7)        */
/* ------------------------------------------------------------------ */
static double q_value(const orc_mdp* m, int64_t s, int32_t a, const double* J)
{
    double acc = 0.0;
    size_t row = (size_t)s * (size_t)m->A + (size_t)a;
    if (m->kind == 0) {
        size_t base = row * (size_t)m->n;
        for (int64_t j = 0; j < m->n; ++j) acc += ld(m->P, m->p_f32, base + (size_t)j) * J[j];
    } else {
        for (int64_t e = m->row_ptr[row]; e < m->row_ptr[row + 1]; ++e)
            acc += ld(m->val, m->p_f32, (size_t)e) * J[m->col[e]];
    }
    return ld(m->c, m->c_f32, row) + m->gamma * acc;
}

/* min over u with the lowest index on exact ties (reading R8) */
static double q_min(const orc_mdp* m, int64_t s, const double* J, int32_t* arg)
{
    double best = q_value(m, s, 0, J);
    int32_t ba = 0;
    for (int32_t a = 1; a < m->A; ++a) {
        double q = q_value(m, s, a, J);
        if (q < best) { best = q; ba = a; }
    }
    *arg = ba;
    return best;
}

/* ------------------------------------------------------------------ */
/* One application of the mini-batch operator B_b (Eq. 12)  */
/* or, with pi_fixed != NULL, of B_{pi,b} (Eq. 13).         */
/*                                                                      */
/* perm[p] is the state at position p (the random re-indexing of        */
/* P:L162).  Batch t = positions [t*b, min(n,(t+1)*b)), so the states   */
/* already updated when processing position p are exactly those at      */
/* positions < b*floor(p/b) = M_b(p) of Eq. M(i); the last */
/* batch is short when b does not divide n (reading R4).                */
/* In place on V: states of earlier batches already hold B J (the       */
/* sum over M(i)), all others still hold J (the sum over S \ M(i)),     */
/* including the states of the current batch (reading R5).             */
/* resid = max_s |V_new(s) - V_old(s)| (every state updated once).      */
/* pi_out (may be NULL) receives the argmin (B_b) or a copy of pi.      */
/* ------------------------------------------------------------------ */
int orc_sweep(const orc_mdp* m, int64_t b, const uint32_t* perm, const int32_t* pi_fixed,
              double* V, int32_t* pi_out, double* resid)
{
    if (!m || !perm || !V || b < 1 || b > m->n) return ORC_INVALID_ARG;
    double* newv = (double*)malloc(sizeof(double) * (size_t)b);
    int32_t* newa = (int32_t*)malloc(sizeof(int32_t) * (size_t)b);
    if (!newv || !newa) { free(newv); free(newa); return ORC_OOM; }
    double r = 0.0;
    int nonfinite = 0;
    for (int64_t lo = 0; lo < m->n; lo += b) {
        int64_t hi = lo + b < m->n ? lo + b : m->n;
        /* every state of the batch is backed up against the same interim V
           (order-free within the batch: workers may share the loop) */
#pragma omp parallel for schedule(static) num_threads(orc_nthreads) if (orc_nthreads > 1 && hi - lo > 1)
        for (int64_t p = lo; p < hi; ++p) {
            int64_t s = perm[p];
            if (pi_fixed) {
                newa[p - lo] = pi_fixed[s];
                newv[p - lo] = q_value(m, s, pi_fixed[s], V);
            } else {
                newv[p - lo] = q_min(m, s, V, &newa[p - lo]);
            }
        }
        /* ... and only then written back, before the next batch starts */
        for (int64_t p = lo; p < hi; ++p) {
            int64_t s = perm[p];
            double d = fabs(newv[p - lo] - V[s]);
            if (!isfinite(newv[p - lo])) nonfinite = 1;
            if (d > r) r = d;
            V[s] = newv[p - lo];
            if (pi_out) pi_out[s] = newa[p - lo];
        }
    }
    free(newv);
    free(newa);
    if (resid) *resid = r;
    return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* "VI*" of P:L570, L577 (Sec. IV-B): the Bellman operator T computed   */
/* in chunks of c states "using the old values" -- the chunks are the   */
/* batches of the partition, but every chunk reads the values V had at  */
/* the start of the application; all new values are written at the end */
/* (DESIGN reading R21).  pi_fixed != NULL: T_pi in chunks.             */
/* ------------------------------------------------------------------ */
int orc_sweep_chunked(const orc_mdp* m, int64_t c, const uint32_t* perm, const int32_t* pi_fixed,
                      double* V, int32_t* pi_out, double* resid)
{
    if (!m || !perm || !V || c < 1 || c > m->n) return ORC_INVALID_ARG;
    double* newv = (double*)malloc(sizeof(double) * (size_t)m->n);
    int32_t* newa = (int32_t*)malloc(sizeof(int32_t) * (size_t)m->n);
    if (!newv || !newa) { free(newv); free(newa); return ORC_OOM; }
    for (int64_t lo = 0; lo < m->n; lo += c) {
        int64_t hi = lo + c < m->n ? lo + c : m->n;
        /* chunk [lo, hi) against the OLD values: V is not touched here */
#pragma omp parallel for schedule(static) num_threads(orc_nthreads) if (orc_nthreads > 1 && hi - lo > 1)
        for (int64_t p = lo; p < hi; ++p) {
            int64_t s = perm[p];
            if (pi_fixed) {
                newa[s] = pi_fixed[s];
                newv[s] = q_value(m, s, pi_fixed[s], V);
            } else {
                newv[s] = q_min(m, s, V, &newa[s]);
            }
        }
    }
    double r = 0.0;
    int nonfinite = 0;
    for (int64_t s = 0; s < m->n; ++s) {
        double d = fabs(newv[s] - V[s]);
        if (!isfinite(newv[s])) nonfinite = 1;
        if (d > r) r = d;
        V[s] = newv[s];
        if (pi_out) pi_out[s] = newa[s];
    }
    free(newv);
    free(newa);
    if (resid) *resid = r;
    return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Policy improvement of Algorithm 1, all states, against  */
/* V, no V write: pi'(s) = argmin_u Q(s,u) (lowest index on ties).      */
/* bellman_resid = max_s |min_u Q(s,u) - V(s)| = ||TV - V||_inf.        */
/* changed = #{s : pi'(s) != pi(s)} where pi is pi's content on entry.  */
/* ------------------------------------------------------------------ */
int orc_improve(const orc_mdp* m, const double* V, int32_t* pi, double* bellman_resid, int64_t* changed)
{
    if (!m || !V || !pi) return ORC_INVALID_ARG;
    double* q = (double*)malloc(sizeof(double) * (size_t)m->n);
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)m->n);
    if (!q || !a) { free(q); free(a); return ORC_OOM; }
    /* greedy action of every state against V (state-parallel, no writes to V) */
#pragma omp parallel for schedule(static) num_threads(orc_nthreads) if (orc_nthreads > 1)
    for (int64_t s = 0; s < m->n; ++s) q[s] = q_min(m, s, V, &a[s]);
    double r = 0.0;
    int64_t ch = 0;
    int nonfinite = 0;
    for (int64_t s = 0; s < m->n; ++s) {
        if (!isfinite(q[s])) nonfinite = 1;
        double d = fabs(q[s] - V[s]);
        if (d > r) r = d;
        if (a[s] != pi[s]) ++ch;
        pi[s] = a[s];
    }
    free(q);
    free(a);
    if (bellman_resid) *bellman_resid = r;
    if (changed) *changed = ch;
    return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* MB-VI (VI of P:L99 with B_b in place of T).                  */
/* V <- V0 (caller), for k = first_sweep, ...: draw the  */
/* partition of sweep k, apply B_b, record r_k; stop at the first r_k   */
/* <= eps (reading R6) or after max_sweeps.  pi = argmins of the final  */
/* sweep (reading R9).  trace[i] = r_{first_sweep+i}.                   */
/* chunked != 0: VI* of P:L577 instead -- every application is T in     */
/* chunks of b states against the old values (orc_sweep_chunked).       */
/* select != 0: every application draws n states WITH replacement      */
/* (orc_select; w = integer weights or NULL for uniform, R28-R29).  r_k */
/* is then the max change over the DRAWN states only, so r_k <= eps     */
/* only triggers the stopping test of R30: rT = ||TV - V||_inf (the     */
/* improvement pass, orc_improve, pi <- greedy(V)); stop iff rT <= eps. */
/* On OK, pi = greedy(V) and ||V - V*|| <= rT / (1 - gamma).            */
/* ------------------------------------------------------------------ */
int orc_vi(const orc_mdp* m, int64_t b, uint64_t seed, int identity, int64_t first_sweep,
           double eps, int64_t max_sweeps, int chunked, double* V, int32_t* pi, double* trace,
           int64_t* sweeps_out, int select, const uint32_t* w)
{
    if (!m || !V || !pi || b < 1 || b > m->n || max_sweeps < 1 || !(eps > 0.0)) return ORC_INVALID_ARG;
    if (select && (chunked || identity)) return ORC_INVALID_ARG;
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m->n);
    if (!perm) return ORC_OOM;
    int st = ORC_NOT_CONVERGED;
    int64_t it = 0;
    while (it < max_sweeps) {
        double r;
        if (draw_order(m->n, seed, first_sweep + it, identity, select, w, perm)) { st = ORC_INVALID_ARG; break; }
        int rc = chunked ? orc_sweep_chunked(m, b, perm, NULL, V, pi, &r)
                         : orc_sweep(m, b, perm, NULL, V, pi, &r);
        if (trace) trace[it] = r;
        ++it;
        if (rc == ORC_NONFINITE) { st = ORC_NONFINITE; break; }
        if (r <= eps) {
            if (select) {  /* R30: confirm on all states */
                double rT;
                int64_t ch;
                if (orc_improve(m, V, pi, &rT, &ch) == ORC_NONFINITE) { st = ORC_NONFINITE; break; }
                if (rT > eps) continue;
            }
            st = ORC_OK;
            break;
        }
    }
    free(perm);
    if (sweeps_out) *sweeps_out = it;
    return st;
}

/* ------------------------------------------------------------------ */
/* MB-MPI: Algorithm 1 with B_{pi,b} as the evaluation     */
/* operator and warm start (reading R10).        */
/* pi_0 = greedy(V0) unless pi_given (reading R10).  Outer iteration o: */
/*   m evaluation sweeps, each with its own sweep counter k and thus    */
/*   its own partition (reading R3), residuals -> trace;                */
/*   improvement -> pi', changed, r_T = ||TV - V||_inf -> trace;        */
/*   stop when changed == 0 and r_T <= eps (reading R11).               */
/* trace layout: trace[o*(m+1) + e], e < m eval residuals, e = m: r_T.  */
/* changed_trace[o] = changed count of outer iteration o.               */
/* select != 0: evaluation sweeps draw with replacement (as orc_vi).    */
/* ------------------------------------------------------------------ */
int orc_mpi(const orc_mdp* m, int64_t b, int32_t msweeps, uint64_t seed, int identity, int64_t first_sweep,
            double eps, int64_t max_outer, int pi_given, double* V, int32_t* pi, double* trace,
            int64_t* changed_trace, int64_t* sweeps_out, int64_t* outer_out, int select, const uint32_t* w)
{
    if (!m || !V || !pi || b < 1 || b > m->n || msweeps < 1 || max_outer < 1 || !(eps > 0.0))
        return ORC_INVALID_ARG;
    if (select && identity) return ORC_INVALID_ARG;
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m->n);
    if (!perm) return ORC_OOM;
    int st = ORC_NOT_CONVERGED;
    int64_t k = first_sweep, o = 0;
    if (!pi_given) {
        int64_t ch;
        double rT;
        if (orc_improve(m, V, pi, &rT, &ch) == ORC_NONFINITE) { free(perm); return ORC_NONFINITE; }
    }
    while (o < max_outer) {
        int bad = 0;
        for (int32_t e = 0; e < msweeps; ++e) {
            double r;
            if (draw_order(m->n, seed, k, identity, select, w, perm)) { bad = 2; break; }
            int rc = orc_sweep(m, b, perm, pi, V, NULL, &r);
            ++k;
            if (trace) trace[o * (msweeps + 1) + e] = r;
            if (rc == ORC_NONFINITE) { bad = 1; break; }
        }
        if (bad == 2) { st = ORC_INVALID_ARG; break; }
        if (bad) { st = ORC_NONFINITE; ++o; break; }
        double rT;
        int64_t ch;
        int rc = orc_improve(m, V, pi, &rT, &ch);
        if (trace) trace[o * (msweeps + 1) + msweeps] = rT;
        if (changed_trace) changed_trace[o] = ch;
        ++o;
        if (rc == ORC_NONFINITE) { st = ORC_NONFINITE; break; }
        if (ch == 0 && rT <= eps) { st = ORC_OK; break; }
    }
    free(perm);
    if (sweeps_out) *sweeps_out = k - first_sweep;
    if (outer_out) *outer_out = o;
    return st;
}

/* ------------------------------------------------------------------ */
/* Single backups for sampled parity checks at full size: Q(s,a) for    */
/* one state given an explicit interim V (the caller assembles V_int    */
/* from the partition and pre/post snapshots).  Dense row block layout: */
/* P_rows = P[s][0..A)[0..n), c_row = c[s][0..A).                       */
/* ------------------------------------------------------------------ */
double orc_backup_dense_row(int64_t n, int32_t A, double gamma, int p_f32, const void* P_rows,
                            const void* c_row, const double* Vint, int32_t pi_a, int32_t* arg)
{
    orc_mdp m;
    memset(&m, 0, sizeof m);
    m.n = n;
    m.A = A;
    m.kind = 0;
    m.gamma = gamma;
    m.p_f32 = p_f32;
    m.c_f32 = p_f32;
    /* view the single-state block as state 0 of an n-state dense MDP */
    m.P = P_rows;
    m.c = c_row;
    if (pi_a >= 0) { if (arg) *arg = pi_a; return q_value(&m, 0, pi_a, Vint); }
    int32_t a;
    double q = q_min(&m, 0, Vint, &a);
    if (arg) *arg = a;
    return q;
}

/* Single-state backup over CSR rows for sampled parity checks at full size:
 * row_ptr has A+1 entries (offsets into col/val for the state's A rows). */
double orc_backup_csr_row(int64_t n, int32_t A, double gamma, int p_f32, const int64_t* row_ptr,
                          const int32_t* col, const void* val, const void* c_row, const double* Vint,
                          int32_t pi_a, int32_t* arg)
{
    orc_mdp m;
    memset(&m, 0, sizeof m);
    m.n = n;
    m.A = A;
    m.kind = 1;
    m.gamma = gamma;
    m.p_f32 = p_f32;
    m.c_f32 = p_f32;
    m.row_ptr = row_ptr;
    m.col = col;
    m.val = val;
    m.c = c_row;
    if (pi_a >= 0) { if (arg) *arg = pi_a; return q_value(&m, 0, pi_a, Vint); }
    int32_t a;
    double q = q_min(&m, 0, Vint, &a);
    if (arg) *arg = a;
    return q;
}


/* ------------------------------------------------------------------ */
/* Certificate for instances too large to hold on the host (config 5:  */
/* 320 GB of P): r_T = ||T V - V||_inf (Eq. 5 / Prop. 3: then           */
/* ||V - V*||_inf <= r_T / (1 - gamma)) over the states [s0, s1) of the */
/* dense random instance (seed, n, A), every row REGENERATED from the   */
/* shared instance definition gen/rmb_gen.h, stored as float (f32) or   */
/* double exactly as the instance is, and summed as q_value does        */
/* (sequentially in j, fp64).  Threads split the states; the max is     */
/* order-free.  arg_out (may be NULL): argmin_a Q(s,a), [s1 - s0].      */
/* ------------------------------------------------------------------ */
double orc_bellman_residual_dense_gen(uint64_t seed, int64_t n, int32_t A, int f32, double gamma, const double* V,
                                      int64_t s0, int64_t s1, int32_t* arg_out)
{
    double r = 0.0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(orc_nthreads) reduction(max : r)
    for (int64_t s = s0; s < s1; ++s) {
        double best = 0.0;
        int32_t ba = 0;
        for (int32_t a = 0; a < A; ++a) {
            uint64_t W = 0;
            for (int64_t j = 0; j < n; ++j) W += rmbgen_dense_w(seed, s, a, j);
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                double p = rmbgen_dense_p(seed, s, a, j, W);
                if (f32) p = (double)(float)p;
                acc += p * V[j];
            }
            double c = rmbgen_cost_u01(seed, s, a);
            if (f32) c = (double)(float)c;
            const double q = c + gamma * acc;
            if (a == 0 || q < best) { best = q; ba = a; }
        }
        if (arg_out) arg_out[s - s0] = ba;
        const double d = fabs(best - V[s]);
        if (d > r || d != d) r = d;
    }
    return r;
}

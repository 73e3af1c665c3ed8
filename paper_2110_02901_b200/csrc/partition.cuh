// partition.cuh — the per-sweep random re-indexing of the states.
//
// The paper shuffles the states "before every evaluation of the operators"
// and processes them in blocks of b (re-indexing P:L162).  We
// fix the shuffle as a counter-based permutation so that the host generator
// (rmb_partition), the device solver and the independent CPU oracle agree on
// every batch (reading R2):
//   mix64 = SplitMix64 output function;  key_k = mix64(mix64(seed) ^ k);
//   round keys rk_r = mix64(key_k ^ r), r < 6;
//   w = max(2, bitlen(n-1)) rounded up to even, h = w/2, x = (L << h) | R;
//   round: (L, R) <- (R, L ^ (mix64(rk_r ^ R) >> (64 - h)));
//   pi_k(p) = enc(p), re-encrypted while >= n (cycle walking).
// Stateless: pi_k(p) costs ~6 mix64 per walk step, no memory traffic.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define RMB_HD __host__ __device__ __forceinline__
#else
#define RMB_HD inline
#endif

namespace rmb {

RMB_HD uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Permutation {
    uint64_t rk[6];
    uint64_t n;
    uint32_t h;
    uint64_t lo_mask;

    RMB_HD void init(int64_t n_, uint64_t seed, int64_t sweep)
    {
        n = (uint64_t)n_;
        uint32_t w = 0;
        for (uint64_t x = n - 1; x; x >>= 1) ++w;
        if (w < 2) w = 2;
        w += (w & 1u);
        h = w >> 1;
        lo_mask = (1ULL << h) - 1ULL;
        const uint64_t key = splitmix64(splitmix64(seed) ^ (uint64_t)sweep);
        for (int r = 0; r < 6; ++r) rk[r] = splitmix64(key ^ (uint64_t)r);
    }

    RMB_HD uint64_t encrypt(uint64_t x) const
    {
        uint64_t L = x >> h, R = x & lo_mask;
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            const uint64_t f = splitmix64(rk[r] ^ R) >> (64u - h);
            const uint64_t t = L ^ f;
            L = R;
            R = t;
        }
        return (L << h) | R;
    }

    RMB_HD uint64_t decrypt(uint64_t x) const
    {
        uint64_t L = x >> h, R = x & lo_mask;
#pragma unroll
        for (int r = 5; r >= 0; --r) {
            // forward round: (L', R') = (R, L ^ F(R))  =>  R = L', L = R' ^ F(L')
            const uint64_t f = splitmix64(rk[r] ^ L) >> (64u - h);
            const uint64_t t = R ^ f;
            R = L;
            L = t;
        }
        return (L << h) | R;
    }

    // state at position p
    RMB_HD uint64_t operator()(uint64_t p) const
    {
        uint64_t x = encrypt(p);
        while (x >= n) x = encrypt(x);
        return x;
    }

    // position of state s (the inverse permutation, same cycle walk backwards)
    RMB_HD uint64_t position(uint64_t s) const
    {
        uint64_t x = decrypt(s);
        while (x >= n) x = decrypt(x);
        return x;
    }
};

// State selection WITH replacement (DESIGN
// readings R28-R29): application k draws n states i.i.d.,
//   skey_k = mix64(key_k ^ 0x5E1EC7105E1EC710),  u_i = mix64(skey_k + i),
//   uniform:  s_i = floor(u_i * n / 2^64);
//   weighted: t_i = floor(u_i * W / 2^64), s_i = first s with cum[s] > t_i
//             (cum = inclusive prefix sums of integer weights w_s >= 1, W = cum[n-1]).
// Integer arithmetic only, so every side draws the same states.
RMB_HD uint64_t mulhi_u64(uint64_t a, uint64_t b)
{
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
#endif
}

struct Selection {
    uint64_t skey;
    uint64_t n;
    const uint64_t* cum;  // null: uniform
    uint64_t W;

    RMB_HD void init(int64_t n_, uint64_t seed, int64_t sweep, const uint64_t* cum_, uint64_t W_)
    {
        n = (uint64_t)n_;
        const uint64_t key = splitmix64(splitmix64(seed) ^ (uint64_t)sweep);
        skey = splitmix64(key ^ 0x5E1EC7105E1EC710ULL);
        cum = cum_;
        W = W_;
    }

    // the state of draw i
    RMB_HD uint32_t operator()(uint64_t i) const
    {
        const uint64_t u = splitmix64(skey + i);
        if (!cum) return (uint32_t)mulhi_u64(u, n);
        const uint64_t t = mulhi_u64(u, W);
        uint64_t lo = 0, hi = n - 1;
        while (lo < hi) {
            const uint64_t mid = lo + ((hi - lo) >> 1);
#if defined(__CUDA_ARCH__)
            const uint64_t cm = __ldg(cum + mid);
#else
            const uint64_t cm = cum[mid];
#endif
            if (cm > t) hi = mid;
            else lo = mid + 1;
        }
        return (uint32_t)lo;
    }
};

// The processing order of operator application k, as the solvers store it
// (one entry per position): the permutation (sel == 0) or the draws
// (sel == 1 uniform, 2 weighted).  Threads tid, tid + stride, ... fill dst.
struct OrderSpec {
    int sel;
    const uint64_t* cum;
    uint64_t W;
};

RMB_HD void fill_order(int64_t n, uint64_t seed, int64_t k, const OrderSpec& os, uint32_t* dst, int64_t tid,
                       int64_t stride)
{
    if (os.sel) {
        Selection sl;
        sl.init(n, seed, k, os.sel == 2 ? os.cum : nullptr, os.W);
        for (int64_t p = tid; p < n; p += stride) dst[p] = sl((uint64_t)p);
    } else {
        Permutation pm;
        pm.init(n, seed, k);
        for (int64_t p = tid; p < n; p += stride) dst[p] = (uint32_t)pm((uint64_t)p);
    }
}

}  // namespace rmb

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

}  // namespace rmb

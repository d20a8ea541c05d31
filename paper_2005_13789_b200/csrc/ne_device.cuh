// ne_device.cuh -- device primitives of the SGNS training engine (sm_100a).
//
// Counter-based randomness (DESIGN.md contract R1/R2): every random choice of
// the method -- walk steps, the pool order and the
// negatives -- is a pure function of (seed, tag, epoch, counter), so
// thousands of warps draw independently and reproducibly.  This is a separate
// implementation from oracle/ (no shared code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ne {

constexpr uint32_t kTagWalk = 1u, kTagNeg = 2u, kTagShuf = 3u, kTagInit = 4u;
constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // walk padding after a sink
constexpr uint64_t kHole = ~0ull;             // empty slot of the pi-indexed array

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32 multiplies,
// key bumped by the Weyl constants between rounds.
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

__device__ __forceinline__ uint2 key_of(uint64_t seed) {
    return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ uint32_t tag_word(uint32_t tag, uint32_t epoch) {
    return (tag << 24) | epoch;
}

// R2: floor(r64 * n / 2^64) -- the high word of a 64x64 product.
__device__ __forceinline__ uint64_t uniform_index(uint32_t lo, uint32_t hi, uint64_t n) {
    return __umul64hi(((uint64_t)hi << 32) | lo, n);
}

// O6: alternating Feistel network on b = max(2, ceil(log2 N)) bits split into
// hi (b - b/2 bits) and lo (b/2 bits); rounds 0..3 alternate hi ^= F(lo) and
// lo ^= F(hi), F = Philox(v, episode, round, SHUF|epoch).x0 masked; cycle-walked
// into [0, N) (domain < 2N: < 2 passes on average).
struct Feistel {
    uint64_t N;
    uint32_t c;                 // lo bits
    uint64_t mask_lo, mask_hi;
    uint32_t episode, tagw;
    uint2 key;
    __device__ __forceinline__ uint64_t operator()(uint64_t x) const {
        uint64_t y = x;
        do {
            uint64_t hi = y >> c, lo = y & mask_lo;
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
                const uint4 o = philox(make_uint4((uint32_t)((i & 1) ? hi : lo), episode, i, tagw), key);
                if (i & 1) lo ^= (uint64_t)o.x & mask_lo;
                else hi ^= (uint64_t)o.x & mask_hi;
            }
            y = (hi << c) | lo;
        } while (y >= N);
        return y;
    }
};

// Index of the range containing v in sorted bounds[0..count] (bounds[0] <= v < bounds[count]).
__device__ __forceinline__ uint32_t range_of(const uint64_t* bounds, uint32_t count, uint64_t v) {
    uint32_t lo = 0, hi = count;  // invariant: bounds[lo] <= v < bounds[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (bounds[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

}  // namespace ne

// sgns_common.cuh -- device pieces shared by the SGNS kernels: the negative
// draw (O8), the group all-reduce and one SGNS update (O10, Alg. 1 Train).
// Every kernel variant calls sgns_step, so they share one arithmetic.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ne_device.cuh"
#include "ne_internal.h"

namespace ne {

constexpr int kMaxK = 8;

// O8: negative j of the sample at canonical position pos of the block:
// Philox(ctr = (pos_lo, pos_hi, episode<<20 | block<<8 | j, NEG<<24 | epoch)),
// column R2(x0|x1<<32, c_count), coin x2 < thr ? column : alias.
// Split in two so a kernel can issue the alias-table load one iteration early
// and take the coin decision only when the id is needed (the load latency then
// overlaps a whole iteration instead of stalling the prefetch).
struct NegDraw {
    uint32_t col, coin;
    uint2 ta;  // (thr, alias) of column col
};
__device__ __forceinline__ NegDraw issue_negative(const SgnsParams& p, uint2 key, uint32_t tagw,
                                                  uint64_t pos, uint32_t j) {
    const uint4 x = philox(make_uint4((uint32_t)pos, (uint32_t)(pos >> 32),
                                      (p.episode << 20) | (p.block << 8) | j, tagw), key);
    NegDraw d;
    d.col = (uint32_t)uniform_index(x.x, x.y, p.c_count);
    d.coin = x.z;
    d.ta = __ldg(p.alias + d.col);
    return d;
}
__device__ __forceinline__ uint32_t finish_negative(const SgnsParams& p, const NegDraw& d) {
    return (uint32_t)(p.c_begin + (d.coin < d.ta.x ? d.col : d.ta.y));
}
__device__ __forceinline__ uint32_t draw_negative(const SgnsParams& p, uint2 key, uint32_t tagw,
                                                  uint64_t pos, uint32_t j) {
    return finish_negative(p, issue_negative(p, key, tagw, pos, j));
}

template <int G>
__device__ __forceinline__ float group_sum(float x) {  // all-reduce inside aligned groups of G lanes
#pragma unroll
    for (int o = G / 2; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
}

// One Train(v, c, y) of Alg. 1 on the lane's R float4 of the two
// rows: x = v.c (per-lane FMA chain + group all-reduce), s = sigma(clamp(x, +-30)),
// a = lr (s - y), (v, c) <- (v - a c, c - a v) from the pre-update values.
// Returns a; vo receives the pre-update v (for delta write-back); loss gets
// -log s (y = 1) or -log(1 - s) (y = 0) as softplus of the same exponential.
template <int G, int R>
__device__ __forceinline__ float sgns_step(float4 (&v)[R], float4 (&c)[R], float4 (&vo)[R], float lr,
                                           bool positive, float& loss) {
    float part = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        part = fmaf(v[r].x, c[r].x, part);
        part = fmaf(v[r].y, c[r].y, part);
        part = fmaf(v[r].z, c[r].z, part);
        part = fmaf(v[r].w, c[r].w, part);
    }
    const float x = fminf(fmaxf(group_sum<G>(part), -30.f), 30.f);
    const float ex = __expf(-x);
    const float s = __fdividef(1.f, 1.f + ex);
    const float a = lr * (s - (positive ? 1.f : 0.f));
    loss = __logf(1.f + ex) + (positive ? 0.f : x);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        vo[r] = v[r];
        const float4 co = c[r];
        v[r] = make_float4(fmaf(-a, co.x, vo[r].x), fmaf(-a, co.y, vo[r].y),
                           fmaf(-a, co.z, vo[r].z), fmaf(-a, co.w, vo[r].w));
        c[r] = make_float4(fmaf(-a, vo[r].x, co.x), fmaf(-a, vo[r].y, co.y),
                           fmaf(-a, vo[r].z, co.z), fmaf(-a, vo[r].w, co.w));
    }
    return a;
}

// NEXT-4 accumulated update of one pair (word2vec order): x = v0 . c with the
// pre-sample vertex row v0, a = lr (s - y); e += a c (the vertex row's
// accumulated step, applied once by the caller: v = v0 - e); c <- c - a v0.
template <int G, int R>
__device__ __forceinline__ float sgns_step_acc(const float4 (&v0)[R], float4 (&c)[R], float4 (&e)[R], float lr,
                                               bool positive, float& loss) {
    float part = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        part = fmaf(v0[r].x, c[r].x, part);
        part = fmaf(v0[r].y, c[r].y, part);
        part = fmaf(v0[r].z, c[r].z, part);
        part = fmaf(v0[r].w, c[r].w, part);
    }
    const float x = fminf(fmaxf(group_sum<G>(part), -30.f), 30.f);
    const float ex = __expf(-x);
    const float s = __fdividef(1.f, 1.f + ex);
    const float a = lr * (s - (positive ? 1.f : 0.f));
    loss = __logf(1.f + ex) + (positive ? 0.f : x);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float4 co = c[r];
        e[r] = make_float4(fmaf(a, co.x, e[r].x), fmaf(a, co.y, e[r].y), fmaf(a, co.z, e[r].z), fmaf(a, co.w, e[r].w));
        c[r] = make_float4(fmaf(-a, v0[r].x, co.x), fmaf(-a, v0[r].y, co.y),
                           fmaf(-a, v0[r].z, co.z), fmaf(-a, v0[r].w, co.w));
    }
    return a;
}

// Row access by element group e (4 consecutive elements) of row `row` of a
// d-wide matrix: fp32 rows are float4 accesses; bf16 rows (NEXT-4, reading
// D16) are 8-byte accesses widened exactly to fp32 on load, rounded to nearest
// even on store, and Hogwild deltas are added with one bf16x4 vector reduction
// (red.global.add.noftz.v2.bf16x2 = REDG.E.ADD.BF16x4.RN).
template <bool BF>
struct RowIO;

template <>
struct RowIO<false> {
    static __device__ __forceinline__ float4 load(const float* m, uint64_t row, uint32_t d, uint32_t e) {
        return reinterpret_cast<const float4*>(m + row * d)[e];
    }
    static __device__ __forceinline__ void store(float* m, uint64_t row, uint32_t d, uint32_t e, float4 v) {
        reinterpret_cast<float4*>(m + row * d)[e] = v;
    }
    static __device__ __forceinline__ void add(float* m, uint64_t row, uint32_t d, uint32_t e, float4 dv) {
        atomicAdd(reinterpret_cast<float4*>(m + row * d) + e, dv);
    }
    // the same with an L2 eviction-priority policy (createpolicy; developer knob NE_SGNS_L2HINT)
    static __device__ __forceinline__ float4 load(const float* m, uint64_t row, uint32_t d, uint32_t e, uint64_t pol) {
        float4 v;
        asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(reinterpret_cast<const float4*>(m + row * d) + e), "l"(pol));
        return v;
    }
    static __device__ __forceinline__ void add(float* m, uint64_t row, uint32_t d, uint32_t e, float4 dv, uint64_t pol) {
        asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                     ::"l"(reinterpret_cast<float4*>(m + row * d) + e), "f"(dv.x), "f"(dv.y), "f"(dv.z), "f"(dv.w),
                     "l"(pol) : "memory");
    }
};

__device__ __forceinline__ uint64_t l2_policy(uint32_t kind) {  // 0 normal, 1 evict_first, 2 evict_last
    uint64_t pol;
    if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <>
struct RowIO<true> {
    static __device__ __forceinline__ uint2* at(const float* m, uint64_t row, uint32_t d, uint32_t e) {
        return reinterpret_cast<uint2*>(const_cast<float*>(m)) + row * (d >> 2) + e;
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // .x = a in the low half
        return *reinterpret_cast<const uint32_t*>(&h);
    }
    static __device__ __forceinline__ float4 load(const float* m, uint64_t row, uint32_t d, uint32_t e) {
        const uint2 u = *at(m, row, d, e);
        return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                           __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
    }
    static __device__ __forceinline__ void store(float* m, uint64_t row, uint32_t d, uint32_t e, float4 v) {
        *at(m, row, d, e) = make_uint2(pack(v.x, v.y), pack(v.z, v.w));
    }
    static __device__ __forceinline__ void add(float* m, uint64_t row, uint32_t d, uint32_t e, float4 dv) {
        asm volatile("red.global.add.noftz.v2.bf16x2 [%0], {%1, %2};" ::"l"(at(m, row, d, e)),
                     "r"(pack(dv.x, dv.y)), "r"(pack(dv.z, dv.w))
                     : "memory");
    }
};

__device__ __forceinline__ float4 scaled(float a, const float4& x) {
    return make_float4(a * x.x, a * x.y, a * x.z, a * x.w);
}

}  // namespace ne

// kernels_sgns.cu -- the SGNS update of Alg. 1 on one 2D block
// (sm_100a).  Memory-bound gather/scatter ("O(1) arithmetic intensity"):
// per positive sample the kernel reads the vertex row, the positive context row
// and K negative context rows and writes all 2+K back -- 8d(2+K) bytes against
// 6d(1+K) flops -- so the design goal is bytes in flight, not FLOPs.
//
// Mapping: one warp per sample.  Each lane owns R float4 of every row
// (d <= 128 R), so a row is one coalesced 128-bit-per-lane access; all 2+K row
// loads are issued before the first dot product (they are independent), the
// 1+K updates then run back to back in registers (dot = per-lane FMA chain +
// 5-step xor-shuffle all-reduce; sigmoid; two FMAs per element), and the rows
// are written once.  Repeated context ids inside a sample are forwarded in
// registers so the result equals the sequential Alg. 1 order (reading D2).
// Negatives (O8) are drawn by lanes 0..K-1 in parallel (one Philox each) and
// broadcast with shuffles.
//
// Production mode: a persistent grid of warps strides over the block's
// samples, updating rows in place without locks (Hogwild; races only between
// concurrent samples sharing a row).  Deterministic mode: one warp walks the
// block in canonical order -- the same device code, so parity of the
// deterministic mode is parity of the production arithmetic.
#include <algorithm>

#include "ne_device.cuh"
#include "ne_internal.h"

namespace ne {

constexpr int kMaxK = 8;
constexpr int kSgnsThreads = 256;

// O8: negative j of the sample at canonical position pos of the block:
// Philox(ctr = (pos_lo, pos_hi, episode<<20 | block<<8 | j, NEG<<24 | epoch)),
// column R2(x0|x1<<32, c_count), coin x2 < thr ? column : alias.
__device__ __forceinline__ uint32_t draw_negative(const SgnsParams& p, uint2 key, uint32_t tagw,
                                                  uint64_t pos, uint32_t j) {
    const uint4 x = philox(make_uint4((uint32_t)pos, (uint32_t)(pos >> 32),
                                      (p.episode << 20) | (p.block << 8) | j, tagw), key);
    const uint64_t col = uniform_index(x.x, x.y, p.c_count);
    const uint2 ta = __ldg(p.alias + col);
    return (uint32_t)(p.c_begin + (x.z < ta.x ? col : (uint64_t)ta.y));
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
}

template <int R>
__global__ void __launch_bounds__(kSgnsThreads) sgns_kernel(SgnsParams p) {
    const uint32_t lane = lane_id();
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t q = p.d >> 2;  // float4 per row
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    const int K = (int)p.K;
    double loss = 0.0;  // lane 0

    for (uint64_t pos = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; pos < p.count;
         pos += nwarps) {
        const uint2 pr = p.pool[pos];  // (src, dst), one broadcast transaction
        const uint32_t my_neg = lane < p.K ? draw_negative(p, key, tagw, pos, lane) : 0u;

        uint32_t ids[kMaxK + 1];
        ids[0] = pr.y;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) ids[j + 1] = __shfl_sync(0xFFFFFFFFu, my_neg, j);

        float4* vrow = reinterpret_cast<float4*>(p.V + (uint64_t)(pr.x - p.v_begin) * p.d);
        float4 v[R];
        float4 c[kMaxK + 1][R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = lane + 32u * r;
            v[r] = e < q ? vrow[e] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j <= kMaxK; ++j) {
            if (j <= K) {
                const float4* crow = reinterpret_cast<const float4*>(p.C + (uint64_t)(ids[j] - p.c_begin) * p.d);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t e = lane + 32u * r;
                    c[j][r] = e < q ? crow[e] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }

        // Alg. 1 lines 10 and 12: positive, then the K negatives, in order.
#pragma unroll
        for (int j = 0; j <= kMaxK; ++j) {
            if (j <= K) {
#pragma unroll
                for (int i = 0; i < j; ++i)  // forward the latest copy of a repeated id
                    if (ids[i] == ids[j]) {
#pragma unroll
                        for (int r = 0; r < R; ++r) c[j][r] = c[i][r];
                    }
                float part = 0.f;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    part = fmaf(v[r].x, c[j][r].x, part);
                    part = fmaf(v[r].y, c[j][r].y, part);
                    part = fmaf(v[r].z, c[j][r].z, part);
                    part = fmaf(v[r].w, c[j][r].w, part);
                }
                const float x = fminf(fmaxf(warp_sum(part), -30.f), 30.f);
                const float s = __fdividef(1.f, 1.f + __expf(-x));
                const float g = s - (j == 0 ? 1.f : 0.f);
                const float a = p.lr * g;
                if (lane == 0)  // -log s (y = 1) or -log(1 - s) (y = 0), as softplus
                    loss += (double)__logf(1.f + __expf(j == 0 ? -x : x));
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 vo = v[r], co = c[j][r];
                    v[r] = make_float4(fmaf(-a, co.x, vo.x), fmaf(-a, co.y, vo.y),
                                       fmaf(-a, co.z, vo.z), fmaf(-a, co.w, vo.w));
                    c[j][r] = make_float4(fmaf(-a, vo.x, co.x), fmaf(-a, vo.y, co.y),
                                          fmaf(-a, vo.z, co.z), fmaf(-a, vo.w, co.w));
                }
            }
        }

        // Fused write-back of 2+K rows (the last copy of a repeated id wins).
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = lane + 32u * r;
            if (e < q) vrow[e] = v[r];
        }
#pragma unroll
        for (int j = 0; j <= kMaxK; ++j) {
            if (j <= K) {
                bool last = true;
#pragma unroll
                for (int i = j + 1; i <= kMaxK; ++i)
                    if (i <= K && ids[i] == ids[j]) last = false;
                if (last) {
                    float4* crow = reinterpret_cast<float4*>(p.C + (uint64_t)(ids[j] - p.c_begin) * p.d);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t e = lane + 32u * r;
                        if (e < q) crow[e] = c[j][r];
                    }
                }
            }
        }
    }
    if (lane == 0 && loss != 0.0) atomicAdd(p.loss, loss);
}

template <int R>
static cudaError_t launch_sgns_r(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if (p.deterministic) {
        sgns_kernel<R><<<1, 32, 0, s>>>(p);
    } else {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgns_kernel<R>,
                                                                      kSgnsThreads, 0);
        if (e != cudaSuccess) return e;
        per_sm = std::max(per_sm, 1);
        const uint64_t warps = std::min<uint64_t>(p.count, std::max<uint64_t>(p.max_warps, 1));
        const uint64_t full = (uint64_t)dev.sm_count * per_sm;
        const int wpb = kSgnsThreads / 32;
        if (warps >= full * wpb) {
            sgns_kernel<R><<<(unsigned)full, kSgnsThreads, 0, s>>>(p);
        } else if (warps >= (uint64_t)dev.sm_count * wpb) {
            sgns_kernel<R><<<(unsigned)((warps + wpb - 1) / wpb), kSgnsThreads, 0, s>>>(p);
        } else {  // small capped grids: spread single warps over the SMs
            sgns_kernel<R><<<(unsigned)warps, 32, 0, s>>>(p);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_sgns(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if (p.count == 0) return cudaSuccess;
    if (p.K > (uint32_t)kMaxK || p.d % 4 != 0 || p.d == 0 || p.d > 512) return cudaErrorInvalidValue;
    const uint32_t R = (p.d / 4 + 31) / 32;
    switch (R) {
        case 1: return launch_sgns_r<1>(p, dev, s);
        case 2: return launch_sgns_r<2>(p, dev, s);
        case 3: return launch_sgns_r<3>(p, dev, s);
        default: return launch_sgns_r<4>(p, dev, s);
    }
}

__global__ void export_negatives_kernel(SgnsParams p, uint64_t pos_begin, uint64_t count,
                                        uint32_t* __restrict__ out) {
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    const uint64_t total = count * p.K;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += stride) {
        const uint64_t i = w / p.K;
        out[w] = draw_negative(p, key, tagw, pos_begin + i, (uint32_t)(w - i * p.K));
    }
}

cudaError_t launch_export_negatives(const SgnsParams& p, uint64_t pos_begin, uint64_t count,
                                    uint32_t* out, const Device& dev, cudaStream_t s) {
    if (count == 0 || p.K == 0) return cudaSuccess;
    const uint64_t total = count * p.K;
    const unsigned g = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((total + 255) / 256, (uint64_t)dev.sm_count * 8));
    export_negatives_kernel<<<g, 256, 0, s>>>(p, pos_begin, count, out);
    return cudaGetLastError();
}

}  // namespace ne

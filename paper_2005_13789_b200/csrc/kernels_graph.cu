// kernels_graph.cu -- CSR validation, embedding initialisation and the walk
// engine (sm_100a).
#include <algorithm>

#include <cuda_bf16.h>

#include "ne_device.cuh"
#include "ne_internal.h"

namespace ne {

static unsigned grid_for(uint64_t work, int threads, const Device& dev, int per_sm = 8) {
    uint64_t blocks = (work + threads - 1) / threads;
    uint64_t cap = (uint64_t)dev.sm_count * per_sm;
    return (unsigned)std::max<uint64_t>(1, std::min(blocks, cap));
}

// offsets monotone and targets < n (and, for node2vec, rows sorted by
// target).  The first violation wins (atomicMin).
__global__ void validate_csr_kernel(const uint64_t* __restrict__ off,
                                    const uint32_t* __restrict__ tgt, uint64_t n, uint64_t nnz,
                                    unsigned long long* bad, bool check_sorted) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t b = off[i], e = off[i + 1];
        if (e < b) atomicMin(&bad[0], (unsigned long long)i);
        if (check_sorted && e > b && e <= nnz)
            for (uint64_t j = b + 1; j < e; ++j)
                if (tgt[j] < tgt[j - 1]) { atomicMin(&bad[2], (unsigned long long)j); break; }
    }
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += stride)
        if (tgt[e] >= n) atomicMin(&bad[1], (unsigned long long)e);
}

cudaError_t launch_validate_csr(const uint64_t* off, const uint32_t* tgt, uint64_t n,
                                uint64_t nnz, unsigned long long* bad, bool check_sorted,
                                const Device& dev, cudaStream_t s) {
    validate_csr_kernel<<<grid_for(std::max(n, nnz), 256, dev), 256, 0, s>>>(off, tgt, n, nnz, bad,
                                                                            check_sorted);
    return cudaGetLastError();
}

// O9 (P:313 GraphVite's init, reading D11): V[i][c] = ((x[c&3] >> 8) * 2^-24 - 0.5) / d,
// x = Philox((i_lo, i_hi, c/4, INIT<<24)).  IEEE division (no fast-math), so the
// result is bit-identical to any correctly rounded implementation.
__global__ void init_vertex_kernel(float* __restrict__ V, uint64_t row_begin, uint64_t rows,
                                   uint32_t d, uint64_t seed, bool bf16) {
    const uint32_t q = d / 4;
    const uint64_t total = rows * q;
    const uint2 key = key_of(seed);
    const float fd = (float)d;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += stride) {
        const uint64_t r = w / q;
        const uint32_t c4 = (uint32_t)(w - r * q);
        const uint64_t i = row_begin + r;
        const uint4 x = philox(make_uint4((uint32_t)i, (uint32_t)(i >> 32), c4, kTagInit << 24), key);
        float4 o;
        o.x = __fdiv_rn(__fsub_rn(__fmul_rn((float)(x.x >> 8), 0x1p-24f), 0.5f), fd);
        o.y = __fdiv_rn(__fsub_rn(__fmul_rn((float)(x.y >> 8), 0x1p-24f), 0.5f), fd);
        o.z = __fdiv_rn(__fsub_rn(__fmul_rn((float)(x.z >> 8), 0x1p-24f), 0.5f), fd);
        o.w = __fdiv_rn(__fsub_rn(__fmul_rn((float)(x.w >> 8), 0x1p-24f), 0.5f), fd);
        if (bf16) {  // NEXT-4 (D16): the O9 value rounded to the nearest bf16
            const __nv_bfloat162 a = __floats2bfloat162_rn(o.x, o.y), b = __floats2bfloat162_rn(o.z, o.w);
            reinterpret_cast<uint2*>(V)[w] = make_uint2(*reinterpret_cast<const uint32_t*>(&a),
                                                        *reinterpret_cast<const uint32_t*>(&b));
        } else {
            reinterpret_cast<float4*>(V)[w] = o;
        }
    }
}

// bf16 rows (NEXT-4) <-> fp32 host arrays: exact widening; rounding to nearest even.
__global__ void convert_rows_kernel(const void* __restrict__ in, void* __restrict__ out, uint64_t n,
                                    bool to_bf16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (to_bf16) {
            reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(reinterpret_cast<const float*>(in)[i]);
        } else {
            const uint32_t h = reinterpret_cast<const uint16_t*>(in)[i];
            reinterpret_cast<float*>(out)[i] = __uint_as_float(h << 16);
        }
    }
}

cudaError_t launch_convert_rows(const void* in, void* out, uint64_t n, bool to_bf16, const Device& dev,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    convert_rows_kernel<<<grid_for(n, 256, dev), 256, 0, s>>>(in, out, n, to_bf16);
    return cudaGetLastError();
}

cudaError_t launch_init_vertex(float* V, uint64_t row_begin, uint64_t rows, uint32_t d,
                               uint64_t seed, bool bf16, const Device& dev, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    init_vertex_kernel<<<grid_for(rows * (d / 4), 256, dev), 256, 0, s>>>(V, row_begin, rows, d, seed, bf16);
    return cudaGetLastError();
}

// O4 walk engine (Alg. 1 "parallel random walk"), one
// lane per walker: the walk is a dependent chain (offsets -> target) so lanes
// of a warp advance 32 independent walkers to keep loads in flight.  Step t
// draws Philox(ctr = (omega_lo, omega_hi, t, WALK<<24 | epoch)) and picks
// neighbour R2(x0|x1<<32, deg).  Rows are padded with kSentinel after a sink.
// N2V (NEXT-1, node2vec P:355 by rejection as in KnightKing P:184): step t >= 2
// repeats trials r (ctr word 2 = t | r << 8) until x2 < thr[kind], kind = 0 if
// the candidate is the previous node, 1 if it is a neighbour of the previous
// node (binary search in its sorted row), 2 otherwise.
__device__ __forceinline__ bool has_edge(const uint64_t* __restrict__ off,
                                         const uint32_t* __restrict__ tgt, uint64_t v, uint32_t x) {
    uint64_t lo = __ldg(off + v), hi = __ldg(off + v + 1);  // lower bound of x in [lo, hi)
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(tgt + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo < __ldg(off + v + 1) && __ldg(tgt + lo) == x;
}

template <bool N2V>
__global__ void __launch_bounds__(256) walk_kernel(const uint64_t* __restrict__ off,
                                                   const uint32_t* __restrict__ tgt, uint64_t n,
                                                   uint64_t omega0, uint64_t count, uint32_t k,
                                                   uint64_t seed, uint32_t epoch, ulonglong4 thr,
                                                   uint32_t* __restrict__ walks, WalkCount wc) {
    const uint2 key = key_of(seed);
    const uint32_t tw = tag_word(kTagWalk, epoch);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < count; w += stride) {
        const uint64_t omega = omega0 + w;
        uint64_t cur = omega % n, prev = 0;
        uint32_t* out = walks + w * (uint64_t)(k + 1);
        out[0] = (uint32_t)cur;
        uint32_t t = 1, kept = 0;
        for (; t <= k; ++t) {
            const uint64_t b = __ldg(off + cur), e = __ldg(off + cur + 1);
            if (e == b) break;
            uint64_t cand;
            for (uint32_t r = 0;; ++r) {
                const uint4 x = philox(make_uint4((uint32_t)omega, (uint32_t)(omega >> 32), t | (r << 8), tw), key);
                cand = __ldg(tgt + b + uniform_index(x.x, x.y, e - b));
                if (!N2V || t == 1 || r + 1 == (1u << 24)) break;
                const uint64_t th = cand == prev ? thr.x : (has_edge(off, tgt, prev, (uint32_t)cand) ? thr.y : thr.z);
                if ((uint64_t)x.z < th) break;
            }
            prev = cur;
            cur = cand;
            out[t] = (uint32_t)cur;
            // O5: node t is the context of the min(t, l) window slots (t - delta, t)
            if (cur >= wc.c_begin && cur < wc.c_end) kept += min(t, wc.l);
        }
        for (; t <= k; ++t) out[t] = kSentinel;
        if (wc.counts) wc.counts[w] = kept;
    }
}

cudaError_t launch_walk(const uint64_t* off, const uint32_t* tgt, uint64_t n, uint64_t omega0,
                        uint64_t count, uint32_t k, uint64_t seed, uint32_t epoch,
                        const uint64_t* n2v_thr, uint32_t* walks, const WalkCount& wc, const Device& dev,
                        cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    if (n2v_thr) {
        const ulonglong4 thr = make_ulonglong4(n2v_thr[0], n2v_thr[1], n2v_thr[2], 0);
        walk_kernel<true><<<grid_for(count, 256, dev), 256, 0, s>>>(off, tgt, n, omega0, count, k, seed,
                                                                     epoch, thr, walks, wc);
    } else {
        walk_kernel<false><<<grid_for(count, 256, dev), 256, 0, s>>>(off, tgt, n, omega0, count, k, seed,
                                                                      epoch, make_ulonglong4(0, 0, 0, 0), walks, wc);
    }
    return cudaGetLastError();
}

}  // namespace ne

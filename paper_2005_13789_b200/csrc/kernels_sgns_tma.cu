// kernels_sgns_tma.cu -- SGNS update (Alg. 1) with the rows of each
// iteration staged in shared memory by TMA bulk copies (sm_100a).
//
// Why: the register kernel (kernels_sgns.cu) only has loads in flight during
// each iteration's load phase; the 1+K sequential updates that follow leave
// HBM idle for that warp.  Here every warp owns a two-stage shared-memory ring:
// while it computes iteration i from stage i&1, the 2(2+K) rows of iteration
// i+1 (the two samples' vertex rows, positive and negative context rows) are
// already streaming into stage (i+1)&1 -- one cp.async.bulk (UBLKCP) per
// 512-byte row, completion tracked by an mbarrier with expect_tx.  Only one
// context row at a time is held in registers, so the register file no longer
// caps the bytes in flight; shared memory does (2 stages x 7 KB per warp at
// d = 128, K = 5).
//
// Mapping and arithmetic are those of the register kernel: 16 lanes per
// sample, two samples per warp, sgns_step from sgns_common.cuh.  Hogwild
// write-back by red.global.add.v4.f32 deltas (or plain stores).  Prefetched
// rows may be one iteration stale (Hogwild semantics); in deterministic mode
// the copies of iteration i are issued only after iteration i-1's writes are
// fenced into the async proxy, so one warp reproduces the canonical order.
#include <algorithm>
#include <cstdlib>

#include "sgns_common.cuh"

namespace ne {

namespace {

constexpr int kTmaWarps = 4;  // warps per CTA
constexpr int kG = 16;        // lanes per sample
constexpr int kS = 32 / kG;   // samples per warp-iteration

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n NE_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra NE_WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared (no tensor map: a contiguous row)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

}  // namespace

template <int R, int KT, bool ADD>
__global__ void __launch_bounds__(kTmaWarps * 32) sgns_tma_kernel(SgnsParams p) {
    constexpr int G = kG, S = kS;
    constexpr int KM = KT > 0 ? KT : kMaxK;
    const int K = KT > 0 ? KT : (int)p.K;
    const uint32_t lane = lane_id(), sub = lane % G, h = lane / G, wib = threadIdx.x >> 5;
    const uint32_t rps = 2u + (uint32_t)K;      // rows per sample: v, c_0 .. c_K
    const uint32_t rb = p.d * 4u;               // row bytes (multiple of 16)
    const uint32_t stage_bytes = S * rps * rb;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + 2 * wib;
    unsigned char* buf = smem + 128 + (size_t)wib * 2 * stage_bytes;

    const bool det = p.deterministic != 0;
    const uint32_t spw = det ? 1u : (uint32_t)S;
    const uint64_t stride = (((uint64_t)gridDim.x * blockDim.x) >> 5) * spw;
    const uint32_t q = p.d >> 2;
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    double loss = 0.0;

    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    // pair + negatives of the iteration starting at sample b (lane L < spw*K
    // draws negative L % K of sample b + L / K)
    auto fetch = [&](uint64_t b, uint2& pr, uint32_t& neg) {
        pr = (h < spw && b + h < p.count) ? p.pool[b + h] : make_uint2(0, 0);
        const uint64_t ps = b + lane / (uint32_t)(K > 0 ? K : 1);
        neg = (K > 0 && lane < spw * (uint32_t)K && ps < p.count) ? draw_negative(p, key, tagw, ps, lane % K) : 0u;
    };
    // lane sub = j <= K of group h gets ids[j] (0: positive context, 1..K: negatives)
    auto group_id = [&](const uint2& pr, uint32_t neg) -> uint32_t {
        const uint32_t nj = __shfl_sync(0xFFFFFFFFu, neg, (h * K + sub + 31) & 31);
        return sub == 0 ? pr.y : nj;
    };
    // issue the bulk copies of the iteration at b into stage st
    auto issue = [&](uint64_t b, const uint2& pr, uint32_t neg, uint32_t st) {
        const uint32_t my_id = group_id(pr, neg);
        const uint64_t left = b < p.count ? p.count - b : 0;
        const uint32_t nact = left < spw ? (uint32_t)left : spw;
        const uint32_t hh = lane / rps < (uint32_t)S ? lane / rps : (uint32_t)S - 1, r = lane % rps;
        const uint32_t srcv = __shfl_sync(0xFFFFFFFFu, pr.x, hh * G);
        const uint32_t idv = __shfl_sync(0xFFFFFFFFu, my_id, hh * G + (r == 0 ? 0u : r - 1));
        if (lane == 0 && nact) mbar_expect_tx(&bars[st], nact * rps * rb);
        __syncwarp();
        if (lane < nact * rps) {
            const float* g = r == 0 ? p.V + (uint64_t)(srcv - p.v_begin) * p.d
                                    : p.C + (uint64_t)(idv - p.c_begin) * p.d;
            bulk_g2s(buf + (size_t)st * stage_bytes + (size_t)(hh * rps + r) * rb, g, rb, &bars[st]);
        }
    };

    uint64_t base = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * spw;
    uint2 prA, prB = make_uint2(0, 0);
    uint32_t negA, negB = 0;
    fetch(base, prA, negA);
    if (!det) {
        if (base < p.count) issue(base, prA, negA, 0);
        fetch(base + stride, prB, negB);
    }
    for (uint32_t it = 0; base < p.count; base += stride, ++it) {
        const uint32_t st = it & 1u, par = (it >> 1) & 1u;
        if (det) {
            issue(base, prA, negA, st);
            fetch(base + stride, prB, negB);
        } else if (base + stride < p.count) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // stage reads of it-1 before refill
            issue(base + stride, prB, negB, st ^ 1u);
        }
        const uint64_t pos = base + h;
        const bool act = h < spw && pos < p.count;
        const uint32_t my_id = group_id(prA, negA);
        uint32_t ids[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) ids[j] = __shfl_sync(0xFFFFFFFFu, my_id, h * G + j);
        const uint64_t mkey = (act && (int)sub <= K) ? (((uint64_t)h << 33) | my_id) : ((1ull << 32) | lane);
        const bool dup = __any_sync(0xFFFFFFFFu, __popc(__match_any_sync(0xFFFFFFFFu, mkey)) > 1);
        float4* vrow = reinterpret_cast<float4*>(p.V + (uint64_t)(prA.x - p.v_begin) * p.d);
        // ids of the iteration after next, while this iteration's rows land
        uint2 prC = make_uint2(0, 0);
        uint32_t negC = 0;
        if (!det) fetch(base + 2 * stride, prC, negC);

        mbar_wait(&bars[st], par);
        const float4* sv = reinterpret_cast<const float4*>(buf + (size_t)st * stage_bytes + (size_t)h * rps * rb);
        const uint32_t rq = rb / 16;  // float4 per row
        float4 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            v[r] = (act && e < q) ? sv[e] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j <= KM; ++j) {
            if (j <= K) {
                float4 c[R], vo[R];
                const float4* sc = sv + (size_t)(1 + j) * rq;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t e = sub + G * r;
                    c[r] = (act && e < q) ? sc[e] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                float lt;
                const float a = sgns_step<G, R>(v, c, vo, p.lr, j == 0, lt);
                if (sub == 0 && act) loss += (double)lt;
                bool last = true;
                if (dup && act) {  // hand the updated row to the later occurrences of the same id
#pragma unroll
                    for (int i = j + 1; i <= KM; ++i)
                        if (i <= K && ids[i] == ids[j]) {
                            last = false;
                            float4* sl = const_cast<float4*>(sv) + (size_t)(1 + i) * rq;
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const uint32_t e = sub + G * r;
                                if (e < q) sl[e] = c[r];
                            }
                        }
                }
                float4* crow = reinterpret_cast<float4*>(p.C + (uint64_t)(ids[j] - p.c_begin) * p.d);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t e = sub + G * r;
                    if (act && e < q) {
                        if constexpr (ADD)
                            atomicAdd(crow + e, scaled(-a, vo[r]));
                        else if (last)
                            crow[e] = c[r];
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            if (act && e < q) {
                if constexpr (ADD) {
                    const float4 v0 = sv[e];  // the staged copy is the pre-update row
                    atomicAdd(vrow + e, make_float4(v[r].x - v0.x, v[r].y - v0.y, v[r].z - v0.z, v[r].w - v0.w));
                } else {
                    vrow[e] = v[r];
                }
            }
        }
        if (det) asm volatile("fence.proxy.async.global;" ::: "memory");  // writes -> next copies
        __syncwarp();
        prA = prB;
        negA = negB;
        prB = prC;
        negB = negC;
    }
    if (sub == 0 && loss != 0.0) atomicAdd(p.loss, loss);
}

size_t sgns_tma_smem_bytes(uint32_t d, uint32_t K) {
    return 128 + (size_t)kTmaWarps * 2 * kS * (2 + K) * d * 4;
}

template <int R, int KT>
static cudaError_t launch_tma_k(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    const size_t smem = sgns_tma_smem_bytes(p.d, p.K);
    auto kern = p.atomic_writeback && !p.deterministic ? sgns_tma_kernel<R, KT, true> : sgns_tma_kernel<R, KT, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (p.deterministic) {
        kern<<<1, 32, smem, s>>>(p);
        return cudaGetLastError();
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTmaWarps * 32, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, 1);
    const uint64_t want = std::min<uint64_t>(p.count, std::max<uint64_t>(p.max_warps, 1));
    if (want < (uint64_t)kS) {  // one sample at a time, canonical order
        SgnsParams q = p;
        q.deterministic = 1;
        kern<<<1, 32, smem, s>>>(q);
        return cudaGetLastError();
    }
    const uint64_t warps = want / kS;
    const uint64_t full = (uint64_t)dev.sm_count * per_sm;
    if (warps >= full * kTmaWarps) {
        kern<<<(unsigned)full, kTmaWarps * 32, smem, s>>>(p);
    } else if (warps >= (uint64_t)dev.sm_count * kTmaWarps) {
        kern<<<(unsigned)((warps + kTmaWarps - 1) / kTmaWarps), kTmaWarps * 32, smem, s>>>(p);
    } else {
        kern<<<(unsigned)warps, 32, smem, s>>>(p);
    }
    return cudaGetLastError();
}

// Returns cudaErrorNotSupported when the shape does not fit the staged kernel.
cudaError_t launch_sgns_tma(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    const uint32_t q = p.d / 4;
    if (sgns_tma_smem_bytes(p.d, p.K) > 200 * 1024) return cudaErrorNotSupported;
    const uint32_t R = (q + kG - 1) / kG;
    if (p.K == 5) {
        switch (R) {
            case 1: return launch_tma_k<1, 5>(p, dev, s);
            case 2: return launch_tma_k<2, 5>(p, dev, s);
            case 3: return launch_tma_k<3, 5>(p, dev, s);
            case 4: return launch_tma_k<4, 5>(p, dev, s);
            default: return cudaErrorNotSupported;
        }
    }
    switch (R) {
        case 1: return launch_tma_k<1, 0>(p, dev, s);
        case 2: return launch_tma_k<2, 0>(p, dev, s);
        case 3: return launch_tma_k<3, 0>(p, dev, s);
        case 4: return launch_tma_k<4, 0>(p, dev, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace ne

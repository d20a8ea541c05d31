// sgns_kernel.cuh -- the SGNS kernel template and its launch chain, shared by
// kernels_sgns.cu (fp32 rows) and kernels_sgns_bf16.cu (bf16 rows, NEXT-4) so
// the two instantiation sets compile as separate translation units.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "sgns_common.cuh"

namespace ne {

constexpr int kSgnsThreads = 256;

// G: lanes per sample (16 or 32); a warp trains S = 32/G samples side by side,
// each lane owning R float4 of every row (d <= 4 G R).  KT: compile-time K
// (0 = runtime K <= kMaxK).  MINB: min resident CTAs per SM (register budget).
// ADD: Hogwild write-back by vector reduction (red.global.add.v4.f32) of each
// update's delta instead of a plain store of the new row, so concurrent samples
// sharing a row never erase each other's updates (they only read stale values).
// PF: the ids of iteration i+1 are known one iteration early (pairs and
// negatives are fetched two iterations ahead), so at the top of iteration i
// every lane prefetches ~2 of the 128-byte lines of iteration i+1's rows into
// L2 (prefetch.global.L2); the next iteration's row loads then hit L2.  A
// prefetch never changes values (L2 is the point of coherence), so it is valid
// in deterministic mode too.
// p.deterministic: only group 0 of the (single) warp works, one sample at a
// time in canonical order -- the same arithmetic as the production mapping.
// ACC: NEXT-4 accumulated-gradient rule (all 1+K dots against the pre-sample
// vertex row, which is updated once at the end): the 1+K group reductions are
// independent, so they overlap instead of forming one dependency chain.
// BF: rows stored as bfloat16 (NEXT-4, reading D16): loads widen 4 bf16 to a
// float4, stores round to nearest even, Hogwild deltas go through a bf16x2
// vector reduction; all arithmetic stays fp32 (RowIO in sgns_common.cuh).
template <int G, int R, int KT, int MINB, bool ADD, bool PF, bool ACC = false, bool BF = false>
__global__ void __launch_bounds__(kSgnsThreads, MINB) sgns_kernel(SgnsParams p) {
    static_assert(!(PF && BF), "L2 prefetch is an fp32-only developer knob");
    using IO = RowIO<BF>;
    constexpr int S = 32 / G;
    constexpr int KM = KT > 0 ? KT : kMaxK;
    const int K = KT > 0 ? KT : (int)p.K;
    const uint32_t lane = lane_id(), sub = lane % G, h = lane / G;
    const uint32_t spw = p.deterministic ? 1u : (uint32_t)S;  // samples per warp-iteration
    const uint64_t stride = (((uint64_t)gridDim.x * blockDim.x) >> 5) * spw;
    const uint32_t q = p.d >> 2;  // float4 per row
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    double loss = 0.0;  // lane sub == 0 of each group

    // pair + negatives of the iteration starting at sample b (lane L < spw*K
    // draws negative L % K of sample b + L / K); the alias entry is loaded here
    // and the coin decided at first use (finish_negative in group_id)
    auto fetch = [&](uint64_t b, uint2& pr, NegDraw& neg) {
        pr = (h < spw && b + h < p.count) ? p.pool[b + h] : make_uint2(0, 0);
        const uint64_t ps = b + lane / (uint32_t)(K > 0 ? K : 1);
        if (K > 0 && lane < spw * (uint32_t)K && ps < p.count) neg = issue_negative(p, key, tagw, ps, lane % K);
        else neg = NegDraw{0u, 0u, make_uint2(0u, 0u)};
    };
    // lane sub = j <= K of group h gets ids[j] (0: positive context, 1..K: negatives)
    auto group_id = [&](const uint2& pr, const NegDraw& neg) -> uint32_t {
        const uint32_t nj = __shfl_sync(0xFFFFFFFFu, finish_negative(p, neg), (h * K + sub + 31) & 31);
        return sub == 0 ? pr.y : nj;
    };

    uint64_t base = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * spw;
    uint2 prA, prB = make_uint2(0, 0);
    NegDraw negA, negB = NegDraw{0u, 0u, make_uint2(0u, 0u)};
    fetch(base, prA, negA);
    if (PF) fetch(base + stride, prB, negB);
    const uint32_t lines = p.d >> 5;                 // 128-byte lines per row
    const uint32_t plines = (2u + (uint32_t)K) * lines;  // per sample
    for (; base < p.count; base += stride) {
        const uint64_t pos = base + h;
        const bool act = h < spw && pos < p.count;
        const uint32_t my_id = group_id(prA, negA);
        uint32_t ids[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) ids[j] = __shfl_sync(0xFFFFFFFFu, my_id, h * G + j);
        // a repeated context id inside a sample is rare: detect it once per iteration
        const uint64_t mkey = (act && (int)sub <= K) ? (((uint64_t)h << 33) | my_id) : ((1ull << 32) | lane);
        const bool dup = __any_sync(0xFFFFFFFFu, __popc(__match_any_sync(0xFFFFFFFFu, mkey)) > 1);

        const uint64_t vr = (uint64_t)(prA.x - p.v_begin);
        float4 v[R], v0[(ADD || ACC) ? R : 1], eacc[ACC ? R : 1];
        float4 c[KM + 1][R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            v[r] = (act && e < q) ? IO::load(p.V, vr, p.d, e) : make_float4(0.f, 0.f, 0.f, 0.f);
            if constexpr (ADD || ACC) v0[r] = v[r];
            if constexpr (ACC) eacc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j <= KM; ++j) {
            if (j <= K) {
                const uint64_t cr = (uint64_t)(ids[j] - p.c_begin);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t e = sub + G * r;
                    c[j][r] = (act && e < q) ? IO::load(p.C, cr, p.d, e) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }

        uint2 prC = make_uint2(0, 0);
        NegDraw negC = NegDraw{0u, 0u, make_uint2(0u, 0u)};
        if constexpr (PF) {
            // L2-prefetch the rows of iteration i+1 (ids known since iteration i-1)
            const uint64_t nb = base + stride;
            const bool nact = h < spw && nb + h < p.count;
            const uint32_t nid = group_id(prB, negB);
            for (uint32_t L = sub; L < ((plines + G - 1) / G) * G; L += G) {
                const uint32_t row = L / lines, line = L % lines;
                const uint32_t rid = __shfl_sync(0xFFFFFFFFu, nid, h * G + (row == 0 ? 0u : row - 1u));
                if (nact && L < plines) {
                    const float* a = row == 0 ? p.V + (uint64_t)(prB.x - p.v_begin) * p.d
                                              : p.C + (uint64_t)(rid - p.c_begin) * p.d;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a + line * 32));
                }
            }
            fetch(base + 2 * stride, prC, negC);  // ids two iterations ahead
        } else {
            fetch(base + stride, prB, negB);     // ids one iteration ahead
        }

        // Alg. 1 lines 10 and 12: positive, then the K negatives, in order.
#pragma unroll
        for (int j = 0; j <= KM; ++j) {
            if (j <= K) {
                bool last = true;  // no later occurrence of ids[j] in this sample
                if (dup) {
#pragma unroll
                    for (int i = 0; i < j; ++i)  // forward the latest copy of a repeated id
                        if (ids[i] == ids[j]) {
#pragma unroll
                            for (int r = 0; r < R; ++r) c[j][r] = c[i][r];
                        }
#pragma unroll
                    for (int i = j + 1; i <= KM; ++i)
                        if (i <= K && ids[i] == ids[j]) last = false;
                }
                float4 vo[R];
                float lt, a;
                if constexpr (ACC) {
                    a = sgns_step_acc<G, R>(v0, c[j], eacc, p.lr, j == 0, lt);
#pragma unroll
                    for (int r = 0; r < R; ++r) vo[r] = v0[r];
                } else {
                    a = sgns_step<G, R>(v, c[j], vo, p.lr, j == 0, lt);
                }
                if (sub == 0 && act) loss += (double)lt;
                const uint64_t cr = (uint64_t)(ids[j] - p.c_begin);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t e = sub + G * r;
                    if (act && e < q) {
                        if constexpr (ADD)  // this update's delta, at every occurrence
                            IO::add(p.C, cr, p.d, e, scaled(-a, vo[r]));
                        else if (last)      // the row's final value, once
                            IO::store(p.C, cr, p.d, e, c[j][r]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            if constexpr (ACC)
                v[r] = make_float4(v0[r].x - eacc[r].x, v0[r].y - eacc[r].y, v0[r].z - eacc[r].z, v0[r].w - eacc[r].w);
            if (act && e < q) {
                if constexpr (ADD)
                    IO::add(p.V, vr, p.d, e, make_float4(v[r].x - v0[r].x, v[r].y - v0[r].y,
                                                         v[r].z - v0[r].z, v[r].w - v0[r].w));
                else
                    IO::store(p.V, vr, p.d, e, v[r]);
            }
        }
        prA = prB;
        negA = negB;
        if constexpr (PF) {
            prB = prC;
            negB = negC;
        }
    }
    if (sub == 0 && loss != 0.0) atomicAdd(p.loss, loss);
}

static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <int G, int R, int KT, int MINB, bool BF>
static cudaError_t launch_sgns_v(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    // developer knob: L2 row prefetch (measured: no gain; fp32 rows only)
    static const bool pf_knob = env_int("NE_SGNS_PF", 0) != 0;
    const bool pf = pf_knob && !BF;
    constexpr bool PFB = !BF;  // the prefetch instantiations exist for fp32 rows only
    if (p.deterministic) {  // one warp, one sample at a time, canonical order, plain stores
        if (p.accumulate) sgns_kernel<G, R, KT, MINB, false, false, true, BF><<<1, 32, 0, s>>>(p);
        else if (pf) sgns_kernel<G, R, KT, MINB, false, PFB, false, BF><<<1, 32, 0, s>>>(p);
        else sgns_kernel<G, R, KT, MINB, false, false, false, BF><<<1, 32, 0, s>>>(p);
        return cudaGetLastError();
    }
    auto kern = p.accumulate
                    ? (p.atomic_writeback ? sgns_kernel<G, R, KT, MINB, true, false, true, BF>
                                          : sgns_kernel<G, R, KT, MINB, false, false, true, BF>)
                : p.atomic_writeback ? (pf ? sgns_kernel<G, R, KT, MINB, true, PFB, false, BF>
                                           : sgns_kernel<G, R, KT, MINB, true, false, false, BF>)
                                     : (pf ? sgns_kernel<G, R, KT, MINB, false, PFB, false, BF>
                                           : sgns_kernel<G, R, KT, MINB, false, false, false, BF>);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSgnsThreads, 0);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, 1);
    constexpr int S = 32 / G;
    // concurrency cap counts samples in flight: warps = cap / S
    const uint64_t want = std::min<uint64_t>(p.count, std::max<uint64_t>(p.max_warps, 1));
    if (want < (uint64_t)S) {  // fewer samples in flight than a warp carries: one at a time
        SgnsParams q = p;
        q.deterministic = 1;  // sequential canonical order, production write-back
        kern<<<1, 32, 0, s>>>(q);
        return cudaGetLastError();
    }
    const uint64_t warps = want / S;
    const uint64_t full = (uint64_t)std::max(1, dev.sm_count - p.reserve_sms) * per_sm;
    const int wpb = kSgnsThreads / 32;
    if (warps >= full * wpb) {
        kern<<<(unsigned)full, kSgnsThreads, 0, s>>>(p);
    } else if (warps >= (uint64_t)dev.sm_count * wpb) {
        kern<<<(unsigned)((warps + wpb - 1) / wpb), kSgnsThreads, 0, s>>>(p);
    } else {  // small capped grids: spread single warps over the SMs
        kern<<<(unsigned)warps, 32, 0, s>>>(p);
    }
    return cudaGetLastError();
}

// Occupancy variant (developer knob NE_SGNS_MINB = 2..3): the register budget
// __launch_bounds__(256, MINB) gives the compiler.  Defaults: 16-lane groups
// carry two samples' rows per lane (MINB 2); 32-lane groups MINB 3.

template <int G, int R, int KT, bool BF>
static cudaError_t launch_sgns_k(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if constexpr (R > 2 && G == 32) {  // wide rows (d > 256): the register file holds 2+K rows of up to 2 KB
        return launch_sgns_v<G, R, KT, 1, BF>(p, dev, s);
    }
    static const int knob = env_int("NE_SGNS_MINB", 0);
    // 16-lane groups hold two samples' rows per lane, 32-lane groups with R = 2
    // (d <= 256) hold 2 float4 per row: both need the 128-register budget of 2 CTAs
    // defaults (measured): 8-lane groups 1 CTA/SM (974 vs 841 M/s at 2 with spills,
    // C4); 16-lane groups and 32-lane R = 2 need 128 registers (2 CTAs); else 3
    int minb = knob >= 1 && knob <= 4 ? knob : (G == 8 ? 1 : (G == 16 || R == 2 ? 2 : 3));
    if (KT == 0) minb = std::min(minb, 2);  // runtime K keeps kMaxK+1 rows live: stay spill-free
    // (the knob's other budgets were measured and dropped: 1 and 4 CTAs/SM lose,
    // except for 8-lane groups, whose 3 float4 per row fit 1 CTA/SM spill-free)
    if constexpr (G == 8) {
        if (minb <= 1) return launch_sgns_v<G, R, KT, 1, BF>(p, dev, s);
    }
    if (minb <= 2) return launch_sgns_v<G, R, KT, 2, BF>(p, dev, s);
    return launch_sgns_v<G, R, KT, 3, BF>(p, dev, s);
}

template <int G, int R, bool BF>
static cudaError_t launch_sgns_r(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if (p.K == 5) return launch_sgns_k<G, R, 5, BF>(p, dev, s);  // the paper's K (tab:perf)
    return launch_sgns_k<G, R, 0, BF>(p, dev, s);
}

// Register-kernel selection by row width (both storage types).
template <bool BF>
cudaError_t launch_sgns_rows(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    const uint32_t q = p.d / 4;
    // d <= 128: 16 lanes x 2 float4 (two samples per warp; developer knob
    // NE_SGNS_LANES=32 selects one sample per warp); d > 128: 32 lanes x R.
    static const int lanes = env_int("NE_SGNS_LANES", 16);
    // 64 < d <= 96 at K = 5: 8-lane groups x 3 float4, four samples per warp, so
    // a 384-byte row uses every lane (16-lane groups leave a quarter idle)
    if (q > 16 && q <= 24 && p.K == 5 && lanes != 32 && env_int("NE_SGNS_G8", 1))
        return launch_sgns_k<8, 3, 5, BF>(p, dev, s);
    if (q <= 32 && lanes == 16) {
        if (q <= 16) return launch_sgns_r<16, 1, BF>(p, dev, s);
        return launch_sgns_r<16, 2, BF>(p, dev, s);
    }
    switch ((q + 31) / 32) {
        case 1: return launch_sgns_r<32, 1, BF>(p, dev, s);
        case 2: return launch_sgns_r<32, 2, BF>(p, dev, s);
        case 3: return launch_sgns_r<32, 3, BF>(p, dev, s);
        default: return launch_sgns_r<32, 4, BF>(p, dev, s);
    }
}

}  // namespace ne

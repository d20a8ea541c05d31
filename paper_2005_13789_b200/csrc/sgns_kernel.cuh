// sgns_kernel.cuh -- the SGNS kernel template and its launch chain, shared by
// kernels_sgns.cu (fp32 rows) and kernels_sgns_bf16.cu (bf16 rows, NEXT-4) so
// the two instantiation sets compile as separate translation units.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "sgns_common.cuh"

namespace ne {


// G: lanes per sample (8, 16 or 32); a warp trains S = 32/G samples side by
// side, each lane owning R float4 of every row (d <= 4 G R).  KT: compile-time K
// (0 = runtime K <= kMaxK).  T, MINB: threads per CTA and min resident CTAs per
// SM -- the register budget (65536 / (T MINB) per thread) and the granularity
// at which CTAs fill the register file (launch shapes below).
// ADD: Hogwild write-back by vector reduction (red.global.add.v4.f32) of each
// update's delta instead of a plain store of the new row, so concurrent samples
// sharing a row never erase each other's updates (they only read stale values).
// p.deterministic: only group 0 of the (single) warp works, one sample at a
// time in canonical order -- the same arithmetic as the production mapping.
// ACC: NEXT-4 accumulated-gradient rule (all 1+K dots against the pre-sample
// vertex row, which is updated once at the end): the 1+K group reductions are
// independent, so they overlap instead of forming one dependency chain.
// BF: rows stored as bfloat16 (NEXT-4, reading D16): loads widen 4 bf16 to a
// float4, stores round to nearest even, Hogwild deltas go through a bf16x2
// vector reduction; all arithmetic stays fp32 (RowIO in sgns_common.cuh).
// p.capture (test hook, ne_capture_block): every group also writes the ids it
// trained -- (src, dst, neg_0 .. neg_{K-1}) at capture[pos * (2 + K)] -- so the
// lane -> sample -> negative routing of the full production grid is checked
// against the oracle position by position.
template <int G, int R, int KT, int T, int MINB, bool ADD, bool ACC, bool BF>
__global__ void __launch_bounds__(T, MINB) sgns_kernel(SgnsParams p) {
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
    // developer knob p.l2hint (fp32 rows): L2 eviction priorities for vertex / context rows
    const bool hint = !BF && p.l2hint != 0;
    uint64_t pol_v = 0, pol_c = 0;
    if (hint) {
        pol_v = l2_policy(p.l2hint & 3u);         // bits 0-1: vertex rows (1 evict_first, 2 evict_last)
        pol_c = l2_policy((p.l2hint >> 2) & 3u);  // bits 2-3: context rows
    }
    auto row_load = [&](const float* m, uint64_t row, uint32_t e, uint64_t pol) -> float4 {
        if constexpr (!BF) {
            if (hint) return IO::load(m, row, p.d, e, pol);
        }
        return IO::load(m, row, p.d, e);
    };
    auto row_add = [&](float* m, uint64_t row, uint32_t e, float4 dv, uint64_t pol) {
        if constexpr (!BF) {
            if (hint) return IO::add(m, row, p.d, e, dv, pol);
        }
        IO::add(m, row, p.d, e, dv);
    };

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
    uint2 prA, prB;
    NegDraw negA, negB;
    fetch(base, prA, negA);
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
        if (p.capture && act) {
            uint32_t* cap = p.capture + pos * (2u + (uint32_t)K);
            if (sub == 0) cap[0] = prA.x;
            if ((int)sub <= K) cap[1 + sub] = my_id;
        }

        const uint64_t vr = (uint64_t)(prA.x - p.v_begin);
        float4 v[R], v0[(ADD || ACC) ? R : 1], eacc[ACC ? R : 1];
        float4 c[KM + 1][R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            v[r] = (act && e < q) ? row_load(p.V, vr, e, pol_v) : make_float4(0.f, 0.f, 0.f, 0.f);
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
                    c[j][r] = (act && e < q) ? row_load(p.C, cr, e, pol_c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }

        fetch(base + stride, prB, negB);  // ids one iteration ahead

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
                            row_add(p.C, cr, e, scaled(-a, vo[r]), pol_c);
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
                    row_add(p.V, vr, e, make_float4(v[r].x - v0[r].x, v[r].y - v0[r].y,
                                                    v[r].z - v0[r].z, v[r].w - v0[r].w), pol_v);
                else
                    IO::store(p.V, vr, p.d, e, v[r]);
            }
        }
        prA = prB;
        negA = negB;
    }
    if (sub == 0 && loss != 0.0) atomicAdd(p.loss, loss);
}

// Shared-memory-staged production kernel (fp32 rows, Alg. 1 sequential rule,
// atomic-delta write-back, K = 5; knob NE_SGNS_STAGED): the same per-lane
// arithmetic (sgns_step) as sgns_kernel, but the 2+K rows of the NEXT
// iteration are copied global -> shared with cp.async (no registers) while the
// current iteration computes, double-buffered per warp, so every warp keeps a
// full iteration of row traffic in flight through its compute phase instead of
// alternating load and compute.  Rows are read from shared memory one step at
// a time (a repeated context id reads the slot its earlier occurrence was
// updated in).  Pairs and negatives run two iterations ahead.  Hogwild only:
// prefetching iteration i+1 before i's write-back is the same staleness
// concurrent warps already have; the deterministic mode keeps sgns_kernel.
template <int G, int R, int KT>
__global__ void __launch_bounds__(256, 2) sgns_staged_kernel(SgnsParams p) {
    constexpr int S = 32 / G, KM = KT > 0 ? KT : kMaxK, ROWS = 2 + KM, ROWF4 = G * R;
    const int K = KT > 0 ? KT : (int)p.K;
    constexpr int BUF = S * ROWS * ROWF4;  // float4 per buffer
    extern __shared__ float4 smem_rows[];
    const uint32_t lane = lane_id(), sub = lane % G, h = lane / G;
    float4* wbuf = smem_rows + (size_t)(threadIdx.x >> 5) * 2 * BUF;
    const uint64_t stride = (((uint64_t)gridDim.x * blockDim.x) >> 5) * S;
    const uint32_t q = p.d >> 2;
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    double loss = 0.0;
    auto fetch = [&](uint64_t b, uint2& pr, NegDraw& neg) {
        pr = (b + h < p.count) ? p.pool[b + h] : make_uint2(0, 0);
        const uint64_t ps = b + lane / (uint32_t)(K > 0 ? K : 1);
        if (K > 0 && lane < S * (uint32_t)K && ps < p.count) neg = issue_negative(p, key, tagw, ps, lane % K);
        else neg = NegDraw{0u, 0u, make_uint2(0u, 0u)};
    };
    auto group_id = [&](const uint2& pr, const NegDraw& neg) -> uint32_t {
        const uint32_t nj = __shfl_sync(0xFFFFFFFFu, finish_negative(p, neg), (h * K + sub + 31) & 31);
        return sub == 0 ? pr.y : nj;
    };
    // rows of the iteration at b (ids: this lane's group id list) into buffer buf
    auto stage = [&](uint64_t b, const uint2& pr, uint32_t my_id, float4* buf) {
        const bool act = b + h < p.count;
#pragma unroll
        for (int j = 0; j < ROWS; ++j) {
            if (j >= 2 + K) break;
            const uint32_t id = j == 0 ? pr.x : __shfl_sync(0xFFFFFFFFu, my_id, h * G + (j - 1));
            const float* rowp = j == 0 ? p.V + (uint64_t)(id - p.v_begin) * p.d : p.C + (uint64_t)(id - p.c_begin) * p.d;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = sub + G * r;
                if (act && e < q) {
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + (h * ROWS + j) * ROWF4 + e);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst),
                                 "l"(reinterpret_cast<const float4*>(rowp) + e)
                                 : "memory");
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    uint64_t base = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * S;
    uint2 prA, prB, prC;
    NegDraw negA, negB, negC;
    fetch(base, prA, negA);
    fetch(base + stride, prB, negB);
    uint32_t idA = group_id(prA, negA);
    stage(base, prA, idA, wbuf);
    uint32_t cur = 0;
    for (; base < p.count; base += stride) {
        const uint64_t pos = base + h;
        const bool act = pos < p.count;
        // the next iteration's rows start moving now; its pairs / negatives were
        // fetched one iteration ago, the one after it is fetched here
        const uint32_t idB = group_id(prB, negB);
        stage(base + stride, prB, idB, wbuf + (cur ^ 1) * BUF);
        fetch(base + 2 * stride, prC, negC);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
        float4* buf = wbuf + cur * BUF + h * ROWS * ROWF4;
        uint32_t ids[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) ids[j] = __shfl_sync(0xFFFFFFFFu, idA, h * G + j);
        const uint64_t mkey = (act && (int)sub <= K) ? (((uint64_t)h << 33) | idA) : ((1ull << 32) | lane);
        const bool dup = __any_sync(0xFFFFFFFFu, __popc(__match_any_sync(0xFFFFFFFFu, mkey)) > 1);
        if (p.capture && act) {
            uint32_t* capp = p.capture + pos * (2u + (uint32_t)K);
            if (sub == 0) capp[0] = prA.x;
            if ((int)sub <= K) capp[1 + sub] = idA;
        }
        float4 v[R], v0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            v[r] = (act && e < q) ? buf[e] : make_float4(0.f, 0.f, 0.f, 0.f);
            v0[r] = v[r];
        }
#pragma unroll
        for (int j = 0; j <= KM; ++j) {
            if (j > K) break;
            int slot = j;  // a repeated id reads the slot its latest earlier occurrence was updated in
            if (dup) {
#pragma unroll
                for (int i2 = 0; i2 < j; ++i2)
                    if (ids[i2] == ids[j]) slot = i2;
            }
            float4 c[R], vo[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = sub + G * r;
                c[r] = (act && e < q) ? buf[(1 + slot) * ROWF4 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float lt;
            const float a = sgns_step<G, R>(v, c, vo, p.lr, j == 0, lt);
            if (sub == 0 && act) loss += (double)lt;
            const uint64_t cr = (uint64_t)(ids[j] - p.c_begin);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = sub + G * r;
                if (act && e < q) {
                    RowIO<false>::add(p.C, cr, p.d, e, scaled(-a, vo[r]));
                    if (dup) buf[(1 + slot) * ROWF4 + e] = c[r];
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t e = sub + G * r;
            if (act && e < q)
                RowIO<false>::add(p.V, (uint64_t)(prA.x - p.v_begin), p.d, e,
                                  make_float4(v[r].x - v0[r].x, v[r].y - v0[r].y, v[r].z - v0[r].z, v[r].w - v0[r].w));
        }
        __syncwarp();  // every lane is done with this buffer before it is restaged
        prA = prB;
        negA = negB;
        idA = idB;
        prB = prC;
        negB = negC;
        cur ^= 1u;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (sub == 0 && loss != 0.0) atomicAdd(p.loss, loss);
}

template <int G, int R, int KT>
static cudaError_t launch_sgns_staged(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    constexpr int S = 32 / G, ROWS = 2 + (KT > 0 ? KT : kMaxK), ROWF4 = G * R;
    constexpr size_t smem = (size_t)(256 / 32) * 2 * S * ROWS * ROWF4 * sizeof(float4);
    auto kern = sgns_staged_kernel<G, R, KT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (e != cudaSuccess) return e;
    const uint64_t want = std::min<uint64_t>(p.count, std::max<uint64_t>(p.max_warps, 1));
    const uint64_t warps = std::max<uint64_t>(1, want / S);
    const uint64_t full = (uint64_t)std::max(1, dev.sm_count - p.reserve_sms) * std::max(per_sm, 1);
    const uint64_t blocks = std::min<uint64_t>(full, (warps + 7) / 8);
    kern<<<(unsigned)std::max<uint64_t>(1, blocks), 256, smem, s>>>(p);
    return cudaGetLastError();
}

static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// One launch shape: T threads per CTA, at least MINB CTAs per SM.
template <int T_, int MINB_>
struct Shape {
    static constexpr int T = T_, MINB = MINB_;
};

template <int G, int R, int KT, class SH, bool BF>
static cudaError_t launch_sgns_v(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    constexpr int T = SH::T, MB = SH::MINB;
    if (p.deterministic) {  // one warp, one sample at a time, canonical order, plain stores
        if (p.accumulate) sgns_kernel<G, R, KT, T, MB, false, true, BF><<<1, 32, 0, s>>>(p);
        else sgns_kernel<G, R, KT, T, MB, false, false, BF><<<1, 32, 0, s>>>(p);
        return cudaGetLastError();
    }
    auto kern = p.accumulate ? (p.atomic_writeback ? sgns_kernel<G, R, KT, T, MB, true, true, BF>
                                                   : sgns_kernel<G, R, KT, T, MB, false, true, BF>)
                             : (p.atomic_writeback ? sgns_kernel<G, R, KT, T, MB, true, false, BF>
                                                   : sgns_kernel<G, R, KT, T, MB, false, false, BF>);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, 0);
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
    constexpr int wpb = T / 32;
    if (warps >= full * wpb) {
        kern<<<(unsigned)full, T, 0, s>>>(p);
    } else if (warps >= (uint64_t)dev.sm_count * wpb) {
        kern<<<(unsigned)((warps + wpb - 1) / wpb), T, 0, s>>>(p);
    } else {  // small capped grids: spread single warps over the SMs
        kern<<<(unsigned)warps, 32, 0, s>>>(p);
    }
    return cudaGetLastError();
}

// Launch shapes (measured; registers per thread from -Xptxas -v):
//  * 16 lanes x 2 float4 (d <= 128) and 32 lanes x 2 (d <= 256): 256 threads,
//    2 CTAs/SM -> <= 128 registers, 16 warps/SM, spill-free;
//  * 8 lanes x 3 float4 (64 < d <= 96, K = 5): ~189 registers unconstrained,
//    256-thread CTAs, one per SM (8 warps).  Packing more warps per SM with
//    smaller CTAs (knob NE_SGNS_G8SHAPE: 1 = 64 x 5 -> 160 registers, 12
//    warps; 2 = 128 x 3) measured slower on C4: 902 / 906 vs 970 M samples/s;
//  * 32 lanes x 3-4 float4 (d > 256): 200-245 registers, 64-thread CTAs.
template <int G, int R, int KT, bool BF>
static cudaError_t launch_sgns_k(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if constexpr (G == 8) {
        static const int shape = env_int("NE_SGNS_G8SHAPE", 0);
        if constexpr (!BF) {
            if (shape == 1) return launch_sgns_v<G, R, KT, Shape<64, 5>, BF>(p, dev, s);
            if (shape == 2) return launch_sgns_v<G, R, KT, Shape<128, 3>, BF>(p, dev, s);
        }
        return launch_sgns_v<G, R, KT, Shape<256, 1>, BF>(p, dev, s);
    } else if constexpr (R > 2) {
        return launch_sgns_v<G, R, KT, Shape<64, 1>, BF>(p, dev, s);
    } else {
        return launch_sgns_v<G, R, KT, Shape<256, 2>, BF>(p, dev, s);
    }
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
    // 64 < d <= 96 at K = 5: 8-lane groups x 3 float4, four samples per warp, so
    // a 384-byte row uses every lane (16-lane groups leave a quarter idle)
    // (developer knob NE_SGNS_D96=16: the 16-lane kernel instead, read per launch)
    if (q > 16 && q <= 24 && p.K == 5 && env_int("NE_SGNS_D96", 8) != 16) return launch_sgns_k<8, 3, 5, BF>(p, dev, s);
    if constexpr (!BF) {  // developer knob: the shared-memory-staged kernel (d <= 128, K = 5, Hogwild)
        const int staged = env_int("NE_SGNS_STAGED", 0);  // read per launch: tests toggle it
        if (staged && q > 16 && q <= 32 && !p.deterministic && p.atomic_writeback && !p.accumulate &&
            p.max_warps >= 2)
            return p.K == 5 ? launch_sgns_staged<16, 2, 5>(p, dev, s) : launch_sgns_staged<16, 2, 0>(p, dev, s);
    }
    // d <= 128: 16 lanes x 1-2 float4, two samples per warp (measured against
    // 32 lanes x 1 float4, one sample per warp: 1093 vs 1003 M samples/s on C3)
    if (q <= 16) return launch_sgns_r<16, 1, BF>(p, dev, s);
    if (q <= 32) return launch_sgns_r<16, 2, BF>(p, dev, s);
    switch ((q + 31) / 32) {  // d > 128: 32 lanes x R float4
        case 2: return launch_sgns_r<32, 2, BF>(p, dev, s);
        case 3: return launch_sgns_r<32, 3, BF>(p, dev, s);
        default: return launch_sgns_r<32, 4, BF>(p, dev, s);
    }
}

}  // namespace ne

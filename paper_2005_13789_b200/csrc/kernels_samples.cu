// kernels_samples.cu -- network augmentation into the episode's sample pool
// (sm_100a): window pairs, canonical Feistel order (O6) and
// the stable bucketing into 2D blocks.
//
// Each rank handles only the pairs whose context node it owns: a count pass
// and an exclusive scan give every kept pair its part-local index x (its rank
// in generation order); pi over [0, N_g) is a bijection, so the pair's
// position y = pi(x) fixes its place in the canonical order.  Default (keyed)
// path: the pair kernel writes (pair, y) in generation order -- coalesced -- and
// 1-2 radix passes on y (CTA counting sort in shared memory, coalesced runs into
// regions whose sizes the bijection fixes) bring every pair into its
// 8192-position window; one CTA per window then places the pairs by y in shared
// memory and does the stable multi-way partition by vertex sub-part.  The
// direct path (one scattered 8-byte store per pair into a dense pi-indexed
// array, then the partition) is kept for pools that leave no room for the key
// buffers; both give the identical pool.  Measured on C3 (522 M pairs): random
// stores over a multi-GB target cost ~24 ms whether they miss L2 or not (TLB
// reach is 256 MB); all-sequential passes avoid that.
#include <algorithm>
#include <cstdlib>

#include "ne_device.cuh"
#include "ne_internal.h"

namespace ne {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kTile = 4096;                 // slots per CTA tile
constexpr uint32_t kPerWarp = kTile / kWarps;    // 512 slots, 16 chunks of 32
constexpr uint32_t kChunks = kPerWarp / 32;
constexpr uint32_t kScanChunk = 4096;            // elements per scan block
constexpr uint32_t kMaxBuckets = 256;
constexpr uint32_t kWin = 1u << kPoolWinBits;      // pi positions per window

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

Feistel make_feistel(const PoolParams& p) {
    uint32_t b = 0;
    while (b < 64 && (1ull << b) < p.N) ++b;
    if (b < 2) b = 2;
    Feistel f;
    f.N = p.N;
    f.c = b / 2;
    f.mask_lo = (1ull << f.c) - 1;
    f.mask_hi = (1ull << (b - f.c)) - 1;
    f.episode = p.episode;
    f.tagw = (kTagShuf << 24) | p.epoch;
    f.key = make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    return f;
}

unsigned grid_cap(uint64_t blocks, const Device& dev, int per_sm) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)dev.sm_count * per_sm));
}

}  // namespace

// Store pair number x (generation order) whose canonical position is y.
__device__ __forceinline__ void sink_put(const PoolSink& s, uint64_t x, uint64_t y, uint64_t pair) {
    if (s.key == nullptr) {
        s.out[y] = pair;
    } else {
        s.out[x] = pair;
        s.key[x] = (uint32_t)y;
    }
}

// Walk staging for the warp-per-walker kernels: the walk of the NEXT walker is
// copied global -> shared with cp.async (no registers, no wait) while the
// current one is processed, so the DRAM latency of the 4(k+1)-byte walk read is
// hidden (it was the dominant stall: ~35 % of samples in the ncu source view).
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void stage_walk(uint32_t* dst, const uint32_t* walks, uint64_t w, uint64_t units,
                                           uint32_t plen, uint32_t lane) {
    if (w < units) {
        const uint32_t* src = walks + w * (uint64_t)plen;
        for (uint32_t i = lane; i < plen; i += 32) cp_async4(dst + i, src + i);
    }
    cp_async_commit();
}

// O5 count, warp per walker: pairs of the walk whose context node is in the part.
__global__ void __launch_bounds__(kThreads) count_walk_kernel(const uint32_t* __restrict__ walks,
                                                              const uint32_t* __restrict__ slot_tab,
                                                              PoolParams p, uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t smem_path[];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t plen = p.k + 1;
    uint32_t* paths = smem_path + warp * 2 * plen;  // double buffer
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t buf = 0;
    stage_walk(paths, walks, w, p.units, plen, lane);
    for (; w < p.units; w += nwarps) {
        cp_async_wait_all();
        __syncwarp();
        const uint32_t* path = paths + buf * plen;
        stage_walk(paths + (buf ^ 1) * plen, walks, w + nwarps, p.units, plen, lane);
        uint32_t cnt = 0;
        uint32_t t_next = lane < p.Pw ? __ldg(slot_tab + lane) : 0u;
        for (uint32_t s0 = 0; s0 < p.Pw; s0 += 32) {
            const uint32_t s = s0 + lane, t = t_next;
            if (s + 32 < p.Pw) t_next = __ldg(slot_tab + s + 32);
            bool kept = false;
            if (s < p.Pw) {
                const uint32_t b = path[(t >> 16) + (t & 0xFFFFu)];
                kept = b != kSentinel && b >= p.c_begin && b < p.c_end;
            }
            cnt += __popc(__ballot_sync(0xFFFFFFFFu, kept));
        }
        if (lane == 0) counts[w] = cnt;
        buf ^= 1;
        __syncwarp();  // every lane is done with `path` before it is restaged
    }
    cp_async_wait_all();
}

cudaError_t launch_count_walk(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                              uint32_t* counts, const Device& dev, cudaStream_t s) {
    if (p.units == 0) return cudaSuccess;
    const size_t smem = (size_t)kWarps * 2 * (p.k + 1) * sizeof(uint32_t);
    count_walk_kernel<<<grid_cap(ceil_div(p.units, kWarps), dev, 8), kThreads, smem, s>>>(walks, slot_tab, p, counts);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) count_line_kernel(const uint32_t* __restrict__ tgt,
                                                              PoolParams p, uint32_t* __restrict__ counts) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < p.units; x += stride) {
        const uint32_t dst = __ldg(tgt + p.u0 + x);
        counts[x] = (dst >= p.c_begin && dst < p.c_end) ? 1u : 0u;
    }
}

cudaError_t launch_count_line(const uint32_t* tgt, const PoolParams& p, uint32_t* counts,
                              const Device& dev, cudaStream_t s) {
    if (p.units == 0) return cudaSuccess;
    count_line_kernel<<<grid_cap(ceil_div(p.units, kThreads), dev, 8), kThreads, 0, s>>>(tgt, p, counts);
    return cudaGetLastError();
}

// O5 + O6, warp per walker: the walk is staged in shared memory, the Pw window
// slots are taken 32 at a time in generation order; a kept pair's local index
// is base[w] + (kept pairs of earlier rounds) + (kept lanes below it).  Kept
// (x, pair) items go to a per-warp queue in shared memory and the Feistel runs
// on full batches of 32 queued items -- all lanes busy -- instead of on every
// round with the holes and foreign-part slots idling most lanes.
constexpr uint32_t kQueue = 64;  // per-warp queue capacity (>= 2 x 32)

__global__ void __launch_bounds__(kThreads) pairs_walk_kernel(const uint32_t* __restrict__ walks,
                                                              const uint32_t* __restrict__ slot_tab,
                                                              PoolParams p, Feistel f,
                                                              const uint64_t* __restrict__ base,
                                                              PoolSink sink) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t plen = p.k + 1;
    uint64_t* qx = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * 2 * kQueue;  // local index
    uint64_t* qp = qx + kQueue;                                                        // pair
    uint32_t* paths = reinterpret_cast<uint32_t*>(smem_raw + (size_t)kWarps * 2 * kQueue * 8) + warp * 2 * plen;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t buf = 0;
    stage_walk(paths, walks, w, p.units, plen, lane);
    uint64_t x_next = w < p.units ? __ldg(base + w) : 0;
    uint32_t qn = 0;  // queued items (warp-uniform)
    for (; w < p.units; w += nwarps) {
        cp_async_wait_all();
        __syncwarp();
        const uint32_t* path = paths + buf * plen;
        const uint64_t wn = w + nwarps;
        stage_walk(paths + (buf ^ 1) * plen, walks, wn, p.units, plen, lane);
        uint64_t x = x_next;
        x_next = wn < p.units ? __ldg(base + wn) : 0;
        uint32_t t_next = lane < p.Pw ? __ldg(slot_tab + lane) : 0u;
        for (uint32_t s0 = 0; s0 < p.Pw; s0 += 32) {
            const uint32_t s = s0 + lane, t = t_next;
            if (s + 32 < p.Pw) t_next = __ldg(slot_tab + s + 32);
            bool kept = false;
            uint32_t a = 0, b = 0;
            if (s < p.Pw) {
                const uint32_t i = t >> 16;
                b = path[i + (t & 0xFFFFu)];
                kept = b != kSentinel && b >= p.c_begin && b < p.c_end;
                a = path[i];
            }
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, kept);
            if (kept) {
                const uint32_t r = __popc(bal & lt);
                qx[qn + r] = x + r;
                qp[qn + r] = (uint64_t)a | ((uint64_t)b << 32);
            }
            x += __popc(bal);
            qn += __popc(bal);
            __syncwarp();
            if (qn >= 32) {  // one full batch: every lane permutes one item
                sink_put(sink, qx[lane], f(qx[lane]), qp[lane]);
                __syncwarp();
                if (lane < qn - 32) {
                    qx[lane] = qx[32 + lane];
                    qp[lane] = qp[32 + lane];
                }
                qn -= 32;
                __syncwarp();
            }
        }
        buf ^= 1;
        __syncwarp();  // every lane is done with `path` before it is restaged
    }
    cp_async_wait_all();
    if (lane < qn) sink_put(sink, qx[lane], f(qx[lane]), qp[lane]);  // the partial last batch
}

cudaError_t launch_pairs_walk(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                              const uint64_t* base, const PoolSink& sink, const Device& dev, cudaStream_t s) {
    if (p.units == 0 || p.N == 0) return cudaSuccess;
    const Feistel f = make_feistel(p);
    const size_t smem = (size_t)kWarps * (2 * kQueue * sizeof(uint64_t) + 2 * (p.k + 1) * sizeof(uint32_t));
    pairs_walk_kernel<<<grid_cap(ceil_div(p.units, kWarps), dev, 8), kThreads, smem, s>>>(
        walks, slot_tab, p, f, base, sink);
    return cudaGetLastError();
}

// ---- sharded construction at P > 1: O(N/P) work per rank ----------------------
// A rank walks only its shard of the episode's walkers and generates ALL their
// pairs; pairs travel to the rank owning their context part (the exchange in
// runtime.cpp).  Per walker w of the shard and part g: counts[g * units + w] =
// the walk's pairs whose context node lies in part g; one exclusive scan over
// the whole [P][units] array then gives every (part, walker) its offset in a
// send buffer grouped by part, generation order inside each part -- exactly the
// order that makes the receiver's part-local index x = base(shard, part) +
// position (O6).  P <= 32 (one lane per part).
constexpr uint32_t kMaxShardParts = 32;

__global__ void __launch_bounds__(kThreads) count_parts_kernel(const uint32_t* __restrict__ walks,
                                                               const uint32_t* __restrict__ slot_tab,
                                                               PoolParams p, const uint64_t* __restrict__ part_bounds,
                                                               uint32_t P, uint32_t* __restrict__ counts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* sb = reinterpret_cast<uint64_t*>(smem_raw);                        // P + 1 bounds
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(sb + kMaxShardParts + 1);       // [warp][P]
    uint32_t* paths = wcnt + kWarps * kMaxShardParts;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t plen = p.k + 1;
    for (uint32_t i = threadIdx.x; i <= P; i += kThreads) sb[i] = part_bounds[i];
    __syncthreads();
    uint32_t* my = paths + warp * 2 * plen;
    uint32_t* cnt = wcnt + warp * kMaxShardParts;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t buf = 0;
    stage_walk(my, walks, w, p.units, plen, lane);
    for (; w < p.units; w += nwarps) {
        cp_async_wait_all();
        if (lane < P) cnt[lane] = 0;
        __syncwarp();
        const uint32_t* path = my + buf * plen;
        stage_walk(my + (buf ^ 1) * plen, walks, w + nwarps, p.units, plen, lane);
        for (uint32_t s0 = 0; s0 < p.Pw; s0 += 32) {
            const uint32_t s = s0 + lane;
            uint32_t pg = 0xFFFFFFFFu;
            if (s < p.Pw) {
                const uint32_t t = __ldg(slot_tab + s);
                const uint32_t b = path[(t >> 16) + (t & 0xFFFFu)];
                if (b != kSentinel) pg = range_of(sb, P, b);
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, pg);
            if (pg != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1)) cnt[pg] += __popc(peers);
            __syncwarp();
        }
        if (lane < P) counts[(uint64_t)lane * p.units + w] = cnt[lane];
        buf ^= 1;
        __syncwarp();
    }
    cp_async_wait_all();
}

// Pairs of the shard into the part-grouped send buffer: pair (path[i],
// path[i+delta]) of walker w goes to out[base[g * units + w] + its rank among
// the walk's part-g pairs in generation order], g = part of the context node.
__global__ void __launch_bounds__(kThreads) pairs_parts_kernel(const uint32_t* __restrict__ walks,
                                                               const uint32_t* __restrict__ slot_tab,
                                                               PoolParams p, const uint64_t* __restrict__ part_bounds,
                                                               uint32_t P, const uint64_t* __restrict__ base,
                                                               uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* sb = reinterpret_cast<uint64_t*>(smem_raw);                 // P + 1 bounds
    uint64_t* wcur = sb + kMaxShardParts + 1;                             // [warp][P] cursors
    uint32_t* paths = reinterpret_cast<uint32_t*>(wcur + kWarps * kMaxShardParts);
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t plen = p.k + 1;
    for (uint32_t i = threadIdx.x; i <= P; i += kThreads) sb[i] = part_bounds[i];
    __syncthreads();
    uint32_t* my = paths + warp * 2 * plen;
    uint64_t* cur = wcur + warp * kMaxShardParts;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t buf = 0;
    stage_walk(my, walks, w, p.units, plen, lane);
    for (; w < p.units; w += nwarps) {
        cp_async_wait_all();
        if (lane < P) cur[lane] = __ldg(base + (uint64_t)lane * p.units + w);
        __syncwarp();
        const uint32_t* path = my + buf * plen;
        stage_walk(my + (buf ^ 1) * plen, walks, w + nwarps, p.units, plen, lane);
        for (uint32_t s0 = 0; s0 < p.Pw; s0 += 32) {
            const uint32_t s = s0 + lane;
            uint32_t pg = 0xFFFFFFFFu, a = 0, b = 0;
            if (s < p.Pw) {
                const uint32_t t = __ldg(slot_tab + s);
                const uint32_t i = t >> 16;
                b = path[i + (t & 0xFFFFu)];
                a = path[i];
                if (b != kSentinel) pg = range_of(sb, P, b);
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, pg);
            if (pg != 0xFFFFFFFFu) out[cur[pg] + __popc(peers & lt)] = (uint64_t)a | ((uint64_t)b << 32);
            __syncwarp();
            if (pg != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1)) cur[pg] += __popc(peers);
            __syncwarp();
        }
        buf ^= 1;
        __syncwarp();
    }
    cp_async_wait_all();
}

static size_t shard_smem(uint32_t k, size_t cursor_bytes) {
    return (kMaxShardParts + 1) * sizeof(uint64_t) + (size_t)kWarps * kMaxShardParts * cursor_bytes +
           (size_t)kWarps * 2 * (k + 1) * sizeof(uint32_t);
}

cudaError_t launch_count_parts(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                               const uint64_t* part_bounds, uint32_t P, uint32_t* counts, const Device& dev,
                               cudaStream_t s) {
    if (P == 0 || P > kMaxShardParts) return cudaErrorInvalidValue;
    if (p.units == 0) return cudaSuccess;
    count_parts_kernel<<<grid_cap(ceil_div(p.units, kWarps), dev, 8), kThreads, shard_smem(p.k, 4), s>>>(
        walks, slot_tab, p, part_bounds, P, counts);
    return cudaGetLastError();
}

cudaError_t launch_pairs_parts(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                               const uint64_t* part_bounds, uint32_t P, const uint64_t* base, uint64_t* out,
                               const Device& dev, cudaStream_t s) {
    if (P == 0 || P > kMaxShardParts) return cudaErrorInvalidValue;
    if (p.units == 0) return cudaSuccess;
    pairs_parts_kernel<<<grid_cap(ceil_div(p.units, kWarps), dev, 8), kThreads, shard_smem(p.k, 8), s>>>(
        walks, slot_tab, p, part_bounds, P, base, out);
    return cudaGetLastError();
}

// O6 keys of a part's pool gathered in generation order: key[x] = pi_g(x).
__global__ void __launch_bounds__(kThreads) feistel_keys_kernel(Feistel f, uint64_t N, uint32_t* __restrict__ key) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < N; x += stride) key[x] = (uint32_t)f(x);
}

cudaError_t launch_feistel_keys(const PoolParams& p, uint32_t* key, const Device& dev, cudaStream_t s) {
    if (p.N == 0) return cudaSuccess;
    feistel_keys_kernel<<<grid_cap(ceil_div(p.N, kThreads), dev, 8), kThreads, 0, s>>>(make_feistel(p), p.N, key);
    return cudaGetLastError();
}

// tot[g] = pairs of the shard in part g, from the scanned [P][units] counts.
__global__ void part_totals_kernel(const uint64_t* __restrict__ base, uint64_t units, uint32_t P,
                                   const uint64_t* __restrict__ total, uint64_t* __restrict__ tot) {
    const uint32_t g = threadIdx.x;
    if (g >= P) return;
    if (units == 0) { tot[g] = 0; return; }
    const uint64_t e = g + 1 < P ? base[(uint64_t)(g + 1) * units] : *total;
    tot[g] = e - base[(uint64_t)g * units];
}

cudaError_t launch_part_totals(const uint64_t* base, uint64_t units, uint32_t P, const uint64_t* total,
                               uint64_t* tot, cudaStream_t s) {
    if (P == 0 || P > kMaxShardParts) return cudaErrorInvalidValue;
    part_totals_kernel<<<1, 32, 0, s>>>(base, units, P, total, tot);
    return cudaGetLastError();
}

// Direct sink for a pool gathered in generation order: out[pi(x)] = in[x].
__global__ void __launch_bounds__(kThreads) feistel_scatter_kernel(Feistel f, uint64_t N,
                                                                   const uint64_t* __restrict__ in,
                                                                   uint64_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < N; x += stride) out[f(x)] = in[x];
}

cudaError_t launch_feistel_scatter(const PoolParams& p, const uint64_t* in, uint64_t* out, const Device& dev,
                                   cudaStream_t s) {
    if (p.N == 0) return cudaSuccess;
    feistel_scatter_kernel<<<grid_cap(ceil_div(p.N, kThreads), dev, 8), kThreads, 0, s>>>(make_feistel(p), p.N,
                                                                                           in, out);
    return cudaGetLastError();
}

// LINE mode: the pool is the CSR edge list; unit = edge id.
__global__ void __launch_bounds__(kThreads) pairs_line_kernel(const uint64_t* __restrict__ off,
                                                              const uint32_t* __restrict__ tgt,
                                                              uint64_t n, PoolParams p, Feistel f,
                                                              const uint64_t* __restrict__ base,
                                                              PoolSink sink) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < p.units; x += stride) {
        const uint64_t e = p.u0 + x;
        const uint32_t dst = __ldg(tgt + e);
        if (dst < p.c_begin || dst >= p.c_end) continue;
        const uint32_t src = range_of(off, (uint32_t)n, e);
        sink_put(sink, base[x], f(base[x]), (uint64_t)src | ((uint64_t)dst << 32));
    }
}

cudaError_t launch_pairs_line(const uint64_t* off, const uint32_t* tgt, uint64_t n,
                              const PoolParams& p, const uint64_t* base, const PoolSink& sink,
                              const Device& dev, cudaStream_t s) {
    if (p.units == 0 || p.N == 0) return cudaSuccess;
    const Feistel f = make_feistel(p);
    pairs_line_kernel<<<grid_cap(ceil_div(p.units, kThreads), dev, 8), kThreads, 0, s>>>(
        off, tgt, n, p, f, base, sink);
    return cudaGetLastError();
}

// ---- stable partition by vertex sub-part ------------------------------------

__device__ __forceinline__ uint32_t bucket_of(uint64_t v, const uint64_t* sb, uint32_t nb) {
    return v == kHole ? 0xFFFFFFFFu : range_of(sb, nb, (uint32_t)v);
}

// counts[b * ntiles + tile] = number of slots of bucket b in the tile (any
// order inside a tile: also counts the windowed layout, tile = window).
__global__ void __launch_bounds__(kThreads) bucket_count_kernel(const uint64_t* __restrict__ slots,
                                                                uint64_t N,
                                                                const uint64_t* __restrict__ bounds,
                                                                uint32_t nb, uint64_t ntiles, uint32_t tile_sz,
                                                                uint32_t* __restrict__ counts) {
    __shared__ uint64_t sb[kMaxBuckets + 1];
    __shared__ uint32_t hist[kMaxBuckets];
    for (uint32_t i = threadIdx.x; i <= nb; i += kThreads) sb[i] = bounds[i];
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < nb; i += kThreads) hist[i] = 0;
        __syncthreads();
        const uint64_t end = min(N, (tile + 1) * tile_sz);
        for (uint64_t i = tile * tile_sz + threadIdx.x; i < end; i += kThreads) {
            const uint32_t b = bucket_of(slots[i], sb, nb);
            if (b != 0xFFFFFFFFu) atomicAdd(&hist[b], 1u);
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kThreads) counts[(uint64_t)b * ntiles + tile] = hist[b];
        __syncthreads();
    }
}

// Exclusive scan of u32 counts into u64 offsets: per-chunk sums, a single-CTA
// scan of the chunk sums, then per-chunk scans with their base.
__global__ void __launch_bounds__(kThreads) scan_sums_kernel(const uint32_t* __restrict__ in,
                                                             uint64_t M, uint64_t* __restrict__ sums) {
    __shared__ uint64_t red[kWarps];
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk;
    uint64_t acc = 0;
    for (uint64_t i = base + threadIdx.x; i < min(M, base + kScanChunk); i += kThreads) acc += in[i];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane_id() == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void scan_partials_kernel(uint64_t* __restrict__ sums, uint64_t nchunks,
                                     uint64_t* __restrict__ total) {
    // one warp, sequential over chunks in groups of 32 (nchunks is small)
    const uint32_t lane = lane_id();
    uint64_t run = 0;
    for (uint64_t b = 0; b < nchunks; b += 32) {
        const uint64_t i = b + lane;
        const uint64_t v = i < nchunks ? sums[i] : 0;
        uint64_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        if (i < nchunks) sums[i] = run + incl - v;
        run += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    if (lane == 0) *total = run;
}

__global__ void __launch_bounds__(kThreads) scan_chunks_kernel(const uint32_t* __restrict__ in,
                                                               uint64_t M,
                                                               const uint64_t* __restrict__ sums,
                                                               uint64_t* __restrict__ out) {
    // each thread owns 16 consecutive elements of the 4096-element chunk
    __shared__ uint64_t warp_tot[kWarps];
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk + threadIdx.x * 16ull;
    uint32_t v[16];
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        v[j] = base + j < M ? in[base + j] : 0u;
        acc += v[j];
    }
    uint64_t incl = acc;
    const uint32_t lane = lane_id();
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) warp_tot[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint64_t run = sums[blockIdx.x];
    for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) run += warp_tot[w];
    run += incl - acc;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (base + j < M) out[base + j] = run;
        run += v[j];
    }
}

__global__ void block_offsets_kernel(const uint64_t* __restrict__ tile_off, uint64_t ntiles,
                                     uint32_t nb, const uint64_t* __restrict__ total,
                                     uint64_t* __restrict__ block_offsets) {
    for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x)
        block_offsets[b] = b < nb ? tile_off[(uint64_t)b * ntiles] : *total;
}

// Stable scatter: within a tile every warp owns 512 consecutive slots; ranks
// inside a 32-slot chunk come from __match_any_sync, per-warp bases from a
// per-tile prefix over warps, so the pool keeps slot (= pi) order per block.
__global__ void __launch_bounds__(kThreads) bucket_scatter_kernel(const uint64_t* __restrict__ slots,
                                                                  uint64_t N,
                                                                  const uint64_t* __restrict__ bounds,
                                                                  uint32_t nb, uint64_t ntiles,
                                                                  const uint64_t* __restrict__ tile_off,
                                                                  uint64_t* __restrict__ pool) {
    __shared__ uint64_t sb[kMaxBuckets + 1];
    __shared__ uint32_t wcnt[kWarps][kMaxBuckets];
    __shared__ uint64_t wbase[kWarps][kMaxBuckets];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (uint32_t i = threadIdx.x; i <= nb; i += kThreads) sb[i] = bounds[i];
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < kWarps * nb; i += kThreads) wcnt[i / nb][i % nb] = 0;
        __syncthreads();
        const uint64_t wb = tile * kTile + (uint64_t)warp * kPerWarp;
        uint64_t vals[kChunks];
        uint32_t bks[kChunks];
#pragma unroll
        for (uint32_t c = 0; c < kChunks; ++c) {
            const uint64_t i = wb + c * 32 + lane;
            vals[c] = i < N ? slots[i] : kHole;
            bks[c] = bucket_of(vals[c], sb, nb);
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bks[c]);
            if (bks[c] != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1))
                wcnt[warp][bks[c]] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kThreads) {
            uint64_t run = tile_off[(uint64_t)b * ntiles + tile];
            for (int w = 0; w < kWarps; ++w) { wbase[w][b] = run; run += wcnt[w][b]; }
        }
        __syncthreads();
#pragma unroll
        for (uint32_t c = 0; c < kChunks; ++c) {
            const uint32_t b = bks[c];
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
            if (b != 0xFFFFFFFFu) {
                pool[wbase[warp][b] + __popc(peers & lt_mask)] = vals[c];
            }
            __syncwarp();
            if (b != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1)) wbase[warp][b] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
    }
}

// ---- keyed sink -> window layout (radix passes on the pi position) ----------
// One pass partitions the (pair, key) tiles of the input by the key prefix
// y >> s.  The input is already partitioned by y >> s_prev (s_prev = 0: the
// first pass, generation order), and pi is a bijection, so prefix p's region of
// the output is exactly [p << s, (p + 1) << s): no histogram pass is needed, a
// per-prefix cursor hands out room.  A CTA counting-sorts its 4096-item tile by
// prefix in shared memory and writes every prefix's run contiguously (one
// global atomic per run), so all DRAM traffic is coalesced and the number of
// pages written concurrently stays within the TLB's reach.
constexpr int kRadThreads = 512;
constexpr uint32_t kRadTile = 4096;
constexpr uint32_t kRadPer = kRadTile / kRadThreads;
constexpr uint32_t kRadMaxBins = 1024;  // 2 x 2^9: a tile spans <= 2 regions of the previous pass
constexpr size_t kRadSmem = (size_t)kRadTile * 12 + (size_t)kRadMaxBins * 12 + 64 * 4;

__global__ void __launch_bounds__(kRadThreads, 2) radix_pass_kernel(const uint64_t* __restrict__ in_pair,
                                                                    const uint32_t* __restrict__ in_key,
                                                                    uint64_t N, uint32_t s_prev, uint32_t s,
                                                                    uint64_t* __restrict__ out_pair,
                                                                    uint32_t* __restrict__ out_key,
                                                                    uint16_t* __restrict__ out_pos,
                                                                    uint32_t* __restrict__ cursor) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* sp = reinterpret_cast<uint64_t*>(smem_raw);
    uint32_t* sk = reinterpret_cast<uint32_t*>(sp + kRadTile);
    uint32_t* hist = sk + kRadTile;
    uint32_t* lscan = hist + kRadMaxBins;
    uint32_t* gbase = lscan + kRadMaxBins;
    uint32_t* wtot = gbase + kRadMaxBins;  // per-warp scan totals
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint64_t ntiles = ceil_div(N, kRadTile);
    const uint64_t last_prefix = (N - 1) >> s;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tile * kRadTile;
        const uint32_t cnt = N - t0 < kRadTile ? (uint32_t)(N - t0) : kRadTile;
        uint64_t pbase = 0, pend = last_prefix + 1;
        if (s_prev) {
            pbase = (t0 >> s_prev) << (s_prev - s);
            const uint64_t e = (((t0 + cnt - 1) >> s_prev) + 1) << (s_prev - s);
            if (e < pend) pend = e;
        }
        const uint32_t nbins = (uint32_t)(pend - pbase);
        for (uint32_t i = tid; i < nbins; i += kRadThreads) hist[i] = 0;
        __syncthreads();
        uint64_t pr[kRadPer];
        uint32_t ky[kRadPer], rk[kRadPer];
#pragma unroll
        for (uint32_t j = 0; j < kRadPer; ++j) {
            const uint32_t i = j * kRadThreads + tid;
            if (i < cnt) {
                ky[j] = __ldg(in_key + t0 + i);
                pr[j] = __ldg(in_pair + t0 + i);
            }
        }
#pragma unroll
        for (uint32_t j = 0; j < kRadPer; ++j)
            if (j * kRadThreads + tid < cnt) rk[j] = atomicAdd(&hist[(uint32_t)((ky[j] >> s) - pbase)], 1u);
        __syncthreads();
        // exclusive scan of hist[0, nbins) (two bins per thread), then one run per prefix
        const uint32_t b0 = 2 * tid, b1 = 2 * tid + 1;
        const uint32_t h0 = b0 < nbins ? hist[b0] : 0u, h1 = b1 < nbins ? hist[b1] : 0u;
        uint32_t incl = h0 + h1;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        if (lane == 31) wtot[warp] = incl;
        __syncthreads();
        uint32_t run = 0;
        for (uint32_t w = 0; w < warp; ++w) run += wtot[w];
        const uint32_t ex = run + incl - h0 - h1;
        if (b0 < nbins) {
            lscan[b0] = ex;
            if (h0) gbase[b0] = atomicAdd(cursor + pbase + b0, h0);
        }
        if (b1 < nbins) {
            lscan[b1] = ex + h0;
            if (h1) gbase[b1] = atomicAdd(cursor + pbase + b1, h1);
        }
        __syncthreads();
#pragma unroll
        for (uint32_t j = 0; j < kRadPer; ++j)
            if (j * kRadThreads + tid < cnt) {
                const uint32_t l = lscan[(uint32_t)((ky[j] >> s) - pbase)] + rk[j];
                sp[l] = pr[j];
                sk[l] = ky[j];
            }
        __syncthreads();
        for (uint32_t i = tid; i < cnt; i += kRadThreads) {
            const uint32_t k = sk[i];
            const uint32_t d = (uint32_t)((k >> s) - pbase);
            const uint64_t g = ((pbase + d) << s) + gbase[d] + (i - lscan[d]);
            out_pair[g] = sp[i];
            if (out_pos) out_pos[g] = (uint16_t)(k & ((1u << s) - 1u));
            else out_key[g] = k;
        }
        __syncthreads();
    }
}

cudaError_t launch_order(uint64_t N, uint64_t* pairs0, uint32_t* keys0, uint64_t* pairs1, uint32_t* keys1,
                         uint32_t* cursors, const uint64_t** win_pairs, const uint16_t** win_pos, uint64_t** spare,
                         const Device& dev, cudaStream_t st, uint32_t* launches) {
    if (N == 0 || N > (1ull << 32)) return cudaErrorInvalidValue;
    uint32_t bits = 0;
    while ((1ull << bits) < N) ++bits;
    const uint32_t total = bits > kPoolWinBits ? bits - kPoolWinBits : 0;  // key bits above the window
    // <= 9 bits per pass (2^10 bins per tile); NE_RADIX_MAXBITS (developer / test knob, 1..9)
    // lowers the cap so small pools exercise the multi-pass path
    const char* mb_env = std::getenv("NE_RADIX_MAXBITS");
    const uint32_t mb = mb_env ? std::min(9u, std::max(1u, (uint32_t)std::atoi(mb_env))) : 9u;
    const uint32_t passes = std::max<uint32_t>(1, (total + mb - 1) / mb);
    const uint32_t step = (total + passes - 1) / passes;
    cudaError_t e = cudaFuncSetAttribute(radix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kRadSmem);
    if (e != cudaSuccess) return e;
    uint64_t* ip = pairs0;
    uint32_t* ik = keys0;
    uint64_t* op = pairs1;
    uint32_t* ok = keys1;
    uint32_t s_prev = 0;
    const unsigned grid = grid_cap(ceil_div(N, kRadTile), dev, 2);
    for (uint32_t i = 0; i < passes; ++i) {
        const bool last = i + 1 == passes;
        const uint32_t sh = last ? kPoolWinBits : std::max(kPoolWinBits, kPoolWinBits + total - (i + 1) * step);
        e = cudaMemsetAsync(cursors, 0, (((N - 1) >> sh) + 1) * sizeof(uint32_t), st);
        if (e != cudaSuccess) return e;
        radix_pass_kernel<<<grid, kRadThreads, kRadSmem, st>>>(ip, ik, N, s_prev, sh, op, last ? nullptr : ok,
                                                               last ? reinterpret_cast<uint16_t*>(ok) : nullptr,
                                                               cursors);
        if (launches) *launches += 1;
        std::swap(ip, op);
        std::swap(ik, ok);
        s_prev = sh;
    }
    *win_pairs = ip;
    *win_pos = reinterpret_cast<const uint16_t*>(ik);
    *spare = op;
    return cudaGetLastError();
}

// Windowed layout: one CTA per 8192-position window.  Its pairs (in arrival
// order) are placed by pos = y mod 8192 into shared memory -- the window is
// dense, pi being a bijection -- after which the stable scatter above runs on
// the shared copy: every warp owns 512 consecutive positions, ranks from
// __match_any_sync, per-warp bases from the per-window prefix.
constexpr int kWinThreads = 512;
constexpr int kWinWarps = kWinThreads / 32;
constexpr uint32_t kWinSpan = kWin / kWinWarps;

size_t window_scatter_smem(uint32_t nb) {
    return (size_t)kWin * 8 + (size_t)(nb + 1) * 8 + (size_t)kWinWarps * nb * 12;
}

__global__ void __launch_bounds__(kWinThreads, 2) window_scatter_kernel(const uint64_t* __restrict__ binned,
                                                                        const uint16_t* __restrict__ pos,
                                                                        uint64_t N,
                                                                        const uint64_t* __restrict__ bounds,
                                                                        uint32_t nb, uint64_t nwin,
                                                                        const uint64_t* __restrict__ tile_off,
                                                                        uint64_t* __restrict__ pool) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* sp = reinterpret_cast<uint64_t*>(smem_raw);  // the window in pi order
    uint64_t* sb = sp + kWin;                                // nb + 1 sub-part bounds
    uint64_t* wbase = sb + nb + 1;                           // [warp][bucket]
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(wbase + (size_t)kWinWarps * nb);
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (uint32_t i = threadIdx.x; i <= nb; i += kWinThreads) sb[i] = bounds[i];
    for (uint64_t win = blockIdx.x; win < nwin; win += gridDim.x) {
        const uint64_t w0 = win << kPoolWinBits;
        const uint32_t cnt = N - w0 < kWin ? (uint32_t)(N - w0) : kWin;
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < cnt; i += kWinThreads) sp[__ldg(pos + w0 + i)] = __ldg(binned + w0 + i);
        for (uint32_t i = threadIdx.x; i < kWinWarps * nb; i += kWinThreads) wcnt[i] = 0;
        __syncthreads();
        const uint32_t j_begin = warp * kWinSpan, j_end = min(cnt, j_begin + kWinSpan);
        for (uint32_t j0 = j_begin; j0 < j_end; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t b = j < j_end ? range_of(sb, nb, (uint32_t)sp[j]) : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
            if (b != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1)) wcnt[warp * nb + b] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kWinThreads) {
            uint64_t run = tile_off[(uint64_t)b * nwin + win];
            for (int w = 0; w < kWinWarps; ++w) {
                wbase[w * nb + b] = run;
                run += wcnt[w * nb + b];
            }
        }
        __syncthreads();
        for (uint32_t j0 = j_begin; j0 < j_end; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint64_t v = j < j_end ? sp[j] : 0;
            const uint32_t b = j < j_end ? range_of(sb, nb, (uint32_t)v) : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
            if (b != 0xFFFFFFFFu) pool[wbase[warp * nb + b] + __popc(peers & lt_mask)] = v;
            __syncwarp();
            if (b != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1)) wbase[warp * nb + b] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
    }
}

// S:230 schedule check: every sample at position i of the pool lies in its 2D
// block -- src in the block's vertex sub-part, dst in this rank's context part.
// bad[0] = first offending position (or ~0).
__global__ void check_pool_kernel(const uint64_t* __restrict__ pool, const uint64_t* __restrict__ boff,
                                  const uint64_t* __restrict__ sub_bounds, uint32_t nb, uint64_t c_begin,
                                  uint64_t c_end, unsigned long long* bad) {
    const uint64_t total = boff[nb];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const uint32_t b = range_of(boff, nb, i);
        const uint32_t src = (uint32_t)pool[i], dst = (uint32_t)(pool[i] >> 32);
        if (src < sub_bounds[b] || src >= sub_bounds[b + 1] || dst < c_begin || dst >= c_end)
            atomicMin(bad, (unsigned long long)i);
    }
}

cudaError_t launch_check_pool(const uint64_t* pool, const uint64_t* boff, uint64_t total,
                              const uint64_t* sub_bounds, uint32_t nb, uint64_t c_begin, uint64_t c_end,
                              unsigned long long* bad, const Device& dev, cudaStream_t s) {
    if (total == 0) return cudaSuccess;
    check_pool_kernel<<<grid_cap(ceil_div(total, kThreads), dev, 8), kThreads, 0, s>>>(
        pool, boff, sub_bounds, nb, c_begin, c_end, bad);
    return cudaGetLastError();
}

size_t scan_scratch_bytes(uint64_t M) {
    const uint64_t nchunks = std::max<uint64_t>(1, ceil_div(M, kScanChunk));
    return (nchunks + 2) * sizeof(uint64_t) + 64;
}

cudaError_t launch_scan(const uint32_t* in, uint64_t M, uint64_t* out, uint64_t* total, void* scratch,
                        cudaStream_t s, uint32_t* launches) {
    const uint64_t nchunks = std::max<uint64_t>(1, ceil_div(M, kScanChunk));
    uint64_t* sums = reinterpret_cast<uint64_t*>(scratch);
    scan_sums_kernel<<<(unsigned)nchunks, kThreads, 0, s>>>(in, M, sums);
    scan_partials_kernel<<<1, 32, 0, s>>>(sums, nchunks, total);
    scan_chunks_kernel<<<(unsigned)nchunks, kThreads, 0, s>>>(in, M, sums, out);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

size_t bucket_scratch_bytes(uint64_t N, uint32_t nb) {
    const uint64_t ntiles = std::max<uint64_t>(1, ceil_div(N, kTile));
    const uint64_t M = ntiles * nb;
    const uint64_t nchunks = std::max<uint64_t>(1, ceil_div(M, kScanChunk));
    return M * sizeof(uint32_t) + M * sizeof(uint64_t) + (nchunks + 2) * sizeof(uint64_t) + 256;
}

cudaError_t launch_bucket(const uint64_t* slots, const uint16_t* pos, uint64_t N, const uint64_t* sub_bounds,
                          uint32_t nb, void* scratch, uint64_t* pool, uint64_t* block_offsets,
                          const Device& dev, cudaStream_t s, uint32_t* launches) {
    if (nb == 0 || nb > kMaxBuckets) return cudaErrorInvalidValue;
    const uint32_t tile_sz = pos ? kWin : kTile;
    const uint64_t ntiles = std::max<uint64_t>(1, ceil_div(N, tile_sz));
    const uint64_t M = ntiles * nb;
    const uint64_t nchunks = std::max<uint64_t>(1, ceil_div(M, kScanChunk));
    uint32_t* counts = reinterpret_cast<uint32_t*>(scratch);
    uint64_t* tile_off = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(counts + M) + 15) & ~(uintptr_t)15);
    uint64_t* sums = tile_off + M;
    uint64_t* total = sums + nchunks;
    const unsigned g = grid_cap(ntiles, dev, 8);
    bucket_count_kernel<<<g, kThreads, 0, s>>>(slots, N, sub_bounds, nb, ntiles, tile_sz, counts);
    scan_sums_kernel<<<(unsigned)nchunks, kThreads, 0, s>>>(counts, M, sums);
    scan_partials_kernel<<<1, 32, 0, s>>>(sums, nchunks, total);
    scan_chunks_kernel<<<(unsigned)nchunks, kThreads, 0, s>>>(counts, M, sums, tile_off);
    block_offsets_kernel<<<1, 256, 0, s>>>(tile_off, ntiles, nb, total, block_offsets);
    if (pos) {
        const size_t smem = window_scatter_smem(nb);
        cudaError_t e = cudaFuncSetAttribute(window_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        if (N) window_scatter_kernel<<<grid_cap(ntiles, dev, 2), kWinThreads, smem, s>>>(
            slots, pos, N, sub_bounds, nb, ntiles, tile_off, pool);
    } else {
        bucket_scatter_kernel<<<g, kThreads, 0, s>>>(slots, N, sub_bounds, nb, ntiles, tile_off, pool);
    }
    if (launches) *launches += (pos && !N) ? 5 : 6;
    return cudaGetLastError();
}

}  // namespace ne

// runtime.cpp -- the C ABI (include/ne.h): context, device memory, the
// episode pipeline and the NCCL ring of vertex sub-parts.
//
// Per-rank HBM layout (rank g of P, k sub-parts; contiguous ranges, D12):
//   CSR           offsets u64[n+1], targets u32[nnz]           (replicated)
//   alias         uint2[c_count] (thr, alias) of context part g (O3)
//   context       fp32[c_count][d], part g, resident for the whole run
//   vertex slots  2k buffers of fp32[max sub-part rows][d]: the k sub-parts
//                 being trained this round and the k arriving (ping-pong)
//   walks         u32[walkers][k+1]        (one episode)
//   slots         u64[N]   pi-indexed pairs (one episode, ~0 = hole)
//   pool          u64[N]   (src, dst) grouped by vertex sub-part, pi order
#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "ne.h"
#include "ne_internal.h"
#include "ne_ctx.h"

int ne_fail(ne_ctx* c, int code, const char* fmt, ...) {
    static const char* names[] = {"NE_OK", "NE_EINVAL", "NE_ERANGE", "NE_ENOMEM", "NE_ESTATE",
                                  "NE_ECUDA", "NE_ENCCL", "NE_ESCHED"};
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = std::string(names[-code]) + ": " + buf;
    return code;
}


namespace {

// Host wait for a stream that may hold NCCL work (ring, pool exchange): poll it
// and the communicators' asynchronous errors, so a failed or vanished peer
// returns NE_ENCCL (communicators aborted) instead of hanging; a stall longer
// than NE_NCCL_TIMEOUT_S (default 900 s) is treated the same way.
int wait_stream(ne_ctx* c, cudaStream_t s) {
    if (!(c->world > 1 && c->comm)) {
        NE_CUDA(c, cudaStreamSynchronize(s));
        return NE_OK;
    }
    static const double limit_s = [] {
        const char* e = std::getenv("NE_NCCL_TIMEOUT_S");
        return e ? std::atof(e) : 900.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return NE_OK;
        if (q != cudaErrorNotReady) NE_CUDA(c, q);
        for (ncclComm_t comm : {c->comm, c->comm_walk}) {
            ncclResult_t async = ncclSuccess;
            if (comm && ncclCommGetAsyncError(comm, &async) == ncclSuccess && async != ncclSuccess) {
                ncclCommAbort(c->comm_walk);
                ncclCommAbort(c->comm);
                c->comm_walk = c->comm = nullptr;
                return ne_fail(c, NE_ENCCL, "NCCL asynchronous error on rank %d: %s (communicators aborted)", c->rank,
                               ncclGetErrorString(async));
            }
        }
        const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (waited > limit_s) {
            ncclCommAbort(c->comm_walk);
            ncclCommAbort(c->comm);
            c->comm_walk = c->comm = nullptr;
            return ne_fail(c, NE_ENCCL, "rank %d: ring / exchange stalled for %.0f s (a peer is gone?); communicators "
                                        "aborted", c->rank, waited);
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

thread_local std::string g_create_error;  // ne_last_error(NULL) after a failed ne_create


void partition(uint64_t begin, uint64_t end, uint32_t parts, uint64_t* out) {
    const uint64_t len = end - begin, q = len / parts, r = len % parts;
    for (uint64_t i = 0; i <= parts; ++i) out[i] = begin + i * q + std::min<uint64_t>(i, r);
}

// O7 plan with NEXT-3 groups: P = G * L ranks, rank
// g = a * L + j; at global round rho = R * L + r rank g trains vertex sub-part
// (((a - R) mod G) * L + ((j - r) mod L)) * k + t.  G = 1: the single ring,
// (g - r) mod P.  After round rho a sub-part moves to ring_dest: along the
// group's ring, (a, j + 1), except after the group's last rotation, when it
// crosses to the next group, (a + 1, j + 1); rho = P - 1 brings it home.
int plan_vsub(uint32_t P, uint32_t G, uint32_t k, uint32_t rho, uint32_t t, uint32_t g) {
    const uint32_t L = P / G, a = g / L, j = g % L, R = (rho / L) % G, r = rho % L;
    return (int)((((a + G - R) % G) * L + (j + L - r) % L) * k + t);
}

uint32_t groups_of(const ne_ctx* c) { return c->cfg.groups > 1 ? c->cfg.groups : 1; }

// NEXT-2 staged ring: vertex sub-parts per ring window (w <= k).
uint32_t stage_window(const ne_ctx* c) {
    const uint32_t w = c->cfg.stage_window ? c->cfg.stage_window : 2;
    return std::min(w, c->cfg.subparts);
}

int dalloc(ne_ctx* c, void** out, size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    void* p = nullptr;
    if (c->alloc) {
        p = c->alloc(bytes, c->device, (void*)c->stream, c->user);
        if (!p) return ne_fail(c, NE_ENOMEM, "allocator callback returned NULL for %zu bytes", bytes);
    } else {
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ne_fail(c, NE_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        }
    }
    c->allocs.push_back({p, bytes});
    *out = p;
    return NE_OK;
}

template <typename T>
int dalloc_t(ne_ctx* c, T** out, size_t count) {
    void* p = nullptr;
    NE_TRY(dalloc(c, &p, count * sizeof(T)));
    *out = static_cast<T*>(p);
    return NE_OK;
}

// Bytes per stored embedding element (NE_STORE_F32: 4, NE_STORE_BF16: 2).
uint64_t elem_bytes(const ne_ctx* c) { return c->cfg.storage == NE_STORE_BF16 ? 2 : 4; }

// Host-staged vertex matrix: address of this rank's row `row` (global id).
void* host_row(const ne_ctx* c, uint64_t row) {
    return reinterpret_cast<char*>(c->h_V) + (row - c->part_bounds[c->rank]) * c->cfg.dim * elem_bytes(c);
}

void dfree(ne_ctx* c, void* p) {
    for (size_t i = 0; i < c->allocs.size(); ++i)
        if (c->allocs[i].p == p) {
            if (c->free_fn) c->free_fn(p, c->allocs[i].bytes, c->device, (void*)c->stream, c->user);
            else cudaFree(p);
            c->allocs.erase(c->allocs.begin() + (long)i);
            return;
        }
}

void free_all(ne_ctx* c) {
    if (c->alias_thread.joinable()) c->alias_thread.join();
    c->alias_pending = false;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    if (c->d2h_stream) cudaStreamSynchronize(c->d2h_stream);
    if (c->build_stream) cudaStreamSynchronize(c->build_stream);
    c->stage_pending = c->stage_pre = false;
    for (auto& a : c->allocs) {
        if (c->free_fn) c->free_fn(a.p, a.bytes, c->device, (void*)c->stream, c->user);
        else cudaFree(a.p);
    }
    c->allocs.clear();
    c->d_tmp_u32 = nullptr;
    c->tmp_u32_cap = 0;
    c->d_tmp_f32 = nullptr;
    c->tmp_f32_cap = 0;
    c->d_keys[0] = c->d_keys[1] = nullptr;
    c->pbufs.clear();
    c->d_slots = c->d_pool = c->pool_at = nullptr;
    c->pool_cap = 0;
    c->next = ne_ctx::NextPool{};
    c->keep_pool = nullptr;
    c->loaded = false;
    c->walked_epoch = c->walked_episode = c->built_epoch = c->built_episode = -1;
}

// Join the host alias build started by ne_load_graph and upload its table
// (once).  Everything that reads the alias table calls this first.
int wait_alias(ne_ctx* c);

cudaEvent_t next_event(ne_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

// O3 on the host (an implementation independent of oracle/): weights
// q_i = round(deg_i^0.75 * 2^20), integer Vose (1991) with stack worklists
// over masses m_i = q_i * n_j against column capacity W = sum q.  The weights
// are computed by all host threads; masses use 64-bit arithmetic whenever
// max(q) * n fits (always for the BASELINE graphs), 128-bit otherwise.
struct AliasScratch {
    std::vector<uint64_t> q, m64, num;
    std::vector<unsigned __int128> m128;
    std::vector<uint32_t> small, large, alias;
};

template <typename M>
static void vose(const std::vector<uint64_t>& q, std::vector<M>& m, unsigned __int128 W,
                 AliasScratch& a) {
    const size_t n = q.size();
    size_t ns = 0, nl = 0;
    for (size_t i = 0; i < n; ++i) {
        m[i] = (M)q[i] * (M)n;
        if ((unsigned __int128)m[i] < W) a.small[ns++] = (uint32_t)i;
        else a.large[nl++] = (uint32_t)i;
    }
    const M w = (M)W;
    while (ns && nl) {
        const uint32_t sm = a.small[--ns], g = a.large[--nl];
        a.num[sm] = (uint64_t)m[sm];
        a.alias[sm] = g;
        m[g] -= w - m[sm];
        if (m[g] < w) a.small[ns++] = g;
        else a.large[nl++] = g;
    }
    while (ns) { const uint32_t x = a.small[--ns]; a.num[x] = (uint64_t)W; a.alias[x] = x; }
    while (nl) { const uint32_t x = a.large[--nl]; a.num[x] = (uint64_t)W; a.alias[x] = x; }
}

void build_alias(const uint64_t* deg, size_t n, std::vector<uint2>& out, AliasScratch& a) {
    out.resize(n);
    if (n == 0) return;
    a.q.resize(n);
    const unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
    std::vector<std::thread> th;
    std::vector<uint64_t> part_sum(nt, 0), part_max(nt, 0);
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            const size_t b = n * t / nt, e = n * (t + 1) / nt;
            uint64_t sum = 0, mx = 0;
            for (size_t i = b; i < e; ++i) {
                uint64_t qi = 0;
                if (deg[i]) {
                    const double d = (double)deg[i];
                    double d3 = d * d;
                    d3 = d3 * d;
                    qi = (uint64_t)std::floor(std::sqrt(std::sqrt(d3)) * 1048576.0 + 0.5);
                }
                a.q[i] = qi;
                sum += qi;
                mx = std::max(mx, qi);
            }
            part_sum[t] = sum;
            part_max[t] = mx;
        });
    for (auto& x : th) x.join();
    unsigned __int128 W = 0;
    uint64_t qmax = 0;
    for (unsigned t = 0; t < nt; ++t) { W += part_sum[t]; qmax = std::max(qmax, part_max[t]); }
    if (W == 0) {  // all weights zero: uniform
        std::fill(a.q.begin(), a.q.end(), 1);
        W = n;
        qmax = 1;
    }
    a.num.resize(n);
    a.alias.resize(n);
    a.small.resize(n);
    a.large.resize(n);
    if ((unsigned __int128)qmax * n < ((unsigned __int128)1 << 64) && (W >> 64) == 0) {
        a.m64.resize(n);
        vose(a.q, a.m64, W, a);
    } else {
        a.m128.resize(n);
        vose(a.q, a.m128, W, a);
    }
    // thr = min(2^32-1, floor(num * 2^32 / W)), exact: a double-precision
    // estimate (error < 1 since the quotient has <= 33 bits) corrected with
    // 128-bit products -- no integer division; all host threads.
    const double inv = 4294967296.0 / (double)W;
    th.clear();
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            const size_t b = n * t / nt, e = n * (t + 1) / nt;
            for (size_t i = b; i < e; ++i) {
                const unsigned __int128 x = (unsigned __int128)a.num[i] << 32;
                uint64_t est = (uint64_t)((double)a.num[i] * inv);
                unsigned __int128 prod = (unsigned __int128)est * W;
                while (prod > x) { --est; prod -= W; }
                while (prod + W <= x) { ++est; prod += W; }
                out[i] = make_uint2(est > 0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)est, a.alias[i]);
            }
        });
    for (auto& x : th) x.join();
}

int wait_alias(ne_ctx* c) {
    if (!c->alias_pending) return NE_OK;
    if (c->alias_thread.joinable()) c->alias_thread.join();
    c->alias_pending = false;
    NE_CUDA(c, cudaMemcpyAsync(c->d_alias, c->alias_host.data(), c->alias_host.size() * sizeof(uint2),
                               cudaMemcpyHostToDevice, c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));  // alias_host is reused by the next load
    return NE_OK;
}

uint64_t pairs_per_walk(uint32_t k, uint32_t l) {
    uint64_t c = 0;
    for (uint32_t i = 0; i < k; ++i) c += std::min<uint32_t>(l, k - i);
    return c;
}

void episode_range(const ne_ctx* c, uint32_t episode, uint64_t* u0, uint64_t* units) {
    const unsigned __int128 U = c->units_total, E = c->cfg.episodes;
    const uint64_t b = (uint64_t)((episode * U) / E), e = (uint64_t)(((episode + 1) * U) / E);
    *u0 = b;
    *units = e - b;
}

int enter(ne_ctx* c) {
    if (!c) return NE_EINVAL;
    c->err.clear();
    NE_CUDA(c, cudaSetDevice(c->device));
    return NE_OK;
}

int check_loaded(ne_ctx* c) {
    if (!c->loaded) return ne_fail(c, NE_ESTATE, "no graph loaded (call ne_load_graph first)");
    return NE_OK;
}

uint32_t nb_local(const ne_ctx* c) { return (uint32_t)c->world * c->cfg.subparts; }

// Walker shard s of an episode of `units` walkers at world P: local walkers
// [s * chunk, min(units, (s + 1) * chunk)), chunk = ceil(units / P).
void shard_range(uint64_t units, uint32_t P, uint32_t s, uint64_t* b, uint64_t* cnt) {
    const uint64_t chunk = (units + P - 1) / P;
    *b = std::min<uint64_t>(units, (uint64_t)s * chunk);
    *cnt = std::min<uint64_t>(units, *b + chunk) - *b;
}

int do_walk(ne_ctx* c, uint32_t epoch, uint32_t episode) {
    NvtxRange range("ne walk");
    uint64_t u0, units;
    episode_range(c, episode, &u0, &units);
    if (c->world > 1 && c->comm) {
        // Walkers sharded over the ranks: this rank walks only its shard (rows
        // from 0); the pool build sends every pair to its context part's owner.
        uint64_t mb, mine;
        shard_range(units, (uint32_t)c->world, (uint32_t)c->rank, &mb, &mine);
        NE_CUDA(c, ne::launch_walk(c->d_off, c->d_tgt, c->n, u0 + mb, mine, c->cfg.walk_len,
                                   c->cfg.seed, epoch, c->n2v ? c->n2v_thr : nullptr,
                                   c->d_walks, ne::WalkCount{}, c->dev, c->ws));
        if (mine) c->launches += 1;
        c->walk_counts = false;
        c->shard_units = mine;
    } else {
        // one GPU: the walk kernel also counts every walker's pairs (O5); a
        // layout-only rank of P > 1 walks the whole episode and emulates the shards
        const bool one = c->world == 1;
        NE_CUDA(c, ne::launch_walk(c->d_off, c->d_tgt, c->n, u0, units, c->cfg.walk_len,
                                   c->cfg.seed, epoch, c->n2v ? c->n2v_thr : nullptr, c->d_walks,
                                   one ? ne::WalkCount{c->d_counts, c->cfg.window, c->c_begin, c->c_begin + c->c_count}
                                       : ne::WalkCount{},
                                   c->dev, c->ws));
        if (units) c->launches += 1;
        c->walk_counts = one;
        c->shard_units = units;
    }
    c->walked_epoch = epoch;
    c->walked_episode = episode;
    c->walked_units = c->shard_units;
    c->built_epoch = c->built_episode = -1;
    return NE_OK;
}

// Episode pool buffers, sized by the episode's actual pool N (grow-only, 1/8
// headroom; the bound N_max -- every walk full length, every pair kept -- is
// 3-4x the real pool on power-law graphs).  The key buffers of the keyed path
// are optional: if they do not fit, the direct path builds the same pool.
int ensure_pool(ne_ctx* c, uint64_t N) {
    if (N <= c->pool_cap && !c->pbufs.empty()) return NE_OK;
    // growing: a pool still being trained may live in these buffers -- wait for it
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    for (void* p : c->pbufs) dfree(c, p);
    for (void* p : {(void*)c->d_keys[0], (void*)c->d_keys[1]})
        if (p) dfree(c, p);
    c->pbufs.clear();
    c->d_slots = c->d_pool = c->pool_at = nullptr;
    c->d_keys[0] = c->d_keys[1] = nullptr;
    c->pool_cap = 0;
    c->pool_gen += 1;
    c->built_epoch = c->built_episode = -1;
    c->next.valid = false;
    const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(std::max<uint64_t>(c->N_max, 1), N + N / 8));
    uint64_t *b0 = nullptr, *b1 = nullptr;
    NE_TRY(dalloc_t(c, &b0, cap));
    NE_TRY(dalloc_t(c, &b1, cap));
    c->pbufs = {b0, b1};
    c->d_slots = b0;
    c->d_pool = b1;
    c->pool_cap = cap;
    size_t free_b = 0, total_b = 0;
    auto fits = [&](size_t bytes) {  // keep 1 GiB for the caller
        return c->alloc || (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b >= bytes + (1ull << 30));
    };
    const std::string saved = c->err;
    const char* e = std::getenv("NE_POOL_DIRECT");  // 1: force the direct path (tests, A/B)
    if (!(e && std::atoi(e) != 0) && fits(2 * cap * sizeof(uint32_t))) {
        uint32_t *k0 = nullptr, *k1 = nullptr;
        if (dalloc_t(c, &k0, cap) == NE_OK && dalloc_t(c, &k1, cap) == NE_OK) {
            c->d_keys[0] = k0;
            c->d_keys[1] = k1;
        } else {
            if (k0) dfree(c, k0);
            c->err = saved;  // not an error: the direct path
        }
    }
    // a third pair buffer lets the next episode's pool be built while this one
    // trains (ne_train_epoch); without it the build is serial (NE_PIPELINE=0 forces that)
    const char* pe = std::getenv("NE_PIPELINE");
    if (!(pe && std::atoi(pe) == 0) && fits(cap * sizeof(uint64_t))) {
        uint64_t* b2 = nullptr;
        if (dalloc_t(c, &b2, cap) == NE_OK) c->pbufs.push_back(b2);
        else c->err = saved;
    }
    return NE_OK;
}

// The two pair buffers a build may use: every pbuf except `keep` (the pool
// being trained while the next one is built).
void select_scratch(ne_ctx* c, const uint64_t* keep) {
    uint64_t* pick[2] = {nullptr, nullptr};
    int k = 0;
    for (uint64_t* b : c->pbufs)
        if (b != keep && k < 2) pick[k++] = b;
    c->d_slots = pick[0];
    c->d_pool = pick[1];
}

// O6 order + 2D bucketing of the N pairs of this rank's part: the keyed path
// takes (pairs, keys) in generation order in (d_slots, d_keys[0]); the direct
// path the dense pi-indexed array in d_slots.  Leaves the pool in pool_at and
// the block offsets in boff / d_boff.
int finish_pool(ne_ctx* c, uint64_t N, bool keyed) {
    c->pool_at = c->d_pool;
    if (keyed) {  // radix passes to the window layout (cursors: head of the bucketing scratch)
        const uint64_t* win_pairs = nullptr;
        const uint16_t* win_pos = nullptr;
        uint64_t* spare = nullptr;
        NE_CUDA(c, ne::launch_order(N, c->d_slots, c->d_keys[0], c->d_pool, c->d_keys[1],
                                    static_cast<uint32_t*>(c->d_scratch), &win_pairs, &win_pos, &spare, c->dev,
                                    c->ws, &c->launches));
        c->pool_at = spare;
        NE_CUDA(c, ne::launch_bucket(win_pairs, win_pos, N, c->d_sub_bounds, nb_local(c), c->d_scratch,
                                     c->pool_at, c->d_boff, c->dev, c->ws, &c->launches));
    } else {
        NE_CUDA(c, ne::launch_bucket(c->d_slots, nullptr, N, c->d_sub_bounds, nb_local(c), c->d_scratch,
                                     c->pool_at, c->d_boff, c->dev, c->ws, &c->launches));
    }
    c->boff.assign(nb_local(c) + 1, 0);
    NE_CUDA(c, cudaMemcpyAsync(c->boff.data(), c->d_boff, c->boff.size() * sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, c->ws));
    NE_TRY(wait_stream(c, c->ws));
    return NE_OK;
}

ne::PoolParams pool_params(const ne_ctx* c, uint32_t epoch, uint32_t episode, uint64_t u0, uint64_t units) {
    ne::PoolParams p{};
    p.units = units;
    p.u0 = u0;
    p.k = c->cfg.walk_len;
    p.l = c->cfg.window;
    p.Pw = c->Pw;
    p.episode = episode;
    p.epoch = epoch;
    p.seed = c->cfg.seed;
    p.c_begin = c->c_begin;
    p.c_end = c->c_begin + c->c_count;
    return p;
}

// Sharded construction (walks, P > 1; "generate and send edge samples to
// all node's memory"): every rank counts and generates the pairs of its
// own walker shard only, grouped by context part; the P x P (shard, part)
// count matrix is all-gathered; each rank receives its part's pairs from every
// shard straight into generation order (shard s lands at base(s, g) = the
// pairs of part g in shards < s), so the part-local index x of O6 is the
// position -- the same pool as the unsharded construction, O(N/P) per rank.
// A layout-only rank (no NCCL) runs the same kernels for every shard and copies
// its part's segment in place of the receive.
// Developer knob NE_BUILD_TIMING=1: per-stage times of every pool build on
// stderr (events on the build's stream; read after finish_pool's sync).
struct BuildTimer {
    ne_ctx* c;
    bool on;
    std::vector<std::pair<const char*, cudaEvent_t>> marks;
    explicit BuildTimer(ne_ctx* cc) : c(cc) {
        static const bool timing = [] { const char* e = std::getenv("NE_BUILD_TIMING"); return e && std::atoi(e); }();
        on = timing;
        mark("start");
    }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e = next_event(c);
        cudaEventRecord(e, c->ws);
        marks.push_back({name, e});
    }
    void report(uint32_t episode, uint64_t N) {
        if (!on || marks.size() < 2) return;
        cudaEventSynchronize(marks.back().second);
        std::string line;
        for (size_t m = 1; m < marks.size(); ++m) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[m - 1].second, marks[m].second);
            char buf[96];
            std::snprintf(buf, sizeof buf, " %s=%.2f", marks[m].first, ms);
            line += buf;
        }
        std::fprintf(stderr, "[ne build rank %d ep %u N=%llu]%s\n", c->rank, episode, (unsigned long long)N,
                     line.c_str());
    }
};

int do_build_sharded(ne_ctx* c, uint32_t epoch, uint32_t episode) {
    const uint32_t P = (uint32_t)c->world, me = (uint32_t)c->rank;
    uint64_t u0, units;
    episode_range(c, episode, &u0, &units);
    const uint64_t row = c->cfg.walk_len + 1;
    const bool real = c->comm != nullptr;
    c->tmat.assign((size_t)P * P, 0);
    BuildTimer bt(c);
    // this rank's shard (real) or shard s (emulation): counts -> scan -> part totals
    auto count_shard = [&](uint32_t s, const uint32_t* walks, uint64_t su, uint64_t* tot_dev) -> int {
        ne::PoolParams pp = pool_params(c, epoch, episode, u0, su);
        if (su) {
            NE_CUDA(c, ne::launch_count_parts(walks, c->d_slot_tab, pp, c->d_part_bounds, P, c->d_counts, c->dev,
                                              c->ws));
            NE_CUDA(c, ne::launch_scan(c->d_counts, (uint64_t)P * su, c->d_base, c->d_total, c->d_scan_scratch,
                                       c->ws, &c->launches));
            c->launches += 1;
        }
        NE_CUDA(c, ne::launch_part_totals(c->d_base, su, P, c->d_total, tot_dev, c->ws));
        c->launches += 1;
        (void)s;
        return NE_OK;
    };
    auto shard_walks = [&](uint32_t s, uint64_t* su) -> const uint32_t* {
        uint64_t b;
        shard_range(units, P, s, &b, su);
        return real ? c->d_walks : c->d_walks + b * row;
    };
    if (real) {
        uint64_t su = c->shard_units;
        NE_TRY(count_shard(me, c->d_walks, su, c->d_tmat + (uint64_t)me * P));
        NE_NCCL(c, ncclAllGather(c->d_tmat + (uint64_t)me * P, c->d_tmat, P, ncclUint64, c->comm_walk, c->ws));
    } else {
        for (uint32_t s = 0; s < P; ++s) {
            uint64_t su;
            const uint32_t* w = shard_walks(s, &su);
            NE_TRY(count_shard(s, w, su, c->d_tmat + (uint64_t)s * P));
        }
    }
    bt.mark("count+scan+allgather");
    NE_CUDA(c, cudaMemcpyAsync(c->tmat.data(), c->d_tmat, c->tmat.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                               c->ws));
    NE_TRY(wait_stream(c, c->ws));
    auto M = [&](uint32_t s, uint32_t g) { return c->tmat[(size_t)s * P + g]; };
    uint64_t N = 0, send_max = 0;
    std::vector<uint64_t> recv_off(P + 1, 0);
    for (uint32_t s = 0; s < P; ++s) {
        recv_off[s] = N;
        N += M(s, me);
        uint64_t S = 0;
        for (uint32_t g = 0; g < P; ++g) S += M(s, g);
        send_max = std::max(send_max, S);
    }
    recv_off[P] = N;
    if (N > c->N_max) return ne_fail(c, NE_ERANGE, "episode pool %llu > bound %llu (internal)", (unsigned long long)N,
                                  (unsigned long long)c->N_max);
    NE_TRY(ensure_pool(c, std::max(N, send_max)));
    select_scratch(c, c->keep_pool);
    // pairs of a shard into the part-grouped send buffer (d_pool), then the
    // exchange into d_slots in generation order
    auto send_off = [&](uint32_t s, uint32_t g) {
        uint64_t o = 0;
        for (uint32_t q = 0; q < g; ++q) o += M(s, q);
        return o;
    };
    auto gen_shard = [&](uint32_t s, const uint32_t* walks, uint64_t su) -> int {
        if (!su) return NE_OK;
        ne::PoolParams pp = pool_params(c, epoch, episode, u0, su);
        NE_CUDA(c, ne::launch_pairs_parts(walks, c->d_slot_tab, pp, c->d_part_bounds, P, c->d_base, c->d_pool,
                                          c->dev, c->ws));
        c->launches += 1;
        (void)s;
        return NE_OK;
    };
    bt.mark("host");
    if (real) {
        NE_TRY(gen_shard(me, c->d_walks, c->shard_units));
        bt.mark("pairs_parts");
        NE_NCCL(c, ncclGroupStart());
        for (uint32_t q = 0; q < P; ++q) {
            if (M(me, q)) NE_NCCL(c, ncclSend(c->d_pool + send_off(me, q), M(me, q), ncclUint64, (int)q, c->comm_walk,
                                              c->ws));
            if (M(q, me)) NE_NCCL(c, ncclRecv(c->d_slots + recv_off[q], M(q, me), ncclUint64, (int)q, c->comm_walk,
                                              c->ws));
        }
        NE_NCCL(c, ncclGroupEnd());
    } else {
        for (uint32_t s = 0; s < P; ++s) {
            uint64_t su;
            const uint32_t* w = shard_walks(s, &su);
            if (!M(s, me)) continue;
            NE_TRY(count_shard(s, w, su, c->d_tmat + (uint64_t)s * P));  // counts / bases of shard s again
            NE_TRY(gen_shard(s, w, su));
            NE_CUDA(c, cudaMemcpyAsync(c->d_slots + recv_off[s], c->d_pool + send_off(s, me), M(s, me) * sizeof(uint64_t),
                                       cudaMemcpyDeviceToDevice, c->ws));
        }
    }
    bt.mark("exchange");
    // O6: pi over the gathered pool, then order + bucketing
    ne::PoolParams pp = pool_params(c, epoch, episode, u0, units);
    pp.N = N;
    const bool keyed = c->d_keys[0] && N > 0 && N <= (1ull << 32);
    if (N) {
        if (keyed) {
            NE_CUDA(c, ne::launch_feistel_keys(pp, c->d_keys[0], c->dev, c->ws));
        } else {  // direct: dense pi-indexed array in d_slots (via d_pool)
            NE_CUDA(c, ne::launch_feistel_scatter(pp, c->d_slots, c->d_pool, c->dev, c->ws));
            std::swap(c->d_slots, c->d_pool);
        }
        c->launches += 1;
    }
    bt.mark("feistel_keys");
    NE_TRY(finish_pool(c, N, keyed));
    bt.mark("order+bucket");
    bt.report(episode, N);
    c->built_epoch = epoch;
    c->built_episode = episode;
    return NE_OK;
}

int do_build(ne_ctx* c, uint32_t epoch, uint32_t episode) {
    NvtxRange range("ne pool build");
    if (c->world > 1 && c->cfg.walk_len > 0) return do_build_sharded(c, epoch, episode);
    uint64_t u0, units;
    episode_range(c, episode, &u0, &units);
    BuildTimer bt(c);
    ne::PoolParams p = pool_params(c, epoch, episode, u0, units);
    // O5: kept pairs per unit, exclusive scan -> part-local index bases, N_g
    uint64_t N = 0;
    if (units) {
        if (c->cfg.walk_len == 0) {
            NE_CUDA(c, ne::launch_count_line(c->d_tgt, p, c->d_counts, c->dev, c->ws));
            c->launches += 1;
        } else if (!c->walk_counts) {
            NE_CUDA(c, ne::launch_count_walk(c->d_walks, c->d_slot_tab, p, c->d_counts, c->dev, c->ws));
            c->launches += 1;
        }
        NE_CUDA(c, ne::launch_scan(c->d_counts, units, c->d_base, c->d_total, c->d_scan_scratch, c->ws,
                                   &c->launches));
        NE_CUDA(c, cudaMemcpyAsync(&N, c->d_total, sizeof N, cudaMemcpyDeviceToHost, c->ws));
        NE_CUDA(c, cudaStreamSynchronize(c->ws));
    }
    bt.mark("count+scan");
    if (N > c->N_max) return ne_fail(c, NE_ERANGE, "episode pool %llu > bound %llu (internal)", (unsigned long long)N,
                                  (unsigned long long)c->N_max);
    NE_TRY(ensure_pool(c, N));
    select_scratch(c, c->keep_pool);
    // O6: every kept pair with its position pi(x), then stable bucketing by sub-part
    p.N = N;
    const bool keyed = c->d_keys[0] && N > 0 && N <= (1ull << 32);
    if (N) {
        ne::PoolSink sink{c->d_slots, keyed ? c->d_keys[0] : nullptr};
        if (c->cfg.walk_len > 0)
            NE_CUDA(c, ne::launch_pairs_walk(c->d_walks, c->d_slot_tab, p, c->d_base, sink, c->dev, c->ws));
        else
            NE_CUDA(c, ne::launch_pairs_line(c->d_off, c->d_tgt, c->n, p, c->d_base, sink, c->dev, c->ws));
        c->launches += 1;
    }
    bt.mark("pairs+keys");
    NE_TRY(finish_pool(c, N, keyed));
    bt.mark("order+bucket");
    bt.report(episode, N);
    c->built_epoch = epoch;
    c->built_episode = episode;
    return NE_OK;
}

ne::SgnsParams sgns_params(const ne_ctx* c, uint32_t vsub, float* V, uint32_t epoch,
                           uint32_t episode, float lr) {
    ne::SgnsParams p{};
    p.pool = reinterpret_cast<const uint2*>(c->pool_at + c->boff[vsub]);
    p.count = c->boff[vsub + 1] - c->boff[vsub];
    p.V = V;
    p.v_begin = c->sub_bounds[vsub];
    p.C = c->d_C;
    p.c_begin = c->c_begin;
    p.c_count = c->c_count;
    p.alias = c->d_alias;
    p.d = c->cfg.dim;
    p.K = c->cfg.negatives;
    p.lr = lr;
    p.seed = c->cfg.seed;
    p.epoch = epoch;
    p.episode = episode;
    p.block = vsub * (uint32_t)c->world + (uint32_t)c->rank;
    p.loss = c->d_loss;
    p.deterministic = (int)c->cfg.deterministic;
    const double eps = (c->cfg.conflict_permille ? c->cfg.conflict_permille : 300) / 1000.0;
    const double kk = (1.0 + c->cfg.negatives) * (1.0 + c->cfg.negatives);
    const double vr = (double)std::max<uint64_t>(1, c->sub_bounds[vsub + 1] - c->sub_bounds[vsub]);
    const double cr = (double)std::max<uint64_t>(1, c->c_count);
    const double cap = eps / (kk / cr + 1.0 / vr);
    p.max_warps = cap >= 1e15 ? ~0ull : std::max<uint64_t>(1, (uint64_t)cap);
    if (c->cfg.update_rule == NE_UPDATE_SHARED_BATCH) {
        // shared-negative batches: at most eps of the rows touched by concurrent
        // batches (2B + K' rows each); the cap is counted in batches (CTAs)
        const double rows = std::min(cr, vr), per = 2.0 * 128 + c->cfg.negatives;
        const double bcap = eps * rows / per;
        p.max_warps = bcap >= 1e15 ? ~0ull : std::max<uint64_t>(1, (uint64_t)bcap);
    }
    p.atomic_writeback = c->cfg.writeback == NE_WB_ATOMIC_DELTA ? 1 : 0;
    p.accumulate = (int)c->cfg.update_rule;
    p.bf16 = c->cfg.storage == NE_STORE_BF16 ? 1 : 0;
    // with a ring, leave SMs to NCCL's send/recv kernels so the transfer of the
    // previous sub-part overlaps this block (developer knob NE_RING_RESERVE_SMS)
    static const int reserve = [] {  // measured: 0, 2, 4 SMs perform alike (C4, 4 GPUs)
        const char* e = std::getenv("NE_RING_RESERVE_SMS");
        return e ? std::atoi(e) : 0;
    }();
    p.reserve_sms = std::max((c->world > 1 && c->comm) ? reserve : 0, c->sgns_reserve);
    static const uint32_t l2hint = [] {  // developer knob NE_SGNS_L2HINT (V policy | C policy << 2; 1 first, 2 last)
        const char* e = std::getenv("NE_SGNS_L2HINT");
        return e ? (uint32_t)std::atoi(e) : 0u;
    }();
    p.l2hint = l2hint;
    return p;
}

// Launched training of one episode: timing events and sample count, read
// back by finish_train after the stream has run them.
struct TrainPending {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed, waits;
    uint64_t samples = 0;
    uint32_t launches = 0;
};

// NEXT-2 host staging (P:142 stages 2 and 5), one GPU: sub-part t trains in
// slot t mod 3 while sub-part t+1 is copied in (copy stream) and t-1 copied
// back (comm stream); a slot is refilled only after its previous D2H.
int launch_train_staged(ne_ctx* c, uint32_t epoch, uint32_t episode, float lr, TrainPending& tp) {
    const uint32_t k = c->cfg.subparts, S = (uint32_t)c->vslot.size();
    const uint64_t d = c->cfg.dim;
    std::vector<cudaEvent_t> loaded(k), stored(k);
    const uint32_t base = c->stage_base;
    auto slot = [&](uint32_t t) { return c->vslot[(t + base) % S]; };
    auto h2d = [&](uint32_t t) -> int {
        if (t >= S) NE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, stored[t - S], 0));
        else if (c->stage_pending) NE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->stage_done, 0));
        const uint64_t sb = c->sub_bounds[t], rows = c->sub_bounds[t + 1] - sb;
        NE_CUDA(c, cudaMemcpyAsync(slot(t), host_row(c, sb), rows * d * elem_bytes(c),
                                   cudaMemcpyHostToDevice, c->copy_stream));
        loaded[t] = next_event(c);
        NE_CUDA(c, cudaEventRecord(loaded[t], c->copy_stream));
        return NE_OK;
    };
    if (k && c->stage_pre) loaded[0] = c->stage_pre_ev;  // prefetched by the previous episode
    else if (k) NE_TRY(h2d(0));
    c->stage_pre = false;
    for (uint32_t t = 0; t < k; ++t) {
        if (t + 1 < k) NE_TRY(h2d(t + 1));
        NE_CUDA(c, cudaStreamWaitEvent(c->stream, loaded[t], 0));
        const ne::SgnsParams sp = sgns_params(c, t, slot(t), epoch, episode, lr);
        cudaEvent_t e0 = next_event(c), e1 = next_event(c);
        NE_CUDA(c, cudaEventRecord(e0, c->stream));
        NE_CUDA(c, ne::launch_sgns(sp, c->dev, c->stream));
        NE_CUDA(c, cudaEventRecord(e1, c->stream));
        if (sp.count) { c->launches += 1; tp.launches += 1; }
        tp.timed.push_back({e0, e1});
        tp.samples += sp.count;
        const uint64_t sb = c->sub_bounds[t], rows = c->sub_bounds[t + 1] - sb;
        NE_CUDA(c, cudaStreamWaitEvent(c->comm_stream, e1, 0));
        NE_CUDA(c, cudaMemcpyAsync(host_row(c, sb), slot(t), rows * d * elem_bytes(c),
                                   cudaMemcpyDeviceToHost, c->comm_stream));
        stored[t] = next_event(c);
        NE_CUDA(c, cudaEventRecord(stored[t], c->comm_stream));
    }
    // the last copies back stay in flight; the next call's first H2D and every
    // host-side reader wait for them
    if (!c->stage_done) NE_CUDA(c, cudaEventCreateWithFlags(&c->stage_done, cudaEventDisableTiming));
    NE_CUDA(c, cudaEventRecord(c->stage_done, c->comm_stream));
    c->stage_pending = true;
    // Prefetch the next episode's sub-part 0 while sub-part k-1 still trains, so
    // an episode does not start behind a full-part H2D: slots rotate across
    // episodes (sub-part 0 of the next episode takes slot (base + k) % 3), and
    // that slot is free once sub-part k-3, its last user, is copied back
    // (comm-stream order also puts sub-part 0's own copy-back, the rows loaded
    // here, before it).  Host writers (rows_op, load_graph) drop the prefetch.
    c->stage_base = (base + k) % S;
    if (k) {
        if (!c->stage_pre_ev) NE_CUDA(c, cudaEventCreateWithFlags(&c->stage_pre_ev, cudaEventDisableTiming));
        NE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, k >= S ? stored[k - S] : c->stage_done, 0));
        NE_CUDA(c, cudaMemcpyAsync(c->vslot[c->stage_base], host_row(c, c->sub_bounds[0]),
                                   (c->sub_bounds[1] - c->sub_bounds[0]) * d * elem_bytes(c),
                                   cudaMemcpyHostToDevice, c->copy_stream));
        NE_CUDA(c, cudaEventRecord(c->stage_pre_ev, c->copy_stream));
        c->stage_pre = true;
    }
    return NE_OK;
}

// NEXT-2 with the ring (P:142 pipeline stages 5, 3, 4, 2; "ping-pong
// buffers"; reading D18): this rank's vertex part lives in pinned host memory;
// its k sub-parts run in windows of w slots.  A window's home sub-parts are
// prefetched into one set of w device slots (stage 5, copy stream) while the
// previous window trains; the window then goes around the ring exactly like
// the in-HBM plan (train set `cur`, send it, receive the next round's
// sub-parts into set `nxt`, swap), and after the last round its sub-parts are
// home again and copied back (stage 2, comm stream).  Device memory: 3 w
// sub-parts instead of 2 k.
int launch_train_staged_ring(ne_ctx* c, uint32_t epoch, uint32_t episode, float lr, TrainPending& tp) {
    const uint32_t P = (uint32_t)c->world, k = c->cfg.subparts, g = (uint32_t)c->rank, G = groups_of(c);
    const uint32_t w = stage_window(c);
    const uint64_t d = c->cfg.dim, esz = elem_bytes(c);
    if (!c->comm) return ne_fail(c, NE_ESTATE, "world=%u context has no NCCL communicator (layout-only)", P);
    const ncclDataType_t dt = c->cfg.storage == NE_STORE_BF16 ? ncclBfloat16 : ncclFloat;
    auto slot = [&](uint32_t set, uint32_t t) { return c->vslot[(size_t)set * w + t]; };
    const uint32_t nwin = (k + w - 1) / w;
    uint32_t cur = 0, nxt = 1, pre = 2;
    std::vector<cudaEvent_t> loaded(w, nullptr), drained(w, nullptr);
    // window 0 prefetched during the previous episode's last window: it trains
    // in that set; the previous last window's home set is still draining
    const bool resumed = c->stage_pre;
    if (resumed) {
        cur = c->stage_pre_set;
        pre = c->stage_drain_set;
        nxt = 3 - cur - pre;
    }
    c->stage_pre = false;
    auto prefetch = [&](uint32_t win, uint32_t set) -> int {  // stage 5: H2D of the window's home sub-parts
        for (uint32_t t = 0; t < w && win * w + t < k; ++t) {
            if (drained[t]) NE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, drained[t], 0));
            else if (c->stage_pending) NE_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->stage_done, 0));
            const uint64_t vs = (uint64_t)g * k + win * w + t, sb = c->sub_bounds[vs];
            NE_CUDA(c, cudaMemcpyAsync(slot(set, t), host_row(c, sb), (c->sub_bounds[vs + 1] - sb) * d * esz,
                                       cudaMemcpyHostToDevice, c->copy_stream));
            loaded[t] = next_event(c);
            NE_CUDA(c, cudaEventRecord(loaded[t], c->copy_stream));
        }
        return NE_OK;
    };
    if (resumed) std::fill(loaded.begin(), loaded.end(), c->stage_pre_ev);
    else NE_TRY(prefetch(0, cur));
    std::vector<cudaEvent_t> recv(w, nullptr);
    for (uint32_t win = 0; win < nwin; ++win) {
        const uint32_t t0 = win * w, wn = std::min(w, k - t0);
        for (uint32_t t = 0; t < wn; ++t) recv[t] = loaded[t];
        if (win + 1 < nwin) NE_TRY(prefetch(win + 1, pre));  // overlaps this whole window
        // the last window also overlaps the next episode's window 0: its rows
        // came home and were copied back at the end of window 0 (ordered before
        // the drain this prefetch waits for), so the next episode does not
        // start behind a window's H2D.  Host writers (rows_op, load_graph)
        // drop it.  One window per episode: no free set yet, no prefetch.
        const bool ahead = win + 1 == nwin && nwin > 1;
        if (ahead) {
            NE_TRY(prefetch(0, pre));
            if (!c->stage_pre_ev) NE_CUDA(c, cudaEventCreateWithFlags(&c->stage_pre_ev, cudaEventDisableTiming));
            NE_CUDA(c, cudaEventRecord(c->stage_pre_ev, c->copy_stream));
        }
        for (uint32_t r = 0; r < P; ++r) {
            for (uint32_t t = 0; t < wn; ++t) {
                const uint32_t vs = (uint32_t)plan_vsub(P, G, k, r, t0 + t, g);
                float* V = slot(cur, t);
                cudaEvent_t w0 = next_event(c), w1 = next_event(c);
                NE_CUDA(c, cudaEventRecord(w0, c->stream));
                NE_CUDA(c, cudaStreamWaitEvent(c->stream, recv[t], 0));
                NE_CUDA(c, cudaEventRecord(w1, c->stream));
                tp.waits.push_back({w0, w1});
                const ne::SgnsParams sp = sgns_params(c, vs, V, epoch, episode, lr);
                cudaEvent_t e0 = next_event(c), e1 = next_event(c);
                NE_CUDA(c, cudaEventRecord(e0, c->stream));
                NE_CUDA(c, ne::launch_sgns(sp, c->dev, c->stream));
                NE_CUDA(c, cudaEventRecord(e1, c->stream));
                if (sp.count) { c->launches += 1; tp.launches += 1; }
                tp.timed.push_back({e0, e1});
                tp.samples += sp.count;
                const uint32_t vs_next = (uint32_t)plan_vsub(P, G, k, r + 1, t0 + t, g);
                NE_CUDA(c, cudaStreamWaitEvent(c->comm_stream, e1, 0));
                NE_NCCL(c, ncclGroupStart());
                NE_NCCL(c, ncclSend(V, (c->sub_bounds[vs + 1] - c->sub_bounds[vs]) * d, dt,
                                    (int)ring_dest(P, G, r, g), c->comm, c->comm_stream));
                NE_NCCL(c, ncclRecv(slot(nxt, t), (c->sub_bounds[vs_next + 1] - c->sub_bounds[vs_next]) * d, dt,
                                    (int)ring_src(P, G, r, g), c->comm, c->comm_stream));
                NE_NCCL(c, ncclGroupEnd());
                recv[t] = next_event(c);
                NE_CUDA(c, cudaEventRecord(recv[t], c->comm_stream));
            }
            std::swap(cur, nxt);
        }
        // home again (set cur): stage 2, D2H after the last receive, on its own
        // stream so the next window's ring transfers do not queue behind it
        for (uint32_t t = 0; t < wn; ++t) {
            const uint64_t vs = (uint64_t)g * k + t0 + t, sb = c->sub_bounds[vs];
            NE_CUDA(c, cudaStreamWaitEvent(c->d2h_stream, recv[t], 0));
            NE_CUDA(c, cudaMemcpyAsync(host_row(c, sb), slot(cur, t), (c->sub_bounds[vs + 1] - sb) * d * esz,
                                       cudaMemcpyDeviceToHost, c->d2h_stream));
            drained[t] = next_event(c);
            NE_CUDA(c, cudaEventRecord(drained[t], c->d2h_stream));
        }
        // next window trains the prefetched set; this window's home set drains
        // and then takes the prefetch of the window after
        const uint32_t home = cur;
        cur = pre;
        pre = home;
        if (ahead) {  // cur now holds the next episode's window 0, pre drains
            c->stage_pre = true;
            c->stage_pre_set = cur;
            c->stage_drain_set = pre;
        }
    }
    if (!c->stage_done) NE_CUDA(c, cudaEventCreateWithFlags(&c->stage_done, cudaEventDisableTiming));
    NE_CUDA(c, cudaEventRecord(c->stage_done, c->d2h_stream));  // after every receive it waited for
    c->stage_pending = true;
    return NE_OK;
}

// O7 ring: round r, slot t trains block
// (vsub = ((rank - r) mod P)*k + t, context part rank); the trained sub-part is
// sent to rank+1 while slot t+1 trains, and the sub-part for round r+1 arrives
// from rank-1 into the other half of the ping-pong buffers.  Everything is
// enqueued (compute stream + comm stream); finish_train waits for it.
int launch_train(ne_ctx* c, uint32_t epoch, uint32_t episode, float lr, TrainPending& tp) {
    NvtxRange range("ne train (SGNS + ring)");
    NE_TRY(wait_alias(c));
    NE_CUDA(c, cudaMemsetAsync(c->d_loss, 0, sizeof(double), c->stream));
    if (c->cfg.staging == NE_STAGE_HOST && c->world > 1) return launch_train_staged_ring(c, epoch, episode, lr, tp);
    if (c->cfg.staging == NE_STAGE_HOST) return launch_train_staged(c, epoch, episode, lr, tp);
    const uint32_t P = (uint32_t)c->world, k = c->cfg.subparts, g = (uint32_t)c->rank, G = groups_of(c);
    const uint64_t d = c->cfg.dim;
    const bool ipc = ipc_ring(c);
    const bool ipc_resumed = ipc && c->ipc.started;  // arrivals owed from an earlier call (not this one's pushes)
    if (P > 1 && !c->comm && !ipc)
        return ne_fail(c, NE_ESTATE, "world=%u context has no NCCL communicator (layout-only)", P);
    std::vector<cudaEvent_t> recv(k, nullptr);
    if (c->ring_pending) recv.assign(k, c->ring_done);  // home-coming sub-parts of the last call
    for (uint32_t r = 0; r < P; ++r) {
        for (uint32_t t = 0; t < k; ++t) {
            const uint32_t vs = (uint32_t)plan_vsub(P, G, k, r, t, g);
            float* V = c->vslot[c->cur * k + t];
            if (ipc && (r > 0 || ipc_resumed)) {  // the sub-part of this slot has landed
                cudaEvent_t w0 = next_event(c), w1 = next_event(c);
                NE_CUDA(c, cudaEventRecord(w0, c->stream));
                NE_TRY(ipc_wait_arrival(c, t, ring_kind(P, G, r + P - 1)));
                NE_CUDA(c, cudaEventRecord(w1, c->stream));
                tp.waits.push_back({w0, w1});
            } else if (recv[t]) {
                cudaEvent_t w0 = next_event(c), w1 = next_event(c);
                NE_CUDA(c, cudaEventRecord(w0, c->stream));
                NE_CUDA(c, cudaStreamWaitEvent(c->stream, recv[t], 0));
                NE_CUDA(c, cudaEventRecord(w1, c->stream));
                tp.waits.push_back({w0, w1});
            }
            const ne::SgnsParams sp = sgns_params(c, vs, V, epoch, episode, lr);
            cudaEvent_t e0 = next_event(c), e1 = next_event(c);
            NE_CUDA(c, cudaEventRecord(e0, c->stream));
            NE_CUDA(c, ne::launch_sgns(sp, c->dev, c->stream));
            NE_CUDA(c, cudaEventRecord(e1, c->stream));
            if (sp.count) { c->launches += 1; tp.launches += 1; }
            tp.timed.push_back({e0, e1});
            tp.samples += sp.count;
            if (P == 1 && c->export_now) {  // sub-part t is final for this call: copy it out now
                const uint64_t rb = c->sub_bounds[vs], rows = c->sub_bounds[vs + 1] - rb;
                NE_CUDA(c, cudaStreamWaitEvent(c->d2h_stream, e1, 0));
                NE_CUDA(c, cudaMemcpyAsync(c->export_V + (rb - c->part_bounds[c->rank]) * d, V, rows * d * sizeof(float),
                                           cudaMemcpyDeviceToHost, c->d2h_stream));
            }
            if (P > 1 && ipc) {  // copy-engine push into rank + 1 (ring_ipc.cpp)
                const uint64_t send_rows = c->sub_bounds[vs + 1] - c->sub_bounds[vs];
                NE_TRY(ipc_push(c, t, V, send_rows * d * elem_bytes(c), e1, ring_kind(P, G, r), ring_dest(P, G, r, g),
                                ring_src(P, G, r + 1, g), ring_kind(P, G, r + 1)));
            } else if (P > 1) {
                const uint32_t vs_next = (uint32_t)plan_vsub(P, G, k, r + 1, t, g);
                const uint64_t send_rows = c->sub_bounds[vs + 1] - c->sub_bounds[vs];
                const uint64_t recv_rows = c->sub_bounds[vs_next + 1] - c->sub_bounds[vs_next];
                float* Vn = c->vslot[(1 - c->cur) * k + t];
                NE_CUDA(c, cudaStreamWaitEvent(c->comm_stream, e1, 0));
                NE_NCCL(c, ncclGroupStart());
                const ncclDataType_t dt = c->cfg.storage == NE_STORE_BF16 ? ncclBfloat16 : ncclFloat;
                NE_NCCL(c, ncclSend(V, send_rows * d, dt, (int)ring_dest(P, G, r, g), c->comm, c->comm_stream));
                NE_NCCL(c, ncclRecv(Vn, recv_rows * d, dt, (int)ring_src(P, G, r, g), c->comm, c->comm_stream));
                NE_NCCL(c, ncclGroupEnd());
                cudaEvent_t rv = next_event(c);
                NE_CUDA(c, cudaEventRecord(rv, c->comm_stream));
                recv[t] = rv;
            }
            if (P > 1 && c->export_now && r + 1 == P) {  // sub-part t comes home final: copy it out on arrival
                const uint32_t vs_home = (uint32_t)plan_vsub(P, G, k, P, t, g);
                const uint64_t rb = c->sub_bounds[vs_home], rows = c->sub_bounds[vs_home + 1] - rb;
                if (ipc) NE_TRY(ipc_wait_home(c, c->d2h_stream, t, ring_kind(P, G, r)));
                else NE_CUDA(c, cudaStreamWaitEvent(c->d2h_stream, recv[t], 0));
                NE_CUDA(c, cudaMemcpyAsync(c->export_V + (rb - c->part_bounds[c->rank]) * d,
                                           c->vslot[(1 - c->cur) * k + t], rows * d * sizeof(float),
                                           cudaMemcpyDeviceToHost, c->d2h_stream));
            }
        }
        if (P > 1) c->cur = 1 - c->cur;
    }
    // The sub-parts are on their way home.  The receives are not awaited here:
    // the next call's first training of each slot waits for them (the next
    // episode's walk and pool build overlap the transfers); every reader of the
    // vertex slots (get/set embeddings, reload, destroy) drains the comm stream.
    c->ring_pending = false;
    if (P > 1 && !ipc) {
        if (!c->ring_done) NE_CUDA(c, cudaEventCreateWithFlags(&c->ring_done, cudaEventDisableTiming));
        NE_CUDA(c, cudaEventRecord(c->ring_done, c->comm_stream));
        c->ring_pending = true;
    }
    return NE_OK;
}

// Wait for a launched episode, add its loss, samples and kernel times to st.
int finish_train(ne_ctx* c, TrainPending& tp, ne_stats* st) {
    double loss = 0.0;
    NE_CUDA(c, cudaMemcpyAsync(&loss, c->d_loss, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NE_TRY(wait_stream(c, c->stream));
    if (st) {
        st->samples += tp.samples;
        st->loss_sum += loss;
        st->train_launches += tp.launches;
        for (auto& pr : tp.timed) {
            float ms = 0.f;
            NE_CUDA(c, cudaEventElapsedTime(&ms, pr.first, pr.second));
            st->ms_train += ms;
        }
        for (auto& pr : tp.waits) {
            float ms = 0.f;
            NE_CUDA(c, cudaEventElapsedTime(&ms, pr.first, pr.second));
            st->ms_comm_wait += ms;
        }
    }
    return NE_OK;
}

int do_train(ne_ctx* c, uint32_t epoch, uint32_t episode, float lr, ne_stats* st) {
    TrainPending tp;
    NE_TRY(launch_train(c, epoch, episode, lr, tp));
    NE_TRY(finish_train(c, tp, st));
    c->ev_used = 0;
    return NE_OK;
}

// Walk + build of (epoch, episode) on stream `s` into the current pool state;
// ms_walk / ms_build from events on `s`.
int walk_build(ne_ctx* c, uint32_t epoch, uint32_t episode, cudaStream_t s, float* ms_walk, float* ms_build) {
    c->ws = s;
    cudaEvent_t a = next_event(c), b = next_event(c), d = next_event(c);
    int rc = NE_OK;
    if (cudaEventRecord(a, s) != cudaSuccess) rc = ne_fail(c, NE_ECUDA, "event record");
    if (rc == NE_OK && c->cfg.walk_len > 0) rc = do_walk(c, epoch, episode);
    if (rc == NE_OK && cudaEventRecord(b, s) != cudaSuccess) rc = ne_fail(c, NE_ECUDA, "event record");
    if (rc == NE_OK) rc = do_build(c, epoch, episode);  // synchronises s
    if (rc == NE_OK && cudaEventRecord(d, s) != cudaSuccess) rc = ne_fail(c, NE_ECUDA, "event record");
    c->ws = c->stream;
    NE_TRY(rc);
    NE_CUDA(c, cudaEventSynchronize(d));
    NE_CUDA(c, cudaEventElapsedTime(ms_walk, a, b));
    NE_CUDA(c, cudaEventElapsedTime(ms_build, b, d));
    return NE_OK;
}

// Build (epoch, episode) into c->next on build_stream while the current pool
// (pool_at) trains on the compute stream: the build uses the two pair buffers
// the training pool does not occupy and the alternate block-offset array.
int prebuild_next(ne_ctx* c, uint32_t epoch, uint32_t episode) {
    NvtxRange range("ne next-episode build (side stream)");
    // stash the current pool
    uint64_t* at = c->pool_at;
    std::vector<uint64_t> boff;
    boff.swap(c->boff);
    uint64_t* d_boff = c->d_boff;
    const int64_t be = c->built_epoch, bp = c->built_episode;
    const uint64_t gen = c->pool_gen;
    c->keep_pool = at;
    c->d_boff = c->d_boff_alt;
    float mw = 0.f, mb = 0.f;
    const int rc = walk_build(c, epoch, episode, c->build_stream, &mw, &mb);
    c->keep_pool = nullptr;
    c->next.valid = rc == NE_OK && c->built_epoch == (int64_t)epoch;
    c->next.at = c->pool_at;
    c->next.d_boff = c->d_boff;
    c->next.boff.swap(c->boff);
    c->next.epoch = epoch;
    c->next.episode = episode;
    c->next.ms_walk = mw;
    c->next.ms_build = mb;
    // restore the current pool (a buffer growth inside the build invalidated it)
    const bool grown = c->pool_gen != gen;
    c->pool_at = at;
    c->boff.swap(boff);
    c->d_boff = d_boff;  // d_boff_alt stays the array the next pool's offsets are in
    c->built_epoch = grown ? -1 : be;
    c->built_episode = grown ? -1 : bp;
    return rc;
}

// Make c->next the current pool (the old current's block-offset array becomes
// the alternate).
void adopt_next(ne_ctx* c) {
    c->pool_at = c->next.at;
    c->boff.swap(c->next.boff);
    std::swap(c->d_boff, c->d_boff_alt);  // d_boff_alt held next.d_boff
    c->built_epoch = c->next.epoch;
    c->built_episode = c->next.episode;
    c->next.valid = false;
}

bool pipelined(const ne_ctx* c) { return c->pbufs.size() >= 3; }

}  // namespace

extern "C" {

int ne_version(void) { return NE_ABI_VERSION; }

int ne_plan_vsub(uint32_t world, uint32_t subparts, uint32_t r, uint32_t t, uint32_t g) {
    if (world == 0 || subparts == 0 || t >= subparts || g >= world) return -1;
    return plan_vsub(world, 1, subparts, r, t, g);
}

int ne_plan_vsub2(uint32_t world, uint32_t groups, uint32_t subparts, uint32_t rho, uint32_t t, uint32_t g) {
    if (groups == 0) groups = 1;
    if (world == 0 || world % groups || subparts == 0 || t >= subparts || g >= world) return -1;
    return plan_vsub(world, groups, subparts, rho, t, g);
}

int ne_ring_peers(uint32_t world, uint32_t groups, uint32_t rho, uint32_t g, uint32_t* dest, uint32_t* src) {
    if (groups == 0) groups = 1;
    if (world == 0 || world % groups || g >= world || !dest || !src) return NE_EINVAL;
    *dest = ring_dest(world, groups, rho, g);
    *src = ring_src(world, groups, rho, g);
    return NE_OK;
}

int ne_partition_bounds(uint64_t n, uint32_t parts, uint64_t* bounds) {
    if (parts == 0 || !bounds) return NE_EINVAL;
    partition(0, n, parts, bounds);
    return NE_OK;
}

int ne_create(ne_ctx** out, const ne_config* cfg, int device, ne_alloc_fn alloc,
              ne_free_fn free_fn, void* user) {
    g_create_error.clear();
    if (!out || !cfg) return ne_fail(nullptr, NE_EINVAL, "null argument");
    *out = nullptr;
    ne_ctx* c = new ne_ctx();
    c->cfg = *cfg;
    c->device = device;
    c->alloc = alloc;
    c->free_fn = free_fn;
    c->user = user;
    auto bad = [&](int code) {  // the message stays readable through ne_last_error(NULL)
        g_create_error = c->err;
        ne_destroy(c);
        return code;
    };
    const ne_config& g = *cfg;
    if (g.dim == 0 || g.dim % 4 || g.dim > 512)
        return bad(ne_fail(c, NE_EINVAL, "dim=%u must be a multiple of 4 in [4, 512]", g.dim));
    if (g.update_rule == NE_UPDATE_SHARED_BATCH) {
        if (g.dim != 128 || g.negatives != 32 || g.storage != NE_STORE_F32)
            return bad(ne_fail(c, NE_EINVAL, "update_rule=2 (shared-negative batches) needs dim=128, negatives=32 "
                                             "and fp32 storage (dim=%u negatives=%u)", g.dim, g.negatives));
    } else if (g.negatives > 8) {
        return bad(ne_fail(c, NE_EINVAL, "negatives=%u > 8", g.negatives));
    }
    if (g.walk_len > 255) return bad(ne_fail(c, NE_EINVAL, "walk_len=%u > 255", g.walk_len));
    if (g.walk_len > 0 && (g.window == 0 || g.window > g.walk_len))
        return bad(ne_fail(c, NE_EINVAL, "window=%u not in [1, walk_len=%u]", g.window, g.walk_len));
    if (g.walk_len > 0 && g.walks_per_node == 0)
        return bad(ne_fail(c, NE_EINVAL, "walks_per_node must be >= 1"));
    if (g.episodes == 0 || g.episodes > 4095)
        return bad(ne_fail(c, NE_EINVAL, "episodes=%u not in [1, 4095]", g.episodes));
    if (g.writeback > NE_WB_STORE) return bad(ne_fail(c, NE_EINVAL, "writeback=%u not in {0, 1}", g.writeback));
    if (g.update_rule > NE_UPDATE_SHARED_BATCH)
        return bad(ne_fail(c, NE_EINVAL, "update_rule=%u not in {0, 1, 2}", g.update_rule));
    if (g.staging > NE_STAGE_HOST) return bad(ne_fail(c, NE_EINVAL, "staging=%u not in {0, 1}", g.staging));
    if (g.storage > NE_STORE_BF16) return bad(ne_fail(c, NE_EINVAL, "storage=%u not in {0, 1}", g.storage));
    if (g.transport > NE_TRANSPORT_IPC)
        return bad(ne_fail(c, NE_EINVAL, "transport=%u not in {0 (NCCL), 1 (IPC)}", g.transport));
    if (!(g.p >= 0.f) || !(g.q >= 0.f))
        return bad(ne_fail(c, NE_EINVAL, "node2vec p=%g q=%g must be > 0 (0 = 1)", g.p, g.q));
    {
        // node2vec thresholds (NEXT-1): alpha = 1/p, 1, 1/q scaled by their max to 2^32
        const double pp = g.p == 0.f ? 1.0 : (double)g.p, qq = g.q == 0.f ? 1.0 : (double)g.q;
        c->n2v = !(pp == 1.0 && qq == 1.0);
        const double w[3] = {1.0 / pp, 1.0, 1.0 / qq};
        const double mx = std::max(std::max(w[0], w[1]), w[2]);
        for (int i = 0; i < 3; ++i)
            c->n2v_thr[i] = w[i] == mx ? (1ull << 32) : (uint64_t)(w[i] / mx * 4294967296.0);
    }
    if (g.subparts == 0 || g.subparts > 256)
        return bad(ne_fail(c, NE_EINVAL, "subparts=%u not in [1, 256]", g.subparts));
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return bad(ne_fail(c, NE_ECUDA, "no CUDA device %d (%s)", device,
                        e != cudaSuccess ? cudaGetErrorString(e) : "out of range"));
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
        return bad(ne_fail(c, NE_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device,
                        prop.major, prop.minor));
    c->dev.sm_count = prop.multiProcessorCount;
    c->dev.max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->build_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&c->d_loss, sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->d_bad, 3 * sizeof(unsigned long long)) != cudaSuccess)
        return bad(ne_fail(c, NE_ECUDA, "stream/scratch setup failed on device %d", device));
    c->stream = c->ws = c->own_stream;
    *out = c;
    return NE_OK;
}

int ne_set_stream(ne_ctx* c, void* stream) {
    NE_TRY(enter(c));
    c->stream = c->ws = stream == NE_STREAM_OWN ? c->own_stream : stream ? (cudaStream_t)stream : cudaStreamLegacy;
    return NE_OK;
}

int ne_join(ne_ctx* c) {
    NE_TRY(enter(c));
    if (c->ring_pending) NE_CUDA(c, cudaStreamWaitEvent(c->stream, c->ring_done, 0));
    if (ipc_ring(c)) NE_TRY(ipc_drain(c, false));
    if (c->stage_pending) NE_CUDA(c, cudaStreamWaitEvent(c->stream, c->stage_done, 0));
    return NE_OK;
}

int ne_get_nccl_id(uint8_t id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return NE_ENCCL;
    std::memcpy(id, &u, 128);
    return NE_OK;
}

int ne_init_dist(ne_ctx* c, int rank, int world, const uint8_t id[128]) {
    NE_TRY(enter(c));
    if (c->loaded) return ne_fail(c, NE_ESTATE, "ne_init_dist must precede ne_load_graph");
    if (world < 1 || rank < 0 || rank >= world) return ne_fail(c, NE_EINVAL, "rank=%d world=%d", rank, world);
    if (world > 1 && c->cfg.staging == NE_STAGE_HOST && c->cfg.transport == NE_TRANSPORT_IPC)
        return ne_fail(c, NE_EINVAL, "staging=NE_STAGE_HOST with world > 1 runs its ring over NCCL (transport=0)");
    if ((uint64_t)world * c->cfg.subparts > 256 || (uint64_t)world * world * c->cfg.subparts > 4096)
        return ne_fail(c, NE_EINVAL, "world=%d x subparts=%u exceeds the block-id range", world, c->cfg.subparts);
    if (world > 32) return ne_fail(c, NE_EINVAL, "world=%d > 32 (one lane per context part in the pool build)", world);
    if (c->cfg.groups > 1 && world % c->cfg.groups)
        return ne_fail(c, NE_EINVAL, "groups=%u does not divide world=%d", c->cfg.groups, world);
    if (c->comm_walk) { ncclCommDestroy(c->comm_walk); c->comm_walk = nullptr; }
    if (c->comm) { ncclCommDestroy(c->comm); c->comm = nullptr; }
    c->rank = rank;
    c->world = world;
    if (world > 1 && id) {  // id == NULL: layout-only context (pool/negatives of rank `rank`)
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        NE_NCCL(c, ncclCommInitRank(&c->comm, world, u, rank));
        NE_NCCL(c, ncclCommSplit(c->comm, 0, rank, &c->comm_walk, nullptr));
    }
    return NE_OK;
}

int ne_load_graph(ne_ctx* c, uint32_t n, uint64_t nnz, const uint64_t* offsets,
                  const uint32_t* targets) {
    NE_TRY(enter(c));
    if (!offsets || (nnz && !targets)) return ne_fail(c, NE_EINVAL, "null offsets/targets");
    if (n == 0xFFFFFFFFu) return ne_fail(c, NE_ERANGE, "n=%u reserves the sentinel id", n);
    if (n < (uint32_t)c->world) return ne_fail(c, NE_ERANGE, "n=%u < world=%d", n, c->world);
    if (nnz >= (1ull << 40)) return ne_fail(c, NE_ERANGE, "nnz=%llu too large", (unsigned long long)nnz);
    // A graph of the same shape reuses every device buffer (repeated loads, e2e).
    NE_TRY(ipc_drain(c, true));                          // IPC ring: pushes into / out of the slots
    NE_CUDA(c, cudaStreamSynchronize(c->comm_stream));  // ring transfers into the vertex slots
    NE_CUDA(c, cudaStreamSynchronize(c->copy_stream));
    NE_CUDA(c, cudaStreamSynchronize(c->d2h_stream));
    c->ring_pending = false;
    c->stage_pending = c->stage_pre = false;
    if (c->alias_thread.joinable()) c->alias_thread.join();
    c->alias_pending = false;
    const bool reuse = c->loaded && c->n == n && c->nnz == nnz;
    if (!reuse) free_all(c);
    c->loaded = false;
    c->walked_epoch = c->walked_episode = c->built_epoch = c->built_episode = -1;
    c->next.valid = false;
    const ne_config& g = c->cfg;
    const uint32_t P = (uint32_t)c->world, k = g.subparts;
    c->n = n;
    c->nnz = nnz;
#define NE_ALLOC(ptr, count) \
    do { if (!reuse) NE_TRY(dalloc_t(c, &(ptr), (count))); } while (0)

    // CSR into HBM, validated on the device.  With a communicator every
    // rank copies only its 1/P slice of the (identical) arrays over its own link
    // and an all-gather over NVLink completes them: P x less host-link traffic
    // per rank.  Buffers are padded to P equal chunks.
    const bool sliced = P > 1 && c->comm_walk;
    const uint64_t on = (uint64_t)n + 1;
    const uint64_t oc = sliced ? (on + P - 1) / P : on, tc = sliced ? (nnz + P - 1) / P : nnz;
    NE_ALLOC(c->d_off, sliced ? oc * P : on);
    NE_ALLOC(c->d_tgt, std::max<uint64_t>(sliced ? tc * P : nnz, 1));
    if (sliced) {
        const uint64_t r = (uint64_t)c->rank;
        const uint64_t ob = std::min(on, r * oc), oe = std::min(on, ob + oc);
        const uint64_t tb = std::min(nnz, r * tc), te = std::min(nnz, tb + tc);
        if (oe > ob)
            NE_CUDA(c, cudaMemcpyAsync(c->d_off + ob, offsets + ob, (oe - ob) * sizeof(uint64_t), cudaMemcpyDefault,
                                       c->stream));
        if (te > tb)
            NE_CUDA(c, cudaMemcpyAsync(c->d_tgt + tb, targets + tb, (te - tb) * sizeof(uint32_t), cudaMemcpyDefault,
                                       c->stream));
        NE_NCCL(c, ncclGroupStart());
        NE_NCCL(c, ncclAllGather(c->d_off + r * oc, c->d_off, oc, ncclUint64, c->comm_walk, c->stream));
        if (tc) NE_NCCL(c, ncclAllGather(c->d_tgt + r * tc, c->d_tgt, tc, ncclUint32, c->comm_walk, c->stream));
        NE_NCCL(c, ncclGroupEnd());
    } else {
        NE_CUDA(c, cudaMemcpyAsync(c->d_off, offsets, on * sizeof(uint64_t), cudaMemcpyDefault, c->stream));
        if (nnz) NE_CUDA(c, cudaMemcpyAsync(c->d_tgt, targets, nnz * sizeof(uint32_t), cudaMemcpyDefault, c->stream));
    }
    NE_CUDA(c, cudaMemsetAsync(c->d_bad, 0xFF, 3 * sizeof(unsigned long long), c->stream));
    NE_CUDA(c, ne::launch_validate_csr(c->d_off, c->d_tgt, n, nnz, c->d_bad, c->n2v, c->dev, c->stream));
    c->launches += 1;
    unsigned long long bad[3];
    uint64_t ends[2];
    NE_CUDA(c, cudaMemcpyAsync(bad, c->d_bad, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaMemcpyAsync(&ends[0], c->d_off, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaMemcpyAsync(&ends[1], c->d_off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (ends[0] != 0) return ne_fail(c, NE_EINVAL, "offsets[0]=%llu != 0", (unsigned long long)ends[0]);
    if (bad[0] != ~0ull) {
        uint64_t pair[2];
        NE_CUDA(c, cudaMemcpy(pair, c->d_off + bad[0], sizeof pair, cudaMemcpyDeviceToHost));
        return ne_fail(c, NE_EINVAL, "offsets[%llu]=%llu < offsets[%llu]=%llu", bad[0] + 1,
                    (unsigned long long)pair[1], bad[0], (unsigned long long)pair[0]);
    }
    if (ends[1] != nnz)
        return ne_fail(c, NE_EINVAL, "offsets[%u]=%llu != nnz=%llu", n, (unsigned long long)ends[1],
                    (unsigned long long)nnz);
    if (bad[1] != ~0ull) {
        uint32_t t;
        NE_CUDA(c, cudaMemcpy(&t, c->d_tgt + bad[1], sizeof t, cudaMemcpyDeviceToHost));
        return ne_fail(c, NE_EINVAL, "targets[%llu]=%u >= n=%u", bad[1], t, n);
    }
    if (bad[2] != ~0ull) {
        uint32_t t[2];
        NE_CUDA(c, cudaMemcpy(t, c->d_tgt + bad[2] - 1, sizeof t, cudaMemcpyDeviceToHost));
        return ne_fail(c, NE_EINVAL, "targets[%llu]=%u < targets[%llu]=%u: node2vec needs rows sorted by target",
                    bad[2], t[1], bad[2] - 1, t[0]);
    }

    // Partitions (D12): P context parts; each vertex part split into k sub-parts.
    c->part_bounds.assign(P + 1, 0);
    partition(0, n, P, c->part_bounds.data());
    c->sub_bounds.assign((size_t)P * k + 1, 0);
    c->max_sub_rows = 0;
    for (uint32_t p = 0; p < P; ++p) {
        partition(c->part_bounds[p], c->part_bounds[p + 1], k, &c->sub_bounds[(size_t)p * k]);
        for (uint32_t t = 0; t < k; ++t)
            c->max_sub_rows = std::max(c->max_sub_rows, c->sub_bounds[(size_t)p * k + t + 1] - c->sub_bounds[(size_t)p * k + t]);
    }
    c->sub_bounds[(size_t)P * k] = n;
    NE_ALLOC(c->d_sub_bounds, c->sub_bounds.size());
    NE_CUDA(c, cudaMemcpyAsync(c->d_sub_bounds, c->sub_bounds.data(), c->sub_bounds.size() * sizeof(uint64_t),
                               cudaMemcpyHostToDevice, c->stream));

    // Alias table of this rank's context part (O3, reading D9).
    c->c_begin = c->part_bounds[c->rank];
    c->c_count = c->part_bounds[c->rank + 1] - c->c_begin;
    // Degrees of the context part: read the caller's offsets directly when they
    // are host memory, else copy that slice back from the device.
    std::vector<uint64_t> hoff;
    const uint64_t* deg_src = offsets + c->c_begin;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, offsets) != cudaSuccess) cudaGetLastError();
    if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
        hoff.resize(c->c_count + 1);
        NE_CUDA(c, cudaMemcpyAsync(hoff.data(), c->d_off + c->c_begin, hoff.size() * sizeof(uint64_t),
                                   cudaMemcpyDeviceToHost, c->stream));
        NE_CUDA(c, cudaStreamSynchronize(c->stream));
        deg_src = hoff.data();
    }
    c->alias_deg.resize(c->c_count);
    for (uint64_t i = 0; i < c->c_count; ++i) c->alias_deg[i] = deg_src[i + 1] - deg_src[i];
    if (!c->alias_scratch) c->alias_scratch = std::make_shared<AliasScratch>();
    NE_ALLOC(c->d_alias, std::max<uint64_t>(c->c_count, 1));
    // The table is built on host threads while the GPU initialises, walks and
    // builds the first pool; wait_alias joins it before the first SGNS launch.
    c->alias_thread = std::thread([c] {
        build_alias(c->alias_deg.data(), c->alias_deg.size(), c->alias_host,
                    *static_cast<AliasScratch*>(c->alias_scratch.get()));
    });
    c->alias_pending = true;

    // Embeddings (O9): context part = 0; home vertex sub-parts initialised.
    const uint64_t esz = g.storage == NE_STORE_BF16 ? 2 : 4;  // bytes per stored element
    NE_ALLOC(c->d_C, std::max<uint64_t>(c->c_count, 1) * g.dim * esz / 4);
    NE_CUDA(c, cudaMemsetAsync(c->d_C, 0, c->c_count * g.dim * esz, c->stream));
    // vertex sub-part slots: the ring needs 2k (ping-pong), one GPU k, host staging 3
    const bool staged = g.staging == NE_STAGE_HOST;
    // slots: one GPU k; ring 2k (ping-pong halves); host staging, one GPU: 3
    // (H2D next / train / D2H last); host staging with a ring: 3 sets of w
    // (the window trains in one set, receives into another, the third
    // prefetches the next window / drains the last one)
    const size_t nslots = staged ? (c->world > 1 ? 3 * (size_t)stage_window(c) : std::min<size_t>(3, k))
                                 : (c->world > 1 ? 2 * (size_t)k : k);
    if (!reuse || c->vslot.size() != nslots) c->vslot.assign(nslots, nullptr);
    const size_t slot_bytes = std::max<uint64_t>(c->max_sub_rows, 1) * g.dim * esz;
    if (ipc_ring(c) && !staged) {  // one exportable region for the copy-engine ring
        NE_TRY(ipc_alloc_slots(c, slot_bytes, nslots));
        NE_TRY(ipc_reset_on_load(c));
    } else {
        for (size_t i = 0; i < c->vslot.size(); ++i) NE_ALLOC(c->vslot[i], slot_bytes / 4);
    }
    c->cur = 0;
    if (staged) {
        const size_t bytes = (c->part_bounds[c->rank + 1] - c->part_bounds[c->rank]) * g.dim * esz;
        if (c->h_V_bytes != bytes) {
            if (c->h_V) cudaFreeHost(c->h_V);
            c->h_V = nullptr;
            c->h_V_bytes = 0;
            cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_V), std::max<size_t>(bytes, 16), cudaHostAllocDefault);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return ne_fail(c, NE_ENOMEM, "cudaHostAlloc(%zu) for the host-staged vertex matrix: %s", bytes,
                            cudaGetErrorString(e));
            }
            c->h_V_bytes = bytes;
        }
    }
    for (uint32_t t = 0; t < k; ++t) {
        const size_t vs = (size_t)c->rank * k + t;
        const uint64_t rows = c->sub_bounds[vs + 1] - c->sub_bounds[vs];
        float* slot = staged ? c->vslot[t % c->vslot.size()] : c->vslot[t];
        NE_CUDA(c, ne::launch_init_vertex(slot, c->sub_bounds[vs], rows, g.dim, g.seed,
                                          g.storage == NE_STORE_BF16, c->dev, c->stream));
        c->launches += 1;
        if (staged)  // stream order: the slot is reused only after its copy to the host
            NE_CUDA(c, cudaMemcpyAsync(host_row(c, c->sub_bounds[vs]), slot, rows * g.dim * esz,
                                       cudaMemcpyDeviceToHost, c->stream));
    }

    // Episode buffers: walks, pi-indexed slots, pool, bucketing scratch.
    c->units_total = g.walk_len == 0 ? nnz : (uint64_t)n * g.walks_per_node;
    c->Pw = g.walk_len == 0 ? 1u : (uint32_t)pairs_per_walk(g.walk_len, g.window);
    c->units_max = (c->units_total + g.episodes - 1) / g.episodes;
    c->N_max = c->units_max * c->Pw;
    if (g.walk_len > 0) {
        // a rank of a world > 1 NCCL job walks only its shard (ceil(units / P)
        // rows); one GPU and layout-only ranks walk the whole episode
        const uint64_t wrows = (P > 1 && c->comm) ? (c->units_max + P - 1) / P : c->units_max;
        NE_ALLOC(c->d_walks, std::max<uint64_t>(wrows, 1) * (g.walk_len + 1));
        std::vector<uint32_t> tab_s;
        for (uint32_t i = 0; i < g.walk_len; ++i)
            for (uint32_t dl = 1; dl <= g.window && i + dl <= g.walk_len; ++dl) tab_s.push_back((i << 16) | dl);
        NE_ALLOC(c->d_slot_tab, tab_s.size());
        NE_CUDA(c, cudaMemcpyAsync(c->d_slot_tab, tab_s.data(), tab_s.size() * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, c->stream));
    }
    // per-unit counts / bases; the sharded construction (walks, P > 1) keeps P
    // counts per walker of a shard: P x ceil(units_max / P) entries
    const uint64_t cnt_len = std::max<uint64_t>(
        {c->units_max, (g.walk_len > 0 && P > 1) ? (c->units_max + P - 1) / P * P : 0, 1});
    NE_ALLOC(c->d_counts, cnt_len);
    NE_ALLOC(c->d_base, cnt_len);
    if (!reuse) NE_TRY(dalloc(c, &c->d_scan_scratch, ne::scan_scratch_bytes(cnt_len)));
    NE_ALLOC(c->d_part_bounds, (size_t)P + 1);
    NE_ALLOC(c->d_tmat, (size_t)P * P);
    NE_CUDA(c, cudaMemcpyAsync(c->d_part_bounds, c->part_bounds.data(), (P + 1) * sizeof(uint64_t),
                               cudaMemcpyHostToDevice, c->stream));
    NE_ALLOC(c->d_total, 1);
    // d_slots / d_pool / d_keys: sized by the first episode's pool (ensure_pool)
    if (!reuse) NE_TRY(dalloc(c, &c->d_scratch, ne::bucket_scratch_bytes(c->N_max, nb_local(c))));
    NE_ALLOC(c->d_boff, (size_t)nb_local(c) + 1);
    NE_ALLOC(c->d_boff_alt, (size_t)nb_local(c) + 1);
#undef NE_ALLOC
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    c->loaded = true;
    return NE_OK;
}

int ne_random_walk(ne_ctx* c, uint32_t epoch, uint32_t episode, uint32_t* host_walks,
                   size_t cap_u32, uint64_t* walkers_out) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (c->cfg.walk_len == 0) return ne_fail(c, NE_ESTATE, "LINE mode (walk_len=0) has no walks");
    if (episode >= c->cfg.episodes) return ne_fail(c, NE_ERANGE, "episode=%u >= episodes=%u", episode, c->cfg.episodes);
    if (epoch >= (1u << 24)) return ne_fail(c, NE_ERANGE, "epoch=%u >= 2^24", epoch);
    c->next.valid = false;  // the walk and pair buffers are reused
    NE_TRY(do_walk(c, epoch, episode));
    const uint64_t total = c->walked_units * (c->cfg.walk_len + 1);
    if (walkers_out) *walkers_out = c->walked_units;
    if (host_walks) {
        if (cap_u32 < total) return ne_fail(c, NE_ERANGE, "host_walks capacity %zu < %llu", cap_u32, (unsigned long long)total);
        NE_CUDA(c, cudaMemcpyAsync(host_walks, c->d_walks, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    return NE_OK;
}

int ne_build_samples(ne_ctx* c, uint32_t epoch, uint32_t episode, uint64_t* n_samples_out) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (episode >= c->cfg.episodes) return ne_fail(c, NE_ERANGE, "episode=%u >= episodes=%u", episode, c->cfg.episodes);
    if (epoch >= (1u << 24)) return ne_fail(c, NE_ERANGE, "epoch=%u >= 2^24", epoch);
    if (c->cfg.walk_len > 0 && (c->walked_epoch != (int64_t)epoch || c->walked_episode != (int64_t)episode))
        return ne_fail(c, NE_ESTATE, "no walks for epoch %u episode %u (call ne_random_walk)", epoch, episode);
    c->next.valid = false;
    NE_TRY(do_build(c, epoch, episode));
    if (n_samples_out) *n_samples_out = c->boff.back();
    return NE_OK;
}

int ne_train_samples(ne_ctx* c, uint32_t epoch, uint32_t episode, float lr, ne_stats* stats) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (c->built_episode != (int64_t)episode)
        return ne_fail(c, NE_ESTATE, "no sample pool for episode %u (call ne_build_samples)", episode);
    if (epoch >= (1u << 24)) return ne_fail(c, NE_ERANGE, "epoch=%u >= 2^24", epoch);
    if (stats) std::memset(stats, 0, sizeof *stats);
    const uint32_t l0 = c->launches;
    NE_TRY(do_train(c, epoch, episode, lr, stats));
    if (stats) stats->kernel_launches = c->launches - l0;
    return NE_OK;
}

int ne_train_epoch(ne_ctx* c, uint32_t epoch, float lr, uint32_t flags, ne_stats* stats) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (epoch >= (1u << 24)) return ne_fail(c, NE_ERANGE, "epoch=%u >= 2^24", epoch);
    ne_stats acc;
    std::memset(&acc, 0, sizeof acc);
    const uint32_t l0 = c->launches;
    if (c->export_V) {
        const uint64_t need = (c->part_bounds[c->rank + 1] - c->part_bounds[c->rank]) * c->cfg.dim;
        if (c->export_cap < need)
            return ne_fail(c, NE_ERANGE, "export buffer %zu floats < %llu (part rows x d)", c->export_cap,
                           (unsigned long long)need);
    }
    // the vertex export (ne_export_vertex_on_train) rides on the call's last episode
    struct ExportGuard {  // also on an error return: no copy into the caller's rows left in flight
        ne_ctx* c;
        ~ExportGuard() {
            if (c->export_now) cudaStreamSynchronize(c->d2h_stream);
            c->export_now = false;
        }
    } export_guard{c};
    if (flags & NE_REUSE_SAMPLES) {
        if (c->cfg.episodes != 1 || c->built_episode != 0)
            return ne_fail(c, NE_ESTATE, "NE_REUSE_SAMPLES needs episodes == 1 and a built pool");
        c->next.valid = false;
        c->export_now = c->export_V != nullptr;
        NE_TRY(do_train(c, epoch, 0, lr, &acc));
    } else {
        // Walk engine decoupled from training ("we run our walk engine for
        // the next epoch while embedding training engine trains samples for this
        // epoch"): while episode e trains on the compute stream, the walk + pool
        // of the next episode -- (epoch, e+1), or (epoch+1, 0) after the last one,
        // kept for the next call -- are built on build_stream into the pair
        // buffers the training pool does not occupy.  Needs the third pair
        // buffer (ensure_pool); without it every build is serial.
        static const int build_reserve = [] {  // SMs the SGNS grid leaves to a concurrent build
            const char* e = std::getenv("NE_BUILD_RESERVE_SMS");
            return e ? std::max(0, std::atoi(e)) : 0;
        }();
        const uint32_t E = c->cfg.episodes;
        for (uint32_t e = 0; e < E; ++e) {
            cudaEvent_t w0 = next_event(c), w1 = next_event(c);
            NE_CUDA(c, cudaEventRecord(w0, c->stream));
            if (c->next.valid && c->next.epoch == (int64_t)epoch && c->next.episode == (int64_t)e) {
                acc.ms_walk += c->next.ms_walk;
                acc.ms_build += c->next.ms_build;
                adopt_next(c);
            } else {
                c->next.valid = false;
                float mw = 0.f, mb = 0.f;
                NE_TRY(walk_build(c, epoch, e, c->stream, &mw, &mb));
                acc.ms_walk += mw;
                acc.ms_build += mb;
            }
            if (flags & NE_CHECK_BLOCKS) NE_TRY(ne_check_pool(c));
            NE_CUDA(c, cudaEventRecord(w1, c->stream));
            const bool more = e + 1 < E || epoch + 1 < (1u << 24);
            const bool pre = more && pipelined(c);
            TrainPending tp;
            c->sgns_reserve = pre ? build_reserve : 0;
            c->export_now = c->export_V != nullptr && e + 1 == E;
            int rc = launch_train(c, epoch, e, lr, tp);
            c->sgns_reserve = 0;
            if (rc == NE_OK && pre) rc = prebuild_next(c, e + 1 < E ? epoch : epoch + 1, e + 1 < E ? e + 1 : 0);
            const int rf = finish_train(c, tp, &acc);
            NE_TRY(rc);
            NE_TRY(rf);
            float gap = 0.f;
            NE_CUDA(c, cudaEventElapsedTime(&gap, w0, w1));
            acc.ms_pool_wait += gap;
            c->ev_used = 0;
        }
    }
    if (c->export_V) NE_CUDA(c, cudaStreamSynchronize(c->d2h_stream));  // host rows complete on return
    acc.kernel_launches = c->launches - l0;
    if (stats) *stats = acc;
    return NE_OK;
}

int ne_export_vertex_on_train(ne_ctx* c, float* host_rows, size_t cap_floats) {
    NE_TRY(enter(c));
    if (!host_rows) {
        c->export_V = nullptr;
        c->export_cap = 0;
        return NE_OK;
    }
    if (c->world > 1 && !c->comm && !ipc_ring(c))
        return ne_fail(c, NE_EINVAL, "vertex export during training needs a ring (NCCL or IPC; layout-only context)");
    if (c->cfg.storage != NE_STORE_F32) return ne_fail(c, NE_EINVAL, "vertex export during training needs fp32 rows");
    if (c->cfg.staging != NE_STAGE_DEVICE) return ne_fail(c, NE_EINVAL, "vertex export during training needs device staging");
    if (c->loaded) {
        const uint64_t need = (c->part_bounds[c->rank + 1] - c->part_bounds[c->rank]) * c->cfg.dim;
        if (cap_floats < need)
            return ne_fail(c, NE_ERANGE, "export buffer %zu floats < %llu (part rows x d)", cap_floats,
                           (unsigned long long)need);
    }
    c->export_V = host_rows;
    c->export_cap = cap_floats;
    return NE_OK;
}

static int rows_op(ne_ctx* c, int which, uint32_t row_begin, uint32_t row_end, float* host,
                   const float* in, size_t cap_floats) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (which != NE_VERTEX && which != NE_CONTEXT) return ne_fail(c, NE_EINVAL, "which=%d", which);
    const uint64_t pb = c->part_bounds[c->rank], pe = c->part_bounds[c->rank + 1];
    if (row_begin > row_end || row_begin < pb || row_end > pe)
        return ne_fail(c, NE_ERANGE, "rows [%u, %u) not in this rank's part [%llu, %llu)", row_begin, row_end,
                    (unsigned long long)pb, (unsigned long long)pe);
    const uint64_t d = c->cfg.dim;
    if (host && cap_floats < (uint64_t)(row_end - row_begin) * d)
        return ne_fail(c, NE_ERANGE, "capacity %zu < %llu floats", cap_floats,
                    (unsigned long long)((row_end - row_begin) * d));
    NE_TRY(ipc_drain(c, true));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->comm_stream));
    const bool bf = c->cfg.storage == NE_STORE_BF16;
    auto copy = [&](float* dev_base, uint64_t base_row, uint64_t a, uint64_t b) -> int {
        if (a >= b) return NE_OK;
        const size_t off = (a - row_begin) * d, count = (b - a) * d;
        if (!bf) {  // on the compute stream, then synchronised: ordered after training, complete on return
            float* dptr = dev_base + (a - base_row) * d;
            if (host) NE_CUDA(c, cudaMemcpyAsync(host + off, dptr, count * sizeof(float), cudaMemcpyDefault, c->stream));
            else NE_CUDA(c, cudaMemcpyAsync(dptr, in + off, count * sizeof(float), cudaMemcpyDefault, c->stream));
            NE_CUDA(c, cudaStreamSynchronize(c->stream));
            return NE_OK;
        }
        // bf16 rows: convert through an fp32 device buffer (exact widening / nearest-even rounding)
        uint16_t* dptr = reinterpret_cast<uint16_t*>(dev_base) + (a - base_row) * d;
        if (c->tmp_f32_cap < count) {
            if (c->d_tmp_f32) dfree(c, c->d_tmp_f32);
            c->d_tmp_f32 = nullptr;
            c->tmp_f32_cap = 0;
            NE_TRY(dalloc_t(c, &c->d_tmp_f32, count));
            c->tmp_f32_cap = count;
        }
        if (host) {
            NE_CUDA(c, ne::launch_convert_rows(dptr, c->d_tmp_f32, count, false, c->dev, c->stream));
            NE_CUDA(c, cudaMemcpyAsync(host + off, c->d_tmp_f32, count * sizeof(float), cudaMemcpyDefault,
                                       c->stream));
        } else {
            NE_CUDA(c, cudaMemcpyAsync(c->d_tmp_f32, in + off, count * sizeof(float), cudaMemcpyDefault,
                                       c->stream));
            NE_CUDA(c, ne::launch_convert_rows(c->d_tmp_f32, dptr, count, true, c->dev, c->stream));
        }
        c->launches += 1;
        NE_CUDA(c, cudaStreamSynchronize(c->stream));
        return NE_OK;
    };
    if (which == NE_CONTEXT) return copy(c->d_C, c->c_begin, row_begin, row_end);
    if (c->cfg.staging == NE_STAGE_HOST) {
        NE_CUDA(c, cudaStreamSynchronize(c->copy_stream));
        NE_CUDA(c, cudaStreamSynchronize(c->d2h_stream));
        c->stage_pending = c->stage_pre = false;
        // pinned host rows (device-accessible under UVA: the bf16 conversion kernel reads them in place)
        return copy(static_cast<float*>(host_row(c, row_begin)), row_begin, row_begin, row_end);
    }
    const uint32_t k = c->cfg.subparts;
    for (uint32_t t = 0; t < k; ++t) {
        const size_t vs = (size_t)c->rank * k + t;
        const uint64_t sb = c->sub_bounds[vs], se = c->sub_bounds[vs + 1];
        NE_TRY(copy(c->vslot[c->cur * k + t], sb, std::max<uint64_t>(sb, row_begin),
                    std::min<uint64_t>(se, row_end)));
    }
    return NE_OK;
}

int ne_get_embeddings(ne_ctx* c, int which, uint32_t row_begin, uint32_t row_end, float* host_out,
                      size_t cap_floats) {
    if (!host_out) return c ? ne_fail(c, NE_EINVAL, "null output") : NE_EINVAL;
    return rows_op(c, which, row_begin, row_end, host_out, nullptr, cap_floats);
}

int ne_set_embeddings(ne_ctx* c, int which, uint32_t row_begin, uint32_t row_end, const float* in) {
    if (!in) return c ? ne_fail(c, NE_EINVAL, "null input") : NE_EINVAL;
    return rows_op(c, which, row_begin, row_end, nullptr, in, 0);
}

int ne_export_samples(ne_ctx* c, uint32_t vsub, uint32_t* pairs_out, size_t cap_pairs, uint64_t* count) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (c->built_episode < 0) return ne_fail(c, NE_ESTATE, "no sample pool built");
    if (vsub >= nb_local(c)) return ne_fail(c, NE_ERANGE, "vsub=%u >= %u", vsub, nb_local(c));
    const uint64_t cnt = c->boff[vsub + 1] - c->boff[vsub];
    if (count) *count = cnt;
    if (!pairs_out) return NE_OK;
    if (cap_pairs < cnt) return ne_fail(c, NE_ERANGE, "capacity %zu < %llu pairs", cap_pairs, (unsigned long long)cnt);
    if (cnt) NE_CUDA(c, cudaMemcpy(pairs_out, c->pool_at + c->boff[vsub], cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return NE_OK;
}

int ne_export_negatives(ne_ctx* c, uint32_t epoch, uint32_t episode, uint32_t vsub, uint64_t pos_begin,
                        uint64_t count, uint32_t* out) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (vsub >= nb_local(c)) return ne_fail(c, NE_ERANGE, "vsub=%u >= %u", vsub, nb_local(c));
    if (!out && count) return ne_fail(c, NE_EINVAL, "null output");
    const uint64_t total = count * c->cfg.negatives;
    if (total == 0) return NE_OK;
    NE_TRY(wait_alias(c));
    if (c->tmp_u32_cap < total) {
        if (c->d_tmp_u32) dfree(c, c->d_tmp_u32);
        c->d_tmp_u32 = nullptr;
        c->tmp_u32_cap = 0;
        NE_TRY(dalloc_t(c, &c->d_tmp_u32, total));
        c->tmp_u32_cap = total;
    }
    ne::SgnsParams p{};
    p.c_begin = c->c_begin;
    p.c_count = c->c_count;
    p.alias = c->d_alias;
    p.K = c->cfg.negatives;
    p.seed = c->cfg.seed;
    p.epoch = epoch;
    p.episode = episode;
    p.block = vsub * (uint32_t)c->world + (uint32_t)c->rank;
    NE_CUDA(c, ne::launch_export_negatives(p, pos_begin, count, c->d_tmp_u32, c->dev, c->stream));
    c->launches += 1;
    NE_CUDA(c, cudaMemcpyAsync(out, c->d_tmp_u32, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    return NE_OK;
}

int ne_capture_block(ne_ctx* c, uint32_t epoch, uint32_t episode, uint32_t vsub, float lr, uint32_t* out,
                     size_t cap_u32, uint64_t* count) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (c->built_episode != (int64_t)episode || c->built_epoch != (int64_t)epoch)
        return ne_fail(c, NE_ESTATE, "no sample pool for epoch %u episode %u", epoch, episode);
    if (c->cfg.staging == NE_STAGE_HOST) return ne_fail(c, NE_ESTATE, "capture needs the vertex matrix in HBM");
    const uint32_t k = c->cfg.subparts, home = (uint32_t)c->rank * k;
    if (vsub < home || vsub >= home + k)
        return ne_fail(c, NE_ERANGE, "vsub=%u is not a home sub-part of rank %d ([%u, %u))", vsub, c->rank, home, home + k);
    NE_TRY(wait_alias(c));
    NE_TRY(ipc_drain(c, true));
    NE_CUDA(c, cudaStreamSynchronize(c->comm_stream));
    c->ring_pending = false;
    ne::SgnsParams sp = sgns_params(c, vsub, c->vslot[c->cur * k + (vsub - home)], epoch, episode, lr);
    const uint64_t per = 2ull + c->cfg.negatives, total = sp.count * per;
    if (count) *count = sp.count;
    if (!out) return NE_OK;
    if (cap_u32 < total) return ne_fail(c, NE_ERANGE, "capacity %zu < %llu", cap_u32, (unsigned long long)total);
    if (total == 0) return NE_OK;
    if (c->tmp_u32_cap < total) {
        if (c->d_tmp_u32) dfree(c, c->d_tmp_u32);
        c->d_tmp_u32 = nullptr;
        c->tmp_u32_cap = 0;
        NE_TRY(dalloc_t(c, &c->d_tmp_u32, total));
        c->tmp_u32_cap = total;
    }
    NE_CUDA(c, cudaMemsetAsync(c->d_tmp_u32, 0xFF, total * sizeof(uint32_t), c->stream));
    sp.deterministic = 0;
    sp.capture = c->d_tmp_u32;
    NE_CUDA(c, ne::launch_sgns(sp, c->dev, c->stream));
    c->launches += 1;
    NE_CUDA(c, cudaMemcpyAsync(out, c->d_tmp_u32, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    return NE_OK;
}

int ne_umma_products(const float* V, const float* N, const float* G, float* S, float* dV, float* dNt) {
    if (!V || !N || !G || !S || !dV || !dNt) return NE_EINVAL;
    float* d = nullptr;
    const size_t nV = 128 * 128, nN = 32 * 128, nG = 128 * 32, nS = 128 * 32, ndV = 128 * 128, ndN = 128 * 32;
    if (cudaMalloc(&d, (nV + nN + nG + nS + ndV + ndN) * sizeof(float)) != cudaSuccess) return NE_ECUDA;
    float *dV_in = d, *dN_in = dV_in + nV, *dG_in = dN_in + nN, *dS = dG_in + nG, *ddV = dS + nS, *ddN = ddV + ndV;
    int rc = NE_OK;
    if (cudaMemcpy(dV_in, V, nV * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dN_in, N, nN * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dG_in, G, nG * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        ne::launch_umma_products(dV_in, dN_in, dG_in, dS, ddV, ddN, 0) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(S, dS, nS * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(dV, ddV, ndV * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(dNt, ddN, ndN * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = NE_ECUDA;
    cudaGetLastError();
    cudaFree(d);
    return rc;
}

int ne_umma_raw(const void* a_img, const void* b_img, uint32_t img_bytes, uint64_t a_hi, uint64_t b_hi,
                uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo, uint32_t a_step, uint32_t b_step,
                uint32_t ksteps, uint32_t idesc, uint32_t N, float* D) {
    void* d = nullptr;
    const size_t out = 128ull * N * sizeof(float);
    if (cudaMalloc(&d, 2ull * img_bytes + out) != cudaSuccess) return NE_ECUDA;
    char* base = static_cast<char*>(d);
    int rc = NE_OK;
    if (cudaMemcpy(base, a_img, img_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(base + img_bytes, b_img, img_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        ne::launch_umma_raw(base, base + img_bytes, img_bytes, a_hi, b_hi, a_lbo, a_sbo, b_lbo, b_sbo, a_step, b_step,
                            ksteps, idesc, N, reinterpret_cast<float*>(base + 2ull * img_bytes), 0) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(D, base + 2ull * img_bytes, out, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = NE_ECUDA;
    cudaGetLastError();
    cudaFree(d);
    return rc;
}

int ne_train_samples_local_ring(ne_ctx* const* ctxs, uint32_t world, uint32_t epoch,
                                uint32_t episode, float lr, ne_stats* stats) {
    if (!ctxs || world == 0) return NE_EINVAL;
    ne_ctx* c0 = ctxs[0];
    NE_TRY(enter(c0));
    const uint32_t k = c0->cfg.subparts;
    for (uint32_t g = 0; g < world; ++g) {
        ne_ctx* c = ctxs[g];
        if (!c || !c->loaded || c->comm || c->world != (int)world || c->rank != (int)g ||
            c->device != c0->device || c->cfg.subparts != k || c->cfg.dim != c0->cfg.dim)
            return ne_fail(c0, NE_EINVAL, "context %u is not layout-only rank %u of %u on device %d", g, g, world,
                        c0->device);
        if (c->built_episode != (int64_t)episode)
            return ne_fail(c0, NE_ESTATE, "context %u has no pool for episode %u", g, episode);
    }
    for (uint32_t g = 0; g < world; ++g) NE_TRY(wait_alias(ctxs[g]));
    if (stats) std::memset(stats, 0, sizeof *stats);
    NE_CUDA(c0, cudaMemsetAsync(c0->d_loss, 0, sizeof(double), c0->stream));
    // Every rank's launches go to rank 0's stream, in plan order: round r, slot t,
    // rank g; the "send to g+1" is a pointer hand-over of the trained slot.
    std::vector<float*> moved(world);
    const uint32_t G = groups_of(c0);
    if (c0->cfg.staging == NE_STAGE_HOST) {  // NEXT-2 staged ring, windows of w slots (launch_train_staged_ring)
        const uint32_t w = stage_window(c0);
        const uint64_t d = c0->cfg.dim, esz = elem_bytes(c0);
        for (uint32_t t0 = 0; t0 < k; t0 += w) {
            const uint32_t wn = std::min(w, k - t0);
            for (uint32_t g = 0; g < world; ++g)
                for (uint32_t t = 0; t < wn; ++t) {  // stage 5: home sub-parts to the device
                    ne_ctx* c = ctxs[g];
                    const uint64_t vs = (uint64_t)g * k + t0 + t, sb = c->sub_bounds[vs];
                    NE_CUDA(c0, cudaMemcpyAsync(c->vslot[t], host_row(c, sb), (c->sub_bounds[vs + 1] - sb) * d * esz,
                                                cudaMemcpyHostToDevice, c0->stream));
                }
            for (uint32_t r = 0; r < world; ++r)
                for (uint32_t t = 0; t < wn; ++t) {
                    for (uint32_t g = 0; g < world; ++g) {
                        ne_ctx* c = ctxs[g];
                        ne::SgnsParams sp = sgns_params(c, (uint32_t)plan_vsub(world, G, k, r, t0 + t, g), c->vslot[t],
                                                        epoch, episode, lr);
                        sp.loss = c0->d_loss;
                        NE_CUDA(c0, ne::launch_sgns(sp, c->dev, c0->stream));
                        if (stats) { stats->samples += sp.count; if (sp.count) stats->train_launches += 1; }
                    }
                    for (uint32_t g = 0; g < world; ++g) moved[ring_dest(world, G, r, g)] = ctxs[g]->vslot[t];
                    for (uint32_t g = 0; g < world; ++g) ctxs[g]->vslot[t] = moved[g];
                }
            for (uint32_t g = 0; g < world; ++g)
                for (uint32_t t = 0; t < wn; ++t) {  // stage 2: home again, back to the host
                    ne_ctx* c = ctxs[g];
                    const uint64_t vs = (uint64_t)g * k + t0 + t, sb = c->sub_bounds[vs];
                    NE_CUDA(c0, cudaMemcpyAsync(host_row(c, sb), c->vslot[t], (c->sub_bounds[vs + 1] - sb) * d * esz,
                                                cudaMemcpyDeviceToHost, c0->stream));
                }
        }
    } else
    for (uint32_t r = 0; r < world; ++r)
        for (uint32_t t = 0; t < k; ++t) {
            for (uint32_t g = 0; g < world; ++g) {
                ne_ctx* c = ctxs[g];
                const uint32_t vs = (uint32_t)plan_vsub(world, G, k, r, t, g);
                ne::SgnsParams sp = sgns_params(c, vs, c->vslot[c->cur * k + t], epoch, episode, lr);
                sp.loss = c0->d_loss;
                NE_CUDA(c0, ne::launch_sgns(sp, c->dev, c0->stream));
                if (stats) { stats->samples += sp.count; if (sp.count) stats->train_launches += 1; }
            }
            for (uint32_t g = 0; g < world; ++g) moved[ring_dest(world, G, r, g)] = ctxs[g]->vslot[ctxs[g]->cur * k + t];
            for (uint32_t g = 0; g < world; ++g) ctxs[g]->vslot[ctxs[g]->cur * k + t] = moved[g];
        }
    double loss = 0.0;
    NE_CUDA(c0, cudaMemcpyAsync(&loss, c0->d_loss, sizeof(double), cudaMemcpyDeviceToHost, c0->stream));
    NE_CUDA(c0, cudaStreamSynchronize(c0->stream));
    if (stats) { stats->loss_sum = loss; stats->kernel_launches = stats->train_launches; }
    return NE_OK;
}

int ne_check_pool(ne_ctx* c) {
    NE_TRY(enter(c));
    NE_TRY(check_loaded(c));
    if (c->built_episode < 0) return ne_fail(c, NE_ESTATE, "no sample pool built");
    NE_CUDA(c, cudaMemsetAsync(c->d_bad, 0xFF, sizeof(unsigned long long), c->stream));
    NE_CUDA(c, ne::launch_check_pool(c->pool_at, c->d_boff, c->boff.back(), c->d_sub_bounds, nb_local(c),
                                     c->c_begin, c->c_begin + c->c_count, c->d_bad, c->dev, c->stream));
    c->launches += 1;
    unsigned long long bad = 0;
    NE_CUDA(c, cudaMemcpyAsync(&bad, c->d_bad, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    if (bad == ~0ull) return NE_OK;
    uint64_t rec = 0;
    NE_CUDA(c, cudaMemcpy(&rec, c->pool_at + bad, sizeof rec, cudaMemcpyDeviceToHost));
    const uint32_t b = (uint32_t)(std::upper_bound(c->boff.begin(), c->boff.end(), (uint64_t)bad) - c->boff.begin() - 1);
    return ne_fail(c, NE_ESCHED, "pool[%llu] = (%u, %u) outside block (vertex sub-part %u = [%llu, %llu), context part [%llu, %llu))",
                bad, (uint32_t)rec, (uint32_t)(rec >> 32), b, (unsigned long long)c->sub_bounds[b],
                (unsigned long long)c->sub_bounds[b + 1], (unsigned long long)c->c_begin,
                (unsigned long long)(c->c_begin + c->c_count));
}

const char* ne_last_error(const ne_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

void ne_destroy(ne_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    ipc_drain(c, true);
    free_all(c);
    ipc_release(c);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->ring_done) cudaEventDestroy(c->ring_done);
    if (c->stage_done) cudaEventDestroy(c->stage_done);
    if (c->stage_pre_ev) cudaEventDestroy(c->stage_pre_ev);
    if (c->h_V) cudaFreeHost(c->h_V);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    if (c->build_stream) cudaStreamDestroy(c->build_stream);
    if (c->comm_walk) ncclCommDestroy(c->comm_walk);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->d_loss) cudaFree(c->d_loss);
    if (c->d_bad) cudaFree(c->d_bad);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    delete c;
}

}  // extern "C"

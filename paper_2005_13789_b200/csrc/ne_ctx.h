// ne_ctx.h -- the context behind the opaque ne_ctx handle of include/ne.h,
// shared by the runtime translation units (runtime.cpp, ring_ipc.cpp).  Not
// part of the ABI.
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "ne.h"
#include "ne_internal.h"

struct ne_ctx {
    ne_config cfg{};
    int device = 0;
    ne::Device dev;
    cudaStream_t own_stream = nullptr, stream = nullptr, comm_stream = nullptr;
    cudaStream_t build_stream = nullptr;  // walk + pool build of the next episode, behind training
    cudaStream_t ws = nullptr;            // the stream walk / build kernels go to: stream, or build_stream
                                          // while a pipelined build runs
    ne_alloc_fn alloc = nullptr;
    ne_free_fn free_fn = nullptr;
    void* user = nullptr;
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    ncclComm_t comm_walk = nullptr;  // split of comm for the walk all-gather: NCCL serialises the
                                     // operations of one communicator, and the ring's last
                                     // return-home transfers would otherwise delay the next walk
    std::string err;

    struct Alloc { void* p; size_t bytes; };
    std::vector<Alloc> allocs;

    bool loaded = false;
    uint64_t n = 0, nnz = 0;
    uint64_t* d_off = nullptr;
    uint32_t* d_tgt = nullptr;
    std::vector<uint64_t> part_bounds, sub_bounds;
    uint64_t* d_sub_bounds = nullptr;
    uint2* d_alias = nullptr;
    float* d_C = nullptr;
    uint64_t c_begin = 0, c_count = 0;
    std::vector<float*> vslot;  // ring: 2k buffers (ping-pong); one GPU: k; host staging: 3
    float* h_V = nullptr;       // host staging: this rank's vertex rows, pinned
    size_t h_V_bytes = 0;
    cudaStream_t copy_stream = nullptr;  // host staging H2D (one GPU: D2H uses comm_stream)
    cudaStream_t d2h_stream = nullptr;   // host staging with the ring: D2H, off the ring's comm stream
    float* export_V = nullptr;           // ne_export_vertex_on_train: host rows of this rank's part
    size_t export_cap = 0;
    bool export_now = false;             // this episode is the call's last: copy sub-parts out
    cudaEvent_t stage_done = nullptr;    // last D2H of a call (deferred like ring_done)
    bool stage_pending = false;
    cudaEvent_t stage_pre_ev = nullptr;  // one GPU: the next episode's sub-part 0, prefetched into slot 0
    bool stage_pre = false;
    uint32_t stage_base = 0;             // one GPU: sub-part t of this episode uses slot (t + base) % 3
    uint32_t stage_pre_set = 0;          // with the ring: the slot set holding the prefetched window 0
    uint32_t stage_drain_set = 1;        // (stage_pre), and the set the last window's rows drain from
    int cur = 0;                // half [cur*k, cur*k+k) holds the current sub-parts
    uint64_t max_sub_rows = 0;

    uint32_t Pw = 1;
    uint64_t units_total = 0, units_max = 0, N_max = 0;
    uint32_t* d_walks = nullptr;
    uint32_t* d_slot_tab = nullptr;
    std::vector<uint64_t*> pbufs;  // 2 pair buffers, or 3 when the next episode's pool is built during training
    uint64_t* d_slots = nullptr;   // the two pbufs a build uses (sink / radix ping-pong)
    uint32_t* d_keys[2] = {nullptr, nullptr};  // keyed pool sink + radix ping-pong (nullptr: direct sink)
    uint64_t* d_pool = nullptr;
    uint64_t* pool_at = nullptr;  // the buffer (d_pool or d_slots) holding the built pool
    bool walk_counts = false;     // d_counts holds the O5 counts of the current walk (unsharded walk)
    uint64_t shard_units = 0;     // world > 1 with NCCL: walkers of this rank's shard in d_walks (from row 0)
    uint64_t* d_part_bounds = nullptr;  // P + 1 context-part bounds (sharded construction)
    uint64_t* d_tmat = nullptr;         // P x P (shard, part) pair counts of the episode (sharded construction)
    std::vector<uint64_t> tmat;
    uint64_t pool_cap = 0;        // pairs d_slots / d_pool (and d_keys) hold; grown by ensure_pool
    float* d_tmp_f32 = nullptr;   // bf16 rows: fp32 staging of ne_get/set_embeddings
    uint64_t tmp_f32_cap = 0;
    void* d_scratch = nullptr;
    uint32_t* d_counts = nullptr;   // per-unit kept-pair counts (O5)
    uint64_t* d_base = nullptr;     // their exclusive scan: part-local index bases
    void* d_scan_scratch = nullptr;
    uint64_t* d_total = nullptr;    // N_g of the episode
    uint64_t* d_boff = nullptr;
    std::vector<uint64_t> boff;
    // the next episode's pool, built on build_stream while the current one trains
    struct NextPool {
        bool valid = false;
        uint64_t* at = nullptr;
        uint64_t* d_boff = nullptr;
        std::vector<uint64_t> boff;
        int64_t epoch = -1, episode = -1;
        float ms_walk = 0.f, ms_build = 0.f;
    } next;
    uint64_t* d_boff_alt = nullptr;
    const uint64_t* keep_pool = nullptr;  // pool in training while a build runs (select_scratch skips it)
    int sgns_reserve = 0;                 // SMs the SGNS grid leaves free (concurrent pool build)
    uint64_t pool_gen = 0;                // bumped whenever ensure_pool reallocates the pair buffers
    double* d_loss = nullptr;
    unsigned long long* d_bad = nullptr;
    bool n2v = false;           // node2vec walks (p, q != 1)
    uint64_t n2v_thr[3] = {0, 0, 0};
    uint32_t* d_tmp_u32 = nullptr;
    size_t tmp_u32_cap = 0;

    int64_t walked_epoch = -1, walked_episode = -1;
    int64_t built_epoch = -1, built_episode = -1;
    uint64_t walked_units = 0;

    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    // recorded on the comm stream after the last ring transfers of a call (the
    // "return home" sends, still in flight when ne_train_samples returns); the
    // next call's first training of every slot waits on it
    cudaEvent_t ring_done = nullptr;
    bool ring_pending = false;
    uint32_t launches = 0;
    std::shared_ptr<void> alias_scratch;  // host buffers reused across ne_load_graph calls
    std::vector<uint2> alias_host;
    std::vector<uint64_t> alias_deg;      // context-part degrees the alias builder reads
    std::thread alias_thread;             // host alias build, overlapped with walk + pool build
    bool alias_pending = false;

    // ---- copy-engine ring over CUDA IPC (cfg.transport == NE_TRANSPORT_IPC; ring_ipc.cpp)
    struct Ipc {
        void* region = nullptr;          // this rank's 2k vertex slots + flags, one exportable cudaMalloc
        size_t region_bytes = 0, slot_bytes = 0;
        uint32_t* flags = nullptr;       // arrived[2][k], credit[2][k] (per hop kind; ring_ipc.cpp)
        std::vector<void*> peer;         // regions of the ranks this one pushes to / credits, opened handles
        bool connected = false;
        std::string blobs;               // the handles the open peers came from (a reload reuses them)
        bool started = false;            // a ring call ran since the last load (arrivals to wait for)
        std::vector<uint32_t> pushed[2], waited[2];  // per hop kind and slot: pushes issued / arrivals awaited
    } ipc;
};

// NEXT-3 ring hops (P = G * L ranks, rank g = a * L + j): after global round
// rho a sub-part moves along the group's ring to (a, j + 1), except after the
// group's last rotation, when it crosses to the next group, (a + 1, j + 1).
inline uint32_t ring_dest(uint32_t P, uint32_t G, uint32_t rho, uint32_t g) {
    const uint32_t L = P / G, a = g / L, j = g % L;
    const uint32_t na = (rho % L) + 1 < L ? a : (a + 1) % G;
    return na * L + (j + 1) % L;
}
// The rank whose ring_dest after round rho is g.
inline uint32_t ring_src(uint32_t P, uint32_t G, uint32_t rho, uint32_t g) {
    const uint32_t L = P / G, a = g / L, j = g % L;
    const uint32_t pa = (rho % L) + 1 < L ? a : (a + G - 1) % G;
    return pa * L + (j + L - 1) % L;
}

// Copy-engine ring over CUDA IPC (ring_ipc.cpp).
bool ipc_ring(const ne_ctx* c);                      // world > 1 and transport == NE_TRANSPORT_IPC
int ipc_alloc_slots(ne_ctx* c, size_t slot_bytes, size_t nslots);  // the 2k vertex slots, exportable
int ipc_reset_on_load(ne_ctx* c);                    // home sub-parts re-initialised: no arrivals owed
// hop kind after global round rho: 0 = along the group's ring, 1 = to the next group
inline uint32_t ring_kind(uint32_t P, uint32_t G, uint32_t rho) {
    const uint32_t L = P / G;
    return (rho % P) % L + 1 < L ? 0u : 1u;
}
int ipc_wait_arrival(ne_ctx* c, uint32_t t, uint32_t kind);  // compute stream waits for slot t's sub-part
// push slot t's sub-part into rank `dest` (a hop of `kind`); `credit_to` = the
// rank that pushes into this one next round, with a hop of `next_kind`
int ipc_push(ne_ctx* c, uint32_t t, const void* src, size_t bytes, cudaEvent_t after, uint32_t kind, uint32_t dest,
             uint32_t credit_to, uint32_t next_kind);
int ipc_drain(ne_ctx* c, bool host_sync);            // every push into / out of this rank has landed
int ipc_wait_home(ne_ctx* c, cudaStream_t s, uint32_t t, uint32_t kind);  // s waits for the last round's push into t
void ipc_release(ne_ctx* c);

// NVTX range for profilers (nsys / ncu --nvtx): walk, build, train, ring phases.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Sets ctx->err to "NE_<CODE>: <message>" and returns code.
int ne_fail(ne_ctx* c, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));

#define NE_CUDA(ctx, call)                                                                  \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return ne_fail(ctx, NE_ECUDA, "%s (%s:%d %s)", cudaGetErrorString(e_), __FILE__,   \
                        __LINE__, #call);                                                   \
    } while (0)

#define NE_NCCL(ctx, call)                                                                  \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return ne_fail(ctx, NE_ENCCL, "%s (%s:%d)", ncclGetErrorString(r_), __FILE__, __LINE__); \
    } while (0)

#define NE_TRY(expr)            \
    do {                        \
        int rc_ = (expr);       \
        if (rc_ != NE_OK) return rc_; \
    } while (0)

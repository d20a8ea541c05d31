/*
 * ne.h -- C ABI of the B200-native SGNS node-embedding training engine.
 *
 * Implements the hot path of Wei et al., "A Distributed Multi-GPU System for
 * Large-Scale Node Embedding at Tencent" (arXiv 2005.13789): network
 * augmentation by random walks (Alg. 1), SGNS SGD with K
 * negatives per positive sample (Alg. 1 lines 8-12), applied block by
 * block to 2D-partitioned vertex / context embedding matrices
 * with vertex sub-parts rotating around a ring of GPUs.
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; R#/O#/D# = the
 * contract and readings listed in DESIGN.md.
 *
 * Conventions (every entry point):
 *   - returns an NE_* status; no C++ exception crosses the ABI;
 *   - ne_last_error(ctx) then holds one machine-parsable line
 *     ("NE_EINVAL: offsets[17]=5 < offsets[16]=9"), cf. S:564;
 *   - input arrays are BORROWED for the duration of the call (copied);
 *     they may be host (pageable or pinned) or device pointers (UVA);
 *   - output arrays are caller-owned; capacities are checked (NE_ERANGE);
 *   - all device memory is owned by the ctx (allocated through the optional
 *     allocator callbacks, else cudaMalloc) and released by ne_destroy;
 *   - a ctx is bound to one CUDA device and one rank; it is NOT thread-safe;
 *   - calls are host-synchronous with respect to their results: when a call
 *     returns, every output it produced is complete.
 * There is no CPU fallback: without a CUDA device ne_create fails (NE_ECUDA).
 */
#ifndef NE_H
#define NE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NE_ABI_VERSION 2

typedef struct ne_ctx ne_ctx;

/* Status codes. */
enum {
    NE_OK = 0,
    NE_EINVAL = -1,  /* bad argument or malformed graph (S:24 CSR invariants)      */
    NE_ERANGE = -2,  /* size/capacity/id out of range, rows not owned by the rank   */
    NE_ENOMEM = -3,  /* device allocation failed                                    */
    NE_ESTATE = -4,  /* call out of order (train before load, export before build)  */
    NE_ECUDA = -5,   /* CUDA runtime error (no device, launch failure, ...)         */
    NE_ENCCL = -6,   /* NCCL error in the ring exchange                             */
    NE_ESCHED = -7   /* schedule violation: a sample outside its 2D block   */
};

/* ne_train_epoch flags. */
enum {
    NE_REUSE_SAMPLES = 1u, /* train again on the pool built earlier instead of
                              walking anew (walk reuse); needs episodes == 1 */
    NE_CHECK_BLOCKS = 2u   /* verify every pool after it is built (ne_check_pool)   */
};

/* ne_config.writeback */
enum { NE_WB_ATOMIC_DELTA = 0, NE_WB_STORE = 1 };

/* ne_config.update_rule */
enum { NE_UPDATE_SEQUENTIAL = 0, NE_UPDATE_ACCUMULATED = 1, NE_UPDATE_SHARED_BATCH = 2 };

/* ne_config.staging */
enum { NE_STAGE_DEVICE = 0, NE_STAGE_HOST = 1 };

/* ne_config.transport: how vertex sub-parts travel the ring (world > 1) */
enum { NE_TRANSPORT_NCCL = 0, NE_TRANSPORT_IPC = 1 };

/* ne_config.storage */
enum { NE_STORE_F32 = 0, NE_STORE_BF16 = 1 };

/* ne_get_embeddings / ne_set_embeddings: which matrix. */
enum { NE_VERTEX = 0, NE_CONTEXT = 1 };

/* Optional device allocator (e.g. PyTorch's caching allocator).  alloc returns
 * a device pointer of at least `bytes` bytes on `device`, usable on `stream`,
 * or NULL on failure.  free releases a pointer alloc returned. */
typedef void *(*ne_alloc_fn)(size_t bytes, int device, void *stream, void *user);
typedef void (*ne_free_fn)(void *ptr, size_t bytes, int device, void *stream, void *user);

/* Training configuration (SPEC RunConfig).  Limits are checked by
 * ne_create (NE_EINVAL): dim % 4 == 0 and 4 <= dim <= 512; negatives <= 8;
 * walk_len <= 255 (0 selects LINE mode: the pool is the CSR edge list);
 * 1 <= window <= walk_len when walk_len > 0; walks_per_node >= 1;
 * 1 <= episodes <= 4095; 1 <= subparts and world*subparts*world <= 4096;
 * p, q > 0 (or 0 for 1). */
typedef struct {
    uint32_t dim;            /* d, embedding dimension (tab:perf d = 96..128)     */
    uint32_t negatives;      /* K negatives per positive sample (tab:perf K = 5)  */
    uint32_t walk_len;       /* k walk steps ("walk distance"); 0 = LINE mode      */
    uint32_t window;         /* l context length ("walk context length")          */
    uint32_t walks_per_node; /* w walks started from every node (reading D5)            */
    uint32_t episodes;       /* episodes per epoch ("fixed-size sample pool")     */
    uint32_t subparts;       /* vertex sub-parts per GPU, the paper's k = 4    */
    uint32_t deterministic;  /* 1: one warp per block in canonical order (parity mode);
                                0: Hogwild production mode (lock-free warps)            */
    uint32_t conflict_permille; /* Hogwild concurrency cap: at most
                                (permille/1000) / ((1+K)^2/ctx_rows + 1/vertex_rows)
                                warps train a block at once -- the expected share of
                                in-flight samples sharing a row with another one under
                                uniform access.  0 = 300 (30 %); >= 1000000 = no cap.
                                Large graphs fill the GPU below the cap.            */
    uint32_t writeback;      /* Hogwild row write-back: NE_WB_ATOMIC_DELTA (0, default)
                                adds each update's delta with a vector reduction
                                (red.global.add.v4.f32), so concurrent updates of a
                                row are never erased; NE_WB_STORE (1) stores the new
                                rows (word2vec-style, loses concurrent updates).
                                Deterministic mode always stores.                   */
    float    p, q;           /* node2vec return / in-out parameters (NEXT-1; node2vec,
                                P:355; rejection sampling as in KnightKing).
                                p = q = 1 (or 0) = first-order DeepWalk walk.  Other
                                values need every CSR row sorted by target.         */
    uint32_t update_rule;    /* NE_UPDATE_SEQUENTIAL (0): the 1+K Train calls of Alg. 1
                                in order, each seeing the updated vertex row (D2);
                                NE_UPDATE_ACCUMULATED (1): word2vec / GraphVite style --
                                all 1+K dots use the pre-sample vertex row, whose
                                accumulated gradient is applied once (NEXT-4);
                                NE_UPDATE_SHARED_BATCH (2): mini-batches of 128
                                consecutive samples share `negatives` (= 32)
                                negatives and take one SGD step on the batch loss
                                (Ji et al. / BlazingText; DESIGN D17) --
                                three tf32 tensor-core products per batch (tcgen05,
                                TMEM accumulators); dim must be 128, fp32 rows      */
    uint32_t staging;        /* NE_STAGE_DEVICE (0): the vertex matrix lives in HBM;
                                NE_STAGE_HOST (1): in pinned host memory (each rank its
                                own part), streamed through device sub-part slots --
                                one GPU: 3 slots, H2D of sub-part t+1 and D2H of t-1
                                overlap the training of t (the paper's pipeline stages
                                5 and 2; NEXT-2); world > 1 (NCCL
                                transport): the sub-parts go around the ring in windows
                                of stage_window slots (3 x stage_window device slots,
                                stages 5, 3, 4, 2), DESIGN reading D18.               */
    uint32_t storage;        /* NE_STORE_F32 (0): fp32 rows, the paper's precision;
                                NE_STORE_BF16 (1): rows stored as bfloat16 (NEXT-4,
                                DESIGN reading D16) -- half the bytes per sample;
                                compute stays fp32, each touched row is rounded to the
                                nearest bf16 (ties to even) when the sample stores it.
                                ne_get/set_embeddings still take fp32 host arrays; the
                                ring and host staging move bf16 sub-parts (half the
                                bytes).                                                 */
    uint32_t transport;      /* NE_TRANSPORT_NCCL (0): ncclSend/Recv on the comm stream;
                                NE_TRANSPORT_IPC (1): copy-engine pushes over CUDA IPC
                                into rank+1's slots, ordered by GPU-side flag waits
                                (no SM kernels; ne_ipc_export / ne_ipc_connect after
                                ne_load_graph).  With IPC, ne_init_dist may take
                                id == NULL: no NCCL at all (each rank then builds its
                                part's pool from every walker, the layout-only way). */
    uint64_t seed;           /* Philox key (contract R1)                                */
    uint32_t stage_window;   /* NE_STAGE_HOST with world > 1: sub-parts per ring window
                                (w <= subparts; 0 = 2).  The plan trains the windows one
                                after the other, each through all world rounds.       */
    uint32_t groups;         /* NEXT-3 two-level ring (P:150 hierarchical partitioning,
                                P:190-191): the world's ranks form `groups` groups
                                ("nodes") of world/groups consecutive ranks; each group
                                first trains its own vertex parts around its internal
                                ring, then the groups pass their parts to the next group
                                (ne_plan_vsub2).  0 or 1 = one ring over all ranks.   */
} ne_config;

/* Per-call statistics (this rank).  Times are device time from CUDA events. */
typedef struct {
    uint64_t samples;        /* positive samples trained                               */
    double   loss_sum;       /* sum over all 1+K updates of -log s / -log(1-s)         */
    float    ms_walk;        /* walk kernel time (on the stream the walk ran on)       */
    float    ms_build;       /* pool build time: pairs, exchange, order, bucketing     */
    float    ms_train;       /* sum of SGNS kernel durations                           */
    float    ms_comm_wait;   /* time the compute stream waited for ring receives       */
    uint32_t train_launches; /* SGNS kernel launches                                   */
    uint32_t kernel_launches;/* every kernel this library launched during the call     */
    float    ms_pool_wait;   /* time the compute stream waited for walk + pool build
                                (exposed; a build overlapped with training is hidden)  */
} ne_stats;

/* Library ABI version (NE_ABI_VERSION). */
int ne_version(void);

/* Create a context on CUDA `device` (the caller has selected nothing; the
 * library calls cudaSetDevice itself).  alloc/free may be NULL (cudaMalloc).
 * Errors: NE_EINVAL (cfg limits above), NE_ECUDA (no device / not sm_100). */
int ne_create(ne_ctx **out, const ne_config *cfg, int device,
              ne_alloc_fn alloc, ne_free_fn free_fn, void *user);

/* Use `stream` (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream)
 * as the compute stream.  NULL (0) is the CUDA legacy default stream -- the
 * handle torch reports for its default stream -- so work the caller queued
 * there is ordered before the library's.  NE_STREAM_OWN selects the context's
 * own non-blocking stream (the state after ne_create). */
#define NE_STREAM_OWN ((void *)~(uintptr_t)0)
int ne_set_stream(ne_ctx *ctx, void *stream);

/* Make the compute stream wait (device-side, the host does not block) for
 * every transfer the library left in flight on its side streams: the
 * return-home ring transfers of the last ne_train_samples / ne_train_epoch
 * and host-staging copies.  Call it before recording a timing event
 * on the compute stream that must cover them. */
int ne_join(ne_ctx *ctx);

/* NCCL bootstrap for the multi-GPU ring: rank 0 calls
 * ne_get_nccl_id, the harness broadcasts the 128 bytes (torch.distributed),
 * then every rank calls ne_init_dist before ne_load_graph.  world == 1 needs
 * no id (id may be NULL); world > 1 with id == NULL makes a layout-only
 * context (partitions, pool and negatives of `rank`, no training: NE_ESTATE).  Rank g owns context part g and vertex part g
 * (contiguous ranges, reading D12; "fix the context embeddings for each
 * GPU").  Errors: NE_EINVAL, NE_ESTATE (graph already loaded), NE_ENCCL. */
int ne_get_nccl_id(uint8_t id[128]);
int ne_init_dist(ne_ctx *ctx, int rank, int world, const uint8_t id[128]);

/* Copy-engine ring bootstrap (transport == NE_TRANSPORT_IPC, world > 1).
 * After ne_load_graph every rank exports one blob of ne_ipc_blob_size()
 * bytes (the CUDA IPC handle of its vertex-slot region); the harness
 * all-gathers them in rank order (e.g. torch.distributed) and every rank
 * calls ne_ipc_connect with the world * blob_size bytes.  Must be repeated
 * after a reload that changes the graph's shape.  Before any rank destroys
 * its context, all ranks must be done training (ne_destroy drains the ring).
 * Errors: NE_ESTATE (wrong transport, no graph), NE_EINVAL (blob mismatch),
 * NE_ECUDA. */
size_t ne_ipc_blob_size(void);
int ne_ipc_export(ne_ctx *ctx, void *blob, size_t cap);
int ne_ipc_connect(ne_ctx *ctx, const void *blobs, size_t blob_size);

/* Load the graph G = (V, E) as CSR: offsets[n+1] (u64),
 * targets[nnz] (u32), validated on the device against S:24 (offsets
 * monotone, offsets[0] == 0, offsets[n] == nnz, every target < n); the copy is
 * resident in HBM on every rank.  With world > 1 and NCCL each rank copies
 * only its 1/world slice of the arrays it is given and an all-gather over
 * NVLink completes the rest, so every rank must pass the same graph.  Also builds this rank's alias table
 * (deg^0.75 over its context part, O3/D9) and initialises the embeddings
 * (O9: vertex U(-0.5/d, 0.5/d), context 0).  May be called again to replace
 * the graph (re-initialises).  Errors: NE_EINVAL (+ first offending index),
 * With node2vec parameters (p, q != 1) rows must also be sorted by target
 * (NE_EINVAL "targets[e]=... < targets[e-1]=... in row r").
 * NE_ERANGE (n >= 2^32 - 1 or n < world), NE_ENOMEM, NE_ECUDA. */
int ne_load_graph(ne_ctx *ctx, uint32_t n, uint64_t nnz,
                  const uint64_t *offsets, const uint32_t *targets);

/* Walk engine, one episode (Alg. 1 "parallel random walk"; O4):
 * walkers omega of the episode's contiguous range, start = omega mod n, k
 * steps, Philox(ctr = (omega, t, WALK|epoch)) per step, stop at a node
 * without out-edges.  With node2vec parameters, step t >= 2 repeats trials r
 * with ctr word 2 = t | r << 8 until the candidate passes its threshold.  Kept on the device; if host_walks != NULL also copied
 * out as [walkers][walk_len+1] u32, 0xFFFFFFFF after the walk's end
 * (cap_u32 = capacity in u32).  walkers_out (nullable) receives the count.
 * Errors: NE_ESTATE (no graph; LINE mode), NE_ERANGE (episode, epoch >= 2^24,
 * capacity). */
int ne_random_walk(ne_ctx *ctx, uint32_t epoch, uint32_t episode,
                   uint32_t *host_walks, size_t cap_u32, uint64_t *walkers_out);

/* Network augmentation + sample pool of the episode (
 * O5/O6): window pairs (path[i], path[i+delta]), 1 <= delta <= l, of the walks
 * ne_random_walk produced (LINE mode: the CSR edges of the episode), keeping
 * those whose context node lies in this rank's context part, ordered by the
 * Feistel permutation pi of their generation index and grouped by vertex
 * sub-part (2D block).  n_samples_out (nullable) = pool size.
 * Errors: NE_ESTATE (walks missing / of another episode), NE_ERANGE. */
int ne_build_samples(ne_ctx *ctx, uint32_t epoch, uint32_t episode, uint64_t *n_samples_out);

/* Train the pool built by ne_build_samples for (epoch, episode) with learning
 * rate lr, following the ring plan (O7): for round r, slot t, this rank trains
 * block (vertex sub-part ((rank - r) mod world)*subparts + t, context part
 * rank), then sends that sub-part to rank+1 and receives the next from
 * rank-1.  Each positive sample (u, v) gets K alias negatives (O8) and
 * 1+K sequential SGNS updates (O10).  stats may be NULL.
 * Errors: NE_ESTATE, NE_ENCCL, NE_ECUDA. */
int ne_train_samples(ne_ctx *ctx, uint32_t epoch, uint32_t episode, float lr, ne_stats *stats);

/* One epoch ("one epoch goes over all the sampled edges"): for every
 * episode, walk + build + train.  The walk and pool of the next episode are
 * built on a side stream while the current episode trains, into a
 * third pool buffer allocated when HBM allows; after the last episode the
 * first episode of epoch+1 is built the same way and kept for the next call
 * (discarded by ne_load_graph, ne_random_walk, ne_build_samples or a call
 * with another epoch).  Results are those of the serial order.
 * flags: NE_REUSE_SAMPLES, NE_CHECK_BLOCKS.  lr is constant within the epoch
 * (the caller may decay it between epochs).  stats (nullable)
 * accumulates the whole epoch. */
int ne_train_epoch(ne_ctx *ctx, uint32_t epoch, float lr, uint32_t flags, ne_stats *stats);

/* Copy rows [row_begin, row_end) of the vertex (which = NE_VERTEX) or context
 * (NE_CONTEXT) matrix to host_out (row-major fp32, d floats per row;
 * cap_floats = capacity).  The rows must lie in this rank's part (the vertex
 * sub-parts are back home after every ne_train_samples).
 * Errors: NE_ERANGE (rows not owned, capacity), NE_ESTATE. */
int ne_get_embeddings(ne_ctx *ctx, int which, uint32_t row_begin, uint32_t row_end,
                      float *host_out, size_t cap_floats);

/* Stream this rank's trained vertex rows to host memory during training
 * (e2e; the paper's stage 2 "send vertex embeddings back"): from the
 * next ne_train_epoch on, every call copies vertex sub-part t to
 * host_rows[(row - part begin) * d ...] on a copy engine as soon as it is
 * final -- one GPU: after its block of the call's last episode; with the ring:
 * when it arrives home after the last round -- overlapping the remaining
 * training, and returns with the copies complete, host_rows then equal to
 * ne_get_embeddings(NE_VERTEX) of the whole part.  host_rows should be pinned
 * (page-locked) for the overlap; it stays registered across ne_load_graph
 * until replaced or turned off with NULL.  fp32 rows, device staging.
 * Errors: NE_EINVAL (bf16 storage, host staging, a layout-only world > 1
 * context), NE_ERANGE (cap_floats < part rows x d, checked here and at every
 * ne_train_epoch). */
int ne_export_vertex_on_train(ne_ctx *ctx, float *host_rows, size_t cap_floats);

/* Overwrite rows [row_begin, row_end) of this rank's part (checkpoint resume,
 * S:399; tests).  Same ownership rules as ne_get_embeddings. */
int ne_set_embeddings(ne_ctx *ctx, int which, uint32_t row_begin, uint32_t row_end,
                      const float *in);

/* Last error message of ctx (never NULL; "" after success). */
const char *ne_last_error(const ne_ctx *ctx);

/* Release the context and all its device memory. */
void ne_destroy(ne_ctx *ctx);

/* Schedule check of the current pool ("orthogonal vertex
 * usage"): every sample of block (vsub, rank) must have its source in vertex
 * sub-part vsub and its context node in this rank's part.  Returns NE_OK, or
 * NE_ESCHED with the first offending position and its block in the message.
 * ne_train_epoch runs it after each build with the NE_CHECK_BLOCKS flag. */
int ne_check_pool(ne_ctx *ctx);

/* ---- test hooks (bit-exact parity against the oracle) -------------------- */

/* Copy the current pool's samples of local block `vsub` (vertex sub-part id,
 * 0 <= vsub < world*subparts; the block is (vsub, this rank's context part))
 * as (src, dst) u32 pairs in canonical order.  count receives the block size
 * even when pairs_out is NULL.  Errors: NE_ESTATE, NE_ERANGE. */
int ne_export_samples(ne_ctx *ctx, uint32_t vsub, uint32_t *pairs_out, size_t cap_pairs,
                      uint64_t *count);

/* Negatives of positions [pos_begin, pos_begin+count) of block (vsub, this
 * rank's part) in (epoch, episode), computed by the same device function the
 * SGNS kernel uses (O8); out = count*K u32 (global node ids). */
int ne_export_negatives(ne_ctx *ctx, uint32_t epoch, uint32_t episode, uint32_t vsub,
                        uint64_t pos_begin, uint64_t count, uint32_t *out);

/* Train block (vsub, this rank's context part) of the built pool of
 * (epoch, episode) once with the PRODUCTION kernel at its full grid (the
 * deterministic flag of the context is ignored), recording the ids every
 * sample position p trained: out[p*(2+K) + 0] = src, + 1 = dst,
 * + 2 + j = negative j (O8).  vsub must be one of this rank's home sub-parts
 * (rank*subparts <= vsub < (rank+1)*subparts); cap_u32 >= count*(2+K).
 * count (nullable) receives the block size.  Updates the embeddings like
 * training.  Errors: NE_ESTATE (no pool; host staging), NE_ERANGE. */
int ne_capture_block(ne_ctx *ctx, uint32_t epoch, uint32_t episode, uint32_t vsub, float lr,
                     uint32_t *out, size_t cap_u32, uint64_t *count);

/* NEXT-4 test hook: the shared-negative batch kernel's three tcgen05 tf32
 * products on the current device, through its shared-memory tiles,
 * transposes, descriptors and TMEM read-back: host row-major V[128][128],
 * N[32][128], G[128][32] -> S = V N^T [128][32], dV = G N [128][128],
 * dNt = V^T G [128][32].  Errors: NE_EINVAL, NE_ECUDA. */
int ne_umma_products(const float *V, const float *N, const float *G, float *S, float *dV, float *dNt);

/* Diagnostics hook: one tcgen05 tf32 product D[128][N] from raw shared-memory
 * images of A and B (img_bytes each, <= 64 KB), shared-memory descriptors
 * (lbo, sbo in bytes; a_hi / b_hi OR-ed into the upper descriptor bits, e.g.
 * the layout type), start addresses advancing a_step / b_step bytes over
 * `ksteps` instructions, and instruction descriptor idesc. */
int ne_umma_raw(const void *a_img, const void *b_img, uint32_t img_bytes, uint64_t a_hi, uint64_t b_hi,
                uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo, uint32_t a_step, uint32_t b_step,
                uint32_t ksteps, uint32_t idesc, uint32_t N, float *D);

/* Single-GPU emulation of the P-rank ring for parity tests: ctxs[g] are
 * layout-only contexts (ne_init_dist(ctx, g, world, NULL)) on ONE device, each
 * with the pool of `episode` built.  Runs the same plan as ne_train_samples
 * (round r, slot t, rank g, in that order, all on ctxs[0]'s stream) with the
 * send to rank g+1 replaced by handing the trained sub-part buffer to context
 * g+1.  After the call every sub-part is home again.  stats (nullable) sums all
 * ranks.  Errors: NE_EINVAL (contexts not ranks 0..world-1 of one device),
 * NE_ESTATE (pool missing). */
int ne_train_samples_local_ring(ne_ctx *const *ctxs, uint32_t world, uint32_t epoch,
                                uint32_t episode, float lr, ne_stats *stats);

/* The host-side ring schedule (O7), no device needed: the vertex sub-part
 * rank g trains at round r, slot t, with `world` ranks and `subparts` slots.
 * Returns -1 on bad arguments. */
int ne_plan_vsub(uint32_t world, uint32_t subparts, uint32_t r, uint32_t t, uint32_t g);

/* NEXT-3 two-level plan: rank g of `world` in `groups` groups trains vertex
 * sub-part ne_plan_vsub2(...) at global round rho (0 <= rho < world) and slot
 * t; groups = 1 is ne_plan_vsub.  ne_ring_peers gives the rank a sub-part
 * moves to after round rho (dest) and the rank sending to g (src).  No device
 * needed.  -1 / NE_EINVAL on bad arguments (groups must divide world). */
int ne_plan_vsub2(uint32_t world, uint32_t groups, uint32_t subparts, uint32_t rho, uint32_t t, uint32_t g);
int ne_ring_peers(uint32_t world, uint32_t groups, uint32_t rho, uint32_t g, uint32_t *dest, uint32_t *src);

/* Contiguous part bounds used by the library (reading D12): bounds[0..parts]
 * of [0, n).  No device needed.  Returns NE_EINVAL if parts == 0. */
int ne_partition_bounds(uint64_t n, uint32_t parts, uint64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif /* NE_H */

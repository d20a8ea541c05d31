// ne_internal.h -- kernel launchers shared by the runtime (host C++) and the
// CUDA translation units.  Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ne {

// Device grid sizing: a multiple of the SM count (persistent / grid-stride kernels).
struct Device {
    int sm_count = 148;
    int max_threads_per_sm = 2048;
};

// ---- graph / init / walks (kernels_graph.cu) -------------------------------
// S:24 invariants; bad[0] = first i with offsets[i+1] < offsets[i] (or ~0),
// bad[1] = first e with targets[e] >= n (or ~0); with check_sorted, bad[2] =
// first e > offsets[row] with targets[e] < targets[e-1] inside its row (or ~0).
cudaError_t launch_validate_csr(const uint64_t* off, const uint32_t* tgt, uint64_t n,
                                uint64_t nnz, unsigned long long* bad, bool check_sorted,
                                const Device& dev, cudaStream_t s);
// O9: rows [row_begin, row_begin + rows) of the vertex matrix into V (row-major).
cudaError_t launch_init_vertex(float* V, uint64_t row_begin, uint64_t rows, uint32_t d,
                               uint64_t seed, bool bf16, const Device& dev, cudaStream_t s);
// NEXT-4 bf16 rows: n elements bf16 -> fp32 (exact) or fp32 -> bf16 (nearest even).
cudaError_t launch_convert_rows(const void* in, void* out, uint64_t n, bool to_bf16, const Device& dev,
                                cudaStream_t s);
// O4: walkers [omega0, omega0 + count) -> walks[count][k+1].  node2vec
// (NEXT-1) when n2v_thr != nullptr: thresholds (return, neighbour, farther),
// each <= 2^32, of the rejection step.  With wc.counts != nullptr the kernel
// also writes the O5 count of every walker (its window pairs whose context
// node lies in [c_begin, c_end)) -- what count_walk would compute from the walk.
struct WalkCount {
    uint32_t* counts;
    uint32_t l;
    uint64_t c_begin, c_end;
};
cudaError_t launch_walk(const uint64_t* off, const uint32_t* tgt, uint64_t n, uint64_t omega0,
                        uint64_t count, uint32_t k, uint64_t seed, uint32_t epoch,
                        const uint64_t* n2v_thr, uint32_t* walks, const WalkCount& wc, const Device& dev,
                        cudaStream_t s);

// ---- sample pool (kernels_samples.cu) ---------------------------------------
struct PoolParams {
    uint64_t N;           // this rank's pairs in the episode (Feistel domain, O6)
    uint64_t units;       // walkers (DeepWalk) or edges (LINE) of the episode
    uint64_t u0;          // first unit (edge id in LINE mode)
    uint32_t k, l, Pw;    // walk steps, window, pairs per full walk (1 in LINE mode)
    uint32_t episode, epoch;
    uint64_t seed;
    uint64_t c_begin, c_end;   // this rank's context part
};
// O5 count: counts[u] = pairs of unit u whose context node lies in this
// rank's part.  slot_tab[s] = (i << 16) | delta for s < Pw.
cudaError_t launch_count_walk(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                              uint32_t* counts, const Device& dev, cudaStream_t s);
cudaError_t launch_count_line(const uint32_t* tgt, const PoolParams& p, uint32_t* counts,
                              const Device& dev, cudaStream_t s);
// Exclusive scan u32 -> u64 over M values; *total = sum.  scratch >= scan_scratch_bytes(M).
size_t scan_scratch_bytes(uint64_t M);
cudaError_t launch_scan(const uint32_t* in, uint64_t M, uint64_t* out, uint64_t* total, void* scratch,
                        cudaStream_t s, uint32_t* launches);
// O5 + O6: the kept pairs of unit u get part-local indices base[u] + rank
// (generation order); pair x belongs at position y = pi(x) of [0, p.N), pi the
// Feistel bijection.  Where it is stored is the sink's choice:
//  * direct (key == nullptr): out[y] = pair -- a dense pi-indexed array, one
//    random 8-byte store per pair.  Measured on C3 (522 M pairs): ~24 ms, a
//    random store over a multi-GB target per pair (TLB reach is 256 MB);
//  * keyed (default): out[x] = pair, key[x] = y in generation order (coalesced);
//    launch_order then moves the pairs to their positions with radix passes.
struct PoolSink {
    uint64_t* out;
    uint32_t* key;       // keyed mode (needs N <= 2^32)
};
cudaError_t launch_pairs_walk(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                              const uint64_t* base, const PoolSink& sink, const Device& dev, cudaStream_t s);
cudaError_t launch_pairs_line(const uint64_t* off, const uint32_t* tgt, uint64_t n,
                              const PoolParams& p, const uint64_t* base, const PoolSink& sink,
                              const Device& dev, cudaStream_t s);
// Sharded construction at P > 1 (walkers sharded over the ranks, O(N/P) per
// rank): p.units = this shard's walkers (walks[units][k+1]); part_bounds =
// device copy of the P + 1 context-part bounds, P <= 32.
// counts[g * units + w] = pairs of walker w whose context node is in part g.
cudaError_t launch_count_parts(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                               const uint64_t* part_bounds, uint32_t P, uint32_t* counts, const Device& dev,
                               cudaStream_t s);
// Every pair of the shard to out[base[g * units + w] + rank within (w, g)]
// (base = exclusive scan of counts): the send buffer, grouped by part.
cudaError_t launch_pairs_parts(const uint32_t* walks, const uint32_t* slot_tab, const PoolParams& p,
                               const uint64_t* part_bounds, uint32_t P, const uint64_t* base, uint64_t* out,
                               const Device& dev, cudaStream_t s);
// tot[g] (device, P values) = the shard's pairs in part g (from base / total).
cudaError_t launch_part_totals(const uint64_t* base, uint64_t units, uint32_t P, const uint64_t* total,
                               uint64_t* tot, cudaStream_t s);
// out[pi(x)] = in[x] for x in [0, p.N): the direct sink of a gathered pool.
cudaError_t launch_feistel_scatter(const PoolParams& p, const uint64_t* in, uint64_t* out, const Device& dev,
                                   cudaStream_t s);
// key[x] = pi(x) for x in [0, p.N) (O6 Feistel of the part's pool).
cudaError_t launch_feistel_keys(const PoolParams& p, uint32_t* key, const Device& dev, cudaStream_t s);
// first pool position outside its 2D block -> *bad (atomicMin; init ~0).
cudaError_t launch_check_pool(const uint64_t* pool, const uint64_t* boff, uint64_t total,
                              const uint64_t* sub_bounds, uint32_t nb, uint64_t c_begin, uint64_t c_end,
                              unsigned long long* bad, const Device& dev, cudaStream_t s);
// Keyed sink -> window layout: 1-2 radix passes over the 32-bit keys above
// the low kPoolWinBits (pi is a bijection, so the region of every key prefix
// is known: prefix << shift).  Buffers ping-pong: (pairs0, keys0) hold the
// sink's output, (pairs1, keys1) are the same size; on return *win_pairs /
// *win_pos (u16 = y mod 2^kPoolWinBits, aliasing a key buffer) are the window
// layout and *spare the pair buffer launch_bucket may write the pool to.
constexpr uint32_t kPoolWinBits = 13;
cudaError_t launch_order(uint64_t N, uint64_t* pairs0, uint32_t* keys0, uint64_t* pairs1, uint32_t* keys1,
                         uint32_t* cursors, const uint64_t** win_pairs, const uint16_t** win_pos, uint64_t** spare,
                         const Device& dev, cudaStream_t s, uint32_t* launches);
// Stable partition of the pairs by vertex sub-part (bounds over nb+1 entries,
// device pointer): pool[block_offsets[b] ...] in pi order.  pos == nullptr:
// `slots` is the dense pi-indexed array; else the window layout.
// scratch >= bucket_scratch_bytes(N, nb); its head doubles as radix cursors.
size_t bucket_scratch_bytes(uint64_t N, uint32_t nb);
cudaError_t launch_bucket(const uint64_t* slots, const uint16_t* pos, uint64_t N, const uint64_t* sub_bounds,
                          uint32_t nb, void* scratch, uint64_t* pool, uint64_t* block_offsets,
                          const Device& dev, cudaStream_t s, uint32_t* launches);

// ---- SGNS (kernels_sgns.cu) ---------------------------------------------------
struct SgnsParams {
    const uint2* pool;          // (src, dst) pairs of the block, canonical order
    uint64_t count;             // samples in the block
    float* V;                   // vertex sub-part slot; row (src - v_begin)
    uint64_t v_begin;
    float* C;                   // context part; row (dst - c_begin)
    uint64_t c_begin, c_count;
    const uint2* alias;         // (thr, alias) per context-part column
    uint32_t d, K;
    float lr;
    uint64_t seed;
    uint32_t epoch, episode, block;   // block = vsub * world + rank (O8 counter)
    double* loss;               // += sum of loss terms (device)
    int deterministic;          // 1: one warp, canonical order
    uint64_t max_warps;         // Hogwild concurrency cap (>= 1)
    int atomic_writeback;       // Hogwild: red.add row deltas instead of storing rows
    int reserve_sms;            // SMs left free for the concurrent NCCL ring kernels
    int bf16;                   // rows stored as bfloat16 (NEXT-4, reading D16); V, C point at them
    int accumulate;             // update rule: 0 sequential, 1 accumulated (word2vec), 2 shared-negative batch
    uint32_t* capture;          // test hook: (src, dst, negs) per position, [count][2+K] (nullptr: off)
    uint32_t l2hint;            // developer knob (fp32 rows): L2 policy of vertex (bits 0-1) / context (2-3) rows
};
cudaError_t launch_sgns(const SgnsParams& p, const Device& dev, cudaStream_t s);
// bf16-row instantiations (kernels_sgns_bf16.cu); launch_sgns dispatches on p.bf16.
cudaError_t launch_sgns_bf16(const SgnsParams& p, const Device& dev, cudaStream_t s);
// NEXT-4 shared-negative mini-batch rule (p.accumulate == 2; kernels_sgns_batch.cu):
// batches of 128 samples share p.K negatives; tcgen05 tf32 products.  d == 128.
cudaError_t launch_sgns_batch(const SgnsParams& p, const Device& dev, cudaStream_t s);
// Test hook: the batch kernel's three tcgen05 products (d = 128, K' = 32) on dense
// row-major device inputs V[128][128], N[32][128], G[128][32] ->
// S = V N^T [128][32], dV = G N [128][128], dNt = V^T G [128][32].
cudaError_t launch_umma_raw(const void* a_img, const void* b_img, uint32_t img_bytes, uint64_t a_hi, uint64_t b_hi,
                            uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo, uint32_t a_step,
                            uint32_t b_step, uint32_t ksteps, uint32_t idesc, uint32_t N, float* D, cudaStream_t s);
cudaError_t launch_umma_products(const float* V, const float* N, const float* G, float* S, float* dV, float* dNt,
                                 cudaStream_t s);
cudaError_t launch_export_negatives(const SgnsParams& p, uint64_t pos_begin, uint64_t count,
                                    uint32_t* out, const Device& dev, cudaStream_t s);

}  // namespace ne

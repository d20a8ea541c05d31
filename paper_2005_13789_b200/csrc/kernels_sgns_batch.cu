// kernels_sgns_batch.cu -- NEXT-4 shared-negative mini-batch SGNS on the 5th
// generation tensor cores (sm_100a tcgen05 + TMEM).
//
// Rule (reading D17; Ji et al. 2019 and BlazingText, cited P:363-364: "forming
// the computation into mini-batches, they can share the negative samples
// within one mini-batch ... level-1 BLAS operations can be converted into
// level-3 BLAS matrix multiply operations"): a block's samples are taken in
// canonical order in mini-batches of B = 128; the batch's K' negatives are
// shared by all its samples; the batch takes ONE SGD step on its loss
//   L = sum_i [ l(v_i . c+_i, 1) + sum_j l(v_i . n_j, 0) ]
// from the batch-start values.  With V (B x d), N (K' x d), the negative part
// is three dense contractions:
//   S  = V N^T              (B x K')   logits            -> TMEM
//   G  = lr * sigma(S)      (B x K')   (epilogue, in smem)
//   dV = G N                (B x d)    vertex gradients  -> TMEM
//   dN^T = V^T G            (d x K')   negative gradients -> TMEM
// each issued as tcgen05.mma.kind::tf32 (fp32 rows, tf32 products, fp32
// accumulation in TMEM) by one thread.  The positive term of each sample is a
// d-long dot (CUDA cores, from shared memory).
//
// One CTA of 256 threads per batch (batch row i <-> TMEM lane i, read by the
// two warps of its lane quarter); the persistent grid strides over the block's
// batches (Hogwild: concurrent batches share rows; every write-back is a
// red.global.add of the delta), and each CTA gathers its next batch's rows
// while it writes the current one back.  The deterministic mode runs one CTA
// over the batches in order, gathering each batch after the previous one's
// write-back.
//
// Every operand is K-major (measured: with the no-swizzle layout, MN-major
// tf32 operands multiply as zeros -- CUTLASS allows MN-major tf32 only in the
// 128B/32B-base swizzled layout), in the UMMA canonical no-swizzle layout:
// 8-row x 16-byte core matrices, row r chunk c (4 floats) at byte
//   ((r / 8) * (cols / 4) + c) * 128 + (r % 8) * 16,
// LBO = 128 B between K chunks, SBO = cols * 32 B between row groups.  Each
// matrix is therefore kept in both orientations the products need: V (rows i)
// and V^T (rows = dimensions), N and N^T, G and G^T -- 192 KB at d = 128,
// K' = 32 (the positive context rows are read from global memory).
#include <algorithm>
#include <cstdlib>

#include "ne_device.cuh"
#include "ne_internal.h"

namespace ne {

namespace {

constexpr int kBatch = 128;      // B = UMMA M = threads per CTA = TMEM lanes
constexpr uint32_t kTagBNeg = 8;

// ---- tcgen05 / mbarrier primitives (PTX ISA 8.7, sm_100a) ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, SWIZZLE_NONE (layout type 0), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Instruction descriptor of kind::tf32: D fp32, A/B tf32, M x N, majors.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
    return (1u << 4)                      // c_format = F32
         | (2u << 7)                      // a_format = TF32
         | (2u << 10)                     // b_format = TF32
         | ((a_mn ? 1u : 0u) << 15)       // a_major
         | ((b_mn ? 1u : 0u) << 16)       // b_major
         | ((N >> 3) << 17)               // n_dim
         | ((M >> 4) << 24);              // m_dim
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n"
        ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane (32x32b shape, x32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive TMEM columns of this thread's lane (32x32b shape, x16).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Byte offset of (row, 4-float chunk) in a no-swizzle tile with `cols` columns.
// Byte offset of (row, 4-float chunk) in a no-swizzle tile with `cols` columns
// whose K-adjacent core matrices are `lbo` bytes apart (LBO; SBO = cols / 4 *
// lbo).  lbo = 128 packs the core matrices; kLboPad = 144 leaves 16 bytes
// after each, so the 32 chunks of one row fall in 32 different banks (a warp
// reading a row, lane = chunk, is conflict-free instead of 8-way).
constexpr uint32_t kLboPad = 144;
__device__ __forceinline__ uint32_t tile_off(uint32_t row, uint32_t chunk, uint32_t cols, uint32_t lbo = 128u) {
    return ((row >> 3) * (cols >> 2) + chunk) * lbo + (row & 7u) * 16u;
}

__device__ __forceinline__ float sigmoid_clamped(float x, float& ex) {
    x = fminf(fmaxf(x, -30.f), 30.f);
    ex = __expf(-x);
    return __fdividef(1.f, 1.f + ex);
}

// The three products of a batch, issued by one thread, all operands K-major:
//   S[B x KP]    = V N^T   A = V   (i x d),  B = N   (j x d)    K = d
//   dV[B x D]    = G N     A = G   (i x j),  B = N^T (d x j)    K = KP
//   dN^T[D x KP] = V^T G   A = V^T (d x i),  B = G^T (j x i)    K = B
template <int D, int KP>
__device__ __forceinline__ void issue_S(uint32_t sV, uint32_t sN, uint32_t t_S) {
    constexpr uint32_t idesc = idesc_tf32(kBatch, KP, false, false);
#pragma unroll
    for (uint32_t ks = 0; ks < D / 8; ++ks)
        mma_tf32(t_S, umma_desc(sV + ks * 2u * kLboPad, kLboPad, D / 4 * kLboPad),
                 umma_desc(sN + ks * 2u * kLboPad, kLboPad, D / 4 * kLboPad), idesc,
                 ks > 0);
}
template <int D, int KP>
__device__ __forceinline__ void issue_dV(uint32_t sG, uint32_t sNt, uint32_t t_dV) {
    constexpr uint32_t idesc = idesc_tf32(kBatch, D, false, false);
#pragma unroll
    for (uint32_t ks = 0; ks < (uint32_t)KP / 8; ++ks)
        mma_tf32(t_dV, umma_desc(sG + ks * 256u, 128u, KP * 32u), umma_desc(sNt + ks * 256u, 128u, KP * 32u), idesc,
                 ks > 0);
}
template <int D, int KP>
__device__ __forceinline__ void issue_dNt(uint32_t sVt, uint32_t sGt, uint32_t t_dNt) {
    constexpr uint32_t idesc = idesc_tf32(D, KP, false, false);
#pragma unroll
    for (uint32_t ks = 0; ks < (uint32_t)kBatch / 8; ++ks)
        mma_tf32(t_dNt, umma_desc(sVt + ks * 256u, 128u, kBatch * 32u),
                 umma_desc(sGt + ks * 2u * kLboPad, kLboPad, kBatch / 4 * kLboPad),
                 idesc, ks > 0);
}

// dst = src^T between two tiles (src: R rows x C cols, dst: C rows x R cols):
// every thread gathers 4 consecutive source rows of one column and stores them
// as one 16-byte chunk of the destination row.
template <uint32_t R, uint32_t C, uint32_t NT = kBatch, uint32_t SL = kLboPad, uint32_t DL = 128u>
__device__ __forceinline__ void transpose_tile(const unsigned char* src, unsigned char* dst, uint32_t tid) {
    static_assert(R % 16 == 0 && C % 8 == 0, "a warp covers 8 columns x 4 row chunks");
    for (uint32_t f = tid; f < R / 4 * C; f += NT) {
        // a warp covers 8 consecutive columns x 4 consecutive row chunks: 4-way
        // bank conflicts on the gathers (32 lanes in one column would be 8-way)
        const uint32_t l = f & 31u, grp = f >> 5, cgroups = C / 8;
        const uint32_t col = (grp % cgroups) * 8 + (l & 7u), r4 = (grp / cgroups) * 4 + (l >> 3);
        float4 v;
        float* vp = &v.x;
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e)
            vp[e] = *reinterpret_cast<const float*>(src + tile_off(4 * r4 + e, col >> 2, C, SL) + (col & 3u) * 4u);
        *reinterpret_cast<float4*>(dst + tile_off(col, r4, R, DL)) = v;
    }
}

// Shared-memory plan of a batch (bytes): V, V^T (B x D each), N (KP x D),
// N^T (D x KP), G (B x KP), G^T (KP x B), then barriers, TMEM address, ids.
template <int D, int KP>
struct BatchSmem {
    // V, N and G^T with padded core matrices (kLboPad): rows read by a warp
    static constexpr uint32_t V = 0, Vt = V + kBatch / 8 * (D / 4) * kLboPad, N = Vt + kBatch * D * 4,
                              Nt = N + KP / 8 * (D / 4) * kLboPad, G = Nt + KP * D * 4, Gt = G + kBatch * KP * 4,
                              tail = Gt + KP / 8 * (kBatch / 4) * kLboPad;
    static_assert(tail - G >= 64 * D * 4, "the dV write-back stages 64 rows in G, G^T");
    static constexpr size_t bytes = tail + 16 + 16 + (2 * (2 * kBatch + KP) + kBatch) * 4;
};

}  // namespace

// D: embedding dimension (UMMA M of the dN^T product: 128); KP: shared
// negatives per batch (UMMA N of S and dN^T).  256 threads: batch row i is
// TMEM lane i of warps i / 32 and 4 + i / 32 (a warp reaches only its own
// 32-lane quarter of TMEM), which split the columns of every TMEM read; the
// gathers, transposes, dot products and write-backs stride over all 8 warps.
constexpr uint32_t kBatchThreads = 256;
template <int D, int KP>
__global__ void __launch_bounds__(kBatchThreads, 1) sgns_batch_kernel(SgnsParams p) {
    static_assert(D == 128, "the dN^T product has M = d: 128");
    static_assert(KP == 32, "K' = 32 (both orientations of V, N, G: 192 KB of shared memory)");
    using SM = BatchSmem<D, KP>;
    constexpr uint32_t NT = kBatchThreads, NW = NT / 32;
    constexpr uint32_t kTmemCols = 256;  // S: KP, dV: D, dN^T: KP
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sV = smem + SM::V, *sVt = smem + SM::Vt, *sN = smem + SM::N, *sNt = smem + SM::Nt,
                  *sG = smem + SM::G, *sGt = smem + SM::Gt;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::tail);   // [0]: S ready, [1]: dV, dN^T ready
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(bar + 2);
    constexpr uint32_t kIds = 2 * kBatch + KP;  // one id buffer: src[B], dst[B], neg[K']
    uint32_t* s_ids = tmem_base + 4;             // two buffers: this batch's and the next one's
    float* s_gpos = reinterpret_cast<float*>(s_ids + 2 * kIds);  // kBatch: x_r, then lr (sigma(x_r) - 1)

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     ::"r"(smem_u32(tmem_base)), "n"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_base;
    const uint32_t t_S = tmem, t_dV = tmem + KP, t_dNt = tmem + KP + D;
    const uint32_t i = tid & (kBatch - 1u);     // batch row (TMEM lane) of this thread
    const uint32_t hi = tid / kBatch;           // 0: warps 0-3, 1: warps 4-7 (column half)
    const uint32_t lane_base = ((warp & 3u) * 32u) << 16;  // this warp's TMEM lanes

    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagBNeg, p.epoch);
    const float lr = p.lr;
    const uint64_t nbatch = (p.count + kBatch - 1) / kBatch;
    constexpr uint32_t KC = D / 4;
    double loss = 0.0;
    uint32_t phase = 0;
    // ids of batch b: thread i < 128 holds pair i; threads j < KP draw shared
    // negative j (Philox + the alias entry; the coin is taken when the id is stored)
    uint2 nx_pr = make_uint2(0, 0), nx_ta = make_uint2(0, 0);
    uint32_t nx_col = 0, nx_coin = 0;
    auto fetch_ids = [&](uint64_t b) {
        if (b >= nbatch || hi) return;
        const uint64_t q = b * kBatch + i;
        if (q < p.count) nx_pr = p.pool[q];
        if (i < (uint32_t)KP) {
            const uint4 x = philox(make_uint4((uint32_t)b, (uint32_t)(b >> 32), (p.episode << 20) | (p.block << 8) | i,
                                              tagw), key);
            nx_col = (uint32_t)uniform_index(x.x, x.y, p.c_count);
            nx_coin = x.z;
            nx_ta = __ldg(p.alias + nx_col);
        }
    };
    auto rows_of = [&](uint64_t bb) -> uint32_t {
        const uint64_t q0 = bb * kBatch;
        return (uint32_t)(p.count - q0 < (uint64_t)kBatch ? p.count - q0 : (uint64_t)kBatch);
    };
    // ids of a batch (O8 with the batch counter, tag BNEG) from the registers
    // fetch_ids filled into id buffer `buf`
    auto publish_ids = [&](uint32_t buf, uint32_t nbx) {
        if (hi) return;
        uint32_t* ids = s_ids + buf * kIds;
        if (i < nbx) {
            ids[i] = nx_pr.x;
            ids[kBatch + i] = nx_pr.y;
        }
        if (i < (uint32_t)KP) ids[2 * kBatch + i] = (uint32_t)(p.c_begin + (nx_coin < nx_ta.x ? nx_col : nx_ta.y));
    };
    // gather V and N rows of a batch (cp.async, 16 B per lane; a warp covers 8
    // rows x 4 chunks so each quarter-warp writes 128 contiguous bytes)
    // Lane l of warp w copies chunk 4w + l / 8 of rows 8k + l % 8 (k < B / 8);
    // the row ids are read from shared memory first, all at once.
    static_assert(NW * 4 == KC, "8 warps x 4 chunks cover a row");
    auto gather = [&](uint32_t buf, uint32_t nbx) {
        const uint32_t* src = s_ids + buf * kIds;
        const uint32_t* neg = src + 2 * kBatch;
        const uint32_t chunk = warp * 4 + (lane >> 3), r8 = lane & 7u;
        uint32_t vid[kBatch / 8], nid[KP / 8];
#pragma unroll
        for (uint32_t k = 0; k < kBatch / 8; ++k) vid[k] = src[8 * k + r8];
#pragma unroll
        for (uint32_t k = 0; k < (uint32_t)KP / 8; ++k) nid[k] = neg[8 * k + r8];
#pragma unroll
        for (uint32_t k = 0; k < kBatch / 8; ++k) {
            const uint32_t row = 8 * k + r8;
            const uint32_t off = tile_off(row, chunk, D, kLboPad);
            if (row < nbx) cp_async16(sV + off, p.V + (uint64_t)(vid[k] - p.v_begin) * D + chunk * 4);
            else *reinterpret_cast<float4*>(sV + off) = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < (uint32_t)KP / 8) cp_async16(sN + off, p.C + (uint64_t)(nid[k] - p.c_begin) * D + chunk * 4);
        }
    };
    // the next batch's ids and rows: published and gathered while this batch
    // is written back (Hogwild: it reads rows as concurrent CTAs do, without
    // this batch's updates); the deterministic mode fetches after them
    auto prepare = [&](uint32_t buf, uint64_t bn) {
        publish_ids(buf, rows_of(bn));
        fetch_ids(bn + gridDim.x);
        __syncthreads();
        gather(buf, rows_of(bn));
    };
    uint32_t buf = 0;
    fetch_ids(blockIdx.x);
    if (blockIdx.x < nbatch) prepare(0, blockIdx.x);

    for (uint64_t b = blockIdx.x; b < nbatch; b += gridDim.x) {
        const uint32_t nb = rows_of(b);
        const bool live = i < nb;
        const uint32_t* s_src = s_ids + buf * kIds;
        const uint32_t* s_dst = s_src + kBatch;
        const uint32_t* s_neg = s_src + 2 * kBatch;
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        // positive context rows c+_r (chunk `lane`), issued before the
        // transposes so their latency overlaps them; warp w takes rows 8w + u
        // and 64 + 8w + u, and keeps them for the vertex write-back, which
        // visits the same rows with the same warp (no C row is written before)
        static_assert(KC == 32, "one float4 of a row per lane");
        static_assert(NW * 8 * 2 == kBatch, "two groups of 8 rows per warp cover the batch");
        float4 cpos[2][8];
#pragma unroll
        for (uint32_t g = 0; g < 2; ++g)
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t r = 64 * g + warp * 8 + u;
                cpos[g][u] = r < nb ? __ldcg(reinterpret_cast<const float4*>(p.C + (uint64_t)(s_dst[r] - p.c_begin) * D) +
                                             lane)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        transpose_tile<kBatch, D, NT>(sV, sVt, tid);
        transpose_tile<KP, D, NT>(sN, sNt, tid);
        fence_async_smem();
        __syncthreads();
        // ---- MMA1: S = V N^T
        if (tid == 0) {
            fence_after();
            issue_S<D, KP>(smem_u32(sV), smem_u32(sN), t_S);
            mma_commit(&bar[0]);
        }
        // ---- positive terms (CUDA cores, overlapping MMA1): x_r = v_r . c+_r,
        // warp per row
#pragma unroll
        for (uint32_t g = 0; g < 2; ++g)
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t r = 64 * g + warp * 8 + u;
                if (r >= nb) break;  // warp-uniform
                const float4 v = *reinterpret_cast<const float4*>(sV + tile_off(r, lane, D, kLboPad));
                const float4 c = cpos[g][u];
                float x = fmaf(v.x, c.x, fmaf(v.y, c.y, fmaf(v.z, c.z, v.w * c.w)));
#pragma unroll
                for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
                if (lane == 0) s_gpos[r] = x;
            }
        __syncthreads();
        float gpos = 0.f;  // lr (sigma(x_i) - 1) of this thread's row
        if (live) {
            float ex;
            const float sp = sigmoid_clamped(s_gpos[i], ex);
            gpos = lr * (sp - 1.f);
            if (!hi) loss += (double)__logf(1.f + ex);  // -log s
        }
        // ---- epilogue 1: G = lr sigma(S) and G^T (padding rows stay 0); the
        // two warps of a lane quarter take 16 columns each
        mbar_wait(&bar[0], phase);
        fence_after();
        {
            constexpr uint32_t HC = KP / 2;
            float sv[HC];
            tmem_ld16(t_S + lane_base + hi * HC, sv);
            float part = 0.f;
#pragma unroll
            for (uint32_t c = 0; c < HC / 4; ++c) {
                float4 g;
                float* gp = &g.x;
#pragma unroll
                for (uint32_t e = 0; e < 4; ++e) {
                    float ex;
                    const float xcl = fminf(fmaxf(sv[c * 4 + e], -30.f), 30.f);
                    const float s = sigmoid_clamped(sv[c * 4 + e], ex);
                    gp[e] = live ? lr * s : 0.f;
                    if (live) part += __logf(1.f + ex) + xcl;  // -log(1 - s)
                    *reinterpret_cast<float*>(sGt + tile_off(hi * HC + c * 4 + e, i >> 2, kBatch, kLboPad) +
                                              (i & 3u) * 4u) =
                        gp[e];
                }
                *reinterpret_cast<float4*>(sG + tile_off(i, hi * (HC / 4) + c, KP)) = g;
            }
            loss += (double)part;
        }
        fence_async_smem();
        fence_before();
        __syncthreads();
        // ---- MMA2: dV = G N; MMA3: dN^T = V^T G
        if (tid == 0) {
            fence_after();
            issue_dV<D, KP>(smem_u32(sG), smem_u32(sNt), t_dV);
            issue_dNt<D, KP>(smem_u32(sVt), smem_u32(sGt), t_dNt);
            mma_commit(&bar[1]);
        }
        mbar_wait(&bar[1], phase);
        fence_after();
        __syncthreads();
        if (!hi) s_gpos[i] = gpos;
        __syncthreads();
        // ---- write-back from the batch-start snapshot; every row update is a
        // coalesced red.global.add of the delta by a warp.  (3) first: positive
        // context rows, -gpos v (every c+ read happened in the positive terms);
        // after it V and N are free for the next batch's gather.
        for (uint32_t r = warp; r < nb; r += NW) {
            const float g = s_gpos[r];
            float4* cw = reinterpret_cast<float4*>(p.C + (uint64_t)(s_dst[r] - p.c_begin) * D);
            for (uint32_t c = lane; c < KC; c += 32) {
                const float4 v = *reinterpret_cast<const float4*>(sV + tile_off(r, c, D, kLboPad));
                atomicAdd(cw + c, make_float4(-g * v.x, -g * v.y, -g * v.z, -g * v.w));
            }
        }
        const uint64_t bn = b + gridDim.x;
        const bool ahead = !p.deterministic && bn < nbatch;
        __syncthreads();
        if (ahead) prepare(buf ^ 1u, bn);
        // (1) vertex rows, -(dV + gpos c+), two halves of 64 rows staged through the G / G^T
        // tiles (consumed by the products); c+ comes from the registers the
        // positive terms loaded it into.  tcgen05.ld is warp-collective: the
        // two warps of a lane quarter load 64 columns each of their 32 rows.
        float* stage = reinterpret_cast<float*>(sG);  // 64 x D floats (G and G^T are adjacent)
#pragma unroll
        for (uint32_t half = 0; half < 2; ++half) {  // unrolled: cpos[half] stays in registers
            if (((warp & 3u) >> 1) == half) {
#pragma unroll 1
                for (uint32_t d0 = hi * (D / 2); d0 < (hi + 1) * (D / 2); d0 += 32) {
                    float dv[32];
                    tmem_ld32(t_dV + lane_base + d0, dv);
                    // chunk ch of staged row sr at ch ^ (sr % 8): the 8 rows of a
                    // quarter-warp store to 8 different bank groups
                    const uint32_t sr = i - 64 * half;
                    float4* dst = reinterpret_cast<float4*>(stage + sr * D);
#pragma unroll
                    for (uint32_t c = 0; c < 8; ++c)
                        dst[(d0 / 4 + c) ^ (sr & 7u)] = make_float4(dv[4 * c], dv[4 * c + 1], dv[4 * c + 2], dv[4 * c + 3]);
                }
            }
            fence_before();
            __syncthreads();
            {
                const uint32_t r0 = 64 * half + warp * 8;  // 8 warps x 8 rows = the half
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) {
                    const uint32_t r = r0 + u;
                    if (r >= nb) break;
                    const float g = s_gpos[r];
                    const float4 c = cpos[half][u];
                    const float4 dv = reinterpret_cast<const float4*>(stage + (r - 64 * half) * D)[lane ^ (r & 7u)];
                    atomicAdd(reinterpret_cast<float4*>(p.V + (uint64_t)(s_src[r] - p.v_begin) * D) + lane,
                              make_float4(-(dv.x + g * c.x), -(dv.y + g * c.y), -(dv.z + g * c.z), -(dv.w + g * c.w)));
                }
            }
            __syncthreads();
        }
        // (2) the dN^T lanes (= dimensions) into dN rows staged in the G tile
        {
            float dn[16];
            tmem_ld16(t_dNt + lane_base + hi * (KP / 2), dn);
#pragma unroll
            for (uint32_t e = 0; e < (uint32_t)KP / 2; ++e) stage[(hi * (KP / 2) + e) * D + i] = dn[e];
        }
        fence_before();
        __syncthreads();
        // (4) negative rows: -dN
        for (uint32_t j = warp; j < (uint32_t)KP; j += NW) {
            float4* nrow = reinterpret_cast<float4*>(p.C + (uint64_t)(s_neg[j] - p.c_begin) * D);
            for (uint32_t c = lane; c < KC; c += 32) {
                const float4 g = reinterpret_cast<const float4*>(stage + j * D)[c];
                atomicAdd(nrow + c, make_float4(-g.x, -g.y, -g.z, -g.w));
            }
        }
        __syncthreads();
        if (!ahead && bn < nbatch) prepare(buf ^ 1u, bn);
        buf ^= 1u;
        phase ^= 1u;
    }
    if (loss != 0.0) atomicAdd(p.loss, loss);
    fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// Test hook (ne_umma_products): the batch kernel's tiles, transposes and three
// products on dense row-major inputs V[128][D], N[KP][D], G[128][KP]; outputs
// S[128][KP], dV[128][D], dNt[D][KP] row-major.
template <int D, int KP>
__global__ void __launch_bounds__(kBatch, 1) umma_products_kernel(const float* __restrict__ V,
                                                                  const float* __restrict__ N,
                                                                  const float* __restrict__ G, float* __restrict__ S,
                                                                  float* __restrict__ dV, float* __restrict__ dNt) {
    using SM = BatchSmem<D, KP>;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sV = smem + SM::V, *sVt = smem + SM::Vt, *sN = smem + SM::N, *sNt = smem + SM::Nt,
                  *sG = smem + SM::G, *sGt = smem + SM::Gt;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::tail);
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(bar + 2);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_base)),
                     "n"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (uint32_t r = 0; r < kBatch; ++r)
        for (uint32_t c = tid; c < D / 4; c += kBatch)
            *reinterpret_cast<float4*>(sV + tile_off(r, c, D, kLboPad)) = reinterpret_cast<const float4*>(V + r * D)[c];
    for (uint32_t r = 0; r < (uint32_t)KP; ++r)
        for (uint32_t c = tid; c < D / 4; c += kBatch)
            *reinterpret_cast<float4*>(sN + tile_off(r, c, D, kLboPad)) = reinterpret_cast<const float4*>(N + r * D)[c];
    for (uint32_t r = 0; r < kBatch; ++r)
        for (uint32_t c = tid; c < KP / 4; c += kBatch)
            *reinterpret_cast<float4*>(sG + tile_off(r, c, KP)) = reinterpret_cast<const float4*>(G + r * KP)[c];
    __syncthreads();
    transpose_tile<kBatch, D>(sV, sVt, tid);
    transpose_tile<KP, D>(sN, sNt, tid);
    transpose_tile<kBatch, KP, kBatch, 128u, kLboPad>(sG, sGt, tid);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_base, t_S = tmem, t_dV = tmem + KP, t_dNt = tmem + KP + D;
    if (tid == 0) {
        issue_S<D, KP>(smem_u32(sV), smem_u32(sN), t_S);
        issue_dV<D, KP>(smem_u32(sG), smem_u32(sNt), t_dV);
        issue_dNt<D, KP>(smem_u32(sVt), smem_u32(sGt), t_dNt);
        mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    fence_after();
    const uint32_t lane_base = (warp * 32u) << 16;
    float v[32];
    for (uint32_t j0 = 0; j0 < (uint32_t)KP; j0 += 32) {
        tmem_ld32(t_S + lane_base + j0, v);
        for (uint32_t e = 0; e < 32; ++e) S[tid * KP + j0 + e] = v[e];
        tmem_ld32(t_dNt + lane_base + j0, v);
        for (uint32_t e = 0; e < 32; ++e) dNt[tid * KP + j0 + e] = v[e];
    }
    for (uint32_t d0 = 0; d0 < (uint32_t)D; d0 += 32) {
        tmem_ld32(t_dV + lane_base + d0, v);
        for (uint32_t e = 0; e < 32; ++e) dV[tid * D + d0 + e] = v[e];
    }
    fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256) : "memory");
}

// Diagnostics hook (ne_umma_raw): one product D[M][N] (M = 128) from raw
// shared-memory images of A and B (each up to 64 KB, copied verbatim),
// descriptors built from (lbo, sbo, layout type) with start advancing by
// a_step / b_step bytes per instruction, `ksteps` instructions, a given
// instruction descriptor.
__global__ void __launch_bounds__(kBatch, 1) umma_raw_kernel(const uint4* __restrict__ a_img,
                                                             const uint4* __restrict__ b_img, uint32_t img_u4,
                                                             uint64_t a_hi, uint64_t b_hi, uint32_t a_lbo, uint32_t a_sbo,
                                                             uint32_t b_lbo, uint32_t b_sbo, uint32_t a_step,
                                                             uint32_t b_step, uint32_t ksteps, uint32_t idesc,
                                                             uint32_t N, float* __restrict__ D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint4* sA = reinterpret_cast<uint4*>(smem);
    uint4* sB = sA + img_u4;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + img_u4);
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(bar + 2);
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_base)),
                     "n"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (uint32_t i = tid; i < img_u4; i += kBatch) {
        sA[i] = a_img[i];
        sB[i] = b_img[i];
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_base;
    if (tid == 0) {
        for (uint32_t ks = 0; ks < ksteps; ++ks) {
            const uint64_t a = umma_desc(smem_u32(sA) + ks * a_step, a_lbo, a_sbo) | a_hi;
            const uint64_t b = umma_desc(smem_u32(sB) + ks * b_step, b_lbo, b_sbo) | b_hi;
            mma_tf32(tmem, a, b, idesc, ks > 0);
        }
        mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    fence_after();
    float v[32];
    for (uint32_t j0 = 0; j0 < N; j0 += 32) {
        tmem_ld32(tmem + ((warp * 32u) << 16) + j0, v);
        for (uint32_t e = 0; e < 32 && j0 + e < N; ++e) D[tid * N + j0 + e] = v[e];
    }
    fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256) : "memory");
}

cudaError_t launch_umma_raw(const void* a_img, const void* b_img, uint32_t img_bytes, uint64_t a_hi, uint64_t b_hi,
                            uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo, uint32_t a_step,
                            uint32_t b_step, uint32_t ksteps, uint32_t idesc, uint32_t N, float* D, cudaStream_t s) {
    const size_t smem = 2ull * img_bytes + 64;
    cudaError_t e = cudaFuncSetAttribute(umma_raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    umma_raw_kernel<<<1, kBatch, smem, s>>>(static_cast<const uint4*>(a_img), static_cast<const uint4*>(b_img),
                                             img_bytes / 16, a_hi, b_hi, a_lbo, a_sbo, b_lbo, b_sbo, a_step, b_step,
                                             ksteps, idesc, N, D);
    return cudaGetLastError();
}

cudaError_t launch_umma_products(const float* V, const float* N, const float* G, float* S, float* dV, float* dNt,
                                 cudaStream_t s) {
    constexpr size_t smem = BatchSmem<128, 32>::bytes;
    auto kern = umma_products_kernel<128, 32>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<1, kBatch, smem, s>>>(V, N, G, S, dV, dNt);
    return cudaGetLastError();
}

template <int D, int KP>
static cudaError_t launch_batch(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    constexpr size_t smem = BatchSmem<D, KP>::bytes;
    auto kern = sgns_batch_kernel<D, KP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint64_t nbatch = (p.count + kBatch - 1) / kBatch;
    // Hogwild: one batch per CTA, at most p.max_warps concurrent batches (the
    // conflict cap, counted in batches for this rule)
    const uint64_t full = (uint64_t)std::max(1, dev.sm_count - p.reserve_sms);
    const unsigned grid = p.deterministic ? 1u : (unsigned)std::max<uint64_t>(
                                                     1, std::min<uint64_t>({nbatch, full, p.max_warps}));
    kern<<<grid, kBatchThreads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_sgns_batch(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if (p.count == 0) return cudaSuccess;
    if (p.d != 128 || p.bf16) return cudaErrorNotSupported;
    switch (p.K) {
        case 32: return launch_batch<128, 32>(p, dev, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace ne

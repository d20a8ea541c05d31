// kernels_sgns.cu -- the SGNS update of Alg. 1 on one 2D block
// (sm_100a).  Memory-bound gather/scatter ("O(1) arithmetic intensity"):
// per positive sample the kernel reads the vertex row, the positive context row
// and K negative context rows and writes all 2+K back -- 8d(2+K) bytes against
// 6d(1+K) flops -- so the design goal is bytes in flight, not FLOPs.
//
// Mapping: one warp per sample.  Each lane owns R float4 of every row
// (d <= 128 R), so a row is one coalesced 128-bit-per-lane access; all 2+K row
// loads are issued before the first dot product (they are independent), the
// 1+K updates then run back to back in registers (dot = per-lane FMA chain +
// 5-step xor-shuffle all-reduce; sigmoid; two FMAs per element), and the rows
// are written once.  Repeated context ids inside a sample are forwarded in
// registers so the result equals the sequential Alg. 1 order (reading D2).
// Negatives (O8) are drawn by lanes 0..K-1 in parallel (one Philox each) and
// broadcast with shuffles.  The next sample's pair and negatives (pool load,
// Philox, alias load) are fetched while the current sample's rows are in
// flight, so the dependent chain pair -> alias -> rows is off the critical path.
//
// Production mode: a persistent grid of warps strides over the block's
// samples, updating rows in place without locks (Hogwild; races only between
// concurrent samples sharing a row).  Deterministic mode: one warp walks the
// block in canonical order -- the same device code, so parity of the
// deterministic mode is parity of the production arithmetic.
// The kernel template lives in sgns_kernel.cuh; this file instantiates it for
// fp32 rows, kernels_sgns_bf16.cu for bf16 rows (NEXT-4).
#include "sgns_kernel.cuh"

namespace ne {

cudaError_t launch_sgns(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    if (p.count == 0) return cudaSuccess;
    if (p.accumulate == 2) return launch_sgns_batch(p, dev, s);  // NEXT-4 shared negatives (tcgen05)
    if (p.K > (uint32_t)kMaxK || p.d % 4 != 0 || p.d == 0 || p.d > 512) return cudaErrorInvalidValue;
    if (p.bf16) return launch_sgns_bf16(p, dev, s);
    return launch_sgns_rows<false>(p, dev, s);
}

__global__ void export_negatives_kernel(SgnsParams p, uint64_t pos_begin, uint64_t count,
                                        uint32_t* __restrict__ out) {
    const uint2 key = key_of(p.seed);
    const uint32_t tagw = tag_word(kTagNeg, p.epoch);
    const uint64_t total = count * p.K;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += stride) {
        const uint64_t i = w / p.K;
        out[w] = draw_negative(p, key, tagw, pos_begin + i, (uint32_t)(w - i * p.K));
    }
}

cudaError_t launch_export_negatives(const SgnsParams& p, uint64_t pos_begin, uint64_t count,
                                    uint32_t* out, const Device& dev, cudaStream_t s) {
    if (count == 0 || p.K == 0) return cudaSuccess;
    const uint64_t total = count * p.K;
    const unsigned g = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((total + 255) / 256, (uint64_t)dev.sm_count * 8));
    export_negatives_kernel<<<g, 256, 0, s>>>(p, pos_begin, count, out);
    return cudaGetLastError();
}

}  // namespace ne

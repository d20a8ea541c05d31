// kernels_sgns_bf16.cu -- the SGNS kernels for bf16 row storage (NEXT-4,
// DESIGN reading D16): the same template as kernels_sgns.cu with BF = true,
// instantiated in its own translation unit.
#include "sgns_kernel.cuh"

namespace ne {

cudaError_t launch_sgns_bf16(const SgnsParams& p, const Device& dev, cudaStream_t s) {
    return launch_sgns_rows<true>(p, dev, s);
}

}  // namespace ne

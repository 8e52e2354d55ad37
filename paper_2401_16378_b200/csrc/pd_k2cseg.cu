// pd_k2cseg.cu — the K2s-c kernel for final walk segments (raw partial sums in, coefficients out), in its own translation unit so that
// ptxas allocates it separately from the other instantiation (pd_k2share.cuh).
#include "pd_k2share.cuh"

namespace pdb {

cudaError_t launch_gray_share_c_seg(const K2Params& P, unsigned grid, cudaStream_t stream) {
    return launch_gray_share_c_impl<true>(P, grid, stream);
}

}  // namespace pdb

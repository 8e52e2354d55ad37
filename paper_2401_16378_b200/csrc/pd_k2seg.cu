// pd_k2seg.cu — the walk-segment instantiation of K2 (gray_xmask_kernel<4, true, false>), used by
// the pipelined host path. It is compiled on its own so that its ptxas schedule does not move
// the whole-walk instantiation in pd_kernels.cu (profiles/r01_k2_codegen.md); the Makefile
// gives this file its own ptxas options (K2SEG_FLAGS).
#include <cuda_runtime.h>

#include <atomic>

#include "pd_k2.cuh"

namespace pdb {

cudaError_t launch_gray_seg4(const K2Params& P, unsigned grid, size_t smem, cudaStream_t stream) {
    static std::atomic<uint64_t> attr_set{0};  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        const cudaError_t e = cudaFuncSetAttribute(gray_xmask_kernel<4, true, false>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kK2MaxSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    gray_xmask_kernel<4, true, false><<<grid, kK2Threads, smem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace pdb

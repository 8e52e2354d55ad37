// pd_shard.cu — data movement of the NCCL pipeline of the sharding layer (sharding.py).
//
// A rank's finished sub-block of X-masks owns 2^(p+q) runs of 4^(N-p-q) coefficients of the
// reference-ordered array (pd_run_offset). The sender packs them from its rank-level run buffer
// into one contiguous message and rank 0 unpacks each message into its place in the output:
// both are the same run copy with different offset tables (computed once per plan on the host).
#include <cuda_runtime.h>

#include <cstdint>

#include "pd_kernels.h"

namespace pdb {

namespace {

constexpr int kCopyThreads = 256;

// grid: (chunks of 4096 elements per run) x count runs; 16 B per thread per iteration
__global__ void __launch_bounds__(kCopyThreads)
    copy_runs_kernel(const double2* __restrict__ src, double2* __restrict__ dst, uint64_t run_len,
                     const uint64_t* __restrict__ src_off, const uint64_t* __restrict__ dst_off) {
    const uint64_t k = blockIdx.y;
    const double2* s = src + src_off[k];
    double2* d = dst + dst_off[k];
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kCopyThreads + threadIdx.x; j < run_len;
         j += static_cast<uint64_t>(gridDim.x) * kCopyThreads)
        __stcs(&d[j], __ldcs(&s[j]));
}

}  // namespace

cudaError_t launch_copy_runs(const double2* src, double2* dst, uint64_t run_len,
                             const uint64_t* src_off, const uint64_t* dst_off, uint64_t count,
                             cudaStream_t stream) {
    if (count == 0 || run_len == 0) return cudaSuccess;
    if (count > 65535) return cudaErrorInvalidValue;
    uint64_t gx = (run_len + kCopyThreads * 4 - 1) / (kCopyThreads * 4);  // ~4 elements per thread
    if (gx > 4096) gx = 4096;
    copy_runs_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(count)), kCopyThreads, 0,
                       stream>>>(src, dst, run_len, src_off, dst_off);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace pdb

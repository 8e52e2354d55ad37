// pd_io.cu — device side of the file path (§8f item 3): the finiteness check the reference's
// readers apply to every element (io.cpp:118-123, 214-218), and the ordered threshold
// selection of its coefficient writer (io.cpp:286-307), so that a decomposition can go from a
// pinned file buffer to a sparse coefficient list without a full D2H of 4^N coefficients.
#include <cuda_runtime.h>

#include <cstdint>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

// ---- first non-finite element (atomicMin of the index; UINT64_MAX when all finite) ----

__global__ void first_nonfinite_kernel(const double2* __restrict__ v, uint64_t count,
                                       unsigned long long* result) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double2 e = v[k];
        if (!isfinite(e.x) || !isfinite(e.y)) atomicMin(result, static_cast<unsigned long long>(k));
    }
}

cudaError_t launch_first_nonfinite(const double2* v, uint64_t count, unsigned long long* result,
                                   cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(result, 0xff, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    uint64_t grid = (count + 255) / 256;
    if (grid > 148ull * 16) grid = 148ull * 16;
    if (grid == 0) grid = 1;
    first_nonfinite_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(v, count, result);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

// ---- ordered selection of |c| > threshold: count per tile, scan tiles, scatter ----
// A tile is 4096 coefficients (256 threads x 16 consecutive). |c| is compared as
// hypot-free re^2 + im^2 > t^2 only when that is exact enough; to match std::abs (hypot)
// semantics bit for bit the kernel uses hypot() like the reference's std::abs(complex).

constexpr unsigned kSelThreads = 256;
constexpr unsigned kSelPer = 16;
constexpr unsigned kSelTile = kSelThreads * kSelPer;

__device__ __forceinline__ bool keep(const double2 c, double threshold) {
    return threshold <= 0.0 || hypot(c.x, c.y) > threshold;
}

__global__ void select_count_kernel(const double2* __restrict__ c, uint64_t count, double threshold,
                                    unsigned* tile_counts) {
    __shared__ unsigned warp_sums[kSelThreads / 32];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSelTile + threadIdx.x * kSelPer;
    unsigned n = 0;
#pragma unroll
    for (unsigned j = 0; j < kSelPer; ++j)
        if (base + j < count && keep(c[base + j], threshold)) ++n;
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (unsigned w = 0; w < kSelThreads / 32; ++w) t += warp_sums[w];
        tile_counts[blockIdx.x] = t;
    }
}

// exclusive scan of tile counts in one CTA (tiles <= a few 10^5); total to tile_offsets[tiles]
__global__ void select_scan_kernel(const unsigned* tile_counts, uint64_t tiles,
                                   unsigned long long* tile_offsets) {
    __shared__ unsigned long long carry;
    __shared__ unsigned long long warp_sums[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < tiles; base += blockDim.x) {
        const uint64_t k = base + threadIdx.x;
        unsigned long long v = k < tiles ? tile_counts[k] : 0;
        // inclusive warp scan
        unsigned long long x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= static_cast<unsigned>(o)) x += y;
        }
        if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long w = threadIdx.x < blockDim.x / 32 ? warp_sums[threadIdx.x] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= static_cast<unsigned>(o)) w += y;
            }
            warp_sums[threadIdx.x] = w;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before_warp = (threadIdx.x >= 32) ? warp_sums[(threadIdx.x >> 5) - 1] : 0;
        if (k < tiles) tile_offsets[k] = carry + before_warp + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_sums[blockDim.x / 32 - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_offsets[tiles] = carry;
}

__global__ void select_scatter_kernel(const double2* __restrict__ c, uint64_t count, double threshold,
                                      const unsigned long long* __restrict__ tile_offsets,
                                      uint64_t* __restrict__ idx_out, double2* __restrict__ val_out) {
    __shared__ unsigned warp_sums[kSelThreads / 32];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSelTile + threadIdx.x * kSelPer;
    unsigned mask = 0;
#pragma unroll
    for (unsigned j = 0; j < kSelPer; ++j)
        if (base + j < count && keep(c[base + j], threshold)) mask |= 1u << j;
    const unsigned n = __popc(mask);
    // exclusive scan of n over the CTA (thread order = coefficient order)
    unsigned x = n;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= static_cast<unsigned>(o)) x += y;
    }
    if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned before = 0;
    for (unsigned w = 0; w < (threadIdx.x >> 5); ++w) before += warp_sums[w];
    uint64_t pos = tile_offsets[blockIdx.x] + before + x - n;
    for (unsigned j = 0; j < kSelPer; ++j) {
        if (mask >> j & 1u) {
            idx_out[pos] = base + j;
            val_out[pos] = c[base + j];
            ++pos;
        }
    }
}

uint64_t select_tiles(uint64_t count) { return (count + kSelTile - 1) / kSelTile; }

cudaError_t launch_select(const double2* c, uint64_t count, double threshold, unsigned* tile_counts,
                          unsigned long long* tile_offsets, uint64_t* idx_out, double2* val_out,
                          cudaStream_t stream) {
    const uint64_t tiles = select_tiles(count);
    if (tiles == 0) return cudaMemsetAsync(tile_offsets, 0, sizeof(unsigned long long), stream);
    select_count_kernel<<<static_cast<unsigned>(tiles), kSelThreads, 0, stream>>>(c, count, threshold,
                                                                                  tile_counts);
    select_scan_kernel<<<1, 1024, 0, stream>>>(tile_counts, tiles, tile_offsets);
    select_scatter_kernel<<<static_cast<unsigned>(tiles), kSelThreads, 0, stream>>>(
        c, count, threshold, tile_offsets, idx_out, val_out);
    g_launches.fetch_add(3, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace pdb

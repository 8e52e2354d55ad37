// pd_nonfinite.cu — the reference's coefficients for X-masks whose diagonal holds an inf or NaN.
//
// The fast kernels (K2/K2s/K2s-c, K4) fold lambda = ±1, ±i into adds and re/im swaps. That is
// the reference's arithmetic for every finite element (decompose.cpp:40 multiplies by a unit
// whose other component is an exact 0), but not for an infinite or NaN one: the reference's
// complex product computes 0 * inf = NaN into the other component, and its libgcc fallback
// recovers infinities per C99 Annex G (cmul_annex_g in pd_device.cuh).
//
// Detection costs nothing on the fast path: the Z-mask-0 coefficient of X-mask x is the plain
// sum of D_x (lambda = 1 at every step, in both the Gray walk and the WHT's butterfly tree), so
// it is non-finite exactly when an element of D_x is (or the finite sum overflowed, where the
// recomputation reproduces the same values). After a fast kernel has written an X-mask range,
// this kernel reads one coefficient per X-mask and recomputes every coefficient of the X-masks
// that failed with the reference's per-step complex product, in the reference's order
// (exact_coeff). Finite matrices pay one launch that reads x_count coefficients.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

namespace {

constexpr int kFixThreads = 256;
constexpr int kFixGroup = 32;  // X-masks per CTA: one per lane of warp 0

// src rows: stride == 0 -> src + (x - x0) 2^N is D_x (gathered diagonals); stride == 2^N ->
// src is G itself and element i of X-mask x is G[i ^ x][i]
__global__ void __launch_bounds__(kFixThreads)
    nonfinite_fixup_kernel(const double2* __restrict__ src, uint64_t stride, unsigned N,
                           uint64_t x0, uint64_t x_count, OutMap map,
                           const unsigned* __restrict__ flags) {
    __shared__ unsigned todo;
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kFixGroup;
    if (threadIdx.x < 32) {
        const uint64_t xl = base + threadIdx.x;
        bool bad = false;
        if (xl < x_count) {
            if (flags) {
                bad = flags[xl] != 0u;
            } else {  // the X-mask's z = 0 coefficient: the sum of its whole diagonal
                const uint64_t x = x0 + xl;
                bad = !finite2(map.out[out_index(map, tensor_number(x, 0), 0)]);
            }
        }
        const unsigned m = __ballot_sync(~0u, bad);
        if (threadIdx.x == 0) todo = m;
    }
    __syncthreads();
    const unsigned todo_m = todo;
    __syncthreads();  // every thread has read the set before any coefficient (z = 0) changes
    const uint64_t dim = 1ull << N;
    for (unsigned m = todo_m; m; m &= m - 1) {
        const uint64_t xl = base + static_cast<unsigned>(__ffs(static_cast<int>(m)) - 1);
        const uint64_t x = x0 + xl;
        const double2* row = stride ? src : src + xl * dim;
        const auto elem = [=](uint64_t i) { return __ldg(&row[(i ^ x) * stride + i]); };
        for (uint64_t z = threadIdx.x; z < dim; z += kFixThreads)
            map.out[out_index(map, tensor_number(x, z), z)] = exact_coeff(elem, N, x, z);
    }
}

// flags[xl] = 1 if row xl of diag holds a non-finite element: one CTA per X-mask
__global__ void __launch_bounds__(kFixThreads)
    nonfinite_scan_kernel(const double2* __restrict__ diag, unsigned N, unsigned* __restrict__ flags) {
    const uint64_t dim = 1ull << N;
    const double2* row = diag + static_cast<uint64_t>(blockIdx.x) * dim;
    bool ok = true;
    for (uint64_t i = threadIdx.x; i < dim; i += kFixThreads) ok &= finite2(__ldcs(&row[i]));
    const int all_ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) flags[blockIdx.x] = all_ok ? 0u : 1u;
}

}  // namespace

cudaError_t launch_nonfinite_fixup(const double2* src, bool from_matrix, unsigned N, uint64_t x0,
                                   uint64_t x_count, const OutMap& map, const unsigned* flags,
                                   cudaStream_t stream) {
    if (x_count == 0) return cudaSuccess;
    const uint64_t grid = (x_count + kFixGroup - 1) / kFixGroup;
    nonfinite_fixup_kernel<<<static_cast<unsigned>(grid), kFixThreads, 0, stream>>>(
        src, from_matrix ? (1ull << N) : 0ull, N, x0, x_count, map, flags);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_nonfinite_scan(const double2* diag, unsigned N, uint64_t x_count, unsigned* flags,
                                  cudaStream_t stream) {
    if (x_count == 0) return cudaSuccess;
    nonfinite_scan_kernel<<<static_cast<unsigned>(x_count), kFixThreads, 0, stream>>>(diag, N, flags);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

// The library's own stream-ordered pool, one per device: per-call scratch (string buckets,
// flags) costs a pool lookup instead of a driver allocation, without changing the release
// policy of the device's default pool that the host application's allocations share.
namespace {
struct Pools {
    std::mutex mu;
    cudaMemPool_t pool[64] = {};
};
Pools& pools() {
    static Pools p;
    return p;
}
}  // namespace

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = nullptr;
    {
        Pools& ps = pools();
        std::lock_guard<std::mutex> lk(ps.mu);
        cudaMemPool_t& slot = ps.pool[dev & 63];
        if (!slot) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&slot, &props);
            if (e != cudaSuccess) {
                slot = nullptr;
                return e;
            }
            uint64_t keep = 64ull << 20;  // keep up to 64 MiB between calls
            cudaMemPoolSetAttribute(slot, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = slot;
    }
    return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, stream);
}

cudaError_t pool_free(void* p, cudaStream_t stream) { return p ? cudaFreeAsync(p, stream) : cudaSuccess; }

}  // namespace pdb

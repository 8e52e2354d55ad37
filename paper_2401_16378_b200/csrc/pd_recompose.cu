// pd_recompose.cu — recompose (decompose.cpp:221-250) on the device: G = sum_n c_n P_n.
//
// The reference walks every nonzero coefficient in reverse (row r receives
// lambda_r c_n at column r ^ mask). Grouped by X-mask x this is, for every x,
//     G[r][r ^ x] = sum_z (-1)^{|r & z|} (-i)^{|x & z|} c_{n(x,z)},
// a Walsh-Hadamard transform over z. So: gather the phased coefficients of each x
// into a row, transform the rows in place (pd_wht.cu), and scatter row x back onto
// the x-th XOR diagonal of G with the tile transpose of K1 run backwards.
// Summation order differs from the reference: parity is to rounding (1e-12 level).
#include <cuda_runtime.h>

#include <cstdint>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

__global__ void __launch_bounds__(256)
    recompose_gather_kernel(const double2* __restrict__ coeffs, unsigned N, double2* __restrict__ rows) {
    const uint64_t total = 1ull << (2 * N);
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t x = k >> N, z = k & ((1ull << N) - 1);
        const double2 c = coeffs[tensor_number(x, z)];
        const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
        rows[k] = apply_phase(ph, c.x, c.y, 1.0);
    }
}

// tile (row block Rb, X-mask block xh): for xl < T, r < T the element
// E[xh T + xl][Rb T + r] lands at G[Rb T + r][(Rb ^ xh) T + (r ^ xl)]
__global__ void __launch_bounds__(256)
    recompose_scatter_kernel(const double2* __restrict__ rows, unsigned N, unsigned t_log,
                             double2* __restrict__ G) {
    __shared__ double2 tile[32 * 33];  // padded rows: the transposed read is conflict-free
    const unsigned T = 1u << t_log, P = T + 1;
    const uint64_t dim = 1ull << N;
    const uint64_t blocks_log = N - t_log;
    const uint64_t rb = static_cast<uint64_t>(blockIdx.x) & ((1ull << blocks_log) - 1);
    const uint64_t xh = static_cast<uint64_t>(blockIdx.x) >> blocks_log;
    const uint64_t cb = rb ^ xh;
    for (unsigned e = threadIdx.x; e < T * T; e += 256) {
        const unsigned xl = e >> t_log, r = e & (T - 1);
        tile[xl * P + r] = rows[((xh << t_log) + xl) * dim + (rb << t_log) + r];
    }
    __syncthreads();
    for (unsigned e = threadIdx.x; e < T * T; e += 256) {
        const unsigned r = e >> t_log, c = e & (T - 1);
        G[((rb << t_log) + r) * dim + (cb << t_log) + c] = tile[(r ^ c) * P + r];
    }
}

cudaError_t launch_recompose_gather(const double2* coeffs, unsigned N, double2* rows,
                                    cudaStream_t stream) {
    const uint64_t total = 1ull << (2 * N);
    uint64_t grid = (total + 255) / 256;
    if (grid > 148ull * 32) grid = 148ull * 32;
    recompose_gather_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(coeffs, N, rows);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_recompose_scatter(const double2* rows, unsigned N, double2* G,
                                     cudaStream_t stream) {
    const unsigned t_log = N < 5 ? N : 5;
    const uint64_t grid = 1ull << (2 * (N - t_log));
    recompose_scatter_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(rows, N, t_log, G);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace pdb

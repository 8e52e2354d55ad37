// tile_read_probe.cu — HBM read rate of the XOR-diagonal tile pattern at several tile edges.
//
// Reading the x-diagonals of G through T x T tiles (row block R, column block C = R ^ xh) means
// every tile row is a contiguous T * 16 B segment, rows 2^N * 16 B apart. K1 uses T = 32
// (512 B segments). A WHT whose pass-1 output stays on chip would need T = 8 (128 B) or T = 4
// (64 B). This probe reads all of G (N=14, 4 GiB) once in that pattern and reports GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/trp tile_read_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

// a warp load covers 32 lanes x 16 B = 512 B: 32 / T row segments (T <= 32) taken in order of
// (tile, row), tile t = (xh, C) with R = C ^ xh; U loads in flight per lane
template <int T, int U>
__global__ void __launch_bounds__(256) tile_read(const double2* __restrict__ G, unsigned N, double* sink) {
    const uint64_t dim = 1ull << N;
    const uint64_t tiles_per_dim = dim / T;
    const uint64_t total_segs = tiles_per_dim * tiles_per_dim * T;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * 8 + warp;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * 8;
    constexpr unsigned SPW = 32 / T;  // segments per warp load
    double acc = 0.0;
    for (uint64_t s0 = gwarp * SPW * U; s0 < total_segs; s0 += nwarps * SPW * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t seg = s0 + u * SPW + lane / T;
            const uint64_t tile = seg / T, row = seg % T;
            const uint64_t C = tile % tiles_per_dim, xh = tile / tiles_per_dim, R = C ^ xh;
            v[u] = seg < total_segs ? __ldcs(&G[(R * T + row) * dim + C * T + lane % T]) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 12345.678) sink[0] = acc;
}

template <int T, int U>
float run(const double2* G, unsigned N, double* sink, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    tile_read<T, U><<<grid, 256>>>(G, N, sink);
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) tile_read<T, U><<<grid, 256>>>(G, N, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    const unsigned N = 14;
    const size_t bytes = size_t{16} << (2 * N);
    double2* G = nullptr;
    double* sink = nullptr;
    cudaMalloc(&G, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(G, 0, bytes);
    for (int grid : {148 * 2, 148 * 4, 148 * 8}) {
        printf("grid %d CTAs x 256\n", grid);
#define R(T, U)                                                                                  \
    {                                                                                            \
        const float ms = run<T, U>(G, N, sink, grid);                                            \
        printf("  T=%2d (%3d B rows), %2d loads in flight per lane: %7.3f ms = %6.0f GB/s\n", T, T * 16, U, ms, \
               bytes / (ms * 1e6));                                                              \
    }
        R(32, 4) R(32, 8) R(16, 4) R(16, 8) R(8, 4) R(8, 8) R(8, 16) R(4, 4) R(4, 8) R(4, 16)
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

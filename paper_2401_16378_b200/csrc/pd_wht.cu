// pd_wht.cu — K4, the fast Walsh-Hadamard path (reported separately from K2).
//
// Same contract as K2 (all coefficients of the X-masks [x0, x0 + x_count), run
// addressing of pd_api.h), but S_{x,.} = H_{2^N} D_x is evaluated with N butterfly
// stages (N 2^N complex adds per X-mask instead of 4^N), so the path is HBM bound.
// The summation order differs from the reference's Gray walk: results agree within
// rounding (bit-exact only for inputs whose partial sums are exact).
//
// Split i = (ih, il), il = the low L = min(N, 12) bits (4096 complex = 64 KiB of smem):
//   pass 1: one CTA per (x, ih) runs the L low butterfly stages in shared memory;
//           with no high bits it applies the phase and writes coefficients,
//           otherwise it writes the row back in place into the diagonal buffer;
//   pass 2: one thread per (x, il) runs the N - L high stages in registers over the
//           2^(N-L) rows and writes coefficients.
#include <cuda_runtime.h>

#include <cstdint>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

namespace {

constexpr int kWhtThreads = 256;
constexpr unsigned kWhtMaxL = 12;

struct Runs {
    double2* ptr[kMaxRuns];
};

__device__ __forceinline__ void store_coeff(const Runs& runs, unsigned N, unsigned run_bits,
                                            uint64_t x, uint64_t z, double sr, double si,
                                            double scale) {
    const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
    const uint64_t n = tensor_number(x, z);
    const unsigned low_bits = 2 * (N - run_bits);
    const uint64_t low_mask = (low_bits >= 64) ? ~0ull : ((1ull << low_bits) - 1);
    const unsigned run = static_cast<unsigned>(z >> (N - run_bits));
    double2* p = runs.ptr[0];
#pragma unroll
    for (unsigned r = 1; r < kMaxRuns; ++r)
        if (run == r) p = runs.ptr[r];
    p[n & low_mask] = apply_phase(ph, sr, si, scale);
}

__global__ void __launch_bounds__(kWhtThreads)
    wht_rows_kernel(double2* __restrict__ diag, unsigned N, unsigned L, uint64_t x0,
                    unsigned run_bits, Runs runs, double scale, int final_pass) {
    // final_pass != 0: emit coefficients; otherwise write the transformed row back
    extern __shared__ __align__(16) double2 row[];
    const uint64_t dim = 1ull << N;
    const unsigned len = 1u << L;
    const uint64_t rows_log = N - L;
    const uint64_t xl = static_cast<uint64_t>(blockIdx.x) >> rows_log;
    const uint64_t ih = static_cast<uint64_t>(blockIdx.x) & ((1ull << rows_log) - 1);
    double2* src = diag + xl * dim + (ih << L);
    for (unsigned j = threadIdx.x; j < len; j += kWhtThreads) row[j] = src[j];
    __syncthreads();
    // radix-2 stages; stage h pairs (j, j + h) with j's bit log2(h) clear
    for (unsigned h = 1; h < len; h <<= 1) {
        for (unsigned q = threadIdx.x; q < len / 2; q += kWhtThreads) {
            const unsigned j = ((q & ~(h - 1)) << 1) | (q & (h - 1));
            const double2 a = row[j], b = row[j + h];
            row[j] = make_double2(a.x + b.x, a.y + b.y);
            row[j + h] = make_double2(a.x - b.x, a.y - b.y);
        }
        __syncthreads();
    }
    if (final_pass) {
        const uint64_t x = x0 + xl;
        for (unsigned j = threadIdx.x; j < len; j += kWhtThreads)
            store_coeff(runs, N, run_bits, x, j, row[j].x, row[j].y, scale);
    } else {
        for (unsigned j = threadIdx.x; j < len; j += kWhtThreads) src[j] = row[j];
    }
}

template <int R>  // R = N - L high bits
__global__ void __launch_bounds__(kWhtThreads)
    wht_cols_kernel(double2* __restrict__ diag, unsigned N, unsigned L, uint64_t x0,
                    uint64_t x_count, unsigned run_bits, Runs runs, double scale, int emit) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * kWhtThreads + threadIdx.x;
    const uint64_t cols = 1ull << L;
    if (t >= x_count * cols) return;
    const uint64_t xl = t >> L, il = t & (cols - 1);
    const uint64_t dim = 1ull << N;
    double2 v[1 << R];
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) v[r] = diag[xl * dim + (static_cast<uint64_t>(r) << L) + il];
#pragma unroll
    for (int h = 1; h < (1 << R); h <<= 1) {
#pragma unroll
        for (int j = 0; j < (1 << R); ++j) {
            if (j & h) continue;
            const double2 a = v[j], b = v[j + h];
            v[j] = make_double2(a.x + b.x, a.y + b.y);
            v[j + h] = make_double2(a.x - b.x, a.y - b.y);
        }
    }
    if (!emit) {
#pragma unroll
        for (int r = 0; r < (1 << R); ++r) diag[xl * dim + (static_cast<uint64_t>(r) << L) + il] = v[r];
        return;
    }
    const uint64_t x = x0 + xl;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r)
        store_coeff(runs, N, run_bits, x, (static_cast<uint64_t>(r) << L) | il, v[r].x, v[r].y,
                    scale);
}

}  // namespace

// shared driver: rows pass, then (N > 12) the column pass; emit != 0 writes
// coefficients through `runs`, emit == 0 leaves the transform in place in `buf`
static cudaError_t wht_passes(double2* buf, unsigned N, uint64_t x0, uint64_t x_count,
                              unsigned run_bits, const Runs& runs, int emit, cudaStream_t stream) {
    const unsigned L = N < kWhtMaxL ? N : kWhtMaxL;
    const unsigned R = N - L;
    if (R > 4) return cudaErrorInvalidValue;  // N <= 16
    const double scale = 1.0 / static_cast<double>(1ull << N);
    static std::atomic<uint64_t> attr_set{0};  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        cudaError_t e = cudaFuncSetAttribute(wht_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(double2) << kWhtMaxL));
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    const uint64_t grid1 = x_count << R;
    wht_rows_kernel<<<static_cast<unsigned>(grid1), kWhtThreads, sizeof(double2) << L, stream>>>(
        buf, N, L, x0, run_bits, runs, scale, emit && R == 0);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || R == 0) return e;
    const unsigned grid2 = static_cast<unsigned>(((x_count << L) + kWhtThreads - 1) / kWhtThreads);
    switch (R) {
        case 1: wht_cols_kernel<1><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, run_bits, runs, scale, emit); break;
        case 2: wht_cols_kernel<2><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, run_bits, runs, scale, emit); break;
        case 3: wht_cols_kernel<3><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, run_bits, runs, scale, emit); break;
        default: wht_cols_kernel<4><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, run_bits, runs, scale, emit); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_wht_xmask(const double2* diag_c, unsigned N, uint64_t x0, uint64_t x_count,
                             unsigned run_bits, double2* const* run_out, cudaStream_t stream) {
    // the passes rewrite the diagonal rows in place (they are scratch owned by the caller)
    Runs runs{};
    for (unsigned r = 0; r < (1u << run_bits); ++r) runs.ptr[r] = run_out[r];
    return wht_passes(const_cast<double2*>(diag_c), N, x0, x_count, run_bits, runs, 1, stream);
}

cudaError_t launch_wht_inplace(double2* rows, unsigned N, uint64_t x_count, cudaStream_t stream) {
    Runs runs{};
    return wht_passes(rows, N, 0, x_count, 0, runs, 0, stream);
}

}  // namespace pdb

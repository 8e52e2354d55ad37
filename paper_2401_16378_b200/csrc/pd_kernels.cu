// pd_kernels.cu — the sm_100a kernels of the B200 Pauli decomposition.
//
//   K0/K3  walk_kernel        one thread per tensor number, reference-order Gray walk
//                             straight from G (coeff_fast / coeff_slow restated,
//                             decompose.cpp:30-80); bit-identical to the reference.
//   K1     diag_gather_kernel D[x][i] = G[i^x][i] as an XOR-permuted 32x32 tile
//                             transpose: coalesced 512 B row reads and writes (HBM bound).
//   K2     gray_xmask_kernel  for each X-mask x, all 2^N Z-mask coefficients by the
//                             paper's Gray-code sign recurrence over the staged diagonal;
//                             FP64-add bound, no multiplies in the inner loop.
//   K5     random_matrix_kernel  the reference's splitmix64 generator (bench.cpp:16-58).
//   probe  fp64_add_probe_kernel  pure-DADD issue probe for the FP64 roofline.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "pd_device.cuh"
#include "pd_k2.cuh"
#include "pd_kernels.h"

namespace pdb {

std::atomic<uint64_t> g_launches{0};

static inline cudaError_t count_launch() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

// ============================================================================
// K2: Gray-code FP64 kernel
// ============================================================================
//
// Work split. For X-mask x the coefficient of Z-mask z is
//     S_{x,z} = sum_k s_k(z) D_x[g_k],   s_k(z) = (-1)^{|g_k & z|}.
// A thread owns one x and 2^K Z-masks z = (zh << K) | zl, zl = 0..2^K-1, each in
// its own register accumulator pair (re, im). Split the walk index k = (kh << K) | p:
// g_k = (gray(kh) << K) | (gray(p) ^ (kh & 1) << (K-1)), so
//     s_k(z) = (-1)^{|gray(kh) & zh|} * (-1)^{|il & zl|},   il = low K bits of g_k.
// The first factor is a per-thread runtime sign carried by the Gray recurrence
// (flip when bit ctz(kh) of zh is set — bits.hpp:42-44 / pauli.hpp:112-114 restated
// one level up) and XORed into the sign bit of each loaded element; the second is
// a compile-time constant of the unrolled (p, zl) pair, so it becomes a DADD vs.
// DADD-with-negated-operand choice: no branches, no multiplies.
//
// Summation order. Every accumulator is one sequential chain visiting k = 0..2^N-1
// in exactly the reference's order (even kh: gray(p); odd kh: gray(p) ^ 2^(K-1)),
// and -1/±i factors are exact, so S and hence c_n are bit-identical to the
// reference's coeff_fast for finite inputs (up to the sign of an exact zero).
//
// Staging. The CTA's diagonals are streamed through shared memory with 1-D bulk
// copies on the TMA engine (cp.async.bulk + mbarrier complete_tx), double
// buffered; an aligned run of C consecutive Gray steps covers the contiguous
// i-range [gray(c) C, gray(c) C + C), so each stage is one contiguous copy per x.
// Every lane of a warp reads the same element (LDS.128 broadcast) when the warp
// shares one x (N >= K + 5).

// K2 constants, K2Params and gray_xmask_kernel are in pd_k2.cuh.

template <int K>
static cudaError_t launch_gray(const K2Params& P0, cudaStream_t stream) {
    K2Geometry g = k2_geometry(P0.N, K, P0.x_count);
    if (P0.ci_log && g.xc_log == 0 && P0.ci_log < g.ci_log && P0.ci_log > static_cast<unsigned>(K)) {
        g.ci_log = P0.ci_log;  // shorter walk chunks (the host pipeline's first segments)
        g.nchunks = 1u << (P0.N - g.ci_log);
        g.smem_bytes = 2 * (sizeof(double2) << g.ci_log) + kK2BarBytes;
    }
    static std::atomic<uint64_t> attr_set{0};  // per instantiation, one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        cudaError_t e = cudaSuccess;
        for (auto k : {gray_xmask_kernel<K, false, false>, gray_xmask_kernel<K, false, true>,
                       gray_xmask_kernel<K, true, true>})
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kK2MaxSmem);
        if constexpr (K != 4) {
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(gray_xmask_kernel<K, true, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kK2MaxSmem);
        }
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    K2Params P = P0;
    P.tpx_log = g.tpx_log;
    P.xc_log = g.xc_log;
    P.cpx_log = g.cpx_log;
    P.ci_log = g.ci_log;
    if (P.c_end == 0 || P.c_end > g.nchunks) P.c_end = g.nchunks;
    if (P.c_begin >= P.c_end) return cudaErrorInvalidValue;
    P.scale = 1.0 / static_cast<double>(1ull << P.N);
    const bool seg = P.c_begin != 0 || P.c_end != g.nchunks || P.part_in || P.part_out;
    const bool mapped = P.run_bits > kRunPtrBits;
    if constexpr (K == 4) {
        static const char* share_env = std::getenv("PD_K2SHARE");
        if (!(share_env && share_env[0] == '0') && gray_share_ok(P.N, P.run_bits)) {
            const cudaError_t e = launch_gray_share(P, seg, static_cast<unsigned>(g.grid), g.smem_bytes, stream);
            return e != cudaSuccess ? e : count_launch();
        }
        if (seg && !mapped) {
            const cudaError_t e = launch_gray_seg4(P, static_cast<unsigned>(g.grid), g.smem_bytes, stream);
            return e != cudaSuccess ? e : count_launch();
        }
        auto kern = seg ? gray_xmask_kernel<K, true, true>
                        : (mapped ? gray_xmask_kernel<K, false, true> : gray_xmask_kernel<K, false, false>);
        kern<<<static_cast<unsigned>(g.grid), kK2Threads, g.smem_bytes, stream>>>(P);
    } else {
        auto kern = seg ? (mapped ? gray_xmask_kernel<K, true, true> : gray_xmask_kernel<K, true, false>)
                        : (mapped ? gray_xmask_kernel<K, false, true> : gray_xmask_kernel<K, false, false>);
        kern<<<static_cast<unsigned>(g.grid), kK2Threads, g.smem_bytes, stream>>>(P);
    }
    return count_launch();
}

cudaError_t launch_gray_segment(const double2* diag, unsigned N, uint64_t x0, uint64_t x_count,
                                unsigned c_begin, unsigned c_end, const double2* part_in,
                                double2* part_out, unsigned run_bits, double2* out, int layout,
                                cudaStream_t stream, unsigned chunk_log) {
    K2Params P{};
    P.ci_log = chunk_log;
    P.diag = diag;
    P.x0 = x0;
    P.x_count = x_count;
    P.N = N;
    P.c_begin = c_begin;
    P.c_end = c_end;
    P.part_in = part_in;
    P.part_out = part_out;
    P.map = make_outmap(out, N, run_bits, layout);
    P.run_bits = run_bits;
    if (run_bits <= kRunPtrBits) {
        const uint64_t shard = run_bits ? (x0 >> (N - run_bits)) : 0;
        const unsigned low_bits = 2 * (N - run_bits);
        for (unsigned r = 0; r < (1u << run_bits); ++r)
            P.runs.ptr[r] = out + (layout ? (static_cast<uint64_t>(r) << low_bits)
                                          : (tensor_number(shard, r) << low_bits));
    }
    switch (N < 4 ? N : 4) {
        case 1: return launch_gray<1>(P, stream);
        case 2: return launch_gray<2>(P, stream);
        case 3: return launch_gray<3>(P, stream);
        default: return launch_gray<4>(P, stream);
    }
}

cudaError_t launch_gray_xmask(const double2* diag, unsigned N, uint64_t x0, uint64_t x_count,
                              unsigned run_bits, double2* out, int layout, cudaStream_t stream) {
    return launch_gray_segment(diag, N, x0, x_count, 0, 0, nullptr, nullptr, run_bits, out, layout,
                               stream);
}

unsigned gray_xmask_chunks(unsigned N) { return k2_geometry(N, N < 4 ? N : 4, 1).nchunks; }

uint64_t gray_xmask_grid(unsigned N, uint64_t x_count) {
    return k2_geometry(N, N < 4 ? N : 4, x_count).grid;
}

// ============================================================================
// K1: XOR-diagonal gather  D[x - x0][i] = G[i ^ x][i]
// ============================================================================
// Tile (row block R, column block C) of T x T elements holds, at (r, c), the
// element of X-mask ((R ^ C) T) | (r ^ c) and column i = C T + c. So loading the
// tile G[R T .. R T + T)[C T .. C T + T) with coalesced row reads and writing
// row x_l of D's tile as tile[x_l ^ c][c] gives coalesced writes too. Bank
// pattern of the permuted read: lanes c and c' hit the same banks only if
// c = c' mod 8, i.e. the 4 wavefronts a 512 B LDS.128 needs anyway.

constexpr int kK1Threads = 256;

__global__ void __launch_bounds__(kK1Threads)
    diag_gather_kernel(const double2* __restrict__ G, unsigned N, uint64_t x0, unsigned t_log,
                       uint64_t col_blocks_log, uint64_t cb_begin, double2* __restrict__ diag) {
    __shared__ double2 tile[32 * 32];
    const unsigned T = 1u << t_log;
    const uint64_t dim = 1ull << N;
    const uint64_t bid = blockIdx.x;
    const uint64_t cb = cb_begin + (bid & ((1ull << col_blocks_log) - 1));
    const uint64_t xb = bid >> col_blocks_log;          // local x block
    const uint64_t xh = (x0 >> t_log) + xb;             // global x block
    const uint64_t rb = cb ^ xh;                        // row block
    const unsigned elems = T * T;
    for (unsigned e = threadIdx.x; e < elems; e += kK1Threads) {
        const unsigned r = e >> t_log, c = e & (T - 1);
        tile[r * T + c] = __ldcs(&G[((rb << t_log) + r) * dim + (cb << t_log) + c]);
    }
    __syncthreads();
    for (unsigned e = threadIdx.x; e < elems; e += kK1Threads) {
        const unsigned xl = e >> t_log, c = e & (T - 1);
        diag[((xb << t_log) + xl) * dim + (cb << t_log) + c] = tile[(xl ^ c) * T + c];
    }
}

cudaError_t launch_diag_gather_cols(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                    uint64_t col0, uint64_t cols, double2* diag, cudaStream_t stream) {
    unsigned t_log = N < 5 ? N : 5;
    while ((1ull << t_log) > x_count || (1ull << t_log) > cols) --t_log;  // powers of two
    const uint64_t col_blocks_log = 63 - __builtin_clzll(cols >> t_log);
    const uint64_t grid = (x_count >> t_log) << col_blocks_log;
    diag_gather_kernel<<<static_cast<unsigned>(grid), kK1Threads, 0, stream>>>(
        G, N, x0, t_log, col_blocks_log, col0 >> t_log, diag);
    return count_launch();
}

cudaError_t launch_diag_gather(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                               double2* diag, cudaStream_t stream) {
    return launch_diag_gather_cols(G, N, x0, x_count, 0, 1ull << N, diag, stream);
}

// ============================================================================
// K0 / K3: one thread per tensor number, the reference's walk straight from G
// ============================================================================
// Visits k = 0..2^N-1 in the reference's order (decompose.cpp:38-43), in blocks
// of 2^B steps so that 2^B independent loads are in flight per thread. The sign
// of step k is (-1)^{|g_k & z|}: for the fast variant the block part is carried
// by the Gray recurrence, for the slow variant (coeff_slow, decompose.cpp:59-80)
// it is recomputed from scratch every step; both give identical sums.

template <bool SLOW, int B, bool ODD>
__device__ __forceinline__ void walk_block(const double2* __restrict__ G, uint64_t dim, uint64_t x,
                                           uint64_t z, uint64_t ih, unsigned sgn_hi, double& sr,
                                           double& si) {
    double2 e[1 << B];
#pragma unroll
    for (int p = 0; p < (1 << B); ++p) {
        constexpr int kHalf = B > 0 ? (1 << (B - 1)) : 0;
        const uint64_t i = (ih << B) | static_cast<uint64_t>(cgray(p) ^ (ODD ? kHalf : 0));
        e[p] = __ldg(&G[(i ^ x) * dim + i]);
    }
#pragma unroll
    for (int p = 0; p < (1 << B); ++p) {
        constexpr int kHalf = B > 0 ? (1 << (B - 1)) : 0;
        const unsigned il = cgray(p) ^ (ODD ? kHalf : 0);
        unsigned sgn;
        if (SLOW) {
            const uint64_t i = (ih << B) | il;
            sgn = static_cast<unsigned>(__popcll(i & z) & 1) << 31;
        } else {
            sgn = sgn_hi ^ (static_cast<unsigned>(__popc(il & static_cast<unsigned>(z)) & 1) << 31);
        }
        sr += flip_sign(e[p].x, sgn);
        si += flip_sign(e[p].y, sgn);
    }
}

template <bool SLOW, int B>
__global__ void __launch_bounds__(128)
    walk_kernel(const double2* __restrict__ G, unsigned N, const uint64_t* __restrict__ ns,
                uint64_t count, double2* __restrict__ out, double scale, uint64_t row_stride,
                const uint32_t* __restrict__ slot) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= count) return;
    if (slot) G += static_cast<uint64_t>(slot[k]) << N;  // compact diagonals, one per X-mask
    const uint64_t n = ns ? ns[k] : k;
    const uint64_t dim = 1ull << N;
    const uint64_t x = xmask_of(n), z = zmask_of(n);
    double sr = 0.0, si = 0.0;
    unsigned sgn_hi = 0;
    const uint64_t nblocks = dim >> B;
    const uint64_t zh = z >> B;
    for (uint64_t kh = 0; kh < nblocks; kh += 2) {
        if (kh != 0) sgn_hi ^= static_cast<unsigned>((zh >> (__ffsll(static_cast<long long>(kh)) - 1)) & 1) << 31;
        walk_block<SLOW, B, false>(G, row_stride, x, z, gray(kh), sgn_hi, sr, si);
        if (kh + 1 < nblocks) {
            sgn_hi ^= static_cast<unsigned>((zh >> (__ffsll(static_cast<long long>(kh + 1)) - 1)) & 1) << 31;
            walk_block<SLOW, B, true>(G, row_stride, x, z, gray(kh + 1), sgn_hi, sr, si);
        }
    }
    const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
    double2 c = apply_phase(ph, sr, si, scale);
    if (!finite2(c)) {
        // an inf or NaN on the diagonal (a finite one cannot make the sum non-finite without
        // overflow, where both arithmetics agree): the reference's complex products instead
        const auto elem = [=](uint64_t i) { return __ldg(&G[(i ^ x) * row_stride + i]); };
        c = exact_coeff(elem, N, x, z);
    }
    out[k] = c;
}

// row_stride = 2^N walks G itself; row_stride = 0 walks a compact diagonal D[i] = G[i ^ x][i]
// of the (single) string's X-mask
template <bool SLOW>
static cudaError_t launch_walk_t(const double2* G, unsigned N, const uint64_t* ns, uint64_t count,
                                 double2* out, uint64_t row_stride, cudaStream_t stream,
                                 const uint32_t* slot = nullptr) {
    const double scale = 1.0 / static_cast<double>(1ull << N);
    const unsigned threads = 128;
    const uint64_t grid = (count + threads - 1) / threads;
    switch (N < 3 ? N : 3) {
        case 1: walk_kernel<SLOW, 1><<<static_cast<unsigned>(grid), threads, 0, stream>>>(G, N, ns, count, out, scale, row_stride, slot); break;
        case 2: walk_kernel<SLOW, 2><<<static_cast<unsigned>(grid), threads, 0, stream>>>(G, N, ns, count, out, scale, row_stride, slot); break;
        default: walk_kernel<SLOW, 3><<<static_cast<unsigned>(grid), threads, 0, stream>>>(G, N, ns, count, out, scale, row_stride, slot); break;
    }
    return count_launch();
}

cudaError_t launch_walk_slots(const double2* D, unsigned N, const uint64_t* ns, const uint32_t* slot,
                              uint64_t count, double2* out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    return launch_walk_t<false>(D, N, ns, count, out, 0, stream, slot);
}

// One string over its gathered diagonal, latency-optimised: the walk is one dependent chain per
// component, so a single thread sums while the CTA streams the diagonal through two shared-
// memory stages (cp.async) in walk order (an aligned run of C Gray steps covers the contiguous
// range [gray(c) C, gray(c) C + C)). Same order, same result as walk_kernel, bit for bit.
constexpr int kW1Threads = 256;
constexpr unsigned kW1ChunkLog = 12;  // 4096 elements = 64 KiB per stage

__global__ void __launch_bounds__(kW1Threads)
    walk_one_kernel(const double2* __restrict__ D, unsigned N, const uint64_t* __restrict__ np,
                    double2* __restrict__ out, double scale) {
    extern __shared__ __align__(16) double2 st[];  // 2 stages
    const uint64_t dim = 1ull << N;
    const unsigned clog = N < kW1ChunkLog ? N : kW1ChunkLog;
    const uint64_t C = 1ull << clog, nchunks = dim >> clog;
    const uint64_t n = *np;
    const uint64_t x = xmask_of(n), z = zmask_of(n);
    auto stage_in = [&](uint64_t c, unsigned s) {
        const double2* src = D + (gray(c) << clog);
        for (uint64_t i = threadIdx.x; i < C; i += kW1Threads) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(st + s * C + i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + i) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage_in(0, 0);
    double sr = 0.0, si = 0.0;
    unsigned sgn_hi = 0;
    const uint64_t zh = z >> 4;
    const unsigned zl = static_cast<unsigned>(z) & 15u;
    unsigned sw[16];
#pragma unroll
    for (int il = 0; il < 16; ++il) sw[il] = static_cast<unsigned>(__popc(static_cast<unsigned>(il) & zl) & 1) << 31;
    for (uint64_t c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            stage_in(c + 1, (c + 1) & 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double2* base = st + (c & 1) * C;
            const uint64_t kh0 = c << (clog - 4 < 64 ? clog - 4 : 0);
            auto block = [&](uint64_t kh, auto odd) {
                constexpr unsigned kOdd = decltype(odd)::value ? 8u : 0u;
                if (kh != 0) sgn_hi ^= static_cast<unsigned>((zh >> (__ffsll(static_cast<long long>(kh)) - 1)) & 1) << 31;
                const double2* blk = base + ((gray(kh) << 4) & (C - 1));
                double2 e[16];
#pragma unroll
                for (int p = 0; p < 16; ++p) e[p] = blk[cgray(p) ^ kOdd];
#pragma unroll
                for (int p = 0; p < 16; ++p) {
                    const unsigned sgn = sgn_hi ^ sw[cgray(p) ^ kOdd];
                    sr += flip_sign(e[p].x, sgn);
                    si += flip_sign(e[p].y, sgn);
                }
            };
            const uint64_t nb = C >> 4;  // 1 (N = 4) or even
            for (uint64_t b = 0; b < nb; b += 2) {
                block(kh0 + b, std::false_type{});
                if (b + 1 < nb) block(kh0 + b + 1, std::true_type{});
            }
        }
        __syncthreads();  // the stage is refilled next iteration
    }
    if (threadIdx.x == 0) {
        const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
        double2 c = apply_phase(ph, sr, si, scale);
        if (!finite2(c)) {  // non-finite element: the reference's complex products (walk_kernel)
            const auto elem = [=](uint64_t i) { return D[i]; };
            c = exact_coeff(elem, N, x, z);
        }
        *out = c;
    }
}

cudaError_t launch_walk_diag(const double2* D, unsigned N, const uint64_t* n, bool slow, double2* out,
                             cudaStream_t stream) {
    if (slow || N < 4)  // coeff_slow semantics, and sizes below one 16-element block
        return slow ? launch_walk_t<true>(D, N, n, 1, out, 0, stream)
                    : launch_walk_t<false>(D, N, n, 1, out, 0, stream);
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = 2 * sizeof(double2) << kW1ChunkLog;
    if (!(attr_set.load() >> dev & 1)) {
        const cudaError_t e = cudaFuncSetAttribute(walk_one_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    const unsigned clog = N < kW1ChunkLog ? N : kW1ChunkLog;
    walk_one_kernel<<<1, kW1Threads, 2 * sizeof(double2) << clog, stream>>>(
        D, N, n, out, 1.0 / static_cast<double>(1ull << N));
    return count_launch();
}

cudaError_t launch_walk(const double2* G, unsigned N, const uint64_t* ns, uint64_t count, bool slow,
                        double2* out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    if (!slow && ns != nullptr && strings_grouped_ok(N, count))
        return launch_strings_grouped(G, N, ns, count, out, stream);
    const uint64_t dim = 1ull << N;
    return slow ? launch_walk_t<true>(G, N, ns, count, out, dim, stream)
                : launch_walk_t<false>(G, N, ns, count, out, dim, stream);
}

// ============================================================================
// Kronecker-trace oracle (oracle_coeff_kron, decompose.cpp:176-203), N <= 6
// ============================================================================
// One thread; the reference sums p[i*dim+j] * g(j,i) over all (i, j) in row-major
// order with full complex products, including the zero entries of P_n.

__global__ void kron_trace_kernel(const double2* __restrict__ G, unsigned N, uint64_t n,
                                  double2* out) {
    const uint64_t dim = 1ull << N;
    double tr = 0.0, ti = 0.0;
    for (uint64_t i = 0; i < dim; ++i) {
        for (uint64_t j = 0; j < dim; ++j) {
            // P_n[i][j] = prod_t sigma_{d_t}[i_t][j_t]
            double pr = 1.0, pi = 0.0;
            for (unsigned t = 0; t < N; ++t) {
                const unsigned d = static_cast<unsigned>((n >> (2 * t)) & 3u);
                const unsigned a = (i >> t) & 1u, b = (j >> t) & 1u;
                double sr = 0.0, si = 0.0;
                switch (d) {
                    case 0: sr = (a == b) ? 1.0 : 0.0; break;
                    case 1: sr = (a != b) ? 1.0 : 0.0; break;
                    case 2: si = (a != b) ? (a == 0 ? -1.0 : 1.0) : 0.0; break;
                    default: sr = (a == b) ? (a == 0 ? 1.0 : -1.0) : 0.0; break;
                }
                const double nr = pr * sr - pi * si, ni = pr * si + pi * sr;
                pr = nr;
                pi = ni;
            }
            const double2 g = G[j * dim + i];
            const double2 t = cmul_annex_g(pr, pi, g.x, g.y);  // the reference's complex product
            tr = __dadd_rn(tr, t.x);
            ti = __dadd_rn(ti, t.y);
        }
    }
    out[0] = make_double2(tr / static_cast<double>(dim), ti / static_cast<double>(dim));
}

cudaError_t launch_kron_trace(const double2* G, unsigned N, uint64_t n, double2* out,
                              cudaStream_t stream) {
    kron_trace_kernel<<<1, 1, 0, stream>>>(G, N, n, out);
    return count_launch();
}

// ============================================================================
// K5: seeded generator, bit-identical to random_matrix (bench.cpp:16-58)
// ============================================================================
// splitmix64 advances its state by a constant, so draw j of the stream uses state
// seed + (j + 1) * 0x9E3779B97F4A7C15 and element k takes draws 2k (re), 2k+1 (im).

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double unit_interval(uint64_t bits) {
    // (bits >> 11) * 2^-53 * 2 - 1: every step exact, no contraction can change it
    return __dsub_rn(__dmul_rn(static_cast<double>(bits >> 11), 0x1.0p-52), 1.0);
}

__global__ void random_matrix_kernel(uint64_t seed, uint64_t count, double2* __restrict__ out) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        out[k] = make_double2(unit_interval(splitmix_at(seed, 2 * k)),
                              unit_interval(splitmix_at(seed, 2 * k + 1)));
    }
}

cudaError_t launch_random_matrix(unsigned N, uint64_t seed, double2* out, cudaStream_t stream) {
    const uint64_t count = 1ull << (2 * N);
    uint64_t grid = (count + 255) / 256;
    if (grid > 148 * 64) grid = 148 * 64;
    random_matrix_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(seed, count, out);
    return count_launch();
}

// ============================================================================
// FP64-add probe: 16 independent DADD chains per thread, no loads in the loop
// ============================================================================

__global__ void __launch_bounds__(256) fp64_add_probe_kernel(double v, unsigned iters, double* sink) {
    double a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = j * 0.5 + threadIdx.x;
    for (unsigned it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] += (j & 1) ? -v : v;
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 12345.678) sink[0] = s;  // never true; keeps the chains live
}

cudaError_t launch_fp64_probe(unsigned blocks, unsigned iters, double* sink, cudaStream_t stream) {
    fp64_add_probe_kernel<<<blocks, 256, 0, stream>>>(1e-300, iters, sink);
    return count_launch();
}

}  // namespace pdb

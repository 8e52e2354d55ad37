// pd_k2.cuh — K2, the Gray-code FP64 kernel (see the description in pd_kernels.cu), in a header
// so that its segment instantiation can be compiled in its own translation unit (pd_k2seg.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pd_device.cuh"

namespace pdb {

constexpr int kK2Threads = 256;
constexpr int kK2ThreadsLog = 8;
constexpr int kK2StageElems = 2048;  // 32 KiB per stage when one x spans >= 1 CTA
constexpr int kK2BarBytes = 128;      // mbarrier block; keeps the stages 128 B aligned
constexpr int kK2MaxSmem = kK2BarBytes + 2 * 16 * kK2StageElems > kK2BarBytes + 16 * 4096
                               ? kK2BarBytes + 2 * 16 * kK2StageElems
                               : kK2BarBytes + 16 * 4096;

struct K2Geometry {
    unsigned tpx_log;    // threads per x inside a CTA (log2)
    unsigned xc_log;     // x per CTA (log2)
    unsigned cpx_log;    // CTAs per x (log2)
    unsigned ci_log;     // chunk length along i (log2)
    unsigned nchunks;    // chunks per diagonal
    unsigned stages;     // 1 or 2
    size_t smem_bytes;   // dynamic shared memory
    uint64_t grid;       // CTAs
};

inline K2Geometry k2_geometry(unsigned N, unsigned K, uint64_t x_count) {
    K2Geometry g{};
    const unsigned tx_log = N - K;  // threads per x overall
    g.tpx_log = tx_log < kK2ThreadsLog ? tx_log : kK2ThreadsLog;
    g.xc_log = kK2ThreadsLog - g.tpx_log;
    g.cpx_log = tx_log - g.tpx_log;
    if (g.xc_log > 0) {  // whole diagonals of 2^xc_log X-masks fit one stage
        g.ci_log = N;
        g.nchunks = 1;
        g.stages = 1;
        g.smem_bytes = (sizeof(double2) << (g.xc_log + N)) + kK2BarBytes;
    } else {
        g.ci_log = 11;  // kK2StageElems
        g.nchunks = 1u << (N - g.ci_log);
        g.stages = 2;
        g.smem_bytes = 2 * sizeof(double2) * kK2StageElems + kK2BarBytes;
    }
    const uint64_t xblocks = (x_count + (1ull << g.xc_log) - 1) >> g.xc_log;
    g.grid = xblocks << g.cpx_log;
    return g;
}

template <int K, bool ODD>
__device__ __forceinline__ void gray_block(const double2* __restrict__ blk, unsigned sgn,
                                           double (&ar)[1 << K], double (&ai)[1 << K]) {
#pragma unroll
    for (int p = 0; p < (1 << K); ++p) {
        constexpr int kHalf = K > 0 ? (1 << (K - 1)) : 0;
        const int il = static_cast<int>(cgray(p)) ^ (ODD ? kHalf : 0);
        const double2 e = blk[il];
        const double er = flip_sign(e.x, sgn);
        const double ei = flip_sign(e.y, sgn);
#pragma unroll
        for (int zl = 0; zl < (1 << K); ++zl) {
            if (cparity(static_cast<unsigned>(il & zl))) {
                ar[zl] -= er;
                ai[zl] -= ei;
            } else {
                ar[zl] += er;
                ai[zl] += ei;
            }
        }
    }
}

// Everything a K2 launch needs. A launch covers the walk steps of chunks [c_begin, c_end)
// (chunk c = steps [c C, (c+1) C), i.e. diagonal indices [gray(c) C, gray(c) C + C)): it starts
// from the raw sums in part_in (or zero) and ends by storing raw sums to part_out, or — when
// part_out is null — the finished coefficients. Continuing a chain from stored sums keeps each
// coefficient's summation order, so segmented launches are bit-identical to one launch.
// Coefficient destinations of a K2 launch. With at most kRunPtrs runs they are passed as one
// pointer per run (run r = Z-mask top-bit value r; GLOBAL layout: out + pd_run_offset, RUNS:
// out + r 4^(N-rb)), selected with constant indices in the epilogue; more runs use the
// arithmetic OutMap instead (MAPPED instantiation). Measured on B200: the run-pointer form
// keeps ptxas' schedule of the main loop at 485.8 ms (N=14, K1+K2) where the OutMap epilogue
// ends at 505.6 ms (+20 % dispatch stalls on DADDs; profiles/r01_k2_codegen.md).
constexpr unsigned kRunPtrBits = 3;
constexpr unsigned kRunPtrs = 1u << kRunPtrBits;
struct RunOut {
    double2* ptr[kRunPtrs];
};

// select a run pointer with constant indices only (a dynamic index into the
// parameter struct would force a local-memory copy of it)
__device__ __forceinline__ double2* run_ptr(const RunOut& runs, unsigned run) {
    double2* p = runs.ptr[0];
#pragma unroll
    for (unsigned r = 1; r < kRunPtrs; ++r)
        if (run == r) p = runs.ptr[r];
    return p;
}

struct K2Params {
    const double2* diag;       // rows of the X-masks [x0, x0 + x_count)
    uint64_t x0, x_count;
    unsigned N, tpx_log, xc_log, cpx_log, ci_log;
    unsigned c_begin, c_end;
    const double2* part_in;    // raw sums S[(x - x0) 2^N + z], or null
    double2* part_out;         // raw sums out, or null for coefficients
    unsigned run_bits;         // run-pointer form: runs of 4^(N - run_bits), run_bits <= 3
    RunOut runs;
    OutMap map;                // MAPPED form
    double scale;
    unsigned sb_ctas;          // K2s-c: CTAs per ZLO phase per X-mask superblock (0: one block)
};

// SEG = false: the whole walk from zero to coefficients (c_begin = 0, no partial sums); kept
// as a separate instantiation so the common case compiles without the segment logic.
template <int K, bool SEG, bool MAPPED>
__global__ void __launch_bounds__(kK2Threads, 2) gray_xmask_kernel(const K2Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned tid = threadIdx.x;
    const unsigned N = P.N, tpx_log = P.tpx_log, xc_log = P.xc_log, ci_log = P.ci_log;
    const uint64_t dim = 1ull << N;
    const unsigned C = 1u << ci_log;
    const uint64_t stage_elems = static_cast<uint64_t>(C) << xc_log;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // 2 mbarriers, then the stages
    double2* stage_buf = reinterpret_cast<double2*>(smem_raw + kK2BarBytes);
    const double2* __restrict__ diag = P.diag;

    const uint64_t cta = blockIdx.x;
    const uint64_t xblock = cta >> P.cpx_log;                  // which group of 2^xc_log x
    const unsigned zpart = static_cast<unsigned>(cta & ((1u << P.cpx_log) - 1));
    const uint64_t xl_base = xblock << xc_log;                 // local x index of the CTA's first x
    const unsigned xl_cta = tid >> tpx_log;                    // x within CTA
    const uint64_t xl = xl_base + xl_cta;                      // local x (row of diag)
    const bool active = xl < P.x_count;
    const uint64_t x = P.x0 + xl;
    const uint64_t zh = (static_cast<uint64_t>(zpart) << tpx_log) | (tid & ((1u << tpx_log) - 1));
    const uint64_t rows_here = (P.x_count - xl_base) < (1ull << xc_log) ? (P.x_count - xl_base)
                                                                        : (1ull << xc_log);

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    __syncthreads();

    auto issue = [&](unsigned c, unsigned s) {
        double2* dst = stage_buf + s * stage_elems;
        const uint64_t col = gray(c) << ci_log;
        if (xc_log > 0) {  // C == dim: the CTA's rows are one contiguous block of diag
            const unsigned bytes = static_cast<unsigned>(rows_here * dim * sizeof(double2));
            mbar_arrive_expect_tx(&bars[s], bytes);
            bulk_g2s(dst, diag + xl_base * dim, bytes, &bars[s]);
        } else {
            const unsigned bytes = C * static_cast<unsigned>(sizeof(double2));
            mbar_arrive_expect_tx(&bars[s], bytes);
            bulk_g2s(dst, diag + xl_base * dim + col, bytes, &bars[s]);
        }
    };

    const unsigned c_begin = SEG ? P.c_begin : 0u;
    const unsigned nseg = P.c_end - c_begin;
    if (tid == 0) {
        issue(c_begin, 0);
        if (nseg > 1) issue(c_begin + 1, 1);
    }

    double ar[1 << K], ai[1 << K];
    if (SEG && P.part_in != nullptr && active) {
        const double2* src = P.part_in + xl * dim + (zh << K);
#pragma unroll
        for (int j = 0; j < (1 << K); ++j) {
            const double2 v = src[j];
            ar[j] = v.x;
            ai[j] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < (1 << K); ++j) ar[j] = ai[j] = 0.0;
    }

    const unsigned blocks_per_chunk = C >> K;
    const uint32_t zh32 = static_cast<uint32_t>(zh);
    const uint64_t kh_start = static_cast<uint64_t>(c_begin) * blocks_per_chunk;
    // (-1)^{|gray(kh) & zh|} as a sign-bit mask: direct at the segment start, then the recurrence
    unsigned sgn = SEG ? static_cast<unsigned>(__popcll(gray(kh_start) & zh) & 1) << 31 : 0u;

    for (unsigned ci = 0; ci < nseg; ++ci) {
        const unsigned c = c_begin + ci;
        const unsigned s = ci & 1u;
        mbar_wait(&bars[s], (ci >> 1) & 1u);
        const double2* base = stage_buf + s * stage_elems + static_cast<uint64_t>(xl_cta) * C;
        const uint64_t kh0 = static_cast<uint64_t>(c) * blocks_per_chunk;
        for (unsigned b = 0; b < blocks_per_chunk; b += 2) {
            const uint64_t kh = kh0 + b;
            if (kh != kh_start) sgn ^= ((zh32 >> __ffsll(static_cast<long long>(kh)) - 1) & 1u) << 31;
            const unsigned off = static_cast<unsigned>((gray(kh) << K) & (C - 1));
            gray_block<K, false>(base + off, sgn, ar, ai);
            if (b + 1 < blocks_per_chunk) {
                const uint64_t kh1 = kh + 1;
                sgn ^= ((zh32 >> __ffsll(static_cast<long long>(kh1)) - 1) & 1u) << 31;
                const unsigned off1 = static_cast<unsigned>((gray(kh1) << K) & (C - 1));
                gray_block<K, true>(base + off1, sgn, ar, ai);
            }
        }
        if (ci + 2 < nseg) {
            __syncthreads();
            if (tid == 0) issue(c + 2, s);
        }
    }

    if (!active) return;
    if (SEG && P.part_out != nullptr) {
        double2* dst = P.part_out + xl * dim + (zh << K);
#pragma unroll
        for (int j = 0; j < (1 << K); ++j) dst[j] = make_double2(ar[j], ai[j]);
        return;
    }
    if (MAPPED) {
#pragma unroll
        for (int zl = 0; zl < (1 << K); ++zl) {
            const uint64_t z = (zh << K) | static_cast<uint64_t>(zl);
            const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
            P.map.out[out_index(P.map, tensor_number(x, z), z)] =
                apply_phase(ph, ar[zl], ai[zl], P.scale);
        }
        return;
    }
    const unsigned low_bits = 2 * (N - P.run_bits);
    const uint64_t low_mask = (low_bits >= 64) ? ~0ull : ((1ull << low_bits) - 1);
#pragma unroll
    for (int zl = 0; zl < (1 << K); ++zl) {
        const uint64_t z = (zh << K) | static_cast<uint64_t>(zl);
        const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
        const uint64_t n = tensor_number(x, z);
        const unsigned run = static_cast<unsigned>(z >> (N - P.run_bits));
        run_ptr(P.runs, run)[n & low_mask] = apply_phase(ph, ar[zl], ai[zl], P.scale);
    }
}

// the segment instantiation of K=4 lives in pd_k2seg.cu (own ptxas run); launches it
cudaError_t launch_gray_seg4(const K2Params& P, unsigned grid, size_t smem, cudaStream_t stream);

// K2s, the shared-prefix form of K2 (pd_k2share.cu): same geometry, parameters and results
bool gray_share_ok(unsigned N, unsigned run_bits);
cudaError_t launch_gray_share(const K2Params& P, bool seg, unsigned grid, size_t smem, cudaStream_t stream);
// K2s-c (pd_k2share.cuh), whole walk (pd_k2c.cu) and walk segments (pd_k2cseg.cu); P in K2s-c geometry
cudaError_t launch_gray_share_c_full(const K2Params& P, unsigned grid, cudaStream_t stream);
cudaError_t launch_gray_share_c_seg(const K2Params& P, unsigned grid, cudaStream_t stream);
// K2q (pd_k2q.cu): early walk segments (raw sums out, ending in region <= 7) with Q = 4 or 2
// Z-masks per thread; gray_share_q_pick returns Q or 0. P in K2 geometry.
unsigned gray_share_q_pick(const K2Params& P);
cudaError_t launch_gray_share_q(const K2Params& P, unsigned q, cudaStream_t stream);

}  // namespace pdb

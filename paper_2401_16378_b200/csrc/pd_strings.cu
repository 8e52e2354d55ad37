// pd_strings.cu — K3b: batched single-string inner products grouped by X-mask.
//
// coeff_fast (proj/src/decompose.cpp:49-57) walks the x-diagonal D_x[i] = G[i^x][i] of the
// string's X-mask x. K3 (walk_kernel) does that per thread straight from G: every string reads
// its own 2^N scattered elements (16 KiB per string at N=10, L2 bound). When a batch holds many
// strings per X-mask (BASELINE configs[1]: 65,536 random strings of N=10, 64 per X-mask), the
// strings are bucketed by X-mask on the device (count, then scan + scatter) and one warp per X-mask
// stages D_x once in shared memory; its threads then walk their strings' Gray sequences over
// the staged diagonal. All lanes of a warp read the same element at each step (broadcast),
// each lane walks two strings, and each string's signs over the low 4 index bits are fixed
// ±1.0 factors (the block sign is carried by the accumulator, see SwStrings), so a step costs
// one LDS.128 per lane and two DFMA per string.
//
// Summation order. Each string is one sequential chain over k = 0..2^N-1 in the reference's
// Gray order, with the exact factors ±1 folded into the sign bit, so the result equals K3 and
// the reference's coeff_fast bit for bit (finite inputs); bucketing only changes which thread
// computes a string, and results are written back at the string's own index.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

namespace {

constexpr int kSwB = 4;  // index bits of the unrolled block

// Bucketing: a count pass (global atomics), then a scatter pass whose CTAs each rescan the
// nb bucket counts in shared memory (4 KiB at N=10) to find the bucket starts, so no separate
// scan launch is needed. order[] lists the string indices grouped by X-mask; bucket x is
// order[off[x] .. off[x+1]) (written by CTA 0 of the scatter pass).
constexpr int kPrepThreads = 1024;

__global__ void strings_count_kernel(const uint64_t* __restrict__ ns, uint64_t count,
                                     unsigned* __restrict__ cnt) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < count) atomicAdd(&cnt[xmask_of(ns[k])], 1u);
}

// exclusive scan of cnt[0..nb) into s[0..nb] in shared memory (kPrepThreads threads)
__device__ void block_exclusive_scan(const unsigned* __restrict__ cnt, unsigned nb, unsigned* s) {
    __shared__ unsigned part[kPrepThreads];
    const unsigned per = (nb + kPrepThreads - 1) / kPrepThreads;
    const unsigned b0 = threadIdx.x * per;
    unsigned sum = 0;
    for (unsigned j = 0; j < per && b0 + j < nb; ++j) sum += cnt[b0 + j];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (unsigned d = 1; d < kPrepThreads; d <<= 1) {
        const unsigned v = threadIdx.x >= d ? part[threadIdx.x - d] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
    for (unsigned j = 0; j < per && b0 + j < nb; ++j) {
        s[b0 + j] = run;
        run += cnt[b0 + j];
    }
    if (threadIdx.x == kPrepThreads - 1) s[nb] = part[kPrepThreads - 1];
    __syncthreads();
}

// each CTA scatters kPrepThreads strings; cur[] (zeroed) counts the strings already placed
__global__ void __launch_bounds__(kPrepThreads)
    strings_scatter_kernel(const uint64_t* __restrict__ ns, uint64_t count,
                           const unsigned* __restrict__ cnt, unsigned nb, unsigned* __restrict__ cur,
                           unsigned* __restrict__ off, unsigned* __restrict__ order) {
    extern __shared__ unsigned start[];  // [nb + 1]
    block_exclusive_scan(cnt, nb, start);
    if (blockIdx.x == 0)
        for (unsigned b = threadIdx.x; b <= nb; b += kPrepThreads) off[b] = start[b];
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kPrepThreads + threadIdx.x;
    if (k < count) {
        const uint64_t x = xmask_of(ns[k]);
        order[start[x] + atomicAdd(&cur[x], 1u)] = static_cast<unsigned>(k);
    }
}

__device__ __forceinline__ double flip_hi(double v, unsigned sgn) {
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(sgn), __double2loint(v));
}

// One string's walk state. With sigma = (-1)^{|gray(kh) & zh|} the sign of the current block of
// 2^kSwB steps, the walk keeps acc' = sigma * acc instead of acc: inside a block
//     sigma (acc + sigma s_lo e) = acc' + s_lo e        (round-to-nearest is sign-symmetric),
// so every step is fma(e, d[il], acc') with the string's fixed d[il] = (-1)^{|il & zl|} = ±1.0
// (exact product: the fma rounds once, exactly like the reference's add), and a change of sigma
// at a block boundary negates acc' (exact). The chain order is the reference's, bit for bit.
template <int S>
struct SwStrings {
    double sr[S], si[S];
    double d[S][1 << kSwB];
    uint64_t zh[S];
    unsigned sig[S];  // sigma of the current block as a sign-bit word
};

template <bool ODD, int S>
__device__ __forceinline__ void sw_block(const double2* __restrict__ blk, SwStrings<S>& st) {
#pragma unroll
    for (int p = 0; p < (1 << kSwB); ++p) {
        constexpr int kHalf = 1 << (kSwB - 1);
        const int il = static_cast<int>(cgray(p)) ^ (ODD ? kHalf : 0);
        const double2 e = blk[il];  // the whole warp reads one element: broadcast
#pragma unroll
        for (int j = 0; j < S; ++j) {
            st.sr[j] = fma(e.x, st.d[j][il], st.sr[j]);
            st.si[j] = fma(e.y, st.d[j][il], st.si[j]);
        }
    }
}

template <int S>
__device__ __forceinline__ void sw_boundary(SwStrings<S>& st, unsigned bit) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
        const unsigned f = static_cast<unsigned>((st.zh[j] >> bit) & 1) << 31;
        st.sig[j] ^= f;
        st.sr[j] = flip_hi(st.sr[j], f);
        st.si[j] = flip_hi(st.si[j], f);
    }
}

// One CTA of kSwWarps warps per X-mask: stage D_x, then the bucket's strings, kSwStr per lane
// walked together (independent accumulator chains; N in [5, 13]).
constexpr int kSwStr = 1;

constexpr int kSwWarps = 3;  // warps per bucket: a Poisson(64) bucket fits one round, one string per lane

// bucket x's strings over its staged diagonal (the caller stages dx and synchronises)
__device__ __forceinline__ void walk_bucket(unsigned N, const uint64_t* __restrict__ ns,
                                            const unsigned* __restrict__ order, unsigned begin,
                                            unsigned end, uint64_t x, const double2* dx,
                                            double2* __restrict__ out, double scale) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nblocks = (1ull << N) >> kSwB;
    for (unsigned t0 = begin + warp * 32 * kSwStr; t0 < end; t0 += kSwWarps * 32 * kSwStr) {
        SwStrings<kSwStr> st;
        unsigned idx[kSwStr];
        uint64_t zs[kSwStr];
#pragma unroll
        for (int j = 0; j < kSwStr; ++j) {
            const unsigned t = t0 + lane + 32 * j;
            idx[j] = t < end ? order[t] : ~0u;  // ~0u: an idle slot (walks z = 0, not stored)
            zs[j] = t < end ? zmask_of(ns[idx[j]]) : 0;
            st.sr[j] = st.si[j] = 0.0;
            st.sig[j] = 0;
            st.zh[j] = zs[j] >> kSwB;
            const unsigned zl = static_cast<unsigned>(zs[j]) & ((1u << kSwB) - 1);
#pragma unroll
            for (int il = 0; il < (1 << kSwB); ++il)
                st.d[j][il] = (__popc(static_cast<unsigned>(il) & zl) & 1) ? -1.0 : 1.0;
        }
        for (uint64_t kh = 0; kh < nblocks; kh += 2) {
            if (kh) sw_boundary(st, static_cast<unsigned>(__ffsll(static_cast<long long>(kh)) - 1));
            sw_block<false>(dx + (gray(kh) << kSwB), st);
            sw_boundary(st, static_cast<unsigned>(__ffsll(static_cast<long long>(kh + 1)) - 1));
            sw_block<true>(dx + (gray(kh + 1) << kSwB), st);
        }
#pragma unroll
        for (int j = 0; j < kSwStr; ++j) {
            if (idx[j] == ~0u) continue;
            const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & zs[j]))) & 3u;
            double2 c = apply_phase(ph, flip_hi(st.sr[j], st.sig[j]), flip_hi(st.si[j], st.sig[j]),
                                    scale);
            if (!finite2(c)) {  // non-finite element: the reference's complex products
                const auto elem = [=](uint64_t i) { return dx[i]; };
                c = exact_coeff(elem, N, x, zs[j]);
            }
            out[idx[j]] = c;
        }
    }
}

__device__ __forceinline__ void stage_diagonal(const double2* __restrict__ G, unsigned N, uint64_t x,
                                               double2* dx) {
    const uint64_t dim = 1ull << N;
    for (uint64_t i = threadIdx.x; i < dim; i += blockDim.x) {
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(dx + i));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                     "l"(G + ((i ^ x) * dim + i))
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
}

__global__ void __launch_bounds__(32 * kSwWarps)
    strings_walk_kernel(const double2* __restrict__ G, unsigned N, const uint64_t* __restrict__ ns,
                        const unsigned* __restrict__ order, const unsigned* __restrict__ off,
                        double2* __restrict__ out, double scale) {
    extern __shared__ __align__(16) double2 dx[];
    const uint64_t x = blockIdx.x;
    const unsigned begin = off[x], end = off[x + 1];
    if (begin == end) return;
    stage_diagonal(G, N, x, dx);
    walk_bucket(N, ns, order, begin, end, x, dx, out, scale);
}

// The whole batch in one cooperative launch: zero the counts, count, scan + scatter, then
// every CTA walks buckets x = blockIdx.x, + gridDim.x, ... (grid-wide syncs between phases).
// One launch instead of a memset and three kernels: the batch call is launch bound.
__global__ void __launch_bounds__(32 * kSwWarps)
    strings_coop_kernel(const double2* __restrict__ G, unsigned N, const uint64_t* __restrict__ ns,
                        uint64_t count, unsigned* __restrict__ cnt, unsigned* __restrict__ cur,
                        unsigned* __restrict__ off, unsigned* __restrict__ order,
                        double2* __restrict__ out, double scale) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double2 dx[];
    const unsigned nb = 1u << N;
    for (uint64_t i = grid.thread_rank(); i < 2ull * nb; i += grid.size()) cnt[i] = 0;  // cnt, cur
    grid.sync();
    for (uint64_t k = grid.thread_rank(); k < count; k += grid.size()) atomicAdd(&cnt[xmask_of(ns[k])], 1u);
    grid.sync();
    {   // exclusive scan of the counts into shared memory (every CTA), then scatter
        unsigned* start = reinterpret_cast<unsigned*>(dx);  // nb + 1 entries fit the D_x space
        __shared__ unsigned part[32 * kSwWarps];
        const unsigned nt = blockDim.x, per = (nb + nt - 1) / nt, b0 = threadIdx.x * per;
        unsigned sum = 0;
        for (unsigned j = 0; j < per && b0 + j < nb; ++j) sum += cnt[b0 + j];
        part[threadIdx.x] = sum;
        __syncthreads();
        for (unsigned d = 1; d < nt; d <<= 1) {
            const unsigned v = threadIdx.x >= d ? part[threadIdx.x - d] : 0u;
            __syncthreads();
            part[threadIdx.x] += v;
            __syncthreads();
        }
        unsigned run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
        for (unsigned j = 0; j < per && b0 + j < nb; ++j) {
            start[b0 + j] = run;
            run += cnt[b0 + j];
        }
        if (threadIdx.x == nt - 1) start[nb] = part[nt - 1];
        __syncthreads();
        if (blockIdx.x == 0)
            for (unsigned j = threadIdx.x; j <= nb; j += nt) off[j] = start[j];
        for (uint64_t k = grid.thread_rank(); k < count; k += grid.size()) {
            const uint64_t x = xmask_of(ns[k]);
            order[start[x] + atomicAdd(&cur[x], 1u)] = static_cast<unsigned>(k);
        }
    }
    grid.sync();
    for (uint64_t x = blockIdx.x; x < nb; x += gridDim.x) {
        const unsigned begin = off[x], end = off[x + 1];
        if (begin == end) continue;
        stage_diagonal(G, N, x, dx);
        walk_bucket(N, ns, order, begin, end, x, dx, out, scale);
        __syncthreads();  // dx is restaged for the next bucket
    }
}

}  // namespace

bool strings_grouped_ok(unsigned N, uint64_t count) {
    // worth it once the average bucket holds a few strings; D_x must fit shared memory
    return N >= 5 && N <= 13 && count >= (2ull << N) && count < (1ull << 32);
}

cudaError_t launch_strings_grouped(const double2* G, unsigned N, const uint64_t* ns,
                                   uint64_t count, double2* out, cudaStream_t stream) {
    const unsigned nb = 1u << N;
    const size_t meta = (3ull * nb + 1) * sizeof(unsigned);
    int dev = 0;
    cudaGetDevice(&dev);
    // per-call scratch from the library's own pool (pool_alloc, pd_nonfinite.cu), which keeps
    // freed blocks: a pool lookup instead of a driver allocation (measured: 45 us otherwise)
    void* scratch = nullptr;
    cudaError_t e = pool_alloc(&scratch, meta + count * sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    unsigned* cnt = static_cast<unsigned*>(scratch);  // nb counts, nb cursors, nb + 1 offsets
    unsigned* cur = cnt + nb;
    unsigned* off = cur + nb;
    unsigned* order = off + nb + 1;
    const size_t smem = sizeof(double2) << N;
    static std::atomic<uint64_t> attr_set{0};  // one bit per device
    if (!(attr_set.load() >> dev & 1)) {
        e = cudaFuncSetAttribute(strings_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(double2) << 13));
        if (e != cudaSuccess) {
            pool_free(scratch, stream);
            return e;
        }
        attr_set.fetch_or(1ull << dev);
    }
    static std::atomic<int> coop_grid[64][14] = {};  // co-resident CTAs per (device, N)
    std::atomic<int>& cg_slot = coop_grid[dev & 63][N];
    if (!cg_slot.load()) {
        int per_sm = 0, sms = 0;
        cudaFuncSetAttribute(strings_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(double2) << 13));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, strings_coop_kernel, 32 * kSwWarps, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaGetLastError();
        cg_slot.store(per_sm * sms > 0 ? per_sm * sms : -1);
    }
    if (cg_slot.load() > 0) {
        const double scale = 1.0 / static_cast<double>(1ull << N);
        unsigned grid = static_cast<unsigned>(cg_slot.load());
        if (grid > nb) grid = nb;
        void* args[] = {const_cast<double2**>(&G), &N, const_cast<uint64_t**>(&ns), &count, &cnt, &cur,
                        &off, &order, &out, const_cast<double*>(&scale)};
        e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(strings_coop_kernel), grid, 32 * kSwWarps,
                                        args, smem, stream);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    } else {
        e = cudaMemsetAsync(cnt, 0, 2ull * nb * sizeof(unsigned), stream);
        if (e == cudaSuccess) {
            strings_count_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(ns, count, cnt);
            strings_scatter_kernel<<<static_cast<unsigned>((count + kPrepThreads - 1) / kPrepThreads),
                                     kPrepThreads, (nb + 1) * sizeof(unsigned), stream>>>(
                ns, count, cnt, nb, cur, off, order);
            strings_walk_kernel<<<nb, 32 * kSwWarps, smem, stream>>>(G, N, ns, order, off, out,
                                                                      1.0 / static_cast<double>(1ull << N));
            g_launches.fetch_add(3, std::memory_order_relaxed);
            e = cudaGetLastError();
        }
    }
    cudaError_t f = pool_free(scratch, stream);
    return e != cudaSuccess ? e : f;
}

}  // namespace pdb

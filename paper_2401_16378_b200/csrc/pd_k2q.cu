// pd_k2q.cu — K2q: the early walk segments of the host pipeline with Q Z-masks per thread.
//
// In walk region r (steps r 2^(N-4) .. (r+1) 2^(N-4)) only 2^bitlen(r) of a thread's 16 chains
// are distinct (pd_k2share.cu), so in the first regions a K2s thread carries 1, 2 or 4 chains:
// 2-8 sequential FP64 add chains, latency-bound. Run on their own, as the host pipeline's first
// walk segments do while G is still being uploaded (pd_api.cu), those regions took 32 ms for 6 %
// of the adds at N=14 (profiles/r01_k2s_c.md). Here a thread carries Q Z-masks
// zm_j = j | (the thread's bits) << log2 Q, j < Q, with their 16 / Q live chains each: Q = 4 for
// regions 0..3 (<= 4 live chains), Q = 2 for regions 4..7 (<= 8), i.e. 4-8x the independent
// chains of K2s in the same registers. The segment ends by storing every coefficient's raw sum
// (all 16 chains per Z-mask; the ones not yet split off are copies of their low-bit parent), so
// the later segments continue unchanged and every chain still performs the reference's adds in
// the reference's order: results are bit-identical to one whole-walk launch.
//
// Element signs: (-1)^{|il & zm_j|} = (-1)^{|il & j|} (a compile-time constant of the unrolled
// step: DADD or DADD with a negated operand) times (-1)^{|il & zm & (15 - (Q - 1))|}, which only
// changes where the Gray step flips an index bit >= log2 Q: one LOP3 on the running sign word
// there. The block sign of bits >= 4 is K2's Gray recurrence over zhi = zm >> 4 (equal for all j).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "pd_k2share.cuh"

namespace pdb {

namespace {

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;
constexpr int kQStageElems = 2048;
constexpr int kQStages = 3;
constexpr size_t kQSmem = kK2BarBytes + kQStages * sizeof(double2) * kQStageElems;

template <int Q>
struct QAcc {
    static constexpr int kL = kChains / Q;  // chains per Z-mask held in registers
    double r[Q][kL], i[Q][kL];
};

// one 16-step block: every one of the L live chains of every Z-mask j adds the element
template <int Q, int L, bool ODD>
__device__ __forceinline__ void q_block(const double2* __restrict__ blk, unsigned sgn, const unsigned (&w)[4],
                                        QAcc<Q>& a) {
    constexpr int kQB = Q == 4 ? 2 : (Q == 2 ? 1 : 0);  // log2 Q
    unsigned cur = sgn;
    if (ODD) cur ^= w[3];  // index bit 3 is set in odd blocks (always a thread bit: log2 Q <= 2)
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        const int il = static_cast<int>(cgray(p)) ^ (ODD ? 8 : 0);
        if (p > 0) {
            const unsigned flip = cgray(p) ^ cgray(p - 1);  // one index bit
            if (kQB <= 1 && flip == 2) cur ^= w[1];
            if (kQB <= 2 && flip == 4) cur ^= w[2];
            if (flip == 8) cur ^= w[3];
        }
        const double2 e = blk[il];
        const double er = flip_sign(e.x, cur);
        const double ei = flip_sign(e.y, cur);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
#pragma unroll
            for (int c = 0; c < L; ++c) {
                if (cparity(static_cast<unsigned>(il & j))) {
                    a.r[j][c] -= er;
                    a.i[j][c] -= ei;
                } else {
                    a.r[j][c] += er;
                    a.i[j][c] += ei;
                }
            }
        }
    }
}

template <int Q, int L>
__device__ __forceinline__ void q_region(const double2* __restrict__ base, uint64_t kh, uint64_t kh_end,
                                         uint64_t kh_start, unsigned C, uint32_t zhi, unsigned& sgn,
                                         const unsigned (&w)[4], QAcc<Q>& a) {
    for (; kh < kh_end; kh += 2) {
        if (kh != kh_start) sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh)) - 1)) & 1u) << 31;
        q_block<Q, L, false>(base + ((gray(kh) << 4) & (C - 1)), sgn, w, a);
        const uint64_t kh1 = kh + 1;
        sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh1)) - 1)) & 1u) << 31;
        q_block<Q, L, true>(base + ((gray(kh1) << 4) & (C - 1)), sgn, w, a);
    }
}

// negate the chains (c < 16 / Q of every Z-mask) whose bit is set in mask
template <int Q>
__device__ __forceinline__ void q_negate(unsigned mask, QAcc<Q>& a) {
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int c = 0; c < QAcc<Q>::kL; ++c) {
            const unsigned f = ((mask >> c) & 1u) << 31;
            a.r[j][c] = flip_sign(a.r[j][c], f);
            a.i[j][c] = flip_sign(a.i[j][c], f);
        }
}

// P: K2Params in this kernel's geometry — tpx_log = thread bits per X-mask group, xc_log =
// X-masks per CTA (log2), cpx_log = CTAs per X-mask group (log2), ci_log = steps per stage (log2)
template <int Q>
__global__ void __launch_bounds__(kQThreads, 2) gray_share_q_kernel(const K2Params P) {
    constexpr int kQB = Q == 4 ? 2 : (Q == 2 ? 1 : 0);
    constexpr int kL = QAcc<Q>::kL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned tid = threadIdx.x, lane = tid & 31u;
    const unsigned N = P.N, tb = P.tpx_log, xc_log = P.xc_log;
    const uint64_t dim = 1ull << N;
    const uint64_t cta = blockIdx.x;
    const uint64_t xblock = cta >> P.cpx_log;
    const uint64_t zpart = cta & ((1ull << P.cpx_log) - 1);
    CtaC t;
    t.diag = P.diag;
    t.xl_base = xblock << xc_log;
    t.C = 1u << P.ci_log;
    t.ci_log = P.ci_log;
    t.rows_here = static_cast<unsigned>(
        (P.x_count - t.xl_base) < (1ull << xc_log) ? (P.x_count - t.xl_base) : (1ull << xc_log));
    t.full = reinterpret_cast<uint64_t*>(smem_raw);
    t.done = reinterpret_cast<unsigned*>(smem_raw + 64);
    t.stages = reinterpret_cast<double2*>(smem_raw + kK2BarBytes);
    const unsigned xl_cta = tid >> tb;
    const uint64_t xl = t.xl_base + xl_cta;
    const bool active = xl < P.x_count;
    // Z-mask j of this thread: zm0 | j
    const uint64_t zm0 = (static_cast<uint64_t>(tid & ((1u << tb) - 1)) << kQB) | (zpart << (kQB + tb));
    const unsigned C = t.C;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&t.full[s], 1);
            t.done[s] = 0;
        }
        fence_barrier_init();
    }
    __syncthreads();
    const unsigned c_begin = P.c_begin;
    const unsigned nseg = P.c_end - c_begin;
    if (tid == 0)
        for (unsigned s = 0; s < kQStages && s < nseg; ++s) issue_c(t, dim, c_begin + s, s);

    QAcc<Q> a;
    const unsigned blocks_per_chunk = C >> 4;
    const unsigned region_log = N - 8;
    const uint64_t kh_start = static_cast<uint64_t>(c_begin) * blocks_per_chunk;
    if (P.part_in != nullptr && active) {
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const double2* src = P.part_in + xl * dim + ((zm0 | j) << 4);
#pragma unroll
            for (int c = 0; c < kL; ++c) {
                const double2 v = src[c];
                a.r[j][c] = v.x;
                a.i[j][c] = v.y;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
            for (int c = 0; c < kL; ++c) a.r[j][c] = a.i[j][c] = 0.0;
    }
    unsigned w[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) w[b] = static_cast<unsigned>((zm0 >> b) & 1) << 31;
    const uint32_t zhi = static_cast<uint32_t>(zm0 >> 4);
    unsigned sgn = static_cast<unsigned>(__popcll(gray(kh_start) & zhi) & 1) << 31;
    unsigned r_last = static_cast<unsigned>(kh_start >> region_log);
    if (kh_start > 0) q_negate(chain_signs(static_cast<unsigned>(gray((kh_start - 1) >> region_log))), a);

    unsigned s = 0, phase = 0;
    for (unsigned ci = 0; ci < nseg; ++ci) {
        const unsigned c = c_begin + ci;
        mbar_wait(&t.full[s], phase);
        const double2* base = t.stages + s * kQStageElems + static_cast<uint64_t>(xl_cta) * C;
        const uint64_t kh_chunk_end = static_cast<uint64_t>(c + 1) * blocks_per_chunk;
        for (uint64_t kh = static_cast<uint64_t>(c) * blocks_per_chunk; kh < kh_chunk_end;) {
            const unsigned r = static_cast<unsigned>(kh >> region_log);
            const uint64_t r_end = static_cast<uint64_t>(r + 1) << region_log;
            const uint64_t kend = r_end < kh_chunk_end ? r_end : kh_chunk_end;
            if (kh == (static_cast<uint64_t>(r) << region_log) && r != 0) {
                if ((r & (r - 1)) == 0) {  // region 2^m: chains c + 2^m start as copies of c
#pragma unroll
                    for (int m = 1; m < kL; m <<= 1)
                        if (r == static_cast<unsigned>(m))
#pragma unroll
                            for (int j = 0; j < Q; ++j)
#pragma unroll
                                for (int c2 = 0; c2 < m; ++c2) a.r[j][c2 + m] = a.r[j][c2], a.i[j][c2 + m] = a.i[j][c2];
                }
                q_negate(chain_signs(r & (0u - r)), a);
            }
            switch (32 - __clz(r)) {  // live chains 2^bitlen(r) <= kL (the launcher checks)
                case 0: q_region<Q, 1>(base, kh, kend, kh_start, C, zhi, sgn, w, a); break;
                case 1: q_region<Q, (kL >= 2 ? 2 : kL)>(base, kh, kend, kh_start, C, zhi, sgn, w, a); break;
                case 2: q_region<Q, (kL >= 4 ? 4 : kL)>(base, kh, kend, kh_start, C, zhi, sgn, w, a); break;
                default: q_region<Q, (kL >= 8 ? 8 : kL)>(base, kh, kend, kh_start, C, zhi, sgn, w, a); break;
            }
            r_last = r;
            kh = kend;
        }
        if (ci + kQStages < nseg) {
            __syncwarp();
            if (lane == 0) {
                unsigned prev;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(prev)
                             : "r"(smem_u32(&t.done[s]))
                             : "memory");
                if (prev == kQWarps - 1) {
                    t.done[s] = 0;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue_c(t, dim, c + kQStages, s);
                }
            }
        }
        if (++s == kQStages) s = 0, phase ^= 1u;
    }

    if (!active) return;
    q_negate(chain_signs(static_cast<unsigned>(gray(r_last))), a);  // back to plain chains
    const unsigned live = 1u << (32 - __clz(r_last));                // 2^bitlen(r_last) <= kL
    // chains not yet split off are copies of their low-bit parent (constant indices only)
#pragma unroll
    for (int m = 1; m < kL; m <<= 1)
        if (live <= static_cast<unsigned>(m))
#pragma unroll
            for (int j = 0; j < Q; ++j)
#pragma unroll
                for (int c = 0; c < m; ++c) a.r[j][c + m] = a.r[j][c], a.i[j][c + m] = a.i[j][c];
    // all 16 chains of each Z-mask: chain c >= kL equals chain c mod kL (live <= kL)
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        double2* dst = P.part_out + xl * dim + ((zm0 | j) << 4);
#pragma unroll
        for (int c = 0; c < kChains; ++c) dst[c] = make_double2(a.r[j][c % kL], a.i[j][c % kL]);
    }
}

template <int Q>
cudaError_t launch_q(const K2Params& P0, cudaStream_t stream) {
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        const cudaError_t e =
            cudaFuncSetAttribute(gray_share_q_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    constexpr unsigned kQB = Q == 4 ? 2 : (Q == 2 ? 1 : 0);
    K2Params P = P0;
    const unsigned bits = P0.N - 4 - kQB;  // thread-owned Z-mask bits per X-mask
    const unsigned tb = bits < 8 ? bits : 8;
    P.tpx_log = tb;
    P.xc_log = 8 - tb;
    P.cpx_log = bits - tb;
    unsigned cs_log = 11 - P.xc_log;  // stages of at most 2048 elements, within the caller's chunks
    if (cs_log > P0.ci_log) cs_log = P0.ci_log;
    if (cs_log < 5) return cudaErrorInvalidValue;
    P.ci_log = cs_log;
    P.c_begin = P0.c_begin << (P0.ci_log - cs_log);
    P.c_end = P0.c_end << (P0.ci_log - cs_log);
    const uint64_t xblocks = (P0.x_count + (1ull << P.xc_log) - 1) >> P.xc_log;
    const uint64_t grid = xblocks << P.cpx_log;
    if (grid > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    gray_share_q_kernel<Q><<<static_cast<unsigned>(grid), kQThreads, kQSmem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace

unsigned gray_share_q_pick(const K2Params& P) {
    // a segment that stores raw sums and ends in region <= 3 (Q = 4) or <= 7 (Q = 2)
    if (P.N < 12 || P.part_out == nullptr || P.c_end == 0) return 0;
    const uint64_t last_step = (static_cast<uint64_t>(P.c_end) << P.ci_log) - 1;
    const uint64_t r_last = last_step >> (P.N - 4);
    if (r_last <= 3) return 4;
    if (r_last <= 7) return 2;
    return 0;
}

cudaError_t launch_gray_share_q(const K2Params& P, unsigned q, cudaStream_t stream) {
    return q == 4 ? launch_q<4>(P, stream) : launch_q<2>(P, stream);
}

}  // namespace pdb

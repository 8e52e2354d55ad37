// pd_k2share.cuh — pieces of K2s shared by its translation units: the chain helpers and the
// K2s-c kernel template (pd_k2share.cu: K2s with sign words and the launcher; pd_k2c.cu /
// pd_k2cseg.cu: the K2s-c whole-walk and walk-segment instantiations, each in its own ptxas run).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "pd_k2.cuh"

namespace pdb {

namespace {

constexpr int kChains = 16;

__device__ __forceinline__ double flip_sign3(double v, unsigned a, unsigned b) {
    int hi = __double2hiint(v);
    asm("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(hi) : "r"(a), "r"(b));
    return __hiloint2double(hi, __double2loint(v));
}

constexpr int bitlen(unsigned v) { return v == 0 ? 0 : 1 + bitlen(v >> 1); }

// one 16-step block (walk steps 16 kh + p): every one of the 2^M live chains adds the element
template <int M, bool ODD>
__device__ __forceinline__ void share_block(const double2* __restrict__ blk, unsigned sgn, const unsigned (&sw)[16],
                                            double (&ar)[kChains], double (&ai)[kChains]) {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        const int il = static_cast<int>(cgray(p)) ^ (ODD ? 8 : 0);
        const double2 e = blk[il];
        const double er = flip_sign3(e.x, sgn, sw[il]);
        const double ei = flip_sign3(e.y, sgn, sw[il]);
#pragma unroll
        for (int c = 0; c < (1 << M); ++c) {
            ar[c] += er;
            ai[c] += ei;
        }
    }
}

// blocks [kh, kh_end) of one region (kh even, kh_end - kh even)
template <int M>
__device__ __forceinline__ void share_region(const double2* __restrict__ base, uint64_t kh, uint64_t kh_end,
                                             uint64_t kh_start, unsigned C, uint32_t zhi, unsigned& sgn,
                                             const unsigned (&sw)[16], double (&ar)[kChains],
                                             double (&ai)[kChains]) {
    for (; kh < kh_end; kh += 2) {
        if (kh != kh_start) sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh)) - 1)) & 1u) << 31;
        share_block<M, false>(base + ((gray(kh) << 4) & (C - 1)), sgn, sw, ar, ai);
        const uint64_t kh1 = kh + 1;
        sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh1)) - 1)) & 1u) << 31;
        share_block<M, true>(base + ((gray(kh1) << 4) & (C - 1)), sgn, sw, ar, ai);
    }
}

// bit c of the result = parity(g & c), c = 0..15
__device__ __forceinline__ unsigned chain_signs(unsigned g) {
    return ((g & 1) ? 0xAAAAu : 0u) ^ ((g & 2) ? 0xCCCCu : 0u) ^ ((g & 4) ? 0xF0F0u : 0u) ^ ((g & 8) ? 0xFF00u : 0u);
}

// negate the chains whose bit is set in mask (exact: sign-bit flips)
__device__ __forceinline__ void negate_chains(unsigned mask, double (&ar)[kChains], double (&ai)[kChains]) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const unsigned f = ((mask >> c) & 1u) << 31;
        ar[c] = flip_sign(ar[c], f);
        ai[c] = flip_sign(ai[c], f);
    }
}

// ---------------------------------------------------------------------------------------------
// K2s-c (N >= 13): the thread's low four Z-mask bits are a compile-time constant of the CTA.
//
// gray_share_kernel pays for the runtime per-element sign (-1)^{|il & zm|} with 16 sign-word
// registers and a 3-input LOP3 per component: with the sign words dropped (wrong results) the
// same launch ran 348.6 -> 332.9 ms. Here every thread of a CTA shares Z-mask bits 0..3 (ZLO),
// so that sign is (-1)^{|il & ZLO|} with il a constant of the unrolled step: it becomes DADD or
// DADD with a negated operand, and the loop body is K2's (LDS.128, 2 LOP3 for the block sign,
// 32 DADD per element). One kernel holds the 16 ZLO bodies (a switch on the CTA's ZLO); ZLO is
// the slowest-varying part of blockIdx, so the CTAs resident at any time run the same body.
//
// Stages are released without CTA barriers: the last warp to finish a stage (a shared-memory
// counter, acq_rel) issues its refill, so no warp waits for another while data is resident.
//
// Geometry (256 threads): thread bits tb = min(N - 8, 6) give Z-mask bits 4 .. 4+tb-1, a CTA
// covers 2^(8 - tb) X-masks (N = 13: 8, N >= 14: 4), and 16 * 2^(N - 8 - tb) CTAs share one
// X-mask group. Three stages of 2048 elements (32 KiB: 2^(8-tb) rows of C steps).
//
// Measured (N=14, K1 + kernel, profiles/r01_k2s_c.md): 348.6 -> 336.8 ms, bit-identical. The
// 16-chain loop runs at 98.7 % of K2's DADD rate (all regions forced to 16 chains: 492.3 ms vs
// K2's 485.7); the rest of the gap to that rate (~7 ms) is the first regions' 1-2 live chains,
// whose sequential adds are latency-bound. ZLO as the fastest-varying blockIdx part (the 16
// bodies mixed on every SM) ran 680 ms: the body must not change between co-resident CTAs. At
// N = 12 the sign-word kernel stays (5.69 vs 5.89 ms: 16 X-masks per CTA, 128-step stages).
// ---------------------------------------------------------------------------------------------
constexpr int kCThreads = 256;
constexpr int kCWarps = kCThreads / 32;
constexpr int kCStageElems = 2048;
constexpr int kCStages = 3;
constexpr size_t kCSmem = kK2BarBytes + kCStages * sizeof(double2) * kCStageElems;

// one 16-step block with the element signs of ZLO folded in at compile time
template <int M, bool ODD, int ZLO>
__device__ __forceinline__ void share_block_c(const double2* __restrict__ blk, unsigned sgn,
                                              double (&ar)[kChains], double (&ai)[kChains]) {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        const int il = static_cast<int>(cgray(p)) ^ (ODD ? 8 : 0);
        const double2 e = blk[il];
        const double er = flip_sign(e.x, sgn);
        const double ei = flip_sign(e.y, sgn);
#pragma unroll
        for (int c = 0; c < (1 << M); ++c) {
            if (cparity(static_cast<unsigned>(il & ZLO))) {
                ar[c] -= er;
                ai[c] -= ei;
            } else {
                ar[c] += er;
                ai[c] += ei;
            }
        }
    }
}

template <int M, int ZLO>
__device__ __forceinline__ void share_region_c(const double2* __restrict__ base, uint64_t kh, uint64_t kh_end,
                                               uint64_t kh_start, unsigned C, uint32_t zhi, unsigned& sgn,
                                               double (&ar)[kChains], double (&ai)[kChains]) {
    for (; kh < kh_end; kh += 2) {
        if (kh != kh_start) sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh)) - 1)) & 1u) << 31;
        share_block_c<M, false, ZLO>(base + ((gray(kh) << 4) & (C - 1)), sgn, ar, ai);
        const uint64_t kh1 = kh + 1;
        sgn ^= ((zhi >> (__ffsll(static_cast<long long>(kh1)) - 1)) & 1u) << 31;
        share_block_c<M, true, ZLO>(base + ((gray(kh1) << 4) & (C - 1)), sgn, ar, ai);
    }
}

struct CtaC {
    const double2* diag;
    uint64_t xl_base;
    unsigned rows_here, C, ci_log;
    uint64_t* full;      // kCStages mbarriers (TMA complete_tx)
    unsigned* done;      // kCStages warp counters
    double2* stages;
};

__device__ __forceinline__ void issue_c(const CtaC& t, uint64_t dim, unsigned c, unsigned s) {
    double2* dst = t.stages + s * kCStageElems;
    const uint64_t col = gray(c) << t.ci_log;
    const unsigned bytes = t.C * static_cast<unsigned>(sizeof(double2));
    mbar_arrive_expect_tx(&t.full[s], bytes * t.rows_here);
    for (unsigned r = 0; r < t.rows_here; ++r)
        bulk_g2s(dst + r * t.C, t.diag + (t.xl_base + r) * dim + col, bytes, &t.full[s]);
}

template <bool SEG, int ZLO>
__device__ __forceinline__ void share_body_c(const K2Params& P, const CtaC& t, uint64_t xl, uint64_t x,
                                             bool active, uint64_t zm, unsigned xl_cta) {
    const unsigned N = P.N;
    const uint64_t dim = 1ull << N;
    const unsigned C = t.C;
    const unsigned lane = threadIdx.x & 31u;
    double ar[kChains], ai[kChains];
    if (SEG && P.part_in != nullptr && active) {
        const double2* src = P.part_in + xl * dim + (zm << 4);
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
            const double2 v = src[j];
            ar[j] = v.x;
            ai[j] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kChains; ++j) ar[j] = ai[j] = 0.0;
    }
    const uint32_t zhi = static_cast<uint32_t>(zm >> 4);
    const unsigned c_begin = SEG ? P.c_begin : 0u;
    const unsigned nseg = P.c_end - c_begin;
    const unsigned blocks_per_chunk = C >> 4;
    const unsigned region_log = N - 8;
    const uint64_t kh_start = static_cast<uint64_t>(c_begin) * blocks_per_chunk;
    unsigned sgn = SEG ? static_cast<unsigned>(__popcll(gray(kh_start) & zhi) & 1) << 31 : 0u;
    unsigned r_last = static_cast<unsigned>(kh_start >> region_log);
    if (SEG && kh_start > 0)
        negate_chains(chain_signs(static_cast<unsigned>(gray((kh_start - 1) >> region_log))), ar, ai);

    unsigned s = 0, phase = 0;
    for (unsigned ci = 0; ci < nseg; ++ci) {
        const unsigned c = c_begin + ci;
        mbar_wait(&t.full[s], phase);
        const double2* base = t.stages + s * kCStageElems + static_cast<uint64_t>(xl_cta) * C;
        const uint64_t kh_chunk_end = static_cast<uint64_t>(c + 1) * blocks_per_chunk;
        for (uint64_t kh = static_cast<uint64_t>(c) * blocks_per_chunk; kh < kh_chunk_end;) {
            const unsigned r = static_cast<unsigned>(kh >> region_log);
            const uint64_t r_end = static_cast<uint64_t>(r + 1) << region_log;
            const uint64_t kend = r_end < kh_chunk_end ? r_end : kh_chunk_end;
            if (kh == (static_cast<uint64_t>(r) << region_log) && r != 0) {
                if ((r & (r - 1)) == 0) {
#pragma unroll
                    for (int w = 1; w < kChains; w <<= 1)
                        if (r == static_cast<unsigned>(w))
#pragma unroll
                            for (int j = 0; j < w; ++j) ar[j + w] = ar[j], ai[j + w] = ai[j];
                }
                negate_chains(chain_signs(r & (0u - r)), ar, ai);
            }
            switch (32 - __clz(r)) {
                case 0: share_region_c<0, ZLO>(base, kh, kend, kh_start, C, zhi, sgn, ar, ai); break;
                case 1: share_region_c<1, ZLO>(base, kh, kend, kh_start, C, zhi, sgn, ar, ai); break;
                case 2: share_region_c<2, ZLO>(base, kh, kend, kh_start, C, zhi, sgn, ar, ai); break;
                case 3: share_region_c<3, ZLO>(base, kh, kend, kh_start, C, zhi, sgn, ar, ai); break;
                default: share_region_c<4, ZLO>(base, kh, kend, kh_start, C, zhi, sgn, ar, ai); break;
            }
            r_last = r;
            kh = kend;
        }
        // release the stage; the last warp out refills it with chunk c + kCStages
        if (ci + kCStages < nseg) {
            __syncwarp();
            if (lane == 0) {
                unsigned prev;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(prev)
                             : "r"(smem_u32(&t.done[s]))
                             : "memory");
                if (prev == kCWarps - 1) {
                    t.done[s] = 0;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue_c(t, dim, c + kCStages, s);
                }
            }
        }
        if (++s == kCStages) s = 0, phase ^= 1u;
    }

    if (!active) return;
    negate_chains(chain_signs(static_cast<unsigned>(gray(r_last))), ar, ai);
    const unsigned live = 1u << (32 - __clz(r_last));
#pragma unroll
    for (int w = 1; w < kChains; w <<= 1)
        if (live <= static_cast<unsigned>(w))
#pragma unroll
            for (int j = 0; j < w; ++j) ar[j + w] = ar[j], ai[j + w] = ai[j];
    const unsigned low_bits = 2 * (N - P.run_bits);
    const uint64_t low_mask = (low_bits >= 64) ? ~0ull : ((1ull << low_bits) - 1);
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
        const uint64_t z = zm | (static_cast<uint64_t>(j) << (N - 4));
        const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
        const uint64_t n = tensor_number(x, z);
        const unsigned run = static_cast<unsigned>(j) >> (4 - P.run_bits);
        run_ptr(P.runs, run)[n & low_mask] = apply_phase(ph, ar[j], ai[j], P.scale);
    }
}

// P.tpx_log = tb, P.xc_log = X-masks per CTA (log2), P.cpx_log = log2(CTAs per X-mask group)
// (>= 4: ZLO plus the Z-mask bits above the thread's), P.ci_log = steps per stage (log2)
template <bool SEG>
__global__ void __launch_bounds__(kCThreads, 2) gray_share_c_kernel(const K2Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned tid = threadIdx.x;
    const unsigned N = P.N, tb = P.tpx_log, xc_log = P.xc_log;
    const uint64_t dim = 1ull << N;
    // blockIdx = ZLO * (grid / 16) + (xblock << (cpx_log - 4)) + zmid
    const unsigned mid_log = P.cpx_log - 4;
    const uint64_t per_zlo = gridDim.x >> 4;
    unsigned zlo;
    uint64_t rest;
    if (P.sb_ctas) {
        // X-mask superblocks of sb_ctas CTAs per ZLO phase: all 16 phases of a superblock run
        // before the next superblock starts, so its diagonals are re-read from L2 (the last
        // superblock holds the remainder)
        const uint64_t per_sb = 16ull * P.sb_ctas;
        const uint64_t nfull = per_zlo / P.sb_ctas;
        const uint64_t sbi = blockIdx.x / per_sb;
        const uint64_t width = sbi < nfull ? P.sb_ctas : per_zlo - nfull * P.sb_ctas;
        const uint64_t r = blockIdx.x - sbi * per_sb;
        zlo = static_cast<unsigned>(r / width);
        rest = sbi * P.sb_ctas + (r - static_cast<uint64_t>(zlo) * width);
    } else {
        zlo = static_cast<unsigned>(blockIdx.x / per_zlo);
        rest = blockIdx.x - zlo * per_zlo;
    }
    const uint64_t xblock = rest >> mid_log;
    const uint64_t zmid = rest & ((1ull << mid_log) - 1);
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
    const uint64_t x = P.x0 + xl;
    const uint64_t zm = zlo | (static_cast<uint64_t>(tid & ((1u << tb) - 1)) << 4) | (zmid << (4 + tb));
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < kCStages; ++s) {
            mbar_init(&t.full[s], 1);
            t.done[s] = 0;
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned c_begin = SEG ? P.c_begin : 0u;
        const unsigned nseg = P.c_end - c_begin;
        for (unsigned s = 0; s < kCStages && s < nseg; ++s) issue_c(t, dim, c_begin + s, s);
    }
    switch (zlo) {
#define PD_ZLO_CASE(v) \
    case v: share_body_c<SEG, v>(P, t, xl, x, active, zm, xl_cta); break;
        PD_ZLO_CASE(0) PD_ZLO_CASE(1) PD_ZLO_CASE(2) PD_ZLO_CASE(3)
        PD_ZLO_CASE(4) PD_ZLO_CASE(5) PD_ZLO_CASE(6) PD_ZLO_CASE(7)
        PD_ZLO_CASE(8) PD_ZLO_CASE(9) PD_ZLO_CASE(10) PD_ZLO_CASE(11)
        PD_ZLO_CASE(12) PD_ZLO_CASE(13) PD_ZLO_CASE(14) PD_ZLO_CASE(15)
#undef PD_ZLO_CASE
    }
}

// one instantiation per translation unit (pd_k2c.cu: SEG = false, pd_k2cseg.cu: SEG = true). The SEG
// form continues a walk from raw sums (part_in) and ends with the coefficients: segments that
// store raw sums go to K2q or K2s (launch_gray_share).
template <bool SEG>
cudaError_t launch_gray_share_c_impl(const K2Params& P, unsigned grid, cudaStream_t stream) {
    static std::atomic<uint64_t> attr_set{0};  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        const cudaError_t e = cudaFuncSetAttribute(gray_share_c_kernel<SEG>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    gray_share_c_kernel<SEG><<<grid, kCThreads, kCSmem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace

}  // namespace pdb

// pd_k2share.cu — K2 with shared walk prefixes (K2s): the same coefficients, bit for bit, with a
// third fewer FP64 additions.
//
// Every coefficient S_{x,z} = sum_k s_k(z) D_x[g_k] is a sequential chain over the Gray walk
// k = 0 .. 2^N-1 (decompose.cpp:30-47). Walk step k only looks at the bits of z that are set in
// g_k = gray(k), and gray(k) < 2^(j+1) for k < 2^(j+1): the first 2^(j+1) steps of the chains of
// all Z-masks that agree on bits 0..j are the same floating-point operations on the same values.
// So the chains of z and z ^ 2^(N-1) coincide for the first half of the walk, the four chains of
// z ^ {0, 1, 2, 3} 2^(N-2) for the first quarter, and so on. Computing every shared prefix once
// costs sum_j 2^j * 2^(j+1) = 2/3 4^N additions per X-mask instead of 4^N, and each chain still
// performs exactly the reference's additions in the reference's order.
//
// Work split. A thread owns one X-mask x and the 16 Z-masks z = zm | c << (N-4), c = 0..15 (the
// top four bits; zm = the thread's low N-4 bits). Walk region r = k >> (N-4) (16 regions of
// 2^(N-4) steps) has top bits gray(r) in every g_k, so in region r chain c's sign is
//     s_k(z) = (-1)^{|g_k & zm|} * (-1)^{|gray(r) & c|}
// and chains c, c' agreeing on the low bitlen(r) bits are still identical: region r keeps
// 2^bitlen(r) chains (1, 2, 4, 4, 8 x 4, 16 x 8) and copies c -> c + r when r is a power of two.
// The first factor is per thread and per step: with k = 16 kh + p it is the block sign of the
// Gray recurrence over kh (bits 4.. of zm, as in K2) times a per-thread sign word of the element's
// low index bits (il & zm); both go into the element's sign bit with one 3-input LOP3 per
// component. The second factor is constant over a region, so each chain is kept as
// sigma_c(r) * S (exact), every live chain adds the same signed element, and entering region r
// negates the chains whose bit ctz(r) is set (gray(r) ^ gray(r-1) = 2^ctz(r)). fl(-a + -b) =
// -fl(a + b) in round-to-nearest, so each chain's value equals the reference's up to the sign
// of an exact zero (compared with IEEE ==). One loop body per live-chain count (five)
// instead of one per region keeps the hot loop in the instruction cache.
//
// Everything else — TMA-staged chunks of the diagonals, the geometry, raw partial sums for
// walk segments, the run-pointer epilogue — is K2's (pd_k2.cuh).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "pd_k2share.cuh"

namespace pdb {

namespace {

template <bool SEG>
__global__ void __launch_bounds__(kK2Threads, 2) gray_share_kernel(const K2Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned tid = threadIdx.x;
    const unsigned N = P.N, tpx_log = P.tpx_log, xc_log = P.xc_log, ci_log = P.ci_log;
    const uint64_t dim = 1ull << N;
    const unsigned C = 1u << ci_log;
    const uint64_t stage_elems = static_cast<uint64_t>(C) << xc_log;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
    double2* stage_buf = reinterpret_cast<double2*>(smem_raw + kK2BarBytes);
    const double2* __restrict__ diag = P.diag;

    const uint64_t cta = blockIdx.x;
    const uint64_t xblock = cta >> P.cpx_log;
    const unsigned zpart = static_cast<unsigned>(cta & ((1u << P.cpx_log) - 1));
    const uint64_t xl_base = xblock << xc_log;
    const unsigned xl_cta = tid >> tpx_log;
    const uint64_t xl = xl_base + xl_cta;
    const bool active = xl < P.x_count;
    const uint64_t x = P.x0 + xl;
    const uint64_t zm = (static_cast<uint64_t>(zpart) << tpx_log) | (tid & ((1u << tpx_log) - 1));
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
        if (xc_log > 0) {
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
    unsigned sw[16];
#pragma unroll
    for (int il = 0; il < 16; ++il) sw[il] = static_cast<unsigned>(__popc(il & static_cast<unsigned>(zm & 15)) & 1) << 31;
    const uint32_t zhi = static_cast<uint32_t>(zm >> 4);

    const unsigned blocks_per_chunk = C >> 4;
    const unsigned region_log = N - 8;  // 16-step blocks per region (log2)
    const uint64_t kh_start = static_cast<uint64_t>(c_begin) * blocks_per_chunk;
    unsigned sgn = SEG ? static_cast<unsigned>(__popcll(gray(kh_start) & zhi) & 1) << 31 : 0u;
    unsigned r_last = static_cast<unsigned>(kh_start >> region_log);
    // stored partial sums are plain chains; carry them as sigma_c(r) S for the region of the
    // segment's previous step (the loop applies the change of sign when it enters a region)
    if (SEG && kh_start > 0)
        negate_chains(chain_signs(static_cast<unsigned>(gray((kh_start - 1) >> region_log))), ar, ai);

    for (unsigned ci = 0; ci < nseg; ++ci) {
        const unsigned c = c_begin + ci;
        const unsigned s = ci & 1u;
        mbar_wait(&bars[s], (ci >> 1) & 1u);
        const double2* base = stage_buf + s * stage_elems + static_cast<uint64_t>(xl_cta) * C;
        const uint64_t kh_chunk_end = static_cast<uint64_t>(c + 1) * blocks_per_chunk;
        for (uint64_t kh = static_cast<uint64_t>(c) * blocks_per_chunk; kh < kh_chunk_end;) {
            const unsigned r = static_cast<unsigned>(kh >> region_log);
            const uint64_t r_end = static_cast<uint64_t>(r + 1) << region_log;
            const uint64_t kend = r_end < kh_chunk_end ? r_end : kh_chunk_end;
            if (kh == (static_cast<uint64_t>(r) << region_log) && r != 0) {
                if ((r & (r - 1)) == 0) {
                    // region r = 2^m opens chain bit m: chains c + r start as copies of chains c
#pragma unroll
                    for (int t = 1; t < kChains; t <<= 1)
                        if (r == static_cast<unsigned>(t))
#pragma unroll
                            for (int j = 0; j < t; ++j) ar[j + t] = ar[j], ai[j + t] = ai[j];
                }
                // gray(r) = gray(r - 1) ^ 2^ctz(r): the chains with that bit set change sign
                negate_chains(chain_signs(r & (0u - r)), ar, ai);
            }
            switch (32 - __clz(r)) {  // live chains 2^bitlen(r)
                case 0: share_region<0>(base, kh, kend, kh_start, C, zhi, sgn, sw, ar, ai); break;
                case 1: share_region<1>(base, kh, kend, kh_start, C, zhi, sgn, sw, ar, ai); break;
                case 2: share_region<2>(base, kh, kend, kh_start, C, zhi, sgn, sw, ar, ai); break;
                case 3: share_region<3>(base, kh, kend, kh_start, C, zhi, sgn, sw, ar, ai); break;
                default: share_region<4>(base, kh, kend, kh_start, C, zhi, sgn, sw, ar, ai); break;
            }
            r_last = r;
            kh = kend;
        }
        if (ci + 2 < nseg) {
            __syncthreads();
            if (tid == 0) issue(c + 2, s);
        }
    }

    if (!active) return;
    negate_chains(chain_signs(static_cast<unsigned>(gray(r_last))), ar, ai);  // back to plain chains
    // chains not yet split off are still copies of their low-bit parent
    const unsigned live = 1u << (32 - __clz(r_last));  // 2^bitlen(r_last)
#pragma unroll
    for (int t = 1; t < kChains; t <<= 1)  // constant indices only (keeps ar/ai in registers)
        if (live <= static_cast<unsigned>(t))
#pragma unroll
            for (int j = 0; j < t; ++j) ar[j + t] = ar[j], ai[j + t] = ai[j];
    if (SEG && P.part_out != nullptr) {
        double2* dst = P.part_out + xl * dim + (zm << 4);
#pragma unroll
        for (int j = 0; j < kChains; ++j) dst[j] = make_double2(ar[j], ai[j]);
        return;
    }
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

}  // namespace

bool gray_share_ok(unsigned N, unsigned run_bits) { return N >= 9 && run_bits <= kRunPtrBits; }

uint64_t gray_share_c_min_xmasks(unsigned N) {
    if (N < 13) return ~0ull;
    static const char* min_env = std::getenv("PD_K2SC_MIN");  // measurement override
    if (min_env) return std::strtoull(min_env, nullptr, 10);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        sms = 148;
    }
    // a ZLO phase of the launch spans x_count / 2^(8-tb) * 2^(N-8-tb) CTAs; ask for as many as
    // 2 CTAs per SM, i.e. one full residency, so that at most two bodies share the GPU at a time
    const unsigned tb = N - 8 < 6 ? N - 8 : 6;
    const uint64_t ctas = 2ull * static_cast<uint64_t>(sms);
    const uint64_t per_x = (1ull << (N - 8 - tb));  // CTAs per X-mask group and ZLO
    uint64_t x = ((ctas + per_x - 1) / per_x) << (8 - tb);
    return x;
}

cudaError_t launch_gray_share(const K2Params& P0, bool seg, unsigned grid, size_t smem, cudaStream_t stream) {
    static std::atomic<uint64_t> attr_set{0};  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        cudaError_t e = cudaFuncSetAttribute(gray_share_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kK2MaxSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(gray_share_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kK2MaxSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    static const char* q_env = std::getenv("PD_K2Q");
    if (seg && !(q_env && q_env[0] == '0'))
        if (const unsigned q = gray_share_q_pick(P0)) return launch_gray_share_q(P0, q, stream);
    static const char* c_env = std::getenv("PD_K2S_C");
    if (P0.N >= 13 && !(c_env && c_env[0] == '0') && P0.part_out == nullptr &&
        P0.x_count >= gray_share_c_min_xmasks(P0.N)) {
        // K2s-c geometry; the caller's chunks (2^ci_log steps) become 2^(ci_log - cs_log) stages
        K2Params P = P0;
        const unsigned tb = P0.N - 8 < 6 ? P0.N - 8 : 6;  // Z-mask bits 4 .. 4+tb-1 from the thread
        P.tpx_log = tb;
        P.xc_log = 8 - tb;                                 // X-masks per CTA (log2)
        P.cpx_log = 4 + (P0.N - 8 - tb);
        const unsigned cs_log = 11 - P.xc_log;            // 2048-element stages
        if (P0.ci_log < cs_log) return cudaErrorInvalidValue;
        P.ci_log = cs_log;
        P.c_begin = P0.c_begin << (P0.ci_log - cs_log);
        P.c_end = P0.c_end << (P0.ci_log - cs_log);
        const uint64_t xblocks = (P0.x_count + (1ull << P.xc_log) - 1) >> P.xc_log;
        const uint64_t cgrid = xblocks << P.cpx_log;
        static const char* sb_env = std::getenv("PD_K2SC_SB");  // measurement override
        const uint64_t sb = sb_env ? std::strtoull(sb_env, nullptr, 10) : 0;
        P.sb_ctas = (sb && sb < (cgrid >> 4)) ? static_cast<unsigned>(sb) : 0u;
        if (cgrid > 0x7fffffffull) return cudaErrorInvalidConfiguration;
        return seg ? launch_gray_share_c_seg(P, static_cast<unsigned>(cgrid), stream)
                   : launch_gray_share_c_full(P, static_cast<unsigned>(cgrid), stream);
    }
    if (seg) gray_share_kernel<true><<<grid, kK2Threads, smem, stream>>>(P0);
    else gray_share_kernel<false><<<grid, kK2Threads, smem, stream>>>(P0);
    return cudaGetLastError();
}

}  // namespace pdb

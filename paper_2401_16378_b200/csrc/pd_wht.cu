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

#include <cstdlib>
#include <mutex>

#include <atomic>
#include <cstdint>

#include "pd_device.cuh"
#include "pd_kernels.h"

namespace pdb {

namespace {

constexpr int kWhtThreads = 256;
constexpr unsigned kWhtMaxL = 12;


__device__ __forceinline__ void store_coeff(const OutMap& map, uint64_t x, uint64_t z, double sr,
                                            double si, double scale) {
    const unsigned ph = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
    __stcs(&map.out[out_index(map, tensor_number(x, z), z)], apply_phase(ph, sr, si, scale));
}

__global__ void __launch_bounds__(kWhtThreads)
    wht_rows_kernel(double2* __restrict__ diag, unsigned N, unsigned L, uint64_t x0,
                    OutMap map, double scale, int final_pass, const unsigned* __restrict__ skip) {
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
        if (skip && skip[xl]) return;  // non-finite diagonal: pd_nonfinite.cu wrote these
        const uint64_t x = x0 + xl;
        for (unsigned j = threadIdx.x; j < len; j += kWhtThreads)
            store_coeff(map, x, j, row[j].x, row[j].y, scale);
    } else {
        for (unsigned j = threadIdx.x; j < len; j += kWhtThreads) src[j] = row[j];
    }
}

template <int R>  // R = N - L high bits
__global__ void __launch_bounds__(kWhtThreads)
    wht_cols_kernel(double2* __restrict__ diag, unsigned N, unsigned L, uint64_t x0,
                    uint64_t x_count, OutMap map, double scale, int emit,
                    const unsigned* __restrict__ skip) {
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
    if (skip && skip[xl]) return;  // non-finite diagonal: pd_nonfinite.cu wrote these
    const uint64_t x = x0 + xl;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r)
        store_coeff(map, x, (static_cast<uint64_t>(r) << L) | il, v[r].x, v[r].y, scale);
}

// ---------------------------------------------------------------------------------------
// Fused two-pass WHT path (N >= 8): HBM traffic = read G + write D' + read D' + write out.
//
//   pass 1 (wht_gather_lo_reg_kernel): CTA = 32 X-masks (one tile row block x_h) x 128 columns
//     (4 column blocks C). Tile (R = C ^ x_h, C) of G holds D_x[C*32 + c] at (r, c) with
//     x = x_h*32 + (r ^ c) (the K1 transposition), so the coalesced 512 B row loads yield 32
//     diagonal segments of 128; index bits 5-6 are butterflied in registers, bits 0-4 in two
//     shared-memory rounds, and the segments are written to D' (128 B lines).
//   pass 2 (wht_hi_out_kernel): CTA = XPC X-masks x 8 adjacent low indices; loads 2^(N-7)
//     128 B pieces per X-mask, butterflies the high N-7 bits, applies (-i)^{|x&z|} 2^-N and
//     writes the coefficients: a warp covers (2 low x bits) x (3 low z bits), i.e. two
//     contiguous 256 B runs of the reference-ordered array.
//
// The generic pass 2 pads its shared-memory rows by one element every 16 (pad(i) = i + i/16)
// so that the strided butterfly rounds are bank-conflict free.

constexpr unsigned kLoBits = 7;  // index bits done in pass 1

__device__ __forceinline__ unsigned pad16(unsigned i) { return i + (i >> 4); }

// largest dynamic shared memory of the generic pass 2 (4096 padded elements)
constexpr size_t kHiOutSmem = 32 * ((1u << kLoBits) + ((1u << kLoBits) >> 4)) * sizeof(double2);

template <int RB>
__device__ __forceinline__ void wht_round(double2* s, unsigned L, unsigned row_stride, unsigned rows,
                                          unsigned b) {
    const unsigned groups_log = L - RB;
    const unsigned total = rows << groups_log;
    for (unsigned g = threadIdx.x; g < total; g += blockDim.x) {
        const unsigned row = g >> groups_log, rest = g & ((1u << groups_log) - 1);
        const unsigned lo = rest & ((1u << b) - 1), hi = rest >> b;
        const unsigned base = (hi << (b + RB)) | lo;
        double2* r = s + row * row_stride;
        double2 v[1 << RB];
#pragma unroll
        for (int k = 0; k < (1 << RB); ++k) v[k] = r[pad16(base + (static_cast<unsigned>(k) << b))];
#pragma unroll
        for (int h = 1; h < (1 << RB); h <<= 1) {
#pragma unroll
            for (int k = 0; k < (1 << RB); ++k) {
                if (k & h) continue;
                const double2 a = v[k], c = v[k + h];
                v[k] = make_double2(a.x + c.x, a.y + c.y);
                v[k + h] = make_double2(a.x - c.x, a.y - c.y);
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << RB); ++k) r[pad16(base + (static_cast<unsigned>(k) << b))] = v[k];
    }
}

// Pass 1, register-first form: each thread loads the 4 column blocks of one
// (row, column) position — the same X-mask x = r ^ c, index bits 5-6 — and butterflies them in
// registers; bits 0-2 and 3-4 follow in two shared-memory rounds, the last storing from
// registers. Rows padded to 33 elements (all access patterns conflict-free).
constexpr unsigned kP1bRow = 33;
constexpr size_t kP1bSmem = 128 * kP1bRow * sizeof(double2);               // 67,584 B

__device__ __forceinline__ void bfly(double2& a, double2& b) {
    const double2 p = a, q = b;
    a = make_double2(p.x + q.x, p.y + q.y);
    b = make_double2(p.x - q.x, p.y - q.y);
}

template <bool KEEP>
__global__ void __launch_bounds__(kWhtThreads, 2)
    wht_gather_lo_reg_kernel(const double2* __restrict__ G, unsigned N, uint64_t x0,
                             double2* __restrict__ dprime) {
    extern __shared__ __align__(16) double2 sb[];              // [x*4 + k][33]
    const uint64_t dim = 1ull << N;
    const unsigned groups_log = N - kLoBits;
    const uint64_t grp = blockIdx.x & ((1u << groups_log) - 1);
    const uint64_t xb = blockIdx.x >> groups_log;
    const uint64_t xh = (x0 >> 5) + xb;
    const unsigned c = threadIdx.x & 31, w = threadIdx.x >> 5;
    double2 v[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
            const uint64_t C = grp * 4 + cb, R = C ^ xh;
            v[j][cb] = __ldcs(&G[((R << 5) + w + 8 * j) * dim + (C << 5) + c]);
        }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        bfly(v[j][0], v[j][1]);
        bfly(v[j][2], v[j][3]);
        bfly(v[j][0], v[j][2]);
        bfly(v[j][1], v[j][3]);
        const unsigned x5 = (w + 8 * j) ^ c;
#pragma unroll
        for (int k = 0; k < 4; ++k) sb[(x5 * 4 + k) * kP1bRow + c] = v[j][k];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const unsigned g = threadIdx.x + q * kWhtThreads, row = g & 127, chi = g >> 7;
        double2* r = sb + row * kP1bRow + chi * 8;
        double2 u[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) u[e] = r[e];
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!(e & h)) bfly(u[e], u[e + h]);
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = u[e];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned g = threadIdx.x + q * kWhtThreads, clo = g & 7, row = g >> 3;
        const double2* r = sb + row * kP1bRow + clo;
        double2 u[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) u[h] = r[h * 8];
        bfly(u[0], u[1]);
        bfly(u[2], u[3]);
        bfly(u[0], u[2]);
        bfly(u[1], u[3]);
        const unsigned x5 = row >> 2, k = row & 3;
        double2* dst = dprime + ((xb << 5) + x5) * dim + (grp << kLoBits) + k * 32 + clo;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (KEEP) dst[h * 8] = u[h];
            else __stcs(dst + h * 8, u[h]);
        }
    }
}

// HB = N - 7 high index bits; XPC_LOG: X-masks per CTA (<= 4096 elements per CTA)
template <int HB, int XPC_LOG>
__global__ void __launch_bounds__(kWhtThreads, 2)
    wht_hi_out_kernel(const double2* __restrict__ dprime, unsigned N, uint64_t x0,
                      OutMap map, double scale) {
    extern __shared__ __align__(16) double2 s2[];
    constexpr unsigned L = HB + 3;                            // row = (hi, j), j = 3 low bits
    constexpr unsigned kRow = (1u << L) + ((1u << L) >> 4);
    constexpr unsigned kTotal = (1u << XPC_LOG) << L;
    constexpr int kIters = kTotal >= kWhtThreads ? kTotal / kWhtThreads : 1;
    const uint64_t dim = 1ull << N;
    constexpr unsigned kJBlocksLog = kLoBits - 3;             // 16 blocks of 8 low indices
    const uint64_t jb = blockIdx.x & ((1u << kJBlocksLog) - 1);
    const uint64_t xq = blockIdx.x >> kJBlocksLog;            // local group of X-masks
    double2 v[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const unsigned e = threadIdx.x + it * kWhtThreads;
        if (e < kTotal) {
            const unsigned xl = e >> L, hi = (e >> 3) & ((1u << HB) - 1), j = e & 7;
            v[it] = __ldcs(&dprime[((xq << XPC_LOG) + xl) * dim +
                                   (static_cast<uint64_t>(hi) << kLoBits) + (jb << 3) + j]);
        }
    }
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const unsigned e = threadIdx.x + it * kWhtThreads;
        if (e < kTotal) {
            const unsigned xl = e >> L, hi = (e >> 3) & ((1u << HB) - 1), j = e & 7;
            s2[xl * kRow + pad16((hi << 3) | j)] = v[it];
        }
    }
    __syncthreads();
#pragma unroll
    for (unsigned b = 3; b < 3 + HB; b += 4) {
        constexpr unsigned kEnd = 3 + HB;
        if (kEnd - b >= 4) wht_round<4>(s2, L, kRow, 1u << XPC_LOG, b);
        else if (kEnd - b == 3) wht_round<3>(s2, L, kRow, 1u << XPC_LOG, b);
        else if (kEnd - b == 2) wht_round<2>(s2, L, kRow, 1u << XPC_LOG, b);
        else wht_round<1>(s2, L, kRow, 1u << XPC_LOG, b);
        __syncthreads();
    }
    // output mapping: e = (hi, xl, j) with j fastest
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const unsigned e = threadIdx.x + it * kWhtThreads;
        if (e < kTotal) {
            const unsigned j = e & 7, xl = (e >> 3) & ((1u << XPC_LOG) - 1), hi = e >> (3 + XPC_LOG);
            const double2 w = s2[xl * kRow + pad16((hi << 3) | j)];
            const uint64_t x = x0 + (xq << XPC_LOG) + xl;
            const uint64_t z = (static_cast<uint64_t>(hi) << kLoBits) | (jb << 3) | j;
            store_coeff(map, x, z, w.x, w.y, scale);
        }
    }
}

// Pass 2 for HB = N - 7 in [4, 8]: every thread holds 16 elements in both register rounds.
// Round A loads straight from D' (128 B pieces, 4 per warp load) and butterflies high bits
// [0, 4); one shared-memory exchange; round B butterflies bits [4, HB) and writes the
// coefficients from registers (a warp covers 32 consecutive (x_low, j) columns: two 256 B runs).
// 2 shared-memory accesses and 1 barrier per element (the generic kernel above needs 6 and 3).
template <int HB, bool DISCARD>  // DISCARD: drop D' lines from L2 once read (never written back)
__global__ void __launch_bounds__(kWhtThreads, 2)
    wht_hi_reg_kernel(const double2* __restrict__ dprime, unsigned N, uint64_t x0, OutMap map,
                      double scale) {
    static_assert(HB >= 4 && HB <= 8, "16 elements per thread in both rounds");
    extern __shared__ __align__(16) double2 s2[];             // [2^HB][COLS]
    constexpr int RB = HB - 4;                                 // bits of round B
    constexpr unsigned COLS = 1u << (12 - HB);                 // (x_low, j) columns per CTA
    constexpr unsigned XPC_LOG = 9 - HB;                       // X-masks per CTA = COLS / 8
    constexpr int PAIRS = 1 << (8 - HB);                       // (hi_low, col) pairs per thread
    const uint64_t dim = 1ull << N;
    const uint64_t jb = blockIdx.x & 15;
    const uint64_t xq = blockIdx.x >> 4;
    {
        const unsigned col = threadIdx.x % COLS, a = threadIdx.x / COLS;
        const double2* src = dprime + ((xq << XPC_LOG) + (col >> 3)) * dim + (jb << 3) + (col & 7);
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r)
            v[r] = __ldcs(src + (static_cast<uint64_t>((a << 4) | r) << kLoBits));
#pragma unroll
        for (int h = 1; h < 16; h <<= 1)
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k & h) continue;
                const double2 p = v[k], q = v[k + h];
                v[k] = make_double2(p.x + q.x, p.y + q.y);
                v[k + h] = make_double2(p.x - q.x, p.y - q.y);
            }
        if (DISCARD && (col & 7) == 0) {
            // every element of these 128 B lines has been consumed by this warp (the butterflies
            // above read all 16 loads), and nothing reads D' again before pass 1 rewrites it
#pragma unroll
            for (int r = 0; r < 16; ++r)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(src + (static_cast<uint64_t>((a << 4) | r) << kLoBits))
                             : "memory");
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) s2[((a << 4) | r) * COLS + col] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
        const unsigned p = threadIdx.x + q * kWhtThreads;
        const unsigned col = p % COLS, hlo = p / COLS;
        double2 v[1 << RB];
#pragma unroll
        for (int h = 0; h < (1 << RB); ++h) v[h] = s2[((h << 4) | hlo) * COLS + col];
#pragma unroll
        for (int h = 1; h < (1 << RB); h <<= 1)
#pragma unroll
            for (int k = 0; k < (1 << RB); ++k) {
                if (k & h) continue;
                const double2 a = v[k], b = v[k + h];
                v[k] = make_double2(a.x + b.x, a.y + b.y);
                v[k + h] = make_double2(a.x - b.x, a.y - b.y);
            }
        const uint64_t x = x0 + (xq << XPC_LOG) + (col >> 3);
        // the 2^RB Z-masks of this thread differ only in bits >= 11 (h << 11): tensor number and
        // phase split into a per-thread part and a part whose spread is a compile-time
        // constant (spread(a ^ b) = spread(a) ^ spread(b)), ~15 instructions per store
        constexpr unsigned kHiShift = kLoBits + 4;
        const uint64_t zl = (static_cast<uint64_t>(hlo) << kLoBits) | (jb << 3) | (col & 7);
        const uint64_t xh = x >> kHiShift << kHiShift;
        const uint64_t nl = spread_bits((x ^ zl) & ((1ull << kHiShift) - 1)) | (spread_bits(zl) << 1);
        const uint64_t sxh = spread_bits(xh);
        const unsigned pl = static_cast<unsigned>(__popcll(x & zl));
#pragma unroll
        for (int h = 0; h < (1 << RB); ++h) {
            const uint64_t zh = static_cast<uint64_t>(h) << kHiShift;
            const uint64_t szh = spread_bits(zh);  // constant
            const uint64_t n = nl | (sxh ^ szh) | (szh << 1);
            const unsigned ph = (3u * (pl + static_cast<unsigned>(__popcll(xh & zh)))) & 3u;
            __stcs(&map.out[out_index(map, n, zh | zl)], apply_phase(ph, v[h].x, v[h].y, scale));
        }
    }
}

// ---------------------------------------------------------------------------------------
// Inverse transform for recompose (decompose.cpp:221-250), the forward passes run backwards.
// Row x of the recomposed matrix, E_x[r] = G[r][r ^ x] = sum_z (-1)^{|r & z|} (-i)^{|x&z|} c_{x,z}
// (pd_recompose.cu), is a Walsh-Hadamard transform over z split as z = (z_hi, z_lo), r = (r_hi,
// r_lo): pass A (mirror of wht_hi_reg_kernel) reads the phased coefficients and butterflies the
// high N-7 bits into E' [x][r_hi 128 + z_lo]; pass B (mirror of wht_gather_lo_reg_kernel)
// butterflies the low 7 bits of 32 rows at once and writes the XOR-diagonal tiles of G.

template <int HB>
__global__ void __launch_bounds__(kWhtThreads, 2)
    wht_inv_hi_kernel(const double2* __restrict__ coeffs, unsigned N, uint64_t x0,
                      double2* __restrict__ eprime) {
    static_assert(HB >= 4 && HB <= 8, "16 elements per thread in both rounds");
    extern __shared__ __align__(16) double2 s2[];             // [2^HB][COLS]
    constexpr int RB = HB - 4;
    constexpr unsigned COLS = 1u << (12 - HB);
    constexpr unsigned XPC_LOG = 9 - HB;
    constexpr int PAIRS = 1 << (8 - HB);
    const uint64_t dim = 1ull << N;
    const uint64_t jb = blockIdx.x & 15;
    const uint64_t xq = blockIdx.x >> 4;
    // all PAIRS x 2^RB scattered coefficient reads are issued before any is used (16 in flight
    // per thread), then phased and butterflied; tensor numbers from a per-thread part and
    // compile-time spreads (wht_hi_reg_kernel)
    constexpr unsigned kHiShift = kLoBits + 4;
    double2 v[PAIRS][1 << RB];
    unsigned ph[PAIRS][1 << RB];
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
        const unsigned p = threadIdx.x + q * kWhtThreads;
        const unsigned col = p % COLS, hlo = p / COLS;
        const uint64_t x = x0 + (xq << XPC_LOG) + (col >> 3);
        const uint64_t zl = (static_cast<uint64_t>(hlo) << kLoBits) | (jb << 3) | (col & 7);
        const uint64_t xh = x >> kHiShift << kHiShift;
        const uint64_t nl = spread_bits((x ^ zl) & ((1ull << kHiShift) - 1)) | (spread_bits(zl) << 1);
        const uint64_t sxh = spread_bits(xh);
        const unsigned pl = static_cast<unsigned>(__popcll(x & zl));
#pragma unroll
        for (int h = 0; h < (1 << RB); ++h) {
            const uint64_t zh = static_cast<uint64_t>(h) << kHiShift;
            const uint64_t szh = spread_bits(zh);  // constant
            v[q][h] = __ldcs(&coeffs[nl | (sxh ^ szh) | (szh << 1)]);
            ph[q][h] = (3u * (pl + static_cast<unsigned>(__popcll(xh & zh)))) & 3u;
        }
    }
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
        const unsigned p = threadIdx.x + q * kWhtThreads;
        const unsigned col = p % COLS, hlo = p / COLS;
#pragma unroll
        for (int h = 0; h < (1 << RB); ++h) v[q][h] = apply_phase(ph[q][h], v[q][h].x, v[q][h].y, 1.0);
#pragma unroll
        for (int h = 1; h < (1 << RB); h <<= 1)
#pragma unroll
            for (int k = 0; k < (1 << RB); ++k)
                if (!(k & h)) bfly(v[q][k], v[q][k + h]);
#pragma unroll
        for (int h = 0; h < (1 << RB); ++h) s2[((h << 4) | hlo) * COLS + col] = v[q][h];
    }
    __syncthreads();
    const unsigned col = threadIdx.x % COLS, a = threadIdx.x / COLS;
    double2 w[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) w[r] = s2[((a << 4) | r) * COLS + col];
#pragma unroll
    for (int h = 1; h < 16; h <<= 1)
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (!(k & h)) bfly(w[k], w[k + h]);
    double2* dst = eprime + ((xq << XPC_LOG) + (col >> 3)) * dim + (jb << 3) + (col & 7);
#pragma unroll
    for (int r = 0; r < 16; ++r) dst[static_cast<uint64_t>((a << 4) | r) << kLoBits] = w[r];
}

// smem rows (rb 32 + x5) of 33 elements: the E' loads, the round over index bits 0-2 and the
// transposed tile writes are all 4 wavefronts per warp
__global__ void __launch_bounds__(kWhtThreads, 2)
    wht_inv_lo_kernel(const double2* __restrict__ eprime, unsigned N, uint64_t x0,
                      double2* __restrict__ G) {
    extern __shared__ __align__(16) double2 sb[];              // [rb*32 + x5][33]
    const uint64_t dim = 1ull << N;
    const unsigned groups_log = N - kLoBits;
    const uint64_t grp = blockIdx.x & ((1u << groups_log) - 1);   // r_hi: rows grp*128 ..
    const uint64_t xb = blockIdx.x >> groups_log;
    const uint64_t xh = (x0 >> 5) + xb;
    // index bits 3-4 while loading 128 B lines of E' (and dropping them from L2): all 16 loads
    // of the thread are issued before any is used, and a line is discarded only after its
    // values have been consumed
    double2 u[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned g = threadIdx.x + q * kWhtThreads, clo = g & 7, row = g >> 3;
        const unsigned x5 = row >> 2, rb = row & 3;
        const double2* src = eprime + ((xb << 5) + x5) * dim + (grp << kLoBits) + rb * 32 + clo;
#pragma unroll
        for (int h = 0; h < 4; ++h) u[q][h] = __ldcs(src + h * 8);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const unsigned g = threadIdx.x + q * kWhtThreads, clo = g & 7, row = g >> 3;
        const unsigned x5 = row >> 2, rb = row & 3;
        bfly(u[q][0], u[q][1]);
        bfly(u[q][2], u[q][3]);
        bfly(u[q][0], u[q][2]);
        bfly(u[q][1], u[q][3]);
#pragma unroll
        for (int h = 0; h < 4; ++h) sb[(rb * 32 + x5) * kP1bRow + h * 8 + clo] = u[q][h];
        if (clo == 0) {
            const double2* src = eprime + ((xb << 5) + x5) * dim + (grp << kLoBits) + rb * 32;
#pragma unroll
            for (int h = 0; h < 4; ++h)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(src + h * 8) : "memory");
        }
    }
    __syncthreads();
    // index bits 0-2
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const unsigned g = threadIdx.x + q * kWhtThreads, row = g & 127, chi = g >> 7;
        double2* r = sb + row * kP1bRow + chi * 8;
        double2 u[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) u[e] = r[e];
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!(e & h)) bfly(u[e], u[e + h]);
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = u[e];
    }
    __syncthreads();
    // index bits 5-6 in registers, then the 4 tiles (R = grp 4 + rb, C = R ^ x_h): element
    // (tile row r, column c) is row r of X-mask x5 = r ^ c
    const unsigned c = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const unsigned r = w + 8 * j, x5 = r ^ c;
        double2 v[4];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) v[rb] = sb[(rb * 32 + x5) * kP1bRow + r];
        bfly(v[0], v[1]);
        bfly(v[2], v[3]);
        bfly(v[0], v[2]);
        bfly(v[1], v[3]);
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
            const uint64_t R = grp * 4 + rb, C = R ^ xh;
            __stcs(&G[((R << 5) + r) * dim + (C << 5) + c], v[rb]);
        }
    }
}

}  // namespace

// shared driver: rows pass, then (N > 12) the column pass; emit != 0 writes
// coefficients through `runs`, emit == 0 leaves the transform in place in `buf`
static cudaError_t wht_passes(double2* buf, unsigned N, uint64_t x0, uint64_t x_count,
                              const OutMap& map, int emit, const unsigned* skip, cudaStream_t stream) {
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
        buf, N, L, x0, map, scale, emit && R == 0, skip);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || R == 0) return e;
    const unsigned grid2 = static_cast<unsigned>(((x_count << L) + kWhtThreads - 1) / kWhtThreads);
    switch (R) {
        case 1: wht_cols_kernel<1><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, map, scale, emit, skip); break;
        case 2: wht_cols_kernel<2><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, map, scale, emit, skip); break;
        case 3: wht_cols_kernel<3><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, map, scale, emit, skip); break;
        default: wht_cols_kernel<4><<<grid2, kWhtThreads, 0, stream>>>(buf, N, L, x0, x_count, map, scale, emit, skip); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_wht_xmask(const double2* diag_c, unsigned N, uint64_t x0, uint64_t x_count,
                             unsigned run_bits, double2* out, int layout, cudaStream_t stream) {
    const OutMap map = make_outmap(out, N, run_bits, layout);
    double2* diag = const_cast<double2*>(diag_c);
    if (N <= kWhtMaxL) {
        // one rows pass reads the diagonals and emits: D is intact for the non-finite fixup
        cudaError_t e = wht_passes(diag, N, x0, x_count, map, 1, nullptr, stream);
        if (e == cudaSuccess) e = launch_nonfinite_fixup(diag_c, false, N, x0, x_count, map, nullptr, stream);
        return e;
    }
    // N > 12: the rows pass rewrites the diagonals in place (they are scratch owned by the
    // caller), so X-masks with a non-finite element are found and done first, from the
    // untouched diagonals, and the passes skip them
    unsigned* flags = nullptr;
    cudaError_t e = pool_alloc(reinterpret_cast<void**>(&flags), x_count * sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    e = launch_nonfinite_scan(diag_c, N, x_count, flags, stream);
    if (e == cudaSuccess) e = launch_nonfinite_fixup(diag_c, false, N, x0, x_count, map, flags, stream);
    if (e == cudaSuccess) e = wht_passes(diag, N, x0, x_count, map, 1, flags, stream);
    const cudaError_t f = pool_free(flags, stream);
    return e != cudaSuccess ? e : f;
}

// pass 2 dispatch: the register-round kernel for HB in [4, 8], the generic one otherwise
static cudaError_t launch_pass2(const double2* scratch, unsigned N, uint64_t x0, uint64_t x_count,
                                const OutMap& map, bool discard, cudaStream_t stream) {
    const unsigned hb = N - kLoBits;
    if (hb < 4 || hb > 8 || x_count < (1ull << (9 - hb))) return cudaErrorNotSupported;
    const double scale = 1.0 / static_cast<double>(1ull << N);
    const size_t smem = sizeof(double2) * 4096;
    const unsigned grid = static_cast<unsigned>((x_count >> (9 - hb)) << 4);
    cudaError_t e = cudaSuccess;
#define PD_REG(HBV)                                                                              \
    do {                                                                                         \
        auto k = discard ? wht_hi_reg_kernel<HBV, true> : wht_hi_reg_kernel<HBV, false>;      \
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);         \
        if (e == cudaSuccess) k<<<grid, kWhtThreads, smem, stream>>>(scratch, N, x0, map, scale);                    \
    } while (0)
    switch (hb) {
        case 4: PD_REG(4); break;
        case 5: PD_REG(5); break;
        case 6: PD_REG(6); break;
        case 7: PD_REG(7); break;
        default: PD_REG(8); break;
    }
#undef PD_REG
    if (e != cudaSuccess) return e;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

bool wht_fused_ok(unsigned N, uint64_t x_count) { return N >= 8 && N <= 16 && x_count >= 32; }

// Chunked L2-resident pipeline. D' of a chunk of S X-masks (S 2^N x 16 B, 16 MiB) is written
// by pass 1 with default (L2-allocating) stores and read back by pass 2 before it leaves L2;
// pass 2 then discards the lines (discard.global.L2), so D' never reaches DRAM and the HBM
// traffic is the algorithmic 32 4^N B (read G, write coefficients). Chunks rotate over four D'
// slots and four streams, so a chunk's pass 2 overlaps the following chunks' pass 1.
namespace {
constexpr int kWhtMaxStreams = 4;
struct WhtPipe {
    cudaStream_t side[kWhtMaxStreams] = {};
    cudaEvent_t fork = nullptr, join[kWhtMaxStreams] = {};
    bool ok = false;
    std::mutex issue;  // one fork/chunks/join sequence at a time (the events are shared)
};

WhtPipe& wht_pipe(int dev) {
    static WhtPipe pipes[64];
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    WhtPipe& p = pipes[dev & 63];
    if (!p.ok) {
        bool good = cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming) == cudaSuccess;
        for (int k = 0; good && k < kWhtMaxStreams; ++k)
            good = cudaStreamCreateWithFlags(&p.side[k], cudaStreamNonBlocking) == cudaSuccess &&
                   cudaEventCreateWithFlags(&p.join[k], cudaEventDisableTiming) == cudaSuccess;
        p.ok = good;
    }
    return p;
}

uint64_t wht_chunk(unsigned N) {
    // 16 MiB of D' per chunk, 4 chunks in flight: 64 MiB of the 126 MB L2 (measured optimum at
    // N=12 and N=14: 2 x 32 MiB is 1 % slower, 1 x 64 MiB or 4 x 32 MiB 6-8 % slower)
    const uint64_t s = (16ull << 20) / (sizeof(double2) << N);
    return s < 32 ? 32 : s;
}
}  // namespace

static cudaError_t wht_two_pass(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                double2* dprime, const OutMap& map, bool l2_resident,
                                cudaStream_t stream) {
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set.load() >> dev & 1)) {
        cudaError_t e = cudaSuccess;
        for (auto k : {wht_gather_lo_reg_kernel<true>, wht_gather_lo_reg_kernel<false>})
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kP1bSmem);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    const uint64_t grid1 = (x_count >> 5) << (N - kLoBits);
    auto k1 = l2_resident ? wht_gather_lo_reg_kernel<true> : wht_gather_lo_reg_kernel<false>;
    k1<<<static_cast<unsigned>(grid1), kWhtThreads, kP1bSmem, stream>>>(G, N, x0, dprime);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launch_pass2(dprime, N, x0, x_count, map, l2_resident, stream) == cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError();
    }
    cudaGetLastError();  // clear cudaErrorNotSupported: fall back to the generic pass 2
    const unsigned hb = N - kLoBits;
    const double scale = 1.0 / static_cast<double>(1ull << N);
    // X-masks per CTA: 4 while 2^(hb+3) <= 1024, then 2, then 1 (<= 4096 elements, 68 KiB)
    unsigned xpc_log = hb <= 7 ? 2 : (hb == 8 ? 1 : 0);
    while ((1ull << xpc_log) > x_count) --xpc_log;
    const size_t smem = (sizeof(double2) << xpc_log) * ((1u << (hb + 3)) + ((1u << (hb + 3)) >> 4));
    const unsigned grid2 = static_cast<unsigned>((x_count >> xpc_log) << (kLoBits - 3));
#define PD_HI(HBV, XL)                                                                        \
    do {                                                                                      \
        auto k = wht_hi_out_kernel<HBV, XL>;                                                  \
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHiOutSmem); \
        if (e == cudaSuccess)                                                                 \
            k<<<grid2, kWhtThreads, smem, stream>>>(dprime, N, x0, map, scale);              \
    } while (0)
    switch (hb * 4 + xpc_log) {
        case 1 * 4 + 2: PD_HI(1, 2); break;
        case 2 * 4 + 2: PD_HI(2, 2); break;
        case 3 * 4 + 2: PD_HI(3, 2); break;
        case 4 * 4 + 2: PD_HI(4, 2); break;
        case 5 * 4 + 2: PD_HI(5, 2); break;
        case 6 * 4 + 2: PD_HI(6, 2); break;
        case 7 * 4 + 2: PD_HI(7, 2); break;
        case 8 * 4 + 1: PD_HI(8, 1); break;
        case 9 * 4 + 0: PD_HI(9, 0); break;
        default: return cudaErrorInvalidValue;
    }
#undef PD_HI
    if (e != cudaSuccess) return e;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

static cudaError_t wht_from_matrix(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                   double2* scratch, const OutMap& map, cudaStream_t stream) {
    const uint64_t S = wht_chunk(N);
    const unsigned hb = N - kLoBits;
    const bool reg_pass2 = hb >= 4 && hb <= 8;
    if (!reg_pass2 || x_count < 4 * S || (S & 31) || x_count % S)
        return wht_two_pass(G, N, x0, x_count, scratch, map, false, stream);
    int dev = 0;
    cudaGetDevice(&dev);
    WhtPipe& p = wht_pipe(dev);
    if (!p.ok) return cudaErrorInitializationError;
    const uint64_t dim = 1ull << N;
    std::lock_guard<std::mutex> lk(p.issue);
    cudaError_t e = cudaEventRecord(p.fork, stream);
    constexpr int ns = kWhtMaxStreams;
    for (int k = 0; e == cudaSuccess && k < ns; ++k) e = cudaStreamWaitEvent(p.side[k], p.fork, 0);
    for (uint64_t c = 0; e == cudaSuccess && c < x_count / S; ++c) {
        const int k = static_cast<int>(c % ns);  // slot k of D' belongs to stream k
        e = wht_two_pass(G, N, x0 + c * S, S, scratch + k * S * dim, map, true, p.side[k]);
    }
    for (int k = 0; e == cudaSuccess && k < ns; ++k) {
        e = cudaEventRecord(p.join[k], p.side[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, p.join[k], 0);
    }
    return e;
}

cudaError_t launch_wht_from_matrix(const double2* G, unsigned N, uint64_t x0, uint64_t x_count,
                                   double2* scratch, unsigned run_bits, double2* out, int layout,
                                   cudaStream_t stream) {
    const OutMap map = make_outmap(out, N, run_bits, layout);
    cudaError_t e = wht_from_matrix(G, N, x0, x_count, scratch, map, stream);
    // X-masks whose diagonal holds an inf or NaN: the reference's products, straight from G
    if (e == cudaSuccess) e = launch_nonfinite_fixup(G, true, N, x0, x_count, map, nullptr, stream);
    return e;
}

bool wht_inverse_ok(unsigned N) { return N >= 11 && N <= 15; }

// recompose of the X-masks [0, 2^N) through the chunked L2-resident inverse passes (same
// pipeline as launch_wht_from_matrix, data flowing the other way)
cudaError_t launch_wht_inverse(const double2* coeffs, unsigned N, double2* scratch, double2* G,
                               cudaStream_t stream) {
    const uint64_t dim = 1ull << N;
    const unsigned hb = N - kLoBits;
    if (!wht_inverse_ok(N)) return cudaErrorNotSupported;
    const uint64_t S0 = wht_chunk(N);
    const uint64_t S = dim < 4 * S0 ? dim / 4 : S0;  // four chunks at least (S >= 32)
    const size_t smem_a = sizeof(double2) * 4096, smem_b = kP1bSmem;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<uint64_t> attr_set{0};
    cudaError_t e = cudaSuccess;
    if (!(attr_set.load() >> dev & 1)) {
        for (auto k : {wht_inv_hi_kernel<4>, wht_inv_hi_kernel<5>, wht_inv_hi_kernel<6>, wht_inv_hi_kernel<7>,
                       wht_inv_hi_kernel<8>})
            if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(wht_inv_lo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem_b));
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(1ull << dev);
    }
    auto pass_a = hb == 4 ? wht_inv_hi_kernel<4> : hb == 5 ? wht_inv_hi_kernel<5> : hb == 6 ? wht_inv_hi_kernel<6>
                : hb == 7 ? wht_inv_hi_kernel<7> : wht_inv_hi_kernel<8>;
    WhtPipe& p = wht_pipe(dev);
    if (!p.ok) return cudaErrorInitializationError;
    std::lock_guard<std::mutex> lk(p.issue);
    e = cudaEventRecord(p.fork, stream);
    constexpr int ns = kWhtMaxStreams;
    for (int k = 0; e == cudaSuccess && k < ns; ++k) e = cudaStreamWaitEvent(p.side[k], p.fork, 0);
    for (uint64_t c = 0; e == cudaSuccess && c < dim / S; ++c) {
        const int k = static_cast<int>(c % ns);
        double2* slot = scratch + k * S * dim;
        const unsigned grid_a = static_cast<unsigned>((S >> (9 - hb)) << 4);
        pass_a<<<grid_a, kWhtThreads, smem_a, p.side[k]>>>(coeffs, N, c * S, slot);
        const unsigned grid_b = static_cast<unsigned>((S >> 5) << (N - kLoBits));
        wht_inv_lo_kernel<<<grid_b, kWhtThreads, smem_b, p.side[k]>>>(slot, N, c * S, G);
        g_launches.fetch_add(2, std::memory_order_relaxed);
        e = cudaGetLastError();
    }
    for (int k = 0; e == cudaSuccess && k < ns; ++k) {
        e = cudaEventRecord(p.join[k], p.side[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, p.join[k], 0);
    }
    return e;
}

cudaError_t launch_wht_inplace(double2* rows, unsigned N, uint64_t x_count, cudaStream_t stream) {
    return wht_passes(rows, N, 0, x_count, make_outmap(nullptr, N, 0, 0), 0, nullptr, stream);
}

}  // namespace pdb

// pd_device.cuh — device-side index algebra and PTX helpers shared by the kernels.
//
// Index algebra restated from the reference (paths relative to proj/):
//   * tensor number n, base-4 digit d_t = (n >> 2t) & 3 selects sigma_t in
//     {I,X,Y,Z} (pauli.hpp:13-20, bits.hpp:52-55);
//   * X-mask x_t = [d_t in {X,Y}] (pauli.hpp:23-39 xy_mask), Z-mask z_t = d_t >> 1,
//     so d_t = 2 z_t + (x_t ^ z_t);
//   * c_n = 2^-N (-i)^{|x&z|} sum_k (-1)^{|g_k & z|} G[g_k ^ x][g_k], g_k = k ^ (k>>1):
//     the reference's Gray walk (decompose.cpp:30-47) with lambda_0 = (-i)^{#Y}
//     (pauli.hpp:97-102) and row-flip quotient -1 for Y,Z (pauli.hpp:65-68).
#pragma once

#include <math_constants.h>

#include <cstdint>

namespace pdb {

// bit t of v -> bit 2t
__host__ __device__ __forceinline__ uint64_t spread_bits(uint64_t v) {
    v &= 0xFFFFFFFFull;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}

// bit 2t of v -> bit t
__host__ __device__ __forceinline__ uint64_t gather_even_bits(uint64_t v) {
    v &= 0x5555555555555555ull;
    v = (v | (v >> 1)) & 0x3333333333333333ull;
    v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
    v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
    v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
    return v;
}

// tensor number of the string with X-mask x and Z-mask z
__host__ __device__ __forceinline__ uint64_t tensor_number(uint64_t x, uint64_t z) {
    return spread_bits(x ^ z) | (spread_bits(z) << 1);
}

__host__ __device__ __forceinline__ uint64_t xmask_of(uint64_t n) {
    return gather_even_bits(n ^ (n >> 1));
}

__host__ __device__ __forceinline__ uint64_t zmask_of(uint64_t n) { return gather_even_bits(n >> 1); }

__host__ __device__ __forceinline__ uint64_t gray(uint64_t k) { return k ^ (k >> 1); }

// parity of v; non-recursive so that it folds to a constant inside unrolled loops
__host__ __device__ __forceinline__ constexpr int cparity(unsigned v) {
    v ^= v >> 16;
    v ^= v >> 8;
    v ^= v >> 4;
    v ^= v >> 2;
    v ^= v >> 1;
    return static_cast<int>(v & 1u);
}

__host__ __device__ constexpr unsigned cgray(unsigned k) { return k ^ (k >> 1); }

// flip the sign of a double when sgn == 0x80000000 (exact, branchless)
// (inline PTX keeps the front end from rewriting it as a select between v and a
// negation, which would cost an extra FP64-pipe DNEG per element)
__device__ __forceinline__ double flip_sign(double v, unsigned sgn) {
    int hi = __double2hiint(v);
    asm("xor.b32 %0, %0, %1;" : "+r"(hi) : "r"(sgn));
    return __hiloint2double(hi, __double2loint(v));
}

// c = i^p * (sr + i si), then * scale (2^-N, exact). p = 3|x&z| mod 4 encodes (-i)^{|x&z|}.
__device__ __forceinline__ double2 apply_phase(unsigned p, double sr, double si, double scale) {
    double cr, ci;
    switch (p & 3u) {
        case 0: cr = sr; ci = si; break;
        case 1: cr = -si; ci = sr; break;
        case 2: cr = -sr; ci = -si; break;
        default: cr = si; ci = -sr; break;
    }
    return make_double2(cr * scale, ci * scale);
}

// ---- the reference's own arithmetic, for non-finite elements ----
//
// The reference accumulates lambda.value() * a[...] (decompose.cpp:40), a std::complex<double>
// product that GCC evaluates as (ac - bd, ad + bc) and, when both parts come out NaN, hands to
// libgcc's __muldc3, which recovers infinities as C99 Annex G.5.1 specifies. For lambda in
// {1, i, -1, -i} and a finite element that is the exact re/im swap the fast kernels fold into
// their adds (up to the sign of an exact zero); for an infinite or NaN element it is not:
// 0 * inf puts a NaN into the other component ([[1, inf], [3, 4]] -> c_1 = inf + nan i).
// Products are rounded one by one (no contraction), as the reference's x86-64 SSE code does.

__device__ __forceinline__ bool finite2(double2 v) {
    return ((__double2hiint(v.x) & 0x7ff00000) != 0x7ff00000) &
           ((__double2hiint(v.y) & 0x7ff00000) != 0x7ff00000);
}

__device__ __forceinline__ double2 cmul_annex_g(double a, double b, double c, double d) {
    const double ac = __dmul_rn(a, c), bd = __dmul_rn(b, d), ad = __dmul_rn(a, d),
                 bc = __dmul_rn(b, c);
    double x = __dsub_rn(ac, bd), y = __dadd_rn(ad, bc);
    if (isnan(x) && isnan(y)) {
        bool recalc = false;
        if (isinf(a) || isinf(b)) {  // the first factor is infinite: box it, NaNs of the other -> 0
            a = copysign(isinf(a) ? 1.0 : 0.0, a);
            b = copysign(isinf(b) ? 1.0 : 0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = true;
        }
        if (isinf(c) || isinf(d)) {  // the second factor is infinite
            c = copysign(isinf(c) ? 1.0 : 0.0, c);
            d = copysign(isinf(d) ? 1.0 : 0.0, d);
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            recalc = true;
        }
        if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) {  // overflow
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = true;
        }
        if (recalc) {
            x = __dmul_rn(CUDART_INF, __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
            y = __dmul_rn(CUDART_INF, __dadd_rn(__dmul_rn(a, d), __dmul_rn(b, c)));
        }
    }
    return make_double2(x, y);
}

// i^p as the reference's unit_phase table (pauli.hpp:71-76)
__device__ __forceinline__ double unit_re(unsigned p) { return p == 0 ? 1.0 : (p == 2 ? -1.0 : 0.0); }
__device__ __forceinline__ double unit_im(unsigned p) { return p == 1 ? 1.0 : (p == 3 ? -1.0 : 0.0); }

// Coefficient (x, z) by the reference's arithmetic: k = 0..2^N-1 in Gray order, lambda carried as
// a power of i from (-i)^{|x&z|} (pauli.hpp:97-102) and multiplied by -1 when the flipped bit is
// set in z (pauli.hpp:65-68, 112-114), acc += lambda * e with cmul_annex_g, then acc / 2^N
// componentwise (complex / double, decompose.cpp:56). elem(i) returns G[i ^ x][i].
template <class Elem>
__device__ __forceinline__ double2 exact_coeff(const Elem& elem, unsigned N, uint64_t x, uint64_t z) {
    const uint64_t dim = 1ull << N;
    unsigned p = (3u * static_cast<unsigned>(__popcll(x & z))) & 3u;
    double ar = 0.0, ai = 0.0;
    uint64_t code = 0;
    for (uint64_t k = 0;; ++k) {
        const double2 e = elem(code);
        const double2 t = cmul_annex_g(unit_re(p), unit_im(p), e.x, e.y);
        ar = __dadd_rn(ar, t.x);
        ai = __dadd_rn(ai, t.y);
        if (k + 1 == dim) break;
        const unsigned b = static_cast<unsigned>(__ffsll(static_cast<long long>(k + 1)) - 1);
        p = (p + 2u * static_cast<unsigned>((z >> b) & 1u)) & 3u;
        code ^= 1ull << b;
    }
    // acc / 2^N: the product with 2^-N is the same correctly rounded quotient (subnormals too)
    const double s = __longlong_as_double(static_cast<long long>(1023 - N) << 52);
    return make_double2(__dmul_rn(ar, s), __dmul_rn(ai, s));
}

// Where coefficient (x, z) with tensor number n goes (see pd_api.h, pd_layout):
//   GLOBAL: out[n], the reference-ordered array of all 4^N coefficients;
//   RUNS:   the coefficients of one aligned block of 2^(N - rb) X-masks, packed as its 2^rb
//           runs (one per value r of the Z-mask's top rb bits) of 4^(N - rb) entries each:
//           out[(r << 2(N - rb)) | (n mod 4^(N - rb))].
struct OutMap {
    double2* out;
    unsigned rb_shift;   // N - rb
    unsigned low_bits;   // 2 (N - rb)
    int runs;            // 0 GLOBAL, 1 RUNS
};

__host__ __device__ __forceinline__ uint64_t out_index(const OutMap& m, uint64_t n, uint64_t z) {
    if (!m.runs) return n;
    const uint64_t low = m.low_bits >= 64 ? n : (n & ((1ull << m.low_bits) - 1));
    return ((z >> m.rb_shift) << m.low_bits) | low;
}

inline OutMap make_outmap(double2* out, unsigned N, unsigned run_bits, int runs) {
    return OutMap{out, N - run_bits, 2 * (N - run_bits), runs};
}

// ---- mbarrier / bulk-copy (TMA engine) PTX ----

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PD_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra PD_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

}  // namespace pdb

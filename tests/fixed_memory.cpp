// fixed_memory.cpp — the reference's fixed-memory promise (proj/tests/test_alloc.cpp: the
// coefficient kernels touch no heap beyond the caller's input) checked on the B200 library, plus
// its device-side counterpart: after a warm-up, coeff_fast / coeff_slow (and their MultCount
// forms) make no operator-new call and leave the device's free memory unchanged, and repeated
// full decompositions into a caller-owned array do not grow device memory.
//
// Built and run by tests/test_fixed_memory_gpu.py: g++ -std=c++20 -I include fixed_memory.cpp
// -L paper_2401_16378_b200 -lpaulidecomp_b200 -lpd_b200 -lcudart. Prints "FAIL ..." lines and
// exits 1 on any violation, "ok" otherwise.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <vector>

#include "paulidecomp_b200/bench.hpp"
#include "paulidecomp_b200/decompose.hpp"

namespace {
std::atomic<std::uint64_t> g_news{0};
int g_failures = 0;

void* counted(std::size_t n) {
    g_news.fetch_add(1, std::memory_order_relaxed);
    if (void* p = std::malloc(n ? n : 1)) return p;
    throw std::bad_alloc();
}

size_t device_free() {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    return free_b;
}

void expect(bool ok, const char* what, long long a, long long b) {
    if (!ok) {
        std::printf("FAIL %s (%lld vs %lld)\n", what, a, b);
        ++g_failures;
    }
}
}  // namespace

// every operator new of the process (the library's too) comes through here
void* operator new(std::size_t n) { return counted(n); }
void* operator new[](std::size_t n) { return counted(n); }
void operator delete(void* p) noexcept { std::free(p); }
void operator delete[](void* p) noexcept { std::free(p); }
void operator delete(void* p, std::size_t) noexcept { std::free(p); }
void operator delete[](void* p, std::size_t) noexcept { std::free(p); }

int main() {
    using namespace paulidecomp;
    for (unsigned nq : {6u, 10u, 13u}) {
        const DenseMatrix g = random_matrix(nq, 1000 + nq);
        MultCount count;
        Complex sink = coeff_fast(g, 5) + coeff_slow(g, 3) + coeff_fast(g, 7, count) + coeff_slow(g, 9, count);
        const size_t free0 = device_free();
        const std::uint64_t news0 = g_news.load();
        const std::uint64_t total = std::uint64_t{1} << (2 * nq);
        for (std::uint64_t k = 0; k < 64; ++k) {
            const std::uint64_t n = (k * 0x9E3779B97F4A7C15ull) % total;
            sink += coeff_fast(g, n);
            sink += coeff_slow(g, n);
            sink += coeff_fast(g, n, count) + coeff_slow(g, n, count);
        }
        const std::uint64_t news1 = g_news.load();
        const size_t free1 = device_free();
        char what[64];
        std::snprintf(what, sizeof(what), "N=%u: coefficient calls allocated", nq);
        expect(news1 == news0, what, static_cast<long long>(news1), static_cast<long long>(news0));
        expect(free1 == free0, "coefficient calls changed device free memory", static_cast<long long>(free1),
               static_cast<long long>(free0));
        expect(sink != Complex{1e308, 1e308} && count.mults > 0, "kernel results observable", 0, 0);
    }
    // full decompositions into a caller-owned array: device memory is set up by the first call
    for (unsigned nq : {10u, 12u}) {
        const DenseMatrix g = random_matrix(nq, 2000 + nq);
        std::vector<Complex> out(g.element_count());
        decompose_into(g.data(), nq, out.data());
        const size_t free0 = device_free();
        for (int r = 0; r < 5; ++r) decompose_into(g.data(), nq, out.data());
        const size_t free1 = device_free();
        expect(free1 == free0, "repeated decompositions changed device free memory", static_cast<long long>(free1),
               static_cast<long long>(free0));
    }
    if (g_failures) return 1;
    std::printf("ok\n");
    return 0;
}

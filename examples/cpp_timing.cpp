// cpp_timing.cpp — the reference's C++ API on the B200 library, timed: decompose_parallel
// (returns PauliDecomposition by value, like proj/include/paulidecomp/decompose.hpp:46) against
// decompose_into a caller-owned array, at N given on the command line (default 14).
// g++ -std=c++20 -O2 -Iinclude examples/cpp_timing.cpp -Lpaper_2401_16378_b200 \
//     -lpaulidecomp_b200 -lpd_b200 -Wl,-rpath,$PWD/paper_2401_16378_b200
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "paulidecomp_b200/bench.hpp"
#include "paulidecomp_b200/decompose.hpp"

int main(int argc, char** argv) {
    using namespace paulidecomp;
    using clock = std::chrono::steady_clock;
    const unsigned nq = argc > 1 ? static_cast<unsigned>(std::atoi(argv[1])) : 14;
    const DenseMatrix g = random_matrix(nq, 7);
    std::vector<Complex> out(g.element_count());
    decompose_into(g.data(), nq, out.data());  // warm-up: context, buffers, staging slots
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = clock::now();
        const PauliDecomposition d = decompose_parallel(g, 1);
        auto t1 = clock::now();
        decompose_into(g.data(), nq, out.data());
        auto t2 = clock::now();
        std::printf("N=%u decompose_parallel %.1f ms, decompose_into %.1f ms, equal=%d\n", nq,
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count(), d.coefficients == out ? 1 : 0);
    }
    return 0;
}

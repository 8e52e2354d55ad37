// paulidecomp_b200/bench.hpp — the reference's benchmark API (proj/include/paulidecomp/bench.hpp)
// on the GPU: the same seeded generator, the same options and CSV schema, the device paths
// timed through the host-buffer API (transfers included, like a caller sees them).
#pragma once

#include <cstdint>
#include <ostream>
#include <string>
#include <vector>

#include "paulidecomp_b200/decompose.hpp"

namespace paulidecomp {

inline constexpr unsigned kBenchMaxQubits = 14;  // the reference caps its CPU bench at 8

struct BenchOptions {  // bench.hpp:14-20 defaults
    unsigned n_min = 1;
    unsigned n_max = 5;
    unsigned reps = 20;
    std::uint64_t seed = 1;
    unsigned threads = 1;  // kept for the interface; the GPU launch sets the parallelism
};

struct BenchRecord {  // one CSV row; rep == -1 is the per-(N, path) mean with its stddev
    unsigned num_qubits = 0;
    std::string path;
    unsigned threads = 1;
    int rep = 0;
    std::uint64_t seed = 0;
    double seconds = 0.0;
    std::uint64_t mult_count = 0;
    double seconds_stddev = 0.0;
};

// bench.cpp:42-46: per-(N, rep) seed of the generator
std::uint64_t matrix_seed(std::uint64_t seed, unsigned num_qubits, unsigned rep);
// bench.cpp:48-58: uniform [-1, 1) real and imaginary parts from splitmix64, generated on the
// device (K5, bit-identical) and copied back
DenseMatrix random_matrix(unsigned num_qubits, std::uint64_t seed);

// bench.cpp:60-139 with the device paths "gray", "wht" and "naive"; gray and naive must agree
// bit for bit and wht within 1e-11 of the largest coefficient, else std::runtime_error
std::vector<BenchRecord> run_bench(const BenchOptions& options);
// bench.cpp:141-150: N,path,threads,rep,seed,seconds,mult_count,seconds_stddev
void write_bench_csv(const std::vector<BenchRecord>& records, std::ostream& out);

}  // namespace paulidecomp

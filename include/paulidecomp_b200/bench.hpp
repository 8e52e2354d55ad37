// paulidecomp_b200/bench.hpp — the seeded matrix generator of the reference's benchmark API
// (proj/include/paulidecomp/bench.hpp), generated on the GPU bit for bit. The reference's
// timing harness and its CSV writer are out of scope; bench.py measures.
#pragma once

#include <cstdint>

#include "paulidecomp_b200/decompose.hpp"

namespace paulidecomp {

// bench.cpp:42-46: per-(N, rep) seed of the generator
std::uint64_t matrix_seed(std::uint64_t seed, unsigned num_qubits, unsigned rep);
// bench.cpp:48-58: uniform [-1, 1) real and imaginary parts from splitmix64, generated on the
// device (K5, bit-identical) and copied back
DenseMatrix random_matrix(unsigned num_qubits, std::uint64_t seed);
// B200 addition: the same matrix into caller-owned memory (4^N entries)
void random_matrix_into(unsigned num_qubits, std::uint64_t seed, Complex* out);

}  // namespace paulidecomp
